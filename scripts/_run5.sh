mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_grid_kernel -s 5 -c 1 -o gpurun_out/p1pct -f python scripts/planted_profile.py 100000 1000000 1 1 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_grid_kernel -s 5 -c 1 -o gpurun_out/p50pct -f python scripts/planted_profile.py 100000 1000000 50 1 > gpurun_out/ncu2.log 2>&1
