mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_grid_kernel -s 5 -c 1 -o gpurun_out/p1pct_b -f python scripts/planted_profile.py 100000 1000000 1 1 > gpurun_out/ncu7.log 2>&1
