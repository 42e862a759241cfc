mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:op_grid_kernel -s 5 -c 1 -o gpurun_out/p8m -f python scripts/planted_profile.py 800000 8000000 50 1 > gpurun_out/ncu8.log 2>&1
