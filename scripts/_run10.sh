mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:block_kernel -c 1 -o gpurun_out/col -f python scripts/run_one.py colour2000 1 block > gpurun_out/ncu10.log 2>&1
