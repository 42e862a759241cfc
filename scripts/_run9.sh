mkdir -p gpurun_out
for c in colour2000 ham200 queens8; do YAS_PROFILE=1 timeout 120 python scripts/run_one.py $c 1 block >> gpurun_out/r9.log 2>&1; YAS_PROFILE=1 timeout 120 python scripts/run_one.py $c 1 block >> gpurun_out/r9.log 2>&1; done
YAS_PROFILE=1 timeout 300 python scripts/run_one.py rand100k 1 grid >> gpurun_out/r9.log 2>&1
YAS_PROFILE=1 timeout 300 python scripts/run_one.py rand100k 1 grid >> gpurun_out/r9.log 2>&1
