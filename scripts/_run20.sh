timeout 600 python -m pytest tests/test_gpu_cubes.py tests/test_multiproc.py -x -q 2>&1 | tail -2 > gpurun_out/r20.log
for k in 4 8; do echo "searches/SM=$k" >> gpurun_out/r20.log; YAS_SEARCHES_PER_SM=$k timeout 120 python scripts/enum_timing.py 12 2>&1 | tail -3 >> gpurun_out/r20.log; YAS_SEARCHES_PER_SM=$k timeout 120 python scripts/enum_timing.py 10 2>&1 | tail -2 >> gpurun_out/r20.log; done
