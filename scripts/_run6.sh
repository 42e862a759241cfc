mkdir -p gpurun_out
timeout 300 python scripts/pass_trace.py 100000 1000000 50 > gpurun_out/pt50.log 2>&1
timeout 300 python scripts/pass_trace.py 100000 1000000 1 > gpurun_out/pt1.log 2>&1
timeout 300 python scripts/pass_trace.py 800000 8000000 50 > gpurun_out/pt8m.log 2>&1
