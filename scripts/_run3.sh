mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt3.log 2>&1; echo "rc=$?" >> gpurun_out/pt3.log
timeout 300 python scripts/planted_profile.py 100000 1000000 50 4 > gpurun_out/prof1m.log 2>&1
timeout 300 python scripts/planted_profile.py 800000 8000000 50 3 > gpurun_out/prof8m.log 2>&1
timeout 300 python scripts/planted_profile.py 100000 1000000 1 3 > gpurun_out/prof1m_1pct.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err
