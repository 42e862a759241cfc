for w in r4a p8 enum fm; do timeout 240 python scripts/_dbg_bench.py $w >> gpurun_out/dbg.log 2>&1; echo "$w rc=$?" >> gpurun_out/dbg.log; done
