for m in a b c; do timeout 150 python scripts/_dbg2.py $m >> gpurun_out/dbg2.log 2>&1; echo "$m rc=$?" >> gpurun_out/dbg2.log; done
