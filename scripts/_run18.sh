for kb in 96 48 24 12; do for c in colour2000 ham200; do YAS_SMEM_KB=$kb python scripts/run_one.py $c 1 block 2>&1 | sed "s/^/kb=$kb /" >> gpurun_out/r18.log; done; done
