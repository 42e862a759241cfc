#!/bin/bash
# One GPU-box pass: tests, smoke, bench, reference arm, launch list, ncu captures of the
# three kernel shapes (grid propagation, cube enumeration, single search), sanitizers.
#   scripts/gpu_round.sh [tests] [bench] [ncu] [san]   (default: all)
mkdir -p gpurun_out
want() { [ $# -eq 0 ] && return 0; for a in "${ARGS[@]}"; do [ "$a" = "$1" ] && return 0; done; [ ${#ARGS[@]} -eq 0 ]; }
ARGS=("$@")
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
if want tests; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
if want bench; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
  timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
if want ncu; then
  # reports stay on the box (/tmp/ncu, too large to copy back); summaries come back
  mkdir -p /tmp/ncu
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/bench_ncu.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:op_grid_kernel -s 5 -c 1 -o /tmp/ncu/planted_grid -f python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/ncu_planted.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_kernel -s 1 -c 1 -o /tmp/ncu/q12_cubes -f python scripts/enum_timing.py 12 > gpurun_out/ncu_q12.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_kernel -c 1 -o /tmp/ncu/ham200_block -f python scripts/run_one.py ham200 > gpurun_out/ncu_ham200.log 2>&1
  for r in planted_grid q12_cubes ham200_block; do
    [ -f /tmp/ncu/$r.ncu-rep ] && timeout 300 python scripts/summarize_ncu.py /tmp/ncu/$r.ncu-rep gpurun_out/ncu_$r >> gpurun_out/ncu_summaries.log 2>&1
  done
fi
if want san; then
  for t in memcheck synccheck initcheck; do
    timeout 400 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_run.py > gpurun_out/san_$t.log 2>&1; echo "rc=$?" >> gpurun_out/san_$t.log
  done
  timeout 500 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_run.py --quick > gpurun_out/san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.log
fi
ls -la gpurun_out
