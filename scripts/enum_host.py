"""Developer probe: host-side laps of repeated q12 enumerations (YAS_PROFILE=1 set here)."""
import os
import sys
import time

os.environ["YAS_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01786_b200 as Y  # noqa: E402
from workloads import instances as I  # noqa: E402

prog = Y.parse_program(I.queens(int(sys.argv[1]) if len(sys.argv) > 1 else 12))
for k in range(4):
    t = time.perf_counter()
    r = Y.solve(prog, Y.SolverConfig(max_models=0))
    print(f"call {k}: wall {(time.perf_counter() - t) * 1e3:.1f} ms device {r.stats.device_ms:.1f} ms models {len(r.models)}",
          file=sys.stderr, flush=True)
