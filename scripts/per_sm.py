"""Developer probe: q12 enumeration per YAS_SEARCHES_PER_SM setting."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01786_b200 as Y  # noqa: E402
from workloads import instances as I  # noqa: E402

prog = Y.parse_program(I.queens(12))
for per in ("2", "4", "6", "8", "16"):
    os.environ["YAS_SEARCHES_PER_SM"] = per
    best = None
    for rep in range(3):
        t = time.perf_counter()
        r = Y.solve(prog, Y.SolverConfig(max_models=0))
        w = (time.perf_counter() - t) * 1e3
        if rep and (best is None or w < best[0]):
            best = (w, r.stats.device_ms, len(r.models), r.stats.cubes)
    print(f"per_sm={per}: wall {best[0]:.1f} ms device {best[1]:.1f} ms models {best[2]} cubes {best[3]}", flush=True)
