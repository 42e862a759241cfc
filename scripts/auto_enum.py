"""Developer probe: plain enumeration (SolverConfig(max_models=0), the drop-in default:
automatic cube split) vs the explicit row ladder, queens 8/12/13."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01786_b200 as Y  # noqa: E402
from workloads import instances as I  # noqa: E402

for n in (8, 12, 13):
    prog = Y.parse_program(I.queens(n))
    for name, cfg in (("default", Y.SolverConfig(max_models=0)), ("rows", Y.SolverConfig(max_models=0, cube_atoms=n))):
        best = None
        for rep in range(3):
            t = time.perf_counter()
            r = Y.solve(prog, cfg)
            w = (time.perf_counter() - t) * 1e3
            if rep and (best is None or w < best[0]):
                best = (w, r.stats.device_ms, len(r.models), r.stats.cubes)
        print(f"queens{n} {name}: wall {best[0]:.1f} ms device {best[1]:.1f} ms models {best[2]} cubes {best[3]}", flush=True)
