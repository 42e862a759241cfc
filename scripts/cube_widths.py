"""Developer probe: cube enumeration time per ladder width / depth.
    python scripts/cube_widths.py n"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01786_b200 as Y  # noqa: E402
from workloads import instances as I  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
prog = Y.parse_program(I.queens(n))
for k, d in ((4, 0), (6, 0), (8, 0), (8, 5), (12, 0), (12, 3), (16, 0), (24, 0)):
    cfg = Y.SolverConfig(max_models=0, cube_atoms=k, cube_depth=d)
    best = None
    for rep in range(3):
        t = time.perf_counter()
        r = Y.solve(prog, cfg)
        w = (time.perf_counter() - t) * 1e3
        if rep and (best is None or w < best[0]):
            best = (w, r.stats.device_ms, len(r.models), r.stats.cubes, r.stats.passes)
    print(f"queens{n} k={k} depth={d}: wall {best[0]:.1f} ms device {best[1]:.1f} ms models {best[2]} cubes {best[3]} "
          f"passes {best[4]}", flush=True)
