"""Developer probe: cube enumeration time per searches-per-SM setting
(YAS_SEARCHES_PER_SM: 8 = 128-thread CTAs, 16 = one warp per search).

    python scripts/enum_variants.py [n ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01786_b200 as Y  # noqa: E402
from workloads import instances as I  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [8, 12]:
    prog = Y.parse_program(I.queens(n))
    for per_sm in ("8", "16"):
        os.environ["YAS_SEARCHES_PER_SM"] = per_sm
        best = None
        for rep in range(4):
            t = time.perf_counter()
            r = Y.solve(prog, Y.SolverConfig(max_models=0, cube_atoms=n))
            wall = (time.perf_counter() - t) * 1e3
            if rep and (best is None or wall < best[0]):
                best = (wall, r.stats.device_ms, len(r.models), r.stats.cubes, r.stats.passes)
        print(f"queens{n} per_sm={per_sm}: wall {best[0]:.1f} ms, device {best[1]:.1f} ms, models {best[2]}, "
              f"cubes {best[3]}, passes {best[4]}", flush=True)
