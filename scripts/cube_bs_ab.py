"""Developer probe: cube enumeration with 64- vs 128-thread searches (YAS_CUBE_BS128)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01786_b200 as Y  # noqa: E402
from workloads import instances as I  # noqa: E402

for n in (8, 12, 13):
    prog = Y.parse_program(I.queens(n))
    for mode in ("64", "128", "64", "128"):
        if mode == "128":
            os.environ["YAS_CUBE_BS128"] = "1"
        else:
            os.environ.pop("YAS_CUBE_BS128", None)
        best = None
        for rep in range(3):
            t = time.perf_counter()
            r = Y.solve(prog, Y.SolverConfig(max_models=0))
            w = (time.perf_counter() - t) * 1e3
            if rep and (best is None or w < best[0]):
                best = (w, r.stats.device_ms, len(r.models))
        print(f"queens{n} {mode}-thread searches: wall {best[0]:.1f} ms device {best[1]:.1f} ms models {best[2]}", flush=True)
