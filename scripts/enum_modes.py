"""Developer probe: cube enumeration time per (mode, heuristic) variant.
    python scripts/enum_modes.py [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01786_b200 as Y  # noqa: E402
from workloads import instances as I  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
prog = Y.parse_program(I.queens(n))
H = {"occ": Y.HeuristicKind.occurrence_count, "jw": Y.HeuristicKind.jeroslow_wang, "act": Y.HeuristicKind.activity}
for mode in ("fwd", "res"):
    for heur in ("occ", "jw", "act"):
        cfg = Y.SolverConfig(max_models=0, cube_atoms=n, mode=Y.LearnMode[mode], heuristic=Y.HeuristicConfig(H[heur]))
        best = None
        for rep in range(3):
            t = time.perf_counter()
            r = Y.solve(prog, cfg)
            w = (time.perf_counter() - t) * 1e3
            if rep and (best is None or w < best[0]):
                best = (w, r.stats.device_ms, len(r.models), r.stats.passes, r.stats.conflicts, r.stats.decisions)
        print(f"queens{n} {mode}/{heur}: wall {best[0]:.1f} ms device {best[1]:.1f} ms models {best[2]} passes {best[3]} "
              f"conflicts {best[4]} decisions {best[5]}", flush=True)
