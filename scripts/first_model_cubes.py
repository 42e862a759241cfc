"""Developer probe: first answer set by one search (reference trajectory) vs the
cube-parallel mode (cube_atoms, max_models=1) on the structured configs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01786_b200 as Y  # noqa: E402
from workloads import instances as I  # noqa: E402

for name, text in (("colour2000", I.colouring(2000, 4.0, 3, 1)), ("ham200", I.hamiltonian(200, 1.0, 1))):
    prog = Y.parse_program(text)
    for label, cfg in (("one search", Y.SolverConfig()), ("cubes k=3", Y.SolverConfig(cube_atoms=3)),
                       ("cubes k=8", Y.SolverConfig(cube_atoms=8)), ("cubes k=16", Y.SolverConfig(cube_atoms=16))):
        best = None
        for rep in range(3):
            t = time.perf_counter()
            r = Y.solve(prog, cfg)
            w = (time.perf_counter() - t) * 1e3
            if rep and (best is None or w < best[0]):
                best = (w, r.stats.device_ms, r.status.name, r.stats.searches, Y.verify_model(prog, r.models[0]))
        print(f"{name} {label}: wall {best[0]:.1f} ms device {best[1]:.1f} ms {best[2]} searches {best[3]} "
              f"answer set {best[4]}", flush=True)
