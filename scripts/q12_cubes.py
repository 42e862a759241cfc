import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01786_b200 as Y
from workloads import instances as I
prog = Y.parse_program(I.queens(int(sys.argv[1]) if len(sys.argv) > 1 else 12))
for spec in sys.argv[2:]:
    k, d = map(int, spec.split(":"))
    t = time.time()
    r = Y.solve(prog, Y.SolverConfig(max_models=0, cube_atoms=k, cube_depth=d))
    s = r.stats
    print(f"k={k} d={d}: models={len(r.models)} uniq={len(set(tuple(m.atom_ids) for m in r.models))} wall={(time.time()-t)*1e3:.0f}ms "
          f"dev={s.device_ms:.0f}ms launches={s.launches} searches={s.searches} passes={s.passes} checks={s.checks}", flush=True)
