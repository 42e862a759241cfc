"""Run one configuration through the public API (profiling helper).
   python scripts/run_one.py queens8 [n_models] [engine] [mode] [heur] [cube_atoms]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01786_b200 as Y
from workloads import instances as I
name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
engine = sys.argv[3] if len(sys.argv) > 3 else "auto"
mode = sys.argv[4] if len(sys.argv) > 4 else "fwd"
heur = sys.argv[5] if len(sys.argv) > 5 else "occ"
cubes = int(sys.argv[6]) if len(sys.argv) > 6 else 0
prog = Y.parse_program(I.CONFIGS[name]())
cfg = Y.SolverConfig(mode=Y.LearnMode[mode], heuristic=Y.HeuristicConfig({"occ": Y.HeuristicKind.occurrence_count,
      "jw": Y.HeuristicKind.jeroslow_wang, "act": Y.HeuristicKind.activity}[heur]), max_models=n, engine=engine,
      cube_atoms=cubes)
t = time.time()
r = Y.solve(prog, cfg)
s = r.stats
print(f"{name}: {r.status.name} models={len(r.models)} wall={(time.time()-t)*1e3:.1f}ms dev={s.device_ms:.1f}ms "
      f"launches={s.launches} passes={s.passes} dec={s.decisions} confl={s.conflicts} props={s.propagations} "
      f"checks={s.checks} searches={s.searches}")
