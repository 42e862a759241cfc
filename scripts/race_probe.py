"""Developer probe: the grid-engine part of sanitize_run.py alone (racecheck bisection)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1909_01786_b200 as Y  # noqa: E402

part = sys.argv[1] if len(sys.argv) > 1 else "grid"
stores = []
if part != "solves":
    with open(os.path.join(ROOT, "tests", "golden", "propstores.json")) as f:
        stores = json.load(f)["test_propagate"][:3]
for st in stores:
    p = Y.Propagator(Y.NogoodStore.build(st["nogoods"], 10), 1, part)
    o = p.initial_propagation()
    if not o.violated:
        o = p.propagate_and_check(1)
    print("store ok", flush=True)
if part != "solves":
    s, seeded, dec = Y.NogoodStore.planted(500, 5000, 50)
    p = Y.Propagator(s, 16, part)
    p.push_decision(dec)
    p.assign_propagated(seeded, 2)
    p.seed([dec] + seeded)
    print("planted", p.propagate_and_check(2).violated, flush=True)

if part == "solves":
    from workloads import instances as I  # noqa: E402
    which = sys.argv[2]
    if which == "corpus":
        with open(os.path.join(ROOT, "tests", "golden", "corpus.json")) as f:
            corpus = json.load(f)[:6]
        for prog in corpus:
            r = Y.solve(Y.parse_program(prog["text"]), Y.SolverConfig(max_models=0))
            print(prog["name"], len(r.models), flush=True)
    elif which == "cubes":
        print(len(Y.solve(Y.parse_program(I.queens(6)), Y.SolverConfig(max_models=0, cube_atoms=6, cube_depth=1)).models))
    elif which == "gridsolve":
        print(len(Y.solve(Y.parse_program(I.queens(5)), Y.SolverConfig(max_models=0, engine="grid")).models))
    elif which == "portfolio":
        col = Y.parse_program(I.colouring(30, 4.0, 3, 7))
        print(Y.solve(col, Y.SolverConfig(portfolio=3)).status)
