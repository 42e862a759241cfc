"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
both engines on small cases — the propagator API on random and planted stores,
full solves of a corpus slice in every mode, a cube enumeration and a portfolio.
Kept small because the sanitizers replay every access.

    compute-sanitizer --tool racecheck python scripts/sanitize_run.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1909_01786_b200 as Y  # noqa: E402
from workloads import instances as I  # noqa: E402


def golden(name):
    with open(os.path.join(ROOT, "tests", "golden", name + ".json")) as f:
        return json.load(f)


def main():
    quick = "--quick" in sys.argv  # racecheck replays every shared-memory access: a smaller slice
    part = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--part=")), "all")  # bisection
    checks = 0
    for engine in ("block", "grid") if part in ("all", "prop") else ():
        for st in golden("propstores")["test_propagate"][:6 if quick else 20]:
            p = Y.Propagator(Y.NogoodStore.build(st["nogoods"], 10), 1, engine)
            o = p.initial_propagation()
            if not o.violated:
                o = p.propagate_and_check(1)
                if not o.violated and st["decision"]:
                    p.push_decision(st["decision"])
                    p.seed([st["decision"]])
                    p.propagate_and_check(2)
            assert p.trail() == st["trail"], engine
            checks += 1
            if part != "all":
                print(engine, "store", checks, flush=True)
        s, seeded, dec = Y.NogoodStore.planted(500 if quick else 2000, 5000 if quick else 20000, 50)
        p = Y.Propagator(s, 16, engine)
        p.push_decision(dec)
        p.assign_propagated(seeded, 2)
        p.seed([dec] + seeded)
        assert not p.propagate_and_check(2).violated
        checks += 1
    for prog in golden("corpus")[:6 if quick else 24] if part in ("all", "corpus") else []:
        for mode in ("fwd", "res"):
            r = Y.solve(Y.parse_program(prog["text"]), Y.SolverConfig(max_models=0, mode=Y.LearnMode[mode]))
            assert sorted(m.atom_ids for m in r.models) == sorted(prog["family"]), prog["name"]
            checks += 1
    if part in ("all", "solves"):
        r = Y.solve(Y.parse_program(I.queens(6)), Y.SolverConfig(max_models=0, cube_atoms=6, cube_depth=1))
        assert len(r.models) == 4
        r = Y.solve(Y.parse_program(I.queens(5)), Y.SolverConfig(max_models=0, engine="grid"))
        assert len(r.models) == 10
        col = Y.parse_program(I.colouring(30, 4.0, 3, 7))
        r = Y.solve(col, Y.SolverConfig(portfolio=3))
        assert r.status == Y.solve(col, Y.SolverConfig()).status
    print(f"sanitize_run: {checks + 3} workloads ok")


if __name__ == "__main__":
    main()
