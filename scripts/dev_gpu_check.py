"""Developer GPU check: quick parity probes against the committed goldens.

    python scripts/dev_gpu_check.py [section ...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1909_01786_b200 as Y  # noqa: E402
from workloads import instances as I  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")
STAT_KEYS = ["decisions", "propagations", "conflicts", "learned_count", "learned_length_sum", "restarts", "models",
             "passes", "duplicate_learned", "blocking_nogoods", "res_learned", "fwd_learned", "fwd_fallbacks",
             "uip_check_failures", "fwd_decision_only_failures", "asserting_failures"]


def load(name):
    with open(os.path.join(G, name + ".json")) as f:
        return json.load(f)


def t_basic():
    s = Y.NogoodStore.build([[1, 2], [1, -2]], 2)
    p = Y.Propagator(s, 1, engine="block")
    p.push_decision(1)
    p.seed([1])
    o = p.propagate_and_check(2)
    print("race:", o.violated, p.cells()[2], o.conflicts, "expect True -2 [1]")


def t_prop(engine="block"):
    data = load("propstores")
    for key in ("test_propagate", "criterion5"):
        bad = 0
        for i, st in enumerate(data[key]):
            s = Y.NogoodStore.build(st["nogoods"], 10)
            p = Y.Propagator(s, 1, engine=engine)
            o = p.initial_propagation()
            ok = o.violated == bool(st["init_violated"]) and sorted(o.conflicts) == sorted(st["init_conflicts"])
            ok &= o.propagations == st["init_props"]
            if ok and not o.violated:
                o = p.propagate_and_check(1)
                ok &= o.violated == bool(st["l1_violated"]) and sorted(o.conflicts) == sorted(st["l1_conflicts"])
                ok &= o.propagations == st["l1_props"] and o.passes == st["l1_passes"]
                if ok and not o.violated and st["decision"]:
                    p.push_decision(st["decision"])
                    p.seed([st["decision"]])
                    o = p.propagate_and_check(2)
                    ok &= o.violated == bool(st["l2_violated"]) and sorted(o.conflicts) == sorted(st["l2_conflicts"])
                    ok &= o.propagations == st["l2_props"] and o.passes == st["l2_passes"]
            ok &= p.cells() == st["cells"] and p.trail() == st["trail"]
            rs = p.reasons()
            ok &= rs == st["reasons"]
            d, ov = p.deps(0)
            ok &= [x | (1 << 63 if v else 0) for x, v in zip(d, ov)] == st["deps"]
            if not ok:
                bad += 1
                if bad <= 3:
                    print("MISMATCH", key, i, st["nogoods"], "cells", p.cells(), st["cells"], "trail", p.trail(),
                          st["trail"], "reasons", rs, st["reasons"])
        print(f"propstores/{key}/{engine}: {len(data[key])} stores, {bad} mismatches")


def t_configs():
    data = load("configs")
    for key, exp in data.items():
        name, mode, heur = key.split("/")
        text = {"queens8": lambda: I.queens(8), "colour2000": lambda: I.colouring(2000, 4.0, 3, 1),
                "ham200": lambda: I.hamiltonian(200, 1.0, 1)}[name]()
        prog = Y.parse_program(text)
        cfg = Y.SolverConfig(mode=Y.LearnMode[mode],
                             heuristic=Y.HeuristicConfig({"occ": Y.HeuristicKind.occurrence_count,
                                                          "jw": Y.HeuristicKind.jeroslow_wang,
                                                          "act": Y.HeuristicKind.activity}[heur]),
                             max_models=0 if name == "queens8" else 1, engine="block")
        t0 = time.time()
        r = Y.solve(prog, cfg)
        dt = time.time() - t0
        models = [m.atom_ids for m in r.models]
        same_models = models == exp["models"]
        diffs = {k: (getattr(r.stats, k), exp["stats"][k]) for k in STAT_KEYS if getattr(r.stats, k) != exp["stats"][k]}
        print(f"{key}: models {'OK' if same_models else 'DIFF'} ({len(models)}/{len(exp['models'])}), "
              f"stat diffs {diffs}, {dt*1e3:.1f} ms wall, dev {r.stats.device_ms:.1f} ms, launches {r.stats.launches}")


def t_planted():
    for exp in load("planted"):
        for engine in ("block", "grid"):
            s, seeded, dec = Y.NogoodStore.planted(exp["atoms"], exp["nogoods"], exp["pct"])
            p = Y.Propagator(s, 16, engine=engine)
            p.push_decision(dec)
            p.assign_propagated(seeded, 2, [], False, 0)
            p.seed([dec] + seeded)
            o = p.propagate_and_check(2)
            tr = p.trail()
            h = 0xcbf29ce484222325
            for c in tr:
                h = ((h ^ (c & 0xFFFFFFFF)) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
            ok = (o.propagations == exp["propagations"] and o.passes == exp["passes"] and h == exp["trail_digest"]
                  and len(tr) == exp["trail"])
            print(f"planted {exp['pct']}% {engine}: {'OK' if ok else 'DIFF'} props {o.propagations}/{exp['propagations']}"
                  f" passes {o.passes}/{exp['passes']} checks {o.checks} dev {o.device_ms:.3f} ms")


if __name__ == "__main__":
    secs = sys.argv[1:] or ["basic", "prop", "configs", "planted"]
    for s in secs:
        t0 = time.time()
        try:
            globals()["t_" + s]()
        except Exception as e:  # report and continue
            import traceback
            traceback.print_exc()
            print("FAILED", s, e)
        print(f"-- {s} {time.time()-t0:.1f}s", flush=True)
