"""Regenerate the committed golden fixtures from the UNMODIFIED reference.

Runs oracle/_ref/aspine_ref (built by `make -C oracle ref` from
/root/reference/proj/src) and stores its outputs as small JSON files here, so
the parity tests can run on a machine without /root/reference (the GPU box).

    python tests/golden/make_golden.py            # all fixtures
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref", "aspine_ref")
sys.path.insert(0, ROOT)

from workloads import instances as I  # noqa: E402

MODES = [("fwd", "occ"), ("res", "occ"), ("fwd", "jw"), ("res", "jw"), ("fwd", "act"), ("res", "act")]


def ref(args, stdin=None):
    out = subprocess.run([REF] + args, input=stdin, capture_output=True, text=True, check=False)
    if out.returncode not in (0, 2):
        raise RuntimeError(out.stderr)
    return json.loads(out.stdout)


def solve_text(text, opts):
    return ref(["solve", "-"] + opts, stdin=text)


def corpus():
    """Acceptance corpus (acceptance_main.cpp:51-65) with full-enumeration results per mode x heuristic."""
    progs = ref(["corpus"])
    for p in progs:
        runs = {}
        for mode, heur in MODES:
            r = solve_text(p["text"], ["-n", "0", "--mode", mode, "--heur", heur, "--verify"])
            runs[f"{mode}/{heur}"] = {"status": r["status"], "models": r["models"], "stats": r["stats"]}
        p["runs"] = runs
    return progs


def extras():
    """Restarts, fanout, deps-words overflow, capacity: small programs x options."""
    progs = ref(["corpus"])
    cases = []
    opts = [
        ["--restarts", "1:1.5"], ["--restarts", "3:2", "--mode", "res"], ["--fanout", "3"],
        ["--fanout", "2", "--heur", "act"], ["--deps-words", "1"], ["--mode", "res", "--heur", "act", "--decay", "0.8"],
    ]
    for i, p in enumerate(progs):
        if i % 5:
            continue
        for o in opts:
            r = solve_text(p["text"], ["-n", "0"] + o)
            cases.append({"name": p["name"], "text": p["text"], "opts": o, "status": r["status"],
                          "models": r["models"], "stats": r["stats"]})
    php = I.pigeonhole(3, 2)
    for o in (["--restarts", "1:1.5"], ["--restarts", "1:1.5", "--mode", "res"], ["--cap", "0"]):
        r = solve_text(php, ["-n", "0"] + o)
        cases.append({"name": "php32", "text": php, "opts": o, "status": r["status"], "models": r["models"],
                      "stats": r["stats"], "error": r["error"]})
    return cases


def configs():
    out = {}
    q8 = I.queens(8)
    for mode, heur in MODES:
        r = solve_text(q8, ["-n", "0", "--mode", mode, "--heur", heur, "--trace"])
        out[f"queens8/{mode}/{heur}"] = {"status": r["status"], "models": r["models"], "stats": r["stats"],
                                         "trace": r["trace"]}
    for name, text in (("colour2000", I.colouring(2000, 4.0, 3, 1)), ("ham200", I.hamiltonian(200, 1.0, 1))):
        r = solve_text(text, ["-n", "1", "--no-models"])
        r1 = solve_text(text, ["-n", "1"])
        out[f"{name}/fwd/occ"] = {"status": r["status"], "models": r1["models"], "stats": r["stats"]}
    return out


def propstores():
    return {
        "test_propagate": ref(["propstores", "0xc105e001", "300", "10", "4"]),
        "criterion5": ref(["propstores", "0xc7059a7e", "1000", "10", "4"]),
    }


def dumps():
    """compile_completion + NogoodStore::build goldens for the corpus and the config instances."""
    progs = ref(["corpus"])
    texts = [(p["name"], p["text"]) for p in progs]
    texts += [("queens8", I.queens(8)), ("queens5", I.queens(5)), ("ham12", I.hamiltonian(12, 1.0, 3)),
              ("colour30", I.colouring(30, 4.0, 3, 7)), ("php43", I.pigeonhole(4, 3))]
    out = []
    for name, text in texts:
        d = ref(["dump", "-"], stdin=text)
        d["name"], d["text"] = name, text
        out.append(d)
    return out


def planted():
    return [ref(["planted", "20000", "200000", str(p), "0x1b00b5"]) for p in (1, 10, 50, 90)]


def model_set_digest(models):
    """Order-independent digest of a set of answer sets: FNV-1a over the sorted
    models, each a sorted atom-id list closed by a 0 (tests/_util.py mirrors it)."""
    h = 0xcbf29ce484222325
    for m in sorted(tuple(sorted(x)) for x in models):
        for a in list(m) + [0]:
            h = ((h ^ (a & 0xFFFFFFFF)) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def pins():
    """Parity pins for every configuration bench.py reports (VERDICT r1 "next" #1):
    full-size planted fixpoints (1M at 1/10/50/90 %, 8M at 50 %) with trail, reason
    and Deps digests; config 4a's first model and SolveStats; all 14,200 answer sets
    of queens(12) as count + model-set digest (the reference needs minutes here)."""
    out = {"planted_1m": [ref(["planted", "100000", "1000000", str(p), "0x1b00b5"]) for p in (1, 10, 50, 90)],
           "planted_8m": [ref(["planted", "800000", "8000000", "50", "0x1b00b5"])]}
    r = solve_text(I.random_program(), ["-n", "1"])
    out["rand4a"] = {"status": r["status"], "stats": r["stats"], "model_len": len(r["models"][0]),
                     "model_digest": model_set_digest(r["models"])}
    for n in (12,):
        r = solve_text(I.queens(n), ["-n", "0"])
        out[f"queens{n}"] = {"status": r["status"], "models": len(r["models"]),
                             "model_set_digest": model_set_digest(r["models"]), "stats": r["stats"]}
    out["queens13"] = queens13_by_cubes()
    return out


def queens13_by_cubes():
    """queens(13), the multi-GPU scaling workload: a single reference enumeration
    runs for hours here, so the reference solves every cube of the ladder split
    (one `aspine_ref cubes` process per core); the cubes partition the answer
    sets, and the union must hold 73,712 distinct models (OEIS A000170)."""
    import tempfile
    import paper_1909_01786_b200 as Y
    text = I.queens(13)
    prog = Y.parse_program(text)
    cubes = Y.cubes(prog, 13, 0, want=4 * 148 * 8)
    nproc = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as d:
        lp, cf = os.path.join(d, "q13.lp"), os.path.join(d, "cubes.txt")
        with open(lp, "w") as f:
            f.write(text)
        with open(cf, "w") as f:
            for c in cubes:
                f.write(" ".join(prog.name(abs(l)) for l in c if l) + "\n")
        procs = [subprocess.Popen([REF, "cubes", lp, cf, str(k), str(nproc)], stdout=subprocess.PIPE, text=True)
                 for k in range(nproc)]
        models = [m for p in procs for m in json.loads(p.communicate()[0])["models"]]
    assert len({tuple(m) for m in models}) == len(models) == 73712
    return {"status": "SAT", "models": len(models), "model_set_digest": model_set_digest(models),
            "source": f"reference, {len(cubes)} cubes solved one by one on {nproc} processes"}


def main():
    targets = sys.argv[1:] or ["corpus", "extras", "configs", "propstores", "planted", "dumps", "pins"]
    for t in targets:
        data = globals()[t]()
        with open(os.path.join(HERE, f"{t}.json"), "w") as f:
            json.dump(data, f, separators=(",", ":"))
        print(t, "written")


if __name__ == "__main__":
    main()
