"""Config 5 CPU reference, measured in full once per round on the GPU box host:
the unmodified reference (oracle/_ref/aspine_ref) enumerating all 14,200 answer
sets of queens(12) with one worker (its fastest setting), split into load and
SolveStats::wall_ms (run only, /root/reference/proj/src/solver.cpp:249,300-301).
Writes profiles/r02_q12_reference_full.json, which bench.py cites next to its
nproc cube-split CPU run (too long to repeat inside every bench run).

    python scripts/cpu_q12_reference.py
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from workloads import instances as I  # noqa: E402


def main():
    text = I.queens(12)
    t = time.perf_counter()
    p = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "aspine_ref"), "solve", "-", "-n", "0", "--no-models"],
                       input=text, capture_output=True, text=True, check=True)
    wall = (time.perf_counter() - t) * 1e3
    r = json.loads(p.stdout)
    model = None
    with open("/proc/cpuinfo") as f:
        for line in f:
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    out = {"instance": "queens12, all answer sets, workers=1 (reference, unmodified)", "models": r["stats"]["models"],
           "run_ms": r["run_ms"][0], "parse_ms": r["parse_ms"], "process_wall_ms": wall, "cores": 1,
           "host_nproc": os.cpu_count(), "cpu_model": model, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "stats": r["stats"]}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "r02_q12_reference_full.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
