"""yasmin-b200 benchmark (driver contract: one JSON line from rank 0).

Headline metric (BASELINE.json): nogood checks/s of propagation-to-fixpoint on
the synthetic 1M-nogood / 100k-atom planted store (config 4b),
with the HBM roofline of the propagation kernel; the same line carries the
enumeration result (12-queens, all 14,200 answer sets, cube-split over the N
GPUs) and the first-model configurations, each next to the reference CPU solver
timed on this host.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl yasmin|reference]

A "step" is one propagate_and_check call to fixpoint over the planted store.
The propagation path does not shard (one fixpoint), so with N > 1 every rank
runs a replica ("weak" scaling); enumeration cubes are partitioned over ranks
and only the model count / time are all-reduced (NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PLANTED = dict(atoms=100_000, nogoods=1_000_000, pct=50, seed=0x1B00B5)
WORKLOAD = "planted store: 1M nogoods, 100k atoms, len U[2,6], 50% of H seeded at level 2 (SURVEY.md App. C, 4b)"
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "aspine_ref")


def pins():
    """Reference outputs at full size (tests/golden/pins.json, make_golden.py pins)."""
    with open(os.path.join(ROOT, "tests", "golden", "pins.json")) as f:
        return json.load(f)


def fnv(words, h=0xcbf29ce484222325):
    for c in words:
        h = ((h ^ (int(c) & 0xFFFFFFFF)) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def planted_parity(prop, o, exp):
    """Untimed: the fixpoint equals the reference's (counts + trail / reason / Deps digests)."""
    tr = prop.trail()
    reasons = prop.reasons()
    d0, ovf = prop.deps(0)
    rs, ds = [], []
    for lit in tr:
        x = abs(lit)
        rs.append(reasons[x] if reasons[x] >= 0 else -1)
        ds += [d0[x] & 0xFFFFFFFF, d0[x] >> 32, 1 if ovf[x] else 0]
    got = (o.propagations, o.passes, len(tr), fnv(tr), fnv(rs), fnv(ds))
    want = (exp["propagations"], exp["passes"], exp["trail"], exp["trail_digest"], exp["reason_digest"],
            exp["deps_digest"])
    return got == want


def model_set_digest(models):
    words = []
    for m in sorted(tuple(sorted(x)) for x in models):
        words += list(m) + [0]
    return fnv(words)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if os.environ.get("BENCH_DIST_BACKEND") == "gloo":  # rank-logic check on a box with fewer GPUs
            local %= max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def allreduce(vals, op="max", world=1):
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist
    gloo = dist.get_backend() == "gloo"
    t = torch.tensor(vals, dtype=torch.float64, device="cpu" if gloo else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return t.tolist()


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def run_reference_planted(reps):
    """Unmodified reference (oracle/_ref): Propagator::propagate_and_check on the same store."""
    out = subprocess.run([REF_BIN, "planted", str(PLANTED["atoms"]), str(PLANTED["nogoods"]), str(PLANTED["pct"]),
                          hex(PLANTED["seed"]), str(reps)], capture_output=True, text=True, check=True)
    return json.loads(out.stdout)


def planted_checks():
    from oracle import port  # the count of items is a property of the workload
    return port.planted(PLANTED["atoms"], PLANTED["nogoods"], PLANTED["pct"], PLANTED["seed"])


def reference_arm(args, rank, world):
    if rank != 0:
        return
    reps = args.warmup + args.steps
    if os.path.exists(REF_BIN):
        ref = run_reference_planted(reps)
        times = ref["prop_ms"][args.warmup:]
        kind = "reference"
    else:  # restatement of the reference algorithm (oracle port), timed in-process
        from oracle import port
        times = []
        for i in range(reps):
            t = time.perf_counter()
            port.planted(PLANTED["atoms"], PLANTED["nogoods"], PLANTED["pct"], PLANTED["seed"])
            if i >= args.warmup:
                times.append((time.perf_counter() - t) * 1e3)
        kind = "port"
    checks = planted_checks()["checks"]
    ms = statistics.mean(times)
    value = checks / (ms / 1e3)
    line = {
        "impl": "reference", "metric": "nogood checks/sec", "value": value, "unit": "checks/s", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "solver": "aspine Propagator workers=1"},
        "cpu_baseline": {"value": value, "unit": "checks/s", "cores": 1, "kind": kind,
                         "sample": f"{args.steps} full propagate_and_check calls ({checks} checks each)"},
        "e2e": {"value": value, "unit": "checks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def log(msg):
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def main():
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("BENCH_WATCHDOG_S", "1500")), exit=True)  # a hung section names itself on stderr
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="yasmin", choices=["yasmin", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="skip enumeration / first-model sections")
    args = ap.parse_args()
    if args.impl == "reference":  # CPU only: no process group needed; rank 0 runs it
        reference_arm(args, int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")))
        return
    rank, world, local = dist_setup(args.gpus)

    import torch
    import paper_1909_01786_b200 as Y
    from workloads import instances as I

    torch.cuda.set_device(local)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    store, seeded_list, dec = Y.NogoodStore.planted(**PLANTED)
    prop = Y.Propagator(store, 16, engine="grid", device=local)
    # step inputs live in pinned host memory: the seeded assignment and the
    # frontier (decision first), as int32
    seeded = torch.tensor(seeded_list, dtype=torch.int32).pin_memory().numpy()
    frontier = torch.tensor([dec] + seeded_list, dtype=torch.int32).pin_memory().numpy()

    def prepare():
        prop.reset()
        prop.push_decision(dec)
        prop.assign_propagated(seeded, 2)
        prop.seed(frontier)

    for _ in range(args.warmup):
        prepare()
        prop.flush()
        flush.zero_()
        torch.cuda.synchronize()
        o = prop.propagate_and_check(2)
    # exact literal count of the checked nogoods (roofline bytes), untimed
    prop.count_literals(True)
    prepare()
    lits_per_step = prop.propagate_and_check(2).checked_lits
    prop.count_literals(False)
    barrier(world)
    torch.cuda.synchronize()
    dev_ms, checks, lits, launches = [], 0, 0, 0
    t0 = time.perf_counter()
    with Clocks(local) as clk:
        for _ in range(args.steps):
            prepare()
            prop.flush()  # the prepare calls run as their own kernel, outside the propagation's timing
            flush.zero_()  # L2 flushed between timed iterations
            torch.cuda.synchronize()
            o = prop.propagate_and_check(2)  # one kernel launch: all passes to fixpoint
            launches += 2  # the batched prepare calls, the propagation (torch's L2 flush not counted)
            dev_ms.append(o.device_ms)
            checks += o.checks
            lits += lits_per_step
            assert not o.violated
    torch.cuda.synchronize()
    barrier(world)
    wall = time.perf_counter() - t0
    total_ms = allreduce([sum(dev_ms)], "max", world)[0]
    all_checks = allreduce([float(checks)], "sum", world)[0]
    value = all_checks / (total_ms / 1e3)
    avg_ms = statistics.mean(dev_ms)
    algo_bytes = (12 * checks + 4 * lits) / args.steps  # per launch, SURVEY.md §8(d)
    peak, peak_kind = peaks()
    achieved = algo_bytes / (avg_ms / 1e3) / 1e9
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", "r02_planted_grid.json")
    if os.path.exists(prof_json):
        with open(prof_json) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    # ---- e2e through the public API with host buffers ----------------------
    e2e_ms = []
    trail_buf = torch.empty(prop.atoms + 1, dtype=torch.int32).pin_memory().numpy()
    moved = []
    for _ in range(args.steps):
        flush.zero_()  # L2 flushed before every step, as for `value` (outside the timed region)
        torch.cuda.synchronize()
        b0 = prop.transfers()
        t = time.perf_counter()
        prepare()  # H2D: decision + seeded assignment + frontier
        o = prop.propagate_and_check(2)
        tr = prop.trail_array(trail_buf)  # D2H: the fixpoint trail, into pinned host memory
        e2e_ms.append((time.perf_counter() - t) * 1e3)
        b1 = prop.transfers()
        moved.append((b1[0] - b0[0], b1[1] - b0[1]))
    e2e_max = allreduce([statistics.mean(e2e_ms)], "max", world)[0]
    exp1m = next(e for e in pins()["planted_1m"] if e["pct"] == PLANTED["pct"])
    parity = {"planted_1m": planted_parity(prop, o, exp1m) and checks == 1_077_320 * args.steps}
    h2d = max(m[0] for m in moved)  # counted by the library at each copy
    d2h = max(m[1] for m in moved)

    line = {
        "metric": "nogood checks/sec", "value": value, "unit": "checks/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "parallelism": f"replicas x{world} (propagation does not shard)",
                   "engine": "grid (1 CTA/SM, cooperative)", "l2": "flushed between steps (512 MiB write)",
                   "timed": "propagate_and_check kernel, CUDA events on its stream"},
        "checks_per_step": checks / args.steps, "passes_per_step": o.passes,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_kind,
                     "algorithmic_bytes_per_launch": algo_bytes,
                     "bytes_model": "12 B/check (occurrence + offset + guard) + 4 B/literal of checked nogoods"},
        "e2e": {"value": (all_checks / args.steps) / (e2e_max / 1e3), "unit": "checks/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_max,
                "bytes": "counted by the propagator at every copy (yas_propagator_transfers)",
                "l2": "flushed before every step, outside the timed region"},
        "clocks": clk.summary(), "gpu_launches": launches, "bracket_wall_s": wall,
        "parity": parity,
    }

    log("cpu baseline")
    if rank == 0:
        try:
            if os.path.exists(REF_BIN):
                ref = run_reference_planted(3)
                cpu_ms = statistics.mean(ref["prop_ms"])
                kind = "reference"
            else:
                from oracle import port
                t = time.perf_counter()
                port.planted(**PLANTED)
                cpu_ms = (time.perf_counter() - t) * 1e3
                kind = "port"
            line["cpu_baseline"] = {"value": checks / args.steps / (cpu_ms / 1e3), "unit": "checks/s", "cores": 1,
                                    "kind": kind, "sample": "3 full propagate_and_check calls on the same store "
                                                            "(workers=1, the reference's fastest setting)",
                                    "ms_per_call": cpu_ms}
        except Exception as e:  # never let the baseline break the line
            line["cpu_baseline"] = {"value": None, "unit": "checks/s", "cores": 1, "kind": "reference",
                                    "sample": f"failed: {e}"}

    if not args.no_extras:
        del prop
        log("planted 8M")
        line["planted_8m"] = planted_large(Y, torch, flush, local)
        parity["planted_8m"] = line["planted_8m"].pop("parity")
        log("enumeration")
        line["enumeration"] = enumeration(Y, I, rank, world, local)
        line["enumeration_q8"] = enumeration(Y, I, rank, world, local, n=8)
        parity["queens12"] = line["enumeration"].pop("parity")
        parity["queens8"] = line["enumeration_q8"].pop("parity")
        log("enumeration q13 (scaling workload)")
        line["enumeration_q13"] = enumeration(Y, I, rank, world, local, n=13)
        parity["queens13"] = line["enumeration_q13"].pop("parity")
        if rank == 0:
            log("random program 4a")
            line["random_program_4a"] = random_program(Y, I, local)
            parity["rand4a"] = line["random_program_4a"].pop("parity")
            log("first model")
            line["first_model"] = first_model(Y, I, local)
        log("done")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def planted_large(Y, torch, flush, local, steps=5):
    """Config 4b scaled past the 126 MB L2: 8M nogoods / 800k atoms (fat
    occurrence entries alone are 512 MB), same recipe and seeding."""
    cfg = dict(atoms=800_000, nogoods=8_000_000, pct=50, seed=0x1B00B5)
    store, seeded_list, dec = Y.NogoodStore.planted(**cfg)
    prop = Y.Propagator(store, 16, engine="grid", device=local)
    seeded = torch.tensor(seeded_list, dtype=torch.int32).pin_memory().numpy()
    frontier = torch.tensor([dec] + seeded_list, dtype=torch.int32).pin_memory().numpy()

    def run():
        prop.reset()
        prop.push_decision(dec)
        prop.assign_propagated(seeded, 2)
        prop.seed(frontier)
        prop.flush()
        flush.zero_()
        torch.cuda.synchronize()
        return prop.propagate_and_check(2)

    for _ in range(2):
        run()
    prop.count_literals(True)
    lits = run().checked_lits
    prop.count_literals(False)
    outs = [run() for _ in range(steps)]
    parity = planted_parity(prop, outs[-1], pins()["planted_8m"][0])
    ms = statistics.mean(o.device_ms for o in outs)
    checks = outs[-1].checks
    peak, _ = peaks()
    achieved = (12 * checks + 4 * lits) / (ms / 1e3) / 1e9
    out = {"workload": "planted 8M nogoods / 800k atoms, 50% seeded (exceeds L2)", "checks_per_step": checks,
           "passes": outs[-1].passes, "ms_per_step": ms, "checks_per_s": checks / (ms / 1e3),
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak},
           "l2": "flushed before every step", "parity": parity}
    if os.path.exists(REF_BIN):  # one reference call on the same store (bounded: ~1 s)
        r = subprocess.run([REF_BIN, "planted", str(cfg["atoms"]), str(cfg["nogoods"]), str(cfg["pct"]),
                            hex(cfg["seed"]), "1"], capture_output=True, text=True, check=True)
        ref_ms = json.loads(r.stdout)["prop_ms"][0]
        out["cpu_reference"] = {"ms_per_call": ref_ms, "checks_per_s": checks / (ref_ms / 1e3), "cores": 1}
    return out


def random_program(Y, I, local):
    """Config 4a: the 100k-atom / 111k-rule random program (986k nogoods),
    solved to its first answer set by propagation alone (grid engine)."""
    text = I.random_program()
    t = time.perf_counter()
    prog = Y.parse_program(text)
    load_ms = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    Y.solve(prog, Y.SolverConfig(device=local))
    solve_ms = (time.perf_counter() - t) * 1e3  # first call: completion + store build + upload + search + result
    t = time.perf_counter()
    r = Y.solve(prog, Y.SolverConfig(device=local))
    solve_cached_ms = (time.perf_counter() - t) * 1e3  # the program keeps its compiled store
    lits = Y.solve(prog, Y.SolverConfig(device=local, count_lits=True)).stats.checked_lits  # untimed
    dev = [Y.solve(prog, Y.SolverConfig(device=local)).stats.device_ms for _ in range(3)]
    dev_ms = statistics.mean(dev)
    algo = 12 * r.stats.checks + 4 * lits
    peak, _ = peaks()
    exp = pins()["rand4a"]
    keys = [k for k in exp["stats"] if k not in ("wall_ms", "watch_replacements")]
    parity = (r.status.name.upper() == exp["status"] and all(getattr(r.stats, k) == exp["stats"][k] for k in keys)
              and len(r.models) == 1 and model_set_digest([r.models[0].atom_ids]) == exp["model_digest"])
    out = {"status": r.status.name, "device_ms": dev_ms, "passes": r.stats.passes,
           "checks": r.stats.checks, "checks_per_s": r.stats.checks / (dev_ms / 1e3),
           "parse_ms": load_ms, "solve_wall_ms": solve_ms, "solve_wall_ms_compiled": solve_cached_ms,
           "decisions": r.stats.decisions, "parity": parity,
           "roofline": {"bound": "hbm", "achieved": algo / (dev_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": algo / (dev_ms / 1e3) / 1e9 / peak, "algorithmic_bytes_per_launch": algo,
                        "checked_lits": lits, "timed": "whole solve kernel (initial propagation + 54 passes + "
                                                       "model), CUDA events, mean of 3, L2 warm"}}
    if os.path.exists(REF_BIN):
        p = subprocess.run([REF_BIN, "solve", "-", "-n", "1", "--no-models", "--reps", "2"], input=text,
                           capture_output=True, text=True, check=True)
        ref = json.loads(p.stdout)
        out["cpu_reference_run_ms"] = statistics.mean(ref["run_ms"])
        out["cpu_reference_parse_ms"] = ref["parse_ms"]
        out["cpu_reference_solve_wall_ms"] = statistics.mean(ref["solve_ms"])  # compile + build + run
        out["same_trajectory"] = all(getattr(r.stats, k) == ref["stats"][k]
                                     for k in ("decisions", "propagations", "conflicts", "passes"))
    return out


def cpu_cube_split(Y, text, cubes):
    """Config 5 CPU side: the same cube set, one reference solve per cube,
    on every host core (one process each); wall time of the whole set and the model set."""
    import tempfile
    prog = Y.parse_program(text)
    nproc = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as d:
        lp, cf = os.path.join(d, "p.lp"), os.path.join(d, "cubes.txt")
        with open(lp, "w") as f:
            f.write(text)
        with open(cf, "w") as f:
            for c in cubes:
                f.write(" ".join(prog.name(abs(l)) for l in c if l) + "\n")
        t = time.perf_counter()
        procs = [subprocess.Popen([REF_BIN, "cubes", lp, cf, str(k), str(nproc)], stdout=subprocess.PIPE, text=True)
                 for k in range(nproc)]
        outs = [json.loads(p.communicate()[0]) for p in procs]
        wall = (time.perf_counter() - t) * 1e3
    models = [m for o in outs for m in o["models"]]
    return {"cores": nproc, "processes": nproc, "cubes": len(cubes), "wall_ms": wall,
            "models": len(models), "model_set_digest": model_set_digest(models)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


_FLEET = None


def fleet(Y, rank, world, local):
    """The product's multi-GPU path: one fleet of all ranks (rank 0's GPU holds the
    shared cube queue, NCCL for the final all-reduce; gloo process group on a
    shared-GPU check)."""
    global _FLEET
    if world == 1:
        return None
    if _FLEET is None:
        import torch.distributed as dist
        if dist.get_backend() == "gloo":
            _FLEET = Y.Fleet.from_process_group(local)
        else:
            uid = [Y.Fleet.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            _FLEET = Y.Fleet.nccl(uid[0], rank, world, local)
    return _FLEET


def enumeration(Y, I, rank, world, local, n=12):
    """n-queens, all answer sets through the unchanged reference call (max_models=0):
    automatic ladder cubes from one queue shared by every GPU (SolverConfig.fleet);
    the model count comes from the product's own all-reduce, time is the max over ranks."""
    from paper_1909_01786_b200 import aspine as A
    text = I.queens(n)
    fl = fleet(Y, rank, world, local)
    # the drop-in default: a plain enumeration (max_models=0) is cube-split automatically,
    # ladders over the rows ("at least one queen per row" constraints)
    cfg = Y.SolverConfig(max_models=0, device=local, fleet=fl)
    Y.solve(Y.parse_program(text), cfg)  # warm-up (module load, allocations)
    barrier(world)
    t = time.perf_counter()
    prog = Y.parse_program(text)
    r = Y.solve(prog, cfg)
    wall = (time.perf_counter() - t) * 1e3
    n_models = r.stats.fleet_models
    cubes = allreduce([float(r.stats.cubes)], "sum", world)[0]
    wall_max, dev_max = allreduce([wall, r.stats.device_ms], "max", world)
    out = {"instance": f"queens{n} (all answer sets)", "models": int(n_models),
           "expected_models": {8: 92, 10: 724, 12: 14200, 13: 73712}.get(n),
           "wall_ms": wall_max, "device_ms": dev_max, "cubes": int(cubes), "n_gpus": world,
           "passes_rank0": r.stats.passes, "cube_queue": "shared (fleet)" if fl is not None else "one GPU"}
    # parity: the union of every rank's models against the reference's model set
    ids = [list(m.atom_ids) for m in r.models]
    if world > 1:
        import torch.distributed as dist
        parts = [None] * world
        dist.all_gather_object(parts, ids)
        ids = [m for part in parts for m in part]
    if n >= 12:
        exp = pins()[f"queens{n}"]
        out["parity"] = len(ids) == exp["models"] and model_set_digest(ids) == exp["model_set_digest"]
    else:
        with open(os.path.join(ROOT, "tests", "golden", "configs.json")) as f:
            exp8 = json.load(f)["queens8/fwd/occ"]["models"]
        out["parity"] = sorted(ids) == sorted(exp8)
    if rank == 0 and os.path.exists(REF_BIN):
        if n <= 8:  # the whole single-thread enumeration is a bounded sample
            p = subprocess.run([REF_BIN, "solve", "-", "-n", "0", "--no-models", "--reps", "3"], input=text,
                               capture_output=True, text=True, check=True)
            ref = json.loads(p.stdout)
            out["cpu_reference"] = {"sample": f"queens{n}, all models, workers=1, mean of 3",
                                    "run_ms": statistics.mean(ref["run_ms"]), "cores": 1}
        else:
            # the same cube set on every host core (one reference process per core); the
            # full single-thread run (~3 min) is measured once by scripts/cpu_q12_reference.py
            cubes_all = A.cubes(prog, 0, 0, want=4 * 148 * 8 * world)  # the same automatic cube set
            cs = cpu_cube_split(Y, text, cubes_all)
            cs["parity"] = cs["models"] == out["expected_models"] and (
                cs["model_set_digest"] == pins()[f"queens{n}"]["model_set_digest"])
            cs["cpu_model"] = cpu_model()
            out["cpu_reference_cube_split"] = cs
            full = os.path.join(ROOT, "profiles", "r02_q12_reference_full.json")
            if n == 12 and os.path.exists(full):
                with open(full) as f:
                    out["cpu_reference_full"] = json.load(f)
        out["models_per_s"] = n_models / (wall_max / 1e3)
    return out


def first_model(Y, I, local):
    out = {}
    for name, text in (("colour2000", I.colouring(2000, 4.0, 3, 1)), ("ham200", I.hamiltonian(200, 1.0, 1))):
        prog = Y.parse_program(text)
        Y.solve(prog, Y.SolverConfig(device=local))
        t = time.perf_counter()
        r = Y.solve(prog, Y.SolverConfig(device=local))
        entry = {"status": r.status.name, "wall_ms": (time.perf_counter() - t) * 1e3, "device_ms": r.stats.device_ms,
                 "decisions": r.stats.decisions, "passes": r.stats.passes}
        if os.path.exists(REF_BIN):
            p = subprocess.run([REF_BIN, "solve", "-", "-n", "1", "--no-models", "--reps", "3"], input=text,
                               capture_output=True, text=True, check=True)
            ref = json.loads(p.stdout)
            entry["cpu_reference_run_ms"] = statistics.mean(ref["run_ms"])
            entry["same_trajectory"] = all(getattr(r.stats, k) == ref["stats"][k]
                                           for k in ("decisions", "propagations", "conflicts", "passes"))
        # extra mode: six concurrent searches over (mode, heuristic), first one reports;
        # an answer set, not the reference's first one
        t = time.perf_counter()
        rp = Y.solve(prog, Y.SolverConfig(device=local, portfolio=6))
        entry["portfolio6"] = {"status": rp.status.name, "wall_ms": (time.perf_counter() - t) * 1e3,
                               "device_ms": rp.stats.device_ms, "winner_variant": rp.stats.portfolio_variant}
        out[name] = entry
    return out


if __name__ == "__main__":
    main()
