"""Developer probe: planted-store propagation (config 4b recipe) at growing store sizes,
L2 flushed before every call: time, checks/s and the roofline fraction of the bench's
bytes model (12 B/check + 4 B/literal).
    python scripts/planted_scale.py [nogoods_in_millions ...]"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1909_01786_b200 as Y  # noqa: E402

peak = 6456.8
try:
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f).get("hbm_gbs", peak))
except (OSError, ValueError):
    pass
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for m in [int(x) for x in sys.argv[1:]] or [1, 8, 32]:
    t0 = time.time()
    store, seeded, dec = Y.NogoodStore.planted(100_000 * m, 1_000_000 * m, 50)
    prop = Y.Propagator(store, 16, engine="grid")
    sd = torch.tensor(seeded, dtype=torch.int32).pin_memory().numpy()
    fr = torch.tensor([dec] + seeded, dtype=torch.int32).pin_memory().numpy()
    build_s = time.time() - t0

    def run():
        prop.reset(); prop.push_decision(dec); prop.assign_propagated(sd, 2); prop.seed(fr)
        prop.flush()
        flush.zero_()
        torch.cuda.synchronize()
        return prop.propagate_and_check(2)

    run()
    prop.count_literals(True)
    lits = run().checked_lits
    prop.count_literals(False)
    outs = [run() for _ in range(5)]
    ms = statistics.mean(o.device_ms for o in outs)
    o = outs[-1]
    gbs = (12 * o.checks + 4 * lits) / (ms / 1e3) / 1e9
    print(json.dumps({"nogoods": 1_000_000 * m, "atoms": 100_000 * m, "ms": round(ms, 4), "passes": o.passes,
                      "checks": o.checks, "propagations": o.propagations, "checks_per_s": o.checks / (ms / 1e3),
                      "achieved_gbs": round(gbs, 1), "frac": round(gbs / peak, 4), "build_s": round(build_s, 1)}),
          flush=True)
    del prop, store
