"""Developer probe: per-pass phase timeline of a grid propagation (planted store).

    python scripts/pass_trace.py atoms nogoods pct
Prints per pass: T, F and for each phase the slowest block's work time and the
barrier time (last arrival -> first departure ... last departure)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1909_01786_b200 as Y  # noqa: E402

atoms, nogoods, pct = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (100_000, 1_000_000, 50)
store, seeded, dec = Y.NogoodStore.planted(atoms, nogoods, pct)
prop = Y.Propagator(store, 16, engine="grid")
sd = np.asarray(seeded, dtype=np.int32)
fr = np.asarray([dec] + seeded, dtype=np.int32)
import torch  # noqa: E402  (L2 flush, as in bench.py: timings with cold L2)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for rep in range(3):
    prop.reset(); prop.push_decision(dec); prop.assign_propagated(sd, 2); prop.seed(fr)
    if rep == 2:
        prop.pass_trace(True)
    prop.flush()
    flush.zero_()
    torch.cuda.synchronize()
    o = prop.propagate_and_check(2)
tr = prop.pass_trace().astype(np.int64)
print(f"kernel {o.device_ms * 1e3:.1f} us, passes {o.passes}")
phases = [("expand", 0, 1, 2), ("resolve", 2, 3, 4), ("select", 4, 5, 6), ("place", 6, 7, 8)]
tot = {}
for p in range(min(o.passes, 64)):
    t = tr[p]
    if not t[:, 0].any():
        break
    T, F = int(t[0, 9]) >> 32, int(t[0, 9]) & 0xffffffff
    if not t[1:, 0].any():  # solo pass: block 0 only
        t = t[:1]
    parts = []
    for name, a, b, c in phases:
        work = (t[:, b] - t[:, a])
        arrive_last = t[:, b].max()
        leave = t[:, c]
        barrier = leave.max() - arrive_last
        parts.append(f"{name} work max {work.max() / 1e3:6.2f} med {np.median(work) / 1e3:5.2f} bar {barrier / 1e3:5.2f}")
        tot[name] = tot.get(name, 0) + (t[:, c].max() - t[:, a].min())
    print(f"pass {p:3d} T={T:8d} F={F:7d} | " + " | ".join(parts))
print("phase totals (us):", {k: round(v / 1e3, 1) for k, v in tot.items()})
d = prop.pass_debug.astype(np.int64)
print("expand, warp 0 of block 0 (cycles since expand start): search | first batch: pe, trig+entry, claims+mirror, decide, props, scans | end")
for p in range(min(o.passes, 64)):
    if d[p, 0]:
        print(f"pass {p:3d}: " + " ".join(f"{int(d[p, k] - d[p, 0]):6d}" for k in range(1, 9)))
