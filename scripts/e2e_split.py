"""Developer probe: where the end-to-end planted call goes (host staging, the batched
prepare kernel, the propagation kernel, the trail read-back)."""
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1909_01786_b200 as Y  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
store, seeded, dec = Y.NogoodStore.planted(100_000, 1_000_000, 50)
prop = Y.Propagator(store, 16, engine="grid")
sd = torch.tensor(seeded, dtype=torch.int32).pin_memory().numpy()
fr = torch.tensor([dec] + seeded, dtype=torch.int32).pin_memory().numpy()
buf = torch.empty(prop.atoms + 1, dtype=torch.int32).pin_memory().numpy()
rows = []
for rep in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prop.reset(); prop.push_decision(dec); prop.assign_propagated(sd, 2); prop.seed(fr)
    t1 = time.perf_counter()
    prop.flush(); torch.cuda.synchronize()
    t2 = time.perf_counter()
    o = prop.propagate_and_check(2)
    t3 = time.perf_counter()
    tr = prop.trail_array(buf)
    t4 = time.perf_counter()
    if rep >= 2:
        rows.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, o.device_ms, (t4 - t3) * 1e3))
names = ["record+stage", "prepare kernel (wall)", "propagate (wall)", "propagate (device)", "trail D2H"]
for k, n in enumerate(names):
    print(f"{n}: {statistics.mean(r[k] for r in rows):.3f} ms")
