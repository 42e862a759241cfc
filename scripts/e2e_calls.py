"""Developer probe: host-side cost of each call of the end-to-end planted step
(bench.py's e2e loop), L2 flushed before every step."""
import os
import statistics
import sys
import time

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
names = ["reset", "push_decision", "assign", "seed", "propagate", "trail", "total"]
rows = []
for rep in range(25):
    flush.zero_()
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    prop.reset(); t.append(time.perf_counter())
    prop.push_decision(dec); t.append(time.perf_counter())
    prop.assign_propagated(sd, 2); t.append(time.perf_counter())
    prop.seed(fr); t.append(time.perf_counter())
    o = prop.propagate_and_check(2); t.append(time.perf_counter())
    prop.trail_array(buf); t.append(time.perf_counter())
    if rep >= 5:
        rows.append([(t[k + 1] - t[k]) * 1e6 for k in range(6)] + [(t[6] - t[0]) * 1e6, o.device_ms * 1e3])
for k, n in enumerate(names + ["device (events)"]):
    print(f"{n:>16}: {statistics.mean(r[k] for r in rows):8.1f} us")
