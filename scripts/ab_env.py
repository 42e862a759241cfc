"""Developer probe: planted-store propagation A/B over an environment switch read
at every launch (e.g. YAS_PREFETCH_CLAIMS), L2 flushed before every call.
    python scripts/ab_env.py VAR [atoms nogoods pct]"""
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1909_01786_b200 as Y  # noqa: E402

var = sys.argv[1]
atoms, nogoods, pct = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (100_000, 1_000_000, 50)
store, seeded, dec = Y.NogoodStore.planted(atoms, nogoods, pct)
prop = Y.Propagator(store, 16, engine="grid")
sd = np.asarray(seeded, dtype=np.int32)
fr = np.asarray([dec] + seeded, dtype=np.int32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
times = {"0": [], "1": []}
for rep in range(24):
    mode = "01"[rep % 2]
    os.environ[var] = mode
    prop.reset(); prop.push_decision(dec); prop.assign_propagated(sd, 2); prop.seed(fr)
    prop.flush()
    flush.zero_()
    torch.cuda.synchronize()
    o = prop.propagate_and_check(2)
    if rep >= 4:
        times[mode].append(o.device_ms * 1e3)
for m, t in times.items():
    print(f"{var}={m}: mean {statistics.mean(t):.1f} us, min {min(t):.1f} us (n={len(t)}), passes {o.passes}")
