"""Developer probe: warm-up calls then one planted propagation (ncu target).
    python scripts/planted_once.py atoms nogoods pct"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1909_01786_b200 as Y  # noqa: E402

atoms, nogoods, pct = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (100_000, 1_000_000, 50)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
store, seeded, dec = Y.NogoodStore.planted(atoms, nogoods, pct)
prop = Y.Propagator(store, 16, engine="grid")
sd = np.asarray(seeded, dtype=np.int32)
fr = np.asarray([dec] + seeded, dtype=np.int32)
for rep in range(4):
    prop.reset(); prop.push_decision(dec); prop.assign_propagated(sd, 2); prop.seed(fr)
    prop.flush()
    flush.zero_()
    torch.cuda.synchronize()
    o = prop.propagate_and_check(2)
print(f"{o.device_ms * 1e3:.1f} us, passes {o.passes}, checks {o.checks}")
