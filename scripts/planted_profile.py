"""Developer probe: planted-store propagation time, phase split and e2e cost.

    python scripts/planted_profile.py [atoms nogoods pct] [reps]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1909_01786_b200 as Y  # noqa: E402

atoms, nogoods, pct = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (100_000, 1_000_000, 50)
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
t = time.perf_counter()
store, seeded, dec = Y.NogoodStore.planted(atoms, nogoods, pct)
print(f"store built in {time.perf_counter() - t:.2f}s, seeded {len(seeded)}")
prop = Y.Propagator(store, 16, engine="grid")
sd = np.asarray(seeded, dtype=np.int32)
fr = np.asarray([dec] + seeded, dtype=np.int32)
for r in range(reps):
    t0 = time.perf_counter()
    prop.reset(); prop.push_decision(dec); prop.assign_propagated(sd, 2); prop.seed(fr)
    t1 = time.perf_counter()
    o = prop.propagate_and_check(2)
    t2 = time.perf_counter()
    tr = prop.trail_array()
    t3 = time.perf_counter()
    split = ""
    print(f"rep {r}: kernel {o.device_ms * 1e3:.1f}us passes={o.passes} checks={o.checks} viol={o.violated} "
          f"trail={len(tr)} | {split} | host: prepare {1e3 * (t1 - t0):.2f}ms propagate {1e3 * (t2 - t1):.2f}ms "
          f"trail {1e3 * (t3 - t2):.2f}ms")
