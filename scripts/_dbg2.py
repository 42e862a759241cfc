import os, sys, time, json, faulthandler
faulthandler.dump_traceback_later(90, exit=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1909_01786_b200 as Y
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
mode = sys.argv[1]
if mode in ("a", "b"):
    store, seeded, dec = Y.NogoodStore.planted(**bench.PLANTED)
    prop = Y.Propagator(store, 16, engine="grid")
    prop.reset(); prop.push_decision(dec); prop.assign_propagated(seeded, 2); prop.seed([dec] + seeded)
    o = prop.propagate_and_check(2)
    print("1M ok", o.passes, flush=True)
    if mode == "b":
        del prop
t = time.time()
print(json.dumps(bench.planted_large(Y, torch, flush, 0, steps=2)), time.time() - t, flush=True)
