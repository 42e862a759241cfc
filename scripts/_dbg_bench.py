import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1909_01786_b200 as Y
from paper_1909_01786_b200 import instances as I
which = sys.argv[1]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
t = time.time()
if which == "p8":
    print(json.dumps(bench.planted_large(Y, torch, flush, 0)), flush=True)
elif which == "enum":
    print(json.dumps(bench.enumeration(Y, I, 0, 1, 0)), flush=True)
elif which == "r4a":
    print(json.dumps(bench.random_program(Y, I, 0)), flush=True)
elif which == "fm":
    print(json.dumps(bench.first_model(Y, I, 0)), flush=True)
print(which, "took", time.time() - t, flush=True)
