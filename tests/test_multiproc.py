"""Multi-process cube split on CPU (gloo, world size 2): the host partition of
cubes across ranks and the final count all-reduce. The per-rank solve itself
needs a GPU and is covered by tests/test_gpu_cubes.py."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1909_01786_b200 as Y
    from paper_1909_01786_b200 import aspine as A
    from workloads import instances as I
    p = Y.parse_program(I.queens(6))
    mine = A.cubes(p, 6, 2, rank, world)
    n = torch.tensor([len(mine)], dtype=torch.int64)
    dist.all_reduce(n)
    gathered = [None] * world
    dist.all_gather_object(gathered, [tuple(c) for c in mine])
    if rank == 0:
        q.put((int(n.item()), gathered))
    dist.destroy_process_group()


def test_cube_partition_allreduce_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    total, gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert total == 49
    cubes = [c for part in gathered for c in part]
    assert len(cubes) == 49 and len(set(cubes)) == 49
    assert not set(gathered[0]) & set(gathered[1])
