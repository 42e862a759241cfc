"""Multi-GPU enumeration and portfolio inside the product: several
GPUs of one process (SolverConfig.devices) or several processes (Fleet) take cubes
from ONE queue in the home GPU's memory and all-reduce counts and flags at the end.
The GPU boxes here have one B200, so the "GPUs" are the same device listed twice
and the processes share it; the queue, claim and collectives are the same code
that runs over NVLink peers on an 8-GPU node. Answer-set sets must equal the
reference's (tests/golden), exactly as for the single-GPU cube split."""
import os
import socket

import pytest

import paper_1909_01786_b200 as Y
from workloads import instances as I

from _util import golden, model_set_digest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_devices_one_queue_queens8():
    exp = sorted(golden("configs")["queens8/fwd/occ"]["models"])
    r = Y.solve(Y.parse_program(I.queens(8)), Y.SolverConfig(max_models=0, cube_atoms=8, devices=[0, 0]))
    got = sorted(m.atom_ids for m in r.models)
    assert got == exp
    assert r.stats.devices == 2 and r.stats.fleet_models == 92
    total = len(Y.cubes(Y.parse_program(I.queens(8)), 8, 0, want=4 * 148 * 8 * 2))
    assert r.stats.cubes == r.stats.searches == total  # every cube searched exactly once over both GPUs


def test_two_devices_one_queue_queens10():
    r = Y.solve(Y.parse_program(I.queens(10)), Y.SolverConfig(max_models=0, cube_atoms=10, devices=[0, 0]))
    ids = [tuple(m.atom_ids) for m in r.models]
    assert len(ids) == 724 and len(set(ids)) == 724


def test_two_devices_portfolio_reports_one_answer_set():
    prog = Y.parse_program(I.colouring(200, 4.0, 3, 1))
    r = Y.solve(prog, Y.SolverConfig(portfolio=3, devices=[0, 0]))
    assert r.status == Y.SolveStatus.sat and len(r.models) == 1 and Y.verify_model(prog, r.models[0])
    assert r.stats.devices == 2 and r.stats.portfolio_variant >= 0 and r.stats.fleet_winner == 0


def test_nccl_fleet_of_one():
    f = Y.Fleet.nccl(Y.Fleet.unique_id(), 0, 1, 0)
    assert f.info() == {"rank": 0, "world": 1, "device": 0, "dynamic": True}
    assert f.allreduce([3, 4], "sum") == [3, 4]
    exp = sorted(golden("configs")["queens8/fwd/occ"]["models"])
    r = Y.solve(Y.parse_program(I.queens(8)), Y.SolverConfig(max_models=0, cube_atoms=8, fleet=f))
    assert sorted(m.atom_ids for m in r.models) == exp and r.stats.fleet_models == 92 and r.stats.fleet_ranks == 1
    with pytest.raises(ValueError):
        Y.solve(Y.parse_program(I.queens(8)), Y.SolverConfig(max_models=0, cube_atoms=8, fleet=f, devices=[0, 0]))
    f.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1909_01786_b200 as Y
    from workloads import instances as I
    try:
        f = Y.Fleet.from_process_group(0)
        info = f.info()
        r = Y.solve(Y.parse_program(I.queens(10)), Y.SolverConfig(max_models=0, cube_atoms=10, fleet=f))
        enum = ([list(m.atom_ids) for m in r.models], r.stats.fleet_models, r.stats.searches, r.stats.fleet_ranks)
        prog = Y.parse_program(I.colouring(200, 4.0, 3, 1))
        p = Y.solve(prog, Y.SolverConfig(portfolio=2, fleet=f))
        port = (p.status.name, [list(m.atom_ids) for m in p.models], p.stats.fleet_winner,
                all(Y.verify_model(prog, m) for m in p.models))
        f.close()
        q.put((rank, info, enum, port))
    except Exception as e:  # surfaced by the parent
        q.put((rank, repr(e), None, None))
    dist.destroy_process_group()


def test_fleet_two_processes_share_one_queue():
    """Two processes on the GPU, gloo as the transport: one cube queue (CUDA IPC),
    model sets union to the reference's 724 with no overlap, counts all-reduced;
    a two-process portfolio reports exactly one winner."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, info, enum, port_ in out:
        assert enum is not None, info
        assert info["dynamic"] and info["world"] == 2
    models = [tuple(m) for _, _, enum, _ in out for m in enum[0]]
    assert len(models) == 724 and len(set(models)) == 724
    assert all(enum[1] == 724 and enum[3] == 2 for _, _, enum, _ in out)
    assert sum(enum[2] for _, _, enum, _ in out) == out[0][2][2] + out[1][2][2]
    winners = {port_[2] for _, _, _, port_ in out}
    assert len(winners) == 1 and winners.pop() in (0, 1)
    reported = [port_ for _, _, _, port_ in out if port_[1]]
    assert len(reported) == 1 and reported[0][0] == "sat" and reported[0][3]
    assert all(port_[0] == "sat" for _, _, _, port_ in out)


def test_queens12_two_devices_model_set():
    exp = golden("pins")["queens12"]
    r = Y.solve(Y.parse_program(I.queens(12)), Y.SolverConfig(max_models=0, cube_atoms=12, devices=[0, 0]))
    ids = [m.atom_ids for m in r.models]
    assert len(ids) == exp["models"] and model_set_digest(ids) == exp["model_set_digest"]
