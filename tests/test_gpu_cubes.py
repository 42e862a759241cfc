"""Cube-split enumeration: answer-set sets and counts must equal the reference's
single-search enumeration (trajectories differ by design)."""
import pytest

import paper_1909_01786_b200 as Y
from workloads import instances as I

from _util import golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k,depth", [(1, 1), (4, 2), (8, 1), (8, 2), (8, 3), (5, 0)])
def test_queens8_cube_split_model_set(k, depth):
    exp = golden("configs")["queens8/fwd/occ"]["models"]
    r = Y.solve(Y.parse_program(I.queens(8)), Y.SolverConfig(max_models=0, cube_atoms=k, cube_depth=depth))
    got = sorted(m.atom_ids for m in r.models)
    assert got == sorted(exp) and len(got) == 92
    if depth:
        assert r.stats.searches == (k + 1) ** depth


def test_cube_split_by_rank_partitions_models():
    exp = sorted(golden("configs")["queens8/fwd/occ"]["models"])
    parts = []
    for rank in range(3):
        r = Y.solve(Y.parse_program(I.queens(8)), Y.SolverConfig(max_models=0, cube_atoms=8, cube_depth=2, rank=rank, world=3))
        parts.append(sorted(m.atom_ids for m in r.models))
    allm = sorted(m for p in parts for m in p)
    assert allm == exp


def test_corpus_cube_split_matches_families():
    for prog in golden("corpus")[::5]:
        r = Y.solve(Y.parse_program(prog["text"]), Y.SolverConfig(max_models=0, cube_atoms=3, cube_depth=2))
        assert sorted(m.atom_ids for m in r.models) == sorted(prog["family"]), prog["name"]


def test_queens10_count():
    r = Y.solve(Y.parse_program(I.queens(10)), Y.SolverConfig(max_models=0, cube_atoms=10, cube_depth=2))
    assert len(r.models) == 724 and len({tuple(m.atom_ids) for m in r.models}) == 724
    for m in r.models[:50]:
        assert Y.verify_model(Y.parse_program(I.queens(10)), m)


def test_corpus_generic_cubes_match_families():
    """Every corpus program split over rule heads as well as choice pairs (the
    passive ":- not a." cubes included): the union of the cubes' answer sets is
    the brute-force family (acceptance_main.cpp:85-123)."""
    bad = []
    for prog in golden("corpus"):
        p = Y.parse_program(prog["text"])
        r = Y.solve(p, Y.SolverConfig(max_models=0, cube_atoms=2, cube_depth=3))
        got = sorted(m.atom_ids for m in r.models)
        if got != sorted(prog["family"]) or len({tuple(m) for m in got}) != len(got):
            bad.append(prog["name"])
    assert not bad, bad[:10]


def test_cube_parallel_first_models():
    """cube_atoms with max_models >= 1: every cube searched in parallel, the first
    max_models answer sets found anywhere are reported (an extra mode, like the
    portfolio: answer sets of the program, not necessarily the reference's first)."""
    for text in (I.hamiltonian(200, 1.0, 1), I.colouring(2000, 4.0, 3, 1)):
        prog = Y.parse_program(text)
        r = Y.solve(prog, Y.SolverConfig(max_models=1, cube_atoms=8))
        assert r.status == Y.SolveStatus.sat and len(r.models) == 1 and Y.verify_model(prog, r.models[0])
    q = Y.parse_program(I.queens(8))
    r = Y.solve(q, Y.SolverConfig(max_models=3, cube_atoms=8))
    ids = [tuple(m.atom_ids) for m in r.models]
    assert len(ids) == 3 and len(set(ids)) == 3 and all(Y.verify_model(q, m) for m in r.models)
    php = Y.parse_program(I.pigeonhole(5, 4))  # no answer set: every cube fails
    r = Y.solve(php, Y.SolverConfig(max_models=1, cube_atoms=4))
    assert r.status == Y.SolveStatus.unsat and not r.models
    r = Y.solve(Y.parse_program(I.queens(8)), Y.SolverConfig(max_models=2, cube_atoms=8, devices=[0, 0]))
    assert len(r.models) == 2
