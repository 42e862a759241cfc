"""Bit-exact parity on every configuration bench.py reports, against the UNMODIFIED
reference run at full size (tests/golden/pins.json, made by make_golden.py pins):

* config 4b, planted 1M nogoods at 1/10/50/90 % seeds and 8M at 50 %: propagation
  count, pass count, trail length and the FNV digests of the trail literals, of the
  reasons and of Deps word 0 + overflow, in trail order
  (/root/reference/proj/src/propagate.cpp:170-205, oracle/ref_harness.cpp cmd_planted);
* config 4a, the 986k-nogood random program: first answer set and every SolveStats
  counter (/root/reference/proj/src/solver.cpp:248-303);
* config 5, queens(12): all 14,200 answer sets of the cube-split enumeration as a
  model-set digest, and each model checked to be an answer set
  (/root/reference/proj/src/solver.cpp:216-246, oracle.cpp is_answer_set).
"""
import pytest

import paper_1909_01786_b200 as Y
from workloads import instances as I

from _util import STAT_KEYS, golden, model_set_digest, stats_diff, trail_digests

pytestmark = pytest.mark.gpu


def planted_run(exp, engine):
    s, seeded, dec = Y.NogoodStore.planted(exp["atoms"], exp["nogoods"], exp["pct"])
    assert len(seeded) == exp["seeded"]
    p = Y.Propagator(s, 16, engine)
    p.push_decision(dec)
    p.assign_propagated(seeded, 2)
    p.seed([dec] + seeded)
    o = p.propagate_and_check(2)
    assert not o.violated and not o.conflicts
    assert (o.propagations, o.passes) == (exp["propagations"], exp["passes"])
    assert trail_digests(p) == (exp["trail"], exp["trail_digest"], exp["reason_digest"], exp["deps_digest"])
    return o


@pytest.mark.parametrize("pct", [1, 10, 50, 90])
def test_planted_1m_matches_reference(pct):
    exp = next(e for e in golden("pins")["planted_1m"] if e["pct"] == pct)
    o = planted_run(exp, "grid")
    if pct == 50:
        assert o.checks == 1_077_320  # the reference's item count


def test_planted_1m_block_engine_matches_reference():
    """The single-CTA engine reaches the same fixpoint on the full-size store."""
    planted_run(next(e for e in golden("pins")["planted_1m"] if e["pct"] == 50), "block")


def test_planted_8m_matches_reference():
    planted_run(golden("pins")["planted_8m"][0], "grid")


def test_random_program_4a_first_model():
    exp = golden("pins")["rand4a"]
    r = Y.solve(Y.parse_program(I.random_program()), Y.SolverConfig())
    assert r.status.name.upper() == exp["status"] and len(r.models) == 1
    assert not stats_diff(r.stats, exp["stats"]), stats_diff(r.stats, exp["stats"])
    assert len(r.models[0].atom_ids) == exp["model_len"]
    assert model_set_digest([r.models[0].atom_ids]) == exp["model_digest"]


def test_queens12_cube_split_model_set():
    exp = golden("pins")["queens12"]
    prog = Y.parse_program(I.queens(12))
    r = Y.solve(prog, Y.SolverConfig(max_models=0, cube_atoms=12))
    ids = [m.atom_ids for m in r.models]
    assert len(ids) == exp["models"] == 14_200 and r.status.name.upper() == exp["status"]
    assert len({tuple(m) for m in ids}) == len(ids)
    assert model_set_digest(ids) == exp["model_set_digest"]
    for m in r.models:
        assert Y.verify_model(prog, m)


def test_stat_keys_cover_reference_counters():
    """Every counter of the pinned 4a run is compared except wall time and watches."""
    exp = golden("pins")["rand4a"]["stats"]
    assert set(exp) - set(STAT_KEYS) == {"wall_ms", "watch_replacements"}


def test_queens13_two_devices_model_set():
    """queens(13) (73,712 answer sets), the scaling workload, through one shared
    cube queue over two GPUs of the process (the same B200 listed twice here)."""
    exp = golden("pins")["queens13"]
    r = Y.solve(Y.parse_program(I.queens(13)), Y.SolverConfig(max_models=0, cube_atoms=13, devices=[0, 0]))
    ids = [m.atom_ids for m in r.models]
    assert len(ids) == exp["models"] == 73_712
    assert model_set_digest(ids) == exp["model_set_digest"]
