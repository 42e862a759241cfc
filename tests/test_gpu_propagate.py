"""Propagation on the device vs the reference Propagator (P/tests/test_propagate.cpp),
through the C-ABI. Both engines: one CTA per search ("block") and whole grid ("grid")."""
import pytest

import paper_1909_01786_b200 as Y

from _util import golden, trail_digests

pytestmark = pytest.mark.gpu
ENGINES = ["block", "grid"]


def fnv(trail):
    h = 0xcbf29ce484222325
    for c in trail:
        h = ((h ^ (c & 0xFFFFFFFF)) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


@pytest.mark.parametrize("engine", ENGINES)
def test_initial_propagation_forces_unit_complements(engine):
    p = Y.Propagator(Y.NogoodStore.build([[1], [2]], 2), 1, engine)
    o = p.initial_propagation()
    assert not o.violated and p.cells()[1:] == [-1, -1] and o.propagations == 2 and len(p.frontier()) == 2


@pytest.mark.parametrize("engine", ENGINES)
def test_inconsistent_units_violate_with_pseudo_id(engine):
    p = Y.Propagator(Y.NogoodStore.build([[1], [-1]], 1), 1, engine)
    o = p.initial_propagation()
    assert o.violated and len(o.conflicts) == 1 and o.conflicts[0] < 0


@pytest.mark.parametrize("engine", ENGINES)
def test_learned_units_replayed(engine):
    p = Y.Propagator(Y.NogoodStore.build([[1, 2]], 3), 1, engine)
    lid = p.add_learned([3])
    assert lid == 1
    o = p.initial_propagation()
    assert not o.violated and p.cells()[3] == -1
    again = p.initial_propagation()
    assert not again.violated and p.frontier() == []


@pytest.mark.parametrize("engine", ENGINES)
def test_unit_propagation_copies_deps(engine):
    p = Y.Propagator(Y.NogoodStore.build([[1, 2]], 2), 2, engine)
    p.push_decision(1)
    p.seed([1])
    o = p.propagate_and_check(2)
    assert not o.violated and p.cells()[2] == -2 and p.reasons()[2] == 0 and o.propagations == 1
    d, _ = p.deps(0)
    assert d[1] == d[2] == 0b10


@pytest.mark.parametrize("engine", ENGINES)
def test_race_first_in_item_order_wins(engine):
    p = Y.Propagator(Y.NogoodStore.build([[1, 2], [1, -2]], 2), 1, engine)
    p.push_decision(1)
    p.seed([1])
    o = p.propagate_and_check(2)
    assert o.violated and p.cells()[2] == -2 and o.conflicts == [1]


@pytest.mark.parametrize("engine", ENGINES)
def test_violation_and_chain(engine):
    p = Y.Propagator(Y.NogoodStore.build([[1, 2, 3]], 3), 1, engine)
    p.push_decision(1)
    p.push_decision(2)
    p.assign_propagated([3], 3, [0b100])
    p.seed([3])
    o = p.propagate_and_check(3)
    assert o.violated and o.conflicts == [0]
    q = Y.Propagator(Y.NogoodStore.build([[1, 2], [-2, -3], [3, 4]], 4), 1, engine)
    q.push_decision(1)
    q.seed([1])
    o = q.propagate_and_check(2)
    assert not o.violated and o.propagations == 3 and o.passes >= 3
    assert q.cells()[2:] == [-2, 2, -2]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("key", ["test_propagate", "criterion5"])
def test_random_stores_match_reference(engine, key):
    """300 + 1000 random stores: outcome, cells, trail order, reasons and Deps."""
    for st in golden("propstores")[key]:
        p = Y.Propagator(Y.NogoodStore.build(st["nogoods"], 10), 1, engine)
        o = p.initial_propagation()
        assert o.violated == bool(st["init_violated"])
        assert sorted(o.conflicts) == sorted(st["init_conflicts"]) and o.propagations == st["init_props"]
        if not o.violated:
            o = p.propagate_and_check(1)
            assert (o.violated, o.propagations, o.passes) == (bool(st["l1_violated"]), st["l1_props"], st["l1_passes"])
            assert sorted(o.conflicts) == sorted(st["l1_conflicts"])
            if not o.violated and st["decision"]:
                p.push_decision(st["decision"])
                p.seed([st["decision"]])
                o = p.propagate_and_check(2)
                assert (o.violated, o.propagations, o.passes) == (bool(st["l2_violated"]), st["l2_props"],
                                                                  st["l2_passes"])
                assert sorted(o.conflicts) == sorted(st["l2_conflicts"])
        assert p.cells() == st["cells"] and p.trail() == st["trail"] and p.reasons() == st["reasons"]
        d, ov = p.deps(0)
        assert [x | (1 << 63 if v else 0) for x, v in zip(d, ov)] == st["deps"]


@pytest.mark.parametrize("engine", ENGINES)
def test_planted_fixpoint_matches_reference(engine):
    """200k-nogood planted stores (App. C recipe) at 1/10/50/90 % seeds: identical
    propagation count, pass count, trail (FNV digest of the literal sequence) and the
    reasons and Deps of the trail atoms (digests in trail order)."""
    for exp in golden("planted"):
        s, seeded, dec = Y.NogoodStore.planted(exp["atoms"], exp["nogoods"], exp["pct"])
        p = Y.Propagator(s, 16, engine)
        p.push_decision(dec)
        p.assign_propagated(seeded, 2)
        p.seed([dec] + seeded)
        o = p.propagate_and_check(2)
        tr = p.trail()
        assert not o.violated
        assert (o.propagations, o.passes, len(tr)) == (exp["propagations"], exp["passes"], exp["trail"])
        assert fnv(tr) == exp["trail_digest"]
        assert trail_digests(p) == (exp["trail"], exp["trail_digest"], exp["reason_digest"], exp["deps_digest"])


def test_planted_1m_properties():
    """Full-size config 4b (1M nogoods, 100k atoms, 50 % seed): size-independent
    properties — H satisfies every nogood, so no conflict may appear, every
    propagated literal agrees with the planted assignment, and the fixpoint is
    closed (re-propagating the whole trail derives nothing new)."""
    s, seeded, dec = Y.NogoodStore.planted(100_000, 1_000_000, 50)
    p = Y.Propagator(s, 16, "grid")
    p.push_decision(dec)
    p.assign_propagated(seeded, 2)
    p.seed([dec] + seeded)
    o = p.propagate_and_check(2)
    assert not o.violated and o.checks > 500_000
    tr = p.trail()
    H = {abs(l): l for l in [dec] + seeded}
    cells = p.cells()
    # every assignment is consistent with H where H is known
    for lit in tr:
        if abs(lit) in H:
            assert H[abs(lit)] == lit
    before = len(tr)
    p.seed(tr)
    o2 = p.propagate_and_check(2)
    assert not o2.violated and o2.propagations == 0 and len(p.trail()) == before


@pytest.mark.parametrize("engine", ENGINES)
def test_assign_keeps_first_occurrence_and_leaves_assigned_atoms(engine):
    """assign_propagated (assignment.cpp:135-144) on a batch: a repeated atom and an
    atom that is already assigned do not change the assignment or the trail."""
    import numpy as np
    p = Y.Propagator(Y.NogoodStore.build([[1, 2], [3, 4]], 5), 1, engine)
    p.push_decision(1)
    p.assign_propagated(np.array([3, -3, 5, 3, -1], dtype=np.int32), 2)
    assert p.trail() == [1, 3, 5]
    assert p.cells()[1:] == [2, 0, 2, 0, 2]
    p.assign_propagated([4, 5], 2)  # 5 agreed, 4 new
    assert p.trail() == [1, 3, 5, 4]


@pytest.mark.parametrize("engine", ENGINES)
def test_reset_clears_whole_deps_rows(engine):
    """After reset every Deps row is empty again (a fresh Assignment), also for rows that
    were written with more words than their atom's level needs: Deps passed to
    assign_propagated, and propagation at a level below the current decision level."""
    def run(p, wide):
        if wide:
            for a in range(50, 120):  # decision levels 2..71: Deps words 0 and 1
                p.push_decision(a)
            p.assign_propagated([1], 2, deps=[0, 1 << 5])
            p.seed([1])
            p.propagate_and_check(2)  # atom 2 at level 2, Deps from atom 1 (word 1)
            assert p.deps(1)[0][2] == 1 << 5
            p.reset()
        p.push_decision(1)
        p.seed([1])
        o = p.propagate_and_check(2)
        return o.propagations, p.trail(), [p.deps(w)[0] for w in range(2)]

    store = Y.NogoodStore.build([[1, -2]], 200)
    fresh = run(Y.Propagator(store, 2, engine), False)
    assert fresh[1] == [1, 2] and fresh[2][0][2] == 2 and fresh[2][1][2] == 0  # decision bit cdl-1 = 1
    assert run(Y.Propagator(store, 2, engine), True) == fresh


@pytest.mark.parametrize("engine", ENGINES)
def test_batched_calls_match_flushed_calls(engine):
    """Recorded calls launched as one batch (bulk inputs uploaded early, staging buffers growing
    mid-batch) give the same fixpoint as the same calls launched one by one."""
    import numpy as np
    store, seeded, dec = Y.NogoodStore.planted(20_000, 200_000, 50)
    sd = np.asarray(seeded, dtype=np.int32)
    out = []
    for flush_each in (True, False):
        p = Y.Propagator(store, 16, engine)
        for rep in range(2):
            p.reset()
            p.push_decision(dec)
            p.assign_propagated(sd[:64], 2)  # small, then a bulk input larger than the staging so far
            if flush_each:
                p.flush()
            p.assign_propagated(sd[64:], 2)
            if flush_each:
                p.flush()
            p.seed(np.concatenate([[dec], sd]).astype(np.int32))
            if flush_each:
                p.flush()
            o = p.propagate_and_check(2)
            out.append((o.violated, o.propagations, o.passes, fnv(p.trail())))
    assert out[0] == out[1] == out[2] == out[3]


def test_grid_pass_trace_diagnostics():
    """The per-pass phase stamps of whole-grid propagation are readable and ordered."""
    store, seeded, dec = Y.NogoodStore.planted(20_000, 200_000, 50)
    p = Y.Propagator(store, 16, "grid")
    p.pass_trace(True)
    p.push_decision(dec)
    p.assign_propagated(seeded, 2)
    p.seed([dec] + seeded)
    o = p.propagate_and_check(2)
    tr = p.pass_trace()
    assert tr.shape[0] == 64 and tr.shape[2] == 10 and not o.violated
    first = tr[0, 0]
    assert first[0] > 0 and all(first[k] <= first[k + 1] for k in range(0, 8))
    assert (int(first[9]) & 0xFFFFFFFF) == 1 + len(seeded)  # F of pass 0


# ---- argument checking on the low-level API ------------------------
@pytest.mark.parametrize("engine", ENGINES)
def test_add_learned_canonicalises_and_rejects_bad_sets(engine):
    p = Y.Propagator(Y.NogoodStore.build([[1, 2]], 4), 1, engine)
    # repeats are dropped and the order does not matter (Nogood::make)
    assert p.add_learned([3, 4, 3]) == 1
    assert p.add_learned([4, 3]) == 2  # an equal set is appended again (duplicate census only)
    for bad in ([], [0], [5], [-9, 1], [2, -2]):
        with pytest.raises(ValueError):
            p.add_learned(bad)
    p.push_decision(-4)
    p.seed([-4])
    o = p.propagate_and_check(2)  # the session stays usable after rejected calls
    assert not o.violated


@pytest.mark.parametrize("engine", ENGINES)
def test_seed_out_of_range_and_over_capacity(engine):
    p = Y.Propagator(Y.NogoodStore.build([[1, 2]], 2), 1, engine)
    with pytest.raises(ValueError):
        p.seed([3])
    with pytest.raises(ValueError):
        p.seed([0])
    p.seed([1, 2, 1])          # A + 1 = 3 frontier literals: accepted
    p.seed([2])                # the fourth exceeds the frontier capacity: reported by the next result
    with pytest.raises(ValueError):
        p.propagate_and_check(1)
    p.reset()
    p.push_decision(1)
    p.seed([1])
    o = p.propagate_and_check(2)
    assert not o.violated and p.cells()[2] == -2


def test_unbounded_learned_capacity_solves():
    prog = Y.parse_program("a :- not b.\nb :- not a.\n:- a.\n")
    r = Y.solve(prog, Y.SolverConfig(max_models=0, learned_capacity=2**64 - 1))
    assert [m.atom_ids for m in r.models] == [[2]]
