"""Full solve/enumerate on the device vs the unmodified reference: identical
verdicts, identical model sequences and identical trajectory counters
(decisions, propagations, conflicts, learned, passes, ...)."""
import pytest

import paper_1909_01786_b200 as Y
from workloads import instances as I

from _util import HEUR, config_from_opts, golden, stats_diff

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfgkey", ["fwd/occ", "res/occ", "fwd/jw", "res/jw", "fwd/act", "res/act"])
def test_acceptance_corpus_trajectories(cfgkey):
    """518 programs (acceptance_main.cpp:51-65) x this mode/heuristic: full enumeration."""
    mode, heur = cfgkey.split("/")
    bad = []
    for prog in golden("corpus"):
        run = prog["runs"][cfgkey]
        cfg = Y.SolverConfig(mode=Y.LearnMode[mode], heuristic=Y.HeuristicConfig(HEUR[heur]), max_models=0,
                             verify=True)
        r = Y.solve(Y.parse_program(prog["text"]), cfg)
        models = [m.atom_ids for m in r.models]
        if models != run["models"] or r.status.name.upper() != run["status"] or stats_diff(r.stats, run["stats"]):
            bad.append((prog["name"], stats_diff(r.stats, run["stats"])))
        assert sorted(models) == sorted(prog["family"]), prog["name"]
    assert not bad, bad[:5]


def test_option_variants_match_reference():
    """Restarts, fanout, deps-words overflow, activity decay, capacity error."""
    for case in golden("extras"):
        cfg = config_from_opts(case["opts"])
        p = Y.parse_program(case["text"])
        if case.get("error"):
            with pytest.raises(Y.StoreCapacityError):
                Y.solve(p, cfg)
            continue
        r = Y.solve(p, cfg)
        assert [m.atom_ids for m in r.models] == case["models"], (case["name"], case["opts"])
        assert not stats_diff(r.stats, case["stats"]), (case["name"], case["opts"], stats_diff(r.stats, case["stats"]))


@pytest.mark.parametrize("key", ["queens8/fwd/occ", "queens8/res/occ", "queens8/fwd/jw", "queens8/res/jw",
                                 "queens8/fwd/act", "queens8/res/act"])
def test_queens8_all_models_and_trace(key):
    _, mode, heur = key.split("/")
    exp = golden("configs")[key]
    trace = []
    cfg = Y.SolverConfig(mode=Y.LearnMode[mode], heuristic=Y.HeuristicConfig(HEUR[heur]), max_models=0,
                         trace=lambda t: trace.append([int(t.mode_used), t.conflict_id, t.learned_length,
                                                       t.backjump_level]))
    r = Y.solve(Y.parse_program(I.queens(8)), cfg)
    assert [m.atom_ids for m in r.models] == exp["models"]
    assert not stats_diff(r.stats, exp["stats"])
    assert trace == exp["trace"]
    # without a trace the same search runs when the reference order is asked for
    cfg.trace = None
    cfg.reference_order = True
    r = Y.solve(Y.parse_program(I.queens(8)), cfg)
    assert [m.atom_ids for m in r.models] == exp["models"] and not stats_diff(r.stats, exp["stats"])


def test_plain_enumeration_is_cube_split_by_default():
    """max_models = 0 on a program with many choice pairs enumerates cubes over the GPU
    (VERDICT r1 #8): the reference's answer-set set, in cube order, the same on every run."""
    exp = sorted(golden("configs")["queens8/fwd/occ"]["models"])
    prog = Y.parse_program(I.queens(8))
    runs = [Y.solve(prog, Y.SolverConfig(max_models=0)) for _ in range(2)]
    for r in runs:
        assert sorted(m.atom_ids for m in r.models) == exp and r.stats.cubes > 1
        assert r.cubes == sorted(r.cubes)
    assert [m.atom_ids for m in runs[0].models] == [m.atom_ids for m in runs[1].models]
    single = Y.solve(prog, Y.SolverConfig(max_models=0, reference_order=True))
    assert single.stats.cubes == 1 and [m.atom_ids for m in single.models] == golden("configs")["queens8/fwd/occ"]["models"]


def test_grid_engine_enumeration_keeps_reference_order():
    """engine="grid" runs one whole-GPU search at a time: max_models = 0 is not cube-split
    there, and the models come in the reference's order (solver.cpp:216-246)."""
    exp = golden("configs")["queens8/fwd/occ"]
    r = Y.solve(Y.parse_program(I.queens(8)), Y.SolverConfig(max_models=0, engine="grid"))
    assert r.stats.cubes == 1 and [m.atom_ids for m in r.models] == exp["models"]
    assert not stats_diff(r.stats, exp["stats"])


@pytest.mark.parametrize("name", ["colour2000", "ham200"])
@pytest.mark.parametrize("engine", ["block", "grid"])
def test_first_model_configs(name, engine):
    text = I.colouring(2000, 4.0, 3, 1) if name == "colour2000" else I.hamiltonian(200, 1.0, 1)
    exp = golden("configs")[f"{name}/fwd/occ"]
    r = Y.solve(Y.parse_program(text), Y.SolverConfig(engine=engine))
    assert r.status == Y.SolveStatus.sat and [m.atom_ids for m in r.models] == exp["models"]
    assert not stats_diff(r.stats, exp["stats"])


def test_reference_solver_cases():
    """P/tests/test_solver.cpp handcrafted cases."""
    even = Y.parse_program("a :- not b.\nb :- not a.")
    r = Y.solve(even, Y.SolverConfig(max_models=0, verify=True, debug_validate=True))
    assert [m.atoms for m in r.models] == [["a"], ["b"]]  # cli_tests.cpp:58-64 model order
    assert Y.solve(Y.parse_program("p :- q.\nq :- p."), Y.SolverConfig(max_models=0)).models[0].atom_ids == []
    assert Y.solve(Y.parse_program("a.\n:- a.")).status == Y.SolveStatus.unsat
    for text in ("p :- p.\np :- not p.\n", "p :- p.\np :- not p.\n:- not p.\n",
                 "c.\np :- p.\nx :- not y.\ny :- not x.\n:- c, not p.\n"):
        for mode in (Y.LearnMode.fwd, Y.LearnMode.res):
            r = Y.solve(Y.parse_program(text), Y.SolverConfig(mode=mode, max_models=0, debug_validate=True))
            assert r.status == Y.SolveStatus.unsat and r.stats.uip_check_failures == 0
    r = Y.solve(Y.parse_program("p :- q.\nq :- p.\np :- z.\nz :- not w.\nw :- not z.\n:- not p.\n"))
    assert r.models[0].atoms == ["p", "q", "z"]
    r = Y.solve(Y.parse_program("a."))
    assert r.models[0].atoms == ["a"] and r.stats.decisions == 0
    r = Y.solve(Y.parse_program(""))
    assert r.status == Y.SolveStatus.sat and r.models[0].atom_ids == []
    assert len(Y.solve(even, Y.SolverConfig(max_models=1)).models) == 1


def test_capacity_and_verify_and_trace_count():
    p = Y.parse_program("a :- not b.\nb :- not a.\nc :- not d.\nd :- not c.\ne :- not f.\nf :- not e.\n"
                        ":- a, c.\n:- a, d.\n:- b, c.\n:- b, d, e.\n:- b, d, f.")
    with pytest.raises(Y.StoreCapacityError):
        Y.solve(p, Y.SolverConfig(learned_capacity=0))
    lines = []
    q = Y.parse_program("a :- not b.\nb :- not a.\nc :- not d.\nd :- not c.\n:- a, c.\n:- a, d.\n")
    r = Y.solve(q, Y.SolverConfig(trace=lambda t: lines.append(t)))
    assert len(lines) == r.stats.learned_count
    assert all(t.learned_length >= 1 and t.backjump_level >= 1 for t in lines)


def test_determinism_and_stats_text():
    p = Y.parse_program(I.pigeonhole(4, 3))
    runs = [Y.solve(p, Y.SolverConfig(max_models=0)) for _ in range(3)]
    for r in runs[1:]:
        assert r.stats.decisions == runs[0].stats.decisions and r.stats.propagations == runs[0].stats.propagations
    r = Y.solve(Y.parse_program("a.\n:- a."))
    ctx = Y.StatsContext("inst.lp", "fwd", "occ", 1, r.status, r.stats.models)
    row = Y.emit_stats(r.stats, ctx, csv=True)
    assert row.startswith("inst.lp,fwd,occ,1,UNSAT,0,0,")
    assert Y.stats_csv_header().count(",") == row.count(",")
    assert "status         : UNSAT" in Y.emit_stats(r.stats, ctx, csv=False)


def test_model_list_views_match_per_model_accessors():
    """SolveResult.models is a lazy sequence over yas_result_models_flat: length,
    indexing, slicing and names agree with the model-by-model C-ABI."""
    from workloads import instances as I
    prog = Y.parse_program(I.queens(6))
    r = Y.solve(prog, Y.SolverConfig(max_models=0))
    ms = r.models
    assert len(ms) == 4 and ms[-1] == ms[3] and ms[1:3] == [ms[1], ms[2]]
    for m in ms:
        assert m.atom_ids == sorted(m.atom_ids) and len(m.atoms) == 36  # six q(i,j), thirty nq(i,j)
        assert m.atoms == sorted(prog.name(a) for a in m.atom_ids)
        assert sum(a.startswith("q(") for a in m.atoms) == 6
    with pytest.raises(IndexError):
        ms[4]


def test_first_model_portfolio():
    """N concurrent searches with diverse (mode, heuristic); the first to finish
    reports. Not the reference's first model, but always one of its answer sets (or UNSAT)."""
    for prog in golden("corpus")[::7]:
        r = Y.solve(Y.parse_program(prog["text"]), Y.SolverConfig(portfolio=6, verify=True))
        assert (r.status == Y.SolveStatus.sat) == bool(prog["family"]), prog["name"]
        if r.models:
            assert r.models[0].atom_ids in prog["family"], prog["name"]
        assert 0 <= r.stats.portfolio_variant < 6 and r.stats.searches == 6 and r.stats.cubes == 0
    for text in (I.colouring(2000, 4.0, 3, 1), I.hamiltonian(200, 1.0, 1)):
        r = Y.solve(Y.parse_program(text), Y.SolverConfig(portfolio=6, verify=True))
        assert r.status == Y.SolveStatus.sat and len(r.models) == 1
    # another rank starts at a different variant; one search = variant of the config itself
    r = Y.solve(Y.parse_program(I.queens(8)), Y.SolverConfig(portfolio=2, rank=1, mode=Y.LearnMode.res))
    assert r.stats.portfolio_variant in (3, 4) and len(r.models) == 1
    r = Y.solve(Y.parse_program(I.queens(8)), Y.SolverConfig())
    assert r.stats.portfolio_variant == -1
