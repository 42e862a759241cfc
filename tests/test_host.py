"""Host side of the drop-in boundary (CPU only): parser, completion compiler and
store builder must produce exactly the reference's atom ids, nogood ids, CSR
layout, guards and unit lists."""
import pytest

import paper_1909_01786_b200 as Y
from paper_1909_01786_b200 import aspine as A
from workloads import instances as I

from _util import golden


# ---- parser: P/tests/test_program.cpp ----------------------------------------
def test_parses_facts_rules_constraints():
    p = Y.parse_program("a.\nb :- a, not c.\n:- b, c.")
    assert p.atom_count() == 3 and p.rule_count() == 2 and p.constraint_count() == 1
    (h0, p0, n0), (h1, p1, n1) = p.rules()
    assert (h0, p0, n0) == (1, [], [])
    assert h1 == p.find("b") and p1 == [p.find("a")] and n1 == [p.find("c")]
    assert p.constraints()[0][1] == [p.find("b"), p.find("c")]


def test_interning_order_and_duplicates():
    p = Y.parse_program("x :- y, not z.\ny.\n")
    assert (p.find("x"), p.find("y"), p.find("z")) == (1, 2, 3)
    q = Y.parse_program("a :- b, b, not c, not c.")
    assert q.rules()[0][1:] == ([2], [3])
    s = Y.parse_program("a :- not a.")
    assert s.rules() == [(1, [], [1])]


def test_comments_blank_lines_and_parenthesised_names():
    p = Y.parse_program("% a comment line\n\nat(1,2) :- step(1), not wall(1,2).  % trailing comment\n")
    assert p.atom_count() == 3 and p.find("at(1,2)") == 1 and p.find("wall(1,2)") == 3


@pytest.mark.parametrize("text,line", [
    ("a.\nb :- \nc.", 2), ("a.\nb :- ,c.\n", 2), ("a. b.", 1), ("a :- not .", 1), ("a :- b", 1),
    ("p(1 :- q.", 1), ("x(a b).", 1), (":- .", 1), ("ok.\n\n% c\nbad :- x,", 4)])
def test_syntax_errors_carry_line_numbers(text, line):
    with pytest.raises(Y.ParseError) as e:
        Y.parse_program(text)
    assert e.value.line == line
    assert str(e.value).startswith(f"line {line}: ")


def test_tp_step_and_validate():
    p = Y.parse_program("a.\nb :- a.")
    assert Y.tp_step(p, []) == [1] and Y.tp_step(p, [1]) == [1, 2]
    q = Y.parse_program("a :- not b.\nb :- not a.")
    assert Y.tp_step(q, [1]) == [1]
    assert Y.validate(Y.parse_program("b :- a.")) == ["atom a has no rules"]
    assert "rule 1 body is inconsistent" in Y.validate(Y.parse_program("a :- b, not b."))
    assert Y.validate(Y.parse_program("a.")) == []
    assert Y.validate(Y.parse_program("")) == ["empty program"]


def test_print_matches_reference_and_round_trips():
    """print_program(parse_program(text)) equals the reference's output; a second
    round trip is a fixpoint (test_program.cpp print/parse round-trip)."""
    for d in golden("dumps"):
        p = Y.parse_program(d["text"])
        printed = Y.print_program(p)
        assert printed == d["printed"], d["name"]
        assert Y.print_program(Y.parse_program(printed)) == printed


# ---- completion + store goldens: test_completion.cpp:19-37, test_store.cpp:62 --
def test_completion_golden_dump():
    p = Y.parse_program("a :- b, not c.")
    assert p.rule_aux(0) == {"b": 4, "t": 5, "n": 6, "vacuous": False}
    assert p.total_atoms() == 6
    assert Y.dump_nogoods(p) == (
        "{F b_r(1), T t_r(1), T n_r(1)} completion\n{T b_r(1), F t_r(1)} completion\n"
        "{T b_r(1), F n_r(1)} completion\n{F b, T t_r(1)} completion\n{T b, F t_r(1)} completion\n"
        "{T c, T n_r(1)} completion\n{F c, F n_r(1)} completion\n{F a, T b_r(1)} completion\n"
        "{T a, F b_r(1)} completion\n{T b} completion\n{T c} completion\n")
    assert p.census() == ((7, 4, 0), (7, 4, 0))


def test_store_golden_csv():
    s = Y.NogoodStore.build([[1, 2, 3], [-4], [1, -2], [-3, 5]], 5)
    assert s.dump_csv() == "offsets,0,2,4,7\npool,1,-2,-3,5,1,2,3\n"
    assert s.static_units() == [-4] and s.static_class_bounds() == [0, 2, 3, 3]
    e = Y.NogoodStore.build([], 3)
    assert e.dump_csv() == "offsets,0\npool\n" and e.size() == 0


def test_vacuous_nogood_rejected():
    with pytest.raises(ValueError):
        Y.NogoodStore.build([[1, -1]], 2)


def test_dumps_match_reference_for_corpus_and_instances():
    """Every program: aux ids, census, dump_nogoods text and the CSR store."""
    for d in golden("dumps"):
        p = Y.parse_program(d["text"])
        assert p.atom_count() == d["atoms"] and p.total_atoms() == d["total_atoms"], d["name"]
        assert [list(p.rule_aux(r).values()) for r in range(p.rule_count())] == [
            [b, t, n, bool(v)] for b, t, n, v in d["aux"]], d["name"]
        census, counts = p.census()
        assert list(census) == d["census"] and list(counts) == d["counts"], d["name"]
        assert Y.dump_nogoods(p) == d["dump"], d["name"]
        assert Y.store_csv(p) == d["csv"], d["name"]


def test_store_units_guards_and_occurrences():
    """Static units, unit ids, class bounds and occurrence lists vs the reference build."""
    for d in golden("dumps")[::7]:
        p = Y.parse_program(d["text"])
        # rebuild the store through the low-level API from the compiled nogoods
        csv = d["csv"].splitlines()
        offs = [int(x) for x in csv[0].split(",")[1:]]
        pool = [int(x) for x in csv[1].split(",")[1:]] if "," in csv[1] else []
        ngs = [pool[offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
        s = Y.NogoodStore.build(ngs, d["total_atoms"], guards=d["store_guards"])
        assert s.dump_csv() == d["csv"]
        assert s.static_class_bounds()[:3] == d["bounds"][:3]
        ids = set()
        for a in range(1, d["total_atoms"] + 1):
            for lit in (a, -a):
                for c in range(4):
                    occ = s.occurrences(lit, c)
                    assert occ == sorted(occ)
                    for i in occ:
                        assert lit in ngs[i] and min(len(ngs[i]), 4) - 1 == c
                        ids.add((lit, i))
        assert len(ids) == len(pool)


def test_planted_store_matches_reference_generator():
    for exp in golden("planted"):
        s, seeded, dec = Y.NogoodStore.planted(exp["atoms"], exp["nogoods"], exp["pct"])
        assert s.size() + len(s.static_units()) == exp["nogoods"] and len(seeded) == exp["seeded"]
        assert abs(dec) == 1


def test_ladder_cubes_partition_and_encoding():
    p = Y.parse_program(I.queens(6))
    one = A.cubes(p, 6, 1)
    assert len(one) == 7
    names = [[p.name(x) for x in c if x] for c in one]
    # cube i: F q(1,1..i-1) as ":- q(1,j).", T q(1,i) as ":- nq(1,i)."; last cube: all F
    assert names[0] == ["nq(1,1)"] and names[2] == ["q(1,1)", "q(1,2)", "nq(1,3)"]
    assert names[6] == [f"q(1,{j})" for j in range(1, 7)]
    two = A.cubes(p, 6, 2)
    assert len(two) == 49 and len({tuple(c) for c in two}) == 49
    parts = [A.cubes(p, 6, 2, r, 3) for r in range(3)]
    assert sorted(tuple(c) for part in parts for c in part) == sorted(tuple(c) for c in two)
    assert len(A.cubes(p, 6, 0, want=300)) == 343


def test_cubes_without_choice_pairs_use_rule_heads():
    """Programs without even-loop pairs still shard: atoms that head a rule split as
    ":- a." (+a, asserts F a) and ":- not a." (-a, a passive unit nogood {F a})."""
    p = Y.parse_program("p :- q.\nq :- not r.\nr :- s.\n")
    assert [p.name(a) for a in (1, 2, 3, 4)] == ["p", "q", "r", "s"]
    assert A.cubes(p, 2, 1) == [[-1, 0], [1, -2], [1, 2]]
    assert len(A.cubes(p, 1, 0, want=8)) == 8  # p, q, r: three levels of width 1
    # pairs come first, then the remaining rule heads
    q = Y.parse_program("a :- not b.\nb :- not a.\nc :- a.\n")
    assert A.cubes(q, 2, 1) == [[2, 0], [1, -3], [1, 3]]


def test_automatic_cubes_follow_at_least_one_groups():
    """k = 0: ladders over "at least one of" constraint groups (a queens row, a node's
    colours): each level asks which member of a group is the first true one."""
    q = Y.parse_program(I.queens(8))
    auto = A.cubes(q, 0, 1)
    assert len(auto) == 9 and auto == A.cubes(q, 8, 1)  # rows are already first, in atom order
    col = Y.parse_program(I.colouring(30, 4.0, 3, 7))
    c = A.cubes(col, 0, 2)
    assert len(c) == 16 and len(c[0]) == 6  # three colours per node, two nodes deep
    names = [[col.name(abs(x)) for x in cube if x] for cube in c]
    assert {n.split("(")[1].split(",")[0] for cube in names for n in cube} == {"1", "2"}  # nodes 1 and 2


# ---- invalid ids raise instead of aborting the host process --------
def test_tp_step_and_verify_reject_out_of_range_ids():
    p = Y.parse_program("a :- not b.\nb :- not a.\n")
    with pytest.raises(ValueError):
        Y.tp_step(p, [7])
    with pytest.raises(ValueError):
        Y.tp_step(p, [0])
    with pytest.raises(ValueError):
        Y.verify_model(p, Y.Model([1, 9], []))
    assert Y.tp_step(p, []) == [1, 2]
    assert Y.verify_model(p, Y.Model([1], ["a"]))


def _first_occurrence_names(text):
    """Atom names in first-occurrence order (head, then body left to right), by a
    plain Python scan of the canonical format (program.cpp:141-174 semantics)."""
    import re
    atom = re.compile(r"[A-Za-z_][A-Za-z0-9_]*(?:\([A-Za-z0-9_,()]*\)[A-Za-z0-9_]*)*")
    seen, order = set(), []
    for line in text.split("\n"):
        line = line.split("%", 1)[0]
        for m in atom.finditer(line):
            name = m.group(0)
            if name == "not" and line[m.end():m.end() + 1] == " ":
                continue
            if name not in seen:
                seen.add(name)
                order.append(name)
    return order


def test_parallel_parse_keeps_first_occurrence_ids():
    """Large programs are tokenized and interned by every host thread; ids must
    still follow first occurrence exactly, and the program must print back to
    the same statements."""
    for text in (I.random_program(), I.queens(12), I.hamiltonian(200, 1.0, 1)):
        p = Y.parse_program(text)
        names = _first_occurrence_names(text)
        assert p.atom_count() == len(names)
        assert [p.name(i) for i in range(1, p.atom_count() + 1)] == names
        q = Y.parse_program(Y.print_program(p))
        assert Y.print_program(q) == Y.print_program(p)
    with pytest.raises(Y.ParseError) as e:
        Y.parse_program(I.random_program() + "a :- b c.\n" + "d :- e\n")
    assert e.value.line == I.random_program().count("\n") + 1
