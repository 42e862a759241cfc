"""`aspine` CLI drop-in, mirroring /root/reference/proj/tests/cli_tests.cpp:58-106."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1909_01786_b200", "_lib", "aspine")
EVEN = "a :- not b.\nb :- not a.\n"


def run(args, stdin=None, tmp=None):
    p = subprocess.run([BIN] + args, input=stdin, capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout


@pytest.fixture()
def files(tmp_path):
    (tmp_path / "even.lp").write_text(EVEN)
    (tmp_path / "unsat.lp").write_text("a.\n:- a.\n")
    (tmp_path / "bad.lp").write_text("a :- \n")
    return tmp_path


def test_usage_parse_and_io_errors(files):
    assert run(["solve", "--no-such-flag", "x"])[0] == 2
    assert run(["solve", "--devices", "0,x", str(files / "even.lp")])[0] == 2
    assert run(["solve", str(files / "bad.lp")])[0] == 2
    assert run(["solve", str(files / "missing.lp")])[0] == 1
    assert run([])[0] == 2


def test_oracle_subcommand(files):
    rc, out = run(["oracle", str(files / "even.lp")])
    assert rc == 10 and "Answer: 1\na\n" in out and "Answer: 2\nb\n" in out and out.endswith("SATISFIABLE\n")
    assert run(["oracle", str(files / "unsat.lp")])[0] == 20


@pytest.mark.gpu
def test_solve_exit_codes_and_output(files):
    rc, out = run(["solve", str(files / "even.lp"), "-n", "0", "--verify"])
    assert rc == 10 and "Answer: 1\na\n" in out and "Answer: 2\nb\n" in out and "SATISFIABLE\n" in out
    rc, out = run(["solve", str(files / "unsat.lp")])
    assert rc == 20 and "UNSATISFIABLE\n" in out
    rc, out = run(["solve", "-", "-n", "1"], stdin=EVEN)
    assert rc == 10 and "Answer: 1\n" in out and "Answer: 2\n" not in out
    rc, out = run(["solve", str(files / "even.lp"), "-n", "0", "--stats", "csv", "--mode", "res", "--heur", "jw"])
    assert rc == 10 and "instance,mode,heuristic,workers,status," in out and ",res,jw,1,SAT,2," in out
    rc, _ = run(["solve", str(files / "even.lp"), "--workers", "4", "--restarts", "geometric:2:2", "-n", "0"])
    assert rc == 10


@pytest.mark.gpu
def test_enumeration_on_two_devices(files, tmp_path):
    """--devices: one cube queue over the listed GPUs (the same B200 twice here)."""
    from workloads import instances as I
    (tmp_path / "q6.lp").write_text(I.queens(6))
    rc, out = run(["solve", str(tmp_path / "q6.lp"), "-n", "0", "--cubes", "6", "--devices", "0,0"])
    assert rc == 10 and out.count("Answer:") == 4


@pytest.mark.gpu
def test_reference_order_flag(tmp_path):
    """--reference-order: a -n 0 enumeration that would be cube-split runs as one search and prints
    the models in the reference's order (the API's reference_order=True run); without the flag the
    same answer sets come in cube order."""
    import paper_1909_01786_b200 as Y
    from workloads import instances as I
    text = I.queens(8)
    (tmp_path / "q8.lp").write_text(text)
    want = [" ".join(m.atoms) for m in Y.solve(Y.parse_program(text), Y.SolverConfig(max_models=0, reference_order=True)).models]

    def answers(out):
        lines = out.splitlines()
        return [lines[i + 1] for i, ln in enumerate(lines) if ln.startswith("Answer:")]

    rc, out = run(["solve", str(tmp_path / "q8.lp"), "-n", "0", "--reference-order"])
    assert rc == 10 and answers(out) == want and len(want) == 92
    rc, out = run(["solve", str(tmp_path / "q8.lp"), "-n", "0"])
    assert rc == 10 and sorted(answers(out)) == sorted(want)
