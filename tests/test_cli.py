"""The command-line front end (proj/tools/condmpc_cli.cpp): the problem
file container round-trips bit-exactly (problem_io.cpp), validation matches problem.cpp:100-158,
invalid input exits 4 before any device work. CPU only."""
import io
import math

import numpy as np
import pytest

from paper_2209_13049_b200 import cli, problem as P


def _eq(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


def test_heat_problem_file_round_trips_bit_exactly():
    data = P.build_heat_problem(P.HeatParams(N=3, T=7))
    buf = io.StringIO()
    cli.write_problem(buf, data)
    text = buf.getvalue()
    assert text.startswith("condmpc-problem v1\nT 7\nA 27 27\n")
    back = cli.read_problem(text)
    for f in ("A", "B", "Q", "Qf", "R", "S", "E", "F", "K"):
        assert _eq(getattr(back, f), getattr(data, f)), f
    for f in ("gl", "gu", "xl", "xu", "ul", "uu", "x_bar"):
        assert _eq(getattr(back, f), np.asarray(getattr(data, f), dtype=float).ravel()), f
    assert _eq(back.w, np.asarray(data.w).reshape(7, -1)) and back.T == 7


def test_infinite_bounds_and_awkward_doubles():
    rng = np.random.default_rng(1)
    data = P.LqProblemData.basic(A=rng.uniform(-1, 1, (3, 3)), B=[[1e-300], [1.0 / 3.0], [-0.0]],
                                 Q=np.eye(3), R=[[0.1]], Qf=np.eye(3), x_bar=[0.1, 2e22, -7.5], T=4)
    data.xl[1] = -5.0
    buf = io.StringIO()
    cli.write_problem(buf, data)
    back = cli.read_problem(buf.getvalue())
    assert _eq(back.B, data.B) and _eq(back.x_bar, data.x_bar)
    assert math.isinf(back.xu[0]) and back.xl[1] == -5.0 and math.isinf(back.ul[0])


@pytest.mark.parametrize("text,msg", [
    ("nope\n", "missing header"),
    ("condmpc-problem v1\nA 1 1 2\n", "missing entry 'T'"),
    ("condmpc-problem v1\nT 2\nA 1 1 x\n", "expected number"),
    ("condmpc-problem v1\nT 2\nA 1 1 1\nA 1 1 1\n", "duplicate entry"),
    ("condmpc-problem v1\nT -2\n", "nonnegative integer"),
])
def test_parse_errors(text, msg):
    with pytest.raises(cli.ParseError, match=msg):
        cli.read_problem(text)


def test_validation_rules():
    data = P.build_heat_problem(P.HeatParams(N=2, T=3))
    assert cli.validate_problem(data) == []
    bad = data.copy()
    bad.Q[0, 1] += 1.0
    assert any(i.field == "Q" for i in cli.validate_problem(bad))
    bad = data.copy()
    bad.xl[0], bad.xu[0] = 5.0, 1.0
    assert any(i.field == "xl/xu" for i in cli.validate_problem(bad))
    bad = data.copy()
    bad.x_bar[0] = -1e9
    assert any(i.field == "x_bar" for i in cli.validate_problem(bad))
    bad = data.copy()
    bad.A = np.zeros((2, 2))
    assert cli.validate_problem(bad)[0].field == "dims"


def test_invalid_input_exits_4(tmp_path):
    p = tmp_path / "bad.txt"
    p.write_text("not a problem\n")
    assert cli.main(["solve", str(p)]) == 4
    assert cli.main(["solve", str(tmp_path / "missing.txt")]) == 4
    data = P.build_heat_problem(P.HeatParams(N=2, T=3))
    data.R = -np.eye(6)
    q = tmp_path / "neg.txt"
    with open(q, "w") as f:
        cli.write_problem(f, data)
    assert cli.main(["solve", str(q)]) == 4          # stage cost not PSD
    assert cli.main(["solve", str(q), "--backend", "eigen"]) == 4
    assert cli.main(["frobnicate"]) == 4


def test_gen_writes_a_readable_file(tmp_path):
    out = tmp_path / "heat.txt"
    assert cli.main(["gen", "--N", "2", "--T", "5", "--dump", str(out)]) == 0
    back = cli.read_problem(out.read_text())
    assert back.T == 5 and back.A.shape == (8, 8) and cli.validate_problem(back) == []
