"""The command-line front end on the device: `solve` (device-built QP) gives the library's
result and the reference's exit code / CSV schema; `bench` prints the 11-column CSV."""
import numpy as np
import pytest

from paper_2209_13049_b200 import cli, ipm, problem as P

pytestmark = pytest.mark.gpu


def test_cli_solve_matches_the_library(tmp_path, capsys):
    data = P.build_heat_problem(P.HeatParams(N=3, T=10))
    f = tmp_path / "heat.txt"
    with open(f, "w") as fh:
        cli.write_problem(fh, data)
    rc = cli.main(["solve", str(f), "--csv", "--log-iters"])
    out = capsys.readouterr().out
    ref = ipm.solve(P.build_dense_qp(data))
    assert rc == 0 and f"iterations  {ref.iter}" in out
    lines = out.splitlines()
    assert cli.CSV_HEADER in lines
    rec = lines[lines.index(cli.CSV_HEADER) + 1].split(",")
    assert len(rec) == 11 and rec[-1] == "converged" and int(rec[5]) == ref.iter
    assert abs(float(rec[8]) - ref.objective) <= 1e-8 * (1 + abs(ref.objective))
    # max_iter exit code
    assert cli.main(["solve", str(f), "--max-iter", "2"]) == 2


def test_cli_bench_grid(capsys):
    assert cli.main(["bench", "--N", "2", "--T", "5,10"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == cli.CSV_HEADER
    rows = [l.split(",") for l in out[1:3]]
    assert all(len(r) == 11 and r[-1] == "converged" for r in rows)
    assert any(l.startswith("# slope log total_s / log T at N=2") for l in out)
