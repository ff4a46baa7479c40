"""Command-line front end: the reference's `condmpc` tool
(proj/tools/condmpc_cli.cpp) on the B200 path.

    python -m paper_2209_13049_b200.cli solve FILE [--tol --mu-init --max-iter --backend cuda]
                                              [--log-iters] [--csv] [--dump QPFILE]
    python -m paper_2209_13049_b200.cli bench [--N 2,3,4] [--T 10,50] [--reps 1] [--setpoint 350]
    python -m paper_2209_13049_b200.cli gen [--N 4] [--T 50] [--setpoint 350] [--dump FILE]

Same subcommands, flags, outputs and exit codes (0 converged, 2 max_iter, 3 factorization
failure, 4 invalid input, 5 line-search failure; condmpc_cli.cpp:18-32). The problem file is
the reference's `condmpc-problem v1` container (problem_io.cpp:13-190): one entry per field,
`name rows cols` then the values row-major, `inf`/`-inf` for infinite bounds, shortest
round-trip decimal (Python's repr) so finite doubles survive a write/read bit-exactly.
`solve` builds the dense QP on the device (cmpc_build_qp) and recovers nothing on the host;
the CSV keeps the reference's 11 columns (bench.hpp:29-30); GPU timings go to `#` lines.
`verify` (the enumeration-oracle cross-check) is test infrastructure here: tests/.
"""
from __future__ import annotations

import argparse
import math
import statistics
import sys
from dataclasses import dataclass

import numpy as np

from . import problem as P

MAGIC = "condmpc-problem v1"
CSV_HEADER = "name,N,T,n_x,n_u,iter,total_s,linalg_s,objective,kkt_error,status"
EXIT = {"converged": 0, "max_iter": 2, "factorization_failure": 3, "line_search_failure": 5}
INVALID = 4


class ParseError(RuntimeError):
    """problem_io.hpp:11-13."""


# ------------------------------------------------------------------ problem file
def _fmt(v: float) -> str:
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    if v == int(v) and abs(v) < 1e16:
        return repr(int(v)) if not (v == 0 and math.copysign(1, v) < 0) else "-0"
    return repr(float(v))


def _write_matrix(out, name, m):
    m = np.atleast_2d(np.asarray(m, dtype=np.float64))
    if m.ndim == 2 and m.shape[0] == 1 and name in _VECTORS:
        m = m.T
    out.write(f"{name} {m.shape[0]} {m.shape[1]}\n")
    for i in range(m.shape[0]):
        out.write(" ".join(_fmt(x) for x in m[i]) + "\n")


_VECTORS = {"gl", "gu", "xl", "xu", "ul", "uu", "x_bar"}
_MATRICES = ["A", "B", "Q", "Qf", "R", "S", "E", "F"]


def write_problem(out, data: P.LqProblemData):
    """problem_io.cpp:77-106."""
    out.write(MAGIC + "\n")
    out.write(f"T {int(data.T)}\n")
    for f in _MATRICES:
        _write_matrix(out, f, getattr(data, f))
    for f in ("gl", "gu", "xl", "xu", "ul", "uu"):
        _write_matrix(out, f, np.asarray(getattr(data, f), dtype=np.float64).reshape(-1, 1))
    _write_matrix(out, "w", np.asarray(data.w, dtype=np.float64).reshape(int(data.T), -1))
    _write_matrix(out, "x_bar", np.asarray(data.x_bar, dtype=np.float64).reshape(-1, 1))
    _write_matrix(out, "K", data.K)


def read_problem(text: str) -> P.LqProblemData:
    """problem_io.cpp:115-184 (the same errors)."""
    lines = text.split("\n", 1)
    if lines[0].rstrip("\r") != MAGIC:
        raise ParseError(f"problem file: missing header '{MAGIC}'")
    toks = lines[1].split() if len(lines) > 1 else []
    pos = 0

    def nxt(what):
        nonlocal pos
        if pos >= len(toks):
            raise ParseError("problem file: unexpected end of input")
        pos += 1
        return toks[pos - 1]

    def index(what):
        t = nxt(what)
        if not t.isdigit():
            raise ParseError(f"problem file: expected nonnegative integer for {what}, got '{t}'")
        return int(t)

    def number(what):
        t = nxt(what)
        try:
            return float(t)
        except ValueError:
            raise ParseError(f"problem file: expected number for {what}, got '{t}'") from None

    entries, T = {}, None
    while pos < len(toks):
        name = nxt("name")
        if name == "T":
            T = index("T")
            continue
        r, c = index(name + " rows"), index(name + " cols")
        m = np.array([number(name) for _ in range(r * c)], dtype=np.float64).reshape(r, c)
        if name in entries:
            raise ParseError(f"problem file: duplicate entry '{name}'")
        entries[name] = m
    if T is None:
        raise ParseError("problem file: missing entry 'T'")

    def take(name):
        if name not in entries:
            raise ParseError(f"problem file: missing entry '{name}'")
        return entries.pop(name)

    def take_vector(name):
        m = take(name)
        if m.shape[1] > 1:
            raise ParseError(f"problem file: '{name}' must have one column")
        return m[:, 0].copy() if m.shape[1] == 1 else np.zeros(0)

    kw = {f: take(f) for f in _MATRICES}
    kw.update({f: take_vector(f) for f in ("gl", "gu", "xl", "xu", "ul", "uu")})
    kw["w"] = take("w")
    kw["x_bar"] = take_vector("x_bar")
    kw["K"] = take("K")
    if entries:
        raise ParseError(f"problem file: unknown entry '{sorted(entries)[0]}'")
    return P.LqProblemData(T=T, **kw)


def write_dense_qp(out, qp):
    """problem_io.cpp write_dense_qp: the reduced QP in the same container."""
    out.write("condmpc-qp v1\n")
    _write_matrix(out, "H", qp.H)
    _write_matrix(out, "h", np.asarray(qp.h).reshape(-1, 1))
    out.write(f"h0 1 1\n{_fmt(qp.h0)}\n")
    _write_matrix(out, "J", qp.J)
    _write_matrix(out, "d", np.asarray(qp.d).reshape(-1, 1))


# ------------------------------------------------------------------ validation
@dataclass
class Issue:
    field: str
    message: str


def _psd(m):
    """problem.cpp is_positive_semidefinite: sym + 1e-10 I admits a Cholesky factorization."""
    try:
        np.linalg.cholesky(m + 1e-10 * np.eye(m.shape[0]))
        return True
    except np.linalg.LinAlgError:
        return False


def validate_problem(data: P.LqProblemData) -> list:
    """problem.cpp:100-158."""
    try:
        d = P.dims(data)
    except Exception as err:  # DimensionError
        return [Issue("dims", str(err))]
    out = []
    for f in ("A", "B", "Q", "Qf", "R", "S", "E", "F", "K"):
        if np.isnan(getattr(data, f)).any():
            out.append(Issue(f, f"{f} contains NaN"))
    if np.isnan(data.x_bar).any():
        out.append(Issue("x_bar", "x_bar contains NaN"))
    for t, wt in enumerate(np.asarray(data.w).reshape(data.T, -1)):
        if np.isnan(wt).any():
            out.append(Issue("w", f"w contains NaN at step {t}"))
    for f in ("Q", "Qf", "R"):
        m = getattr(data, f)
        if np.abs(m - m.T).max(initial=0.0) > 1e-12 * max(1.0, np.abs(m).max(initial=0.0)):
            out.append(Issue(f, f"{f} not symmetric"))
    if not out:
        stage = np.block([[data.Q, data.S], [data.S.T, data.R]])
        if not _psd(stage):
            out.append(Issue("Q/S/R", "stage cost matrix [Q S; S' R] not positive semidefinite"))
        if not _psd(data.Qf):
            out.append(Issue("Qf", "Qf not positive semidefinite"))
    for lo, hi, ln, hn in ((data.xl, data.xu, "xl", "xu"), (data.ul, data.uu, "ul", "uu"),
                           (data.gl, data.gu, "gl", "gu")):
        for i in range(len(lo)):
            if np.isfinite(lo[i]) and np.isfinite(hi[i]) and lo[i] > hi[i]:
                out.append(Issue(f"{ln}/{hn}", f"{ln} > {hn} at index {i}"))
    for i in range(d.n_x):
        if np.isfinite(data.xl[i]) and data.x_bar[i] < data.xl[i]:
            out.append(Issue("x_bar", f"x_bar violates xl at index {i}"))
        if np.isfinite(data.xu[i]) and data.x_bar[i] > data.xu[i]:
            out.append(Issue("x_bar", f"x_bar violates xu at index {i}"))
    return out


# ------------------------------------------------------------------ commands
def _opts(a):
    from . import ipm
    return ipm.IpmOptions(tol=a.tol, mu_init=a.mu_init, max_iter=a.max_iter, backend=a.backend)


def _csv(name, N, T, nx, nu, r) -> str:
    return (f"{name},{N},{T},{nx},{nu},{r.iter},{r.total_seconds!r},{r.linalg_seconds!r},"
            f"{r.objective!r},{r.kkt_error!r},{r.status.name}")


def cmd_solve(a) -> int:
    from . import ipm
    try:
        with open(a.file) as f:
            data = read_problem(f.read())
    except (OSError, ParseError, ValueError) as err:
        print(f"error: {err}", file=sys.stderr)
        return INVALID
    issues = validate_problem(data)
    if issues:
        print("invalid problem:\n" + "".join(f"  {i.field}: {i.message}\n" for i in issues),
              end="", file=sys.stderr)
        return INVALID
    opts = _opts(a)
    if a.log_iters:
        opts.log = lambda r: print(r.iter, repr(r.mu), repr(r.alpha), repr(r.alpha_z),
                                   repr(r.kkt_error), repr(r.objective))
    if a.dump:
        with open(a.dump, "w") as f:
            write_dense_qp(f, P.build_dense_qp(data))
    dq = ipm.DeviceQp.from_problem(data)
    try:
        r = dq.solve(opts)
    finally:
        dq.close()
    print(f"status      {r.status.name}\niterations  {r.iter}\ntotal_s     {r.total_seconds!r}\n"
          f"linalg_s    {r.linalg_seconds!r}\nobjective   {r.objective!r}\nkkt_error   {r.kkt_error!r}")
    if a.csv:
        d = P.dims(data)
        print(CSV_HEADER)
        print(_csv(a.file, 0, d.T, d.n_x, d.n_u, r))
        print(f"# device_s {r.device_seconds!r} syrk_s {r.syrk_seconds!r} chol_s {r.chol_seconds!r} "
              f"launches {r.launches} syncs {r.syncs}")
    return EXIT.get(r.status.name, INVALID)


def cmd_bench(a) -> int:
    """bench.cpp run_heat_grid / write_csv / write_summary: N-major, T next, reps innermost."""
    from . import ipm
    opts = _opts(a)
    rows = []
    print(CSV_HEADER)
    for N in a.N:
        for T in a.T:
            for _ in range(a.reps):
                params = P.HeatParams(N=N, T=T, setpoint=a.setpoint)
                try:
                    data = P.build_heat_problem(params)
                    r = ipm.solve_problem(data, opts)
                    line = _csv("heat3d", N, T, N ** 3, 6, r)
                    rows.append((N, T, N ** 3, r))
                except Exception as err:  # the sweep keeps going (bench.hpp:32-34)
                    line = f"heat3d,{N},{T},{N ** 3},6,0,0,0,0,0,error: {err}"
                print(line, flush=True)
    ok = [(N, T, nx, r) for N, T, nx, r in rows if r.status.name == "converged"]
    if not ok:
        print("# no converged runs")
        return 0
    cells = {}
    for N, T, nx, r in ok:
        cells.setdefault((N, T), []).append(r)
    for (N, T), rs in sorted(cells.items()):
        print(f"# N={N} T={T} median total_s {statistics.median(x.total_seconds for x in rs)!r} "
              f"median linalg_s {statistics.median(x.linalg_seconds for x in rs)!r} "
              f"median device_s {statistics.median(x.device_seconds for x in rs)!r}")
    for N in sorted({k[0] for k in cells}):
        pts = sorted((T, statistics.median(x.total_seconds for x in cells[(N, T)]))
                     for (n, T) in cells if n == N)
        if len(pts) >= 2:
            lx, ly = np.log([p[0] for p in pts]), np.log([p[1] for p in pts])
            print(f"# slope log total_s / log T at N={N}: {np.polyfit(lx, ly, 1)[0]!r}")
    return 0


def cmd_gen(a) -> int:
    data = P.build_heat_problem(P.HeatParams(N=a.N, T=a.T, setpoint=a.setpoint))
    if a.dump:
        with open(a.dump, "w") as f:
            write_problem(f, data)
    else:
        write_problem(sys.stdout, data)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="condmpc", description="condensed-space interior-point MPC solver")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def ipm_flags(p):
        p.add_argument("--tol", type=float, default=1e-8, help="KKT tolerance")
        p.add_argument("--mu-init", type=float, default=1e-1, help="initial barrier parameter")
        p.add_argument("--max-iter", type=int, default=200, help="iteration cap")
        p.add_argument("--backend", default="cuda",
                       help="factorization backend: cuda (the reference's reference/eigen select it too)")

    s = sub.add_parser("solve", help="solve a problem file")
    s.add_argument("file")
    ipm_flags(s)
    s.add_argument("--log-iters", action="store_true")
    s.add_argument("--csv", action="store_true")
    s.add_argument("--dump", default="")
    ints = lambda t: [int(x) for x in t.split(",")]
    b = sub.add_parser("bench", help="run the heat-cube benchmark grid, CSV to stdout")
    b.add_argument("--N", type=ints, default=[2, 3, 4])
    b.add_argument("--T", type=ints, default=[10, 50])
    b.add_argument("--reps", type=int, default=1)
    b.add_argument("--setpoint", type=float, default=350.0)
    ipm_flags(b)
    g = sub.add_parser("gen", help="emit a heat-cube problem file")
    g.add_argument("--N", type=int, default=4)
    g.add_argument("--T", type=int, default=50)
    g.add_argument("--setpoint", type=float, default=350.0)
    g.add_argument("--dump", default="")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else INVALID
    from . import linalg
    if getattr(a, "backend", "cuda") not in linalg.BACKEND_NAMES:
        print(f"error: unknown factorization backend: {a.backend}", file=sys.stderr)
        return INVALID
    if getattr(a, "reps", 1) < 1 or (a.cmd == "gen" and (a.N < 1 or a.T < 1)):
        print("error: value must be positive", file=sys.stderr)
        return INVALID
    try:
        return {"solve": cmd_solve, "bench": cmd_bench, "gen": cmd_gen}[a.cmd](a)
    except Exception as err:
        print(f"error: {err}", file=sys.stderr)
        return INVALID


if __name__ == "__main__":
    sys.exit(main())
