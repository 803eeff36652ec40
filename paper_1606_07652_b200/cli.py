"""`blfmm` command-line driver, GPU backend: the `fmm-matvec` and `solve`
subcommands of /root/reference/proj/tools/blfmm_cli.cpp.

Same flags, defaults, artifact format and exit codes as the reference:
  - CSV artifacts open with `#` metadata lines (version, command line, seed,
    timestamp), then the command's `#` stats lines, then one `%.17g` value
    per line (blfmm_cli.cpp:46-74, 400-412, 433-447);
  - errors go to stderr as ONE JSON line; exit 0 iff every embedded check
    passed, 1 for failed checks / accuracy_error (with "achieved"), 2 for
    usage / IO / argument errors (blfmm_cli.cpp:160-168, 705-737);
  - `--dump-expansions` writes the upsweep multipoles of levels 2..L for
    every box in the reference's row-major box order (386-396).
Points files hold x[,y[,z]] lines (the reference reads d <= 2; a third column
is this backend's 3-D extension) and get the reference's padded tight bounds
(geometry.cpp:160-198).

    python -m paper_1606_07652_b200.cli fmm-matvec --kernel imq:c=1 \\
        --points pts.csv --weights w.csv --mode mlfmm --levels 3 --out u.csv
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time

import numpy as np

VERSION = "0.1.0"
PI = 3.14159265358979323846


class _Usage(Exception):
    pass


def fmt(v: float) -> str:
    return "%.17g" % v


def _csv_header(cmdline: str, seed: int) -> list[str]:
    return ["# blfmm " + VERSION, "# command: " + cmdline, "# seed: %d" % seed,
            "# generated: " + time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())]


def read_vector_csv(path: str) -> np.ndarray:
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise RuntimeError("cannot open " + path)
    return np.array([float(s) for s in lines if s and s[0] != "#"], dtype=np.float64)


def infer_dimension(path: str) -> int:
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise RuntimeError("cannot open " + path)
    for s in lines:
        if s and s[0] != "#":
            return 1 + s.count(",")
    raise RuntimeError("no data lines in " + path)


def read_points_csv(path: str, d: int):
    """geometry.cpp:160-198: tight bounds padded by 1e-9 max(1, extent)."""
    from . import api as B
    rows = []
    for s in open(path).read().splitlines():
        if not s or s[0] == "#":
            continue
        parts = s.split(",")
        if len(parts) != d:
            raise RuntimeError("expected %d columns in %s" % (d, path))
        rows.append([float(v) for v in parts])
    x = np.asarray(rows, dtype=np.float64).reshape(-1, d)
    lo, hi = [0.0, 0.0, 0.0], [1.0, 1.0, 1.0]
    if x.shape[0]:
        for k in range(d):
            a, b = float(x[:, k].min()), float(x[:, k].max())
            pad = 1e-9 * max(1.0, b - a)
            lo[k], hi[k] = a - pad, b + pad
    return B.PointSet(d, x, B.BoundingBox(tuple(lo), tuple(hi)))


def cmd_fmm_matvec(a, cmdline: str) -> int:
    """blfmm_cli.cpp:353-413."""
    from . import api as B
    from .solver import default_leaf_level
    k = B.parse_kernel_spec(a.kernel)
    ps = read_points_csv(a.points, infer_dimension(a.points))
    w = read_vector_csv(a.weights)
    if w.shape[0] != ps.size():
        raise ValueError("weights length %d != point count %d" % (w.shape[0], ps.size()))
    if a.dump_expansions and a.mode != "mlfmm":
        raise ValueError("--dump-expansions needs --mode mlfmm")
    n = ps.size()
    m = a.m if a.m > 0 else B.choose_truncation(n)
    if a.mode == "direct":
        res = B.direct_matvec(k, ps, w, False, a.sigma)
    elif a.mode == "single":
        level = a.levels if a.levels > 0 else default_leaf_level(n, ps.d, False)
        tree = B.build_tree(ps, level)
        res = B.fmm_matvec_single(B.SumRequest(k, a.sigma, ps, w, m), tree)
    else:
        level = a.levels if a.levels > 0 else default_leaf_level(n, ps.d, True)
        if level < 3:
            raise ValueError("mlfmm needs --levels >= 3")
        tree = B.build_tree(ps, level)
        grids = B.make_level_grids(k, a.sigma, m, ps.d, level, B.GridMode.shared, a.stencil_k)
        req = B.SumRequest(k, a.sigma, ps, w, m)
        if a.dump_expansions:
            plan = B.Plan(ps, level, k, a.sigma, m, c_table=grids.factors[level].c_vals)
            plan.execute(w)
            out = _csv_header(cmdline, a.seed) + ["level,box,node,coeff_re,coeff_im"]
            for lvl in range(2, level + 1):
                ex = plan.expansions(lvl, 0)
                for box in range(ex.shape[0]):
                    for node in range(ex.shape[1]):
                        z = ex[box, node]
                        out.append("%d,%d,%d,%s,%s" % (lvl, box, node, fmt(z.real), fmt(z.imag)))
            _write(a.dump_expansions, out)
        res = B.mlfmm_matvec(req, tree, grids)
    fails = []
    out = _csv_header(cmdline, a.seed)
    out += ["# mode: " + a.mode, "# near_pairs: %d" % res.stats.near_pairs,
            "# far_work: %d" % res.stats.far_work,
            "# max_imag_residual: " + fmt(res.stats.max_imag_residual)]
    for v in np.asarray(res.values, dtype=np.float64):
        if not math.isfinite(v):
            fails.append("non-finite output value")
        out.append(fmt(v))
    _write(a.out, out)
    return _finish("fmm-matvec", fails)


def cmd_solve(a, cmdline: str) -> int:
    """blfmm_cli.cpp:416-448 over solver.solve_interpolation (GPU matvec)."""
    from . import api as B
    from . import solver as S
    ps = read_points_csv(a.points, infer_dimension(a.points))
    prob = S.InterpolationProblem(kernel=B.parse_kernel_spec(a.kernel), ps=ps,
                                  rhs=read_vector_csv(a.rhs),
                                  backend={"dense": S.Backend.dense,
                                           "single_fmm": S.Backend.single_fmm,
                                           "mlfmm": S.Backend.mlfmm}[a.backend],
                                  tol=a.tol, max_iter=a.max_iter, sigma=a.sigma,
                                  m_per_dim=a.m, leaf_level=a.levels)
    lam, st = S.solve_interpolation(prob)
    fails = []
    out = _csv_header(cmdline, a.seed)
    out += ["# backend: " + a.backend, "# method: " + st.method,
            "# iterations: %d" % st.iterations, "# matvecs: %d" % st.matvecs,
            "# residual: " + fmt(st.residual), "# converged: %d" % (1 if st.converged else 0)]
    for v in lam:
        if not math.isfinite(v):
            fails.append("non-finite coefficient")
        out.append(fmt(v))
    if not st.converged:
        fails.append("solver did not converge")
    _write(a.out, out)
    return _finish("solve", fails)


def _lround(v: float) -> int:
    return int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))


def _write(path: str, lines: list[str]):
    try:
        with open(path, "w") as f:
            f.write("\n".join(lines) + "\n")
    except OSError:
        raise RuntimeError("cannot open " + path)


def _finish(command: str, fails: list[str]) -> int:
    if not fails:
        return 0
    print(json.dumps({"command": command, "error": "embedded checks failed",
                      "failures": fails}), file=sys.stderr)
    return 1


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise _Usage(message)


def _range(lo, hi, typ):
    def conv(s):
        v = typ(s)
        if not (lo <= v <= hi):
            raise argparse.ArgumentTypeError("%s not in [%s, %s]" % (s, lo, hi))
        return v
    return conv


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="blfmm", description="band-limited kernel FMM driver (GPU backend)")
    ap.add_argument("--version", action="version", version=VERSION)
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p, kernel_required=True):
        p.add_argument("--kernel", required=kernel_required, help="kernel spec, name:param=value")
        p.add_argument("--sigma", type=_range(1e-6, 1e6, float), default=None,
                       help="frequency cutoff")
        p.add_argument("--seed", type=int, default=1234, help="RNG seed")
        p.add_argument("--threads", type=_range(0, 256, int), default=0,
                       help="accepted for compatibility (the GPU path ignores it)")

    mv = sub.add_parser("fmm-matvec", help="one kernel summation")
    common(mv)
    mv.add_argument("--points", required=True, help="points CSV, x[,y[,z]] lines")
    mv.add_argument("--weights", required=True, help="one weight per line")
    mv.add_argument("--mode", choices=["single", "direct", "mlfmm"], default="single")
    mv.add_argument("--m", type=_range(0, 16384, int), default=0,
                    help="frequency nodes (0: sqrt-N rule)")
    mv.add_argument("--levels", type=_range(0, 12, int), default=0,
                    help="leaf level (0: from N)")
    mv.add_argument("--stencil-k", dest="stencil_k", type=_range(2, 64, int), default=10,
                    help="interpolation stencil")
    mv.add_argument("--dump-expansions", dest="dump_expansions", default="",
                    help="write per-level multipole coefficients (mlfmm)")
    mv.add_argument("--out", required=True, help="output CSV")

    so = sub.add_parser("solve", help="fit interpolation weights")
    common(so)
    so.add_argument("--points", required=True)
    so.add_argument("--rhs", required=True, help="one value per line")
    so.add_argument("--backend", choices=["dense", "single_fmm", "mlfmm"], default="dense")
    so.add_argument("--tol", type=_range(1e-15, 1.0, float), default=1e-8)
    so.add_argument("--max-iter", dest="max_iter", type=_range(1, 100000, int), default=2000)
    so.add_argument("--m", type=_range(0, 16384, int), default=0)
    so.add_argument("--levels", type=_range(0, 12, int), default=0)
    so.add_argument("--out", required=True, help="coefficients CSV")
    return ap


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    cmdline = " ".join(["blfmm"] + list(argv))
    try:
        a = build_parser().parse_args(argv)
    except _Usage as e:
        print(json.dumps({"error": str(e), "command": "parse"}), file=sys.stderr)
        return 2
    import os
    for attr in ("points", "weights", "rhs"):
        p = getattr(a, attr, None)
        if p is not None and not os.path.isfile(p):
            print(json.dumps({"error": "%s: File does not exist: %s" % ("--" + attr, p),
                              "command": "parse"}), file=sys.stderr)
            return 2
    # per-command defaults (blfmm_cli.cpp:695-700): solve defers sigma to the library
    if a.sigma is None:
        a.sigma = 0.0 if a.command == "solve" else PI
    from .api import AccuracyError
    try:
        if a.command == "fmm-matvec":
            return cmd_fmm_matvec(a, cmdline)
        return cmd_solve(a, cmdline)
    except AccuracyError as e:
        print(json.dumps({"error": str(e), "achieved": float(getattr(e, "achieved", math.nan)),
                          "command": cmdline}), file=sys.stderr)
        return 1
    except Exception as e:  # std::exception -> 2 (blfmm_cli.cpp:731-735)
        print(json.dumps({"error": str(e), "command": cmdline}), file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
