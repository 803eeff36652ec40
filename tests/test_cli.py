"""The `blfmm` CLI drop-in (paper_1606_07652_b200/cli.py) run end to end, as
the reference's tests/test_cli.cpp drives its binary: artifact formats,
exit codes, single-line JSON errors (test_cli.cpp:229-318)."""
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1606_07652_b200 import inputs as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_cli(args, cwd):
    r = subprocess.run([sys.executable, "-m", "paper_1606_07652_b200.cli"] + args, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout, r.stderr


def read_values(path):
    return np.array([float(s) for s in open(path).read().splitlines() if s and s[0] != "#"])


def read_csv(path):
    return [s.split(",") for s in open(path).read().splitlines() if s and s[0] != "#"]


@pytest.fixture()
def fixture_files(tmp_path):
    """test_cli.cpp:104-118: 256 jittered 1-D points, weights, smooth rhs."""
    x = I.generate_quasiuniform(256, 1, 424242, 0.35)[:, 0]
    pts, w, rhs = tmp_path / "pts.csv", tmp_path / "w.csv", tmp_path / "rhs.csv"
    pts.write_text("".join("%.17g\n" % v for v in x))
    w.write_text("".join("%.17g\n" % (2.0 * I.uniform01(99, j) - 1.0) for j in range(256)))
    rhs.write_text("".join("%.17g\n" % math.sin(math.pi * v) for v in x))
    return pts, w, rhs


def test_usage_errors_are_single_line_json(tmp_path, fixture_files):
    pts, w, _ = fixture_files
    rc, _, err = run_cli(["fmm-matvec", "--points", str(pts), "--weights", str(w),
                          "--out", str(tmp_path / "u.csv")], tmp_path)  # --kernel missing
    assert rc == 2
    j = json.loads(err)
    assert j["command"] == "parse" and err.count("\n") == 1
    rc, _, err = run_cli(["fmm-matvec", "--kernel", "imq:c=1", "--points", str(tmp_path / "no"),
                          "--weights", str(w), "--out", str(tmp_path / "u.csv")], tmp_path)
    assert rc == 2 and "error" in json.loads(err)
    rc, _, err = run_cli(["fmm-matvec", "--kernel", "imq:c=1", "--points", str(pts),
                          "--weights", str(w), "--mode", "bogus", "--out", "x"], tmp_path)
    assert rc == 2


def test_dump_expansions_needs_mlfmm(tmp_path, fixture_files):
    pts, w, _ = fixture_files
    rc, _, err = run_cli(["fmm-matvec", "--mode", "single", "--dump-expansions", "x.csv",
                          "--kernel", "imq:c=1", "--points", str(pts), "--weights", str(w),
                          "--out", str(tmp_path / "u.csv")], tmp_path)
    assert rc == 2
    assert "--dump-expansions needs --mode mlfmm" in json.loads(err)["error"]


def test_weight_count_mismatch(tmp_path, fixture_files):
    pts, _, _ = fixture_files
    w = tmp_path / "w3.csv"
    w.write_text("1\n2\n3\n")
    rc, _, err = run_cli(["fmm-matvec", "--kernel", "imq:c=1", "--points", str(pts),
                          "--weights", str(w), "--out", str(tmp_path / "u.csv")], tmp_path)
    assert rc == 2 and "weights length 3 != point count 256" in json.loads(err)["error"]


@pytest.mark.gpu
def test_fmm_matvec_modes_agree_and_dump(tmp_path, fixture_files):
    """test_cli.cpp:229-291 on the GPU backend."""
    pts, w, _ = fixture_files
    common = ["--kernel", "imq:c=1", "--points", str(pts), "--weights", str(w),
              "--sigma", "3.14159265358979", "--m", "64"]
    ud, us, um, ex = (tmp_path / f for f in ("ud.csv", "us.csv", "um.csv", "exp.csv"))
    assert run_cli(["fmm-matvec", "--mode", "direct"] + common + ["--out", str(ud)], tmp_path)[0] == 0
    assert run_cli(["fmm-matvec", "--mode", "single", "--levels", "3"] + common +
                   ["--out", str(us)], tmp_path)[0] == 0
    rc, _, err = run_cli(["fmm-matvec", "--mode", "mlfmm", "--levels", "3", "--dump-expansions",
                          str(ex)] + common + ["--out", str(um)], tmp_path)
    assert rc == 0, err
    d, s, m = read_values(ud), read_values(us), read_values(um)
    assert d.size == s.size == m.size == 256
    scale = np.abs(d).max()
    assert np.abs(s - m).max() < 1e-10 * scale  # shared grids telescope
    ds = np.abs(d - s).max()
    assert 1e-4 * scale < ds < 5e-2 * scale  # the sigma = pi mollification gap
    text = open(um).read()
    for key in ("# blfmm 0.1.0", "# command: ", "# seed: 1234", "# generated: ", "# mode: mlfmm",
                "# near_pairs: ", "# far_work: ", "# max_imag_residual: "):
        assert key in text
    rows = read_csv(ex)
    assert rows[0] == ["level", "box", "node", "coeff_re", "coeff_im"]
    assert len(rows) - 1 == (4 + 8) * 64
    for r in rows[1:]:
        assert 2 <= int(r[0]) <= 3 and math.isfinite(float(r[3])) and math.isfinite(float(r[4]))
    # reruns agree except for the timestamp line
    um2 = tmp_path / "um2.csv"
    run_cli(["fmm-matvec", "--mode", "mlfmm", "--levels", "3"] + common + ["--out", str(um2)],
            tmp_path)
    strip = lambda t: [l for l in t.splitlines() if not l.startswith("# generated:")
                       and not l.startswith("# command:")]
    assert strip(open(um).read()) == strip(open(um2).read())


@pytest.mark.gpu
def test_solve_writes_converged_coefficients(tmp_path, fixture_files):
    pts, _, rhs = fixture_files
    lam = tmp_path / "lambda.csv"
    # band-capturing Gaussian (sigma covers the spectrum, as tests/test_solver.py)
    band = ["--kernel", "gaussian:c=256", "--sigma", "203", "--m", "2112", "--levels", "3"]
    rc, _, err = run_cli(["solve"] + band + ["--points", str(pts), "--rhs", str(rhs),
                          "--backend", "mlfmm", "--tol", "1e-6", "--out", str(lam)], tmp_path)
    assert rc == 0, err
    text = open(lam).read()
    assert "# method: cg" in text and "# converged: 1" in text
    assert read_values(lam).size == 256
    # an unreachable iteration cap surfaces as a one-line JSON accuracy error, exit 1
    rc, _, err = run_cli(["solve"] + band + ["--points", str(pts), "--rhs", str(rhs),
                          "--backend", "mlfmm", "--tol", "1e-12", "--max-iter", "2",
                          "--out", str(lam)], tmp_path)
    assert rc == 1
    assert '"achieved"' in err and err.count("\n") == 1


@pytest.mark.gpu
def test_solve_reference_case_tps_dense(tmp_path, fixture_files):
    """test_cli.cpp:293-318 verbatim: `solve --kernel tps:beta=2 --backend dense
    --tol 1e-8` converges with GMRES; `--max-iter 2` fails with a one-line JSON
    error carrying "achieved" and exit code 1."""
    pts, _, rhs = fixture_files
    lam = tmp_path / "lambda.csv"
    rc, _, err = run_cli(["solve", "--kernel", "tps:beta=2", "--points", str(pts), "--rhs",
                          str(rhs), "--backend", "dense", "--tol", "1e-8", "--out", str(lam)],
                         tmp_path)
    assert rc == 0, err
    text = open(lam).read()
    assert read_values(lam).size == 256
    assert "# method: gmres" in text and "# converged: 1" in text
    rc, _, err = run_cli(["solve", "--kernel", "tps:beta=2", "--points", str(pts), "--rhs",
                          str(rhs), "--backend", "dense", "--tol", "1e-8", "--max-iter", "2",
                          "--out", str(lam)], tmp_path)
    assert rc == 1
    assert '"achieved"' in err and err.find("\n") == len(err) - 1  # single line


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [1, 2])
def test_fmm_matvec_outputs_match_reference(tmp_path, oracle, dim):
    """The CLI's artifacts against the REFERENCE library (compiled from its
    sources; the oracle restatement where it is absent): u of every mode
    (direct / single / mlfmm, rel-l2 <= 1e-10 against direct_matvec /
    fmm_matvec_single / mlfmm_matvec on the same tight-bounds domain), the
    near_pairs / far_work header lines, and the --dump-expansions multipoles
    in reference box order (upsweep, mlfmm.cpp:201-266)."""
    n = 512 if dim == 1 else 1024
    x = np.stack([I.generate_quasiuniform(n, 1, 7 + q, 0.35)[:, 0] for q in range(dim)], 1)
    w = np.array([2.0 * I.uniform01(1999, j) - 1.0 for j in range(n)])
    pts, wf = tmp_path / "pts.csv", tmp_path / "w.csv"
    pts.write_text("".join(",".join("%.17g" % v for v in row) + "\n" for row in x))
    wf.write_text("".join("%.17g\n" % v for v in w))
    spec, sigma, m, lev = "imq:c=0.5", 3.14159265358979, 16 if dim == 2 else 64, 3
    lo = [x[:, k].min() - 1e-9 * max(1.0, np.ptp(x[:, k])) for k in range(dim)]
    hi = [x[:, k].max() + 1e-9 * max(1.0, np.ptp(x[:, k])) for k in range(dim)]
    common = ["--kernel", spec, "--points", str(pts), "--weights", str(wf),
              "--sigma", "%.17g" % sigma, "--m", str(m)]
    outs = {}
    for mode in ("direct", "single", "mlfmm"):
        extra = ["--levels", str(lev)] if mode != "direct" else []
        if mode == "mlfmm":
            extra += ["--dump-expansions", str(tmp_path / "exp.csv")]
        rc, _, err = run_cli(["fmm-matvec", "--mode", mode] + common + extra +
                             ["--out", str(tmp_path / f"u_{mode}.csv")], tmp_path)
        assert rc == 0, err
        outs[mode] = read_values(tmp_path / f"u_{mode}.csv")
    header = open(tmp_path / "u_mlfmm.csv").read()
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    if oracle.ref_available():
        rd = oracle.ref_direct(x, w, spec)[0]
        rs, sst = oracle.ref_single(x, w, spec, sigma, m, lev, lo=lo, hi=hi)
        rm, mst = oracle.ref_mlfmm(x, w, spec, sigma, m, lev, lo=lo, hi=hi)
        ex = [oracle.ref_expansions(x, w, spec, sigma, m, lev, l, 0, lo=lo, hi=hi)
              for l in range(2, lev + 1)]
    else:
        rd = oracle.direct(x, w, spec)
        rs, sst, _ = oracle.mlfmm(x, w, spec, sigma, m, lev, lo=lo, hi=hi)
        rm, mst, _ = oracle.mlfmm(x, w, spec, sigma, m, lev, lo=lo, hi=hi)
        ex = None
    assert rel(outs["direct"], rd) <= 1e-12
    assert rel(outs["single"], rs) <= 1e-10
    assert rel(outs["mlfmm"], rm) <= 1e-10
    assert f"# near_pairs: {mst['near_pairs']}" in header
    assert f"# far_work: {mst['far_work']}" in header
    if ex is not None:
        rows = read_csv(tmp_path / "exp.csv")[1:]
        got = {}
        for r in rows:
            got[(int(r[0]), int(r[1]), int(r[2]))] = float(r[3]) + 1j * float(r[4])
        for li, l in enumerate(range(2, lev + 1)):
            ref = ex[li]
            g = np.array([[got[(l, b, e)] for e in range(ref.shape[1])] for b in range(ref.shape[0])])
            assert np.linalg.norm(g - ref) <= 1e-10 * max(np.linalg.norm(ref), 1e-300)
