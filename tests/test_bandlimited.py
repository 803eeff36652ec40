"""Band-limited kernel Phi_sigma and the O(N^2) band-limited / hybrid oracles
(the radial table and direct_matvec_hybrid).

Reference behaviour: eval_bandlimited (bandlimit.cpp:307-334), the radial
table (bandlimit.cpp:229-262), direct_matvec(use_bandlimited=true)
(fmm.cpp:57-70) and direct_matvec_hybrid (fmm.cpp:77-113). Golden values:
test_bandlimit.cpp:120-141 (eval_bandlimited at sigma = pi) and
tests/golden/bandlimited_1d_ref.npz (outputs of the reference itself, made by
tests/golden/make_golden.py). The CPU tests exercise the library's host
plan-time math; the GPU tests the O(N^2) kernel through the C ABI.

Tolerances: Phi_sigma values against the reference's golden numbers at the
reference tests' own epsilons (1e-12 Gaussian, 1e-10 IMQ / MQ; measured
~1e-15); GPU oracles against the reference's outputs at rel-l2 <= 1e-12
(same table arithmetic, the table values differ by quadrature rounding only).
"""
import math
import os

import numpy as np
import pytest

from paper_1606_07652_b200 import inputs as I

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "bandlimited_1d_ref.npz")


def rel_l2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def rel_linf(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


# test_bandlimit.cpp:120-141, sigma = pi, refinement 2048 (the d=1 default)
EVAL_GOLDEN = [
    ("gaussian:c=1", 0.0, 0.97367892507825857, 1e-12),
    ("gaussian:c=1", 0.5, 0.78500162347256436, 1e-12),
    ("imq:c=1", 0.0, 0.98325045404027081, 1e-10),
    ("imq:c=1", 0.25, 0.96143728916669926, 1e-10),
    ("imq:c=1", 0.5, 0.90069708853343813, 1e-10),
    ("imq:c=1", 1.0, 0.71632964302991934, 1e-10),
    ("mq:c=1", 0.0, 1.0048404606633916, 1e-10),
    ("mq:c=1", 0.5, 1.1164784549388851, 1e-10),
]


@pytest.mark.parametrize("spec,x,want,eps", EVAL_GOLDEN)
def test_eval_bandlimited_reference_values(blfmm, spec, x, want, eps):
    v = blfmm.eval_bandlimited(blfmm.parse_kernel_spec(spec), math.pi, x)
    assert abs(v - want) <= eps * abs(want)
    # even in x
    assert blfmm.eval_bandlimited(blfmm.parse_kernel_spec(spec), math.pi, -x) == v


def test_eval_bandlimited_validation(blfmm):
    k = blfmm.parse_kernel_spec("imq:c=1")
    with pytest.raises(blfmm.InvalidArgument):
        blfmm.eval_bandlimited(k, 0.0, 0.5)
    with pytest.raises(blfmm.InvalidArgument):
        blfmm.eval_bandlimited(k, math.pi, 0.5, refinement=512)  # below reference resolution
    with pytest.raises(blfmm.DomainError):  # d = 2 band integral: not on this library's path
        blfmm.eval_bandlimited(k, math.pi, (0.5, 0.5), d=2)
    with pytest.raises(blfmm.DomainError):
        blfmm.eval_bandlimited(blfmm.parse_kernel_spec("tps"), math.pi, 0.5)


def test_radial_table_matches_reference(blfmm, oracle):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    for spec, sigma in [("gaussian:c=1", math.pi), ("imq:c=0.1", math.pi), ("mq:c=0.05", 5.0)]:
        k = blfmm.parse_kernel_spec(spec)
        step, vals = blfmm.bandlimited_radial_table(k, sigma, 1.0, 1024)
        assert step == 1.0 / 1024 and vals.shape == (1027,)
        for i in (0, 1, 17, 500, 1023, 1026):
            want = oracle.ref_eval_bandlimited(spec, sigma, i * step, 1024)
            assert abs(vals[i] - want) <= 1e-13 * max(1.0, abs(want)), (spec, i)


def test_direct_bandlimited_refuses_d2_before_any_device_work(blfmm):
    k = blfmm.parse_kernel_spec("gaussian:c=1")
    ps = blfmm.PointSet(2, I.generate_quasiuniform(9, 2, 8, 0.0))
    with pytest.raises(blfmm.DomainError):
        blfmm.direct_matvec(k, ps, np.ones(9), use_bandlimited=True, sigma=math.pi)
    with pytest.raises(blfmm.DomainError):
        blfmm.direct_matvec_hybrid(k, ps, blfmm.build_tree(ps, 2), np.ones(9), math.pi)
    ps1 = blfmm.PointSet(1, np.zeros((0, 1)))
    r = blfmm.direct_matvec(k, ps1, np.zeros(0), use_bandlimited=True, sigma=math.pi)
    assert r.values.shape == (0,)


# ------------------------------------------------------------------- GPU
def _cases():
    z = np.load(GOLDEN)
    for i in range(int(z["ncases"])):
        yield (z[f"x_{i}"], z[f"w_{i}"], str(z[f"spec_{i}"]), float(z[f"sigma_{i}"]),
               int(z[f"refinement_{i}"]), int(z[f"leaf_{i}"]), z[f"band_{i}"],
               z[f"hybrid_{i}"] if f"hybrid_{i}" in z else None)


@pytest.mark.gpu
def test_gpu_bandlimited_and_hybrid_match_reference(blfmm):
    for x, w, spec, sigma, refinement, leaf, band, hybrid in _cases():
        k = blfmm.parse_kernel_spec(spec)
        ps = blfmm.PointSet(1, x)
        r = blfmm.direct_matvec(k, ps, w, use_bandlimited=True, sigma=sigma,
                                refinement=refinement)
        assert r.stats.near_pairs == len(w) ** 2
        # Points outside the domain put distances past rmax, where both
        # implementations extrapolate the end interval's cubic with t up to
        # ~400: rounding-level table differences grow by ~t^3/6.
        outside = x.min() < 0.0 or x.max() > 1.0
        tol = 1e-8 if outside else 1e-12
        assert rel_l2(r.values, band) <= tol, (spec, len(w))
        if hybrid is not None:
            h = blfmm.direct_matvec_hybrid(k, ps, blfmm.build_tree(ps, leaf), w, sigma,
                                           refinement)
            assert rel_l2(h.values, hybrid) <= tol, (spec, len(w), leaf)


@pytest.mark.gpu
def test_gpu_band_table_path_matches_eval_bandlimited(blfmm):
    # test_fmm.cpp:68-87
    k = blfmm.parse_kernel_spec("gaussian:c=1")
    x = I.generate_quasiuniform(16, 1, 8, 0.5)
    w = I.uniform_weights(16, 3)
    r = blfmm.direct_matvec(k, blfmm.PointSet(1, x), w, use_bandlimited=True, sigma=math.pi,
                            refinement=4096)
    for i in range(16):
        want = sum(w[j] * blfmm.eval_bandlimited(k, math.pi, x[i, 0] - x[j, 0])
                   for j in range(16))
        assert abs(r.values[i] - want) <= 1e-8 * abs(want)


@pytest.mark.gpu
def test_gpu_hybrid_near_keeps_kernel(blfmm):
    # test_fmm.cpp:89-107: two points in leaf 0, two in leaf 3 (level 2)
    k = blfmm.parse_kernel_spec("imq:c=1")
    x = np.array([[0.05], [0.1], [0.9], [0.95]])
    w = np.array([1.0, -2.0, 0.5, 1.5])
    ps = blfmm.PointSet(1, x)
    r = blfmm.direct_matvec_hybrid(k, ps, blfmm.build_tree(ps, 2), w, math.pi, 4096)
    for i in range(4):
        want = 0.0
        for j in range(4):
            d = x[i, 0] - x[j, 0]
            near = (i < 2) == (j < 2)
            want += w[j] * (1.0 / math.sqrt(d * d + 1.0) if near
                            else blfmm.eval_bandlimited(k, math.pi, d))
        assert abs(r.values[i] - want) <= 1e-8 * abs(want)


@pytest.mark.gpu
def test_gpu_single_level_matches_hybrid_oracle(blfmm):
    # test_fmm.cpp:131-152: the fast method converges to the hybrid oracle in M
    k = blfmm.parse_kernel_spec("imq:c=1")
    x = I.generate_quasiuniform(256, 1, 2026, 0.35)
    w = I.uniform_weights(256, 99)
    ps = blfmm.PointSet(1, x)
    tree = blfmm.build_tree(ps, 4)
    oracle = blfmm.direct_matvec_hybrid(k, ps, tree, w, math.pi, 4096).values
    e = {}
    for m in (64, 128):
        req = blfmm.SumRequest(k, math.pi, ps, w, m)
        e[m] = rel_linf(blfmm.fmm_matvec_single(req, tree).values, oracle)
    assert e[64] < 1e-3
    assert e[128] * 2.0 <= e[64]
    band = blfmm.direct_matvec(k, ps, w, use_bandlimited=True, sigma=math.pi,
                               refinement=4096).values
    req = blfmm.SumRequest(k, math.pi, ps, w, 128)
    assert rel_linf(blfmm.fmm_matvec_single(req, tree).values, band) < 5e-2


@pytest.mark.gpu
def test_gpu_mlfmm_matches_hybrid_oracle(blfmm):
    # test_mlfmm.cpp:426-437 (measured 8.8e-4 by the reference)
    k = blfmm.parse_kernel_spec("imq:c=1")
    x = I.generate_quasiuniform(1024, 1, 2026, 0.35)
    w = I.uniform_weights(1024, 99)
    ps = blfmm.PointSet(1, x)
    tree = blfmm.build_tree(ps, 5)
    grids = blfmm.make_level_grids(k, math.pi, 64, 1, 5)
    r = blfmm.mlfmm_matvec(blfmm.SumRequest(k, math.pi, ps, w, 64), tree, grids)
    oracle = blfmm.direct_matvec_hybrid(k, ps, tree, w, math.pi, 4096).values
    assert rel_linf(r.values, oracle) < 1e-3
    assert r.stats.far_work > 0
