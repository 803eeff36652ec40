"""The C-ABI library loads, exports every symbol include/blfmm_gpu.h
declares, and its host-side plan math (kernel-spec grammar, translation
spectrum) matches the oracle. No GPU compute here; without a device every
compute entry point must fail loudly (no CPU fallback)."""
import ctypes as ct
import math
import os
import re

import numpy as np
import pytest

from paper_1606_07652_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "blfmm_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(blfmm_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = ct.CDLL(_capi.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_capi.EXPORTS), "ctypes table out of sync with the header"
    assert _capi.lib().blfmm_abi_version() == 4


def test_library_is_sm100a():
    import subprocess
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH],
                       capture_output=True, text=True)
    assert "sm_100a" in r.stdout


@pytest.mark.parametrize("spec,t,shape", [("gaussian:c=16", 0, 16.0), ("GA", 0, 1.0),
                                          ("IMQ:c=0.1", 2, 0.1), ("multiquadric:c=0.05", 1, 0.05),
                                          ("mq", 1, 1.0), ("tps:beta=4", 3, 4.0),
                                          ("wendland:eps=0.5", 4, 0.5)])
def test_parse_kernel_spec(blfmm, spec, t, shape):
    k = blfmm.parse_kernel_spec(spec)
    assert int(k.type) == t and k.shape == shape


@pytest.mark.parametrize("bad", ["foo", "imq:eps=1", "imq:c=-1", "imq:c=0", "tps:beta=3",
                                 "imq:c=1x", "imq:c", "gaussian:c=inf"])
def test_parse_kernel_spec_rejects(blfmm, bad):
    # kernels.cpp:48-103 throws std::invalid_argument on junk
    with pytest.raises(blfmm.InvalidArgument):
        blfmm.parse_kernel_spec(bad)


@pytest.mark.parametrize("spec,d,m,sigma", [
    ("gaussian:c=16", 2, 64, math.pi), ("gaussian:c=64", 3, 58, 101.8),
    ("imq:c=0.1", 3, 16, math.pi), ("mq:c=0.05", 2, 16, math.pi), ("imq:c=1", 2, 12, math.pi),
    ("imq:c=1", 1, 8, math.pi), ("mq:c=1", 3, 6, math.pi), ("imq:c=0.5", 3, 7, math.pi)])
def test_translation_spectrum_matches_oracle(blfmm, oracle, spec, d, m, sigma):
    k = blfmm.parse_kernel_spec(spec)
    c = blfmm.translation_coefficients(k, blfmm.make_quadrature(sigma, m, d)).c_vals
    o = oracle.c_table(spec, sigma, m, d)
    assert np.abs(c - o).max() <= 1e-13 * np.abs(o).max()


def test_translation_spectrum_frozen(blfmm):
    # test_bandlimit.cpp:207-217
    k = blfmm.parse_kernel_spec("gaussian:c=1")
    c = blfmm.translation_coefficients(k, blfmm.make_quadrature(2.0, 4, 1)).c_vals
    assert abs(c[3] - 0.2196956447338612) <= 1e-13 * 0.2196956447338612
    assert abs(c[2] - math.sqrt(math.pi) / (2 * math.pi)) <= 1e-13


def test_unsupported_kernel_is_domain_error(blfmm):
    k = blfmm.parse_kernel_spec("tps:beta=2")
    with pytest.raises(blfmm.DomainError):
        blfmm.translation_coefficients(k, blfmm.make_quadrature(math.pi, 8, 2))


def test_validation_errors(blfmm):
    with pytest.raises(blfmm.InvalidArgument):
        blfmm.make_quadrature(0.0, 8, 2)
    with pytest.raises(blfmm.InvalidArgument):
        blfmm.make_quadrature(1.0, 1, 2)
    ps = blfmm.PointSet(3, np.zeros((4, 3)))
    with pytest.raises(blfmm.InvalidArgument):
        blfmm.build_tree(ps, 1)
    with pytest.raises(blfmm.InvalidArgument):
        blfmm.build_tree(ps, 9)  # d*L > 24
    with pytest.raises(blfmm.InvalidArgument):
        blfmm.choose_truncation(3)
    assert blfmm.choose_truncation(101) == 12 and blfmm.choose_truncation(256) == 16


def test_boxtree_index_helpers(blfmm):
    # geometry.cpp:201-262 / test_geometry.cpp:194-205, 286-292
    ps = blfmm.PointSet(2, np.zeros((1, 2)))
    t = blfmm.build_tree(ps, 2)
    assert t.leaf_of((0.3, 0.8)) == 7 and t.leaf_of((1.0, 1.0)) == 15
    assert t.children(1, 3) == [10, 11, 14, 15]
    assert t.parent(2, 15) == 3
    t1 = blfmm.build_tree(blfmm.PointSet(1, np.zeros((1, 1))), 2)
    assert t1.side(2, 0) == 0.25 and abs(t1.center(2, 1)[0] - 0.375) < 1e-15


def test_no_gpu_fails_loudly(blfmm):
    """Without a CUDA device the product must raise, never fall back."""
    from tests.conftest import cuda_available
    if cuda_available():
        pytest.skip("a GPU is present")
    ps = blfmm.PointSet(2, np.random.default_rng(0).random((64, 2)))
    with pytest.raises(blfmm.CudaError):
        blfmm.Plan(ps, 3, blfmm.parse_kernel_spec("gaussian:c=16"), math.pi, 8)
