"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref, the
reference's own sources compiled with the repo's Boost.Math shim).

Run in the build container (needs /root/reference):
    make -C oracle && python tests/golden/make_golden.py
The fixtures are small and committed; the GPU box never reads /root/reference.
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as po  # noqa: E402
from paper_1606_07652_b200 import inputs as I  # noqa: E402


def mlfmm_fixture(name, x, w, spec, sigma, m, leaf, with_direct=False, mode=0, stencil=10):
    v, st = po.ref_mlfmm(x, w, spec, sigma, m, leaf, mode=mode, stencil=stencil)
    extra = {}
    if with_direct:
        dv, _ = po.ref_direct(x, w, spec)
        extra["direct"] = dv
    if mode == 1:  # the reference's own per-level C tables (LevelGrids::factors)
        extra["ctab"] = po.ref_level_c_tables(spec, sigma, m, x.shape[1], leaf, mode, stencil)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), kind="mlfmm", x=x, w=w, spec=spec,
                        sigma=sigma, m=m, leaf=leaf, values=v, near_pairs=st["near_pairs"],
                        far_work=st["far_work"], max_imag=st["max_imag_residual"],
                        grid_mode=mode, stencil_k=stencil, **extra)
    print(name, x.shape, st)


def bandlimited_fixture(name, cases):
    """Band-limited (fmm.cpp:57-70) and hybrid (fmm.cpp:77-113) O(N^2) oracles
    of the reference, d = 1: one npz holding every case (x_i, w_i, spec_i, ...)."""
    out = {}
    for i, (x, w, spec, sigma, refinement, leaf) in enumerate(cases):
        out[f"x_{i}"] = x
        out[f"w_{i}"] = w
        out[f"spec_{i}"] = spec
        out[f"sigma_{i}"] = sigma
        out[f"refinement_{i}"] = refinement
        out[f"leaf_{i}"] = leaf
        out[f"band_{i}"] = po.ref_direct_bl(x, w, spec, sigma, refinement)
        if leaf >= 2:
            out[f"hybrid_{i}"] = po.ref_direct_bl(x, w, spec, sigma, refinement, leaf)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), kind="bandlimited", ncases=len(cases),
                        **out)
    print(name, len(cases), "cases")


def bandlimited_main():
    cases = [
        # test_fmm.cpp:68-87 (band-limited table path)
        (I.generate_quasiuniform(16, 1, 8, 0.5), I.uniform_weights(16, 3), "gaussian:c=1",
         math.pi, 4096, -1),
        # test_fmm.cpp:89-107 (two points in leaf 0, two in leaf 3, level 2)
        (np.array([[0.05], [0.1], [0.9], [0.95]]), np.array([1.0, -2.0, 0.5, 1.5]), "imq:c=1",
         math.pi, 4096, 2),
        # test_fmm.cpp:131-152 (256-point IMQ fixture, 16 leaves)
        (I.generate_quasiuniform(256, 1, 2026, 0.35), I.uniform_weights(256, 99), "imq:c=1",
         math.pi, 4096, 4),
        # test_mlfmm.cpp:426-437 (1024-point fixture, 32 leaves)
        (I.generate_quasiuniform(1024, 1, 2026, 0.35), I.uniform_weights(1024, 99), "imq:c=1",
         math.pi, 4096, 5),
        # MQ (tail form) and a narrow Gaussian, uniform points
        (I.uniform_points(2048, 1, 71), I.uniform_weights(2048, 72), "mq:c=0.05", math.pi, 1024,
         6),
        (I.uniform_points(1500, 1, 73), I.uniform_weights(1500, 74), "gaussian:c=16", 20.0, 1024,
         5),
        # edge cases: a single point (r = 0 only), and points outside the domain
        # [0, 1] (clamped leaves, distances past rmax: the table's end interval)
        (np.array([[0.5]]), np.array([2.0]), "imq:c=1", math.pi, 1024, 2),
        (I.uniform_points(300, 1, 75) * 1.4 - 0.2, I.uniform_weights(300, 76), "imq:c=0.5",
         math.pi, 1024, 3),
    ]
    bandlimited_fixture("bandlimited_1d_ref", cases)


def main():
    assert po.ref_available(), "build oracle/_ref first (make -C oracle)"
    bandlimited_main()
    W = I.WORKLOADS["P1"]
    x, w = W.make()
    mlfmm_fixture("p1_gaussian_2d_ref", x, w, W.kernel, W.sigma, W.m, W.leaf, with_direct=True)
    W = I.WORKLOADS["P1b"]
    x, w = W.make()
    mlfmm_fixture("p1b_gaussian_2d_bandcapture_ref", x, w, W.kernel, W.sigma, W.m, W.leaf,
                  with_direct=True)
    W = I.WORKLOADS["P4"]
    x, w = W.make(8192)
    mlfmm_fixture("p4_mq_2d_small_ref", x, w, W.kernel, W.sigma, W.m, 4)
    x = I.generate_quasiuniform(256, 2, 77, 0.4)
    w = I.uniform_weights(256, 8)
    mlfmm_fixture("telescope_imq_2d_ref", x, w, "imq:c=1", math.pi, 12, 3)
    x = I.uniform_points(2048, 2, 31)
    w = I.uniform_weights(2048, 32)
    mlfmm_fixture("imq_2d_small_ref", x, w, "imq:c=0.1", math.pi, 16, 4)
    x = I.generate_quasiuniform(1024, 1, 2026, 0.35)
    w = I.uniform_weights(1024, 99)
    mlfmm_fixture("imq_1d_ref", x, w, "imq:c=1", math.pi, 64, 5)
    # GridMode::scaled (halved band per level, Lagrange transfers)
    x = I.generate_quasiuniform(512, 1, 55, 0.4)
    w = I.uniform_weights(512, 56)
    mlfmm_fixture("scaled_gaussian_1d_ref", x, w, "gaussian:c=1", math.pi, 16, 5, mode=1,
                  stencil=6)
    x = I.uniform_points(1024, 2, 61)
    w = I.uniform_weights(1024, 62)
    mlfmm_fixture("scaled_imq_2d_ref", x, w, "imq:c=1", math.pi, 12, 4, mode=1, stencil=10)
    x = I.uniform_points(600, 2, 63)
    w = I.uniform_weights(600, 64)
    mlfmm_fixture("scaled_mq_2d_global_stencil_ref", x, w, "mq:c=0.5", math.pi, 8, 3, mode=1,
                  stencil=8)


if __name__ == "__main__":
    main()
