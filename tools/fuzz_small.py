"""Seeded sweep of small configurations (dimension, nodes per axis, leaf level,
point count, kernel, right-hand sides, point distribution) through the GPU
matvec against the CPU oracle: a robustness check of the kernel-selection
boundaries (M = 16 / even M <= 64 / odd / large M, 1..3 dimensions, tiny and
empty leaves). Prints one line per case; exit code = number of failures.
usage: fuzz_small.py [ncases] [seed]"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1606_07652_b200 as B  # noqa: E402
from oracle import pyoracle  # noqa: E402


def cases(ncases, seed):
    rng = np.random.default_rng(seed)
    ms = {1: [2, 3, 8, 16, 17, 64, 300, 2048, 20000], 2: [2, 5, 8, 15, 16, 17, 20, 33, 64, 100],
          3: [2, 3, 6, 8, 15, 16, 17, 18, 20, 31, 34]}
    for _ in range(ncases):
        d = int(rng.integers(1, 4))
        m = int(rng.choice(ms[d]))
        leaf = int(rng.integers(2, 5 if d < 3 else 4))
        n = int(rng.choice([1, 7, 60, 700, 3000]))
        spec = str(rng.choice(["gaussian:c=9", "imq:c=0.3", "mq:c=0.2"]))
        nrhs = int(rng.choice([1, 1, 1, 2, 8]))
        dist = str(rng.choice(["uniform", "cluster", "edge"]))
        yield d, m, leaf, n, spec, nrhs, dist, int(rng.integers(1 << 30))


def points(d, n, dist, seed):
    rng = np.random.default_rng(seed)
    if dist == "uniform":
        x = rng.random((n, d))
    elif dist == "cluster":
        x = np.clip(0.5 + 0.03 * rng.standard_normal((n, d)), 0.0, 1.0)
    else:  # points on the domain faces and corners (clamp binning)
        x = rng.random((n, d))
        x[rng.random((n, d)) < 0.3] = 1.0
        x[rng.random((n, d)) < 0.1] = 0.0
    return x


def mode_cases(ncases, seed):
    """Second sweep: API modes on top of the geometry - scaled grids (M^d <= 6400),
    the single-level sum, a non-unit domain with points outside it (clamp
    binning), odd / DMMA-sized right-hand-side counts, the stats-free device call."""
    rng = np.random.default_rng(seed)
    ms = {1: [4, 8, 16, 33, 64], 2: [4, 8, 16, 17, 20, 64], 3: [4, 6, 8, 16, 18]}
    for _ in range(ncases):
        d = int(rng.integers(1, 4))
        m = int(rng.choice(ms[d]))
        leaf = int(rng.integers(2, 5 if d < 3 else 4))
        n = int(rng.choice([5, 90, 1200]))
        spec = str(rng.choice(["gaussian:c=9", "imq:c=0.3", "mq:c=0.2"]))
        mode = str(rng.choice(["scaled", "single", "domain", "rhs", "device"]))
        yield d, m, leaf, n, spec, mode, int(rng.integers(1 << 30))


def run_mode_case(d, m, leaf, n, spec, mode, s):
    import torch
    rng = np.random.default_rng(s)
    x = rng.random((n, d))
    k = B.parse_kernel_spec(spec)
    lo = hi = None
    nrhs, grid_mode, stencil = 1, 0, 10
    if mode == "domain":
        lo, hi = np.full(d, -0.5), np.full(d, 1.75)
        x = -0.7 + 2.8 * x  # some points outside the box: clamped into edge leaves
    if mode == "rhs":
        nrhs = int(rng.choice([3, 5, 16, 32]))
    if mode == "scaled":
        if m ** d > 6400 or m % 2:
            m = 8
        grid_mode, stencil = 1, int(rng.integers(3, min(m, 10) + 1))
    w = rng.uniform(-1, 1, (nrhs, n) if nrhs > 1 else n)
    lo3 = None if lo is None else tuple(lo) + (0.0,) * (3 - d)
    hi3 = None if hi is None else tuple(hi) + (1.0,) * (3 - d)
    dom = B.BoundingBox(lo3 or (0.0,) * 3, hi3 or (1.0,) * 3)
    plan = B.Plan(B.PointSet(d, x, dom), leaf, k, math.pi, m, nrhs=nrhs, grid_mode=grid_mode,
                  stencil_k=stencil)
    if mode == "single":
        res = plan.execute(w, single=True)
        ctab = B.translation_coefficients(k, B.make_quadrature(math.pi, m, d)).c_vals
        ov, ost = pyoracle.single(x, w, spec, math.pi, m, leaf, c_table_in=ctab)
    else:
        res = plan.execute(w)
        if grid_mode:
            ov, ost, _ = pyoracle.mlfmm(x, w, spec, math.pi, m, leaf, lo, hi, mode=1,
                                        stencil=stencil)
        else:
            ctab = B.translation_coefficients(k, B.make_quadrature(math.pi, m, d)).c_vals
            ov, ost, _ = pyoracle.mlfmm(x, w, spec, math.pi, m, leaf, lo, hi, c_table_in=ctab)
    v = np.asarray(res.values).reshape(nrhs, n)
    if mode == "device":  # the stats-free device call (graph capture on the second use)
        lam = torch.from_numpy(np.ascontiguousarray(np.asarray(w).reshape(nrhs, n))).cuda()
        out = torch.empty_like(lam)
        for _ in range(3):
            plan.execute_device(lam.data_ptr(), out.data_ptr(), stats=False)
        torch.cuda.synchronize()
        v = out.cpu().numpy()
    ov = np.asarray(ov).reshape(nrhs, n)
    err = max(np.linalg.norm(v[r] - ov[r]) / max(np.linalg.norm(ov[r]), 1e-300)
              for r in range(nrhs))
    tol = 1e-10
    ok = err <= tol and res.stats.near_pairs == ost["near_pairs"] and \
        res.stats.far_work == ost["far_work"]
    return ok, err


def main():
    ncases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    fails = 0
    for d, m, leaf, n, spec, nrhs, dist, s in cases(ncases, seed):
        tag = f"d={d} M={m} L={leaf} n={n} {spec} nrhs={nrhs} {dist}"
        try:
            x = points(d, n, dist, s)
            w = np.random.default_rng(s + 1).uniform(-1, 1, (nrhs, n) if nrhs > 1 else n)
            k = B.parse_kernel_spec(spec)
            plan = B.Plan(B.PointSet(d, x), leaf, k, math.pi, m, nrhs=nrhs)
            res = plan.execute(w)
            ctab = B.translation_coefficients(k, B.make_quadrature(math.pi, m, d)).c_vals
            ov, ost, _ = pyoracle.mlfmm(x, w, spec, math.pi, m, leaf, c_table_in=ctab)
            v = np.asarray(res.values).reshape(nrhs, n)
            ov = np.asarray(ov).reshape(nrhs, n)
            err = max(np.linalg.norm(v[r] - ov[r]) / max(np.linalg.norm(ov[r]), 1e-300)
                      for r in range(nrhs))
            ok = err <= 1e-10 and res.stats.near_pairs == ost["near_pairs"] and \
                res.stats.far_work == ost["far_work"]
            print(("ok   " if ok else "FAIL ") + tag + f" rel-l2 {err:.2e} kernels {plan.kernels()['p2m']}/"
                  f"{plan.kernels()['l2p']}", flush=True)
            fails += 0 if ok else 1
        except Exception as e:  # noqa: BLE001
            print("FAIL " + tag + f" {type(e).__name__}: {str(e)[:160]}", flush=True)
            fails += 1
    for d, m, leaf, n, spec, mode, s in mode_cases(ncases, seed + 1000):
        tag = f"mode={mode} d={d} M={m} L={leaf} n={n} {spec}"
        try:
            ok, err = run_mode_case(d, m, leaf, n, spec, mode, s)
            print(("ok   " if ok else "FAIL ") + tag + f" rel-l2 {err:.2e}", flush=True)
            fails += 0 if ok else 1
        except Exception as e:  # noqa: BLE001
            print("FAIL " + tag + f" {type(e).__name__}: {str(e)[:160]}", flush=True)
            fails += 1
    print(f"{fails} failures of {2 * ncases}")
    return fails


if __name__ == "__main__":
    sys.exit(min(main(), 100))
