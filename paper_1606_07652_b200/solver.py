"""Krylov interpolation solve on the GPU matvec (first "next" row).

Mirrors ``solve_interpolation`` (/root/reference/proj/core/src/solver.cpp:243-300)
and its Krylov loops ``run_cg`` (43-88) and ``run_gmres`` (90-203): CG when the
kernel is positive definite, restarted GMRES(300) with Givens rotations
otherwise; the same backend rules (dense / single-level FMM / multilevel FMM,
sigma <= 0 -> pi, m <= 0 -> choose_truncation(N), leaf level from N), the same
stopping tests and the same errors (invalid_argument, accuracy_error with the
best residual). The plan (tree, grids, C table, expansion buffers) is built
once and reused by every iteration, and all Krylov vectors stay on the device.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _capi

from .api import (AccuracyError, InvalidArgument, KernelType, Plan, PointSet, RadialKernel,
                  choose_truncation, direct_matvec)


class Backend(enum.IntEnum):
    dense = 0
    single_fmm = 1
    mlfmm = 2


@dataclass
class InterpolationProblem:
    kernel: RadialKernel
    ps: PointSet | None = None
    rhs: np.ndarray = field(default_factory=lambda: np.zeros(0))
    backend: Backend = Backend.dense
    tol: float = 1e-10
    max_iter: int = 2000
    sigma: float = 0.0
    m_per_dim: int = 0
    leaf_level: int = 0


@dataclass
class SolveStats:
    iterations: int = 0
    residual: float = 0.0
    matvecs: int = 0
    method: str = ""
    converged: bool = False


def positive_definite(k: RadialKernel) -> bool:
    """kernels.cpp:334-337 (Gaussian, IMQ, Wendland)."""
    return k.type in (KernelType.Gaussian, KernelType.IMQ, KernelType.WendlandC2,
                      KernelType.Wendland31)


def run_cg(apply, b, tol: float, max_iter: int):
    """solver.cpp:43-88 on torch tensors (any device)."""
    import torch
    stats = SolveStats(method="cg")
    x = torch.zeros_like(b)
    bnorm = torch.linalg.vector_norm(b).item()
    if bnorm == 0.0:
        stats.converged = True
        return x, stats
    r = b.clone()
    p = b.clone()
    rr = torch.dot(r, r).item()
    best = math.sqrt(rr) / bnorm
    for it in range(max_iter):
        ap = apply(p)
        stats.matvecs += 1
        pap = torch.dot(p, ap).item()
        if pap <= 0.0:  # not PD to working precision
            break
        alpha = rr / pap
        x.add_(p, alpha=alpha)
        r.sub_(ap, alpha=alpha)
        rr_new = torch.dot(r, r).item()
        stats.iterations = it + 1
        rel = math.sqrt(rr_new) / bnorm
        best = min(best, rel)
        if rel <= tol:
            stats.residual = rel
            stats.converged = True
            return x, stats
        beta = rr_new / rr
        rr = rr_new
        p.mul_(beta).add_(r)
    stats.residual = best
    raise AccuracyError("cg did not reach tolerance", best)


def run_gmres(apply, b, tol: float, max_iter: int):
    """solver.cpp:90-203: restarted GMRES (restart 300), Givens rotations."""
    import torch
    stats = SolveStats(method="gmres")
    n = b.shape[0]
    x = torch.zeros_like(b)
    bnorm = torch.linalg.vector_norm(b).item()
    if bnorm == 0.0:
        stats.converged = True
        return x, stats
    restart = min(max_iter, 300)
    best = math.inf
    total_it = 0
    while total_it < max_iter:
        if total_it == 0:
            r = b.clone()
        else:
            r = b - apply(x)
            stats.matvecs += 1
        beta = torch.linalg.vector_norm(r).item()
        if beta / bnorm <= tol:
            stats.residual = beta / bnorm
            stats.converged = True
            return x, stats
        m = min(restart, max_iter - total_it)
        V = torch.zeros((m + 1, n), dtype=b.dtype, device=b.device)
        V[0] = r / beta
        H = np.zeros((m + 1, m + 1))  # H[k][j] = column k, row j (as the reference)
        cs, sn, g = [], [], [beta]
        k = 0
        while k < m:
            w = apply(V[k])
            stats.matvecs += 1
            # modified Gram-Schmidt, one projection at a time (as the reference)
            for j in range(k + 1):
                d = torch.dot(w, V[j])
                H[k][j] = d.item()
                w = w - d * V[j]
            wn = torch.linalg.vector_norm(w).item()
            H[k][k + 1] = wn
            breakdown = wn < 1e-14 * beta
            if not breakdown:
                V[k + 1] = w / wn
            for j in range(k):
                t = cs[j] * H[k][j] + sn[j] * H[k][j + 1]
                H[k][j + 1] = -sn[j] * H[k][j] + cs[j] * H[k][j + 1]
                H[k][j] = t
            denom = math.hypot(H[k][k], H[k][k + 1])
            cs.append(H[k][k] / denom)
            sn.append(H[k][k + 1] / denom)
            H[k][k] = denom
            H[k][k + 1] = 0.0
            g.append(-sn[k] * g[k])
            g[k] = cs[k] * g[k]
            total_it += 1
            stats.iterations = total_it
            rel = abs(g[k + 1]) / bnorm
            best = min(best, rel)
            k += 1
            if rel <= tol or breakdown:
                break
        y = np.zeros(k)
        for j in range(k - 1, -1, -1):
            s = g[j]
            for l in range(j + 1, k):
                s -= H[l][j] * y[l]
            y[j] = s / H[j][j]
        x = x + torch.mv(V[:k].T, torch.as_tensor(y, dtype=b.dtype, device=b.device))
        res = (torch.linalg.vector_norm(b - apply(x)).item()) / bnorm
        stats.matvecs += 1
        best = min(best, res)
        if res <= tol:
            stats.residual = res
            stats.converged = True
            return x, stats
    stats.residual = best
    raise AccuracyError("gmres did not reach tolerance", best)


def default_leaf_level(n: int, d: int, multilevel: bool) -> int:
    """Leaf level when the caller gives none. d <= 2: the reference's rules
    (multilevel lround(log2(n/32)), solver.cpp:280 / blfmm_cli.cpp:377-380;
    single level lround(log2(sqrt n))), kept for parity. d = 3 (no reference
    counterpart): the same targets counted in 8^L boxes - about 32 points per
    leaf (multilevel) or sqrt(n) leaves (single level) - clamped to the
    plan's d*L <= 24 box cap (geometry.cpp:266-267)."""
    if d <= 2:
        if multilevel:
            return max(3, _lround(math.log2(float(n) / 32.0)))
        return max(2, _lround(math.log2(math.sqrt(float(n)))))
    if multilevel:
        return min(8, max(3, _lround(math.log2(max(float(n) / 32.0, 1.0)) / 3.0)))
    return min(8, max(2, _lround(math.log2(max(float(n), 1.0)) / 6.0)))


def _lround(v: float) -> int:
    """std::lround: half away from zero (Python's round() is half-to-even)."""
    return int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))


def _device_apply(plan: Plan):
    """x -> A x on the device. The operand is staged into one persistent input
    buffer and the product lands in one persistent output buffer, so every
    iteration hands the plan the same device pointers and replays its captured
    CUDA graph; the caller gets a fresh tensor (a device copy)."""
    import ctypes as ct

    import torch
    stream = torch.cuda.current_stream()
    sp = ct.c_void_p(stream.cuda_stream)
    bufs = {}

    def apply(x):
        if "in" not in bufs or bufs["in"].shape != x.shape or bufs["in"].dtype != x.dtype:
            bufs["in"] = torch.empty_like(x, memory_format=torch.contiguous_format)
            bufs["out"] = torch.empty_like(bufs["in"])
        bufs["in"].copy_(x)
        plan.execute_device(bufs["in"].data_ptr(), bufs["out"].data_ptr(), stream=sp)
        return bufs["out"].clone()
    return apply


def solve_interpolation(prob: InterpolationProblem):
    """solver.cpp:243-300. Returns (lambda [numpy], SolveStats)."""
    if prob.ps is None:
        raise InvalidArgument("problem has no point set")
    ps = prob.ps
    n = ps.size()
    rhs = np.ascontiguousarray(prob.rhs, dtype=np.float64)
    if rhs.shape != (n,):
        raise InvalidArgument("rhs length != point count")
    if not prob.tol > 0.0:
        raise InvalidArgument("tol must be positive")
    sigma = prob.sigma if prob.sigma > 0.0 else math.pi
    m = prob.m_per_dim if prob.m_per_dim > 0 else choose_truncation(n)
    if prob.backend != Backend.dense:
        # the Krylov loop runs in the C++ library (blfmm_solve: device vectors,
        # the plan's matvec, deterministic reductions)
        multilevel = prob.backend == Backend.mlfmm
        level = prob.leaf_level if prob.leaf_level > 0 else default_leaf_level(n, ps.d, multilevel)
        plan = Plan(ps, level, prob.kernel, sigma, m)
        return solve_on_plan(plan, rhs, prob.tol, prob.max_iter, positive_definite(prob.kernel))
    # Backend.dense (the reference assembles the matrix with Eigen, solver.cpp:
    # 207-262): the same loops in the library on the matrix-free O(N^2) device
    # kernel (blfmm_solve_dense), every kernel type, N <= 8192
    return solve_dense(prob.kernel, ps, rhs, prob.tol, prob.max_iter)


def solve_dense(kernel, ps, rhs, tol: float, max_iter: int):
    """blfmm_solve_dense: CG / restarted GMRES on A_ij = phi(|x_i - x_j|)."""
    import ctypes as ct
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    coords = np.ascontiguousarray(ps.pts, dtype=np.float64)
    x = np.zeros_like(rhs)
    st = _capi.SolveStatsC()
    spd = positive_definite(kernel)
    dp = ct.POINTER(ct.c_double)
    rc = _capi.lib().blfmm_solve_dense(
        ps.d, ps.size(), coords.ctypes.data_as(dp), int(kernel.type), float(kernel.shape),
        _capi.SOLVE_CG if spd else _capi.SOLVE_GMRES, rhs.ctypes.data_as(dp),
        x.ctypes.data_as(dp), float(tol), int(max_iter), ct.byref(st), -1)
    stats = SolveStats(iterations=st.iterations, residual=st.residual, matvecs=st.matvecs,
                       method="cg" if st.method == _capi.SOLVE_CG else "gmres",
                       converged=bool(st.converged))
    _capi.check(rc)
    return x, stats


def solve_on_plan(plan: Plan, rhs, tol: float, max_iter: int, spd: bool):
    """blfmm_solve: CG (spd) or restarted GMRES on the plan's matvec, in the
    library. Returns (x, SolveStats); raises AccuracyError (best residual) when
    the tolerance is not reached, as the reference."""
    import ctypes as ct
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    x = np.zeros_like(rhs)
    st = _capi.SolveStatsC()
    rc = _capi.lib().blfmm_solve(plan.handle, _capi.SOLVE_CG if spd else _capi.SOLVE_GMRES,
                                 rhs.ctypes.data_as(ct.POINTER(ct.c_double)),
                                 x.ctypes.data_as(ct.POINTER(ct.c_double)), float(tol),
                                 int(max_iter), ct.byref(st))
    stats = SolveStats(iterations=st.iterations, residual=st.residual, matvecs=st.matvecs,
                       method="cg" if st.method == _capi.SOLVE_CG else "gmres",
                       converged=bool(st.converged))
    _capi.check(rc)
    return x, stats
