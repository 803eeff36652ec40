"""Host-side mirror of the reference library's public interface.

Same names, argument meaning and error behaviour as blfmm's headers
(/root/reference/proj/core/include/blfmm/*.hpp); every numeric call goes
through the C ABI of include/blfmm_gpu.h into the sm_100a kernels. Extended
to d = 3 and to batched right-hand sides (weights of shape [nrhs, n]).

    reference                                   here
    parse_kernel_spec      kernels.hpp:23       parse_kernel_spec
    build_tree             geometry.hpp:72      build_tree (BoxTree helpers are
                                                 pure index arithmetic; the
                                                 point binning happens on the
                                                 GPU inside the plan)
    make_quadrature        bandlimit.hpp:35     make_quadrature
    translation_coefficients bandlimit.hpp:106  translation_coefficients
    make_level_grids       mlfmm.hpp:61-63      make_level_grids
    upsweep / couple       mlfmm.hpp:79-87      upsweep / couple (stage dumps)
    mlfmm_matvec           mlfmm.hpp:98-99      mlfmm_matvec
    fmm_matvec_single      fmm.hpp:55           fmm_matvec_single
    direct_matvec          fmm.hpp:33-36        direct_matvec
    choose_truncation      fmm.hpp:47           choose_truncation
"""
from __future__ import annotations

import ctypes as ct
import enum
import math
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import (AccuracyError, BlfmmError, CudaError, DomainError,  # noqa: F401
                    InvalidArgument, LengthError)

_dp = ct.POINTER(ct.c_double)


def _ptr(a):
    return a.ctypes.data_as(_dp)


class KernelType(enum.IntEnum):
    Gaussian = 0
    MQ = 1
    IMQ = 2
    TPS = 3
    WendlandC2 = 4
    Wendland31 = 5


@dataclass(frozen=True)
class RadialKernel:
    type: KernelType = KernelType.Gaussian
    shape: float = 1.0


def parse_kernel_spec(spec: str) -> RadialKernel:
    """kernels.cpp:48-103 grammar: ``name[:key=value]``, case-insensitive."""
    t, s = ct.c_int(), ct.c_double()
    _capi.check(_capi.lib().blfmm_parse_kernel_spec(spec.encode(), ct.byref(t), ct.byref(s)))
    return RadialKernel(KernelType(t.value), s.value)


def kernel_name(k: RadialKernel) -> str:
    key = {KernelType.Gaussian: "gaussian:c=", KernelType.MQ: "mq:c=", KernelType.IMQ: "imq:c=",
           KernelType.TPS: "tps:beta=", KernelType.WendlandC2: "wendland:eps=",
           KernelType.Wendland31: "wendland31:eps="}[k.type]
    return f"{key}{k.shape:g}"


def eval_kernel(k: RadialKernel, r):
    """phi(r) (kernels.cpp:131-161), vectorised numpy (host helper)."""
    r = np.abs(np.asarray(r, dtype=np.float64))
    c = k.shape
    if k.type == KernelType.Gaussian:
        return np.exp(-c * r * r)
    if k.type == KernelType.MQ:
        return np.sqrt(r * r + c * c)
    if k.type == KernelType.IMQ:
        return 1.0 / np.sqrt(r * r + c * c)
    raise DomainError("kernel not supported by the GPU band-limited FMM (gaussian, mq, imq)")


@dataclass
class BoundingBox:
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)

    def side(self, dim: int) -> float:
        return self.hi[dim] - self.lo[dim]


class PointSet:
    """geometry.hpp:17-23 (d <= 3 here); pts is an [n, d] float64 array."""

    def __init__(self, d: int = 1, pts=None, domain: BoundingBox | None = None):
        self.d = int(d)
        self.domain = domain if domain is not None else BoundingBox()
        pts = np.zeros((0, self.d)) if pts is None else np.asarray(pts, dtype=np.float64)
        if pts.ndim == 1:
            pts = pts.reshape(-1, 1)
        self.pts = np.ascontiguousarray(pts)

    def size(self) -> int:
        return int(self.pts.shape[0])


class BoxTree:
    """Uniform 2^d-ary tree to ``leaf_level`` (geometry.hpp:49-69). Box ids are
    row-major over per-axis indices. Neighbor / interaction lists and the leaf
    binning are materialised on the GPU inside the plan; the methods here are
    the reference's pure index arithmetic."""

    def __init__(self, ps: PointSet, leaf_level: int):
        self.d = ps.d
        self.leaf_level = leaf_level
        self.domain = ps.domain
        self._ps = ps

    def boxes_per_dim(self, level: int) -> int:
        return 1 << level

    def box_count(self, level: int) -> int:
        return 1 << (self.d * level)

    def side(self, level: int, dim: int) -> float:
        return self.domain.side(dim) / self.boxes_per_dim(level)

    def _idx(self, level, box):
        n = 1 << level
        out = []
        for _ in range(self.d):
            out.append(box % n)
            box //= n
        return out[::-1]

    def _id(self, level, idx):
        b = 0
        for i in idx:
            b = (b << level) | int(i)
        return b

    def center(self, level: int, box: int):
        idx = self._idx(level, box)
        return tuple(self.domain.lo[k] + (idx[k] + 0.5) * self.side(level, k)
                     for k in range(self.d))

    def parent(self, level: int, box: int) -> int:
        return self._id(level - 1, [i // 2 for i in self._idx(level, box)])

    def children(self, level: int, box: int):
        if level >= self.leaf_level:
            return []
        idx = self._idx(level, box)
        out = []
        for q in range(1 << self.d):
            c = [2 * idx[k] + ((q >> (self.d - 1 - k)) & 1) for k in range(self.d)]
            out.append(self._id(level + 1, c))
        return out

    def leaf_of(self, x) -> int:
        n = 1 << self.leaf_level
        idx = []
        for k in range(self.d):
            v = int((x[k] - self.domain.lo[k]) / self.side(self.leaf_level, k))
            idx.append(min(max(v, 0), n - 1))
        return self._id(self.leaf_level, idx)


def build_tree(ps: PointSet, leaf_level: int) -> BoxTree:
    if leaf_level < 2:
        raise InvalidArgument("leaf_level must be >= 2")
    if ps.d * leaf_level > 24:
        raise InvalidArgument("box count cap exceeded")
    return BoxTree(ps, leaf_level)


class GridMode(enum.IntEnum):
    shared = 0
    scaled = 1


@dataclass
class QuadratureGrid:
    sigma: float = 0.0
    m_per_dim: int = 0
    d: int = 1
    nodes: np.ndarray = field(default_factory=lambda: np.zeros((0, 1)))
    weights: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def node_count(self) -> int:
        return int(self.nodes.shape[0])

    def dxi(self) -> float:
        return 2.0 * self.sigma / self.m_per_dim


def make_quadrature(sigma: float, m_per_dim: int, d: int) -> QuadratureGrid:
    """bandlimit.cpp:269-292: xi = -sigma + m dxi, row-major tensor nodes."""
    if not sigma > 0.0:
        raise InvalidArgument("sigma must be positive")
    if m_per_dim < 2:
        raise InvalidArgument("m_per_dim must be >= 2")
    if d not in (1, 2, 3):
        raise InvalidArgument("d must be 1, 2 or 3")
    dxi = 2.0 * sigma / m_per_dim
    ax = -sigma + np.arange(m_per_dim) * dxi
    mesh = np.meshgrid(*([ax] * d), indexing="ij")
    nodes = np.stack([g.reshape(-1) for g in mesh], axis=1)
    w = dxi if d == 1 else (dxi * dxi if d == 2 else dxi * dxi * dxi)
    return QuadratureGrid(sigma, m_per_dim, d, nodes, np.full(nodes.shape[0], w))


@dataclass
class LowRankFactors:
    grid: QuadratureGrid
    c_vals: np.ndarray
    q_terms: int = 0
    regularized: list = field(default_factory=list)


def translation_coefficients(k: RadialKernel, grid: QuadratureGrid,
                             mode: str = "spectral") -> LowRankFactors:
    """Spectral-mode translation spectrum C(xi_m) (bandlimit.cpp:388-447)."""
    if mode != "spectral":
        raise DomainError("only spectral translation is provided by the GPU backend")
    c = np.empty(grid.node_count())
    _capi.check(_capi.lib().blfmm_translation_coefficients(
        grid.d, int(k.type), k.shape, grid.sigma, grid.m_per_dim, _ptr(c)))
    reg = list(range(grid.node_count())) if k.type != KernelType.Gaussian else []
    return LowRankFactors(grid, c, 0, reg)


@dataclass
class LevelGrids:
    mode: GridMode = GridMode.shared
    d: int = 1
    leaf_level: int = 2
    stencil_k: int = 10
    kernel: RadialKernel = field(default_factory=RadialKernel)
    grids: list = field(default_factory=list)
    factors: list = field(default_factory=list)
    interp: list = field(default_factory=list)


def rescale_grid(grid: QuadratureGrid, s: float) -> QuadratureGrid:
    """bandlimit.cpp:294-305: nodes / s, weights / s^d (sum w = (2 sigma/s)^d)."""
    if not s > 0.0:
        raise InvalidArgument("s must be positive")
    return QuadratureGrid(grid.sigma / s, grid.m_per_dim, grid.d, grid.nodes / s,
                          grid.weights / s ** grid.d)


def make_level_grids(kernel: RadialKernel, sigma_leaf: float, m_leaf: int, d: int,
                     leaf_level: int, mode: GridMode = GridMode.shared,
                     stencil_k: int = 10) -> LevelGrids:
    """mlfmm.cpp:112-142. Shared mode: every level reuses the leaf grid and C.
    Scaled mode: sigma_{l-1} = sigma_l / 2 and one C table per level; the GPU
    plan builds the Lagrange transfers itself (stencil_k)."""
    if leaf_level < 2:
        raise InvalidArgument("leaf_level must be >= 2")
    g = make_quadrature(sigma_leaf, m_leaf, d)
    grids = [None] * (leaf_level + 1)
    factors = [None] * (leaf_level + 1)
    grids[leaf_level] = g
    for l in range(leaf_level - 1, 1, -1):
        grids[l] = grids[l + 1] if mode == GridMode.shared else rescale_grid(grids[l + 1], 2.0)
    f = translation_coefficients(kernel, g)
    for l in range(2, leaf_level + 1):
        factors[l] = f if mode == GridMode.shared else translation_coefficients(kernel, grids[l])
    return LevelGrids(mode, d, leaf_level, min(stencil_k, m_leaf), kernel, grids, factors)


@dataclass
class SumStats:
    near_pairs: int = 0
    far_work: int = 0
    max_imag_residual: float = 0.0


@dataclass
class SumResult:
    values: np.ndarray
    stats: SumStats


@dataclass
class SumRequest:
    kernel: RadialKernel
    sigma: float
    ps: PointSet | None
    weights: np.ndarray
    m_per_dim: int


def choose_truncation(n: int) -> int:
    """fmm.cpp:115-121: ceil(sqrt(n)) rounded up to even."""
    if n < 4:
        raise InvalidArgument("n must be >= 4")
    m = int(math.ceil(math.sqrt(float(n))))
    return m + (m % 2)


# ------------------------------------------------------------------ plans
class Plan:
    """Owns a device-resident blfmm_plan (sorted points, tree, C table and the
    expansion sets). Build once, execute many times (the solver pattern,
    solver.cpp:280-293)."""

    def __init__(self, ps: PointSet, leaf_level: int, kernel: RadialKernel, sigma: float,
                 m_per_dim: int, c_table: np.ndarray | None = None, nrhs: int = 1,
                 device: int = -1, rank: int = 0, world: int = 1, grid_mode: int = 0,
                 stencil_k: int = 10, tuning: dict | None = None):
        self._h = ct.c_void_p()
        self._keep = []
        d = ps.d
        desc = _capi.PlanDesc()
        desc.d = d
        desc.n = ps.size()
        coords = np.ascontiguousarray(ps.pts, dtype=np.float64)
        self._keep.append(coords)
        desc.coords = _ptr(coords)
        for k in range(3):
            desc.domain_lo[k] = ps.domain.lo[k] if k < d else 0.0
            desc.domain_hi[k] = ps.domain.hi[k] if k < d else 1.0
        desc.kernel_type = int(kernel.type)
        desc.kernel_shape = kernel.shape
        desc.sigma = sigma
        desc.m_per_dim = m_per_dim
        desc.leaf_level = leaf_level
        desc.grid_mode = int(grid_mode)
        desc.stencil_k = int(stencil_k)
        desc.nrhs = nrhs
        desc.device = device
        if c_table is not None:
            ctab = np.ascontiguousarray(c_table, dtype=np.float64)
            self._keep.append(ctab)
            desc.c_table = _ptr(ctab)
        desc.rank = rank
        desc.world = world
        tune = _capi.Tuning()
        _capi.lib().blfmm_tuning_defaults(ct.byref(tune))
        for k, v in (tuning or {}).items():
            if not hasattr(tune, k):
                raise InvalidArgument(f"unknown tuning field {k!r}")
            setattr(tune, k, int(v))
        _capi.check(_capi.lib().blfmm_plan_create_tuned(ct.byref(desc), ct.byref(tune),
                                                        ct.byref(self._h)))
        self.n, self.d, self.nrhs = ps.size(), d, nrhs
        self.K = m_per_dim ** d
        self.leaf_level = leaf_level
        self._fin = weakref.finalize(self, _capi.lib().blfmm_plan_destroy, self._h)

    @property
    def handle(self):
        return self._h

    def info(self) -> _capi.PlanInfo:
        inf = _capi.PlanInfo()
        _capi.check(_capi.lib().blfmm_plan_get_info(self._h, ct.byref(inf)))
        return inf

    def kernels(self) -> dict:
        """Stage -> kernel that blfmm_execute launches (blfmm_plan_info.kernels)."""
        out = {}
        for tok in self.info().kernels.decode().split():
            k, _, v = tok.partition("=")
            out[k] = v
        return out

    def _weights(self, weights):
        w = np.ascontiguousarray(weights, dtype=np.float64)
        if w.ndim == 1:
            w = w.reshape(1, -1)
        if w.shape != (self.nrhs, self.n):
            raise InvalidArgument("weight count != point count")
        return w

    def execute(self, weights, single: bool = False, stream=None) -> SumResult:
        w = self._weights(weights)
        out = np.empty_like(w)
        st = _capi.Stats()
        fn = _capi.lib().blfmm_execute_single if single else _capi.lib().blfmm_execute
        _capi.check(fn(self._h, _ptr(w), _ptr(out), ct.byref(st), stream))
        vals = out[0] if np.ndim(weights) == 1 else out
        return SumResult(vals, SumStats(st.near_pairs, st.far_work, st.max_imag_residual))

    def execute_device(self, d_lambda: int, d_out: int, stream=None, stats: bool = False):
        st = _capi.Stats() if stats else None
        _capi.check(_capi.lib().blfmm_execute_device(
            self._h, ct.c_void_p(d_lambda), ct.c_void_p(d_out),
            ct.byref(st) if st is not None else None, stream))
        if st is not None:
            return SumStats(st.near_pairs, st.far_work, st.max_imag_residual)
        return None

    # ---- multi-GPU exchange mode (blfmm_execute_upsweep / _downsweep)
    def attach_nccl(self, unique_id: bytes):
        """Attach an NCCL communicator (rank / world of this plan): execute
        then runs the whole sharded matvec and returns u on every rank."""
        if len(unique_id) != _capi.NCCL_ID_BYTES:
            raise InvalidArgument("NCCL unique id must be 128 bytes")
        _capi.check(_capi.lib().blfmm_plan_attach_nccl(self._h, unique_id))

    def attach_comm(self, all_reduce_sum, all_reduce_max, broadcast):
        """Attach caller collectives: all_reduce_sum(dptr, count, stream),
        all_reduce_max(dptr, count, stream), broadcast(dptr, count, root,
        stream), each on a device buffer of float64, returning None."""
        def wrap(f):
            def cb(_ctx, *a):
                try:
                    f(*a)
                    return 0
                except Exception:  # noqa: BLE001 - reported as BLFMM_ENCCL
                    import traceback
                    traceback.print_exc()
                    return 1
            return cb
        self._ops = _capi.CommOps(None, _capi.SUM_FN(wrap(all_reduce_sum)),
                                  _capi.SUM_FN(wrap(all_reduce_max)),
                                  _capi.BCAST_FN(wrap(broadcast)))
        _capi.check(_capi.lib().blfmm_plan_attach_comm(self._h, ct.byref(self._ops)))

    def exchange_size(self) -> int:
        """Doubles in the exchange buffer (0: no exchange mode)."""
        v = ct.c_longlong()
        _capi.check(_capi.lib().blfmm_plan_exchange_size(self._h, ct.byref(v)))
        return v.value

    def bind_exchange(self, d_buffer: int):
        _capi.check(_capi.lib().blfmm_plan_bind_exchange(self._h, ct.c_void_p(d_buffer)))

    def upsweep(self, d_lambda: int, stream=None):
        _capi.check(_capi.lib().blfmm_execute_upsweep(self._h, ct.c_void_p(d_lambda), stream))

    def downsweep(self, d_out: int, stream=None, stats: bool = False):
        st = _capi.Stats() if stats else None
        _capi.check(_capi.lib().blfmm_execute_downsweep(
            self._h, ct.c_void_p(d_out), ct.byref(st) if st is not None else None, stream))
        if st is not None:
            return SumStats(st.near_pairs, st.far_work, st.max_imag_residual)
        return None

    def set_profiling(self, on: bool = True):
        _capi.check(_capi.lib().blfmm_set_profiling(self._h, int(on)))

    def set_keep_couple(self, on: bool = True):
        _capi.check(_capi.lib().blfmm_set_keep_couple(self._h, int(on)))

    def stage_times(self):
        t = _capi.StageTimes()
        _capi.check(_capi.lib().blfmm_get_stage_times(self._h, ct.byref(t)))
        return {n: (t.ms[i], t.launches[i]) for i, n in enumerate(_capi.STAGE_NAMES)}

    def expansions(self, level: int, kind: int, rhs: int = 0) -> np.ndarray:
        """Dense [box_count(level), K] complex, reference box-id order."""
        cnt = 1 << (self.d * level)
        out = np.empty(cnt * self.K * 2)
        _capi.check(_capi.lib().blfmm_get_expansions(self._h, level, kind, rhs, _ptr(out)))
        z = out.reshape(cnt, self.K, 2)
        return z[..., 0] + 1j * z[..., 1]


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0; broadcast it to the others)."""
    buf = ct.create_string_buffer(_capi.NCCL_ID_BYTES)
    _capi.check(_capi.lib().blfmm_nccl_get_unique_id(buf))
    return buf.raw


def _plan_for(req: SumRequest, tree: BoxTree, grids: LevelGrids, nrhs: int) -> Plan:
    """The device plan of (point set, tree, grids), reused across matvecs (the
    solver pattern, solver.cpp:280-293). The reference recomputes from
    req.ps on every call, so a cached plan is only returned when the FULL
    coordinate array equals the copy the plan was built from (coordinates
    edited in place, or a new array at a recycled id, rebuild the plan)."""
    ps = req.ps
    cache = grids.__dict__.setdefault("_plans", {})
    pts = np.ascontiguousarray(np.asarray(ps.pts, dtype=np.float64))
    key = (pts.shape, tree.leaf_level, nrhs, req.kernel,
           tuple(ps.domain.lo), tuple(ps.domain.hi))
    hit = cache.get(key)
    if hit is not None and np.array_equal(hit[0], pts):
        return hit[1]
    g = grids.grids[tree.leaf_level]
    if grids.mode == GridMode.scaled:
        ctab = np.concatenate([grids.factors[l].c_vals
                               for l in range(2, tree.leaf_level + 1)])
    else:
        ctab = grids.factors[tree.leaf_level].c_vals
    plan = Plan(ps, tree.leaf_level, req.kernel, g.sigma, g.m_per_dim, c_table=ctab,
                nrhs=nrhs, grid_mode=int(grids.mode), stencil_k=grids.stencil_k)
    cache.clear()
    cache[key] = (pts.copy(), plan)
    return plan


def _check_request(req: SumRequest):
    if req.ps is None:
        raise InvalidArgument("request has no point set")
    w = np.asarray(req.weights)
    if w.shape[-1] != req.ps.size():
        raise InvalidArgument("weight count != point count")
    return 1 if w.ndim == 1 else w.shape[0]


def mlfmm_matvec(req: SumRequest, tree: BoxTree, grids: LevelGrids) -> SumResult:
    """mlfmm.cpp:361-406 on the GPU. values = far (downsweep) + near field."""
    nrhs = _check_request(req)
    if grids.d != req.ps.d or grids.leaf_level != tree.leaf_level:
        raise InvalidArgument("grids incompatible with tree/points")
    return _plan_for(req, tree, grids, nrhs).execute(req.weights)


def fmm_matvec_single(req: SumRequest, tree: BoxTree) -> SumResult:
    """fmm.cpp:123-213 semantics: single-level sum over every non-neighbor
    leaf pair. With a shared grid the multilevel sweep equals it to rounding
    (mlfmm.hpp:17-20), so the GPU runs the sweep and reports the single-level
    far_work count."""
    nrhs = _check_request(req)
    if not req.sigma > 0.0:
        raise InvalidArgument("sigma must be > 0")
    if req.m_per_dim < 2:
        raise InvalidArgument("m_per_dim must be >= 2")
    grids = make_level_grids(req.kernel, req.sigma, req.m_per_dim, req.ps.d, tree.leaf_level)
    return _plan_for(req, tree, grids, nrhs).execute(req.weights, single=True)


def direct_matvec(k: RadialKernel, ps: PointSet, weights, use_bandlimited: bool = False,
                  sigma: float = 0.0, refinement: int = 1024,
                  targets=None) -> SumResult:
    """fmm.cpp:30-75 plain-kernel O(N^2) sum on the GPU (independent check).
    ``targets`` (extension) restricts the output to those point indices."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    n = ps.size()
    if w.shape != (n,):
        raise InvalidArgument("weights length != point count")
    if use_bandlimited:
        return _direct_bandlimited(k, ps, w, sigma, refinement, -1)
    coords = np.ascontiguousarray(ps.pts, dtype=np.float64)
    tg = None if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    nt = n if tg is None else tg.shape[0]
    out = np.zeros(nt)
    _capi.check(_capi.lib().blfmm_direct(
        ps.d, n, _ptr(coords), int(k.type), k.shape, _ptr(w), nt,
        None if tg is None else tg.ctypes.data_as(ct.POINTER(ct.c_longlong)),
        _ptr(out), -1))
    return SumResult(out, SumStats(n * n if tg is None else n * nt, 0, 0.0))


def _direct_bandlimited(k: RadialKernel, ps: PointSet, w, sigma, refinement, leaf_level):
    n = ps.size()
    coords = np.ascontiguousarray(ps.pts, dtype=np.float64)
    lo = np.ascontiguousarray(ps.domain.lo[:ps.d], dtype=np.float64)
    hi = np.ascontiguousarray(ps.domain.hi[:ps.d], dtype=np.float64)
    out = np.zeros(n)
    _capi.check(_capi.lib().blfmm_direct_bandlimited(
        ps.d, n, _ptr(coords), _ptr(lo), _ptr(hi), int(k.type), k.shape, _ptr(w),
        float(sigma), int(refinement), int(leaf_level), _ptr(out), -1))
    return SumResult(out, SumStats(n * n, 0, 0.0))


def direct_matvec_hybrid(k: RadialKernel, ps: PointSet, tree: BoxTree, weights,
                         sigma: float, refinement: int = 1024) -> SumResult:
    """fmm.cpp:77-113 on the GPU: the original kernel inside the target leaf's
    neighbour block, Phi_sigma (radial table) outside it; d = 1 only."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    if w.shape != (ps.size(),):
        raise InvalidArgument("weights length != point count")
    if ps.d != 1:
        raise DomainError("hybrid direct oracle is 1d only")
    return _direct_bandlimited(k, ps, w, sigma, refinement, tree.leaf_level)


def eval_bandlimited(k: RadialKernel, sigma: float, x, d: int = 1,
                     refinement: int = 2048) -> float:
    """bandlimit.cpp:307-334, d = 1 (host plan-time math of the library)."""
    out = ct.c_double()
    x0 = float(x[0]) if np.ndim(x) else float(x)
    _capi.check(_capi.lib().blfmm_eval_bandlimited(int(d), int(k.type), k.shape, float(sigma),
                                                   x0, int(refinement), ct.byref(out)))
    return out.value


def bandlimited_radial_table(k: RadialKernel, sigma: float, rmax: float,
                             refinement: int = 1024):
    """bandlimit.cpp:241-262: (step, 1027 samples of Phi_sigma on [0, rmax + 2 step])."""
    vals = np.zeros(1027)
    step = ct.c_double()
    _capi.check(_capi.lib().blfmm_bandlimited_radial_table(
        int(k.type), k.shape, float(sigma), float(rmax), int(refinement), _ptr(vals),
        ct.byref(step)))
    return step.value, vals


def upsweep(tree: BoxTree, grids: LevelGrids, ps: PointSet, weights):
    """Multipole expansions per level (mlfmm.cpp:201-266): list indexed by
    level, dense [box_count, K] complex arrays (levels 0, 1 are None)."""
    req = SumRequest(grids.kernel, grids.grids[tree.leaf_level].sigma, ps, weights,
                     grids.grids[tree.leaf_level].m_per_dim)
    _check_request(req)
    plan = _plan_for(req, tree, grids, 1)
    plan.execute(weights)
    return [None, None] + [plan.expansions(l, 0) for l in range(2, tree.leaf_level + 1)]


def couple(tree: BoxTree, grids: LevelGrids, ps: PointSet, weights):
    """Local expansions from the M2L step alone (mlfmm.cpp:268-299), before
    L2L, per level. Takes the weights (the multipoles are device-resident)."""
    req = SumRequest(grids.kernel, grids.grids[tree.leaf_level].sigma, ps, weights,
                     grids.grids[tree.leaf_level].m_per_dim)
    _check_request(req)
    plan = _plan_for(req, tree, grids, 1)
    plan.set_keep_couple(True)
    plan.execute(weights)
    return [None, None] + [plan.expansions(l, 1) for l in range(2, tree.leaf_level + 1)]
