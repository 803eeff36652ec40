"""Multi-GPU (one process per GPU) band-limited FMM matvec.

Sharding: the leaves, sorted by Morton key, are split into
`world` contiguous ranges of equal estimated cost (blfmm_partition; the same
deterministic split on every rank). Each rank's plan builds the full tree,
runs the upsweep, and evaluates the downsweep (couple / L2L / L2P) and the
near field for its own range only, writing zeros elsewhere. The exchange is
one all-reduce(sum) of the output vector over NCCL (NVLink) — the ranks'
supports are disjoint, so the sum is the matvec bit for bit.

Round-1 scope: the upsweep (P2M + M2M) is replicated on every rank instead
of exchanging leaf / coarse-level multipoles (the halo + coarse all-reduce
design is the next step).
"""
from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _capi
from .api import InvalidArgument, Plan, PointSet, RadialKernel


def leaf_cost(npts: np.ndarray, nsrc: np.ndarray, K: int) -> np.ndarray:
    """Per-leaf cost model used by the plan (blfmm.cu, plan_build_tree):
    near pairs x 20 + points x 2K (P2M/L2P) + 100 K (translations)."""
    npts = np.asarray(npts, dtype=np.float64)
    return 20.0 * npts * np.asarray(nsrc, dtype=np.float64) + 2.0 * npts * K + 100.0 * K


def partition(cost: np.ndarray, world: int) -> np.ndarray:
    """Contiguous equal-cost split of a cost vector: bounds[0..world]."""
    cost = np.ascontiguousarray(cost, dtype=np.float64)
    if world < 1:
        raise InvalidArgument("world must be >= 1")
    bounds = np.zeros(world + 1, dtype=np.int64)
    _capi.check(_capi.lib().blfmm_partition(
        cost.ctypes.data_as(ct.POINTER(ct.c_double)), cost.shape[0], world,
        bounds.ctypes.data_as(ct.POINTER(ct.c_longlong))))
    return bounds


def assemble(local_out, group=None):
    """Sum the ranks' disjoint partial outputs in place (all-reduce)."""
    import torch.distributed as dist
    dist.all_reduce(local_out, op=dist.ReduceOp.SUM, group=group)
    return local_out


class ShardedMatvec:
    """u = A lambda over `world` ranks (torch.distributed process group)."""

    def __init__(self, ps: PointSet, leaf_level: int, kernel: RadialKernel, sigma: float,
                 m_per_dim: int, nrhs: int = 1, group=None, device: int = -1):
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.plan = Plan(ps, leaf_level, kernel, sigma, m_per_dim, nrhs=nrhs, device=device,
                         rank=self.rank, world=self.world)

    def owned_points(self) -> np.ndarray:
        inf = self.plan.info()
        idx = np.zeros(inf.owned_end - inf.owned_begin, dtype=np.int64)
        if idx.size:
            _capi.check(_capi.lib().blfmm_plan_owned_points(
                self.plan.handle, idx.ctypes.data_as(ct.POINTER(ct.c_longlong))))
        return idx

    def device(self, lam, out, stream=None):
        """lam / out: device tensors [nrhs, n]; out is assembled on every rank."""
        self.plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=stream)
        if self.world > 1:
            assemble(out, self.group)
        return out
