"""Multi-GPU (one process per GPU) band-limited FMM matvec.

Sharding: the leaves, sorted by Morton key, are split into
`world` contiguous ranges of equal estimated cost (blfmm_partition; the same
deterministic split on every rank). Each rank's plan builds the full tree,
runs the upsweep, and evaluates the downsweep (couple / L2L / L2P) and the
near field for its own range only, writing zeros elsewhere. The exchange is
one all-reduce(sum) of the output vector over NCCL (NVLink) — the ranks'
supports are disjoint, so the sum is the matvec bit for bit.

Exchange mode (leaf level >= 3, the default here): the upsweep is partitioned
as well. Each rank runs P2M on its leaves plus a two-leaf halo, keeps complete
multipoles at levels L and L-1 where its downsweep reads them, and writes
partial multipoles of the coarse levels (its own leaves only) into an exchange
buffer; one NCCL all-reduce of that buffer is the upper-level expansion
exchange, after which the downsweep runs. With the telescoped 3-D downsweep
(blfmm_plan_info.telescoped) the leaf locals need only the root multipole, so
the buffer holds level 1 alone (8 expansions, 0.3 MB for P3); otherwise levels
1..L-2. Without exchange mode
(blfmm_execute on a world > 1 plan) the upsweep is replicated instead.
"""
from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _capi
from .api import InvalidArgument, Plan, PointSet, RadialKernel


def leaf_cost(npts: np.ndarray, nsrc: np.ndarray, K: int) -> np.ndarray:
    """Per-leaf cost model used by the plan (blfmm.cu, plan_build_tree), in
    units of one near-field pair and calibrated on the P3 kernels: near pairs
    + 1.1 K per point (P2M / L2P) + 19 K per leaf (translations), with K the
    stored nodes per expansion (blfmm_plan_info.stored_nodes)."""
    npts = np.asarray(npts, dtype=np.float64)
    return npts * np.asarray(nsrc, dtype=np.float64) + 1.1 * npts * K + 19.0 * K


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
                 m_per_dim: int, nrhs: int = 1, group=None, device: int = -1,
                 exchange: bool = True, rank: int | None = None, world: int | None = None):
        import torch
        import torch.distributed as dist
        self.group = group
        init = dist.is_available() and dist.is_initialized()
        self.rank = rank if rank is not None else (dist.get_rank(group) if init else 0)
        self.world = world if world is not None else (dist.get_world_size(group) if init else 1)
        self.plan = Plan(ps, leaf_level, kernel, sigma, m_per_dim, nrhs=nrhs, device=device,
                         rank=self.rank, world=self.world)
        self.xbuf = None
        if exchange and self.world > 1 and self.plan.exchange_size() > 0:
            dev = torch.device("cuda", device) if device >= 0 else torch.device("cuda")
            self.xbuf = torch.zeros(self.plan.exchange_size(), dtype=torch.float64, device=dev)
            self.plan.bind_exchange(self.xbuf.data_ptr())

    def owned_points(self) -> np.ndarray:
        inf = self.plan.info()
        idx = np.zeros(inf.owned_end - inf.owned_begin, dtype=np.int64)
        if idx.size:
            _capi.check(_capi.lib().blfmm_plan_owned_points(
                self.plan.handle, idx.ctypes.data_as(ct.POINTER(ct.c_longlong))))
        return idx

    def device(self, lam, out, stream=None):
        """lam / out: device tensors [nrhs, n]; out is assembled on every rank.
        Stream ordering: the library orders its work after / before `stream`
        (NULL = the default stream), where the NCCL calls are enqueued."""
        if self.xbuf is not None:
            self.plan.upsweep(lam.data_ptr(), stream=stream)
            assemble(self.xbuf, self.group)  # upper-level expansion exchange
            self.plan.downsweep(out.data_ptr(), stream=stream)
        else:
            self.plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=stream)
        if self.world > 1:
            assemble(out, self.group)
        return out
