"""Multi-GPU (one process per GPU) band-limited FMM matvec.

Sharding: the leaves, sorted by Morton key, are split into
`world` contiguous ranges of equal estimated cost (blfmm_partition; the same
deterministic split on every rank). The distributed matvec itself runs INSIDE
the C++ library (blfmm_plan_attach_nccl / blfmm_plan_attach_comm, then
blfmm_execute): each rank's plan runs P2M on its leaves plus a two-leaf halo,
writes the partial upper-level multipoles into its exchange buffer, one NCCL
all-reduce of that buffer is the upper-level expansion exchange (level 1
only with the telescoped 3-D downsweep: 0.3 MB for P3; levels 1..L-2
otherwise), the rank evaluates the downsweep and the near field of its own
leaves, and the owned sorted slices of u are gathered (one broadcast per
rank and right-hand side) and scattered to the caller's order on every rank.

This module is the Python caller of that path: ShardedMatvec attaches NCCL
when the torch process group runs NCCL (the unique id travels through the
process group), and otherwise host collectives over the torch process group
(gloo: CPU tests, and several ranks sharing one GPU, whose kernels never wait
on each other - the collectives run on the host between the library's
phases).
"""
from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _capi
from .api import InvalidArgument, Plan, PointSet, RadialKernel, nccl_unique_id


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


def _device_view(dptr: int, count: int):
    """A torch tensor over `count` float64 at a raw device pointer (no copy)."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (count,), "typestr": "<f8",
                                    "data": (dptr, False), "version": 3}
    return torch.as_tensor(_View(), device="cuda")


def attach_torch_collectives(plan: Plan, group=None):
    """Library collectives over a torch.distributed process group through host
    copies (any backend; gloo for the CPU / shared-GPU tests)."""
    import torch
    import torch.distributed as dist

    def _sync(stream):
        torch.cuda.ExternalStream(stream).synchronize() if stream else torch.cuda.synchronize()

    def all_reduce(op):
        def f(dptr, count, stream):
            _sync(stream)
            t = _device_view(dptr, count)
            h = t.cpu()
            dist.all_reduce(h, op=op, group=group)
            t.copy_(h)
            torch.cuda.synchronize()
        return f

    def broadcast(dptr, count, root, stream):
        _sync(stream)
        t = _device_view(dptr, count)
        h = t.cpu()
        dist.broadcast(h, src=dist.get_global_rank(group, root) if group is not None else root,
                       group=group)
        t.copy_(h)
        torch.cuda.synchronize()

    plan.attach_comm(all_reduce(dist.ReduceOp.SUM), all_reduce(dist.ReduceOp.MAX), broadcast)


class ShardedMatvec:
    """u = A lambda over `world` ranks (torch.distributed process group): one
    plan per rank with the library's distributed execute attached. Every rank
    passes the full lambda and receives the full u (caller order)."""

    def __init__(self, ps: PointSet, leaf_level: int, kernel: RadialKernel, sigma: float,
                 m_per_dim: int, nrhs: int = 1, group=None, device: int = -1,
                 comm: str = "auto", rank: int | None = None, world: int | None = None):
        import torch.distributed as dist
        self.group = group
        init = dist.is_available() and dist.is_initialized()
        self.rank = rank if rank is not None else (dist.get_rank(group) if init else 0)
        self.world = world if world is not None else (dist.get_world_size(group) if init else 1)
        self.plan = Plan(ps, leaf_level, kernel, sigma, m_per_dim, nrhs=nrhs, device=device,
                         rank=self.rank, world=self.world)
        self.comm = "none"
        if self.world > 1:
            backend = dist.get_backend(group) if init else "none"
            use_nccl = comm == "nccl" or (comm == "auto" and backend == "nccl")
            if use_nccl:
                obj = [nccl_unique_id() if self.rank == 0 else None]
                dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0)
                                           if group is not None else 0, group=group)
                self.plan.attach_nccl(obj[0])
                self.comm = "nccl"
            else:
                attach_torch_collectives(self.plan, group)
                self.comm = "torch-host"

    def owned_points(self) -> np.ndarray:
        inf = self.plan.info()
        idx = np.zeros(inf.owned_end - inf.owned_begin, dtype=np.int64)
        if idx.size:
            _capi.check(_capi.lib().blfmm_plan_owned_points(
                self.plan.handle, idx.ctypes.data_as(ct.POINTER(ct.c_longlong))))
        return idx

    def device(self, lam, out, stream=None, stats: bool = False):
        """lam / out: device tensors [nrhs, n]; out holds u on every rank."""
        return self.plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=stream,
                                        stats=stats)

    def __call__(self, weights):
        """Host weights [n] or [nrhs, n] -> SumResult (u on every rank)."""
        return self.plan.execute(weights)
