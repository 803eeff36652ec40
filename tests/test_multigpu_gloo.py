"""Multi-rank path on CPU (gloo, world_size 2 and 3): the host-side sharding
logic the GPU ranks use - the deterministic Morton-range partition
(blfmm_partition, host-only code of the C-ABI library) and the gather of the
ranks' owned slices of u (one broadcast per rank, as blfmm_execute does on a
plan with a communicator) - with the CPU oracle standing in for each rank's
kernels."""
import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1606_07652_b200 import inputs as I


def morton_of(idx, d, L):
    key = 0
    for b in range(L - 1, -1, -1):
        for k in range(d):
            key = (key << 1) | ((idx[k] >> b) & 1)
    return key


def leaf_tables(oracle, x, L):
    """Nonempty leaves in Morton order with point lists and near-source counts."""
    d = x.shape[1]
    pts = oracle.tree_lists(x, L, L, 2)
    nbr = oracle.tree_lists(x, L, L, 0)
    n = 1 << L
    leaves = [b for b in range(len(pts)) if len(pts[b])]

    def coords(b):
        out = []
        for _ in range(d):
            out.append(b % n)
            b //= n
        return out[::-1]

    leaves.sort(key=lambda b: morton_of(coords(b), d, L))
    npts = np.array([len(pts[b]) for b in leaves])
    nsrc = np.array([sum(len(pts[q]) for q in nbr[b]) for b in leaves])
    return leaves, pts, npts, nsrc


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    from oracle import pyoracle as po
    from paper_1606_07652_b200 import distributed as D

    W = I.WORKLOADS["P3"]
    x, w = W.make(6000)
    L, M = 3, 6
    leaves, pts, npts, nsrc = leaf_tables(po, x, L)
    bounds = D.partition(D.leaf_cost(npts, nsrc, M ** 3), world)
    # every rank derives the same split
    allb = [torch.zeros(world + 1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allb, torch.from_numpy(bounds))
    assert all(torch.equal(b, allb[0]) for b in allb)
    owned = np.concatenate([pts[b] for b in leaves[bounds[rank]:bounds[rank + 1]]] or
                           [np.zeros(0, dtype=np.int64)])
    full, _, _ = po.mlfmm(x, w, W.kernel, W.sigma, M, L)
    # gather: rank q broadcasts its owned slice (known sizes on every rank)
    u = np.full_like(full, np.nan)
    for q in range(world):
        own_q = np.concatenate([pts[b] for b in leaves[bounds[q]:bounds[q + 1]]] or
                               [np.zeros(0, dtype=np.int64)])
        buf = torch.from_numpy(full[own_q].copy() if q == rank else np.zeros(len(own_q)))
        dist.broadcast(buf, src=q)
        u[own_q] = buf.numpy()
    if rank == 0:
        np.savez(result_path, assembled=u, full=full, bounds=bounds,
                 counts=np.array([len(owned)]))
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_partition_and_owned_slice_gather(tmp_path, oracle, world):
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, free_port(), out), nprocs=world, join=True)
    r = np.load(out)
    assert np.array_equal(r["assembled"], r["full"])  # every target owned once: exact
    b = r["bounds"]
    assert b[0] == 0 and np.all(np.diff(b) > 0)


def test_partition_properties(oracle):
    from paper_1606_07652_b200 import distributed as D
    rng = np.random.default_rng(0)
    cost = rng.random(1000) ** 3
    for world in (1, 2, 3, 8):
        b = D.partition(cost, world)
        assert b[0] == 0 and b[-1] == 1000 and np.all(np.diff(b) >= 0)
        parts = [cost[b[r]:b[r + 1]].sum() for r in range(world)]
        assert max(parts) - min(parts) <= 2 * cost.max() + 1e-12
    with pytest.raises(Exception):
        D.partition(cost, 0)
