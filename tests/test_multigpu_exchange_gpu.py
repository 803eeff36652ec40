"""The sharded matvec's real orchestration (ShardedMatvec: upsweep, all-reduce
of the exchange buffer, downsweep, all-reduce of u) with world_size 2. Both
ranks share the one GPU of the test box, so the collective is gloo (host-side
reduction of the CUDA tensors): no kernel of one rank waits on the other's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, out_path, name, n, leaf):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1606_07652_b200 as B
    from paper_1606_07652_b200 import distributed as D
    from paper_1606_07652_b200 import inputs as I
    W = I.WORKLOADS[name]
    x, w = W.make(n)
    k = B.parse_kernel_spec(W.kernel)
    sm = D.ShardedMatvec(B.PointSet(W.d, x), leaf, k, W.sigma, W.m, device=0)
    assert sm.xbuf is not None and sm.world == world
    lam = torch.from_numpy(np.ascontiguousarray(w.reshape(1, -1))).cuda()
    out = torch.empty_like(lam)
    for _ in range(2):  # second call reuses the plan and buffers
        sm.device(lam, out)
    torch.cuda.synchronize()
    if rank == 0:
        np.save(out_path, out.cpu().numpy()[0])
    dist.barrier()
    dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,n,leaf", [("P3", 60000, 4), ("P4", 40000, 5)])
def test_two_rank_exchange_matvec(blfmm, tmp_path, name, n, leaf):
    from paper_1606_07652_b200 import inputs as I
    W = I.WORKLOADS[name]
    x, w = W.make(n)
    full = blfmm.Plan(blfmm.PointSet(W.d, x), leaf, blfmm.parse_kernel_spec(W.kernel),
                      W.sigma, W.m).execute(w).values
    out = str(tmp_path / "u.npy")
    mp.spawn(_worker, args=(2, _port(), out, name, n, leaf), nprocs=2, join=True)
    got = np.load(out)
    assert np.linalg.norm(got - full) / np.linalg.norm(full) <= 1e-13
