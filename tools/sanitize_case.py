"""Small plans for compute-sanitizer (memcheck / racecheck / synccheck, one
tool per run): P3-shape (3-D IMQ blobs: half spectrum, fused P2M + leaf M2M,
column couple, shared-memory L2P, persistent symmetric near field incl. the
CTA-shared items, stats GEMM) and P4-shape (2-D MQ: generated-phase DMMA
P2M / L2P, separable couple, 2-D symmetric near field), plus a 4-RHS plan
(batched near field, table-staged P2M / L2P) and a 2-rank exchange-mode
upsweep/downsweep on one device (host-side sum of the exchange buffers).

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_07652_b200 as B  # noqa: E402
from paper_1606_07652_b200 import inputs as I  # noqa: E402


def run(name, n, leaf, nrhs=None, tuning=None):
    W = I.WORKLOADS[name]
    x, w = W.make(n)
    if nrhs is not None:
        w = np.ascontiguousarray(np.atleast_2d(w)[:nrhs]) if np.ndim(w) == 2 else \
            np.stack([w * (q + 1) for q in range(nrhs)])
    plan = B.Plan(B.PointSet(W.d, x), leaf, B.parse_kernel_spec(W.kernel), W.sigma, W.m,
                  nrhs=1 if np.ndim(w) == 1 else w.shape[0], tuning=tuning)
    r1 = plan.execute(w)
    r2 = plan.execute(w)  # graph replay
    assert np.array_equal(r1.values, r2.values)
    print(name, n, leaf, plan.kernels(), float(np.linalg.norm(r1.values)), flush=True)


def main():
    run("P3", 40000, 4)                      # symmetric near items incl. > 96-point leaves
    run("P3", 12000, 3, tuning={"couple_tile": 0})
    run("P4", 60000, 5)
    run("P5", 8192, 3, nrhs=4)
    run("P2p", 6000, 3)
    # exchange mode, 2 ranks on one device: upsweep both, sum the exchange
    # buffers on the device (the all-reduce), downsweep both, sum u
    W = I.WORKLOADS["P3"]
    x, w = W.make(30000)
    k = B.parse_kernel_spec(W.kernel)
    plans = [B.Plan(B.PointSet(3, x), 4, k, W.sigma, W.m, rank=r, world=2) for r in range(2)]
    lam = torch.from_numpy(w.reshape(1, -1).copy()).cuda()
    bufs = [torch.zeros(p.exchange_size(), dtype=torch.float64, device="cuda") for p in plans]
    outs = [torch.zeros_like(lam) for _ in plans]
    for p, b in zip(plans, bufs):
        p.bind_exchange(b.data_ptr())
    for p in plans:
        p.upsweep(lam.data_ptr())
    torch.cuda.synchronize()
    tot = bufs[0] + bufs[1]
    for b in bufs:
        b.copy_(tot)
    for p, o in zip(plans, outs):
        p.downsweep(o.data_ptr())
    torch.cuda.synchronize()
    u = (outs[0] + outs[1]).cpu().numpy()[0]
    full = B.Plan(B.PointSet(3, x), 4, k, W.sigma, W.m).execute(w).values
    print("exchange rel", float(np.linalg.norm(u - full) / np.linalg.norm(full)), flush=True)


if __name__ == "__main__":
    main()
