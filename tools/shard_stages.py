"""Per-rank stage times of the sharded P3 matvec (replicated-upsweep form, one
rank at a time on one GPU, profiling mode): shows which stage makes a rank
slow (load balance of the Morton-range partition)."""
import ctypes as ct
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_07652_b200 as B  # noqa: E402
from paper_1606_07652_b200 import inputs as I  # noqa: E402

W = I.WORKLOADS["P3"]
x, w = W.make()
n = x.shape[0]
k = B.parse_kernel_spec(W.kernel)
ps = B.PointSet(W.d, x)
lam = torch.from_numpy(np.ascontiguousarray(w.reshape(1, n))).cuda()
out = torch.empty_like(lam)
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for rank in range(world):
    plan = B.Plan(ps, W.leaf, k, W.sigma, W.m, rank=rank, world=world)
    plan.set_profiling(True)
    for _ in range(2):
        plan.execute_device(lam.data_ptr(), out.data_ptr(), stats=True)
    torch.cuda.synchronize()
    st = plan.stage_times()
    inf = plan.info()
    print(rank, inf.owned_end - inf.owned_begin, inf.near_pairs,
          {kk: round(v[0], 3) for kk, v in st.items()}, flush=True)
    del plan
