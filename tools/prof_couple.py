"""One P3 matvec per leaf-couple variant (blfmm_tuning.couple_tile), for an
ncu capture of the couple kernels: python tools/prof_couple.py 0 1"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_07652_b200 as B  # noqa: E402
from paper_1606_07652_b200 import inputs as I  # noqa: E402

W = I.WORKLOADS[os.environ.get("WL", "P3")]
x, w = W.make()
lam = torch.from_numpy(np.ascontiguousarray(w.reshape(W.nrhs, -1))).cuda()
out = torch.empty_like(lam)
for v in [int(a) for a in sys.argv[1:]]:
    plan = B.Plan(B.PointSet(W.d, x), W.leaf, B.parse_kernel_spec(W.kernel), W.sigma, W.m,
                  nrhs=W.nrhs, tuning={"couple_tile": v, "graphs": 0})
    plan.execute_device(lam.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    print(v, plan.kernels()["couple"], float(out[0, :4].sum()), flush=True)
    del plan
