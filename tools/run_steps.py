"""Minimal matvec loop for profiling (ncu) and quick timing: builds the plan of
a BASELINE workload and runs `--steps` matvecs through blfmm_execute_device."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_07652_b200 as B  # noqa: E402
from paper_1606_07652_b200 import inputs as I  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="P3")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--scaled", type=int, default=0, help="GridMode::scaled with this stencil")
    ap.add_argument("--stats", type=int, default=0,
                    help="request SumStats (the L2P imaginary-residual GEMM runs)")
    args = ap.parse_args()
    W = I.WORKLOADS[args.workload]
    x, w = W.make(args.n)
    n = x.shape[0]
    plan = B.Plan(B.PointSet(W.d, x), W.leaf, B.parse_kernel_spec(W.kernel), W.sigma, W.m,
                  nrhs=W.nrhs, grid_mode=1 if args.scaled else 0,
                  stencil_k=args.scaled if args.scaled else 10)
    lam = torch.from_numpy(np.ascontiguousarray(w.reshape(W.nrhs, n))).cuda()
    out = torch.empty_like(lam)
    s = torch.cuda.Stream()
    import ctypes as ct
    sp = ct.c_void_p(s.cuda_stream)
    plan.set_profiling(True)
    for i in range(args.steps):
        st = plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp, stats=args.stats)
        print(i, {k: round(v[0], 3) for k, v in plan.stage_times().items()}, flush=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
