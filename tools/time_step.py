"""Device-timed matvec loop (no per-stage fences): prints ms per matvec for a
BASELINE workload, then one serialised per-stage profile. --tuning takes a
JSON dict of blfmm_tuning fields for A/B runs."""
import json
import argparse
import ctypes as ct
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_07652_b200 as B  # noqa: E402
from paper_1606_07652_b200 import inputs as I  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="P3")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--tag", default="")
    ap.add_argument("--scaled", type=int, default=0, help="GridMode::scaled with this stencil")
    ap.add_argument("--tuning", default="{}")
    args = ap.parse_args()
    W = I.WORKLOADS[args.workload]
    x, w = W.make()
    n = x.shape[0]
    plan = B.Plan(B.PointSet(W.d, x), W.leaf, B.parse_kernel_spec(W.kernel), W.sigma, W.m,
                  nrhs=W.nrhs, grid_mode=1 if args.scaled else 0,
                  stencil_k=args.scaled if args.scaled else 10,
                  tuning=json.loads(args.tuning))
    lam = torch.from_numpy(np.ascontiguousarray(w.reshape(W.nrhs, n))).cuda()
    out = torch.empty_like(lam)
    s = torch.cuda.Stream()
    sp = ct.c_void_p(s.cuda_stream)
    for _ in range(3):
        plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(args.steps):
            plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp)
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    plan.set_profiling(True)
    plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp)
    st = {k: round(v[0], 3) for k, v in plan.stage_times().items()}
    print(f"{args.tag} {args.workload} ms/matvec {ms:.4f} stages {st} kernels {plan.kernels()}",
          flush=True)


if __name__ == "__main__":
    main()
