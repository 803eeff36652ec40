"""A/B of the telescoped leaf-couple variants (blfmm_tuning.couple_tile):
agreement with the per-parent kernel (variant 0) on several workloads and the
per-stage couple time. Usage: python tools/ab_couple.py [variants...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_07652_b200 as B  # noqa: E402
from paper_1606_07652_b200 import inputs as I  # noqa: E402


def run(W, x, w, leaf, var, steps=10):
    plan = B.Plan(B.PointSet(W.d, x), leaf, B.parse_kernel_spec(W.kernel), W.sigma, W.m,
                  nrhs=W.nrhs, tuning={"couple_tile": var})
    lam = torch.from_numpy(np.ascontiguousarray(w.reshape(W.nrhs, -1))).cuda()
    out = torch.empty_like(lam)
    for _ in range(3):
        plan.execute_device(lam.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        plan.execute_device(lam.data_ptr(), out.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    plan.set_profiling(True)
    acc = 0.0
    for _ in range(steps):
        plan.execute_device(lam.data_ptr(), out.data_ptr())
        acc += plan.stage_times()["m2l_l2l"][0] / steps
    vals = out.cpu().numpy().copy()
    k = plan.kernels()["couple"]
    del plan
    return ms, acc, vals, k


def main():
    only = [a for a in sys.argv[1:] if not a.lstrip("-").isdigit()]
    vars_ = [int(a) for a in sys.argv[1:] if a.lstrip("-").isdigit()] or [0, 1, 2, 3, 4]
    for name, n, leaf in [("P3", None, 6), ("P3", 200000, 5), ("P2p", None, 4), ("P5", None, 4),
                          ("P2", None, 4)]:
        if only and name not in only:
            continue
        W = I.WORKLOADS[name]
        x, w = W.make(n) if n else W.make()
        base = None
        for v in vars_:
            ms, cms, vals, k = run(W, x, w, leaf, v)
            if base is None:
                base = vals
            err = np.linalg.norm(vals - base) / np.linalg.norm(base)
            print(f"{name} n={x.shape[0]} leaf={leaf} var={v} {k}: step {ms:.4f} ms, "
                  f"couple {cms:.4f} ms, rel vs first {err:.2e}", flush=True)


if __name__ == "__main__":
    main()
