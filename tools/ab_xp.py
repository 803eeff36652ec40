"""A/B of development experiment switches (BLFMM_XP0..3, development builds:
BLFMM_DEV_KNOBS=1 at build time): one plan per setting of a BASELINE workload,
stage times of the median step and the result's rel-l2 against the first
setting.  usage: ab_xp.py WORKLOAD "0,0,0,0" "1,0,1,0:{\"near_ctas_per_sm\": 1}" ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_07652_b200 as B  # noqa: E402
from paper_1606_07652_b200 import inputs as I  # noqa: E402


def run(wl, xp, steps=7, tuning=None):
    for i, v in enumerate(xp):
        os.environ[f"BLFMM_XP{i}"] = str(v)
    W = I.WORKLOADS[wl]
    x, w = W.make(None)
    n = x.shape[0]
    plan = B.Plan(B.PointSet(W.d, x), W.leaf, B.parse_kernel_spec(W.kernel), W.sigma, W.m,
                  nrhs=W.nrhs, tuning=tuning)
    lam = torch.from_numpy(np.ascontiguousarray(w.reshape(W.nrhs, n))).cuda()
    out = torch.empty_like(lam)
    s = torch.cuda.Stream()
    import ctypes as ct
    sp = ct.c_void_p(s.cuda_stream)
    # serialised stage profile
    plan.set_profiling(True)
    st = []
    for _ in range(3):
        plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp, stats=0)
        st.append({k: v[0] for k, v in plan.stage_times().items()})
    plan.set_profiling(False)
    stages = {k: round(float(np.median([q[k] for q in st])), 3) for k in st[0]}
    ts = []
    for _ in range(steps + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp, stats=0)
            e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    u = out.cpu().numpy().copy()
    del plan
    return float(np.median(ts[3:])), stages, u


def main():
    wl = sys.argv[1]
    ref = None
    for spec in sys.argv[2:]:
        head, _, tj = spec.partition(":")
        xp = [int(v) for v in head.split(",")]
        import json
        ms, stages, u = run(wl, xp, tuning=json.loads(tj) if tj else None)
        if ref is None:
            ref = u
        err = np.linalg.norm(u - ref) / np.linalg.norm(ref)
        print(f"{wl} xp={spec} step {ms:.3f} ms rel-vs-first {err:.2e} {stages}", flush=True)


if __name__ == "__main__":
    main()
