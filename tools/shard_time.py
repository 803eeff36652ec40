"""Per-rank device time of the sharded P3 matvec, measured one rank at a time
on ONE GPU (no collective: the exchange buffer is left as this rank's partial
sums, which does not change the work). Projects the N-GPU step as
max over ranks (upsweep + downsweep) + the two all-reduces (estimated from
their byte counts). Exchange mode = distributed.ShardedMatvec's default."""
import argparse
import ctypes as ct
import json
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
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    W = I.WORKLOADS[args.workload]
    x, w = W.make()
    n = x.shape[0]
    k = B.parse_kernel_spec(W.kernel)
    ps = B.PointSet(W.d, x)
    lam = torch.from_numpy(np.ascontiguousarray(w.reshape(W.nrhs, n))).cuda()
    out = torch.empty_like(lam)
    s = torch.cuda.Stream()
    sp = ct.c_void_p(s.cuda_stream)
    res = {}
    for world in [int(v) for v in args.worlds.split(",")]:
        per = []
        for rank in range(world):
            plan = B.Plan(ps, W.leaf, k, W.sigma, W.m, nrhs=W.nrhs, rank=rank, world=world)
            xs = plan.exchange_size()
            xb = torch.zeros(max(xs, 1), dtype=torch.float64, device="cuda")
            if xs:
                plan.bind_exchange(xb.data_ptr())
            for _ in range(2):
                plan.upsweep(lam.data_ptr(), stream=sp)
                plan.downsweep(out.data_ptr(), stream=sp)
            torch.cuda.synchronize()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            up = dn = 0.0
            for _ in range(args.steps):
                with torch.cuda.stream(s):
                    e0.record(s)
                    plan.upsweep(lam.data_ptr(), stream=sp)
                    e1.record(s)
                    plan.downsweep(out.data_ptr(), stream=sp)
                    e2.record(s)
                torch.cuda.synchronize()
                up += e0.elapsed_time(e1)
                dn += e1.elapsed_time(e2)
            per.append({"rank": rank, "upsweep_ms": up / args.steps,
                        "downsweep_ms": dn / args.steps, "xbuf_MB": xs * 8 / 1e6})
            del plan
        mx = max(p["upsweep_ms"] + p["downsweep_ms"] for p in per)
        xmb = max(p["xbuf_MB"] for p in per)
        # all-reduce estimate: ring/NVLS bus traffic ~2x bytes at ~400 GB/s effective
        ar_ms = 2 * (xmb + 8.0 * n * W.nrhs / 1e6) / 400e3 * 1e3
        res[world] = {"per_rank": per, "max_rank_ms": mx, "allreduce_est_ms": ar_ms,
                      "projected_ms": mx + ar_ms}
        print(json.dumps({"world": world, "max_rank_ms": round(mx, 3),
                          "min_rank_ms": round(min(p["upsweep_ms"] + p["downsweep_ms"] for p in per), 3),
                          "allreduce_est_ms": round(ar_ms, 3), "projected_ms": round(mx + ar_ms, 3)}),
              flush=True)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "shard_time.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
