#!/usr/bin/env python
"""Benchmark of the B200 band-limited FMM RBF matvec (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload P3] [--no-cpu-baseline]

One step = one band-limited multilevel FMM matvec (P2M, M2M, M2L+L2L, L2P,
near-field P2P) of the workload with a prebuilt plan (tree + grids + C table,
the reference's bench_matvec.cpp:48-61 convention). Metric: evals/s =
nrhs * N^2 / t_step (BASELINE.json). Default workload: configs[2] of
BASELINE.json (3D IMQ c=0.1, N=1,048,576 blob mixture) — the configuration
the metric ("at N=1M 3D") is quoted on; it fits one B200.

--impl reference times the reference's CPU path on this host (the oracle
port: the reference itself is d <= 2 only, so its 3-D path is the
restatement in oracle/), with all host threads, and prints the same line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1606_07652_b200 import inputs as I  # noqa: E402

METRIC = "FMM RBF matvec evals/s (N^2/time)"
UNIT = "evals/s"


def peaks():
    p = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
    except Exception:
        pass
    return p


def fp64_peak():
    """Measured FP64 DFMA peak (profiles/fp64_peak.json, written by
    tools/fp64_peak.py on a B200), TFLOP/s."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self, which):
        """Wall-clock bounds of the timed region (samples outside are dropped)."""
        import datetime
        setattr(self, which, datetime.datetime.now())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        import datetime
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0 = getattr(self, "t0", None)
        t1 = getattr(self, "t1", None)
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f")
                if t0 and t1 and not (t0 - datetime.timedelta(milliseconds=150) <= ts <= t1):
                    continue
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        under = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(under) if under else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def far_bytes(info, K, nrhs):
    """Algorithmic HBM bytes of the far-field translation kernels per matvec
    (SURVEY §8d): M2M reads children + writes parents (levels L..1); the fused
    M2L+L2L kernel reads V_l once, reads the parent's G_{l-1} once and writes
    one expansion (G_l, or L_L at the leaf) per box, levels 1..L."""
    L = info.leaf_level
    B = [info.boxes[l] for l in range(L + 1)]
    cb = 16 * K * nrhs
    m2m = sum((B[l] + B[l - 1]) * cb for l in range(2, L + 1))
    if getattr(info, "telescoped", 0):
        # telescoped: k_root reads V_1 and writes C V_0; the leaf couple reads
        # V_L once and writes L_L (no intermediate G levels)
        m2l = (B[1] + 1) * cb + 2 * B[L] * cb
    else:
        m2l = sum(2 * B[l] * cb + (B[l - 1] * cb if l >= 2 else 0) for l in range(1, L + 1))
    return m2m, m2l


def run_ours(args, W, world, rank, local):
    import torch

    import paper_1606_07652_b200 as B

    # test-only overrides: run the N>1 code path on a single-GPU box
    # (BLFMM_BENCH_DEVICE pins every rank to one device; BLFMM_DIST_BACKEND=gloo
    # keeps ranks that share a GPU from waiting on each other's kernels)
    if os.environ.get("BLFMM_BENCH_DEVICE") is not None:
        local = int(os.environ["BLFMM_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("BLFMM_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    x, w = W.make()
    n, nrhs = W.n, W.nrhs
    k = B.parse_kernel_spec(W.kernel)
    t0 = time.perf_counter()
    sharded = None
    if world > 1:
        # the library's distributed execute (blfmm_plan_attach_nccl): partitioned
        # upsweep, NCCL all-reduce of the level-1 expansions, owned downsweep +
        # near field, NCCL broadcast gather of the owned slices of u
        from paper_1606_07652_b200 import distributed as Dst
        sharded = Dst.ShardedMatvec(B.PointSet(W.d, x), W.leaf, k, W.sigma, W.m, nrhs=nrhs,
                                    device=local, rank=rank, world=world)
        plan = sharded.plan
    else:
        plan = B.Plan(B.PointSet(W.d, x), W.leaf, k, W.sigma, W.m, nrhs=nrhs, device=local)
    plan_s = time.perf_counter() - t0
    info = plan.info()
    K = W.m ** W.d
    w2 = np.ascontiguousarray(w.reshape(nrhs, n))
    lam = torch.from_numpy(w2).to(dev)
    out = torch.empty_like(lam)
    # a dedicated (non-default) stream: the library orders its own stream
    # after/before it with events, so events on it bracket the whole matvec
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sp = ct_stream(stream)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def step():
        if sharded is not None:
            sharded.device(lam, out, stream=sp)
        else:
            plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        # keep the GPU busy while nvidia-smi starts sampling, then time
        t_start = time.perf_counter()
        while time.perf_counter() - t_start < 0.5:
            step()
            torch.cuda.synchronize(dev)
        barrier()
        clk.mark("t0")
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        clk.mark("t1")
    barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # Informational: the same matvec with the SumStats requested every step
    # (max|Im| of the far field: the half-spectrum L2P adds its imaginary-
    # residual GEMM, plus one D2H read and host sync per call).
    ms_stats = None
    if sharded is None:
        torch.cuda.synchronize(dev)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp, stats=True)
        s0.record(stream)
        for _ in range(args.steps):
            plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp, stats=True)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        ms_stats = s0.elapsed_time(s1) / args.steps

    # Stage profile (CUDA events recorded by the library on the launch stream),
    # same command, separate pass of `steps` matvecs.
    plan.set_profiling(True)
    acc = {}
    launches = 0
    for _ in range(args.steps):
        plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp)
        for name, (t, nl) in plan.stage_times().items():
            a = acc.setdefault(name, [0.0, 0])
            a[0] += t / args.steps
            a[1] = nl
    plan.set_profiling(False)
    launches = sum(v[1] for v in acc.values())

    # End to end through the C ABI with host (pinned) buffers: H2D of lambda
    # and D2H of the result inside the timed region, every step.
    hl = torch.from_numpy(w2).pin_memory()
    ho = torch.empty_like(hl).pin_memory()
    lam_np, out_np = hl.numpy(), ho.numpy()
    for _ in range(max(1, args.warmup // 2)):
        plan.execute(lam_np if nrhs > 1 else lam_np[0], stream=sp)
    torch.cuda.synchronize(dev)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        if world == 1:
            e2e_call(B, plan, lam_np, out_np, sp)
        else:  # sharded, same C ABI call: H2D, distributed matvec, D2H
            e2e_call(B, plan, lam_np, out_np, sp)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # The level-by-level couple + L2L sweep (mlfmm.cpp:268-340, SURVEY §7's
    # graded path; the default telescoped form equals it to rounding, DESIGN.md
    # §5.4): same matvec on a plan built with tuning telescope = 0.
    ms_sweep = None
    if world == 1 and info.telescoped:
        sw_plan = B.Plan(B.PointSet(W.d, x), W.leaf, k, W.sigma, W.m, nrhs=nrhs, device=local,
                         tuning={"telescope": 0})
        for _ in range(2):
            sw_plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp)
        torch.cuda.synchronize(dev)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            sw_plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        ms_sweep = s0.elapsed_time(s1) / args.steps
        del sw_plan

    # parity spot checks (cheap): GPU direct O(N^2) on 1024 sampled targets
    rng = np.random.default_rng(7)
    tg = np.sort(rng.choice(n, size=min(1024, n), replace=False))
    dv = B.direct_matvec(k, B.PointSet(W.d, x), w2[0], targets=tg).values
    fmm_vals = (out_np[0] if world == 1 else out.cpu().numpy()[0]).copy()
    rel_direct = float(np.linalg.norm(fmm_vals[tg] - dv) / np.linalg.norm(dv))

    evals = nrhs * float(n) * float(n)
    value = evals / (ms / 1e3)
    pk = peaks()
    m2m_b, m2l_b = far_bytes(info, info.stored_nodes, nrhs)
    stage = {k_: {"ms": round(v[0], 4), "launches": v[1]} for k_, v in acc.items()}
    top = max(acc.items(), key=lambda kv: kv[1][0])[0]
    hbm_peak = pk.get("hbm_gbs", 6650.0)
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in pk else "fallback 6.65 TB/s"
    fp = fp64_peak() or {}
    dmma_peak, dfma_peak = fp.get("dmma_tflops", 37.2), fp.get("dfma_tflops", 37.2)
    fp_src = ("profiles/fp64_peak.json (measured on B200 by tools/fp64_peak.cu; "
              "MEASURED_PEAKS.json has no FP64 figure)" if fp else "nominal 37.2 TFLOP/s")
    L = info.leaf_level
    Bx = [info.boxes[l] for l in range(L + 1)]
    cb = 16 * info.stored_nodes * nrhs
    # algorithmic work per stage: P2M / L2P one
    # complex MAC (8 flops) per point and grid node of the full K = M^d grid;
    # M2M (levels L-1 -> 1, the leaf level is fused into P2M) and the couple
    # bytes from the stored expansions; near field F_k flops per pair
    near_fk = {"imq": 19, "mq": 16, "gaussian": 15}.get(W.kernel.split(":")[0], 16)
    work = {
        "p2m": ("k_p2m", "tensor", 8.0 * n * K * nrhs, "TFLOP/s", dmma_peak, fp_src),
        "m2m": ("k_m2m", "hbm", float(sum((Bx[l] + Bx[l - 1]) * cb for l in range(2, L))),
                "GB/s", hbm_peak, hbm_src),
        "m2l_l2l": ("k_couple", "hbm", float(m2l_b), "GB/s", hbm_peak, hbm_src),
        "l2p": ("k_l2p", "tensor", 8.0 * n * K * nrhs, "TFLOP/s", dmma_peak, fp_src),
        "near": ("k_near", "fp64", float(near_fk) * info.near_pairs * nrhs, "TFLOP/s",
                 dfma_peak, fp_src),
    }
    stage_roof = {}
    for name, (kern, bound, amount, unit, peak_v, src) in work.items():
        t_ms = acc.get(name, [0, 0])[0]
        if t_ms <= 0 or amount <= 0:
            continue
        ach = amount / (t_ms / 1e3) / (1e9 if unit == "GB/s" else 1e12)
        stage_roof[name] = {"kernel": kern + "*", "bound": bound, "achieved": round(ach, 2),
                            "peak": peak_v, "unit": unit, "frac": round(ach / peak_v, 4),
                            "traffic": load_traffic(kern),
                            ("algorithmic_bytes" if unit == "GB/s" else "algorithmic_flops"): amount,
                            "peak_source": src, "ms": round(t_ms, 4)}
        if unit == "TFLOP/s":
            # reference-equivalent work (the reference's full-grid / ordered-pair
            # count) vs the FP64 work the kernel executes (half spectrum,
            # symmetric pairs, operand formation), from the committed ncu
            # capture of one matvec: physical rate = this run's time x the
            # capture's physical / algorithmic ratio
            ph = load_physical(kern)
            if ph:
                phys = ph["flops"] / (t_ms / 1e3) / 1e12
                stage_roof[name]["physical"] = {
                    "executed_fp64_flops": ph["flops"], "achieved": round(phys, 2),
                    "frac": round(phys / peak_v, 4),
                    "fp64_pipe_pct": ph.get("fp64_pipe_pct"),
                    "dmma_pipe_pct": ph.get("dmma_pipe_pct"),
                    "source": os.path.relpath(TRAFFIC_PROFILE, ROOT)}
    roof = None
    if top in stage_roof:
        roof = dict(stage_roof[top], dominant_stage=top)
    elif "m2l_l2l" in stage_roof:
        roof = dict(stage_roof["m2l_l2l"], dominant_stage=top)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
        "config": {"workload": W.name, "d": W.d, "kernel": W.kernel, "n": n, "nrhs": nrhs,
                   "sigma": W.sigma, "m_per_dim": W.m, "K": K, "leaf_level": W.leaf,
                   "points": W.points, "grid_mode": "shared",
                   "parallelism": (f"morton-range x{world} (halo P2M + NCCL all-reduce of "
                                   f"level-1 multipoles (telescoped) + broadcast gather of "
                                   f"the owned slices of u, inside libblfmm_gpu)")
                                  if world > 1 else "single",
                   "l2": "per-step working set (expansions %.1f GB) >> 126 MB L2" %
                         (info.device_bytes / 1e9),
                   "nonempty_boxes": [info.boxes[l] for l in range(2, W.leaf + 1)]},
        "e2e": {"value": evals / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": 8 * n * nrhs,
                "d2h_bytes_per_step": 8 * n * nrhs,
                "api": ("blfmm_execute (C ABI, host buffers, stats NULL)" if world == 1 else
                        "blfmm_execute on a plan with an NCCL communicator (C ABI, host "
                        "buffers): H2D + upsweep + NCCL expansion all-reduce + downsweep + "
                        "NCCL gather of u + D2H")},
        "ms_per_step_with_stats": ms_stats,
        "ms_per_step_level_sweep": ms_sweep,
        "kernels": plan.kernels(),
        "gpu_launches": launches * args.steps,
        "stages_ms": stage,
        "roofline": roof,
        "stage_rooflines": stage_roof,
        "plan_seconds": plan_s,
        "parity": {"rel_l2_vs_gpu_direct_1024_targets": rel_direct,
                   "note": "rel_l2_vs_oracle: this matvec against one full CPU matvec "
                           "(cpu_baseline leg, same inputs and C table; bar 1e-10). "
                           "vs direct: informational (band-limited far field vs the plain "
                           "kernel)"},
        "_values_rhs0": fmm_vals,
        "stats": {"near_pairs": info.near_pairs, "far_work": info.far_work,
                  "il_pairs_nonempty": info.il_pairs},
    }
    if world == 1 and W.name == "P3" and not args.no_extra_workloads:
        # the other GPU configs of BASELINE.json, short runs on the same box
        # (not the headline; P1 is the reference's own CPU-sized case)
        line["workloads"] = {}
        for name in ("P2", "P4", "P5"):
            line["workloads"][name] = time_workload(B, I.WORKLOADS[name], 10, 3, dev, stream, sp)
    near_ms = acc.get("near", [0, 0])[0]
    if near_ms > 0:
        line["near_field_fp64"] = {"pairs": info.near_pairs, "ms": near_ms,
                                   "pairs_per_s": info.near_pairs * nrhs / (near_ms / 1e3),
                                   "flops_per_pair": near_fk, "peak_tflops": dfma_peak}
    return line, clk.summary()


def time_workload(B, W, steps, warmup, dev, stream, sp):
    """Short device-resident timing of another BASELINE config (same
    protocol as the headline: prebuilt plan, inputs in HBM, CUDA events on the
    launch stream) plus its serialised per-stage profile."""
    import torch
    x, w = W.make()
    n, nrhs = W.n, W.nrhs
    k = B.parse_kernel_spec(W.kernel)
    t0 = time.perf_counter()
    plan = B.Plan(B.PointSet(W.d, x), W.leaf, k, W.sigma, W.m, nrhs=nrhs, device=dev.index)
    plan_s = time.perf_counter() - t0
    lam = torch.from_numpy(np.ascontiguousarray(w.reshape(nrhs, n))).to(dev)
    out = torch.empty_like(lam)
    for _ in range(warmup):
        plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    plan.set_profiling(True)
    acc = {}
    for _ in range(steps):
        plan.execute_device(lam.data_ptr(), out.data_ptr(), stream=sp)
        for name, (t, nl) in plan.stage_times().items():
            a = acc.setdefault(name, [0.0, 0])
            a[0] += t / steps
            a[1] = nl
    plan.set_profiling(False)
    info = plan.info()
    evals = nrhs * float(n) * float(n)
    res = {"value": evals / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": steps,
           "warmup": warmup, "plan_seconds": plan_s,
           "config": {"workload": W.name, "d": W.d, "kernel": W.kernel, "n": n, "nrhs": nrhs,
                      "sigma": W.sigma, "m_per_dim": W.m, "leaf_level": W.leaf,
                      "points": W.points},
           "kernels": plan.kernels(),
           "stages_ms": {k_: {"ms": round(v[0], 4), "launches": v[1]} for k_, v in acc.items()},
           "near_pairs": info.near_pairs, "near_sym_items": info.near_sym_items}
    del plan
    torch.cuda.synchronize(dev)
    return res


def e2e_call(B, plan, lam_np, out_np, sp):
    # u only (stats = NULL: no max|Im| diagnostic), as a Krylov caller uses it
    import ctypes as ct
    from paper_1606_07652_b200 import _capi
    _capi.check(_capi.lib().blfmm_execute(
        plan.handle, lam_np.ctypes.data_as(ct.POINTER(ct.c_double)),
        out_np.ctypes.data_as(ct.POINTER(ct.c_double)), None, sp))


def ct_stream(stream):
    import ctypes as ct
    return ct.c_void_p(stream.cuda_stream)


TRAFFIC_PROFILE = os.path.join(ROOT, "profiles", "r02_ncu_step_metrics.json")


def load_traffic(prefix):
    """DRAM bytes (read + write) per matvec of the kernels whose name starts
    with `prefix` (all launches of one step, matching `achieved`), from the
    committed ncu capture (tools/ncu_dram_summary.py), or None."""
    try:
        with open(TRAFFIC_PROFILE) as f:
            s = json.load(f)
        hits = [v["dram_bytes_total"] for k_, v in s["kernels"].items() if k_.startswith(prefix)]
        return float(sum(hits)) if hits else None
    except Exception:
        return None


def load_physical(prefix):
    """Executed FP64 work of the kernels whose name starts with `prefix` in the
    committed one-matvec ncu capture: physical flops (DMMA m8n8k4 = 512, DFMA
    = 2, DADD / DMUL = 1), the capture's kernel time, and the FP64 / DMMA
    pipe utilisation (time-weighted), or None."""
    try:
        with open(TRAFFIC_PROFILE) as f:
            s = json.load(f)
        hits = [v for k_, v in s["kernels"].items() if k_.startswith(prefix)]
        if not hits or not all("fp64_flops_physical" in v for v in hits):
            return None
        ms = sum(v["ms_total"] for v in hits)
        out = {"flops": sum(v["fp64_flops_physical"] for v in hits), "ncu_ms": ms}
        for key in ("fp64_pipe_pct", "dmma_pipe_pct"):
            if all(key in v for v in hits):
                out[key] = round(sum(v[key] * v["ms_total"] for v in hits) / max(ms, 1e-12), 2)
        return out
    except Exception:
        return None


def cpu_model():
    """CPU model string of this host (lscpu), for the baseline lines."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_matvec(W, x=None, w=None):
    """One FULL (unsampled) CPU matvec of the workload on this host's cores:
    the reference's own mlfmm_matvec (compiled from its sources) for d <= 2,
    the oracle restatement of it (oracle/blfmm_oracle.cpp, same loop
    structure, std::polar per term) for d = 3, where the reference's 2-D
    point type cannot run. Tree and grids are built outside the timed call
    (bench_matvec.cpp:48-61). Multiple right-hand sides are separate calls
    in the reference; one is timed and multiplied by nrhs.
    Returns (seconds for all nrhs, values of rhs 0, kind)."""
    from oracle import pyoracle as po
    if x is None:
        x, w = W.make()
    w1 = np.ascontiguousarray(np.asarray(w).reshape(W.nrhs, W.n)[0])
    if W.d <= 2 and po.ref_available():
        vals, st = po.ref_mlfmm(x, w1, W.kernel, W.sigma, W.m, W.leaf)
        return st["seconds"] * W.nrhs, vals, "reference"
    ctab = po.c_table(W.kernel, W.sigma, W.m, W.d)
    t0 = time.perf_counter()
    vals, _, secs = po.mlfmm(x, w1, W.kernel, W.sigma, W.m, W.leaf, c_table_in=ctab)
    t = time.perf_counter() - t0
    return t * W.nrhs, vals, "port"


def run_reference(args, W):
    from oracle import pyoracle as po
    cores = os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(cores)  # torchrun exports 1
    cores = po.set_threads(cores)
    x, w = W.make()
    times = []
    kind = "port"
    # every step is one full, unsampled CPU matvec; one untimed warm-up call
    # (first-touch allocation) however large --warmup is: a CPU call has no
    # JIT or cache state to warm beyond that
    warm = min(args.warmup, 1)
    for s in range(warm + args.steps):
        t, _, kind = cpu_matvec(W, x, w)
        if s >= warm:
            times.append(t)
    t = statistics.median(times)
    evals = W.nrhs * float(W.n) ** 2
    v = evals / t
    sample = ("full mlfmm_matvec call per step (the reference compiled from its sources)"
              if kind == "reference" else
              "full oracle mlfmm_matvec per step (the reference restated for d=3; unsampled)")
    if W.nrhs > 1:
        sample += f"; rhs 1 of {W.nrhs} timed, x{W.nrhs} (the reference takes one rhs per call)"
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "warmup_run": warm, "ms_per_step": t * 1e3,
            "ms_per_step_min": min(times) * 1e3, "ms_per_step_max": max(times) * 1e3,
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "impl": "reference",
            "config": {"workload": W.name, "d": W.d, "kernel": W.kernel, "n": W.n, "nrhs": W.nrhs,
                       "sigma": W.sigma, "m_per_dim": W.m, "leaf_level": W.leaf},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="P3", choices=sorted(I.WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-workloads", action="store_true",
                    help="skip the short P2 / P4 / P5 timings appended to the P3 line")
    args = ap.parse_args()
    world, rank, local = dist_env()
    W = I.WORKLOADS[args.workload]
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args, W)), flush=True)
        return
    line, clocks = run_ours(args, W, world, rank, local)
    line["clocks"] = clocks
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only
            from oracle import pyoracle as po
            cores = po.set_threads(os.cpu_count() or 1)
            x, w = W.make()
            t, vals, kind = cpu_matvec(W, x, w)
            line["cpu_baseline"] = {
                "value": W.nrhs * float(W.n) ** 2 / t, "unit": UNIT, "cores": cores,
                "kind": kind, "cpu_model": cpu_model(), "seconds_per_matvec": t,
                "sample": "one full, unsampled CPU matvec of the same workload (" +
                          ("the reference compiled from its sources" if kind == "reference"
                           else "oracle restatement of the reference, d=3") + ")" +
                          (f"; rhs 1 of {W.nrhs} timed, x{W.nrhs}" if W.nrhs > 1 else "")}
            # parity of the benchmarked matvec against that CPU result (same
            # inputs, same C table): the north-star bar is rel-l2 <= 1e-10
            gv = line.pop("_values_rhs0")
            err = float(np.linalg.norm(gv - vals) / np.linalg.norm(vals))
            line["parity"]["rel_l2_vs_oracle"] = err
            line["parity"]["oracle_kind"] = kind
            line["parity"]["pass"] = err <= 1e-10
        line.pop("_values_rhs0", None)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
