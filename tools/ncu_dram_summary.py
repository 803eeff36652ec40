"""Summarise an ncu --csv metrics log (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum per launch, and when captured the
executed FP64 work: DMMA warp instructions, DFMA / DADD / DMUL thread
instructions, FP64 / DMMA pipe utilisation) into per-kernel JSON: launches,
total ms, DRAM bytes total / per launch, physical FP64 flops (DMMA m8n8k4 =
512 flops, DFMA = 2, DADD / DMUL = 1). Usage:
  python tools/ncu_dram_summary.py LOG.csv OUT.json "source description"
"""
import csv
import json
import re
import sys
from collections import defaultdict

TIME = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
        "second": 1e3, "s": 1e3}
BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name):
    m = re.match(r"(?:void\s+)?(?:[\w:]+::)?(\w+)", name)
    return m.group(1) if m else name


def main():
    src, out, desc = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr = rows[0]
    ki, ii = hdr.index("Kernel Name"), hdr.index("ID")
    mi, ui, vi = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    launches = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        lid = int(r[ii])
        names[lid] = short(r[ki])
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            launches[lid]["ms"] = v * TIME.get(r[ui], 1.0)
        elif r[mi].startswith("dram__bytes"):
            launches[lid][r[mi]] = v * BYTES.get(r[ui], 1.0)
        else:
            launches[lid][r[mi]] = v
    k = defaultdict(lambda: {"launches": 0, "ms_total": 0.0, "dram_bytes_total": 0.0})
    DMMA = "sm__inst_executed_pipe_tensor_subpipe_dmma.sum"
    OPS = {"smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": 2.0,
           "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": 1.0,
           "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": 1.0}
    PCT = {"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active":
               "dmma_pipe_pct"}
    for lid, m in launches.items():
        e = k[names[lid]]
        e["launches"] += 1
        e["ms_total"] += m.get("ms", 0.0)
        e["dram_bytes_total"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        if DMMA in m or any(o in m for o in OPS):
            e.setdefault("dmma_inst", 0.0)
            e.setdefault("fp64_flops_physical", 0.0)
            e["dmma_inst"] += m.get(DMMA, 0.0)
            e["fp64_flops_physical"] += 512.0 * m.get(DMMA, 0.0) + sum(
                w * m.get(o, 0.0) for o, w in OPS.items())
        for mn, key in PCT.items():
            if mn in m:  # time-weighted mean over the kernel's launches
                e.setdefault(key + "_x_ms", 0.0)
                e[key + "_x_ms"] += m[mn] * m.get("ms", 0.0)
    for e in k.values():
        e["dram_bytes_per_launch"] = e["dram_bytes_total"] / max(1, e["launches"])
        for key in ("fp64_pipe_pct", "dmma_pipe_pct"):
            if key + "_x_ms" in e:
                e[key] = round(e.pop(key + "_x_ms") / max(e["ms_total"], 1e-12), 2)
        e["ms_total"] = round(e["ms_total"], 6)
    json.dump({"source": desc, "kernels": k}, open(out, "w"), indent=1)
    for n, e in sorted(k.items(), key=lambda kv: -kv[1]["ms_total"])[:12]:
        print(f"{n:24s} {e['launches']:4d} {e['ms_total']:9.4f} ms  {e['dram_bytes_total']/1e9:8.3f} GB")


if __name__ == "__main__":
    main()
