"""Summarise an ncu --csv metrics log (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum per launch) into per-kernel JSON:
launches, total ms, DRAM bytes total / per launch. Usage:
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
    k = defaultdict(lambda: {"launches": 0, "ms_total": 0.0, "dram_bytes_total": 0.0})
    for lid, m in launches.items():
        e = k[names[lid]]
        e["launches"] += 1
        e["ms_total"] += m.get("ms", 0.0)
        e["dram_bytes_total"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    for e in k.values():
        e["dram_bytes_per_launch"] = e["dram_bytes_total"] / max(1, e["launches"])
        e["ms_total"] = round(e["ms_total"], 6)
    json.dump({"source": desc, "kernels": k}, open(out, "w"), indent=1)
    for n, e in sorted(k.items(), key=lambda kv: -kv[1]["ms_total"])[:12]:
        print(f"{n:24s} {e['launches']:4d} {e['ms_total']:9.4f} ms  {e['dram_bytes_total']/1e9:8.3f} GB")


if __name__ == "__main__":
    main()
