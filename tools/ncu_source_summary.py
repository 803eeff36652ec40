"""Compact text summary of one `ncu --set full` report from its CSV pages:
per launch the headline counters of the raw page (time, registers, grid,
occupancy, DMMA / FP64 pipe, DRAM bytes, L1 / L2 hit rates, shared-memory
wavefronts and bank conflicts, warp stalls per issue), and from the source
page the share of warp-stall samples by SASS opcode and by stall reason.
usage: ncu_source_summary.py RAW.csv SOURCE.csv > SUMMARY.txt"""
import csv
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "DMMA warp instructions"),
]


def raw_page(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return
    hdr, units, data = rows[0], rows[1], rows[2:]
    for d in data:
        print("== launch:", d[hdr.index("Kernel Name")][:110])
        for key, label in WANT:
            if key in hdr:
                i = hdr.index(key)
                print(f"   {label:24s} {d[i]} {units[i]}")
        st = []
        for i, h in enumerate(hdr):
            if "smsp__average_warps_issue_stalled" in h and h.endswith("_per_issue_active.ratio") \
                    and d[i] not in ("", "n/a"):
                st.append((float(d[i].replace(",", "")),
                           h.replace("smsp__average_warps_issue_stalled_", "")
                            .replace("_per_issue_active.ratio", "")))
        st.sort(reverse=True)
        print("   stalls per issue:", ", ".join(f"{n} {v:.2f}" for v, n in st[:6]))


def source_page(path):
    rows = list(csv.reader(open(path)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    seen = set()
    for b in blocks:
        if b["name"] in seen or len(b["rows"]) < 2:
            continue
        seen.add(b["name"])
        hdr, data = b["rows"][0], b["rows"][1:]
        si, src, ex = (hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"),
                       hdr.index("Instructions Executed"))
        tot = sum(int(d[si]) for d in data if d[si].isdigit()) or 1
        print("== source:", b["name"][:110], "| stall samples", tot)
        agg = {}
        for d in data:
            t = d[src].split()
            if not t:
                continue
            op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
            a = agg.setdefault(op, [0, 0])
            a[0] += int(d[si]) if d[si].isdigit() else 0
            a[1] += int(d[ex]) if d[ex].isdigit() else 0
        print("   by opcode:", ", ".join(
            f"{op} {100 * s / tot:.1f}% (x{e})"
            for op, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:8]))
        rs = {h: sum(int(d[i]) for d in data if d[i].isdigit())
              for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
        print("   by reason:", ", ".join(
            f"{k.replace('stall_', '')} {100 * v / tot:.1f}%"
            for k, v in sorted(rs.items(), key=lambda kv: -kv[1])[:7]))


if __name__ == "__main__":
    raw_page(sys.argv[1])
    source_page(sys.argv[2])
