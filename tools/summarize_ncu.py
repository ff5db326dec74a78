"""Summarise ncu outputs (launch lists and --set full reports) into
profiles/*.md so the numbers behind bench.py's roofline are reviewable.

usage:
  python tools/summarize_ncu.py launches <launches.csv> <out.md> [title]
  python tools/summarize_ncu.py full <report.ncu-rep> <out.md> [title]
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
       "launch__occupancy_limit_shared_mem", "lts__t_sector_hit_rate.pct"]


def launches(path, out, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    d = OrderedDict()
    for r in rows[1:]:
        d.setdefault((int(r[ii]), r[ki].split("(")[0].replace("(anonymous namespace)::", "")), {})[r[mi]] = float(
            r[vi].replace(",", ""))
    lines = [f"# {title}", "", f"source: `{path}` (ncu --metrics, --clock-control none; cold-cache, serialised "
             "launches: compare shares, not absolute times)", "",
             "| id | kernel | time ms | share | metrics |", "|---|---|---|---|---|"]
    tot = sum(m.get("gpu__time_duration.sum", 0) for m in d.values())
    for (i, k), m in d.items():
        t = m.get("gpu__time_duration.sum", 0)
        extra = ", ".join(f"{n.split('__')[1]}={v:.4g}" for n, v in m.items() if n != "gpu__time_duration.sum")
        lines.append(f"| {i} | `{k[-60:]}` | {t / 1e6:.3f} | {t / tot * 100:.1f}% | {extra} |")
    lines.append("")
    lines.append(f"total {tot / 1e6:.3f} ms over {len(d)} launches")
    open(out, "w").write("\n".join(lines) + "\n")


def full(path, out, title):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    lines = [f"# {title}", "", f"source: `{path}` (ncu --set full --clock-control none)", ""]
    for r in rows[2:]:
        lines.append(f"## `{r[hdr.index('Kernel Name')][:110]}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for m in RAW:
            if m in hdr:
                lines.append(f"| {m} | {r[hdr.index(m)]} | {units[hdr.index(m)]} |")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        lines.append("")
        lines.append("top stall reasons (pc samples): " + ", ".join(f"{n} {int(v)}" for v, n in stalls[:6]))
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    title = sys.argv[4] if len(sys.argv) > 4 else dst
    (launches if kind == "launches" else full)(src, dst, title)
