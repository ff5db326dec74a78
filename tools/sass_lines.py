"""Instructions executed and stall samples per source line of one kernel in an
ncu report, each SASS instruction counted once (inlined helpers are listed
under every line of their inline stack; an instruction is charged to the
innermost attribution inside [LO, HI], the kernel body):
python tools/sass_lines.py REPORT KERNEL_REGEX SOURCE.cu LO HI [MIN_PCT]"""
import csv
import re
import subprocess
import sys

rep, kre, src, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
min_pct = float(sys.argv[6]) if len(sys.argv) > 6 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fn = [i for i, r in enumerate(rows) if r and r[0] == "Function Name"]
sec = next(i for i in fn if re.search(kre, rows[i][1]))
end = next((i for i in fn if i > sec), len(rows))
hdr = rows[sec + 1]
si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
by_addr = {}
cur = None
for r in rows[sec + 2:end]:
    if not r:
        continue
    if r[0]:
        try:
            cur = int(r[0])
        except ValueError:
            cur = None
    if cur is None or len(r) <= ii:
        continue
    try:
        addr = int(r[2], 16)
        ins, smp = float(r[ii] or 0), float(r[si] or 0)
    except ValueError:
        continue
    a = by_addr.setdefault(addr, [[], ins, smp, r[3].strip()])
    a[0].append(cur)
acc = {}
for addr, (lines, ins, smp, sass) in by_addr.items():
    inside = [x for x in lines if lo <= x <= hi]
    ln = max(inside) if inside else max(lines)
    a = acc.setdefault(ln, [0.0, 0.0])
    a[0] += ins
    a[1] += smp
ti = sum(a[0] for a in acc.values()) or 1.0
ts = sum(a[1] for a in acc.values()) or 1.0
text = open(src).read().splitlines()
print(f"total instructions {ti:.4g}, samples {ts:.4g}")
for ln in sorted(acc):
    i, s = acc[ln]
    if 100 * i / ti >= min_pct or 100 * s / ts >= min_pct:
        print(f"{ln:5d} {100 * i / ti:5.1f}% {100 * s / ts:5.1f}%  {text[ln - 1].strip()[:100] if ln <= len(text) else ''}")
