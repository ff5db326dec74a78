"""Per-basic-block instruction/stall breakdown of one kernel in an ncu report
(source page, SASS view): python tools/sass_hot.py REPORT KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"],
                     capture_output=True, text=True).stdout
import re

rows = list(csv.reader(out.splitlines()))
# the page lists each matching kernel (possibly twice): keep the first section
# whose name matches the pattern
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
sec = next(i for i in starts if re.search(kre, rows[i][1]))
end = next((i for i in starts if i > sec), len(rows))
rows = rows[sec:end]
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[hi]
ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
seq = []
for r in rows[hi + 1:]:
    try:
        seq.append((float(r[ie]), float(r[ss]), r[1].strip()))
    except (ValueError, IndexError):
        continue
tot_i = sum(v for v, _, _ in seq) or 1
tot_s = sum(s for _, s, _ in seq) or 1
blocks, cur, prev = [], [], None
for k, (v, s, src) in enumerate(seq):
    if prev is not None and abs(v - prev) > 0.05 * max(v, prev, 1):
        blocks.append(cur)
        cur = []
    cur.append((k, v, s, src))
    prev = v
blocks.append(cur)
res = sorted(((sum(v for _, v, _, _ in b), sum(s for _, _, s, _ in b), b) for b in blocks), key=lambda t: -t[0])
print(f"total warp-instr {tot_i:.4g}, stall samples {tot_s:.4g}")
for vi, si, b in res[:top]:
    print(f"{vi / tot_i * 100:5.1f}% instr {si / tot_s * 100:5.1f}% stall  sass {b[0][0]}-{b[-1][0]} n={len(b)} "
          f"x{b[0][1]:.3g}  {b[0][3][:60]}")
if len(sys.argv) > 4:
    lo, hi2 = map(int, sys.argv[4].split("-"))
    for k, (v, s, src) in enumerate(seq[lo:hi2 + 1], lo):
        print(f"{k:5d} {v:10.4g} {s:7.0f}  {src}")
