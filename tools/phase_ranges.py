"""Per-phase share of a kernel's stall samples, warp instructions, SIMT
efficiency (thread instructions per warp instruction) and excess shared-memory
wavefronts (bank conflicts), phases given as source line ranges:
python tools/phase_ranges.py REPORT.ncu-rep LO:HI:NAME ...
(lines outside every range, e.g. inlined helpers above the kernel, are
reported as "other")."""
import csv
import subprocess
import sys

rep, specs = sys.argv[1], sys.argv[2:]
ph = [(int(a), int(b), n) for a, b, n in (s.split(":", 2) for s in specs)]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
ti = hdr.index("Thread Instructions Executed")
cw = hdr.index("L1 Wavefronts Shared Excessive")
acc, tot = {}, [0.0, 0.0]
for r in rows:
    try:
        ln = int(r[0])
        s, i, t, c = (float(r[k] or 0) for k in (si, ii, ti, cw))
    except (ValueError, IndexError):
        continue
    name = next((n for a, b, n in ph if a <= ln <= b), "other")
    a = acc.setdefault(name, [0.0] * 4)
    for k, v in enumerate((s, i, t, c)):
        a[k] += v
    tot[0] += s
    tot[1] += i
for k, a in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    print(f"| {k} | {100 * a[0] / tot[0]:.1f} % | {a[1] / 1e9:.3f} G ({100 * a[1] / tot[1]:.1f} %) | "
          f"{a[2] / max(a[1], 1):.1f} | {a[3] / 1e6:.1f} M |")
