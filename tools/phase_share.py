"""Share of warp-stall samples (~ time) and executed instructions per phase
of a kernel, phases delimited by marker comments in the source file:
python tools/phase_share.py REPORT SOURCE.cu KERNEL_REGEX 'marker1' 'marker2' ..."""
import csv
import re
import subprocess
import sys

rep, src, kre = sys.argv[1], sys.argv[2], sys.argv[3]
markers = sys.argv[4:]
lines = open(src).read().splitlines()
starts = []
for m in markers:
    starts.append(next(i + 1 for i, l in enumerate(lines) if m in l))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fn = [i for i, r in enumerate(rows) if r and r[0] == "Function Name"]
sec = next(i for i in fn if re.search(kre, rows[i][1]))
end = next((i for i in fn if i > sec), len(rows))
hdr = rows[sec + 1]
si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
acc = {}
tot_s = tot_i = 0.0
for r in rows[sec + 2:end]:
    if not r or not r[0]:
        continue
    try:
        ln, smp, ins = int(r[0]), float(r[si]), float(r[ii])
    except ValueError:
        continue
    ph = "pre"
    for name, st in zip(markers, starts):
        if ln >= st:
            ph = name
    if ln < min(starts) or ln > len(lines):
        ph = "other(%s)" % ("header" if ln < min(starts) else "?")
    a = acc.setdefault(ph, [0.0, 0.0])
    a[0] += smp
    a[1] += ins
    tot_s += smp
    tot_i += ins
for k, (smp, ins) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    print(f"{k[:50]:50s} samples {100 * smp / tot_s:5.1f}%  instr {100 * ins / tot_i:5.1f}%")
