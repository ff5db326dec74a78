"""profiles/traffic.json from an ncu launch list of one bench step
(`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,... --csv`):
DRAM bytes (read + write) per pipeline stage, summed over each stage's
launches in launch order (bench.py reports the dominant stage's value).

usage: python tools/traffic.py LAUNCHES.csv [OUT.json]"""
import csv
import json
import sys


def stage_of(name, seen):
    if "k_synth" in name or "k_march_init" in name or "k_minmax" in name or "k_quantise" in name:
        return None
    if "k_tile_segment" in name or "k_hop_codes" in name:
        return "tile_segment"
    if "k_tt_succ" in name or "k_tt_jump" in name:
        seen.add("B")
        return "exit_resolve"
    if "E" in seen:
        return None  # the step ended with its emission (later launches: other bench legs)
    if "k_emit_chunks" in name:
        seen.add("E")
        return "march"
    if "k_ms_ids" in name:
        seen.add("D")
        return "march"
    if "D" in seen:
        return "march"
    return "finalize_ids" if "B" in seen else "extrema_sort"


def main():
    src = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic.json"
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = {}
    names = {}
    for r in rows[1:]:
        if r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            per[int(r[ii])] = per.get(int(r[ii]), 0.0) + float(r[vi].replace(",", ""))
            names[int(r[ii])] = r[ki]
    seen, tot = set(), {}
    for i in sorted(per):
        st = stage_of(names[i], seen)
        if st:
            tot[st] = tot.get(st, 0.0) + per[i]
    d = {"_source": f"{src} (dram__bytes_read.sum + dram__bytes_write.sum per launch, cfg5 1024^3), summed over "
                    "each stage's kernels in launch order"}
    d.update(tot)
    d["_total"] = sum(tot.values())
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
