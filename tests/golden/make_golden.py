"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference and oracle/_ref, built by
`make -C oracle ref`). Outputs are committed; nothing at test time reads
/root/reference.

* fig1.json — the 4x4 "Fig. 1" fixture of the reference test-suite
  (proj/tests/fixtures.hpp:25-115), parsed from that file: order values,
  expected desc/asc labels, the descending and Morse-Smale separator
  polylines and the ascending boundary edges.
* case_*.npz — 3-D cases run through the compiled reference library
  (oracle/_ref/libplmss_ref.so, proj/src/*.cpp unchanged): the float32 field,
  desc/asc/maxima/minima, ms_region/region_keys, per-cell codes, and for the
  separator / boundary meshes either the full arrays (small cases) or their
  SHA-256 digests plus counts (larger cases), so fixtures stay small.
"""
from __future__ import annotations

import hashlib
import json
import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure)
from paper_2303_15491_b200.configs import CONFIGS, host_field, scaled  # noqa: E402

FIXTURES = "/root/reference/proj/tests/fixtures.hpp"


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def parse_fig1() -> dict:
    src = open(FIXTURES).read()

    def arr(name):
        m = re.search(name + r"\s*=\s*\{([^}]*)\}", src)
        return [float(x) for x in m.group(1).replace("\n", " ").split(",") if x.strip()]

    def segs(fn):
        body = src[src.index(fn):]
        body = body[: body.index("return out;")]
        consts = {}
        for name, a, b in re.findall(r"(b\d[xy]) = ([\d.]+) / ([\d.]+)", body):
            consts[name] = float(a) / float(b)
        block = body[body.index("segs = {{") + len("segs = {"):]
        block = block[: block.index("}};") + 1]
        rows = re.findall(r"\{([^{}]*?)\}", block)
        out = []
        for r in rows:
            vals = [consts[t.strip()] if t.strip() in consts else float(t) for t in r.split(",")]
            if len(vals) == 4:
                out.append(vals)
        return out

    bnd = re.findall(r"\{(\d+), (\d+), (\d+)\}", src[src.index("fig1_asc_boundaries"):])
    return dict(
        dims=[4, 4, 1],
        order=arr("kFig1Order"),
        desc=[int(x) for x in arr("kFig1Desc")],
        asc=[int(x) for x in arr("kFig1Asc")],
        desc_separators=segs("fig1_desc_separators"),
        ms_separators=segs("fig1_ms_separators"),
        asc_boundaries=[[int(a), int(b), int(c)] for a, b, c in bnd],
        source="proj/tests/fixtures.hpp:25-115",
    )


def cases():
    rng = np.random.default_rng(20240317)
    out = []
    out.append(("noise_6x5x4", (6, 5, 4), rng.random(120).astype(np.float32), True))
    ties = rng.integers(0, 4, size=9 * 8 * 7).astype(np.float32)
    ties[rng.random(ties.size) < 0.2] = -0.0
    ties[ties == 0] = np.where(rng.random(int((ties == 0).sum())) < 0.5, -0.0, 0.0)
    out.append(("ties_9x8x7", (9, 8, 7), ties, True))
    out.append(("noise_12x12x12", (12, 12, 12), rng.random(12 ** 3).astype(np.float32), False))
    out.append(("gauss_17x13x11", (17, 13, 11), host_field(scaled(CONFIGS["cfg1"], (17, 13, 11))), False))
    out.append(("cfg1_64", (64, 64, 64), host_field(CONFIGS["cfg1"]), False))
    q = host_field(scaled(CONFIGS["cfg4"], (24, 20, 16)))
    out.append(("quant_24x20x16", (24, 20, 16), q, False))
    out.append(("slab_2x3x9", (2, 3, 9), rng.random(54).astype(np.float32), True))
    return out


def run_case(ref: oracle.Reference, name, dims, field, full):
    vals = field.astype(np.float64)
    rank = ref.compute_order(vals)
    seg = ref.segment(dims, rank, direction=2, workers=3, combine=True)
    rec = dict(name=name, dims=np.array(dims, np.int64), field=field.astype(np.float32))
    for k in ("desc", "asc", "maxima", "minima", "ms_region", "region_keys"):
        rec[k] = seg[k]
    sep = ref.emit_separators(dims, seg["ms_region"], workers=2)
    rec["codes"] = sep["codes"]
    rec["sep_count"] = np.int64(len(sep["source_cells"]))
    bnd = ref.emit_boundaries(dims, seg["asc"], workers=2)
    bms = ref.emit_boundaries(dims, seg["ms_region"], workers=2)
    sp = (2.0, 1.0, 3.0)
    og = (0.5, -1.25, 0.0)
    sep_sp = ref.emit_separators(dims, seg["ms_region"], workers=2, spacing=sp, origin=og)
    for tag, m in (("sep", sep), ("sepsp", sep_sp), ("bnd_asc", bnd), ("bnd_ms", bms)):
        for k in ("points", "indices", "regions", "source_cells"):
            if full:
                rec[f"{tag}_{k}"] = m[k]
            rec[f"{tag}_{k}_sha256"] = np.array(digest(m[k]))
        rec[f"{tag}_n"] = np.int64(len(m["source_cells"]))
    # union mode: asc then desc separators (marching.cpp:344-347)
    for tag, lab in (("sep_asc", seg["asc"]), ("sep_desc", seg["desc"])):
        m = ref.emit_separators(dims, lab, workers=2)
        rec[f"{tag}_n"] = np.int64(len(m["source_cells"]))
        for k in ("points", "regions", "source_cells"):
            rec[f"{tag}_{k}_sha256"] = np.array(digest(m[k]))
    return rec


def main():
    fig1 = parse_fig1()
    with open(os.path.join(HERE, "fig1.json"), "w") as f:
        json.dump(fig1, f, indent=1)
    ref = oracle.Reference()
    for name, dims, field, full in cases():
        rec = run_case(ref, name, dims, field, full)
        np.savez_compressed(os.path.join(HERE, f"case_{name}.npz"), **rec)
        print(name, dims, "tris", int(rec["sep_count"]), "regions", len(rec["region_keys"]))


if __name__ == "__main__":
    main()
