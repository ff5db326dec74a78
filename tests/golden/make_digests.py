"""Full-size oracle digests of the five BASELINE configs -> tests/golden/cfgN_digest.json.

TEST INFRASTRUCTURE (run in the build container; needs oracle/_ref, i.e.
/root/reference, and ~45 GB of RAM for cfg5). The GPU tests and bench.py
compare the device pipeline against these digests on the GPU box, where
neither /root/reference nor the host RAM for the oracle exists.

Per config:
* the field, from the host half of the input definition
  (include/plmss_synth.h via oracle orc_synth) — its digest pins the device
  generator to the same bytes;
* labels (desc, asc, maxima, minima), dense MS ids and region keys from the
  full-size C restatement (oracle/plmss_oracle_big.c); for cfg1-cfg4 also
  from the compiled reference itself (compute_order + segment(Both) +
  combine_ms, proj/src/{orderfield,segmentation}.cpp) and required equal —
  cfg5 needs ~100 GB in the reference's int64 / 128-bit layout, so its labels
  rest on the restatement (pinned by the cfg1-cfg4 equality);
* MS separator records (cell << 6 | recipe row, lo, hi) from the compiled
  reference's emit_separators in z-chunks (rows checked
  against the reference's own points, oracle/ref_capi.cpp cap_records_chunk)
  and required equal to the restatement's records chunk by chunk.

Digests: paper_2303_15491_b200/digest.py (chunked SHA-256 of the raw
little-endian bytes: u32 labels, u64 keys asc << 32 | desc, 16-byte records).

usage: python tests/golden/make_digests.py [cfg1 cfg2 ...] [--workers N]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2303_15491_b200.configs import CONFIGS  # noqa: E402
from paper_2303_15491_b200.digest import ChunkedSha256, digest  # noqa: E402


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def make(name: str, workers: int, chunk_layers: int) -> dict:
    cfg = CONFIGS[name]
    X, Y, Z = cfg.dims
    XY = X * Y
    R = oracle.Restatement()
    F = oracle.Reference()
    t0 = time.time()
    f = R.synth(cfg)
    log(name, "field", f"{time.time() - t0:.1f}s")
    out = {"config": name, "workload": cfg.name, "dims": list(cfg.dims), "field": digest(f)}
    s = R.segment_u32(cfg.dims, f)
    log(name, "segment", f"{time.time() - t0:.1f}s", "sweeps", s["sweeps"])
    ms, keys = R.combine_ms_u32(s["asc"], s["desc"])
    log(name, "combine", f"{time.time() - t0:.1f}s", "regions", keys.size)
    sources = {"labels": "restatement (oracle/plmss_oracle_big.c)"}
    if cfg.n <= (1 << 27):
        rank = F.compute_order(f.astype(np.float64))
        ref = F.segment(cfg.dims, rank, direction=2, workers=workers, combine=True)
        del rank
        ok = (np.array_equal(ref["desc"], s["desc"]) and np.array_equal(ref["asc"], s["asc"])
              and np.array_equal(ref["maxima"], s["maxima"]) and np.array_equal(ref["minima"], s["minima"])
              and np.array_equal(ref["ms_region"], ms))
        rk = ref["region_keys"]
        ok = ok and np.array_equal((rk[:, 0].astype(np.uint64) << np.uint64(32)) | rk[:, 1].astype(np.uint64), keys)
        if not ok:
            raise SystemExit(f"{name}: restatement labels differ from the compiled reference")
        del ref
        sources["labels"] = "compiled reference (orderfield/segmentation.cpp) == restatement"
        log(name, "reference labels equal", f"{time.time() - t0:.1f}s")
    out.update(n_maxima=int(s["maxima"].size), n_minima=int(s["minima"].size), n_regions=int(keys.size),
               desc=digest(s["desc"]), asc=digest(s["asc"]), ms=digest(ms), maxima=digest(s["maxima"]),
               minima=digest(s["minima"]), region_keys=digest(keys))
    del s, f
    # separators, z-chunk by z-chunk: reference records == restatement records
    h = ChunkedSha256()
    total = 0
    chunk_counts = []
    for cz0 in range(0, Z - 1, chunk_layers):
        cz1 = min(cz0 + chunk_layers, Z - 1)
        lab = ms[cz0 * XY:(cz1 + 1) * XY].astype(np.int64)
        rec = F.records_chunk(cfg.dims, lab, cz0, cz1, workers=workers)
        mine = R.separator_records(cfg.dims, ms, cz0, cz1)
        if not np.array_equal(rec, mine):
            raise SystemExit(f"{name}: reference / restatement records differ in cube layers [{cz0}, {cz1})")
        h.update(rec)
        total += rec.size
        chunk_counts.append(int(rec.size))
    sources["separators"] = "compiled reference emit_separators in z-chunks == restatement"
    out.update(n_tris=total, tris=h.hexdigest(), tri_chunk_layers=chunk_layers, tri_chunk_counts=chunk_counts,
               sources=sources, digest="chunked sha256 (paper_2303_15491_b200/digest.py), raw little-endian")
    log(name, "separators", total, f"{time.time() - t0:.1f}s")
    return out


def add_geometry(name: str, workers: int, chunk_layers: int) -> dict:
    """Digests of the reference SeparatingMesh arrays (marching.hpp:65-76:
    points, regions, source_cells) of an existing digest file's config, from
    the compiled reference's emit_separators in z-chunks; the chunks' records
    must reproduce the file's record digest."""
    path = os.path.join(HERE, f"{name}_digest.json")
    out = json.load(open(path))
    cfg = CONFIGS[name]
    X, Y, Z = cfg.dims
    XY = X * Y
    R = oracle.Restatement()
    F = oracle.Reference()
    t0 = time.time()
    s = R.segment_u32(cfg.dims, R.synth(cfg))
    ms, _ = R.combine_ms_u32(s["asc"], s["desc"])
    del s
    hs = {k: ChunkedSha256() for k in ("tris", "points", "regions", "source_cells")}
    for cz0 in range(0, Z - 1, chunk_layers):
        cz1 = min(cz0 + chunk_layers, Z - 1)
        rec, geo = F.records_chunk(cfg.dims, ms[cz0 * XY:(cz1 + 1) * XY].astype(np.int64), cz0, cz1,
                                   workers=workers, geometry=True)
        hs["tris"].update(rec)
        for k in ("points", "regions", "source_cells"):
            hs[k].update(geo[k])
        del rec, geo
        for h in hs.values():
            h.drain()
    got = {k: h.hexdigest() for k, h in hs.items()}
    if got.pop("tris") != out["tris"]:
        raise SystemExit(f"{name}: geometry pass records differ from the stored record digest")
    out["geometry"] = dict(got, source="compiled reference emit_separators in z-chunks (SeparatingMesh arrays: "
                                       "points f64 x3 per corner, regions i64 x2, source_cells i64)")
    log(name, "geometry", f"{time.time() - t0:.1f}s")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--chunk-layers", type=int, default=16)
    ap.add_argument("--geometry", action="store_true", help="add SeparatingMesh digests to existing files")
    args = ap.parse_args()
    for name in args.configs:
        d = add_geometry(name, args.workers, args.chunk_layers) if args.geometry else \
            make(name, args.workers, args.chunk_layers)
        with open(os.path.join(HERE, f"{name}_digest.json"), "w") as fh:
            json.dump(d, fh, indent=1)
            fh.write("\n")


if __name__ == "__main__":
    main()
