"""One pipeline case for compute-sanitizer (tools/sanitize.sh): a BASELINE
config's field generated on the device, the fused pipeline with the given
options, every output digest compared with tests/golden/<cfg>_digest.json;
then the staged reference-API kernels (segment, combine_ms,
emit_separators) on a sub-volume. Exit 0 only when everything matches.

usage: python tools/sanitize_case.py cfg1 [--spec 0|1|2] [--path 0|1|2] [--staged]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--spec", type=int, default=1)
    ap.add_argument("--path", type=int, default=0)
    ap.add_argument("--staged", action="store_true")
    a = ap.parse_args()
    import torch

    import paper_2303_15491_b200 as P
    from paper_2303_15491_b200.configs import CONFIGS

    cfg = CONFIGS[a.config]
    g = json.load(open(os.path.join(ROOT, "tests", "golden", f"{a.config}_digest.json")))
    ctx = P.Context(0)
    f = P.synth_field(cfg.dims, kind=cfg.kind, gaussians=cfg.gaussians() if cfg.kind == "gaussians" else None,
                      noise_amp=cfg.noise, seed=cfg.seed, levels=cfg.levels, ctx=ctx)
    ctx.set_option(P.OPT_SPECULATIVE_SWEEPS, a.spec)
    ctx.set_option(P.OPT_COMBINE_PATH, a.path)
    res = P.pipeline(cfg.dims, f, ctx=ctx)
    got = P.result_digests(ctx, res)
    bad = [k for k in ("desc", "asc", "ms", "maxima", "minima", "region_keys", "tris") if got[k] != g[k]]
    print(f"{a.config} spec={a.spec} path={a.path}: sweeps={res.sweeps} tris={res.n_tris} "
          f"regions={res.n_regions} mismatched={bad}", flush=True)
    ok = not bad
    if a.staged:
        # the reference-API kernels (staged path) on the first 24 layers
        X, Y, _ = cfg.dims
        dims = (X, Y, 24)
        sub = f[: X * Y * 24].clone()
        seg = P.segment(dims, sub, direction=P.BOTH, ctx=ctx)
        seg = P.combine_ms(seg, ctx=ctx)
        rec = P.emit_separators(dims, seg.ms_region, ctx=ctx)
        torch.cuda.synchronize()
        pres = P.pipeline(dims, sub, ctx=ctx)
        out = P.fetch(ctx, pres)
        same = all(torch.equal((getattr(seg, k).to(torch.int64) & 0xFFFFFFFF).cpu(),
                               (out[o].to(torch.int64) & 0xFFFFFFFF).cpu())
                   for k, o in (("desc", "desc"), ("asc", "asc"), ("ms_region", "ms")))
        same = same and torch.equal(rec.cpu(), out["tris"].view(torch.int64).reshape(-1, 2).cpu())
        print(f"staged API vs fused on {dims}: labels and records equal={same}, records={rec.shape[0]}", flush=True)
        ok = ok and same
    ctx.close()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
