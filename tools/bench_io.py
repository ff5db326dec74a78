"""Measurement of the callers either side of the path:
volume ingest, label / OBJ writers and point welding, B200 implementation vs
the compiled reference (oracle/_ref, CPU) on the same inputs. Prints one JSON
object. Run on the GPU box: python tools/bench_io.py [--dims 512 512 256]."""
import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=3):
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs=3, default=[512, 512, 256])
    ap.add_argument("--sep-dims", type=int, nargs=3, default=[128, 128, 128])
    args = ap.parse_args()
    import torch

    import oracle
    import paper_2303_15491_b200 as P
    from paper_2303_15491_b200 import configs

    ctx = P.default_context(0)
    ref = oracle.Reference()
    res = {"host_threads": os.cpu_count()}
    tmp = tempfile.mkdtemp(dir="/tmp")
    # ---- read_volume: f32le file (page cache warm) -> device f32 / host f64
    dims = tuple(args.dims)
    n = int(np.prod(dims))
    c2 = configs.scaled(configs.CONFIGS["cfg2"], dims)
    f = P.synth_field(dims, "gaussians", gaussians=c2.gaussians(), noise_amp=c2.noise, seed=c2.seed, ctx=ctx)
    path = os.path.join(tmp, "vol.raw")
    f.cpu().numpy().astype("<f4").tofile(path)
    t_mine, d = timed(lambda: (P.read_volume(path, dims, "f32le", ctx=ctx), torch.cuda.synchronize()))
    t_ref, v = timed(lambda: ref.read_volume(path, dims, "f32le"), reps=1)
    assert np.array_equal(P.read_volume(path, dims, "f32le", out="f64", ctx=ctx).cpu().numpy(), v)
    res["read_volume"] = {"bytes": 4 * n, "b200_GBps": 4 * n / t_mine / 1e9, "reference_GBps": 4 * n / t_ref / 1e9,
                          "note": "file in page cache; B200: pread into pinned chunks, H2D + convert on device"}
    # ---- write_labels from the device segmentation
    seg = P.segment(dims, f, ctx=ctx)
    lp, rp = os.path.join(tmp, "mine.lbl"), os.path.join(tmp, "ref.lbl")
    t_mine, _ = timed(lambda: P.write_labels(lp, seg.asc, seg.desc, ctx=ctx))
    asc = (seg.asc.to(torch.int64) & 0xFFFFFFFF).cpu().numpy()
    desc = (seg.desc.to(torch.int64) & 0xFFFFFFFF).cpu().numpy()
    t_ref, _ = timed(lambda: ref.write_labels(rp, asc, desc), reps=1)
    same = open(lp, "rb").read() == open(rp, "rb").read()
    res["write_labels"] = {"bytes": 20 + 16 * n, "b200_GBps": (20 + 16 * n) / t_mine / 1e9,
                           "reference_GBps": (20 + 16 * n) / t_ref / 1e9, "identical": same}
    # ---- separators of a smaller field: weld_points and write_surface_obj
    sd = tuple(args.sep_dims)
    c1 = configs.scaled(configs.CONFIGS["cfg1"], sd)
    fs = P.synth_field(sd, "gaussians", gaussians=c1.gaussians(), noise_amp=c1.noise, seed=c1.seed, ctx=ctx)
    r = P.pipeline(sd, fs, ctx=ctx)
    out = P.fetch(ctx, r)
    m = P.materialize_separators(sd, out["tris"], ctx=ctx)
    pts, idx = m["points"], m["indices"]
    hp, hi = pts.cpu().numpy(), idx.cpu().numpy()

    def weld():
        p2, i2 = P.weld_points(pts.clone(), idx.clone(), ctx=ctx)
        torch.cuda.synchronize()
        return p2, i2

    t_mine, (wp, wi) = timed(weld)
    t_ref, (rp2, ri2) = timed(lambda: ref.weld_points(hp, hi), reps=1)
    res["weld_points"] = {"points": int(pts.shape[0]), "unique": int(wp.shape[0]),
                          "b200_Mpoints_s": pts.shape[0] / t_mine / 1e6, "reference_Mpoints_s": pts.shape[0] / t_ref / 1e6,
                          "identical": bool(np.array_equal(wp.cpu().numpy().view(np.uint64), rp2.view(np.uint64))
                                            and np.array_equal(wi.cpu().numpy(), ri2))}
    op, orf = os.path.join(tmp, "mine.obj"), os.path.join(tmp, "ref.obj")
    t_mine, _ = timed(lambda: P.write_surface_obj(op, wp, wi, m["regions"], ctx=ctx), reps=1)
    t_ref, _ = timed(lambda: ref.write_surface_obj(orf, wp.cpu().numpy(), wi.cpu().numpy(),
                                                   m["regions"].cpu().numpy()), reps=1)
    sz = os.path.getsize(op)
    res["write_surface_obj"] = {"bytes": sz, "b200_MBps": sz / t_mine / 1e6, "reference_MBps": sz / t_ref / 1e6,
                                "identical": open(op, "rb").read() == open(orf, "rb").read()}
    res["dims"], res["sep_dims"] = list(dims), list(sd)
    print(json.dumps(res))
    for fn in os.listdir(tmp):
        os.remove(os.path.join(tmp, fn))
    os.rmdir(tmp)


if __name__ == "__main__":
    main()
