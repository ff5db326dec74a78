"""The z-slab (multi-GPU) pipeline on the device: plmss_b200_slab_* through
B200SlabBackend, ranks run in lockstep in one process
(distributed.run_ranks_inprocess: no kernel of one rank waits on another, so
the results are those of world GPUs), and over NCCL at world size 1.

Checked against the single-volume oracle (small grids, bit for bit per rank)
and against the committed full-size oracle digests (BASELINE configs split
over up to 8 slabs): the concatenated rank outputs must equal the
single-volume outputs exactly."""
import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from test_distributed import check_rank, make_field, whole_volume

pytestmark = pytest.mark.gpu


def run_slabs(plmss, dims, world, field, combine_path=0):
    from paper_2303_15491_b200.distributed import (B200SlabBackend, run_ranks_inprocess, slab_bounds,
                                                   slab_field_buffer, slab_step)

    X, Y, Z = dims
    gens, ctxs = [], []
    for r in range(world):
        z0, z1 = slab_bounds(Z, world, r)
        ctx = plmss.Context(0)
        ctx.set_option(plmss.OPT_COMBINE_PATH, combine_path)
        ctxs.append(ctx)
        buf = slab_field_buffer(dims, world, r, "cuda", field[z0 * X * Y: z1 * X * Y])
        gens.append(slab_step(B200SlabBackend(ctx), dims, r, world, buf))
    res = run_ranks_inprocess(gens)
    torch.cuda.synchronize()
    return res, ctxs


CASES = [((12, 10, 96), 3, "gauss", 0), ((9, 8, 70), 2, "noise", 0), ((32, 33, 128), 4, "ties", 0),
         ((40, 24, 100), 3, "noise", 2), ((16, 12, 64), 1, "gauss", 0), ((20, 16, 160), 5, "ties", 2),
         ((8, 8, 33), 2, "noise", 0)]


@pytest.mark.parametrize("dims,world,kind,path", CASES)
def test_slab_ranks_match_single_volume_oracle(plmss, gpu, dims, world, kind, path):
    field = make_field(dims, kind, 3 * world + sum(dims))
    res, ctxs = run_slabs(plmss, dims, world, torch.from_numpy(field).cuda(), path)
    ref = whole_volume(dims, field)
    for r in res:
        check_rank(r, ref, dims)
    for c in ctxs:
        c.close()


def test_slab_stage1_matches_oracle_backend(plmss, gpu):
    """The device slab_segment outputs (extremum lists, boundary layers with
    portals) equal the numpy stage backend's word for word."""
    from paper_2303_15491_b200.distributed import B200SlabBackend, halo_bounds, slab_bounds
    from slab_oracle import OracleSlabBackend

    dims, world = (36, 20, 128), 4
    X, Y, Z = dims
    field = make_field(dims, "ties", 5)
    for r in range(world):
        z0, z1 = slab_bounds(Z, world, r)
        h0, h1 = halo_bounds(Z, world, r)
        buf = torch.from_numpy(field[h0 * X * Y: h1 * X * Y].copy())
        g = B200SlabBackend(gpu).segment(dims, z0, z1, buf.cuda())
        o = OracleSlabBackend().segment(dims, z0, z1, buf)
        for k in ("maxima", "minima", "boundary"):
            assert torch.equal(g[k].cpu(), o[k]), (r, k)
        assert (g["n_max"], g["n_min"]) == (o["n_max"], o["n_min"])


def test_slab_rejects_unaligned_and_out_of_order(plmss, gpu):
    import ctypes as C

    a = plmss.api
    info = a.PlmssSlabInfo()
    d = a._dims((16, 16, 64))
    f = torch.zeros(16 * 16 * 64, device="cuda")
    with pytest.raises(ValueError):
        a._check(a.lib().plmss_b200_slab_segment(gpu.h, d.ctypes.data, 16, 48, a._ptr(f), C.byref(info)))
    with pytest.raises(RuntimeError):  # stage 3 before stage 1/2
        a._check(a.lib().plmss_b200_slab_ids(gpu.h, None, 0, C.byref(info)))


def test_slab_over_nccl_world1_matches_pipeline(plmss, gpu):
    """TorchComm over NCCL (world size 1) with device tensors."""
    import socket

    import torch.distributed as dist

    from paper_2303_15491_b200.configs import CONFIGS, scaled
    from paper_2303_15491_b200.distributed import B200SlabBackend, ms_segmentation, slab_field_buffer

    if dist.is_initialized() or not dist.is_nccl_available():
        pytest.skip("a process group is already open / NCCL unavailable")
    cfg = scaled(CONFIGS["cfg2"], (96, 80, 64))
    f = plmss.synth_field(cfg.dims, kind=cfg.kind, gaussians=cfg.gaussians(), noise_amp=cfg.noise, seed=cfg.seed,
                          ctx=gpu)
    res = plmss.pipeline(cfg.dims, f, ctx=gpu)
    out = plmss.fetch(gpu, res)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        ctx = plmss.Context(0)
        s = ms_segmentation(slab_field_buffer(cfg.dims, 1, 0, "cuda", f), cfg.dims, B200SlabBackend(ctx))
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()
    for k in ("desc", "asc", "ms"):
        assert torch.equal(getattr(s, k).cpu(), out[k].cpu()), k
    assert s.tri_total == res.n_tris
    assert torch.equal(s.tris.cpu(), out["tris"].cpu())
    assert torch.equal(s.region_keys.cpu(), out["region_keys"].cpu())
    ctx.close()


# full-size configs split over slabs: (config, world, combine path)
FULL = [("cfg2", 1, 0), ("cfg2", 2, 0), ("cfg2", 8, 0), ("cfg2", 4, 2), ("cfg4", 8, 0), ("cfg3", 4, 0),
        ("cfg5", 8, 0)]


@pytest.mark.parametrize("name,world,path", FULL)
def test_slab_full_size_matches_oracle_digests(plmss, gpu, name, world, path):
    from paper_2303_15491_b200.configs import CONFIGS
    from paper_2303_15491_b200.digest import ChunkedSha256, digest_device

    p = os.path.join(GOLDEN, f"{name}_digest.json")
    if not os.path.exists(p):
        pytest.skip(f"{p} not generated")
    g = json.load(open(p))
    cfg = CONFIGS[name]
    gpu.release()  # the single-volume tests' buffers (cfg3: ~100 GB) are not needed here
    torch.cuda.empty_cache()
    f = plmss.synth_field(cfg.dims, kind=cfg.kind, gaussians=cfg.gaussians() if cfg.kind == "gaussians" else None,
                          noise_amp=cfg.noise, seed=cfg.seed, levels=cfg.levels, ctx=gpu)
    torch.cuda.synchronize()
    res, ctxs = run_slabs(plmss, cfg.dims, world, f, path)
    del f
    try:
        h = {k: ChunkedSha256() for k in ("desc", "asc", "ms", "tris")}
        for r in res:
            for k in h:
                t = getattr(r, k).reshape(-1)
                for i in range(0, t.numel(), 1 << 28):
                    h[k].update(t[i:i + (1 << 28)].cpu().numpy()).drain()
        got = {k: v.hexdigest() for k, v in h.items()}
        got["maxima"] = digest_device(res[0].maxima)
        got["minima"] = digest_device(res[0].minima)
        got["region_keys"] = digest_device(res[0].region_keys)
        assert res[0].tri_total == g["n_tris"]
        assert (res[0].maxima.numel(), res[0].minima.numel(), res[0].region_keys.numel()) == \
            (g["n_maxima"], g["n_minima"], g["n_regions"])
        bad = [k for k in got if got[k] != g[k]]
        assert not bad, f"{name} over {world} slabs: digests differ for {bad}"
    finally:
        del res
        for c in ctxs:
            c.close()
