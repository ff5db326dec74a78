"""Multi-rank z-slab path (paper_2303_15491_b200/distributed.py) on CPU:
gloo at world sizes 1-3 (one process per rank, the product TorchComm) and the
in-process lockstep runner at larger world sizes. Every rank's slice of
desc / asc / ms, the global extremum lists, region table and separator
records must equal the single-volume oracle bit for bit. The per-slab
compute is the numpy stage backend (tests/slab_oracle.py, the contract of
B200SlabBackend); the exchange / resolve / merge logic is the product code."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make_field(dims, kind, seed):
    rng = np.random.default_rng(seed)
    n = int(np.prod(dims))
    if kind == "noise":
        return rng.random(n).astype(np.float32)
    if kind == "ties":
        return rng.integers(0, 3, n).astype(np.float32)
    from paper_2303_15491_b200.configs import CONFIGS, host_field, scaled

    return host_field(scaled(CONFIGS["cfg1"], dims))


def whole_volume(dims, field):
    """Single-process oracle: labels, ids, region keys, separator records."""
    import oracle

    R = oracle.Restatement()
    s = R.segment_u32(dims, field)
    ms, keys = R.combine_ms_u32(s["asc"], s["desc"])
    rec = R.separator_records(dims, ms, 0, dims[2] - 1)
    tris = np.empty((rec.size, 2), np.uint64)
    tris[:, 0] = rec["cellrow"]
    tris[:, 1] = rec["lo"].astype(np.uint64) | (rec["hi"].astype(np.uint64) << np.uint64(32))
    return dict(s, ms=ms, keys=keys, tris=tris)


def check_rank(res, ref, dims):
    X, Y, _ = dims
    sl = slice(res.z0 * X * Y, res.z1 * X * Y)
    u32 = lambda t: t.cpu().numpy().view(np.uint32)  # noqa: E731
    assert np.array_equal(u32(res.desc), ref["desc"][sl]), "desc"
    assert np.array_equal(u32(res.asc), ref["asc"][sl]), "asc"
    assert np.array_equal(u32(res.ms), ref["ms"][sl]), "ms"
    assert np.array_equal(u32(res.maxima), ref["maxima"]), "maxima"
    assert np.array_equal(u32(res.minima), ref["minima"]), "minima"
    assert np.array_equal(res.region_keys.cpu().numpy().view(np.uint64), ref["keys"]), "region keys"
    assert res.tri_total == ref["tris"].shape[0], "triangle total"
    rs = slice(res.tri_base, res.tri_base + res.tris.shape[0])
    assert np.array_equal(res.tris.cpu().numpy().view(np.uint64), ref["tris"][rs]), "records"


def _worker(rank, world, port, dims, field, errq):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2303_15491_b200.distributed import ms_segmentation, slab_bounds, slab_field_buffer
        from slab_oracle import OracleSlabBackend

        X, Y, Z = dims
        z0, z1 = slab_bounds(Z, world, rank)
        buf = slab_field_buffer(dims, world, rank, "cpu", torch.from_numpy(field[z0 * X * Y: z1 * X * Y].copy()))
        res = ms_segmentation(buf, dims, OracleSlabBackend())
        check_rank(res, whole_volume(dims, field), dims)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # report to the parent
        import traceback

        errq.put(f"rank {rank}: {ex}\n{traceback.format_exc()}")
        raise


CASES = [(1, (7, 6, 5), "noise"), (2, (9, 8, 40), "noise"), (3, (10, 7, 96), "ties"), (2, (16, 12, 64), "gauss"),
         (3, (6, 5, 70), "noise"), (2, (5, 4, 33), "ties")]


@pytest.mark.parametrize("world,dims,kind", CASES)
def test_zslab_gloo_ranks_match_single_volume_oracle(world, dims, kind):
    field = make_field(dims, kind, sum(dims) + world)
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, field, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)


@pytest.mark.parametrize("world,dims,kind", [(4, (8, 7, 128), "noise"), (5, (6, 9, 150), "ties"),
                                             (3, (12, 10, 96), "gauss")])
def test_zslab_inprocess_ranks_match_single_volume_oracle(world, dims, kind):
    """The lockstep runner (used on one GPU for the device parity tests)."""
    from paper_2303_15491_b200.distributed import run_ranks_inprocess, slab_bounds, slab_field_buffer, slab_step
    from slab_oracle import OracleSlabBackend

    field = make_field(dims, kind, 7 * world + sum(dims))
    X, Y, Z = dims
    gens = []
    for r in range(world):
        z0, z1 = slab_bounds(Z, world, r)
        buf = slab_field_buffer(dims, world, r, "cpu", torch.from_numpy(field[z0 * X * Y: z1 * X * Y].copy()))
        gens.append(slab_step(OracleSlabBackend(), dims, r, world, buf))
    ref = whole_volume(dims, field)
    for res in run_ranks_inprocess(gens):
        check_rank(res, ref, dims)


def test_slab_bounds_are_whole_brick_layers():
    from paper_2303_15491_b200.distributed import halo_bounds, slab_bounds

    for Z in (2, 31, 32, 33, 100, 1024):
        nb = (Z + 31) // 32
        for world in range(1, min(nb, 9) + 1):
            bounds = [slab_bounds(Z, world, r) for r in range(world)]
            assert bounds[0][0] == 0 and bounds[-1][1] == Z
            for (a0, a1), (b0, b1) in zip(bounds, bounds[1:]):
                assert a1 == b0 and a0 % 32 == 0 and a1 % 32 == 0 and a1 > a0
            for r, (z0, z1) in enumerate(bounds):
                assert halo_bounds(Z, world, r) == (max(z0 - 1, 0), min(z1 + 1, Z))
    with pytest.raises(ValueError):
        slab_bounds(64, 3, 0)
