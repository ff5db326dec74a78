"""Multi-rank z-slab path (paper_2303_15491_b200/distributed.py) on CPU with
gloo, world sizes 1-3: every rank's slice of desc/asc/ms, the global extrema
lists, region table and separator records must equal the single-process
oracle bit for bit. The per-slab compute is the CPU restatement (test
backend); the exchange / resolve / merge logic is the product code."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


class OracleBackend:
    """Test stand-in for B200Backend: same contract, CPU restatement."""

    def __init__(self):
        import oracle

        self.R = oracle.Restatement()

    def segment_slab(self, dims, field_ext, halo_lo, halo_hi):
        X, Y, Z = dims
        XY = X * Y
        d, a = self.R.seed_hops(dims, values=field_ext.numpy().astype(np.float64))
        if halo_lo:
            d[:XY] = np.arange(XY)
            a[:XY] = np.arange(XY)
        if halo_hi:
            d[-XY:] = np.arange(X * Y * (Z - 1), X * Y * Z)
            a[-XY:] = np.arange(X * Y * (Z - 1), X * Y * Z)
        self.R.lib.orc_compress(d.size, d, a)
        return torch.from_numpy(d), torch.from_numpy(a)

    def march_slab(self, dims, ms_ext):
        e = self.R.emit_separators(dims, ms_ext.numpy().astype(np.int64))
        return (torch.from_numpy(e["source_cells"].copy()), torch.from_numpy(e["regions"][:, 0].copy()),
                torch.from_numpy(e["regions"][:, 1].copy()))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dims, field, errq):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2303_15491_b200.distributed import ms_segmentation, slab_bounds

        X, Y, Z = dims
        z0, z1 = slab_bounds(Z, world, rank)
        own = torch.from_numpy(field[z0 * X * Y: z1 * X * Y].copy())
        res = ms_segmentation(own, dims, OracleBackend())
        # single-process oracle of the whole volume
        import oracle

        R = oracle.Restatement()
        s = R.segment(dims, values=field.astype(np.float64))
        ms, keys = R.combine_ms(s["asc"], s["desc"])
        e = R.emit_separators(dims, ms)
        sl = slice(z0 * X * Y, z1 * X * Y)
        assert np.array_equal(res.desc.numpy(), s["desc"][sl]), "desc"
        assert np.array_equal(res.asc.numpy(), s["asc"][sl]), "asc"
        assert np.array_equal(res.ms.numpy(), ms[sl]), "ms"
        assert np.array_equal(res.maxima.numpy(), s["maxima"]), "maxima"
        assert np.array_equal(res.minima.numpy(), s["minima"]), "minima"
        assert np.array_equal(res.region_keys.numpy(), keys), "region keys"
        assert res.tri_total == len(e["source_cells"]), "triangle total"
        rs = slice(res.tri_base, res.tri_base + res.cells.shape[0])
        assert np.array_equal(res.cells.numpy(), e["source_cells"][rs]), "cells"
        assert np.array_equal(res.lo.numpy(), e["regions"][rs, 0]), "lo"
        assert np.array_equal(res.hi.numpy(), e["regions"][rs, 1]), "hi"
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # report to the parent
        import traceback

        errq.put(f"rank {rank}: {ex}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world,dims,kind", [(1, (7, 6, 5), "noise"), (2, (9, 8, 12), "noise"),
                                             (3, (10, 7, 9), "ties"), (2, (16, 12, 10), "gauss"),
                                             (3, (6, 5, 4), "noise")])
def test_zslab_ranks_match_single_process_oracle(world, dims, kind):
    rng = np.random.default_rng(sum(dims) + world)
    n = int(np.prod(dims))
    if kind == "noise":
        field = rng.random(n).astype(np.float32)
    elif kind == "ties":
        field = rng.integers(0, 3, n).astype(np.float32)
    else:
        from paper_2303_15491_b200.configs import CONFIGS, host_field, scaled

        field = host_field(scaled(CONFIGS["cfg1"], dims))
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
