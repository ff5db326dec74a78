"""TEST INFRASTRUCTURE: a numpy backend with the contract of
paper_2303_15491_b200.distributed.B200SlabBackend (the four stages of the
z-slab pipeline, include/plmss_b200.h plmss_b200_slab_*) built on the CPU
restatement (oracle/), so the exchange / resolve / merge logic of the product
code runs on CPU with gloo (tests/test_distributed.py), and the device stages
can be compared with it stage by stage (tests/test_gpu_parity.py).

Stage semantics restated from the reference algorithm on a slab: steepest
hops (segmentation.cpp:60-85) over the slab plus its halo layers, halo
vertices as terminals, path compression to the fixpoint
(segmentation.cpp:87-168): every owned vertex ends at an owned extremum or
at the halo vertex where its chain leaves the slab (a portal).
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
from oracle import _dims
from paper_2303_15491_b200.distributed import FINAL, PORTAL

MASK = FINAL | PORTAL


class OracleSlabBackend:
    def __init__(self):
        self.R = oracle.Restatement()

    # stage 1
    def segment(self, dims, z0, z1, field_buf):
        X, Y, Z = (int(v) for v in dims)
        XY = X * Y
        h0, h1 = max(z0 - 1, 0), min(z1 + 1, Z)  # the buffer's layers (distributed.halo_bounds)
        nzx, lo, nz = h1 - h0, z0 - h0, z1 - z0
        self.dims, self.z0, self.z1, self.XY, self.nz, self.lo = (X, Y, Z), z0, z1, XY, nz, lo
        f = np.ascontiguousarray(field_buf.numpy().reshape(-1), dtype=np.float32)
        d = np.empty(nzx * XY, np.uint32)
        a = np.empty(nzx * XY, np.uint32)
        bad = self.R.lib.orc_seed_hops_f32(_dims((X, Y, nzx)), f, d, a)
        if bad >= 0:
            raise ValueError(f"non-finite scalar value at vertex {bad + h0 * XY}")
        idx = np.arange(nzx * XY, dtype=np.uint32)
        layer = idx // XY
        halo = (layer < lo) | (layer >= lo + nz)
        d[halo] = idx[halo]
        a[halo] = idx[halo]
        for p in (d, a):
            while True:
                q = p[p]
                if np.array_equal(q, p):
                    break
                p[:] = q
        own = slice(lo * XY, (lo + nz) * XY)
        self.ld, self.la = d[own].copy(), a[own].copy()
        oi = idx[own]
        self.max_ext = oi[self.ld == oi]  # ascending
        self.min_ext = oi[self.la == oi]
        gshift = np.int64(z0 * XY - lo * XY)
        self.sweeps = 1

        def value(lab, ext):
            z = lab // XY
            out = np.empty(lab.size, np.uint32)
            h = (z < lo) | (z >= lo + nz)
            side = (z[h] >= lo + nz).astype(np.uint32)
            out[h] = FINAL | PORTAL | (side * XY + lab[h] % XY)
            out[~h] = FINAL | np.searchsorted(ext, lab[~h]).astype(np.uint32)
            return out

        first, last = slice(0, XY), slice((nz - 1) * XY, nz * XY)
        bnd = np.stack([value(self.ld[first], self.max_ext), value(self.ld[last], self.max_ext),
                        value(self.la[first], self.min_ext), value(self.la[last], self.min_ext)])
        self.bnd = bnd
        self.vd, self.va = value(self.ld, self.max_ext), value(self.la, self.min_ext)
        return {"n_max": int(self.max_ext.size), "n_min": int(self.min_ext.size),
                "maxima": torch.from_numpy((self.max_ext.astype(np.int64) + gshift).astype(np.uint32).view(np.int32)),
                "minima": torch.from_numpy((self.min_ext.astype(np.int64) + gshift).astype(np.uint32).view(np.int32)),
                "boundary": torch.from_numpy(bnd.view(np.int32).copy()), "sweeps": self.sweeps}

    # stage 2
    def resolve(self, G, world, rank, max_counts, min_counts, maxima, minima):
        XY = self.XY
        G = G.numpy().view(np.uint32).reshape(world, 4, XY)
        pre = [np.concatenate([[0], np.cumsum(max_counts)]), np.concatenate([[0], np.cumsum(min_counts)])]

        def final(v, dr):
            out = np.empty(v.size, np.int64)
            port = (v & PORTAL) != 0
            out[~port] = (v[~port] & ~np.uint32(FINAL)).astype(np.int64) + pre[dr][rank]
            r = np.full(int(port.sum()), rank, np.int64)
            p = (v[port] & ~np.uint32(MASK)).astype(np.int64)
            res = np.empty(p.size, np.int64)
            todo = np.arange(p.size)
            for _ in range(1 << 20):
                if todo.size == 0:
                    break
                side = p[todo] >= XY
                xy = p[todo] - side * XY
                r2 = np.where(side, r[todo] + 1, r[todo] - 1)
                assert ((r2 >= 0) & (r2 < world)).all(), "portal chain leaves the volume"
                w = G[r2, dr * 2 + np.where(side, 0, 1), xy]
                fin = (w & PORTAL) == 0
                res[todo[fin]] = (w[fin] & ~np.uint32(FINAL)).astype(np.int64) + pre[dr][r2[fin]]
                r[todo[~fin]] = r2[~fin]
                p[todo[~fin]] = (w[~fin] & ~np.uint32(MASK)).astype(np.int64)
                todo = todo[~fin]
            out[port] = res
            return out

        self.rd, self.ra = final(self.vd, 0), final(self.va, 1)
        mx = maxima.numpy().view(np.uint32)
        mn = minima.numpy().view(np.uint32)
        self.maxima_all, self.minima_all = mx, mn
        self._desc = mx[self.rd]
        self._asc = mn[self.ra]
        self.pair = (self.ra.astype(np.uint64) << np.uint64(32)) | self.rd.astype(np.uint64)
        keys = np.unique(self.pair)
        return torch.from_numpy(keys.view(np.int64)), int(keys.size)

    # stage 3
    def ids(self, keys_all):
        u = np.unique(keys_all.numpy().view(np.uint64))
        self._ms = np.searchsorted(u, self.pair).astype(np.uint32)
        rk = (self.minima_all[(u >> np.uint64(32)).astype(np.int64)].astype(np.uint64) << np.uint64(32)) | \
            self.maxima_all[(u & np.uint64(0xFFFFFFFF)).astype(np.int64)].astype(np.uint64)
        has_up = self.z1 < self.dims[2]
        self._ms_ext = torch.zeros(self.nz * self.XY + (self.XY if has_up else 0), dtype=torch.int32)
        self._ms_ext[: self.nz * self.XY] = torch.from_numpy(self._ms.view(np.int32))
        return torch.from_numpy(rk.view(np.int64))

    def ms_ext(self):
        return self._ms_ext

    def ms(self):
        return self._ms_ext[: self.nz * self.XY]

    def desc(self):
        return torch.from_numpy(self._desc.view(np.int32))

    def asc(self):
        return torch.from_numpy(self._asc.view(np.int32))

    # stage 4
    def emit(self):
        X, Y, _ = self.dims
        lab = self._ms_ext.numpy().view(np.uint32)
        nzm = lab.size // self.XY
        if nzm < 2:
            return torch.empty((0, 2), dtype=torch.int64)
        rec = self.R.separator_records((X, Y, nzm), lab, 0, nzm - 1)
        cube0 = np.uint64(self.z0 * (X - 1) * (Y - 1))
        out = np.empty((rec.size, 2), np.uint64)
        out[:, 0] = rec["cellrow"] + ((np.uint64(6) * cube0) << np.uint64(6))
        out[:, 1] = rec["lo"].astype(np.uint64) | (rec["hi"].astype(np.uint64) << np.uint64(32))
        return torch.from_numpy(out.view(np.int64))
