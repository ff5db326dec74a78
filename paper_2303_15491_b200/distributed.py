"""Z-slab decomposition of the full Morse-Smale segmentation over ranks.

One process per GPU (torch.distributed, NCCL on B200 / gloo on CPU). Rank r
owns the z-layers [z0, z1) = [Z*r/P, Z*(r+1)/P) — whole layers, so rank order
is the reference's global vertex and cell order. Exchange
steps, each one collective:

1. field halo: the neighbours' boundary layers (one X*Y layer each way,
   point-to-point);
2. slab segmentation on the device with the halo layers as terminals
   (plmss_b200_segment_slab): every owned label is then a root of the slab or
   a halo vertex;
3. boundary graph: all_gather of every rank's two boundary layers of labels;
   every rank resolves the (acyclic: strictly monotone chains) boundary graph
   by pointer jumping and fixes its halo-pointing labels — one exchange, no
   iteration across ranks;
4. extrema: all_gather of counts and the per-rank sorted lists (rank order is
   id order);
5. Morse-Smale ids: all_gather of each rank's sorted unique (asc, desc) keys,
   global sorted merge -> identical dense ids everywhere (combine_ms order);
6. marching: the next rank's first layer of ids (point-to-point), local
   separator records for the owned cube layers, global cell ids, and base
   offsets from an all_gather of the per-rank counts.

The per-slab device work is delegated to a backend (``B200Backend`` below, the
product path over the C-ABI). Everything here is plain tensor plumbing and
runs unchanged on CPU tensors with gloo (tests/test_distributed.py).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


def slab_bounds(Z: int, world: int, rank: int):
    """Owned z-layers of a rank (the even split of parallel.hpp:27-29)."""
    return Z * rank // world, Z * (rank + 1) // world


@dataclass
class SlabResult:
    z0: int
    z1: int
    desc: torch.Tensor        # int64 global extremum ids of the owned vertices
    asc: torch.Tensor
    ms: torch.Tensor          # int64 dense region ids of the owned vertices
    maxima: torch.Tensor      # global, ascending (identical on every rank)
    minima: torch.Tensor
    region_keys: torch.Tensor  # (R, 2) int64 (min id, max id), global
    cells: torch.Tensor       # this rank's separator records, reference order
    lo: torch.Tensor
    hi: torch.Tensor
    tri_base: int             # offset of this rank's records in the global list
    tri_total: int


class B200Backend:
    """Per-slab device work through libplmss_b200 (the product path)."""

    def __init__(self, ctx=None):
        from . import api

        self.api = api
        self.ctx = ctx or api.default_context()

    def segment_slab(self, dims, field_ext: torch.Tensor, halo_lo: bool, halo_hi: bool):
        import ctypes as C

        a = self.api
        d = a._dims(dims)
        n = int(np.prod(d))
        desc = torch.empty(n, dtype=torch.int32, device=field_ext.device)
        asc = torch.empty(n, dtype=torch.int32, device=field_ext.device)
        sweeps = C.c_int32()
        a._check(a.lib().plmss_b200_segment_slab(self.ctx.h, d.ctypes.data, a._key_type(field_ext),
                                                 a._ptr(field_ext), int(halo_lo), int(halo_hi), a._ptr(desc),
                                                 a._ptr(asc), C.byref(sweeps)))
        return desc.to(torch.int64) & 0xFFFFFFFF, asc.to(torch.int64) & 0xFFFFFFFF

    def local_regions(self, asc: torch.Tensor, desc: torch.Tensor, N: int):
        """combine_ms on this slab's (global-id) labels: local dense ids and
        the sorted distinct keys asc * N + desc they index."""
        a = self.api
        seg = a.SegmentationResult(desc=desc.to(torch.int32), asc=asc.to(torch.int32))
        a.combine_ms(seg, ctx=self.ctx)
        k = seg.region_keys
        uniq = (k >> 32) * N + (k & 0xFFFFFFFF)
        return seg.ms_region.to(torch.int64) & 0xFFFFFFFF, uniq

    def march_slab(self, dims, ms_ext: torch.Tensor):
        recs = self.api.emit_separators(dims, ms_ext.contiguous(), ctx=self.ctx)
        return recs[:, 0] >> 6, recs[:, 1], recs[:, 2]


def _all_gather_var(t: torch.Tensor, group=None):
    """all_gather of variable-length 1-D/2-D tensors (pad to the max)."""
    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(x.item()) for x in ns]
    m = max(ns) if ns else 0
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return [o[:k] for o, k in zip(outs, ns)]


def _exchange_layers(bottom: torch.Tensor, top: torch.Tensor, rank: int, world: int, group=None):
    """Send my bottom layer down and top layer up; return (from_below,
    from_above) — the neighbours' top / bottom layers (None at the ends)."""
    ops, below, above = [], None, None
    if rank > 0:
        below = torch.empty_like(top)
        ops.append(dist.P2POp(dist.isend, bottom.contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, below, rank - 1, group))
    if rank + 1 < world:
        above = torch.empty_like(bottom)
        ops.append(dist.P2POp(dist.isend, top.contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, above, rank + 1, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return below, above


def ms_segmentation(field_owned: torch.Tensor, dims, backend, group=None) -> SlabResult:
    """Full MS segmentation of a z-slab decomposed volume. ``field_owned`` is
    this rank's owned layers (x fastest), ``dims`` the global (X, Y, Z)."""
    X, Y, Z = (int(v) for v in dims)
    XY, N = X * Y, X * Y * Z
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    z0, z1 = slab_bounds(Z, world, rank)
    nz = z1 - z0
    f = field_owned.reshape(nz, XY)
    dev = f.device

    # 1. field halo
    below, above = _exchange_layers(f[0], f[-1], rank, world, group)
    parts = ([below[None]] if below is not None else []) + [f] + ([above[None]] if above is not None else [])
    f_ext = torch.cat(parts).reshape(-1)
    lo = 1 if below is not None else 0
    nz_ext = nz + lo + (1 if above is not None else 0)
    zbase = z0 - lo  # global layer of extended layer 0

    # 2. slab segmentation (halo layers are terminals)
    d_ext, a_ext = backend.segment_slab((X, Y, nz_ext), f_ext, below is not None, above is not None)
    off = zbase * XY
    own = slice(lo * XY, (lo + nz) * XY)
    desc = d_ext[own] + off
    asc = a_ext[own] + off

    # 3. boundary graph over every rank's bottom and top owned layers
    bnd = torch.stack([desc[:XY], desc[-XY:], asc[:XY], asc[-XY:]])
    allb = [torch.empty_like(bnd) for _ in range(world)]
    dist.all_gather(allb, bnd, group=group)
    layers = []  # global z of each boundary row, rank-major: bottom, top
    for r in range(world):
        a0, a1 = slab_bounds(Z, world, r)
        layers += [a0, a1 - 1]
    layer_slot = torch.full((Z,), -1, dtype=torch.int64, device=dev)
    for i, zl in enumerate(layers):
        if layer_slot[zl] < 0:
            layer_slot[zl] = i
    nodes_d = torch.stack([b[k] for b in allb for k in (0, 1)]).reshape(-1)
    nodes_a = torch.stack([b[k] for b in allb for k in (2, 3)]).reshape(-1)

    def slot_of(g):  # global vertex id -> boundary slot (or -1)
        s = layer_slot[g // XY]
        return torch.where(s >= 0, s * XY + g % XY, torch.full_like(g, -1))

    def resolve(nodes):
        lab = nodes.clone()
        for _ in range(64):
            s = slot_of(lab)
            nxt = torch.where(s >= 0, lab[s.clamp(min=0)], lab)
            if torch.equal(nxt, lab):
                return lab
            lab = nxt
        raise RuntimeError("boundary graph did not converge")

    fin_d, fin_a = resolve(nodes_d), resolve(nodes_a)

    def fix(lab, fin):  # owned labels that point at halo vertices
        z = lab // XY
        halo = (z < z0) | (z >= z1)
        s = slot_of(lab)
        return torch.where(halo, fin[s.clamp(min=0)], lab)

    desc, asc = fix(desc, fin_d), fix(asc, fin_a)

    # 4. extrema (owned roots, id order; rank order = global order)
    ids = torch.arange(z0 * XY, z1 * XY, dtype=torch.int64, device=dev)
    maxima = torch.cat(_all_gather_var(ids[desc == ids], group))
    minima = torch.cat(_all_gather_var(ids[asc == ids], group))

    # 5. Morse-Smale ids: lexicographic (asc, desc) == key asc * N + desc
    # The device combine_ms indexes its rank maps by slab-local vertex index,
    # so it only applies while global ids equal local ones (one rank).
    local_regions = getattr(backend, "local_regions", None) if world == 1 else None
    if local_regions is not None:  # dense local ids from the device hash (no sort of the slab)
        local, uniq = local_regions(asc, desc, N)
    else:
        key = asc * N + desc
        uniq, local = torch.unique(key, return_inverse=True)
    gkeys = torch.unique(torch.cat(_all_gather_var(uniq, group)))
    ms = torch.searchsorted(gkeys, uniq)[local]
    region_keys = torch.stack([gkeys // N, gkeys % N], dim=1)

    # 6. marching: owned cube layers need the next rank's first layer of ids
    _, ms_above = _exchange_layers(ms[:XY], ms[-XY:], rank, world, group)
    ms_ext = torch.cat([ms] + ([ms_above] if ms_above is not None else []))
    nz_m = nz + (1 if ms_above is not None else 0)
    if nz_m >= 2:
        cells, tlo, thi = backend.march_slab((X, Y, nz_m), ms_ext)
        cells = cells + 6 * (X - 1) * (Y - 1) * z0
    else:
        cells = tlo = thi = torch.empty(0, dtype=torch.int64, device=dev)
    cnt = torch.tensor([cells.shape[0]], dtype=torch.int64, device=dev)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    cnts = [int(c.item()) for c in cnts]
    return SlabResult(z0, z1, desc, asc, ms, maxima, minima, region_keys, cells, tlo, thi, sum(cnts[:rank]),
                      sum(cnts))
