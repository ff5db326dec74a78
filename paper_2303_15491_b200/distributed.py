"""Z-slab decomposition of the full Morse-Smale segmentation over ranks
(SURVEY.md §8(e)): one process per GPU, torch.distributed over NCCL for the
exchanges, the fused brick pipeline on every slab (include/plmss_b200.h,
plmss_b200_slab_*).

Rank r owns whole 32-layer brick layers [z0, z1) (slab_bounds: the even split
of parallel.hpp:27-29 applied to brick layers), so rank order is the
reference's global vertex and cell order. One step:

0. field halo: the neighbours' boundary layers of f (point-to-point, into
   the slab buffer's halo layers);
1. slab_segment (device): pass A on the slab's bricks with the halo layers as
   real data, the sorted extremum lists, the terminal forest inside the slab;
   a chain that leaves the slab ends at a portal (the halo vertex it enters);
   -> all_gather: extremum counts, extremum lists, boundary layers (the
   resolved value of every vertex of the first / last owned layer);
2. slab_resolve (device): every portal followed through the gathered boundary
   layers to its extremum (chains are strictly monotone, so one exchange
   suffices: no iteration across ranks), desc / asc, region tokens, the
   slab's distinct (rank_min, rank_max) pairs;
   -> all_gather of the pairs;
3. slab_ids (device): the global region table in the combine_ms order
   (segmentation.cpp:170-196); ms holds globally consistent region tokens
   (dense mode) or the dense ids (hash mode);
   -> the next rank's first layer of ms (point-to-point) into ms's extra layer;
4. slab_emit (device): the dense ids (from the tokens, in the count pass),
   separator records of the owned cube layers with global cell ids, reference
   order (marching.cpp:116-215); concatenated in rank order they are the
   single-volume record list.

The step is written once, as a generator (``slab_step``) that yields its
collectives. ``TorchComm`` runs it over torch.distributed (NCCL on B200,
gloo on CPU); ``run_ranks_inprocess`` runs world ranks in one process,
advancing every rank to its next collective and performing it in memory —
ranks never wait on each other inside a kernel, so this reproduces the
multi-GPU results exactly on one device (tests/test_gpu_parity.py). Backends:
``B200SlabBackend`` (the product path, C-ABI); tests/test_distributed.py has a
numpy backend with the same contract for the gloo tests.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

BRICK = 32
FINAL, PORTAL = 0x80000000, 0x40000000  # boundary-layer value flags (fused.cu kFinal / kPortal)


def slab_bounds(Z: int, world: int, rank: int):
    """Owned z-layers [z0, z1) of a rank: brick layers split evenly
    (parallel.hpp:27-29 on ceil(Z / 32) units), the last slab clipped to Z."""
    nb = (Z + BRICK - 1) // BRICK
    if world > nb:
        raise ValueError(f"{world} ranks for {nb} brick layers: at most one rank per 32 z-layers")
    b0, b1 = nb * rank // world, nb * (rank + 1) // world
    return b0 * BRICK, min(b1 * BRICK, Z)


def halo_bounds(Z: int, world: int, rank: int):
    """Field layers a rank's slab buffer holds: [z0 - 1, z1 + 1) clipped."""
    z0, z1 = slab_bounds(Z, world, rank)
    return max(z0 - 1, 0), min(z1 + 1, Z)


@dataclass
class SlabResult:
    z0: int
    z1: int
    desc: torch.Tensor         # owned vertices: vertex id of the maximum (uint32 in int32 storage)
    asc: torch.Tensor          # ... of the minimum
    ms: torch.Tensor           # owned vertices: dense MS region id
    maxima: torch.Tensor       # global sorted extremum lists (identical on every rank)
    minima: torch.Tensor
    region_keys: torch.Tensor  # global (asc << 32 | desc) per region, sorted (int64 storage)
    tris: torch.Tensor         # this rank's separator records (T, 2) int64: [cell << 6 | row, lo | hi << 32]
    tri_base: int              # offset of this rank's records in the global list
    tri_total: int
    sweeps: int


# ------------------------------------------------------------ the step -----
def slab_step(backend, dims, rank: int, world: int, field_buf: torch.Tensor):
    """One z-slab step as a generator of collectives (module docstring).
    ``field_buf`` holds halo_bounds(Z, world, rank) layers with this rank's
    owned layers filled; the halo layers are filled by step 0."""
    X, Y, Z = (int(v) for v in dims)
    XY = X * Y
    z0, z1 = slab_bounds(Z, world, rank)
    h0, h1 = halo_bounds(Z, world, rank)
    lo = z0 - h0
    f = field_buf.view(h1 - h0, XY)
    # 0. field halo
    yield ("exchange", f[lo], f[lo + z1 - z0 - 1], f[0] if lo else None, f[-1] if h1 > z1 else None)
    # 1. the slab
    s = backend.segment(dims, z0, z1, field_buf)
    counts = yield ("allgather", torch.tensor([s["n_max"], s["n_min"]], dtype=torch.int64, device=f.device))
    counts = counts.cpu().numpy()
    maxima = yield ("allgather_var", s["maxima"], [int(c) for c in counts[:, 0]])
    minima = yield ("allgather_var", s["minima"], [int(c) for c in counts[:, 1]])
    G = yield ("allgather", s["boundary"])
    # 2. portals, labels, the slab's region pairs
    keys, nk = backend.resolve(G, world, rank, counts[:, 0].copy(), counts[:, 1].copy(), maxima, minima)
    nks = yield ("allgather", torch.tensor([nk], dtype=torch.int64, device=f.device))
    keys_all = yield ("allgather_var", keys, [int(c) for c in nks.cpu().numpy().reshape(-1)])
    # 3. dense ids
    region_keys = backend.ids(keys_all)
    # 4. marching: the next rank's first layer of ids
    ms_ext = backend.ms_ext()
    nz = z1 - z0
    yield ("exchange", ms_ext[:XY], None, None, ms_ext[nz * XY:(nz + 1) * XY] if z1 < Z else None)
    tris = backend.emit()
    nts = yield ("allgather", torch.tensor([tris.shape[0]], dtype=torch.int64, device=f.device))
    nts = [int(c) for c in nts.cpu().numpy().reshape(-1)]
    return SlabResult(z0, z1, backend.desc(), backend.asc(), backend.ms(), maxima, minima, region_keys, tris,
                      sum(nts[:rank]), sum(nts), s["sweeps"])


# ------------------------------------------------------- communicators -----
class TorchComm:
    """The step's collectives over torch.distributed (NCCL / gloo)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allgather(self, t):
        out = torch.empty(self.world * t.numel(), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous().view(-1), group=self.group)
        return out.view((self.world,) + tuple(t.shape))

    def allgather_var(self, t, counts):
        m = max(max(counts), 1)
        pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        out = self.allgather(pad)
        return torch.cat([out[r, : counts[r]] for r in range(self.world)])

    def exchange(self, send_down, send_up, recv_below, recv_above):
        """send_down -> rank - 1 (its recv_above), send_up -> rank + 1 (its
        recv_below); None entries skip a direction, ends skip the edge."""
        ops = []
        r, w, g = self.rank, self.world, self.group
        if r > 0 and send_down is not None:
            ops.append(dist.P2POp(dist.isend, send_down.contiguous(), r - 1, g))
        if r > 0 and recv_below is not None:
            ops.append(dist.P2POp(dist.irecv, recv_below, r - 1, g))
        if r + 1 < w and send_up is not None:
            ops.append(dist.P2POp(dist.isend, send_up.contiguous(), r + 1, g))
        if r + 1 < w and recv_above is not None:
            ops.append(dist.P2POp(dist.irecv, recv_above, r + 1, g))
        if ops:
            for q in dist.batch_isend_irecv(ops):
                q.wait()

    def run(self, gen):
        """Drive a step generator to completion; returns its result."""
        try:
            req = next(gen)
            while True:
                kind = req[0]
                if kind == "allgather":
                    res = self.allgather(req[1])
                elif kind == "allgather_var":
                    res = self.allgather_var(req[1], req[2])
                elif kind == "exchange":
                    self.exchange(*req[1:])
                    res = None
                else:
                    raise ValueError(kind)
                req = gen.send(res)
        except StopIteration as e:
            return e.value


def run_ranks_inprocess(gens):
    """Run the step generators of all ranks in one process: every rank is
    advanced to its next collective, the collective is performed in memory,
    and the results are sent back (lockstep; the ranks' device work never
    waits on another rank inside a kernel)."""
    world = len(gens)
    reqs = [next(g) for g in gens]
    results = [None] * world
    done = [False] * world
    while not all(done):
        kinds = {r[0] for r, d in zip(reqs, done) if not d}
        if len(kinds) != 1 or any(done):
            raise RuntimeError(f"ranks diverged: {kinds}")
        kind = kinds.pop()
        if kind == "allgather":
            stacked = torch.stack([r[1].to(reqs[0][1].device) for r in reqs])
            outs = [stacked.to(r[1].device) for r in reqs]
        elif kind == "allgather_var":
            cat = torch.cat([r[1][: r[2][i]].to(reqs[0][1].device) for i, r in enumerate(reqs)])
            outs = [cat.to(r[1].device) for r in reqs]
        elif kind == "exchange":
            for i, r in enumerate(reqs):
                _, sd, su, rb, ra = r
                if i > 0 and rb is not None:
                    rb.copy_(reqs[i - 1][2])
                if i + 1 < world and ra is not None:
                    ra.copy_(reqs[i + 1][1])
            outs = [None] * world
        else:
            raise ValueError(kind)
        for i, g in enumerate(gens):
            try:
                reqs[i] = g.send(outs[i])
            except StopIteration as e:
                results[i] = e.value
                done[i] = True
    return results


def ms_segmentation(field_buf: torch.Tensor, dims, backend, group=None) -> SlabResult:
    """Full MS segmentation of a z-slab decomposed volume on this rank:
    ``field_buf`` holds halo_bounds(Z, world, rank) layers (owned ones
    filled), ``dims`` the global (X, Y, Z)."""
    comm = TorchComm(group)
    return comm.run(slab_step(backend, dims, comm.rank, comm.world, field_buf))


# --------------------------------------------------------- B200 backend ----
class _DevView:
    """Zero-copy torch view of context-owned device memory."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr or 0), False),
                                         "version": 3}


def _view(ptr, n, dtype, device):
    ts = {torch.int32: "<i4", torch.int64: "<i8"}[dtype]
    if n == 0 or not ptr:
        return torch.empty(0, dtype=dtype, device=device)
    return torch.as_tensor(_DevView(ptr, n, ts), device=device)


class B200SlabBackend:
    """The slab stages through libplmss_b200 (the product path). Device
    outputs are views of buffers owned by this backend / its context, valid
    until the next step."""

    def __init__(self, ctx=None):
        from . import api

        self.api = api
        self.ctx = ctx or api.default_context()
        self.info = api.PlmssSlabInfo()
        self._bufs = {}
        self.dev = torch.device(f"cuda:{self.ctx.device}")

    def _buf(self, name, n):
        b = self._bufs.get(name)
        if b is None or b.numel() < n:
            b = self._bufs[name] = torch.empty(max(n, 1), dtype=torch.int32, device=self.dev)
        return b[:n]

    def segment(self, dims, z0, z1, field_buf):
        a = self.api
        d = a._dims(dims)
        self.XY = int(d[0]) * int(d[1])
        self.nz = z1 - z0
        self.has_up = z1 < int(d[2])
        a._check(a.lib().plmss_b200_slab_segment(self.ctx.h, d.ctypes.data, z0, z1, a._ptr(field_buf),
                                                 C.byref(self.info)))
        i = self.info
        return {"n_max": i.n_maxima, "n_min": i.n_minima,
                "maxima": _view(i.d_maxima, i.n_maxima, torch.int32, self.dev),
                "minima": _view(i.d_minima, i.n_minima, torch.int32, self.dev),
                "boundary": _view(i.d_boundary, 4 * self.XY, torch.int32, self.dev).view(4, self.XY),
                "sweeps": i.sweeps}

    def resolve(self, G, world, rank, max_counts, min_counts, maxima, minima):
        a = self.api
        n = self.nz * self.XY
        desc, asc = self._buf("desc", n), self._buf("asc", n)
        ms = self._buf("ms", n + (self.XY if self.has_up else 0))
        self._keep = (G, maxima, minima)  # alive until slab_emit
        mc = np.ascontiguousarray(max_counts, dtype=np.int64)
        nc = np.ascontiguousarray(min_counts, dtype=np.int64)
        a._check(a.lib().plmss_b200_slab_resolve(self.ctx.h, a._ptr(G.contiguous()), world, rank, mc.ctypes.data,
                                                 nc.ctypes.data, a._ptr(maxima), a._ptr(minima), a._ptr(desc),
                                                 a._ptr(asc), a._ptr(ms), C.byref(self.info)))
        return _view(self.info.d_keys, self.info.n_keys, torch.int64, self.dev), self.info.n_keys

    def ids(self, keys_all):
        a = self.api
        a._check(a.lib().plmss_b200_slab_ids(self.ctx.h, a._ptr(keys_all), keys_all.numel(), C.byref(self.info)))
        return _view(self.info.d_region_keys, self.info.n_regions, torch.int64, self.dev)

    def ms_ext(self):
        """ms of the owned layers + the next rank's first layer (region
        tokens in dense mode, ids in hash mode: exchanged as they are)."""
        return self._bufs["ms"][: self.nz * self.XY + (self.XY if self.has_up else 0)]

    def ms(self):
        """Dense MS ids of the owned vertices (after emit)."""
        return self._bufs["ids"][: self.nz * self.XY]

    def desc(self):
        return self._bufs["desc"][: self.nz * self.XY]

    def asc(self):
        return self._bufs["asc"][: self.nz * self.XY]

    def emit(self):
        a = self.api
        ids = self._buf("ids", self.nz * self.XY + (self.XY if self.has_up else 0))
        a._check(a.lib().plmss_b200_slab_emit(self.ctx.h, a._ptr(ids), C.byref(self.info)))
        self._keep = None
        return _view(self.info.d_tris, 2 * self.info.n_tris, torch.int64, self.dev).view(-1, 2)


def slab_field_buffer(dims, world: int, rank: int, device, owned: Optional[torch.Tensor] = None):
    """A rank's field buffer (halo_bounds layers); ``owned`` copied in."""
    X, Y, Z = (int(v) for v in dims)
    h0, h1 = halo_bounds(Z, world, rank)
    z0, z1 = slab_bounds(Z, world, rank)
    buf = torch.empty((h1 - h0) * X * Y, dtype=torch.float32, device=device)
    if owned is not None:
        buf[(z0 - h0) * X * Y:(z1 - h0) * X * Y].copy_(owned.reshape(-1))
    return buf
