"""Chunked SHA-256 digests of large result arrays (harness utility: the
full-size parity tests and bench.py compare the device outputs against the
committed oracle digests, tests/golden/cfg*_digest.json, without moving the
arrays or the oracle to the GPU box).

digest(bytes) = sha256( sha256(block_0) || sha256(block_1) || ... ) with
64 MiB blocks of the raw little-endian bytes, so blocks hash in parallel and
a stream of arrays (e.g. separator records produced chunk by chunk) hashes
identically to the concatenated array.
"""
from __future__ import annotations

import hashlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np

BLOCK = 1 << 26
_POOL = ThreadPoolExecutor(max_workers=16)


def _h(mv) -> bytes:
    return hashlib.sha256(mv).digest()


class ChunkedSha256:
    """Streaming form: update() with consecutive pieces, hexdigest() at the end."""

    def __init__(self):
        self._pending = bytearray()
        self._futs = []
        self.nbytes = 0

    def update(self, data) -> "ChunkedSha256":
        if isinstance(data, (bytes, bytearray)):
            mv = memoryview(data)
        else:
            mv = memoryview(np.ascontiguousarray(data).reshape(-1).view(np.uint8))
        self.nbytes += mv.nbytes
        if self._pending:
            take = min(BLOCK - len(self._pending), mv.nbytes)
            self._pending += mv[:take]
            mv = mv[take:]
            if len(self._pending) == BLOCK:
                self._futs.append(_POOL.submit(_h, bytes(self._pending)))
                self._pending = bytearray()
        full = (mv.nbytes // BLOCK) * BLOCK
        if full:
            buf = mv[:full]
            # keep the source alive while its blocks hash
            self._futs += [_POOL.submit(_h, buf[i:i + BLOCK]) for i in range(0, full, BLOCK)]
        if mv.nbytes > full:
            self._pending += mv[full:]
        return self

    def drain(self, keep_blocks: int = 64) -> "ChunkedSha256":
        """Wait for all but the last keep_blocks block hashes (bounds the host
        memory held by pending blocks when streaming large arrays)."""
        for f in self._futs[:-keep_blocks] if keep_blocks else self._futs:
            f.result()
        return self

    def hexdigest(self) -> str:
        if self._pending:
            self._futs.append(_POOL.submit(_h, bytes(self._pending)))
            self._pending = bytearray()
        top = hashlib.sha256()
        for f in self._futs:
            top.update(f.result())
        return top.hexdigest()


def digest(a) -> str:
    """Chunked SHA-256 of an array's raw bytes."""
    return ChunkedSha256().update(a).hexdigest()


def digest_device(t, piece_bytes: int = 1 << 30) -> str:
    """Chunked SHA-256 of a CUDA tensor's bytes, copied to the host in pieces."""
    h = ChunkedSha256()
    flat = t.reshape(-1).view(__import__("torch").uint8)
    for i in range(0, flat.numel(), piece_bytes):
        h.update(flat[i:i + piece_bytes].cpu().numpy())
        h.drain(4 * max(piece_bytes // BLOCK, 1))  # bound host memory
    return h.hexdigest()
