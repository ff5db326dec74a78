"""The five BASELINE.json workloads as seeded synthetic inputs.

The reference benchmarks real datasets (Miranda 512^3, Foot 256^3,
PAPER.md:1118,1123) that are not available here; BASELINE.json names seeded
synthetic stand-ins with the same sizes. Parameters are drawn with the
reference's RNG convention, std::mt19937_64 and u = (rng() >> 11) * 2^-53
(proj/src/synth.cpp:15-17), in the order (cx, cy, cz, sigma, amp) per
Gaussian. The field itself is include/plmss_synth.h: separable Gaussians
from float32 axis tables, per-voxel noise from a counter-based splitmix64
hash of (seed, vertex id); the device (csrc/synth.cu), the oracle's C loop
and host_field() below produce identical bytes.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the published 64-bit Mersenne Twister)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _MASK64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _MASK64
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64

    def uniform01(self) -> float:
        return float(self() >> 11) * 2.0 ** -53


@dataclass(frozen=True)
class Config:
    name: str
    dims: tuple
    kind: str          # "gaussians" | "uniform"
    n_gauss: int = 0
    sigma: tuple = (0.0, 0.0)
    noise: float = 0.0
    levels: int = 0
    seed: int = 0

    @property
    def n(self) -> int:
        return int(np.prod(self.dims))

    def gaussians(self) -> np.ndarray:
        """(n_gauss, 5) array of (cx, cy, cz, sigma, amp): centres uniform in
        the volume [0, n-1]^3, sigma and amplitude uniform in their ranges."""
        rng = MT19937_64(self.seed)
        out = np.zeros((self.n_gauss, 5), np.float64)
        for k in range(self.n_gauss):
            cx = rng.uniform01() * (self.dims[0] - 1)
            cy = rng.uniform01() * (self.dims[1] - 1)
            cz = rng.uniform01() * (self.dims[2] - 1)
            s = self.sigma[0] + (self.sigma[1] - self.sigma[0]) * rng.uniform01()
            a = -1.0 + 2.0 * rng.uniform01()
            out[k] = (cx, cy, cz, s, a)
        return out


CONFIGS = {
    "cfg1": Config("cfg1_64_gauss8", (64, 64, 64), "gaussians", 8, (4.0, 12.0), 1e-3, 0, 1),
    "cfg2": Config("cfg2_256_gauss64", (256, 256, 256), "gaussians", 64, (6.0, 24.0), 1e-4, 0, 2),
    "cfg3": Config("cfg3_512_white_noise", (512, 512, 512), "uniform", seed=3),
    "cfg4": Config("cfg4_512_gauss64_q64", (512, 512, 512), "gaussians", 64, (12.0, 48.0), 0.0, 64, 4),
    "cfg5": Config("cfg5_1024_gauss512", (1024, 1024, 1024), "gaussians", 512, (16.0, 64.0), 1e-5, 0, 5),
}


def scaled(cfg: Config, dims: tuple, name: str | None = None) -> Config:
    """Same distribution on a smaller grid (sigma scaled with the extent) —
    used for CPU-sized parity cases and the bounded CPU-baseline sample."""
    f = (min(dims) - 1) / (min(cfg.dims) - 1)
    return Config(name or f"{cfg.name}@{'x'.join(map(str, dims))}", tuple(dims), cfg.kind, cfg.n_gauss,
                  (cfg.sigma[0] * f, cfg.sigma[1] * f), cfg.noise, cfg.levels, cfg.seed)


def splitmix64_np(x: np.ndarray) -> np.ndarray:
    x = (x + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


_INV_FACT = [1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0, 1.0 / 40320.0, 1.0 / 5040.0,
             1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 1.0 / 2.0, 1.0, 1.0]


def synth_exp_np(x: np.ndarray) -> np.ndarray:
    """plmss_synth_exp (include/plmss_synth.h) elementwise, same IEEE ops."""
    x = np.minimum(np.asarray(x, np.float64), 0.0)
    t = x * 1.4426950408889634
    n = np.trunc(t - 0.5)
    r = (x - n * 6.93147180369123816490e-01) - n * 1.90821492927058770002e-10
    p = np.full_like(r, 1.0 / 6227020800.0)
    for c in _INV_FACT:
        p = p * r + c
    n = n.astype(np.int64)
    sub = n < -1022
    p = np.where(sub, p * 2.0 ** -600, p)
    e = np.where(sub, n + 600, n)
    out = p * np.ldexp(1.0, e)
    return np.where(x < -740.0, 0.0, out)


def axis_table_np(c: float, sigma: float, length: int) -> np.ndarray:
    d = np.arange(length, dtype=np.float64) - c
    return synth_exp_np(-(d * d) / (2.0 * sigma * sigma)).astype(np.float32)


def host_field(cfg: Config) -> np.ndarray:
    """The input definition of include/plmss_synth.h in numpy — the same
    bytes as the device generator (csrc/synth.cu) and the oracle's C loop:
    float32 separable Gaussian sums (every product / sum rounded), double
    noise, optional quantisation. Practical up to ~256^3 on the host."""
    X, Y, Z = cfg.dims
    v = np.arange(cfg.n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u = (splitmix64_np(np.uint64(cfg.seed) ^ (v * np.uint64(0xD1B54A32D192ED03))) >> np.uint64(11)).astype(
            np.float64) * 2.0 ** -53
    if cfg.kind == "uniform":
        return u.astype(np.float32)
    s = np.zeros((Z, Y, X), np.float32)
    for cx, cy, cz, sig, amp in cfg.gaussians():
        ex, ey, ez = axis_table_np(cx, sig, X), axis_table_np(cy, sig, Y), axis_table_np(cz, sig, Z)
        w = np.float32(amp) * (ey[None, :] * ez[:, None])  # (Z, Y), float32 products
        s = s + ex[None, None, :] * w[:, :, None]
    f = (s.reshape(-1).astype(np.float64) + cfg.noise * (2.0 * u - 1.0)).astype(np.float32)
    if cfg.levels:
        lo, hi = float(f.min()), float(f.max())
        t = (f.astype(np.float64) - lo) / (hi - lo) if hi > lo else np.zeros_like(f, dtype=np.float64)
        f = np.clip(np.floor(t * cfg.levels), 0, cfg.levels - 1).astype(np.float32)
    return f
