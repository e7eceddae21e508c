"""Seeded synthetic inputs for the BASELINE.json configs.

The reference's evaluation photos are not available (and are not recreated); these generators
stand in with the shapes and value distributions BASELINE.json names.  Images are generated in
fp64 with numpy's PCG64, stored as fp32 (the configs' pixel type), and converted ONCE on the host
to the u8 raster the reference consumes (proj/include/zinpaint/image.hpp:11-16).  The oracle and
the GPU always see the same bytes.

Shared by tests/ and bench.py; neither product nor oracle code.
"""
from __future__ import annotations

import numpy as np


def _round_half_away(x: np.ndarray) -> np.ndarray:
    return np.floor(x + 0.5)  # llround for the non-negative values used here


def value_noise(h: int, w: int, cell: float, rng: np.random.Generator) -> np.ndarray:
    """Bilinear lattice value noise in [0, 1] with lattice spacing `cell` pixels."""
    gh, gw = int(np.ceil(h / cell)) + 2, int(np.ceil(w / cell)) + 2
    lat = rng.random((gh, gw))
    y = np.arange(h) / cell
    x = np.arange(w) / cell
    y0, x0 = np.floor(y).astype(int), np.floor(x).astype(int)
    fy, fx = (y - y0)[:, None], (x - x0)[None, :]
    fy = fy * fy * (3 - 2 * fy)
    fx = fx * fx * (3 - 2 * fx)
    a = lat[y0][:, x0]
    b = lat[y0][:, x0 + 1]
    c = lat[y0 + 1][:, x0]
    d = lat[y0 + 1][:, x0 + 1]
    return (a * (1 - fx) + b * fx) * (1 - fy) + (c * (1 - fx) + d * fx) * fy


def sinusoids(h: int, w: int, rng: np.random.Generator, count: int = 8, size: int = 256):
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    f = rng.uniform(1, 16, count)
    a = rng.uniform(0.1, 0.5, count)
    th = rng.uniform(0, 2 * np.pi, count)
    ph = rng.uniform(0, 2 * np.pi, count)
    v = np.zeros((h, w))
    for i in range(count):
        v += a[i] * np.sin(2 * np.pi * f[i] * (xx * np.cos(th[i]) + yy * np.sin(th[i])) / size + ph[i])
    return v, a.sum()


def cfg1(seed: int = 1, size: int = 256, hole: int = 48):
    """256^2 grayscale: 8 seeded sinusoids + N(0, 0.05^2); centred 48x48 hole; K=9, D=8."""
    rng = np.random.default_rng(seed)
    v, _ = sinusoids(size, size, rng, 8, size)
    v = (v + rng.normal(0.0, 0.05, v.shape)).astype(np.float32).astype(np.float64)
    img = _round_half_away(255.0 * (v - v.min()) / (v.max() - v.min())).astype(np.uint8)
    known = np.ones((size, size), dtype=np.uint8)
    o = (size - hole) // 2
    known[o:o + hole, o:o + hole] = 0
    return img, known, dict(patch_size=9, dims=8, knn=80)


def cfg2(seed: int = 2, size: int = 1024, disks: int = 12):
    """1024^2 RGB: per channel 8 sinusoids + value noise, clamped [0,1]; 12 disk holes r~U[20,60];
    K=11 (11x11x3 patches), D=12."""
    rng = np.random.default_rng(seed)
    chans = []
    for _ in range(3):
        s, asum = sinusoids(size, size, rng, 8, size)
        nz = 0.6 * value_noise(size, size, 64.0, rng) + 0.4 * value_noise(size, size, 16.0, rng)
        v = 0.5 + 0.35 * s / asum + 0.3 * (nz - 0.5)
        chans.append(np.clip(v, 0.0, 1.0))
    v = np.stack(chans, axis=-1).astype(np.float32).astype(np.float64)
    img = _round_half_away(255.0 * v).astype(np.uint8)
    known = np.ones((size, size), dtype=np.uint8)
    yy, xx = np.mgrid[0:size, 0:size]
    for _ in range(disks):
        cx, cy = rng.uniform(0, size, 2)
        r = rng.uniform(20, 60)
        known[(xx - cx) ** 2 + (yy - cy) ** 2 < r * r] = 0
    return img, known, dict(patch_size=11, dims=12, knn=80)


def cfg4(seed: int = 4, size: int = 4096, frac: float = 0.05, block: int = 16):
    """4096^2 u16-range value noise, 5 octaves; 5% of the 16x16 blocks removed; u8 = v16 >> 8;
    K=9, D=8."""
    rng = np.random.default_rng(seed)
    v = np.zeros((size, size))
    amp, tot = 1.0, 0.0
    cell = size / 8.0
    for _ in range(5):
        v += amp * value_noise(size, size, cell, rng)
        tot += amp
        amp *= 0.5
        cell /= 2.0
    v16 = np.clip(np.floor(v / tot * 65535.0), 0, 65535).astype(np.uint16)
    img = (v16 >> 8).astype(np.uint8)
    nb = size // block
    total = nb * nb
    drop = rng.choice(total, size=int(round(frac * total)), replace=False)
    known = np.ones((size, size), dtype=np.uint8)
    for b in drop:
        by, bx = divmod(int(b), nb)
        known[by * block:(by + 1) * block, bx * block:(bx + 1) * block] = 0
    return img, known, dict(patch_size=9, dims=8, knn=80)


def cfg5_points(n: int, dims_in: int = 125, seed: int = 5):
    """cfg5 vectors: x = Q diag(0.9^(k/2)) z, Q seeded orthogonal, z ~ N(0, I) (fp32)."""
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.normal(size=(dims_in, dims_in)))
    scale = 0.9 ** (np.arange(dims_in) / 2.0)
    z = rng.normal(size=(n, dims_in)).astype(np.float32)
    return (z * scale.astype(np.float32)) @ q.T.astype(np.float32)


def cfg5_descriptors(n: int, D: int, nq: int, seed: int = 5, dims_in: int = 125, miss: float = 0.4):
    """cfg5 stand-in for the k-NN sweep: the quantised top-D principal coordinates of
    x = Q diag(0.9^(k/2)) z (their PCA basis is Q's first D columns, eigenvalues 0.9^k), and
    nq held-out queries with 40% of their 125 coordinates unknown -> mean (make_query semantics,
    proj/src/builder.cpp:110-127), projected and quantised with the dictionary's lo/hi."""
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.normal(size=(dims_in, dims_in)))
    scale = 0.9 ** (np.arange(dims_in) / 2.0)
    y = rng.standard_normal((n, D), dtype=np.float32)
    y *= scale[:D].astype(np.float32)
    lo, hi = y.min(0), y.max(0)
    inv = (255.0 / (hi - lo)).astype(np.float32)

    def quant(v):
        c = np.clip(v.astype(np.float32), lo, hi)
        c -= lo
        c *= inv
        c += np.float32(0.5)
        return np.floor(c).astype(np.uint8)

    coords = np.empty((n, D), dtype=np.uint8)
    for b in range(0, n, 1 << 21):
        coords[b:b + (1 << 21)] = quant(y[b:b + (1 << 21)])
    zq = rng.standard_normal((nq, dims_in))
    xq = (zq * scale) @ Q.T
    xq[rng.random((nq, dims_in)) < miss] = 0.0  # unknown -> mean (the distribution mean is 0)
    queries = quant(xq @ Q[:, :D])
    return coords, queries


def small_image(h: int, w: int, channels: int, seed: int, hole_frac: float = 0.1):
    """Small textured image + random rectangular holes, for parity tests."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w]
    base = 110 + 50 * np.sin(0.23 * xx + 0.11 * yy) + 30 * np.cos(0.05 * xx * (1 + 0.3 * np.sin(0.07 * yy)))
    chans = [base + 15 * c + rng.integers(-8, 9, size=(h, w)) for c in range(channels)]
    img = np.clip(np.stack(chans, -1) if channels > 1 else chans[0], 0, 255).astype(np.uint8)
    known = np.ones((h, w), dtype=np.uint8)
    target = hole_frac * h * w
    while (known == 0).sum() < target:
        rh, rw = rng.integers(2, 8), rng.integers(3, 14)
        y0, x0 = rng.integers(0, h - rh), rng.integers(0, w - rw)
        known[y0:y0 + rh, x0:x0 + rw] = 0
    return img, known
