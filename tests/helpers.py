"""Shared numpy helpers for the parity tests (test code, not product)."""
from __future__ import annotations

import numpy as np


def morton_words(coords: np.ndarray) -> list[np.ndarray]:
    """Interleaved Morton address (level 7 first, dim 0 first) as uint64 words, MSW first.

    Restates the explicit interleave oracle of proj/tests/support/oracles.hpp:33-39.
    """
    coords = np.asarray(coords, dtype=np.uint8)
    n, D = coords.shape
    bits = []
    for level in range(7, -1, -1):
        for d in range(D):
            bits.append((coords[:, d] >> level) & 1)
    nb = len(bits)
    words = []
    for start in range(0, nb, 64):
        w = np.zeros(n, dtype=np.uint64)
        chunk = bits[start:start + 64]
        for b in chunk:
            w = (w << np.uint64(1)) | b.astype(np.uint64)
        words.append(w)
    return words


def is_morton_sorted(coords: np.ndarray, keys: np.ndarray) -> bool:
    """Adjacent pairs ordered by (Morton address, packed key) -- zcurve.cpp:116-125."""
    if len(keys) < 2:
        return True
    words = morton_words(coords)
    less = np.zeros(len(keys) - 1, dtype=bool)
    equal = np.ones(len(keys) - 1, dtype=bool)
    for w in words:
        a, b = w[:-1], w[1:]
        less |= equal & (a < b)
        equal &= a == b
    less |= equal & (keys[:-1] < keys[1:])
    return bool(less.all())


def fillfront(known: np.ndarray) -> list[tuple[int, int]]:
    """KNOWN pixels with an UNKNOWN 4-neighbour, row-major (proj/src/image.cpp:49-61)."""
    k = known != 0
    h, w = k.shape
    unk = ~k
    nb = np.zeros_like(k)
    nb[:, 1:] |= unk[:, :-1]
    nb[:, :-1] |= unk[:, 1:]
    nb[1:, :] |= unk[:-1, :]
    nb[:-1, :] |= unk[1:, :]
    ys, xs = np.nonzero(k & nb)
    return list(zip(xs.tolist(), ys.tolist()))


def pca_of(mi, layouts=range(8)):
    pm = np.stack([mi.layout(l)["mean"] for l in layouts])
    pc = np.stack([mi.layout(l)["components"] for l in layouts])
    return pm, pc
