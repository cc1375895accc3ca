"""Sampled index blocks S_u, S_l (SURVEY §8(c) Q9, §8(d) "Synthetic inputs").

The paper never says which components were "sampled"; the
caller supplies the blocks.  Default recipe: distinct, sorted, seeded-uniform
subsets of [0, 2^h) drawn from a Philox stream keyed ``seed + 1000``; the
full range when n == 2^h.
"""
from __future__ import annotations

import numpy as np


def sample_block(h: int, n: int, seed: int) -> np.ndarray:
    """``n`` distinct sorted indices in [0, 2^h) as uint64."""
    if n < 0 or n > (1 << h):
        raise ValueError("block larger than the half space")
    if n == (1 << h):
        return np.arange(n, dtype=np.uint64)
    rng = np.random.Generator(np.random.Philox(seed + 1000))
    if h <= 24:
        picked = rng.choice(1 << h, size=n, replace=False)
    else:
        picked = np.unique(rng.integers(0, 1 << h, size=n + n // 4 + 64, dtype=np.uint64))
        while picked.size < n:
            more = rng.integers(0, 1 << h, size=n, dtype=np.uint64)
            picked = np.unique(np.concatenate([picked, more]))
        picked = rng.permutation(picked)[:n]
    return np.sort(np.asarray(picked, dtype=np.uint64))
