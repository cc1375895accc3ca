"""Sampler over a reconstructed amplitude block (ORACLE — test infrastructure only).

The paper's "sampling" is amplitude extraction; drawing outcomes
proportional to p = |a|^2 within the sampled block is the north-star
extension.  Definition used by both sides:

* Uniforms: Philox4x32-10 (Salmon et al., Random123), counter
  (k mod 2^32, k >> 32, 0, 0), key (seed mod 2^32, seed >> 32);
  u_k = (((out1 << 32) | out0) >> 11) * 2^-53 in [0, 1).
* C[i, :]  = inclusive prefix sum of p[i, :] in column order (sequential fp64)
  r_i      = C[i, n_l - 1];  R = inclusive sequential prefix of r;  W = R[-1]
* draw k:  t = u_k * W;  i = first i with R[i] > t (none: last i with r_i > 0)
           t2 = t - R[i-1] (t for i = 0);  j = first j with C[i, j] > t2
           (none: last j with p[i, j] > 0);  x = (S_u[i] << h_l) | S_l[j].

Strict '>' on an inclusive prefix never selects a zero-mass row or column.
"""
from __future__ import annotations

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK32 = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """Philox4x32 with 10 rounds on uint64 arrays holding 32-bit words.

    ctr: tuple of 4 arrays (or ints), key: tuple of 2 arrays (or ints).
    Round: (hi0, lo0) = M0*c0, (hi1, lo1) = M1*c2,
           c <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); key bumped by (W0, W1)
           between rounds (Random123 philox4x32_R, R = 10).
    """
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & MASK32 for x in ctr)
    k0, k1 = (np.asarray(x, dtype=np.uint64) & MASK32 for x in key)
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
        p0 = np.uint64(M0) * c0
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & MASK32, lo1, (hi0 ^ c3 ^ k1) & MASK32, lo0
    return c0, c1, c2, c3


def uniforms(seed: int, n: int, start: int = 0) -> np.ndarray:
    """u_k for k in [start, start + n)."""
    k = np.arange(start, start + n, dtype=np.uint64)
    seed = int(seed)
    out0, out1, _, _ = philox4x32_10((k & MASK32, k >> np.uint64(32), 0, 0),
                                     (seed & MASK32, (seed >> 32) & MASK32))
    v = (out1 << np.uint64(32)) | out0
    return (v >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def prefix_tables(p: np.ndarray):
    """C (row-wise inclusive prefix), R (prefix of row masses), W — sequential order."""
    p = np.asarray(p, dtype=np.float64)
    C = np.cumsum(p, axis=1)
    r = C[:, -1].copy()
    R = np.cumsum(r)
    return C, r, R, float(R[-1])


def draw(p: np.ndarray, seed: int, n_draws: int):
    """Row and column indices of n_draws samples from the block p[n_u, n_l]."""
    p = np.asarray(p, dtype=np.float64)
    C, r, R, W = prefix_tables(p)
    if not W > 0.0:
        raise ValueError("block has zero total mass")
    u = uniforms(seed, n_draws)
    t = u * W
    rows = np.searchsorted(R, t, side="right")
    last_row = int(np.nonzero(r > 0)[0][-1])
    rows = np.where(rows >= p.shape[0], last_row, rows)
    Rprev = np.where(rows > 0, R[np.maximum(rows - 1, 0)], 0.0)
    t2 = t - Rprev
    cols = np.empty(n_draws, dtype=np.int64)
    for k in range(n_draws):
        i = rows[k]
        j = int(np.searchsorted(C[i], t2[k], side="right"))
        if j >= p.shape[1]:
            j = int(np.nonzero(p[i] > 0)[0][-1])
        cols[k] = j
    return rows.astype(np.int64), cols, W


def sample(p, S_u, S_l, h_l: int, seed: int, n_draws: int):
    """Bitstrings x = (S_u[i] << h_l) | S_l[j] of n_draws samples, and the block mass W."""
    rows, cols, W = draw(p, seed, n_draws)
    S_u = np.asarray(S_u, dtype=np.uint64)
    S_l = np.asarray(S_l, dtype=np.uint64)
    x = (S_u[rows] << np.uint64(h_l)) | S_l[cols]
    return x.astype(np.uint64), W
