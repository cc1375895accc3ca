"""Porter-Thomas / Gumbel statistics (ORACLE — test infrastructure only).

Eq. 7: f(z) = (1/alpha) exp(z - (e^z + alpha - 1)/alpha), alpha = 1,
for z = ln(N p), N = 2^n (Fig. 5 caption P:227).  For alpha = 1 the CDF is
F(z) = 1 - exp(-e^z) (integral of f with w = e^z).
"""
import numpy as np


def gumbel_pdf(z, alpha: float = 1.0):
    z = np.asarray(z, dtype=np.float64)
    return (1.0 / alpha) * np.exp(z - (np.exp(z) + alpha - 1.0) / alpha)


def gumbel_cdf(z):
    """F(z) = 1 - exp(-e^z), evaluated as -expm1(-e^z) (no cancellation in the left tail)."""
    z = np.asarray(z, dtype=np.float64)
    return -np.expm1(-np.exp(z))


def log_transform(p, n_qubits: int):
    p = np.asarray(p, dtype=np.float64).ravel()
    p = p[p > 0]
    return np.log(p) + n_qubits * np.log(2.0)


def ks_distance(z) -> float:
    """Kolmogorov-Smirnov distance of the sample z against F(z) = 1 - exp(-e^z)."""
    z = np.sort(np.asarray(z, dtype=np.float64))
    n = z.size
    F = gumbel_cdf(z)
    hi = np.arange(1, n + 1) / n - F
    lo = F - np.arange(0, n) / n
    return float(max(hi.max(), lo.max()))


def porter_thomas(p, n_qubits: int, z_lo: float, z_hi: float, n_bins: int) -> dict:
    """The f1 analyzer's quantities, written out (Fig. 5, Eq. 7):
    x = N p (N = 2^n); mean and population variance of x over all entries; the histogram
    of z = ln(N p) over the p > 0 entries in n_bins equal bins of [z_lo, z_hi) (bin =
    floor((z - z_lo) n_bins / (z_hi - z_lo))); Eq. 7's expected count per bin
    n_pos (F(e_k+1) - F(e_k)); the exact KS distance of z against F."""
    p = np.asarray(p, dtype=np.float64).ravel()
    x = p * 2.0 ** n_qubits
    z = log_transform(p, n_qubits)
    scale = n_bins / (z_hi - z_lo)
    b = np.floor((z - z_lo) * scale)
    inside = (b >= 0) & (b < n_bins)
    hist = np.bincount(b[inside].astype(np.int64), minlength=n_bins).astype(np.uint64)
    edges = z_lo + np.arange(n_bins + 1) * ((z_hi - z_lo) / n_bins)
    expected = z.size * np.diff(gumbel_cdf(edges))
    return {"count": p.size, "zeros": int(np.sum(p == 0)), "mean_Np": float(np.mean(x)),
            "var_Np": float(np.var(x)), "below": int(np.sum(b < 0)), "above": int(np.sum(b >= n_bins)),
            "hist": hist, "expected": expected, "ks": ks_distance(z) if z.size else 0.0, "z": z,
            "edges": edges}
