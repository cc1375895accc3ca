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
    z = np.asarray(z, dtype=np.float64)
    return 1.0 - np.exp(-np.exp(z))


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
