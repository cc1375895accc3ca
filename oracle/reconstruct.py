"""Reconstruction of sampled amplitudes from branch slices (ORACLE — test infrastructure only).

"The final state of the original circuit is equal to the addition of all
transformed circuits" (Fig. 1 caption); per copy the sampled upper and
lower results are combined by a tensor product and "added to the resultant
vector".  For sampled blocks this is

    A[i, j] = sum_b U[b, i] * L[b, j]      (complex, no conjugation)

written here as the literal accumulation loop over b in fp64 (complex128).
"""
import numpy as np


def branch_sum(U: np.ndarray, L: np.ndarray) -> np.ndarray:
    U = np.asarray(U, dtype=np.complex128)
    L = np.asarray(L, dtype=np.complex128)
    if U.shape[0] != L.shape[0]:
        raise ValueError("branch counts differ")
    A = np.zeros((U.shape[1], L.shape[1]), dtype=np.complex128)
    for b in range(U.shape[0]):
        A += np.outer(U[b], L[b])
    return A


def probabilities(A: np.ndarray) -> np.ndarray:
    """p = |a|^2 (P:118 'probability amplitude of the sampled components')."""
    A = np.asarray(A, dtype=np.complex128)
    return A.real * A.real + A.imag * A.imag
