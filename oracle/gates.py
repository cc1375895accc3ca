"""Gate matrices, written out from their definitions (ORACLE — test infrastructure only).

* H  = [[1, 1], [1, -1]] / sqrt(2)                   layer 0 (P:48 n_1 = 1)
* SX = X^(1/2) = 1/2 [[1+i, 1-i], [1-i, 1+i]]       the paper's "X gate" (Q6; Ref. [6] gate set)
* SY = Y^(1/2) = 1/2 [[1+i, -1-i], [1+i, 1+i]]      the paper's "Y gate" (Q6)
* T  = diag(1, (1+i)/sqrt(2))                        P:86 "T_{1,1} = (1+i)/sqrt 2"
* CZ = diag(1, 1, 1, -1)                             P:100 "CZ_{1,1,1,1} = -1"
* P0 = diag(1, 0), P1 = diag(0, 1), Z = diag(1, -1), I  (Eq. 1)

Matrices are indexed M[out, in] in the computational basis |0>, |1>
(two-qubit: basis |q0 q1> with q0 the more significant).
"""
import numpy as np

S2 = np.sqrt(2.0)

H = np.array([[1, 1], [1, -1]], dtype=np.complex128) / S2
SX = 0.5 * np.array([[1 + 1j, 1 - 1j], [1 - 1j, 1 + 1j]], dtype=np.complex128)
SY = 0.5 * np.array([[1 + 1j, -1 - 1j], [1 + 1j, 1 + 1j]], dtype=np.complex128)
T = np.array([[1, 0], [0, (1 + 1j) / S2]], dtype=np.complex128)
I2 = np.eye(2, dtype=np.complex128)
Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)
P0 = np.array([[1, 0], [0, 0]], dtype=np.complex128)
P1 = np.array([[0, 0], [0, 1]], dtype=np.complex128)
CZ = np.diag(np.array([1, 1, 1, -1], dtype=np.complex128))

# kind codes of the C-ABI / workloads (SX=1, SY=2, T=3, CZ=4) plus oracle-only branch gates
SINGLE = {1: SX, 2: SY, 3: T, "SX": SX, "SY": SY, "T": T, "H": H,
          "P0": P0, "P1": P1, "Z": Z, "I": I2}
