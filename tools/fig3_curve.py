"""Fig. 3(a) of the paper: relative complexity vs depth of the 2-, 3- and 4-part schemes
of the 64-qubit grid, from the planner of the C-ABI (host only, no GPU).

    python tools/fig3_curve.py [--grid 8x8] [--depths 1-40] > profiles/fig3_complexity.csv

Columns per scheme: c_total (all cut CZs), the paper's measure "the partition with the maximum
number of qubits" + c_total (every copy of the circuit is t sub-circuits; P:114, P:199 counts
max part + c, +1 for the 2 halves = 49 at 64q d22), and this library's log2 of the leaf
amplitudes it evolves (each part forks only on the cuts of its own boundaries).
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_06952_b200 import qsim as Q  # noqa: E402
from workloads import generate  # noqa: E402

SCHEMES = {"2-part": [4], "3-part": [3, 5], "4-part": [2, 4, 6]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="8x8")
    ap.add_argument("--depths", default="1-40")
    a = ap.parse_args()
    rows, cols = map(int, a.grid.split("x"))
    d0, d1 = map(int, a.depths.split("-"))
    hdr = ["depth"]
    for name in SCHEMES:
        hdr += [f"{name}_c", f"{name}_paper_Ne", f"{name}_log2_leaf_amps"]
    print(",".join(hdr))
    for d in range(d0, d1 + 1):
        circ = generate(rows, cols, d, 0)
        ctx = Q.qsim_create(Q.QSIM_C64, 0)
        row = [str(d)]
        try:
            Q.qsim_load_circuit(ctx, rows, cols, d, circ.gate_array())
            for name, rc in SCHEMES.items():
                p = Q.qsim_multipart_plan(ctx, rc)
                c = sum(p["boundary_cuts"])
                t = len(rc) + 1
                ne = max(p["part_qubits"]) + c + math.log2(t)
                row += [str(c), f"{ne:.3f}", f"{p['log2_states']:.3f}"]
        finally:
            Q.qsim_destroy(ctx)
        print(",".join(row))


if __name__ == "__main__":
    main()
