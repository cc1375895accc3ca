"""ORACLE — plain, slow, obviously-correct CPU reference for the partitioned simulator
of arXiv:1802.06952 ("64-qubit quantum circuit simulation", Chen et al.).

THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import or execute anything in this package.  The product
path (``paper_1802_06952_b200``) never imports it and shares no code with it;
the only shared module is ``workloads`` (seeded input generators, no method
arithmetic).

Precision: complex128 / float64 throughout (the paper ran in double: a 32-qubit
copy is 128 GB = 2 x 2^32 x 16 B).

Modules
  gates        2x2 / 4x4 matrices of the gate set
  statevector  full state vector, gate by gate, no fusion (Supp. A Eq. 4)
  partition    cut list, branch half-circuits, flat partitioned simulator
               (Supp. A Eqs. 7-8)
  multipart    t-way partitions (rows in bands), A = sum_b prod_k psi^k_b[S_k]
               (Fig. 3; DESIGN.md R-f4)
  reconstruct  A[i,j] = sum_b U_b[i] L_b[j] (Fig. 1 caption P:175)
  sampler      Philox4x32-10 + two-level inverse CDF over |a|^2
  stats        Porter-Thomas / Gumbel Eq. 7

Parity pins (``tests/test_oracle.py``) tie each function to something other
than itself: the Fig. 1 worked example, Fig. 4 / Table 2 printed values, the
CZ identity (Eq. 1), brute-force branch-sum identity on tiny grids, the
depth<=3 closed form, norm invariants, Random123 Philox known-answer vectors.
Functions without such a pin say "parity unpinned" in their docstring.
"""
