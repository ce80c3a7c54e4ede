"""CPU ORACLE for the BBWADG hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call or execute anything in this package.
The product path (``paper_1808_08645_b200``) never imports it and has no CPU
fallback.  The oracle shares no code with the CUDA library (no kernels,
headers, tables, constants or pre/post-processing); the only shared code is the
input-synthesis package ``workloads/``.

What it computes (PAPER.md; ``P:n`` = PAPER.md line n):

* the semi-discrete WADG right-hand side of Eq. WADGform for the
  acoustic system Eq. awave with penalty fluxes Eq. sdf,
  written as its plain dense definition:
    - volume:  -(sum_ij G_ij D_j) u with D_j = M^-1 S_j, dense;
    - surface: sum_f (J_f/J) L^f F with L^f = M^-1 M_f, applied by
      face quadrature at PHYSICAL face points, the neighbour's polynomial
      evaluated at the same physical points (no coefficient face maps);
    - WADG:    (M^k)^-1 M^k_{c^2} = P_q diag(c^2_M(x_q)) V_q  (Eq. pwadg
      P:250-254, with the weight c^2 -- DESIGN.md R1/R2) on a rule exact to
      degree 2N+M, which makes it EXACTLY the L2 projection of c^2_M * r_p
      onto P^N that BBWADG computes;
* the low-storage RK update the paper cites (Carpenter-Kennedy (5,4),
  DESIGN.md R13);
* diagnostics: WADG energy, semi-discrete energy rate, L2 error.

Precision: dense reference operators that contain M^-1 are formed by solving
with mixed-precision iterative refinement (fp64 Cholesky, 80-bit long double
residuals, exact integer mass matrix, mpmath quadrature nodes) and rounded to
fp64 once; everything per element runs in fp64.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): see DESIGN.md "Oracle pins".
"""
