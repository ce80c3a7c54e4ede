"""Seeded synthetic inputs shared by the oracle tests and the product path.

This package is the ONLY code both sides may use.
It holds no arithmetic of the BBWADG hot path (volume derivative, surface flux /
lift, WADG multiply-project, LSRK): it only synthesises the DATA the hot path is
run on, with the shapes and structure of the paper's workloads:

* ``kuhn``   -- Kuhn-cube tetrahedral meshes on [-1,1]^3 (vertex + element arrays),
                Morton-ordered cubes (BASELINE.json configs 1-5).
* ``media``  -- wavespeed fields c^2(x) (smooth, frequency-k, layered) and their
                per-element degree-M Bernstein coefficients, the *input* c^2_M
                that ``bbwadg_setup`` takes (PAPER.md P:284-286 says the
                approximation is "computed and stored once in a pre-processing
                step"; BASELINE.json north_star passes "c^2 coefficients").
* ``states`` -- initial states and manufactured-solution source data.

The per-element L2 projections used to synthesise c^2_M, initial states and the
manufactured source are input preparation (they run once, outside the timed hot
path, on the host) and are implemented here independently of both ``oracle/``
and the CUDA library.
"""
