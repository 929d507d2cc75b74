"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU (numpy, fp64) implementation of the hot path of
Dolgov & Savostyanov, "Parallel cross interpolation for high-precision calculation of
high-dimensional integrals" (arXiv:1903.11554, /root/reference/PAPER.md).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product path
(``paper_1903_11554_b200``) never imports it, and this package never imports the product.
The two share no code; the only common module is ``workloads`` (seeded grid/config
generators, which hold none of the method's arithmetic).

Modules
  integrand  -- the Ising integrands on u-nodes (§5.1 eq. (9)-(10); BASELINE.json
                configs in the (4/d!) t-form), the per-entry definition of the tensor A,
                full-grid brute force (§4.1 eq. (5)).
  cross      -- counter-based initial pivots, fibers A(I_{<=k-1}, i_k, I_{>k}), the
                greedy pivot search of Alg. 2 (random samples, then rook search on the
                cross error), the dimension-parallel sweeps of
                Alg. 6 (every superblock appends at most one pivot per sweep from the index
                sets of the previous sweep, lines 624-641), and the TT quadrature (§4.1
                product of (2d-1) matrices, lines 689-693).

Parity status: every function is pinned by ``tests/test_oracle_*.py`` against closed
forms, brute force, mpmath or determinant/volume identities (DESIGN.md §"Oracle pins").
No function is "parity unpinned".
"""
