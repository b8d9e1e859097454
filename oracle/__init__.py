"""CPU oracle for arXiv 2405.19246 (L1 multi-marginal OT, fast tensor-vector products).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import, call,
link or execute anything under ``oracle/``.  The product path
(``paper_2405_19246_b200``) never touches it and shares no code with it.

Everything is plain fp64 and follows the paper (``P:n`` = line n of PAPER.md):

* ``dense``   -- O1: the definitions written out.  Cost tensor,
                 kernel tensor, tensor-vector products J_k
                 (P:1023-1028), plan, W,
                 generalized Sinkhorn (Algorithm 1; l-marginal
                 update scheme P:1029-1035).  Dense N**l tensors, tiny N only.
* ``paper3``  -- O2: Algorithms 2 (FTVP-1), 3 (FTVP-2)
                 and 5 (FTVP-LOG) for l = 3, step by step in the
                 paper's notation, with the typo fixes listed in DESIGN.md §2;
                 Algorithm 4 driver.
* ``regions`` -- O3: §4.2's l!-region separation with the
                 per-region nested first-order recursions ("region chains"),
                 in the normalised form of Algorithm 2 (relative powers of
                 lambda only).  Plain, log-domain and cost (E-weighted,
                 P:1103-1125) variants; C implementation ``regions.c``.
* ``subset``  -- O4: the subset-lattice DP over the 2^(l-1) placement states,
                 written as plain subset sums; plain, log-domain and tangent variants; C
                 implementation ``subset.c``.  Pinned against O1 and O3; the fast oracle for
                 full-size parity and the timed CPU baseline.
* ``sinkhorn`` -- O5: Gauss-Seidel Sinkhorn driver over any of the above,
                 residual (Algorithm 1 line 7 generalised), cost W.
* ``comonotone`` -- closed-form unregularised optimum W_0 of the 1-D pairwise
                 L1 MMOT (sanity pin: W_eta >= W_0).
* ``grid2d``  -- O6: 2-D grids (§4.1), l = 3: the product written out, Algorithm 6
                 (FTVP_2d) with Algorithm 2 inside, the 2-D cost (reading A21), Sinkhorn.
* ``points``  -- non-uniform 1-D grids (footnote P:182): one decay per grid edge;
                 brute force and the subset recursion with per-edge weights, Sinkhorn driver.

Every function and the tests that pin it are listed in DESIGN.md §2b; none is "parity unpinned".
"""
from . import dense, paper3, regions, subset, sinkhorn, comonotone, grid2d  # noqa: F401
