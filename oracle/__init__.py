"""CPU oracle for the matrix-free neo-Hookean path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference package ``sdmefem``
(arXiv 2104.13466 companion code) for the hot path: 1D bases, structured DOF
map, dense element kernels (f_int, consistent tangent, consistent mass),
assembly, Jacobi-PCG, Newmark/Newton, and the explicit lumped-mass
penalty-contact loop.  Every function cites the reference
file:line it follows.

Rules:
* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import anything here, and
  only as the checker or the timed CPU baseline -- never as the product path.
* Parity is pinned: ``tests/golden/*.npz`` hold vectors produced by the real
  reference (``tests/golden/make_golden.py``, run in the build container where
  ``/root/reference`` exists), and ``tests/test_oracle_golden.py`` checks this
  restatement against them.
"""
