"""CPU oracle for the GraphBLAST hot path -- TEST INFRASTRUCTURE ONLY.

This package restates the reference's algorithms (``/root/reference/pkg/src/
graphalg``) on the CPU so the CUDA product path can be checked against it:

* ``oracle.port``   -- numpy restatement of the operator layer (kernels.py),
  the algorithms (algorithms.py) and the R-MAT input pipeline (io.py).
* ``oracle.cgraph`` -- ctypes loader for ``oracle/cgraph.c``, a plain-C
  restatement of the scale-dependent pieces (bit-exact R-MAT + preprocess +
  CSR, direction-optimizing BFS, FastSV CC, sparsified Bellman-Ford SSSP,
  PageRank, degree-ordered triangle count) used at RMAT scales the numpy port
  cannot reach, and as the ``cpu_baseline`` / ``--impl reference`` timing arm.

Parity is PINNED against outputs of the real reference package, produced in
the build container by ``tests/golden/make_golden.py`` (``tests/golden/``):
``tests/test_oracle.py`` checks the numpy port (operator cases, generator,
algorithms at s8-s12); ``tests/test_oracle_pins.py`` checks the C oracle --
BFS (two sources) s8-s20, SSSP / CC / TC / PageRank s8-s20, the reference
weights at s16/s18/s20, the non-integral SSSP variant and all 20 PageRank
iterates at s16/s20, the uniform family at s14/s16 and the reference's s22
BFS / CC / PageRank digests.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package.  The product package (``paper_1908_01407_b200``)
never imports it: there is no CPU fallback.
"""
