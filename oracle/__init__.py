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

Parity is PINNED: ``tests/test_oracle.py`` checks both against the golden
fixtures in ``tests/golden/`` that ``tests/golden/make_golden.py`` produced by
running the real reference package in the build container.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package.  The product package (``paper_1908_01407_b200``)
never imports it: there is no CPU fallback.
"""
