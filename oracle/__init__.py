"""CPU oracle for the Grünwald–Letnikov history stepper — TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the reference `fracgrid` hot path
(`/root/reference/pkg/src/fracgrid/{coefficients,schedule,grid,solver}.py`) so that
the B200 product path can be checked against it.  It is the *checker*, never the
thing measured or shipped:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
  ``--impl reference`` legs may import it;
* the product package ``paper_1004_5128_b200`` never imports it and has no CPU
  fallback — it fails loudly if its CUDA library is missing.

Two restatements live here:

``fg_oracle.py``  NumPy, op-for-op with the reference (same ``np.einsum`` contraction,
                  same contiguous/gather split, same scalar evaluation order), so the
                  2D linear-decay path is *bitwise* equal to ``fracgrid.solver.run``.
``fg_oracle.c``   plain C (``-ffp-contract=off``), the same per-element sequential
                  accumulation order, OpenMP over grid points; bitwise equal to the
                  NumPy restatement and used as the timed CPU baseline.

Parity is pinned: ``tests/golden/make_golden.py`` imports the real reference in the
build container and freezes its outputs under ``tests/golden/``; the CPU test-suite
checks both restatements against those fixtures bit for bit.
"""
