"""Swap this package's GPU ``run`` in under the reference's own drivers.

The reference's callers bind ``run`` by name — ``fracgrid.benchmark``
(/root/reference/pkg/src/fracgrid/benchmark.py:17, called at :63 and :179) and
``fracgrid.cli`` (cli.py:73, called at :237) — and catch the reference's
``DivergenceError`` (benchmark.py:114-128 records the cell as a NaN row,
cli.py:469-479 exits with code 3).  ``install`` rebinds those two names; the
errors this package raises are instances of the reference's classes whenever
``fracgrid`` is loaded (``_engine.error_class``), so the handlers keep working.

    import fracgrid
    from paper_1004_5128_b200 import integrate
    undo = integrate.install(fracgrid)     # run_comparison / gamma_sweep / CLI on the GPU
    ...
    undo()                                 # restore the reference's NumPy run
"""

from __future__ import annotations

import importlib

from .solver import run as gpu_run

CALLERS = ("benchmark", "cli")  # the reference modules that import ``run`` by name


def install(fracgrid=None, run=gpu_run):
    """Rebind ``run`` in the reference's driver modules; returns an undo callable.

    ``fracgrid`` is the reference package (imported by name when omitted).  Only
    caller modules that exist and define ``run`` are touched.
    """
    if fracgrid is None:
        fracgrid = importlib.import_module("fracgrid")
    saved = []
    for name in CALLERS:
        mod = getattr(fracgrid, name, None)
        if mod is None:
            try:
                mod = importlib.import_module(f"{fracgrid.__name__}.{name}")
            except ImportError:
                continue
        if hasattr(mod, "run"):
            saved.append((mod, mod.run))
            mod.run = run

    def undo() -> None:
        for mod, fn in saved:
            mod.run = fn

    return undo
