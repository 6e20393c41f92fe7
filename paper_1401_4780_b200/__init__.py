"""paper_1401_4780_b200 — B200-native AsyRK (asynchronous parallel randomized
Kaczmarz) hot path behind the reference's interfaces.

Python surface, mirroring the reference package ``asyrk``
(ref/python/asyrk/__init__.py:11-43, ref/bindings/module.cpp:281-318) for the
hot path:

* ``solve_rk(m, n, rows, cols, vals, b, epochs=100, target=0.0, seed=0,
  sampling="uniform")`` — deterministic device worker, iterates bit-identical
  to the reference's ``rk_solve``.
* ``solve_parallel(m, n, rows, cols, vals, b, threads=1, gamma=1.0,
  epochs=100, target=0.0, seed=0, variant="full-row")`` — ``threads``
  concurrent warp-workers (``threads == 1``: the deterministic worker).
* ``system_stats(m, n, rows, cols, vals)``, ``step_params(..., tau)`` —
  device compute_stats with the dense spectrum (lambda_max, lambda_min,
  sigma_r) from the device one-sided Jacobi SVD.
* ``lsq(m, n, rows, cols, vals, b, epochs=5000, target=0.0, seed=0)`` —
  least squares through the augmented system, solved on the device.
* ``simulate(m, n, rows, cols, vals, b, iterations, tau, gamma,
  delay="uniform", variant="single", seed=0)`` — the bounded-delay replay on
  the device, bit-identical to the reference's ``simulate``.

Device extensions: ``solve_parallel_device`` (sampling / precision /
snapshot interval / x_star), ``lambda_max``, ``residuals``,
``max_feasible_tau``, ``dense_spectrum``, ``lsq(..., sigma_r=, threads=,
gamma=)``; and :mod:`paper_1401_4780_b200.capi` for the C ABI
(device-resident systems, timing). Errors surface as
``ValueError("<ErrorCodeName>: message")`` like the reference.

The compiled extension is required: importing this package without it fails
loudly (there is no CPU fallback).
"""
import os as _os
import sys as _sys

_HERE = _os.path.dirname(_os.path.abspath(__file__))

try:
    from . import _asyrk  # type: ignore[attr-defined]
except ImportError as _e:  # pragma: no cover - exercised only when unbuilt
    raise ImportError(
        "paper_1401_4780_b200: the CUDA extension (_asyrk / libasyrk_b200.so) is not built; "
        "run `python -c 'import __graft_entry__ as g; g.build()'` from the repo root"
    ) from _e

solve_rk = _asyrk.solve_rk
solve_parallel = _asyrk.solve_parallel
solve_parallel_device = _asyrk.solve_parallel_device
lambda_max = _asyrk.lambda_max
residuals = _asyrk.residuals
max_feasible_tau = _asyrk.max_feasible_tau
system_stats = _asyrk.system_stats
step_params = _asyrk.step_params
simulate = _asyrk.simulate
lsq = _asyrk.lsq
dense_spectrum = _asyrk.dense_spectrum

__all__ = [
    "solve_rk",
    "solve_parallel",
    "system_stats",
    "step_params",
    "simulate",
    "lsq",
    "solve_parallel_device",
    "dense_spectrum",
    "lambda_max",
    "residuals",
    "max_feasible_tau",
]
__version__ = "0.1.0"
