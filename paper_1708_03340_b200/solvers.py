"""CG with truncation after every operation -- the reference solver loop
(solvers.py:110-231) as the direct caller of the truncation hot path.

The loop is backend-generic exactly like the reference's: it only calls the
eleven Backend methods, so it runs on ``GpuBackend`` (default; every add /
apply / truncate / inner product on the B200) or on any other backend object.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

from .arith import TruncationControl
from .backend import GpuBackend


@dataclass
class RelativeTruncation:
    """Truncation to a RELATIVE accuracy: every truncate call uses
    eps = rel * ||Y|| for its own input Y (the reference takes an
    absolute eps, solvers.py:196), optionally capped."""

    rel: float
    max_rank: int | None = None


@dataclass
class SolverConfig:
    """solvers.py:110-135 (the fields the CG loop uses)."""

    truncation: object  # TruncationControl or RelativeTruncation
    eps_stop: float = 1e-8
    max_cg_steps: int = 25


@dataclass
class TraceEntry:
    step: int
    true_rel_residual: float
    internal_residual: float
    max_rank: int
    seconds: float


@dataclass
class ConvergenceTrace:
    entries: list = field(default_factory=list)
    aborted: str | None = None

    def record(self, step, true_rel, internal, max_rank, seconds):
        self.entries.append(TraceEntry(step, true_rel, internal, max_rank, seconds))

    @property
    def floor(self) -> float:
        return min(e.true_rel_residual for e in self.entries)


def _true_residual(backend, op, x, b_neg, norm_b: float, ctl) -> float:
    """solvers.py:163-170: |A x - b| / |b| recomputed in tree arithmetic."""
    ax = backend.truncate(backend.apply(op, x), ctl)
    return backend.norm(backend.add(ax, b_neg)) / norm_b


def cg_solve(op, rhs, cfg: SolverConfig, backend=None, trace_residuals: bool = True):
    """solvers.py:172-186: X0 = rhs; stops when the internal residual norm drops to
    ``eps_stop`` or after ``max_cg_steps``; a non-positive curvature aborts."""
    backend = backend or GpuBackend()
    a = backend.lift_operator(op)
    b = backend.lift(rhs)
    trace = ConvergenceTrace()
    x = _cg_loop(a, b, cfg, backend, trace if trace_residuals else None)
    return backend.retrieve(x), trace


def _cg_loop(a, b, cfg: SolverConfig, backend, trace):
    """solvers.py:189-231."""
    ctl = cfg.truncation
    t0 = time.perf_counter()
    if trace is not None:
        b_neg = backend.scale(b, -1.0)
        norm_b = backend.norm(b)
    x = b
    r = backend.truncate(backend.add(b, backend.scale(backend.apply(a, x), -1.0)), ctl)
    d = r
    rr = backend.inner_product(r, r)
    if trace is not None:
        trace.record(0, _true_residual(backend, a, x, b_neg, norm_b, ctl), math.sqrt(max(0.0, rr)),
                     backend.max_rank(x), time.perf_counter() - t0)
    j = 0
    while math.sqrt(max(0.0, rr)) > cfg.eps_stop and j < cfg.max_cg_steps:
        z = backend.truncate(backend.apply(a, d), ctl)
        dz = backend.inner_product(d, z)
        if dz <= 0.0:
            if trace is not None:
                trace.aborted = f"non-positive curvature <D,AD> = {dz:.3e} at step {j}"
            break
        alpha = rr / dz
        x = backend.truncate(backend.add(x, backend.scale(d, alpha)), ctl)
        r_new = backend.truncate(backend.add(r, backend.scale(z, -alpha)), ctl)
        rr_new = backend.inner_product(r_new, r_new)
        beta = rr_new / rr
        d = backend.truncate(backend.add(backend.scale(d, beta), r_new), ctl)
        r, rr = r_new, rr_new
        j += 1
        if trace is not None:
            trace.record(j, _true_residual(backend, a, x, b_neg, norm_b, ctl), math.sqrt(max(0.0, rr)),
                         backend.max_rank(x), time.perf_counter() - t0)
    return x


__all__ = ["SolverConfig", "RelativeTruncation", "ConvergenceTrace", "TraceEntry", "cg_solve"]
