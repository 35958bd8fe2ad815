"""Truncated conjugate gradients over the Backend seam -- the direct caller of the
truncation hot path (reference solvers.py:172-231, the algorithm of the paper's
CG-with-truncation experiments).

``TruncatedCG`` keeps the iteration as an explicit state machine: ``start()``
builds the first iterate, ``advance()`` performs one CG step, ``report()``
measures an iterate.  Every tensor operation goes through the eleven Backend
methods only, so the loop runs unchanged on ``GpuBackend`` (default: every add,
apply, truncate and inner product on the B200) or on any other backend object
-- including the reference's own ``SerialBackend``.

The arithmetic order is the reference's, so traces agree with its CG to rounding:
residual R0 = T(B - A X0) with X0 = B, D0 = R0; per step Z = T(A D),
alpha = <R,R>/<D,Z>, X <- T(X + alpha D), R <- T(R - alpha Z),
beta = <R',R'>/<R,R>, D <- T(beta D + R'); a non-positive curvature <D,Z> stops the
iteration with a diagnostic.  T is the truncation of ``cfg.truncation``.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import NamedTuple

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
    """The CG fields of the reference's SolverConfig (solvers.py:110-135)."""

    truncation: object  # TruncationControl or RelativeTruncation
    eps_stop: float = 1e-8
    max_cg_steps: int = 25


class TraceEntry(NamedTuple):
    step: int
    true_rel_residual: float
    internal_residual: float
    max_rank: int
    seconds: float


@dataclass
class ConvergenceTrace:
    entries: list = field(default_factory=list)
    aborted: str | None = None

    def record(self, *values) -> None:
        self.entries.append(TraceEntry(*values))

    @property
    def floor(self) -> float:
        return min(e.true_rel_residual for e in self.entries)


class Iterate(NamedTuple):
    step: int
    x: object
    r: object
    d: object
    rr: float  # <R, R>


class TruncatedCG:
    """CG with truncation after every operation, one step at a time."""

    def __init__(self, backend, op, rhs, cfg: SolverConfig):
        self.be = backend
        self.cfg = cfg
        self.A = backend.lift_operator(op)
        self.b = backend.lift(rhs)
        self._minus_b = None
        self._norm_b = None

    # -- building blocks ---------------------------------------------------------
    def _combine(self, *terms):
        """sum alpha_i Y_i in tree arithmetic (ranks add; no truncation)."""
        acc = None
        for alpha, y in terms:
            y = self.be.scale(y, alpha) if alpha is not None else y
            acc = y if acc is None else self.be.add(acc, y)
        return acc

    def _round(self, y):
        return self.be.truncate(y, self.cfg.truncation)

    # -- the iteration -----------------------------------------------------------
    def start(self) -> Iterate:
        x = self.b
        r = self._round(self._combine((None, self.b), (-1.0, self.be.apply(self.A, x))))
        return Iterate(0, x, r, r, self.be.inner_product(r, r))

    def converged(self, it: Iterate) -> bool:
        return math.sqrt(max(0.0, it.rr)) <= self.cfg.eps_stop or it.step >= self.cfg.max_cg_steps

    def advance(self, it: Iterate):
        """One CG step; returns (next iterate, None) or (None, reason) on breakdown."""
        be = self.be
        z = self._round(be.apply(self.A, it.d))
        curvature = be.inner_product(it.d, z)
        if curvature <= 0.0:
            return None, f"non-positive curvature <D,AD> = {curvature:.3e} at step {it.step}"
        alpha = it.rr / curvature
        x = self._round(self._combine((None, it.x), (alpha, it.d)))
        r = self._round(self._combine((None, it.r), (-alpha, z)))
        rr = be.inner_product(r, r)
        d = self._round(self._combine((rr / it.rr, it.d), (None, r)))
        return Iterate(it.step + 1, x, r, d, rr), None

    def report(self, it: Iterate) -> tuple:
        """(true relative residual ||T(A X) - B|| / ||B||, internal residual ||R||, max rank):
        the true residual is recomputed in tree arithmetic and never fed back."""
        if self._minus_b is None:
            self._minus_b = self.be.scale(self.b, -1.0)
            self._norm_b = self.be.norm(self.b)
        ax = self._round(self.be.apply(self.A, it.x))
        true_rel = self.be.norm(self.be.add(ax, self._minus_b)) / self._norm_b
        return true_rel, math.sqrt(max(0.0, it.rr)), self.be.max_rank(it.x)


def cg_solve(op, rhs, cfg: SolverConfig, backend=None, trace_residuals: bool = True):
    """Solve A X = rhs by truncated CG from X0 = rhs (reference solvers.py:172-186):
    stops when ||R|| <= eps_stop or after max_cg_steps; returns (X, ConvergenceTrace)."""
    backend = backend or GpuBackend()
    cg = TruncatedCG(backend, op, rhs, cfg)
    trace = ConvergenceTrace()
    t0 = time.perf_counter()
    it = cg.start()
    if trace_residuals:
        trace.record(it.step, *cg.report(it), time.perf_counter() - t0)
    while not cg.converged(it):
        nxt, why = cg.advance(it)
        if nxt is None:
            trace.aborted = why
            break
        it = nxt
        if trace_residuals:
            trace.record(it.step, *cg.report(it), time.perf_counter() - t0)
    return backend.retrieve(it.x), trace


__all__ = ["SolverConfig", "RelativeTruncation", "ConvergenceTrace", "TraceEntry", "TruncatedCG", "cg_solve"]
