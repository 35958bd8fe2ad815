"""``GpuBackend`` -- the solver plugin seam of the reference (solvers.py:28-106).

Every solver of the reference package takes ``backend=`` and only calls these
eleven methods (``lift``, ``retrieve``, ``lift_operator``, ``apply``, ``add``,
``scale``, ``truncate``, ``inner_product``, ``norm``, ``leaf_map``,
``max_rank``).  ``GpuBackend`` implements them with the device-resident
``HTensor`` of this package, so ``htucker.solvers.cg_solve(op, rhs, cfg,
backend=GpuBackend(...))`` runs its whole loop on the B200 while the solver code
stays the reference's own.

Host objects are duck-typed: anything with ``tree.d``, ``leaves``, ``transfer``
and ``root_matrix`` (the reference ``HTensor``, format.py:50-132) lifts; an
operator additionally carries per-leaf lists of matrices with ``kind`` and
``data`` (the reference ``GeneralizedMatrix``, format.py:135-180).
``retrieve`` returns a device ``HTensor`` unless a ``host_factory(tree, leaves,
transfer, root)`` was given (e.g. ``htucker.HTensor``), in which case the
result is rebuilt on the host with the tree object the tensor was lifted with.
"""

from __future__ import annotations

import numpy as np

from . import arith
from .arith import TruncationControl
from .format import GeneralizedMatrix, HTensor, HTOperator
from .tree import build_balanced_tree


def _ctl(ctl) -> TruncationControl:
    """Accept the reference TruncationControl (eps / max_rank attributes) too."""
    if isinstance(ctl, TruncationControl):
        return ctl
    return TruncationControl(eps=getattr(ctl, "eps", None), max_rank=getattr(ctl, "max_rank", None))


def _gmat(m) -> GeneralizedMatrix:
    if isinstance(m, GeneralizedMatrix):
        return m
    kind = getattr(m, "kind", None)
    if kind == "dense":
        return GeneralizedMatrix.dense(m.data)
    if kind == "diagonal":
        return GeneralizedMatrix.diagonal(m.data)
    if kind == "csr":
        return GeneralizedMatrix.csr(m.data)
    return GeneralizedMatrix.dense(np.asarray(m))


class GpuBackend:
    """Solver arithmetic on one B200 (reference SerialBackend semantics: every
    operation returns a new tensor; ``truncate`` returns the truncated tensor)."""

    def __init__(self, host_factory=None, device=None):
        self.host_factory = host_factory
        self.device = device
        self._host_trees: dict = {}

    # -- movement ------------------------------------------------------------
    def lift(self, tensor) -> HTensor:
        if isinstance(tensor, HTensor):
            return tensor
        d = int(tensor.tree.d)
        self._host_trees[d] = tensor.tree
        return HTensor(build_balanced_tree(d), dict(tensor.leaves), dict(tensor.transfer), tensor.root_matrix,
                       getattr(tensor, "orthogonal", False), device=self.device)

    def retrieve(self, h: HTensor):
        if self.host_factory is None:
            return h
        leaves, transfer, root = h.to_numpy()
        tree = self._host_trees.get(h.tree.d, h.tree)
        return self.host_factory(tree, leaves, transfer, root)

    def lift_operator(self, op) -> HTOperator:
        if isinstance(op, HTOperator):
            return op
        d = int(op.tree.d)
        leaves = {t: [_gmat(m) for m in cols] for t, cols in op.leaves.items()}
        return HTOperator(build_balanced_tree(d), leaves, dict(op.transfer), op.root_matrix, device=self.device)

    # -- arithmetic (solvers.py:44-66) --------------------------------------
    def apply(self, op, x):
        return arith.apply_operator(op, x)

    def add(self, x, y):
        return arith.add(x, y)

    def scale(self, x, alpha: float):
        return arith.scale(x, float(alpha))

    def truncate(self, x, ctl):
        rel = getattr(ctl, "rel", None)
        if rel is not None:  # relative accuracy: eps = rel * ||x|| for this input, ||x|| taken on the device
            return arith.truncate(x, TruncationControl.relative_accuracy(rel, max_rank=ctl.max_rank))
        return arith.truncate(x, _ctl(ctl))

    def inner_product(self, x, y) -> float:
        return arith.inner_product(x, y)

    def norm(self, x) -> float:
        return arith.norm(x)

    def leaf_map(self, x, dim: int, matrix):
        return arith.leaf_map(x, dim, matrix)

    def max_rank(self, x) -> int:
        return x.max_rank


__all__ = ["GpuBackend"]
