"""Parameter-dependent diffusion model problem (BASELINE config C4), host-side setup.

  -div(a(x; p) grad u) = 1 on the unit square, u = 0 on the boundary, with a
  piecewise-constant coefficient a = p_mu on the mu-th cell of a 3 x 3 grid of
  subdomains and each p_mu sampled on a grid of values.

P1 finite elements on a uniform mesh (each square cell split into two right
triangles) give stiffness matrices K_mu of the subdomains; the parametric
operator is the affine family  A = A_0 (x) I (x) ... (x) I + sum_mu K_mu (x) D_mu
with D_mu = diag(grid_mu), stored as an HT operator of minimal ranks in the tree
of the reference's cookie problem (d = 10: parameter modes 1..9, space last;
reference cookie.py:189-300 builds the same family, and its test CG drives it
through solvers.cg_solve).  The reference ships a Q1 assembler for circular
"cookies"; the P1 / 3 x 3-subdomain variant is BASELINE C4's own statement.

These are problem-setup utilities (numpy / scipy on the host); the solve itself
runs through ``solvers.cg_solve`` on ``GpuBackend``.
"""

from __future__ import annotations

import numpy as np

from .format import GeneralizedMatrix, HTensor, HTOperator
from .tree import build_balanced_tree

N_PARAMS = 9
SPATIAL_DIM = 10


def p1_diffusion_matrices(cells: int = 64, sub: int = 3):
    """Stiffness matrices of the ``sub x sub`` subdomains and the load vector of
    the unit source, Dirichlet nodes eliminated: ``(cells - 1)**2`` unknowns
    (3969 for the 64 x 64 mesh of C4).  Returns (list of scipy CSR, ndarray)."""
    import scipy.sparse as sp

    h = 1.0 / cells
    ni = cells - 1

    def dof(ix, iy):  # interior numbering, None on the boundary
        if ix <= 0 or iy <= 0 or ix >= cells or iy >= cells:
            return None
        return (iy - 1) * ni + (ix - 1)

    # reference-triangle gradients: the P1 stiffness of a right triangle with legs h
    # is independent of h in 2-D: for vertices (right angle, x-leg, y-leg)
    k_right = np.array([[1.0, -0.5, -0.5], [-0.5, 0.5, 0.0], [-0.5, 0.0, 0.5]])
    rows = [[] for _ in range(sub * sub)]
    cols = [[] for _ in range(sub * sub)]
    vals = [[] for _ in range(sub * sub)]
    load = np.zeros(ni * ni)
    area = 0.5 * h * h
    for cy in range(cells):
        for cx in range(cells):
            mu = min(int((cy + 0.5) * sub / cells), sub - 1) * sub + min(int((cx + 0.5) * sub / cells), sub - 1)
            # lower-left triangle: right angle at (cx, cy); upper-right: right angle at (cx+1, cy+1)
            for tri in (((cx, cy), (cx + 1, cy), (cx, cy + 1)), ((cx + 1, cy + 1), (cx, cy + 1), (cx + 1, cy))):
                ids = [dof(*v) for v in tri]
                for a in range(3):
                    if ids[a] is None:
                        continue
                    load[ids[a]] += area / 3.0
                    for b in range(3):
                        if ids[b] is None:
                            continue
                        rows[mu].append(ids[a])
                        cols[mu].append(ids[b])
                        vals[mu].append(k_right[a, b])
    mats = [sp.csr_matrix((vals[m], (rows[m], cols[m])), shape=(ni * ni, ni * ni)) for m in range(sub * sub)]
    for m in mats:
        m.sum_duplicates()
        m.sort_indices()
    return mats, load


def parameter_grids(points: int = 16, lo: float = 0.1, hi: float = 1.0):
    """BASELINE C4: 16 samples uniform in [0.1, 1.0] per parameter (np.linspace)."""
    return [np.linspace(lo, hi, points) for _ in range(N_PARAMS)]


def _params(node):
    return [mu for mu in node.dims if mu <= N_PARAMS]


def _has_space(node):
    return node.interval[1] == SPATIAL_DIM


def _columns(node):
    """Column meaning of an operator node: slot 0 is the identity (parameter-only
    nodes) or the complete partial operator (nodes containing space); the other
    slots are the parameters owned (parameter-only nodes) or still outside (space)."""
    if _has_space(node):
        return [0] + [mu for mu in range(1, N_PARAMS + 1) if mu not in set(node.dims)]
    return [0] + _params(node)


def affine_operator(matrices, grids, device=None) -> HTOperator:
    """HT operator of ``matrices[0] (x) I + sum_mu matrices[mu] (x) diag(grids[mu-1])``
    (``matrices`` = [A_0, A_1 .. A_9]) with minimal ranks: 2 at the parameter leaves,
    1 + (number of parameters outside) for the nodes containing space (10 at the
    spatial leaf), 1 + (parameters owned) elsewhere."""
    if len(matrices) != N_PARAMS + 1 or len(grids) != N_PARAMS:
        raise ValueError("expected 10 matrices and 9 parameter grids")
    tree = build_balanced_tree(SPATIAL_DIM)
    leaves = {}
    for mu in range(1, N_PARAMS + 1):
        g = np.asarray(grids[mu - 1], dtype=np.float64)
        leaves[tree.leaf_for_dim(mu).index] = [GeneralizedMatrix.diagonal(np.ones(g.size)),
                                               GeneralizedMatrix.diagonal(g)]
    leaves[tree.leaf_for_dim(SPATIAL_DIM).index] = [GeneralizedMatrix.csr(m) for m in matrices]
    transfer, root = {}, None
    for node in tree.nodes:
        if node.is_leaf:
            continue
        left, right = tree.sons(node.index)
        if _has_space(left):
            raise ValueError("the spatial mode must sit in the right subtree")
        ct, cl, cr = _columns(node), _columns(left), _columns(right)
        it = {c: i for i, c in enumerate(ct)}
        il = {c: i for i, c in enumerate(cl)}
        ir = {c: i for i, c in enumerate(cr)}
        core = np.zeros((len(ct), len(cl), len(cr)))
        core[0, 0, 0] = 1.0  # identity (x) identity, or identity (x) complete
        if _has_space(node):
            for mu in _params(left):  # absorb: parameter mu of the left son meets slot mu on the right
                core[0, il[mu], ir[mu]] = 1.0
            for nu in ct[1:]:  # pass-through slots of parameters still outside
                core[it[nu], 0, ir[nu]] = 1.0
        else:
            for mu in _params(left):
                core[it[mu], il[mu], 0] = 1.0
            for mu in _params(right):
                core[it[mu], 0, ir[mu]] = 1.0
        if node.is_root:
            root = core[0]
        else:
            transfer[node.index] = core
    return HTOperator(tree, leaves, transfer, root, device=device)


def constant_rhs(load, grids, device=None) -> HTensor:
    """Rank-1 right-hand side: the load vector on the spatial leaf, ones on every
    parameter leaf (the source does not depend on the parameters)."""
    tree = build_balanced_tree(SPATIAL_DIM)
    leaves = {tree.leaf_for_dim(mu).index: np.ones((len(grids[mu - 1]), 1)) for mu in range(1, N_PARAMS + 1)}
    leaves[tree.leaf_for_dim(SPATIAL_DIM).index] = np.asarray(load, dtype=np.float64).reshape(-1, 1)
    transfer = {n.index: np.ones((1, 1, 1)) for n in tree.inner_nodes}
    return HTensor(tree, leaves, transfer, np.ones((1, 1)), device=device)


__all__ = ["p1_diffusion_matrices", "parameter_grids", "affine_operator", "constant_rhs", "N_PARAMS", "SPATIAL_DIM"]


def laplace_sum_operator(tree, n: int, device=None) -> HTOperator:
    """BASELINE config C3's operator: sum_mu I (x) .. (x) L_mu (x) .. (x) I with
    L = tridiag(-1, 2, -1) of size n, in HT format of ranks 2 (root 1) -- the
    same construction the reference's tests use for Laplace-like operators
    (format.py:183-250 layout): leaf columns [I, L]; every transfer tensor
    H[0,0,0] = H[1,1,0] = H[1,0,1] = 1; root [[0, 1], [1, 0]]."""
    import scipy.sparse as sp

    lap = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")
    lap.sort_indices()
    leaves = {leaf.index: [GeneralizedMatrix.diagonal(np.ones(n)), GeneralizedMatrix.csr(lap)]
              for leaf in tree.leaves}
    h = np.zeros((2, 2, 2))
    h[0, 0, 0] = h[1, 1, 0] = h[1, 0, 1] = 1.0
    transfer = {node.index: h.copy() for node in tree.nodes if not node.is_leaf and not node.is_root}
    return HTOperator(tree, leaves, transfer, np.array([[0.0, 1.0], [1.0, 0.0]]), device=device)


# -- evaluation over the parameter directions (reference cookie.py:359-426) ----------


def _spatial_readout(x: HTensor, leaf_weights: dict, param_rows: list) -> "torch.Tensor":
    """X contracted over every parameter mode, the spatial (last) mode left open: one
    device upward pass per spatial index (``ht_evaluate_weighted``); parameter leaves
    contribute the weighted row w^T U (leaf_weights[mu]) or the frame row U[i, :]
    (param_rows[mu]).  Same value as the reference's _upward_spatial_pass
    (cookie.py:362-380), reassociated per spatial entry."""
    import ctypes

    import torch

    from . import _lib
    from .arith import _stream

    d = x.tree.d
    n_sp = x.shape[d - 1]
    idx = torch.zeros((n_sp, d), dtype=torch.int64)
    for mu, i in enumerate(param_rows):
        if i is not None:
            idx[:, mu] = int(i)
    idx[:, d - 1] = torch.arange(n_sp, dtype=torch.int64)
    idx = idx.to(x.device).contiguous()
    ws = [None] * d
    for mu, w in leaf_weights.items():
        ws[mu] = torch.as_tensor(w, dtype=torch.float64).to(x.device).contiguous()
    ptrs = (ctypes.c_void_p * d)(*[w.data_ptr() if w is not None else None for w in ws])
    out = torch.empty(n_sp, dtype=torch.float64, device=x.device)
    _lib.check(_lib.load().ht_evaluate_weighted(x._c(), ctypes.cast(ptrs, ctypes.c_void_p), idx.data_ptr(),
                                                 n_sp, out.data_ptr(), _stream()), "evaluate_weighted")
    return out


def extract_solution(x: HTensor, param_indices) -> "torch.Tensor":
    """Spatial vector at one parameter-index combination (0-based), on the device
    (reference cookie.py:383-404): ValueError unless d-1 indices, IndexError when one
    is out of bounds, as there."""
    d = x.tree.d
    param_indices = tuple(int(i) for i in param_indices)
    if len(param_indices) != d - 1:
        raise ValueError(f"need {d - 1} parameter indices")
    shape = x.shape
    for mu, i in enumerate(param_indices):
        if not 0 <= i < shape[mu]:
            raise IndexError(f"parameter index {i} out of bounds for dimension {mu + 1} of size {shape[mu]}")
    return _spatial_readout(x, {}, list(param_indices))


def parameter_mean(x: HTensor, weights=None) -> "torch.Tensor":
    """Weighted contraction over all parameter grids (default uniform), on the device
    (reference cookie.py:407-426): ValueError on a weight vector of the wrong length."""
    d = x.tree.d
    shape = x.shape
    lw = {}
    for mu in range(d - 1):
        n = shape[mu]
        w = np.full(n, 1.0 / n) if weights is None else np.asarray(
            weights[mu].cpu() if hasattr(weights[mu], "cpu") else weights[mu], dtype=float)
        if w.shape != (n,):
            raise ValueError(f"weight length {w.shape} mismatches dimension {mu + 1} of size {n}")
        lw[mu] = w
    return _spatial_readout(x, lw, [None] * (d - 1))
