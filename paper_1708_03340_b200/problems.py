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


def distinct_parameter_grids(points: int = 16):
    """C4 with the parameter symmetry broken: parameter i samples [0.1 + 0.013 i,
    1.0 - 0.007 i] (still inside [0.1, 1.0]), so no two parameter modes are
    interchangeable and the truncations' kept subspaces are unique."""
    return [np.linspace(0.1 + 0.013 * i, 1.0 - 0.007 * i, points) for i in range(N_PARAMS)]


def kron_sum_operator(tree, terms: list, factors: dict, sizes: dict, device=None) -> HTOperator:
    """HT operator of a sum of Kronecker products  sum_j (x)_mu F_{j,mu}  with minimal ranks.

    ``terms[j]`` maps a mode mu (1-based) to a key of ``factors`` (the matrix F_{j,mu},
    a GeneralizedMatrix); modes a term does not mention carry the identity of size
    ``sizes[mu]``.  Construction (the matricisation view of an HT operator): at node t
    the operator is  sum_j L_j (x) R_j  with L_j / R_j the restrictions of term j to the
    modes inside / outside t.  Grouping the terms by their outside restriction R gives
    the column space of the matricisation: one column  sum_{j: R_j = R} L_j  per distinct
    R, with duplicates removed; this is the node's frame (ranks 1 + |params| and
    1 + |params outside| for C4's affine family).  Each transfer tensor then solves
    column_i(t) = sum_{j,l} B[i,j,l] column_j(s1) (x) column_l(s2) exactly (the columns
    are formal sums of elementary Kronecker products, so this is a small linear system
    over those products with 0/1 solutions).  Columns are ordered by the first term
    they contain."""
    d = tree.d
    cols = {}
    for node in tree.nodes:
        inside = tuple(node.dims)
        outside = tuple(mu for mu in range(1, d + 1) if mu not in set(inside))
        groups, first = {}, {}
        for j, term in enumerate(terms):
            key = tuple(term.get(mu) for mu in outside)
            u = tuple(term.get(mu) for mu in inside)
            g = groups.setdefault(key, {})
            g[u] = g.get(u, 0) + 1
            first.setdefault(key, j)
        frame = []
        for key in sorted(groups, key=first.get):
            if groups[key] not in frame:
                frame.append(groups[key])
        cols[node.index] = frame

    def leaf_matrix(formal, mu):
        """A leaf column: one factor, or a weighted sum of factors (terms that share
        everything outside this mode)."""
        mats = [(c, GeneralizedMatrix.diagonal(np.ones(sizes[mu])) if key is None else factors[key])
                for (key,), c in formal.items()]
        if len(mats) == 1 and mats[0][0] == 1:
            return mats[0][1]
        kinds = {g.kind for _, g in mats}
        if kinds == {"diagonal"}:
            return GeneralizedMatrix.diagonal(sum(c * g.data for c, g in mats))
        if "dense" not in kinds:
            import scipy.sparse as sp

            return GeneralizedMatrix.csr(sum(c * sp.csr_matrix(g.to_dense()) if g.kind == "diagonal" else c * g.data
                                             for c, g in mats))
        return GeneralizedMatrix.dense(sum(c * g.to_dense() for c, g in mats))

    leaves, transfer, root = {}, {}, None
    for node in tree.nodes:
        if node.is_leaf:
            leaves[node.index] = [leaf_matrix(f, node.dims[0]) for f in cols[node.index]]
            continue
        s1, s2 = node.sons
        n1 = len(tree.node(s1).dims)
        left, right, parent = cols[s1], cols[s2], cols[node.index]
        pairs = [(j, l) for j in range(len(left)) for l in range(len(right))]
        keys = {}
        for j, l in pairs:
            for u in left[j]:
                for v in right[l]:
                    keys.setdefault(u + v, len(keys))
        for f in parent:
            for uv in f:
                keys.setdefault(uv, len(keys))
        M = np.zeros((len(keys), len(pairs)))
        for c, (j, l) in enumerate(pairs):
            for u, a in left[j].items():
                for v, b in right[l].items():
                    M[keys[u + v], c] += a * b
        core = np.zeros((len(parent), len(left), len(right)))
        for i, f in enumerate(parent):
            rhs = np.zeros(len(keys))
            for uv, a in f.items():
                rhs[keys[uv]] = a
            sol = np.linalg.lstsq(M, rhs, rcond=None)[0]
            sol = np.round(sol)  # integer coefficients: exact 0/1 transfer tensors
            if not np.allclose(M @ sol, rhs):
                raise ValueError(f"node {node.index}: column {i} is not in the span of its sons' frames")
            core[i] = sol.reshape(len(left), len(right))
        assert n1 == len(tree.node(s1).dims)
        if node.is_root:
            root = core[0]
        else:
            transfer[node.index] = core
    return HTOperator(tree, leaves, transfer, root, device=device)


def affine_operator(matrices, grids, device=None) -> HTOperator:
    """HT operator of the affine family  A_0 (x) I + sum_mu A_mu (x) diag(grid_mu)
    (``matrices`` = [A_0, A_1 .. A_9] on the spatial mode, the last of the d = 10
    modes; parameter mu is mode mu): ten Kronecker terms handed to kron_sum_operator.
    Minimal ranks: 2 at the parameter leaves, 10 at the spatial leaf, 1 + (parameters
    owned) at parameter-only nodes, 1 + (parameters outside) at nodes holding space."""
    if len(matrices) != N_PARAMS + 1 or len(grids) != N_PARAMS:
        raise ValueError("expected 10 matrices and 9 parameter grids")
    tree = build_balanced_tree(SPATIAL_DIM)
    if SPATIAL_DIM not in tree.node(tree.node(0).sons[1]).dims:
        raise ValueError("the spatial mode must sit in the right subtree")
    factors = {("A", m): GeneralizedMatrix.csr(a) for m, a in enumerate(matrices)}
    factors.update({("D", mu): GeneralizedMatrix.diagonal(np.asarray(grids[mu - 1], dtype=np.float64))
                    for mu in range(1, N_PARAMS + 1)})
    terms = [{SPATIAL_DIM: ("A", 0)}] + [{SPATIAL_DIM: ("A", mu), mu: ("D", mu)} for mu in range(1, N_PARAMS + 1)]
    sizes = {mu: len(grids[mu - 1]) for mu in range(1, N_PARAMS + 1)}
    sizes[SPATIAL_DIM] = matrices[0].shape[0]
    return kron_sum_operator(tree, terms, factors, sizes, device=device)


def rank_one_tensor(tree, vectors: dict, device=None) -> HTensor:
    """The elementary tensor (x)_mu v_mu (``vectors[mu]``, 1-based modes) in HT format:
    every rank 1, every transfer tensor and the root equal to 1."""
    leaves = {tree.leaf_for_dim(mu).index: np.asarray(v, dtype=np.float64).reshape(-1, 1)
              for mu, v in vectors.items()}
    transfer = {n.index: np.ones((1, 1, 1)) for n in tree.inner_nodes}
    return HTensor(tree, leaves, transfer, np.ones((1, 1)), device=device)


def constant_rhs(load, grids, device=None) -> HTensor:
    """C4's right-hand side load (x) 1 (x) ... (x) 1: the source does not depend on the
    parameters (spatial mode last)."""
    tree = build_balanced_tree(SPATIAL_DIM)
    vectors = {mu: np.ones(len(grids[mu - 1])) for mu in range(1, N_PARAMS + 1)}
    vectors[SPATIAL_DIM] = load
    return rank_one_tensor(tree, vectors, device=device)


__all__ = ["p1_diffusion_matrices", "parameter_grids", "distinct_parameter_grids", "affine_operator",
           "kron_sum_operator", "rank_one_tensor", "constant_rhs", "N_PARAMS", "SPATIAL_DIM"]


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
