"""CPU oracle: a numpy restatement of the reference HT arithmetic.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_1708_03340_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` legs use it, and only as the checker or
the timed CPU baseline.

Every function restates the algorithm of the reference package
``/root/reference/pkg/src/htucker`` (arXiv 1708.03340) and cites the
``file:line`` it follows.  Dense linear algebra goes through the same
LAPACK/BLAS entry points the reference uses (numpy 2.3.5 ->
scipy-openblas 0.3.30: ``dgeqrf``/``dorgqr`` for QR, ``dsyevd`` for the
symmetric eigenproblem, ``dgemm`` for contractions).

Pinning: the oracle is checked against fixtures produced by running the
reference itself in the build container (``tests/golden/make_golden.py``,
``tests/test_oracle_golden.py``) and against the SPEC's known answers.

Conventions (reference ``arith.py:10-12``, ``kernels.py:5-9``): leaf frames
``U[t]`` are ``(n, k)`` C-order; transfer tensors ``B[t]`` are
``(k_t, k_s1, k_s2)`` indexed ``B[i, j, l]`` with ``i`` the node's own rank;
the root matrix is ``(k_s1, k_s2)``; composite indices run last-mode-fastest.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# dimension tree (reference tree.py:55-101, 139-145)
# ---------------------------------------------------------------------------


@dataclass
class Tree:
    """Balanced dimension tree with breadth-first node ids (root = 0).

    ``interval[t]`` is the inclusive 1-based mode range, ``sons[t]`` is None
    for leaves, ``level[t]`` the depth.  Split of ``{mu..nu}`` at
    ``(mu + nu - 1) // 2`` (tree.py:55-57).
    """

    d: int
    interval: list = field(default_factory=list)
    father: list = field(default_factory=list)
    sons: list = field(default_factory=list)
    level: list = field(default_factory=list)

    @property
    def n_nodes(self) -> int:
        return len(self.interval)

    def is_leaf(self, t: int) -> bool:
        return self.sons[t] is None

    def leaf_of_dim(self, mu: int) -> int:
        for t in range(self.n_nodes):
            if self.sons[t] is None and self.interval[t][0] == mu:
                return t
        raise KeyError(mu)

    def leaves_by_dim(self) -> list:
        return [self.leaf_of_dim(mu) for mu in range(1, self.d + 1)]

    def inner_ids(self) -> list:
        return [t for t in range(1, self.n_nodes) if self.sons[t] is not None]

    def levels(self) -> list:
        depth = max(self.level)
        out = [[] for _ in range(depth + 1)]
        for t in range(self.n_nodes):
            out[self.level[t]].append(t)
        return out


def balanced_tree(d: int) -> Tree:
    """tree.py:78-101 (BFS construction) restated with an explicit queue."""
    if d < 2:
        raise ValueError(f"tensor dimension must be >= 2, got {d}")
    tr = Tree(d)
    queue = [((1, d), None, 0)]
    head = 0
    while head < len(queue):
        (mu, nu), fa, lev = queue[head]
        t = head
        head += 1
        tr.interval.append((mu, nu))
        tr.father.append(fa)
        tr.level.append(lev)
        tr.sons.append(None)
        if fa is not None:
            tr.sons[fa] = tr.sons[fa] + (t,)  # left son is queued (and numbered) first
        if mu != nu:
            cut = (mu + nu - 1) // 2
            queue.append(((mu, cut), t, lev + 1))
            queue.append(((cut + 1, nu), t, lev + 1))
            tr.sons[t] = ()
    return tr


# ---------------------------------------------------------------------------
# container (reference format.py:50-132)
# ---------------------------------------------------------------------------


@dataclass
class HT:
    """HT tensor: ``U`` leaf frames, ``B`` transfer tensors, ``root`` matrix."""

    tree: Tree
    U: dict
    B: dict
    root: np.ndarray
    orthogonal: bool = False

    def rank(self, t: int) -> int:
        if t == 0:
            return 1
        return self.U[t].shape[1] if self.tree.is_leaf(t) else self.B[t].shape[0]

    @property
    def ranks(self) -> dict:
        return {t: self.rank(t) for t in range(1, self.tree.n_nodes)}

    @property
    def shape(self) -> tuple:
        return tuple(self.U[t].shape[0] for t in self.tree.leaves_by_dim())

    def arrays(self):
        """(node id, array) in BFS id order -- the storage order used everywhere."""
        for t in range(self.tree.n_nodes):
            if t == 0:
                yield t, self.root
            elif self.tree.is_leaf(t):
                yield t, self.U[t]
            else:
                yield t, self.B[t]

    def check(self) -> None:
        """format.py:101-119 rank-chain invariant."""
        tr = self.tree
        for t in range(tr.n_nodes):
            if tr.is_leaf(t):
                continue
            s1, s2 = tr.sons[t]
            got = self.root.shape if t == 0 else self.B[t].shape[1:]
            if tuple(got) != (self.rank(s1), self.rank(s2)):
                raise ValueError(f"rank chain broken at node {t}")


def storage(x: HT) -> int:
    """format.py:459-464."""
    return int(sum(a.size for _, a in x.arrays()))


# ---------------------------------------------------------------------------
# dense primitives (reference kernels.py:24-54, 92-121)
# ---------------------------------------------------------------------------


def qr_signfixed(a: np.ndarray):
    """kernels.py:24-32: Householder QR (LAPACK dgeqrf+dorgqr), diag(R) >= 0."""
    q, r = np.linalg.qr(np.asarray(a, dtype=np.float64), mode="reduced")
    s = np.ones(r.shape[0])
    s[np.diagonal(r) < 0.0] = -1.0
    return q * s[None, :], r * s[:, None]


def eig_desc(s: np.ndarray, rtol: float = 1e-12):
    """kernels.py:35-54: symmetric check, dsyevd, stable descending, clamp >= 0."""
    s = np.asarray(s, dtype=np.float64)
    if s.ndim != 2 or s.shape[0] != s.shape[1]:
        raise ValueError(f"matrix is not square: {s.shape}")
    bound = rtol * max(1.0, float(np.max(np.abs(s), initial=0.0)))
    if float(np.max(np.abs(s - s.T), initial=0.0)) > bound:
        raise ValueError("matrix is not symmetric within tolerance")
    lam, vec = np.linalg.eigh(0.5 * (s + s.T))
    perm = np.argsort(-lam, kind="stable")
    return vec[:, perm], np.clip(lam[perm], 0.0, None)


def m23(b: np.ndarray) -> np.ndarray:
    """kernels.py:107-115: (k_t,k1,k2) -> (k1*k2, k_t), mode 3 fastest."""
    kt, k1, k2 = b.shape
    return np.transpose(b, (1, 2, 0)).reshape(k1 * k2, kt)


def m23_inv(m: np.ndarray, k1: int, k2: int) -> np.ndarray:
    """kernels.py:118-121."""
    return np.transpose(m.reshape(k1, k2, m.shape[1]), (2, 0, 1))


# ---------------------------------------------------------------------------
# truncation control (reference arith.py:32-88)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Ctl:
    """arith.py:32-66: absolute ``eps`` and/or ``max_rank`` (int or per-node dict)."""

    eps: float | None = None
    max_rank: object = None

    def __post_init__(self):
        if self.eps is None and self.max_rank is None:
            raise ValueError("truncation needs eps and/or max_rank")
        if self.eps is not None and self.eps <= 0:
            raise ValueError("eps must be positive")

    def cap(self, t: int):
        if self.max_rank is None:
            return None
        if isinstance(self.max_rank, dict):
            return int(self.max_rank[t])
        return int(self.max_rank)


def pick_rank(lam: np.ndarray, ctl: Ctl, t: int, n_nonroot: int) -> int:
    """arith.py:69-88: smallest r with tail(lam[r:]) <= eps^2/(2d-2); cap; >= 1."""
    k = lam.shape[0]
    r = k
    if ctl.eps is not None:
        budget = ctl.eps ** 2 / n_nonroot
        tail = np.append(np.cumsum(lam[::-1])[::-1], 0.0)  # tail[r] = sum lam[r:]
        r = int(np.argmax(tail <= budget))
    c = ctl.cap(t)
    if c is not None:
        r = min(r, c)
    return max(1, min(r, k))


# ---------------------------------------------------------------------------
# node kernels (reference arith.py:105-213)
# ---------------------------------------------------------------------------


def node_orth_inner(b, r1, r2):
    """arith.py:130-141: absorb son R factors (modes 2,3), QR of M23."""
    b2 = np.einsum("pj,ijl->ipl", r1, b, optimize=True)
    b3 = np.einsum("ql,ipl->ipq", r2, b2, optimize=True)
    q, r = qr_signfixed(m23(b3))
    return m23_inv(q, r1.shape[0], r2.shape[0]), r


def node_gram_sons(core, g):
    """arith.py:148-158 / PAPER:715-723: reduced Gramians of both sons."""
    t1 = np.tensordot(g, core, axes=(1, 0))
    g1 = np.einsum("ijl,iql->jq", core, t1, optimize=True)
    g2 = np.einsum("ijl,ijq->lq", core, t1, optimize=True)
    return 0.5 * (g1 + g1.T), 0.5 * (g2 + g2.T)


def node_project_inner(b, qt, q1, q2):
    """arith.py:161-170: (Q_t^T, Q1^T, Q2^T) applied to modes 1, 2, 3 in that order."""
    c = np.tensordot(qt.T, b, axes=(1, 0))
    c = np.einsum("ja,iab->ijb", q1.T, c, optimize=True)
    return np.einsum("lb,ijb->ijl", q2.T, c, optimize=True)


def node_phi_inner(ba, bc, p1, p2):
    """arith.py:109-118: Phi_t[i,i'] = sum B_a[i,j,l] P1[j,j'] P2[l,l'] B_c[i',j',l']."""
    s = np.tensordot(ba, p1, axes=(1, 0))        # (ka, la, jc)
    s = np.tensordot(s, p2, axes=(1, 0))         # (ka, jc, lc)
    return np.tensordot(s, bc, axes=((1, 2), (1, 2)))


def node_add_inner(ba, bc):
    """arith.py:177-183: block-diagonal embedding."""
    out = np.zeros(tuple(x + y for x, y in zip(ba.shape, bc.shape)))
    out[: ba.shape[0], : ba.shape[1], : ba.shape[2]] = ba
    out[ba.shape[0]:, ba.shape[1]:, ba.shape[2]:] = bc
    return out


def node_add_root(ra, rc):
    """arith.py:186-192."""
    out = np.zeros((ra.shape[0] + rc.shape[0], ra.shape[1] + rc.shape[1]))
    out[: ra.shape[0], : ra.shape[1]] = ra
    out[ra.shape[0]:, ra.shape[1]:] = rc
    return out


def node_apply_inner(h, b):
    """arith.py:204-209: Kronecker transfer tensor, operator index slow."""
    p, q, r = h.shape
    i, j, l = b.shape
    return (h[:, None, :, None, :, None] * b[None, :, None, :, None, :]).reshape(p * i, q * j, r * l)


# ---------------------------------------------------------------------------
# operators (reference format.py:135-250)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class GMat:
    """format.py:135-180: 'dense' | 'diagonal' | 'csr' linear map."""

    kind: str
    data: object

    @property
    def shape(self):
        if self.kind == "diagonal":
            return (self.data.shape[0], self.data.shape[0])
        return self.data.shape

    def matmat(self, x):
        if self.kind == "diagonal":
            return self.data[:, None] * x
        if self.kind == "csr":
            return np.asarray(self.data @ x)
        return self.data @ x

    def dense(self):
        if self.kind == "diagonal":
            return np.diag(self.data)
        if self.kind == "csr":
            return self.data.toarray()
        return np.asarray(self.data)


@dataclass
class HTOp:
    """format.py:183-250: leaf lists of GMat columns + transfer/root like HT."""

    tree: Tree
    W: dict
    H: dict
    root: np.ndarray

    def rank(self, t):
        if t == 0:
            return 1
        return len(self.W[t]) if self.tree.is_leaf(t) else self.H[t].shape[0]

    @property
    def col_sizes(self):
        return tuple(self.W[t][0].shape[1] for t in self.tree.leaves_by_dim())


# ---------------------------------------------------------------------------
# level-wise drivers (reference arith.py:246-395)
# ---------------------------------------------------------------------------


def _bottom_up(tr: Tree):
    for lev in reversed(tr.levels()):
        yield from lev


def _same_shape(a: HT, c: HT):
    """arith.py:398-402."""
    if a.tree.d != c.tree.d:
        raise ValueError(f"tensor dimensions differ: {a.tree.d} vs {c.tree.d}")
    if a.shape != c.shape:
        raise ValueError(f"tensor shapes differ: {a.shape} vs {c.shape}")


def add(a: HT, c: HT) -> HT:
    """arith.py:355-365 (Lemma 3)."""
    _same_shape(a, c)
    tr = a.tree
    U = {t: np.concatenate([a.U[t], c.U[t]], axis=1) for t in a.U}
    B = {t: node_add_inner(a.B[t], c.B[t]) for t in a.B}
    return HT(tr, U, B, node_add_root(a.root, c.root))


def scale(a: HT, alpha: float) -> HT:
    """arith.py:368-371 (keeps the orthogonal flag, shares arrays)."""
    return HT(a.tree, a.U, a.B, alpha * a.root, a.orthogonal)


def subtract(a: HT, c: HT) -> HT:
    """arith.py:374-375."""
    return add(a, scale(c, -1.0))


def inner_product(a: HT, c: HT) -> float:
    """arith.py:246-265 with phi_leaf/phi_inner/phi_root (arith.py:105-123)."""
    _same_shape(a, c)
    tr = a.tree
    phi = {}
    for t in _bottom_up(tr):
        if tr.is_leaf(t):
            phi[t] = a.U[t].T @ c.U[t]
        elif t == 0:
            s1, s2 = tr.sons[0]
            return float(np.sum((phi[s1].T @ a.root @ phi[s2]) * c.root))
        else:
            s1, s2 = tr.sons[t]
            phi[t] = node_phi_inner(a.B[t], c.B[t], phi[s1], phi[s2])
    raise AssertionError


def norm(a: HT) -> float:
    """arith.py:268-270."""
    return math.sqrt(max(0.0, inner_product(a, a)))


def orthogonalize(a: HT) -> HT:
    """arith.py:273-296: bottom-up QR sweep; R factors travel to the fathers."""
    tr = a.tree
    U, B, R = {}, {}, {}
    root = a.root
    for t in _bottom_up(tr):
        if tr.is_leaf(t):
            U[t], R[t] = qr_signfixed(a.U[t])
        elif t == 0:
            s1, s2 = tr.sons[0]
            root = R[s1] @ a.root @ R[s2].T  # arith.py:144-145
        else:
            s1, s2 = tr.sons[t]
            B[t], R[t] = node_orth_inner(a.B[t], R[s1], R[s2])
    return HT(tr, U, B, root, orthogonal=True)


def reduced_gramians(a: HT) -> dict:
    """arith.py:299-322 (compute_bhat): top-down, root seeded with G=[[1]]."""
    if not a.orthogonal:
        raise ValueError("tensor is not orthogonal; call orthogonalize() first")
    tr = a.tree
    G = {}
    for lev in tr.levels():
        for t in lev:
            if tr.is_leaf(t):
                continue
            if t == 0:
                core, own = a.root[None, :, :], np.ones((1, 1))
            else:
                core, own = a.B[t], G[t]
            s1, s2 = tr.sons[t]
            G[s1], G[s2] = node_gram_sons(core, own)
    return G


def truncate(a: HT, ctl: Ctl, return_info: bool = False):
    """arith.py:325-352: orthogonalize, Gramians, eig + rank per node, project."""
    if not a.orthogonal:
        a = orthogonalize(a)
    tr = a.tree
    G = reduced_gramians(a)
    nnr = tr.n_nodes - 1
    Q, lams = {}, {}
    for t in range(1, tr.n_nodes):
        vec, lam = eig_desc(G[t])
        Q[t] = vec[:, : pick_rank(lam, ctl, t, nnr)]
        lams[t] = lam
    U = {t: a.U[t] @ Q[t] for t in a.U}
    B = {t: node_project_inner(a.B[t], Q[t], Q[tr.sons[t][0]], Q[tr.sons[t][1]]) for t in a.B}
    s1, s2 = tr.sons[0]
    out = HT(tr, U, B, Q[s1].T @ a.root @ Q[s2], orthogonal=False)
    if return_info:
        return out, {"eigenvalues": lams, "gramians": G, "orthogonalized": a}
    return out


def apply_operator(op: HTOp, a: HT) -> HT:
    """arith.py:378-395 (Lemma 4): ranks multiply, operator index slow."""
    tr = a.tree
    if op.tree.d != tr.d:
        raise ValueError(f"operator dimension {op.tree.d} != tensor dimension {tr.d}")
    if op.col_sizes != a.shape:
        raise ValueError("operator column sizes do not match tensor shape")
    U = {t: np.concatenate([w.matmat(a.U[t]) for w in op.W[t]], axis=1) for t in a.U}
    B = {t: node_apply_inner(op.H[t], a.B[t]) for t in a.B}
    return HT(tr, U, B, np.kron(op.root, a.root))


def evaluate_entry(a: HT, index) -> float:
    """arith.py:221-243: leaf rows combined upward."""
    tr = a.tree
    rows = {}
    for t in _bottom_up(tr):
        if tr.is_leaf(t):
            rows[t] = a.U[t][index[tr.interval[t][0] - 1], :]
        elif t == 0:
            s1, s2 = tr.sons[0]
            return float(rows[s1] @ a.root @ rows[s2])
        else:
            s1, s2 = tr.sons[t]
            rows[t] = np.einsum("qjl,j,l->q", a.B[t], rows[s1], rows[s2])
    raise AssertionError


def _upward_spatial_pass(a: HT, leaf_values: dict) -> np.ndarray:
    """cookie.py:362-380: parameter leaves contribute row vectors, the spatial (last)
    leaf its full frame; nodes holding the spatial mode carry (n x k_t) matrices
    (einsum "qjl,j,nl->nq"), the root returns v2 @ (B_D^T v1)."""
    tr = a.tree
    vals = dict(leaf_values)
    for t in _bottom_up(tr):
        if tr.is_leaf(t):
            continue
        s1, s2 = tr.sons[t]
        v1, v2 = vals[s1], vals[s2]
        if t == 0:
            return v2 @ (a.root.T @ v1)
        if tr.interval[t][1] == tr.d:
            vals[t] = np.einsum("qjl,j,nl->nq", a.B[t], v1, v2)
        else:
            vals[t] = np.einsum("qjl,j,l->q", a.B[t], v1, v2)
    raise AssertionError


def extract_solution(a: HT, param_indices) -> np.ndarray:
    """cookie.py:383-404: spatial vector at one parameter-index combination."""
    tr = a.tree
    param_indices = tuple(int(i) for i in param_indices)
    if len(param_indices) != tr.d - 1:
        raise ValueError(f"need {tr.d - 1} parameter indices")
    vals = {}
    for mu in range(1, tr.d):
        f = a.U[tr.leaf_of_dim(mu)]
        if not 0 <= param_indices[mu - 1] < f.shape[0]:
            raise IndexError(f"parameter index {param_indices[mu - 1]} out of bounds")
        vals[tr.leaf_of_dim(mu)] = f[param_indices[mu - 1], :]
    vals[tr.leaf_of_dim(tr.d)] = a.U[tr.leaf_of_dim(tr.d)]
    return _upward_spatial_pass(a, vals)


def parameter_mean(a: HT, weights=None) -> np.ndarray:
    """cookie.py:407-426: weighted contraction over all parameter grids (default
    uniform)."""
    tr = a.tree
    vals = {}
    for mu in range(1, tr.d):
        f = a.U[tr.leaf_of_dim(mu)]
        w = np.full(f.shape[0], 1.0 / f.shape[0]) if weights is None else np.asarray(weights[mu - 1], float)
        if w.shape != (f.shape[0],):
            raise ValueError(f"weight length {w.shape} mismatches dimension {mu}")
        vals[tr.leaf_of_dim(mu)] = w @ f
    vals[tr.leaf_of_dim(tr.d)] = a.U[tr.leaf_of_dim(tr.d)]
    return _upward_spatial_pass(a, vals)


def to_dense(a: HT) -> np.ndarray:
    """format.py:342-383: explicit frames bottom-up (desk-scale only)."""
    tr = a.tree
    F = {}
    for t in _bottom_up(tr):
        if tr.is_leaf(t):
            F[t] = a.U[t]
            continue
        s1, s2 = tr.sons[t]
        if t == 0:
            full = np.einsum("jl,aj,bl->ab", a.root, F[s1], F[s2])
            return full.reshape(a.shape)
        F[t] = np.einsum("qjl,aj,bl->abq", a.B[t], F[s1], F[s2]).reshape(
            F[s1].shape[0] * F[s2].shape[0], -1)
    raise AssertionError


# ---------------------------------------------------------------------------
# derived quantities used by the parity gates (SURVEY §8(c) gaps 3-4)
# ---------------------------------------------------------------------------


def hierarchical_singular_values(a: HT) -> dict:
    """sigma_t = sqrt(lambda(Bhat_t)) of the orthogonalized tensor (kernels.py:35-54,
    arith.py:273-322); the reference computes these inside truncate (arith.py:340-343)
    and discards them."""
    o = a if a.orthogonal else orthogonalize(a)
    G = reduced_gramians(o)
    return {t: np.sqrt(eig_desc(G[t])[1]) for t in G}


def orth_difference_norm(x: HT, y: HT) -> float:
    """||x - y||_F via the root of orthogonalize(x - y) (SURVEY finding 0.3.3)."""
    return float(np.linalg.norm(orthogonalize(subtract(x, y)).root))


# ---------------------------------------------------------------------------
# CG with truncation (solvers.py:172-231): the direct caller of the hot path
# ---------------------------------------------------------------------------


def ones_htensor(tr: Tree, n: int) -> HT:
    """Rank-1 all-ones tensor (the reference's constant right-hand side shape)."""
    U = {t: np.ones((n, 1)) for t in tr.leaves_by_dim()}
    B = {t: np.ones((1, 1, 1)) for t in tr.inner_ids()}
    return HT(tr, U, B, np.ones((1, 1)))


def cg_solve(op: HTOp, rhs: HT, ctl, eps_stop: float, max_steps: int):
    """solvers.py:183-231 (_cg_loop with trace): X0 = rhs, truncation after every
    add / apply, stop on sqrt(<R,R>) <= eps_stop or max_steps, abort on <D,AD> <= 0.
    ``ctl`` is a Ctl or a callable y -> Ctl (per-call control, e.g. relative eps).
    Returns (X, internal residuals, true relative residuals)."""
    def trunc(y):
        return truncate(y, ctl(y) if callable(ctl) else ctl)

    b = rhs
    b_neg = scale(b, -1.0)
    norm_b = norm(b)

    def true_res(x):  # solvers.py:163-170
        ax = trunc(apply_operator(op, x))
        return norm(add(ax, b_neg)) / norm_b

    x = b
    r = trunc(add(b, scale(apply_operator(op, x), -1.0)))
    d = r
    rr = inner_product(r, r)
    internal, true = [math.sqrt(max(0.0, rr))], [true_res(x)]
    j = 0
    while math.sqrt(max(0.0, rr)) > eps_stop and j < max_steps:
        z = trunc(apply_operator(op, d))
        dz = inner_product(d, z)
        if dz <= 0.0:
            break
        alpha = rr / dz
        x = trunc(add(x, scale(d, alpha)))
        r_new = trunc(add(r, scale(z, -alpha)))
        rr_new = inner_product(r_new, r_new)
        beta = rr_new / rr
        d = trunc(add(scale(d, beta), r_new))
        r, rr = r_new, rr_new
        j += 1
        internal.append(math.sqrt(max(0.0, rr)))
        true.append(true_res(x))
    return x, internal, true


# ---------------------------------------------------------------------------
# seeded generators
# ---------------------------------------------------------------------------


def _pow2_scale(v: float) -> float:
    return 2.0 ** (-round(math.log2(v)))


def gaussian_htensor(tr: Tree, n, k, seed: int, scaled: bool = True) -> HT:
    """N(0,1) factors in random_htensor's node order (format.py:283-300) from
    ``PCG64(seed).standard_normal``; with ``scaled`` leaves are multiplied by
    2^-round(log2 sqrt(n)) and transfer/root tensors by 2^-round(log2 k) --
    an exact power-of-two rescale that keeps large-d sums finite."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    if np.isscalar(n):
        sizes = {t: int(n) for t in tr.leaves_by_dim()}
    else:
        sizes = {tr.leaf_of_dim(mu): int(n[mu - 1]) for mu in range(1, tr.d + 1)}
    ranks = ({t: int(k[t]) for t in range(1, tr.n_nodes)} if isinstance(k, dict)
             else {t: int(k) for t in range(1, tr.n_nodes)})
    U, B, root = {}, {}, None
    for t in range(tr.n_nodes):
        if tr.is_leaf(t):
            nn, kk = sizes[t], ranks[t]
            if kk > nn:
                raise ValueError(f"leaf rank {kk} exceeds size {nn} at node {t}")
            U[t] = rng.standard_normal((nn, kk))
            if scaled:
                U[t] *= _pow2_scale(math.sqrt(nn))
            continue
        s1, s2 = tr.sons[t]
        k1, k2 = ranks[s1], ranks[s2]
        if t == 0:
            root = rng.standard_normal((k1, k2))
            if scaled:
                root *= _pow2_scale(max(k1, k2))
            continue
        kt = ranks[t]
        if kt > k1 * k2:
            raise ValueError(f"rank {kt} at node {t} exceeds structural bound {k1 * k2}")
        B[t] = rng.standard_normal((kt, k1, k2))
        if scaled:
            B[t] *= _pow2_scale(kt)
    return HT(tr, U, B, root)


def laplace_operator(tr: Tree, n: int) -> HTOp:
    """Sum_mu I x .. x L_mu x .. x I with L = tridiag(-1, 2, -1) of size n, as an
    HT operator of ranks 2 (SURVEY §8(c) gap 5): leaves [I, L]; inner
    H[0,0,0] = H[1,1,0] = H[1,0,1] = 1; root [[0,1],[1,0]]."""
    import scipy.sparse as sp

    lap = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")
    lap.sort_indices()
    W = {t: [GMat("diagonal", np.ones(n)), GMat("csr", lap)] for t in tr.leaves_by_dim()}
    H = {}
    for t in tr.inner_ids():
        h = np.zeros((2, 2, 2))
        h[0, 0, 0] = h[1, 1, 0] = h[1, 0, 1] = 1.0
        H[t] = h
    return HTOp(tr, W, H, np.array([[0.0, 1.0], [1.0, 0.0]]))


def c1_inputs():
    """BASELINE config 0 (C1): d=8, n=64, k=10, A seed 0, C seed 1,
    X = add(scale(A, 2), scale(C, 1e-10)), ranks 20 -> fixed_rank(10)."""
    tr = balanced_tree(8)
    a = gaussian_htensor(tr, 64, 10, 0)
    c = gaussian_htensor(tr, 64, 10, 1)
    return a, c, add(scale(a, 2.0), scale(c, 1e-10))


def c2_inputs(d: int, n: int = 1000, k: int = 50, seed_base: int | None = None):
    """BASELINE config 1 (C2): A seed 2p, C seed 2p+1 (p = log2 d), X = add(A, C)."""
    tr = balanced_tree(d)
    p = int(round(math.log2(d)))
    s = 2 * p if seed_base is None else seed_base
    a = gaussian_htensor(tr, n, k, s)
    c = gaussian_htensor(tr, n, k, s + 1)
    return a, c, add(a, c)


def c5_inputs(d: int = 256, n: int = 2048, k: int = 100):
    """BASELINE config 4 (C5): four rank-k Gaussian tensors, seeds 0..3; the caller sums
    them in the fixed order ((A0 + A1) + A2) + A3 (rank 4k)."""
    tr = balanced_tree(d)
    return [gaussian_htensor(tr, n, k, s) for s in range(4)]
