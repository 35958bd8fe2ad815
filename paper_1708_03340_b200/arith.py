"""HT arithmetic on the GPU -- the drop-in for the reference ``htucker.arith``.

Same functions, signatures, semantics and exceptions as the reference
(arith.py:32-402); every one dispatches to the C ABI of ``libht_b200.so``
(include/ht_b200.h), whose level-batched sm_100a kernels do all the floating
point work.  Host code here only sizes workspaces, allocates outputs and reads
back the values the reference returns to the host (ranks in accuracy mode,
inner products).
"""

from __future__ import annotations

import ctypes
import os
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .format import F64, HTensor, HTOperator, node_shape


# ---------------------------------------------------------------------------
# truncation control (reference arith.py:32-66)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class TruncationControl:
    """Per-node rank choice: absolute ``eps`` (budget eps^2/(2d-2) per node) and/or
    a ``max_rank`` cap (int or per-node-id dict).  At least one must be set."""

    eps: float | None = None
    max_rank: int | dict | None = None
    # eps is relative to the norm of the tensor being truncated (HT_CTL_RELATIVE_EPS:
    # ||x|| is read off the orthogonalised root on the device; an extension of the
    # reference control, which only has an absolute eps)
    eps_is_relative: bool = False

    def __post_init__(self):
        if self.eps is None and self.max_rank is None:
            raise ValueError("truncation needs eps and/or max_rank")
        if self.eps is not None and self.eps <= 0:
            raise ValueError("eps must be positive")

    @staticmethod
    def fixed_rank(max_rank) -> "TruncationControl":
        return TruncationControl(eps=None, max_rank=max_rank)

    @staticmethod
    def accuracy(eps: float, max_rank=None) -> "TruncationControl":
        return TruncationControl(eps=eps, max_rank=max_rank)

    @staticmethod
    def relative(rel: float, norm_value: float, max_rank=None) -> "TruncationControl":
        """Relative accuracy rel*||Y|| (C3/C4 configs); the reference only has absolute eps."""
        return TruncationControl(eps=rel * norm_value, max_rank=max_rank)

    @staticmethod
    def relative_accuracy(rel: float, max_rank=None) -> "TruncationControl":
        """eps = rel * ||x|| for whatever tensor x the control is applied to; the norm is
        taken on the device inside the truncation (no separate inner product)."""
        return TruncationControl(eps=rel, max_rank=max_rank, eps_is_relative=True)

    def cap_for(self, node_id: int):
        if self.max_rank is None:
            return None
        if isinstance(self.max_rank, dict):
            return int(self.max_rank[node_id])
        return int(self.max_rank)

    def _c(self, nn: int):
        per = None
        cap = 0
        if isinstance(self.max_rank, dict):
            per = _lib.i64_array([0] + [int(self.max_rank[t]) for t in range(1, nn)])
        elif self.max_rank is not None:
            cap = int(self.max_rank)
            if cap <= 0:
                cap = 1  # select_rank keeps at least one column (arith.py:88)
        c = _lib.CTruncCtl(float(self.eps) if self.eps is not None else 0.0, cap,
                           ctypes.cast(per, ctypes.POINTER(ctypes.c_int64)) if per is not None else None)
        if self.eps_is_relative and self.eps is not None:
            c.flags = _lib.CTL_RELATIVE_EPS
        return c, per


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


_POISON_WS = os.environ.get("HT_POISON_WORKSPACE") == "1"


def _ws(nbytes: int, dev) -> torch.Tensor:
    w = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
    if _POISON_WS:  # debugging aid: NaN-fill so reads of unwritten workspace show up
        w.fill_(0xFF)
    return w


def _sizes_by_node(x: HTensor) -> dict:
    sz = x.__dict__.get("_sizes_cached")
    if sz is None:
        sz = {leaf.index: int(x.node_array(leaf.index).shape[0]) for leaf in x.tree.leaves}
        x._sizes_cached = sz
    return dict(sz)


def _check_compatible(a: HTensor, c: HTensor) -> None:
    """arith.py:398-402."""
    if a.tree.d != c.tree.d:
        raise ValueError(f"tensor dimensions differ: {a.tree.d} vs {c.tree.d}")
    if a.shape != c.shape:
        raise ValueError(f"tensor shapes differ: {a.shape} vs {c.shape}")


def _stream():
    return _lib.stream_handle()


# ---------------------------------------------------------------------------
# drop-in API
# ---------------------------------------------------------------------------


def add(a: HTensor, c: HTensor, out: HTensor | None = None, lazy: bool | None = None) -> HTensor:
    """arith.py:355-365: frames concatenate, transfers embed block-diagonally.  By
    default (``set_lazy_add``) the result is a ``SumHTensor``: the block-diagonal transfer
    tensors are not written until something other than ``truncate`` reads them.  ``out``
    (optional, an extension of the reference API): an existing tensor of the sum's
    shapes to write into -- an ordinary ``HTensor`` (materialised sum; pipelines reuse
    device buffers, and fixed buffers let the truncation replay its captured CUDA graphs
    without re-pointing them) or a ``SumHTensor`` returned by an earlier ``add`` of
    tensors of these shapes (its leaf arena is reused)."""
    return _add(a, c, 1.0, out, lazy)


def subtract(a: HTensor, c: HTensor) -> HTensor:
    """arith.py:374-375: add(a, scale(c, -1)) in one launch."""
    return _add(a, c, -1.0)


def _check_out(out: HTensor, tree, sizes: dict, ranks: dict) -> None:
    rl = out._rank_list()
    if out.tree.d != tree.d or _sizes_by_node(out) != sizes or \
            any(rl[t] != ranks[t] for t in range(1, len(tree.nodes))):
        raise ValueError("out tensor has the wrong shapes for this result")


_lazy_add = os.environ.get("HT_LAZY_ADD", "1") != "0"
# sums whose materialised transfer tensors are smaller than this many values are embedded
# at once: a tiny truncation is launch-latency-bound, and the block form costs it a few
# extra launches (C1: 0.35 ms materialised, 0.38 ms in block form)
_lazy_add_min_values = int(os.environ.get("HT_LAZY_ADD_MIN_VALUES", str(1 << 20)))


def set_lazy_add(on: bool, min_values: int | None = None) -> None:
    """``add`` / ``subtract`` return a ``SumHTensor`` (block-form sum, consumed in place by
    ``truncate``; default for sums whose transfer tensors hold at least ``min_values``
    values) or materialise the block-diagonal embedding at once."""
    global _lazy_add, _lazy_add_min_values
    _lazy_add = bool(on)
    if min_values is not None:
        _lazy_add_min_values = int(min_values)


def _transfer_values(a: HTensor, c: HTensor) -> int:
    tree, ra, rc = a.tree, a._rank_list(), c._rank_list()
    tot = 0
    for node in tree.inner_nodes:
        s1, s2 = node.sons
        tot += (ra[node.index] + rc[node.index]) * (ra[s1] + rc[s1]) * (ra[s2] + rc[s2])
    return tot


def _add(a: HTensor, c: HTensor, alpha_c: float, out: HTensor | None = None, lazy: bool | None = None) -> HTensor:
    _check_compatible(a, c)
    if lazy is None:
        if out is not None:
            lazy = isinstance(out, SumHTensor) and out._dense is None
        else:
            lazy = _lazy_add and (_transfer_values(a, c) >= _lazy_add_min_values
                                  or any(isinstance(t, SumHTensor) and t._dense is None for t in (a, c)))
    if lazy:
        terms = _sum_terms(a, 1.0) + _sum_terms(c, float(alpha_c))
        assert terms[0][0] == 1.0  # the first block carries no coefficient (as in the eager embedding)
        return SumHTensor._build(terms, a, c, out if isinstance(out, SumHTensor) else None)
    if isinstance(out, _LazyHTensor) and out._dense is None:
        raise ValueError("out tensor has the wrong shapes for this result")
    lib = _lib.load()
    tree = a.tree
    ra, rc = a._rank_list(), c._rank_list()
    ranks = {t: ra[t] + rc[t] for t in range(1, len(tree.nodes))}
    if out is None:
        out = HTensor.empty(tree, _sizes_by_node(a), ranks, device=a.device)
    else:
        _check_out(out, tree, _sizes_by_node(a), ranks)
        out.orthogonal = False
    _lib.check(lib.ht_add(a._c(), c._c(), float(alpha_c), out._c(), _stream()), "add")
    return out


def scale(a: HTensor, alpha: float) -> HTensor:
    """arith.py:368-371: alpha applied to the root matrix; leaves/transfers shared."""
    lib = _lib.load()
    root = a.root_matrix
    new_root = torch.empty_like(root)
    _lib.check(lib.ht_scale(root.data_ptr(), new_root.data_ptr(), root.numel(), float(alpha), _stream()), "scale")
    nodes = dict(a._nodes)
    nodes[0] = new_root
    return HTensor._wrap(a.tree, nodes, a.orthogonal)


def _bilinear_terms(x: HTensor) -> list | None:
    """[(alpha, term)] of an unmaterialised block-form sum, else None."""
    if "SumHTensor" in globals() and isinstance(x, SumHTensor) and x._dense is None:
        return list(x._terms)
    return None


def _inner_product_bilinear(a: HTensor, c: HTensor) -> torch.Tensor | None:
    """<sum_i a_i A_i, sum_j c_j C_j> = sum_ij a_i c_j <A_i, C_j> for block-form sums: the
    terms' (smaller-rank) inner products instead of a materialisation plus one inner
    product at the summed ranks.  None when neither operand is an unmaterialised sum."""
    ta, tc = _bilinear_terms(a), _bilinear_terms(c)
    if ta is None and tc is None:
        return None
    same = a is c
    ta = ta if ta is not None else [(1.0, a)]
    tc = tc if tc is not None else [(1.0, c)]
    acc = None
    for i, (al, x) in enumerate(ta):
        for j, (be, y) in enumerate(tc):
            if same and j < i:
                continue  # <A_i, A_j> = <A_j, A_i>
            w = al * be * (2.0 if same and j > i else 1.0)
            v = inner_product_device(x, y) * w
            acc = v if acc is None else acc + v
    return acc


def inner_product(a: HTensor, c: HTensor) -> float:
    """arith.py:246-265 (returns a host float; one device->host read)."""
    _check_compatible(a, c)
    bil = _inner_product_bilinear(a, c)
    if bil is not None:
        v = float(bil.item())
        _lib.check_status()
        return v
    lib = _lib.load()
    nbytes = ctypes.c_size_t(0)
    _lib.check(lib.ht_inner_product_workspace_size(a._c(), c._c(), ctypes.byref(nbytes)), "inner_product")
    ws = _ws(nbytes.value, a.device)
    res = torch.empty(1, dtype=F64, device=a.device)
    host = ctypes.c_double(0.0)
    _lib.check(lib.ht_inner_product(a._c(), c._c(), ws.data_ptr(), ws.numel(), res.data_ptr(),
                                    ctypes.byref(host), _stream()), "inner_product")
    _lib.check_status()  # host synchronisation point: errors of queued truncations surface here
    return float(host.value)


def inner_product_device(a: HTensor, c: HTensor) -> torch.Tensor:
    """Asynchronous variant: the inner product as a 1-element device tensor."""
    _check_compatible(a, c)
    bil = _inner_product_bilinear(a, c)
    if bil is not None:
        return bil
    lib = _lib.load()
    nbytes = ctypes.c_size_t(0)
    _lib.check(lib.ht_inner_product_workspace_size(a._c(), c._c(), ctypes.byref(nbytes)), "inner_product")
    ws = _ws(nbytes.value, a.device)
    res = torch.empty(1, dtype=F64, device=a.device)
    _lib.check(lib.ht_inner_product(a._c(), c._c(), ws.data_ptr(), ws.numel(), res.data_ptr(), None, _stream()),
               "inner_product")
    return res


def norm(a: HTensor) -> float:
    """arith.py:268-270."""
    return math.sqrt(max(0.0, inner_product(a, a)))


def orthogonalize(a: HTensor) -> HTensor:
    """arith.py:273-296: bottom-up batched Householder QR sweep."""
    lib = _lib.load()
    tree = a.tree
    nn = len(tree.nodes)
    rbuf = (ctypes.c_int64 * nn)()
    _lib.check(lib.ht_orth_ranks(a._c_trunc(), rbuf), "orthogonalize")
    ranks = {t: int(rbuf[t]) for t in range(1, nn)}
    out = HTensor.empty(tree, _sizes_by_node(a), ranks, orthogonal=True, device=a.device)
    nbytes = ctypes.c_size_t(0)
    _lib.check(lib.ht_orthogonalize_workspace_size(a._c_trunc(), ctypes.byref(nbytes)), "orthogonalize")
    ws = _ws(nbytes.value, a.device)
    _lib.check(lib.ht_orthogonalize(a._c_trunc(), ws.data_ptr(), ws.numel(), out._c(), _stream()), "orthogonalize")
    return out


def compute_bhat(a: HTensor) -> dict:
    """arith.py:299-322: reduced Gramians (device tensors) of every non-root node."""
    if not a.orthogonal:
        raise ValueError("tensor is not orthogonal; call orthogonalize() first")
    lib = _lib.load()
    tree = a.tree
    nn = len(tree.nodes)
    G = {t: torch.empty((a.rank(t), a.rank(t)), dtype=F64, device=a.device) for t in range(1, nn)}
    ptrs = _lib.ptr_array([0] + [G[t].data_ptr() for t in range(1, nn)])
    nbytes = ctypes.c_size_t(0)
    _lib.check(lib.ht_gramians_workspace_size(a._c(), ctypes.byref(nbytes)), "compute_bhat")
    ws = _ws(nbytes.value, a.device)
    _lib.check(lib.ht_gramians(a._c(), ws.data_ptr(), ws.numel(), ptrs, _stream()), "compute_bhat")
    return G


class _TruncState:
    """Workspace + ranks after phase 1 of a truncation (orth, Gramians, eig, select)."""

    def __init__(self, a: HTensor, ctl: TruncationControl):
        lib = _lib.load()
        self.a = a
        self.ctl = ctl
        nn = len(a.tree.nodes)
        self.cctl, self._keep = ctl._c(nn)
        nbytes = ctypes.c_size_t(0)
        _lib.check(lib.ht_truncate_workspace_size(a._c_trunc(), ctypes.byref(nbytes)), "truncate")
        self.ws = _ws(nbytes.value, a.device)
        rbuf = (ctypes.c_int64 * nn)()
        self.static = lib.ht_truncate_static_ranks(a._c_trunc(), ctypes.byref(self.cctl), rbuf) == 1
        self.ranks = {t: int(rbuf[t]) for t in range(1, nn)}
        self.phase1_done = False

    def run_phase1(self):
        lib = _lib.load()
        nn = len(self.a.tree.nodes)
        rbuf = (ctypes.c_int64 * nn)()
        _lib.check(lib.ht_truncate_ranks(self.a._c_trunc(), ctypes.byref(self.cctl), self.ws.data_ptr(), self.ws.numel(),
                                         rbuf, _stream()), "truncate")
        self.ranks = {t: int(rbuf[t]) for t in range(1, nn)}
        self.phase1_done = True


def truncate(a: HTensor, ctl: TruncationControl, out: HTensor | None = None) -> HTensor:
    """arith.py:325-352: orthogonalize if needed, reduced Gramians, batched
    eigendecompositions + rank choice, projection.  Result not orthogonal.  ``out``
    (optional, an extension of the reference API): an existing tensor of the result's
    shapes to write into -- only when the ranks follow from the control and the shapes
    (fixed-rank control), as they do not depend on the data then."""
    lib = _lib.load()
    st = _TruncState(a, ctl)
    if out is not None:
        if not st.static:
            raise ValueError("truncate(out=...) needs a control whose ranks follow from the shapes (max_rank only)")
        _check_out(out, a.tree, _sizes_by_node(a), st.ranks)
        out.orthogonal = False
    if st.static:
        if out is None:
            out = HTensor.empty(a.tree, _sizes_by_node(a), st.ranks, device=a.device)
        _lib.check(lib.ht_truncate(a._c_trunc(), ctypes.byref(st.cctl), st.ws.data_ptr(), st.ws.numel(), out._c(),
                                   _stream()), "truncate")
        return out
    st.run_phase1()
    out = HTensor.empty(a.tree, _sizes_by_node(a), st.ranks, device=a.device)
    _lib.check(lib.ht_truncate_project(a._c_trunc(), ctypes.byref(st.cctl), st.ws.data_ptr(), st.ws.numel(), out._c(),
                                       _stream()), "truncate")
    return out


def hierarchical_singular_values(a: HTensor) -> dict:
    """sigma_t = sqrt(lambda(Bhat_t)) per non-root node, descending (device tensors).
    The reference computes these inside truncate (arith.py:340-343) and discards them."""
    lib = _lib.load()
    st = _TruncState(a, TruncationControl.fixed_rank(1))
    st.cctl.flags = _lib.CTL_RELATIVE_SIGMA  # every sigma to relative accuracy (Jacobi on graded nodes)
    st.run_phase1()
    nn = len(a.tree.nodes)
    rbuf = (ctypes.c_int64 * nn)()
    _lib.check(lib.ht_orth_ranks(a._c_trunc(), rbuf), "orth ranks")
    ko = {t: (int(rbuf[t]) if not a.orthogonal else a.rank(t)) for t in range(1, nn)}
    total = sum(ko.values())
    lam = torch.empty(total, dtype=F64, device=a.device)
    _lib.check(lib.ht_truncate_eigenvalues(a._c_trunc(), st.ws.data_ptr(), st.ws.numel(), lam.data_ptr(), _stream()),
               "eigenvalues")
    out, off = {}, 0
    for t in range(1, nn):
        out[t] = torch.sqrt(lam[off:off + ko[t]])
        off += ko[t]
    return out


class _LazyHTensor(HTensor):
    """An ``HTensor`` whose transfer tensors and root are held in a structured form
    (Kronecker products / diagonal blocks) until something other than ``truncate`` /
    ``hierarchical_singular_values`` reads them.  Leaf frames are ordinary arrays in
    ``_leaf_arena``; ``_lazy`` keeps the C structs (and everything they point to) alive.
    Subclasses provide ``_materialize_now() -> HTensor``."""

    def _init_lazy(self, tree, sizes: dict, ranks: dict, dev, leaf_arena=None):
        nn = len(tree.nodes)
        self.tree = tree
        self.orthogonal = False
        self._cstruct = None
        self._dense = None
        self._ranks_cached = [1] + [ranks[t] for t in range(1, nn)]
        self._sizes_cached = dict(sizes)
        self._shape_cached = tuple(sizes[tree.leaf_for_dim(mu).index] for mu in range(1, tree.d + 1))
        self._lazy_dev = dev
        offs, total = {}, 0
        for t in sorted(leaf.index for leaf in tree.leaves):  # node-id order, 256-byte aligned frames
            offs[t] = total
            total += (sizes[t] * ranks[t] + 31) // 32 * 32
        if leaf_arena is None:
            leaf_arena = torch.empty(total, dtype=F64, device=dev)
        self._leaf_arena = leaf_arena
        base = leaf_arena.data_ptr()
        self._n_arr = _lib.i64_array(self._shape_cached)
        self._rk_arr = _lib.i64_array(self._ranks_cached)
        # leaf pointers; inner nodes get a placeholder (`base`) in the struct handed to the
        # node-masked kernels that fill the leaves, and NULL in the lazy struct
        self._leaf_ptrs = [base + 8 * offs[t] if t in offs else None for t in range(nn)]
        self._leaf_mask = (ctypes.c_uint8 * nn)(*[1 if t in offs else 0 for t in range(nn)])
        ph = _lib.ptr_array([p if p is not None else base for p in self._leaf_ptrs])
        self._leaf_cs = (_lib.CTensor(tree.d, ctypes.cast(self._n_arr, ctypes.POINTER(ctypes.c_int64)),
                                      ctypes.cast(self._rk_arr, ctypes.POINTER(ctypes.c_int64)),
                                      ctypes.cast(ph, ctypes.POINTER(ctypes.c_void_p)), 0), ph)

    def _lazy_struct(self, kron=None, sum_=None) -> _lib.CTensor:
        ptrs = _lib.ptr_array([p if p is not None else 0 for p in self._leaf_ptrs])
        cs = _lib.CTensor(self.tree.d, ctypes.cast(self._n_arr, ctypes.POINTER(ctypes.c_int64)),
                          ctypes.cast(self._rk_arr, ctypes.POINTER(ctypes.c_int64)),
                          ctypes.cast(ptrs, ctypes.POINTER(ctypes.c_void_p)), 0,
                          ctypes.cast(ctypes.pointer(kron), ctypes.c_void_p) if kron is not None else None,
                          ctypes.cast(ctypes.pointer(sum_), ctypes.c_void_p) if sum_ is not None else None)
        return cs, ptrs

    @property
    def is_materialized(self) -> bool:
        return self._dense is not None

    def _materialize(self) -> HTensor:
        if self._dense is None:
            self._dense = self._materialize_now()
            self._lazy = None
        return self._dense

    @property
    def _nodes(self):
        return self._materialize()._nodes

    @property
    def _arena(self):
        return self._materialize()._arena

    @property
    def device(self) -> torch.device:
        return self._dense.device if self._dense is not None else self._lazy_dev

    def _shape(self, t: int) -> tuple:
        if self._dense is not None:
            return self._dense._shape(t)
        node = self.tree.node(t)
        rl = self._ranks_cached
        if node.is_leaf:
            return (self._sizes_cached[t], rl[t])
        s1, s2 = node.sons
        return (rl[s1], rl[s2]) if node.is_root else (rl[t], rl[s1], rl[s2])

    def _c_trunc(self) -> _lib.CTensor:
        if self._dense is not None:
            return self._c()
        if self._lazy_dev.index != torch.cuda.current_device():
            raise ValueError(f"HTensor lives on cuda:{self._lazy_dev.index} but the current device is "
                             f"cuda:{torch.cuda.current_device()}; call under torch.cuda.device(...)")
        return self._lazy[0]


class AppliedHTensor(_LazyHTensor):
    """``apply_operator(op, x)`` with its transfer tensors kept in Kronecker form.

    The leaf frames V_t = [W_r U_t]_r are computed at once; the transfer tensors and
    the root F_t = H_t (x) B_t (reference arith.py:204-213) are NOT written to memory.
    ``truncate`` / ``hierarchical_singular_values`` consume H_t and B_t in place (the
    orthogonalisation sweep's first mode product runs against the small B_t; SURVEY
    K10b, ``ht_tensor.kron`` in include/ht_b200.h).  Anything else that reads the
    tensor (``transfer``, ``to_numpy``, ``add``, ``inner_product`` ...) materialises it
    first and from then on it is an ordinary ``HTensor``: the values are those of the
    eager ``apply_operator`` either way.  ``op`` and ``x`` are referenced (not copied)
    until then, so they must not be overwritten in place (``truncate(..., out=x)``).
    """

    @classmethod
    def _build(cls, op: HTOperator, x: HTensor) -> "AppliedHTensor":
        lib = _lib.load()
        tree = x.tree
        nn = len(tree.nodes)
        ranks = {t: op.rank(t) * x.rank(t) for t in range(1, nn)}
        sizes = {leaf.index: int(op.leaf_shape(leaf.index)[0]) for leaf in tree.leaves}
        obj = cls.__new__(cls)
        cop, cx = op._c(), x._c()
        obj._init_lazy(tree, sizes, ranks, x.device)
        obj._op, obj._x = op, x
        # leaf frames through the node-masked apply (inner nodes masked off)
        _lib.check(lib.ht_apply_operator_sharded(ctypes.byref(cop), cx, obj._leaf_mask, obj._leaf_cs[0], _stream()),
                   "apply_operator")
        src = _lib.CKronSrc(ctypes.pointer(cop), ctypes.pointer(cx))
        cs, ptrs = obj._lazy_struct(kron=src)
        obj._lazy = (cs, ptrs, src, cop, cx)
        return obj

    def _materialize_now(self) -> HTensor:
        lib = _lib.load()
        ranks = {t: self._ranks_cached[t] for t in range(1, len(self.tree.nodes))}
        out = HTensor.empty(self.tree, self._sizes_cached, ranks, device=self._lazy_dev)
        _lib.check(lib.ht_apply_operator(ctypes.byref(self._op._c()), self._x._c(), out._c(), _stream()),
                   "apply_operator")
        self._op = self._x = None
        return out


class SumHTensor(_LazyHTensor):
    """``add(a, c)`` (and sums of sums) held in block form: the leaf frames
    [U_1 .. U_p] are concatenated at once, the block-diagonal transfer tensors and root
    (reference arith.py:173-192) are NOT written to memory -- 1 - 1/p^2 of every inner
    node would be structural zeros.  ``truncate`` / ``hierarchical_singular_values``
    run the orthogonalisation sweep's mode products on the diagonal blocks
    (``ht_tensor.sum`` in include/ht_b200.h); anything else
    materialises the sum with the ordinary embedding kernel (same values as the eager
    ``add``).  The terms are referenced, not copied: overwrite them only after the
    sum has been consumed."""

    @classmethod
    def _build(cls, terms: list, a, c, out: "SumHTensor | None" = None) -> "SumHTensor":
        """terms: [(alpha, ordinary HTensor)]; a, c: the two operands of this add (ordinary
        tensors or unmaterialised sums), whose leaf frames are concatenated."""
        lib = _lib.load()
        tree = terms[0][1].tree
        nn = len(tree.nodes)
        ranks = {t: sum(x.rank(t) for _, x in terms) for t in range(1, nn)}
        sizes = _sizes_by_node(terms[0][1])
        if out is not None and out._dense is None and out._ranks_cached[1:] == [ranks[t] for t in range(1, nn)] \
                and out._sizes_cached == sizes and out._lazy_dev == terms[0][1].device:
            obj, arena = out, out._leaf_arena
        else:
            obj, arena = cls.__new__(cls), None
        obj._init_lazy(tree, sizes, ranks, terms[0][1].device, arena)
        obj._terms = list(terms)
        _lib.check(lib.ht_add_sharded(_leaf_view(a), _leaf_view(c), 1.0, obj._leaf_mask, obj._leaf_cs[0], _stream()),
                   "add")
        structs = [x._c() for _, x in terms]
        tarr = (ctypes.POINTER(_lib.CTensor) * len(terms))(*[ctypes.pointer(cs) for cs in structs])
        alphas = (ctypes.c_double * len(terms))(*[float(al) for al, _ in terms])
        src = _lib.CSumSrc(len(terms), tarr, alphas)
        cs, ptrs = obj._lazy_struct(sum_=src)
        obj._lazy = (cs, ptrs, src, tarr, alphas, structs)
        return obj

    def _materialize_now(self) -> HTensor:
        acc = None
        for alpha, x in self._terms:
            acc = x if acc is None else _add(acc, x, alpha, lazy=False)
        self._terms = None
        return acc


def _leaf_view(x: HTensor) -> _lib.CTensor:
    """C view good for the leaf frames of x (what the node-masked add reads)."""
    if isinstance(x, _LazyHTensor) and x._dense is None:
        return x._leaf_cs[0]
    return x._c()


def _sum_terms(x: HTensor, alpha: float) -> list:
    if isinstance(x, SumHTensor) and x._dense is None and alpha in (1.0, -1.0):
        return [(alpha * al, t) for al, t in x._terms]
    if isinstance(x, _LazyHTensor):
        x = x._materialize()
    return [(alpha, x)]


_lazy_apply = os.environ.get("HT_LAZY_APPLY", "1") != "0"


def set_lazy_apply(on: bool) -> None:
    """``apply_operator`` returns an ``AppliedHTensor`` (Kronecker-form transfer tensors,
    consumed in place by ``truncate``; default) or materialises every F_t at once."""
    global _lazy_apply
    _lazy_apply = bool(on)


def apply_operator(op: HTOperator, a: HTensor, lazy: bool | None = None) -> HTensor:
    """arith.py:378-395 (Lemma 4): ranks multiply, operator index slow.  ``lazy`` (default:
    ``set_lazy_apply``, on) keeps the transfer tensors H_t (x) B_t unmaterialised until
    something other than ``truncate`` reads them (``AppliedHTensor``)."""
    tree = a.tree
    if op.tree.d != tree.d:
        raise ValueError(f"operator dimension {op.tree.d} != tensor dimension {tree.d}")
    if op.col_sizes != a.shape:
        raise ValueError(f"operator column sizes {op.col_sizes} do not match tensor shape {a.shape}")
    if _lazy_apply if lazy is None else lazy:
        return AppliedHTensor._build(op, a)
    lib = _lib.load()
    ranks = {t: op.rank(t) * a.rank(t) for t in range(1, len(tree.nodes))}
    sizes = {leaf.index: int(op.leaf_shape(leaf.index)[0]) for leaf in tree.leaves}
    out = HTensor.empty(tree, sizes, ranks, device=a.device)
    _lib.check(lib.ht_apply_operator(ctypes.byref(op._c()), a._c(), out._c(), _stream()), "apply_operator")
    return out


_QR_MODES = {"auto": 0, "householder": 1, "cholqr2": 2}
_qr_mode = "auto"


def set_qr_mode(mode: str) -> None:
    """QR policy of the orthogonalisation sweep (process-wide): ``"auto"`` (default)
    runs Cholesky-QR on DMMA GEMMs where eligible (second pass only where the
    estimated condition number exceeds 20) and re-runs the sweep with Householder QR
    when its device-side check fails; ``"cholqr2"`` always runs both passes;
    ``"householder"`` always uses the Householder tree-TSQR.  All return the
    reference's sign-fixed QR (kernels.py:24-32) up to rounding."""
    global _qr_mode
    if mode not in _QR_MODES:
        raise ValueError(f"qr mode must be one of {sorted(_QR_MODES)}")
    _lib.check(_lib.load().ht_set_qr_mode(_QR_MODES[mode]), "set_qr_mode")
    _qr_mode = mode


def get_qr_mode() -> str:
    return _qr_mode


def set_implicit_q(on: bool) -> None:
    """Implicit-Q truncation (process-wide, default on): the Cholesky-QR sweep keeps the
    absorbed transfer tensors and R^-1 instead of forming Q = M23(B') R^-1, and the
    Gramian / projection phases fold R^-1 into their small operands.  Off forms Q
    explicitly; both compute reference arith.py:325-352."""
    _lib.check(_lib.load().ht_set_implicit_q(1 if on else 0), "set_implicit_q")


_EIG_MODES = {"auto": 0, "jacobi": 1}
_eig_mode = "auto"


def set_eig_mode(mode: str) -> None:
    """Eigensolver policy of truncate (process-wide): ``"auto"`` (default) runs the
    tridiagonal fast path and redoes graded / near-degenerate nodes with Jacobi;
    ``"jacobi"`` uses Jacobi everywhere.  Both match sym_eig_desc (kernels.py:35-54)."""
    global _eig_mode
    if mode not in _EIG_MODES:
        raise ValueError(f"eig mode must be one of {sorted(_EIG_MODES)}")
    _lib.check(_lib.load().ht_set_eig_mode(_EIG_MODES[mode]), "set_eig_mode")
    _eig_mode = mode


def get_eig_mode() -> str:
    return _eig_mode


def evaluate_entries(a: HTensor, indices) -> torch.Tensor:
    """X[i] for a batch of 0-based multi-indices (B x d, host or device), on the device.
    Batched form of the reference's evaluate_entry (arith.py:221-243); IndexError on
    an out-of-bounds index, as there."""
    idx = torch.as_tensor(indices, dtype=torch.int64)
    if idx.dim() == 1:
        idx = idx[None, :]
    if idx.dim() != 2 or idx.shape[1] != a.tree.d:
        raise IndexError(f"indices must be B x {a.tree.d}")
    shape = torch.tensor(a.shape, dtype=torch.int64, device=idx.device)
    if idx.numel() and (bool((idx < 0).any()) or bool((idx >= shape).any())):
        bad = idx[((idx < 0) | (idx >= shape)).any(dim=1)][0].tolist()
        raise IndexError(f"index {tuple(bad)} out of bounds for shape {a.shape}")
    idx = idx.to(a.device).contiguous()
    out = torch.empty(idx.shape[0], dtype=F64, device=a.device)
    _lib.check(_lib.load().ht_evaluate_entries(a._c(), idx.data_ptr(), idx.shape[0], out.data_ptr(), _stream()),
               "evaluate_entries")
    return out


def evaluate_entry(a: HTensor, index) -> float:
    """One tensor entry (reference arith.py:221-243)."""
    index = tuple(int(i) for i in index)
    if len(index) != a.tree.d or any(not 0 <= i < n for i, n in zip(index, a.shape)):
        raise IndexError(f"index {index} out of bounds for shape {a.shape}")
    v = float(evaluate_entries(a, [index])[0].item())
    _lib.check_status()
    return v


def synchronize() -> None:
    """Wait for the queued work of the current stream and raise any error a queued
    truncation recorded (fixed-rank truncations do not read their status back)."""
    _lib.check_status()


def set_graph_mode(on: bool) -> None:
    """CUDA-graph replay of repeated fixed-rank truncations (process-wide, default on).
    Same kernels and arguments as the eager launches, so results are identical."""
    _lib.check(_lib.load().ht_set_graph_mode(1 if on else 0), "set_graph_mode")


def set_graph_relocation(on: bool) -> None:
    """Re-point cached truncation graphs at moved buffers instead of capturing a graph per
    address combination (process-wide; off by default, ``HT_RELOC=1`` turns it on)."""
    _lib.check(_lib.load().ht_set_graph_relocation(1 if on else 0), "set_graph_relocation")


def graph_relocations() -> int:
    """How many cached truncation graphs were relocated to new buffer addresses."""
    return int(_lib.load().ht_graph_relocations())


def graph_stats() -> tuple:
    """(captures, replays) of the truncation graph cache."""
    c, r = ctypes.c_int64(0), ctypes.c_int64(0)
    _lib.check(_lib.load().ht_graph_stats(ctypes.byref(c), ctypes.byref(r)), "graph_stats")
    return int(c.value), int(r.value)


def qr_fallback_count() -> int:
    """How many Cholesky-QR2 sweeps were recomputed with Householder QR."""
    return int(_lib.load().ht_qr_fallback_count())


def gemm(A: torch.Tensor, B: torch.Tensor, out: torch.Tensor | None = None, alpha=1.0, beta=0.0) -> torch.Tensor:
    """C = alpha A B + beta C on the DMMA kernel (row-major 2-D CUDA float64)."""
    lib = _lib.load()
    M, K = A.shape
    K2, N = B.shape
    if K != K2:
        raise ValueError("inner dimensions differ")
    if out is None:
        out = torch.empty((M, N), dtype=F64, device=A.device)
    _lib.check(lib.ht_gemm_strided(M, N, K, 1, float(alpha), A.data_ptr(), A.stride(0), A.stride(1), 0,
                                   B.data_ptr(), B.stride(0), B.stride(1), 0, float(beta), out.data_ptr(),
                                   out.stride(0), out.stride(1), 0, _stream()), "gemm")
    return out


def leaf_map(x: HTensor, dim: int, matrix) -> HTensor:
    """Replace the frame of mode ``dim`` by ``matrix @ U`` (solvers.py:58-62)."""
    leaf = x.tree.leaf_for_dim(dim)
    M = matrix if isinstance(matrix, torch.Tensor) else torch.as_tensor(np.asarray(matrix, dtype=np.float64))
    M = M.to(x.device, F64).contiguous()
    U = x.node_array(leaf.index)
    nodes = dict(x._nodes)
    nodes[leaf.index] = gemm(M, U)
    return HTensor._wrap(x.tree, nodes, False)


def _check_all():
    return _lib.load()


__all__ = ["set_graph_relocation", "AppliedHTensor", "SumHTensor", "set_lazy_apply", "set_lazy_add", "TruncationControl", "add", "subtract", "scale", "inner_product", "inner_product_device", "norm",
           "orthogonalize", "compute_bhat", "truncate", "hierarchical_singular_values", "apply_operator",
           "gemm", "leaf_map", "synchronize"]
