"""Device-resident HT containers (mirror of the reference ``htucker.format``).

:class:`HTensor` keeps the reference constructor ``HTensor(tree, leaves,
transfer, root_matrix, orthogonal=False)`` (format.py:50-132) but stores every
node array in HBM as a float64 CUDA tensor.  Arrays created by this package
live in one contiguous *arena* per tensor (node arrays in breadth-first id
order, C-order -- exactly the layout the C ABI expects), so host<->device
transfer of a whole tensor is a single copy.  Node arrays may also be shared
between tensors (``scale`` reuses leaves and transfers like arith.py:370-371).
"""

from __future__ import annotations

import ctypes
import math
import os
from collections.abc import Mapping

import numpy as np
import torch

from . import _lib

_POISON = os.environ.get("HT_POISON_WORKSPACE") == "1"
from .tree import DimensionTree, build_balanced_tree

F64 = torch.float64


def _device(device=None) -> torch.device:
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1708_03340_b200 needs a CUDA device (B200); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def node_shape(tree: DimensionTree, t: int, sizes: dict, ranks: dict) -> tuple:
    """C-order shape of node ``t`` given leaf sizes (by node id) and ranks (by node id)."""
    node = tree.node(t)
    if node.is_leaf:
        return (sizes[t], ranks[t])
    s1, s2 = node.sons
    if node.is_root:
        return (ranks[s1], ranks[s2])
    return (ranks[t], ranks[s1], ranks[s2])


class _ArenaViews(Mapping):
    """Node arrays of an arena-backed tensor, built as views on first access.

    Outputs of add / truncate / apply are arena-backed; building all 2d-1 views
    eagerly cost ~0.6 ms of host time per d=64 call, so only the arena, the offsets
    and the shapes are kept until a node array is actually asked for.
    """

    __slots__ = ("arena", "offsets", "shapes", "_views")

    def __init__(self, arena: torch.Tensor, offsets: list, shapes: list):
        self.arena, self.offsets, self.shapes = arena, offsets, shapes
        self._views = [None] * len(shapes)

    def __getitem__(self, t):
        v = self._views[t]
        if v is None:
            o, s = self.offsets[t], self.shapes[t]
            v = self.arena[o:o + math.prod(s)].view(s)
            self._views[t] = v
        return v

    def __iter__(self):
        return iter(range(len(self.shapes)))

    def __len__(self):
        return len(self.shapes)

    def __contains__(self, t):
        return isinstance(t, int) and 0 <= t < len(self.shapes)

    def get(self, t, default=None):
        return self[t] if t in self else default

    def pointers(self) -> list:
        base = self.arena.data_ptr()
        return [base + 8 * o for o in self.offsets]


def _arena_views(arena: torch.Tensor, shapes: list) -> _ArenaViews:
    offsets, off = [], 0
    for s in shapes:
        offsets.append(off)
        off += math.prod(s)
    return _ArenaViews(arena, offsets, shapes)


class HTensor:
    """A tensor in hierarchical Tucker format, resident on the GPU.

    ``leaves``/``transfer``/``root_matrix`` accept numpy arrays or torch tensors
    (copied to the device in one transfer) exactly like the reference
    constructor; the attributes hold CUDA float64 tensors.
    """

    def __init__(self, tree: DimensionTree, leaves: dict, transfer: dict, root_matrix,
                 orthogonal: bool = False, *, device=None):
        self.tree = tree
        self.orthogonal = bool(orthogonal)
        arrays = {}
        for t, u in leaves.items():
            arrays[int(t)] = u
        for t, b in transfer.items():
            arrays[int(t)] = b
        arrays[0] = root_matrix
        if all(isinstance(v, torch.Tensor) and v.is_cuda and v.dtype == F64 for v in arrays.values()):
            self._nodes = {t: v.contiguous() for t, v in arrays.items()}
            self._arena = None
        else:
            self._nodes, self._arena = _upload(tree, arrays, _device(device))
        self._cstruct = None
        self.validate()

    # -- internal constructors -------------------------------------------------

    @classmethod
    def _wrap(cls, tree, nodes: dict, orthogonal: bool, arena=None) -> "HTensor":
        obj = cls.__new__(cls)
        obj.tree = tree
        obj.orthogonal = bool(orthogonal)
        obj._nodes = nodes
        obj._arena = arena
        obj._cstruct = None
        return obj

    @classmethod
    def empty(cls, tree: DimensionTree, sizes_by_node: dict, ranks: dict, orthogonal: bool = False,
              device=None) -> "HTensor":
        """Allocate an uninitialised tensor (one arena) with the given leaf sizes / ranks."""
        dev = _device(device)
        shapes = [node_shape(tree, t, sizes_by_node, ranks) for t in range(len(tree.nodes))]
        total = sum(math.prod(s) for s in shapes)
        arena = torch.empty(total, dtype=F64, device=dev)
        if _POISON:  # debugging aid (HT_POISON_WORKSPACE=1): outputs start as NaN
            arena.fill_(float("nan"))
        return cls._wrap(tree, _arena_views(arena, shapes), orthogonal, arena)

    @classmethod
    def from_numpy(cls, tree, leaves, transfer, root_matrix, orthogonal=False, device=None) -> "HTensor":
        return cls(tree, leaves, transfer, root_matrix, orthogonal, device=device)

    # -- reference attributes --------------------------------------------------

    @property
    def leaves(self) -> dict:
        return {n.index: self._nodes[n.index] for n in self.tree.nodes if n.is_leaf}

    @property
    def transfer(self) -> dict:
        return {n.index: self._nodes[n.index] for n in self.tree.inner_nodes}

    @property
    def root_matrix(self) -> torch.Tensor:
        return self._nodes[0]

    def node_array(self, t: int) -> torch.Tensor:
        return self._nodes[t]

    def _shape(self, t: int) -> tuple:
        n = self._nodes
        return n.shapes[t] if isinstance(n, _ArenaViews) else tuple(n[t].shape)

    def _rank_list(self) -> list:
        """Ranks by node id, computed once (node shapes never change: HTensors are
        immutable by convention, format.py:19)."""
        rl = self.__dict__.get("_ranks_cached")
        if rl is None:
            rl = []
            for t in range(len(self.tree.nodes)):
                node = self.tree.node(t)
                if node.is_root:
                    rl.append(1)
                elif node.is_leaf:
                    rl.append(int(self._shape(t)[1]))
                else:
                    rl.append(int(self._shape(t)[0]))
            self._ranks_cached = rl
        return rl

    def rank(self, node_id: int) -> int:
        return self._rank_list()[node_id]

    @property
    def ranks(self) -> dict:
        return {n.index: self.rank(n.index) for n in self.tree.non_root}

    @property
    def max_rank(self) -> int:
        return max(self.ranks.values())

    @property
    def shape(self) -> tuple:
        sh = self.__dict__.get("_shape_cached")
        if sh is None:
            sh = tuple(int(self._shape(self.tree.leaf_for_dim(mu).index)[0]) for mu in range(1, self.tree.d + 1))
            self._shape_cached = sh
        return sh

    @property
    def device(self) -> torch.device:
        if self._arena is not None:
            return self._arena.device
        return self._nodes[0].device

    def validate(self) -> None:
        """format.py:101-119: rank chain along every edge."""
        tree = self.tree
        for node in tree.nodes:
            if node.is_leaf:
                if node.index not in self._nodes:
                    raise ValueError(f"missing leaf frame for node {node.index}")
                if self._nodes[node.index].dim() != 2:
                    raise ValueError(f"leaf {node.index} must be a matrix")
                continue
            s1, s2 = node.sons
            k1, k2 = self.rank(s1), self.rank(s2)
            arr = self._nodes.get(node.index)
            if arr is None:
                raise ValueError(f"missing array for node {node.index}")
            got = tuple(arr.shape) if node.is_root else tuple(arr.shape[1:])
            if got != (k1, k2):
                raise ValueError(f"rank chain broken at node {node.index}: transfer sees {got}, "
                                 f"sons have ranks ({k1}, {k2})")

    def copy(self) -> "HTensor":
        nodes = {t: v.clone() for t, v in self._nodes.items()}
        return HTensor._wrap(self.tree, nodes, self.orthogonal)

    def storage_size(self) -> int:
        return int(sum(v.numel() for v in self._nodes.values()))

    # -- host transfer ---------------------------------------------------------

    def to_numpy(self):
        """(leaves, transfer, root_matrix) as numpy dicts -- one D2H copy when arena-backed.
        A host synchronisation point: errors left by queued truncations are raised here."""
        if self.device.type == "cuda":
            with torch.cuda.device(self.device):
                _lib.check_status()
        if isinstance(self._nodes, _ArenaViews):
            host = self._arena.cpu().numpy()
            out = {}
            for t, (o, s) in enumerate(zip(self._nodes.offsets, self._nodes.shapes)):
                out[t] = host[o:o + math.prod(s)].reshape(s)
        elif self._arena is not None:
            host = self._arena.cpu().numpy()
            out, off = {}, 0
            for t in range(len(self.tree.nodes)):
                a = self._nodes[t]
                out[t] = host[off:off + a.numel()].reshape(tuple(a.shape))
                off += a.numel()
        else:
            out = {t: v.cpu().numpy() for t, v in self._nodes.items()}
        leaves = {n.index: out[n.index] for n in self.tree.nodes if n.is_leaf}
        transfer = {n.index: out[n.index] for n in self.tree.inner_nodes}
        return leaves, transfer, out[0]

    # -- pinned host arenas (end-to-end path) ----------------------------------

    @classmethod
    def from_host_arena(cls, tree: DimensionTree, sizes_by_node: dict, ranks: dict, host: torch.Tensor,
                        orthogonal: bool = False, device=None) -> "HTensor":
        """Upload a flat host buffer (node arrays in BFS id order, C-order; ideally
        pinned) with ONE asynchronous host->device copy."""
        out = cls.empty(tree, sizes_by_node, ranks, orthogonal, device)
        if host.numel() != out._arena.numel():
            raise ValueError("host arena size does not match the tensor shapes")
        out._arena.copy_(host, non_blocking=True)
        return out

    def load_host_arena(self, host: torch.Tensor) -> "HTensor":
        """Overwrite this tensor's values from a flat host buffer (one async H2D copy on
        the current stream; shapes must match).  Lets pipelines reuse device buffers."""
        if self._arena is None or host.numel() != self._arena.numel():
            raise ValueError("host arena size does not match the tensor shapes")
        self._arena.copy_(host, non_blocking=True)
        return self

    def to_host_arena(self, host: torch.Tensor | None = None) -> torch.Tensor:
        """Copy the whole tensor into a flat (pinned) host buffer with one D2H copy."""
        if self._arena is None:
            flat = torch.cat([self._nodes[t].reshape(-1) for t in range(len(self.tree.nodes))])
        else:
            flat = self._arena
        if host is None:
            host = torch.empty(flat.numel(), dtype=F64, pin_memory=True)
        host.copy_(flat, non_blocking=True)
        return host

    def arena_numel(self) -> int:
        """Number of float64 values of the tensor (all node arrays)."""
        if self._arena is not None:
            return int(self._arena.numel())
        return sum(int(self._nodes[t].numel()) for t in range(len(self.tree.nodes)))

    def host_layout(self):
        """(sizes_by_node, ranks) needed to rebuild this tensor from a host arena."""
        return ({leaf.index: int(self._shape(leaf.index)[0]) for leaf in self.tree.leaves},
                {t: self.rank(t) for t in range(1, len(self.tree.nodes))})

    # -- C ABI -----------------------------------------------------------------

    def _check_resident(self) -> torch.device:
        """Every node array must be a float64 CUDA tensor on one device (the C ABI takes
        raw device pointers); host-resident tensors are rejected instead of faulting."""
        if isinstance(self._nodes, _ArenaViews):
            arrays = [self._arena]
        else:
            arrays = [self._nodes[t] for t in range(len(self.tree.nodes))]
        dev = arrays[0].device
        for a in arrays:
            if not a.is_cuda or a.dtype != F64 or a.device != dev:
                raise ValueError(f"HTensor node arrays must be float64 CUDA tensors on one device; got "
                                 f"{a.dtype} on {a.device} (host-resident tensors cannot be passed to the kernels)")
            if not a.is_contiguous():
                raise ValueError("HTensor node arrays must be contiguous (C-order)")
        return dev

    def _c(self) -> _lib.CTensor:
        if self._cstruct is None:
            dev = self._check_resident()
            tree = self.tree
            n = _lib.i64_array(self.shape)
            ranks = _lib.i64_array([1] + [self.rank(t) for t in range(1, len(tree.nodes))])
            if isinstance(self._nodes, _ArenaViews):
                ptrs = _lib.ptr_array(self._nodes.pointers())
            else:
                ptrs = _lib.ptr_array([self._nodes[t].data_ptr() for t in range(len(tree.nodes))])
            cs = _lib.CTensor(tree.d, ctypes.cast(n, ctypes.POINTER(ctypes.c_int64)),
                              ctypes.cast(ranks, ctypes.POINTER(ctypes.c_int64)),
                              ctypes.cast(ptrs, ctypes.POINTER(ctypes.c_void_p)), int(self.orthogonal))
            self._cstruct = (cs, n, ranks, ptrs, dev.index)
        if self._cstruct[4] != torch.cuda.current_device():
            raise ValueError(f"HTensor lives on cuda:{self._cstruct[4]} but the current device is "
                             f"cuda:{torch.cuda.current_device()}; call under torch.cuda.device(...)")
        cs = self._cstruct[0]
        cs.orthogonal = int(self.orthogonal)
        return cs

    def _c_trunc(self) -> _lib.CTensor:
        """The C view the truncation entry points take (``AppliedHTensor`` overrides it
        with its Kronecker form)."""
        return self._c()

    def __repr__(self) -> str:
        return (f"HTensor(d={self.tree.d}, shape={self.shape}, max_rank={self.max_rank}, "
                f"orthogonal={self.orthogonal}, device={self.device})")


def _upload(tree: DimensionTree, arrays: dict, dev: torch.device):
    """Pack node arrays (numpy / torch) into one pinned buffer and copy it to HBM."""
    host = {}
    for t, a in arrays.items():
        if isinstance(a, torch.Tensor):
            a = a.detach().to("cpu", F64).numpy()
        host[t] = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    total = sum(a.size for a in host.values())
    if dev.type != "cuda":  # host-resident container (I/O, CPU tests); no kernel runs on it
        arena = torch.from_numpy(np.concatenate([host[t].ravel() for t in range(len(tree.nodes))]
                                                if host else np.zeros(0))).to(dev)
        nodes, off = {}, 0
        for t in range(len(tree.nodes)):
            nodes[t] = arena[off:off + host[t].size].view(host[t].shape)
            off += host[t].size
        return nodes, arena
    pinned = torch.empty(total, dtype=F64, pin_memory=True)
    buf = pinned.numpy()
    off = 0
    layout = {}
    for t in range(len(tree.nodes)):
        if t not in host:
            raise ValueError(f"missing array for node {t}")
        a = host[t]
        buf[off:off + a.size] = a.ravel()
        layout[t] = (off, a.shape)
        off += a.size
    arena = torch.empty(total, dtype=F64, device=dev)
    arena.copy_(pinned, non_blocking=True)
    nodes = {t: arena[o:o + math.prod(s)].view(s) for t, (o, s) in layout.items()}
    # keep the pinned buffer alive until the asynchronous copy has executed
    _PINNED_KEEPALIVE.append((torch.cuda.current_stream(dev).record_event(), pinned))
    _trim_keepalive()
    return nodes, arena


_PINNED_KEEPALIVE: list = []


def _trim_keepalive():
    while _PINNED_KEEPALIVE and _PINNED_KEEPALIVE[0][0].query():
        _PINNED_KEEPALIVE.pop(0)


# ---------------------------------------------------------------------------
# operators (reference format.py:135-250)
# ---------------------------------------------------------------------------


class GeneralizedMatrix:
    """A linear map R^n -> R^m stored dense, diagonal or CSR (format.py:135-180)."""

    def __init__(self, kind: str, data):
        if kind not in ("dense", "diagonal", "csr"):
            raise ValueError(f"unknown kind {kind}")
        self.kind = kind
        self.data = data
        self._dev = None

    @staticmethod
    def dense(mat) -> "GeneralizedMatrix":
        return GeneralizedMatrix("dense", np.asarray(mat, dtype=np.float64))

    @staticmethod
    def diagonal(vec) -> "GeneralizedMatrix":
        return GeneralizedMatrix("diagonal", np.asarray(vec, dtype=np.float64).ravel())

    @staticmethod
    def csr(mat) -> "GeneralizedMatrix":
        import scipy.sparse as sp

        m = sp.csr_matrix(mat, dtype=np.float64)
        m.sort_indices()
        return GeneralizedMatrix("csr", m)

    @property
    def shape(self) -> tuple:
        if self.kind == "diagonal":
            n = self.data.shape[0]
            return (n, n)
        return tuple(self.data.shape)

    def to_dense(self) -> np.ndarray:
        if self.kind == "diagonal":
            return np.diag(self.data)
        if self.kind == "csr":
            return self.data.toarray()
        return np.asarray(self.data)

    def device_struct(self, dev) -> _lib.CGmat:
        """Upload once; returns the ht_gmat descriptor (keeps the device arrays alive)."""
        if self._dev is None:
            rows, cols = self.shape
            if self.kind == "dense":
                vals = torch.as_tensor(np.ascontiguousarray(self.data), dtype=F64).to(dev)
                self._dev = (_lib.CGmat(0, rows, cols, rows * cols, vals.data_ptr(), None, None), vals)
            elif self.kind == "diagonal":
                vals = torch.as_tensor(self.data, dtype=F64).to(dev)
                self._dev = (_lib.CGmat(1, rows, cols, rows, vals.data_ptr(), None, None), vals)
            else:
                vals = torch.as_tensor(self.data.data, dtype=F64).to(dev)
                ip = torch.as_tensor(self.data.indptr.astype(np.int32)).to(dev)
                ix = torch.as_tensor(self.data.indices.astype(np.int32)).to(dev)
                self._dev = (_lib.CGmat(2, rows, cols, int(self.data.nnz), vals.data_ptr(), ip.data_ptr(),
                                        ix.data_ptr()), vals, ip, ix)
        return self._dev[0]


class HTOperator:
    """Tree-format linear operator (format.py:183-250): leaf columns are
    :class:`GeneralizedMatrix` lists; transfer tensors / root live on the GPU."""

    def __init__(self, tree: DimensionTree, leaves: dict, transfer: dict, root_matrix, *, device=None):
        self.tree = tree
        self.leaves = {int(t): list(cols) for t, cols in leaves.items()}
        dev = _device(device)
        self._dev = dev
        self.transfer = {int(t): torch.as_tensor(np.asarray(b, dtype=np.float64) if not isinstance(b, torch.Tensor)
                                                 else b, dtype=F64).to(dev).contiguous()
                         for t, b in transfer.items()}
        self.root_matrix = torch.as_tensor(np.asarray(root_matrix, dtype=np.float64)
                                           if not isinstance(root_matrix, torch.Tensor) else root_matrix,
                                           dtype=F64).to(dev).contiguous()
        self._cstruct = None
        self.validate()

    def rank(self, node_id: int) -> int:
        node = self.tree.node(node_id)
        if node.is_root:
            return 1
        if node.is_leaf:
            return len(self.leaves[node_id])
        return int(self.transfer[node_id].shape[0])

    @property
    def ranks(self) -> dict:
        return {n.index: self.rank(n.index) for n in self.tree.non_root}

    def leaf_shape(self, node_id: int) -> tuple:
        return self.leaves[node_id][0].shape

    @property
    def row_sizes(self) -> tuple:
        return tuple(self.leaf_shape(self.tree.leaf_for_dim(mu).index)[0] for mu in range(1, self.tree.d + 1))

    @property
    def col_sizes(self) -> tuple:
        return tuple(self.leaf_shape(self.tree.leaf_for_dim(mu).index)[1] for mu in range(1, self.tree.d + 1))

    def validate(self) -> None:
        tree = self.tree
        for node in tree.nodes:
            if node.is_leaf:
                cols = self.leaves.get(node.index)
                if not cols:
                    raise ValueError(f"missing leaf columns for node {node.index}")
                if len({c.shape for c in cols}) != 1:
                    raise ValueError(f"leaf {node.index} mixes column shapes")
                continue
            s1, s2 = node.sons
            got = tuple(self.root_matrix.shape) if node.is_root else tuple(self.transfer[node.index].shape[1:])
            if got != (self.rank(s1), self.rank(s2)):
                raise ValueError(f"rank chain broken at operator node {node.index}")

    def _c(self) -> _lib.COperator:
        if self._cstruct is None:
            tree = self.tree
            nn = len(tree.nodes)
            ranks = _lib.i64_array([1] + [self.rank(t) for t in range(1, nn)])
            col_arrays = []
            leaf_ptrs = (ctypes.POINTER(_lib.CGmat) * nn)()
            for t in range(nn):
                if tree.node(t).is_leaf:
                    arr = (_lib.CGmat * len(self.leaves[t]))(*[g.device_struct(self._dev) for g in self.leaves[t]])
                    col_arrays.append(arr)
                    leaf_ptrs[t] = ctypes.cast(arr, ctypes.POINTER(_lib.CGmat))
            node_ptrs = _lib.ptr_array([self.root_matrix.data_ptr() if t == 0 else
                                        (self.transfer[t].data_ptr() if t in self.transfer else 0)
                                        for t in range(nn)])
            cs = _lib.COperator(tree.d, ctypes.cast(ranks, ctypes.POINTER(ctypes.c_int64)),
                                ctypes.cast(leaf_ptrs, ctypes.POINTER(ctypes.POINTER(_lib.CGmat))),
                                ctypes.cast(node_ptrs, ctypes.POINTER(ctypes.c_void_p)))
            self._cstruct = (cs, ranks, col_arrays, leaf_ptrs, node_ptrs)
        return self._cstruct[0]

    def __repr__(self) -> str:
        return f"HTOperator(d={self.tree.d}, rows={self.row_sizes}, cols={self.col_sizes})"


# ---------------------------------------------------------------------------
# constructors (reference format.py:262-336)
# ---------------------------------------------------------------------------


def _uniform_ranks(tree, k) -> dict:
    if isinstance(k, dict):
        return {n.index: int(k[n.index]) for n in tree.non_root}
    return {n.index: int(k) for n in tree.non_root}


def _leaf_sizes(tree, n) -> dict:
    if np.isscalar(n):
        return {leaf.index: int(n) for leaf in tree.leaves}
    sizes = list(n)
    if len(sizes) != tree.d:
        raise ValueError(f"need {tree.d} leaf sizes, got {len(sizes)}")
    return {tree.leaf_for_dim(mu).index: int(sizes[mu - 1]) for mu in range(1, tree.d + 1)}


def _draw_factors(tree: DimensionTree, n, k, draw, leaf_scale=None, core_scale=None):
    """Factors in the reference's node order (format.py:271-301), one ``draw(shape)``
    per node; optional exact power-of-two rescales of leaves / transfer tensors."""
    ranks = _uniform_ranks(tree, k)
    sizes = _leaf_sizes(tree, n)
    leaves, transfer, root = {}, {}, None
    for node in tree.nodes:
        if node.is_leaf:
            nm, km = sizes[node.index], ranks[node.index]
            if km > nm:
                raise ValueError(f"leaf rank {km} exceeds size {nm} at node {node.index}")
            leaves[node.index] = draw((nm, km))
            if leaf_scale:
                leaves[node.index] *= leaf_scale(nm)
            continue
        s1, s2 = node.sons
        k1, k2 = ranks[s1], ranks[s2]
        if node.is_root:
            root = draw((k1, k2))
            if core_scale:
                root *= core_scale(max(k1, k2))
            continue
        kt = ranks[node.index]
        if kt > k1 * k2:
            raise ValueError(f"rank {kt} at node {node.index} exceeds structural bound {k1 * k2}")
        transfer[node.index] = draw((kt, k1, k2))
        if core_scale:
            transfer[node.index] *= core_scale(kt)
    return leaves, transfer, root


def random_htensor(tree: DimensionTree, n, k, seed: int, device=None) -> HTensor:
    """Uniform [-1, 1] entries from PCG64(seed) in the reference's node order
    (format.py:271-301): the same seed gives the same tensor as the reference."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    leaves, transfer, root = _draw_factors(tree, n, k, lambda shp: rng.uniform(-1.0, 1.0, size=shp))
    return HTensor(tree, leaves, transfer, root, device=device)


def _pow2(x: float) -> float:
    return 2.0 ** -round(math.log2(x))


def gaussian_factors(tree: DimensionTree, n, k, seed: int, scaled: bool = True):
    """Host (numpy) factors of the benchmark tensors: N(0,1) from
    PCG64(seed) in the reference's node order; with ``scaled`` leaves x 2^-round(log2 sqrt n)
    and transfer/root tensors x 2^-round(log2 k) (exact, keeps large-d sums finite).
    Returns (leaves, transfer, root) dicts keyed by node id."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    return _draw_factors(tree, n, k, rng.standard_normal,
                         (lambda nm: _pow2(math.sqrt(nm))) if scaled else None,
                         _pow2 if scaled else None)


def gaussian_htensor(tree: DimensionTree, n, k, seed: int, scaled: bool = True, device=None) -> HTensor:
    leaves, transfer, root = gaussian_factors(tree, n, k, seed, scaled)
    return HTensor(tree, leaves, transfer, root, device=device)


def identity_htoperator(tree: DimensionTree, n) -> HTOperator:
    """Rank-1 identity operator (format.py:330-336)."""
    sizes = _leaf_sizes(tree, n)
    leaves = {leaf.index: [GeneralizedMatrix.diagonal(np.ones(sizes[leaf.index]))] for leaf in tree.leaves}
    transfer = {node.index: np.ones((1, 1, 1)) for node in tree.inner_nodes}
    return HTOperator(tree, leaves, transfer, np.ones((1, 1)))


def storage_size(tensor: HTensor) -> int:
    """format.py:459-464: sum n k + sum k_t k1 k2 + k1 k2."""
    return tensor.storage_size()


__all__ = ["HTensor", "HTOperator", "GeneralizedMatrix", "random_htensor", "gaussian_htensor", "gaussian_factors",
           "identity_htoperator",
           "storage_size", "build_balanced_tree", "DimensionTree"]


# ---------------------------------------------------------------------------
# HT01 binary interchange (reference format.py:467-553): little-endian; magic
# "HT01", u32 d, u64 reserved 0, d u64 leaf sizes in dimension order, 2d-1 u64
# ranks in BFS node order (root 1), then every node array in id order as f64 with
# the first index fastest (matrices column-major, transfer tensors mode 1 fastest).
# Host-side packing of one device->host copy of the tensor's arena; deserialize
# uploads the arrays as one arena.
# ---------------------------------------------------------------------------

HT01_MAGIC = b"HT01"


class ParseError(ValueError):
    """Malformed HT01 data; carries the byte offset of the first problem (format.py:37-42)."""

    def __init__(self, message: str, offset: int):
        super().__init__(f"{message} (byte offset {offset})")
        self.offset = offset


def serialized_size(tensor: HTensor) -> int:
    """Exact byte length of :func:`serialize`: 16-byte header, the two index tables,
    then 8 bytes per stored float."""
    d = tensor.tree.d
    return 16 + 8 * d + 8 * (2 * d - 1) + 8 * storage_size(tensor)


def serialize(tensor: HTensor) -> bytes:
    import struct

    tree = tensor.tree
    d = tree.d
    leaves, transfer, root = tensor.to_numpy()
    parts = [HT01_MAGIC, struct.pack("<IQ", d, 0)]
    parts.append(np.array([leaves[tree.leaf_for_dim(mu).index].shape[0] for mu in range(1, d + 1)],
                          dtype="<u8").tobytes())
    parts.append(np.array([1] + [tensor.rank(t) for t in range(1, len(tree.nodes))], dtype="<u8").tobytes())
    for node in tree.nodes:
        arr = root if node.is_root else (leaves[node.index] if node.is_leaf else transfer[node.index])
        parts.append(np.asarray(arr, dtype="<f8").ravel(order="F").tobytes())
    return b"".join(parts)


def deserialize(blob: bytes, device=None) -> HTensor:
    """Inverse of :func:`serialize` (raises :class:`ParseError` with the byte offset)."""
    import struct

    blob = bytes(blob)
    if len(blob) < 4 or blob[:4] != HT01_MAGIC:
        raise ParseError("bad magic", 0)
    if len(blob) < 16:
        raise ParseError("truncated header", len(blob))
    (d,) = struct.unpack_from("<I", blob, 4)
    if d < 2:
        raise ParseError(f"invalid dimension {d}", 4)
    tree = build_balanced_tree(d)
    off = 16
    nn = 2 * d - 1
    if len(blob) < off + 8 * (d + nn):
        raise ParseError("truncated index tables", len(blob))
    sizes = np.frombuffer(blob, dtype="<u8", count=d, offset=off).astype(np.int64)
    off += 8 * d
    ranks = np.frombuffer(blob, dtype="<u8", count=nn, offset=off).astype(np.int64)
    if ranks[0] != 1:
        raise ParseError(f"root rank must be 1, found {ranks[0]}", off)
    off += 8 * nn
    leaves, transfer, root = {}, {}, None
    for node in tree.nodes:
        t = node.index
        if node.is_root:
            shape = (int(ranks[node.sons[0]]), int(ranks[node.sons[1]]))
        elif node.is_leaf:
            shape = (int(sizes[node.dim - 1]), int(ranks[t]))
        else:
            shape = (int(ranks[t]), int(ranks[node.sons[0]]), int(ranks[node.sons[1]]))
        count = math.prod(shape)
        if len(blob) < off + 8 * count:
            raise ParseError("truncated payload", len(blob))
        arr = np.frombuffer(blob, dtype="<f8", count=count, offset=off).reshape(shape, order="F")
        off += 8 * count
        if node.is_root:
            root = np.ascontiguousarray(arr)
        elif node.is_leaf:
            leaves[t] = np.ascontiguousarray(arr)
        else:
            transfer[t] = np.ascontiguousarray(arr)
    if off != len(blob):
        raise ParseError(f"{len(blob) - off} trailing bytes", off)
    return HTensor(tree, leaves, transfer, root, device=device)
