"""Tree-parallel (sharded) HT truncation across GPUs -- the paper's design.

arXiv 1708.03340 assigns one compute node per tree node and passes R factors up,
reduced Gramians down and truncated bases up the dimension tree (reference
dist.py:239-333, message waves RFACTOR_UP / BHAT_DOWN / QTRUNC_UP).  On B200
the 2d-1 "workers" collapse into level-batched kernels on one GPU, and the
tree is split across G = 2, 4 or 8 GPUs: GPU g owns the subtree under the g-th
node of level log2(G); GPU 0 additionally owns the G-1 nodes above (root
included).  Per truncation there are three waves of G-1 point-to-point
messages (K x K R factors up, K x K Gramians down, K x K eigenvector blocks +
ranks up), carried by ``torch.distributed`` (NCCL over NVLink, or gloo in the
CPU tests).  Everything else is local.

The protocol (:func:`sharded_truncate`) is written against a small engine
interface so the same code drives the GPU (``GpuShardEngine``: the C-ABI
``ht_truncate_sharded``/``ht_truncate_slot``) and the CPU test engine.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .arith import TruncationControl, _ws
from .format import F64, HTensor, node_shape
from .tree import DimensionTree

ORTH, GRAM, EIG, PROJECT = 0, 1, 2, 3
SLOT_R, SLOT_G, SLOT_EV, SLOT_LAM, SLOT_RANKS, SLOT_ORTH = 0, 1, 2, 3, 4, 5


# ---------------------------------------------------------------------------
# shard map
# ---------------------------------------------------------------------------


@dataclass
class ShardMap:
    """Subtree-per-rank placement.

    ``roots[g]`` is the node whose subtree rank g owns; ``top`` are the nodes
    above level log2(world) (owned by rank 0, root included).
    """

    tree: DimensionTree
    world: int
    roots: list = field(default_factory=list)
    top: list = field(default_factory=list)
    owner: list = field(default_factory=list)

    @classmethod
    def build(cls, tree: DimensionTree, world: int) -> "ShardMap":
        if world < 1 or world & (world - 1):
            raise ValueError("world size must be a power of two")
        L = int(round(math.log2(world)))
        levels = tree.levels_top_down()
        if L > tree.depth or len(levels[L]) != world:
            raise ValueError(f"tree of d={tree.d} has {len(levels[L]) if L <= tree.depth else 0} nodes on level "
                             f"{L}; cannot shard over {world} ranks (use replicas)")
        sm = cls(tree, world)
        sm.roots = list(levels[L])
        sm.top = [t for lev in levels[:L] for t in lev]
        sm.owner = [0] * len(tree.nodes)
        for g, r in enumerate(sm.roots):
            for t in tree.subtree(r):
                sm.owner[t] = g
        return sm

    def subtree(self, g: int) -> list:
        return self.tree.subtree(self.roots[g])

    def owned(self, g: int) -> list:
        return sorted(self.subtree(g) + (self.top if g == 0 else []))

    def mask(self, nodes) -> np.ndarray:
        m = np.zeros(len(self.tree.nodes), dtype=np.uint8)
        m[list(nodes)] = 1
        return m


# ---------------------------------------------------------------------------
# sharded tensor: metadata for every node, storage only for owned nodes
# ---------------------------------------------------------------------------


class ShardedHTensor:
    """One rank's share of an HT tensor: full shape metadata, arrays of owned nodes only."""

    def __init__(self, tree: DimensionTree, sizes: dict, ranks: dict, arrays: dict, orthogonal: bool = False):
        self.tree = tree
        self.sizes = {int(t): int(v) for t, v in sizes.items()}   # leaf node id -> n
        self.ranks = {int(t): int(v) for t, v in ranks.items()}   # non-root node id -> k
        self.arrays = arrays                                     # owned node id -> torch tensor
        self.orthogonal = orthogonal
        dev = next(iter(arrays.values())).device if arrays else torch.device("cpu")
        self._dummy = torch.zeros(1, dtype=F64, device=dev)
        self._cs = None

    @classmethod
    def from_host(cls, tree: DimensionTree, leaves: dict, transfer: dict, root, nodes, device=None,
                  pin: bool = False) -> "ShardedHTensor":
        """Upload only the owned nodes' host arrays (numpy or torch) to this rank's GPU."""
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        sizes = {t: int(a.shape[0]) for t, a in leaves.items()}
        ranks = {t: int(a.shape[1]) for t, a in leaves.items()}
        ranks.update({t: int(a.shape[0]) for t, a in transfer.items()})
        host = dict(leaves)
        host.update(transfer)
        host[0] = root
        arrays = {}
        for t in sorted(nodes):
            h = torch.as_tensor(np.ascontiguousarray(host[t]), dtype=F64)
            arrays[t] = h.to(dev, non_blocking=False)
        return cls(tree, sizes, ranks, arrays, False)

    @classmethod
    def from_htensor(cls, x: HTensor, nodes) -> "ShardedHTensor":
        sizes, ranks = x.host_layout()
        return cls(x.tree, sizes, ranks, {t: x.node_array(t) for t in nodes}, x.orthogonal)

    def shape(self, t: int) -> tuple:
        return node_shape(self.tree, t, self.sizes, self.ranks)

    @property
    def device(self) -> torch.device:
        return self._dummy.device

    def nbytes(self) -> int:
        return sum(a.numel() * 8 for a in self.arrays.values())

    def orth_ranks(self) -> dict:
        """Ranks after orthogonalisation (shape-only; arith.py:280-297 rank shrink)."""
        nn = len(self.tree.nodes)
        if self.orthogonal:
            return dict(self.ranks)
        rbuf = (ctypes.c_int64 * nn)()
        _lib.check(_lib.load().ht_orth_ranks(self._c(), rbuf), "orth ranks")
        return {t: int(rbuf[t]) for t in range(1, nn)}

    def _c(self):
        if self._cs is None:
            tree = self.tree
            nn = len(tree.nodes)
            n = _lib.i64_array([self.sizes[tree.leaf_for_dim(mu).index] for mu in range(1, tree.d + 1)])
            r = _lib.i64_array([1] + [self.ranks[t] for t in range(1, nn)])
            ptrs = _lib.ptr_array([(self.arrays[t] if t in self.arrays else self._dummy).data_ptr()
                                   for t in range(nn)])
            cs = _lib.CTensor(tree.d, ctypes.cast(n, ctypes.POINTER(ctypes.c_int64)),
                              ctypes.cast(r, ctypes.POINTER(ctypes.c_int64)),
                              ctypes.cast(ptrs, ctypes.POINTER(ctypes.c_void_p)), int(self.orthogonal))
            self._cs = (cs, n, r, ptrs)
        return self._cs[0]


def sharded_add(a: ShardedHTensor, c: ShardedHTensor, alpha_c: float = 1.0) -> ShardedHTensor:
    """Owned-node HT add (arith.py:160-193); communication-free (reference dist.py add
    protocol sends no messages).  Nodes owned here must be the same in a and c."""
    if set(a.arrays) != set(c.arrays):
        raise ValueError("sharded add: operands own different nodes")
    lib = _lib.load()
    ranks = {t: a.ranks[t] + c.ranks[t] for t in a.ranks}
    arrays = {t: torch.empty(node_shape(a.tree, t, a.sizes, ranks), dtype=F64, device=a.device)
              for t in a.arrays}
    out = ShardedHTensor(a.tree, a.sizes, ranks, arrays, False)
    mask = np.zeros(len(a.tree.nodes), dtype=np.uint8)
    mask[list(a.arrays)] = 1
    _lib.check(lib.ht_add_sharded(a._c(), c._c(), float(alpha_c), mask.ctypes.data_as(ctypes.c_void_p), out._c(),
                                  _lib.stream_handle()), "sharded add")
    return out


# ---------------------------------------------------------------------------
# GPU engine: the C-ABI sharded phases on one device
# ---------------------------------------------------------------------------


def _mask(nn: int, nodes) -> np.ndarray:
    m = np.zeros(nn, dtype=np.uint8)
    m[list(nodes)] = 1
    return np.ascontiguousarray(m)


def _ptr(m: np.ndarray):
    return m.ctypes.data_as(ctypes.c_void_p)


def shard_workspace_bytes(tree: DimensionTree, sizes: dict, ranks: dict, owned, orthogonal: bool = False) -> int:
    """Truncate workspace of one shard (host-only query, no device needed): the plan
    holds the owned nodes and their sons' message slots only."""
    nn = len(tree.nodes)
    n = _lib.i64_array([sizes[tree.leaf_for_dim(mu).index] for mu in range(1, tree.d + 1)])
    r = _lib.i64_array([1] + [ranks[t] for t in range(1, nn)])
    cs = _lib.CTensor(tree.d, ctypes.cast(n, ctypes.POINTER(ctypes.c_int64)),
                      ctypes.cast(r, ctypes.POINTER(ctypes.c_int64)), None, int(orthogonal))
    m = _mask(nn, owned) if owned is not None else None
    nbytes = ctypes.c_size_t(0)
    _lib.check(_lib.load().ht_truncate_workspace_size_sharded(ctypes.byref(cs), _ptr(m) if m is not None else None,
                                                              ctypes.byref(nbytes)), "shard workspace size")
    return int(nbytes.value)


class GpuShardEngine:
    """One rank's truncation state on its GPU: the C-ABI phases over a workspace
    planned for the nodes this rank owns (plus the message slots of their sons)."""

    def __init__(self, x: ShardedHTensor, ctl: TruncationControl, owned=None):
        self.lib = _lib.load()
        self.x = x
        self.ctl = ctl
        nn = len(x.tree.nodes)
        self.cctl, self._keep = ctl._c(nn)
        self.owned = _mask(nn, sorted(owned if owned is not None else x.arrays))
        nbytes = ctypes.c_size_t(0)
        _lib.check(self.lib.ht_truncate_workspace_size_sharded(x._c(), _ptr(self.owned), ctypes.byref(nbytes)),
                   "sharded truncate")
        self.ws = _ws(nbytes.value, x._dummy.device)
        self._slots = {}

    def phase(self, ph: int, nodes, out: ShardedHTensor | None = None):
        m = _mask(len(self.x.tree.nodes), nodes)
        _lib.check(self.lib.ht_truncate_sharded(self.x._c(), ctypes.byref(self.cctl), self.ws.data_ptr(),
                                                self.ws.numel(), ph, _ptr(m), _ptr(self.owned),
                                                out._c() if out is not None else None, _lib.stream_handle()),
                   f"sharded truncate phase {ph}")

    def slot(self, kind: int, node: int) -> torch.Tensor:
        key = (kind, node)
        if key in self._slots:
            return self._slots[key]
        ptr = ctypes.c_void_p(0)
        cnt = ctypes.c_int64(0)
        _lib.check(self.lib.ht_truncate_slot(self.x._c(), ctypes.c_void_p(self.ws.data_ptr()), _ptr(self.owned),
                                             kind, node, ctypes.byref(ptr), ctypes.byref(cnt)), "workspace slot")
        off = ptr.value - self.ws.data_ptr()
        if kind == SLOT_RANKS:
            v = self.ws[off:off + 4 * cnt.value].view(torch.int32)
        else:
            v = self.ws[off:off + 8 * cnt.value].view(F64)
        self._slots[key] = v
        return v

    def ranks(self) -> np.ndarray:
        torch.cuda.current_stream().synchronize()
        return self.slot(SLOT_RANKS, 0).cpu().numpy()

    def orth_rank(self, t: int) -> int:
        return int(self.slot(SLOT_LAM, t).numel())

    def allocate_out(self, ranks: dict, nodes) -> ShardedHTensor:
        x = self.x
        arrays = {}
        for t in nodes:
            shape = node_shape(x.tree, t, x.sizes, ranks)
            arrays[t] = torch.empty(shape, dtype=F64, device=x._dummy.device)
        return ShardedHTensor(x.tree, x.sizes, ranks, arrays, False)


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------


class TorchComm:
    """Point-to-point over torch.distributed (NCCL on GPUs, gloo on CPU).

    A message wave is one ``exchange``: every send and receive of the wave is posted
    at once through ``batch_isend_irecv`` (one NCCL group: the G-1 transfers of a wave
    overlap instead of running back to back).  On NCCL the waits only order the
    current stream (no host blocking); gloo waits on the host."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def _global(self, r: int) -> int:
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def exchange(self, sends=(), recvs=()):
        d = self.dist
        ops = [d.P2POp(d.isend, t.contiguous(), self._global(p), self.group) for t, p in sends]
        bufs = []
        for t, p in recvs:
            b = t if t.is_contiguous() else torch.empty_like(t, memory_format=torch.contiguous_format)
            bufs.append((t, b))
            ops.append(d.P2POp(d.irecv, b, self._global(p), self.group))
        if ops:
            for w in d.batch_isend_irecv(ops):
                w.wait()
        for t, b in bufs:
            if b is not t:
                t.copy_(b)

    def send(self, t: torch.Tensor, dst: int):
        self.exchange(sends=[(t, dst)])

    def recv_into(self, t: torch.Tensor, src: int):
        self.exchange(recvs=[(t, src)])

    def broadcast(self, t: torch.Tensor, src: int = 0):
        self.dist.broadcast(t, self._global(src), group=self.group)

    def all_gather(self, t: torch.Tensor) -> list:
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return out


# ---------------------------------------------------------------------------
# the protocol (engine- and transport-agnostic)
# ---------------------------------------------------------------------------


def static_ranks(tree: DimensionTree, orth_ranks: dict, ctl: TruncationControl):
    """Kept ranks when they follow from the shapes (no eps): min(cap, k'), >= 1."""
    if ctl.eps is not None:
        return None
    out = {}
    for t in range(1, len(tree.nodes)):
        cap = ctl.cap_for(t)
        out[t] = max(1, min(orth_ranks[t], cap if cap is not None else orth_ranks[t]))
    return out


def sharded_truncate(engine, comm, smap: ShardMap, ctl: TruncationControl, orth_ranks: dict):
    """One truncation (arith.py:325-352) with the tree split over comm.world ranks.

    Returns this rank's ShardedHTensor of the truncated tensor (owned nodes), with
    the kept rank of EVERY node in its metadata.  Three message waves (reference
    dist.py:239-333: RFACTOR_UP / BHAT_DOWN / QTRUNC_UP): R factors of the shard roots
    up to rank 0, their reduced Gramians down, their eigenvector blocks (and, with an
    accuracy control, kept ranks) up.  Each wave is one batched exchange."""
    r, G = comm.rank, comm.world
    tree = smap.tree
    nn = len(tree.nodes)
    sub = smap.subtree(r)
    others = range(1, G)
    # wave 1: bottom-up orthogonalisation, R of the shard root goes up
    engine.phase(ORTH, sub)
    if r != 0:
        comm.exchange(sends=[(engine.slot(SLOT_R, smap.roots[r]), 0)])
    else:
        comm.exchange(recvs=[(engine.slot(SLOT_R, smap.roots[g]), g) for g in others])
        if smap.top:
            engine.phase(ORTH, smap.top)
            engine.phase(GRAM, smap.top)
    # wave 2: reduced Gramians of the shard roots go down
    if r != 0:
        comm.exchange(recvs=[(engine.slot(SLOT_G, smap.roots[r]), 0)])
    else:
        comm.exchange(sends=[(engine.slot(SLOT_G, smap.roots[g]), g) for g in others])
    inner_sub = [t for t in sub if not tree.node(t).is_leaf]
    engine.phase(GRAM, inner_sub)
    owned = smap.owned(r)
    engine.phase(EIG, [t for t in owned if t != 0])
    # wave 3: eigenvector blocks of the shard roots go up (the kept ranks follow from the
    # shapes under a fixed-rank control; with eps they are chosen on the device)
    ranks = static_ranks(tree, orth_ranks, ctl)
    if r != 0:
        comm.exchange(sends=[(engine.slot(SLOT_EV, smap.roots[r]), 0)])
    else:
        comm.exchange(recvs=[(engine.slot(SLOT_EV, smap.roots[g]), g) for g in others])
    if ranks is None:
        # every rank learns every kept rank (the next operation plans with them)
        local = engine.ranks()
        mine = torch.zeros(nn, dtype=torch.float64)
        for t in owned:
            if t != 0:
                mine[t] = float(local[t])
        dev = engine.slot(SLOT_EV, next(t for t in owned if t != 0)).device
        parts = comm.all_gather(mine.to(dev)) if G > 1 else [mine]
        allr = torch.stack([p.cpu() for p in parts]).sum(0)
        ranks = {t: int(allr[t]) for t in range(1, nn)}
    out = engine.allocate_out(ranks, owned)
    engine.phase(PROJECT, owned, out)
    return out


def sharded_inner_product(engine, comm, smap: ShardMap) -> float:
    """<A, C> (arith.py:246-265) with the tree split over comm.world ranks: every rank
    runs the Phi recursion of its subtree, the shard roots' Phi go up in one wave
    (reference dist.py:239-254 GRAM_UP, 516-524), rank 0 finishes the top levels and the
    root, and the value is broadcast so every rank returns it."""
    r, G = comm.rank, comm.world
    engine.phase(smap.subtree(r))
    if r != 0:
        comm.exchange(sends=[(engine.slot(smap.roots[r]), 0)])
    else:
        comm.exchange(recvs=[(engine.slot(smap.roots[g]), g) for g in range(1, G)])
        if smap.top:
            engine.phase(smap.top)
    res = engine.result()
    if G > 1:
        comm.broadcast(res, 0)
    return float(res.item())


class GpuInnerEngine:
    """<A, C> state of one rank: Phi slots of every node, the C-ABI sharded recursion."""

    def __init__(self, a: ShardedHTensor, c: ShardedHTensor):
        self.lib = _lib.load()
        self.a, self.c = a, c
        nbytes = ctypes.c_size_t(0)
        _lib.check(self.lib.ht_inner_product_workspace_size(a._c(), c._c(), ctypes.byref(nbytes)), "inner product")
        self.ws = _ws(nbytes.value, a.device)
        self.res = torch.zeros(1, dtype=F64, device=a.device)

    def phase(self, nodes):
        m = _mask(len(self.a.tree.nodes), nodes)
        _lib.check(self.lib.ht_inner_product_sharded(self.a._c(), self.c._c(), _ptr(m), self.ws.data_ptr(),
                                                     self.ws.numel(), self.res.data_ptr(), _lib.stream_handle()),
                   "sharded inner product")

    def slot(self, node: int) -> torch.Tensor:
        ptr = ctypes.c_void_p(0)
        cnt = ctypes.c_int64(0)
        _lib.check(self.lib.ht_inner_product_slot(self.a._c(), self.c._c(), ctypes.c_void_p(self.ws.data_ptr()),
                                                  node, ctypes.byref(ptr), ctypes.byref(cnt)), "phi slot")
        off = ptr.value - self.ws.data_ptr()
        return self.ws[off:off + 8 * cnt.value].view(F64)

    def result(self) -> torch.Tensor:
        return self.res


def sharded_apply(op, x: ShardedHTensor) -> ShardedHTensor:
    """apply_operator (arith.py:378-395) on the owned nodes: node-local (reference
    dist.py:324-333 _cmd_apply sends no messages).  The operator is replicated."""
    tree = x.tree
    ranks = {t: op.rank(t) * x.ranks[t] for t in x.ranks}
    sizes = {leaf.index: int(op.leaf_shape(leaf.index)[0]) for leaf in tree.leaves}
    arrays = {t: torch.empty(node_shape(tree, t, sizes, ranks), dtype=F64, device=x.device) for t in x.arrays}
    out = ShardedHTensor(tree, sizes, ranks, arrays, False)
    m = _mask(len(tree.nodes), x.arrays)
    _lib.check(_lib.load().ht_apply_operator_sharded(ctypes.byref(op._c()), x._c(), _ptr(m), out._c(),
                                                     _lib.stream_handle()), "sharded apply")
    return out


def sharded_scale(x: ShardedHTensor, alpha: float) -> ShardedHTensor:
    """scale (arith.py:368-371): alpha on the root matrix, on the rank that owns it
    (reference dist.py:334-341 _cmd_scale); leaves and transfers are shared."""
    arrays = dict(x.arrays)
    if 0 in arrays:
        root = arrays[0]
        new = torch.empty_like(root)
        _lib.check(_lib.load().ht_scale(root.data_ptr(), new.data_ptr(), root.numel(), float(alpha),
                                        _lib.stream_handle()), "sharded scale")
        arrays[0] = new
    return ShardedHTensor(x.tree, x.sizes, x.ranks, arrays, x.orthogonal)


def sharded_leaf_map(x: ShardedHTensor, dim: int, matrix) -> ShardedHTensor:
    """leaf_map (solvers.py:58-62): the owner of mode dim's leaf replaces U by M U
    (reference dist.py:342-349 _cmd_leafmap)."""
    from .arith import gemm

    leaf = x.tree.leaf_for_dim(dim).index
    arrays = dict(x.arrays)
    sizes = dict(x.sizes)
    if leaf in arrays:
        M = torch.as_tensor(np.asarray(matrix, dtype=np.float64)).to(x.device).contiguous()
        arrays[leaf] = gemm(M, arrays[leaf])
        sizes[leaf] = int(M.shape[0])
    else:
        sizes[leaf] = int(np.asarray(matrix).shape[0])
    return ShardedHTensor(x.tree, sizes, x.ranks, arrays, False)


class ShardedBackend:
    """The solver Backend seam (solvers.py:28-106) over the tree-sharded tensors: the
    reference's DistBackend role (solvers.py:68-106) with one GPU per subtree.  SPMD:
    every rank runs the same solver loop; values returned to the host (inner products,
    norms, max ranks) are identical on all ranks."""

    def __init__(self, comm, tree: DimensionTree, device=None):
        self.comm = comm
        self.smap = ShardMap.build(tree, comm.world)
        self.owned = self.smap.owned(comm.rank)
        self.device = device

    def lift(self, tensor) -> ShardedHTensor:
        return ShardedHTensor.from_host(self.smap.tree, dict(tensor.leaves), dict(tensor.transfer),
                                        tensor.root_matrix, self.owned, device=self.device)

    def retrieve(self, x: ShardedHTensor):
        """Gather the whole tensor on every rank (host numpy dicts)."""
        tree = x.tree
        nodes = {}
        for g in range(self.comm.world):
            for t in self.smap.owned(g):
                buf = (x.arrays[t].contiguous() if g == self.comm.rank
                       else torch.empty(x.shape(t), dtype=F64, device=x.device))
                if self.comm.world > 1:
                    self.comm.broadcast(buf, g)
                nodes[t] = buf.cpu().numpy()
        leaves = {leaf.index: nodes[leaf.index] for leaf in tree.leaves}
        transfer = {n.index: nodes[n.index] for n in tree.inner_nodes}
        return leaves, transfer, nodes[0]

    def lift_operator(self, op):
        return op

    def apply(self, op, x):
        return sharded_apply(op, x)

    def add(self, x, y):
        return sharded_add(x, y)

    def scale(self, x, alpha: float):
        return sharded_scale(x, alpha)

    def truncate(self, x, ctl):
        rel = getattr(ctl, "rel", None)
        if rel is not None:
            ctl = TruncationControl(eps=rel * self.norm(x), max_rank=ctl.max_rank)
        eng = GpuShardEngine(x, ctl, self.owned)
        return sharded_truncate(eng, self.comm, self.smap, ctl, x.orth_ranks())

    def inner_product(self, x, y) -> float:
        return sharded_inner_product(GpuInnerEngine(x, y), self.comm, self.smap)

    def norm(self, x) -> float:
        return math.sqrt(max(0.0, self.inner_product(x, x)))

    def leaf_map(self, x, dim: int, matrix):
        return sharded_leaf_map(x, dim, matrix)

    def max_rank(self, x) -> int:
        return max(x.ranks.values())


class LocalComm:
    """In-process communicator for G virtual ranks driven sequentially on one device
    (the survey's fake-shard mode): messages are device-to-device copies."""

    def __init__(self, rank: int, world: int, mailbox: dict):
        self.rank, self.world, self.box = rank, world, mailbox

    def send(self, t, dst):
        self.box.setdefault((self.rank, dst), []).append(t.clone())

    def recv_into(self, t, src):
        q = self.box.get((src, self.rank))
        if not q:
            raise RuntimeError(f"rank {self.rank}: no message from {src} (protocol order)")
        t.copy_(q.pop(0))

    def exchange(self, sends=(), recvs=()):
        for t, p in sends:
            self.send(t, p)
        for t, p in recvs:
            self.recv_into(t, p)

    def broadcast(self, t, src=0):
        if self.rank == src:
            for g in range(self.world):
                if g != src:
                    self.send(t, g)
        else:
            self.recv_into(t, src)

    def all_gather(self, t):
        for g in range(self.world):
            if g != self.rank:
                self.send(t, g)
        out = []
        for g in range(self.world):
            if g == self.rank:
                out.append(t.clone())
            else:
                b = torch.empty_like(t)
                self.recv_into(b, g)
                out.append(b)
        return out


def fake_shard_run(world: int, fn):
    """Run ``fn(rank, comm)`` for `world` virtual ranks on the current GPU (the survey's
    fake-shard mode): cooperative threads whose receives block on missing messages,
    device work issued in protocol order.  Returns the per-rank results."""
    import threading

    box: dict = {}
    results = [None] * world
    cv = threading.Condition()

    class BlockingComm(LocalComm):
        def recv_into(self, t, src):
            with cv:
                while not self.box.get((src, self.rank)):
                    cv.wait()
                t.copy_(self.box[(src, self.rank)].pop(0))

        def send(self, t, dst):
            with cv:
                self.box.setdefault((self.rank, dst), []).append(t.clone())
                cv.notify_all()

    errors = []

    def run(g):
        try:
            results[g] = fn(g, BlockingComm(g, world, box))
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)
            with cv:
                cv.notify_all()

    threads = [threading.Thread(target=run, args=(g,)) for g in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    return results


def fake_shard_truncate(x: HTensor, ctl: TruncationControl, world: int):
    """Run the sharded protocol with `world` virtual ranks on the current GPU and
    gather the result into one HTensor (used by tests and as the N>1 reference)."""
    tree = x.tree
    smap = ShardMap.build(tree, world)
    nn = len(tree.nodes)
    rbuf = (ctypes.c_int64 * nn)()
    _lib.check(_lib.load().ht_orth_ranks(x._c(), rbuf), "orth ranks")
    orth = {t: (x.rank(t) if x.orthogonal else int(rbuf[t])) for t in range(1, nn)}
    engines = [GpuShardEngine(ShardedHTensor.from_htensor(x, smap.owned(g)), ctl) for g in range(world)]
    results = fake_shard_run(world, lambda g, comm: sharded_truncate(engines[g], comm, smap, ctl, orth))
    nodes = {}
    for g in range(world):
        for t in smap.owned(g):
            nodes[t] = results[g].arrays[t]
    for g in range(world):  # every rank learned every kept rank
        assert results[g].ranks == results[0].ranks
    return HTensor._wrap(tree, nodes, False)


def fake_shard_inner_product(a: HTensor, c: HTensor, world: int) -> list:
    """<A, C> by the sharded protocol with `world` virtual ranks (each rank's value)."""
    smap = ShardMap.build(a.tree, world)
    engines = [GpuInnerEngine(ShardedHTensor.from_htensor(a, smap.owned(g)),
                              ShardedHTensor.from_htensor(c, smap.owned(g))) for g in range(world)]
    return fake_shard_run(world, lambda g, comm: sharded_inner_product(engines[g], comm, smap))


__all__ = ["ShardMap", "ShardedHTensor", "GpuShardEngine", "GpuInnerEngine", "TorchComm", "LocalComm",
           "ShardedBackend", "sharded_truncate", "sharded_add", "sharded_inner_product", "sharded_apply",
           "sharded_scale", "sharded_leaf_map", "shard_workspace_bytes", "fake_shard_run", "fake_shard_truncate",
           "fake_shard_inner_product", "static_ranks"]
