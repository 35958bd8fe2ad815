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


class GpuShardEngine:
    def __init__(self, x: ShardedHTensor, ctl: TruncationControl):
        self.lib = _lib.load()
        self.x = x
        self.ctl = ctl
        nn = len(x.tree.nodes)
        self.cctl, self._keep = ctl._c(nn)
        nbytes = ctypes.c_size_t(0)
        _lib.check(self.lib.ht_truncate_workspace_size(x._c(), ctypes.byref(nbytes)), "sharded truncate")
        self.ws = _ws(nbytes.value, x._dummy.device)

    def phase(self, ph: int, nodes, out: ShardedHTensor | None = None):
        m = np.ascontiguousarray(np.zeros(len(self.x.tree.nodes), dtype=np.uint8))
        m[list(nodes)] = 1
        _lib.check(self.lib.ht_truncate_sharded(self.x._c(), ctypes.byref(self.cctl), self.ws.data_ptr(),
                                                self.ws.numel(), ph, m.ctypes.data_as(ctypes.c_void_p),
                                                out._c() if out is not None else None, _lib.stream_handle()),
                   f"sharded truncate phase {ph}")

    def slot(self, kind: int, node: int) -> torch.Tensor:
        ptr = ctypes.c_void_p(0)
        cnt = ctypes.c_int64(0)
        _lib.check(self.lib.ht_truncate_slot(self.x._c(), ctypes.c_void_p(self.ws.data_ptr()), kind, node,
                                             ctypes.byref(ptr), ctypes.byref(cnt)), "workspace slot")
        off = ptr.value - self.ws.data_ptr()
        if kind == SLOT_RANKS:
            return self.ws[off:off + 4 * cnt.value].view(torch.int32)
        return self.ws[off:off + 8 * cnt.value].view(F64)

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
    """Point-to-point over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def send(self, t: torch.Tensor, dst: int):
        self.dist.send(t.contiguous(), dst, group=self.group)

    def recv_into(self, t: torch.Tensor, src: int):
        if t.is_contiguous():
            self.dist.recv(t, src, group=self.group)
        else:
            buf = torch.empty_like(t, memory_format=torch.contiguous_format)
            self.dist.recv(buf, src, group=self.group)
            t.copy_(buf)


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

    Returns this rank's ShardedHTensor of the truncated tensor (owned nodes).
    Messages: wave 1 R factors (shard roots -> 0), wave 2 Gramians (0 -> shard
    roots), wave 3 eigenvector blocks + ranks (shard roots -> 0).
    """
    r, G = comm.rank, comm.world
    tree = smap.tree
    sub = smap.subtree(r)
    # wave 1: bottom-up orthogonalisation, R of the shard root goes up
    engine.phase(ORTH, sub)
    if r != 0:
        comm.send(engine.slot(SLOT_R, smap.roots[r]), 0)
    else:
        for g in range(1, G):
            comm.recv_into(engine.slot(SLOT_R, smap.roots[g]), g)
        if smap.top:
            engine.phase(ORTH, smap.top)
            engine.phase(GRAM, smap.top)
        # wave 2: reduced Gramians of the shard roots go down
        for g in range(1, G):
            comm.send(engine.slot(SLOT_G, smap.roots[g]), g)
    if r != 0:
        comm.recv_into(engine.slot(SLOT_G, smap.roots[r]), 0)
    inner_sub = [t for t in sub if not tree.node(t).is_leaf]
    engine.phase(GRAM, inner_sub)
    owned = smap.owned(r)
    engine.phase(EIG, [t for t in owned if t != 0])
    # kept ranks
    ranks = static_ranks(tree, orth_ranks, ctl)
    if ranks is None:
        local = engine.ranks()
        ranks = {t: int(local[t]) for t in owned if t != 0}
    # wave 3: eigenvector blocks (and ranks) of the shard roots go up
    if r != 0:
        s = smap.roots[r]
        comm.send(torch.tensor([ranks[s]], dtype=torch.float64, device=engine.slot(SLOT_EV, s).device), 0)
        comm.send(engine.slot(SLOT_EV, s), 0)
    else:
        for g in range(1, G):
            s = smap.roots[g]
            rk = torch.zeros(1, dtype=torch.float64, device=engine.slot(SLOT_EV, s).device)
            comm.recv_into(rk, g)
            ranks[s] = int(rk.item())
            comm.recv_into(engine.slot(SLOT_EV, s), g)
    full = {t: ranks.get(t, orth_ranks[t]) for t in range(1, len(tree.nodes))}
    out = engine.allocate_out(full, owned)
    engine.phase(PROJECT, owned, out)
    return out


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


def fake_shard_truncate(x: HTensor, ctl: TruncationControl, world: int):
    """Run the sharded protocol with `world` virtual ranks on the current GPU and
    gather the result into one HTensor (used by tests and as the N>1 reference)."""
    import threading

    tree = x.tree
    smap = ShardMap.build(tree, world)
    nn = len(tree.nodes)
    rbuf = (ctypes.c_int64 * nn)()
    _lib.check(_lib.load().ht_orth_ranks(x._c(), rbuf), "orth ranks")
    orth = {t: (x.rank(t) if x.orthogonal else int(rbuf[t])) for t in range(1, nn)}
    box: dict = {}
    results = [None] * world
    engines = [GpuShardEngine(ShardedHTensor.from_htensor(x, smap.owned(g)), ctl) for g in range(world)]
    # The protocol is sequentially consistent: run ranks as cooperative threads that
    # block on missing messages (device work is issued to one stream in order).
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
            results[g] = sharded_truncate(engines[g], BlockingComm(g, world, box), smap, ctl, orth)
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
    nodes = {}
    for g in range(world):
        for t in smap.owned(g):
            nodes[t] = results[g].arrays[t]
    return HTensor._wrap(tree, nodes, False)


__all__ = ["ShardMap", "ShardedHTensor", "GpuShardEngine", "TorchComm", "LocalComm", "sharded_truncate", "sharded_add",
           "fake_shard_truncate", "static_ranks"]
