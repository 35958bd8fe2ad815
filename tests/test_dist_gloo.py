"""Multi-rank sharded truncation (the paper's tree-parallel protocol) on CPU:
world sizes 2 and 4 under gloo, numpy node kernels, compared with the oracle's
serial truncate.  Exercises the real protocol code in paper_1708_03340_b200.dist."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist_
import torch.multiprocessing as mp

from oracle import htucker_oracle as orc


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, d, n, k, cap, eps_rel, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist_.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1708_03340_b200 import build_balanced_tree, dist
        from tests.np_engine import NumpyShardEngine

        tr = orc.balanced_tree(d)
        a = orc.gaussian_htensor(tr, n, k, 3)
        c = orc.gaussian_htensor(tr, n, k, 4)
        x = orc.add(a, c)
        eps = eps_rel * orc.norm(x) if eps_rel else None
        ctl = orc.Ctl(eps=eps, max_rank=cap)
        smap = dist.ShardMap.build(build_balanced_tree(d), world)
        ko = {t: orc.orthogonalize(x).rank(t) for t in range(1, tr.n_nodes)}
        eng = NumpyShardEngine(x, smap.owned(rank), ctl, ko)
        from paper_1708_03340_b200.arith import TruncationControl

        out = dist.sharded_truncate(eng, dist.TorchComm(), smap, TruncationControl(eps=eps, max_rank=cap), ko)
        # gather everything on rank 0
        if rank == 0:
            arrays = {t: out.arrays[t].numpy() for t in out.arrays}
            ranks = dict(out.ranks)
            for g in range(1, world):
                for t in smap.owned(g):
                    shp = torch.zeros(3, dtype=torch.int64)
                    dist_.recv(shp, g)
                    dims = [int(v) for v in shp if v > 0]
                    buf = torch.zeros(dims, dtype=torch.float64)
                    dist_.recv(buf, g)
                    arrays[t] = buf.numpy()
            U = {t: arrays[t] for t in tr.leaves_by_dim()}
            B = {t: arrays[t] for t in tr.inner_ids()}
            got = orc.HT(tr, U, B, arrays[0])
            ref = orc.truncate(x, ctl)
            q.put((got.ranks == ref.ranks, orc.orth_difference_norm(got, ref) / orc.norm(x),
                   eng.rk.tolist()))
        else:
            for t in smap.owned(rank):
                a_ = out.arrays[t]
                shp = torch.zeros(3, dtype=torch.int64)
                shp[: a_.dim()] = torch.tensor(a_.shape)
                dist_.send(shp, 0)
                dist_.send(a_.contiguous(), 0)
    finally:
        dist_.destroy_process_group()


@pytest.mark.parametrize("world,d,cap,eps_rel", [(2, 8, 6, None), (4, 8, 6, None), (2, 16, 5, None),
                                                 (2, 8, 12, 0.3), (4, 16, None, 0.2),
                                                 (2, 3, 4, None), (4, 10, 5, None)])
def test_sharded_truncate_matches_serial(world, d, cap, eps_rel):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, 12, 4, cap, eps_rel, q)) for r in range(world)]
    for p in procs:
        p.start()
    ranks_equal, err, _ = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ranks_equal
    assert err <= 1e-12


def _ip_worker(rank, world, port, d, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist_.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1708_03340_b200 import build_balanced_tree, dist
        from tests.np_engine import NumpyInnerEngine

        tr = orc.balanced_tree(d)
        a = orc.gaussian_htensor(tr, n, 3, 5)
        c = orc.add(orc.gaussian_htensor(tr, n, 2, 6), a)  # different ranks on every node
        smap = dist.ShardMap.build(build_balanced_tree(d), world)
        v = dist.sharded_inner_product(NumpyInnerEngine(a, c), dist.TorchComm(), smap)
        q.put((rank, v, orc.inner_product(a, c)))
    finally:
        dist_.destroy_process_group()


@pytest.mark.parametrize("world,d", [(2, 8), (4, 8), (4, 16), (2, 10), (4, 10)])
def test_sharded_inner_product_matches_serial(world, d):
    """The GRAM_UP wave (reference dist.py:239-254): Phi of the shard roots up, rank 0
    finishes the top levels, every rank returns the same value."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ip_worker, args=(r, world, port, d, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, v, ref in got:
        np.testing.assert_allclose(v, ref, rtol=1e-12)


def test_c5_shard_workspace_fits():
    """C5 (d=256, n=2048, rank 400 -> 100) on 8 GPUs: each rank's truncate workspace is
    planned for its 32-leaf subtree (+ the top nodes on rank 0) and their message slots,
    not the whole tree -- host-only query, no device needed."""
    from paper_1708_03340_b200 import build_balanced_tree, dist

    tree = build_balanced_tree(256)
    sizes = {leaf.index: 2048 for leaf in tree.leaves}
    ranks = {t: 400 for t in range(1, len(tree.nodes))}
    whole = dist.shard_workspace_bytes(tree, sizes, ranks, None)
    smap = dist.ShardMap.build(tree, 8)
    per = [dist.shard_workspace_bytes(tree, sizes, ranks, smap.owned(g)) for g in range(8)]
    assert whole > 100e9  # the whole-tree plan cannot fit one B200
    assert max(per) < 40e9, [f"{b / 1e9:.1f} GB" for b in per]
    assert max(per) < whole / 4


def test_shard_map_layout():
    from paper_1708_03340_b200 import build_balanced_tree, dist

    tr = build_balanced_tree(64)
    for world in (1, 2, 4, 8):
        sm = dist.ShardMap.build(tr, world)
        assert len(sm.roots) == world
        assert len(sm.top) == world - 1
        owned = sorted(t for g in range(world) for t in sm.owned(g))
        assert owned == list(range(len(tr.nodes)))  # a partition of the tree
        assert all(len(sm.subtree(g)) == 2 * (64 // world) - 1 for g in range(world))
    assert len(dist.ShardMap.build(build_balanced_tree(10), 4).roots) == 4  # uneven subtrees are fine
    with pytest.raises(ValueError):
        dist.ShardMap.build(build_balanced_tree(3), 4)  # level 2 has only 2 nodes
    with pytest.raises(ValueError):
        dist.ShardMap.build(build_balanced_tree(8), 3)  # not a power of two
