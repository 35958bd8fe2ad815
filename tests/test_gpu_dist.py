"""Sharded truncation on one B200 in fake-shard mode: G virtual ranks run the real
protocol (masked C-ABI phases + message waves as device copies); the result must
match the single-launch truncation."""

import numpy as np
import pytest

from oracle import htucker_oracle as orc
from tests.htconv import rel_err, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_fake_shard_equals_single_gpu(cuda_ok, world):
    import paper_1708_03340_b200 as htb
    from paper_1708_03340_b200 import dist

    a, c, x = orc.c2_inputs(16, 200, 20)
    xd = htb.add(to_dev(a), to_dev(c))
    ctl = htb.TruncationControl.fixed_rank(20)
    t1 = to_host(htb.truncate(xd, ctl))
    tg = to_host(dist.fake_shard_truncate(xd, ctl, world))
    assert tg.ranks == t1.ranks
    assert rel_err(tg, t1) <= 1e-12
    assert rel_err(tg, orc.truncate(x, orc.Ctl(max_rank=20))) <= 1e-10


def test_fake_shard_accuracy_mode(cuda_ok):
    import paper_1708_03340_b200 as htb
    from paper_1708_03340_b200 import dist

    a, c, x = orc.c2_inputs(8, 100, 12)
    xd = htb.add(to_dev(a), to_dev(c))
    eps = 0.3 * orc.norm(x)
    ctl = htb.TruncationControl.accuracy(eps)
    tg = to_host(dist.fake_shard_truncate(xd, ctl, 4))
    ref = orc.truncate(x, orc.Ctl(eps=eps))
    assert tg.ranks == ref.ranks
    assert rel_err(tg, ref) <= 1e-10


def test_sharded_add_equals_add(cuda_ok):
    import torch

    import paper_1708_03340_b200 as htb
    from paper_1708_03340_b200 import dist

    tree = htb.build_balanced_tree(8)
    fa = htb.gaussian_factors(tree, 30, 4, 5)
    fc = htb.gaussian_factors(tree, 30, 3, 6)
    full = htb.subtract(htb.HTensor(tree, *fa), htb.HTensor(tree, *fc))
    smap = dist.ShardMap.build(tree, 4)
    for g in range(4):
        own = smap.owned(g)
        a = dist.ShardedHTensor.from_host(tree, *fa, own)
        c = dist.ShardedHTensor.from_host(tree, *fc, own)
        s = dist.sharded_add(a, c, -1.0)
        assert set(s.arrays) == set(own)
        for t in own:
            assert torch.equal(s.arrays[t], full.node_array(t))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_fake_shard_inner_product(cuda_ok, world):
    """GRAM_UP wave (reference dist.py:239-254) with virtual ranks: every rank returns
    the serial <A, C>."""
    import paper_1708_03340_b200 as htb
    from paper_1708_03340_b200 import dist

    a, c, x = orc.c2_inputs(16, 120, 9)
    ad, cd = to_dev(a), htb.add(to_dev(c), to_dev(a))
    vals = dist.fake_shard_inner_product(ad, cd, world)
    ref = orc.inner_product(a, orc.add(c, a))
    for v in vals:
        np.testing.assert_allclose(v, ref, rtol=1e-12)
    np.testing.assert_allclose(vals[0], htb.inner_product(ad, cd), rtol=1e-13)


def test_sharded_apply_scale_leaf_map(cuda_ok):
    """Node-local sharded operations (reference dist.py:324-349): apply_operator, scale
    and leaf_map on each shard's nodes equal the single-GPU results bit for bit."""
    import torch

    import paper_1708_03340_b200 as htb
    from paper_1708_03340_b200 import dist, problems

    tree = htb.build_balanced_tree(8)
    f = htb.gaussian_factors(tree, 40, 5, 9)
    full = htb.HTensor(tree, *f)
    op = problems.laplace_sum_operator(tree, 40)
    ref_apply = htb.apply_operator(op, full)
    ref_scale = htb.scale(full, -2.5)
    M = np.random.default_rng(1).standard_normal((40, 40))
    ref_map = htb.leaf_map(full, 3, M)
    smap = dist.ShardMap.build(tree, 4)
    for g in range(4):
        own = smap.owned(g)
        xs = dist.ShardedHTensor.from_host(tree, *f, own)
        ya = dist.sharded_apply(op, xs)
        ys = dist.sharded_scale(xs, -2.5)
        ym = dist.sharded_leaf_map(xs, 3, M)
        for t in own:
            assert torch.equal(ya.arrays[t], ref_apply.node_array(t))
            assert torch.equal(ys.arrays[t], ref_scale.node_array(t))
            assert torch.equal(ym.arrays[t], ref_map.node_array(t))


def test_fake_shard_workspace_is_shard_local(cuda_ok):
    """Each virtual rank's engine plans only its owned nodes and their sons' slots."""
    import paper_1708_03340_b200 as htb
    from paper_1708_03340_b200 import dist

    a, c, x = orc.c2_inputs(32, 200, 20)
    xd = htb.add(to_dev(a), to_dev(c))
    ctl = htb.TruncationControl.fixed_rank(20)
    smap = dist.ShardMap.build(xd.tree, 8)
    whole = dist.GpuShardEngine(dist.ShardedHTensor.from_htensor(xd, range(len(xd.tree.nodes))), ctl).ws.numel()
    for g in range(8):
        eng = dist.GpuShardEngine(dist.ShardedHTensor.from_htensor(xd, smap.owned(g)), ctl)
        # rank 0 also holds the 7 top nodes; the 4 KB-per-node slack is plan-wide
        assert eng.ws.numel() < whole / (2 if g == 0 else 4)
    tg = to_host(dist.fake_shard_truncate(xd, ctl, 8))
    assert rel_err(tg, orc.truncate(x, orc.Ctl(max_rank=20))) <= 1e-10
