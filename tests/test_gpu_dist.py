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
