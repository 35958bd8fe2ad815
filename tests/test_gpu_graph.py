"""CUDA-graph replay of repeated fixed-rank truncations (driver.cu truncate_graph):
replays must reproduce the eager launches bit for bit, and the Cholesky-QR red flag
read behind the ORTH graph must still route rank-deficient input to the Householder
re-run (reference semantics: arith.py:325-352 with kernels.py:24-32's QR)."""

import numpy as np
import pytest

from oracle import htucker_oracle as orc
from tests.htconv import rel_err, to_host

pytestmark = pytest.mark.gpu


def _arrays(t):
    leaves, transfer, root = t.to_numpy()
    return [np.asarray(v) for _, v in sorted(leaves.items())] + \
           [np.asarray(v) for _, v in sorted(transfer.items())] + [np.asarray(root)]


def _truncs(htb, x, ctl, n):
    out = []
    for _ in range(n):
        out.append(_arrays(htb.truncate(x, ctl)))
    return out


@pytest.mark.parametrize("d,n,k", [(8, 300, 24), (16, 200, 40)])
def test_graph_replay_bitwise_equals_eager(cuda_ok, d, n, k):
    import paper_1708_03340_b200 as htb

    tree = htb.build_balanced_tree(d)
    x = htb.add(htb.gaussian_htensor(tree, n, k, 3), htb.gaussian_htensor(tree, n, k, 4))
    ctl = htb.TruncationControl.fixed_rank(k)
    htb.set_graph_mode(False)
    try:
        eager = _truncs(htb, x, ctl, 1)[0]
    finally:
        htb.set_graph_mode(True)
    c0, r0 = htb.graph_stats()
    got = _truncs(htb, x, ctl, 4)
    c1, r1 = htb.graph_stats()
    assert r1 - r0 >= 2, "repeated truncations of one tensor should replay the captured graph"
    assert c1 - c0 <= 2
    for g in got:
        for a, b in zip(g, eager):
            assert np.array_equal(a, b)
    ref = orc.truncate(to_host(x), orc.Ctl(max_rank=k))
    assert rel_err(to_host(htb.truncate(x, ctl)), ref) <= 1e-10


def test_graph_replay_routes_rank_deficient_input_to_householder(cuda_ok):
    import paper_1708_03340_b200 as htb

    tree = htb.build_balanced_tree(8)
    a = htb.gaussian_htensor(tree, 120, 12, 7)
    x = htb.add(a, a)  # rank 24 frames of rank 12: Cholesky-QR must raise its flag
    ctl = htb.TruncationControl.fixed_rank(12)
    f0 = htb.qr_fallback_count()
    outs = _truncs(htb, x, ctl, 4)
    assert htb.qr_fallback_count() - f0 == 4
    # replays take the Householder branch on the device (conditional node), no host check
    from paper_1708_03340_b200 import _lib
    assert _lib.load().ht_graph_device_fallback() == 1
    ref = orc.truncate(to_host(x), orc.Ctl(max_rank=12))
    leaves, transfer, root = htb.truncate(x, ctl).to_numpy()
    for o in outs[1:]:
        for p, q in zip(o, outs[0]):
            assert np.array_equal(p, q)
    got = orc.HT(orc.balanced_tree(8), {t: np.array(v) for t, v in leaves.items()},
                 {t: np.array(v) for t, v in transfer.items()}, np.array(root))
    assert orc.orth_difference_norm(got, ref) / orc.norm(ref) <= 1e-10
