"""Block-form (lazy) sums: ``add`` keeps the block-diagonal transfer
tensors of reference arith.py:173-192 unmaterialised and ``truncate`` runs the sweep's
mode products on the diagonal blocks.  Checked against the CPU oracle (ranks, error
<= 1e-10, sigma rtol 1e-10) and against the materialised path of the library."""

import numpy as np
import pytest

from oracle import htucker_oracle as orc
from tests.htconv import rel_err, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[("auto", True), ("auto", False), ("householder", True)],
                ids=["fast", "explicit_q", "householder"])
def htb(cuda_ok, request):
    import paper_1708_03340_b200 as m

    m.set_qr_mode(request.param[0])
    m.set_implicit_q(request.param[1])
    m.set_lazy_add(True, min_values=0)  # block form for the small test tensors too
    yield m
    m.set_lazy_add(True, min_values=1 << 20)
    m.set_qr_mode("auto")
    m.set_implicit_q(True)


def _sig(s):
    return {t: v.cpu().numpy() for t, v in s.items()}


def test_lazy_sum_values_are_the_eager_ones(htb):
    tr = orc.balanced_tree(6)
    a, c, e = (orc.gaussian_htensor(tr, [9, 10, 11, 12, 13, 14], k, s) for k, s in ((3, 1), (4, 2), (2, 3)))
    da, dc, de = to_dev(a), to_dev(c), to_dev(e)
    lazy = htb.add(da, dc)
    assert isinstance(lazy, htb.SumHTensor) and not lazy.is_materialized
    assert lazy.ranks == {t: 7 for t in range(1, 11)} and lazy.shape == (9, 10, 11, 12, 13, 14)
    eager = htb.add(da, dc, lazy=False)
    assert not isinstance(eager, htb.SumHTensor)
    # three terms with coefficients: a - c + e, against the eager chain and the oracle
    lazy3 = htb.add(htb.subtract(da, dc), de)
    assert isinstance(lazy3, htb.SumHTensor) and not lazy3.is_materialized and lazy3.max_rank == 9
    eager3 = htb.add(htb.add(da, htb.scale(dc, -1.0), lazy=False), de, lazy=False)
    ref3 = orc.add(orc.add(a, orc.scale(c, -1.0)), e)
    for (t, u), (_, v), (_, w) in zip(to_host(lazy3).arrays(), to_host(eager3).arrays(), ref3.arrays()):
        np.testing.assert_array_equal(u, v)
        np.testing.assert_array_equal(u, w)
    for (t, u), (_, v) in zip(to_host(lazy).arrays(), to_host(eager).arrays()):
        np.testing.assert_array_equal(u, v)
    assert lazy.is_materialized


@pytest.mark.parametrize("d,n,ka,kc,r", [(8, 64, 10, 10, 10), (5, 40, 7, 4, 6), (4, 150, 60, 60, 50), (8, 300, 70, 60, 40)],
                         ids=["c1-shape", "unequal-unbalanced", "K120", "K130-gemm-path"])
def test_truncate_lazy_sum(htb, d, n, ka, kc, r):
    tr = orc.balanced_tree(d)
    a, c = orc.gaussian_htensor(tr, n, ka, 11), orc.gaussian_htensor(tr, n, kc, 12)
    x = orc.add(a, orc.scale(c, 0.5))
    xd = htb.add(to_dev(a), htb.scale(to_dev(c), 0.5))
    sig = _sig(htb.hierarchical_singular_values(xd))
    T = htb.truncate(xd, htb.TruncationControl.fixed_rank(r))
    assert not xd.is_materialized
    ref = orc.truncate(x, orc.Ctl(max_rank=r))
    assert to_host(T).ranks == ref.ranks
    assert rel_err(to_host(T), ref) <= 1e-10
    # K > 112: the large-K eigensolver delivers absolute accuracy u ||G|| on ungraded
    # spectra, i.e. u sigma_0^2 / (2 sigma) on the smallest sigma
    atol = 1e-13 if ka + kc <= 112 else 5e-12
    for t, s in orc.hierarchical_singular_values(x).items():
        np.testing.assert_allclose(sig[t], s, rtol=1e-10, atol=atol * s[0])
    eps = 0.3 * orc.norm(x)
    Te = htb.truncate(xd, htb.TruncationControl.accuracy(eps))
    refe = orc.truncate(x, orc.Ctl(eps=eps))
    assert to_host(Te).ranks == refe.ranks
    assert rel_err(to_host(Te), refe) <= 1e-10
    # the materialised path gives the same tensor
    T2 = htb.truncate(htb.add(to_dev(a), htb.scale(to_dev(c), 0.5), lazy=False), htb.TruncationControl.fixed_rank(r))
    assert rel_err(to_host(T), to_host(T2)) <= 1e-12


def test_four_term_sum_c5_shape(htb):
    """C5's input: the sum of four tensors (rank 4k), 15/16 of every transfer tensor
    structurally zero -- here k = 30 (K = 120) on d = 8."""
    tr = orc.balanced_tree(8)
    parts = [orc.gaussian_htensor(tr, 200, 30, s) for s in range(4)]
    x = orc.add(orc.add(orc.add(parts[0], parts[1]), parts[2]), parts[3])
    dp = [to_dev(p) for p in parts]
    xd = htb.add(htb.add(htb.add(dp[0], dp[1]), dp[2]), dp[3])
    assert isinstance(xd, htb.SumHTensor) and len(xd._terms) == 4 and xd.max_rank == 120
    T = htb.truncate(xd, htb.TruncationControl.fixed_rank(30))
    assert not xd.is_materialized
    ref = orc.truncate(x, orc.Ctl(max_rank=30))
    assert to_host(T).ranks == ref.ranks
    assert rel_err(to_host(T), ref) <= 1e-10
    # balanced pairing add(add(a, b), add(c, d)) flattens to the same four blocks
    xd2 = htb.add(htb.add(dp[0], dp[1]), htb.add(dp[2], dp[3]))
    assert len(xd2._terms) == 4
    T2 = htb.truncate(xd2, htb.TruncationControl.fixed_rank(30))
    assert rel_err(to_host(T2), ref) <= 1e-10


def test_rank_deficient_lazy_sum(htb):
    """add(a, a): exactly rank-deficient frames (the Cholesky-QR red flag / Householder path)."""
    tr = orc.balanced_tree(4)
    a = orc.gaussian_htensor(tr, 40, 6, 3)
    da = to_dev(a)
    T = htb.truncate(htb.add(da, da), htb.TruncationControl.fixed_rank(6))
    ref = orc.scale(a, 2.0)
    assert rel_err(to_host(T), ref) <= 1e-10


def test_lazy_sum_out_reuse_and_graph_replay(htb):
    """add(a, c, out=S) refills a SumHTensor's leaf arena; repeated fixed-rank truncations
    of it replay a captured graph and follow the new values."""
    tr = orc.balanced_tree(8)
    ttr = htb.build_balanced_tree(8)
    ctl = htb.TruncationControl.fixed_rank(8)
    da = htb.HTensor(ttr, *htb.gaussian_factors(ttr, 50, 8, 1))
    dc = htb.HTensor(ttr, *htb.gaussian_factors(ttr, 50, 8, 2))
    S = htb.add(da, dc)
    out = htb.truncate(S, ctl)
    for seed in (3, 4, 5, 6):
        a, c = orc.gaussian_htensor(tr, 50, 8, seed), orc.gaussian_htensor(tr, 50, 8, seed + 10)
        ha, hc = to_dev(a), to_dev(c)
        da.load_host_arena(ha.to_host_arena())
        dc.load_host_arena(hc.to_host_arena())
        S2 = htb.add(da, dc, out=S)
        assert S2 is S and not S.is_materialized
        T = htb.truncate(S, ctl, out=out)
        ref = orc.truncate(orc.add(a, c), orc.Ctl(max_rank=8))
        assert rel_err(to_host(T), ref) <= 1e-10


def _ht_with_ranks(tr, sizes, ranks, seed):
    rng = np.random.default_rng(seed)
    U, B = {}, {}
    for t in range(tr.n_nodes):
        if tr.is_leaf(t):
            U[t] = rng.standard_normal((sizes[tr.interval[t][0] - 1], ranks[t]))
        elif t > 0:
            s1, s2 = tr.sons[t]
            B[t] = rng.standard_normal((ranks[t], ranks[s1], ranks[s2])) / ranks[t]
    s1, s2 = tr.sons[0]
    return orc.HT(tr, U, B, rng.standard_normal((ranks[s1], ranks[s2])))


@pytest.mark.parametrize("lazy", [False, True], ids=["eager", "lazy"])
def test_c4_rank_pattern_with_cholqr_fallback(htb, lazy):
    """The first CG residual of C4 (a rank-1 right-hand side plus an applied tensor with
    node-dependent ranks, parameter leaves of size 4, d = 10 unbalanced): a Cholesky-QR
    sweep raises its red flag here, the truncation is redone on the Householder path, and
    the discarded sweep's eigenproblems must not leave a sticky error behind."""
    tr = orc.balanced_tree(10)
    rk = [1, 6, 6, 3, 4, 3, 8, 2, 2, 2, 3, 2, 2, 2, 9, 2, 2, 2, 10]
    sizes = [4] * 9 + [49]
    a = _ht_with_ranks(tr, sizes, {t: 1 for t in range(19)}, 0)
    c = _ht_with_ranks(tr, sizes, {t: rk[t] for t in range(19)}, 1)
    x = orc.add(a, c)
    xd = htb.add(to_dev(a), to_dev(c), lazy=lazy)
    T = htb.truncate(xd, htb.TruncationControl.fixed_rank(20))
    htb.synchronize()  # raises if a stale eigensolver status was left behind
    ref = orc.truncate(x, orc.Ctl(max_rank=20))
    assert to_host(T).ranks == ref.ranks
    assert rel_err(to_host(T), ref) <= 1e-10
    eps = 1e-3 * orc.norm(x)
    Te = htb.truncate(xd, htb.TruncationControl.accuracy(eps, 20))
    refe = orc.truncate(x, orc.Ctl(eps=eps, max_rank=20))
    assert to_host(Te).ranks == refe.ranks
    assert rel_err(to_host(Te), refe) <= 1e-10


def test_inner_product_of_block_form_sums_is_bilinear(htb):
    """<X, Y> for unmaterialised sums runs on the terms (no materialisation) and agrees
    with the oracle's inner product of the materialised sums."""
    tr = orc.balanced_tree(8)
    a, c, e = (orc.gaussian_htensor(tr, 40, k, s) for k, s in ((6, 1), (5, 2), (4, 3)))
    da, dc, de = to_dev(a), to_dev(c), to_dev(e)
    x, xr = htb.subtract(htb.add(da, dc), de), orc.add(orc.add(a, c), orc.scale(e, -1.0))
    y, yr = htb.add(de, da), orc.add(e, a)
    np.testing.assert_allclose(htb.inner_product(x, x), orc.inner_product(xr, xr), rtol=1e-12)
    np.testing.assert_allclose(htb.inner_product(x, y), orc.inner_product(xr, yr), rtol=1e-11)
    np.testing.assert_allclose(htb.inner_product(x, dc), orc.inner_product(xr, c), rtol=1e-11)
    np.testing.assert_allclose(htb.norm(x), orc.norm(xr), rtol=1e-12)
    assert not x.is_materialized and not y.is_materialized


def test_three_unequal_terms_staircase(htb):
    """Three terms of unequal, node-dependent ranks (the staircase of corners has three
    steps of different sizes), fixed-rank (graph-captured on repeat) and accuracy control."""
    tr = orc.balanced_tree(8)
    rk = lambda base: {t: base + (t % 3) for t in range(1, 15)}  # noqa: E731
    a = orc.gaussian_htensor(tr, 60, rk(4), 21)
    c = orc.gaussian_htensor(tr, 60, rk(3), 22)
    e = orc.gaussian_htensor(tr, 60, rk(5), 23)
    x = orc.add(orc.add(a, orc.scale(c, -1.0)), e)
    xd = htb.add(htb.subtract(to_dev(a), to_dev(c)), to_dev(e))
    assert isinstance(xd, htb.SumHTensor) and len(xd._terms) == 3
    ref = orc.truncate(x, orc.Ctl(max_rank=6))
    for _ in range(3):  # eager, capture, replay
        T = htb.truncate(xd, htb.TruncationControl.fixed_rank(6))
        assert to_host(T).ranks == ref.ranks
        assert rel_err(to_host(T), ref) <= 1e-10
    eps = 0.2 * orc.norm(x)
    Te = htb.truncate(xd, htb.TruncationControl.accuracy(eps))
    refe = orc.truncate(x, orc.Ctl(eps=eps))
    assert to_host(Te).ranks == refe.ranks
    assert rel_err(to_host(Te), refe) <= 1e-10
    assert not xd.is_materialized
