"""Kronecker-fused orthogonalisation: ``apply_operator`` keeps the
transfer tensors F_t = H_t (x) B_t (reference arith.py:204-213) unmaterialised and
``truncate`` consumes H_t, B_t in place.  Checked against the CPU oracle (ranks, error
<= 1e-10, sigma rtol 1e-10) and against the materialised path of the library itself."""

import ctypes

import numpy as np
import pytest

from oracle import htucker_oracle as orc
from tests.htconv import rel_err, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["auto", "householder"])
def htb(cuda_ok, request):
    import paper_1708_03340_b200 as m

    m.set_qr_mode(request.param)
    yield m
    m.set_qr_mode("auto")


def _laplace(htb, d, n):
    tr = orc.balanced_tree(d)
    op = orc.laplace_operator(tr, n)
    ttr = htb.build_balanced_tree(d)
    dop = htb.HTOperator(ttr, {t: [htb.GeneralizedMatrix.diagonal(w[0].data), htb.GeneralizedMatrix.csr(w[1].data)]
                                for t, w in op.W.items()}, dict(op.H), op.root)
    return tr, op, dop


def _random_operator(htb, d, sizes, rank, seed):
    """Dense-leaf operator with Gaussian H_t of uniform rank `rank` (exercises every (a, c) job)."""
    tr = orc.balanced_tree(d)
    rng = np.random.default_rng(seed)
    leaves = tr.leaves_by_dim()
    W = {t: [orc.GMat("dense", rng.standard_normal((sizes[i], sizes[i])) / np.sqrt(sizes[i])) for _ in range(rank)]
         for i, t in enumerate(leaves)}
    H = {t: rng.standard_normal((rank, rank, rank)) / rank for t in tr.inner_ids()}
    op = orc.HTOp(tr, W, H, rng.standard_normal((rank, rank)))
    ttr = htb.build_balanced_tree(d)
    dop = htb.HTOperator(ttr, {t: [htb.GeneralizedMatrix.dense(g.data) for g in w] for t, w in W.items()}, H, op.root)
    return tr, op, dop


def _sig(s):
    return {t: v.cpu().numpy() for t, v in s.items()}


def test_lazy_apply_values_are_the_eager_ones(htb):
    tr, op, dop = _laplace(htb, 8, 32)
    x = orc.gaussian_htensor(tr, 32, 6, 3)
    lazy = htb.apply_operator(dop, to_dev(x))
    assert isinstance(lazy, htb.AppliedHTensor) and not lazy.is_materialized
    assert lazy.ranks == {t: 12 for t in range(1, 15)} and lazy.shape == (32,) * 8
    eager = htb.apply_operator(dop, to_dev(x), lazy=False)
    assert not isinstance(eager, htb.AppliedHTensor)
    for (t, u), (_, v) in zip(to_host(lazy).arrays(), to_host(eager).arrays()):
        np.testing.assert_array_equal(u, v)
    assert lazy.is_materialized
    ref = orc.apply_operator(op, x)
    for (t, u), (_, v) in zip(to_host(lazy).arrays(), ref.arrays()):
        np.testing.assert_allclose(u, v, rtol=1e-13, atol=1e-13)


def test_c3_full_size_kron_truncate(htb):
    """BASELINE config C3 (d=16, n=256, k=30, Laplace-sum operator ranks 2 -> rank 60 ->
    eps / cap 30) with F_t never materialised."""
    tr, op, dop = _laplace(htb, 16, 256)
    x = orc.gaussian_htensor(tr, 256, 30, 16)
    yr = orc.apply_operator(op, x)
    eps = 1e-8 * orc.norm(yr)
    y = htb.apply_operator(dop, to_dev(x))
    sig = _sig(htb.hierarchical_singular_values(y))
    T = htb.truncate(y, htb.TruncationControl(eps=eps, max_rank=30))
    assert not y.is_materialized
    ref = orc.truncate(yr, orc.Ctl(eps=eps, max_rank=30))
    assert to_host(T).ranks == ref.ranks
    assert rel_err(to_host(T), ref) <= 1e-10
    for t, s in orc.hierarchical_singular_values(yr).items():
        np.testing.assert_allclose(sig[t], s, rtol=1e-10, atol=1e-13 * s[0])
    # the materialised path of the library gives the same tensor
    T2 = htb.truncate(htb.apply_operator(dop, to_dev(x), lazy=False), htb.TruncationControl(eps=eps, max_rank=30))
    assert to_host(T2).ranks == to_host(T).ranks
    assert rel_err(to_host(T), to_host(T2)) <= 1e-12


@pytest.mark.parametrize("d,n,k,r", [(4, 20, 5, 3), (5, 24, 7, 2), (8, 48, 40, 3), (6, 40, 12, 9)],
                         ids=["d4r3", "d5r2-unbalanced", "d8K120-gemm-path", "d6r9"])
def test_kron_truncate_random_operator(htb, d, n, k, r):
    """Dense Gaussian operator transfer tensors of rank r (every (a, c) job distinct);
    K = r k = 120 takes the grouped-GEMM path (N > 104), r = 9 the C4 operator rank."""
    sizes = [n + i for i in range(d)]
    tr, op, dop = _random_operator(htb, d, sizes, r, seed=d + r)
    x = orc.gaussian_htensor(tr, sizes, k, 5)
    yr = orc.apply_operator(op, x)
    y = htb.apply_operator(dop, to_dev(x))
    T = htb.truncate(y, htb.TruncationControl.fixed_rank(k))
    assert not y.is_materialized
    ref = orc.truncate(yr, orc.Ctl(max_rank=k))
    assert to_host(T).ranks == ref.ranks
    assert rel_err(to_host(T), ref) <= 1e-10
    # accuracy control: ranks chosen from the Gramian spectra of the Kronecker-form input
    eps = 1e-3 * orc.norm(yr)
    Te = htb.truncate(y, htb.TruncationControl.accuracy(eps))
    refe = orc.truncate(yr, orc.Ctl(eps=eps))
    assert to_host(Te).ranks == refe.ranks
    assert rel_err(to_host(Te), refe) <= 1e-10


def test_kron_form_is_rejected_outside_truncate(htb):
    """The C ABI accepts ht_tensor.kron in the truncation entry points only."""
    from paper_1708_03340_b200 import _lib

    tr, op, dop = _laplace(htb, 4, 8)
    x = to_dev(orc.gaussian_htensor(tr, 8, 3, 1))
    y = htb.apply_operator(dop, x)
    lib = _lib.load()
    nbytes = ctypes.c_size_t(0)
    assert lib.ht_inner_product_workspace_size(y._c_trunc(), y._c_trunc(), ctypes.byref(nbytes)) == _lib.HT_ERR_UNSUPPORTED
    assert not y.is_materialized
    # the Python API materialises instead
    ref = orc.apply_operator(op, to_host(x))
    np.testing.assert_allclose(htb.inner_product(y, y), orc.inner_product(ref, ref), rtol=1e-12)
    assert y.is_materialized


def test_relative_eps_on_device(htb):
    """HT_CTL_RELATIVE_EPS: eps = rel ||x|| with ||x|| read off the orthogonalised root on
    the device -- same ranks and tensor as the absolute control with the norm from an
    inner product (C3's control), for a Kronecker-form and an ordinary input."""
    tr, op, dop = _laplace(htb, 16, 256)
    x = orc.gaussian_htensor(tr, 256, 30, 16)
    yr = orc.apply_operator(op, x)
    ref = orc.truncate(yr, orc.Ctl(eps=1e-8 * orc.norm(yr), max_rank=30))
    ctl = htb.TruncationControl.relative_accuracy(1e-8, max_rank=30)
    for lazy in (True, False):
        y = htb.apply_operator(dop, to_dev(x), lazy=lazy)
        T = htb.truncate(y, ctl)
        assert lazy == (isinstance(y, htb.AppliedHTensor) and not y.is_materialized)
        assert to_host(T).ranks == ref.ranks
        assert rel_err(to_host(T), ref) <= 1e-10
    # accuracy-only control on a sum (ranks from the spectra)
    a, c, _ = orc.c1_inputs()
    xs = orc.add(orc.scale(a, 2.0), orc.scale(c, 1e-3))
    xd = htb.add(htb.scale(to_dev(a), 2.0), htb.scale(to_dev(c), 1e-3))
    for rel in (1e-2, 1e-5):
        refs = orc.truncate(xs, orc.Ctl(eps=rel * orc.norm(xs)))
        Ts = htb.truncate(xd, htb.TruncationControl.relative_accuracy(rel))
        assert to_host(Ts).ranks == refs.ranks
        assert rel_err(to_host(Ts), refs) <= 1e-10
