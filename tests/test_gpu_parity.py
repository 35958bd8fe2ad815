"""Tree-level parity of the CUDA path with the CPU oracle and the reference's
golden fixtures (north-star gates: hierarchical singular values rtol 1e-10,
||X_gpu - X_ref|| / ||X_ref|| <= 1e-10 via the orthogonalised difference,
identical truncated ranks)."""

import numpy as np
import pytest

from oracle import htucker_oracle as orc
from tests.goldens import load, node_dict, unpack
from tests.htconv import rel_err, to_dev, to_host

pytestmark = pytest.mark.gpu

SIGMA_RTOL = 1e-10
ERR_TOL = 1e-10


@pytest.fixture(scope="module", params=[("auto", "auto", True), ("auto", "auto", False), ("cholqr2", "auto", True),
                                        ("householder", "jacobi", True)],
                ids=["fast", "explicit_q", "cholqr2", "fallback"])
def htb(cuda_ok, request):
    """Every parity test runs under each kernel policy: the fast paths (Cholesky-QR with
    implicit Q, tridiagonal eigensolver; default), the same with Q formed explicitly, both
    Cholesky-QR passes, and the fallbacks (Householder QR, Jacobi)."""
    import paper_1708_03340_b200 as m

    m.set_qr_mode(request.param[0])
    m.set_eig_mode(request.param[1])
    m.set_implicit_q(request.param[2])
    yield m
    m.set_qr_mode("auto")
    m.set_eig_mode("auto")
    m.set_implicit_q(True)


def _sig_host(sig):
    return {t: v.cpu().numpy() for t, v in sig.items()}


def test_c1_orthogonalize_entrywise(htb):
    z = load("c1.npz")
    _, _, x = orc.c1_inputs()
    o = to_host(htb.orthogonalize(to_dev(x)))
    ro = unpack(z, "Xorth", x.tree, orthogonal=True)
    assert o.orthogonal
    for (t, u), (_, v) in zip(o.arrays(), ro.arrays()):
        assert u.shape == v.shape
        # unique sign-fixed Householder factors: fp64 agreement to ~1e-13
        np.testing.assert_allclose(u, v, rtol=0, atol=1e-12 * max(1.0, np.abs(v).max()))


def test_c1_gramians_entrywise(htb):
    z = load("c1.npz")
    _, _, x = orc.c1_inputs()
    o = htb.orthogonalize(to_dev(x))
    G = htb.compute_bhat(o)
    for t, g in node_dict(z, "bhat", x.tree).items():
        np.testing.assert_allclose(G[t].cpu().numpy(), g, rtol=0, atol=1e-12 * np.abs(g).max())


def test_c1_truncate_gates(htb):
    z = load("c1.npz")
    _, _, x = orc.c1_inputs()
    xd = to_dev(x)
    sig = _sig_host(htb.hierarchical_singular_values(xd))
    for t, lam in node_dict(z, "lam", x.tree).items():
        np.testing.assert_allclose(sig[t], np.sqrt(lam), rtol=SIGMA_RTOL)  # all 20 per node
    T = htb.truncate(xd, htb.TruncationControl.fixed_rank(10))
    assert [T.rank(t) for t in range(1, 15)] == list(z["ranks_T"])
    Th = to_host(T)
    assert rel_err(Th, unpack(z, "T", x.tree)) <= ERR_TOL
    np.testing.assert_allclose(htb.inner_product(T, T), float(z["ip_TT"]), rtol=1e-10)
    np.testing.assert_allclose(htb.norm(xd), float(z["norm_X"]), rtol=1e-10)


def test_add_bitwise_and_scale(htb):
    a, c, x = orc.c1_inputs()
    xd = htb.add(htb.scale(to_dev(a), 2.0), htb.scale(to_dev(c), 1e-10))
    xh = to_host(xd)
    for (t, u), (_, v) in zip(xh.arrays(), x.arrays()):
        np.testing.assert_array_equal(u, v)  # add is bit-exact (no FLOPs, Lemma 3)
    s = to_host(htb.subtract(to_dev(a), to_dev(c)))
    for (t, u), (_, v) in zip(s.arrays(), orc.subtract(a, c).arrays()):
        np.testing.assert_array_equal(u, v)


@pytest.mark.parametrize("case", range(40))
def test_small_sweep_against_reference(htb, case):
    z = load("small.npz")
    p = f"case{case}"
    d = int(z[f"{p}/d"])
    tr = orc.balanced_tree(d)
    a, c = unpack(z, f"{p}/A", tr), unpack(z, f"{p}/C", tr)
    ad, cd = to_dev(a), to_dev(c)
    xd = htb.add(ad, htb.scale(cd, 0.5))
    x = orc.add(a, orc.scale(c, 0.5))
    np.testing.assert_allclose(htb.inner_product(ad, cd), float(z[f"{p}/ip_AC"]), rtol=1e-11, atol=1e-13)
    o = to_host(htb.orthogonalize(xd))
    ro = unpack(z, f"{p}/Xorth", tr, orthogonal=True)
    for (t, u), (_, v) in zip(o.arrays(), ro.arrays()):
        assert u.shape == v.shape
    np.testing.assert_allclose(o.root, ro.root, rtol=0, atol=1e-11 * max(1.0, np.abs(ro.root).max()))
    sig = _sig_host(htb.hierarchical_singular_values(xd))
    for t, lam in node_dict(z, f"{p}/lam", tr).items():
        # Rank-deficient nodes (add of random tensors with k_t > n) have exact-zero
        # eigenvalues that every Gram-based solver returns as round-off noise
        # (~eps * lambda_max): compare in lambda-space with that absolute floor.
        np.testing.assert_allclose(sig[t] ** 2, lam, rtol=1e-9, atol=64 * 2.2e-16 * lam[0])
        big = lam > 1e-4 * lam[0]
        np.testing.assert_allclose(sig[t][big], np.sqrt(lam[big]), rtol=1e-10)
    eps = float(z[f"{p}/eps"])
    for tag, ctl in (("fix", htb.TruncationControl.fixed_rank(2)), ("eps", htb.TruncationControl.accuracy(eps)),
                     ("both", htb.TruncationControl(eps=eps, max_rank=1))):
        T = htb.truncate(xd, ctl)
        assert [T.rank(t) for t in range(1, 2 * d - 1)] == list(z[f"{p}/ranks_{tag}"])
        np.testing.assert_allclose(htb.norm(T), float(z[f"{p}/normT_{tag}"]), rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(orc.orth_difference_norm(x, to_host(T)), float(z[f"{p}/err_{tag}"]),
                                   rtol=1e-6, atol=1e-12)


def test_rank_shrink(htb):
    z = load("shrink.npz")
    tr = orc.balanced_tree(4)
    x = orc.add(unpack(z, "A", tr), unpack(z, "C", tr))
    xd = to_dev(x)
    o = htb.orthogonalize(xd)
    assert [o.rank(t) for t in range(1, 7)] == list(z["ranks_Xorth"])
    oh = to_host(o)
    for t in range(1, 7):
        if tr.is_leaf(t):
            k = oh.U[t].shape[1]
            np.testing.assert_allclose(oh.U[t].T @ oh.U[t], np.eye(k), atol=1e-13)
    T = htb.truncate(xd, htb.TruncationControl.fixed_rank(2))
    assert [T.rank(t) for t in range(1, 7)] == list(z["ranks_T"])
    np.testing.assert_allclose(orc.orth_difference_norm(x, to_host(T)), float(z["err_T"]), rtol=1e-6)


def test_rank_deficient_add_a_a(htb):
    # truncate(add(A, A)) == 2A; exercises exactly rank-deficient frames
    tr = orc.balanced_tree(8)
    a = orc.gaussian_htensor(tr, 64, 10, 5)
    ad = to_dev(a)
    n_fb = htb.qr_fallback_count()
    x2 = htb.add(ad, ad)
    T = htb.truncate(x2, htb.TruncationControl.fixed_rank(10))
    two_a = orc.scale(a, 2.0)
    assert rel_err(to_host(T), two_a) <= 1e-12
    o = to_host(htb.orthogonalize(x2))
    for t, u in o.U.items():  # frames stay orthonormal although [U, U] has rank k
        np.testing.assert_allclose(u.T @ u, np.eye(u.shape[1]), atol=1e-13)
    if htb.get_qr_mode() in ("auto", "cholqr2"):
        # the Cholesky-QR2 red flag must have fired (both sweeps re-run with Householder)
        assert htb.qr_fallback_count() == n_fb + 2


def test_c3_small_operator_then_truncate(htb):
    z = load("c3_small.npz")
    tr = orc.balanced_tree(4)
    x = unpack(z, "X", tr)
    op = orc.laplace_operator(tr, 6)
    ttr = htb.build_balanced_tree(4)
    dop = htb.HTOperator(ttr, {t: [htb.GeneralizedMatrix.diagonal(w[0].data), htb.GeneralizedMatrix.csr(w[1].data)]
                                for t, w in op.W.items()}, dict(op.H), op.root)
    y = htb.apply_operator(dop, to_dev(x))
    for (t, u), (_, v) in zip(to_host(y).arrays(), unpack(z, "Y", tr).arrays()):
        np.testing.assert_allclose(u, v, rtol=1e-15, atol=1e-15)
    ny = htb.norm(y)
    np.testing.assert_allclose(ny, float(z["norm_Y"]), rtol=1e-12)
    T = htb.truncate(y, htb.TruncationControl(eps=1e-8 * ny, max_rank=3))
    assert [T.rank(t) for t in range(1, 7)] == list(z["ranks_T"])
    np.testing.assert_allclose(orc.orth_difference_norm(orc.apply_operator(op, x), to_host(T)), float(z["err_T"]),
                               rtol=1e-6)


def test_dense_operator_leaves(htb):
    tr = orc.balanced_tree(3)
    rng = np.random.default_rng(2)
    x = orc.gaussian_htensor(tr, [4, 5, 6], 2, 3)
    W = {t: [orc.GMat("dense", rng.standard_normal((x.U[t].shape[0] + 1, x.U[t].shape[0]))) for _ in range(2)]
         for t in tr.leaves_by_dim()}
    H = {t: rng.standard_normal((2, 2, 2)) for t in tr.inner_ids()}
    op = orc.HTOp(tr, W, H, rng.standard_normal((2, 2)))
    ref = orc.apply_operator(op, x)
    ttr = htb.build_balanced_tree(3)
    dop = htb.HTOperator(ttr, {t: [htb.GeneralizedMatrix.dense(g.data) for g in w] for t, w in W.items()}, H, op.root)
    y = to_host(htb.apply_operator(dop, to_dev(x)))
    for (t, u), (_, v) in zip(y.arrays(), ref.arrays()):
        np.testing.assert_allclose(u, v, rtol=1e-13, atol=1e-13)


def test_c2_d8_against_reference(htb):
    z = load("c2_d8.npz")
    a, c, x = orc.c2_inputs(8)
    xd = htb.add(to_dev(a), to_dev(c))
    n_fb = htb.qr_fallback_count()
    sig = _sig_host(htb.hierarchical_singular_values(xd))
    for t, lam in node_dict(z, "lam", x.tree).items():
        np.testing.assert_allclose(sig[t], np.sqrt(lam), rtol=SIGMA_RTOL)
    T = htb.truncate(xd, htb.TruncationControl.fixed_rank(50))
    assert htb.qr_fallback_count() == n_fb  # well-conditioned: the Cholesky-QR2 path is kept
    assert [T.rank(t) for t in range(1, 15)] == list(z["ranks_T"])
    np.testing.assert_allclose(htb.inner_product(T, T), float(z["ip_TT"]), rtol=1e-10)
    t_ref = orc.truncate(x, orc.Ctl(max_rank=50))
    assert rel_err(to_host(T), t_ref) <= ERR_TOL


@pytest.mark.slow
def test_c2_d64_headline_shape(htb):
    """BASELINE config C2 at the headline size (d=64, n=1000, k=50 -> rank 100 -> 50)."""
    a, c, x = orc.c2_inputs(64)
    xd = htb.add(to_dev(a), to_dev(c))
    n_fb = htb.qr_fallback_count()
    T = htb.truncate(xd, htb.TruncationControl.fixed_rank(50))
    assert htb.qr_fallback_count() == n_fb
    assert all(T.rank(t) == 50 for t in range(1, 127))
    t_ref = orc.truncate(x, orc.Ctl(max_rank=50))
    assert rel_err(to_host(T), t_ref) <= ERR_TOL
    np.testing.assert_allclose(htb.inner_product(T, T), orc.inner_product(t_ref, t_ref), rtol=1e-10)


def test_c3_full_size(htb):
    """BASELINE config C3 at its full size: d=16, n=256, X rank 30 (Gaussian), the
    Laplace-sum operator (ranks 2) -> Y rank 60, truncated with eps = 1e-8 ||Y|| and
    cap 30 ("whichever comes first")."""
    tr = orc.balanced_tree(16)
    x = orc.gaussian_htensor(tr, 256, 30, 16)
    op = orc.laplace_operator(tr, 256)
    ttr = htb.build_balanced_tree(16)
    dop = htb.HTOperator(ttr, {t: [htb.GeneralizedMatrix.diagonal(w[0].data), htb.GeneralizedMatrix.csr(w[1].data)]
                                for t, w in op.W.items()}, dict(op.H), op.root)
    y = htb.apply_operator(dop, to_dev(x))
    assert y.max_rank == 60
    yr = orc.apply_operator(op, x)
    ny = htb.norm(y)
    np.testing.assert_allclose(ny, orc.norm(yr), rtol=1e-12)
    T = htb.truncate(y, htb.TruncationControl(eps=1e-8 * ny, max_rank=30))
    ref = orc.truncate(yr, orc.Ctl(eps=1e-8 * orc.norm(yr), max_rank=30))
    assert to_host(T).ranks == ref.ranks
    assert rel_err(to_host(T), ref) <= 1e-10
