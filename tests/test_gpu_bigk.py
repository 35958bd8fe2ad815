"""Ranks beyond the shared-memory kernels (K > 112 / 128): the tridiagonal
eigensolver with global scratch, blocked Cholesky-QR, wide QR (rank shrink)."""

import numpy as np
import pytest

from oracle import htucker_oracle as orc
from tests.htconv import rel_err, to_dev, to_host

pytestmark = pytest.mark.gpu


def test_truncate_orthogonal_input_k200(cuda_ok):
    """Orthogonal input (orth phase skipped): Gramians of size 200 go through the
    tridiagonal eigensolver's global-scratch path."""
    import paper_1708_03340_b200 as htb

    tr = orc.balanced_tree(4)
    a = orc.gaussian_htensor(tr, 400, 100, 21)
    c = orc.gaussian_htensor(tr, 400, 100, 22)
    x = orc.orthogonalize(orc.add(a, c))  # ranks 200, orthonormal frames (numpy)
    xd = to_dev(x)
    assert xd.orthogonal
    sig = htb.hierarchical_singular_values(xd)
    G = orc.reduced_gramians(x)
    for t, g in G.items():
        lam = np.linalg.eigvalsh(g)[::-1]
        got = sig[t].cpu().numpy() ** 2
        np.testing.assert_allclose(got, np.clip(lam, 0, None), rtol=0, atol=1e-12 * lam[0])
    T = htb.truncate(xd, htb.TruncationControl.fixed_rank(60))
    ref = orc.truncate(x, orc.Ctl(max_rank=60))
    assert to_host(T).ranks == ref.ranks
    assert rel_err(to_host(T), ref) <= 1e-10


def _sum4(tr, n, k, seeds):
    xs = [orc.gaussian_htensor(tr, n, k, s) for s in seeds]
    x = xs[0]
    for y in xs[1:]:
        x = orc.add(x, y)
    return xs, x


def test_c5_shaped_rank160(cuda_ok):
    """C5's structure at a size the oracle finishes: the sum of four rank-40 tensors
    (rank 160 > 128: blocked Cholesky-QR panels, global-scratch eigensolver) -> 40."""
    import paper_1708_03340_b200 as htb

    tr = orc.balanced_tree(8)
    xs, x = _sum4(tr, 512, 40, (0, 1, 2, 3))
    xd = to_dev(xs[0])
    for y in xs[1:]:
        xd = htb.add(xd, to_dev(y))
    assert xd.max_rank == 160
    o = to_host(htb.orthogonalize(xd))
    for t, u in o.U.items():
        np.testing.assert_allclose(u.T @ u, np.eye(u.shape[1]), atol=1e-13)
    T = htb.truncate(xd, htb.TruncationControl.fixed_rank(40))
    ref = orc.truncate(x, orc.Ctl(max_rank=40))
    assert to_host(T).ranks == ref.ranks
    assert rel_err(to_host(T), ref) <= 1e-10
    sig = htb.hierarchical_singular_values(xd)
    G = orc.reduced_gramians(orc.orthogonalize(x))
    for t, g in G.items():
        lam = np.clip(np.linalg.eigvalsh(g)[::-1], 0, None)
        np.testing.assert_allclose(sig[t].cpu().numpy() ** 2, lam, rtol=0, atol=1e-12 * lam[0])


def test_wide_leaves_rank_shrink(cuda_ok):
    """Short-wide leaf frames (n = 16 < K = 128, the C4 parameter-mode shape) and
    wide inner ranks (240): the sum of eight tensors, truncated to 30."""
    import paper_1708_03340_b200 as htb

    tr = orc.balanced_tree(4)
    n = [16, 200, 16, 200]
    k = {t: 30 for t in range(1, tr.n_nodes)}
    for mu in (1, 3):
        k[tr.leaf_of_dim(mu)] = 16
    xs = [orc.gaussian_htensor(tr, n, k, 40 + s) for s in range(8)]
    x = xs[0]
    xd = to_dev(xs[0])
    for y in xs[1:]:
        x = orc.add(x, y)
        xd = htb.add(xd, to_dev(y))
    T = htb.truncate(xd, htb.TruncationControl.fixed_rank(30))
    ref = orc.truncate(x, orc.Ctl(max_rank=30))
    assert to_host(T).ranks == ref.ranks
    assert rel_err(to_host(T), ref) <= 1e-10


def test_qr_wide_kernel_direct(cuda_ok):
    """ht orthogonalize on leaves with n = 16 and K = 200 (wide QR path)."""
    import paper_1708_03340_b200 as htb

    tr = orc.balanced_tree(2)
    rng = np.random.default_rng(5)
    U = {1: rng.standard_normal((16, 200)), 2: rng.standard_normal((300, 200))}
    root = rng.standard_normal((200, 200)) * 1e-2
    x = orc.HT(tr, U, {}, root)
    o = to_host(htb.orthogonalize(to_dev(x)))
    assert o.U[1].shape == (16, 16)
    np.testing.assert_allclose(o.U[1].T @ o.U[1], np.eye(16), atol=1e-13)
    np.testing.assert_allclose(o.U[2].T @ o.U[2], np.eye(200), atol=1e-13)
    ro = orc.orthogonalize(x)
    assert orc.orth_difference_norm(o, ro) <= 1e-12 * orc.norm(ro)


@pytest.mark.parametrize("k", [69, 75])
@pytest.mark.parametrize("mode", ["householder", "auto"])
def test_bigk_workspace_covers_unmerged_layouts(cuda_ok, k, mode):
    """K = 2k with K = 2 mod 4 (138, 150): node arrays whose byte size is not a multiple
    of 256 make the scratch allocator pad between nodes, so the per-level QR problems do
    not merge at run time -- the workspace query must cover the unmerged plan (it once
    sized the merged one and the Householder panels overran into the output)."""
    import paper_1708_03340_b200 as htb

    tr = orc.balanced_tree(4)
    a = orc.gaussian_htensor(tr, 300, k, 41)
    c = orc.gaussian_htensor(tr, 300, k, 42)
    x = orc.add(a, c)
    htb.set_qr_mode(mode)
    try:
        xd = to_dev(x)
        o = to_host(htb.orthogonalize(xd))
        ro = orc.orthogonalize(x)
        for (t, u), (_, v) in zip(o.arrays(), ro.arrays()):
            np.testing.assert_allclose(u, v, rtol=0, atol=1e-12 * max(1.0, np.abs(v).max()))
        T = htb.truncate(xd, htb.TruncationControl.fixed_rank(k))
        ref = orc.truncate(x, orc.Ctl(max_rank=k))
        assert rel_err(to_host(T), ref) <= 1e-10
    finally:
        htb.set_qr_mode("auto")
