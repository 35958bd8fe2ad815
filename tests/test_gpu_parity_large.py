"""North-star parity gates at the BASELINE configs' full sizes, against fixtures
produced by running the REFERENCE (tests/golden/make_golden.py --large):

* every hierarchical singular value to rtol 1e-10 (sigma = sqrt(lambda(B_hat)),
  reference kernels.py:35-54 on compute_bhat(orthogonalize(X)), arith.py:273-322);
* ||T_gpu - T_ref|| / ||T_ref|| <= 1e-10 through the orthogonalised difference
  (T_ref from the oracle port on the same host arrays; the oracle itself is pinned
  to the same fixtures by tests/test_oracle_golden.py);
* identical truncated ranks, <T,T> and ||X|| against the reference's values.

C2 at d = 64 (the headline), 128 and 256 (n=1000, rank 100 -> 50), and a C5-shaped
d = 8 subtree at the stress test's real node sizes (n = 2048, the 4-way sum of
rank-100 tensors: 2048 x 400 frames, 400^3 transfer tensors, 400 x 400 Gramians).
"""

import numpy as np
import pytest

from oracle import htucker_oracle as orc
from tests.goldens import load, node_dict
from tests.htconv import rel_err, to_dev, to_host

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SIGMA_RTOL = 1e-10
ERR_TOL = 1e-10


@pytest.fixture(scope="module")
def htb(cuda_ok):
    import paper_1708_03340_b200 as m

    m.set_qr_mode("auto")
    m.set_eig_mode("auto")
    return m


def sigma_tolerance(ref: np.ndarray) -> np.ndarray:
    """rtol 1e-10 per sigma, floored by the Gram route's conditioning.

    The reference forms B_hat in fp64 and takes sigma^2 = lambda(B_hat) (arith.py:299-322,
    kernels.py:51): B_hat's entries carry rounding of order eps * lambda_max, so any
    implementation that forms B_hat -- the reference's own LAPACK run included -- fixes
    sigma_i only to a relative eps/2 * (sigma_max / sigma_i)^2 (the accuracy loss the
    paper flags).  Below sigma_max / ~1000 that floor exceeds 1e-10;
    the floor used is 4 eps (sigma_max / sigma_i)^2 (8x the first-order bound)."""
    eps = np.finfo(np.float64).eps
    return np.maximum(SIGMA_RTOL, 4.0 * eps * (ref.max() / ref) ** 2)


def _check(htb, z, xd, x_host, k, tree):
    sig = htb.hierarchical_singular_values(xd)
    lam = node_dict(z, "lam", tree)
    assert len(lam) == tree.n_nodes - 1
    worst = 0.0
    floored = 0
    for t, lt in lam.items():
        ref = np.sqrt(lt)
        got = sig[t].cpu().numpy()
        assert got.shape == ref.shape
        rel = np.abs(got - ref) / ref
        tol = sigma_tolerance(ref)
        floored += int(np.sum(tol > SIGMA_RTOL))
        worst = max(worst, float(np.max(rel)))
        bad = np.nonzero(rel > tol)[0]
        assert bad.size == 0, f"node {t}: sigma {bad[:5]} rel err {rel[bad[:5]]} > tol {tol[bad[:5]]}"
    print(f"  sigmas below the 1e-10-attainable range (floored tolerance): {floored}")
    n_fb = htb.qr_fallback_count()
    T = htb.truncate(xd, htb.TruncationControl.fixed_rank(k))
    assert [T.rank(t) for t in range(1, tree.n_nodes)] == list(z["ranks_T"])
    np.testing.assert_allclose(htb.inner_product(T, T), float(z["ip_TT"]), rtol=1e-10)
    np.testing.assert_allclose(htb.norm(xd), float(z["norm_X"]), rtol=1e-10)
    t_ref = orc.truncate(x_host, orc.Ctl(max_rank=k))
    Th = to_host(T)
    assert Th.ranks == t_ref.ranks
    err = rel_err(Th, t_ref)
    assert err <= ERR_TOL
    # the truncation error itself (a gauge-invariant scalar the reference reported)
    e_gpu = orc.orth_difference_norm(Th, x_host)
    np.testing.assert_allclose(e_gpu, float(z["trunc_err"]), rtol=1e-6)
    return worst, err, htb.qr_fallback_count() - n_fb


@pytest.mark.parametrize("d", [64, 128, 256])
def test_c2_full_size_gates(htb, d):
    z = load(f"c2_d{d}.npz")
    a, c, x = orc.c2_inputs(d)
    xd = htb.add(to_dev(a), to_dev(c))
    worst, err, fb = _check(htb, z, xd, x, 50, x.tree)
    assert fb == 0  # well-conditioned: the Cholesky-QR path is kept
    print(f"C2 d={d}: max sigma rel err {worst:.2e}, ||T_gpu - T_ref||/||T_ref|| {err:.2e}")


def test_c2_d64_householder_path(htb):
    """The headline config through the north star's own algorithm (Householder QR)."""
    z = load("c2_d64.npz")
    a, c, x = orc.c2_inputs(64)
    xd = htb.add(to_dev(a), to_dev(c))
    htb.set_qr_mode("householder")
    try:
        _check(htb, z, xd, x, 50, x.tree)
    finally:
        htb.set_qr_mode("auto")


def test_c5_shaped_subtree_k400(htb):
    """C5 node sizes: d=8, n=2048, X = ((A0 + A1) + A2) + A3 (rank 400) -> rank 100.
    Drives the K > 128 block Gram-Schmidt orthogonalisation on 160000 x 400 frames and
    the global-scratch eigensolver at K = 400."""
    z = load("c5_d8.npz")
    xs = orc.c5_inputs(8)
    x = xs[0]
    for y in xs[1:]:
        x = orc.add(x, y)
    xd = to_dev(xs[0])
    for y in xs[1:]:
        xd = htb.add(xd, to_dev(y))
    assert xd.max_rank == 400
    worst, err, _ = _check(htb, z, xd, x, 100, x.tree)
    print(f"C5 shape: max sigma rel err {worst:.2e}, ||T_gpu - T_ref||/||T_ref|| {err:.2e}")


def test_graded_sigma_beyond_shared_memory_jacobi(htb):
    """Graded Gramians at K > 112 go to the global-scratch Jacobi when every sigma is asked
    for: the construction of C1 (X = 2A + 1e-10 C: the tiny block lives in the root) at
    rank 150.  The sigmas of the root's sons are checked against the host Jacobi on the
    device's own Gramians (relative accuracy of the eigensolver and the routing; the
    Gram-route error of forming B_hat is common to both sides)."""
    from tests.jacobi_host import jacobi_eigvals

    tr = htb.build_balanced_tree(4)
    a = htb.gaussian_htensor(tr, 300, 75, 41)
    c = htb.gaussian_htensor(tr, 300, 75, 42)
    xd = htb.add(htb.scale(a, 2.0), htb.scale(c, 1e-10))
    assert xd.max_rank == 150
    sig = htb.hierarchical_singular_values(xd)
    G = htb.compute_bhat(htb.orthogonalize(xd))
    for t in (1, 2):
        lam = jacobi_eigvals(G[t].cpu().numpy())
        s = np.sqrt(lam)
        assert s[-1] < 1e-8 * s[0]  # graded: a 1e-10-relative tail
        np.testing.assert_allclose(sig[t].cpu().numpy(), s, rtol=1e-9, err_msg=f"node {t}")
