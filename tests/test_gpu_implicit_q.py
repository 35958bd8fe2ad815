"""Implicit-Q truncation (driver.cu OrthPlan::imp): the Cholesky-QR sweep keeps the
absorbed transfer tensors and R^-1 instead of forming Q, and the Gramian / projection
phases fold R^-1 into their small operands.  These cases force each branch of that
scheme -- one Cholesky-QR pass (R^-1 kept), the second pass (explicit Q, R^-1 := I),
the Householder re-run (explicit Q everywhere) -- and check the north-star gates
against the oracle (reference arith.py:325-352) and the explicit-Q path."""

import numpy as np
import pytest

from oracle import htucker_oracle as orc
from tests.htconv import rel_err, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def htb(cuda_ok):
    import paper_1708_03340_b200 as m

    yield m
    m.set_implicit_q(True)
    m.set_qr_mode("auto")


def _graded(d, n, k, decades, seed):
    """Gaussian HT tensor whose transfer tensors have slice i scaled by
    10^(-decades * i / (k - 1)): M23(B_t) then has condition ~10^decades, which sets how
    the Cholesky-QR sweep treats node t (one pass / second pass / Householder)."""
    tr = orc.balanced_tree(d)
    x = orc.gaussian_htensor(tr, n, k, seed)
    for t, b in x.B.items():
        kt = b.shape[0]
        if kt > 1:
            x.B[t] = b * (10.0 ** (-decades * np.arange(kt) / (kt - 1)))[:, None, None]
    return x


def _truncate_both(htb, xd, ctl):
    out = {}
    for imp in (True, False):
        htb.set_implicit_q(imp)
        out[imp] = htb.truncate(xd, ctl)
    htb.set_implicit_q(True)
    return out


def _near_copy(x, delta, seed):
    """x with every factor perturbed by delta * N(0,1): add(x, near_copy) has frames of
    condition ~1/delta (near-collinear columns, which Cholesky-QR cannot scale away)."""
    rng = np.random.default_rng(seed)
    y = orc.HT(x.tree, {t: u + delta * rng.standard_normal(u.shape) for t, u in x.U.items()},
               {t: b + delta * rng.standard_normal(b.shape) for t, b in x.B.items()},
               x.root + delta * rng.standard_normal(x.root.shape))
    return y


@pytest.mark.parametrize("decades,fallback", [(0.0, False), (3.5, False), (None, True)],
                         ids=["one_pass", "second_pass", "householder"])
def test_implicit_q_branches(htb, decades, fallback):
    d, n, k = 8, 120, 12
    if decades is None:  # near-rank-deficient sum: the Cholesky-QR red flag fires
        a = orc.gaussian_htensor(orc.balanced_tree(d), n, k, 3)
        c = _near_copy(a, 1e-9, 4)
    else:  # column-graded transfer tensors: kappa(R) ~ 10^decades (second pass above 300)
        a = _graded(d, n, k, decades, 3)
        c = _graded(d, n, k, decades, 4)
    x = orc.add(a, c)
    xd = htb.add(to_dev(a), to_dev(c))
    n_fb = htb.qr_fallback_count()
    ctl = htb.TruncationControl.fixed_rank(k)
    T = _truncate_both(htb, xd, ctl)
    assert (htb.qr_fallback_count() > n_fb) == fallback
    t_ref = orc.truncate(x, orc.Ctl(max_rank=k))
    for imp, t in T.items():
        assert [t.rank(s) for s in range(1, 2 * d - 1)] == [t_ref.rank(s) for s in range(1, 2 * d - 1)]
        assert rel_err(to_host(t), t_ref) <= 1e-10, imp
    # implicit and explicit agree far below the gate
    assert orc.orth_difference_norm(to_host(T[True]), to_host(T[False])) <= 1e-12 * orc.norm(t_ref)


def test_implicit_q_accuracy_mode_and_sigma(htb):
    d, n, k = 16, 64, 10
    a = _graded(d, n, k, 3.0, 7)
    c = _graded(d, n, k, 0.0, 8)
    x = orc.add(a, orc.scale(c, 1e-3))
    xd = htb.add(to_dev(a), htb.scale(to_dev(c), 1e-3))
    sig = {t: v.cpu().numpy() for t, v in htb.hierarchical_singular_values(xd).items()}
    ref = orc.hierarchical_singular_values(x)
    for t in ref:
        # Gram-route floor: lambda to ~eps * lambda_max absolutely;
        # sigma to rtol 1e-10 where lambda is well above that floor
        lam, lam_ref = sig[t] ** 2, ref[t] ** 2
        np.testing.assert_allclose(lam, lam_ref, rtol=1e-9, atol=64 * 2.2e-16 * lam_ref[0])
        big = lam_ref > 1e-4 * lam_ref[0]
        np.testing.assert_allclose(sig[t][big], ref[t][big], rtol=1e-10)
    eps = 1e-4 * orc.norm(x)
    T = htb.truncate(xd, htb.TruncationControl.accuracy(eps))
    t_ref = orc.truncate(x, orc.Ctl(eps=eps))
    assert [T.rank(s) for s in range(1, 2 * d - 1)] == [t_ref.rank(s) for s in range(1, 2 * d - 1)]
    assert rel_err(to_host(T), t_ref) <= 1e-10


def test_implicit_q_graph_replay_matches_eager(htb):
    """The captured truncation (graph replay) and the eager launches give identical bits."""
    a, c, x = orc.c2_inputs(8, 200, 20)
    xd = htb.add(to_dev(a), to_dev(c))
    ctl = htb.TruncationControl.fixed_rank(20)
    htb.set_graph_mode(False)
    ref = to_host(htb.truncate(xd, ctl))
    htb.set_graph_mode(True)
    outs = [to_host(htb.truncate(xd, ctl)) for _ in range(3)]
    for o in outs:
        for (t, u), (_, v) in zip(o.arrays(), ref.arrays()):
            np.testing.assert_array_equal(u, v)
