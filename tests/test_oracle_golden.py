"""Pin the CPU oracle against fixtures produced by the reference itself
(tests/golden/make_golden.py) and against the SPEC's known answers.
No GPU needed."""

import numpy as np
import pytest

from oracle import htucker_oracle as orc
from tests.goldens import load, node_dict, unpack


def test_spec_known_answers():
    z = load("spec.npz")
    q, r = orc.qr_signfixed(np.array([[3.0], [4.0]]))
    np.testing.assert_allclose(q, [[0.6], [0.8]], rtol=0, atol=1e-15)
    np.testing.assert_allclose(r, [[5.0]], rtol=1e-15)
    np.testing.assert_array_equal(q, z["qr_q"])
    _, lam = orc.eig_desc(np.array([[2.0, 1.0], [1.0, 2.0]]))
    np.testing.assert_allclose(lam, [3.0, 1.0], rtol=1e-15)
    np.testing.assert_allclose(lam, z["eig_lam"], rtol=1e-15)
    t5 = orc.balanced_tree(5)
    assert [tuple(v) for v in z["tree5_intervals"]] == t5.interval
    assert t5.interval[1] == (1, 2) and t5.interval[2] == (3, 5)
    assert [(-1 if f is None else f) for f in t5.father] == list(z["tree5_fathers"])
    t10 = orc.balanced_tree(10)
    assert list(z["tree10_levels"]) == t10.level
    assert [tuple(v) for v in z["tree10_intervals"]] == t10.interval


def test_storage_known_answers():
    # d=8, n=1e4, k=100 -> 14 010 000; d=2, n=5, k=3 -> 39
    tr = orc.balanced_tree(8)
    count = 8 * 10000 * 100 + 6 * 100 ** 3 + 100 ** 2
    assert count == 14_010_000
    tr2 = orc.balanced_tree(2)
    x = orc.gaussian_htensor(tr2, 5, 3, 0)
    assert orc.storage(x) == 39


def test_non_symmetric_raises():
    with pytest.raises(ValueError):
        orc.eig_desc(np.array([[1.0, 2.0], [0.0, 1.0]]))
    with pytest.raises(ValueError):
        orc.Ctl()
    with pytest.raises(ValueError):
        orc.Ctl(eps=-1.0)


@pytest.mark.parametrize("case", range(40))
def test_small_sweep(case):
    z = load("small.npz")
    p = f"case{case}"
    d = int(z[f"{p}/d"])
    tr = orc.balanced_tree(d)
    a = unpack(z, f"{p}/A", tr)
    c = unpack(z, f"{p}/C", tr)
    x = orc.add(a, orc.scale(c, 0.5))
    # add is bit-exact; dense reconstruction and entries
    dense = orc.to_dense(x)
    np.testing.assert_allclose(dense, z[f"{p}/dense_X"], rtol=1e-13, atol=1e-14)
    n = [int(v) for v in z[f"{p}/n"]]
    np.testing.assert_allclose(orc.evaluate_entry(x, [0] * d), z[f"{p}/entry"][0], rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(orc.evaluate_entry(x, [v - 1 for v in n]), z[f"{p}/entry"][1],
                               rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(orc.inner_product(a, c), float(z[f"{p}/ip_AC"]), rtol=1e-12, atol=1e-13)
    # orthogonalised factors entrywise (unique with the sign fix)
    o = orc.orthogonalize(x)
    ro = unpack(z, f"{p}/Xorth", tr, orthogonal=True)
    for t, arr in o.arrays():
        ref_arr = dict(ro.arrays())[t]
        assert arr.shape == ref_arr.shape
    np.testing.assert_allclose(o.root, ro.root, rtol=1e-10, atol=1e-12)
    G = orc.reduced_gramians(o)
    for t, g in node_dict(z, f"{p}/bhat", tr).items():
        np.testing.assert_allclose(G[t], g, rtol=1e-10, atol=1e-12)
    for t, lam in node_dict(z, f"{p}/lam", tr).items():
        np.testing.assert_allclose(orc.eig_desc(G[t])[1], lam, rtol=1e-9, atol=1e-12)
    eps = float(z[f"{p}/eps"])
    for tag, ctl in (("fix", orc.Ctl(max_rank=2)), ("eps", orc.Ctl(eps=eps)),
                     ("both", orc.Ctl(eps=eps, max_rank=1))):
        t_ = orc.truncate(x, ctl)
        assert [t_.rank(t) for t in range(1, 2 * d - 1)] == list(z[f"{p}/ranks_{tag}"])
        np.testing.assert_allclose(orc.norm(t_), float(z[f"{p}/normT_{tag}"]), rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(orc.orth_difference_norm(x, t_), float(z[f"{p}/err_{tag}"]),
                                   rtol=1e-8, atol=1e-12)


def test_rank_shrink():
    z = load("shrink.npz")
    tr = orc.balanced_tree(4)
    a, c = unpack(z, "A", tr), unpack(z, "C", tr)
    x = orc.add(a, c)
    assert [x.rank(t) for t in range(1, 7)] == list(z["ranks_X"])
    o = orc.orthogonalize(x)
    assert [o.rank(t) for t in range(1, 7)] == list(z["ranks_Xorth"])
    ro = unpack(z, "Xorth", tr, orthogonal=True)
    np.testing.assert_allclose(o.root, ro.root, rtol=1e-12, atol=1e-13)
    G = orc.reduced_gramians(o)
    for t, lam in node_dict(z, "lam", tr).items():
        np.testing.assert_allclose(orc.eig_desc(G[t])[1], lam, rtol=1e-9, atol=1e-13)
    t_ = orc.truncate(x, orc.Ctl(max_rank=2))
    assert [t_.rank(t) for t in range(1, 7)] == list(z["ranks_T"])
    np.testing.assert_allclose(orc.orth_difference_norm(x, t_), float(z["err_T"]), rtol=1e-8)


def test_c1_against_reference():
    z = load("c1.npz")
    a, c, x = orc.c1_inputs()
    tr = a.tree
    ga, gc = unpack(z, "A", tr), unpack(z, "C", tr)
    for (t, u), (_, v) in zip(a.arrays(), ga.arrays()):
        np.testing.assert_array_equal(u, v)  # generator reproduces the fixture inputs bit for bit
    for (t, u), (_, v) in zip(c.arrays(), gc.arrays()):
        np.testing.assert_array_equal(u, v)
    o = orc.orthogonalize(x)
    ro = unpack(z, "Xorth", tr, orthogonal=True)
    for (t, u), (_, v) in zip(o.arrays(), ro.arrays()):
        np.testing.assert_allclose(u, v, rtol=0, atol=1e-13 * max(1.0, np.abs(v).max()))
    G = orc.reduced_gramians(o)
    for t, g in node_dict(z, "bhat", tr).items():
        np.testing.assert_allclose(G[t], g, rtol=0, atol=1e-13 * np.abs(g).max())
    sig = orc.hierarchical_singular_values(x)
    for t, lam in node_dict(z, "lam", tr).items():
        np.testing.assert_allclose(sig[t], np.sqrt(lam), rtol=1e-10)  # all 20 per node
    t_ = orc.truncate(x, orc.Ctl(max_rank=10))
    assert [t_.rank(t) for t in range(1, 15)] == list(z["ranks_T"])
    rt = unpack(z, "T", tr)
    assert orc.orth_difference_norm(t_, rt) / float(z["norm_X"]) <= 1e-10
    np.testing.assert_allclose(orc.norm(x), float(z["norm_X"]), rtol=1e-12)
    np.testing.assert_allclose(orc.inner_product(t_, t_), float(z["ip_TT"]), rtol=1e-10)
    np.testing.assert_allclose(orc.orth_difference_norm(x, t_), float(z["trunc_err"]), rtol=1e-6)


def test_c3_small_operator():
    z = load("c3_small.npz")
    tr = orc.balanced_tree(4)
    x = unpack(z, "X", tr)
    op = orc.laplace_operator(tr, 6)
    y = orc.apply_operator(op, x)
    ry = unpack(z, "Y", tr)
    for (t, u), (_, v) in zip(y.arrays(), ry.arrays()):
        np.testing.assert_array_equal(u, v)
    # the operator really is the Laplace sum: dense check
    n, d = 6, 4
    lap = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    full = sum(np.kron(np.kron(np.kron(lap if m == 0 else np.eye(n), lap if m == 1 else np.eye(n)),
                               lap if m == 2 else np.eye(n)), lap if m == 3 else np.eye(n))
               for m in range(d))
    np.testing.assert_allclose(full, z["dense_op"], atol=1e-14)
    np.testing.assert_allclose(orc.to_dense(y).ravel(), full @ orc.to_dense(x).ravel(), rtol=1e-12, atol=1e-12)
    ny = orc.norm(y)
    np.testing.assert_allclose(ny, float(z["norm_Y"]), rtol=1e-12)
    t_ = orc.truncate(y, orc.Ctl(eps=1e-8 * ny, max_rank=3))
    assert [t_.rank(t) for t in range(1, 7)] == list(z["ranks_T"])
    np.testing.assert_allclose(orc.orth_difference_norm(y, t_), float(z["err_T"]), rtol=1e-6)


def test_c2_d8_sigmas():
    z = load("c2_d8.npz")
    a, c, x = orc.c2_inputs(8)
    sig = orc.hierarchical_singular_values(x)
    for t, lam in node_dict(z, "lam", x.tree).items():
        np.testing.assert_allclose(sig[t], np.sqrt(lam), rtol=1e-10)
    t_ = orc.truncate(x, orc.Ctl(max_rank=50))
    assert [t_.rank(t) for t in range(1, 15)] == list(z["ranks_T"])
    np.testing.assert_allclose(orc.inner_product(t_, t_), float(z["ip_TT"]), rtol=1e-10)


def test_c2_d64_sigmas():
    """The headline config (d=64): the oracle's sigmas, ranks and <T,T> against the
    reference-generated fixture (the GPU parity tests compare against both)."""
    z = load("c2_d64.npz")
    a, c, x = orc.c2_inputs(64)
    sig = orc.hierarchical_singular_values(x)
    lam = node_dict(z, "lam", x.tree)
    assert len(lam) == 126
    for t, lt in lam.items():
        np.testing.assert_allclose(sig[t], np.sqrt(lt), rtol=1e-10)
    t_ = orc.truncate(x, orc.Ctl(max_rank=50))
    assert [t_.rank(t) for t in range(1, 127)] == list(z["ranks_T"])
    np.testing.assert_allclose(orc.inner_product(t_, t_), float(z["ip_TT"]), rtol=1e-10)
    np.testing.assert_allclose(orc.orth_difference_norm(x, t_), float(z["trunc_err"]), rtol=1e-8)


def test_oracle_cg_matches_reference_cg():
    """The oracle's CG (solvers.py:172-231 restated) against the reference's own
    cg_solve run in the build container (tests/golden/cg.npz)."""
    z = load("cg.npz")
    tr = orc.balanced_tree(4)
    x, internal, true = orc.cg_solve(orc.laplace_operator(tr, 16), orc.ones_htensor(tr, 16),
                                     orc.Ctl(eps=1e-7, max_rank=6), 1e-10, 8)
    np.testing.assert_allclose(internal, z["internal"], rtol=1e-12)
    np.testing.assert_allclose(true, z["true_rel"], rtol=1e-12)
    assert [x.rank(t) for t in range(1, 7)] == list(z["ranks_X"])
    ref = unpack(z, "Xcg", tr)
    assert orc.orth_difference_norm(x, ref) <= 1e-12 * orc.norm(ref)


def test_readouts_against_reference():
    """Oracle extract_solution / parameter_mean vs the reference's cookie.py:383-426
    on the fixture tensor (d=10, nine 16-point parameter modes, spatial mode last)."""
    from tests.goldens import load, unpack

    z = load("readouts.npz")
    tree = orc.balanced_tree(10)
    x = unpack(z, "X", tree)
    gen = orc.gaussian_htensor(tree, [16] * 9 + [40], 6, seed=31)
    for t in range(1, tree.n_nodes):
        np.testing.assert_array_equal(x.rank(t), gen.rank(t))
    for q, idx in enumerate(z["idx"]):
        np.testing.assert_allclose(orc.extract_solution(x, idx), z[f"sol/{q}"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(orc.parameter_mean(x), z["mean"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(orc.parameter_mean(x, list(z["weights"])), z["wmean"], rtol=1e-13, atol=0)
    with pytest.raises(ValueError):
        orc.extract_solution(x, (0,) * 8)
    with pytest.raises(IndexError):
        orc.extract_solution(x, (0,) * 8 + (16,))
    with pytest.raises(ValueError):
        orc.parameter_mean(x, [np.ones(15)] * 9)
