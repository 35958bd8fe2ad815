"""BASELINE C4 problem setup (host side): the P1 subdomain matrices and the affine
HT operator, pinned against the reference's own operator builder
(cookie.build_ht_operator, tests/golden/c4_operator.npz)."""

import numpy as np
import scipy.sparse as sp

from tests.goldens import load


def test_p1_matrices_properties():
    from paper_1708_03340_b200 import problems

    mats, rhs = problems.p1_diffusion_matrices(cells=64)
    assert len(mats) == 9 and mats[0].shape == (3969, 3969)
    full = sum(mats)
    assert abs(full - full.T).max() < 1e-14  # symmetric
    # the sum over subdomains is the Laplacian: 5-point stencil on interior rows
    d = full.diagonal()
    assert np.allclose(d, 4.0)
    assert np.allclose(np.asarray(full.sum(axis=1)).ravel()[3969 // 2], 0.0)  # interior row sums vanish
    assert np.isclose(rhs.sum(), (1.0 - 2.0 / 64) ** 2, rtol=0.05)  # ~ area of the interior support
    assert np.linalg.eigvalsh(full[:200, :200].toarray()).min() > 0


def test_affine_operator_matches_reference_builder():
    from paper_1708_03340_b200 import problems

    z = load("c4_operator.npz")
    mats, rhs = problems.p1_diffusion_matrices(cells=6)
    for j, m in enumerate(mats):
        np.testing.assert_array_equal(m.toarray(), z[f"K/{j}"])
    np.testing.assert_allclose(rhs, z["load"], rtol=0, atol=0)
    grids = [np.linspace(0.1, 1.0, 4) for _ in range(9)]
    op = problems.affine_operator([sp.csr_matrix(mats[0].shape)] + mats, grids, device="cpu")
    assert np.array_equal(op.root_matrix.numpy(), z["root"])
    assert sorted(op.transfer) == sorted(int(k.split("/")[1]) for k in z.files if k.startswith("B/"))
    for t, b in op.transfer.items():
        np.testing.assert_array_equal(b.numpy(), z[f"B/{t}"])
    for t, cols in op.leaves.items():
        for j, g in enumerate(cols):
            np.testing.assert_array_equal(g.to_dense(), z[f"W/{t}/{j}/dense"])


def test_kron_sum_operator_equals_dense_kronecker_sum():
    """The generic builder on random dense factors: applying the HT operator to a random
    HT tensor equals applying the dense sum of Kronecker products (d=5, ragged tree)."""
    from oracle import htucker_oracle as orc
    from paper_1708_03340_b200 import problems
    from paper_1708_03340_b200.format import GeneralizedMatrix
    from paper_1708_03340_b200.tree import build_balanced_tree

    rng = np.random.default_rng(3)
    d, n = 5, [3, 2, 4, 3, 2]
    tree = build_balanced_tree(d)
    terms = [{1: "a", 4: "b"}, {2: "c"}, {3: "d", 5: "e", 1: "f"}, {}, {4: "g"}]
    mode_of = {"a": 1, "b": 4, "c": 2, "d": 3, "e": 5, "f": 1, "g": 4}
    factors = {k: GeneralizedMatrix.dense(rng.standard_normal((n[m - 1], n[m - 1]))) for k, m in mode_of.items()}
    sizes = {mu: n[mu - 1] for mu in range(1, d + 1)}
    op = problems.kron_sum_operator(tree, terms, factors, sizes, device="cpu")
    dense = np.zeros((int(np.prod(n)),) * 2)
    for term in terms:
        k = np.eye(1)
        for mu in range(1, d + 1):
            k = np.kron(k, factors[term[mu]].to_dense() if mu in term else np.eye(n[mu - 1]))
        dense += k
    otr = orc.balanced_tree(d)
    oop = orc.HTOp(otr, {t: [orc.GMat(g.kind, g.data) for g in cols] for t, cols in op.leaves.items()},
                   {t: b.numpy() for t, b in op.transfer.items()}, op.root_matrix.numpy())
    x = orc.gaussian_htensor(otr, n, 2, 9)
    y = orc.to_dense(orc.apply_operator(oop, x))
    np.testing.assert_allclose(y.ravel(), dense @ orc.to_dense(x).ravel(), rtol=1e-12, atol=1e-12)
    assert max(len(c) for c in op.leaves.values()) <= 3
