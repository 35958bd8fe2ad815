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
