"""BASELINE C4: parameter-dependent diffusion, CG with relative truncation after
every operation, on GpuBackend -- against the oracle's CG on the same operator
(small mesh), and the full 64 x 64 / 16^9 configuration end to end."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import htucker_oracle as orc
from tests.htconv import rel_err

pytestmark = pytest.mark.gpu


def _oracle_operator(op_host_matrices, grids):
    from paper_1708_03340_b200 import problems

    tr = orc.balanced_tree(10)
    op = problems.affine_operator(op_host_matrices, grids, device="cpu")
    W = {t: [orc.GMat(g.kind, g.data) for g in cols] for t, cols in op.leaves.items()}
    H = {t: b.numpy() for t, b in op.transfer.items()}
    return orc.HTOp(tr, W, H, op.root_matrix.numpy())


def test_cg_c4_small_matches_oracle(cuda_ok):
    from paper_1708_03340_b200 import problems
    from paper_1708_03340_b200.backend import GpuBackend
    from paper_1708_03340_b200.solvers import RelativeTruncation, SolverConfig, cg_solve

    mats, load = problems.p1_diffusion_matrices(cells=8)
    grids = problems.parameter_grids(points=4)
    matrices = [sp.csr_matrix(mats[0].shape)] + mats
    op = problems.affine_operator(matrices, grids)
    rhs = problems.constant_rhs(load, grids)
    cfg = SolverConfig(truncation=RelativeTruncation(1e-6, max_rank=20), eps_stop=1e-12, max_cg_steps=5)
    x, trace = cg_solve(op, rhs, cfg, backend=GpuBackend())

    oop = _oracle_operator(matrices, grids)
    tr = orc.balanced_tree(10)
    orhs = orc.HT(tr, *[{t: a for t, a in d.items()} for d in rhs.to_numpy()[:2]], rhs.to_numpy()[2])
    ox, internal, true = orc.cg_solve(oop, orhs, lambda y: orc.Ctl(eps=1e-6 * orc.norm(y), max_rank=20), 1e-12, 5)
    got = [e.internal_residual for e in trace.entries]
    # the first steps agree to the truncation gate; later steps drift by ~1e-7 because
    # every truncation of this parameter-symmetric problem cuts through (near-)degenerate
    # singular values at the rank cap, and CG amplifies the O(1e-15) differences
    np.testing.assert_allclose(got[:2], internal[:2], rtol=1e-10)
    np.testing.assert_allclose(got, internal, rtol=1e-6)
    np.testing.assert_allclose([e.true_rel_residual for e in trace.entries], true, rtol=1e-6)
    leaves, transfer, root = x.to_numpy()
    assert rel_err(orc.HT(tr, leaves, transfer, root), ox) <= 1e-5


@pytest.mark.slow
def test_cg_c4_full_size_matches_reference_trace(cuda_ok):
    """64 x 64 P1 mesh (3969 unknowns), 9 parameters x 16 values (d = 10), 20 CG
    steps with relative truncation 1e-6 (cap 50) -- against the trace of the
    REFERENCE's own cg_solve on the same problem (tests/golden/c4_cg.npz,
    make_golden.py --c4).  Pre-truncation ranks reach 500, so every wide-rank
    kernel (K > 112 QR / eigensolver paths) runs.

    Tolerances: the first three steps (rank cap not yet binding) agree to 1e-10.
    From step 3 on every truncation cuts through (near-)degenerate singular values
    at the cap -- the parameter symmetry of the problem makes them exactly
    degenerate -- so the kept subspace is not unique and CG amplifies the O(eps)
    differences: the reference and the oracle (both LAPACK) already drift 1e-5 apart
    by step 20; the B200 path stays within 1e-2 over the whole trace, with the
    same maximal rank at every step."""
    import os

    from paper_1708_03340_b200 import problems
    from paper_1708_03340_b200.backend import GpuBackend
    from paper_1708_03340_b200.solvers import RelativeTruncation, SolverConfig, cg_solve

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c4_cg.npz"))
    mats, load = problems.p1_diffusion_matrices(cells=64)
    grids = problems.parameter_grids(points=16)
    op = problems.affine_operator([sp.csr_matrix(mats[0].shape)] + mats, grids)
    rhs = problems.constant_rhs(load, grids)
    cfg = SolverConfig(truncation=RelativeTruncation(1e-6, max_rank=50), eps_stop=1e-12, max_cg_steps=20)
    x, trace = cg_solve(op, rhs, cfg, backend=GpuBackend())
    true = np.array([e.true_rel_residual for e in trace.entries])
    internal = np.array([e.internal_residual for e in trace.entries])
    assert trace.aborted is None and len(true) == 21
    np.testing.assert_allclose(true[:3], g["true_rel"][:3], rtol=1e-10)
    np.testing.assert_allclose(internal[:3], g["internal"][:3], rtol=1e-10)
    np.testing.assert_allclose(true, g["true_rel"], rtol=1e-2)
    np.testing.assert_allclose(internal, g["internal"], rtol=1e-2)
    assert [e.max_rank for e in trace.entries] == list(g["max_rank"])
    # the final iterate has drifted by ~1e-3: its eps-chosen ranks may move by one
    assert np.abs(np.array([x.rank(t) for t in range(1, 19)]) - g["ranks_X"]).max() <= 1


@pytest.mark.slow
def test_cg_c4_distinct_grids_holds_parity_for_20_steps(cuda_ok):
    """C4 with the parameter symmetry broken (every parameter on its own grid, see
    problems.distinct_parameter_grids): the kept singular subspaces at the rank cap are
    unique, so the 20-step CG trace must follow the REFERENCE's own cg_solve
    (tests/golden/c4_cg_distinct.npz, make_golden.py --c4) with identical maximal and
    final ranks, and the CG iteration's own residual norms to rtol 1e-10 at every step
    (measured: 4e-12).

    The "true" residual ||T(A X) - B|| / ||B|| is gated at 1e-8 instead (measured: up to
    9e-9 at step 20 under every QR / eigensolver policy): T truncates A X (ranks up to
    500) at eps = 1e-6 ||A X||, where the cut singular values sit near 1e-7 sigma_max,
    i.e. lambda_cut ~ 1e-14 lambda_max in the Gramians -- the fp64 Gram route fixes the
    eigenvectors there only to ~eps lambda_max / lambda_cut, so T(A X) itself is
    determined to ~sigma_cut * 1e-2 ~ 1e-9 by ANY implementation that forms the
    Gramians in fp64.  The oracle port (the reference's own numpy calls in the same
    order) tracks it to 2e-11 only because it repeats the reference's rounding."""
    import os

    from paper_1708_03340_b200 import problems
    from paper_1708_03340_b200.backend import GpuBackend
    from paper_1708_03340_b200.solvers import RelativeTruncation, SolverConfig, cg_solve

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c4_cg_distinct.npz"))
    mats, load = problems.p1_diffusion_matrices(cells=64)
    grids = problems.distinct_parameter_grids(points=16)
    op = problems.affine_operator([sp.csr_matrix(mats[0].shape)] + mats, grids)
    rhs = problems.constant_rhs(load, grids)
    cfg = SolverConfig(truncation=RelativeTruncation(1e-6, max_rank=50), eps_stop=1e-12, max_cg_steps=20)
    x, trace = cg_solve(op, rhs, cfg, backend=GpuBackend())
    true = np.array([e.true_rel_residual for e in trace.entries])
    internal = np.array([e.internal_residual for e in trace.entries])
    assert trace.aborted is None and len(true) == len(g["true_rel"])
    np.testing.assert_allclose(internal, g["internal"], rtol=1e-10)
    np.testing.assert_allclose(true[:9], g["true_rel"][:9], rtol=1e-10)  # before the cut tightens
    np.testing.assert_allclose(true, g["true_rel"], rtol=1e-8)
    assert [e.max_rank for e in trace.entries] == list(g["max_rank"])
    assert [x.rank(t) for t in range(1, 19)] == list(g["ranks_X"])
