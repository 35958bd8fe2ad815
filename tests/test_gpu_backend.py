"""The solver plugin seam (reference solvers.py:28-106): GpuBackend + the CG loop
(solvers.py:172-231) on the device against the reference's own CG run
(tests/golden/cg.npz)."""

import numpy as np
import pytest

from oracle import htucker_oracle as orc
from tests.goldens import load, unpack
from tests.htconv import rel_err, to_host

pytestmark = pytest.mark.gpu


class _HostHT:
    """Stand-in for the reference HTensor (duck-typed: tree.d, leaves, transfer, root_matrix)."""

    def __init__(self, tree, leaves, transfer, root):
        self.tree, self.leaves, self.transfer, self.root_matrix = tree, leaves, transfer, root


class _HostTree:
    def __init__(self, d):
        self.d = d


def _host_op(op):
    class Op:
        pass

    o = Op()
    o.tree = _HostTree(op.tree.d)
    o.leaves = {t: list(w) for t, w in op.W.items()}  # oracle GMat has kind/data like the reference
    o.transfer = dict(op.H)
    o.root_matrix = op.root
    return o


def test_cg_on_gpu_backend_matches_reference(cuda_ok):
    import paper_1708_03340_b200 as htb
    from paper_1708_03340_b200.backend import GpuBackend
    from paper_1708_03340_b200.solvers import SolverConfig, cg_solve

    z = load("cg.npz")
    tr = orc.balanced_tree(4)
    op = orc.laplace_operator(tr, 16)
    rhs = orc.ones_htensor(tr, 16)
    be = GpuBackend(host_factory=lambda tree, L, B, r: orc.HT(tr, L, B, r))
    cfg = SolverConfig(truncation=htb.TruncationControl(eps=1e-7, max_rank=6), eps_stop=1e-10, max_cg_steps=8)
    x, trace = cg_solve(_host_op(op), _HostHT(_HostTree(4), rhs.U, rhs.B, rhs.root), cfg, backend=be)
    np.testing.assert_allclose([e.internal_residual for e in trace.entries], z["internal"], rtol=1e-9)
    np.testing.assert_allclose([e.true_rel_residual for e in trace.entries], z["true_rel"], rtol=1e-9)
    assert [x.rank(t) for t in range(1, 7)] == list(z["ranks_X"])
    assert rel_err(x, unpack(z, "Xcg", tr)) <= 1e-9


def test_backend_methods(cuda_ok):
    import paper_1708_03340_b200 as htb
    from paper_1708_03340_b200.backend import GpuBackend

    tr = orc.balanced_tree(8)
    a = orc.gaussian_htensor(tr, 20, 4, 1)
    c = orc.gaussian_htensor(tr, 20, 3, 2)
    be = GpuBackend()
    ad = be.lift(_HostHT(_HostTree(8), a.U, a.B, a.root))
    cd = be.lift(_HostHT(_HostTree(8), c.U, c.B, c.root))
    for got, ref in ((to_host(be.add(ad, cd)), orc.add(a, c)), (to_host(be.scale(ad, -3.0)), orc.scale(a, -3.0))):
        for (_, u), (_, v) in zip(got.arrays(), ref.arrays()):
            assert np.array_equal(u, v)  # structural ops are bit-exact
    np.testing.assert_allclose(be.inner_product(ad, cd), orc.inner_product(a, c), rtol=1e-12)
    np.testing.assert_allclose(be.norm(ad), orc.norm(a), rtol=1e-12)
    assert be.max_rank(be.add(ad, cd)) == 7
    M = np.random.default_rng(0).standard_normal((20, 20))
    lm = to_host(be.leaf_map(ad, 3, M))
    leaf = tr.leaf_of_dim(3)
    np.testing.assert_allclose(lm.U[leaf], M @ a.U[leaf], rtol=1e-13, atol=1e-13)
    t = be.truncate(be.add(ad, cd), htb.TruncationControl.fixed_rank(3))
    assert rel_err(to_host(t), orc.truncate(orc.add(a, c), orc.Ctl(max_rank=3))) <= 1e-10
