"""Parameter-direction readouts on the device: problems.extract_solution
and problems.parameter_mean through ht_evaluate_weighted, against the oracle and the
reference-generated fixture (reference cookie.py:362-426)."""

import numpy as np
import pytest

from oracle import htucker_oracle as orc
from tests.goldens import load, unpack

pytestmark = pytest.mark.gpu

TOL = 1e-12  # fp64: reassociated sums (entry-wise upward passes vs the reference's matrix pass)


def _device(htb, x):
    tree = htb.build_balanced_tree(x.tree.d)
    return htb.HTensor(tree, x.U, x.B, x.root)


def _close(got, want):
    got = got.cpu().numpy()
    assert got.shape == want.shape
    assert np.abs(got - want).max() <= TOL * np.abs(want).max()


def test_readouts_match_reference_fixture(cuda_ok):
    import paper_1708_03340_b200 as htb
    from paper_1708_03340_b200 import problems

    z = load("readouts.npz")
    x = unpack(z, "X", orc.balanced_tree(10))
    xd = _device(htb, x)
    for q, idx in enumerate(z["idx"]):
        _close(problems.extract_solution(xd, idx), z[f"sol/{q}"])
    _close(problems.parameter_mean(xd), z["mean"])
    _close(problems.parameter_mean(xd, list(z["weights"])), z["wmean"])
    # reference error behaviour (cookie.py:393-400, 418-420)
    with pytest.raises(ValueError):
        problems.extract_solution(xd, (0,) * 8)
    with pytest.raises(IndexError):
        problems.extract_solution(xd, (0,) * 8 + (16,))
    with pytest.raises(ValueError):
        problems.parameter_mean(xd, [np.ones(15)] * 9)


@pytest.mark.parametrize("n_sp,k", [(3969, 30), (1, 1), (257, 50)])
def test_readouts_match_oracle(cuda_ok, n_sp, k):
    """Full C4 spatial size, a one-point / rank-1 edge case, and a rank-50 tensor;
    weights supplied as device tensors; one-hot weights reproduce extract_solution
    (the reference's own identity, cookie.py:410-412)."""
    import torch

    import paper_1708_03340_b200 as htb
    from paper_1708_03340_b200 import problems

    tree = orc.balanced_tree(10)
    sizes = [16] * 9 + [n_sp]
    ranks = {t: (min(k, sizes[tree.interval[t][0] - 1]) if tree.is_leaf(t) else k) for t in range(1, tree.n_nodes)}
    x = orc.gaussian_htensor(tree, sizes, ranks, seed=3 + k)
    xd = _device(htb, x)
    idx = tuple(range(9))
    _close(problems.extract_solution(xd, idx), orc.extract_solution(x, idx))
    rng = np.random.default_rng(k)
    ws = [rng.random(16) for _ in range(9)]
    _close(problems.parameter_mean(xd, [torch.as_tensor(w, device="cuda") for w in ws]),
           orc.parameter_mean(x, ws))
    onehot = [np.eye(16)[i] for i in idx]
    _close(problems.parameter_mean(xd, onehot), orc.extract_solution(x, idx))
