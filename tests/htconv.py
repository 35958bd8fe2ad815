"""Conversions between oracle HT (numpy) and the device HTensor (test helpers)."""

import numpy as np

from oracle import htucker_oracle as orc


def to_dev(x: "orc.HT", orthogonal=None):
    import paper_1708_03340_b200 as htb

    tree = htb.build_balanced_tree(x.tree.d)
    return htb.HTensor(tree, dict(x.U), dict(x.B), x.root, orthogonal=x.orthogonal if orthogonal is None else orthogonal)


def to_host(y) -> "orc.HT":
    leaves, transfer, root = y.to_numpy()
    tr = orc.balanced_tree(y.tree.d)
    return orc.HT(tr, {t: np.array(v) for t, v in leaves.items()}, {t: np.array(v) for t, v in transfer.items()},
                  np.array(root), y.orthogonal)


def rel_err(x_gpu: "orc.HT", x_ref: "orc.HT") -> float:
    """||X_gpu - X_ref|| / ||X_ref|| through the orthogonalised difference."""
    return orc.orth_difference_norm(x_gpu, x_ref) / max(orc.norm(x_ref), 1e-300)
