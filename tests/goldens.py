"""Helpers to unpack the reference-generated fixtures in tests/golden/."""

import os

import numpy as np

from oracle import htucker_oracle as orc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def unpack(z, prefix, tree, orthogonal=False):
    U, B, root = {}, {}, None
    for t in range(tree.n_nodes):
        arr = np.array(z[f"{prefix}/{t}"])
        if t == 0:
            root = arr
        elif tree.is_leaf(t):
            U[t] = arr
        else:
            B[t] = arr
    return orc.HT(tree, U, B, root, orthogonal)


def node_dict(z, prefix, tree):
    return {t: np.array(z[f"{prefix}/{t}"]) for t in range(1, tree.n_nodes) if f"{prefix}/{t}" in z}
