"""B200-native hierarchical Tucker (HT) arithmetic -- drop-in for ``htucker``.

Mirrors the public surface of the reference package (htucker/__init__.py:10-70)
for the north-star path: truncation by hierarchical SVD plus the add, inner
product and operator application that feed it.  All floating point work runs
in hand-written sm_100a kernels (``csrc/``) behind the C ABI in
``include/ht_b200.h``; there is no CPU fallback.
"""

from .arith import (
    TruncationControl,
    add,
    apply_operator,
    compute_bhat,
    evaluate_entries,
    evaluate_entry,
    gemm,
    get_eig_mode,
    get_qr_mode,
    hierarchical_singular_values,
    inner_product,
    inner_product_device,
    leaf_map,
    norm,
    orthogonalize,
    qr_fallback_count,
    scale,
    set_eig_mode,
    set_graph_mode,
    set_implicit_q,
    graph_stats,
    graph_relocations,
    synchronize,
    set_qr_mode,
    subtract,
    truncate,
)
from .format import (
    GeneralizedMatrix,
    HTensor,
    HTOperator,
    ParseError,
    deserialize,
    serialize,
    serialized_size,
    gaussian_factors,
    gaussian_htensor,
    identity_htoperator,
    random_htensor,
    storage_size,
)
from .tree import DimensionTree, build_balanced_tree, nodes_at_level

__all__ = [
    "DimensionTree",
    "GeneralizedMatrix",
    "HTensor",
    "HTOperator",
    "TruncationControl",
    "add",
    "apply_operator",
    "build_balanced_tree",
    "compute_bhat",
    "evaluate_entries",
    "evaluate_entry",
    "deserialize",
    "serialize",
    "serialized_size",
    "ParseError",
    "gaussian_factors",
    "gaussian_htensor",
    "gemm",
    "get_eig_mode",
    "get_qr_mode",
    "hierarchical_singular_values",
    "identity_htoperator",
    "inner_product",
    "inner_product_device",
    "leaf_map",
    "nodes_at_level",
    "norm",
    "orthogonalize",
    "random_htensor",
    "qr_fallback_count",
    "scale",
    "set_eig_mode",
    "set_graph_mode",
    "set_implicit_q",
    "graph_stats",
    "graph_relocations",
    "synchronize",
    "set_qr_mode",
    "storage_size",
    "subtract",
    "truncate",
]

__version__ = "0.1.0"
