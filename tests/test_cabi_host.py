"""No-GPU checks: the C-ABI library loads and exports every symbol the header
declares; host-side tree / control logic mirrors the reference."""

import os
import re

import numpy as np
import pytest

from oracle import htucker_oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ht_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(ht_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    from paper_1708_03340_b200 import _lib

    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTS)
    assert b"sm_100a" in lib.ht_version()


def test_library_has_sm100a_cubin():
    import subprocess

    from paper_1708_03340_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_sass_uses_fp64_tensor_cores():
    import subprocess

    from paper_1708_03340_b200 import _lib

    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "DMMA" in sass


@pytest.mark.parametrize("d", [2, 3, 5, 8, 10, 17, 64, 256])
def test_tree_matches_oracle(d):
    from paper_1708_03340_b200 import build_balanced_tree

    t = build_balanced_tree(d)
    o = orc.balanced_tree(d)
    assert [n.interval for n in t.nodes] == o.interval
    assert [n.father for n in t.nodes] == o.father
    assert [n.level for n in t.nodes] == o.level
    assert [n.sons for n in t.nodes] == o.sons
    assert len(t.nodes) == 2 * d - 1
    assert t.depth == int(np.ceil(np.log2(d)))


def test_tree_matches_reference_fixture():
    from paper_1708_03340_b200 import build_balanced_tree
    from tests.goldens import load

    z = load("spec.npz")
    t10 = build_balanced_tree(10)
    assert [n.level for n in t10.nodes] == list(z["tree10_levels"])
    assert [n.interval for n in t10.nodes] == [tuple(v) for v in z["tree10_intervals"]]


def test_truncation_control_semantics():
    from paper_1708_03340_b200 import TruncationControl

    with pytest.raises(ValueError):
        TruncationControl()
    with pytest.raises(ValueError):
        TruncationControl(eps=0.0)
    c = TruncationControl.fixed_rank({1: 3, 2: 4})
    assert c.cap_for(2) == 4
    assert TruncationControl.accuracy(1e-3, 5).cap_for(7) == 5
    assert TruncationControl.relative(1e-6, 10.0).eps == pytest.approx(1e-5)


def test_static_ranks_and_workspace_queries_without_gpu():
    """Shape-only C-ABI queries run on the host (no device pointers needed)."""
    import ctypes

    from paper_1708_03340_b200 import _lib

    lib = _lib.load()
    d = 8
    n = _lib.i64_array([1000] * d)
    ranks = _lib.i64_array([1] + [100] * (2 * d - 2))
    t = _lib.CTensor(d, ctypes.cast(n, ctypes.POINTER(ctypes.c_int64)),
                     ctypes.cast(ranks, ctypes.POINTER(ctypes.c_int64)), None, 0)
    nb = ctypes.c_size_t(0)
    assert lib.ht_truncate_workspace_size(ctypes.byref(t), ctypes.byref(nb)) == 0
    assert nb.value > 8 * (8 * 1000 * 100 + 6 * 100 ** 3)
    ctl = _lib.CTruncCtl(0.0, 50, None)
    out = (ctypes.c_int64 * (2 * d - 1))()
    assert lib.ht_truncate_static_ranks(ctypes.byref(t), ctypes.byref(ctl), out) == 1
    assert list(out)[1:] == [50] * (2 * d - 2)
    ctl2 = _lib.CTruncCtl(1e-3, 0, None)
    assert lib.ht_truncate_static_ranks(ctypes.byref(t), ctypes.byref(ctl2), out) == 0
    bad = _lib.CTruncCtl(0.0, 0, None)
    assert lib.ht_truncate_static_ranks(ctypes.byref(t), ctypes.byref(bad), out) == _lib.HT_ERR_ARGUMENT
    assert "eps" in _lib.last_error()
    # orthogonalised ranks shrink where k > n (kernels.py:27-28)
    n2 = _lib.i64_array([3, 2, 3, 4])
    r2 = _lib.i64_array([1, 7, 5, 5, 4, 3, 3])
    t2 = _lib.CTensor(4, ctypes.cast(n2, ctypes.POINTER(ctypes.c_int64)),
                      ctypes.cast(r2, ctypes.POINTER(ctypes.c_int64)), None, 0)
    ko = (ctypes.c_int64 * 7)()
    assert lib.ht_orth_ranks(ctypes.byref(t2), ko) == 0
    assert list(ko) == [1, 6, 5, 3, 2, 3, 3]


def test_gaussian_factors_match_oracle_generator():
    import paper_1708_03340_b200 as htb
    from oracle import htucker_oracle as orc

    for d, n, k, seed in [(8, 30, 5, 7), (5, 12, 3, 2)]:
        lv, tf, root = htb.gaussian_factors(htb.build_balanced_tree(d), n, k, seed)
        o = orc.gaussian_htensor(orc.balanced_tree(d), n, k, seed)
        assert all(np.array_equal(lv[t], o.U[t]) for t in o.U)
        assert all(np.array_equal(tf[t], o.B[t]) for t in o.B)
        assert np.array_equal(root, o.root)


def test_kronecker_form_shape_queries_without_gpu():
    """ht_tensor.kron (an unmaterialised apply_operator result, DESIGN 3.4): the
    truncation's shape-only queries accept it, check rank = operator rank * tensor rank,
    and every other entry point rejects it."""
    import ctypes

    from paper_1708_03340_b200 import _lib

    lib = _lib.load()
    d, nn = 4, 7
    n = _lib.i64_array([64] * d)
    xr = _lib.i64_array([1] + [30] * (nn - 1))
    opr = _lib.i64_array([1] + [2] * (nn - 1))
    yr = _lib.i64_array([1] + [60] * (nn - 1))
    i64p = ctypes.POINTER(ctypes.c_int64)
    x = _lib.CTensor(d, ctypes.cast(n, i64p), ctypes.cast(xr, i64p), None, 0)
    op = _lib.COperator(d, ctypes.cast(opr, i64p), None, None)
    src = _lib.CKronSrc(ctypes.pointer(op), ctypes.pointer(x))
    y = _lib.CTensor(d, ctypes.cast(n, i64p), ctypes.cast(yr, i64p), None, 0,
                     ctypes.cast(ctypes.pointer(src), ctypes.c_void_p))
    dense = _lib.CTensor(d, ctypes.cast(n, i64p), ctypes.cast(yr, i64p), None, 0)
    nb, nb_dense = ctypes.c_size_t(0), ctypes.c_size_t(0)
    assert lib.ht_truncate_workspace_size(ctypes.byref(y), ctypes.byref(nb)) == 0
    assert lib.ht_truncate_workspace_size(ctypes.byref(dense), ctypes.byref(nb_dense)) == 0
    assert nb.value >= nb_dense.value  # the E_ac operands live in the sweep's scratch
    ctl = _lib.CTruncCtl(0.0, 30, None)
    out = (ctypes.c_int64 * nn)()
    assert lib.ht_truncate_static_ranks(ctypes.byref(y), ctypes.byref(ctl), out) == 1
    assert list(out)[1:] == [30] * (nn - 1)
    # rank chain of the Kronecker form
    bad_r = _lib.i64_array([1] + [61] * (nn - 1))
    ybad = _lib.CTensor(d, ctypes.cast(n, i64p), ctypes.cast(bad_r, i64p), None, 0,
                        ctypes.cast(ctypes.pointer(src), ctypes.c_void_p))
    assert lib.ht_truncate_workspace_size(ctypes.byref(ybad), ctypes.byref(nb)) == _lib.HT_ERR_SHAPE
    assert "operator rank" in _lib.last_error()
    # not a truncation entry point
    assert lib.ht_inner_product_workspace_size(ctypes.byref(y), ctypes.byref(y), ctypes.byref(nb)) \
        == _lib.HT_ERR_UNSUPPORTED
    assert lib.ht_gramians_workspace_size(ctypes.byref(y), ctypes.byref(nb)) == _lib.HT_ERR_UNSUPPORTED
    # the orthogonalisation sweep itself takes the structured form
    assert lib.ht_orthogonalize_workspace_size(ctypes.byref(y), ctypes.byref(nb)) == 0


def test_block_form_sum_shape_queries_without_gpu():
    """ht_tensor.sum (an unmaterialised add result, DESIGN 3.5): rank = sum of the terms'
    ranks, accepted by the truncation / orthogonalisation queries only."""
    import ctypes

    from paper_1708_03340_b200 import _lib

    lib = _lib.load()
    d, nn = 8, 15
    i64p = ctypes.POINTER(ctypes.c_int64)
    n = _lib.i64_array([200] * d)
    ra, rc = _lib.i64_array([1] + [30] * (nn - 1)), _lib.i64_array([1] + [20] * (nn - 1))
    ry = _lib.i64_array([1] + [50] * (nn - 1))
    a = _lib.CTensor(d, ctypes.cast(n, i64p), ctypes.cast(ra, i64p), None, 0)
    c = _lib.CTensor(d, ctypes.cast(n, i64p), ctypes.cast(rc, i64p), None, 0)
    terms = (ctypes.POINTER(_lib.CTensor) * 2)(ctypes.pointer(a), ctypes.pointer(c))
    alphas = (ctypes.c_double * 2)(1.0, -0.5)
    src = _lib.CSumSrc(2, terms, alphas)
    y = _lib.CTensor(d, ctypes.cast(n, i64p), ctypes.cast(ry, i64p), None, 0, None,
                     ctypes.cast(ctypes.pointer(src), ctypes.c_void_p))
    nb = ctypes.c_size_t(0)
    assert lib.ht_truncate_workspace_size(ctypes.byref(y), ctypes.byref(nb)) == 0 and nb.value > 0
    ctl = _lib.CTruncCtl(0.0, 25, None)
    out = (ctypes.c_int64 * nn)()
    assert lib.ht_truncate_static_ranks(ctypes.byref(y), ctypes.byref(ctl), out) == 1
    assert list(out)[1:] == [25] * (nn - 1)
    bad = _lib.i64_array([1] + [51] * (nn - 1))
    ybad = _lib.CTensor(d, ctypes.cast(n, i64p), ctypes.cast(bad, i64p), None, 0, None,
                        ctypes.cast(ctypes.pointer(src), ctypes.c_void_p))
    assert lib.ht_truncate_workspace_size(ctypes.byref(ybad), ctypes.byref(nb)) == _lib.HT_ERR_SHAPE
    assert "sum of the terms" in _lib.last_error()
    assert lib.ht_inner_product_workspace_size(ctypes.byref(y), ctypes.byref(y), ctypes.byref(nb)) \
        == _lib.HT_ERR_UNSUPPORTED


def test_relative_accuracy_control_sets_the_flag():
    from paper_1708_03340_b200 import TruncationControl, _lib

    c, _ = TruncationControl.relative_accuracy(1e-6, 50)._c(7)
    assert c.flags == _lib.CTL_RELATIVE_EPS and c.eps == 1e-6 and c.max_rank == 50
    c2, _ = TruncationControl.accuracy(1e-6)._c(7)
    assert c2.flags == 0
