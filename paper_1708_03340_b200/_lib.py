"""ctypes binding of the C ABI in ``include/ht_b200.h`` (libht_b200.so).

The shared library is built in-tree by ``build.py`` (nvcc, sm_100a).  There is
no fallback: if the library is missing, or no CUDA device is present, every
compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libht_b200.so")

HT_OK = 0
HT_ERR_SHAPE = 1
HT_ERR_NOT_ORTHOGONAL = 2
HT_ERR_NONCONVERGED = 3
HT_ERR_CUDA = 4
HT_ERR_NOT_SYMMETRIC = 5
HT_ERR_ARGUMENT = 6
HT_ERR_UNSUPPORTED = 7

# Exported symbols (kept in sync with include/ht_b200.h; tests check both).
EXPORTS = (
    "ht_last_error", "ht_version",
    "ht_truncate_workspace_size", "ht_truncate_static_ranks", "ht_truncate_ranks",
    "ht_truncate_project", "ht_truncate", "ht_truncate_eigenvalues",
    "ht_orth_ranks", "ht_orthogonalize_workspace_size", "ht_orthogonalize",
    "ht_gramians_workspace_size", "ht_gramians",
    "ht_add", "ht_add_sharded", "ht_scale",
    "ht_inner_product_workspace_size", "ht_inner_product",
    "ht_apply_operator", "ht_apply_operator_sharded", "ht_inner_product_sharded", "ht_inner_product_slot",
    "ht_qr_workspace_size", "ht_qr_batched", "ht_syev_batched", "ht_gemm_strided",
    "ht_launch_count", "ht_profile_enable", "ht_profile_report", "ht_profile_log",
    "ht_truncate_sharded", "ht_truncate_workspace_size_sharded", "ht_truncate_slot", "ht_set_qr_mode", "ht_set_implicit_q", "ht_qr_fallback_count", "ht_set_eig_mode",
    "ht_set_graph_mode", "ht_graph_stats", "ht_graph_relocations", "ht_set_graph_relocation", "ht_status", "ht_evaluate_entries", "ht_evaluate_weighted", "ht_graph_device_fallback",
)

_i64p = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p


class CTensor(ctypes.Structure):
    # `kron`: ht_kron_src* (NULL for an ordinary tensor; see include/ht_b200.h)
    _fields_ = [("d", ctypes.c_int32), ("n", _i64p), ("rank", _i64p),
                ("node", ctypes.POINTER(ctypes.c_void_p)), ("orthogonal", ctypes.c_int32),
                ("kron", ctypes.c_void_p), ("sum", ctypes.c_void_p)]


class CTruncCtl(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("max_rank", ctypes.c_int64), ("max_rank_per_node", _i64p),
                ("flags", ctypes.c_int32)]


CTL_RELATIVE_SIGMA = 1
CTL_RELATIVE_EPS = 2


class CGmat(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("nnz", ctypes.c_int64), ("values", _vp), ("indptr", _vp), ("indices", _vp)]


class COperator(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("rank", _i64p),
                ("leaf_cols", ctypes.POINTER(ctypes.POINTER(CGmat))),
                ("node", ctypes.POINTER(ctypes.c_void_p))]


class CSumSrc(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int32), ("term", ctypes.POINTER(ctypes.POINTER(CTensor))),
                ("alpha", ctypes.POINTER(ctypes.c_double))]


class CKronSrc(ctypes.Structure):
    _fields_ = [("op", ctypes.POINTER(COperator)), ("x", ctypes.POINTER(CTensor))]


_lock = threading.Lock()
_lib = None


def _declare(lib):
    P = ctypes.POINTER
    sz = P(ctypes.c_size_t)
    t = P(CTensor)
    ctl = P(CTruncCtl)
    sig = {
        "ht_last_error": ([], ctypes.c_char_p),
        "ht_version": ([], ctypes.c_char_p),
        "ht_truncate_workspace_size": ([t, sz], ctypes.c_int),
        "ht_truncate_static_ranks": ([t, ctl, _i64p], ctypes.c_int),
        "ht_truncate_ranks": ([t, ctl, _vp, ctypes.c_size_t, _i64p, _vp], ctypes.c_int),
        "ht_truncate_project": ([t, ctl, _vp, ctypes.c_size_t, t, _vp], ctypes.c_int),
        "ht_truncate": ([t, ctl, _vp, ctypes.c_size_t, t, _vp], ctypes.c_int),
        "ht_truncate_eigenvalues": ([t, _vp, ctypes.c_size_t, _vp, _vp], ctypes.c_int),
        "ht_orth_ranks": ([t, _i64p], ctypes.c_int),
        "ht_orthogonalize_workspace_size": ([t, sz], ctypes.c_int),
        "ht_orthogonalize": ([t, _vp, ctypes.c_size_t, t, _vp], ctypes.c_int),
        "ht_gramians_workspace_size": ([t, sz], ctypes.c_int),
        "ht_gramians": ([t, _vp, ctypes.c_size_t, P(ctypes.c_void_p), _vp], ctypes.c_int),
        "ht_add": ([t, t, ctypes.c_double, t, _vp], ctypes.c_int),
        "ht_add_sharded": ([t, t, ctypes.c_double, _vp, t, _vp], ctypes.c_int),
        "ht_scale": ([_vp, _vp, ctypes.c_int64, ctypes.c_double, _vp], ctypes.c_int),
        "ht_inner_product_workspace_size": ([t, t, sz], ctypes.c_int),
        "ht_inner_product": ([t, t, _vp, ctypes.c_size_t, _vp, P(ctypes.c_double), _vp], ctypes.c_int),
        "ht_apply_operator": ([P(COperator), t, t, _vp], ctypes.c_int),
        "ht_apply_operator_sharded": ([P(COperator), t, _vp, t, _vp], ctypes.c_int),
        "ht_inner_product_sharded": ([t, t, _vp, _vp, ctypes.c_size_t, _vp, _vp], ctypes.c_int),
        "ht_inner_product_slot": ([t, t, _vp, ctypes.c_int32, P(ctypes.c_void_p), _i64p], ctypes.c_int),
        "ht_qr_workspace_size": ([ctypes.c_int64] * 3 + [sz], ctypes.c_int),
        "ht_qr_batched": ([ctypes.c_int64] * 3 + [_vp] + [ctypes.c_int64] * 3 + [_vp] + [ctypes.c_int64] * 3
                          + [_vp] + [ctypes.c_int64] * 2 + [_vp, ctypes.c_size_t, _vp], ctypes.c_int),
        "ht_truncate_sharded": ([t, ctl, _vp, ctypes.c_size_t, ctypes.c_int32, _vp, _vp, t, _vp], ctypes.c_int),
        "ht_truncate_workspace_size_sharded": ([t, _vp, sz], ctypes.c_int),
        "ht_truncate_slot": ([t, _vp, _vp, ctypes.c_int32, ctypes.c_int32, P(ctypes.c_void_p), _i64p], ctypes.c_int),
        "ht_launch_count": ([], ctypes.c_int64),
        "ht_set_qr_mode": ([ctypes.c_int], ctypes.c_int),
        "ht_set_implicit_q": ([ctypes.c_int], ctypes.c_int),
        "ht_qr_fallback_count": ([], ctypes.c_int64),
        "ht_set_eig_mode": ([ctypes.c_int], ctypes.c_int),
        "ht_set_graph_mode": ([ctypes.c_int], ctypes.c_int),
        "ht_evaluate_entries": ([t, _vp, ctypes.c_int64, _vp, _vp], ctypes.c_int),
        "ht_evaluate_weighted": ([t, _vp, _vp, ctypes.c_int64, _vp, _vp], ctypes.c_int),
        "ht_graph_stats": ([_i64p, _i64p], ctypes.c_int),
        "ht_graph_relocations": ([], ctypes.c_int64),
        "ht_set_graph_relocation": ([ctypes.c_int], ctypes.c_int),
        "ht_status": ([ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), _vp], ctypes.c_int),
        "ht_graph_device_fallback": ([], ctypes.c_int),
        "ht_profile_enable": ([ctypes.c_int], ctypes.c_int),
        "ht_profile_report": ([ctypes.c_char_p, ctypes.c_size_t], ctypes.c_int),
        "ht_profile_log": ([ctypes.c_char_p, ctypes.c_size_t], ctypes.c_int),
        "ht_syev_batched": ([ctypes.c_int64, ctypes.c_int64, _vp, _vp, _vp, _vp], ctypes.c_int),
        "ht_gemm_strided": ([ctypes.c_int64] * 4 + [ctypes.c_double, _vp] + [ctypes.c_int64] * 3 + [_vp]
                            + [ctypes.c_int64] * 3 + [ctypes.c_double, _vp] + [ctypes.c_int64] * 3 + [_vp],
                            ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def load(path: str = LIB_PATH):
    """Load libht_b200.so (no GPU needed just to load it)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"libht_b200.so not found at {path}; build it with `python -m paper_1708_03340_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(path)
            _declare(lib)
            _lib = lib
    return _lib


def last_error() -> str:
    return load().ht_last_error().decode()


def check(rc: int, what: str = "") -> None:
    if rc == HT_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc in (HT_ERR_SHAPE, HT_ERR_NOT_ORTHOGONAL, HT_ERR_NOT_SYMMETRIC, HT_ERR_ARGUMENT):
        raise ValueError(msg)
    if rc == HT_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def check_status(stream=None) -> None:
    """Raise the error a queued truncation left in the sticky status word (and clear it)."""
    check(load().ht_status(1, None, stream_handle(stream)), "queued truncation")


def profile_report() -> dict:
    import json

    lib = load()
    n = lib.ht_profile_report(None, 0)
    buf = ctypes.create_string_buffer(n + 1)
    lib.ht_profile_report(buf, n + 1)
    return json.loads(buf.value.decode())


def profile_log() -> list:
    """Launch-order kernel tags recorded while ht_profile_enable(2) was on."""
    import json

    lib = load()
    n = lib.ht_profile_log(None, 0)
    buf = ctypes.create_string_buffer(n + 1)
    lib.ht_profile_log(buf, n + 1)
    return json.loads(buf.value.decode())


def i64_array(values):
    arr = (ctypes.c_int64 * len(values))(*[int(v) for v in values])
    return arr


def ptr_array(values):
    return (ctypes.c_void_p * len(values))(*[int(v) for v in values])


def stream_handle(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def as_np_i64(buf, n):
    return np.array([buf[i] for i in range(n)], dtype=np.int64)
