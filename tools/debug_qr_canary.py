"""Debug: Householder TSQR on a column panel inside a larger column-major matrix, in
place (the block Gram-Schmidt panel call), with canary regions around every buffer."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_03340_b200 import _lib  # noqa: E402

lib = _lib.load()
m, K, c0, w = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
PAD = 1 << 20
CAN = 12345.678
rng = np.random.default_rng(0)
A = rng.standard_normal((K, m))  # column-major m x K  == row-major K x m
buf = torch.full((PAD + m * K + PAD,), CAN, dtype=torch.float64, device="cuda")
buf[PAD:PAD + m * K] = torch.as_tensor(A.ravel()).cuda()
Rb = torch.full((PAD + K * K + PAD,), CAN, dtype=torch.float64, device="cuda")
nb = ctypes.c_size_t(0)
_lib.check(lib.ht_qr_workspace_size(m, w, 1, ctypes.byref(nb)))
ws = torch.full((PAD + nb.value // 8 + 16 + PAD,), CAN, dtype=torch.float64, device="cuda")
base = buf.data_ptr() + 8 * PAD
QJ = base + 8 * c0 * m
RJ = Rb.data_ptr() + 8 * (PAD + c0 * K + c0)
_lib.check(lib.ht_qr_batched(m, w, 1, QJ, 1, m, m * K, QJ, 1, m, m * K, RJ, K, K * K,
                             ws.data_ptr() + 8 * PAD, nb.value, _lib.stream_handle()))
torch.cuda.synchronize()
b = buf.cpu().numpy()
print("canary matrix before", np.all(b[:PAD] == CAN), "after", np.all(b[PAD + m * K:] == CAN))
r = Rb.cpu().numpy()
print("canary R before", np.all(r[:PAD] == CAN), "after", np.all(r[PAD + K * K:] == CAN))
wv = ws.cpu().numpy()
print("canary ws before", np.all(wv[:PAD] == CAN), "after", np.all(wv[PAD + nb.value // 8 + 16:] == CAN))
Q = b[PAD:PAD + m * K].reshape(K, m).T
print("other columns untouched", np.array_equal(Q[:, :c0], A.T[:, :c0]), np.array_equal(Q[:, c0 + w:], A.T[:, c0 + w:]))
Qp = Q[:, c0:c0 + w]
print("orthonormal", np.abs(Qp.T @ Qp - np.eye(w)).max())
R = r[PAD:PAD + K * K].reshape(K, K)
print("R block canary-free rows", np.all(R[c0:c0 + w, c0:c0 + w][np.tril_indices(w, -1)] == 0) or "lower nonzero")
print("reconstruct", np.abs(Qp @ np.triu(R[c0:c0 + w, c0:c0 + w]) - A.T[:, c0:c0 + w]).max())
print("R outside block untouched", np.all(np.delete(R, np.s_[c0:c0 + w], axis=0) == CAN))
