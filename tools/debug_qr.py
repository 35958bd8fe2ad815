"""Debug helper: run ht_qr_batched on one block and inspect V / R / T in the workspace."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1708_03340_b200 import _lib
lib = _lib.load()
m, K = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(0)
A = rng.standard_normal((m, K))
Ad = torch.as_tensor(A).cuda()
kq = min(m, K)
Q = torch.zeros((m, kq), dtype=torch.float64, device='cuda')
R = torch.zeros((kq, K), dtype=torch.float64, device='cuda')
nb = ctypes.c_size_t(0)
_lib.check(lib.ht_qr_workspace_size(m, K, 1, ctypes.byref(nb)))
ws = torch.zeros(nb.value // 8 + 1, dtype=torch.float64, device='cuda')
_lib.check(lib.ht_qr_batched(m, K, 1, Ad.data_ptr(), K, 1, m * K, Q.data_ptr(), kq, 1, m * kq, R.data_ptr(), K, kq * K,
                             ws.data_ptr(), nb.value, _lib.stream_handle()))
torch.cuda.synchronize()
w = ws.cpu().numpy()
P = -(-m // 128)
V = w[:m * K].reshape(K, m).T
Rst = w[m * K:m * K + P * K * K].reshape(P, K, K)
Tst = w[m * K + P * K * K: m * K + 3 * P * K * K].reshape(2 * P, K, K)
q_ref, r_ref = np.linalg.qr(A)
s = np.sign(np.diag(r_ref))
print("R (pre-sign) vs lapack R up to row signs:", np.abs(np.abs(Rst[0][:kq]) - np.abs(r_ref)).max())
Y = np.tril(V, -1)[:, :K].copy()
for j in range(min(m, K)): Y[j, j] = 1
taus = np.diag(Tst[0]).copy()
H = np.eye(m)
for j in range(min(m, K)):
    H = H @ (np.eye(m) - taus[j] * np.outer(Y[:, j], Y[:, j]))
print("H[:, :K] R vs A:", np.abs(H[:, :kq] @ Rst[0][:kq] - A).max())
print("Y T Y^T vs product:", np.abs(np.eye(m) - Y @ Tst[0] @ Y.T - H).max())
Qn, Rn = Q.cpu().numpy(), R.cpu().numpy()
print("Q R vs A:", np.abs(Qn @ Rn - A).max(), " Q^T Q - I:", np.abs(Qn.T @ Qn - np.eye(kq)).max())
print("R vs ref:", np.abs(Rn - r_ref * s[:, None]).max(), " Q vs ref:", np.abs(Qn - q_ref * s[None, :]).max())
