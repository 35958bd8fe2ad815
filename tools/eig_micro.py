"""Microbenchmark of the batched Jacobi eigensolver: nodes x (K x K) Gram matrices."""
import sys, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1708_03340_b200 import _lib
lib = _lib.load()
K, nodes = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (100, 126)))
rng = np.random.default_rng(0)
X = rng.standard_normal((nodes, K + 7, K))
S = torch.as_tensor(np.einsum("nij,nik->njk", X, X)).cuda()
V = torch.empty_like(S); lam = torch.empty((nodes, K), dtype=torch.float64, device='cuda')
def run():
    _lib.check(lib.ht_syev_batched(K, nodes, S.data_ptr(), V.data_ptr(), lam.data_ptr(), _lib.stream_handle()))
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record(); torch.cuda.synchronize()
ref = np.linalg.eigvalsh(S.cpu().numpy())[:, ::-1]
print(json.dumps({"K": K, "nodes": nodes, "ms": e0.elapsed_time(e1), "max_rel_err": float(np.abs(lam.cpu().numpy() - ref).max() / ref.max())}))
