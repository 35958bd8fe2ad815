"""Microbenchmark of the batched QR (C2 inner-node shape by default): m x K, nodes."""
import ctypes, sys, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1708_03340_b200 import _lib
lib = _lib.load()
m, K, nodes = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (10000, 100, 32)))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
A = torch.randn((nodes, K, m), dtype=torch.float64, device='cuda')  # column-major blocks (M23 layout)
Q = torch.empty_like(A)
R = torch.empty((nodes, K, K), dtype=torch.float64, device='cuda')
nb = ctypes.c_size_t(0)
_lib.check(lib.ht_qr_workspace_size(m, K, nodes, ctypes.byref(nb)))
ws = torch.empty(nb.value, dtype=torch.uint8, device='cuda')
def run():
    _lib.check(lib.ht_qr_batched(m, K, nodes, A.data_ptr(), 1, m, m * K, Q.data_ptr(), 1, m, m * K, R.data_ptr(), K,
                                 K * K, ws.data_ptr(), ws.numel(), _lib.stream_handle()))
run(); torch.cuda.synchronize()
lib.ht_profile_enable(1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps): run()
e1.record(); torch.cuda.synchronize()
prof = _lib.profile_report(); lib.ht_profile_enable(0)
flops = nodes * 2 * (2 * m * K * K - 2 / 3 * K ** 3)
ms = e0.elapsed_time(e1) / reps
print(json.dumps({"m": m, "K": K, "nodes": nodes, "ms": ms, "tflops": flops / ms / 1e9,
                  "kernels": {k: round(v["ms"] / reps, 4) for k, v in prof.items()}}))
