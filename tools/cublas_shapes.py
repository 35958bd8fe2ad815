"""cuBLAS (torch.bmm, fp64) on the truncation's hot GEMM shapes, as a yardstick."""
import torch

def bench(b, m, n, k, ta=False, reps=20):
    A = torch.randn(b, k, m, dtype=torch.float64, device="cuda").transpose(1, 2) if ta else \
        torch.randn(b, m, k, dtype=torch.float64, device="cuda")
    B = torch.randn(b, k, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.bmm(A, B)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.bmm(A, B)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"b={b:5d} m={m:6d} n={n:4d} k={k:6d} ta={ta}: {ms*1e3:8.1f} us  {2*b*m*n*k/ms/1e9:6.2f} TF/s", flush=True)

bench(32, 10000, 100, 100)          # Q1 = A R^-1 / mode-3 absorb, level 5
bench(3200, 100, 100, 100)          # mode-2 absorb per slice
bench(32, 100, 100, 10000, ta=True) # Gram A^T A
bench(1, 4096, 4096, 4096)
