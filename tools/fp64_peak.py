"""cuBLAS DGEMM rate (torch.matmul float64) on the box: the FP64 roofline denominator."""
import json
import torch

def main():
    out = {}
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device="cuda")
        b = torch.randn(n, n, dtype=torch.float64, device="cuda")
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[f"dgemm_{n}_tflops"] = 2 * n**3 / best / 1e9
    # batched small DGEMM typical of the HT kernels (100x100x10000)
    a = torch.randn(32, 100, 10000, dtype=torch.float64, device="cuda")
    b = torch.randn(32, 10000, 100, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.bmm(a, b)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); torch.bmm(a, b); e1.record(); torch.cuda.synchronize()
    out["bmm_32x100x10000x100_tflops"] = 2 * 32 * 100 * 100 * 10000 / e0.elapsed_time(e1) / 1e9
    x = torch.empty(2**28, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
    y.copy_(x); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out["copy_gbs"] = 2 * x.numel() * 8 / best / 1e6
    out["device"] = torch.cuda.get_device_name()
    print(json.dumps(out))

if __name__ == "__main__":
    main()
