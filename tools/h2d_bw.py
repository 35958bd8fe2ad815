"""Host<->device copy bandwidth on the box (experiments): the e2e pipeline moves 175 MB
H2D and 88 MB D2H per step through pinned buffers."""
import os
import time

import torch


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


n_in, n_out = 175_240_000 // 8, 87_620_000 // 8
h = torch.empty(n_in, dtype=torch.float64).pin_memory()
d = torch.empty(n_in, dtype=torch.float64, device="cuda")
o = torch.empty(n_out, dtype=torch.float64).pin_memory()
do = torch.empty(n_out, dtype=torch.float64, device="cuda")
o.fill_(1.0)  # touch the pinned pages
streams = [torch.cuda.Stream() for _ in range(4)]


def d2h_chunks(k):
    def f():
        step = (n_out + k - 1) // k
        for i in range(k):
            with torch.cuda.stream(streams[i % len(streams)]):
                o[i * step:(i + 1) * step].copy_(do[i * step:(i + 1) * step], non_blocking=True)
    return f


print(f"pid {os.getpid()}: H2D {timed(lambda: d.copy_(h, non_blocking=True)):.2f} ms  "
      f"D2H 1 chunk {timed(d2h_chunks(1)):.2f}  4 chunks/4 streams {timed(d2h_chunks(4)):.2f}  "
      f"16 chunks {timed(d2h_chunks(16)):.2f} ms")
