"""Host enqueue time vs device time of the C2 truncation."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb

tree = htb.build_balanced_tree(64)
x = htb.add(htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 12)),
            htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 13)))
ctl = htb.TruncationControl.fixed_rank(50)
for _ in range(3):
    htb.truncate(x, ctl)
torch.cuda.synchronize()
n = 10
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(n):
    htb.truncate(x, ctl)
t1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e3*(t1-t0)/n:.3f} ms/step, device {e0.elapsed_time(e1)/n:.3f} ms/step, wall {1e3*(t2-t0)/n:.3f}")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    htb.truncate(x, ctl)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumtime").print_stats(12)

# same loop with a bench-style NVML sampler thread running
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402
with ClockSampler(0) as clk:
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        htb.truncate(x, ctl)
    e1.record()
    torch.cuda.synchronize()
print(f"with sampler: device {e0.elapsed_time(e1)/n:.3f} ms/step", clk.summary())
