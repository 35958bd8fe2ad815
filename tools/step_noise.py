"""Run-to-run spread of the timed C2 d=64 step: repeated 50-step CUDA-event timings,
without and with the bench's NVML clock sampler running.   python tools/step_noise.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1708_03340_b200 as htb  # noqa: E402

tree = htb.build_balanced_tree(64)
x = htb.add(htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 12)),
            htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 13)))
ctl = htb.TruncationControl.fixed_rank(50)
for _ in range(20):
    htb.truncate(x, ctl)
torch.cuda.synchronize()


def timed(n=50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        htb.truncate(x, ctl)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print("arena", hex(x.arena.data_ptr()) if hasattr(x, "arena") else "?", "graphs", htb.graph_stats())
htb.set_graph_mode(False)
print("eager  ", [round(timed(), 3) for _ in range(3)])
htb.set_graph_mode(True)
print("plain  ", [round(timed(), 3) for _ in range(6)])
with bench.ClockSampler(0):
    print("sampler", [round(timed(), 3) for _ in range(6)])
print("plain  ", [round(timed(), 3) for _ in range(6)])

import time  # noqa: E402

torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    htb.truncate(x, ctl)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("host enqueue ms/step %.3f, wall ms/step %.3f" % ((t1 - t0) * 20, (t2 - t0) * 20))
