"""Per-step device times of the first truncations in a fresh process (warm-up study)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb
tree = htb.build_balanced_tree(64)
x = htb.add(htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 12)),
            htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 13)))
ctl = htb.TruncationControl.fixed_rank(50)
t0 = time.perf_counter()
out = []
for i in range(400):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); htb.truncate(x, ctl); e1.record()
    out.append((e0, e1, time.perf_counter() - t0))
torch.cuda.synchronize()
ts = [(a.elapsed_time(b), w) for a, b, w in out]
for i in (0, 1, 2, 3, 5, 10, 20, 50, 100, 150, 200, 300, 399):
    print(i, "%.3f ms  wall %.2f s" % ts[i])
