"""Device ms per C2 truncation step (events, 30 steps after 10 warm-up)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb

tree = htb.build_balanced_tree(64)
x = htb.add(htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 12)),
            htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 13)))
ctl = htb.TruncationControl.fixed_rank(50)
for _ in range(10):
    htb.truncate(x, ctl)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = []
for rep in range(3):
    e0.record()
    for _ in range(30):
        htb.truncate(x, ctl)
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 30)
print(os.environ.get("HT_GEMM_LR", "1"), " ".join(f"{r:.3f}" for r in res))
