"""One C2 truncation step between cudaProfilerStart/Stop, for ncu
(--profile-from-start off).  Usage: python tools/profile_step.py [d]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
tree = htb.build_balanced_tree(d)
p = d.bit_length() - 1
x = htb.add(htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p)),
            htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p + 1)))
ctl = htb.TruncationControl.fixed_rank(50)
for _ in range(2):
    htb.truncate(x, ctl)
torch.cuda.synchronize()
torch.cuda.profiler.start()
htb.truncate(x, ctl)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
