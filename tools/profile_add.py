"""One C2 d=64 add between cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402

tree = htb.build_balanced_tree(64)
a = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 12))
c = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 13))
x = htb.add(a, c)
for _ in range(3):
    htb.add(a, c, out=x)
torch.cuda.synchronize()
torch.cuda.profiler.start()
htb.add(a, c, out=x)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
