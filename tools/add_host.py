"""Host-side profile of add(a, c, out=x) at C2 d=64 (experiments)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402

tree = htb.build_balanced_tree(64)
a = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 12))
c = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 13))
x = htb.add(a, c)
for _ in range(5):
    htb.add(a, c, out=x)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    htb.add(a, c, out=x)
print("host ms per add:", (time.perf_counter() - t0) / 50 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    htb.add(a, c, out=x)
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(12)
