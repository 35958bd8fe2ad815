"""Device time of add (block embedding, HBM-bound) for C2 d=64: ms and GB/s."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402

tree = htb.build_balanced_tree(64)
a = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 12))
c = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 13))
for _ in range(5):
    x = htb.add(a, c)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    x = htb.add(a, c)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
nbytes = 8 * (x.storage_size() if hasattr(x, "storage_size") else 0)
print("add ms %.3f" % ms, "out MB", nbytes / 1e6, "GB/s(out+in)", (nbytes * 1.32) / ms / 1e6 if nbytes else None)
