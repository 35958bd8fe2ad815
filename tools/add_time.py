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

from paper_1708_03340_b200 import _lib  # noqa: E402

lib = _lib.load()
lib.ht_profile_enable(1)
for _ in range(5):
    x = htb.add(a, c)
torch.cuda.synchronize()
rep = _lib.profile_report()
lib.ht_profile_enable(0)
for k, v in rep.items():
    print("kernel", k, "ms/add %.4f" % (v["ms"] / 5), "GB/s %.0f" % (v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] else 0))
