"""One <T,T> of the truncated C2 d=64 tensor between cudaProfilerStart/Stop (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402
from paper_1708_03340_b200 import _lib  # noqa: E402

tree = htb.build_balanced_tree(64)
x = htb.add(htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 12)),
            htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 13)))
T = htb.truncate(x, htb.TruncationControl.fixed_rank(50))
for _ in range(3):
    htb.inner_product_device(T, T)
torch.cuda.synchronize()
lib = _lib.load()
lib.ht_profile_enable(2)
torch.cuda.profiler.start()
htb.inner_product_device(T, T)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
import json
os.makedirs("gpurun_out", exist_ok=True)
json.dump(_lib.profile_log(), open("gpurun_out/tags_ip.json", "w"))
