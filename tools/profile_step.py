"""One C2 truncation step between cudaProfilerStart/Stop, for ncu
(--profile-from-start off).  Also writes the launch-order kernel tags of that step
to gpurun_out/tags.json so ncu launch lists can be attributed to pipeline stages.

    python tools/profile_step.py [d] [dense|block]      (block: the block-form sum, DESIGN 3.5)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402
from paper_1708_03340_b200 import _lib  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
tree = htb.build_balanced_tree(d)
p = d.bit_length() - 1
block = len(sys.argv) > 2 and sys.argv[2] == "block"
x = htb.add(htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p)),
            htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p + 1)), lazy=block)
ctl = htb.TruncationControl.fixed_rank(50)
for _ in range(2):
    htb.truncate(x, ctl)
torch.cuda.synchronize()
lib = _lib.load()
lib.ht_profile_enable(2)
torch.cuda.profiler.start()
htb.truncate(x, ctl)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
tags = _lib.profile_log()
lib.ht_profile_enable(0)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/tags.json", "w") as f:
    json.dump(tags, f)
print("ok", len(tags), "launches")
