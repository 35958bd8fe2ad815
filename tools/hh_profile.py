"""Per-kernel device times (CUDA events per launch, ht_profile_enable) of one C2
truncation under a QR policy: python tools/hh_profile.py [householder|auto] [d]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402
from paper_1708_03340_b200 import _lib  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "householder"
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
tree = htb.build_balanced_tree(d)
p = d.bit_length() - 1
x = htb.add(htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p)),
            htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p + 1)))
ctl = htb.TruncationControl.fixed_rank(50)
htb.set_qr_mode(mode)
for _ in range(2):
    htb.truncate(x, ctl)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    htb.truncate(x, ctl)
e1.record()
torch.cuda.synchronize()
print(f"{mode}: {e0.elapsed_time(e1) / 5:.3f} ms per truncation")
lib = _lib.load()
lib.ht_profile_enable(1)
htb.truncate(x, ctl)
torch.cuda.synchronize()
rep = _lib.profile_report()
lib.ht_profile_enable(0)
tot = sum(v["ms"] for v in rep.values())
for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"{k:28s} {v['ms']:8.3f} ms {v['launches']:5d} launches  {100 * v['ms'] / tot:5.1f}%")
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rep, open(f"gpurun_out/prof_{mode}.json", "w"))
