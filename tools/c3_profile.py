"""Per-kernel device times of the C3 step (d=16, n=256, k=30, Laplace-sum operator):
Kronecker-fused apply + relative-eps truncation.  python tools/c3_profile.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402
from paper_1708_03340_b200 import _lib, problems  # noqa: E402

tree = htb.build_balanced_tree(16)
x = htb.gaussian_htensor(tree, 256, 30, 16)
op = problems.laplace_sum_operator(tree, 256)
ctl = htb.TruncationControl.relative_accuracy(1e-8, max_rank=30)


def step():
    return htb.truncate(htb.apply_operator(op, x), ctl)


for _ in range(5):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    step()
torch.cuda.synchronize()
print(f"fused apply + truncate: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms wall per step")
lib = _lib.load()
lib.ht_profile_enable(1)
step()
torch.cuda.synchronize()
rep = _lib.profile_report()
lib.ht_profile_enable(0)
tot = sum(v["ms"] for v in rep.values())
print(f"kernels {tot:.3f} ms, {sum(v['launches'] for v in rep.values())} launches")
for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"{k:28s} {v['ms']:8.4f} ms {v['launches']:5d} launches  {100 * v['ms'] / tot:5.1f}%")
