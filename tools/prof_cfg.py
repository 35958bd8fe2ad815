"""Per-kernel CUDA-event breakdown (ht_profile_enable) of one truncation of a config:
    python tools/prof_cfg.py c3|c2:<d>|c5
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402
from paper_1708_03340_b200 import _lib, problems  # noqa: E402


def setup(cfg):
    if cfg == "c3":
        tree = htb.build_balanced_tree(16)
        x = htb.gaussian_htensor(tree, 256, 30, 16)
        y = htb.apply_operator(problems.laplace_sum_operator(tree, 256), x)
        return y, htb.TruncationControl(eps=1e-8 * htb.norm(y), max_rank=30)
    if cfg.startswith("c2"):
        d = int(cfg.split(":")[1])
        tree = htb.build_balanced_tree(d)
        p = d.bit_length() - 1
        a = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p))
        c = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p + 1))
        return htb.add(a, c), htb.TruncationControl.fixed_rank(50)
    raise SystemExit(cfg)


x, ctl = setup(sys.argv[1])
lib = _lib.load()
for _ in range(3):
    htb.truncate(x, ctl)
torch.cuda.synchronize()
lib.ht_profile_enable(1)
reps = 5
for _ in range(reps):
    htb.truncate(x, ctl)
torch.cuda.synchronize()
prof = _lib.profile_report()
lib.ht_profile_enable(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    htb.truncate(x, ctl)
e1.record()
torch.cuda.synchronize()
tot = sum(v["ms"] for v in prof.values()) / reps
print(json.dumps({"cfg": sys.argv[1], "step_ms": e0.elapsed_time(e1) / reps, "kernel_sum_ms": tot}))
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"{k:24s} {v['ms'] / reps:8.3f} ms  {v['launches'] / reps:5.1f} launches")
