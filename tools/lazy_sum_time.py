"""Truncation of the block-form (lazy) sum vs the materialised sum at C2 (d, n=1000, k=50),
device time per truncation, plus the per-kernel breakdown of the lazy one:
python tools/lazy_sum_time.py [d]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402
from paper_1708_03340_b200 import _lib  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
tree = htb.build_balanced_tree(d)
p = d.bit_length() - 1
a = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p))
c = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p + 1))
ctl = htb.TruncationControl.fixed_rank(50)


def timed(fn, reps=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


xm = htb.add(a, c, lazy=False)
xl = htb.add(a, c, lazy=True)
Tm = htb.truncate(xm, ctl)
Tl = htb.truncate(xl, ctl)
out = htb.truncate(xl, ctl)
print(f"materialised: truncate {timed(lambda: htb.truncate(xm, ctl, out=out)):.3f} ms, "
      f"add {timed(lambda: htb.add(a, c, out=xm)):.3f} ms")
print(f"block form  : truncate {timed(lambda: htb.truncate(xl, ctl, out=out)):.3f} ms, "
      f"add {timed(lambda: htb.add(a, c, out=xl)):.3f} ms, "
      f"add+truncate {timed(lambda: htb.truncate(htb.add(a, c, out=xl), ctl, out=out)):.3f} ms")
diff = htb.subtract(Tm, Tl)
print("||T_mat - T_lazy|| / ||T|| =", htb.norm(diff) / htb.norm(Tm), "graphs", htb.graph_stats())
lib = _lib.load()
lib.ht_profile_enable(1)
htb.truncate(xl, ctl, out=out)
torch.cuda.synchronize()
rep = _lib.profile_report()
lib.ht_profile_enable(0)
tot = sum(v["ms"] for v in rep.values())
print(f"lazy truncation kernels {tot:.3f} ms, {sum(v['launches'] for v in rep.values())} launches")
for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"])[:14]:
    print(f"  {k:26s} {v['ms']:8.4f} ms {v['launches']:4d} launches")
