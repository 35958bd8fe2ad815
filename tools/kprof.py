"""Per-kernel device times (CUDA events per launch) of add, <T,T> and a truncation at
C2 (d, n=1000, k=50):  python tools/kprof.py [d]"""
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
x = htb.add(a, c)
ctl = htb.TruncationControl.fixed_rank(50)
T = htb.truncate(x, ctl)
lib = _lib.load()


def timed(name, fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    lib.ht_profile_enable(1)
    fn()
    torch.cuda.synchronize()
    rep = _lib.profile_report()
    lib.ht_profile_enable(0)
    tot = sum(v["ms"] for v in rep.values())
    print(f"== {name}: {e0.elapsed_time(e1) / reps:.4f} ms per call (back to back); kernels {tot:.4f} ms")
    for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
        extra = f" {v['bytes'] / v['ms'] / 1e6:.0f} GB/s" if v.get("bytes") else ""
        print(f"   {k:28s} {v['ms']:8.4f} ms {v['launches']:4d} launches{extra}")


timed("add", lambda: htb.add(a, c, out=x))
timed("inner <T,T>", lambda: htb.inner_product_device(T, T))
timed("truncate", lambda: htb.truncate(x, ctl), 5)

if os.environ.get("PER_LAUNCH"):
    lib.ht_profile_enable(5)
    htb.inner_product_device(T, T)
    torch.cuda.synchronize()
    rep = _lib.profile_report()
    lib.ht_profile_enable(0)
    print("== <T,T> per launch")
    for k, v in sorted(rep.items(), key=lambda kv: int(kv[0].split("#")[1])):
        print(f"   {k:28s} {v['ms'] * 1e3:8.1f} us")
