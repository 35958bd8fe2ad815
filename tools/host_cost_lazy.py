"""Host-side cost (wall, no device sync inside the loop) of the e2e step's calls at C2 d=64."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb

tree = htb.build_balanced_tree(64)
a = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 12))
c = htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 13))
ctl = htb.TruncationControl.fixed_rank(50)
xl = htb.add(a, c)
xm = htb.add(a, c, lazy=False)
T = htb.truncate(xl, ctl)
for _ in range(4):
    htb.truncate(htb.add(a, c, out=xl), ctl, out=T)
    htb.truncate(htb.add(a, c, out=xm), ctl, out=T)
torch.cuda.synchronize()


def host(fn, n=50):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = (time.perf_counter() - t0) / n * 1e3
    torch.cuda.synchronize()
    return dt


print(f"lazy add(out=)      host {host(lambda: htb.add(a, c, out=xl)):.3f} ms")
print(f"eager add(out=)     host {host(lambda: htb.add(a, c, out=xm)):.3f} ms")
print(f"truncate(lazy, out) host {host(lambda: htb.truncate(xl, ctl, out=T), 20):.3f} ms")
print(f"truncate(mat, out)  host {host(lambda: htb.truncate(xm, ctl, out=T), 20):.3f} ms")
