"""Pure host cost of one truncate call (Householder QR: no device->host wait inside)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb
from paper_1708_03340_b200 import _lib

tree = htb.build_balanced_tree(64)
x = htb.add(htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 12)),
            htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 13)))
ctl = htb.TruncationControl.fixed_rank(50)
htb.set_qr_mode("householder")
for _ in range(3):
    htb.truncate(x, ctl)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    htb.truncate(x, ctl)
    ts.append(time.perf_counter() - t0)
print("host ms per truncate (enqueue only):", [round(1e3 * t, 3) for t in ts])
lib = _lib.load()
import ctypes
nb = ctypes.c_size_t(0)
t0 = time.perf_counter()
for _ in range(20):
    lib.ht_truncate_workspace_size(x._c(), ctypes.byref(nb))
print("workspace query ms:", round(1e3 * (time.perf_counter() - t0) / 20, 3))
