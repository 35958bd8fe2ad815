"""Debug: orthogonalisation / sigma of the graded sum X = 2A + 1e-10 C at K > 128,
per QR policy (run with CUDA_LAUNCH_BLOCKING=1 to localise a faulting launch)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402
from oracle import htucker_oracle as orc  # noqa: E402
from tests.htconv import to_dev, to_host  # noqa: E402

k, n, mode, graded = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4] == "1"
tr = orc.balanced_tree(4)
a = orc.gaussian_htensor(tr, n, k, 41)
c = orc.gaussian_htensor(tr, n, k, 42)
s = 1e-10 if graded else 1.0
x = orc.add(orc.scale(a, 2.0), orc.scale(c, s))
xd = htb.add(htb.scale(to_dev(a), 2.0), htb.scale(to_dev(c), s))
htb.set_qr_mode(mode)
o = to_host(htb.orthogonalize(xd))
ro = orc.orthogonalize(x)
for t in range(1, 7):
    u, v = (o.U.get(t), ro.U.get(t)) if t in o.U else (o.B[t], ro.B[t])
    print(f"K={2*k} n={n} mode={mode} node {t}: max|diff| {np.abs(u - v).max():.2e}", flush=True)
print("fallbacks", htb.qr_fallback_count())
