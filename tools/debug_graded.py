"""Debug: graded hierarchical singular values (X = 2A + 1e-10 C) at K beyond the
shared-memory Jacobi, per eigensolver policy."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402
from oracle import htucker_oracle as orc  # noqa: E402
from tests.htconv import to_dev  # noqa: E402

for k in [int(v) for v in sys.argv[1:]]:
    tr = orc.balanced_tree(4)
    a = orc.gaussian_htensor(tr, 300, k, 41)
    c = orc.gaussian_htensor(tr, 300, k, 42)
    x = orc.add(orc.scale(a, 2.0), orc.scale(c, 1e-10))
    xd = htb.add(htb.scale(to_dev(a), 2.0), htb.scale(to_dev(c), 1e-10))
    ref = orc.hierarchical_singular_values(x)
    for mode in ("auto", "jacobi"):
        htb.set_eig_mode(mode)
        sig = htb.hierarchical_singular_values(xd)
        for t, s in ref.items():
            got = sig[t].cpu().numpy()
            rel = np.abs(got - s) / s
            print(f"K={2*k} mode={mode} node {t}: max rel {rel.max():.2e} at {rel.argmax()} "
                  f"(tail ratio {s.min()/s.max():.1e})", flush=True)
    htb.set_eig_mode("auto")
