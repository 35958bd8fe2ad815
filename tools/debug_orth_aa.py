import numpy as np
import paper_1708_03340_b200 as htb
from oracle import htucker_oracle as orc
from tests.htconv import to_dev, to_host

tr = orc.balanced_tree(8)
a = orc.gaussian_htensor(tr, 64, 10, 5)
c = orc.gaussian_htensor(tr, 64, 10, 6)
for name, x in (("a+a", htb.add(to_dev(a), to_dev(a))), ("a+c", htb.add(to_dev(a), to_dev(c)))):
    for mode in ("householder", "auto"):
        htb.set_qr_mode(mode)
        n0 = htb.qr_fallback_count()
        o = to_host(htb.orthogonalize(x))
        errs = [np.abs(u.T @ u - np.eye(u.shape[1])).max() for u in o.U.values()]
        errs += [np.abs(b.reshape(b.shape[0], -1) @ b.reshape(b.shape[0], -1).T - np.eye(b.shape[0])).max()
                 for b in o.B.values()]
        print(name, mode, "fallbacks", htb.qr_fallback_count() - n0, "max orth err", max(errs),
              ["%.1e" % e for e in errs])
