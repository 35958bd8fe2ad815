"""Phase timing of the tridiagonal eigensolver inside one C2 truncation (experiments):
loads a library built with -DHT_EIG_TIMING=1 (tools/data/libht_eigtime.so)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_03340_b200 import _lib  # noqa: E402

_lib.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "libht_eigtime.so"))
import torch  # noqa: E402

import paper_1708_03340_b200 as htb  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
tree = htb.build_balanced_tree(d)
p = d.bit_length() - 1
x = htb.add(htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p)),
            htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 2 * p + 1)))
htb.set_graph_mode(False)
for _ in range(2):
    htb.truncate(x, htb.TruncationControl.fixed_rank(50))
torch.cuda.synchronize()
