"""Debug: graph capture / replay / relocation step by step (prints counters after each call)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402
from paper_1708_03340_b200 import _lib  # noqa: E402


def arrays(t):
    leaves, transfer, root = t.to_numpy()
    return [np.asarray(v) for _, v in sorted(leaves.items())] + \
           [np.asarray(v) for _, v in sorted(transfer.items())] + [np.asarray(root)]


def state(tag):
    torch.cuda.synchronize()
    print(tag, "stats", htb.graph_stats(), "reloc", htb.graph_relocations(),
          "mode", _lib.load().ht_graph_device_fallback(), flush=True)


d, n, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
tree = htb.build_balanced_tree(d)
x = htb.add(htb.gaussian_htensor(tree, n, k, 3), htb.gaussian_htensor(tree, n, k, 4))
ctl = htb.TruncationControl.fixed_rank(k)
htb.set_graph_mode(False)
ref = arrays(htb.truncate(x, ctl))
htb.set_graph_mode(True)
state("eager")
keep = []
for i in range(6):
    t = htb.truncate(x, ctl)
    state(f"call {i} out={t._arena.data_ptr():#x}")
    keep.append(t)
    got = arrays(t)
    print("  equal", all(np.array_equal(a, b) for a, b in zip(got, ref)), flush=True)
