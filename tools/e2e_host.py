"""Host-side cost of the bench's end-to-end pipeline (experiments): wall time per step of
each call the e2e loop makes, measured without synchronising (the host should run ahead
of the GPU).   python tools/e2e_host.py [steps]"""
import collections
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1708_03340_b200 as htb  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
tree = htb.build_balanced_tree(64)
fa = htb.gaussian_factors(tree, 1000, 50, 12)
fc = htb.gaussian_factors(tree, 1000, 50, 13)
work = bench._Single(htb, tree, fa, fc, htb.TruncationControl.fixed_rank(50))
for _ in range(5):
    work.step()
work.prepare_e2e()
tot = collections.Counter()
orig = {}
for name in ("add", "truncate"):
    orig[name] = getattr(htb, name)

    def wrap(*a, _n=name, **k):
        t0 = time.perf_counter()
        r = orig[_n](*a, **k)
        tot[_n] += time.perf_counter() - t0
        return r

    setattr(htb, name, wrap)
for n_arena in ("load_host_arena", "to_host_arena"):
    f = getattr(htb.HTensor, n_arena)

    def wrapm(self, *a, _f=f, _n=n_arena, **k):
        t0 = time.perf_counter()
        r = _f(self, *a, **k)
        tot[_n] += time.perf_counter() - t0
        return r

    setattr(htb.HTensor, n_arena, wrapm)
ev = torch.cuda.Event()
ev.record()
work.e2e_run(12, ev)
torch.cuda.synchronize()
tot.clear()
ev.record()
t0 = time.perf_counter()
work.e2e_run(steps, ev)
t_host = time.perf_counter() - t0
torch.cuda.synchronize()
t_all = time.perf_counter() - t0
print(f"host enqueue {1e3 * t_host / steps:.3f} ms/step, wall incl. sync {1e3 * t_all / steps:.3f} ms/step")
for k, v in tot.items():
    print(f"  {k}: {1e3 * v / steps:.3f} ms/step")
print("graph stats", htb.graph_stats(), "relocations", htb.graph_relocations())
