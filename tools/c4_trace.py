"""C4 CG at full size: print the convergence trace (true / internal residual, ranks, time)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import scipy.sparse as sp
from paper_1708_03340_b200 import problems
from paper_1708_03340_b200.backend import GpuBackend
from paper_1708_03340_b200.solvers import RelativeTruncation, SolverConfig, cg_solve

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cells = int(args[0]) if len(args) > 0 else 64
rel = float(args[1]) if len(args) > 1 else 1e-6
cap = int(args[2]) if len(args) > 2 else 50
steps = int(args[3]) if len(args) > 3 else 20
mats, load = problems.p1_diffusion_matrices(cells=cells)
grids = problems.parameter_grids(points=16)
op = problems.affine_operator([sp.csr_matrix(mats[0].shape)] + mats, grids)
rhs = problems.constant_rhs(load, grids)
cfg = SolverConfig(truncation=RelativeTruncation(rel, max_rank=cap), eps_stop=1e-12, max_cg_steps=steps)
import collections, torch
from paper_1708_03340_b200 import _lib


class TimedBackend(GpuBackend):
    """GpuBackend with per-method wall time (synchronised) for the breakdown."""
    acc = collections.defaultdict(lambda: [0, 0.0])

    def __getattribute__(self, name):
        f = super().__getattribute__(name)
        if name in ("apply", "add", "scale", "truncate", "inner_product", "norm"):
            def wrapped(*a, **k):
                torch.cuda.synchronize()
                t = time.perf_counter()
                r = f(*a, **k)
                torch.cuda.synchronize()
                TimedBackend.acc[name][0] += 1
                TimedBackend.acc[name][1] += time.perf_counter() - t
                return r
            return wrapped
        return f


profile = "--profile" in sys.argv
cg_solve(op, rhs, SolverConfig(truncation=cfg.truncation, eps_stop=1e-12, max_cg_steps=2), backend=GpuBackend())
torch.cuda.synchronize()
if profile:
    _lib.load().ht_profile_enable(1)
t0 = time.time()
x, trace = cg_solve(op, rhs, cfg, backend=TimedBackend() if profile else GpuBackend())
torch.cuda.synchronize()
print("wall", time.time() - t0, "aborted", trace.aborted)
if profile:
    rep = _lib.profile_report()
    _lib.load().ht_profile_enable(0)
    print({k: (v[0], round(v[1], 3)) for k, v in TimedBackend.acc.items()})
    items = sorted(rep.items(), key=lambda kv: -kv[1].get("ms", 0) if isinstance(kv[1], dict) else 0)
    for k, v in items[:25]:
        print(k, v)
for e in trace.entries:
    print(e.step, f"{e.true_rel_residual:.4e} {e.internal_residual:.4e}", e.max_rank, f"{e.seconds:.2f}")
