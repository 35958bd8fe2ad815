"""C4 CG at full size: print the convergence trace (true / internal residual, ranks, time)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import scipy.sparse as sp
from paper_1708_03340_b200 import problems
from paper_1708_03340_b200.backend import GpuBackend
from paper_1708_03340_b200.solvers import RelativeTruncation, SolverConfig, cg_solve

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rel = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 50
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
mats, load = problems.p1_diffusion_matrices(cells=cells)
grids = problems.parameter_grids(points=16)
op = problems.affine_operator([sp.csr_matrix(mats[0].shape)] + mats, grids)
rhs = problems.constant_rhs(load, grids)
cfg = SolverConfig(truncation=RelativeTruncation(rel, max_rank=cap), eps_stop=1e-12, max_cg_steps=steps)
t0 = time.time()
x, trace = cg_solve(op, rhs, cfg, backend=GpuBackend())
print("wall", time.time() - t0, "aborted", trace.aborted)
for e in trace.entries:
    print(e.step, f"{e.true_rel_residual:.4e} {e.internal_residual:.4e}", e.max_rank, f"{e.seconds:.2f}")
