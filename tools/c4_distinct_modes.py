"""C4 with distinct parameter grids under each QR / eigensolver policy: max relative
deviation of the 20-step CG trace from the reference's (tests/golden/c4_cg_distinct.npz)."""
import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_03340_b200 as htb  # noqa: E402
from paper_1708_03340_b200 import problems  # noqa: E402
from paper_1708_03340_b200.backend import GpuBackend  # noqa: E402
from paper_1708_03340_b200.solvers import RelativeTruncation, SolverConfig, cg_solve  # noqa: E402

g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c4_cg_distinct.npz"))
mats, load = problems.p1_diffusion_matrices(cells=64)
grids = problems.distinct_parameter_grids(points=16)
op = problems.affine_operator([sp.csr_matrix(mats[0].shape)] + mats, grids)
rhs = problems.constant_rhs(load, grids)
cfg = SolverConfig(truncation=RelativeTruncation(1e-6, max_rank=50), eps_stop=1e-12, max_cg_steps=20)
for qr in sys.argv[1].split(","):
    for eig in sys.argv[2].split(","):
        htb.set_qr_mode(qr)
        htb.set_eig_mode(eig)
        x, trace = cg_solve(op, rhs, cfg, backend=GpuBackend())
        true = np.array([e.true_rel_residual for e in trace.entries])
        internal = np.array([e.internal_residual for e in trace.entries])
        dt = np.abs(true - g["true_rel"]) / g["true_rel"]
        di = np.abs(internal - g["internal"]) / g["internal"]
        print(f"qr={qr} eig={eig}: true {dt.max():.2e} internal {di.max():.2e} per-step true "
              + " ".join(f"{v:.0e}" for v in dt), flush=True)
