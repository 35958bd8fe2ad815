"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py [--c4] [--large]

The fixtures pin both the oracle restatement (``tests/test_oracle_golden.py``)
and, through the oracle, the CUDA path (``tests/test_gpu_parity.py``).  Inputs
are the seeded Gaussian tensors of ``oracle.htucker_oracle.gaussian_htensor``
(or the reference's own ``random_htensor`` for the small-case sweep); the same
host arrays are handed to the reference.  Recorded library versions are stored
in every file under ``meta``.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import htucker as ref  # noqa: E402
from htucker import arith as ref_arith  # noqa: E402
from htucker import kernels as ref_kernels  # noqa: E402

from oracle import htucker_oracle as orc  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def meta():
    import scipy

    cfg = np.show_config(mode="dicts")
    blas = cfg.get("Build Dependencies", {}).get("blas", {})
    return json.dumps({"numpy": np.__version__, "scipy": scipy.__version__,
                       "blas": f"{blas.get('name')} {blas.get('version')}",
                       "generator": "tests/golden/make_golden.py"})


def to_ref(x: orc.HT):
    tree = ref.build_balanced_tree(x.tree.d)
    return ref.HTensor(tree, dict(x.U), dict(x.B), x.root.copy(), orthogonal=x.orthogonal)


def pack(prefix: str, x, out: dict):
    """Flatten an HT (oracle or reference) into npz keys ``prefix/<node>``."""
    tree_n = 2 * x.tree.d - 1
    for t in range(tree_n):
        if t == 0:
            arr = x.root_matrix if hasattr(x, "root_matrix") else x.root
        elif (x.leaves if hasattr(x, "leaves") else x.U).get(t) is not None:
            arr = (x.leaves if hasattr(x, "leaves") else x.U)[t]
        else:
            arr = (x.transfer if hasattr(x, "transfer") else x.B)[t]
        out[f"{prefix}/{t}"] = np.ascontiguousarray(arr)


def ref_sigmas(xr):
    o = ref.orthogonalize(xr)
    bh = ref.compute_bhat(o)
    return o, bh, {t: ref_kernels.sym_eig_desc(bh[t])[1] for t in bh}


def golden_c1():
    a, c, x = orc.c1_inputs()
    ar, cr = to_ref(a), to_ref(c)
    xr = ref.add(ref.scale(ar, 2.0), ref.scale(cr, 1e-10))
    ctl = ref.TruncationControl.fixed_rank(10)
    tr = ref.truncate(xr, ctl)
    o, bh, lam = ref_sigmas(xr)
    out = {"meta": meta()}
    pack("A", a, out)
    pack("C", c, out)
    pack("Xorth", o, out)
    pack("T", tr, out)
    for t in bh:
        out[f"bhat/{t}"] = bh[t]
        out[f"lam/{t}"] = lam[t]
    out["ranks_T"] = np.array([tr.rank(t) for t in range(1, 15)])
    out["norm_X"] = ref.norm(xr)
    out["norm_T"] = ref.norm(tr)
    out["ip_TT"] = ref.inner_product(tr, tr)
    # truncation error through the orthogonalised difference (SURVEY finding 0.3.3)
    out["trunc_err"] = float(np.linalg.norm(ref.orthogonalize(ref.subtract(xr, tr)).root_matrix))
    np.savez_compressed(os.path.join(OUT, "c1.npz"), **out)


def golden_small():
    """The SPEC's intended oracle sweep: d in 2..5, n <= 4, k <= 3,
    reference ``random_htensor`` inputs, every drop-in operation recorded."""
    out = {"meta": meta()}
    case = 0
    for seed in range(40):
        rng = np.random.default_rng(1000 + seed)
        d = int(rng.integers(2, 6))
        n = [int(v) for v in rng.integers(2, 5, size=d)]
        tree = ref.build_balanced_tree(d)
        ka = {t.index: int(min(rng.integers(1, 4), 3)) for t in tree.non_root}
        # keep the generator's structural bounds (format.py:286-287, 296-299)
        for leaf in tree.leaves:
            ka[leaf.index] = min(ka[leaf.index], n[leaf.dim - 1])
        for lev in reversed(tree.levels_top_down()):
            for t in lev:
                node = tree.node(t)
                if not node.is_leaf and not node.is_root:
                    s1, s2 = node.sons
                    ka[t] = min(ka[t], ka[s1] * ka[s2])
        a = ref.random_htensor(tree, n, ka, seed=2 * seed)
        c = ref.random_htensor(tree, n, ka, seed=2 * seed + 1)
        x = ref.add(a, ref.scale(c, 0.5))
        p = f"case{case}"
        out[f"{p}/d"] = d
        out[f"{p}/n"] = np.array(n)
        pack(f"{p}/A", a, out)
        pack(f"{p}/C", c, out)
        o, bh, lam = ref_sigmas(x)
        pack(f"{p}/Xorth", o, out)
        for t in bh:
            out[f"{p}/bhat/{t}"] = bh[t]
            out[f"{p}/lam/{t}"] = lam[t]
        eps = 0.3 * ref.norm(x)
        for tag, ctl in (("fix", ref.TruncationControl.fixed_rank(2)),
                         ("eps", ref.TruncationControl.accuracy(eps)),
                         ("both", ref.TruncationControl(eps=eps, max_rank=1))):
            tr = ref.truncate(x, ctl)
            out[f"{p}/ranks_{tag}"] = np.array([tr.rank(t) for t in range(1, 2 * d - 1)])
            out[f"{p}/normT_{tag}"] = ref.norm(tr)
            out[f"{p}/err_{tag}"] = float(np.linalg.norm(
                ref.orthogonalize(ref.subtract(x, tr)).root_matrix))
        out[f"{p}/eps"] = eps
        out[f"{p}/ip_AC"] = ref.inner_product(a, c)
        out[f"{p}/dense_X"] = ref.to_dense(x)
        out[f"{p}/entry"] = np.array([ref.evaluate_entry(x, tuple(0 for _ in range(d))),
                                      ref.evaluate_entry(x, tuple(v - 1 for v in n))])
        case += 1
    out["count"] = case
    np.savez_compressed(os.path.join(OUT, "small.npz"), **out)


def golden_shrink():
    """Rank shrink in orthogonalize: leaf rank > n and k_t > k1*k2 after add
    (arith.py:135-141, kernels.py:27-28)."""
    tree = ref.build_balanced_tree(4)
    a = ref.random_htensor(tree, [3, 2, 3, 4], {1: 4, 2: 3, 3: 3, 4: 2, 5: 2, 6: 2}, seed=7)
    c = ref.random_htensor(tree, [3, 2, 3, 4], {1: 3, 2: 2, 3: 2, 4: 2, 5: 1, 6: 2}, seed=8)
    x = ref.add(a, c)
    o, bh, lam = ref_sigmas(x)
    out = {"meta": meta()}
    pack("A", a, out)
    pack("C", c, out)
    pack("Xorth", o, out)
    for t in bh:
        out[f"bhat/{t}"] = bh[t]
        out[f"lam/{t}"] = lam[t]
    out["ranks_X"] = np.array([x.rank(t) for t in range(1, 7)])
    out["ranks_Xorth"] = np.array([o.rank(t) for t in range(1, 7)])
    tr = ref.truncate(x, ref.TruncationControl.fixed_rank(2))
    out["ranks_T"] = np.array([tr.rank(t) for t in range(1, 7)])
    out["err_T"] = float(np.linalg.norm(ref.orthogonalize(ref.subtract(x, tr)).root_matrix))
    np.savez_compressed(os.path.join(OUT, "shrink.npz"), **out)


def golden_c2_d8():
    """C2 at d=8 (n=1000, k=50): inputs regenerate from seeds 6/7; store the
    gauge-invariant outputs only (the tensors are ~9 MB each)."""
    a, c, x = orc.c2_inputs(8)
    xr = ref.add(to_ref(a), to_ref(c))
    tr = ref.truncate(xr, ref.TruncationControl.fixed_rank(50))
    _, _, lam = ref_sigmas(xr)
    out = {"meta": meta()}
    for t in lam:
        out[f"lam/{t}"] = lam[t]
    out["ranks_T"] = np.array([tr.rank(t) for t in range(1, 15)])
    out["ip_TT"] = ref.inner_product(tr, tr)
    out["norm_X"] = ref.norm(xr)
    out["trunc_err"] = float(np.linalg.norm(ref.orthogonalize(ref.subtract(xr, tr)).root_matrix))
    np.savez_compressed(os.path.join(OUT, "c2_d8.npz"), **out)


def golden_c2_large(d: int):
    """C2 at d = 64 / 128 / 256 (n=1000, k=50, rank 100 -> 50) through the REFERENCE:
    every hierarchical singular value (sqrt of sym_eig_desc of compute_bhat of the
    orthogonalised sum), the truncated ranks, <T,T>, ||X|| and the truncation error.
    Inputs regenerate from the seeds (2p, 2p+1); only gauge-invariant outputs are kept."""
    a, c, x = orc.c2_inputs(d)
    xr = ref.add(to_ref(a), to_ref(c))
    tr = ref.truncate(xr, ref.TruncationControl.fixed_rank(50))
    _, _, lam = ref_sigmas(xr)
    out = {"meta": meta()}
    for t in lam:
        out[f"lam/{t}"] = lam[t]
    out["ranks_T"] = np.array([tr.rank(t) for t in range(1, 2 * d - 1)])
    out["ip_TT"] = ref.inner_product(tr, tr)
    out["norm_X"] = ref.norm(xr)
    out["trunc_err"] = float(np.linalg.norm(ref.orthogonalize(ref.subtract(xr, tr)).root_matrix))
    np.savez_compressed(os.path.join(OUT, f"c2_d{d}.npz"), **out)


def golden_c5_shape():
    """C5 shape on one shard's worth of tree: d=8, n=2048, the 4-way sum of rank-100
    Gaussian tensors (seeds 0..3, X = ((A0 + A1) + A2) + A3, rank 400) truncated to
    rank 100 -- 2048 x 400 leaf frames, 400^3 transfer tensors, 400 x 400 Gramians."""
    xs = orc.c5_inputs(8)
    xr = to_ref(xs[0])
    for y in xs[1:]:
        xr = ref.add(xr, to_ref(y))
    tr = ref.truncate(xr, ref.TruncationControl.fixed_rank(100))
    _, _, lam = ref_sigmas(xr)
    out = {"meta": meta()}
    for t in lam:
        out[f"lam/{t}"] = lam[t]
    out["ranks_T"] = np.array([tr.rank(t) for t in range(1, 15)])
    out["ip_TT"] = ref.inner_product(tr, tr)
    out["norm_X"] = ref.norm(xr)
    out["trunc_err"] = float(np.linalg.norm(ref.orthogonalize(ref.subtract(xr, tr)).root_matrix))
    np.savez_compressed(os.path.join(OUT, "c5_d8.npz"), **out)


def golden_c3_small():
    """Operator application + truncation (C3 shape, shrunk): d=4, n=6, k=3,
    Laplace-sum operator, eps 1e-8*||Y|| with cap 3."""
    tree = ref.build_balanced_tree(4)
    otr = orc.balanced_tree(4)
    x = orc.gaussian_htensor(otr, 6, 3, 11)
    op = orc.laplace_operator(otr, 6)
    rop = ref.HTOperator(tree, {t: [ref.GeneralizedMatrix.diagonal(w[0].data),
                                    ref.GeneralizedMatrix.csr(w[1].data)] for t, w in op.W.items()},
                         dict(op.H), op.root.copy())
    xr = to_ref(x)
    y = ref.apply_operator(rop, xr)
    ctl = ref.TruncationControl(eps=1e-8 * ref.norm(y), max_rank=3)
    tr = ref.truncate(y, ctl)
    out = {"meta": meta()}
    pack("X", x, out)
    pack("Y", y, out)
    out["dense_op"] = ref.operator_to_dense_matrix(rop)
    out["ranks_T"] = np.array([tr.rank(t) for t in range(1, 7)])
    out["norm_Y"] = ref.norm(y)
    out["err_T"] = float(np.linalg.norm(ref.orthogonalize(ref.subtract(y, tr)).root_matrix))
    _, _, lam = ref_sigmas(y)
    for t in lam:
        out[f"lam/{t}"] = lam[t]
    np.savez_compressed(os.path.join(OUT, "c3_small.npz"), **out)


def golden_cg():
    """The reference's own CG (solvers.cg_solve, SerialBackend) on a small Laplace
    problem: d=4, n=16, rhs = all-ones rank 1, eps 1e-7 absolute + cap 6, 8 steps."""
    from htucker import solvers as ref_solvers

    tree = ref.build_balanced_tree(4)
    otr = orc.balanced_tree(4)
    op = orc.laplace_operator(otr, 16)
    rop = ref.HTOperator(tree, {t: [ref.GeneralizedMatrix.diagonal(w[0].data),
                                    ref.GeneralizedMatrix.csr(w[1].data)] for t, w in op.W.items()},
                         dict(op.H), op.root.copy())
    rhs = to_ref(orc.ones_htensor(otr, 16))
    cfg = ref_solvers.SolverConfig(truncation=ref.TruncationControl(eps=1e-7, max_rank=6), eps_stop=1e-10,
                                   max_cg_steps=8)
    x, trace = ref_solvers.cg_solve(rop, rhs, cfg)
    out = {"meta": meta()}
    pack("Xcg", x, out)
    out["ranks_X"] = np.array([x.rank(t) for t in range(1, 7)])
    out["internal"] = np.array([e.internal_residual for e in trace.entries])
    out["true_rel"] = np.array([e.true_rel_residual for e in trace.entries])
    np.savez_compressed(os.path.join(OUT, "cg.npz"), **out)


def golden_c4_operator():
    """The reference's affine operator builder (cookie.build_ht_operator, compressed)
    on small P1 subdomain matrices: pins problems.affine_operator."""
    from htucker import cookie

    from paper_1708_03340_b200 import problems

    mats, load = problems.p1_diffusion_matrices(cells=6)
    import scipy.sparse as sp

    zero = sp.csr_matrix(mats[0].shape)
    grids = [np.linspace(0.1, 1.0, 4) for _ in range(9)]
    op = cookie.build_ht_operator([zero] + mats, grids)
    out = {"meta": meta(), "load": load}
    for t, a in op.transfer.items():
        out[f"B/{t}"] = np.asarray(a)
    out["root"] = np.asarray(op.root_matrix)
    for t, cols in op.leaves.items():
        for j, g in enumerate(cols):
            out[f"W/{t}/{j}/kind"] = np.array(g.kind)
            out[f"W/{t}/{j}/dense"] = np.asarray(g.to_dense() if hasattr(g, "to_dense") else g.data.toarray())
    for j, m in enumerate(mats):
        out[f"K/{j}"] = m.toarray()
    np.savez_compressed(os.path.join(OUT, "c4_operator.npz"), **out)


def golden_c4_cg(broken: bool = False):
    """BASELINE C4 at full size through the REFERENCE: cookie.build_ht_operator on the
    64 x 64 P1 subdomain matrices, build_rhs_htensor, and solvers.cg_solve for 20
    steps on a SerialBackend whose truncate uses eps = 1e-6 * ||Y|| (cap 50) -- the
    relative-tolerance wrapper C4 asks for (the reference takes an absolute eps).
    Takes a few minutes; writes c4_cg.npz (the residual traces and max ranks)."""
    import scipy.sparse as sp
    from htucker import arith as ref_ar
    from htucker import cookie
    from htucker import solvers as ref_solvers

    from paper_1708_03340_b200 import problems

    class RelBackend(ref_solvers.SerialBackend):
        def truncate(self, x, ctl):
            return ref_ar.truncate(x, ref.TruncationControl(eps=1e-6 * ref_ar.norm(x), max_rank=50))

    mats, load = problems.p1_diffusion_matrices(cells=64)
    # broken: distinct grids per parameter, so no two parameter modes are interchangeable
    # and the kept singular subspaces at the rank cap are unique
    grids = problems.distinct_parameter_grids(points=16) if broken else problems.parameter_grids(points=16)
    op = cookie.build_ht_operator([sp.csr_matrix(mats[0].shape)] + mats, grids)
    rhs = cookie.build_rhs_htensor(load, grids)
    cfg = ref_solvers.SolverConfig(truncation=ref.TruncationControl(eps=1.0, max_rank=50), eps_stop=1e-12,
                                   max_cg_steps=20)
    x, trace = ref_solvers.cg_solve(op, rhs, cfg, backend=RelBackend())
    out = {"meta": meta(),
           "internal": np.array([e.internal_residual for e in trace.entries]),
           "true_rel": np.array([e.true_rel_residual for e in trace.entries]),
           "max_rank": np.array([e.max_rank for e in trace.entries]),
           "ranks_X": np.array([x.rank(t) for t in range(1, 19)])}
    np.savez_compressed(os.path.join(OUT, "c4_cg_distinct.npz" if broken else "c4_cg.npz"), **out)


def golden_readouts():
    """The reference's parameter-direction readouts (cookie.extract_solution /
    parameter_mean) on a seeded Gaussian d=10 tensor of the cookie shape (nine
    16-point parameter modes, spatial mode last): pins the oracle's restatement."""
    from htucker import cookie

    tree = orc.balanced_tree(10)
    x = orc.gaussian_htensor(tree, [16] * 9 + [40], 6, seed=31)
    xr = to_ref(x)
    out = {"meta": meta()}
    pack("X", x, out)
    rng = np.random.default_rng(5)
    idx = [tuple(int(v) for v in rng.integers(0, 16, 9)) for _ in range(3)]
    out["idx"] = np.array(idx)
    for q, ii in enumerate(idx):
        out[f"sol/{q}"] = np.asarray(cookie.extract_solution(xr, ii))
    out["mean"] = np.asarray(cookie.parameter_mean(xr))
    ws = [rng.random(16) for _ in range(9)]
    out["weights"] = np.array(ws)
    out["wmean"] = np.asarray(cookie.parameter_mean(xr, ws))
    np.savez_compressed(os.path.join(OUT, "readouts.npz"), **out)


def golden_spec():
    """Known answers quoted in the SPEC."""
    q, r = ref_kernels.reduced_qr(np.array([[3.0], [4.0]]))
    v, lam = ref_kernels.sym_eig_desc(np.array([[2.0, 1.0], [1.0, 2.0]]))
    t5 = ref.build_balanced_tree(5)
    out = {"meta": meta(), "qr_q": q, "qr_r": r, "eig_lam": lam,
           "tree5_intervals": np.array([n.interval for n in t5.nodes]),
           "tree5_fathers": np.array([-1 if n.father is None else n.father for n in t5.nodes]),
           "tree10_levels": np.array([n.level for n in ref.build_balanced_tree(10).nodes]),
           "tree10_intervals": np.array([n.interval for n in ref.build_balanced_tree(10).nodes])}
    np.savez_compressed(os.path.join(OUT, "spec.npz"), **out)


def golden_io():
    """HT01 bytes (format.py:467-553) and evaluate_entry values (arith.py:221-243) of
    the reference on a ragged d=5 tree with mixed leaf sizes and ranks."""
    tr = orc.balanced_tree(5)
    ranks = {1: 3, 2: 4, 3: 2, 4: 3, 5: 2, 6: 3, 7: 2, 8: 3}
    sizes = {1: 4, 2: 5, 3: 3, 4: 6, 5: 2}
    rng = np.random.default_rng(np.random.PCG64(77))
    rt = ref.build_balanced_tree(5)
    U, B = {}, {}
    for node in rt.nodes:
        t = node.index
        if node.is_root:
            root = rng.standard_normal((ranks[node.sons[0]], ranks[node.sons[1]]))
        elif node.is_leaf:
            U[t] = rng.standard_normal((sizes[node.dim], ranks[t]))
        else:
            B[t] = rng.standard_normal((ranks[t], ranks[node.sons[0]], ranks[node.sons[1]]))
    x = ref.HTensor(rt, U, B, root)
    blob = ref.serialize(x)
    idx = np.array([[0, 0, 0, 0, 0], [3, 4, 2, 5, 1], [1, 2, 0, 3, 1], [2, 0, 1, 4, 0]])
    vals = np.array([ref_arith.evaluate_entry(x, tuple(i)) for i in idx])
    out = {"meta": meta(), "blob": np.frombuffer(blob, dtype=np.uint8), "idx": idx, "vals": vals}
    pack("x", x, out)
    np.savez_compressed(os.path.join(OUT, "io.npz"), **out)


if __name__ == "__main__":
    golden_io()
    golden_spec()
    golden_small()
    golden_shrink()
    golden_c1()
    golden_c3_small()
    golden_c2_d8()
    golden_cg()
    golden_c4_operator()
    golden_readouts()
    if "--c4" in sys.argv:  # minutes of CPU time
        golden_c4_cg()
        golden_c4_cg(broken=True)
    if "--large" in sys.argv:  # minutes of CPU time
        for d in (64, 128, 256):
            golden_c2_large(d)
        golden_c5_shape()
    print("golden fixtures written to", OUT)
