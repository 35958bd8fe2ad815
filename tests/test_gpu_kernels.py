"""Node-kernel parity on the B200 through the C ABI: DMMA GEMM, batched
Householder QR (reduced_qr, kernels.py:24-32), batched Jacobi eig
(sym_eig_desc, kernels.py:35-54).  Floating-point tolerances are stated per test."""

import ctypes

import numpy as np
import pytest

from oracle import htucker_oracle as orc

pytestmark = pytest.mark.gpu


def _t():
    import torch

    return torch


@pytest.fixture(scope="module")
def lib(cuda_ok):
    from paper_1708_03340_b200 import _lib

    return _lib.load()


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (64, 64, 16), (100, 100, 100), (129, 65, 257),
                                   (10000, 100, 100), (100, 100, 10000)])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_gemm_vs_fp64_reference(lib, M, N, K, ta, tb):
    torch = _t()
    from paper_1708_03340_b200 import _lib

    g = torch.Generator().manual_seed(M * 131 + N * 7 + K)
    A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, generator=g).cuda()
    B = torch.randn((N, K) if tb else (K, N), dtype=torch.float64, generator=g).cuda()
    Av = A.t() if ta else A
    Bv = B.t() if tb else B
    C = torch.randn(M, N, dtype=torch.float64, generator=g).cuda()
    ref = 0.5 * (Av.cpu() @ Bv.cpu()) + 2.0 * C.cpu()
    _lib.check(lib.ht_gemm_strided(M, N, K, 1, 0.5, Av.data_ptr(), Av.stride(0), Av.stride(1), 0, Bv.data_ptr(),
                                   Bv.stride(0), Bv.stride(1), 0, 2.0, C.data_ptr(), C.stride(0), C.stride(1), 0,
                                   _lib.stream_handle()))
    torch.cuda.synchronize()
    # fp64: |err| <= 1e-13 * (|A||B| scale) -- accumulation order differs from the CPU
    tol = 1e-13 * np.sqrt(K) * 4
    np.testing.assert_allclose(C.cpu().numpy(), ref.numpy(), rtol=0, atol=tol * max(1.0, np.abs(ref.numpy()).max()))


def _qr_dev(lib, A_np, col_major=False, nodes=1):
    torch = _t()
    from paper_1708_03340_b200 import _lib

    m, K = A_np.shape[-2:]
    kq = min(m, K)
    if col_major:
        A = torch.as_tensor(np.ascontiguousarray(np.swapaxes(A_np, -1, -2))).cuda()  # (nodes, K, m)
        a_r, a_c = 1, m
        Q = torch.empty((nodes, kq, m), dtype=torch.float64, device="cuda")
        q_r, q_c = 1, m
    else:
        A = torch.as_tensor(np.ascontiguousarray(A_np)).cuda()
        a_r, a_c = K, 1
        Q = torch.empty((nodes, m, kq), dtype=torch.float64, device="cuda")
        q_r, q_c = kq, 1
    R = torch.empty((nodes, kq, K), dtype=torch.float64, device="cuda")
    nb = ctypes.c_size_t(0)
    _lib.check(lib.ht_qr_workspace_size(m, K, nodes, ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    _lib.check(lib.ht_qr_batched(m, K, nodes, A.data_ptr(), a_r, a_c, m * K, Q.data_ptr(), q_r, q_c, m * kq,
                                 R.data_ptr(), K, kq * K, ws.data_ptr(), ws.numel(), _lib.stream_handle()))
    torch.cuda.synchronize()
    Qn = Q.cpu().numpy()
    if col_major:
        Qn = np.swapaxes(Qn, -1, -2)
    return Qn, R.cpu().numpy()


@pytest.mark.parametrize("m,K,col", [(64, 20, False), (1000, 100, False), (256, 60, False), (10000, 100, True),
                                     (400, 20, True), (3600, 60, True), (16, 40, False), (5, 3, False),
                                     (130, 112, False), (1, 1, False), (2000, 1, True),
                                     # odd widths (block Gram-Schmidt panels of odd ranks, e.g. K=150 -> 2 x 75)
                                     (300, 75, True), (300, 75, False), (300, 77, True), (500, 101, True),
                                     (130, 111, False), (200, 65, True), (22500, 75, True)])
def test_qr_matches_reduced_qr(lib, m, K, col):
    rng = np.random.default_rng(m * 7 + K)
    nodes = 3
    A = rng.standard_normal((nodes, m, K))
    Q, R = _qr_dev(lib, A, col_major=col, nodes=nodes)
    for i in range(nodes):
        q_ref, r_ref = orc.qr_signfixed(A[i])
        kq = min(m, K)
        # reconstruction and orthonormality (fp64, Householder: O(eps) backward error)
        np.testing.assert_allclose(Q[i] @ R[i], A[i], rtol=0, atol=1e-12 * np.abs(A[i]).max() * np.sqrt(m))
        np.testing.assert_allclose(Q[i].T @ Q[i], np.eye(kq), rtol=0, atol=1e-13 * np.sqrt(m))
        assert np.all(np.diag(R[i]) >= 0.0)
        assert np.allclose(np.tril(R[i], -1), 0.0)
        # unique sign-fixed factors: entrywise agreement with LAPACK
        if kq == K:
            np.testing.assert_allclose(R[i], r_ref, rtol=0, atol=1e-12 * np.abs(r_ref).max())
            np.testing.assert_allclose(Q[i], q_ref, rtol=0, atol=1e-11)


def test_qr_rank_deficient_stays_orthonormal(lib):
    # add(A, A)-style duplicated columns: Gram/Cholesky QR would fail here
    rng = np.random.default_rng(3)
    half = rng.standard_normal((2, 1000, 50))
    A = np.concatenate([half, half], axis=2)
    Q, R = _qr_dev(lib, A, nodes=2)
    for i in range(2):
        np.testing.assert_allclose(Q[i].T @ Q[i], np.eye(100), rtol=0, atol=1e-12)
        np.testing.assert_allclose(Q[i] @ R[i], A[i], rtol=0, atol=1e-11)


def _syev(lib, S):
    torch = _t()
    from paper_1708_03340_b200 import _lib

    nodes, K, _ = S.shape
    Sd = torch.as_tensor(np.ascontiguousarray(S)).cuda()
    V = torch.empty_like(Sd)
    lam = torch.empty((nodes, K), dtype=torch.float64, device="cuda")
    rc = lib.ht_syev_batched(K, nodes, Sd.data_ptr(), V.data_ptr(), lam.data_ptr(), _lib.stream_handle())
    _lib.check(rc)
    return V.cpu().numpy(), lam.cpu().numpy()


@pytest.mark.parametrize("K", [1, 2, 3, 10, 20, 33, 60, 100, 112])
def test_syev_matches_sym_eig_desc(lib, K):
    rng = np.random.default_rng(K)
    nodes = 4
    X = rng.standard_normal((nodes, K + 5, K))
    S = np.einsum("nij,nik->njk", X, X)
    V, lam = _syev(lib, S)
    for i in range(nodes):
        v_ref, l_ref = orc.eig_desc(S[i])
        np.testing.assert_allclose(lam[i], l_ref, rtol=1e-12, atol=1e-13 * l_ref[0])
        np.testing.assert_allclose(V[i].T @ V[i], np.eye(K), atol=1e-13)
        np.testing.assert_allclose(V[i] @ np.diag(lam[i]) @ V[i].T, S[i], atol=1e-12 * l_ref[0])
        # eigenvectors up to sign (gauge, kernels.py:51-54)
        sgn = np.sign(np.sum(V[i] * v_ref, axis=0))
        np.testing.assert_allclose(V[i] * sgn, v_ref, atol=1e-9)


def test_syev_graded_relative_accuracy(lib):
    # graded PSD matrix D A D: Jacobi keeps small eigenvalues to high relative accuracy
    rng = np.random.default_rng(11)
    K = 20
    X = rng.standard_normal((K + 3, K))
    A = X.T @ X
    d = np.logspace(0, -10, K)
    S = (d[:, None] * A * d[None, :])[None]
    _, lam = _syev(lib, S)
    ref = np.linalg.eigvalsh(S[0])[::-1]  # dsyevd is also accurate here (graded, well-ordered)
    np.testing.assert_allclose(lam[0], ref, rtol=1e-8)


@pytest.mark.parametrize("K", [80, 113, 150, 301])
def test_syev_graded_relative_accuracy_any_rank(lib, K):
    """Graded S = D M D (eigenvalues over 16 decades, randomly placed): the Jacobi
    kernels -- shared-memory up to K = 112, global scratch beyond -- deliver every
    eigenvalue to relative accuracy (against the host restatement of the same method,
    tests/jacobi_host.py; LAPACK's dsyevd is only accurate relative to ||S|| here)."""
    from tests.jacobi_host import graded_spd, jacobi_eigvals

    S = np.stack([graded_spd(K, 8, K + i) for i in range(2)])
    V, lam = _syev(lib, S)
    for i in range(2):
        ref = jacobi_eigvals(S[i])
        assert ref[-1] < 1e-14 * ref[0]
        np.testing.assert_allclose(lam[i], ref, rtol=1e-11)
        np.testing.assert_allclose(V[i].T @ V[i], np.eye(K), atol=1e-13)


def test_syev_rejects_nonsymmetric(lib):
    S = np.array([[[1.0, 2.0], [0.0, 1.0]]])
    with pytest.raises(ValueError):
        _syev(lib, S)


def test_qr_merge_keeps_every_node_of_irregularly_spaced_leaves(cuda_ok):
    """Leaf frames of one shape at irregular spacing (pairs 12 doubles apart, the pairs 96 /
    104 apart): the sweep merges each pair into a two-node QR problem, and the second
    merge pass (plan_qrs) must not fuse the two pairs into one re-strided problem that
    would drop a node of each (regression: NaN leaf frames)."""
    import torch

    import paper_1708_03340_b200 as htb
    from oracle import htucker_oracle as orc
    from tests.htconv import to_host

    tr = orc.balanced_tree(4)
    x = orc.gaussian_htensor(tr, 4, 3, 7)
    buf = torch.full((512,), float("nan"), dtype=torch.float64, device="cuda")
    offs = {3: 0, 4: 12, 5: 96, 6: 200}
    leaves = {}
    for t, o in offs.items():
        leaves[t] = buf[o:o + 12].view(4, 3)
        leaves[t].copy_(torch.from_numpy(x.U[t]))
    tree = htb.build_balanced_tree(4)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    xd = htb.HTensor(tree, leaves, {t: dev(b) for t, b in x.B.items()}, dev(x.root))
    for mode in ("householder", "auto"):
        htb.set_qr_mode(mode)
        try:
            o = to_host(htb.orthogonalize(xd))
        finally:
            htb.set_qr_mode("auto")
        ref = orc.orthogonalize(x)
        for (t, u), (_, v) in zip(o.arrays(), ref.arrays()):
            assert np.all(np.isfinite(u)), f"node {t} not written ({mode})"
            np.testing.assert_allclose(u, v, rtol=1e-10, atol=1e-12)
