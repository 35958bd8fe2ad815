"""Host restatement of two-sided cyclic Jacobi with the Demmel-Veselic stopping rule
(test infrastructure): eigenvalues of graded symmetric positive definite matrices to
high RELATIVE accuracy, where LAPACK's dsyevd (the reference's eigh) only guarantees
accuracy relative to ||S||.  Vectorised over the disjoint rotations of a round."""

import numpy as np


def jacobi_eigvals(S: np.ndarray, max_sweeps: int = 60) -> np.ndarray:
    A = np.array(S, dtype=np.float64)
    K = A.shape[0]
    n = K + (K & 1)
    if n != K:  # pad to even order with a decoupled zero
        B = np.zeros((n, n))
        B[:K, :K] = A
        A = B
    tol = np.finfo(np.float64).eps * max(K, 8)
    players = np.arange(n)
    for _ in range(max_sweeps):
        rotated = False
        for r in range(n - 1):
            # round-robin: player 0 fixed, the others rotate
            ring = np.concatenate([[0], np.roll(players[1:], r)])
            p, q = ring[: n // 2], ring[n // 2:][::-1]
            p, q = np.minimum(p, q), np.maximum(p, q)
            app, aqq, apq = A[p, p], A[q, q], A[p, q]
            act = (np.abs(apq) > tol * np.sqrt(np.abs(app)) * np.sqrt(np.abs(aqq))) & (np.abs(apq) > 1e-300)
            if not act.any():
                continue
            rotated = True
            p, q, app, aqq, apq = p[act], q[act], app[act], aqq[act], apq[act]
            tau = (aqq - app) / (2.0 * apq)
            t = np.where(tau >= 0, 1.0, -1.0) / (np.abs(tau) + np.sqrt(1.0 + tau * tau))
            c = 1.0 / np.sqrt(1.0 + t * t)
            s = t * c
            Ap, Aq = A[:, p].copy(), A[:, q].copy()
            A[:, p] = c * Ap - s * Aq
            A[:, q] = s * Ap + c * Aq
            Ap, Aq = A[p, :].copy(), A[q, :].copy()
            A[p, :] = c[:, None] * Ap - s[:, None] * Aq
            A[q, :] = s[:, None] * Ap + c[:, None] * Aq
        if not rotated:
            break
    lam = np.diag(A)[:K]
    return np.sort(np.maximum(lam, 0.0))[::-1]


def graded_spd(K: int, decades: float, seed: int) -> np.ndarray:
    """S = D M D: M a well-conditioned SPD matrix (unit diagonal), D = diag of
    10^-(decades * i / K) in a random order -- eigenvalues spread over 2*decades
    decades, each determined to O(K eps kappa(M)) relative accuracy by the entries."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((K, K))
    M = np.eye(K) + 0.5 * (G @ G.T) / K
    dm = np.sqrt(np.diag(M))
    M = M / dm[:, None] / dm[None, :]
    d = 10.0 ** (-decades * rng.permutation(K) / K)
    return d[:, None] * M * d[None, :]
