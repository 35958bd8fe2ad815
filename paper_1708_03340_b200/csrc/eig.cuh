// Batched symmetric eigensolver (parallel cyclic two-sided Jacobi in shared
// memory) with the reference's post-processing fused in: stable descending
// order, eigenvalues clamped >= 0 (kernels.py:35-54) and the per-node rank
// choice of select_rank (arith.py:69-88) -- all on device, no host sync.
//
// Two kernels: the tridiagonal fast path (eig_tri.cu) and parallel cyclic Jacobi.
// Jacobi is kept for graded Gramians -- e.g. the C1 parity case, whose small
// eigenvalues (~1e-20 relative) are only determined to high RELATIVE accuracy by a
// Jacobi method with the |a_pq| <= eps*sqrt(|a_pp a_qq|) stopping rule
// (Demmel-Veselic) -- and for near-degenerate kept eigenvalues.
#pragma once

#include <vector>

#include "common.cuh"

namespace ht {

struct EigProblem {
  const double* S;  // symmetric K x K, row-major (ld K), node stride s_node
  long long s_node;
  double* V;        // eigenvectors, row-major K x K: V[i*K + j] = i-th entry of eigenvector j
  long long v_node;
  double* lam;      // K eigenvalues, descending, clamped >= 0
  long long l_node;
  int* rank;        // selected rank per node (may be null)
  int* status;      // device int, OR-ed with error bits (may be null)
  int K, nodes;
  double eps;       // absolute truncation accuracy; <= 0: none
  const double* eps_scale2;  // optional device scalar: the budget uses eps^2 * *eps_scale2
                             // (HT_CTL_RELATIVE_EPS: ||x||^2)
  int n_nonroot;    // 2d - 2
  int cap;          // rank cap; <= 0: none
  int* fallback;    // per-node flags (node stride 1): set by the tridiagonal fast path for
                    // nodes the Jacobi kernel must redo; null = Jacobi for every node
  double* work;     // global scratch for K > kEigMaxK (2 K (K+2) doubles per node), or null
  long long w_node;
  int graded_fallback;  // graded spectra go to Jacobi (relative accuracy of every sigma)
};

constexpr int kEigMaxK = 112;      // shared-memory paths (Jacobi; tridiagonal in smem)
constexpr int kEigMaxKBig = 512;   // tridiagonal path with the matrices in global scratch
// tridiagonal path: K x (K|1) matrix + kept-vector rows; Jacobi: A (n x n+1) + V^T (n x n+2), n = K rounded up to even
inline long long eig_work_doubles(int K) { return K > kEigMaxK ? 2LL * (K + 1) * (K + 3) + 8 : 0; }
constexpr int kEigStatusNotSymmetric = 1;
constexpr int kEigStatusNonConverged = 2;

// Eigensolver policy (process-wide): 0 = tridiagonal fast path with Jacobi for the
// nodes it flags (needs EigProblem::fallback), 1 = Jacobi only.
extern int g_eig_mode;

int eig_batched(std::vector<EigProblem>& probs, cudaStream_t stream);
int eig_tri_batched(std::vector<EigProblem>& probs, cudaStream_t stream);

}  // namespace ht
