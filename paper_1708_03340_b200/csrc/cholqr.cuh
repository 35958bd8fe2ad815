// Tall-skinny QR by Cholesky-QR2 on DMMA GEMMs -- the fast path of the
// orthogonalisation sweep (replaces reference kernels.py:24-32 reduced_qr for
// well-conditioned frames; the Householder path of qr.cuh is the fallback).
//
//   W1 = A^T A          (split-K DMMA GEMM)      R1 = chol(W1), Ri = R1^{-1}
//   Q1 = A Ri           (DMMA GEMM)
//   W2 = Q1^T Q1                                 R2 = chol(W2), Ri = R2^{-1}
//   Q  = Q1 Ri,  R = R2 R1
// The second pass only runs (decided on the device, per problem) when the power-
// iteration estimate of kappa(R1) exceeds 20; below that one pass already gives
// ||Q^T Q - I|| <~ 1e-14 (single-pass error ~1e-17 kappa^2 measured).
//
// For full-column-rank A the QR factorisation with diag(R) > 0 is unique, so the
// result is the sign-fixed Householder QR of the reference up to rounding.
// CholeskyQR2 is accurate to O(u) in orthogonality and residual while
// kappa(A) << u^{-1/2}; the factor kernel flags a node (atomicOr on `fail`) when
// a pivot loses more than 10 digits against its column norm, when anything is
// non-finite, or when W2 is not within 0.1 of the identity.  The caller then
// re-runs the whole sweep with Householder QR (exactly rank-deficient frames such
// as add(A, A) always take that route).
#pragma once

#include <vector>

#include "common.cuh"
#include "qr.cuh"

namespace ht {

constexpr int kCholMaxK = 128;  // K x (K+1) doubles resident in shared memory

struct CholQr {
  QrProblem q;  // addressing of A / Q / R (m, K, nodes, strides); q.V unused
  int S = 1;    // split-K of the two Gram GEMMs
  double *P = nullptr, *W = nullptr, *Q1 = nullptr, *R1 = nullptr, *R2 = nullptr, *Ri = nullptr;
};

bool cholqr_eligible(const QrProblem& q);
long long cholqr_workspace_doubles(const CholQr& c);
void cholqr_bind(CholQr& c, double* ws);
// Launch the sequence for all problems; *fail (device int) is OR-ed with 1 on any
// numerical red flag; need2 (device, cs.size() ints) carries the per-problem
// "second pass needed" decision between the kernels.  No host synchronisation.
// two_pass: always run the second pass (testing / ht_set_qr_mode(2)).
int cholqr_run(std::vector<CholQr>& cs, int* fail, int* need2, bool two_pass, cudaStream_t stream);

}  // namespace ht

namespace ht {

// Wide frames (K > kCholInPlaceK, m >= K): block Gram-Schmidt with
// re-orthogonalisation over panels of <= 104 columns, each panel by Cholesky-QR
// (adaptive second pass):  Q_J <- Q_J - Q_< (Q_<^T Q_J)  twice,  R_<J += both
// projections,  [Q_J, R_JJ] = CholQR(Q_J).  Works in place in the output Q.
struct CholBig {
  QrProblem q;
  int np = 0, pw = 0;  // panels, panel width (last panel may be narrower)
  int S = 1;           // split-K of the projection GEMMs
  double *P = nullptr, *Sb = nullptr, *Rp = nullptr;
  CholQr panel;        // workspace / plan of one Cholesky-QR panel (re-bound per panel)
  QrProblem hpanel;    // plan of one Householder-TSQR panel (re-planned per panel width)
  double* hws = nullptr;  // its workspace
};

bool cholbig_eligible(const QrProblem& q);
long long cholbig_workspace_doubles(CholBig& c);  // also fills np, pw, S
void cholbig_bind(CholBig& c, double* ws);
// householder: panels by Householder tree-TSQR (exactly rank-deficient panels keep an
// orthonormal Q), each followed by one more projection + TSQR so that the completion
// directions of deficient panels are orthogonal to the earlier panels too.
int cholbig_run(std::vector<CholBig>& cs, int* fail, int* need2, bool two_pass, cudaStream_t stream,
                bool householder = false);

}  // namespace ht
