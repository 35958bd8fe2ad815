// Batched tall-skinny Householder QR (sign-fixed, explicit thin Q) for the
// leaf frames and the M_{2,3} matricised transfer tensors -- the replacement
// for reference kernels.py:24-32 (numpy dgeqrf+dorgqr, R diagonal >= 0).
//
// Algorithm (communication-avoiding, all Householder, no Gram/Cholesky step so
// rank-deficient frames such as add(A, A) stay exactly orthonormal):
//   1. every node is cut into P row chunks (>= K rows each); one CTA per chunk
//      factors its first sub-block densely and then streams the remaining
//      sub-blocks through a "triangular head" Householder step against its
//      running R (flat TSQR inside the CTA);
//   2. the P chunk R factors are combined by a binary tree of [R_a; R_b]
//      Householder steps (one launch per round, all nodes of a level at once);
//   3. R is sign-fixed (R_jj >= 0) and the sign matrix seeds the backward
//      accumulation of Q: tree rounds top-down, then every chunk applies its
//      reflectors in reverse to produce its rows of Q.
#pragma once

#include <vector>

#include "common.cuh"

namespace ht {

struct QrProblem {
  // A(row, col) of node `nd`: A + nd*a_node + row*a_r + col*a_c   (m x K), read only
  const double* A;
  long long a_r, a_c, a_node;
  // Q(row, col) output (m x kq, kq = min(m, K))
  double* Q;
  long long q_r, q_c, q_node;
  // R output, row-major kq x K with leading dimension r_ld
  double* R;
  long long r_ld, r_node;
  int m, K, nodes;
  int P;  // requested row chunks per node (clamped by the planner)

  // --- filled by qr_plan() ---
  int rpc, ms0, ms, nsub_pc, nsub_total;
  long long v_node, tau_node, st_node;  // workspace strides per node (doubles)
  // --- filled by qr_bind_workspace() ---
  double* V;    // reflector tails, column-major ld = m
  double* tau;  // [nsub_total*K sub-block taus][P*K combine taus]
  double* Rst;  // P blocks K*K (chunk R factors, then combine tails)
  double* W;    // P blocks K*K (backward-accumulation seeds)
};

constexpr int kQrMaxK = 112;  // shared-memory resident path

// Choose chunking / sub-block sizes and the per-node workspace footprint.
int qr_plan(QrProblem& p, int target_ctas);
long long qr_workspace_doubles(const QrProblem& p);
void qr_bind_workspace(QrProblem& p, double* ws);

// Run all problems (each a group of same-shaped nodes) on `stream`.
int qr_batched(std::vector<QrProblem>& probs, cudaStream_t stream);

}  // namespace ht
