// Batched tall-skinny Householder QR (sign-fixed, explicit thin Q) for the
// leaf frames and the M_{2,3}-matricised transfer tensors -- the replacement
// for reference kernels.py:24-32 (numpy dgeqrf + dorgqr, then diag(R) >= 0).
//
// Algorithm: tree TSQR, Householder everywhere (no Gram / Cholesky step, so
// exactly rank-deficient frames such as add(A, A) keep an orthonormal Q).
//   1. Each node is cut into P row blocks of <= 128 rows (all but the last
//      have >= K rows).  One CTA per block runs dense Householder QR with the
//      block held in registers (16 warps x 8 rows, lanes x 4 columns), two
//      CTA barriers per reflector (the dots of reflector j+1 are fused into
//      the update of reflector j), and builds the compact-WY factor T
//      (H_0..H_{K-1} = I - Y T Y^T) in shared memory.
//   2. Block R factors are merged by a binary tree of [R_a; R_b] steps
//      (reflector heads in R_a rows, tails in R_b), one launch per round for
//      all nodes of a tree level.
//   3. R is sign-fixed; diag(sign) seeds Q.  Q is then formed top-down with
//      batched DMMA GEMMs only: per tree pair X = T W_a, W_b = -V_b X,
//      W_a -= X; per block Q = [W; 0] - Y T (Y_top^T W).
#pragma once

#include <vector>

#include "common.cuh"

namespace ht {

struct QrProblem {
  // A(row, col) of node nd: A + nd*a_node + row*a_r + col*a_c  (m x K), read only
  const double* A;
  long long a_r, a_c, a_node;
  // Q(row, col) output (m x kq, kq = min(m, K))
  double* Q;
  long long q_r, q_c, q_node;
  // R output, row-major kq x K (leading dimension r_ld)
  double* R;
  long long r_ld, r_node;
  int m, K, nodes;
  // optional: reflector storage (column-major, ld m, node stride m*K).  May alias
  // A when A is itself column-major scratch (a_r == 1, a_c == m): the kernel reads
  // a block into registers before writing its reflectors back.
  double* V;
  // optional (Cholesky-QR path only): implicit Q.  The factor kernel writes R^{-1}
  // (K x K row-major, node stride K*K) here and the first-pass Q = A R^{-1} is NOT
  // formed: the caller keeps A and folds R^{-1} into its next small operand (see
  // driver.cu, "implicit Q").  A node that needs the second pass gets an explicit Q
  // (written to Q, which then aliases A) and R^{-1} := I.
  double* rinv = nullptr;

  // --- filled by qr_plan() ---
  int P, rpc;
  long long v_node, st_node, t_node, x_node;
  double* Rst;  // P x K x K: block R factors, then combine reflector tails
  double* Tst;  // 2P x K x K: T factors of blocks [0,P) and of combine steps [P + b]
  double* X;    // 3P x K x K: GEMM scratch of the Q formation
  bool own_v;
  // wide-frame QR (qr_wide.cu) with the block in global memory: scratch per node
  double* wide_ws = nullptr;
  long long wide_ws_node = 0;
};

constexpr int kQrMaxK = 112;  // register/shared-memory resident path

int qr_plan(QrProblem& p);
long long qr_workspace_doubles(const QrProblem& p);
void qr_bind_workspace(QrProblem& p, double* ws);
int qr_batched(std::vector<QrProblem>& probs, cudaStream_t stream);

}  // namespace ht
