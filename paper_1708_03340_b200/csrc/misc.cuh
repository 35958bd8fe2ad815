// HBM-bound elementwise kernels of the HT arithmetic: the Lemma-3 block
// embedding of add (arith.py:173-192), the Kronecker transfer tensors of the
// operator application (arith.py:204-213), the leaf images W_r U of diagonal /
// CSR operator columns (arith.py:195-201, format.py:167-173), scaling and dots.
#pragma once

#include <vector>

#include "common.cuh"

namespace ht {

// out(i0,i1,i2) over dims D = A placed at 0 (dims a) + C placed at offset o (dims c), 0 elsewhere.
struct EmbedDesc {
  double* out;
  const double* A;
  const double* C;
  int D0, D1, D2;
  int a0, a1, a2;
  int c0, c1, c2;
  int o0, o1, o2;
  double alpha_c;  // scale applied to the C block
};
int embed_batched(const std::vector<EmbedDesc>& descs, cudaStream_t stream);

// out[(p*ki+i), (q*kj+j), (r*kl+l)] = H[p,q,r] * B[i,j,l]
struct KronDesc {
  double* out;
  const double* H;
  const double* B;
  int kp, kq, kr;
  int ki, kj, kl;
};
int kron_batched(const std::vector<KronDesc>& descs, cudaStream_t stream);

// Stationary operands of a mode product applied to an unmaterialised Kronecker product
// F = H (x) B (arith.py:204-213 consumed in place): with R (ko x rb*ks row-major, ld ldr)
// the factor absorbed into the mode whose operator index is b,
//   E[a][c][J][j] = sum_b H[a,b,c] R[J, b*ks + j]        (ra x rc matrices of ko x ks)
// so that (F x_2 R)[(a,i), J, (c,l)] = sum_j E[a][c][J][j] B[i,j,l].
struct KronFactorDesc {
  const double* H;
  const double* R;
  double* E;
  int ra, rb, rc, ks, ko, ldr;
};
int kron_factor_batched(const std::vector<KronFactorDesc>& descs, cudaStream_t stream);

// Zero-fill of contiguous runs (the structurally zero slabs of a block-form sum's
// absorbed transfer tensors).
struct ZeroDesc {
  double* p;
  long long count;
};
int zero_batched(const std::vector<ZeroDesc>& descs, cudaStream_t stream);

// out (rows x cols row-major) = blockdiag_q(alpha_q * B_q), B_q (r_q x c_q) at (ro_q, co_q);
// `out` must be zero-filled first.
struct RootBlockDesc {
  const double* B;
  double alpha;
  int r, c, ro, co;
};
int root_blocks(double* out, int cols, const std::vector<RootBlockDesc>& blocks, cudaStream_t stream);

// Leaf operator column applied to U (n_in x k row-major), written into columns
// [col0, col0+k) of V (n_out x ldv row-major).  kind 1: diagonal, kind 2: CSR.
struct LeafApplyDesc {
  int kind;
  const double* vals;
  const int* indptr;
  const int* indices;
  const double* U;
  double* V;
  int n_out, k, ldv, col0;
};
int leaf_apply_batched(const std::vector<LeafApplyDesc>& descs, cudaStream_t stream);

int scale_copy(const double* x, double* y, long long n, double alpha, cudaStream_t stream);

// dst(r, c) = src(r, c) for rows x cols per node, arbitrary strides (layout changes)
struct Copy2dDesc {
  const double* src;
  double* dst;
  long long s_r, s_c, s_node, d_r, d_c, d_node;
  int rows, cols, nodes;
};
int copy2d_batched(const std::vector<Copy2dDesc>& descs, cudaStream_t stream);
// p[node * node_stride + i * K + j] = (i == j) for nodes x K x K (skipped when *active == 0)
int identity_batched(double* p, long long node_stride, int K, int nodes, const int* active, cudaStream_t stream);
// out[0] = sum_i a[i] * b[i]   (single CTA, deterministic order)
int dot(const double* a, const double* b, long long n, double* out, cudaStream_t stream);

}  // namespace ht

namespace ht {
// Entry evaluation (reference arith.py:221-243): for each multi-index b the leaf rows
// U_mu[i_mu, :] are combined upward through the transfer tensors in post-order; one
// CTA per entry, the rows of the open subtrees on a shared-memory stack.
constexpr int kEvalMaxNodes = 1023;
constexpr int kEvalMaxDims = 512;
struct EvalTree {
  int nn, d, kmax, depth;
  short post[kEvalMaxNodes];  // node ids in post-order (root last)
  short son1[kEvalMaxNodes], son2[kEvalMaxNodes], dim[kEvalMaxNodes];  // dim: 0-based (leaves)
  short k[kEvalMaxNodes];
  const double* p[kEvalMaxNodes];
  // optional per-dimension leaf weights: the leaf of dimension mu contributes the row
  // w[mu]^T U (w[mu] of length n[mu]) instead of U[idx[mu], :]
  const double* w[kEvalMaxDims];
  int n[kEvalMaxDims];
};
int evaluate_entries(const EvalTree& T, const long long* idx, long long B, double* out, cudaStream_t s);
}  // namespace ht
