// Grouped, doubly-batched, strided FP64 GEMM on DMMA tensor cores (sm_100a).
//
// One descriptor describes   C[b] = alpha * sum_{o<KO} sum_{k<K} A[b](m,o,k) B[b](o,k,n) + beta * C[b]
// for a two-level batch b = (b2, b1).  Every operand is addressed through
// explicit element strides, so the mode products, reduced-Gramian contractions
// and projections of the HT arithmetic (reference arith.py:109-170,
// kernels.py:92-121) are all expressed WITHOUT materialising transposes or
// M_{2,3} reshapes: the C-order bytes of a transfer tensor already are the
// column-major (k1*k2 x k_t) matrix.
#pragma once

#include <vector>

#include "common.cuh"

namespace ht {

struct GemmDesc {
  const double* A;
  const double* B;
  double* C;  // output, or the split-K partial buffer when splits > 1
  long long a_m, a_k, a_o, a_b1, a_b2;
  long long b_k, b_n, b_o, b_b1, b_b2;
  long long c_m, c_n, c_b1, c_b2;
  int M, N, K, KO;
  int nb1, nb2;
  int splits;
  int tiles_m, tiles_n;
  int block_begin;
  int a_tri;  // 0 dense; 1 unit-lower in (m,k); 2 unit-upper in (m,k); 3 identity (A not read)
  int b_tri;  // 0 dense; 1 unit-lower in (k,n): stored for k > n, 1 on the diagonal, 0 above
  double alpha, beta;
  const int* active;  // optional device flag: the GEMM is skipped (every CTA exits) when *active == 0
  int sym;  // C is symmetric (M == N; e.g. A^T A or a reduced Gramian): the long-reduction
            // kernel computes the upper-triangle 16 x 16 blocks only and mirrors them
};

// Sum the split-K partials [splits][batch][M][N] into C (optionally (X+X^T)/2).
struct ReduceDesc {
  const double* P;
  double* C;
  long long c_m, c_n, c_b1, c_b2;
  int S, M, N, nb1, nb2;
  int sym;
  double alpha, beta;
  const int* active;  // optional device flag, as in GemmDesc
};

// Launch a set of GEMMs (any number; split into launches of <= kMaxGemmDescs).
// count_flops = false for launches whose work is conditional on a device flag (the
// profiler then books their time but no algorithmic flops).
int gemm_grouped(std::vector<GemmDesc>& descs, cudaStream_t stream, const char* tag = "gemm_dmma",
                 bool count_flops = true);
// CTA tiles one M x N output uses (tile shape chosen per descriptor)
int gemm_tiles(int M, int N);
int reduce_partials(const std::vector<ReduceDesc>& descs, cudaStream_t stream, const char* tag = "reduce_partials");

constexpr int kMaxGemmDescs = 64;  // one launch for a d=64 level's 2 x 32 son Gramians (params < 32 KB)
constexpr int kGemmBM = 64, kGemmBN = 64, kGemmBK = 16;

// Host helper: a plain (single-batch, KO=1) GEMM descriptor with all strides.
inline GemmDesc gemm_desc(const double* A, long long a_m, long long a_k,
                          const double* B, long long b_k, long long b_n,
                          double* C, long long c_m, long long c_n,
                          int M, int N, int K, double alpha = 1.0, double beta = 0.0) {
  GemmDesc d{};
  d.A = A; d.B = B; d.C = C;
  d.a_m = a_m; d.a_k = a_k;
  d.b_k = b_k; d.b_n = b_n;
  d.c_m = c_m; d.c_n = c_n;
  d.M = M; d.N = N; d.K = K; d.KO = 1;
  d.nb1 = 1; d.nb2 = 1; d.splits = 1;
  d.alpha = alpha; d.beta = beta;
  return d;
}

}  // namespace ht
