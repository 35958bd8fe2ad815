// Stationary-operand streaming GEMM (FP64 DMMA):  C = alpha * X S + beta * C
// for a tall streamed operand X (M x K) and a small stationary operand S (K x N,
// K <= 128, N <= 104) -- the shape of every mode product / projection / Q = A R^-1
// of the HT truncation (reference arith.py:109-170, kernels.py:92-121).
//
// Persistent CTAs (16 warps) own a contiguous range of 128-row output tiles of one
// or more jobs; S stays in shared memory for a whole job, X flows through a 4-stage
// cp.async ring that runs continuously across tile boundaries (the epilogue of one
// tile overlaps the loads of the next), so there is no per-tile pipeline fill and
// no per-tile re-read of S.
//
// Row index m of X and C may be two-level, m = m_hi * M_lo + m_lo, each level with
// its own stride (slices of a transfer tensor); the batch index selects a job
// (X, S, C base pointers advance by their job strides).
#pragma once

#include <vector>

#include "common.cuh"

namespace ht {

struct SsDesc {
  const double* X;
  const double* S;
  double* C;
  long long x_hi, x_lo, x_k, x_job;  // X(m, k) = X[job*x_job + (m / M_lo)*x_hi + (m % M_lo)*x_lo + k*x_k]
  long long s_k, s_n, s_job;         // S(k, n) = S[job*s_job + k*s_k + n*s_n]
  long long c_hi, c_lo, c_n, c_job;  // C(m, n) likewise
  int M, M_lo, N, K, jobs;
  double alpha, beta;
  const int* active;  // optional device flag: skip when *active == 0
  int s_tri;          // 0 dense S; 1: S(k, n) = 0 for k < n; 2: S(k, n) = 0 for k > n
                      // (triangular factors: the zero (k16 x n8) MMA blocks are skipped)
};

constexpr int kSsMaxK = 128;
constexpr int kSsMaxN = 104;

// Launch a set of descriptors (grouped by N <= 56 / N <= 104 variants).
int ss_gemm(std::vector<SsDesc>& descs, cudaStream_t stream, const char* tag, bool count_flops = true);

// Helper for a single-level (M_lo = M) descriptor.
inline SsDesc ss_desc(const double* X, long long x_m, long long x_k, const double* S, long long s_k, long long s_n,
                      double* C, long long c_m, long long c_n, int M, int N, int K) {
  SsDesc d{};
  d.X = X; d.S = S; d.C = C;
  d.x_hi = 0; d.x_lo = x_m; d.x_k = x_k;
  d.s_k = s_k; d.s_n = s_n;
  d.c_hi = 0; d.c_lo = c_m; d.c_n = c_n;
  d.M = M; d.M_lo = M; d.N = N; d.K = K; d.jobs = 1;
  d.alpha = 1.0; d.beta = 0.0;
  return d;
}

}  // namespace ht
