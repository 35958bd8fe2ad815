// QR of short-wide frames (m < K, the rank-shrink case of reference
// arith.py:280-297 / kernels.py:24-32: Q is m x m, R is m x K, diag(R) >= 0).
// One CTA per node holds the whole m x K block -- in shared memory when it fits
// (<= 200 KB), else in a global scratch (L2-resident) -- so neither K nor m (<= 1024)
// is limited to the tall-QR kernels' 112.  Unblocked Householder: reflector j by one
// warp, then every thread updates whole columns; Q accumulated backwards from I_m.
// A rare path (rank shrink at wide ranks): latency, not throughput, matters.
#include <cmath>

#include "prof.cuh"
#include "qr_wide.cuh"

namespace ht {
namespace {

constexpr int WT = 256;
constexpr int MAXD = 32;

struct WideBatch {
  int count;
  int begin[MAXD + 1];
  QrProblem d[MAXD];
};

__global__ void __launch_bounds__(WT) qr_wide_kernel(const __grid_constant__ WideBatch b) {
  extern __shared__ double sm[];
  int di = 0;
  while (di + 1 < b.count && (int)blockIdx.x >= b.begin[di + 1]) ++di;
  const QrProblem& q = b.d[di];
  const int nd = blockIdx.x - b.begin[di];
  const int m = q.m, K = q.K, ap = K + 1;
  // the block lives in shared memory when it fits, else in the node's global scratch
  double* A = q.wide_ws ? q.wide_ws + nd * q.wide_ws_node : sm;  // m x ap (row-major)
  double* V = A + (size_t)m * ap;  // m x m: reflector j in column j (rows j..m-1), 1 on the diagonal
  double* tau = V + m * m;        // m
  double* Qs = tau + m;           // m x m
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Ag = q.A + nd * q.a_node;
  for (int e = tid; e < m * K; e += WT) {
    const int r = e / K, c = e - r * K;
    A[r * ap + c] = Ag[(long long)r * q.a_r + (long long)c * q.a_c];
  }
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    if (warp == 0) {
      double ss = 0.0;
      for (int r = j + 1 + lane; r < m; r += 32) ss = fma(A[r * ap + j], A[r * ap + j], ss);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const double alpha = A[j * ap + j];
      double t = 0.0, beta = alpha, scale = 0.0;
      if (ss > 0.0) {
        beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      for (int r = j + lane; r < m; r += 32) V[r * m + j] = r == j ? 1.0 : A[r * ap + j] * scale;
      if (lane == 0) {
        tau[j] = t;
        A[j * ap + j] = beta;
      }
    }
    __syncthreads();
    const double tj = tau[j];
    if (tj != 0.0)
      for (int c = j + 1 + tid; c < K; c += WT) {
        double w = 0.0;
        for (int r = j; r < m; ++r) w = fma(V[r * m + j], A[r * ap + c], w);
        w *= tj;
        for (int r = j; r < m; ++r) A[r * ap + c] = fma(-w, V[r * m + j], A[r * ap + c]);
      }
    __syncthreads();
  }
  // Q = H_0 ... H_{m-1} I: apply in reverse to the identity, one column per thread
  for (int c = tid; c < m; c += WT) {
    for (int r = 0; r < m; ++r) Qs[r * m + c] = r == c ? 1.0 : 0.0;
    for (int j = m - 1; j >= 0; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      double w = 0.0;
      for (int r = j; r < m; ++r) w = fma(V[r * m + j], Qs[r * m + c], w);
      w *= tj;
      for (int r = j; r < m; ++r) Qs[r * m + c] = fma(-w, V[r * m + j], Qs[r * m + c]);
    }
  }
  __syncthreads();
  // sign fix diag(R) >= 0 (kernels.py:31-32): row j of R and column j of Q
  double* Ro = q.R + nd * q.r_node;
  double* Qo = q.Q + nd * q.q_node;
  for (int e = tid; e < m * K; e += WT) {
    const int r = e / K, c = e - r * K;
    const double sg = A[r * ap + r] < 0.0 ? -1.0 : 1.0;
    Ro[(long long)r * q.r_ld + c] = c >= r ? sg * A[r * ap + c] : 0.0;
  }
  for (int e = tid; e < m * m; e += WT) {
    const int r = e / m, c = e - r * m;
    const double sg = A[c * ap + c] < 0.0 ? -1.0 : 1.0;
    Qo[(long long)r * q.q_r + (long long)c * q.q_c] = sg * Qs[r * m + c];
  }
}

size_t wide_smem(int m, int K) { return sizeof(double) * ((size_t)m * (K + 1) + 2 * (size_t)m * m + m); }
constexpr size_t kWideSmem = 200 * 1024;

bool g_attr = false;

}  // namespace

bool qr_wide_eligible(const QrProblem& q) { return q.m >= 1 && q.m < q.K && q.m <= 1024; }

long long qr_wide_ws_doubles(const QrProblem& q) {
  return wide_smem(q.m, q.K) <= kWideSmem ? 0 : (long long)(wide_smem(q.m, q.K) / sizeof(double)) + 32;
}

int qr_wide_batched(std::vector<QrProblem>& probs, cudaStream_t stream) {
  if (!g_attr) {
    HT_CUDA_CHECK(cudaFuncSetAttribute(qr_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    g_attr = true;
  }
  size_t i = 0;
  while (i < probs.size()) {
    WideBatch b;
    b.count = 0;
    int blocks = 0;
    size_t smem = 0;
    while (i < probs.size() && b.count < MAXD) {
      const QrProblem& p = probs[i++];
      if (!qr_wide_eligible(p) || (wide_smem(p.m, p.K) > kWideSmem && !p.wide_ws)) {
        set_error("qr_wide: frame outside the wide QR (m < K, m <= 1024, scratch for large blocks)");
        return kErrUnsupported;
      }
      b.begin[b.count] = blocks;
      blocks += p.nodes;
      if (!p.wide_ws) smem = std::max(smem, wide_smem(p.m, p.K));
      b.d[b.count++] = p;
    }
    if (!b.count) continue;
    b.begin[b.count] = blocks;
    double flops = 0;
    for (int q = 0; q < b.count; ++q)
      flops += b.d[q].nodes * (2.0 * b.d[q].K * b.d[q].m * b.d[q].m - 2.0 / 3.0 * b.d[q].m * b.d[q].m * b.d[q].m);
    ProfToken tok = prof_begin(stream);
    qr_wide_kernel<<<blocks, WT, smem, stream>>>(b);
    HT_LAUNCH_CHECK();
    prof_end(tok, "qr_wide", stream, flops, 0.0);
  }
  return kOk;
}

}  // namespace ht
