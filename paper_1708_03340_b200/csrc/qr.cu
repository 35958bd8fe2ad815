// Batched streaming-TSQR Householder QR, see qr.cuh for the algorithm.
//
// Reference semantics: kernels.py:24-32 -- Householder QR (dlarfg reflectors as
// in LAPACK dgeqrf), explicit thin Q (dorgqr), then the sign fix diag(R) >= 0.
// Wide input (m < K) gives Q m x m and R m x K (kernels.py:27-28).
#include <algorithm>

#include "qr.cuh"
#include "prof.cuh"

namespace ht {

namespace {

constexpr int QT = 512;        // threads per CTA
constexpr int NW = QT / kWarp;  // 16 warps
constexpr int MAXD = 32;
constexpr int MS = 128;        // sub-block rows (4 rows per lane)
constexpr int NT = MS / kWarp;  // row slots per lane
constexpr int SMEM_MAX_BYTES = 227 * 1024;

struct QrDev {
  const double* A;
  long long a_r, a_c, a_node;
  double* Q;
  long long q_r, q_c, q_node;
  double* R;
  long long r_ld, r_node;
  double* V;
  double* tau;
  double* Rst;
  double* W;
  long long v_node, tau_node, st_node;
  int m, K, P, rpc, nsub_pc, nsub_total;
  int begin, per_node, nodes;
};

struct QrBatch {
  int count;
  int round;
  QrDev d[MAXD];
};

__device__ __forceinline__ int find_desc(const QrBatch& b) {
  int di = 0;
  while (di + 1 < b.count && (int)blockIdx.x >= b.d[di + 1].begin) ++di;
  return di;
}

__device__ __forceinline__ int chunk_rows(const QrDev& q, int c) {
  return c < q.P - 1 ? q.rpc : q.m - (q.P - 1) * q.rpc;
}

__device__ __forceinline__ int nsub_of(int rows) { return rows <= MS ? 1 : 1 + (rows - MS + MS - 1) / MS; }

__device__ __forceinline__ int round_up32(int v) { return (v + 31) & ~31; }

__device__ __forceinline__ double pick(const double (&r)[NT], int slot) {
  double v = r[0];
#pragma unroll
  for (int t = 1; t < NT; ++t)
    if (slot == t) v = r[t];
  return v;
}

// Householder factorisation of the column-major shared block As (pitch p).
//  dense = true : reflector j: head As[j][j], tail rows j+1..nrows-1 (plain dgeqr2)
//  dense = false: reflector j: head R[j][j] (row-major, pitch rp), tail rows 0..nrows-1
//                 (QR of [R; As] with R upper triangular: one flat-TSQR step)
// Writes tau[0..K) (zeros beyond nrefl).  One __syncthreads per reflector: the warp
// owning column j+1 updates it first and immediately computes reflector j+1.
__device__ void hh_factor(double* As, int p, int nrows, int K, int nrefl, bool dense, double* R, int rp,
                          double* taus) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  auto in_tail = [&](int i, int j) { return i < nrows && (!dense || i > j); };
  auto head_ptr = [&](int j, int c) -> double* { return dense ? &As[c * p + j] : &R[j * rp + c]; };

  auto larfg = [&](int j) {
    double ss = 0.0;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int i = lane + t * kWarp;
      if (in_tail(i, j)) {
        const double v = As[j * p + i];
        ss = fma(v, v, ss);
      }
    }
    ss = warp_sum(ss);
    const double alpha = *head_ptr(j, j);
    double tau = 0.0;
    if (ss > 0.0) {
      const double beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
      tau = (beta - alpha) / beta;
      const double scal = 1.0 / (alpha - beta);
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int i = lane + t * kWarp;
        if (in_tail(i, j)) As[j * p + i] *= scal;
      }
      __syncwarp();
      if (lane == 0) *head_ptr(j, j) = beta;
    }
    if (lane == 0) taus[j] = tau;
    __syncwarp();
  };

  for (int j = nrefl + (int)threadIdx.x; j < K; j += blockDim.x) taus[j] = 0.0;
  if (nrefl > 0 && warp == 0) larfg(0);
  __syncthreads();
  for (int j = 0; j < nrefl; ++j) {
    const double tj = taus[j];
    double x[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int i = lane + t * kWarp;
      x[t] = in_tail(i, j) ? As[j * p + i] : 0.0;
    }
    const int c0 = j + 1 + (((warp - (j + 1)) % NW) + NW) % NW;
    for (int c = c0; c < K; c += NW) {
      if (tj != 0.0) {
        double s = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int i = lane + t * kWarp;
          if (i < nrows) s = fma(x[t], As[c * p + i], s);
        }
        double* h = head_ptr(j, c);
        const double hv = *h;
        s = warp_sum(s);
        const double w = tj * (hv + s);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int i = lane + t * kWarp;
          if (in_tail(i, j)) As[c * p + i] = fma(-w, x[t], As[c * p + i]);
        }
        __syncwarp();
        if (lane == 0) *h = hv - w;
        __syncwarp();
      }
      if (c == j + 1 && c < nrefl) larfg(c);
    }
    __syncthreads();
  }
}

// Load rows [row0, row0+nrows) x cols [0, K) of a strided matrix into column-major smem.
__device__ void load_block(double* As, int p, const double* A, long long a_r, long long a_c, int row0, int nrows,
                           int K) {
  const int total = nrows * K;
  if (a_c == 1) {
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int i = e / K, c = e - i * K;
      As[c * p + i] = A[(long long)(row0 + i) * a_r + c];
    }
  } else {
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int c = e / nrows, i = e - c * nrows;
      As[c * p + i] = A[(long long)(row0 + i) * a_r + (long long)c * a_c];
    }
  }
}

__global__ void __launch_bounds__(QT, 1) qr_factor_kernel(const __grid_constant__ QrBatch b) {
  extern __shared__ double sm[];
  const QrDev& q = b.d[find_desc(b)];
  const int local = blockIdx.x - q.begin;
  const int nd = local / q.P, c = local % q.P;
  const int K = q.K, m = q.m;
  const int rows = chunk_rows(q, c), r0 = c * q.rpc;
  const double* A = q.A + nd * q.a_node;
  double* V = q.V + nd * q.v_node;
  double* tg = q.tau + nd * q.tau_node + (long long)c * q.nsub_pc * K;
  double* Rst = q.Rst + nd * q.st_node + (long long)c * K * K;
  const int rp = K + 1;
  double* R = sm;
  double* As = sm + K * rp;
  double* taus = As + K * (MS + 1);

  // sub-block 0: dense Householder QR (its top K rows become the chunk's R rows)
  const int n0 = min(rows, MS);
  const int p0 = round_up32(n0) + 1;
  const int k0 = min(n0, K);
  load_block(As, p0, A, q.a_r, q.a_c, r0, n0, K);
  __syncthreads();
  hh_factor(As, p0, n0, K, k0, true, R, rp, taus);
  for (int e = threadIdx.x; e < k0 * n0; e += blockDim.x) {
    const int col = e / n0, i = e - col * n0;
    if (i > col) V[(long long)col * m + r0 + i] = As[col * p0 + i];
  }
  for (int j = threadIdx.x; j < K; j += blockDim.x) tg[j] = taus[j];
  if (rows > n0) {
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
      const int j = e / K, cc = e - j * K;
      R[j * rp + cc] = cc >= j ? As[cc * p0 + j] : 0.0;
    }
  } else {
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
      const int j = e / K, cc = e - j * K;
      Rst[e] = (j < k0 && cc >= j) ? As[cc * p0 + j] : 0.0;
    }
  }
  __syncthreads();

  // remaining sub-blocks: one flat-TSQR step [R; A_s] each
  int off = n0, s = 1;
  while (off < rows) {
    const int ns = min(MS, rows - off);
    load_block(As, MS + 1, A, q.a_r, q.a_c, r0 + off, ns, K);
    __syncthreads();
    hh_factor(As, MS + 1, ns, K, K, false, R, rp, taus);
    for (int e = threadIdx.x; e < K * ns; e += blockDim.x) {
      const int col = e / ns, i = e - col * ns;
      V[(long long)col * m + r0 + off + i] = As[col * (MS + 1) + i];
    }
    for (int j = threadIdx.x; j < K; j += blockDim.x) tg[(long long)s * K + j] = taus[j];
    __syncthreads();
    off += ns;
    ++s;
  }
  if (rows > n0) {
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
      const int j = e / K, cc = e - j * K;
      Rst[e] = R[j * rp + cc];
    }
  }
}

__device__ __forceinline__ int pairs_in_round(int P, int r) {
  const int h = 1 << r;
  return P > h ? (P - h - 1) / (2 * h) + 1 : 0;
}

// Binary-tree combine of chunk R factors: QR of [R_a; R_b] (round r).
__global__ void __launch_bounds__(QT, 1) qr_combine_kernel(const __grid_constant__ QrBatch b) {
  extern __shared__ double sm[];
  const QrDev& q = b.d[find_desc(b)];
  const int r = b.round;
  const int local = blockIdx.x - q.begin;
  const int nd = local / q.per_node, k = local % q.per_node;
  const int a = k << (r + 1), bb = a + (1 << r);
  const int K = q.K;
  const int rp = K + 1, pb = round_up32(K) + 1;
  double* R = sm;
  double* As = sm + K * rp;
  double* taus = As + K * (MS + 1);
  double* Ra = q.Rst + nd * q.st_node + (long long)a * K * K;
  double* Rb = q.Rst + nd * q.st_node + (long long)bb * K * K;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    const int i = e / K, cc = e - i * K;
    R[i * rp + cc] = Ra[e];
    As[cc * pb + i] = Rb[e];
  }
  __syncthreads();
  hh_factor(As, pb, K, K, K, false, R, rp, taus);
  double* ctau = q.tau + nd * q.tau_node + (long long)q.nsub_total * K + (long long)bb * K;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    const int i = e / K, cc = e - i * K;
    Ra[e] = R[i * rp + cc];
    Rb[cc * K + i] = As[cc * pb + i];  // reflector tails, column-major
  }
  for (int j = threadIdx.x; j < K; j += blockDim.x) ctau[j] = taus[j];
}

// Sign fix (kernels.py:31-32) and the seed diag(s) of the backward accumulation.
__global__ void qr_finalize_kernel(const __grid_constant__ QrBatch b) {
  const QrDev& q = b.d[find_desc(b)];
  const int nd = blockIdx.x - q.begin;
  const int K = q.K, kq = min(q.m, K);
  const double* Rf = q.Rst + nd * q.st_node;
  double* Ro = q.R + nd * q.r_node;
  double* W0 = q.W + nd * q.st_node;
  for (int e = threadIdx.x; e < kq * K; e += blockDim.x) {
    const int j = e / K, c = e - j * K;
    const double s = Rf[j * K + j] < 0.0 ? -1.0 : 1.0;
    Ro[(long long)j * q.r_ld + c] = s * Rf[j * K + c];
  }
  for (int e = threadIdx.x; e < kq * K; e += blockDim.x) {
    const int c = e / K, i = e - c * K;
    W0[(long long)c * K + i] = (i == c) ? (Rf[c * K + c] < 0.0 ? -1.0 : 1.0) : 0.0;
  }
}

// Backward accumulation through one combine round: [W_a; 0] -> [W_a'; W_b].
__global__ void __launch_bounds__(QT, 1) qr_expand_round_kernel(const __grid_constant__ QrBatch b) {
  extern __shared__ double sm[];
  const QrDev& q = b.d[find_desc(b)];
  const int r = b.round;
  const int local = blockIdx.x - q.begin;
  const int nd = local / q.per_node, k = local % q.per_node;
  const int a = k << (r + 1), bb = a + (1 << r);
  const int K = q.K, kq = min(q.m, K);
  const int pb = round_up32(K) + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* Vs = sm;
  double* taus = sm + K * pb;
  const double* Vb = q.Rst + nd * q.st_node + (long long)bb * K * K;
  const double* ct = q.tau + nd * q.tau_node + (long long)q.nsub_total * K + (long long)bb * K;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    const int c = e / K, i = e - c * K;
    Vs[c * pb + i] = Vb[e];
  }
  for (int j = threadIdx.x; j < K; j += blockDim.x) taus[j] = ct[j];
  __syncthreads();
  double* Wa = q.W + nd * q.st_node + (long long)a * K * K;
  double* Wb = q.W + nd * q.st_node + (long long)bb * K * K;
  for (int c = warp; c < kq; c += NW) {
    double wa[NT], wb[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int i = lane + t * kWarp;
      wa[t] = i < K ? Wa[(long long)c * K + i] : 0.0;
      wb[t] = 0.0;
    }
    for (int j = K - 1; j >= 0; --j) {
      const double tj = taus[j];
      if (tj == 0.0) continue;
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int i = lane + t * kWarp;
        if (i < K) s = fma(Vs[j * pb + i], wb[t], s);
      }
      const double hv = __shfl_sync(0xffffffffu, pick(wa, j >> 5), j & 31);
      s = warp_sum(s);
      const double w = tj * (hv + s);
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int i = lane + t * kWarp;
        if (t == (j >> 5) && lane == (j & 31)) wa[t] -= w;
        if (i < K) wb[t] = fma(-w, Vs[j * pb + i], wb[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int i = lane + t * kWarp;
      if (i < K) {
        Wa[(long long)c * K + i] = wa[t];
        Wb[(long long)c * K + i] = wb[t];
      }
    }
  }
}

// Every chunk applies its reflectors in reverse to its seed: rows of the thin Q.
__global__ void __launch_bounds__(QT, 1) qr_expand_chunk_kernel(const __grid_constant__ QrBatch b) {
  extern __shared__ double sm[];
  const QrDev& q = b.d[find_desc(b)];
  const int local = blockIdx.x - q.begin;
  const int nd = local / q.P, c = local % q.P;
  const int K = q.K, m = q.m, kq = min(m, K);
  const int rows = chunk_rows(q, c), r0 = c * q.rpc;
  const int n0 = min(rows, MS), p0 = round_up32(n0) + 1, k0 = min(n0, K);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* V = q.V + nd * q.v_node;
  const double* tg = q.tau + nd * q.tau_node + (long long)c * q.nsub_pc * K;
  double* Wc = q.W + nd * q.st_node + (long long)c * K * K;
  double* Q = q.Q + nd * q.q_node;
  double* Vs = sm;
  double* taus = sm + K * (MS + 1);

  const int nsub = nsub_of(rows);
  for (int s = nsub - 1; s >= 1; --s) {
    const int off = n0 + (s - 1) * MS;
    const int ns = min(MS, rows - off);
    for (int e = threadIdx.x; e < K * ns; e += blockDim.x) {
      const int col = e / ns, i = e - col * ns;
      Vs[col * (MS + 1) + i] = V[(long long)col * m + r0 + off + i];
    }
    for (int j = threadIdx.x; j < K; j += blockDim.x) taus[j] = tg[(long long)s * K + j];
    __syncthreads();
    for (int cc = warp; cc < kq; cc += NW) {
      double wr[NT], qv[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int i = lane + t * kWarp;
        wr[t] = i < K ? Wc[(long long)cc * K + i] : 0.0;
        qv[t] = 0.0;
      }
      for (int j = K - 1; j >= 0; --j) {
        const double tj = taus[j];
        if (tj == 0.0) continue;
        double sdot = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int i = lane + t * kWarp;
          if (i < ns) sdot = fma(Vs[j * (MS + 1) + i], qv[t], sdot);
        }
        const double hv = __shfl_sync(0xffffffffu, pick(wr, j >> 5), j & 31);
        sdot = warp_sum(sdot);
        const double w = tj * (hv + sdot);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int i = lane + t * kWarp;
          if (t == (j >> 5) && lane == (j & 31)) wr[t] -= w;
          if (i < ns) qv[t] = fma(-w, Vs[j * (MS + 1) + i], qv[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int i = lane + t * kWarp;
        if (i < ns) Q[(long long)(r0 + off + i) * q.q_r + (long long)cc * q.q_c] = qv[t];
        if (i < K) Wc[(long long)cc * K + i] = wr[t];
      }
    }
    __syncthreads();
  }

  // sub-block 0: dense reflectors applied in reverse to [W; 0]
  for (int e = threadIdx.x; e < k0 * n0; e += blockDim.x) {
    const int col = e / n0, i = e - col * n0;
    Vs[col * p0 + i] = V[(long long)col * m + r0 + i];
  }
  for (int j = threadIdx.x; j < K; j += blockDim.x) taus[j] = tg[j];
  __syncthreads();
  for (int cc = warp; cc < kq; cc += NW) {
    double qv[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int i = lane + t * kWarp;
      qv[t] = (i < k0) ? Wc[(long long)cc * K + i] : 0.0;
    }
    for (int j = k0 - 1; j >= 0; --j) {
      const double tj = taus[j];
      if (tj == 0.0) continue;
      double sdot = 0.0;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int i = lane + t * kWarp;
        if (i < n0 && i > j) sdot = fma(Vs[j * p0 + i], qv[t], sdot);
      }
      const double hv = __shfl_sync(0xffffffffu, pick(qv, j >> 5), j & 31);
      sdot = warp_sum(sdot);
      const double w = tj * (hv + sdot);
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int i = lane + t * kWarp;
        if (t == (j >> 5) && lane == (j & 31)) qv[t] -= w;
        if (i < n0 && i > j) qv[t] = fma(-w, Vs[j * p0 + i], qv[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int i = lane + t * kWarp;
      if (i < n0) Q[(long long)(r0 + i) * q.q_r + (long long)cc * q.q_c] = qv[t];
    }
  }
}

int nsub_host(int rows) { return rows <= MS ? 1 : 1 + (rows - MS + MS - 1) / MS; }

int pairs_host(int P, int r) {
  const int h = 1 << r;
  return P > h ? (P - h - 1) / (2 * h) + 1 : 0;
}

size_t smem_bytes(int K) { return (size_t)(K * (K + 1) + K * (MS + 1) + K) * sizeof(double); }

bool g_attr_done = false;

int ensure_attrs() {
  if (g_attr_done) return kOk;
  HT_CUDA_CHECK(cudaFuncSetAttribute(qr_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX_BYTES));
  HT_CUDA_CHECK(cudaFuncSetAttribute(qr_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX_BYTES));
  HT_CUDA_CHECK(
      cudaFuncSetAttribute(qr_expand_round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX_BYTES));
  HT_CUDA_CHECK(
      cudaFuncSetAttribute(qr_expand_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX_BYTES));
  g_attr_done = true;
  return kOk;
}

QrDev to_dev(const QrProblem& p) {
  QrDev d{};
  d.A = p.A; d.a_r = p.a_r; d.a_c = p.a_c; d.a_node = p.a_node;
  d.Q = p.Q; d.q_r = p.q_r; d.q_c = p.q_c; d.q_node = p.q_node;
  d.R = p.R; d.r_ld = p.r_ld; d.r_node = p.r_node;
  d.V = p.V; d.tau = p.tau; d.Rst = p.Rst; d.W = p.W;
  d.v_node = p.v_node; d.tau_node = p.tau_node; d.st_node = p.st_node;
  d.m = p.m; d.K = p.K; d.P = p.P; d.rpc = p.rpc; d.nsub_pc = p.nsub_pc; d.nsub_total = p.nsub_total;
  d.nodes = p.nodes;
  return d;
}

enum Phase { kFactor, kCombine, kFinalize, kExpandRound, kExpandChunk };

// LAPACK-equivalent algorithmic flops: dgeqrf (factor) / dorgqr (Q formation)
double qr_flops(int m, int K) {
  const double a = std::max(m, K), b = std::min(m, K);
  return 2.0 * a * b * b - 2.0 / 3.0 * b * b * b;
}

const char* phase_name(int ph) {
  static const char* names[] = {"qr_factor", "qr_combine", "qr_finalize", "qr_expand_round", "qr_expand_chunk"};
  return names[ph];
}

template <typename KernelT>
int launch_phase(KernelT kernel, std::vector<QrProblem>& probs, Phase ph, int round, cudaStream_t stream) {
  size_t i = 0;
  while (i < probs.size()) {
    QrBatch b;
    b.count = 0;
    b.round = round;
    int blocks = 0;
    size_t smem = 0;
    while (i < probs.size() && b.count < MAXD) {
      const QrProblem& p = probs[i++];
      int per = 0;
      switch (ph) {
        case kFactor:
        case kExpandChunk: per = p.P; break;
        case kCombine:
        case kExpandRound: per = pairs_host(p.P, round); break;
        case kFinalize: per = 1; break;
      }
      if (per == 0 || p.nodes == 0) continue;
      QrDev d = to_dev(p);
      d.begin = blocks;
      d.per_node = per;
      blocks += per * p.nodes;
      smem = std::max(smem, smem_bytes(p.K));
      b.d[b.count++] = d;
    }
    if (b.count == 0) continue;
    if (ph == kFinalize) smem = 0;
    double flops = 0, bytes = 0;
    for (int q = 0; q < b.count; ++q) {
      const QrDev& d = b.d[q];
      if (ph == kFactor || ph == kExpandChunk) {
        flops += (double)d.nodes * qr_flops(d.m, d.K);
        bytes += 16.0 * d.nodes * (double)d.m * d.K;
      }
    }
    ProfToken tok = prof_begin(stream);
    kernel<<<blocks, ph == kFinalize ? 256 : QT, smem, stream>>>(b);
    HT_LAUNCH_CHECK();
    prof_end(tok, phase_name(ph), stream, flops, bytes);
  }
  return kOk;
}

}  // namespace

int qr_plan(QrProblem& p, int target_ctas) {
  if (p.K < 1 || p.m < 1) {
    set_error("qr_plan: empty matrix");
    return kErrShape;
  }
  if (p.K > kQrMaxK) {
    set_error("qr_plan: K=" + std::to_string(p.K) + " exceeds the shared-memory QR path (K <= 112)");
    return kErrUnsupported;
  }
  int pmax = std::max(1, p.m / std::max(p.K, MS));
  int want = p.P > 0 ? p.P : std::max(1, ceil_div(target_ctas, std::max(1, p.nodes)));
  p.P = std::min(want, pmax);
  p.rpc = p.m / p.P;
  p.ms0 = MS;
  p.ms = MS;
  p.nsub_pc = nsub_host(p.rpc);
  p.nsub_total = (p.P - 1) * p.nsub_pc + nsub_host(p.m - (p.P - 1) * p.rpc);
  p.v_node = (long long)p.m * p.K;
  p.tau_node = (long long)(p.nsub_total + p.P) * p.K;
  p.st_node = (long long)p.P * p.K * p.K;
  return kOk;
}

long long qr_workspace_doubles(const QrProblem& p) {
  return (long long)p.nodes * (p.v_node + p.tau_node + 2 * p.st_node);
}

void qr_bind_workspace(QrProblem& p, double* ws) {
  p.V = ws;
  ws += (long long)p.nodes * p.v_node;
  p.tau = ws;
  ws += (long long)p.nodes * p.tau_node;
  p.Rst = ws;
  ws += (long long)p.nodes * p.st_node;
  p.W = ws;
}

int qr_batched(std::vector<QrProblem>& probs, cudaStream_t stream) {
  if (probs.empty()) return kOk;
  HT_TRY(ensure_attrs());
  int maxP = 1;
  for (auto& p : probs) maxP = std::max(maxP, p.P);
  int rounds = 0;
  while ((1 << rounds) < maxP) ++rounds;
  HT_TRY(launch_phase(qr_factor_kernel, probs, kFactor, 0, stream));
  for (int r = 0; r < rounds; ++r) HT_TRY(launch_phase(qr_combine_kernel, probs, kCombine, r, stream));
  HT_TRY(launch_phase(qr_finalize_kernel, probs, kFinalize, 0, stream));
  for (int r = rounds - 1; r >= 0; --r) HT_TRY(launch_phase(qr_expand_round_kernel, probs, kExpandRound, r, stream));
  HT_TRY(launch_phase(qr_expand_chunk_kernel, probs, kExpandChunk, 0, stream));
  return kOk;
}

}  // namespace ht
