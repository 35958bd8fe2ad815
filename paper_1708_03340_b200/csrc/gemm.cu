// Grouped FP64 DMMA GEMM (see gemm.cuh).  64x64x16 CTA tile, 8 warps each
// owning a 32x16 sub-tile as 4x2 mma.sync.m8n8k4.f64 fragments; operands are
// staged k-major in shared memory (pitch 68 doubles: conflict-free fragment
// loads), double-buffered with a register prefetch of the next k-tile.
#include <algorithm>

#include "gemm.cuh"
#include "prof.cuh"

namespace ht {

namespace {

constexpr int BM = kGemmBM, BN = kGemmBN, BK = kGemmBK;
constexpr int PITCH = 68;  // 64 + 4: k-rows land in disjoint 8-byte bank groups
constexpr int THREADS = 256;
constexpr int PER_THREAD = BM * BK / THREADS;  // 4

struct GemmBatch {
  int count;
  GemmDesc d[kMaxGemmDescs];
};

struct ReduceBatch {
  int count;
  int block_begin[kMaxGemmDescs + 1];
  ReduceDesc d[kMaxGemmDescs];
};

__global__ void __launch_bounds__(THREADS, 2) gemm_dmma_kernel(const __grid_constant__ GemmBatch batch) {
  __shared__ __align__(16) double As[2][BK][PITCH];
  __shared__ __align__(16) double Bs[2][BK][PITCH];

  int di = 0;
  while (di + 1 < batch.count && (int)blockIdx.x >= batch.d[di + 1].block_begin) ++di;
  const GemmDesc& g = batch.d[di];

  int local = blockIdx.x - g.block_begin;
  const int tn = local % g.tiles_n;
  local /= g.tiles_n;
  const int tm = local % g.tiles_m;
  local /= g.tiles_m;
  const int split = local % g.splits;
  const int b = local / g.splits;
  const int b1 = b % g.nb1, b2 = b / g.nb1;

  const double* A = g.A + b1 * g.a_b1 + b2 * g.a_b2;
  const double* Bp = g.B + b1 * g.b_b1 + b2 * g.b_b2;

  const int m0 = tm * BM, n0 = tn * BN;
  const long long L = (long long)g.K * g.KO;
  const long long per_split = ((L + g.splits - 1) / g.splits + BK - 1) / BK * BK;
  const long long k_begin = split * per_split;
  const long long k_end = min(L, k_begin + per_split);
  const int ntiles = k_end > k_begin ? (int)((k_end - k_begin + BK - 1) / BK) : 0;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps, each 32 x 16

  const bool a_kc = (g.a_k == 1);
  const bool b_kc = (g.b_k == 1);

  double ra[PER_THREAD], rb[PER_THREAD];

  auto load = [&](int t) {
#pragma unroll
    for (int q = 0; q < PER_THREAD; ++q) {
      const int e = tid + q * THREADS;
      {
        const int kk = a_kc ? (e & (BK - 1)) : (e >> 6);
        const int mm = a_kc ? (e >> 4) : (e & (BM - 1));
        const long long f = k_begin + (long long)t * BK + kk;
        const int m = m0 + mm;
        double v = 0.0;
        if (m < g.M && f < k_end) {
          long long o = 0, k = f;
          if (g.KO > 1) { o = f / g.K; k = f - o * g.K; }
          if (g.a_tri == 0) {
            v = __ldg(A + m * g.a_m + k * g.a_k + o * g.a_o);
          } else if (g.a_tri == 3) {
            v = (m == k) ? 1.0 : 0.0;
          } else {
            // implicit unit-diagonal Householder vectors (compact-WY Y factor)
            const bool stored = g.a_tri == 1 ? (m > k) : (k > m);
            v = stored ? __ldg(A + m * g.a_m + k * g.a_k + o * g.a_o) : (m == k ? 1.0 : 0.0);
          }
        }
        ra[q] = v;
      }
      {
        const int kk = b_kc ? (e & (BK - 1)) : (e >> 6);
        const int nn = b_kc ? (e >> 4) : (e & (BN - 1));
        const long long f = k_begin + (long long)t * BK + kk;
        const int n = n0 + nn;
        double v = 0.0;
        if (n < g.N && f < k_end) {
          long long o = 0, k = f;
          if (g.KO > 1) { o = f / g.K; k = f - o * g.K; }
          if (g.b_tri == 0 || k > n) v = __ldg(Bp + k * g.b_k + n * g.b_n + o * g.b_o);
          else v = (k == n) ? 1.0 : 0.0;
        }
        rb[q] = v;
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < PER_THREAD; ++q) {
      const int e = tid + q * THREADS;
      const int akk = a_kc ? (e & (BK - 1)) : (e >> 6);
      const int amm = a_kc ? (e >> 4) : (e & (BM - 1));
      As[buf][akk][amm] = ra[q];
      const int bkk = b_kc ? (e & (BK - 1)) : (e >> 6);
      const int bnn = b_kc ? (e >> 4) : (e & (BN - 1));
      Bs[buf][bkk][bnn] = rb[q];
    }
  };

  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  if (ntiles > 0) {
    load(0);
    store(0);
  }
  __syncthreads();
  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1;
    if (t + 1 < ntiles) load(t + 1);
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][ks + (lane & 3)][wm * 32 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Bs[buf][ks + (lane & 3)][wn * 16 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
    if (t + 1 < ntiles) store(buf ^ 1);
    __syncthreads();
  }

  // epilogue
  if (g.splits == 1) {
    double* C = g.C + b1 * g.c_b1 + b2 * g.c_b2;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int m = m0 + wm * 32 + i * 8 + (lane >> 2);
          const int n = n0 + wn * 16 + j * 8 + 2 * (lane & 3) + v;
          if (m < g.M && n < g.N) {
            double* p = C + m * g.c_m + n * g.c_n;
            double r = g.alpha * acc[i][j][v];
            if (g.beta != 0.0) r += g.beta * *p;
            *p = r;
          }
        }
  } else {
    const long long nbatch = (long long)g.nb1 * g.nb2;
    double* P = g.C + ((long long)split * nbatch + b) * g.M * g.N;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int m = m0 + wm * 32 + i * 8 + (lane >> 2);
          const int n = n0 + wn * 16 + j * 8 + 2 * (lane & 3) + v;
          if (m < g.M && n < g.N) P[(long long)m * g.N + n] = acc[i][j][v];
        }
  }
}

__global__ void reduce_partials_kernel(const __grid_constant__ ReduceBatch rb) {
  int di = 0;
  while (di + 1 < rb.count && (int)blockIdx.x >= rb.block_begin[di + 1]) ++di;
  const ReduceDesc& r = rb.d[di];
  const long long nbatch = (long long)r.nb1 * r.nb2;
  const long long total = nbatch * r.M * r.N;
  const long long stride = (long long)(rb.block_begin[di + 1] - rb.block_begin[di]) * blockDim.x;
  for (long long e = (long long)(blockIdx.x - rb.block_begin[di]) * blockDim.x + threadIdx.x; e < total;
       e += stride) {
    const int n = (int)(e % r.N);
    const int m = (int)((e / r.N) % r.M);
    const long long b = e / ((long long)r.M * r.N);
    double s = 0.0;
    for (int k = 0; k < r.S; ++k) s += r.P[k * total + e];
    if (r.sym) {
      double t = 0.0;
      const long long et = (b * r.M + n) * r.N + m;
      for (int k = 0; k < r.S; ++k) t += r.P[k * total + et];
      s = 0.5 * (s + t);
    }
    const int b1 = (int)(b % r.nb1), b2 = (int)(b / r.nb1);
    double* p = r.C + b1 * r.c_b1 + b2 * r.c_b2 + (long long)m * r.c_m + (long long)n * r.c_n;
    double out = r.alpha * s;
    if (r.beta != 0.0) out += r.beta * *p;
    *p = out;
  }
}

}  // namespace

int gemm_grouped(std::vector<GemmDesc>& descs, cudaStream_t stream, const char* tag) {
  size_t i = 0;
  while (i < descs.size()) {
    GemmBatch batch;
    batch.count = 0;
    int blocks = 0;
    while (i < descs.size() && batch.count < kMaxGemmDescs) {
      GemmDesc d = descs[i++];
      if (d.M <= 0 || d.N <= 0 || d.nb1 <= 0 || d.nb2 <= 0) continue;
      if (d.splits < 1) d.splits = 1;
      if (d.KO < 1) d.KO = 1;
      d.tiles_m = ceil_div(d.M, BM);
      d.tiles_n = ceil_div(d.N, BN);
      d.block_begin = blocks;
      long long nb = (long long)d.tiles_m * d.tiles_n * d.splits * d.nb1 * d.nb2;
      if (nb > (1LL << 30)) {
        set_error("gemm_grouped: grid too large");
        return kErrArgument;
      }
      blocks += (int)nb;
      batch.d[batch.count++] = d;
    }
    if (batch.count == 0) continue;
    double flops = 0, bytes = 0;
    for (int q = 0; q < batch.count; ++q) {
      const GemmDesc& d = batch.d[q];
      const double nb = (double)d.nb1 * d.nb2;
      flops += 2.0 * d.M * d.N * (double)d.K * d.KO * nb;
      bytes += 8.0 * nb * ((double)d.M * d.K * d.KO + (double)d.K * d.KO * d.N + (double)d.M * d.N * d.splits);
    }
    ProfToken tok = prof_begin(stream);
    gemm_dmma_kernel<<<blocks, THREADS, 0, stream>>>(batch);
    HT_LAUNCH_CHECK();
    prof_end(tok, tag, stream, flops, bytes);
  }
  return kOk;
}

int reduce_partials(const std::vector<ReduceDesc>& descs, cudaStream_t stream, const char* tag) {
  size_t i = 0;
  while (i < descs.size()) {
    ReduceBatch rb;
    rb.count = 0;
    int blocks = 0;
    while (i < descs.size() && rb.count < kMaxGemmDescs) {
      const ReduceDesc& d = descs[i++];
      long long total = (long long)d.nb1 * d.nb2 * d.M * d.N;
      if (total <= 0) continue;
      rb.block_begin[rb.count] = blocks;
      blocks += (int)std::min<long long>(ceil_div(total, 256), 4096);
      rb.d[rb.count++] = d;
    }
    if (rb.count == 0) continue;
    rb.block_begin[rb.count] = blocks;
    double bytes = 0;
    for (int q = 0; q < rb.count; ++q)
      bytes += 8.0 * rb.d[q].nb1 * rb.d[q].nb2 * rb.d[q].M * rb.d[q].N * (rb.d[q].S * (rb.d[q].sym ? 2 : 1) + 1);
    ProfToken tok = prof_begin(stream);
    reduce_partials_kernel<<<blocks, 256, 0, stream>>>(rb);
    HT_LAUNCH_CHECK();
    prof_end(tok, tag, stream, 0.0, bytes);
  }
  return kOk;
}

}  // namespace ht
