#include <cstdio>
// Grouped FP64 DMMA GEMM (see gemm.cuh).
//
// CTA tiles are shaped for the HT contractions, whose short dimension is a rank
// (K ~ 100, r ~ 50): 128x104 / 104x128 cover a 100-wide side in one tile
// (96% useful), 128x56 / 56x128 a 50-wide side, 64x64 everything else.  8 warps,
// each owning WM x WN mma.sync.m8n8k4.f64 fragments; operands are staged k-major
// in shared memory (pitch = 4 mod 16 doubles: conflict-free fragment loads)
// through a 3-stage cp.async pipeline with zero-fill for the ragged edges.
#include <algorithm>
#include <cstdlib>

#include "gemm.cuh"
#include "prof.cuh"

namespace ht {

namespace {

constexpr int BK = kGemmBK;  // 16
constexpr int THREADS = 256;
constexpr int STAGES = 3;

__host__ __device__ constexpr int pitch16(int x) { return ((x + 15) / 16) * 16 + 4; }

struct GemmBatch {
  int count;
  GemmDesc d[kMaxGemmDescs];
};

struct ReduceBatch {
  int count;
  int block_begin[kMaxGemmDescs + 1];
  ReduceDesc d[kMaxGemmDescs];
};

__device__ __forceinline__ void cp8(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp8z(double* smem, const double* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Operand fetch with masks (implicit unit-triangular Householder factors, identity).
// Returns the global address to copy from, or null with the constant in `val`.
// (o0, k0): decomposition of the tile's first reduction index f0 = o0*K + k0; within a
// 16-wide tile the outer index advances at most once when K >= 16 (else: divide).
__device__ __forceinline__ void split_f(const GemmDesc& g, long long f0, int kk, long long& o, long long& k) {
  if (g.KO == 1) {
    o = 0;
    k = f0 + kk;
  } else if (g.K >= 16) {
    const long long o0 = f0 / g.K;
    k = f0 - o0 * g.K + kk;
    o = o0;
    if (k >= g.K) {
      k -= g.K;
      ++o;
    }
  } else {
    o = (f0 + kk) / g.K;
    k = f0 + kk - o * g.K;
  }
}

__device__ __forceinline__ const double* a_src(const GemmDesc& g, const double* A, int m, long long f0, int kk,
                                               long long k_end, double& val) {
  val = 0.0;
  if (m >= g.M || f0 + kk >= k_end) return nullptr;
  long long o, k;
  split_f(g, f0, kk, o, k);
  if (g.a_tri == 3) {
    val = (m == k) ? 1.0 : 0.0;
    return nullptr;
  }
  if (g.a_tri == 1 || g.a_tri == 2) {
    const bool stored = g.a_tri == 1 ? (m > k) : (k > m);
    if (!stored) {
      val = (m == k) ? 1.0 : 0.0;
      return nullptr;
    }
  }
  return A + m * g.a_m + k * g.a_k + o * g.a_o;
}

__device__ __forceinline__ const double* b_src(const GemmDesc& g, const double* B, int n, long long f0, int kk,
                                               long long k_end, double& val) {
  val = 0.0;
  if (n >= g.N || f0 + kk >= k_end) return nullptr;
  long long o, k;
  split_f(g, f0, kk, o, k);
  if (g.b_tri == 1 && k <= n) {
    val = (k == n) ? 1.0 : 0.0;
    return nullptr;
  }
  return B + k * g.b_k + n * g.b_n + o * g.b_o;
}

template <int WM, int WN, int WARPS_M, int WARPS_N>
__global__ void __launch_bounds__(THREADS, ((WM * WN == 13 || WM * WN == 14) ? 2 : 1)) gemm_kernel(const __grid_constant__ GemmBatch batch) {
  constexpr int BM = 8 * WM * WARPS_M, BN = 8 * WN * WARPS_N;
  constexpr int PA = pitch16(BM), PB = pitch16(BN);
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                     // [STAGES][BK][PA]
  double* Bs = smem + STAGES * BK * PA;  // [STAGES][BK][PB]

  int di = 0;
  while (di + 1 < batch.count && (int)blockIdx.x >= batch.d[di + 1].block_begin) ++di;
  const GemmDesc& g = batch.d[di];
  if (g.active && *g.active == 0) return;

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

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const bool a_kc = (g.a_k == 1), b_kc = (g.b_k == 1);

  // Fast path (plain operands; two-level reductions with K >= 16): every thread copies
  // fixed tile slots.  Each slot keeps a running global pointer that advances by BK
  // reduction steps per tile (plus the outer-index jump when the inner index wraps),
  // so the steady-state loader is one predicated cp.async and a 64-bit add per slot.
  constexpr int NA = (BM * BK + THREADS - 1) / THREADS, NBB = (BN * BK + THREADS - 1) / THREADS;
  const bool fast = g.a_tri == 0 && g.b_tri == 0 && (g.KO == 1 || g.K >= BK);
  const int gK = g.K;
  const bool two_level = g.KO > 1;
  const long long a_step = (long long)BK * g.a_k, b_step = (long long)BK * g.b_k;
  const long long a_wrap = g.a_o - (long long)gK * g.a_k, b_wrap = g.b_o - (long long)gK * g.b_k;
  const double* pa[NA];
  const double* pb[NBB];
  int kia[NA], kib[NBB];  // current inner reduction index of each slot (two-level case)
  if (fast) {
    const long long o_b = two_level ? k_begin / gK : 0;
    const long long k_b = two_level ? k_begin - o_b * gK : k_begin;
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const int e = tid + q * THREADS;
      const int kk = a_kc ? (e % BK) : (e / BM);
      const int mm = a_kc ? (e / BK) : (e % BM);
      const bool ok = e < BM * BK && m0 + mm < g.M;
      long long k = k_b + kk, o = o_b;
      if (two_level && k >= gK) {
        k -= gK;
        ++o;
      }
      kia[q] = ok ? (int)k : -1;
      pa[q] = A + (long long)(ok ? m0 + mm : 0) * g.a_m + k * g.a_k + o * g.a_o;
    }
#pragma unroll
    for (int q = 0; q < NBB; ++q) {
      const int e = tid + q * THREADS;
      const int kk = b_kc ? (e % BK) : (e / BN);
      const int nn = b_kc ? (e / BK) : (e % BN);
      const bool ok = e < BN * BK && n0 + nn < g.N;
      long long k = k_b + kk, o = o_b;
      if (two_level && k >= gK) {
        k -= gK;
        ++o;
      }
      kib[q] = ok ? (int)k : -1;
      pb[q] = Bp + (long long)(ok ? n0 + nn : 0) * g.b_n + k * g.b_k + o * g.b_o;
    }
    // rows / columns beyond the matrix edge are zero in every stage, once
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const int e = tid + q * THREADS;
      if (kia[q] < 0 && e < BM * BK)
        for (int st = 0; st < STAGES; ++st)
          As[st * BK * PA + (a_kc ? (e % BK) : (e / BM)) * PA + (a_kc ? (e / BK) : (e % BM))] = 0.0;
    }
#pragma unroll
    for (int q = 0; q < NBB; ++q) {
      const int e = tid + q * THREADS;
      if (kib[q] < 0 && e < BN * BK)
        for (int st = 0; st < STAGES; ++st)
          Bs[st * BK * PB + (b_kc ? (e % BK) : (e / BN)) * PB + (b_kc ? (e / BK) : (e % BN))] = 0.0;
    }
  }

  auto load_tile = [&](int t, int stage) {
    double* as = As + stage * BK * PA;
    double* bs = Bs + stage * BK * PB;
    const long long fb = k_begin + (long long)t * BK;
    if (fast) {
      const long long krem_l = k_end - fb;
      const int krem = krem_l < BK ? (int)krem_l : BK;
#pragma unroll
      for (int q = 0; q < NA; ++q) {
        if (kia[q] >= 0) {
          const int e = tid + q * THREADS;
          const int kk = a_kc ? (e % BK) : (e / BM);
          const int mm = a_kc ? (e / BK) : (e % BM);
          const bool ok = kk < krem;
          cp8z(as + kk * PA + mm, ok ? pa[q] : A, ok);
          pa[q] += a_step;
          if (two_level) {
            kia[q] += BK;
            if (kia[q] >= gK) {
              kia[q] -= gK;
              pa[q] += a_wrap;
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < NBB; ++q) {
        if (kib[q] >= 0) {
          const int e = tid + q * THREADS;
          const int kk = b_kc ? (e % BK) : (e / BN);
          const int nn = b_kc ? (e / BK) : (e % BN);
          const bool ok = kk < krem;
          cp8z(bs + kk * PB + nn, ok ? pb[q] : Bp, ok);
          pb[q] += b_step;
          if (two_level) {
            kib[q] += BK;
            if (kib[q] >= gK) {
              kib[q] -= gK;
              pb[q] += b_wrap;
            }
          }
        }
      }
      return;
    }
    for (int e = tid; e < BM * BK; e += THREADS) {
      const int kk = a_kc ? (e % BK) : (e / BM);
      const int mm = a_kc ? (e / BK) : (e % BM);
      double v;
      const double* src = a_src(g, A, m0 + mm, fb, kk, k_end, v);
      double* dst = as + kk * PA + mm;
      if (src) cp8(dst, src);
      else *dst = v;
    }
    for (int e = tid; e < BN * BK; e += THREADS) {
      const int kk = b_kc ? (e % BK) : (e / BN);
      const int nn = b_kc ? (e / BK) : (e % BN);
      double v;
      const double* src = b_src(g, Bp, n0 + nn, fb, kk, k_end, v);
      double* dst = bs + kk * PB + nn;
      if (src) cp8(dst, src);
      else *dst = v;
    }
  };

  double acc[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < WN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ntiles) load_tile(s, s);
    cp_commit();
  }
  const int ar = wm * WM * 8 + (lane >> 2);
  const int br = wn * WN * 8 + (lane >> 2);
  int cst = 0, lst = STAGES - 1;  // compute / load stage (rotating, no divisions)
  for (int t = 0; t < ntiles; ++t) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nt = t + STAGES - 1;
      if (nt < ntiles) load_tile(nt, lst);
      cp_commit();
      if (++lst == STAGES) lst = 0;
    }
    const double* as = As + cst * BK * PA;
    const double* bs = Bs + cst * BK * PB;
    if (++cst == STAGES) cst = 0;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      const int kr = ks + (lane & 3);
      double af[WM], bf[WN];
#pragma unroll
      for (int i = 0; i < WM; ++i) af[i] = as[kr * PA + ar + i * 8];
#pragma unroll
      for (int j = 0; j < WN; ++j) bf[j] = bs[kr * PB + br + j * 8];
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int j = 0; j < WN; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
  }
  cp_wait<0>();

  if (g.splits == 1) {
    double* C = g.C + b1 * g.c_b1 + b2 * g.c_b2;
    const double alpha = g.alpha, beta = g.beta;
    const long long c_m = g.c_m, c_n = g.c_n;
    const int M = g.M, N = g.N;
    // paired 16-byte stores when the row is contiguous and 16-byte aligned
    const bool pair = c_n == 1 && (c_m & 1) == 0 && (((uintptr_t)C) & 15) == 0;
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      const int m = m0 + wm * WM * 8 + i * 8 + (lane >> 2);
      if (m >= M) continue;
      double* row = C + (long long)m * c_m;
#pragma unroll
      for (int j = 0; j < WN; ++j) {
        const int n = n0 + wn * WN * 8 + j * 8 + 2 * (lane & 3);
        if (pair && n + 1 < N) {
          double2 r = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
          double2* p = reinterpret_cast<double2*>(row + n);
          if (beta != 0.0) {
            const double2 o = *p;
            r.x += beta * o.x;
            r.y += beta * o.y;
          }
          *p = r;
        } else {
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            if (n + v < N) {
              double* p = row + (long long)(n + v) * c_n;
              double r = alpha * acc[i][j][v];
              if (beta != 0.0) r += beta * *p;
              *p = r;
            }
          }
        }
      }
    }
  } else {
    const long long nbatch = (long long)g.nb1 * g.nb2;
    double* P = g.C + ((long long)split * nbatch + b) * g.M * g.N;
#pragma unroll
    for (int i = 0; i < WM; ++i)
#pragma unroll
      for (int j = 0; j < WN; ++j)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int m = m0 + wm * WM * 8 + i * 8 + (lane >> 2);
          const int n = n0 + wn * WN * 8 + j * 8 + 2 * (lane & 3) + v;
          if (m < g.M && n < g.N) P[(long long)m * g.N + n] = acc[i][j][v];
        }
  }
}

__global__ void reduce_partials_kernel(const __grid_constant__ ReduceBatch rb) {
  int di = 0;
  while (di + 1 < rb.count && (int)blockIdx.x >= rb.block_begin[di + 1]) ++di;
  const ReduceDesc& r = rb.d[di];
  if (r.active && *r.active == 0) return;
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


// ---- long-reduction kernel ---------------------------------------------------
// C (M x N <= 112 x 112) = sum over a long (split-K) reduction f = (o, k) of
// A(f, m) B(f, n): the reduced-Gramian contractions and the Cholesky-QR Gram
// matrices.  14 warps (7 x 2) each own a 16 x 56 block of one 112 x 112 tile as
// seven m16n8k16 fragments (A fragment reused seven times: 36 LDS per 56 DMMA);
// ~130 registers, so 14 warps per SM hide the operand latency the 8-warp generic
// tile could not.  Both operands are staged through a 3-stage pipeline of 32-deep
// k-chunks (one barrier per 112 DMMA per warp) in 16-byte cp.async pairs, per
// descriptor either along m/n (lm = 1: a_m == b_n == 1, staged [k][m]) or along k
// (lm = 0: a_k == b_k == 1, staged [m][k]); both layouts share one launch so a level's
// two son Gramians fill the machine together.
constexpr int LR_T = 112;        // tile edge
constexpr int LR_BK = 32;
constexpr int LR_STAGES = 3;
constexpr int LR_PM = LR_T + 4;  // [k][m] pitch (4 mod 16 doubles: conflict-free fragments)
constexpr int LR_PK = LR_BK + 4; // [m][k] pitch
constexpr int LR_OPD = (LR_BK * LR_PM > LR_T * LR_PK) ? LR_BK * LR_PM : LR_T * LR_PK;  // doubles per operand-stage

struct LrBatch {
  int count;
  unsigned char lm[kMaxGemmDescs];
  GemmDesc d[kMaxGemmDescs];
};

__device__ __forceinline__ void cp16z(double* smem, const double* gmem, int valid_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid_bytes));
}

// ---- long-reduction kernel, warp-specialised mbarrier pipeline -----------------
// 14 consumer warps, 112 x 112 tiles, m16n8k16; producer warps stage the operands (16-byte cp.async, completion counted on
// a per-stage `full` mbarrier) and the consumers release each stage on an `empty`
// mbarrier: no CTA-wide barrier per k-chunk, consumer warps drift independently and
// the producer runs up to LR_STAGES chunks ahead.
constexpr int LRT_CONSUMERS = 14;
// upper-triangle block pairs of the symmetric variant: warp w computes blocks
// (kBI[2w], kBJ[2w]) and (kBI[2w+1], kBJ[2w+1])
__constant__ unsigned char kBI[28] = {0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 5, 5, 0, 2, 4, 6};
__constant__ unsigned char kBJ[28] = {0, 1, 2, 3, 4, 5, 1, 2, 3, 4, 5, 6, 2, 3, 4, 5, 3, 4, 5, 6, 4, 5, 5, 6, 6, 6, 6, 6};
constexpr int LRT_PRODUCERS = 2;
constexpr int LRT_THREADS = (LRT_CONSUMERS + LRT_PRODUCERS) * 32;

template <int LM>
__device__ __forceinline__ void lrt_body(const GemmDesc& g, int local, double* smem, unsigned long long* full,
                                         unsigned long long* empty) {
  const int split = local % g.splits;
  const int b = local / g.splits;
  const int b1 = b % g.nb1, b2 = b / g.nb1;
  const double* A = g.A + b1 * g.a_b1 + b2 * g.a_b2;
  const double* B = g.B + b1 * g.b_b1 + b2 * g.b_b2;
  const int M = g.M, N = g.N, K = g.K;
  const long long L = (long long)K * g.KO;
  const long long per_split = ((L + g.splits - 1) / g.splits + LR_BK - 1) / LR_BK * LR_BK;
  const long long f_begin = split * per_split;
  const long long f_end = min(L, f_begin + per_split);
  const int nst = f_end > f_begin ? (int)((f_end - f_begin + LR_BK - 1) / LR_BK) : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (warp >= LRT_CONSUMERS) {
    // ---------------- producer warps ----------------
    // 16-byte cp.async pairs (zero-filled past the k-tail and beyond M / N), their
    // completion signalled to full[st] by cp.async.mbarrier.arrive (one per lane)
    long long o = f_begin / K;
    int k = (int)(f_begin - o * K);
    for (int s = 0; s < nst; ++s) {
      const int st = s % LR_STAGES;
      mbar_wait(&empty[st], ((s / LR_STAGES) & 1) ^ 1);
      double* as = smem + st * 2 * LR_OPD;
      double* bs = as + LR_OPD;
      const long long f0 = f_begin + (long long)s * LR_BK;
      const int nv = (int)min((long long)LR_BK, f_end - f0);  // valid k of this chunk
      const int pw = warp - LRT_CONSUMERS;
      if (LM) {
        // k-rows kk = pw, pw + P, ...: lane covers m pairs 2 lane and 2 (lane + 32)
#pragma unroll 4
        for (int kq = 0; kq < LR_BK / LRT_PRODUCERS; ++kq) {
          const int kk = kq * LRT_PRODUCERS + pw;
          const bool fin = kk < nv;
          const bool wrap = k + kk >= K;
          const long long oo = wrap ? o + 1 : o;
          const long long kx = wrap ? k + kk - K : k + kk;
          const double* arow = A + oo * g.a_o + kx * g.a_k;
          const double* brow = B + oo * g.b_o + kx * g.b_k;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = 2 * (lane + 32 * h);
            if (r < LR_T) {
              const int av = fin ? 8 * max(0, min(2, M - r)) : 0;
              const int bv = fin ? 8 * max(0, min(2, N - r)) : 0;
              cp16z(as + kk * LR_PM + r, av ? arow + r : A, av);
              cp16z(bs + kk * LR_PM + r, bv ? brow + r : B, bv);
            }
          }
        }
      } else {
        // lane covers k pair kk = 2 (lane % 16) of rows lane / 16 + 2 q (this warp's half)
        const int kk = 2 * (lane & 15);
        const bool fin = kk < nv;
        const bool wrap = k + kk >= K;
        const long long oo = wrap ? o + 1 : o;
        const long long kx = wrap ? k + kk - K : k + kk;
        const int r0 = (lane >> 4) + LR_T / LRT_PRODUCERS * pw;
        const double* ap = A + oo * g.a_o + kx + (long long)r0 * g.a_m;
        const double* bp = B + oo * g.b_o + kx + (long long)r0 * g.b_n;
        double* ad = as + r0 * LR_PK + kk;
        double* bd = bs + r0 * LR_PK + kk;
#pragma unroll 4
        for (int q = 0; q < LR_T / LRT_PRODUCERS / 2; ++q) {
          const int r = r0 + 2 * q;
          const int av = fin && r < M ? 16 : 0;
          const int bv = fin && r < N ? 16 : 0;
          cp16z(ad, av ? ap : A, av);
          cp16z(bd, bv ? bp : B, bv);
          ap += 2 * g.a_m;
          bp += 2 * g.b_n;
          ad += 2 * LR_PK;
          bd += 2 * LR_PK;
        }
      }
      cp_async_mbar_arrive(&full[st]);
      k += LR_BK;
      while (k >= K) {
        k -= K;
        ++o;
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    return;
  }

  // ---------------- consumer warps ----------------
  const int g8 = lane >> 2, t4 = lane & 3;
  const long long nbatch = (long long)g.nb1 * g.nb2;
  auto store = [&](int m, int n, double r) {
    if (g.splits == 1) {
      double* p = g.C + b1 * g.c_b1 + b2 * g.c_b2 + (long long)m * g.c_m + (long long)n * g.c_n;
      *p = g.beta != 0.0 ? g.alpha * r + g.beta * *p : g.alpha * r;
    } else {
      g.C[((long long)split * nbatch + b) * M * N + (long long)m * N + n] = r;
    }
  };
  auto frag_a = [&](const double* as, int row0, int k16, double (&a)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = row0 + g8 + 8 * (i & 1), k = k16 + t4 + 4 * (i >> 1);
      a[i] = LM ? as[k * LR_PM + m] : as[m * LR_PK + k];
    }
  };
  auto frag_b = [&](const double* bs, int col0, int k16, double (&bq)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int n = col0 + g8, k = k16 + t4 + 4 * i;
      bq[i] = LM ? bs[k * LR_PM + n] : bs[n * LR_PK + k];
    }
  };
  if (g.sym) {
    // Upper-triangle 16 x 16 blocks (I <= J) of the 112 x 112 tile: 28 blocks, two per
    // warp, paired along a block row (A fragment shared) where possible.
    const int I0 = kBI[2 * warp], J0 = kBJ[2 * warp], I1 = kBI[2 * warp + 1], J1 = kBJ[2 * warp + 1];
    const bool same_row = I0 == I1;
    double acc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
    for (int s = 0; s < nst; ++s) {
      const int st = s % LR_STAGES;
      mbar_wait(&full[st], (s / LR_STAGES) & 1);
      const double* as = smem + st * 2 * LR_OPD;
      const double* bs = as + LR_OPD;
#pragma unroll
      for (int k16 = 0; k16 < LR_BK; k16 += 16) {
        double a[8], bq[4];
        frag_a(as, 16 * I0, k16, a);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          frag_b(bs, 16 * J0 + 8 * j, k16, bq);
          dmma_16x8x16(acc[j], a, bq);
        }
        if (!same_row) frag_a(as, 16 * I1, k16, a);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          frag_b(bs, 16 * J1 + 8 * j, k16, bq);
          dmma_16x8x16(acc[2 + j], a, bq);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int I = q ? I1 : I0, J = q ? J1 : J0;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int m = 16 * I + g8 + 8 * f, n = 16 * J + 8 * j + 2 * t4 + v;
            if (m > n || n >= N) continue;
            const double r = acc[2 * q + j][2 * f + v];
            store(m, n, r);
            if (m != n) store(n, m, r);
          }
    }
    return;
  }
  const int wm = warp >> 1, wn = warp & 1;
  const int ar = wm * 16, bc = wn * 56;
  double acc[7][4];
#pragma unroll
  for (int j = 0; j < 7; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
  for (int s = 0; s < nst; ++s) {
    const int st = s % LR_STAGES;
    mbar_wait(&full[st], (s / LR_STAGES) & 1);
    const double* as = smem + st * 2 * LR_OPD;
    const double* bs = as + LR_OPD;
#pragma unroll
    for (int k16 = 0; k16 < LR_BK; k16 += 16) {
      double a[8];
      frag_a(as, ar, k16, a);
#pragma unroll
      for (int j = 0; j < 7; ++j) {
        double bq[4];
        frag_b(bs, bc + 8 * j, k16, bq);
        dmma_16x8x16(acc[j], a, bq);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    const int m = ar + g8 + 8 * f;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 7; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int n = bc + 8 * j + 2 * t4 + v;
        if (n < N) store(m, n, acc[j][2 * f + v]);
      }
  }
}

__global__ void __launch_bounds__(LRT_THREADS, 1) lrt_kernel(const __grid_constant__ LrBatch batch) {
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned long long full[LR_STAGES], empty[LR_STAGES];
  int di = 0;
  while (di + 1 < batch.count && (int)blockIdx.x >= batch.d[di + 1].block_begin) ++di;
  const GemmDesc& g = batch.d[di];
  if (g.active && *g.active == 0) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < LR_STAGES; ++i) {
      mbar_init(&full[i], 32 * LRT_PRODUCERS);  // the producer lanes' cp.async arrivals
      mbar_init(&empty[i], LRT_CONSUMERS);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int local = blockIdx.x - g.block_begin;
  if (batch.lm[di]) lrt_body<1>(g, local, smem, full, empty);
  else lrt_body<0>(g, local, smem, full, empty);
}

// descriptors the long-reduction kernel takes: plain operands, M, N <= 112 (not both
// <= 56), reduction >= 256, and 16-byte pairs: layout 1 (a_m == b_n == 1) or 0
// (a_k == b_k == 1, even K); -1 otherwise
int lr_layout(const GemmDesc& d) {
  if (d.a_tri || d.b_tri || d.M > LR_T || d.N > LR_T || (d.M <= 56 && d.N <= 56)) return -1;
  const int KO = std::max(d.KO, 1);
  if ((long long)d.K * KO < 256 || (KO > 1 && d.K < LR_BK)) return -1;
  auto even = [](long long v) { return (v & 1) == 0; };
  const bool al = (((uintptr_t)d.A | (uintptr_t)d.B) & 15) == 0 && even(d.a_b1) && even(d.a_b2) && even(d.b_b1) &&
                  even(d.b_b2) && even(d.a_o) && even(d.b_o);
  if (!al) return -1;
  if (d.a_m == 1 && d.b_n == 1 && even(d.a_k) && even(d.b_k) && even(d.M) && even(d.N)) return 1;
  if (d.a_k == 1 && d.b_k == 1 && even(d.K) && even(d.a_m) && even(d.b_n)) return 0;
  return -1;
}

size_t lr_smem() { return sizeof(double) * (size_t)LR_STAGES * 2 * LR_OPD; }

int lr_grouped(std::vector<std::pair<GemmDesc, int>>& descs, cudaStream_t stream, const char* tag, bool count_flops) {
  static bool attr = false;
  if (!attr) {
    HT_CUDA_CHECK(cudaFuncSetAttribute(lrt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lr_smem()));
    attr = true;
  }
  size_t i = 0;
  while (i < descs.size()) {
    LrBatch batch;
    batch.count = 0;
    int blocks = 0;
    double flops = 0, bytes = 0;
    while (i < descs.size() && batch.count < kMaxGemmDescs) {
      GemmDesc d = descs[i].first;
      batch.lm[batch.count] = (unsigned char)descs[i].second;
      ++i;
      if (d.splits < 1) d.splits = 1;
      if (d.KO < 1) d.KO = 1;
      if (d.M != d.N) d.sym = 0;
      d.tiles_m = d.tiles_n = 1;
      d.block_begin = blocks;
      blocks += d.splits * d.nb1 * d.nb2;
      const double nbt = (double)d.nb1 * d.nb2;
      // symmetric outputs: the flops of the upper triangle (the mirrored half is not computed)
      flops += (d.sym ? 1.0 * d.M * (d.N + 1) : 2.0 * d.M * d.N) * (double)d.K * d.KO * nbt;
      bytes += 8.0 * nbt * ((double)d.M * d.K * d.KO + (double)d.K * d.KO * d.N + (double)d.M * d.N * d.splits);
      batch.d[batch.count++] = d;
    }
    if (batch.count == 0) continue;
    ProfToken tok = prof_begin(stream);
    lrt_kernel<<<blocks, LRT_THREADS, lr_smem(), stream>>>(batch);
    HT_LAUNCH_CHECK();
    prof_end(tok, tag, stream, count_flops ? flops : 0.0, count_flops ? bytes : 0.0);
  }
  return kOk;
}
// HT_GEMM_LR=0 routes everything through the generic tiles (A/B comparisons)
const int g_lr_enabled = [] {
  const char* e = std::getenv("HT_GEMM_LR");
  return e && e[0] == '0' ? 0 : 1;
}();

// ---- tile configurations ----
int g_half_tiles = 1;
enum Cfg { kC64, kCN104, kCM104, kCN56, kCM56, kCN104h, kCM104h, kNumCfg };

struct CfgInfo {
  int bm, bn;
};
// *h: half-height tiles with 8 warps x (8 x 104) fragments, <= 128 registers, two CTAs
// per SM (one CTA's pipeline fill / epilogue overlaps the other's DMMA main loop)
constexpr CfgInfo kCfg[kNumCfg] = {{64, 64}, {128, 104}, {104, 128}, {128, 56}, {56, 128}, {64, 104}, {104, 64}};

Cfg pick_cfg(const GemmDesc& d) {
  // a handful of rank-sized products (root / top-level GEMMs): latency-bound, so spread
  // each over 64 x 64 tiles (four CTAs for 100 x 100) rather than one big tile
  if (d.M <= 128 && d.N <= 128 && (long long)d.K * std::max(d.KO, 1) <= 256 && (long long)d.nb1 * d.nb2 <= 4)
    return kC64;
  // half-height tiles only pay off for short reductions (the rank-sized K of the mode
  // products and Q = A R^-1); long (split-K) reductions keep the full tiles
  const bool half = g_half_tiles && (long long)d.K * std::max(d.KO, 1) <= 512;
  if (d.N <= 56 && d.M > 56) return kCN56;
  if (d.M <= 56 && d.N > 56) return kCM56;
  if (d.N <= 104 && d.M > 104) return half ? kCN104h : kCN104;
  if (d.M <= 104 && d.N > 104) return half ? kCM104h : kCM104;
  if (d.M <= 64 && d.N <= 64) return kC64;
  if (d.N <= 104 && d.M <= 104) {
    if (half) return d.N >= d.M ? kCM104h : kCN104h;
    return d.N >= d.M ? kCM104 : kCN104;
  }
  return kCN104;
}

size_t smem_for(Cfg c) { return (size_t)STAGES * BK * (pitch16(kCfg[c].bm) + pitch16(kCfg[c].bn)) * sizeof(double); }

template <int WM, int WN, int WMW, int WNW>
int launch_cfg(GemmBatch& batch, int blocks, size_t smem, cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    HT_CUDA_CHECK(cudaFuncSetAttribute(gemm_kernel<WM, WN, WMW, WNW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    attr = true;
  }
  gemm_kernel<WM, WN, WMW, WNW><<<blocks, THREADS, smem, stream>>>(batch);
  HT_LAUNCH_CHECK();
  return kOk;
}

int launch_batch(Cfg c, GemmBatch& batch, int blocks, cudaStream_t stream) {
  const size_t smem = smem_for(c);
  switch (c) {
    case kC64: return launch_cfg<4, 2, 2, 4>(batch, blocks, smem, stream);     // 64 x 64
    case kCN104: return launch_cfg<2, 13, 8, 1>(batch, blocks, smem, stream);  // 128 x 104
    case kCM104: return launch_cfg<13, 2, 1, 8>(batch, blocks, smem, stream);  // 104 x 128
    case kCN56: return launch_cfg<2, 7, 8, 1>(batch, blocks, smem, stream);    // 128 x 56
    case kCM56: return launch_cfg<7, 2, 1, 8>(batch, blocks, smem, stream);    // 56 x 128
    case kCN104h: return launch_cfg<1, 13, 8, 1>(batch, blocks, smem, stream); // 64 x 104
    case kCM104h: return launch_cfg<13, 1, 1, 8>(batch, blocks, smem, stream); // 104 x 64
    default: break;
  }
  set_error("gemm: bad tile config");
  return kErrArgument;
}

}  // namespace

int gemm_tiles(int M, int N) {  // tiles of a long-reduction (split-K planned) GEMM
  GemmDesc d{};
  d.M = M;
  d.N = N;
  d.K = 1 << 20;
  d.KO = 1;
  const Cfg c = pick_cfg(d);
  return ceil_div(M, kCfg[c].bm) * ceil_div(N, kCfg[c].bn);
}

int gemm_grouped(std::vector<GemmDesc>& descs_in, cudaStream_t stream, const char* tag, bool count_flops) {
  if (g_sync_check > 1 || (g_sync_check && getenv("HT_SYNC_DUMP")))
    for (const auto& d : descs_in)
      fprintf(stderr,
              "[gemm %s] M=%d N=%d K=%d KO=%d nb=%d,%d S=%d A=%p(%lld,%lld,%lld,%lld) B=%p(%lld,%lld,%lld,%lld) "
              "C=%p(%lld,%lld,%lld) tri=%d,%d act=%p sym=%d ab=%g,%g\n",
              tag ? tag : "-", d.M, d.N, d.K, d.KO, d.nb1, d.nb2, d.splits, (const void*)d.A, d.a_m, d.a_k, d.a_o,
              d.a_b1, (const void*)d.B, d.b_k, d.b_n, d.b_o, d.b_b1, (void*)d.C, d.c_m, d.c_n, d.c_b1, d.a_tri,
              d.b_tri, (const void*)d.active, d.sym, d.alpha, d.beta);
  std::vector<std::pair<GemmDesc, int>> lr;
  std::vector<GemmDesc> descs;
  for (const auto& d : descs_in) {
    if (d.M <= 0 || d.N <= 0 || d.nb1 <= 0 || d.nb2 <= 0) continue;
    const int l = g_lr_enabled ? lr_layout(d) : -1;
    if (l >= 0) lr.emplace_back(d, l);
    else descs.push_back(d);
  }
  if (!lr.empty()) HT_TRY(lr_grouped(lr, stream, tag, count_flops));
  for (int c = 0; c < kNumCfg; ++c) {
    size_t i = 0;
    while (i < descs.size()) {
      GemmBatch batch;
      batch.count = 0;
      int blocks = 0;
      double flops = 0, bytes = 0;
      while (i < descs.size() && batch.count < kMaxGemmDescs) {
        GemmDesc d = descs[i++];
        if (d.M <= 0 || d.N <= 0 || d.nb1 <= 0 || d.nb2 <= 0) continue;
        if (pick_cfg(d) != (Cfg)c) continue;
        if (d.splits < 1) d.splits = 1;
        if (d.KO < 1) d.KO = 1;
        d.tiles_m = ceil_div(d.M, kCfg[c].bm);
        d.tiles_n = ceil_div(d.N, kCfg[c].bn);
        d.block_begin = blocks;
        const long long nb = (long long)d.tiles_m * d.tiles_n * d.splits * d.nb1 * d.nb2;
        if (nb > (1LL << 30)) {
          set_error("gemm_grouped: grid too large");
          return kErrArgument;
        }
        blocks += (int)nb;
        const double nbt = (double)d.nb1 * d.nb2;
        flops += 2.0 * d.M * d.N * (double)d.K * d.KO * nbt;
        bytes += 8.0 * nbt * ((double)d.M * d.K * d.KO + (double)d.K * d.KO * d.N + (double)d.M * d.N * d.splits);
        batch.d[batch.count++] = d;
      }
      if (batch.count == 0) continue;
      ProfToken tok = prof_begin(stream);
      HT_TRY(launch_batch((Cfg)c, batch, blocks, stream));
      prof_end(tok, tag, stream, count_flops ? flops : 0.0, count_flops ? bytes : 0.0);
    }
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

namespace ht {
// Debugging aid (HT_SYNC_CHECK=3): one fixed split-K long-reduction GEMM on a private
// buffer, synchronised; non-zero if it faults (localises kernels that corrupt state).
int debug_probe() {
  static double* buf = nullptr;
  static bool busy = false;
  if (busy) return 0;
  busy = true;
  if (!buf && cudaMalloc(&buf, sizeof(double) * (150 * 2048 + 8 * 76 * 74)) != cudaSuccess) return 1;
  GemmDesc g = gemm_desc(buf, 2048, 1, buf + 76 * 2048, 1, 2048, buf + 150 * 2048, 74, 1, 76, 74, 2048);
  g.splits = 8;
  g.c_b1 = 76 * 74;
  std::vector<GemmDesc> v{g};
  const int sc = g_sync_check;
  (void)sc;
  int rc = gemm_grouped(v, 0, "probe", false);
  cudaError_t e = cudaDeviceSynchronize();
  busy = false;
  return rc != kOk || e != cudaSuccess;
}
}  // namespace ht
