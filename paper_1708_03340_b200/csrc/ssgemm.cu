// Stationary-operand streaming GEMM (see ssgemm.cuh).
#include <algorithm>
#include <cstdlib>

#include "prof.cuh"
#include "ssgemm.cuh"

namespace ht {
namespace {

#ifndef HT_SS2_DEBUG_NOLOAD
#define HT_SS2_DEBUG_NOLOAD 0
#endif
#ifndef HT_SS2_DEBUG_SMALLC
#define HT_SS2_DEBUG_SMALLC 0
#endif
#ifndef HT_SS2_DEBUG_NOSTORE
#define HT_SS2_DEBUG_NOSTORE 0
#endif
#ifndef HT_SS2_CONS
#define HT_SS2_CONS 8
#endif
#ifndef HT_SS2_STAGES
#define HT_SS2_STAGES 5
#endif
constexpr int SBM = 16 * HT_SS2_CONS;  // rows per output tile (16 per consumer warp: two m8 fragments)
constexpr int SBK = 16;                // k-chunk per pipeline stage
constexpr int kSsMaxDescs = 32;
constexpr int kSMs = 148;
#ifndef SS_DEBUG_NO_EPILOGUE
#define SS_DEBUG_NO_EPILOGUE 0
#endif
#ifndef SS_DEBUG_NO_XLOAD
#define SS_DEBUG_NO_XLOAD 0
#endif

__host__ __device__ constexpr int ss_pitch(int x) { return ((x + 15) / 16) * 16 + 4; }  // 4 mod 16 doubles
constexpr int PX = ss_pitch(SBM);

struct SsBatch {
  int count;
  int tile_begin[kSsMaxDescs + 1];  // prefix sums of jobs * tiles_m
  int tiles_m[kSsMaxDescs];
  int kp;                            // K rounded up to SBK (smem rows of S)
  unsigned char vec[kSsMaxDescs];    // 16-byte X copies are legal for this descriptor
  SsDesc d[kSsMaxDescs];
};

__device__ __forceinline__ void cp8z(double* smem, const double* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0));
}

__device__ __forceinline__ void cp16z(double* smem, const double* gmem, int valid_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid_bytes));
}

constexpr int PK = SBK + 4;  // [m][k] layout pitch (4 mod 16 doubles: conflict-free fragments)
constexpr int XSTAGE = (SBK * PX > SBM * PK) ? SBK * PX : SBM * PK;  // doubles per stage

// X staging.  LAYOUT 0: X m-contiguous (x_lo == 1), staged [k][m]; copies are row
// pairs (m, m+1).  LAYOUT 1: X k-contiguous (x_k == 1), staged [m][k]; copies are k
// pairs.  VEC: pairs are 16-byte aligned and never straddle an M_lo boundary -> one
// 16-byte cp.async per pair, else two 8-byte ones.

// ---- warp-specialised pipeline ------------------------------------------------
// 8 consumer warps x 16 rows with S resident in shared memory; two producer warps
// stage the X chunks (cp.async, completion counted on a
// per-stage `full` mbarrier) and the consumers release each stage on an `empty`
// mbarrier: no CTA-wide barrier per 16-deep k-chunk, so consumer warps drift and the
// producers run up to SS2_STAGES chunks ahead, across tile boundaries.  The only CTA
// barriers left are at job (segment) boundaries, where S is reloaded.
// Triangular stationary operands: the MMA fragments j of k-chunk kc that are not
// structurally zero form one contiguous range [lo, hi) (TRI 1: S(k, n) = 0 for k < n ->
// j < 2 kc + 2; TRI 2: S(k, n) = 0 for k > n -> j >= 2 kc).  Each chunk index gets its
// own fully unrolled, branch-free MMA sequence (a per-fragment skip branch kept ptxas
// from interleaving the fragments' dependent DMMA chains).
template <int NF, int TRI, int KC>
struct TriRange {
  static constexpr int lo = TRI == 2 ? (2 * KC < NF ? 2 * KC : NF) : 0;
  static constexpr int hi = TRI == 1 ? (2 * KC + 2 < NF ? 2 * KC + 2 : NF) : NF;
};

template <int LO, int HI, int J0, int NJ, int PS>
__device__ __forceinline__ void ss_mma_range(double (&acc)[NJ][4], const double (&a)[8], const double* ss, int t4,
                                             int g8) {
  constexpr int lo = LO > J0 ? LO : J0;
  constexpr int hi = HI < J0 + NJ ? HI : J0 + NJ;
#pragma unroll
  for (int j = lo; j < hi; ++j) {
    double bq[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) bq[i] = ss[(t4 + 4 * i) * PS + j * 8 + g8];
    dmma_16x8x16(acc[j - J0], a, bq);
  }
}

template <int NF, int TRI, int PS, int J0, int NJ>
__device__ __forceinline__ void ss_mma_chunk(int kc, double (&acc)[NJ][4], const double (&a)[8], const double* ss,
                                             int t4, int g8) {
  if (TRI == 0) {
    ss_mma_range<0, NF, J0, NJ, PS>(acc, a, ss, t4, g8);
    return;
  }
  switch (kc) {
#define HT_SS_CASE(c)                                                                                          \
  case c:                                                                                                     \
    ss_mma_range<TriRange<NF, TRI, c>::lo, TriRange<NF, TRI, c>::hi, J0, NJ, PS>(acc, a, ss, t4, g8);        \
    break;
    HT_SS_CASE(0) HT_SS_CASE(1) HT_SS_CASE(2) HT_SS_CASE(3) HT_SS_CASE(4) HT_SS_CASE(5) HT_SS_CASE(6)
#undef HT_SS_CASE
    default:  // kc >= 7 (K > 112): every fragment of a TRI 1 chunk, j >= 14 of TRI 2 (none when NF <= 13)
      ss_mma_range<TriRange<NF, TRI, 7>::lo, TriRange<NF, TRI, 7>::hi, J0, NJ, PS>(acc, a, ss, t4, g8);
      break;
  }
}

// (Measured alternatives that lost: n-split consumer warps, 16 warps x half the
// fragments; two consumer groups on alternate tiles half a tile out of phase, to overlap
// one group's epilogue with the other's MMAs: +5 % dense, -5 % triangular.)
constexpr int SS2_CONS = HT_SS2_CONS;
constexpr int SS2_PROD = 2;
constexpr int SS2_T = (SS2_CONS + SS2_PROD) * 32;
constexpr int SS2_STAGES = HT_SS2_STAGES;

// Consumer warp: 16 rows (row group rg) x fragments [J0, J0 + NJ) of every tile of the
// CTA's segment; X chunks from the `full` ring, released on `empty`.
template <int NF, int LAYOUT, int TRI, int PS, int J0, int NJ>
__device__ __forceinline__ void ss2_consume(const SsDesc& g, const double* Xs, const double* Ss,
                                            unsigned long long* full, unsigned long long* empty, unsigned& gs,
                                            int mt0, int seg, int KT, double* C, int rg, int lane) {
  const int K = g.K, N = g.N, M = g.M, M_lo = g.M_lo;
  double acc[NJ][4];
  const int g8 = lane >> 2, t4 = lane & 3;
  const int ar = rg * 16 + g8;
  const double alpha = g.alpha, beta = g.beta;
  auto xa = [&](const double* xs, int rs, int k) -> double {
    return LAYOUT == 0 ? xs[k * PX + ar + 8 * rs] : xs[(ar + 8 * rs) * PK + k];
  };
  for (int mt = mt0; mt < mt0 + seg; ++mt) {
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
    for (int kc = 0; kc < KT; ++kc, ++gs) {
      const int st = gs % SS2_STAGES;
      mbar_wait(&full[st], (gs / SS2_STAGES) & 1);
      const double* xs = Xs + st * XSTAGE;
      const double* ss = Ss + kc * SBK * PS;
      const int kv = K - kc * SBK;
      if (kv >= 12) {
        double a[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = xa(xs, i & 1, t4 + 4 * (i >> 1));
        ss_mma_chunk<NF, TRI, PS, J0, NJ>(kc, acc, a, ss, t4, g8);
      } else {
        int k0 = 0;
        if (kv > 4) {
          double a[4], bq[2];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = xa(xs, i & 1, t4 + 4 * (i >> 1));
#pragma unroll
          for (int j = J0; j < J0 + NJ; ++j) {
            bq[0] = ss[t4 * PS + j * 8 + g8];
            bq[1] = ss[(t4 + 4) * PS + j * 8 + g8];
            dmma_16x8x8(acc[j - J0], a, bq);
          }
          k0 = 8;
        }
        if (kv > k0) {
          double a[2], bq[1];
          a[0] = xa(xs, 0, k0 + t4);
          a[1] = xa(xs, 1, k0 + t4);
#pragma unroll
          for (int j = J0; j < J0 + NJ; ++j) {
            bq[0] = ss[(k0 + t4) * PS + j * 8 + g8];
            dmma_16x8x4(acc[j - J0], a, bq);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (HT_SS2_DEBUG_NOSTORE) {  // timing experiments: keep the MMAs alive, store nothing
      double z = 0.0;
#pragma unroll
      for (int j = 0; j < NJ; ++j) z += acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
      if (alpha == 12345.0) C[lane] = z;
      continue;
    }
    // m-contiguous outputs (c_lo == 1, e.g. t1^T and the projections): lanes g8 and
    // g8 ^ 1 swap one value per fragment so each stores a 16-byte (m, m + 1) pair
    // (dense stationary operands only: the triangular instances are register-bound)
    const bool mpair = TRI == 0 && beta == 0.0 && g.c_lo == 1 && g.c_n != 1 && !(M_lo & 1) && !(g.c_hi & 1) &&
                       !(g.c_n & 1) && !(((uintptr_t)C) & 15);
    if (mpair) {
      const bool odd = g8 & 1;
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const int m0 = (HT_SS2_DEBUG_SMALLC ? 0 : mt * SBM) + rg * 16 + 8 * f + (g8 & ~1);
        const int hi = m0 / M_lo, lo = m0 - hi * M_lo;
        double* crow = C + hi * g.c_hi + lo;
#pragma unroll
        for (int j = J0; j < J0 + NJ; ++j) {
          const double keep = odd ? acc[j - J0][2 * f + 1] : acc[j - J0][2 * f];
          const double got = __shfl_xor_sync(0xffffffffu, odd ? acc[j - J0][2 * f] : acc[j - J0][2 * f + 1], 4);
          const int col = j * 8 + 2 * t4 + (odd ? 1 : 0);
          if (col < N && m0 < M) {
            double* p = crow + (long long)col * g.c_n;
            const double r0 = alpha * (odd ? got : keep), r1 = alpha * (odd ? keep : got);
            if (m0 + 1 < M) *reinterpret_cast<double2*>(p) = make_double2(r0, r1);
            else *p = r0;
          }
        }
      }
    } else
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int m = (HT_SS2_DEBUG_SMALLC ? 0 : mt * SBM) + ar + 8 * f;
      if (m < M) {
        const int hi = m / M_lo, lo = m - hi * M_lo;
        double* crow = C + hi * g.c_hi + lo * g.c_lo;
        const bool pair = g.c_n == 1 && ((((uintptr_t)crow) & 15) == 0);
#pragma unroll
        for (int j = J0; j < J0 + NJ; ++j) {
          const int n = j * 8 + 2 * t4;
          const double v0 = acc[j - J0][2 * f], v1 = acc[j - J0][2 * f + 1];
          if (pair && n + 1 < N) {
            double2 r = make_double2(alpha * v0, alpha * v1);
            double2* p = reinterpret_cast<double2*>(crow + n);
            if (beta != 0.0) {
              const double2 o = *p;
              r.x += beta * o.x;
              r.y += beta * o.y;
            }
            *p = r;
          } else {
            if (n < N) {
              double* p = crow + (long long)n * g.c_n;
              *p = beta != 0.0 ? alpha * v0 + beta * *p : alpha * v0;
            }
            if (n + 1 < N) {
              double* p = crow + (long long)(n + 1) * g.c_n;
              *p = beta != 0.0 ? alpha * v1 + beta * *p : alpha * v1;
            }
          }
        }
      }
    }
  }
}

template <int NF, int LAYOUT, int TRI>
__global__ void __launch_bounds__(SS2_T, 1) ss2_kernel(const __grid_constant__ SsBatch b) {
  constexpr int NP = NF * 8;
  constexpr int PS = ss_pitch(NP);
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned long long full[SS2_STAGES], empty[SS2_STAGES];
  double* Xs = smem;                       // [SS2_STAGES][XSTAGE]
  double* Ss = smem + SS2_STAGES * XSTAGE;  // [kp][PS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int total = b.tile_begin[b.count];
  const int G = gridDim.x;
  int t = (int)((long long)blockIdx.x * total / G);
  const int t_end = (int)((long long)(blockIdx.x + 1) * total / G);
  if (tid == 0) {
    for (int i = 0; i < SS2_STAGES; ++i) {
      mbar_init(&full[i], 32 * SS2_PROD);
      mbar_init(&empty[i], SS2_CONS);
    }
    mbar_fence_init();
  }
  unsigned gs = 0;  // ring position: steps issued / consumed so far (both roles agree)

  while (t < t_end) {
    int di = 0;
    while (di + 1 < b.count && t >= b.tile_begin[di + 1]) ++di;
    const SsDesc& g = b.d[di];
    const int tm = b.tiles_m[di];
    const int local = t - b.tile_begin[di];
    const int job = local / tm, mt0 = local - job * tm;
    const int seg = min(t_end - t, tm - mt0);  // tiles of this (desc, job) in this CTA
    if (g.active && *g.active == 0) {
      t += seg;
      continue;
    }
    const int K = g.K, N = g.N, M = g.M, M_lo = g.M_lo;
    const int KT = (K + SBK - 1) / SBK;
    const double* X = g.X + job * g.x_job;
    const double* S = g.S + job * g.s_job;
    double* C = g.C + job * g.c_job;
    const bool vec = b.vec[di];
    __syncthreads();  // the previous segment is done with S (and the barriers are initialised)
    if (g.s_n == 1 && !(g.s_k & 1) && !(((uintptr_t)S) & 15)) {
      // rows of S contiguous along n: 16-byte copies of (n, n + 1) pairs
      for (int e = tid; e < KT * SBK * (NP / 2); e += SS2_T) {
        const int k = e / (NP / 2), n = 2 * (e - k * (NP / 2));
        const int nv = k < K ? max(0, min(2, N - n)) : 0;
        cp16z(Ss + k * PS + n, nv ? S + (long long)k * g.s_k + n : S, 8 * nv);
      }
    } else {
      for (int e = tid; e < KT * SBK * NP; e += SS2_T) {
        const int k = e / NP, n = e - k * NP;
        const bool ok = k < K && n < N;
        cp8z(Ss + k * PS + n, ok ? S + k * g.s_k + n * g.s_n : S, ok);
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    const int nsteps = seg * KT;

    if (warp >= SS2_CONS) {
      // ---------------- producers ----------------
      const int pl = tid - SS2_CONS * 32;  // 0 .. 63
      int mt = mt0, kc = 0;
      // LAYOUT 0: pair (2 mp, 2 mp + 1), mp = pl, k rows kk = 0..15 (all)
      // LAYOUT 1: rows pl / 8 + 8 q (q < 16), k pair 2 (pl % 8)
      const double* rowp[LAYOUT == 0 ? 2 : 16];
      int rv = 0;             // LAYOUT 0: valid rows of the pair; LAYOUT 1: bit q = row valid
      auto set_rows = [&](int mtile) {
        if (LAYOUT == 0) {
          const int m = mtile * SBM + 2 * pl;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int mm = min(m + u, M - 1);
            const int hi = mm / M_lo, lo = mm - hi * M_lo;
            rowp[u] = X + hi * g.x_hi + lo * g.x_lo;
          }
          rv = max(0, min(2, M - m));
        } else {
          rv = 0;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int m = mtile * SBM + (pl >> 3) + 8 * q;
            const int mm = m < M ? m : 0;
            if (m < M) rv |= 1 << q;
            const int hi = mm / M_lo, lo = mm - hi * M_lo;
            rowp[q] = X + hi * g.x_hi + lo * g.x_lo;
          }
        }
      };
      set_rows(mt);
      for (int s = 0; s < nsteps; ++s, ++gs) {
        const int st = gs % SS2_STAGES;
        mbar_wait(&empty[st], ((gs / SS2_STAGES) & 1) ^ 1);
        double* xs = Xs + st * XSTAGE;
        const int kb = kc * SBK;
        if (HT_SS2_DEBUG_NOLOAD && s >= SS2_STAGES) {
        } else if (LAYOUT == 0) {
          const int r = 2 * pl;
#pragma unroll
          for (int kk = 0; kk < SBK; ++kk) {
            const int nv = kb + kk < K ? rv : 0;
            const long long ko = (long long)(kb + kk) * g.x_k;
            double* dst = xs + kk * PX + r;
            if (vec) {
              cp16z(dst, nv ? rowp[0] + ko : X, 8 * nv);
            } else {
              cp8z(dst, nv > 0 ? rowp[0] + ko : X, nv > 0);
              cp8z(dst + 1, nv > 1 ? rowp[1] + ko : X, nv > 1);
            }
          }
        } else {
          const int kk = 2 * (pl & 7);
          const int kv = max(0, min(2, K - (kb + kk)));
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int r = (pl >> 3) + 8 * q;
            const int nv = (rv >> q) & 1 ? kv : 0;
            double* dst = xs + r * PK + kk;
            if (vec) {
              cp16z(dst, nv ? rowp[q] + kb + kk : X, 8 * nv);
            } else {
              cp8z(dst, nv > 0 ? rowp[q] + kb + kk : X, nv > 0);
              cp8z(dst + 1, nv > 1 ? rowp[q] + kb + kk + 1 : X, nv > 1);
            }
          }
        }
        cp_async_mbar_arrive(&full[st]);
        if (++kc == KT) {
          kc = 0;
          if (++mt < mt0 + seg) set_rows(mt);
        }
      }
    } else {
      // ---------------- consumers ----------------
      ss2_consume<NF, LAYOUT, TRI, PS, 0, NF>(g, Xs, Ss, full, empty, gs, mt0, seg, KT, C, warp, lane);
    }
    t += seg;
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

size_t ss2_smem(int nf, int kp) {
  return sizeof(double) * ((size_t)SS2_STAGES * XSTAGE + (size_t)kp * ss_pitch(nf * 8));
}

template <int NF, int LAYOUT, int TRI>
int launch_ss(SsBatch& b, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    HT_CUDA_CHECK(cudaFuncSetAttribute(ss2_kernel<NF, LAYOUT, TRI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)ss2_smem(NF, kSsMaxK)));
    attr = true;
  }
  const int total = b.tile_begin[b.count];
  const int grid = std::min(total, kSMs);  // persistent: balanced contiguous tile ranges
  ss2_kernel<NF, LAYOUT, TRI><<<grid, SS2_T, ss2_smem(NF, b.kp), s>>>(b);
  HT_LAUNCH_CHECK();
  return kOk;
}

// 16-byte copies of X pairs are legal when every pair start is 16-byte aligned and
// (LAYOUT 0) a row pair never straddles an M_lo boundary.
bool ss_vec_ok(const SsDesc& d, int layout) {
  auto even = [](long long v) { return (v & 1) == 0; };
  if (((uintptr_t)d.X & 15) != 0 || !even(d.x_job) || !even(d.x_hi)) return false;
  if (layout == 0) return even(d.M_lo) && even(d.x_k);
  return even(d.x_lo);
}

}  // namespace

int ss_gemm(std::vector<SsDesc>& descs, cudaStream_t stream, const char* tag, bool count_flops) {
  for (int variant = 0; variant < 12; ++variant) {  // (N <= 56 | N <= 104) x LAYOUT x TRI
    const int nclass = variant / 6, layout = (variant / 3) % 2, tri = variant % 3;
    size_t i = 0;
    while (i < descs.size()) {
      SsBatch b;
      b.count = 0;
      b.tile_begin[0] = 0;
      int kmax = 1;
      double flops = 0, bytes = 0;
      while (i < descs.size() && b.count < kSsMaxDescs) {
        const SsDesc& d = descs[i++];
        if (d.M <= 0 || d.N <= 0 || d.jobs <= 0) continue;
        if (d.K > kSsMaxK || d.N > kSsMaxN || d.K < 1 || (d.x_k != 1 && d.x_lo != 1)) {
          set_error("ss_gemm: operand outside the stationary-operand kernel (K, N or X strides)");
          return kErrUnsupported;
        }
        const int dl = d.x_lo == 1 && d.x_k != 1 ? 0 : 1;  // m-contiguous -> LAYOUT 0
        if ((d.N <= 56 ? 0 : 1) != nclass || dl != layout || d.s_tri != tri) continue;
        const int tm = (d.M + SBM - 1) / SBM;
        b.tiles_m[b.count] = tm;
        b.vec[b.count] = ss_vec_ok(d, layout) ? 1 : 0;
        b.d[b.count] = d;
        b.tile_begin[b.count + 1] = b.tile_begin[b.count] + tm * d.jobs;
        kmax = std::max(kmax, d.K);
        flops += 2.0 * d.M * d.N * (double)d.K * d.jobs;
        bytes += 8.0 * d.jobs * ((double)d.M * d.K + (double)d.K * d.N + (double)d.M * d.N);
        ++b.count;
      }
      if (b.count == 0) continue;
      b.kp = (kmax + SBK - 1) / SBK * SBK;
      ProfToken tok = prof_begin(stream);
      int rc = kErrArgument;
#define HT_SS_CASE(NFv, Lv, Tv) \
  if (nclass == (NFv == 7 ? 0 : 1) && layout == Lv && tri == Tv) rc = launch_ss<NFv, Lv, Tv>(b, stream);
      HT_SS_CASE(7, 0, 0) HT_SS_CASE(7, 0, 1) HT_SS_CASE(7, 0, 2) HT_SS_CASE(7, 1, 0) HT_SS_CASE(7, 1, 1)
      HT_SS_CASE(7, 1, 2) HT_SS_CASE(13, 0, 0) HT_SS_CASE(13, 0, 1) HT_SS_CASE(13, 0, 2) HT_SS_CASE(13, 1, 0)
      HT_SS_CASE(13, 1, 1) HT_SS_CASE(13, 1, 2)
#undef HT_SS_CASE
      HT_TRY(rc);
      prof_end(tok, tag, stream, count_flops ? flops : 0.0, count_flops ? bytes : 0.0);
    }
  }
  return kOk;
}

}  // namespace ht
