// Stationary-operand streaming GEMM (see ssgemm.cuh).
#include <algorithm>

#include "prof.cuh"
#include "ssgemm.cuh"

namespace ht {
namespace {

constexpr int SST = 256;     // 8 warps
constexpr int SBM = 128;     // rows per output tile (16 per warp: two m8 fragments)
constexpr int SBK = 16;      // k-chunk per pipeline stage
constexpr int NQ = SBM * SBK / SST;  // X elements each thread copies per stage
constexpr int SSTAGES = 4;
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
  int chunk;                         // tiles per CTA
  int kp;                            // K rounded up to SBK (smem rows of S)
  SsDesc d[kSsMaxDescs];
};

__device__ __forceinline__ void cp8z(double* smem, const double* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int NF>
__global__ void __launch_bounds__(SST, 1) ss_kernel(const __grid_constant__ SsBatch b) {
  constexpr int NP = NF * 8;
  constexpr int PS = ss_pitch(NP);
  extern __shared__ __align__(16) double smem[];
  double* Xs = smem;                        // [SSTAGES][SBK][PX]
  double* Ss = smem + SSTAGES * SBK * PX;   // [kp][PS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int total = b.tile_begin[b.count];
  int t = blockIdx.x * b.chunk;
  const int t_end = min(total, t + b.chunk);

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
    const bool kcontig = g.x_k == 1;
    __syncthreads();  // the previous segment is done with the shared buffers

    // stationary operand: S(k, n) for k < KT*SBK, n < NP (zero padded)
    for (int e = tid; e < KT * SBK * NP; e += SST) {
      const int k = e / NP, n = e - k * NP;
      const bool ok = k < K && n < N;
      cp8z(Ss + k * PS + n, ok ? S + k * g.s_k + n * g.s_n : S, ok);
    }

    // loader state: rows this thread copies for the tile currently being loaded
    // k-contiguous X: element e = tid + SST*q -> row e/16 = tid/16 + 16q, kk = tid%16
    // m-contiguous X: element e -> kk = e/128 = tid/128 + 2q, row = tid%128
    int ld_tile = -1;
    const double* rowp[NQ];
    bool rowok[NQ];
    auto set_rows = [&](int mt) {
      ld_tile = mt;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int r = kcontig ? (tid / SBK) + (SST / SBK) * q : (tid & 127);
        const int m = mt * SBM + r;
        rowok[q] = m < M;
        const int mm = rowok[q] ? m : 0;
        const int hi = mm / M_lo, lo = mm - hi * M_lo;
        rowp[q] = X + hi * g.x_hi + lo * g.x_lo;
        if (!kcontig) break;
      }
    };
    const int nsteps = seg * KT;
    auto issue = [&](int s) {
      if (s < nsteps && !(SS_DEBUG_NO_XLOAD && s >= SSTAGES)) {
        const int mt = mt0 + s / KT, kc = s - (s / KT) * KT;
        if (mt != ld_tile) set_rows(mt);
        double* xs = Xs + (s % SSTAGES) * SBK * PX;
        const int kb = kc * SBK;
        if (kcontig) {
          const int kk = tid % SBK;
          const bool kok = kb + kk < K;
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const int r = tid / SBK + (SST / SBK) * q;
            const bool ok = kok && rowok[q];
            cp8z(xs + kk * PX + r, ok ? rowp[q] + (kb + kk) : X, ok);
          }
        } else {
          const int r = tid & 127;
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const int kk = (tid >> 7) + (SST / 128) * q;
            const bool ok = rowok[0] && kb + kk < K;
            cp8z(xs + kk * PX + r, ok ? rowp[0] + (long long)(kb + kk) * g.x_k : X, ok);
          }
        }
      }
      cp_commit();
    };
#pragma unroll
    for (int s = 0; s < SSTAGES - 1; ++s) issue(s);  // S travels with the first group

    double acc[NF][4];  // m16n8 accumulators: rows g, g+8 of the warp's 16, cols 2t, 2t+1
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
    const int g8 = lane >> 2, t4 = lane & 3;
    const int ar = warp * 16 + g8;
    const double alpha = g.alpha, beta = g.beta;
    for (int s = 0; s < nsteps; ++s) {
      cp_wait<SSTAGES - 2>();
      __syncthreads();
      issue(s + SSTAGES - 1);
      const double* xs = Xs + (s % SSTAGES) * SBK * PX;
      const int kc = s % KT;
      const double* ss = Ss + kc * SBK * PS;
      const int krem = K - kc * SBK;  // valid k of this chunk (zero-filled beyond)
#pragma unroll
      for (int k16 = 0; k16 < SBK; k16 += 16) {
        const int kv = krem - k16;
        if (kv <= 0) break;
        const double* xk = xs + k16 * PX;
        const double* sk = ss + k16 * PS;
        if (kv >= 12) {  // m16n8k16 (k rows beyond K are zero in shared memory)
          double a[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) a[i] = xk[(t4 + 4 * (i >> 1)) * PX + ar + 8 * (i & 1)];
#pragma unroll
          for (int j = 0; j < NF; ++j) {
            double bq[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) bq[i] = sk[(t4 + 4 * i) * PS + j * 8 + g8];
            dmma_16x8x16(acc[j], a, bq);
          }
        } else {  // tail: k8 and/or k4 steps
          int k0 = 0;
          if (kv > 4) {
            double a[4], bq[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = xk[(t4 + 4 * (i >> 1)) * PX + ar + 8 * (i & 1)];
#pragma unroll
            for (int j = 0; j < NF; ++j) {
              bq[0] = sk[t4 * PS + j * 8 + g8];
              bq[1] = sk[(t4 + 4) * PS + j * 8 + g8];
              dmma_16x8x8(acc[j], a, bq);
            }
            k0 = 8;
          }
          if (kv > k0) {
            double a[2], bq[1];
            a[0] = xk[(k0 + t4) * PX + ar];
            a[1] = xk[(k0 + t4) * PX + ar + 8];
#pragma unroll
            for (int j = 0; j < NF; ++j) {
              bq[0] = sk[(k0 + t4) * PS + j * 8 + g8];
              dmma_16x8x4(acc[j], a, bq);
            }
          }
        }
      }
      if (SS_DEBUG_NO_EPILOGUE && kc == KT - 1 && alpha == 12345.0) {  // keep the MMAs alive
        for (int j = 0; j < NF; ++j) C[j] = acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
      }
      if (kc == KT - 1 && !SS_DEBUG_NO_EPILOGUE) {  // tile done: epilogue, then restart the accumulators
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          const int m = (mt0 + s / KT) * SBM + ar + 8 * f;
          if (m < M) {
            const int hi = m / M_lo, lo = m - hi * M_lo;
            double* crow = C + hi * g.c_hi + lo * g.c_lo;
            const bool pair = g.c_n == 1 && ((((uintptr_t)crow) & 15) == 0);
#pragma unroll
            for (int j = 0; j < NF; ++j) {
              const int n = j * 8 + 2 * t4;
              const double v0 = acc[j][2 * f], v1 = acc[j][2 * f + 1];
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
#pragma unroll
        for (int j = 0; j < NF; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
      }
      if (SS_DEBUG_NO_EPILOGUE && kc == KT - 1)
        for (int j = 0; j < NF; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
    }
    cp_wait<0>();
    t += seg;
  }
}

size_t ss_smem(int nf, int kp) { return sizeof(double) * ((size_t)SSTAGES * SBK * PX + (size_t)kp * ss_pitch(nf * 8)); }

template <int NF>
int launch_ss(SsBatch& b, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    HT_CUDA_CHECK(cudaFuncSetAttribute(ss_kernel<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)ss_smem(NF, kSsMaxK)));
    attr = true;
  }
  const int total = b.tile_begin[b.count];
  const int grid = (total + b.chunk - 1) / b.chunk;
  ss_kernel<NF><<<grid, SST, ss_smem(NF, b.kp), s>>>(b);
  HT_LAUNCH_CHECK();
  return kOk;
}

}  // namespace

int ss_gemm(std::vector<SsDesc>& descs, cudaStream_t stream, const char* tag, bool count_flops) {
  for (int variant = 0; variant < 2; ++variant) {
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
        if (d.K > kSsMaxK || d.N > kSsMaxN || d.K < 1) {
          set_error("ss_gemm: K or N outside the stationary-operand kernel");
          return kErrUnsupported;
        }
        if ((d.N <= 56 ? 0 : 1) != variant) continue;
        const int tm = (d.M + SBM - 1) / SBM;
        b.tiles_m[b.count] = tm;
        b.d[b.count] = d;
        b.tile_begin[b.count + 1] = b.tile_begin[b.count] + tm * d.jobs;
        kmax = std::max(kmax, d.K);
        flops += 2.0 * d.M * d.N * (double)d.K * d.jobs;
        bytes += 8.0 * d.jobs * ((double)d.M * d.K + (double)d.K * d.N + (double)d.M * d.N);
        ++b.count;
      }
      if (b.count == 0) continue;
      const int total = b.tile_begin[b.count];
      b.chunk = std::max(1, (total + kSMs - 1) / kSMs);
      b.kp = (kmax + SBK - 1) / SBK * SBK;
      ProfToken tok = prof_begin(stream);
      HT_TRY(variant == 0 ? launch_ss<7>(b, stream) : launch_ss<13>(b, stream));
      prof_end(tok, tag, stream, count_flops ? flops : 0.0, count_flops ? bytes : 0.0);
    }
  }
  return kOk;
}

}  // namespace ht
