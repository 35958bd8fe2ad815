// Level finish of the reduced-Gramian sweep (see gramfin.cuh).
#include <algorithm>

#include <cooperative_groups.h>

#include "gemm.cuh"
#include "gramfin.cuh"
#include "prof.cuh"

namespace ht {
namespace {

constexpr int kGfThreads = 256;
constexpr int kGfCols = 16;  // rows of G and G~ per CTA
constexpr int kGfMaxDescs = 160;

struct GramFinBatch {
  GramFinDesc d[kGfMaxDescs];
  int count;
};

constexpr int kGfCluster = 8;  // CTAs per son: 8 x 16 rows cover K <= 128
__host__ __device__ constexpr int gf_kp(int K) { return (K + 15) / 16 * 16; }
// pitch 4 mod 16 doubles: both the [m][k] (A) and [k][n] (B) fragment reads are conflict-free
__host__ __device__ constexpr int gf_pitch(int K) { return gf_kp(K) + 4; }

size_t gf_smem(int K) {
  const size_t kp = gf_kp(K), pg = gf_pitch(K);
  return sizeof(double) * (kp * pg + 2 * (size_t)kGfCols * pg);
}

constexpr int kGfChunks = kGramFinMaxK / 16;  // k-chunks of the DMMA products (8)

// One 8-CTA cluster per son; CTA r owns rows I = [16r, 16r + 16) of G and G~, and warp w
// of every CTA owns columns [16w, 16w + 16).
//  (0) the warp's B fragments of R^{-T} (R^{-1} rows of its columns) and the CTA's rows I
//      of R^{-1} start loading (registers / cp.async) before anything else;
//  (1) rows I of G = sum of the split-K partials (each partial byte read once per son,
//      spread over the cluster), written to G;
//  (2) W_I = G_I R^{-T} (16 x K, DMMA; zero blocks of the triangular R^{-1} skipped),
//      pushed into every CTA's copy of W = G R^{-T} (DSMEM stores, no round trip);
//  (3) after the cluster barrier, G~_I = R^{-1}_I W (16 x K, DMMA), written to G~.
__global__ void __cluster_dims__(kGfCluster, 1, 1) __launch_bounds__(kGfThreads)
    gram_finish_kernel(const __grid_constant__ GramFinBatch b) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int di = (int)blockIdx.x / kGfCluster;
  const int rank = (int)cluster.block_rank();
  const GramFinDesc& g = b.d[di];
  const int K = g.K, S = g.S;
  const long long KK = (long long)K * K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int I = rank * kGfCols;  // first row of this CTA
  const int jn = max(0, min(kGfCols, K - I));

  extern __shared__ __align__(16) double sm[];
  const int Kp = gf_kp(K), PG = gf_pitch(K);
  double* W = sm;                          // [Kp][PG]: W = G R^{-T} (filled by the cluster)
  double* Gr = W + (size_t)Kp * PG;        // [16][PG]: rows I of G (zero padded)
  double* Ri = Gr + (size_t)kGfCols * PG;  // [16][PG]: rows I of R^{-1} (zero padded)
  // thread layout of the row-block loops: row tr = tid / 16 (0..15), columns
  // tc + 16u (u < 8): 16 consecutive lanes cover 128 contiguous bytes of a row
  const int tr = tid >> 4, tc = tid & 15;
  const int nt = warp * 16;  // this warp's 16 output columns (8 warps x 16 >= Kp)
  const bool sandwich = g.Rinv != nullptr;

  double bR[kGfChunks][2][4];  // B(k, n) = R^{-1}[n][k] of the warp's columns, all k-chunks
  if (sandwich) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");  // all CTAs started (waited in (2))
#pragma unroll
    for (int c = 0; c < kGfChunks; ++c)
#pragma unroll
      for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int n = nt + 8 * f + g8, k = 16 * c + t4 + 4 * i;
          bR[c][f][i] = (n < K && k < K && k >= n) ? g.Rinv[(long long)n * K + k] : 0.0;
        }
    const double* src = g.Rinv + (long long)min(I + tr, K - 1) * K;
    for (int c = 2 * tc; c < Kp; c += 32) {  // rows I of R^{-1}, 8-byte copies (any alignment)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool ok = tr < jn && c + h < K;
        const unsigned sa = (unsigned)__cvta_generic_to_shared(Ri + tr * PG + c + h);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(ok ? src + c + h : src),
                     "r"(ok ? 8 : 0));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }

  // (1) rows I of G = sum of the partials: all eight loads of a partial in flight, two
  // partials per iteration
  {
    constexpr int kE = kGramFinMaxK / 16;  // 8 columns per thread
    const bool row_ok = tr < jn;
    const double* P = g.P + (long long)(I + (row_ok ? tr : 0)) * K;
    double acc[kE];
#pragma unroll
    for (int u = 0; u < kE; ++u) acc[u] = 0.0;
    if (row_ok) {
      int q = 0;
      for (; q + 1 < S; q += 2) {
        const double* P0 = P + q * KK;
        const double* P1 = P0 + KK;
        double v0[kE], v1[kE];
#pragma unroll
        for (int u = 0; u < kE; ++u) {
          const int c = tc + 16 * u;
          v0[u] = c < K ? P0[c] : 0.0;
          v1[u] = c < K ? P1[c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kE; ++u) acc[u] += v0[u] + v1[u];
      }
      if (q < S) {
#pragma unroll
        for (int u = 0; u < kE; ++u) {
          const int c = tc + 16 * u;
          if (c < K) acc[u] += P[q * KK + c];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kE; ++u) {
      const int c = tc + 16 * u;
      if (row_ok && c < K && g.G) g.G[(long long)(I + tr) * K + c] = acc[u];
      if (sandwich && c < Kp) Gr[tr * PG + c] = (row_ok && c < K) ? acc[u] : 0.0;
    }
  }
  if (!sandwich) return;  // uniform over the cluster: no cluster barrier is pending
  __syncthreads();

  // (2) W_I = G_I R^{-T}  (B(k, n) = R^{-1}[n][k] = 0 for k < n: chunks below nt skipped)
  asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  if (nt < Kp && I < Kp) {
    double acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
    for (int c = 0; c < kGfChunks; ++c) {
      const int k0 = 16 * c;
      if (k0 < nt || k0 >= Kp) continue;
      double a[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = Gr[(g8 + 8 * (i & 1)) * PG + k0 + t4 + 4 * (i >> 1)];
      dmma_16x8x16(acc[0], a, bR[c][0]);
      dmma_16x8x16(acc[1], a, bR[c][1]);
    }
    // push rows I of W into every CTA of the cluster
#pragma unroll 1
    for (int dst = 0; dst < kGfCluster; ++dst) {
      double* Wd = cluster.map_shared_rank(W, dst);
#pragma unroll
      for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          *reinterpret_cast<double2*>(Wd + (I + g8 + 8 * h) * PG + nt + 8 * f + 2 * t4) =
              make_double2(acc[f][2 * h], acc[f][2 * h + 1]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  cluster.sync();  // W complete everywhere (release / acquire); Ri landed
  if (jn == 0) return;
  // (3) G~_I = R^{-1}_I W  (R^{-1}[I + i][k] = 0 for k < I + i: chunks below I skipped)
  if (nt < Kp) {
    double acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    for (int k0 = I; k0 < Kp; k0 += 16) {
      double a[8], bq[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = Ri[(g8 + 8 * (i & 1)) * PG + k0 + t4 + 4 * (i >> 1)];
#pragma unroll
      for (int f = 0; f < 2; ++f) {
#pragma unroll
        for (int i = 0; i < 4; ++i) bq[i] = W[(k0 + t4 + 4 * i) * PG + nt + 8 * f + g8];
        dmma_16x8x16(acc[f], a, bq);
      }
    }
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = g8 + 8 * (v >> 1), c = nt + 8 * f + 2 * t4 + (v & 1);
        if (i < jn && c < K) g.Gt[(long long)(I + i) * K + c] = acc[f][v];
      }
  }
}

}  // namespace

int gram_finish(const std::vector<GramFinDesc>& descs, cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    HT_CUDA_CHECK(cudaFuncSetAttribute(gram_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)gf_smem(kGramFinMaxK)));
    attr = true;
  }
  // The split-K sums run on the wide reduction kernel (every SM shares them; a cluster
  // per son would leave the top levels' tens of partials to 8 SMs); the sandwich then
  // reads the finished G_s (L2-resident) with one cluster per son.
  std::vector<ReduceDesc> red;
  std::vector<GramFinDesc> sw;
  for (const auto& d : descs) {
    if (d.K < 1) continue;
    if (d.Rinv && d.K > kGramFinMaxK) {
      set_error("gram_finish: the R^{-1} sandwich needs K <= 128");
      return kErrArgument;
    }
    const double* G = d.G;
    if (d.G && (d.P != d.G || d.S != 1))
      red.push_back(ReduceDesc{d.P, d.G, d.K, 1, 0, 0, d.S, d.K, d.K, 1, 1, 1, 1.0, 0.0});
    else if (!d.G)
      G = d.P;  // G~ of a G that is already final (a received message)
    if (d.Rinv) {
      GramFinDesc e = d;
      e.P = G;
      e.S = 1;
      e.G = nullptr;
      sw.push_back(e);
    }
  }
  HT_TRY(reduce_partials(red, stream));
  size_t i = 0;
  while (i < sw.size()) {
    GramFinBatch b;
    b.count = 0;
    int kmax = 1;
    double bytes = 0, flops = 0;
    while (i < sw.size() && b.count < kGfMaxDescs) {
      const GramFinDesc& d = sw[i++];
      kmax = std::max(kmax, d.K);
      bytes += 8.0 * d.K * d.K * 3;
      flops += 2.0 * d.K * d.K * d.K;  // two triangular K^3 products
      b.d[b.count++] = d;
    }
    ProfToken tok = prof_begin(stream);
    gram_finish_kernel<<<b.count * kGfCluster, kGfThreads, gf_smem(kmax), stream>>>(b);
    HT_LAUNCH_CHECK();
    prof_end(tok, "gram_sandwich", stream, flops, bytes);
  }
  return kOk;
}

}  // namespace ht
