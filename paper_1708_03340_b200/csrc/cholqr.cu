#include <cstdio>
#include <cstdlib>
// Cholesky-QR2 (see cholqr.cuh).  The GEMMs run on the grouped DMMA kernel of
// gemm.cu; this file holds the batched Cholesky / triangular-inverse kernel and
// the launch sequence.
#include <cmath>
#include <cstdlib>
#include <algorithm>

#include "cholqr.cuh"
#include "gemm.cuh"
#include "prof.cuh"
#include "ssgemm.cuh"
#include "misc.cuh"
#include "cond.cuh"

namespace ht {
namespace {

constexpr int kCholMaxDescs = 48;
// pivot / column-norm^2 below this => kappa(A) ~> 1e5: leave it to Householder
constexpr double kPivotTol = 1e-10;
constexpr double kIdentityTol = 0.1;
// One pass of Cholesky-QR leaves ||Q^T Q - I|| ~ 1e-17 kappa^2 (measured: 3e-15 at
// kappa = 10, 7e-14 at 100).  The second pass runs unless ||R||_F ||R^{-1}||_F
// (>= kappa_2, <= K kappa_2) is at most 300, i.e. kappa_2 <= 300 guaranteed.
constexpr double kKappaOnePass = 300.0;
constexpr int kCholInPlaceK = 104;  // widest output one GEMM tile covers (in-place pass 2)

struct CholDesc {
  const double* W;  // nodes x K x K row-major (only the upper triangle is read)
  double* Rf;       // nodes x K x K: upper Cholesky factor (zeros below)
  double* Ri;       // nodes x K x K: its inverse (upper, zeros below)
  double* Rout;     // optional second copy of Rf (row-major, ld r_ld, node stride r_node)
  long long r_ld, r_node;
  int K, nodes;
  int check_identity;
  const int* active;  // optional: skip unless *active != 0
  int* need2;         // pass 1: OR-ed with 1 when kappa(R) > kappa_max (second pass needed)
  double kappa_max;   // <= 0: second pass always
};

struct CholBatch {
  CholDesc d[kCholMaxDescs];
  int block_begin[kCholMaxDescs + 1];
  int count;
  int* fail;
};

// ---- batched blocked Cholesky ---------------------------------------------------
// One CTA of 8 warps per K x K Gram matrix (the lower triangle is read), the matrix resident in shared memory
// (padded to Kp = 16 * ceil(K / 16), pitch Kp + 4).  Right-looking blocked Cholesky
// W = L L^T with 16-wide panels: the 16 x 16 diagonal block is factored by one warp
// in registers (lane i owns row i; pivot by shuffle, rsqrt, rank-1 update), the panel
// below by a row-per-thread triangular solve, the trailing matrix by DMMA m16n8k16
// tiles.  Then X = L^{-1}: diagonal blocks per warp (column per lane), off-diagonal
// blocks by block distance with DMMA (T = L_{I,*} X_{*,J}, X_{IJ} = -X_{II} T).  X is
// kept transposed in the strict upper triangle (it is R^{-1} = L^{-T} there), its
// diagonal in rinv.  Outputs: R, R^{-1}, the red flag (a pivot loses more than 10
// digits against its column norm, anything non-finite, or -- second pass -- W not
// within 0.1 of I) and the ||R||_F ||R^{-1}||_F estimate that decides the second pass.
#ifndef HT_CHOL_TIMING
#define HT_CHOL_TIMING 0  // 1: block 0 prints its phase times (clock64) -- experiments only
#endif
constexpr int kC2Threads = 256;
constexpr int kC2Warps = kC2Threads / 32;

__host__ __device__ constexpr int c2_pitch(int kp) { return kp + 4; }
size_t chol2_smem(int K) {
  const int kp = (K + 15) / 16 * 16;
  return sizeof(double) * ((size_t)kp * c2_pitch(kp) + 3 * (size_t)kp + (size_t)kC2Warps * 16 * 17);
}

__global__ void __launch_bounds__(kC2Threads, 1) chol2_kernel(const __grid_constant__ CholBatch cb) {
  int di = 0;
  while (di + 1 < cb.count && (int)blockIdx.x >= cb.block_begin[di + 1]) ++di;
  const CholDesc& c = cb.d[di];
  if (c.active && *c.active == 0) return;
  const int node = blockIdx.x - cb.block_begin[di];
  const int K = c.K;
  const int Kp = (K + 15) / 16 * 16, P = c2_pitch(Kp);
  extern __shared__ __align__(16) double sm[];
  double* A = sm;                       // [Kp][P]
  double* d0 = A + (size_t)Kp * P;      // original diagonal
  double* rinv = d0 + Kp;               // 1 / L_ii  (= diagonal of X = L^{-1})
  double* scratch = rinv + 2 * Kp;      // per warp 16 x 17
  __shared__ double red[kC2Warps][2];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const long long off = (long long)node * K * K;
  const double* Wg = c.W + off;
  if (tid == 0) bad = 0;
  long long clk[6] = {clock64(), 0, 0, 0, 0, 0};

  // load: the whole K x K block into A (zero-filled padding) with every copy in flight
  // at once (cp.async, 16-byte pairs when the rows allow); the factorisation reads the
  // lower triangle only (W is symmetric: the Gram GEMMs write both triangles) and the
  // strict upper triangle is overwritten by X = L^{-1} later
  {
    const bool v16 = !(K & 1) && !(((uintptr_t)Wg) & 15);
    const int rw = v16 ? Kp / 2 : Kp;  // copies per row
    for (int e = tid; e < Kp * rw; e += kC2Threads) {
      const int r = e / rw, cc = (e - r * rw) * (v16 ? 2 : 1);
      const unsigned sa = (unsigned)__cvta_generic_to_shared(A + r * P + cc);
      const bool ok = r < K && cc < K;
      const double* src = ok ? Wg + (long long)r * K + cc : Wg;
      if (v16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 16 : 0));
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 8 : 0));
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
  }
  double dev = 0.0;
  bool nonfinite = false;
  for (int r = warp; r < K; r += kC2Warps)
    for (int cc = lane; cc <= r; cc += 32) {
      const double x = A[r * P + cc];
      dev = fmax(dev, fabs(x - (r == cc ? 1.0 : 0.0)));
      nonfinite |= !isfinite(x);
      if (r == cc) d0[r] = x;
    }
  const int any_nonfinite = __syncthreads_or(nonfinite);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
  if (lane == 0) red[warp][0] = dev;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int q = 0; q < kC2Warps; ++q) m = fmax(m, red[q][0]);
    if (any_nonfinite || (c.check_identity && !(m <= kIdentityTol))) bad = 1;
  }

  const int nJ = Kp / 16;
  if (HT_CHOL_TIMING) clk[1] = clock64();
  for (int J = 0; J < nJ; ++J) {
    const int j0 = 16 * J, jb = min(16, K - j0);
    // (a) diagonal block, warp 0, lane i owns row j0 + i; the scaled pivot column is
    // broadcast through shared memory (one STS + LDS.128 reads instead of 15 shuffles)
    if (warp == 0) {
      double x[16];
      double* colb = scratch;  // 16 doubles
      const int i = lane & 15;
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = A[(j0 + i) * P + j0 + k];
      bool flag = false;
      // pivot d -> rsqrt, with the usual check (a failed pivot is replaced and flagged)
      auto pivot = [&](double d, int p, double& dfix) -> double {
        double rs = rsqrt(d);  // issued before the (warp-uniform, rarely taken) check
        const double dd = d0[j0 + p];
        const bool ok = dd > 1e-290 && isfinite(dd) && d > kPivotTol * dd && isfinite(d);
        dfix = d;
        if (!ok) {
          dfix = (dd > 1e-290 && isfinite(dd)) ? dd : 1.0;  // keep going; the node is flagged
          rs = rsqrt(dfix);
          flag = true;
        }
        return rs;
      };
      // software-pipelined: pivot p + 1's diagonal (lane p + 1's own update) and its
      // rsqrt are issued before pivot p's broadcast and rank-1 update of the block
      double dcur, rs = pivot(__shfl_sync(0xffffffffu, x[0], 0), 0, dcur);
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        if (p < jb) {
          const double l = i == p ? dcur * rs : x[p] * rs;
          x[p] = l;
          if (lane == p) rinv[j0 + p] = rs;
          double dnext = 0.0, rsn = 0.0;
          if (p + 1 < jb) {
            const double own = fma(-l, l, x[p + 1]);
            rsn = pivot(__shfl_sync(0xffffffffu, own, p + 1), p + 1, dnext);
          }
          if (lane < 16 && i >= p) colb[i] = l;
          __syncwarp();
#pragma unroll
          for (int j = p + 1; j < 16; ++j)
            if (i >= j) x[j] = fma(-l, colb[j], x[j]);
          __syncwarp();
          dcur = dnext;
          rs = rsn;
        }
      }
      if (lane < jb) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k <= i) A[(j0 + i) * P + j0 + k] = x[k];
      }
      if (flag && lane == 0) bad = 1;
    }
    __syncthreads();
    // (b) panel: rows r >= j0 + 16 solve y L_JJ^T = a
    {
      const int r = j0 + 16 + tid;
      if (r < K) {
        double y[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) y[k] = A[r * P + j0 + k];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          y[k] *= rinv[j0 + k];
#pragma unroll
          for (int k2 = k + 1; k2 < 16; ++k2) y[k2] = fma(-y[k], A[(j0 + k2) * P + j0 + k], y[k2]);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) A[r * P + j0 + k] = y[k];
      }
    }
    __syncthreads();
    // (c) trailing update A[I][cn] -= L[I][J] L[cn][J]^T on the lower tiles (DMMA)
    if (j0 + 16 < K) {
      int tile = warp;
      for (int I = J + 1; I < nJ; ++I) {
        const int ntl = 2 * (I - J);  // n8 tiles cn = 2(J+1) .. 2I+1
        for (; tile < ntl; tile += kC2Warps) {
          const int n0 = 16 * (J + 1) + 8 * tile, i0 = 16 * I;
          double a[8], b[4], acc[4];
#pragma unroll
          for (int q = 0; q < 8; ++q) a[q] = -A[(i0 + g8 + 8 * (q & 1)) * P + j0 + t4 + 4 * (q >> 1)];
#pragma unroll
          for (int q = 0; q < 4; ++q) b[q] = A[(n0 + g8) * P + j0 + t4 + 4 * q];
          acc[0] = A[(i0 + g8) * P + n0 + 2 * t4];
          acc[1] = A[(i0 + g8) * P + n0 + 2 * t4 + 1];
          acc[2] = A[(i0 + g8 + 8) * P + n0 + 2 * t4];
          acc[3] = A[(i0 + g8 + 8) * P + n0 + 2 * t4 + 1];
          dmma_16x8x16(acc, a, b);
          A[(i0 + g8) * P + n0 + 2 * t4] = acc[0];
          A[(i0 + g8) * P + n0 + 2 * t4 + 1] = acc[1];
          A[(i0 + g8 + 8) * P + n0 + 2 * t4] = acc[2];
          A[(i0 + g8 + 8) * P + n0 + 2 * t4 + 1] = acc[3];
        }
        tile -= ntl;
      }
    }
    __syncthreads();
  }

  // X = L^{-1}; X[r][cc] (r > cc) lives at A[cc][r], X[r][r] = rinv[r]
  auto xat = [&](int r, int cc) -> double {  // X element (zero above the diagonal / padding)
    return r >= K ? 0.0 : (r > cc ? A[cc * P + r] : (r == cc ? rinv[r] : 0.0));
  };
  if (HT_CHOL_TIMING) clk[2] = clock64();
  // (d) diagonal blocks: warp w -> block w, lane cc -> column cc
  for (int J = warp; J < nJ; J += kC2Warps) {
    const int j0 = 16 * J;
    const int cc = lane & 15;
    double xc[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      double v = 0.0;
      if (r == cc) v = j0 + r < K ? rinv[j0 + r] : 0.0;
      else if (r > cc && j0 + r < K) {
        double sacc = 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k >= cc && k < r) sacc = fma(A[(j0 + r) * P + j0 + k], xc[k], sacc);
        v = -rinv[j0 + r] * sacc;
      }
      xc[r] = v;
    }
    if (lane < 16) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r > cc) A[(j0 + cc) * P + j0 + r] = xc[r];
    }
  }
  __syncthreads();
  if (HT_CHOL_TIMING) clk[3] = clock64();
  // (e) off-diagonal blocks by block distance: X_IJ = -X_II (sum_k L_Ik X_kJ)
  double* T = scratch + warp * 16 * 17;
  for (int dlt = 1; dlt < nJ; ++dlt) {
    for (int I = dlt + warp; I < nJ; I += kC2Warps) {
      const int Jc = I - dlt, i0 = 16 * I, jc0 = 16 * Jc;
      double acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
      for (int kb = Jc; kb < I; ++kb) {
        const int k0 = 16 * kb;
        double a[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = A[(i0 + g8 + 8 * (q & 1)) * P + k0 + t4 + 4 * (q >> 1)];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double b[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) b[q] = xat(k0 + t4 + 4 * q, jc0 + 8 * h + g8);
          dmma_16x8x16(acc[h], a, b);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        T[g8 * 17 + 8 * h + 2 * t4] = acc[h][0];
        T[g8 * 17 + 8 * h + 2 * t4 + 1] = acc[h][1];
        T[(g8 + 8) * 17 + 8 * h + 2 * t4] = acc[h][2];
        T[(g8 + 8) * 17 + 8 * h + 2 * t4 + 1] = acc[h][3];
      }
      __syncwarp();
      double a[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = -xat(i0 + g8 + 8 * (q & 1), i0 + t4 + 4 * (q >> 1));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double b[4], o[4] = {0, 0, 0, 0};
#pragma unroll
        for (int q = 0; q < 4; ++q) b[q] = T[(t4 + 4 * q) * 17 + 8 * h + g8];
        dmma_16x8x16(o, a, b);
        // X[i0 + row][jc0 + col] -> A[jc0 + col][i0 + row]
        A[(jc0 + 8 * h + 2 * t4) * P + i0 + g8] = o[0];
        A[(jc0 + 8 * h + 2 * t4 + 1) * P + i0 + g8] = o[1];
        A[(jc0 + 8 * h + 2 * t4) * P + i0 + g8 + 8] = o[2];
        A[(jc0 + 8 * h + 2 * t4 + 1) * P + i0 + g8 + 8] = o[3];
      }
      __syncwarp();
    }
    __syncthreads();
  }

  if (HT_CHOL_TIMING) clk[4] = clock64();
  // outputs: R = L^T, R^{-1} = X^T (upper), zeros below; Frobenius norms for kappa
  double* Rf = c.Rf ? c.Rf + off : nullptr;
  double* Ri = c.Ri + off;
  double* Ro = c.Rout ? c.Rout + (long long)node * c.r_node : nullptr;
  double s0 = 0.0, s1 = 0.0;
  for (int e = tid; e < K * K; e += kC2Threads) {
    const int i = e / K, j = e - i * K;
    const double rv = j >= i ? A[j * P + i] : 0.0;
    const double iv = j > i ? A[i * P + j] : (j == i ? rinv[i] : 0.0);
    if (Rf) Rf[e] = rv;
    if (Ro) Ro[(long long)i * c.r_ld + j] = rv;
    Ri[e] = iv;
    s0 = fma(rv, rv, s0);
    s1 = fma(iv, iv, s1);
  }
  if (c.need2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane == 0) { red[warp][0] = s0; red[warp][1] = s1; }
    __syncthreads();
    if (tid == 0) {
      double a0 = 0.0, a1 = 0.0;
      for (int q = 0; q < kC2Warps; ++q) { a0 += red[q][0]; a1 += red[q][1]; }
      if (!(sqrt(a0 * a1) <= c.kappa_max)) atomicOr(c.need2, 1);
    }
  }
  __syncthreads();
  if (tid == 0 && bad) atomicOr(cb.fail, 1);
  if (HT_CHOL_TIMING && tid == 0 && blockIdx.x == 0) {
    clk[5] = clock64();
    printf("chol2 K=%d: load %lld factor %lld inv-diag %lld inv-offdiag %lld out %lld cycles\n", K, clk[1] - clk[0],
           clk[2] - clk[1], clk[3] - clk[2], clk[4] - clk[3], clk[5] - clk[4]);
  }
}

int launch_chol(const std::vector<CholDesc>& ds, int* fail, cudaStream_t s, const char* tag = "cholqr_factor") {
  size_t i = 0;
  while (i < ds.size()) {
    CholBatch b{};
    b.fail = fail;
    int blocks = 0;
    while (i < ds.size() && b.count < kCholMaxDescs) {
      b.d[b.count] = ds[i];
      b.block_begin[b.count] = blocks;
      blocks += ds[i].nodes;
      ++b.count;
      ++i;
    }
    b.block_begin[b.count] = blocks;
    double flops = 0;
    for (int q = 0; q < b.count; ++q) flops += (double)b.d[q].nodes * b.d[q].K * b.d[q].K * b.d[q].K / 1.5;
    ProfToken tok = prof_begin(s);
    static bool attr = false;
    if (!attr) {
      HT_CUDA_CHECK(cudaFuncSetAttribute(chol2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)chol2_smem(kCholMaxK)));
      attr = true;
    }
    int kmax = 1;
    for (int q = 0; q < b.count; ++q) kmax = std::max(kmax, b.d[q].K);
    chol2_kernel<<<blocks, kC2Threads, chol2_smem(kmax), s>>>(b);
    HT_LAUNCH_CHECK();
    prof_end(tok, tag, s, ds[0].active ? 0.0 : flops, 0.0);  // conditional launches: no flop claim
  }
  return kOk;
}

}  // namespace

bool cholqr_eligible(const QrProblem& q) { return q.K >= 1 && q.K <= kCholMaxK && q.m >= 2 * q.K; }

long long cholqr_workspace_doubles(const CholQr& c) {
  const long long K = c.q.K, n = c.q.nodes, m = c.q.m;
  const long long kk = K * K * n;
  return (c.S > 1 ? c.S * kk : 0) + kk + m * K * n + 4 * kk + 5 * 32;
}

void cholqr_bind(CholQr& c, double* ws) {
  const long long K = c.q.K, n = c.q.nodes, m = c.q.m;
  const long long kk = K * K * n;
  auto al = [](double* p) { return (double*)(((uintptr_t)p + 255) & ~(uintptr_t)255); };
  double* p = al(ws);
  if (c.S > 1) {
    c.P = p;
    p = al(p + c.S * kk);
  }
  c.W = p; p = al(p + kk);
  c.Q1 = p; p = al(p + m * K * n);
  c.R1 = p; p = al(p + kk);
  c.R2 = p; p = al(p + kk);
  c.Ri = p;
}

int cholqr_run(std::vector<CholQr>& cs, int* fail, int* need2, bool two_pass, cudaStream_t s) {
  if (cs.empty()) return kOk;
  // need2[p]: problem p needs the second pass (kappa estimate above kKappaOnePass, or K
  // too wide for the in-place second pass)
  HT_CUDA_CHECK(cudaMemsetAsync(need2, 0, sizeof(int) * cs.size(), s));
  // Gram GEMM of X (m x K, element (r, i) at X + r*xr + i*xc, node stride xn) into W
  auto gram = [&](std::vector<GemmDesc>& g, std::vector<ReduceDesc>& r, const CholQr& c, const double* X,
                  long long xr, long long xc, long long xn, const int* active) {
    const int K = c.q.K, m = c.q.m, n = c.q.nodes;
    GemmDesc d = gemm_desc(X, xc, xr, X, xr, xc, c.S > 1 ? c.P : c.W, K, 1, K, K, m);
    d.nb1 = n; d.a_b1 = xn; d.b_b1 = xn; d.c_b1 = (long long)K * K;
    d.splits = c.S;
    d.active = active;
    d.sym = 1;
    g.push_back(d);
    if (c.S > 1) {
      ReduceDesc rd{c.P, c.W, K, 1, (long long)K * K, 0, c.S, K, K, n, 1, 0, 1.0, 0.0};
      rd.active = active;
      r.push_back(rd);
    }
  };
  std::vector<GemmDesc> g;
  std::vector<ReduceDesc> r;
  std::vector<CholDesc> ch;
  // pass 1: W1 = A^T A, R1 = chol(W1) (also written as the final R), kappa estimate
  for (auto& c : cs) gram(g, r, c, c.q.A, c.q.a_r, c.q.a_c, c.q.a_node, nullptr);
  HT_TRY(gemm_grouped(g, s, "gemm_cholqr_gram"));
  HT_TRY(reduce_partials(r, s));
  for (size_t p = 0; p < cs.size(); ++p) {
    const CholQr& c = cs[p];
    CholDesc d{};
    // R1 goes to the output R only (the rarely taken second pass copies it back into
    // c.R1 first): one fewer K x K store per node on the critical path
    d.W = c.W; d.Rf = nullptr; d.Ri = c.q.rinv ? c.q.rinv : c.Ri; d.Rout = c.q.R; d.r_ld = c.q.r_ld;
    d.r_node = c.q.r_node;
    d.K = c.q.K; d.nodes = c.q.nodes;
    d.need2 = need2 + p;
    d.kappa_max = (c.q.K <= kCholInPlaceK && !two_pass) ? kKappaOnePass : 0.0;
    ch.push_back(d);
  }
  HT_TRY(launch_chol(ch, fail, s));
  g.clear(); r.clear(); ch.clear();
  // Q1 = A R1^{-1}, straight into the output when the second pass can run in place
  // (one CTA owns whole output rows: K <= 104), else into scratch.  R1^{-1} is the
  // stationary operand of the streaming GEMM.
  std::vector<SsDesc> sd;
  for (auto& c : cs) {
    const int K = c.q.K, m = c.q.m;
    if (c.q.rinv) continue;  // implicit Q: A and R^{-1} stand for Q
    if (K <= kCholInPlaceK) {
      SsDesc d = ss_desc(c.q.A, c.q.a_r, c.q.a_c, c.Ri, K, 1, c.q.Q, c.q.q_r, c.q.q_c, m, K, K);
      d.jobs = c.q.nodes; d.x_job = c.q.a_node; d.s_job = (long long)K * K; d.c_job = c.q.q_node;
      d.s_tri = 2;  // R^{-1} upper triangular
      sd.push_back(d);
      continue;
    }
    GemmDesc d = gemm_desc(c.q.A, c.q.a_r, c.q.a_c, c.Ri, K, 1, c.Q1, K, 1, m, K, K);
    d.nb1 = c.q.nodes; d.a_b1 = c.q.a_node; d.b_b1 = (long long)K * K; d.c_b1 = (long long)m * K;
    g.push_back(d);
  }
  HT_TRY(ss_gemm(sd, s, "ss_cholqr_q"));
  HT_TRY(gemm_grouped(g, s, "gemm_cholqr_q"));
  g.clear();
  sd.clear();
  // pass 2 (skipped on the device unless need2): W2 = Q1^T Q1, R2 = chol(W2),
  // Q = Q1 R2^{-1}, R = R2 R1.  Inside the library's own graph captures the five
  // launches sit in an IF node taken only when some need2 flag is set; elsewhere they
  // are enqueued and exit on their device flags.
  auto pass2 = [&](cudaStream_t s) -> int {
    // implicit-Q problems form their first-pass Q1 = A R1^{-1} only now (in place when
    // one CTA owns whole rows, else into scratch)
    for (size_t p = 0; p < cs.size(); ++p) {
      const CholQr& c = cs[p];
      if (!c.q.rinv) continue;
      const int K = c.q.K, m = c.q.m;
      if (K <= kCholInPlaceK) {
        SsDesc d = ss_desc(c.q.A, c.q.a_r, c.q.a_c, c.q.rinv, K, 1, c.q.Q, c.q.q_r, c.q.q_c, m, K, K);
        d.jobs = c.q.nodes; d.x_job = c.q.a_node; d.s_job = (long long)K * K; d.c_job = c.q.q_node;
        d.s_tri = 2;
        d.active = need2 + p;
        sd.push_back(d);
      } else {
        GemmDesc d = gemm_desc(c.q.A, c.q.a_r, c.q.a_c, c.q.rinv, K, 1, c.Q1, K, 1, m, K, K);
        d.nb1 = c.q.nodes; d.a_b1 = c.q.a_node; d.b_b1 = (long long)K * K; d.c_b1 = (long long)m * K;
        d.active = need2 + p;
        g.push_back(d);
      }
    }
    HT_TRY(ss_gemm(sd, s, "ss_cholqr2_q", false));
    HT_TRY(gemm_grouped(g, s, "gemm_cholqr2_q", false));
    sd.clear();
    g.clear();
    for (size_t p = 0; p < cs.size(); ++p) {
      const CholQr& c = cs[p];
      if (c.q.K <= kCholInPlaceK) gram(g, r, c, c.q.Q, c.q.q_r, c.q.q_c, c.q.q_node, need2 + p);
      else gram(g, r, c, c.Q1, c.q.K, 1, (long long)c.q.m * c.q.K, need2 + p);
    }
    HT_TRY(gemm_grouped(g, s, "gemm_cholqr2_gram", false));
    HT_TRY(reduce_partials(r, s));
    for (size_t p = 0; p < cs.size(); ++p) {
      const CholQr& c = cs[p];
      CholDesc d{};
      d.W = c.W; d.Rf = c.R2; d.Ri = c.Ri;
      d.K = c.q.K; d.nodes = c.q.nodes;
      d.check_identity = 1;
      d.active = need2 + p;
      ch.push_back(d);
    }
    HT_TRY(launch_chol(ch, fail, s, "cholqr2_factor"));
    g.clear();
    std::vector<GemmDesc> rcopy;
    for (size_t p = 0; p < cs.size(); ++p) {
      const CholQr& c = cs[p];
      const int K = c.q.K, m = c.q.m;
      if (K <= kCholInPlaceK) {  // Q <- Q R2^{-1} in place (each CTA owns whole rows)
        SsDesc d = ss_desc(c.q.Q, c.q.q_r, c.q.q_c, c.Ri, K, 1, c.q.Q, c.q.q_r, c.q.q_c, m, K, K);
        d.jobs = c.q.nodes; d.x_job = c.q.q_node; d.s_job = (long long)K * K; d.c_job = c.q.q_node;
        d.s_tri = 2;
        d.active = need2 + p;
        sd.push_back(d);
      } else {
        GemmDesc d = gemm_desc(c.Q1, K, 1, c.Ri, K, 1, c.q.Q, c.q.q_r, c.q.q_c, m, K, K);
        d.nb1 = c.q.nodes; d.a_b1 = (long long)m * K; d.b_b1 = (long long)K * K;
        d.c_b1 = c.q.q_node;
        d.active = need2 + p;
        g.push_back(d);
      }
      GemmDesc cp = gemm_desc(nullptr, K, 1, c.q.R, c.q.r_ld, 1, c.R1, K, 1, K, K, K);  // R1 = copy of R
      cp.a_tri = 3;
      cp.nb1 = c.q.nodes; cp.b_b1 = c.q.r_node; cp.c_b1 = (long long)K * K;
      cp.active = need2 + p;
      rcopy.push_back(cp);
      GemmDesc e = gemm_desc(c.R2, K, 1, c.R1, K, 1, c.q.R, c.q.r_ld, 1, K, K, K);
      e.nb1 = c.q.nodes; e.a_b1 = (long long)K * K; e.b_b1 = (long long)K * K; e.c_b1 = c.q.r_node;
      e.active = need2 + p;
      g.push_back(e);
    }
    HT_TRY(gemm_grouped(rcopy, s, "gemm_cholqr2_q", false));  // before R is overwritten by R2 R1
    HT_TRY(ss_gemm(sd, s, "ss_cholqr2_q", false));
    HT_TRY(gemm_grouped(g, s, "gemm_cholqr2_q", false));
    // the Q of an implicit problem is explicit now: its R^{-1} stand-in becomes I
    for (size_t p = 0; p < cs.size(); ++p) {
      const CholQr& c = cs[p];
      if (c.q.rinv) HT_TRY(identity_batched(c.q.rinv, (long long)c.q.K * c.q.K, c.q.K, c.q.nodes, need2 + p, s));
    }
    return kOk;
  };
  if (g_own_capture && g_cond_nodes != 0) {
    const int rc = capture_if_any(s, need2, (int)cs.size(), nullptr, pass2);
    if (rc != kOk) g_cond_nodes = 0;  // the capture fails; later captures stay unconditional
    return rc;
  }
  return pass2(s);
}

// ---------------------------------------------------------------------------
// wide frames: block Gram-Schmidt (twice) over Cholesky-QR panels
// ---------------------------------------------------------------------------
namespace {
int split_for(long long tiles, long long reduction) {
  const long long T = std::max<long long>(1, tiles);
  const long long kt = std::max<long long>(1, (reduction + kGemmBK - 1) / kGemmBK);
  long long best_s = 1;
  double best = 1e300;
  for (long long S = 1; S <= std::min<long long>(160, std::max<long long>(1, kt / 4)); ++S) {
    const double cost = (double)((T * S + 147) / 148) * ((double)((kt + S - 1) / S) + 3.0) + 0.02 * S;
    if (cost < best - 1e-9) {
      best = cost;
      best_s = S;
    }
  }
  return (int)best_s;
}
}  // namespace

bool cholbig_eligible(const QrProblem& q) { return q.K > kCholInPlaceK && q.K <= 1024 && q.m >= q.K; }

long long cholbig_workspace_doubles(CholBig& c) {
  const int K = c.q.K;
  c.np = (K + kCholInPlaceK - 1) / kCholInPlaceK;
  c.pw = (K + c.np - 1) / c.np;
  c.pw += c.pw & 1;  // even panel width: every panel starts 16-byte aligned (c0 even)
  const long long n = c.q.nodes;
  const long long c0max = (long long)(c.np - 1) * c.pw;
  c.S = split_for((long long)gemm_tiles((int)c0max, c.pw) * n, c.q.m);
  c.panel = CholQr{};
  c.panel.q = c.q;
  c.panel.q.K = c.pw;
  c.panel.S = split_for((long long)gemm_tiles(c.pw, c.pw) * n, c.q.m);
  c.hpanel = c.q;
  c.hpanel.K = c.pw;
  c.hpanel.V = nullptr;
  c.hpanel.wide_ws = nullptr;
  qr_plan(c.hpanel);
  return (long long)c.S * n * c0max * c.pw + n * c0max * c.pw + n * (long long)c.pw * c.pw +
         std::max(cholqr_workspace_doubles(c.panel), qr_workspace_doubles(c.hpanel)) + 4 * 32;
}

void cholbig_bind(CholBig& c, double* ws) {
  if (g_sync_check && getenv("HT_SYNC_DUMP"))
    fprintf(stderr, "[cholbig] K=%d m=%d nodes=%d np=%d pw=%d S=%d ws=%p doubles=%lld\n", c.q.K, c.q.m, c.q.nodes,
            c.np, c.pw, c.S, (void*)ws, cholbig_workspace_doubles(c));
  const long long n = c.q.nodes;
  const long long c0max = (long long)(c.np - 1) * c.pw;
  auto al = [](double* p) { return (double*)(((uintptr_t)p + 255) & ~(uintptr_t)255); };
  double* p = al(ws);
  c.P = p;
  p = al(p + (long long)c.S * n * c0max * c.pw);
  c.Sb = p;
  p = al(p + n * c0max * c.pw);
  c.Rp = p;
  p = al(p + n * (long long)c.pw * c.pw);
  cholqr_bind(c.panel, p);  // the two panel plans share one workspace (used one at a time)
  c.hws = p;
}

int cholbig_run(std::vector<CholBig>& cs, int* fail, int* need2, bool two_pass, cudaStream_t s, bool householder) {
  for (auto& c : cs) {
    const QrProblem& q = c.q;
    const int m = q.m, K = q.K, n = q.nodes;
    // Q <- A (the sweep works in place in the output), R <- 0
    std::vector<Copy2dDesc> cp{Copy2dDesc{q.A, q.Q, q.a_r, q.a_c, q.a_node, q.q_r, q.q_c, q.q_node, m, K, n}};
    HT_TRY(copy2d_batched(cp, s));
    for (int nd = 0; nd < n; ++nd)
      HT_CUDA_CHECK(cudaMemset2DAsync(q.R + nd * q.r_node, sizeof(double) * q.r_ld, 0, sizeof(double) * K, K, s));
    for (int j = 0; j < c.np; ++j) {
      const int c0 = j * c.pw, w = std::min(c.pw, K - c0);
      if (w <= 0) break;
      double* QJ = q.Q + (long long)c0 * q.q_c;
      double* RJ = q.R + c0;  // rows 0..c0-1 of the column block J
      for (int pass = 0; j > 0 && pass < 2; ++pass) {
        // P = Q_<^T Q_J (split-K partials [S][node][c0][w])
        GemmDesc g = gemm_desc(q.Q, q.q_c, q.q_r, QJ, q.q_r, q.q_c, c.P, w, 1, c0, w, m);
        g.nb1 = n; g.a_b1 = q.q_node; g.b_b1 = q.q_node; g.c_b1 = (long long)c0 * w;
        g.splits = c.S;
        std::vector<GemmDesc> gv{g};
        HT_TRY(gemm_grouped(gv, s, "gemm_bgs_proj"));
        // pass 0: R_<J = P;  pass 1: Sb = P, R_<J += P
        std::vector<ReduceDesc> rd;
        if (pass == 0) {
          rd.push_back(ReduceDesc{c.P, RJ, q.r_ld, 1, q.r_node, 0, c.S, c0, w, n, 1, 0, 1.0, 0.0});
        } else {
          rd.push_back(ReduceDesc{c.P, c.Sb, w, 1, (long long)c0 * w, 0, c.S, c0, w, n, 1, 0, 1.0, 0.0});
          rd.push_back(ReduceDesc{c.P, RJ, q.r_ld, 1, q.r_node, 0, c.S, c0, w, n, 1, 0, 1.0, 1.0});
        }
        HT_TRY(reduce_partials(rd, s));
        // Q_J -= Q_< S
        GemmDesc u = pass == 0 ? gemm_desc(q.Q, q.q_r, q.q_c, RJ, q.r_ld, 1, QJ, q.q_r, q.q_c, m, w, c0, -1.0, 1.0)
                               : gemm_desc(q.Q, q.q_r, q.q_c, c.Sb, w, 1, QJ, q.q_r, q.q_c, m, w, c0, -1.0, 1.0);
        u.nb1 = n; u.a_b1 = q.q_node; u.b_b1 = pass == 0 ? q.r_node : (long long)c0 * w; u.c_b1 = q.q_node;
        std::vector<GemmDesc> uv{u};
        HT_TRY(gemm_grouped(uv, s, "gemm_bgs_update"));
      }
      if (!householder) {
        // [Q_J, R_JJ] = CholQR(Q_J), in place
        CholQr pc = c.panel;
        pc.q.A = QJ; pc.q.a_r = q.q_r; pc.q.a_c = q.q_c; pc.q.a_node = q.q_node;
        pc.q.Q = QJ;
        pc.q.R = q.R + (long long)c0 * q.r_ld + c0;
        pc.q.K = w;
        std::vector<CholQr> pv{pc};
        HT_TRY(cholqr_run(pv, fail, need2, two_pass, s));
        continue;
      }
      // [Q_J, R_JJ] = TSQR(Q_J) in place (Householder: rank-deficient panels stay orthonormal)
      QrProblem hp = c.hpanel;
      hp.A = QJ; hp.a_r = q.q_r; hp.a_c = q.q_c; hp.a_node = q.q_node;
      hp.Q = QJ; hp.q_r = q.q_r; hp.q_c = q.q_c; hp.q_node = q.q_node;
      hp.R = q.R + (long long)c0 * q.r_ld + c0; hp.r_ld = q.r_ld; hp.r_node = q.r_node;
      hp.K = w;
      hp.V = nullptr;
      HT_TRY(qr_plan(hp));
      qr_bind_workspace(hp, c.hws);  // w <= pw: fits the workspace planned for pw
      std::vector<QrProblem> hv{hp};
      HT_TRY(qr_batched(hv, s));
      if (j == 0) continue;
      // completion directions of a deficient panel: project once more and re-factor,
      // R_<J += S R_JJ and R_JJ <- R' R_JJ
      GemmDesc g = gemm_desc(q.Q, q.q_c, q.q_r, QJ, q.q_r, q.q_c, c.P, w, 1, c0, w, m);
      g.nb1 = n; g.a_b1 = q.q_node; g.b_b1 = q.q_node; g.c_b1 = (long long)c0 * w;
      g.splits = c.S;
      std::vector<GemmDesc> gv{g};
      HT_TRY(gemm_grouped(gv, s, "gemm_bgs_proj"));
      std::vector<ReduceDesc> rd{ReduceDesc{c.P, c.Sb, w, 1, (long long)c0 * w, 0, c.S, c0, w, n, 1, 0, 1.0, 0.0}};
      HT_TRY(reduce_partials(rd, s));
      GemmDesc u = gemm_desc(q.Q, q.q_r, q.q_c, c.Sb, w, 1, QJ, q.q_r, q.q_c, m, w, c0, -1.0, 1.0);
      u.nb1 = n; u.a_b1 = q.q_node; u.b_b1 = (long long)c0 * w; u.c_b1 = q.q_node;
      // R_<J += S R_JJ  (R_JJ upper triangular, row-major at (c0, c0))
      const double* RJJ = q.R + (long long)c0 * q.r_ld + c0;
      GemmDesc ra = gemm_desc(c.Sb, w, 1, RJJ, q.r_ld, 1, RJ, q.r_ld, 1, c0, w, w, 1.0, 1.0);
      ra.nb1 = n; ra.a_b1 = (long long)c0 * w; ra.b_b1 = q.r_node; ra.c_b1 = q.r_node;
      std::vector<GemmDesc> uv{u, ra};
      HT_TRY(gemm_grouped(uv, s, "gemm_bgs_update"));
      // R' from the re-factorisation into scratch, then R_JJ <- R' R_JJ
      hp.R = c.Rp; hp.r_ld = w; hp.r_node = (long long)w * w;
      std::vector<QrProblem> hv2{hp};
      HT_TRY(qr_batched(hv2, s));
      std::vector<Copy2dDesc> cr{Copy2dDesc{RJJ, c.Sb, q.r_ld, 1, q.r_node, w, 1, (long long)w * w, w, w, n}};
      HT_TRY(copy2d_batched(cr, s));
      GemmDesc rr = gemm_desc(c.Rp, w, 1, c.Sb, w, 1, q.R + (long long)c0 * q.r_ld + c0, q.r_ld, 1, w, w, w);
      rr.nb1 = n; rr.a_b1 = (long long)w * w; rr.b_b1 = (long long)w * w; rr.c_b1 = q.r_node;
      std::vector<GemmDesc> rv{rr};
      HT_TRY(gemm_grouped(rv, s, "gemm_bgs_update"));
    }
  }
  return kOk;
}

}  // namespace ht
