#include <cstdio>
#include <cstdlib>
// Blocked tree-TSQR Householder QR with DMMA trailing updates (see qr.cuh).
//
// Reference semantics: kernels.py:24-32 -- dlarfg reflectors as in LAPACK dgeqrf,
// explicit thin Q (dorgqr), sign fix diag(R) >= 0; wide input (m < K) gives
// Q m x m and R m x K (kernels.py:27-28).
//
// One CTA owns one "step": either a dense row block (<= 128 rows, dgeqrf on the
// block) or a tree pair [R_a; R_b] (reflector heads in R_a's rows, tails in R_b).
// The step's K columns are processed in panels of 8: warp 0 factors the panel
// in registers (warp-synchronous dlarfg + dots, no CTA barrier per reflector),
// builds the panel's compact-WY T (8 x 8), and all 16 warps apply
// (I - V T V^T)^T to the trailing columns with mma.sync DMMA tiles on shared
// memory.  Q is formed the same way in reverse (I - V T V^T per panel, last
// panel first) by the apply kernel.
#include <algorithm>

#include "prof.cuh"
#include "qr.cuh"

namespace ht {

namespace {

constexpr int QT = 512;         // threads per CTA (apply kernel)
constexpr int QTF = 256;        // threads per CTA (factor kernel: the panel warp needs registers)
constexpr int NB = 8;           // panel width
constexpr int LR = 4;           // rows per lane in the panel warp -> 128 rows
constexpr int BR = kWarp * LR;  // 128 block rows
constexpr int MAXD = 32;
constexpr int SMEM_LIMIT = 227 * 1024;

__host__ __device__ __forceinline__ int pitch_rows(int rows) { return ((rows + 15) & ~15) + 4; }
__host__ __device__ __forceinline__ int npanels(int K) { return (K + NB - 1) / NB; }

struct QrDev {
  const double* A;
  long long a_r, a_c, a_node;
  double* Q;
  long long q_r, q_c, q_node;
  double* R;
  long long r_ld, r_node;
  double* V;
  double* Rst;
  double* Tp;
  double* tau;
  long long v_node, st_node, tp_node, tau_node;
  int m, K, P, rpc;
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

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0));
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Transposed 8-way warp reduction: lane L ends with the total of slot (L >> 2) & 7.
__device__ __forceinline__ double reduce8(const double (&x)[8], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  const unsigned F = 0xffffffffu;
  const double y0 = (b4 ? x[4] : x[0]) + __shfl_xor_sync(F, b4 ? x[0] : x[4], 16);
  const double y1 = (b4 ? x[5] : x[1]) + __shfl_xor_sync(F, b4 ? x[1] : x[5], 16);
  const double y2 = (b4 ? x[6] : x[2]) + __shfl_xor_sync(F, b4 ? x[2] : x[6], 16);
  const double y3 = (b4 ? x[7] : x[3]) + __shfl_xor_sync(F, b4 ? x[3] : x[7], 16);
  const double z0 = (b3 ? y2 : y0) + __shfl_xor_sync(F, b3 ? y0 : y2, 8);
  const double z1 = (b3 ? y3 : y1) + __shfl_xor_sync(F, b3 ? y1 : y3, 8);
  double u = (b2 ? z1 : z0) + __shfl_xor_sync(F, b2 ? z0 : z1, 4);
  u += __shfl_xor_sync(F, u, 2);
  u += __shfl_xor_sync(F, u, 1);
  return u;
}

// C(M x N) = Cinit + sum_k A(m,k) B(k,n) on 8x8 DMMA tiles spread over the CTA's warps.
// ga/gb return operands (0 outside), lc the initial C value, sc stores a result.
template <typename GA, typename GB, typename LC, typename SC>
__device__ __forceinline__ void cta_dmma(int M, int N, int K, GA ga, GB gb, LC lc, SC sc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int tm = (M + 7) >> 3, tn = (N + 7) >> 3;
  const int r = lane >> 2, q = lane & 3;
  for (int tile = warp; tile < tm * tn; tile += nw) {
    const int m0 = (tile / tn) << 3, n0 = (tile % tn) << 3;
    double c0[2], c1[2];
    c0[0] = lc(m0 + r, n0 + 2 * q);
    c0[1] = lc(m0 + r, n0 + 2 * q + 1);
    c1[0] = 0.0;
    c1[1] = 0.0;
    int k = 0;
    for (; k + 8 <= K; k += 8) {
      dmma_8x8x4(c0, ga(m0 + r, k + q), gb(k + q, n0 + r));
      dmma_8x8x4(c1, ga(m0 + r, k + 4 + q), gb(k + 4 + q, n0 + r));
    }
    for (; k < K; k += 4) dmma_8x8x4(c0, ga(m0 + r, k + q), gb(k + q, n0 + r));
    sc(m0 + r, n0 + 2 * q, c0[0] + c1[0]);
    sc(m0 + r, n0 + 2 * q + 1, c0[1] + c1[1]);
  }
}

// ---------------------------------------------------------------------------
// panel factorisation by warp 0 (columns j0 .. j0+nbp-1 of the step)
//  DENSE: head S[j][j], tail rows j+1..nrows-1;  TRI: head R[j][j], tail rows 0..nrows-1.
// Writes the reflectors back into S, tau into taus[j], R heads (TRI), and T_p (8x8) into Tp.
// ---------------------------------------------------------------------------
// One reflector JJ (compile-time) of the panel factorisation.  Panel rows are held
// shifted: lane l, slot t holds panel row r' = l + 32 t, i.e. block row j0 + r' (DENSE)
// or block row r' (TRI), so the head row of reflector JJ (DENSE) is lane JJ, slot 0.
// The tail norm is reduced together with the 7 dot products (one 8-way reduction).
template <bool DENSE, int JJ>
__device__ __forceinline__ void panel_reflector(double (&pv)[NB][LR], double (&trow)[NB], int nr, int j0, int nbp,
                                                double* R, int rp, double* taus) {
  const int lane = threadIdx.x & 31;
  if (JJ < nbp) {
    const int j = j0 + JJ;
    // u = tail of column JJ (rows after the head)
    double u[LR];
#pragma unroll
    for (int t = 0; t < LR; ++t) {
      const int rr = lane + t * kWarp;
      u[t] = (rr < nr && (!DENSE || rr > JJ)) ? pv[JJ][t] : 0.0;
    }
    double x[8];
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      x[c] = 0.0;
      if (c < nbp) {
#pragma unroll
        for (int t = 0; t < LR; ++t) x[c] = fma(u[t], pv[c][t], x[c]);
      }
    }
    const double tot = reduce8(x, lane);
    double dsum[NB], head[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      dsum[c] = __shfl_sync(0xffffffffu, tot, 4 * c);
      head[c] = DENSE ? __shfl_sync(0xffffffffu, pv[c][0], JJ) : ((c < nbp && c >= JJ) ? R[j * rp + j0 + c] : 0.0);
    }
    const double ss = dsum[JJ];
    const double alpha = head[JJ];
    double beta = alpha, tau = 0.0, scal = 0.0;
    if (ss > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
      const double r1 = 1.0 / beta, r2 = 1.0 / (alpha - beta);
      tau = (beta - alpha) * r1;
      scal = r2;
    }
    double wc[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) wc[c] = (c == JJ) ? 0.0 : fma(scal, dsum[c], (DENSE || c > JJ) ? head[c] : 0.0);
    // update the trailing panel columns; store v_JJ (head beta, tail scaled)
#pragma unroll
    for (int t = 0; t < LR; ++t) {
      const int rr = lane + t * kWarp;
      const double v = (DENSE && t == 0 && lane == JJ) ? 1.0 : u[t] * scal;
#pragma unroll
      for (int c = JJ + 1; c < NB; ++c)
        if (c < nbp) pv[c][t] = fma(-tau * wc[c], v, pv[c][t]);
      if (DENSE && t == 0 && lane == JJ) pv[JJ][0] = beta;
      else if (rr < nr && (!DENSE || rr > JJ)) pv[JJ][t] = u[t] * scal;
    }
    if (!DENSE && lane == 0) {
#pragma unroll
      for (int c = JJ + 1; c < NB; ++c)
        if (c < nbp) R[j * rp + j0 + c] = head[c] - tau * wc[c];
      R[j * rp + j] = beta;
    }
    if (lane == 0) taus[j] = tau;
    // T column JJ (dlarft), kept in registers: lane r < 8 holds T row r.
    //   T[r][JJ] = -tau_JJ sum_{l=r}^{JJ-1} T[r][l] G[l][JJ],  G[l][JJ] = v_l^T v_JJ = wc[l]
    double acc = 0.0;
#pragma unroll
    for (int l = 0; l < JJ; ++l)
      if (l >= lane) acc = fma(trow[l], wc[l], acc);
    trow[JJ] = (lane == JJ) ? tau : (lane < JJ ? -tau * acc : 0.0);
  }
  if constexpr (JJ + 1 < NB) panel_reflector<DENSE, JJ + 1>(pv, trow, nr, j0, nbp, R, rp, taus);
}

// ---------------------------------------------------------------------------
// panel factorisation by warp 0 (columns j0 .. j0+nbp-1 of the step)
//  DENSE: head S[j][j], tail rows j+1..nrows-1;  TRI: head R[j][j], tail rows 0..nrows-1.
// Writes the reflectors back into S, tau into taus[j], R heads (TRI), and T_p (8x8) into Tp.
// ---------------------------------------------------------------------------
template <bool DENSE>
__device__ void panel_factor(double* S, int ps, int nrows, int j0, int nbp, double* R, int rp, double* taus,
                             double* Gs, double* Tp) {
  (void)Gs;
  const int lane = threadIdx.x & 31;
  const int off = DENSE ? j0 : 0;   // panel row r' = block row - off
  const int nr = nrows - off;
  double pv[NB][LR];
  double trow[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    trow[c] = 0.0;
#pragma unroll
    for (int t = 0; t < LR; ++t) {
      const int rr = lane + t * kWarp;
      pv[c][t] = (c < nbp && rr < nr) ? S[(j0 + c) * ps + off + rr] : 0.0;
    }
  }
  panel_reflector<DENSE, 0>(pv, trow, nr, j0, nbp, R, rp, taus);
#pragma unroll
  for (int c = 0; c < NB; ++c)
#pragma unroll
    for (int t = 0; t < LR; ++t) {
      const int rr = lane + t * kWarp;
      if (c < nbp && rr < nr) S[(j0 + c) * ps + off + rr] = pv[c][t];
    }
  if (lane < NB) {
#pragma unroll
    for (int c = 0; c < NB; ++c) Tp[lane * NB + c] = (lane < nbp && c < nbp) ? trow[c] : 0.0;
  }
  __syncwarp();
}

// Masked copy of panel V (columns j0..j0+nbp-1) into Vp[r][row] (zero rows beyond nrows,
// unit diagonal and zeros above it in the DENSE case).
template <bool DENSE>
__device__ __forceinline__ void stage_panel_v(const double* S, int ps, int nrows, int j0, int nbp, double* Vp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = warp; r < NB; r += nw)
    for (int row = lane; row < ps; row += kWarp) {
      double v = 0.0;
      if (r < nbp && row < nrows) {
        const int col = j0 + r;
        if (!DENSE || row > col) v = S[col * ps + row];
        else if (row == col) v = 1.0;
      }
      Vp[r * ps + row] = v;
    }
}

// W (8 x nt) = [R head rows] + Vp^T C,  C = S[:, c0:c0+nt]  (all operands zero padded)
__device__ __forceinline__ void dmma_vt_c(const double* Vp, int pv, const double* C, int pc, int krows, int nt,
                                          double* W, int pw, const double* Rh, int rp, int nbp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  const int ntt = (nt + 7) >> 3;
  for (int tile = warp; tile < ntt; tile += nw) {
    const int n0 = tile << 3;
    double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
    if (Rh) {
      if (r < nbp && n0 + 2 * q < nt) c0[0] = Rh[r * rp + n0 + 2 * q];
      if (r < nbp && n0 + 2 * q + 1 < nt) c0[1] = Rh[r * rp + n0 + 2 * q + 1];
    }
    const double* a = Vp + r * pv + q;
    const double* b = C + (n0 + r) * pc + q;
    int k = 0;
    for (; k + 8 <= krows; k += 8) {
      dmma_8x8x4(c0, a[k], b[k]);
      dmma_8x8x4(c1, a[k + 4], b[k + 4]);
    }
    for (; k < krows; k += 4) dmma_8x8x4(c0, a[k], b[k]);
    W[r * pw + n0 + 2 * q] = c0[0] + c1[0];
    W[r * pw + n0 + 2 * q + 1] = c0[1] + c1[1];
  }
}

// C[:, 0:nt] (rows krows) += Vp * Wn   (Wn = -T-scaled W, 8 x nt, zero padded)
__device__ __forceinline__ void dmma_c_plus_v_w(const double* Vp, int pv, const double* Wn, int pw, double* C, int pc,
                                                int krows, int nt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  const int mt = (krows + 7) >> 3, ntt = (nt + 7) >> 3;
  for (int tile = warp; tile < mt * ntt; tile += nw) {
    const int m0 = (tile / ntt) << 3, n0 = (tile % ntt) << 3;
    double acc[2];
    double* c = C + (n0 + 2 * q) * pc + m0 + r;
    acc[0] = c[0];
    acc[1] = c[pc];
    // A(m = row, k = reflector) = Vp[k][row]; B(k, n) = Wn[k][n]
    dmma_8x8x4(acc, Vp[q * pv + m0 + r], Wn[q * pw + n0 + r]);
    dmma_8x8x4(acc, Vp[(q + 4) * pv + m0 + r], Wn[(q + 4) * pw + n0 + r]);
    c[0] = acc[0];
    c[pc] = acc[1];
  }
}

// Apply (I - V T V^T)^T of panel [j0, j0+nbp) to the trailing columns [j0+nbp, K).
template <bool DENSE>
__device__ void trailing_update(double* S, int ps, int nrows, int K, int j0, int nbp, double* R, int rp,
                                const double* Tp, double* W, double* W2, int pw, double* Vp) {
  const int c0 = j0 + nbp;
  const int nt = K - c0;
  if (nt <= 0) return;
  const int krows = (nrows + 3) & ~3;
  dmma_vt_c(Vp, ps, S + c0 * ps, ps, krows, nt, W, pw, DENSE ? nullptr : R + j0 * rp + c0, rp, nbp);
  __syncthreads();
  // W2 = -(T^T W)  (T upper triangular: (T^T W)[r][c] = sum_{l<=r} T[l][r] W[l][c]); TRI: R heads -= T^T W
  const int ntp = (nt + 7) & ~7;
  for (int e = threadIdx.x; e < NB * ntp; e += blockDim.x) {
    const int r = e & (NB - 1), c = e >> 3;
    double acc = 0.0;
    if (r < nbp && c < nt) {
      for (int l = 0; l <= r; ++l) acc = fma(Tp[l * NB + r], W[l * pw + c], acc);
      if (!DENSE) R[(j0 + r) * rp + c0 + c] -= acc;
    }
    W2[r * pw + c] = -acc;
  }
  __syncthreads();
  dmma_c_plus_v_w(Vp, ps, W2, pw, S + c0 * ps, ps, krows, nt);
  __syncthreads();
}

template <bool DENSE>
__device__ void factor_step(double* S, int ps, int nrows, int K, int nrefl, double* R, int rp, double* taus,
                            double* W, double* W2, int pw, double* Gs, double* Tp, double* Tp_out, double* Vp) {
  for (int j0 = 0; j0 < nrefl; j0 += NB) {
    const int nbp = min(NB, nrefl - j0);
    // TRI: R_b stays upper triangular, so panel p only touches its rows < j0 + nbp
    const int prow = DENSE ? nrows : min(nrows, j0 + nbp);
    if (threadIdx.x < kWarp) panel_factor<DENSE>(S, ps, prow, j0, nbp, R, rp, taus, Gs, Tp);
    __syncthreads();
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) Tp_out[(j0 / NB) * NB * NB + e] = Tp[e];
    stage_panel_v<DENSE>(S, ps, prow, j0, nbp, Vp);
    __syncthreads();
    trailing_update<DENSE>(S, ps, prow, K, j0, nbp, R, rp, Tp, W, W2, pw, Vp);
  }
}

struct FactorSmem {
  double *S, *R, *W, *W2, *Gs, *Tp, *taus, *Vp;
  int ps, rp, pw;
};

__host__ __device__ __forceinline__ int pad8(int v) { return (v + 7) & ~7; }

__host__ __device__ inline size_t factor_smem_doubles(int K, bool dense, int rows) {
  const int ps = pitch_rows(dense ? rows : K);
  const int pw = pitch_rows(pad8(K));
  return (size_t)(pad8(K) + (dense ? 8 : 0)) * ps + (dense ? 0 : (size_t)K * (K + 1)) + 2 * NB * pw + 2 * NB * NB + K + 8 +
         (size_t)NB * ps;
}

__device__ FactorSmem carve_factor(double* sm, int K, bool dense, int rows) {
  FactorSmem f;
  f.ps = pitch_rows(dense ? rows : K);
  f.rp = K + 1;
  f.pw = pitch_rows(pad8(K));
  f.S = sm;
  double* p = sm + (size_t)(pad8(K) + (dense ? 8 : 0)) * f.ps;
  f.R = p;
  if (!dense) p += (size_t)K * f.rp;
  f.W = p;
  p += NB * f.pw;
  f.W2 = p;
  p += NB * f.pw;
  f.Gs = p;
  p += NB * NB;
  f.Tp = p;
  p += NB * NB;
  f.taus = p;
  p += K + 8;
  f.Vp = p;
  return f;
}

// round < 0: dense blocks; round >= 0: combine round
__global__ void __launch_bounds__(QTF, 1) qr_factor_kernel(const __grid_constant__ QrBatch b) {
  extern __shared__ double sm[];
  const QrDev& q = b.d[find_desc(b)];
  const int local = blockIdx.x - q.begin;
  const int nd = local / q.per_node, k = local % q.per_node;
  const int K = q.K;
  const int np = npanels(K);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double* Rst = q.Rst + nd * q.st_node;
  double* Tpg = q.Tp + nd * q.tp_node;
  double* taug = q.tau + nd * q.tau_node;

  if (b.round < 0) {
    const int c = k;
    const int row0 = c * q.rpc;
    const int rows = min(q.rpc, q.m - row0);
    const int nrefl = min(rows, K);
    FactorSmem f = carve_factor(sm, K, true, BR);
    const double* A = q.A + nd * q.a_node;
    // column-major smem block; global loads coalesced along rows for column-major A
    for (int col = warp; col < pad8(K) + 8; col += nwarps)
      for (int row = lane; row < f.ps; row += kWarp) {
        const bool ok = row < rows && col < K;
        cp_async8(f.S + col * f.ps + row, ok ? A + (long long)(row0 + row) * q.a_r + (long long)col * q.a_c : A, ok);
      }
    cp_async_wait_all();
    __syncthreads();
    factor_step<true>(f.S, f.ps, rows, K, nrefl, f.R, f.rp, f.taus, f.W, f.W2, f.pw, f.Gs, f.Tp,
                      Tpg + (long long)c * np * NB * NB, f.Vp);
    double* V = q.V + nd * q.v_node;
    double* Rc = Rst + (long long)c * K * K;
    for (int col = warp; col < K; col += nwarps)
      for (int row = lane; row < BR; row += kWarp) {
        const double v = f.S[col * f.ps + row];
        if (row < rows) V[(long long)col * q.m + row0 + row] = v;
        if (row < K) Rc[(long long)row * K + col] = (row < nrefl && col >= row) ? v : 0.0;
      }
    for (int j = threadIdx.x; j < K; j += blockDim.x) taug[(long long)c * K + j] = j < nrefl ? f.taus[j] : 0.0;
  } else {
    const int r = b.round;
    const int ia = k << (r + 1), ib = ia + (1 << r);
    FactorSmem f = carve_factor(sm, K, false, K);
    double* Ra = Rst + (long long)ia * K * K;
    double* Rb = Rst + (long long)ib * K * K;
    for (int i = warp; i < K; i += nwarps)
      for (int col = lane; col < K; col += kWarp) f.R[i * f.rp + col] = Ra[i * K + col];
    for (int col = warp; col < pad8(K); col += nwarps)
      for (int i = lane; i < f.ps; i += kWarp)
        f.S[col * f.ps + i] = (i < K && col < K) ? Rb[(long long)i * K + col] : 0.0;
    __syncthreads();
    factor_step<false>(f.S, f.ps, K, K, K, f.R, f.rp, f.taus, f.W, f.W2, f.pw, f.Gs, f.Tp,
                       Tpg + (long long)(q.P + ib) * np * NB * NB, f.Vp);
    for (int i = warp; i < K; i += nwarps)
      for (int col = lane; col < K; col += kWarp) Ra[i * K + col] = f.R[i * f.rp + col];
    for (int col = warp; col < K; col += nwarps)
      for (int i = lane; i < K; i += kWarp) Rb[(long long)col * K + i] = f.S[col * f.ps + i];  // tails
    for (int j = threadIdx.x; j < K; j += blockDim.x) taug[(long long)(q.P + ib) * K + j] = f.taus[j];
  }
}

// ---------------------------------------------------------------------------
// Q formation: apply the step's panels in reverse (H_p = I - V_p T_p V_p^T, last panel
// first) to [W; 0] (dense block) or to [H; Z] (tree pair: heads H = W_a, tails Z = 0).
// ---------------------------------------------------------------------------
__host__ __device__ inline size_t apply_smem_doubles(int K, bool dense) {
  const int pw = pitch_rows(pad8(K));
  if (dense) {
    const int pc = pitch_rows(BR);
    return (size_t)(pad8(K) + 8) * pc + (size_t)NB * pc + 2 * NB * pw + NB * NB + 8;
  }
  const int pz = pitch_rows(K);
  return (size_t)K * pw + (size_t)pad8(K) * pz + (size_t)NB * pz + 2 * NB * pw + NB * NB + 8;
}

// W2 = -(T W) for upper-triangular T (8 x 8), W (8 x ncols); TRI: heads H += W2
__device__ __forceinline__ void apply_t(const double* Ts, const double* W, double* W2, int pw, int nbp, int ncols,
                                        double* Hh, int ph) {
  const int ntp = (ncols + 7) & ~7;
  for (int e = threadIdx.x; e < NB * ntp; e += blockDim.x) {
    const int r = e & (NB - 1), c = e >> 3;
    double acc = 0.0;
    if (r < nbp && c < ncols) {
      for (int l = r; l < nbp; ++l) acc = fma(Ts[r * NB + l], W[l * pw + c], acc);
      if (Hh) Hh[r * ph + c] -= acc;
    }
    W2[r * pw + c] = -acc;
  }
}

template <bool DENSE>
__device__ void apply_step(double* C, int pc, double* H, int ph, int nrows, int kq, int nrefl, const double* Vg,
                           long long v_ld, const double* Tpg, double* Vs, double* W, double* W2, int pw, double* Ts) {
  for (int p = npanels(nrefl) - 1; p >= 0; --p) {
    const int j0 = p * NB, nbp = min(NB, nrefl - j0);
    const int prow = DENSE ? nrows : min(nrows, j0 + nbp);  // TRI: tails only in rows < j0 + nbp
    {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (int r = warp; r < NB; r += nw)
        for (int row = lane; row < pc; row += kWarp) {
          double v = 0.0;
          if (r < nbp && row < prow) {
            const int col = j0 + r;
            if (!DENSE || row > col) v = Vg[(long long)col * v_ld + row];
            else if (row == col) v = 1.0;
          }
          Vs[r * pc + row] = v;
        }
    }
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) Ts[e] = Tpg[p * NB * NB + e];
    __syncthreads();
    const int krows = (prow + 3) & ~3;
    dmma_vt_c(Vs, pc, C, pc, krows, kq, W, pw, DENSE ? nullptr : H + j0 * ph, ph, nbp);
    __syncthreads();
    apply_t(Ts, W, W2, pw, nbp, kq, DENSE ? nullptr : H + j0 * ph, ph);
    __syncthreads();
    dmma_c_plus_v_w(Vs, pc, W2, pw, C, pc, krows, kq);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(QT, 1) qr_apply_kernel(const __grid_constant__ QrBatch b) {
  extern __shared__ double sm[];
  const QrDev& q = b.d[find_desc(b)];
  const int local = blockIdx.x - q.begin;
  const int nd = local / q.per_node, k = local % q.per_node;
  const int K = q.K, kq = min(q.m, K);
  const int np = npanels(K);
  const int pw = pitch_rows(pad8(K));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double* Q = q.Q + nd * q.q_node;
  const double* Tpg = q.Tp + nd * q.tp_node;
  if (b.round < 0) {
    const int c = k;
    const int row0 = c * q.rpc;
    const int rows = min(q.rpc, q.m - row0);
    const int nrefl = min(rows, K), kr = nrefl;
    const int pc = pitch_rows(BR);
    double* C = sm;
    double* Vs = C + (size_t)(pad8(K) + 8) * pc;
    double* W = Vs + NB * pc;
    double* W2 = W + NB * pw;
    double* Ts = W2 + NB * pw;
    for (int col = warp; col < pad8(K) + 8; col += nwarps)
      for (int row = lane; row < pc; row += kWarp) {
        const bool ok = row < kr && col < kq;
        cp_async8(C + col * pc + row, ok ? Q + (long long)(row0 + row) * q.q_r + (long long)col * q.q_c : Q, ok);
      }
    cp_async_wait_all();
    __syncthreads();
    apply_step<true>(C, pc, nullptr, 0, rows, kq, nrefl, q.V + nd * q.v_node + row0, q.m,
                     Tpg + (long long)c * np * NB * NB, Vs, W, W2, pw, Ts);
    for (int col = warp; col < kq; col += nwarps)
      for (int row = lane; row < rows; row += kWarp)
        Q[(long long)(row0 + row) * q.q_r + (long long)col * q.q_c] = C[col * pc + row];
  } else {
    const int r = b.round;
    const int ia = k << (r + 1), ib = ia + (1 << r);
    const int rows_b = min(q.rpc, q.m - ib * q.rpc);
    const int krb = min(rows_b, K);
    const int pz = pitch_rows(K), ph = pw;
    double* H = sm;                             // heads, row-major K x ph
    double* Z = H + (size_t)K * ph;             // tails, column-major pad8(kq) x pz
    double* Vs = Z + (size_t)pad8(K) * pz;
    double* W = Vs + NB * pz;
    double* W2 = W + NB * pw;
    double* Ts = W2 + NB * pw;
    const long long ra = (long long)ia * q.rpc, rb = (long long)ib * q.rpc;
    for (int row = warp; row < K; row += nwarps)
      for (int col = lane; col < ph; col += kWarp) {
        const bool ok = col < kq;
        cp_async8(H + row * ph + col, ok ? Q + (ra + row) * q.q_r + (long long)col * q.q_c : Q, ok);
      }
    for (int e = threadIdx.x; e < pad8(K) * pz; e += blockDim.x) Z[e] = 0.0;
    cp_async_wait_all();
    __syncthreads();
    apply_step<false>(Z, pz, H, ph, K, kq, K, q.Rst + nd * q.st_node + (long long)ib * K * K, K,
                      Tpg + (long long)(q.P + ib) * np * NB * NB, Vs, W, W2, pw, Ts);
    for (int row = warp; row < K; row += nwarps)
      for (int col = lane; col < kq; col += kWarp) Q[(ra + row) * q.q_r + (long long)col * q.q_c] = H[row * ph + col];
    for (int col = warp; col < kq; col += nwarps)
      for (int row = lane; row < krb; row += kWarp) Q[(rb + row) * q.q_r + (long long)col * q.q_c] = Z[col * pz + row];
  }
}

// sign fix (kernels.py:31-32): R out, and the seed diag(s) in Q's top rows
__global__ void qr_finalize_kernel(const __grid_constant__ QrBatch b) {
  const QrDev& q = b.d[find_desc(b)];
  const int nd = blockIdx.x - q.begin;
  const int K = q.K, kq = min(q.m, K);
  const double* Rf = q.Rst + nd * q.st_node;
  double* Ro = q.R + nd * q.r_node;
  double* Q = q.Q + nd * q.q_node;
  for (int e = threadIdx.x; e < kq * K; e += blockDim.x) {
    const int j = e / K, c = e - j * K;
    const double sg = Rf[j * K + j] < 0.0 ? -1.0 : 1.0;
    Ro[(long long)j * q.r_ld + c] = sg * Rf[j * K + c];
  }
  for (int e = threadIdx.x; e < kq * kq; e += blockDim.x) {
    const int i = e / kq, c = e - i * kq;
    Q[(long long)i * q.q_r + (long long)c * q.q_c] = (i == c) ? (Rf[c * K + c] < 0.0 ? -1.0 : 1.0) : 0.0;
  }
}

int pairs_host(int P, int r) {
  const int h = 1 << r;
  return P > h ? (P - h - 1) / (2 * h) + 1 : 0;
}

bool g_attr_done = false;

QrDev to_dev(const QrProblem& p) {
  QrDev d{};
  d.A = p.A; d.a_r = p.a_r; d.a_c = p.a_c; d.a_node = p.a_node;
  d.Q = p.Q; d.q_r = p.q_r; d.q_c = p.q_c; d.q_node = p.q_node;
  d.R = p.R; d.r_ld = p.r_ld; d.r_node = p.r_node;
  d.V = p.V; d.Rst = p.Rst; d.Tp = p.Tst; d.tau = p.X;
  d.v_node = p.v_node; d.st_node = p.st_node; d.tp_node = p.t_node; d.tau_node = p.x_node;
  d.m = p.m; d.K = p.K; d.P = p.P; d.rpc = p.rpc;
  d.nodes = p.nodes;
  return d;
}

double qr_flops(int m, int K) {
  const double a = std::max(m, K), b = std::min(m, K);
  return 2.0 * a * b * b - 2.0 / 3.0 * b * b * b;
}

enum Kind { kFactor, kApply, kFinalize };

int launch(std::vector<QrProblem>& probs, Kind kind, int round, cudaStream_t stream) {
  size_t i = 0;
  while (i < probs.size()) {
    QrBatch b;
    b.count = 0;
    b.round = round;
    int blocks = 0;
    size_t smem = 0;
    double flops = 0;
    while (i < probs.size() && b.count < MAXD) {
      const QrProblem& p = probs[i++];
      int per;
      if (kind == kFinalize) per = 1;
      else if (round < 0) per = p.P;
      else per = pairs_host(p.P, round);
      if (per == 0 || p.nodes == 0) continue;
      QrDev d = to_dev(p);
      d.begin = blocks;
      d.per_node = per;
      blocks += per * p.nodes;
      const bool dense = round < 0;
      smem = std::max(smem, sizeof(double) * (kind == kFactor ? factor_smem_doubles(p.K, dense, BR)
                                                              : apply_smem_doubles(p.K, dense)));
      if (round < 0 && kind != kFinalize) flops += (double)p.nodes * qr_flops(p.m, p.K);
      b.d[b.count++] = d;
    }
    if (!b.count) continue;
    ProfToken tok = prof_begin(stream);
    if (kind == kFinalize) {
      qr_finalize_kernel<<<blocks, 256, 0, stream>>>(b);
      HT_LAUNCH_CHECK();
      prof_end(tok, "qr_finalize", stream, 0.0, 0.0);
    } else if (kind == kFactor) {
      qr_factor_kernel<<<blocks, QTF, smem, stream>>>(b);
      HT_LAUNCH_CHECK();
      prof_end(tok, round < 0 ? "qr_block_factor" : "qr_tree_factor", stream, flops, 0.0);
    } else {
      qr_apply_kernel<<<blocks, QT, smem, stream>>>(b);
      HT_LAUNCH_CHECK();
      prof_end(tok, round < 0 ? "qr_block_apply" : "qr_tree_apply", stream, flops, 0.0);
    }
  }
  return kOk;
}

}  // namespace

int qr_plan(QrProblem& p) {
  if (p.K < 1 || p.m < 1) {
    set_error("qr_plan: empty matrix");
    return kErrShape;
  }
  if (p.K > kQrMaxK) {
    set_error("qr_plan: K=" + std::to_string(p.K) + " exceeds the shared-memory QR path (K <= 112)");
    return kErrUnsupported;
  }
  int P = ceil_div(p.m, BR);
  int rpc = std::max(ceil_div(p.m, P), std::min(p.K, BR));
  P = ceil_div(p.m, rpc);
  p.P = P;
  p.rpc = rpc;
  const int np = npanels(p.K);
  p.v_node = (long long)p.m * p.K;
  p.st_node = (long long)P * p.K * p.K;
  p.t_node = 2LL * P * np * NB * NB;  // per-panel T factors of blocks and tree pairs
  p.x_node = 2LL * P * p.K;           // taus
  p.own_v = (p.V == nullptr);
  return kOk;
}

long long qr_workspace_doubles(const QrProblem& p) {
  return (long long)p.nodes * ((p.own_v ? p.v_node : 0) + p.st_node + p.t_node + p.x_node) + 1024;
}

void qr_bind_workspace(QrProblem& p, double* ws) {
  if (p.own_v) {
    p.V = ws;
    ws += (long long)p.nodes * p.v_node;
  }
  p.Rst = ws;
  ws += (long long)p.nodes * p.st_node;
  p.Tst = ws;
  ws += (long long)p.nodes * p.t_node;
  p.X = ws;
}

int qr_batched(std::vector<QrProblem>& probs, cudaStream_t stream) {
  if (probs.empty()) return kOk;
  if (g_sync_check && getenv("HT_SYNC_DUMP"))
    for (const auto& p : probs)
      fprintf(stderr,
              "[qr] m=%d K=%d nodes=%d P=%d rpc=%d A=%p(%lld,%lld,%lld) Q=%p(%lld,%lld,%lld) R=%p(%lld,%lld) V=%p "
              "Rst=%p Tst=%p X=%p own=%d vn=%lld stn=%lld tn=%lld xn=%lld\n",
              p.m, p.K, p.nodes, p.P, p.rpc, (const void*)p.A, p.a_r, p.a_c, p.a_node, (void*)p.Q, p.q_r, p.q_c,
              p.q_node, (void*)p.R, p.r_ld, p.r_node, (void*)p.V, (void*)p.Rst, (void*)p.Tst, (void*)p.X,
              (int)p.own_v, p.v_node, p.st_node, p.t_node, p.x_node);
  if (!g_attr_done) {
    HT_CUDA_CHECK(cudaFuncSetAttribute(qr_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
    HT_CUDA_CHECK(cudaFuncSetAttribute(qr_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
    g_attr_done = true;
  }
  int maxP = 1;
  for (auto& p : probs) maxP = std::max(maxP, p.P);
  int rounds = 0;
  while ((1 << rounds) < maxP) ++rounds;
  HT_TRY(launch(probs, kFactor, -1, stream));
  for (int r = 0; r < rounds; ++r) HT_TRY(launch(probs, kFactor, r, stream));
  HT_TRY(launch(probs, kFinalize, 0, stream));
  for (int r = rounds - 1; r >= 0; --r) HT_TRY(launch(probs, kApply, r, stream));
  HT_TRY(launch(probs, kApply, -1, stream));
  return kOk;
}

}  // namespace ht
