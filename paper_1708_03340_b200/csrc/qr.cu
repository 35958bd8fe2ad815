// Tree-TSQR Householder QR with register-resident blocks and compact-WY Q
// formation on DMMA GEMMs (see qr.cuh).
//
// Reference semantics: kernels.py:24-32 -- dlarfg reflectors as in LAPACK
// dgeqrf, explicit thin Q (dorgqr), sign fix diag(R) >= 0; wide input (m < K)
// gives Q m x m and R m x K (kernels.py:27-28).
#include <algorithm>

#include "gemm.cuh"
#include "prof.cuh"
#include "qr.cuh"

namespace ht {

namespace {

constexpr int QT = 512;          // threads per CTA
constexpr int NW = QT / kWarp;   // 16 warps
constexpr int LR = 4;            // row slots per lane: rows lane + 32 t -> 128-row blocks
constexpr int MC = 7;            // column slots per warp: columns w + 16 m -> K <= 112
constexpr int BR = kWarp * LR;   // 128 block rows
constexpr int MAXD = 32;

struct QrDev {
  const double* A;
  long long a_r, a_c, a_node;
  double* Q;
  long long q_r, q_c, q_node;
  double* R;
  long long r_ld, r_node;
  double* V;
  double* Rst;
  double* Tst;
  long long v_node, st_node, t_node;
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

struct Smem {
  double* R;     // K x (K+1) heads of the triangular-head mode
  double* GT;    // K x (K+1): strict upper = G = Y^T Y, strict lower = T^T
  double* vbuf;  // 2 x 128: the current / next reflector (head 1 and zeros included)
  double* taus;  // K
  double* prm;   // 2 x 4: tau of the current / next reflector
  int rp;
};

__device__ __forceinline__ Smem carve(double* sm, int K) {
  Smem s;
  s.rp = K + 1;
  s.R = sm;
  s.GT = s.R + K * s.rp;
  s.vbuf = s.GT + K * s.rp;
  s.taus = s.vbuf + 2 * BR;
  s.prm = s.taus + K;
  return s;
}

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Transposed 8-way warp reduction: afterwards lane L holds the warp total of slot
// (L >> 2) & 7 (lanes 4m..4m+3 hold slot m).  18 shuffles instead of 40.
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

// reflector jj (dlarfg) from the owner warp's column registers; publishes v (with its
// head 1 and zeros) in vbuf[buf] and tau in prm[buf]
template <bool DENSE>
__device__ __forceinline__ void gen_reflector(double (&col)[LR], int jj, int buf, int nrows, const Smem& s) {
  const int lane = threadIdx.x & 31;
  const int rp = s.rp;
  double ss = 0.0;
#pragma unroll
  for (int t = 0; t < LR; ++t) {
    const int row = lane + t * kWarp;
    const bool tail = row < nrows && (!DENSE || row > jj);
    if (tail) ss = fma(col[t], col[t], ss);
  }
  ss = warp_allsum(ss);
  double alpha;
  if (DENSE) {
    double hv = col[0];
#pragma unroll
    for (int t = 1; t < LR; ++t)
      if ((jj >> 5) == t) hv = col[t];
    alpha = __shfl_sync(0xffffffffu, hv, jj & 31);
  } else {
    alpha = s.R[jj * rp + jj];
  }
  double beta = alpha, tau = 0.0, scal = 0.0;
  if (ss > 0.0) {
    beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
    tau = (beta - alpha) / beta;
    scal = 1.0 / (alpha - beta);
  }
#pragma unroll
  for (int t = 0; t < LR; ++t) {
    const int row = lane + t * kWarp;
    const bool tail = row < nrows && (!DENSE || row > jj);
    if (tail) col[t] *= scal;
    double vb = tail ? col[t] : 0.0;
    if (DENSE && row == jj) {
      col[t] = beta;
      vb = 1.0;
    }
    s.vbuf[buf * BR + row] = vb;
  }
  if (lane == 0) {
    s.prm[buf * 4] = tau;
    s.taus[jj] = tau;
    if (!DENSE) s.R[jj * rp + jj] = beta;
  }
}

// Householder factorisation of a register block held column-wise: warp w owns columns
// c = w + 16 m (slot m), lane l owns rows l + 32 t (slot t).
//  DENSE: reflector j has head a[j][j], tail rows j+1..nrows-1 (dgeqr2 on the block).
//  !DENSE: head R[j][j] (shared, upper triangular), tail rows 0..nrows-1 (one TSQR step
//          on [R; a]).
// One CTA barrier per reflector: the owner warp of column j+1 updates it first and
// publishes reflector j+1 in the same interval.  G = Y^T Y (strict upper) and the
// compact-WY T (dlarft, transposed into the strict lower part of GT) are built in the
// same intervals.
template <bool DENSE>
__device__ void factor_core(double (&a)[MC][LR], int nrows, int K, int nrefl, const Smem& s) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int rp = s.rp;
  for (int j = tid; j < K; j += blockDim.x) s.taus[j] = 0.0;

  if (nrefl > 0 && w == 0) gen_reflector<DENSE>(a[0], 0, 0, nrows, s);
  __syncthreads();
  for (int j = 0; j < nrefl; ++j) {
    const int buf = j & 1;
    double vr[LR];
#pragma unroll
    for (int t = 0; t < LR; ++t) vr[t] = s.vbuf[buf * BR + lane + t * kWarp];
    const double tau = s.prm[buf * 4];
    double x[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) x[m] = 0.0;
#pragma unroll
    for (int m = 0; m < MC; ++m) {
      const int c = w + NW * m;
      if (c < K && c != j) {
#pragma unroll
        for (int t = 0; t < LR; ++t) x[m] = fma(vr[t], a[m][t], x[m]);
      }
    }
    const double tot = reduce8(x, lane);
#pragma unroll
    for (int m = 0; m < MC; ++m) {
      const int c = w + NW * m;
      if (c < K && c != j) {
        const double d = __shfl_sync(0xffffffffu, tot, 4 * m);
        if (c > j) {
          const double hd = DENSE ? 0.0 : s.R[j * rp + c];
          const double coef = tau * (d + hd);
#pragma unroll
          for (int t = 0; t < LR; ++t) a[m][t] = fma(-coef, vr[t], a[m][t]);
          if (!DENSE && lane == 0) s.R[j * rp + c] = hd - coef;
          if (c == j + 1 && c < nrefl) gen_reflector<DENSE>(a[m], c, buf ^ 1, nrows, s);
        } else if (lane == 0) {
          s.GT[c * rp + j] = d;  // G[c][j] = v_c^T v_j
        }
      }
    }
    __syncthreads();
  }
  // compact-WY T (dlarft): row i solves T[i][j] = -tau_j sum_{l=i}^{j-1} T[i][l] G[l][j],
  // T[i][i] = tau_i -- rows are independent: one thread per row, no barriers.
  // T[i][j] (i < j) is stored transposed at GT[j][i].
  if (tid < nrefl) {
    const int i = tid;
    for (int j = i + 1; j < nrefl; ++j) {
      double a0 = s.taus[i] * s.GT[i * rp + j], a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int l = i + 1;
      for (; l + 3 < j; l += 4) {
        a0 = fma(s.GT[l * rp + i], s.GT[l * rp + j], a0);
        a1 = fma(s.GT[(l + 1) * rp + i], s.GT[(l + 1) * rp + j], a1);
        a2 = fma(s.GT[(l + 2) * rp + i], s.GT[(l + 2) * rp + j], a2);
        a3 = fma(s.GT[(l + 3) * rp + i], s.GT[(l + 3) * rp + j], a3);
      }
      for (; l < j; ++l) a0 = fma(s.GT[l * rp + i], s.GT[l * rp + j], a0);
      s.GT[j * rp + i] = -s.taus[j] * ((a0 + a1) + (a2 + a3));
    }
  }
  __syncthreads();
}

__device__ void store_T(double* T, const Smem& s, int K, int nrefl) {
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    const int i = e / K, j = e - i * K;
    double v = 0.0;
    if (j < nrefl) {
      if (i < j) v = s.GT[j * s.rp + i];
      else if (i == j) v = s.taus[i];
    }
    T[e] = v;
  }
}

// mode 0: dense QR of one row block; mode 1: combine step [R_a; R_b] of round `round`.
__global__ void __launch_bounds__(QT, 1) qr_step_kernel(const __grid_constant__ QrBatch b) {
  extern __shared__ double sm[];
  const QrDev& q = b.d[find_desc(b)];
  const int local = blockIdx.x - q.begin;
  const int nd = local / q.per_node, k = local % q.per_node;
  const int K = q.K;
  const Smem s = carve(sm, K);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double a[MC][LR];
  double* Rst = q.Rst + nd * q.st_node;
  double* Tst = q.Tst + nd * q.t_node;

  if (b.round < 0) {
    // ---- dense block c = k ----
    const int c = k;
    const int row0 = c * q.rpc;
    const int rows = min(q.rpc, q.m - row0);
    const double* A = q.A + nd * q.a_node;
#pragma unroll
    for (int m = 0; m < MC; ++m) {
      const int col = w + NW * m;
#pragma unroll
      for (int t = 0; t < LR; ++t) {
        const int i = lane + t * kWarp;
        a[m][t] = (i < rows && col < K) ? __ldg(A + (long long)(row0 + i) * q.a_r + (long long)col * q.a_c) : 0.0;
      }
    }
    const int nrefl = min(rows, K);
    factor_core<true>(a, rows, K, nrefl, s);
    double* V = q.V + nd * q.v_node;
    double* Rc = Rst + (long long)c * K * K;
#pragma unroll
    for (int m = 0; m < MC; ++m) {
      const int col = w + NW * m;
      if (col >= K) continue;
#pragma unroll
      for (int t = 0; t < LR; ++t) {
        const int i = lane + t * kWarp;
        if (i < rows) V[(long long)col * q.m + row0 + i] = a[m][t];
        if (i < K) Rc[(long long)i * K + col] = (i < nrefl && col >= i) ? a[m][t] : 0.0;
      }
    }
    store_T(Tst + (long long)c * K * K, s, K, nrefl);
  } else {
    // ---- combine pair (a, b) ----
    const int r = b.round;
    const int ia = k << (r + 1), ib = ia + (1 << r);
    double* Ra = Rst + (long long)ia * K * K;
    double* Rb = Rst + (long long)ib * K * K;
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
      const int i = e / K, c = e - i * K;
      s.R[i * s.rp + c] = Ra[e];
    }
#pragma unroll
    for (int m = 0; m < MC; ++m) {
      const int col = w + NW * m;
#pragma unroll
      for (int t = 0; t < LR; ++t) {
        const int i = lane + t * kWarp;
        a[m][t] = (i < K && col < K) ? Rb[(long long)i * K + col] : 0.0;
      }
    }
    __syncthreads();
    factor_core<false>(a, K, K, K, s);
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
      const int i = e / K, c = e - i * K;
      Ra[e] = s.R[i * s.rp + c];
    }
    // reflector tails of the R_b rows, column-major K x K, into R_b's slot
#pragma unroll
    for (int m = 0; m < MC; ++m) {
      const int col = w + NW * m;
      if (col >= K) continue;
#pragma unroll
      for (int t = 0; t < LR; ++t) {
        const int i = lane + t * kWarp;
        if (i < K) Rb[(long long)col * K + i] = a[m][t];
      }
    }
    store_T(Tst + (long long)(q.P + ib) * K * K, s, K, K);
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

size_t smem_bytes(int K) {
  const int rp = K + 1;
  return (size_t)(2 * K * rp + 2 * BR + K + 8) * sizeof(double);
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
  d.V = p.V; d.Rst = p.Rst; d.Tst = p.Tst;
  d.v_node = p.v_node; d.st_node = p.st_node; d.t_node = p.t_node;
  d.m = p.m; d.K = p.K; d.P = p.P; d.rpc = p.rpc;
  d.nodes = p.nodes;
  return d;
}

double qr_flops(int m, int K) {
  const double a = std::max(m, K), b = std::min(m, K);
  return 2.0 * a * b * b - 2.0 / 3.0 * b * b * b;
}

// round < 0: dense blocks; round >= 0: combine round; round == -2: finalize
int launch(std::vector<QrProblem>& probs, int round, cudaStream_t stream) {
  size_t i = 0;
  while (i < probs.size()) {
    QrBatch b;
    b.count = 0;
    b.round = round == -2 ? 0 : round;
    int blocks = 0;
    size_t smem = 0;
    double flops = 0;
    while (i < probs.size() && b.count < MAXD) {
      const QrProblem& p = probs[i++];
      int per;
      if (round == -2) per = 1;
      else if (round < 0) per = p.P;
      else per = pairs_host(p.P, round);
      if (per == 0 || p.nodes == 0) continue;
      QrDev d = to_dev(p);
      d.begin = blocks;
      d.per_node = per;
      blocks += per * p.nodes;
      smem = std::max(smem, smem_bytes(p.K));
      if (round == -1) flops += (double)p.nodes * qr_flops(p.m, p.K);
      b.d[b.count++] = d;
    }
    if (!b.count) continue;
    ProfToken tok = prof_begin(stream);
    if (round == -2) {
      qr_finalize_kernel<<<blocks, 256, 0, stream>>>(b);
      HT_LAUNCH_CHECK();
      prof_end(tok, "qr_finalize", stream, 0.0, 0.0);
    } else {
      qr_step_kernel<<<blocks, QT, smem, stream>>>(b);
      HT_LAUNCH_CHECK();
      prof_end(tok, round < 0 ? "qr_block_factor" : "qr_tree_combine", stream, flops, 0.0);
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
    set_error("qr_plan: K=" + std::to_string(p.K) + " exceeds the register-resident QR path (K <= 112)");
    return kErrUnsupported;
  }
  int P = ceil_div(p.m, BR);
  int rpc = std::max(ceil_div(p.m, P), std::min(p.K, BR));
  P = ceil_div(p.m, rpc);
  p.P = P;
  p.rpc = rpc;
  p.v_node = (long long)p.m * p.K;
  p.st_node = (long long)P * p.K * p.K;
  p.t_node = 2LL * P * p.K * p.K;
  p.x_node = 3LL * P * p.K * p.K;
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
  if (!g_attr_done) {
    HT_CUDA_CHECK(cudaFuncSetAttribute(qr_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    g_attr_done = true;
  }
  int maxP = 1;
  for (auto& p : probs) maxP = std::max(maxP, p.P);
  int rounds = 0;
  while ((1 << rounds) < maxP) ++rounds;

  // ---- factorisation ----
  HT_TRY(launch(probs, -1, stream));
  for (int r = 0; r < rounds; ++r) HT_TRY(launch(probs, r, stream));
  HT_TRY(launch(probs, -2, stream));

  // ---- Q formation on DMMA GEMMs (compact WY) ----
  // Q(row, col) for row = chunk start + i; W blocks live in Q's top rows of each chunk.
  auto qptr = [](const QrProblem& p, long long row) { return p.Q + row * p.q_r; };
  for (int r = rounds - 1; r >= 0; --r) {
    std::vector<GemmDesc> g1, g2;
    for (auto& p : probs) {
      const int np = pairs_host(p.P, r);
      if (np == 0) continue;
      const int K = p.K, kq = std::min(p.m, K);
      const long long KK = (long long)K * K;
      const long long pair_rows = (long long)p.rpc << (r + 1);
      const long long hb = 1LL << r;
      // last chunk may be short: split off the pair whose b is the last chunk
      const int last_b = (int)((long long)(np - 1) * (2 * hb) + hb);
      const int rows_lastb = std::min(p.rpc, p.m - last_b * p.rpc);
      const bool short_last = rows_lastb < K;
      auto add_pairs = [&](int k0, int cnt, int krb) {
        if (cnt <= 0) return;
        const long long ia0 = (long long)k0 * 2 * hb, ib0 = ia0 + hb;
        double* X = p.X + ia0 * KK;
        // X = T_ab W_a  (K x kq)
        GemmDesc x = gemm_desc(p.Tst + (p.P + ib0) * KK, K, 1, qptr(p, ia0 * p.rpc), p.q_r, p.q_c, X, kq, 1, K,
                               kq, K);
        x.nb1 = cnt; x.a_b1 = 2 * hb * KK; x.b_b1 = pair_rows * p.q_r; x.c_b1 = 2 * hb * KK;
        x.nb2 = p.nodes; x.a_b2 = p.t_node; x.b_b2 = p.q_node; x.c_b2 = p.x_node;
        g1.push_back(x);
        // W_b = -V_b X   (krb x kq); V_b column-major K x K in R_b's slot
        GemmDesc wb = gemm_desc(p.Rst + ib0 * KK, 1, K, X, kq, 1, qptr(p, ib0 * p.rpc), p.q_r, p.q_c, krb, kq, K,
                                -1.0, 0.0);
        wb.nb1 = cnt; wb.a_b1 = 2 * hb * KK; wb.b_b1 = 2 * hb * KK; wb.c_b1 = pair_rows * p.q_r;
        wb.nb2 = p.nodes; wb.a_b2 = p.st_node; wb.b_b2 = p.x_node; wb.c_b2 = p.q_node;
        g2.push_back(wb);
        // W_a -= X
        GemmDesc wa = gemm_desc(nullptr, 0, 0, X, kq, 1, qptr(p, ia0 * p.rpc), p.q_r, p.q_c, K, kq, K, -1.0, 1.0);
        wa.a_tri = 3;
        wa.nb1 = cnt; wa.b_b1 = 2 * hb * KK; wa.c_b1 = pair_rows * p.q_r;
        wa.nb2 = p.nodes; wa.b_b2 = p.x_node; wa.c_b2 = p.q_node;
        g2.push_back(wa);
      };
      if (short_last) {
        add_pairs(0, np - 1, K);
        add_pairs(np - 1, 1, rows_lastb);
      } else {
        add_pairs(0, np, K);
      }
    }
    HT_TRY(gemm_grouped(g1, stream, "gemm_qr_tree"));
    HT_TRY(gemm_grouped(g2, stream, "gemm_qr_tree"));
  }
  {
    // blocks: X1 = Y_top^T W, X2 = T X1, Q = [W; 0] - Y X2
    std::vector<GemmDesc> g1, g2, g3;
    for (auto& p : probs) {
      const int K = p.K, kq = std::min(p.m, K);
      const long long KK = (long long)K * K;
      const int last_rows = p.m - (p.P - 1) * p.rpc;
      auto add_blocks = [&](int c0, int cnt, int rows) {
        if (cnt <= 0) return;
        const int kr = std::min(rows, K);
        double* X1 = p.X + (long long)p.P * KK + (long long)c0 * KK;
        double* X2 = p.X + 2LL * p.P * KK + (long long)c0 * KK;
        const long long row0 = (long long)c0 * p.rpc;
        // X1 (K x kq) = Y[0:kr, :]^T W (kr x kq): A(m,k) = Y(k,m), unit-upper in (m,k)
        GemmDesc a = gemm_desc(p.V + row0, p.m, 1, qptr(p, row0), p.q_r, p.q_c, X1, kq, 1, K, kq, kr);
        a.a_tri = 2;
        a.nb1 = cnt; a.a_b1 = p.rpc; a.b_b1 = (long long)p.rpc * p.q_r; a.c_b1 = KK;
        a.nb2 = p.nodes; a.a_b2 = p.v_node; a.b_b2 = p.q_node; a.c_b2 = p.x_node;
        g1.push_back(a);
        // X2 = T X1
        GemmDesc t = gemm_desc(p.Tst + (long long)c0 * KK, K, 1, X1, kq, 1, X2, kq, 1, K, kq, K);
        t.nb1 = cnt; t.a_b1 = KK; t.b_b1 = KK; t.c_b1 = KK;
        t.nb2 = p.nodes; t.a_b2 = p.t_node; t.b_b2 = p.x_node; t.c_b2 = p.x_node;
        g2.push_back(t);
        // Q rows [0, kr) = W - Y[0:kr] X2  (unit-lower in (m,k))
        GemmDesc top = gemm_desc(p.V + row0, 1, p.m, X2, kq, 1, qptr(p, row0), p.q_r, p.q_c, kr, kq, K, -1.0, 1.0);
        top.a_tri = 1;
        top.nb1 = cnt; top.a_b1 = p.rpc; top.b_b1 = KK; top.c_b1 = (long long)p.rpc * p.q_r;
        top.nb2 = p.nodes; top.a_b2 = p.v_node; top.b_b2 = p.x_node; top.c_b2 = p.q_node;
        g3.push_back(top);
        if (rows > kr) {
          // Q rows [kr, rows) = -Y[kr:rows] X2  (dense part of Y)
          GemmDesc bot = gemm_desc(p.V + row0 + kr, 1, p.m, X2, kq, 1, qptr(p, row0 + kr), p.q_r, p.q_c, rows - kr,
                                   kq, K, -1.0, 0.0);
          bot.nb1 = cnt; bot.a_b1 = p.rpc; bot.b_b1 = KK; bot.c_b1 = (long long)p.rpc * p.q_r;
          bot.nb2 = p.nodes; bot.a_b2 = p.v_node; bot.b_b2 = p.x_node; bot.c_b2 = p.q_node;
          g3.push_back(bot);
        }
      };
      if (last_rows == p.rpc) {
        add_blocks(0, p.P, p.rpc);
      } else {
        add_blocks(0, p.P - 1, p.rpc);
        add_blocks(p.P - 1, 1, last_rows);
      }
    }
    HT_TRY(gemm_grouped(g1, stream, "gemm_qr_block"));
    HT_TRY(gemm_grouped(g2, stream, "gemm_qr_block"));
    HT_TRY(gemm_grouped(g3, stream, "gemm_qr_block"));
  }
  return kOk;
}

}  // namespace ht
