// Batched symmetric eigensolver, fast path: one CTA per K x K matrix (K <= 112),
// everything in shared memory.
//
//   1. Householder tridiagonalisation A = Q T Q^T (lower, dsytd2 order): per column
//      one reflector, the symmetric mat-vec p = tau A22 v by 4 threads per row, and
//      the rank-2 update A22 -= v w^T + w v^T, on the lower triangle only.  Reflectors
//      stay in the lower triangle.
//   2. All K eigenvalues of T by multisection bisection: 4 threads per eigenvalue
//      evaluate Sturm counts at 4 points per round (sign changes of the scaled
//      leading-minor recurrence p_k = (d_k - x) p_{k-1} - e_{k-1}^2 p_{k-2}).
//   3. select_rank (arith.py:69-88) on the device, then eigenvectors of T for the
//      kept ranks only, by twisted factorisation (stationary + progressive LDL^T,
//      twist at min |gamma_k|), four O(K) passes held in the output row itself;
//      close pairs (gap < 1e-5 ||T||) are re-orthogonalised (MGS) in T-space.
//   4. Back-transformation by the reflectors, 4 threads per eigenvector.
//
// Nodes the fast path cannot serve to the reference's accuracy are flagged for the
// Jacobi kernel (eig.cu), which runs next and only on flagged nodes: graded spectra
// (min |lambda| < 1e-6 max |lambda|: the small hierarchical singular values need
// relative accuracy) and near-degenerate kept eigenvalues (gap < 1e-12 ||T||).
#include <cmath>

#include "eig.cuh"
#include "prof.cuh"

namespace ht {
namespace {

constexpr int TT = 512;
#ifndef HT_EIG_TIMING
#define HT_EIG_TIMING 0  // 1: blocks 0-1 print their phase times (clock64) -- experiments only
#endif
constexpr int MAXD = 48;
constexpr int kGroup = 4;  // threads per eigenvalue / eigenvector / mat-vec row
constexpr double kGradedTol = 1e-6;
constexpr double kDegenTol = 1e-12;
constexpr double kClusterTol = 1e-5;

struct TriBatch {
  int count;
  int kmax;  // largest K of the batch (sizes the shared-memory vectors)
  int begin[MAXD + 1];
  EigProblem d[MAXD];
};

__device__ __forceinline__ double quad_sum(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

// Number of eigenvalues of T strictly below x: sign changes of the leading minors
// p_k = (d_k - x) p_{k-1} - e_{k-1}^2 p_{k-2} (T normalised to ||T|| ~ 1), with
// de[k] = (d_k, e_{k-1}^2) read as one 16-byte word.  Three FP64 ops per step; the
// sign test runs on the integer pipe and the exact power-of-two rescale is checked
// every 8 steps (|p| changes by at most 2^16 up / 2^-424 down in 8 steps: inside a
// block |e_k| > eps ||T||, and splits restart the recurrence).  A zero minor counts
// as positive.  `splits`: some e_k = 0 (block-uniform; the common case has none and
// runs the recurrence without the restart select).
__device__ __forceinline__ int sturm_count(const double2* de, int K, double x, bool splits) {
  double pm2 = 1.0, pm1 = de[0].x - x;
  int c = __double_as_longlong(pm1) < 0;
  int k = 1;
  auto step = [&](int kk) {
    const double2 t = de[kk];
    // a split (e_{k-1} = 0) restarts the recurrence for the next block with
    // p_{k-1} = 1: the count adds up over blocks and |p| cannot decay across it
    const double q = (splits && t.y == 0.0) ? 1.0 : pm1;
    const double p = fma(t.x - x, q, -t.y * pm2);
    c += (int)((unsigned)(__double2hiint(p) ^ __double2hiint(q)) >> 31);
    pm2 = q;
    pm1 = p;
  };
  while (k < K) {
    if (k + 8 <= K) {
#pragma unroll
      for (int u = 0; u < 8; ++u) step(k + u);
      k += 8;
    } else {
      for (; k < K; ++k) step(k);
    }
    const double a = fmax(fabs(pm1), fabs(pm2));
    if (a > 0x1p+300) {
      pm1 *= 0x1p-300;
      pm2 *= 0x1p-300;
    } else if (a < 0x1p-300) {
      pm1 *= 0x1p+300;
      pm2 *= 0x1p+300;
    }
  }
  return c;
}

// Back-transformation of one vector slice held in registers: thread `part` of an
// 8-thread group owns rows part + 8q (q < kBtRQ).  Reflectors j of block JB
// (8 JB <= j < 8 JB + 8) touch rows > j, i.e. register q = JB (rows with part >
// j - 8 JB) and all q > JB: the block index is a template parameter so the register
// window is resolved at compile time.  v_j = 1 at row j + 1, A[row][j] below.
constexpr int kBtG = 8, kBtRQ = (kEigMaxK + kBtG - 1) / kBtG;
template <int JB>
__device__ __forceinline__ void bt_block(double (&zr)[kBtRQ], const double* A, const double* tau, int ap, int K,
                                         int part) {
  const int jhi = min(8 * JB + 7, K - 3);
  for (int j = jhi; j >= 8 * JB; --j) {
    const double tj = tau[j];
    if (tj == 0.0) continue;
    double av[kBtRQ];
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int q = JB; q < kBtRQ; ++q) {
      const int row = part + kBtG * q;
      double a;
      if (q == JB) a = row == j + 1 ? 1.0 : (row > j && row < K ? A[row * ap + j] : 0.0);
      else if (q == JB + 1) a = row == j + 1 ? 1.0 : (row < K ? A[row * ap + j] : 0.0);
      else a = row < K ? A[row * ap + j] : 0.0;
      av[q] = a;
      if ((q - JB) & 1) s1 = fma(a, zr[q], s1);
      else s0 = fma(a, zr[q], s0);
    }
    double sj = s0 + s1;
    sj += __shfl_xor_sync(0xffffffffu, sj, 1);
    sj += __shfl_xor_sync(0xffffffffu, sj, 2);
    sj += __shfl_xor_sync(0xffffffffu, sj, 4);
    sj *= tj;
#pragma unroll
    for (int q = JB; q < kBtRQ; ++q) zr[q] = fma(-sj, av[q], zr[q]);
  }
}

template <int JB>
__device__ __forceinline__ void bt_dispatch(int jb, double (&zr)[kBtRQ], const double* A, const double* tau, int ap,
                                            int K, int part) {
  if constexpr (JB >= 0) {
    if (jb == JB) bt_block<JB>(zr, A, tau, ap, K, part);
    else bt_dispatch<JB - 1>(jb, zr, A, tau, ap, K, part);
  }
}

__global__ void __launch_bounds__(TT, 1) tri_eig_kernel(const __grid_constant__ TriBatch b) {
  extern __shared__ double sm[];
  int di = 0;
  while (di + 1 < b.count && (int)blockIdx.x >= b.begin[di + 1]) ++di;
  const EigProblem& e = b.d[di];
  const int nd = blockIdx.x - b.begin[di];
  const int K = e.K;
  const int KM = b.kmax;
  const int ap = K | 1;            // odd pitch
  const int zp = (K + 1) | 1;
  double* dd = sm;                 // [KM] diagonal of T
  double* ee = dd + KM;            // [KM] off-diagonal
  double* e2 = ee + KM;            // [KM] squares
  double* tau = e2 + KM;           // [KM]
  double* vb = tau + KM;           // [2][KM] reflectors (double-buffered)
  double* pb = vb + 2 * KM;        // [KM] p
  double* lam = pb + KM;           // [KM] ascending eigenvalues
  // the matrix and the eigenvectors of T: shared memory up to kEigMaxK, else the
  // node's global scratch (L2-resident)
  const bool big = K > kEigMaxK;
  double* A = big ? e.work + nd * e.w_node : lam + KM;  // K x ap
  double* Z = A + (size_t)K * ap;                        // r x zp, one row per kept pair
  __shared__ double red[TT / 32][2];
  __shared__ double sh[4];
  __shared__ int flags[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- load, symmetry check (kernels.py:46-50), symmetrise -------------------
  long long clk[6] = {clock64(), 0, 0, 0, 0, 0};
  const double* S = e.S + nd * e.s_node;
  double asym = 0.0, amax = 0.0;
  for (int x = tid; x < K * K; x += TT) {
    const int i = x / K, j = x - i * K;
    const double a = S[x], at = S[j * K + i];
    asym = fmax(asym, fabs(a - at));
    amax = fmax(amax, fabs(a));
    if (!isfinite(a)) amax = INFINITY;  // fmax drops NaN: make it visible
    A[i * ap + j] = 0.5 * (a + at);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    asym = fmax(asym, __shfl_xor_sync(0xffffffffu, asym, o));
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  }
  if (lane == 0) { red[warp][0] = asym; red[warp][1] = amax; }
  __syncthreads();
  if (tid == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < TT / 32; ++w) { s0 = fmax(s0, red[w][0]); s1 = fmax(s1, red[w][1]); }
    if (e.status && s0 > 1e-12 * fmax(1.0, s1)) atomicOr(e.status, kEigStatusNotSymmetric);
    if (e.status && !isfinite(s1)) atomicOr(e.status, kEigStatusNonConverged);
    flags[0] = 0;
    flags[1] = isfinite(s1) ? 0 : 1;
  }
  __syncthreads();
  if (flags[1]) {  // non-finite Gramian: flagged above; NaN results, no Jacobi redo
    for (int x = tid; x < K * K; x += TT) e.V[nd * e.v_node + x] = __longlong_as_double(0x7ff8000000000000ll);
    for (int x = tid; x < K; x += TT) e.lam[nd * e.l_node + x] = __longlong_as_double(0x7ff8000000000000ll);
    if (tid == 0) {
      if (e.rank) e.rank[nd] = e.cap > 0 ? min(e.cap, K) : K;
      if (e.fallback) e.fallback[nd] = 0;
    }
    return;
  }

  // ---- 1. tridiagonalisation --------------------------------------------------
  if (HT_EIG_TIMING) clk[1] = clock64();
  // Reflector j from column j (rows j+1..K-1), computed by warp 0 into vbuf[j & 1]
  // while the other warps finish the previous rank-2 update: two barriers per column.
  double* vbuf = vb;
  auto reflector = [&](int j, double* v) {
    const int m = K - j - 1;
    double ss = 0.0;
    for (int k = 1 + lane; k < m; k += 32) {
      const double x = A[(j + 1 + k) * ap + j];
      ss = fma(x, x, ss);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const double alpha = A[(j + 1) * ap + j];
    double t = 0.0, beta = alpha, scale = 0.0;
    if (ss > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
      t = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    for (int k = lane; k < m; k += 32) {
      const double x = k == 0 ? 1.0 : A[(j + 1 + k) * ap + j] * scale;
      v[k] = x;
      if (k > 0) A[(j + 1 + k) * ap + j] = x;  // reflector tail kept in the lower triangle
    }
    if (lane == 0) {
      dd[j] = A[j * ap + j];
      ee[j] = beta;
      tau[j] = t;
    }
  };
  if (K > 2 && warp == 0) reflector(0, vbuf);
  __syncthreads();
  for (int j = 0; j + 2 < K; ++j) {
    const int m = K - j - 1;       // reflector length (rows j+1 .. K-1)
    const double* v = vbuf + (j & 1) * KM;
    double* vn = vbuf + ((j + 1) & 1) * KM;
    const double tj = tau[j];
    if (tj != 0.0) {
      // p = tau * A22 v (4 threads per row) and the per-warp partial of p.v.  Only the
      // lower triangle of A22 is kept current: S[i][k] is row i for k <= i, column i
      // (odd pitch: conflict-free across rows) for k > i.
      {
        for (int i0 = 0; i0 < m; i0 += TT / kGroup) {
          const int i = i0 + tid / kGroup, part = tid % kGroup;
          double acc = 0.0, acc2 = 0.0;
          if (i < m) {
            const double* rowi = A + (size_t)(j + 1 + i) * ap + (j + 1);
            const double* coli = A + (size_t)(j + 1) * ap + (j + 1 + i);
            // uniform trip count across the warp (rows differ in where they switch)
            int k = part;
            for (; k + kGroup < m; k += 2 * kGroup) {
              const int k2 = k + kGroup;
              acc = fma(k <= i ? rowi[k] : coli[(size_t)k * ap], v[k], acc);
              acc2 = fma(k2 <= i ? rowi[k2] : coli[(size_t)k2 * ap], v[k2], acc2);
            }
            if (k < m) acc = fma(k <= i ? rowi[k] : coli[(size_t)k * ap], v[k], acc);
          }
          acc = quad_sum(acc + acc2) * tj;
          if (i < m && part == 0) pb[i] = acc;
        }
      }
      __syncthreads();
      // p.v summed by every warp from pb (same order in each: deterministic)
      double sv = 0.0;
      for (int i = lane; i < m; i += 32) sv = fma(pb[i], v[i], sv);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
      const double c = -0.5 * tj * sv;                     // w = p + c v
      if (warp == 0) {
        // column j+1 (A22 column 0), then the next reflector from it
        for (int r = lane; r < m; r += 32) {
          const double wr = fma(c, v[r], pb[r]), w0 = fma(c, v[0], pb[0]);
          A[(j + 1 + r) * ap + (j + 1)] -= fma(v[r], w0, wr * v[0]);
        }
        __syncwarp();
        if (j + 3 < K) reflector(j + 1, vn);
      } else {
        // rank-2 update of the lower triangle (columns 1 .. r of row r); each lane keeps
        // v and w of its columns in registers, 128 columns per pass
        for (int cb = 1; cb < m; cb += 128) {
          double vq[4], wq[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int cc = cb + lane + 32 * q;
            vq[q] = cc < m ? v[cc] : 0.0;
            wq[q] = cc < m ? fma(c, vq[q], pb[cc]) : 0.0;
          }
          int r = warp - 1;
          if (r < cb) r += ((cb - r + TT / 32 - 2) / (TT / 32 - 1)) * (TT / 32 - 1);
          for (; r < m; r += TT / 32 - 1) {
            const double vr = v[r], wr = fma(c, vr, pb[r]);
            double* ar = A + (size_t)(j + 1 + r) * ap + (j + 1);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int cc = cb + lane + 32 * q;
              if (cc <= r) ar[cc] -= fma(vr, wq[q], wr * vq[q]);
            }
          }
        }
      }
    } else if (warp == 0 && j + 3 < K) {
      reflector(j + 1, vn);
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (K >= 2) {
      dd[K - 2] = A[(K - 2) * ap + K - 2];
      ee[K - 2] = A[(K - 1) * ap + K - 2];
    }
    dd[K - 1] = A[(K - 1) * ap + K - 1];
    ee[K - 1] = 0.0;
  }
  __syncthreads();
  // exact power-of-two normalisation of T (eigenvalues O(1): the Sturm recurrence
  // stays in range); lam is scaled back on output
  if (warp == 0) {
    double mx = 0.0;
    for (int k = lane; k < K; k += 32) mx = fmax(mx, fmax(fabs(dd[k]), fabs(ee[k])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) sh[3] = (mx > 0.0 && isfinite(mx)) ? exp2(-(double)ilogb(mx)) : 1.0;
  }
  __syncthreads();
  const double tscale = sh[3];
  for (int k = tid; k < K; k += TT) {
    dd[k] *= tscale;
    ee[k] *= tscale;
    e2[k] = ee[k] * ee[k];
  }
  __syncthreads();
  // Gershgorin bounds, pivmin
  if (warp == 0) {
    double gl = INFINITY, gu = -INFINITY, em = 0.0;
    for (int k = lane; k < K; k += 32) {
      const double r = (k > 0 ? fabs(ee[k - 1]) : 0.0) + (k + 1 < K ? fabs(ee[k]) : 0.0);
      gl = fmin(gl, dd[k] - r);
      gu = fmax(gu, dd[k] + r);
      if (k + 1 < K) em = fmax(em, ee[k] * ee[k]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
      gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
      em = fmax(em, __shfl_xor_sync(0xffffffffu, em, o));
    }
    if (lane == 0) {
      const double tn = fmax(fabs(gl), fabs(gu));
      const double pad = 2.0 * 2.220446049250313e-16 * tn * K + 1e-300;
      sh[0] = gl - pad;
      sh[1] = gu + pad;
      sh[2] = 2.2250738585072014e-308 * fmax(1.0, em);
      sh[3] = tn;
    }
  }
  __syncthreads();
  // split T at negligible off-diagonals (|e_k| <= eps ||T||, a perturbation inside the
  // absolute accuracy of the reduction): graded Gramians leave long runs of tiny
  // e_k whose products would underflow the Sturm recurrence, and the twisted
  // vectors of eigenvalues shared by several blocks stay confined to their block
  bool split = false;
  for (int k = tid; k + 1 < K; k += TT)
    if (fabs(ee[k]) <= 2.220446049250313e-16 * sh[3]) {
      ee[k] = 0.0;
      e2[k] = 0.0;
      split = true;
    }
  const bool splits = __syncthreads_or(split);
  // (d_k, e_{k-1}^2) pairs for the Sturm recurrence, in the reflector / p buffers
  // (free after the reduction; 16-byte aligned)
  double2* de = reinterpret_cast<double2*>(vb + ((reinterpret_cast<uintptr_t>(vb) >> 3) & 1));
  for (int k = tid; k < K; k += TT) de[k] = make_double2(dd[k], k > 0 ? e2[k - 1] : 0.0);
  __syncthreads();

  // ---- 2. eigenvalues: multisection bisection, 4 threads per eigenvalue ---------
  if (HT_EIG_TIMING) clk[2] = clock64();
  for (int i0 = 0; i0 < K; i0 += TT / kGroup) {
    const int i = i0 + tid / kGroup, part = tid % kGroup;
    const double pivmin = sh[2];
    const double atol = 4.0 * 2.220446049250313e-16 * sh[3] + pivmin;  // absolute accuracy of the reduction
    double lo = sh[0], hi = sh[1];
    const bool act = i < K;
    for (int it = 0; it < 64; ++it) {
      const double w = hi - lo;
      const bool done = !(w > 2.220446049250313e-16 * 2.0 * fmax(fabs(lo), fabs(hi)) + atol);
      if (__all_sync(0xffffffffu, done || !act)) break;
      const double x = lo + w * (double)(part + 1) / (double)(kGroup + 1);
      const int c = act ? sturm_count(de, K, x, splits) : 0;
      // smallest point with count > i becomes hi; the point before it lo
      const unsigned base = (unsigned)(lane & ~(kGroup - 1));
      double nlo = lo, nhi = hi;
      bool found = false;
#pragma unroll
      for (int g = 0; g < kGroup; ++g) {
        const int cg = __shfl_sync(0xffffffffu, c, base + g);
        const double xg = __shfl_sync(0xffffffffu, x, base + g);
        if (!found) {
          if (cg > i) {
            nhi = xg;
            found = true;
          } else {
            nlo = xg;
          }
        }
      }
      if (!done) {
        lo = nlo;
        hi = nhi;
      }
    }
    if (act && part == 0) lam[i] = 0.5 * (lo + hi);
  }
  __syncthreads();
  const double unscale = 1.0 / tscale;  // exact (power of two)

  // ---- outputs: eigenvalues (descending, clamped), rank, fallback decision ------
  double* lamo = e.lam + nd * e.l_node;
  for (int k = tid; k < K; k += TT) lamo[k] = fmax(lam[K - 1 - k] * unscale, 0.0);
  __shared__ int rsel;
  if (tid == 0) {
    int r = K;
    if (e.eps > 0.0) {
      const double budget = e.eps * e.eps * (e.eps_scale2 ? *e.eps_scale2 : 1.0) / e.n_nonroot;
      double tail = 0.0;
      for (int k = K - 1; k >= 0; --k) {  // descending index k <-> ascending K-1-k
        tail += fmax(lam[K - 1 - k] * unscale, 0.0);
        if (tail <= budget) r = k;
        else break;
      }
    }
    if (e.cap > 0) r = min(r, e.cap);
    r = max(1, min(r, K));
    if (e.rank) e.rank[nd] = r;
    rsel = r;
    const double tn = fmax(fabs(lam[0]), fabs(lam[K - 1]));
    int fb = 0, graded = 0;
    if (e.graded_fallback)
      for (int k = 0; k < K; ++k)
        if (fabs(lam[k]) < kGradedTol * tn) graded = 1;  // graded: relative accuracy needed
    // kept eigenpairs (ascending K-r .. K-1) and the boundary pair must be separated
    for (int k = max(0, K - r - 1); k + 1 < K; ++k)
      if (lam[k + 1] - lam[k] < kDegenTol * tn) fb = 1;
    if (!(tn > 0.0) || !isfinite(tn)) fb = 1;  // zero / non-finite matrix: Jacobi
    fb |= graded;
    if (big) {
      // beyond kEigMaxK the Jacobi redo runs out of global scratch (slow): only for
      // graded spectra whose every sigma was asked for (HT_CTL_RELATIVE_SIGMA); close
      // kept pairs are handled by the MGS pass below, to LAPACK's absolute accuracy
      if (fb && !graded && e.status && !(tn >= 0.0)) atomicOr(e.status, kEigStatusNonConverged);
      fb = graded;
    }
    flags[1] = fb;
    if (e.fallback) e.fallback[nd] = fb;
  }
  __syncthreads();
  if (flags[1]) return;  // the Jacobi kernel takes this node
  const int r = rsel;

  // ---- 3. eigenvectors of T (twisted factorisation) --------------------------------
  if (HT_EIG_TIMING) clk[3] = clock64();
  // Fast path (2r <= K, matrices in shared memory): two adjacent lanes per vector run
  // the stationary (D+, lane 0) and progressive (D-, lane 1, into the spare row r + v
  // of Z) recurrences at the same time; gamma / twist, L = e / D+ and U = e / D- are
  // then element-wise, and the two product chains run down and up from the twist
  // concurrently.  Same quantities as the serial passes below.
  const bool pair2 = !big && K >= 2 && 2 * r <= K;
  if (pair2) {
    const int v = tid >> 1, role = tid & 1;
    const bool act = v < r;
    const double sig = act ? lam[K - 1 - v] : 0.0;
    double* z = Z + (size_t)(act ? v : 0) * zp;
    double* w = Z + (size_t)(act ? r + v : 0) * zp;
    const double pivmin = sh[2];
    if (act && role == 0) {  // D+_k (guarded) into z[k]
      double dp = dd[0] - sig;
      if (fabs(dp) < pivmin) dp = -pivmin;
      z[0] = dp;
      for (int k = 0; k + 1 < K; ++k) {
        dp = (dd[k + 1] - sig) - e2[k] / dp;
        if (fabs(dp) < pivmin) dp = -pivmin;
        z[k + 1] = dp;
      }
    } else if (act) {  // guarded D-_k into w[k]
      double dm = dd[K - 1] - sig;
      if (fabs(dm) < pivmin) dm = -pivmin;
      w[K - 1] = dm;
      for (int k = K - 2; k >= 0; --k) {
        const double u = ee[k] / dm;
        const double dmk = (dd[k] - sig) - ee[k] * u;
        dm = fabs(dmk) < pivmin ? -pivmin : dmk;
        w[k] = dm;
      }
    }
    __syncthreads();
    // gamma_k = D+_k + D-_k - (d_k - sig), twist = argmin |gamma| (ties: larger k, as
    // the serial descending scan); lane 0 takes k < K/2, lane 1 the rest
    int twist = K - 1;
    double gmin = INFINITY;
    if (act) {
      const int h = K / 2;
      const int klo = role ? h : 0, khi = role ? K - 1 : h;  // k in [klo, khi)
      if (role) gmin = fabs(z[K - 1]);
      for (int k = khi - 1; k >= klo; --k) {
        const double u = ee[k] / w[k + 1];
        const double dmk = (dd[k] - sig) - ee[k] * u;
        const double g = fabs(z[k] + dmk - (dd[k] - sig));
        if (g < gmin) {
          gmin = g;
          twist = k;
        }
      }
    }
    {
      const double og = __shfl_xor_sync(0xffffffffu, gmin, 1);
      const int ot = __shfl_xor_sync(0xffffffffu, twist, 1);
      if (og < gmin || (og == gmin && ot > twist)) {
        gmin = og;
        twist = ot;
      }
    }
    __syncthreads();  // every gamma is read before z is overwritten
    double part = 0.0;
    if (act && role == 0) {  // z_k = -L_k z_{k+1}, L_k = e_k / D+_k, downward from the twist
      double prev = 1.0;
      for (int k = twist - 1; k >= 0; --k) {
        prev = -(ee[k] / z[k]) * prev;
        z[k] = prev;
        part = fma(prev, prev, part);
      }
    } else if (act) {  // z_{k+1} = -U_k z_k, U_k = e_k / D-_{k+1}, upward from the twist
      double prev = 1.0;
      z[twist] = 1.0;
      for (int k = twist; k + 1 < K; ++k) {
        prev = -(ee[k] / w[k + 1]) * prev;
        z[k + 1] = prev;
        part = fma(prev, prev, part);
      }
    }
    const double nrm = 1.0 + part + __shfl_xor_sync(0xffffffffu, part, 1);
    __syncthreads();
    if (act) {
      const double inv = 1.0 / sqrt(nrm);
      for (int k = role ? twist : 0; k < (role ? K : twist); ++k) z[k] *= inv;
    }
  }
  for (int v = tid; v < r && !pair2; v += TT) {
    const double sig = lam[K - 1 - v];  // descending order: vector v <-> eigenvalue K-1-v
    double* z = Z + v * zp;
    const double pivmin = sh[2];
    if (K == 1) {
      z[0] = 1.0;
      continue;
    }
    // pass 1: stationary D+_k into z[k]
    double dp = dd[0] - sig;
    if (fabs(dp) < pivmin) dp = -pivmin;
    z[0] = dp;
    for (int k = 0; k + 1 < K; ++k) {
      dp = (dd[k + 1] - sig) - e2[k] / dp;
      if (fabs(dp) < pivmin) dp = -pivmin;
      z[k + 1] = dp;
    }
    // pass 2: progressive D-_k, U_k into z[k+1], gamma_k = D+_k + D-_k - (d_k - sig)
    double dm = dd[K - 1] - sig;
    if (fabs(dm) < pivmin) dm = -pivmin;
    int twist = K - 1;
    double gmin = fabs(z[K - 1]);  // gamma_{K-1} = D+_{K-1}
    for (int k = K - 2; k >= 0; --k) {
      const double u = ee[k] / dm;          // U_k
      const double dmk = (dd[k] - sig) - ee[k] * u;
      const double g = z[k] + dmk - (dd[k] - sig);
      z[k + 1] = u;
      dm = fabs(dmk) < pivmin ? -pivmin : dmk;
      if (fabs(g) < gmin) {
        gmin = fabs(g);
        twist = k;
      }
    }
    // pass 3: L_k = e_k / D+_k for k < twist into z[k]
    dp = dd[0] - sig;
    if (fabs(dp) < pivmin) dp = -pivmin;
    for (int k = 0; k < twist; ++k) {
      z[k] = ee[k] / dp;
      dp = (dd[k + 1] - sig) - e2[k] / dp;
      if (fabs(dp) < pivmin) dp = -pivmin;
    }
    // pass 4/5: z_twist = 1, z_k = -L_k z_{k+1} (k < twist), z_{k+1} = -U_k z_k (k >= twist)
    z[twist] = 1.0;
    double nrm = 1.0;
    for (int k = twist - 1; k >= 0; --k) {
      z[k] = -z[k] * z[k + 1];
      nrm = fma(z[k], z[k], nrm);
    }
    for (int k = twist; k + 1 < K; ++k) {
      z[k + 1] = -z[k + 1] * z[k];
      nrm = fma(z[k + 1], z[k + 1], nrm);
    }
    const double inv = 1.0 / sqrt(nrm);
    for (int k = 0; k < K; ++k) z[k] *= inv;
  }
  __syncthreads();
  // Close kept pairs (runs of gap < kClusterTol ||T||), warp 0.  Exactly or nearly
  // degenerate eigenvalues (symmetric problems: T numerically split into blocks
  // sharing an eigenvalue) give (near-)identical twisted vectors, so vector a of a
  // run is refined by two steps of inverse iteration with T - lam_a I, each followed
  // by two Gram-Schmidt passes against the run's earlier vectors; a vector that
  // vanishes under the projection restarts from a pseudo-random one (the solve then
  // pulls it into the cluster's invariant subspace).  Singletons only get a
  // finiteness check.
  if (warp == 0) {
    const double tn = sh[3];
    const double piv = 2.220446049250313e-16 * tn + sh[2];
    double* Dl = vb;  // LDL^T pivots of T - sig I (the reflector buffers are free now)
    auto wsum = [&](double s) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      return s;
    };
    auto nrm2 = [&](const double* z) {
      double s = 0.0;
      for (int k = lane; k < K; k += 32) s = fma(z[k], z[k], s);
      return wsum(s);
    };
    auto project_out = [&](double* za, int v0, int a) {
      for (int pass = 0; pass < 2; ++pass)
        for (int bq = v0; bq < a; ++bq) {
          const double* zb = Z + bq * zp;
          double s = 0.0;
          for (int k = lane; k < K; k += 32) s = fma(za[k], zb[k], s);
          s = wsum(s);
          for (int k = lane; k < K; k += 32) za[k] = fma(-s, zb[k], za[k]);
          __syncwarp();
        }
    };
    int v0 = 0;
    while (v0 < r) {
      int v1 = v0 + 1;
      while (v1 < r && lam[K - 1 - (v1 - 1)] - lam[K - 1 - v1] < kClusterTol * tn) ++v1;
      for (int a = v0; a < v1; ++a) {
        double* za = Z + a * zp;
        const double s0 = nrm2(za);
        if (v1 == v0 + 1 && isfinite(s0) && s0 > 0.0) break;  // singleton, twisted vector fine
        const double sig = lam[K - 1 - a];
        for (int it = 0; it < 3; ++it) {
          // scale to max |z| = 1 first (inverse iteration grows the vector by 1/gap)
          double mx = 0.0;
          for (int k = lane; k < K; k += 32) mx = fmax(mx, fabs(za[k]));
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
          const bool bad = !(mx > 0.0) || !isfinite(mx);
          for (int k = lane; k < K; k += 32) za[k] = bad ? 0.0 : za[k] / mx;
          __syncwarp();
          const double sb = bad ? 0.0 : nrm2(za);
          project_out(za, v0, a);
          double s = nrm2(za);
          if (!(s > 1e-16 * sb)) {  // nothing left outside the earlier vectors: restart
            for (int k = lane; k < K; k += 32) {
              unsigned h = (unsigned)k * 2654435761u ^ (unsigned)(a * 40503 + it * 7919 + 12345);
              h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
              za[k] = (double)(h & 0xffffu) / 65536.0 - 0.5;
            }
            __syncwarp();
            project_out(za, v0, a);
            s = nrm2(za);
          }
          const double inv = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
          for (int k = lane; k < K; k += 32) za[k] *= inv;
          __syncwarp();
          if (it == 2) break;
          // za <- (T - sig I)^{-1} za by LDL^T (pivots guarded at eps ||T||), lane 0
          if (lane == 0) {
            double dk = dd[0] - sig;
            if (fabs(dk) < piv) dk = dk < 0.0 ? -piv : piv;
            Dl[0] = dk;
            for (int k = 1; k < K; ++k) {
              const double l = ee[k - 1] / Dl[k - 1];
              dk = (dd[k] - sig) - l * ee[k - 1];
              if (fabs(dk) < piv) dk = dk < 0.0 ? -piv : piv;
              Dl[k] = dk;
              za[k] = fma(-l, za[k - 1], za[k]);
            }
            za[K - 1] /= Dl[K - 1];
            for (int k = K - 2; k >= 0; --k) za[k] = (za[k] - ee[k] * za[k + 1]) / Dl[k];
          }
          __syncwarp();
        }
      }
      v0 = v1;
    }
  }
  __syncthreads();

  // ---- 4. back-transformation y = H_0 ... H_{K-3} z --------------------------------
  if (HT_EIG_TIMING) clk[4] = clock64();
  if (!big) {
    // 8 threads per vector, the vector in registers (bt_block), so each reflector is
    // one pass over its column (broadcast to the four vectors of a warp) instead of a
    // read-modify-write of z in shared memory
    for (int v0 = 0; v0 < r; v0 += TT / kBtG) {
      const int v = v0 + tid / kBtG, part = tid % kBtG;
      const bool act = v < r;
      double* z = Z + (size_t)(act ? v : 0) * zp;
      double zr[kBtRQ];
#pragma unroll
      for (int q = 0; q < kBtRQ; ++q) {
        const int row = part + kBtG * q;
        zr[q] = (act && row < K) ? z[row] : 0.0;
      }
      for (int jb = (K - 3) / 8; jb >= 0 && K >= 3; --jb) bt_dispatch<kBtRQ - 1>(jb, zr, A, tau, ap, K, part);
      if (act) {
#pragma unroll
        for (int q = 0; q < kBtRQ; ++q) {
          const int row = part + kBtG * q;
          if (row < K) z[row] = zr[q];
        }
      }
    }
  } else {
    const int G = r <= TT / 8 ? 8 : kGroup;  // global-scratch matrices (K > kEigMaxK)
    for (int v0 = 0; v0 < r; v0 += TT / G) {
      const int v = v0 + tid / G, part = tid % G;
      const bool act = v < r;
      double* z = Z + (size_t)(act ? v : 0) * zp;
      for (int j = K - 3; j >= 0; --j) {
        const double tj = tau[j];
        if (tj == 0.0) continue;
        const int m = K - j - 1;
        // v_j: 1 at row j+1, A[(j+1+k)*ap + j] below
        double s = 0.0;
        if (act)
          for (int k = part; k < m; k += G) s = fma(k == 0 ? 1.0 : A[(size_t)(j + 1 + k) * ap + j], z[j + 1 + k], s);
        s += __shfl_xor_sync(0xffffffffu, s, 1);  // all lanes shuffle
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (G == 8) s += __shfl_xor_sync(0xffffffffu, s, 4);
        s *= tj;
        if (act)
          for (int k = part; k < m; k += G) z[j + 1 + k] = fma(-s, k == 0 ? 1.0 : A[(size_t)(j + 1 + k) * ap + j], z[j + 1 + k]);
      }
    }
  }
  __syncthreads();
  double* Vo = e.V + nd * e.v_node;
  for (int x = tid; x < K * r; x += TT) {
    const int row = x / r, c = x - row * r;
    Vo[(long long)row * K + c] = Z[c * zp + row];
  }
  if (HT_EIG_TIMING && tid == 0 && blockIdx.x < 2) {
    clk[5] = clock64();
    printf("tri_eig block %d K=%d r=%d: load %lld tridiag %lld bisect+select %lld eigvec %lld backtr+out %lld cycles\n",
           blockIdx.x, K, r, clk[1] - clk[0], clk[2] - clk[1], clk[3] - clk[2], clk[4] - clk[3], clk[5] - clk[4]);
  }
}

bool g_tri_attr = false;

}  // namespace

int eig_tri_batched(std::vector<EigProblem>& probs, cudaStream_t stream) {
  constexpr size_t kSmemMax = 226 * 1024;  // + the kernel's static shared memory
  if (!g_tri_attr) {
    HT_CUDA_CHECK(cudaFuncSetAttribute(tri_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax));
    g_tri_attr = true;
  }
  // vectors are sized for the batch's largest K; matrices sit in shared memory only
  // for K <= kEigMaxK -- a problem that would push the batch past the limit starts
  // the next batch
  auto mat_bytes = [](int K) {
    return K <= kEigMaxK ? sizeof(double) * ((size_t)K * (K | 1) + (size_t)K * ((K + 1) | 1)) : 0;
  };
  size_t i = 0;
  while (i < probs.size()) {
    TriBatch b;
    b.count = 0;
    b.kmax = 1;
    int blocks = 0;
    size_t mats = 0;
    while (i < probs.size() && b.count < MAXD) {
      const EigProblem& p = probs[i];
      if (p.nodes == 0) {
        ++i;
        continue;
      }
      if (p.K > kEigMaxKBig || (p.K > kEigMaxK && !p.work)) {
        set_error("eigensolver: K=" + std::to_string(p.K) + " needs K <= 512 and a global scratch");
        return kErrUnsupported;
      }
      const int kmax = std::max(b.kmax, p.K);
      const size_t m = std::max(mats, mat_bytes(p.K));
      if (b.count > 0 && sizeof(double) * 8 * (size_t)kmax + 64 + m > kSmemMax) break;
      ++i;
      b.begin[b.count] = blocks;
      blocks += p.nodes;
      b.kmax = kmax;
      mats = m;
      b.d[b.count++] = p;
    }
    const size_t smem = sizeof(double) * 8 * (size_t)b.kmax + 64 + mats;
    if (b.count == 0) continue;
    b.begin[b.count] = blocks;
    double flops = 0;
    for (int q = 0; q < b.count; ++q) flops += 9.0 * b.d[q].nodes * (double)b.d[q].K * b.d[q].K * b.d[q].K;
    ProfToken tok = prof_begin(stream);
    tri_eig_kernel<<<blocks, TT, smem, stream>>>(b);
    HT_LAUNCH_CHECK();
    prof_end(tok, "tridiag_eig", stream, flops, 0.0);
  }
  return kOk;
}

}  // namespace ht
