// Parallel cyclic Jacobi eigensolver, one CTA per matrix (see eig.cuh).
// Each round applies n/2 disjoint rotations (round-robin "circle" ordering);
// the 2x2 blocks of A' = J^T A J are updated once per (pair_i <= pair_j) and
// mirrored, so A stays exactly symmetric.
#include <algorithm>

#include "eig.cuh"
#include "prof.cuh"

namespace ht {

namespace {

constexpr int ET = 512;
constexpr int MAXD = 48;
constexpr int MAX_SWEEPS = 40;

struct EigBatch {
  int count;
  int begin[MAXD + 1];
  EigProblem d[MAXD];
};

__device__ __forceinline__ int circle(int i, int r, int n) {
  // position i of round r in the round-robin schedule over n (even) players
  return i == 0 ? 0 : ((i - 1 + r) % (n - 1)) + 1;
}

// BIG: K > kEigMaxK -- A and V^T live in the node's global scratch (e.work, L2-resident
// at the sizes that need it), only the rotation parameters and the block list stay in
// shared memory.  Same rotations, same order: relative accuracy for graded Gramians at
// any rank up to kEigMaxKBig.
template <bool BIG>
__global__ void __launch_bounds__(ET, 1) jacobi_kernel(const __grid_constant__ EigBatch b) {
  extern __shared__ double sm[];
  int di = 0;
  while (di + 1 < b.count && (int)blockIdx.x >= b.begin[di + 1]) ++di;
  const EigProblem& e = b.d[di];
  const int nd = blockIdx.x - b.begin[di];
  if (e.fallback && e.fallback[nd] == 0) return;  // served by the tridiagonal fast path
  const int K = e.K;
  const int n = K + (K & 1);
  const int ap = n + 1;
  const int half = n / 2;
  const int nblk = half * (half + 1) / 2;
  const int vp_pitch = n + 2;      // even: 16-byte aligned rows for double2 rotations
  double* A = BIG ? e.work + nd * e.w_node : sm;  // n x ap, symmetric
  double* Vt = A + ((n * ap + 1) & ~1);  // n x vp_pitch, rows = eigenvectors (V transposed)
  double* cs = BIG ? sm : Vt + n * vp_pitch;  // [half]
  double* sn = cs + half;
  double* tt = sn + half;
  int* pp = (int*)(tt + half);     // [half]
  int* qq = pp + half;
  unsigned short* blk = (unsigned short*)(qq + half);  // [nblk] packed (bi, bj), bi <= bj
  __shared__ double red[2];
  const int tid = threadIdx.x;

  const double* S = e.S + nd * e.s_node;
  for (int x = tid; x < n * n; x += blockDim.x) {
    const int i = x / n, j = x - i * n;
    A[i * ap + j] = (i < K && j < K) ? S[i * K + j] : 0.0;
    Vt[i * vp_pitch + j] = (i == j) ? 1.0 : 0.0;
  }
  const int tpp = max(1, (int)blockDim.x / half);  // threads per rotation pair in the V update
  const int vk = tid / tpp, vsub = tid - vk * tpp;
  for (int x = tid; x < nblk; x += blockDim.x) {
    int bi = 0, rem = x;
    while (rem >= half - bi) { rem -= half - bi; ++bi; }
    blk[x] = (unsigned short)((bi << 8) | (bi + rem));
  }
  __syncthreads();
  // symmetry check (kernels.py:46-50), then symmetrise as eigh((S + S^T)/2)
  double asym = 0.0, amax = 0.0;
  for (int x = tid; x < K * K; x += blockDim.x) {
    const int i = x / K, j = x - i * K;
    asym = fmax(asym, fabs(A[i * ap + j] - A[j * ap + i]));
    amax = fmax(amax, fabs(A[i * ap + j]));
    if (!isfinite(A[i * ap + j])) amax = INFINITY;  // fmax drops NaN: make it visible
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    asym = fmax(asym, __shfl_xor_sync(0xffffffffu, asym, o));
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  }
  if (tid == 0) { red[0] = 0.0; red[1] = 0.0; }
  __syncthreads();
  if ((tid & 31) == 0) {
    atomicMax((unsigned long long*)&red[0], __double_as_longlong(asym));  // non-negative doubles order as ints
    atomicMax((unsigned long long*)&red[1], __double_as_longlong(amax));
  }
  __syncthreads();
  if (tid == 0 && e.status && red[0] > 1e-12 * fmax(1.0, red[1])) atomicOr(e.status, kEigStatusNotSymmetric);
  if (tid == 0 && e.status && !isfinite(red[1])) atomicOr(e.status, kEigStatusNonConverged);
  for (int x = tid; x < K * K; x += blockDim.x) {
    const int i = x / K, j = x - i * K;
    if (i < j) {
      const double s = 0.5 * (A[i * ap + j] + A[j * ap + i]);
      A[i * ap + j] = s;
      A[j * ap + i] = s;
    }
  }
  __syncthreads();

  const double tol = 2.220446049250313e-16 * (double)max(K, 8);
  bool converged = false;
  for (int sweep = 0; sweep < MAX_SWEEPS; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < n - 1; ++r) {
      if (tid < half) {
        int p = circle(tid, r, n), q = circle(n - 1 - tid, r, n);
        if (p > q) { const int t = p; p = q; q = t; }
        const double apq = A[p * ap + q];
        const double app = A[p * ap + p], aqq = A[q * ap + q];
        double c = 1.0, s = 0.0, t = 0.0;
        // relative (Demmel-Veselic) threshold tol * sqrt(a_pp a_qq), tol = K eps: the
        // eigenvalue perturbation from the neglected a_pq is O(tol^2) relative
        if (fabs(apq) > tol * sqrt(fabs(app)) * sqrt(fabs(aqq)) && fabs(apq) > 1e-300) {
          const double tau = (aqq - app) / (2.0 * apq);
          t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
          rotated = 1;
        }
        pp[tid] = p; qq[tid] = q; cs[tid] = c; sn[tid] = s; tt[tid] = t;
      }
      __syncthreads();
      // A' = J^T A J on the (pair_i, pair_j) 2x2 blocks, i <= j, mirrored
      for (int x = tid; x < nblk; x += blockDim.x) {
        const int code = blk[x];
        const int bi = code >> 8, bj = code & 255;
        const double si = sn[bi], sj = sn[bj];
        if (si == 0.0 && sj == 0.0) continue;
        const int pi = pp[bi], qi = qq[bi];
        if (bi == bj) {
          const double apq = A[pi * ap + qi], t = tt[bi];
          A[pi * ap + pi] -= t * apq;
          A[qi * ap + qi] += t * apq;
          A[pi * ap + qi] = 0.0;
          A[qi * ap + pi] = 0.0;
          continue;
        }
        const double ci = cs[bi], cj = cs[bj];
        const int pj = pp[bj], qj = qq[bj];
        const double x00 = A[pi * ap + pj], x01 = A[pi * ap + qj];
        const double x10 = A[qi * ap + pj], x11 = A[qi * ap + qj];
        const double y00 = ci * x00 - si * x10, y01 = ci * x01 - si * x11;
        const double y10 = si * x00 + ci * x10, y11 = si * x01 + ci * x11;
        const double z00 = cj * y00 - sj * y01, z01 = sj * y00 + cj * y01;
        const double z10 = cj * y10 - sj * y11, z11 = sj * y10 + cj * y11;
        A[pi * ap + pj] = z00; A[pj * ap + pi] = z00;
        A[pi * ap + qj] = z01; A[qj * ap + pi] = z01;
        A[qi * ap + pj] = z10; A[pj * ap + qi] = z10;
        A[qi * ap + qj] = z11; A[qj * ap + qi] = z11;
      }
      // V <- V J: rotate rows p, q of V^T, two columns per thread-iteration (16-byte)
      if (vk < half) {
        const double s = sn[vk];
        if (s != 0.0) {
          const double c = cs[vk];
          double2* vp = reinterpret_cast<double2*>(Vt + pp[vk] * vp_pitch);
          double2* vq = reinterpret_cast<double2*>(Vt + qq[vk] * vp_pitch);
          for (int i = vsub; i < n / 2; i += tpp) {
            const double2 a0 = vp[i], b0 = vq[i];
            vp[i] = make_double2(c * a0.x - s * b0.x, c * a0.y - s * b0.y);
            vq[i] = make_double2(s * a0.x + c * b0.x, s * a0.y + c * b0.y);
          }
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) {
      converged = true;
      break;
    }
  }
  if (!converged) {
    // The relative (Demmel-Veselic) test cannot be met when the small eigenvalues are
    // rounding noise of a numerically rank-deficient Gramian: accept the result if the
    // remaining off-diagonal mass is at the absolute noise level of the matrix.
    double off = 0.0, dmax = 0.0;
    for (int x = tid; x < K * K; x += blockDim.x) {
      const int i = x / K, j = x - i * K;
      if (i != j) off = fmax(off, fabs(A[i * ap + j]));
      else dmax = fmax(dmax, fabs(A[i * ap + i]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      off = fmax(off, __shfl_xor_sync(0xffffffffu, off, o));
      dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    if (tid == 0) { red[0] = 0.0; red[1] = 0.0; }
    __syncthreads();
    if ((tid & 31) == 0) {
      atomicMax((unsigned long long*)&red[0], __double_as_longlong(off));
      atomicMax((unsigned long long*)&red[1], __double_as_longlong(dmax));
    }
    __syncthreads();
    if (tid == 0 && e.status && !(red[0] <= 64.0 * 2.220446049250313e-16 * K * red[1]))
      atomicOr(e.status, kEigStatusNonConverged);
  }

  // stable descending order by eigenvalue, clamp >= 0 (kernels.py:51-53)
  double* lam = e.lam + nd * e.l_node;
  double* Vo = e.V + nd * e.v_node;
  double* lsorted = cs;  // reuse (cs, sn, tt are contiguous: 3*half >= K doubles)
  int* perm = pp;        // pp, qq contiguous: 2*half >= K ints
  for (int i = tid; i < K; i += blockDim.x) {
    const double li = A[i * ap + i];
    int pos = 0;
    for (int j = 0; j < K; ++j) {
      const double lj = A[j * ap + j];
      pos += (lj > li) || (lj == li && j < i);
    }
    const double lc = fmax(li, 0.0);
    lam[pos] = lc;
    lsorted[pos] = lc;
    perm[pos] = i;
  }
  __syncthreads();
  for (int x = tid; x < K * K; x += blockDim.x) {
    const int row = x / K, pos = x - row * K;
    Vo[(long long)row * K + pos] = Vt[perm[pos] * vp_pitch + row];
  }
  __syncthreads();
  if (tid == 0 && e.rank) {
    int r = K;
    if (e.eps > 0.0) {
      const double budget = e.eps * e.eps * (e.eps_scale2 ? *e.eps_scale2 : 1.0) / e.n_nonroot;
      // tails[r] = sum_{i >= r} lam[i], accumulated from the end like numpy's cumsum (arith.py:83-84)
      double tail = 0.0;
      r = K;
      for (int i = K - 1; i >= 0; --i) {
        tail += lsorted[i];
        if (tail <= budget) r = i;
        else break;
      }
    }
    if (e.cap > 0) r = min(r, e.cap);
    r = max(1, min(r, K));
    e.rank[nd] = r;
  }
}

size_t smem_bytes(int K) {
  const int n = K + (K & 1);
  const int half = n / 2;
  const size_t mats = K > kEigMaxK ? 0 : (size_t)(n * (n + 1) + 1 + n * (n + 2));
  return (mats + 3 * half) * sizeof(double) + (size_t)2 * half * sizeof(int) +
         (size_t)(half * (half + 1) / 2) * sizeof(unsigned short) + 64;
}

bool g_attr = false;

}  // namespace

int g_eig_mode = 0;

int eig_batched(std::vector<EigProblem>& probs, cudaStream_t stream) {
  bool tri = g_eig_mode == 0;
  bool big = false;
  for (const auto& p : probs) {
    tri = tri && p.fallback != nullptr && (p.K <= kEigMaxK || p.work);
    big = big || p.K > kEigMaxK;
  }
  for (const auto& p : probs)
    if (p.K > kEigMaxK && (!p.work || p.K > kEigMaxKBig)) {
      set_error("eigensolver: K > 112 needs a global workspace (and K <= 512)");
      return kErrUnsupported;
    }
  (void)big;
  if (tri) HT_TRY(eig_tri_batched(probs, stream));
  else
    for (auto& p : probs) p.fallback = nullptr;
  // the Jacobi kernel serves the nodes the tridiagonal path flagged (or every node in
  // Jacobi mode); K > 112 runs the global-scratch variant
  if (!g_attr) {
    HT_CUDA_CHECK(cudaFuncSetAttribute(jacobi_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    HT_CUDA_CHECK(cudaFuncSetAttribute(jacobi_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    g_attr = true;
  }
  for (int pass = 0; pass < 2; ++pass) {
  const bool bigpass = pass == 1;
  std::vector<EigProblem> sel;
  for (const auto& p : probs)
    if ((p.K > kEigMaxK) == bigpass) sel.push_back(p);
  size_t i = 0;
  while (i < sel.size()) {
    EigBatch b;
    b.count = 0;
    int blocks = 0;
    size_t smem = 0;
    while (i < sel.size() && b.count < MAXD) {
      const EigProblem& p = sel[i++];
      if (p.nodes == 0) continue;
      if (p.K > kEigMaxKBig || p.K < 1) {
        set_error("eig_batched: K=" + std::to_string(p.K) + " outside the Jacobi path (K <= 512)");
        return kErrUnsupported;
      }
      b.begin[b.count] = blocks;
      blocks += p.nodes;
      smem = std::max(smem, smem_bytes(p.K));
      b.d[b.count++] = p;
    }
    if (b.count == 0) continue;
    b.begin[b.count] = blocks;
    double flops = 0, bytes = 0;
    for (int q = 0; q < b.count; ++q) {
      flops += 9.0 * b.d[q].nodes * (double)b.d[q].K * b.d[q].K * b.d[q].K;
      bytes += 24.0 * b.d[q].nodes * (double)b.d[q].K * b.d[q].K;
    }
    ProfToken tok = prof_begin(stream);
    if (bigpass) jacobi_kernel<true><<<blocks, ET, smem, stream>>>(b);
    else jacobi_kernel<false><<<blocks, ET, smem, stream>>>(b);
    HT_LAUNCH_CHECK();
    prof_end(tok, "jacobi_eig", stream, flops, bytes);
  }
  }
  return kOk;
}

}  // namespace ht
