#include <algorithm>

#include "misc.cuh"
#include "prof.cuh"

namespace ht {

namespace {

constexpr int MAXD = 64;

struct EmbedBatch {
  int count;
  int begin[MAXD + 1];
  EmbedDesc d[MAXD];
};

struct KronBatch {
  int count;
  int begin[MAXD + 1];
  KronDesc d[MAXD];
};

struct LeafBatch {
  int count;
  int begin[MAXD + 1];
  LeafApplyDesc d[MAXD];
};

template <typename B>
__device__ __forceinline__ int find(const B& b) {
  int di = 0;
  while (di + 1 < b.count && (int)blockIdx.x >= b.begin[di + 1]) ++di;
  return di;
}

// One warp per output row (i0, i1): the row's A segment, scaled C segment and zeros
// are written with coalesced stores; index arithmetic once per row, not per element.
__global__ void embed_kernel(const __grid_constant__ EmbedBatch b) {
  const int di = find(b);
  const EmbedDesc& e = b.d[di];
  const long long rows = (long long)e.D0 * e.D1;
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  const long long nw = (long long)(b.begin[di + 1] - b.begin[di]) * wpb;
  const bool vec = !((e.D2 | e.a2 | e.c2 | e.o2) & 1) &&
                   !((((uintptr_t)e.out) | ((uintptr_t)e.A) | ((uintptr_t)e.C)) & 15);
  for (long long r = (long long)(blockIdx.x - b.begin[di]) * wpb + (threadIdx.x >> 5); r < rows; r += nw) {
    const int i0 = (int)(r / e.D1), i1 = (int)(r - (long long)i0 * e.D1);
    double* o = e.out + r * e.D2;
    const bool ina = i0 < e.a0 && i1 < e.a1;
    const double* arow = e.A + ((long long)i0 * e.a1 + i1) * e.a2;
    const int j0 = i0 - e.o0, j1 = i1 - e.o1;
    const bool inc = j0 >= 0 && j1 >= 0 && j0 < e.c0 && j1 < e.c1;
    const double* crow = e.C + ((long long)j0 * e.c1 + j1) * e.c2;
    if (vec) {  // even extents and offsets: 16-byte pairs never straddle a segment edge
      for (int p = lane; 2 * p < e.D2; p += 32) {
        const int i2 = 2 * p, j2 = i2 - e.o2;
        double2 v = make_double2(0.0, 0.0);
        if (ina && i2 < e.a2) {
          v = reinterpret_cast<const double2*>(arow)[p];
        } else if (inc && j2 >= 0 && j2 < e.c2) {
          const double2 c = reinterpret_cast<const double2*>(crow)[j2 >> 1];
          v = make_double2(e.alpha_c * c.x, e.alpha_c * c.y);
        }
        reinterpret_cast<double2*>(o)[p] = v;
      }
      continue;
    }
    for (int i2 = lane; i2 < e.D2; i2 += 32) {
      double v = 0.0;
      const int j2 = i2 - e.o2;
      if (ina && i2 < e.a2) v = arow[i2];
      else if (inc && j2 >= 0 && j2 < e.c2) v = e.alpha_c * crow[j2];
      o[i2] = v;
    }
  }
}

__global__ void kron_kernel(const __grid_constant__ KronBatch b) {
  const int di = find(b);
  const KronDesc& k = b.d[di];
  const long long D1 = (long long)k.kq * k.kj, D2 = (long long)k.kr * k.kl;
  const long long total = (long long)k.kp * k.ki * D1 * D2;
  const long long stride = (long long)(b.begin[di + 1] - b.begin[di]) * blockDim.x;
  for (long long x = (long long)(blockIdx.x - b.begin[di]) * blockDim.x + threadIdx.x; x < total; x += stride) {
    const long long i2 = x % D2, rr = x / D2;
    const long long i1 = rr % D1, i0 = rr / D1;
    const int p = (int)(i0 / k.ki), i = (int)(i0 % k.ki);
    const int q = (int)(i1 / k.kj), j = (int)(i1 % k.kj);
    const int r = (int)(i2 / k.kl), l = (int)(i2 % k.kl);
    k.out[x] = k.H[((long long)p * k.kq + q) * k.kr + r] * k.B[((long long)i * k.kj + j) * k.kl + l];
  }
}

__global__ void leaf_apply_kernel(const __grid_constant__ LeafBatch b) {
  const int di = find(b);
  const LeafApplyDesc& e = b.d[di];
  const long long total = (long long)e.n_out * e.k;
  const long long stride = (long long)(b.begin[di + 1] - b.begin[di]) * blockDim.x;
  for (long long x = (long long)(blockIdx.x - b.begin[di]) * blockDim.x + threadIdx.x; x < total; x += stride) {
    const int i = (int)(x / e.k), l = (int)(x % e.k);
    double v;
    if (e.kind == 1) {
      v = e.vals[i] * e.U[(long long)i * e.k + l];
    } else {
      v = 0.0;
      for (int z = e.indptr[i]; z < e.indptr[i + 1]; ++z) v = fma(e.vals[z], e.U[(long long)e.indices[z] * e.k + l], v);
    }
    e.V[(long long)i * e.ldv + e.col0 + l] = v;
  }
}

__global__ void scale_kernel(const double* x, double* y, long long n, double a) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = a * x[i];
}

__global__ void dot_kernel(const double* a, const double* b, long long n, double* out) {
  __shared__ double part[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s = fma(a[i], b[i], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) *out = v;
  }
}

int blocks_for(long long total) { return (int)std::max<long long>(1, std::min<long long>(ceil_div(total, 256), 2048)); }

}  // namespace

int embed_batched(const std::vector<EmbedDesc>& descs, cudaStream_t stream) {
  size_t i = 0;
  while (i < descs.size()) {
    EmbedBatch b;
    b.count = 0;
    int blocks = 0;
    double bytes = 0.0;
    while (i < descs.size() && b.count < MAXD) {
      const EmbedDesc& d = descs[i++];
      const long long total = (long long)d.D0 * d.D1 * d.D2;
      if (total == 0) continue;
      b.begin[b.count] = blocks;
      blocks += (int)std::max<long long>(1, std::min<long long>(ceil_div((long long)d.D0 * d.D1, 8), 2048));
      bytes += 8.0 * ((double)total + (double)d.a0 * d.a1 * d.a2 + (double)d.c0 * d.c1 * d.c2);
      b.d[b.count++] = d;
    }
    if (!b.count) continue;
    b.begin[b.count] = blocks;
    ProfToken tok = prof_begin(stream);
    embed_kernel<<<blocks, 256, 0, stream>>>(b);
    HT_LAUNCH_CHECK();
    prof_end(tok, "embed", stream, 0.0, bytes);
  }
  return kOk;
}

int kron_batched(const std::vector<KronDesc>& descs, cudaStream_t stream) {
  size_t i = 0;
  while (i < descs.size()) {
    KronBatch b;
    b.count = 0;
    int blocks = 0;
    while (i < descs.size() && b.count < MAXD) {
      const KronDesc& d = descs[i++];
      const long long total = (long long)d.kp * d.kq * d.kr * d.ki * d.kj * d.kl;
      if (total == 0) continue;
      b.begin[b.count] = blocks;
      blocks += blocks_for(total);
      b.d[b.count++] = d;
    }
    if (!b.count) continue;
    b.begin[b.count] = blocks;
    ProfToken tok = prof_begin(stream);
    kron_kernel<<<blocks, 256, 0, stream>>>(b);
    HT_LAUNCH_CHECK();
    prof_end(tok, "kron", stream, 0.0, 0.0);
  }
  return kOk;
}

int leaf_apply_batched(const std::vector<LeafApplyDesc>& descs, cudaStream_t stream) {
  size_t i = 0;
  while (i < descs.size()) {
    LeafBatch b;
    b.count = 0;
    int blocks = 0;
    while (i < descs.size() && b.count < MAXD) {
      const LeafApplyDesc& d = descs[i++];
      const long long total = (long long)d.n_out * d.k;
      if (total == 0) continue;
      b.begin[b.count] = blocks;
      blocks += blocks_for(total);
      b.d[b.count++] = d;
    }
    if (!b.count) continue;
    b.begin[b.count] = blocks;
    ProfToken tok = prof_begin(stream);
    leaf_apply_kernel<<<blocks, 256, 0, stream>>>(b);
    HT_LAUNCH_CHECK();
    prof_end(tok, "leaf_apply", stream, 0.0, 0.0);
  }
  return kOk;
}

__global__ void copy2d_kernel(Copy2dDesc d) {
  const long long total = (long long)d.nodes * d.rows * d.cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    // column-fastest for row-major destinations, row-fastest otherwise (coalesced writes)
    long long nd, r, c;
    if (d.d_c == 1) {
      c = e % d.cols;
      r = (e / d.cols) % d.rows;
      nd = e / ((long long)d.cols * d.rows);
    } else {
      r = e % d.rows;
      c = (e / d.rows) % d.cols;
      nd = e / ((long long)d.cols * d.rows);
    }
    d.dst[nd * d.d_node + r * d.d_r + c * d.d_c] = d.src[nd * d.s_node + r * d.s_r + c * d.s_c];
  }
}

int copy2d_batched(const std::vector<Copy2dDesc>& descs, cudaStream_t stream) {
  for (const auto& d : descs) {
    const long long total = (long long)d.nodes * d.rows * d.cols;
    if (total <= 0) continue;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
    ProfToken tok = prof_begin(stream);
    copy2d_kernel<<<blocks, 256, 0, stream>>>(d);
    HT_LAUNCH_CHECK();
    prof_end(tok, "copy2d", stream, 0.0, 16.0 * total);
  }
  return kOk;
}

int scale_copy(const double* x, double* y, long long n, double alpha, cudaStream_t stream) {
  if (n <= 0) return kOk;
  ProfToken tok = prof_begin(stream);
  scale_kernel<<<blocks_for(n), 256, 0, stream>>>(x, y, n, alpha);
  HT_LAUNCH_CHECK();
  prof_end(tok, "scale", stream, 0.0, 16.0 * n);
  return kOk;
}

__global__ void identity_kernel(double* p, long long node_stride, int K, const int* active) {
  if (active && *active == 0) return;
  double* q = p + (long long)blockIdx.y * node_stride;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K * K; e += gridDim.x * blockDim.x)
    q[e] = (e / K == e % K) ? 1.0 : 0.0;
}

int identity_batched(double* p, long long node_stride, int K, int nodes, const int* active, cudaStream_t stream) {
  if (nodes <= 0 || K <= 0) return kOk;
  identity_kernel<<<dim3((K * K + 255) / 256, nodes), 256, 0, stream>>>(p, node_stride, K, active);
  HT_LAUNCH_CHECK();
  return kOk;
}

int dot(const double* a, const double* b, long long n, double* out, cudaStream_t stream) {
  ProfToken tok = prof_begin(stream);
  dot_kernel<<<1, 1024, 0, stream>>>(a, b, n, out);
  HT_LAUNCH_CHECK();
  prof_end(tok, "dot", stream, 2.0 * n, 16.0 * n);
  return kOk;
}

}  // namespace ht

namespace ht {
namespace {
constexpr int kEvalThreads = 256;

__global__ void __launch_bounds__(kEvalThreads) evaluate_kernel(const __grid_constant__ EvalTree T,
                                                                const long long* __restrict__ idx,
                                                                double* __restrict__ out) {
  extern __shared__ double stk[];  // [depth + 2][kmax]
  const long long b = blockIdx.x;
  const long long* ib = idx + b * T.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int top = 0;  // number of rows on the stack
  double result = 0.0;
  for (int q = 0; q < T.nn; ++q) {
    const int t = T.post[q];
    if (T.son1[t] < 0) {  // leaf: row U[i_mu, :], or the weighted row w_mu^T U
      const int mu = T.dim[t];
      const int k = T.k[t];
      const double* w = T.w[mu];
      if (w) {
        const double* U = T.p[t];
        const int n = T.n[mu];
        for (int j = tid; j < k; j += kEvalThreads) {
          double s = 0.0;
          for (int i = 0; i < n; ++i) s = fma(w[i], U[(long long)i * k + j], s);
          stk[top * T.kmax + j] = s;
        }
      } else {
        const long long i = ib[mu];
        for (int j = tid; j < k; j += kEvalThreads) stk[top * T.kmax + j] = T.p[t][i * k + j];
      }
      ++top;
      __syncthreads();
      continue;
    }
    const int k1 = T.k[T.son1[t]], k2 = T.k[T.son2[t]];
    const double* r1 = stk + (top - 2) * T.kmax;
    const double* r2 = stk + (top - 1) * T.kmax;
    const double* Bt = T.p[t];
    if (t == 0) {  // root: r1^T B_D r2, one CTA-wide reduction
      double acc = 0.0;
      for (int e = tid; e < k1 * k2; e += kEvalThreads) acc = fma(r1[e / k2] * Bt[e], r2[e % k2], acc);
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      __shared__ double red[kEvalThreads / 32];
      if (lane == 0) red[warp] = acc;
      __syncthreads();
      if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kEvalThreads / 32; ++w) s += red[w];
        result = s;
      }
      break;
    }
    // inner: row[i] = sum_{j,l} B[i,j,l] r1[j] r2[l]; warp per i, lanes along l (coalesced)
    const int kt = T.k[t];
    double* row = stk + top * T.kmax;  // written above the operands, then moved down
    for (int i = warp; i < kt; i += kEvalThreads / 32) {
      const double* Bi = Bt + (long long)i * k1 * k2;
      double acc = 0.0;
      for (int j = 0; j < k1; ++j) {
        double s = 0.0;
        for (int l = lane; l < k2; l += 32) s = fma(Bi[j * k2 + l], r2[l], s);
        acc = fma(r1[j], s, acc);
      }
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) row[i] = acc;
    }
    __syncthreads();
    double* dst = stk + (top - 2) * T.kmax;
    for (int i = tid; i < kt; i += kEvalThreads) dst[i] = row[i];
    __syncthreads();
    top -= 1;
  }
  if (tid == 0) out[b] = result;
}
}  // namespace

int evaluate_entries(const EvalTree& T, const long long* idx, long long B, double* out, cudaStream_t s) {
  if (B <= 0) return kOk;
  const size_t smem = sizeof(double) * (size_t)(T.depth + 3) * T.kmax;
  if (smem > 200 * 1024) {
    set_error("evaluate_entries: ranks too large for the shared-memory row stack");
    return kErrUnsupported;
  }
  static bool attr = false;
  if (!attr) {
    HT_CUDA_CHECK(cudaFuncSetAttribute(evaluate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  ProfToken tok = prof_begin(s);
  evaluate_kernel<<<(unsigned)B, kEvalThreads, smem, s>>>(T, idx, out);
  HT_LAUNCH_CHECK();
  double flops = 0;
  prof_end(tok, "evaluate", s, flops, 0.0);
  return kOk;
}
}  // namespace ht
