#include <algorithm>
#include <type_traits>

#include "misc.cuh"
#include "prof.cuh"

namespace ht {

namespace {

constexpr int MAXD = 64;

constexpr int kEmbedMaxD = 128;

// Unsigned division by a per-descriptor constant (n < 2^31): q = (umulhi(n, m) + n) >> s.
struct FastDiv {
  unsigned m, s, d;
};

struct EmbedBatch {
  int count;
  int begin[kEmbedMaxD + 1];  // prefix sums of the descriptors' CTA counts
  FastDiv row[kEmbedMaxD];    // units per output row (D2 / W)
  FastDiv d1[kEmbedMaxD];     // D1
  EmbedDesc d[kEmbedMaxD];
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

// Block embedding of add (arith.py:173-192).  The output of a node is one flat run of
// W-double units (W = 2: 16-byte pairs when every extent / offset is even and the bases
// are 16-byte aligned; W = 1 otherwise); each CTA owns a contiguous chunk of one
// descriptor's units and every thread issues the loads of kEmbedU units (A or scaled C
// segment, nothing for the structural zeros -- three quarters of an inner node) before
// any store, so stores are fully coalesced and ~kEmbedU loads per thread are in flight.
constexpr int kEmbedThreads = 256;
constexpr int kEmbedU = 8;  // units per thread per CTA chunk
constexpr int kEmbedChunk = kEmbedThreads * kEmbedU;

__device__ __forceinline__ unsigned fdiv(unsigned n, const FastDiv& f) {
  return (__umulhi(n, f.m) + n) >> f.s;
}

template <int W>
__global__ void __launch_bounds__(kEmbedThreads) embed_kernel(const __grid_constant__ EmbedBatch b) {
  using V = typename std::conditional<W == 2, double2, double>::type;
  int lo = 0, hi = b.count - 1;  // descriptor of this CTA: begin[lo] <= blockIdx.x < begin[lo + 1]
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((int)blockIdx.x >= b.begin[mid]) lo = mid;
    else hi = mid - 1;
  }
  const EmbedDesc& e = b.d[lo];
  const FastDiv fr = b.row[lo], f1 = b.d1[lo];
  const unsigned units = (unsigned)(((long long)e.D0 * e.D1 * e.D2) / W);
  const unsigned u0 = (unsigned)(blockIdx.x - b.begin[lo]) * kEmbedChunk + threadIdx.x;
  const double sc = e.alpha_c;
  V v[kEmbedU];
#pragma unroll
  for (int k = 0; k < kEmbedU; ++k) {
    const unsigned u = u0 + k * kEmbedThreads;
    if constexpr (W == 2) v[k] = make_double2(0.0, 0.0);
    else v[k] = 0.0;
    if (u < units) {
      const unsigned row = fdiv(u, fr);
      const int i2 = (int)(u - row * fr.d) * W;
      const int i0 = (int)fdiv(row, f1), i1 = (int)(row - (unsigned)i0 * f1.d);
      if (i0 < e.a0 && i1 < e.a1 && i2 < e.a2) {
        v[k] = *reinterpret_cast<const V*>(e.A + ((long long)i0 * e.a1 + i1) * e.a2 + i2);
      } else {
        const int j0 = i0 - e.o0, j1 = i1 - e.o1, j2 = i2 - e.o2;
        if (j0 >= 0 && j1 >= 0 && j2 >= 0 && j0 < e.c0 && j1 < e.c1 && j2 < e.c2) {
          const V w = *reinterpret_cast<const V*>(e.C + ((long long)j0 * e.c1 + j1) * e.c2 + j2);
          if constexpr (W == 2) v[k] = make_double2(sc * w.x, sc * w.y);
          else v[k] = sc * w;
        }
      }
    }
  }
  V* out = reinterpret_cast<V*>(e.out);
#pragma unroll
  for (int k = 0; k < kEmbedU; ++k) {
    const unsigned u = u0 + k * kEmbedThreads;
    if (u < units) __stcs(out + u, v[k]);
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

struct KronFactorBatch {
  int count;
  int begin[MAXD + 1];
  KronFactorDesc d[MAXD];
};

__global__ void kron_factor_kernel(const __grid_constant__ KronFactorBatch b) {
  const int di = find(b);
  const KronFactorDesc& k = b.d[di];
  const long long total = (long long)k.ra * k.rc * k.ko * k.ks;
  const long long stride = (long long)(b.begin[di + 1] - b.begin[di]) * blockDim.x;
  for (long long x = (long long)(blockIdx.x - b.begin[di]) * blockDim.x + threadIdx.x; x < total; x += stride) {
    const int j = (int)(x % k.ks);
    long long r = x / k.ks;
    const int J = (int)(r % k.ko);
    r /= k.ko;
    const int c = (int)(r % k.rc), a = (int)(r / k.rc);
    const double* h = k.H + ((long long)a * k.rb) * k.rc + c;
    const double* row = k.R + (long long)J * k.ldr + j;
    double v = 0.0;
    for (int q = 0; q < k.rb; ++q) v = fma(h[(long long)q * k.rc], row[(long long)q * k.ks], v);
    k.E[x] = v;
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

namespace {
FastDiv make_fastdiv(unsigned d) {
  FastDiv f;
  f.d = d;
  unsigned s = 0;
  while ((1ull << s) < d) ++s;
  f.s = s;
  f.m = (unsigned)(((1ull << 32) * ((1ull << s) - d)) / d + 1);
  return f;
}
}  // namespace

int embed_batched(const std::vector<EmbedDesc>& descs, cudaStream_t stream) {
  // W = 2 launches for the 16-byte-pair descriptors, W = 1 for the rest
  for (int W : {2, 1}) {
    size_t i = 0;
    while (i < descs.size()) {
      EmbedBatch b;
      b.count = 0;
      b.begin[0] = 0;
      double bytes = 0.0;
      while (i < descs.size() && b.count < kEmbedMaxD) {
        const EmbedDesc& d = descs[i++];
        const long long n = (long long)d.D0 * d.D1 * d.D2;
        if (n == 0) continue;
        const bool vec = !((d.D2 | d.a2 | d.c2 | d.o2) & 1) &&
                         !((((uintptr_t)d.out) | ((uintptr_t)d.A) | ((uintptr_t)d.C)) & 15);
        if ((W == 2) != vec) continue;
        if (n / W >= (1ll << 31)) {
          set_error("add: node array too large for the embedding kernel");
          return kErrShape;
        }
        b.row[b.count] = make_fastdiv((unsigned)(d.D2 / W));
        b.d1[b.count] = make_fastdiv((unsigned)d.D1);
        b.begin[b.count + 1] = b.begin[b.count] + ceil_div(n / W, kEmbedChunk);
        bytes += 8.0 * ((double)n + (double)d.a0 * d.a1 * d.a2 + (double)d.c0 * d.c1 * d.c2);
        b.d[b.count++] = d;
      }
      if (!b.count) continue;
      ProfToken tok = prof_begin(stream);
      if (W == 2) embed_kernel<2><<<b.begin[b.count], kEmbedThreads, 0, stream>>>(b);
      else embed_kernel<1><<<b.begin[b.count], kEmbedThreads, 0, stream>>>(b);
      HT_LAUNCH_CHECK();
      prof_end(tok, "embed", stream, 0.0, bytes);
    }
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

struct ZeroBatch {
  int count;
  int begin[MAXD + 1];
  ZeroDesc d[MAXD];
};

__global__ void zero_kernel(const __grid_constant__ ZeroBatch b) {
  const int di = find(b);
  const ZeroDesc& z = b.d[di];
  const long long stride = (long long)(b.begin[di + 1] - b.begin[di]) * blockDim.x;
  long long x = (long long)(blockIdx.x - b.begin[di]) * blockDim.x + threadIdx.x;
  if (!(reinterpret_cast<uintptr_t>(z.p) & 15)) {  // 16-byte stores over the aligned body
    double2* p2 = reinterpret_cast<double2*>(z.p);
    const long long n2 = z.count / 2;
    for (long long i = x; i < n2; i += stride) p2[i] = make_double2(0.0, 0.0);
    if ((z.count & 1) && x == 0) z.p[z.count - 1] = 0.0;
  } else {
    for (long long i = x; i < z.count; i += stride) z.p[i] = 0.0;
  }
}

int zero_batched(const std::vector<ZeroDesc>& descs, cudaStream_t stream) {
  size_t i = 0;
  while (i < descs.size()) {
    ZeroBatch b;
    b.count = 0;
    int blocks = 0;
    double bytes = 0;
    while (i < descs.size() && b.count < MAXD) {
      const ZeroDesc& d = descs[i++];
      if (d.count <= 0) continue;
      b.begin[b.count] = blocks;
      blocks += blocks_for(d.count / 8);
      b.d[b.count++] = d;
      bytes += 8.0 * d.count;
    }
    if (!b.count) continue;
    b.begin[b.count] = blocks;
    ProfToken tok = prof_begin(stream);
    zero_kernel<<<blocks, 256, 0, stream>>>(b);
    HT_LAUNCH_CHECK();
    prof_end(tok, "zero_fill", stream, 0.0, bytes);
  }
  return kOk;
}

struct RootBlocks {
  int count;
  RootBlockDesc d[16];
};

__global__ void root_blocks_kernel(double* out, int cols, const __grid_constant__ RootBlocks b) {
  const RootBlockDesc& q = b.d[blockIdx.y];
  const int total = q.r * q.c;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int i = e / q.c, j = e - i * q.c;
    out[(long long)(q.ro + i) * cols + q.co + j] = q.alpha * q.B[e];
  }
}

int root_blocks(double* out, int cols, const std::vector<RootBlockDesc>& blocks, cudaStream_t stream) {
  size_t i = 0;
  while (i < blocks.size()) {
    RootBlocks b;
    b.count = 0;
    int mx = 1;
    while (i < blocks.size() && b.count < 16) {
      mx = std::max(mx, blocks[i].r * blocks[i].c);
      b.d[b.count++] = blocks[i++];
    }
    ProfToken tok = prof_begin(stream);
    root_blocks_kernel<<<dim3(std::min((mx + 255) / 256, 64), b.count), 256, 0, stream>>>(out, cols, b);
    HT_LAUNCH_CHECK();
    prof_end(tok, "root_blocks", stream, 0.0, 0.0);
  }
  return kOk;
}

int kron_factor_batched(const std::vector<KronFactorDesc>& descs, cudaStream_t stream) {
  size_t i = 0;
  while (i < descs.size()) {
    KronFactorBatch b;
    b.count = 0;
    int blocks = 0;
    while (i < descs.size() && b.count < MAXD) {
      const KronFactorDesc& d = descs[i++];
      const long long total = (long long)d.ra * d.rc * d.ko * d.ks;
      if (total == 0) continue;
      b.begin[b.count] = blocks;
      blocks += blocks_for(total);
      b.d[b.count++] = d;
    }
    if (!b.count) continue;
    b.begin[b.count] = blocks;
    ProfToken tok = prof_begin(stream);
    kron_factor_kernel<<<blocks, 256, 0, stream>>>(b);
    HT_LAUNCH_CHECK();
    prof_end(tok, "kron_factor", stream, 0.0, 0.0);
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
  ProfToken tok = prof_begin(stream);
  identity_kernel<<<dim3((K * K + 255) / 256, nodes), 256, 0, stream>>>(p, node_stride, K, active);
  HT_LAUNCH_CHECK();
  prof_end(tok, "identity", stream, 0.0, 0.0);
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
