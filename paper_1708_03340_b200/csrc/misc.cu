#include <algorithm>

#include "misc.cuh"
#include "prof.cuh"

namespace ht {

namespace {

constexpr int MAXD = 64;

struct EmbedBatch {
  int count;
  long long row_begin[MAXD + 1];  // prefix sums of the descriptors' output rows
  unsigned char vec[MAXD];        // even extents / offsets, 16-byte aligned: pair copies
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

// Block embedding of add.  Output rows (i0, i1) of D2 values, all descriptors' rows in
// one global row space; each warp owns a contiguous run of rows (descriptor lookup once
// per run) and works on four rows at a time: every lane issues the loads of all four
// rows (A or scaled C segments; pure-zero rows -- half of every inner node -- load
// nothing) before any store, so ~8 16-byte loads per lane are in flight.
constexpr int kEmbedThreads = 256;
constexpr int kEmbedU = 4;  // rows per warp step

struct RowSrc {
  const double* a;  // A row segment -> output [0, ahi), or null
  const double* c;  // C row segment (indexed from clo) -> output [clo, chi), or null
  int ahi, clo, chi;
  // value pair (i2, i2 + 1) of the output row: exactly one source or zero
  __device__ __forceinline__ bool from_a(int i2) const { return a && i2 < ahi; }
  __device__ __forceinline__ bool from_c(int i2) const { return c && i2 >= clo && i2 < chi; }
};

// (a leaf row has both: U = [U_a, U_c]; an inner row at most one block)
__device__ __forceinline__ RowSrc row_src(const EmbedDesc& e, int i0, int i1) {
  RowSrc s{nullptr, nullptr, 0, 0, 0};
  if (i0 < e.a0 && i1 < e.a1) {
    s.a = e.A + ((long long)i0 * e.a1 + i1) * e.a2;
    s.ahi = e.a2;
  }
  const int j0 = i0 - e.o0, j1 = i1 - e.o1;
  if (j0 >= 0 && j1 >= 0 && j0 < e.c0 && j1 < e.c1) {
    s.c = e.C + ((long long)j0 * e.c1 + j1) * e.c2 - e.o2;
    s.clo = e.o2;
    s.chi = e.o2 + e.c2;
  }
  return s;
}

__global__ void __launch_bounds__(kEmbedThreads, 4) embed_kernel(const __grid_constant__ EmbedBatch b) {
  const int lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * (kEmbedThreads / 32) + (threadIdx.x >> 5);
  const long long nwarps = (long long)gridDim.x * (kEmbedThreads / 32);
  const long long total = b.row_begin[b.count];
  long long r = total * gw / nwarps;
  const long long r_end = total * (gw + 1) / nwarps;
  int di = 0;
  while (di + 1 < b.count && r >= b.row_begin[di + 1]) ++di;
  while (r < r_end) {
    const EmbedDesc& e = b.d[di];
    const long long rd_end = min(r_end, b.row_begin[di + 1]);  // this descriptor's part of the run
    const long long base = b.row_begin[di];
    const bool vec = b.vec[di];
    const int D2 = e.D2;
    // (i0, i1) of the run's first row (one division per run), then stepped per row
    int i0 = (int)((r - base) / e.D1), i1 = (int)((r - base) - (long long)i0 * e.D1);
    auto step = [&]() {
      if (++i1 == e.D1) {
        i1 = 0;
        ++i0;
      }
    };
    if (vec) {
      const int P2 = D2 >> 1;  // 16-byte pairs per row
      for (; r < rd_end; r += kEmbedU) {
        double2 v[kEmbedU][2];  // only the loaded pairs stay live into the store phase
        const double sc = e.alpha_c;
        const int s0 = i0, s1 = i1;  // first row of this step (the long-row path restarts from it)
#pragma unroll
        for (int u = 0; u < kEmbedU; ++u) {
          const RowSrc src = r + u < rd_end ? row_src(e, i0, i1) : RowSrc{nullptr, nullptr, 0, 0, 0};
          step();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int pr = lane + 32 * h, i2 = 2 * pr;
            v[u][h] = make_double2(0.0, 0.0);
            if (pr < P2) {
              if (src.from_a(i2)) {
                v[u][h] = *reinterpret_cast<const double2*>(src.a + i2);
              } else if (src.from_c(i2)) {
                const double2 w = *reinterpret_cast<const double2*>(src.c + i2);
                v[u][h] = make_double2(sc * w.x, sc * w.y);
              }
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kEmbedU; ++u) {
          if (r + u >= rd_end) break;
          double2* o = reinterpret_cast<double2*>(e.out + (r + u - base) * D2);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int pr = lane + 32 * h;
            if (pr < P2) o[pr] = v[u][h];
          }
          if (P2 > 64) {  // rows longer than 128 values
            int q0 = s0, q1 = s1 + u;
            while (q1 >= e.D1) {
              q1 -= e.D1;
              ++q0;
            }
            const RowSrc src = row_src(e, q0, q1);
            for (int pr = lane + 64; pr < P2; pr += 32) {
              const int i2 = 2 * pr;
              double2 w = make_double2(0.0, 0.0);
              if (src.from_a(i2)) {
                w = *reinterpret_cast<const double2*>(src.a + i2);
              } else if (src.from_c(i2)) {
                w = *reinterpret_cast<const double2*>(src.c + i2);
                w.x *= sc;
                w.y *= sc;
              }
              o[pr] = w;
            }
          }
        }
      }
    } else {
      for (; r < rd_end; ++r, step()) {
        const RowSrc sr = row_src(e, i0, i1);
        double* o = e.out + (r - base) * D2;
        for (int i2 = lane; i2 < D2; i2 += 32)
          o[i2] = sr.from_a(i2) ? sr.a[i2] : (sr.from_c(i2) ? e.alpha_c * sr.c[i2] : 0.0);
      }
    }
    r = rd_end;  // (the four-row steps may overshoot the descriptor's last row)
    ++di;
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
    b.row_begin[0] = 0;
    double bytes = 0.0;
    while (i < descs.size() && b.count < MAXD) {
      const EmbedDesc& d = descs[i++];
      const long long rows = (long long)d.D0 * d.D1;
      if (rows * d.D2 == 0) continue;
      b.vec[b.count] = !((d.D2 | d.a2 | d.c2 | d.o2) & 1) &&
                       !((((uintptr_t)d.out) | ((uintptr_t)d.A) | ((uintptr_t)d.C)) & 15);
      b.row_begin[b.count + 1] = b.row_begin[b.count] + rows;
      bytes += 8.0 * ((double)rows * d.D2 + (double)d.a0 * d.a1 * d.a2 + (double)d.c0 * d.c1 * d.c2);
      b.d[b.count++] = d;
    }
    if (!b.count) continue;
    // enough warps to keep ~8 loads per lane in flight on every SM, not more than rows / 4
    const long long rows = b.row_begin[b.count];
    const int blocks = (int)std::max<long long>(1, std::min<long long>(148LL * 8, ceil_div(rows, 4 * 8)));
    ProfToken tok = prof_begin(stream);
    embed_kernel<<<blocks, kEmbedThreads, 0, stream>>>(b);
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
