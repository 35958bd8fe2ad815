// Shared definitions for the B200 (sm_100a) HT-arithmetic kernels.
//
// All arithmetic is IEEE float64.  On sm_100a the only FP64 tensor-core path is
// mma.sync DMMA (tcgen05 has no kind::f64); DMMA and DFMA both measure ~37 TF/s
// on this pool's B200s (profiles/r01_fp64_peak_microbench.jsonl).
#pragma once
#include <cstdio>

#include <cuda_runtime.h>
#include <cstdint>
#include <string>

namespace ht {

constexpr int kWarp = 32;

// Status codes shared with include/ht_b200.h.
enum Status : int {
  kOk = 0,
  kErrShape = 1,
  kErrNotOrthogonal = 2,
  kErrNonConverged = 3,
  kErrCuda = 4,
  kErrNotSymmetric = 5,
  kErrArgument = 6,
  kErrUnsupported = 7,
};

void set_error(const std::string& msg);
const char* last_error();

#define HT_CUDA_CHECK(expr)                                                     \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      ::ht::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));      \
      return ::ht::kErrCuda;                                                    \
    }                                                                           \
  } while (0)

// HT_SYNC_CHECK=1 (debugging): every launch check also synchronises the device, so a
// faulting kernel is reported at its own launch site
extern const int g_sync_check;
int debug_probe();  // HT_SYNC_CHECK=3: a fixed long-reduction GEMM after every launch

#define HT_LAUNCH_CHECK()                                                       \
  do {                                                                          \
    cudaError_t _e = cudaGetLastError();                                        \
    if (_e == cudaSuccess && ::ht::g_sync_check) {                              \
      _e = cudaDeviceSynchronize();                                             \
      if (::ht::g_sync_check > 1) fprintf(stderr, "[launch] %s:%d -> %d\n", __FILE__, __LINE__, (int)_e); \
      if (_e == cudaSuccess && ::ht::g_sync_check > 2 && ::ht::debug_probe() != 0) \
        fprintf(stderr, "[probe] FAILED after %s:%d\n", __FILE__, __LINE__);    \
    }                                                                           \
    if (_e != cudaSuccess) {                                                    \
      ::ht::set_error(std::string("kernel launch (") + __FILE__ + ":" +         \
                      std::to_string(__LINE__) + "): " + cudaGetErrorString(_e)); \
      return ::ht::kErrCuda;                                                    \
    }                                                                           \
  } while (0)

#define HT_TRY(expr)                        \
  do {                                      \
    int _s = (expr);                        \
    if (_s != ::ht::kOk) return _s;         \
  } while (0)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// m16n8kK f64 (K = 16, 8, 4), verified on sm_100a by tools/mma_layout.cu.  With
// g = lane/4, t = lane%4:  a[i] = A[g + 8*(i&1)][t + 4*(i>>1)],  b[i] = B[t + 4i][g],
// c = {C[g][2t], C[g][2t+1], C[g+8][2t], C[g+8][2t+1]}.
__device__ __forceinline__ void dmma_16x8x16(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
// predicated form: no-op when !p (branch-free skipping of structurally zero blocks)
__device__ __forceinline__ void dmma_16x8x16_if(bool p, double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %16, 0;\n"
      " @q mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n}\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]), "r"((int)p));
}
__device__ __forceinline__ void dmma_16x8x8(double (&c)[4], const double* a, const double* b) {
  asm("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], const double* a, const double* b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}


// ---- mbarrier + bulk-async (TMA engine) copy primitives (sm_90+/sm_100a) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* b, unsigned parity) {
  unsigned done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  while (!mbar_try_wait(b, parity)) {
  }
}
// arrive on the mbarrier when all of this thread's prior cp.async copies have landed
// (counted against the barrier's expected arrivals: one per issuing thread per phase)
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
// generic-proxy writes to shared memory -> visible to later async-proxy (bulk copy) writes
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// bulk global -> shared copy (bytes % 16 == 0, both addresses 16-byte aligned),
// completion counted on the mbarrier's transaction count
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace ht
