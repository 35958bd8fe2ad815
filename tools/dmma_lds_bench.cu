// How fast can m16n8k16 f64 MMAs run when their B operands come from shared memory?
// Variants: warps per SM, B from registers vs LDS, with/without a CTA barrier per k16.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma16(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
               "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int NF, bool LDSB, bool BAR, bool LDSA = false>
__global__ void kern(double* out, int iters) {
  __shared__ double sb[16 * 116];
  for (int i = threadIdx.x; i < 16 * 116; i += blockDim.x) sb[i] = 1.0 + i * 1e-9;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double a[8], c[NF][4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (lane + i) * 1e-9;
  for (int j = 0; j < NF; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.0;
  double breg[4] = {1.0, 1.0, 1.0, 1.0};
  for (int it = 0; it < iters; ++it) {
    if (LDSA) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = sb[(t + 4 * (i >> 1)) * 116 + g + 8 * (i & 1) + (it & 1) * 4];
    }
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      double b[4];
      if (LDSB) {
#pragma unroll
        for (int i = 0; i < 4; ++i) b[i] = sb[(t + 4 * i) * 116 + j * 8 + g + (it & 1) * 2];
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) b[i] = breg[i];
      }
      mma16(c[j], a, b);
    }
    if (BAR) __syncthreads();
  }
  double s = 0;
  for (int j = 0; j < NF; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 12345.0) out[0] = s;
}

template <int NF, bool LDSB, bool BAR, bool LDSA = false>
void run(const char* name, int warps, double* out) {
  int iters = 2000;
  const int grid = 148;
  kern<NF, LDSB, BAR, LDSA><<<grid, warps * 32>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<NF, LDSB, BAR, LDSA><<<grid, warps * 32>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 16 * 8 * 16 * NF * (double)iters * warps * grid;
  printf("%-28s warps/SM=%2d  %6.2f TF/s\n", name, warps, fl / ms / 1e9);
}

int main() {
  double* out; cudaMalloc(&out, 8);
  for (int w : {4, 8}) {
    run<13, false, false>("regs B, no barrier", w, out);
    run<13, true, false>("LDS B (moving), no barrier", w, out);
    run<13, true, true>("LDS B (moving), barrier", w, out);
    run<13, true, true, true>("LDS A+B (moving), barrier", w, out);
  }
  return 0;
}
