// Dependent-chain latencies of FP64 ops on the B200 (one warp): cycles per op.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double seed, int n) {
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0, t1;
  // 0: DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
  t1 = clock64(); cyc[0] = t1 - t0;
  // 1: DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  t1 = clock64(); cyc[1] = t1 - t0;
  // 2: shfl chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  t1 = clock64(); cyc[2] = t1 - t0;
  // 3: rsqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 1.0);
  t1 = clock64(); cyc[3] = t1 - t0;
  // 4: sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  t1 = clock64(); cyc[4] = t1 - t0;
  // 5: division chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64(); cyc[5] = t1 - t0;
  // 6: __drcp_rn chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x + 1.0);
  t1 = clock64(); cyc[6] = t1 - t0;
  // 7: DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  t1 = clock64(); cyc[7] = t1 - t0;
  // 8: smem store/load round trip
  __shared__ double s[64];
  t0 = clock64();
  for (int i = 0; i < n; ++i) { s[threadIdx.x] = x; __syncwarp(); x = s[(threadIdx.x + 1) & 31] + 1e-30; __syncwarp(); }
  t1 = clock64(); cyc[8] = t1 - t0;
  // 9: __syncthreads (1 warp)
  t0 = clock64();
  for (int i = 0; i < n; ++i) { __syncthreads(); }
  t1 = clock64(); cyc[9] = t1 - t0;
  out[threadIdx.x] = x;
}
__global__ void kb(long long* cyc, int n) {  // __syncthreads with 8 / 32 warps
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64 * 8);
  const int n = 4096;
  k<<<1, 32>>>(out, cyc, 0.5, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(out, cyc, 0.5, n); cudaDeviceSynchronize();
  const char* names[] = {"dfma", "dmul", "shfl", "rsqrt", "sqrt", "div", "drcp_rn", "dadd", "sts+lds", "bar(1w)"};
  for (int i = 0; i < 10; ++i) printf("%-8s %6.1f cyc\n", names[i], (double)cyc[i] / n);
  for (int t : {256, 512, 1024}) {
    kb<<<1, t>>>(cyc, n); cudaDeviceSynchronize();
    kb<<<1, t>>>(cyc, n); cudaDeviceSynchronize();
    printf("bar(%d thr) %6.1f cyc\n", t, (double)cyc[0] / n);
  }
  return 0;
}
