// FP64 throughput microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) and DFMA.
// Used once to fix the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double x[8];
  double y = 1.0 + threadIdx.x * 1e-12, z = 0.999999;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], z, y);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int bps = 1; bps <= 4; bps *= 2) {
      dim3 grid(sms * bps), block(32 * warps);
      float ms;
      dmma_m8n8k4<<<grid, block>>>(out, 16);
      cudaEventRecord(e0); dmma_m8n8k4<<<grid, block>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid.x * warps;
      printf("{\"kernel\":\"dmma_m8n8k4\",\"warps\":%d,\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", warps, bps, fl / ms / 1e9);
      dmma_m16n8k16<<<grid, block>>>(out, 16);
      cudaEventRecord(e0); dmma_m16n8k16<<<grid, block>>>(out, iters / 4); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 16 * 8 * 16 * 4.0 * (iters / 4) * (double)grid.x * warps;
      printf("{\"kernel\":\"dmma_m16n8k16\",\"warps\":%d,\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", warps, bps, fl / ms / 1e9);
      dfma_loop<<<grid, block>>>(out, 16);
      cudaEventRecord(e0); dfma_loop<<<grid, block>>>(out, iters * 4); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 8 * iters * 4.0 * (double)grid.x * block.x;
      printf("{\"kernel\":\"dfma\",\"warps\":%d,\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", warps, bps, fl / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
