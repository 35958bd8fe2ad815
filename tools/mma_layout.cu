// Verify the operand layout assumed for mma.sync.m16n8k16.row.col.f64 (sm_100a).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[8], b[4], c[4] = {0, 0, 0, 0};
  for (int i = 0; i < 8; ++i) a[i] = A[(g + 8 * (i & 1)) * 16 + (t + 4 * (i >> 1))];  // H1
  for (int i = 0; i < 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];                          // B(k, n) row-major
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  C[g * 8 + 2 * t] = c[0];
  C[g * 8 + 2 * t + 1] = c[1];
  C[(g + 8) * 8 + 2 * t] = c[2];
  C[(g + 8) * 8 + 2 * t + 1] = c[3];
}


template <int KK>
__global__ void kk(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  constexpr int NA = KK / 2, NB = KK / 4;
  double a[8], b[4], c[4] = {0, 0, 0, 0};
  for (int i = 0; i < NA; ++i) a[i] = A[(g + 8 * (i & 1)) * 16 + (t + 4 * (i >> 1))];
  for (int i = 0; i < NB; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  if (KK == 4)
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
  else
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  C[g * 8 + 2 * t] = c[0];
  C[g * 8 + 2 * t + 1] = c[1];
  C[(g + 8) * 8 + 2 * t] = c[2];
  C[(g + 8) * 8 + 2 * t + 1] = c[3];
}

int main() {
  double hA[256], hB[128], hC[128], ref[128];
  for (int i = 0; i < 256; ++i) hA[i] = (double)rand() / RAND_MAX - 0.5;
  for (int i = 0; i < 128; ++i) hB[i] = (double)rand() / RAND_MAX - 0.5;
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int kk = 0; kk < 16; ++kk) s += hA[m * 16 + kk] * hB[kk * 8 + n];
      ref[m * 8 + n] = s;
    }
  double *dA, *dB, *dC;
  cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dC, sizeof(hC));
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  k<<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(hC, dC, sizeof(hC), cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 128; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("m16n8k16 f64 layout H1 max err %.3e (%s)\n", err, err < 1e-12 ? "OK" : "WRONG");
  for (int KK = 4; KK <= 8; KK += 4) {
    for (int m = 0; m < 16; ++m)
      for (int n = 0; n < 8; ++n) {
        double s = 0;
        for (int q = 0; q < KK; ++q) s += hA[m * 16 + q] * hB[q * 8 + n];
        ref[m * 8 + n] = s;
      }
    if (KK == 4) kk<4><<<1, 32>>>(dA, dB, dC); else kk<8><<<1, 32>>>(dA, dB, dC);
    cudaMemcpy(hC, dC, sizeof(hC), cudaMemcpyDeviceToHost);
    double e2 = 0;
    for (int i = 0; i < 128; ++i) e2 = fmax(e2, fabs(hC[i] - ref[i]));
    printf("m16n8k%d f64 layout H1 max err %.3e (%s)\n", KK, e2, e2 < 1e-12 ? "OK" : "WRONG");
  }
  return 0;
}
