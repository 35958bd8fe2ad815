// Standalone reproduction of one split-K GEMM descriptor through ht::gemm_grouped
// (links libht_b200.so).  usage: repro_gemm M N K S [offsetA offsetB]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1708_03340_b200/csrc/gemm.cuh"

int main(int argc, char** argv) {
  const int M = atoi(argv[1]), N = atoi(argv[2]), K = atoi(argv[3]), S = atoi(argv[4]);
  const long long offA = argc > 5 ? atoll(argv[5]) : 0, offB = argc > 6 ? atoll(argv[6]) : 0;
  const long long cols = M + N;
  double* Q;
  cudaMalloc(&Q, sizeof(double) * (cols * K + offA + offB + 4096));
  cudaMemset(Q, 0, sizeof(double) * (cols * K + offA + offB + 4096));
  double* P;
  cudaMalloc(&P, sizeof(double) * (size_t)S * M * N + 4096);
  ht::GemmDesc g = ht::gemm_desc(Q + offA, K, 1, Q + offA + (long long)M * K, 1, K, P, N, 1, M, N, K);
  g.splits = S;
  g.c_b1 = (long long)M * N;
  std::vector<ht::GemmDesc> v{g};
  int rc = ht::gemm_grouped(v, 0, "repro", true);
  cudaError_t e = cudaDeviceSynchronize();
  printf("M=%d N=%d K=%d S=%d rc=%d sync=%s\n", M, N, K, S, rc, cudaGetErrorString(e));
  return e != cudaSuccess;
}
