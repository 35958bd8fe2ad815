// Stand-alone timing of the streaming GEMM on the truncation's shapes (experiments).
#include <cstdio>
#include <vector>
#include "../paper_1708_03340_b200/csrc/ssgemm.cu"
namespace ht {
ProfToken prof_begin(cudaStream_t) { return ProfToken{}; }
void prof_end(const ProfToken&, const char*, cudaStream_t, double, double) {}
void set_error(const std::string& m) { fprintf(stderr, "%s\n", m.c_str()); }
}  // namespace ht
using namespace ht;

int main() {
  const int K = 100, N = 100, nodes = 32, kt = 100, k1 = 100, k2 = 100;
  double *X, *S, *C;
  const size_t big = (size_t)nodes * kt * k1 * k2;
  cudaMalloc(&X, big * 8); cudaMalloc(&C, big * 8); cudaMalloc(&S, (size_t)nodes * K * N * 8);
  cudaMemset(X, 0, big * 8); cudaMemset(S, 0, (size_t)nodes * K * N * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int variant = 0; variant < 2; ++variant) {
    std::vector<SsDesc> v;
    if (variant == 0) {  // mode-3 absorb: X row-major (k-contiguous)
      SsDesc d = ss_desc(X, k2, 1, S, 1, k2, C, N, 1, kt * k1, N, k2);
      d.jobs = nodes; d.x_job = (long long)kt * k1 * k2; d.s_job = K * N; d.c_job = (long long)kt * k1 * N;
      v.push_back(d);
    } else {  // mode-2 absorb: two-level rows, m-contiguous X, column-major C
      SsDesc d = ss_desc(X, 1, k2, S, 1, k1, C, 1, k2, kt * k2, N, k1);
      d.M_lo = k2; d.x_hi = (long long)k1 * k2; d.c_hi = (long long)N * k2;
      d.jobs = nodes; d.x_job = (long long)kt * k1 * k2; d.s_job = K * N; d.c_job = (long long)kt * N * k2;
      v.push_back(d);
    }
    ss_gemm(v, 0, "x");
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) ss_gemm(v, 0, "x");
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
    const double fl = 2.0 * nodes * (double)kt * k1 * k2 * N;
    printf("variant %d (%s): %.1f us  %.2f TF/s  (err %s)\n", variant, variant ? "mode-2" : "mode-3", ms * 1e3,
           fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
