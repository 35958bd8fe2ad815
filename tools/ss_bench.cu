// Stand-alone timing of the streaming GEMM on the truncation's C2 d=64 level-5 shapes
// (32 nodes, K = 100): the Gramian t1 product (dense), the two absorb mode products
// (triangular R^T) and the first projection mode product (N = 50).  Build variants
// with -DHT_SS2_CONS=.. -DHT_SS2_STAGES=.. (experiments only).
#include <cstdio>
#include <vector>
#include "../paper_1708_03340_b200/csrc/ssgemm.cu"
namespace ht {
ProfToken prof_begin(cudaStream_t) { return ProfToken{}; }
void prof_end(const ProfToken&, const char*, cudaStream_t, double, double) {}
void set_error(const std::string& m) { fprintf(stderr, "%s\n", m.c_str()); }
extern const int g_sync_check = 0;
int debug_probe() { return 0; }
}  // namespace ht
using namespace ht;

int main() {
  const int K = 100, nodes = 32;
  const long long K3 = (long long)K * K * K;
  double *X, *S, *C;
  cudaMalloc(&X, nodes * K3 * 8); cudaMalloc(&C, nodes * K3 * 8); cudaMalloc(&S, (size_t)nodes * K * K * 8);
  cudaMemset(X, 0, nodes * K3 * 8); cudaMemset(S, 0, (size_t)nodes * K * K * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"t1 (dense, N=100)", "absorb mode-2 (tri)", "absorb mode-3 (tri)", "project mode-1 (N=50)"};
  for (int variant = 0; variant < 4; ++variant) {
    std::vector<SsDesc> v;
    double frac = 1.0;
    int N = K;
    if (variant == 0) {  // t1^T = M1(B)^T G^T: rows (j,l) contiguous, k = i
      SsDesc d = ss_desc(X, 1, (long long)K * K, S, 1, K, C, 1, (long long)K * K, K * K, K, K);
      d.jobs = nodes; d.x_job = K3; d.s_job = K * K; d.c_job = K3;
      v.push_back(d);
    } else if (variant == 1) {  // T1_i^T = B_i^T R1^T over rows (i, l)
      SsDesc d = ss_desc(X, 1, K, S, 1, K, C, 1, K, K * K, K, K);
      d.M_lo = K; d.x_hi = (long long)K * K; d.c_hi = (long long)K * K; d.s_tri = 1;
      d.jobs = nodes; d.x_job = K3; d.s_job = K * K; d.c_job = K3;
      v.push_back(d); frac = 0.5;
    } else if (variant == 2) {  // Bp = T1 R2^T, rows (i, j) k-contiguous
      SsDesc d = ss_desc(X, K, 1, S, 1, K, C, K, 1, K * K, K, K);
      d.s_tri = 1;
      d.jobs = nodes; d.x_job = K3; d.s_job = K * K; d.c_job = K3;
      v.push_back(d); frac = 0.5;
    } else {  // C1^T = M1(B)^T PEV (N = 50)
      N = 50;
      SsDesc d = ss_desc(X, 1, (long long)K * K, S, N, 1, C, 1, (long long)K * K, K * K, N, K);
      d.jobs = nodes; d.x_job = K3; d.s_job = K * N; d.c_job = (long long)K * K * N;
      v.push_back(d);
    }
    ss_gemm(v, 0, "x");
    cudaEventRecord(e0);
    const int reps = 20;
    for (int r = 0; r < reps; ++r) ss_gemm(v, 0, "x");
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    const double fl = 2.0 * nodes * (double)K * K * K * N;
    const double by = 8.0 * nodes * ((double)K * K * K + (double)K * K * N);
    printf("CONS=%d STAGES=%d %-24s %7.1f us  alg %5.2f TF/s  exec %5.2f TF/s  %5.2f TB/s  (%s)\n", HT_SS2_CONS,
           HT_SS2_STAGES, names[variant], ms * 1e3, fl / ms / 1e9, frac * fl / ms / 1e9, by / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
