// QR of short-wide frames (m < K): rank-shrink orthogonalisation without the
// tall-QR kernels' K <= 112 limit (see qr_wide.cu).
#pragma once

#include <vector>

#include "qr.cuh"

namespace ht {

bool qr_wide_eligible(const QrProblem& q);
// global scratch per node needed when the block does not fit in shared memory (0 if it does)
long long qr_wide_ws_doubles(const QrProblem& q);
// Q (m x m, strides q_r/q_c) and R (m x K row-major, ld r_ld) of every node.
int qr_wide_batched(std::vector<QrProblem>& probs, cudaStream_t stream);

}  // namespace ht
