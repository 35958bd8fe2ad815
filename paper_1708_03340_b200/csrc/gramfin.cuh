// Finishing step of one level of the top-down reduced-Gramian sweep (reference
// arith.py:148-158, 299-322): sum the split-K partials of each son Gramian G_s into
// G_s and, for a son whose orthogonalisation left an implicit Q (driver.cu,
// OrthPlan::imp), also form the operand its own level applies to the absorbed transfer
// tensor:  G~_s = R_s^{-1} G_s R_s^{-T}.
//
// One launch per level for all sons.  A son with the sandwich takes ceil(K/16) CTAs:
// each sums the whole G_s from the partials into shared memory (they are L2-resident,
// just written by the long-reduction GEMM), writes its 16 rows of G_s, computes
// Y = G_s R^{-T}[:, J] (K x 16) and then G~[:, J] = R^{-1} Y for its 16 columns J.
// A son without it takes ceil(K/16) CTAs that only reduce their 16 rows.  The partials
// of a symmetric Gram GEMM are exactly symmetric (lrt_kernel mirrors its blocks), so
// the sum is too.
#pragma once

#include <vector>

#include "common.cuh"

namespace ht {

struct GramFinDesc {
  const double* P;     // S partials, each K x K row-major (partial stride K*K)
  double* G;           // output K x K row-major (may be null with Rinv: G~ only)
  const double* Rinv;  // optional: K x K row-major upper triangular R^{-1}
  double* Gt;          // output G~ (when Rinv)
  int S, K;
};

constexpr int kGramFinMaxK = 128;

int gram_finish(const std::vector<GramFinDesc>& descs, cudaStream_t stream);

}  // namespace ht
