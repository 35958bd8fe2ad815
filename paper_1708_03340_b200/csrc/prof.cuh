// Native launch accounting: a global launch counter (always on) and optional
// per-kernel CUDA-event timing on the launching stream (ht_profile_enable).
#pragma once

#include <cuda_runtime.h>

namespace ht {

struct ProfToken {
  cudaEvent_t a = nullptr;
};

// Call around every kernel launch: begin() records the start event if profiling is
// on; end() records the stop event and attributes algorithmic flops / bytes.
ProfToken prof_begin(cudaStream_t s);
void prof_end(const ProfToken& tok, const char* name, cudaStream_t s, double flops, double bytes);

// true while per-launch timing or the tag log is on (CUDA-graph replay is bypassed then)
bool prof_active();
// launches replayed inside a CUDA graph count like direct ones
void prof_add_launches(long long n);
long long prof_launches();

}  // namespace ht
