// Device-side branches of captured truncations: CUDA conditional (IF) graph nodes.
#pragma once

#include <functional>

#include "common.cuh"

namespace ht {

// -1 untried, 1 conditional nodes work, 0 unavailable (callers enqueue eagerly and
// decide on the host / with device-flagged no-op launches instead)
extern int g_cond_nodes;
// kernels recorded inside IF bodies during the current process (they run only when
// the branch is taken: graph launch counts exclude them)
extern long long g_cond_body_launches;

bool stream_capturing(cudaStream_t s);
// true while the library captures one of its own truncation graphs on this thread
// (device-side branches are used there only, never inside a caller's capture)
extern thread_local bool g_own_capture;

// Inside a stream capture on `s`: append a one-thread kernel that sets the condition
// to (any of flags[0..n) != 0) -- counting taken branches into *taken when non-null --
// and an IF node whose body `body` enqueues on a second capture stream.
int capture_if_any(cudaStream_t s, const int* flags, int n, unsigned long long* taken,
                   const std::function<int(cudaStream_t)>& body);

}  // namespace ht
