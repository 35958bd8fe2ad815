// Relocation of captured CUDA graphs (address-independent graph replay).
//
// A captured truncation bakes the device addresses of its input tensor, output
// tensor and workspace into the arguments of its kernel / memset / memcpy nodes.
// A caller whose buffers come from a caching allocator (the end-to-end pipeline:
// add -> truncate -> read back, every step on fresh buffers) presents the same
// shapes at different addresses on every call.  Instead of capturing again, the
// executable graph is *relocated*: every 8-byte argument word that pointed into
// one of the captured address ranges is shifted by that range group's delta
// (new base - captured base) and written back with cudaGraphExec*NodeSetParams
// (or, where the driver refuses per-node updates inside conditional bodies,
// with the source graph patched and cudaGraphExecUpdate).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace ht {

struct RelocRange {
  uintptr_t lo, hi;  // [lo, hi)
  int group;
};

struct RelocSite {
  uint32_t param;  // kernel parameter index (memset/memcpy: 0 = dst, 1 = src)
  uint32_t off;    // byte offset inside the parameter
  int group;
};

struct RelocNode {
  cudaGraph_t owner = nullptr;
  cudaGraphNode_t node = nullptr;
  int kind = 0;  // 0 kernel, 1 memset, 2 memcpy
  cudaKernelNodeParams kp{};
  std::vector<std::vector<unsigned char>> args;  // captured argument bytes
  cudaMemsetParams ms{};
  cudaMemcpy3DParms mc{};
  std::vector<RelocSite> sites;
};

struct RelocTable {
  bool ok = true;  // false: a node type or argument layout the relocator cannot handle
  std::vector<RelocNode> nodes;  // only nodes with at least one relocation site
  long long kernel_nodes = 0;
};

// Collects the conditional-body graphs captured while `sink` is installed
// (capture_if_any registers each body it creates).
extern thread_local std::vector<cudaGraph_t>* g_body_sink;
// ... and the conditional nodes themselves (cudaGraphNodeGetType does not report them
// on every driver: they are skipped by identity)
extern thread_local std::vector<cudaGraphNode_t>* g_cond_sink;

// Scan `g` (and the registered conditional bodies) for argument words inside `ranges`.
void reloc_scan(cudaGraph_t g, const std::vector<cudaGraph_t>& bodies, const std::vector<cudaGraphNode_t>& conds,
                std::vector<RelocRange> ranges, RelocTable& out);

// Shift every site by delta[group] relative to the captured arguments and update `exec`.
// Returns cudaSuccess or the failing call's error.
cudaError_t reloc_apply(cudaGraphExec_t exec, cudaGraph_t g, RelocTable& t, const std::vector<long long>& delta);

// 1: per-node exec updates were refused once (conditional bodies), whole-graph update in use.
int reloc_update_mode();

}  // namespace ht
