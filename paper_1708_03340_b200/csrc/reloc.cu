// Relocation of captured CUDA graphs -- see reloc.cuh.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <mutex>

#include "reloc.cuh"

namespace ht {

thread_local std::vector<cudaGraph_t>* g_body_sink = nullptr;
thread_local std::vector<cudaGraphNode_t>* g_cond_sink = nullptr;

namespace {

int g_update_mode = -1;  // -1: untried, 0: per-node exec updates work, 1: whole-graph update

bool dbg() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HT_RELOC_DEBUG");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

int find_group(const std::vector<RelocRange>& r, uintptr_t w) {
  // r sorted by lo, disjoint
  auto it = std::upper_bound(r.begin(), r.end(), w, [](uintptr_t v, const RelocRange& x) { return v < x.lo; });
  if (it == r.begin()) return -1;
  --it;
  return w < it->hi ? it->group : -1;
}

void scan_words(const unsigned char* p, size_t size, uint32_t param, const std::vector<RelocRange>& r,
                std::vector<RelocSite>& sites) {
  for (size_t o = 0; o + 8 <= size; o += 8) {
    uint64_t w;
    memcpy(&w, p + o, 8);
    const int g = find_group(r, (uintptr_t)w);
    if (g >= 0) sites.push_back(RelocSite{param, (uint32_t)o, g});
  }
}

void scan_fail(RelocTable& out, const char* what, int type, cudaError_t e) {
  out.ok = false;
  cudaGetLastError();  // a failed query must not surface as the next launch's error
  if (dbg()) fprintf(stderr, "[reloc] not relocatable: %s (node type %d, error %d)\n", what, type, (int)e);
}

void scan_graph(cudaGraph_t g, const std::vector<cudaGraphNode_t>& conds, const std::vector<RelocRange>& r,
                RelocTable& out) {
  size_t n = 0;
  cudaError_t e = cudaGraphGetNodes(g, nullptr, &n);
  if (e != cudaSuccess) return scan_fail(out, "get nodes", -1, e);
  std::vector<cudaGraphNode_t> nodes(n);
  if (n && (e = cudaGraphGetNodes(g, nodes.data(), &n)) != cudaSuccess) return scan_fail(out, "get nodes", -1, e);
  for (cudaGraphNode_t nd : nodes) {
    if (std::find(conds.begin(), conds.end(), nd) != conds.end()) continue;  // bodies scanned separately
    cudaGraphNodeType ty;
    if ((e = cudaGraphNodeGetType(nd, &ty)) != cudaSuccess) return scan_fail(out, "node type", -1, e);
    RelocNode rn;
    rn.owner = g;
    rn.node = nd;
    switch (ty) {
      case cudaGraphNodeTypeKernel: {
        ++out.kernel_nodes;
        rn.kind = 0;
        if ((e = cudaGraphKernelNodeGetParams(nd, &rn.kp)) != cudaSuccess || rn.kp.extra != nullptr)
          return scan_fail(out, "kernel params", (int)ty, e);
        for (size_t i = 0;; ++i) {
          size_t off = 0, sz = 0;
          if (cudaFuncGetParamInfo(rn.kp.func, i, &off, &sz) != cudaSuccess) {
            cudaGetLastError();
            break;
          }
          const unsigned char* src = (const unsigned char*)rn.kp.kernelParams[i];
          rn.args.emplace_back(src, src + sz);
          scan_words(src, sz, (uint32_t)i, r, rn.sites);
        }
        break;
      }
      case cudaGraphNodeTypeMemset: {
        rn.kind = 1;
        if ((e = cudaGraphMemsetNodeGetParams(nd, &rn.ms)) != cudaSuccess)
          return scan_fail(out, "memset params", (int)ty, e);
        const int gr = find_group(r, (uintptr_t)rn.ms.dst);
        if (gr >= 0) rn.sites.push_back(RelocSite{0, 0, gr});
        break;
      }
      case cudaGraphNodeTypeMemcpy: {
        rn.kind = 2;
        if ((e = cudaGraphMemcpyNodeGetParams(nd, &rn.mc)) != cudaSuccess || rn.mc.srcArray || rn.mc.dstArray)
          return scan_fail(out, "memcpy params", (int)ty, e);
        const int gd = find_group(r, (uintptr_t)rn.mc.dstPtr.ptr);
        const int gs = find_group(r, (uintptr_t)rn.mc.srcPtr.ptr);
        if (gd >= 0) rn.sites.push_back(RelocSite{0, 0, gd});
        if (gs >= 0) rn.sites.push_back(RelocSite{1, 0, gs});
        break;
      }
      case cudaGraphNodeTypeConditional:  // bodies are scanned from the registered list
      case cudaGraphNodeTypeEmpty:
      case cudaGraphNodeTypeWaitEvent:
      case cudaGraphNodeTypeEventRecord:
        continue;
      default:  // host / child-graph / allocation nodes: not relocatable
        return scan_fail(out, "node type", (int)ty, cudaSuccess);
    }
    if (!rn.sites.empty()) out.nodes.push_back(std::move(rn));
  }
}

// The node's parameters with every site shifted by its group's delta.
struct Patched {
  std::vector<std::vector<unsigned char>> args;
  std::vector<void*> argp;
  cudaKernelNodeParams kp{};
  cudaMemsetParams ms{};
  cudaMemcpy3DParms mc{};
};

void patch(const RelocNode& n, const std::vector<long long>& delta, Patched& p) {
  if (n.kind == 0) {
    p.args = n.args;
    for (const auto& s : n.sites) {
      uint64_t w;
      memcpy(&w, p.args[s.param].data() + s.off, 8);
      w += (uint64_t)delta[s.group];
      memcpy(p.args[s.param].data() + s.off, &w, 8);
    }
    p.argp.resize(p.args.size());
    for (size_t i = 0; i < p.args.size(); ++i) p.argp[i] = p.args[i].data();
    p.kp = n.kp;
    p.kp.kernelParams = p.argp.data();
    p.kp.extra = nullptr;
  } else if (n.kind == 1) {
    p.ms = n.ms;
    p.ms.dst = (char*)p.ms.dst + delta[n.sites[0].group];
  } else {
    p.mc = n.mc;
    for (const auto& s : n.sites) {
      if (s.param == 0) p.mc.dstPtr.ptr = (char*)p.mc.dstPtr.ptr + delta[s.group];
      else p.mc.srcPtr.ptr = (char*)p.mc.srcPtr.ptr + delta[s.group];
    }
  }
}

cudaError_t apply_exec(cudaGraphExec_t exec, const RelocNode& n, const Patched& p) {
  if (n.kind == 0) return cudaGraphExecKernelNodeSetParams(exec, n.node, &p.kp);
  if (n.kind == 1) return cudaGraphExecMemsetNodeSetParams(exec, n.node, &p.ms);
  return cudaGraphExecMemcpyNodeSetParams(exec, n.node, &p.mc);
}

cudaError_t apply_source(const RelocNode& n, const Patched& p) {
  if (n.kind == 0) return cudaGraphKernelNodeSetParams(n.node, &p.kp);
  if (n.kind == 1) return cudaGraphMemsetNodeSetParams(n.node, &p.ms);
  return cudaGraphMemcpyNodeSetParams(n.node, &p.mc);
}

}  // namespace

void reloc_scan(cudaGraph_t g, const std::vector<cudaGraph_t>& bodies, const std::vector<cudaGraphNode_t>& conds,
                std::vector<RelocRange> ranges, RelocTable& out) {
  out = RelocTable{};
  std::sort(ranges.begin(), ranges.end(), [](const RelocRange& a, const RelocRange& b) { return a.lo < b.lo; });
  // overlapping ranges (aliased node arrays) make the group of a word ambiguous
  for (size_t i = 1; i < ranges.size(); ++i)
    if (ranges[i].lo < ranges[i - 1].hi) {
      out.ok = false;
      return;
    }
  scan_graph(g, conds, ranges, out);
  for (cudaGraph_t b : bodies) {
    if (!out.ok) break;
    scan_graph(b, conds, ranges, out);
  }
  if (dbg()) {
    fprintf(stderr, "[reloc] scan: ok=%d kernel_nodes=%lld patched_nodes=%zu bodies=%zu\n", (int)out.ok,
            out.kernel_nodes, out.nodes.size(), bodies.size());
    for (const auto& n : out.nodes)
      fprintf(stderr, "[reloc]   kind=%d args=%zu sites=%zu func=%p\n", n.kind, n.args.size(), n.sites.size(),
              n.kind == 0 ? n.kp.func : nullptr);
  }
  if (!out.ok) out.nodes.clear();
  cudaGetLastError();
}

cudaError_t reloc_apply(cudaGraphExec_t exec, cudaGraph_t g, RelocTable& t, const std::vector<long long>& delta) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (g_update_mode < 0) {
    const char* e = getenv("HT_RELOC_UPDATE");  // tests: force the whole-graph update path
    if (e && e[0] == '1') g_update_mode = 1;
  }
  std::vector<Patched> ps(t.nodes.size());
  for (size_t i = 0; i < t.nodes.size(); ++i) patch(t.nodes[i], delta, ps[i]);
  if (g_update_mode != 1) {
    cudaError_t e = cudaSuccess;
    for (size_t i = 0; i < t.nodes.size() && e == cudaSuccess; ++i) {
      e = apply_exec(exec, t.nodes[i], ps[i]);
      if (dbg()) fprintf(stderr, "[reloc] exec-set node %zu kind %d -> %d\n", i, t.nodes[i].kind, (int)e);
    }
    if (e == cudaSuccess) {
      g_update_mode = 0;
      return cudaSuccess;
    }
    cudaGetLastError();
    g_update_mode = 1;  // e.g. nodes inside conditional bodies: update the whole graph instead
  }
  for (size_t i = 0; i < t.nodes.size(); ++i) {
    const cudaError_t e = apply_source(t.nodes[i], ps[i]);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return e;
    }
  }
  cudaGraphExecUpdateResultInfo info{};
  const cudaError_t e = cudaGraphExecUpdate(exec, g, &info);
  if (dbg()) fprintf(stderr, "[reloc] exec-update -> %d (result %d)\n", (int)e, (int)info.result);
  if (e != cudaSuccess) cudaGetLastError();
  return e;
}

int reloc_update_mode() { return g_update_mode; }

}  // namespace ht
