#include <atomic>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "ht_b200.h"
#include "prof.cuh"

namespace ht {

namespace {

struct Pending {
  std::string name;
  cudaEvent_t a, b;
  double flops, bytes;
};

struct Entry {
  double ms = 0, flops = 0, bytes = 0;
  long long launches = 0;
};

std::atomic<long long> g_launches{0};
std::mutex g_mu;
bool g_on = false;
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_pool;
std::map<std::string, Entry> g_acc;
bool g_log_on = false;
bool g_per_launch = false;  // bit 2: one report entry per launch ("tag#seq")
long long g_seq = 0;
struct LogEntry {
  std::string name;
  double flops, bytes;
};
std::vector<LogEntry> g_log;  // launch-order tag log (ht_profile_enable bit 1)

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void drain_locked() {
  for (auto& p : g_pending) {
    cudaEventSynchronize(p.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    Entry& e = g_acc[p.name];
    e.ms += ms;
    e.flops += p.flops;
    e.bytes += p.bytes;
    e.launches += 1;
    g_pool.push_back(p.a);
    g_pool.push_back(p.b);
  }
  g_pending.clear();
}

}  // namespace

ProfToken prof_begin(cudaStream_t s) {
  ProfToken t;
  std::lock_guard<std::mutex> g(g_mu);
  if (g_on) {
    t.a = get_event();
    cudaEventRecord(t.a, s);
  }
  return t;
}

void prof_end(const ProfToken& tok, const char* name, cudaStream_t s, double flops, double bytes) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_log_on) {
    std::lock_guard<std::mutex> g(g_mu);
    g_log.push_back({name, flops, bytes});
  }
  if (!tok.a) return;
  std::lock_guard<std::mutex> g(g_mu);
  cudaEvent_t b = get_event();
  cudaEventRecord(b, s);
  if (g_per_launch) {
    char key[160];
    snprintf(key, sizeof key, "%s#%03lld", name, g_seq++);
    g_pending.push_back({key, tok.a, b, flops, bytes});
  } else {
    g_pending.push_back({name, tok.a, b, flops, bytes});
  }
  if (g_pending.size() > 4096) drain_locked();
}

bool prof_active() {
  std::lock_guard<std::mutex> g(g_mu);
  return g_on || g_log_on;
}

void prof_add_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

long long prof_launches() { return g_launches.load(); }

}  // namespace ht

extern "C" {

int64_t ht_launch_count(void) { return ht::g_launches.load(); }

int ht_profile_enable(int on) {
  std::lock_guard<std::mutex> g(ht::g_mu);
  ht::drain_locked();
  ht::g_acc.clear();
  ht::g_log.clear();
  ht::g_on = (on & 1) != 0;
  ht::g_log_on = (on & 2) != 0;
  ht::g_per_launch = (on & 4) != 0;
  ht::g_seq = 0;
  return 0;
}

int ht_profile_log(char* buf, size_t len) {
  std::lock_guard<std::mutex> g(ht::g_mu);
  std::string s = "[";
  for (size_t i = 0; i < ht::g_log.size(); ++i) {
    char tmp[256];
    snprintf(tmp, sizeof(tmp), "%s[\"%s\", %.6e, %.6e]", i ? ", " : "", ht::g_log[i].name.c_str(),
             ht::g_log[i].flops, ht::g_log[i].bytes);
    s += tmp;
  }
  s += "]";
  if (buf && len) {
    size_t n = s.size() < len - 1 ? s.size() : len - 1;
    memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return (int)s.size();
}

int ht_profile_report(char* buf, size_t len) {
  std::lock_guard<std::mutex> g(ht::g_mu);
  ht::drain_locked();
  std::string s = "{";
  bool first = true;
  for (auto& kv : ht::g_acc) {
    char tmp[512];
    snprintf(tmp, sizeof(tmp), "%s\"%s\": {\"ms\": %.6f, \"launches\": %lld, \"flops\": %.6e, \"bytes\": %.6e}",
             first ? "" : ", ", kv.first.c_str(), kv.second.ms, kv.second.launches, kv.second.flops,
             kv.second.bytes);
    s += tmp;
    first = false;
  }
  s += "}";
  if (buf && len) {
    size_t n = s.size() < len - 1 ? s.size() : len - 1;
    memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return (int)s.size();
}

}  // extern "C"
