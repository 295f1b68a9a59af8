// Optional in-library kernel timing: CUDA events recorded on the launching stream around each
// hot-path launch of the model runtime, plus the algorithmic bytes / flops of that launch
// (SURVEY §8(d) d.3).  Disabled by default; bench.py enables it for the timed region.
#include <mutex>
#include <vector>

#include "internal.cuh"
#include "profile.cuh"

namespace mph {
namespace prof {

struct Rec {
  int kind;
  cudaEvent_t a, b;
  double bytes, flops;
};

static std::mutex g_mu;
static bool g_on = false;
static std::vector<Rec> g_recs;
static std::vector<cudaEvent_t> g_pool;

static cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

bool enabled() { return g_on; }
void set_enabled(bool on) { g_on = on; }

Scope::Scope(int kind, cudaStream_t s, double bytes, double flops) : idx_(-1), s_(s) {
  if (!g_on) return;
  std::lock_guard<std::mutex> lk(g_mu);
  Rec r{kind, get_event(), get_event(), bytes, flops};
  cudaEventRecord(r.a, s);
  g_recs.push_back(r);
  idx_ = (int)g_recs.size() - 1;
}

Scope::~Scope() {
  if (idx_ < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  if (idx_ < (int)g_recs.size()) cudaEventRecord(g_recs[idx_].b, s_);
}

}  // namespace prof
}  // namespace mph

using namespace mph;

extern "C" int mph_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(prof::g_mu);
  for (auto& r : prof::g_recs) {
    prof::g_pool.push_back(r.a);
    prof::g_pool.push_back(r.b);
  }
  prof::g_recs.clear();
  prof::g_on = on != 0;
  return MPH_OK;
}

extern "C" int mph_profile_read(int32_t kind, int64_t* count_h, double* total_ms_h, double* total_bytes_h,
                                double* total_flops_h) {
  std::lock_guard<std::mutex> lk(prof::g_mu);
  int64_t n = 0;
  double ms = 0.0, by = 0.0, fl = 0.0;
  for (auto& r : prof::g_recs) {
    if (r.kind != kind) continue;
    float t = 0.0f;
    cudaError_t e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e != cudaSuccess) return fail(MPH_ECUDA, "profile_read: %s (synchronise first)", cudaGetErrorString(e));
    ++n;
    ms += t;
    by += r.bytes;
    fl += r.flops;
  }
  if (count_h) *count_h = n;
  if (total_ms_h) *total_ms_h = ms;
  if (total_bytes_h) *total_bytes_h = by;
  if (total_flops_h) *total_flops_h = fl;
  return MPH_OK;
}
