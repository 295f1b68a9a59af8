// Error reporting, version, launch accounting and device probe of the C-ABI.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace mph {

static thread_local char g_err[1024] = "";
static std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ---- device memory: cudaMalloc or the registered caller allocator (mph_set_allocator)
struct Allocator {
  void* (*alloc)(size_t, void*, void*) = nullptr;
  void (*release)(void*, size_t, void*, void*) = nullptr;
  void* ctx = nullptr;
};
static Allocator g_alloc;
static std::mutex g_alloc_mu;
static std::unordered_map<void*, std::pair<size_t, Allocator>> g_from_caller;  // ptr -> (bytes, provider)

int dev_alloc_bytes(void** p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) return MPH_OK;
  Allocator a;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    a = g_alloc;
  }
  if (a.alloc) {
    void* q = a.alloc(bytes, nullptr, a.ctx);
    if (!q) return fail(MPH_ENOMEM, "caller allocator returned NULL for %zu B", bytes);
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    g_from_caller[q] = {bytes, a};
    *p = q;
    return MPH_OK;
  }
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess)
    return fail(e == cudaErrorMemoryAllocation ? MPH_ENOMEM : MPH_ECUDA, "cudaMalloc(%zu B): %s", bytes,
                cudaGetErrorString(e));
  return MPH_OK;
}

void dev_free(void* p) {
  if (!p) return;
  std::pair<size_t, Allocator> owner{0, Allocator{}};
  bool caller = false;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    auto it = g_from_caller.find(p);
    if (it != g_from_caller.end()) {
      owner = it->second;
      g_from_caller.erase(it);
      caller = true;
    }
  }
  if (caller)
    owner.second.release(p, owner.first, nullptr, owner.second.ctx);
  else
    cudaFree(p);
}

}  // namespace mph

extern "C" {

int mph_version(void) { return MPH_VERSION; }

int mph_set_allocator(void* (*alloc)(size_t, void*, void*), void (*release)(void*, size_t, void*, void*), void* ctx) {
  if ((alloc == nullptr) != (release == nullptr)) return mph::fail(MPH_EINVAL, "set_allocator: give both or neither");
  std::lock_guard<std::mutex> lk(mph::g_alloc_mu);
  mph::g_alloc.alloc = alloc;
  mph::g_alloc.release = release;
  mph::g_alloc.ctx = alloc ? ctx : nullptr;
  return MPH_OK;
}

const char* mph_last_error(void) { return mph::g_err; }

int mph_launch_count(int64_t* count_h) {
  if (!count_h) return mph::fail(MPH_EINVAL, "null count");
  *count_h = mph::g_launches.load();
  return MPH_OK;
}

int mph_device_check(int32_t* sm_count_h) {
  mph::g_err[0] = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return mph::fail(MPH_ECUDA, "no CUDA device: %s", cudaGetErrorString(e));
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, dev);
  if (e != cudaSuccess) return mph::fail(MPH_ECUDA, "cudaGetDeviceProperties: %s", cudaGetErrorString(e));
  if (prop.major != 10 || prop.minor != 0)
    return mph::fail(MPH_ECUDA, "kernels are built for sm_100a; device is sm_%d%d", prop.major, prop.minor);
  if (sm_count_h) *sm_count_h = prop.multiProcessorCount;
  return MPH_OK;
}

}  // extern "C"
