// Error reporting, version, launch accounting and device probe of the C-ABI.
#include <atomic>
#include <cstdarg>
#include <cstdio>

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

}  // namespace mph

extern "C" {

int mph_version(void) { return MPH_VERSION; }

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
