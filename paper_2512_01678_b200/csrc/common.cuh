// Shared device/host helpers for the Morphling B200 kernels (sm_100a only).
// Nothing here is used by oracle/ (and nothing from oracle/ is used here).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/morphling.h"

namespace mph {

// ------------------------------------------------------------------ errors
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);

#define MPH_CUDA_TRY(expr)                                                            \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      return ::mph::fail(MPH_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,        \
                         cudaGetErrorString(_e));                                     \
  } while (0)

#define MPH_TRY(expr)             \
  do {                            \
    int _rc = (expr);             \
    if (_rc != MPH_OK) return _rc; \
  } while (0)

#define MPH_CHECK_ARG(cond, msg)                                 \
  do {                                                           \
    if (!(cond)) return ::mph::fail(MPH_EINVAL, "%s", (msg));    \
  } while (0)

inline int launch_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MPH_ECUDA, "launch %s: %s", what, cudaGetErrorString(e));
  return MPH_OK;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int round_up(int a, int b) { return (a + b - 1) / b * b; }

// Feature rows are padded to a multiple of 8 floats (one 32 B sector), or 4 when w <= 4
// (SURVEY §8 "Per-config shapes"; padded columns are exactly zero, Q26).
inline int pad_width(int w) { return w <= 4 ? 4 : round_up(w, 8); }

// Device memory: cudaMalloc, or the caller's allocator when one is registered
// (mph_set_allocator); the library owns what it allocates (include/morphling.h).
int dev_alloc_bytes(void** p, size_t bytes);
void dev_free(void* p);
template <class T>
int dev_alloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return MPH_OK;
  void* q = nullptr;
  MPH_TRY(dev_alloc_bytes(&q, count * sizeof(T)));
  *p = static_cast<T*>(q);
  return MPH_OK;
}

// Kernel launch counter (bench.py reports gpu_launches from it).
void count_launch(int n = 1);

// ------------------------------------------------------------------ device helpers
#ifdef __CUDACC__
__device__ __forceinline__ float4 ldg_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int ldg_stream_i32(const int* p) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
// L2 eviction-priority hints for streams that are touched once (neighbour ids, SpMM output),
// so they do not push the gathered operand out of L2.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int ldg_stream_i32_hint(const int* p, uint64_t pol) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_f4_hint(float4* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
// The same sums with Blackwell's packed FP32 adds (FADD2: add.rn.f32x2, two lanes of a float4 per
// instruction): round-to-nearest on each element, bit-identical to f4_add, half the instructions.
__device__ __forceinline__ float4 f4_add2(float4 a, float4 b) {
#ifdef MPH_NO_FADD2
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
#endif
  float4 r;
  asm("{\n\t.reg .b64 a0, a1, b0, b1, d0, d1;\n\t"
      "mov.b64 a0, {%4, %5};\n\tmov.b64 a1, {%6, %7};\n\t"
      "mov.b64 b0, {%8, %9};\n\tmov.b64 b1, {%10, %11};\n\t"
      "add.rn.f32x2 d0, a0, b0;\n\tadd.rn.f32x2 d1, a1, b1;\n\t"
      "mov.b64 {%0, %1}, d0;\n\tmov.b64 {%2, %3}, d1;\n\t}"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w));
  return r;
}
__device__ __forceinline__ bool bf16_positive(uint32_t bits16) { return (bits16 & 0x8000u) == 0 && (bits16 & 0x7FFFu); }
__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 f4_zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
// Round to the nearest TF32 value (ties away from zero), kept in an fp32 container: the
// tensor cores then read it exactly instead of truncating the low 13 mantissa bits.
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ float4 f4_tf32(float4 v) {
  return make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
}

// ---- peer-memory flags (NEXT-1, p2p.cu): system-scope release/acquire over NVLink
__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_timer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// One thread waits until flags_row[q] >= seq for every q < world (each peer's monotone step
// counter, written remotely by st_release_sys_u64).  Gives up after 10 s, recording the
// timeout in *err (and every later wait returns at once), so a lost peer cannot hang the GPU.
__device__ __forceinline__ bool p2p_wait_all(const uint64_t* flags_row, int world, uint64_t seq, int* err) {
  if (*(volatile int*)err) return false;
  const uint64_t t0 = global_timer_ns();
  for (int q = 0; q < world; ++q) {
    while (ld_acquire_sys_u64(flags_row + q) < seq) {
      if (global_timer_ns() - t0 > 10000000000ull) {
        atomicExch(err, 1);
        return false;
      }
      __nanosleep(128);
    }
  }
  return true;
}

// Two floats -> two bfloat16 (round to nearest even) packed lo | hi << 16: BF16 GEMM operands.
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// Philox4x32-10 (Salmon et al., SC'11) — the dropout mask of reading Q10.
struct PhiloxOut {
  uint32_t v[4];
};
__device__ __forceinline__ PhiloxOut philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                   uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  PhiloxOut o;
  o.v[0] = c0;
  o.v[1] = c1;
  o.v[2] = c2;
  o.v[3] = c3;
  return o;
}
#endif

// Dropout parameters carried into fused epilogues (Q10).
struct Dropout {
  uint32_t threshold;  // keep iff u32 >= threshold; 0 disables
  float scale;         // 1/(1-p) in f32
  uint32_t key0, key1;
  uint32_t layer, epoch;
  const int32_t* epoch_dev;  // when set (CUDA-graph replay) the epoch is read from device memory
};

}  // namespace mph
