// Bandwidth probe used by bench.py to put the aggregation SpMM on a measured roofline:
// random-row gathers (the SpMM's memory pattern, SURVEY §8(d) d.4 "L2 random-row-gather
// bench") from a table that is either L2-resident or HBM-resident.  Not part of the training
// step.
#include <algorithm>

#include "internal.cuh"

namespace mph {

template <int U>
__global__ void __launch_bounds__(256) k_probe_gather(const float* __restrict__ table, int w4, const int32_t* idx,
                                                      int64_t n_idx, int64_t per_warp, float* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t e0 = warp * per_warp, e1 = min(n_idx, e0 + per_warp);
  float4 acc = f4_zero();
  for (int64_t b = e0; b < e1; b += 32) {
    const int nb = (int)min((int64_t)32, e1 - b);
    const int my = lane < nb ? ldg_stream_i32(idx + b + lane) : 0;
    for (int k0 = 0; k0 < nb; k0 += U) {
      float4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = __shfl_sync(0xffffffffu, my, (k0 + u) & 31);
        x[u] = (k0 + u < nb && lane < w4) ? ldg_f4(reinterpret_cast<const float4*>(table + (int64_t)r * w4 * 4) + lane)
                                          : f4_zero();
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc = f4_add(acc, x[u]);
    }
  }
  if (lane < w4) reinterpret_cast<float4*>(out)[warp * 32 + lane] = acc;
}

// Streaming read of an L2-resident buffer through the L2 -> SM path only (ld.global.cg: no L1
// allocation, so no L1 hits inflate the rate): block b reads chunk (b + pass * 37) mod n_blocks
// on pass `pass`, so no SM re-reads its own chunk; 8 independent 16-byte loads per thread in
// flight.  Its rate is the L2 delivery ceiling the aggregation's gathers are measured against.
__global__ void __launch_bounds__(512) k_probe_l2_stream(const float4* __restrict__ buf, int64_t chunk4,
                                                         int passes, float* out) {
  float4 acc = f4_zero();
  const int nb = gridDim.x;
  for (int p = 0; p < passes; ++p) {
    const float4* c = buf + (int64_t)((blockIdx.x + (int64_t)p * 37) % nb) * chunk4;
    for (int64_t i = threadIdx.x; i < chunk4; i += 8 * (int64_t)blockDim.x) {
      float4 x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t j = i + (int64_t)u * blockDim.x;
        if (j < chunk4) {
          asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(x[u].x), "=f"(x[u].y), "=f"(x[u].z), "=f"(x[u].w)
                       : "l"(c + j));
        } else {
          x[u] = f4_zero();
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = f4_add(acc, x[u]);
    }
  }
  reinterpret_cast<float4*>(out)[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

}  // namespace mph

using namespace mph;

// Reads buf_d [n_floats] (n_floats a multiple of 4 * n_blocks * 4; keep it L2-resident, e.g.
// 48 MB) `passes` times with n_blocks = 2 x SMs blocks of 512 threads; out_d needs
// n_blocks * 512 * 4 floats.  Rate = passes * n_floats * 4 / t.
extern "C" int mph_probe_l2_stream(const float* buf_d, int64_t n_floats, int32_t passes, float* out_d, void* stream) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nb = 2 * sms;
  if (!buf_d || !out_d || passes < 1 || n_floats <= 0 || n_floats % (4 * nb))
    return fail(MPH_EINVAL, "probe_l2_stream arguments (n_floats must be a multiple of %d)", 4 * nb);
  k_probe_l2_stream<<<nb, 512, 0, (cudaStream_t)stream>>>(reinterpret_cast<const float4*>(buf_d), n_floats / 4 / nb,
                                                          passes, out_d);
  count_launch();
  return launch_check("probe_l2_stream");
}

// Gathers rows idx[0..n_idx) (w floats each, w % 4 == 0, w <= 128) of table [n_rows][w] and
// writes one float4 partial per lane per warp into out (needs 128 * n_warps floats; n_warps =
// 148 * 32).  Time it with CUDA events to get gather bandwidth = n_idx * w * 4 / t.
extern "C" int mph_probe_gather(const float* table_d, int64_t n_rows, int32_t w, const int32_t* idx_d, int64_t n_idx,
                                float* out_d, void* stream) {
  if (!table_d || !idx_d || !out_d || n_rows <= 0 || w <= 0 || w % 4 || w > 128 || n_idx < 0)
    return fail(MPH_EINVAL, "probe_gather arguments");
  const int64_t warps = 148 * 32;
  const int64_t per_warp = ceil_div(std::max<int64_t>(n_idx, 1), warps);
  k_probe_gather<8><<<(unsigned)(warps / 8), 256, 0, (cudaStream_t)stream>>>(table_d, w / 4, idx_d, n_idx, per_warp,
                                                                              out_d);
  count_launch();
  return launch_check("probe_gather");
}
