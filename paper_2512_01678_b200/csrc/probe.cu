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

}  // namespace mph

using namespace mph;

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
