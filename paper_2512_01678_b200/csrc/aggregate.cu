// Other aggregation schemes ("GCN uses normalized mean aggregation ...
// GIN employs sum aggregation", "multiple aggregation schemes (mean, max, sum)", Listing 1's
// SAGE "Max" P:165; readings R6-R7).
//
//  * sum / mean run on the aggregation SpMM (spmm.cu) with the scheme's diagonal scales:
//    AGG = diag(post)·Ã·diag(pre), the pre-scale applied by the producer of the operand, as for
//    the GCN's dinv.  gcn: pre = post = D̃^{-1/2}; sum: none; mean: post = D̃^{-1} forward, and
//    for the adjoint Ã·D̃^{-1} pre = D̃^{-1}.
//  * max gets its own pair of kernels, same work items and row structure as the SpMM (warp per
//    row, LPR lanes × VPL float4 across the width, 32/LPR edge slots walking the neighbours in
//    ascending id order):
//      forward   Y[u,c] = max_{v∈Ñ(u)} H[v,c], arg[u,c] = the smallest v attaining it: each slot
//                keeps its first maximum (strict >), slots merge by (value, then smaller id);
//      backward  dH[v,c] = Σ_{u∈Ñ(v)} [arg[u,c] = v]·dY[u,c] — the routing adjoint written as a
//                gather over v's own neighbours (Ã is symmetric), so no atomics: fixed order,
//                deterministic; the ReLU-mask / dropout scale / TF32 epilogue is fused.
#include <algorithm>
#include <climits>

#include "internal.cuh"

namespace mph {

struct MaxArgs {
  const int64_t* row_ptr;
  const int32_t* col;
  const float* in;   // forward: H; backward: dY
  const int32_t* arg;  // backward: arg of the forward
  float* out;
  int32_t* arg_out;  // forward (nullable: arg not recorded)
  const int2* items;
  int* counter;
  int n_items, nv4, ld_in, ld_arg, ld_out;
  // epilogue
  uint32_t flags;
  const float* mask_src;
  int ld_mask;
  float mask_scale;
};

__device__ __forceinline__ void max_take(float& b, int& a, float x, int c) {
  if (x > b || a == INT_MAX) {  // the first neighbour always initialises (also for -inf / NaN rows)
    b = x;
    a = c;
  }
}
__device__ __forceinline__ void max_merge(float& b, int& a, float b2, int a2) {
  if (a2 != INT_MAX && (a == INT_MAX || b2 > b || (b2 == b && a2 < a))) {
    b = b2;
    a = a2;
  }
}

// U gathers per slot in flight per round (the max merge and the routed sum take them in ascending
// edge order, so U changes nothing but the memory-level parallelism)
template <int LPR, int VPL, int U>
__device__ __forceinline__ void max_row(const MaxArgs& a, int row, int lane) {
  constexpr int ES = 32 / LPR;
  const int slot = lane / LPR, sub = lane % LPR;
  const int64_t s = a.row_ptr[row], e = a.row_ptr[row + 1];
  float4 best[VPL];
  int4 arg[VPL];
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    best[j] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    arg[j] = make_int4(INT_MAX, INT_MAX, INT_MAX, INT_MAX);
  }
  for (int64_t base = s; base < e; base += 32) {
    const int nb = (int)min((int64_t)32, e - base);
    const int my_c = (base + lane < e) ? ldg_stream_i32(a.col + base + lane) : 0;
    for (int k0 = 0; k0 < nb; k0 += U * ES) {
      float4 x[U][VPL];
      int cc[U];
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {  // all U gathers in flight before any is used
        const int k = k0 + uu * ES + slot;
        const int c = __shfl_sync(0xffffffffu, my_c, k & 31);  // all lanes shuffle
        cc[uu] = k < nb ? c : INT_MAX;
        const float4* p = reinterpret_cast<const float4*>(a.in + (int64_t)(k < nb ? c : 0) * a.ld_in) + sub;
#pragma unroll
        for (int j = 0; j < VPL; ++j) x[uu][j] = (k < nb && sub + j * LPR < a.nv4) ? ldg_f4(p + j * LPR) : f4_zero();
      }
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        if (cc[uu] == INT_MAX) continue;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          max_take(best[j].x, arg[j].x, x[uu][j].x, cc[uu]);
          max_take(best[j].y, arg[j].y, x[uu][j].y, cc[uu]);
          max_take(best[j].z, arg[j].z, x[uu][j].z, cc[uu]);
          max_take(best[j].w, arg[j].w, x[uu][j].w, cc[uu]);
        }
      }
    }
  }
#pragma unroll
  for (int off = LPR; off < 32; off <<= 1)
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      float b2;
      int a2;
#define MERGE(F)                                           \
  b2 = __shfl_xor_sync(0xffffffffu, best[j].F, off);       \
  a2 = __shfl_xor_sync(0xffffffffu, arg[j].F, off);        \
  max_merge(best[j].F, arg[j].F, b2, a2);
      MERGE(x) MERGE(y) MERGE(z) MERGE(w)
#undef MERGE
    }
  if (slot != 0) return;
  const bool to_tf32 = (a.flags & MPH_EPI_TF32) != 0;
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int c4 = sub + j * LPR;
    if (c4 >= a.nv4) continue;
    reinterpret_cast<float4*>(a.out + (int64_t)row * a.ld_out)[c4] = to_tf32 ? f4_tf32(best[j]) : best[j];
    if (a.arg_out) reinterpret_cast<int4*>(a.arg_out + (int64_t)row * a.ld_arg)[c4] = arg[j];
  }
}

template <int LPR, int VPL, int U>
__device__ __forceinline__ void maxbwd_row(const MaxArgs& a, int row, int lane) {
  constexpr int ES = 32 / LPR;
  const int slot = lane / LPR, sub = lane % LPR;
  const int64_t s = a.row_ptr[row], e = a.row_ptr[row + 1];
  float4 acc[VPL];
#pragma unroll
  for (int j = 0; j < VPL; ++j) acc[j] = f4_zero();
  for (int64_t base = s; base < e; base += 32) {
    const int nb = (int)min((int64_t)32, e - base);
    const int my_c = (base + lane < e) ? ldg_stream_i32(a.col + base + lane) : 0;
    for (int k0 = 0; k0 < nb; k0 += U * ES) {
      float4 x[U][VPL];
      int4 ar[U][VPL];
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        const int k = k0 + uu * ES + slot;
        const int u = __shfl_sync(0xffffffffu, my_c, k & 31);
        const float4* p = reinterpret_cast<const float4*>(a.in + (int64_t)u * a.ld_in) + sub;
        const int4* q = reinterpret_cast<const int4*>(a.arg + (int64_t)u * a.ld_arg) + sub;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const bool ok = k < nb && sub + j * LPR < a.nv4;
          x[uu][j] = ok ? ldg_f4(p + j * LPR) : f4_zero();
          ar[uu][j] = ok ? __ldg(q + j * LPR) : make_int4(-1, -1, -1, -1);
        }
      }
#pragma unroll
      for (int uu = 0; uu < U; ++uu)
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          acc[j].x += ar[uu][j].x == row ? x[uu][j].x : 0.0f;
          acc[j].y += ar[uu][j].y == row ? x[uu][j].y : 0.0f;
          acc[j].z += ar[uu][j].z == row ? x[uu][j].z : 0.0f;
          acc[j].w += ar[uu][j].w == row ? x[uu][j].w : 0.0f;
        }
    }
  }
#pragma unroll
  for (int off = LPR; off < 32; off <<= 1)
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      acc[j].x += __shfl_xor_sync(0xffffffffu, acc[j].x, off);
      acc[j].y += __shfl_xor_sync(0xffffffffu, acc[j].y, off);
      acc[j].z += __shfl_xor_sync(0xffffffffu, acc[j].z, off);
      acc[j].w += __shfl_xor_sync(0xffffffffu, acc[j].w, off);
    }
  if (slot != 0) return;
  const bool to_tf32 = (a.flags & MPH_EPI_TF32) != 0;
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int c4 = sub + j * LPR;
    if (c4 >= a.nv4) continue;
    float4 v = acc[j];
    if (a.flags & MPH_EPI_MASK) {  // ReLU'(H_{l-1}) (Q8) and the dropout keep scale
      const float4 m = reinterpret_cast<const float4*>(a.mask_src + (int64_t)row * a.ld_mask)[c4];
      v.x = m.x > 0.0f ? v.x * a.mask_scale : 0.0f;
      v.y = m.y > 0.0f ? v.y * a.mask_scale : 0.0f;
      v.z = m.z > 0.0f ? v.z * a.mask_scale : 0.0f;
      v.w = m.w > 0.0f ? v.w * a.mask_scale : 0.0f;
    }
    reinterpret_cast<float4*>(a.out + (int64_t)row * a.ld_out)[c4] = to_tf32 ? f4_tf32(v) : v;
  }
}

template <int LPR, int VPL, bool BWD>
__global__ void __launch_bounds__(256) k_aggmax(MaxArgs a) {
  const int lane = threadIdx.x & 31;
  while (true) {
    int it = 0;
    if (lane == 0) it = atomicAdd(a.counter, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= a.n_items) break;
    const int2 rr = a.items[it];
    constexpr int U = VPL == 1 ? 8 : (VPL == 2 ? 4 : 2);
    for (int row = rr.x; row < rr.y; ++row) {
      if (BWD)
        maxbwd_row<LPR, VPL, U>(a, row, lane);
      else
        max_row<LPR, VPL, U>(a, row, lane);
    }
  }
}

template <int LPR, int VPL, bool BWD>
static int launch_max(const MaxArgs& a, cudaStream_t s) {
  static int blocks_per_sm = 0, sms = 0;
  if (!blocks_per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_aggmax<LPR, VPL, BWD>, 256, 0);
    blocks_per_sm = std::max(1, blocks_per_sm);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t grid = std::min<int64_t>((int64_t)sms * blocks_per_sm, ceil_div(a.n_items, 8));
  MPH_CUDA_TRY(cudaMemsetAsync(a.counter, 0, sizeof(int), s));
  k_aggmax<LPR, VPL, BWD><<<(unsigned)std::max<int64_t>(1, grid), 256, 0, s>>>(a);
  count_launch();
  return launch_check(BWD ? "aggregate_max_backward" : "aggregate_max");
}

template <bool BWD>
static int dispatch_max(const MaxArgs& a, cudaStream_t s) {
  const int nv4 = a.nv4;
  if (nv4 <= 1) return launch_max<1, 1, BWD>(a, s);
  if (nv4 <= 2) return launch_max<2, 1, BWD>(a, s);
  if (nv4 <= 4) return launch_max<4, 1, BWD>(a, s);
  if (nv4 <= 8) return launch_max<8, 1, BWD>(a, s);
  if (nv4 <= 16) return launch_max<16, 1, BWD>(a, s);
  if (nv4 <= 32) return launch_max<32, 1, BWD>(a, s);
  if (nv4 <= 64) return launch_max<32, 2, BWD>(a, s);
  if (nv4 <= 96) return launch_max<32, 3, BWD>(a, s);
  return launch_max<32, 4, BWD>(a, s);
}

static int check_common(const mph_graph* g, const float* in, int w, int ld_in, const float* out, int ld_out,
                        const char* what, int w_max) {
  if (!g || !in || !out) return fail(MPH_EINVAL, "%s: null argument", what);
  if (w <= 0 || w % 4 || ld_in % 4 || ld_out % 4 || ld_in < w || ld_out < w || w > w_max)
    return fail(MPH_EINVAL, "%s: w, ld_in, ld_out must be multiples of 4 with ld >= w, w <= %d (w=%d)", what, w_max,
                w);
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(MPH_EINVAL, "%s: operands must be 16-byte aligned", what);
  if (g->local && g->world > 1) return fail(MPH_ENOTSUP, "%s: max aggregation is single-GPU", what);
  return MPH_OK;
}

int aggregate_max_launch(const mph_graph* g, const float* in, int w, int ld_in, float* out, int ld_out, int32_t* arg,
                         int ld_arg, const mph_epilogue* epi, cudaStream_t s) {
  MPH_TRY(check_common(g, in, w, ld_in, out, ld_out, "aggregate_max", 1 << 20));
  if (arg && (ld_arg % 4 || ld_arg < w || (reinterpret_cast<uintptr_t>(arg) & 15)))
    return fail(MPH_EINVAL, "aggregate_max: arg must be 16-byte aligned with ld_arg >= w, multiple of 4");
  if (epi && (epi->flags & ~MPH_EPI_TF32)) return fail(MPH_EINVAL, "aggregate_max: only the TF32 epilogue flag");
  if (g->n_rows == 0) return MPH_OK;
  MPH_TRY(ensure_graph_items(g, s));
  for (int c0 = 0; c0 < w; c0 += 512) {  // column slabs of <= 512 (wide raw features, e.g. Y_1 = MAX(X))
    MaxArgs a{};
    a.row_ptr = g->row_ptr;
    a.col = g->col_idx;
    a.in = in + c0;
    a.out = out + c0;
    a.arg_out = arg ? arg + c0 : nullptr;
    a.items = g->items;
    a.counter = g->item_counter;
    a.n_items = g->n_items;
    a.nv4 = std::min(512, w - c0) / 4;
    a.ld_in = ld_in;
    a.ld_arg = ld_arg;
    a.ld_out = ld_out;
    a.flags = epi ? epi->flags : 0u;
    MPH_TRY(dispatch_max<false>(a, s));
  }
  return MPH_OK;
}

int aggregate_max_backward_launch(const mph_graph* g, const float* dY, int w, int ld_dy, const int32_t* arg, int ld_arg,
                                  float* dH, int ld_out, const mph_epilogue* epi, cudaStream_t s) {
  MPH_TRY(check_common(g, dY, w, ld_dy, dH, ld_out, "aggregate_max_backward", 512));
  if (!arg || ld_arg % 4 || ld_arg < w || (reinterpret_cast<uintptr_t>(arg) & 15))
    return fail(MPH_EINVAL, "aggregate_max_backward: arg must be 16-byte aligned with ld_arg >= w, multiple of 4");
  if (epi && (epi->flags & ~(MPH_EPI_TF32 | MPH_EPI_MASK)))
    return fail(MPH_EINVAL, "aggregate_max_backward: only the MASK and TF32 epilogue flags");
  if (epi && (epi->flags & MPH_EPI_MASK) &&
      (!epi->mask_src || epi->ld_mask % 4 || (reinterpret_cast<uintptr_t>(epi->mask_src) & 15)))
    return fail(MPH_EINVAL, "aggregate_max_backward: mask_src must be 16-byte aligned, ld_mask multiple of 4");
  if (g->n_rows == 0) return MPH_OK;
  MPH_TRY(ensure_graph_items(g, s));
  MaxArgs a{};
  a.row_ptr = g->row_ptr;
  a.col = g->col_idx;
  a.in = dY;
  a.arg = arg;
  a.out = dH;
  a.items = g->items;
  a.counter = g->item_counter;
  a.n_items = g->n_items;
  a.nv4 = w / 4;
  a.ld_in = ld_dy;
  a.ld_arg = ld_arg;
  a.ld_out = ld_out;
  a.flags = epi ? epi->flags : 0u;
  a.mask_src = epi ? epi->mask_src : nullptr;
  a.ld_mask = epi ? epi->ld_mask : 0;
  a.mask_scale = epi ? epi->mask_scale : 1.0f;
  return dispatch_max<true>(a, s);
}

// Column sums of rows [128·b, 128·b + 128) into partial row b (the same [ceil(rows/128)][cols]
// layout as the GEMM COLSUM epilogue; mph_reduce_rows then sums the partials in order).
__global__ void k_colsum_chunks(const float* in, int rows, int cols, int ld, float* part) {
  const int b = blockIdx.x;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    float s = 0.0f;
    const int r1 = min(rows, (b + 1) * 128);
    for (int r = b * 128; r < r1; ++r) s += in[(int64_t)r * ld + c];
    part[(int64_t)b * cols + c] = s;
  }
}

int colsum_chunks_launch(const float* in, int rows, int cols, int ld, float* part, cudaStream_t s) {
  if (rows == 0) return MPH_OK;
  k_colsum_chunks<<<(unsigned)ceil_div(rows, 128), 256, 0, s>>>(in, rows, cols, ld, part);
  count_launch();
  return launch_check("colsum_chunks");
}

int agg_scales(const mph_graph* g, int scheme, int transpose, const float** pre, const float** post) {
  switch (scheme) {
    case MPH_AGG_GCN:
      *pre = g->dinv;
      *post = g->dinv;
      return MPH_OK;
    case MPH_AGG_SUM:
      *pre = nullptr;
      *post = nullptr;
      return MPH_OK;
    case MPH_AGG_MEAN:
      *pre = transpose ? g->dinv1 : nullptr;
      *post = transpose ? nullptr : g->dinv1;
      return MPH_OK;
    default:
      return fail(MPH_EINVAL, "not a linear aggregation scheme: %d", scheme);
  }
}

}  // namespace mph

extern "C" int mph_graph_agg_scales(const mph_graph* g, int32_t scheme, int32_t transpose, const float** pre_d,
                                    const float** post_d) {
  if (!g) return mph::fail(MPH_EINVAL, "null graph");
  const float *pre = nullptr, *post = nullptr;
  MPH_TRY(mph::agg_scales(g, scheme, transpose, &pre, &post));
  if (pre_d) *pre_d = pre;
  if (post_d) *post_d = post;
  return MPH_OK;
}

extern "C" int mph_aggregate(const mph_graph* g, int32_t scheme, int32_t transpose, const float* in_d, int32_t w,
                             int32_t ld_in, float* out_d, int32_t ld_out, const mph_epilogue* epi, void* stream) {
  if (!g) return mph::fail(MPH_EINVAL, "null graph");
  const float *pre = nullptr, *post = nullptr;
  MPH_TRY(mph::agg_scales(g, scheme, transpose, &pre, &post));
  return mph::spmm_launch(g, -1, in_d, w, ld_in, out_d, ld_out, epi, post, (cudaStream_t)stream);
}

extern "C" int mph_aggregate_max(const mph_graph* g, const float* in_d, int32_t w, int32_t ld_in, float* out_d,
                                 int32_t ld_out, int32_t* arg_d, int32_t ld_arg, const mph_epilogue* epi, void* stream) {
  return mph::aggregate_max_launch(g, in_d, w, ld_in, out_d, ld_out, arg_d, ld_arg, epi, (cudaStream_t)stream);
}

extern "C" int mph_aggregate_max_backward(const mph_graph* g, const float* dY_d, int32_t w, int32_t ld_dy,
                                          const int32_t* arg_d, int32_t ld_arg, float* dH_d, int32_t ld_out,
                                          const mph_epilogue* epi, void* stream) {
  return mph::aggregate_max_backward_launch(g, dY_d, w, ld_dy, arg_d, ld_arg, dH_d, ld_out, epi,
                                            (cudaStream_t)stream);
}
