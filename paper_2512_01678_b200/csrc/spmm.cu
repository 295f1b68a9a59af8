// a3/a6 — aggregation SpMM with fused epilogue (Alg. 3; fused message passing
// without |E|xF buffers P:361; T_comp ∝ Σ deg·F P:550-555).
//
// B200 design (differs from the paper's block-per-row):
//  * one warp per output row.  The row's width is covered by LPR lanes holding VPL float4
//    each; the remaining 32/LPR "edge slots" walk different neighbours of the same row, so
//    all 32 lanes stay busy for every width (48-wide rows: 4 lanes x 3 float4 x 8 slots) and
//    every warp-wide load moves up to 512 B.
//  * neighbour ids are read 32 at a time with one coalesced 128 B load (L1 no-allocate); the
//    next 32 are prefetched while the current ones are gathered; each lane issues U×VPL
//    independent 16 B gathers before it consumes any.
//  * persistent warps pull work items from a global counter.  A work item is a run of
//    consecutive rows holding about the same number of edges (built once per graph), so the
//    power-law degree skew (Reddit hubs have 20x the mean degree) never idles a warp the way
//    a block-per-row grid does.  Two item lists: hub-first whole rows (items holding a hub row
//    are served first, so the longest rows start at t = 0 instead of forming the tail), and,
//    for whole-row launches of rows >= 64 wide whose gathered operand exceeds L2/2 (products),
//    a chunked virtual CSR walked in row order: rows longer than S = 256 edges cut into chunks, their partial rows
//    added in chunk order by k_spmm_combine, so the rows gathered at any moment stay a narrow
//    window of the graph and its L2 hits are kept.  Either way the summation order
//    of every row is fixed (deterministic).
//  * per-edge values are pre-scaled by dinv at the producer (T' = dinv ⊙ T), so the kernel
//    reads no per-edge weight: out[u] = dinv[u] · Σ_v T'[v]  ==  (Â·T)[u]  (Q1).
//  * partial sums: a pairwise tree over each group of U gathers, a running sum per slot,
//    and a fixed xor-shuffle tree across slots.
//  * epilogue fused: dinv, bias, ReLU, inverted dropout (Philox, Q10), row scale, TF32 store.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "internal.cuh"

namespace mph {

struct EpiDev {
  uint32_t flags;
  const float* bias;
  const float* row_scale;
  Dropout drop;
  int64_t row0;
  int c4_0;  // float4-column offset of this launch inside the full row (dropout counter)
};

struct SpmmArgs {
  const int64_t* row_ptr;
  const int64_t* row_end;  // row r's entries end at row_end[r] (row_ptr + 1, or a part's virtual row ends)
  int64_t col_len;         // entries in col (the id prefetch never reads past it)
  int contig;              // 1: whole-row launch over the graph's CSR (rows run contiguously through col)
  const int64_t* split;
  const int32_t* col;
  const float* val;   // per-edge values (HAS_VAL kernels only)
  const float* dinv;  // output row scale (nullptr: 1)
  const float* in;
  float* out;
  const int2* items;  // [first_row, end_row) per work item (hubs first), or {-1 - chunk, 0} (split items)
  int* counter;
  int n_items;
  int ld_in, ld_out, n_rows, nv4, part;
  int row_slots;   // 1: narrow rows of a low-degree graph -> k_spmm_rows
  int mid_degree;  // 1: mean degree in [16, 64) (dispatch of 48-wide rows)
  const float* partial;  // part 1 with a BF16 output: part 0's FP32 sums (row stride nv4·4), else nullptr
  uint32_t* bits_out;    // SIGNBITS: sign nibbles, one byte per float4 column, [rows][ld_bits] bytes
  int ld_bits;
  // whole-row launches over the chunked virtual CSR (build_split_items): row_ptr is the virtual
  // row_ptr, vmap[v] the output row of virtual row v, or -1 - chunk for a chunk of a cut row
  const int* vmap;
  float4* chunk_part;    // [chunk][kChunkPartF4] partial row sums
  EpiDev epi;
};

constexpr int kChunkPartF4 = 128;  // float4 per chunk partial: the widest launch (512 columns)

__device__ __forceinline__ float4 apply_dropout(float4 v, const Dropout& d, int64_t grow, int c4) {
  const uint32_t ep = d.epoch_dev ? (uint32_t)*d.epoch_dev : d.epoch;
  PhiloxOut r = philox4x32_10((uint32_t)grow, (uint32_t)c4, d.layer, ep, d.key0, d.key1);
  v.x = r.v[0] >= d.threshold ? v.x * d.scale : 0.0f;
  v.y = r.v[1] >= d.threshold ? v.y * d.scale : 0.0f;
  v.z = r.v[2] >= d.threshold ? v.z * d.scale : 0.0f;
  v.w = r.v[3] >= d.threshold ? v.w * d.scale : 0.0f;
  return v;
}

// Fused epilogue of one aggregated row: the LPR lanes of a slot hold acc[j] = columns
// 4·(sub + j·LPR) .. +3.  part 0 stores raw sums; part 1 adds them to part 0's; then dinv, bias,
// ReLU, dropout, row scale, TF32 (Q1, Q6, Q8, Q10).
constexpr int64_t kRowSlotMaxDegree = 16;  // mean degree (incl. self loop) below which k_spmm_rows serves w <= 64 (arxiv -7 %; products at 26 is 5 % slower with it)

template <int LPR, int VPL, bool SGN = false>
__device__ __forceinline__ void store_row(const SpmmArgs& a, int row, int sub, const float4 (&acc)[VPL], float du,
                                          float rs, uint64_t pol) {
  float4* orow = reinterpret_cast<float4*>(a.out + (int64_t)row * a.ld_out);
  if (a.part == 0) {
#pragma unroll
    for (int j = 0; j < VPL; ++j)
      if (sub + j * LPR < a.nv4) orow[sub + j * LPR] = acc[j];
    return;
  }
  const bool to_tf32 = (a.epi.flags & MPH_EPI_TF32) != 0;
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int c4 = sub + j * LPR;
    if (c4 >= a.nv4) continue;
    float4 v = acc[j];
    if (a.part == 1)
      v = f4_add(v, a.partial ? reinterpret_cast<const float4*>(a.partial + (int64_t)row * a.nv4 * 4)[c4] : orow[c4]);
    v.x *= du;
    v.y *= du;
    v.z *= du;
    v.w *= du;
    if (a.epi.flags & MPH_EPI_BIAS) {
      float4 b = reinterpret_cast<const float4*>(a.epi.bias)[c4];
      v = f4_add(v, b);
    }
    if (a.epi.flags & MPH_EPI_RELU) {
      v.x = fmaxf(v.x, 0.0f);
      v.y = fmaxf(v.y, 0.0f);
      v.z = fmaxf(v.z, 0.0f);
      v.w = fmaxf(v.w, 0.0f);
    }
    if (a.epi.flags & MPH_EPI_DROPOUT) v = apply_dropout(v, a.epi.drop, a.epi.row0 + row, a.epi.c4_0 + c4);
    if (a.epi.flags & MPH_EPI_ROWSCALE) {
      v.x *= rs;
      v.y *= rs;
      v.z *= rs;
      v.w *= rs;
    }
    uint32_t nib;  // SGN: the 4 sign bits of the stored values, one byte per float4 (MPH_EPI_SIGNBITS)
    if (a.epi.flags & MPH_EPI_BF16) {  // BF16 row (only feeds BF16 GEMMs); out/ld_out in bf16 elements
      uint2* o16 = reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(a.out) + (int64_t)row * a.ld_out);
      const uint2 q = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
      o16[c4] = q;
      nib = (uint32_t)bf16_positive(q.x & 0xFFFFu) | ((uint32_t)bf16_positive(q.x >> 16) << 1) |
            ((uint32_t)bf16_positive(q.y & 0xFFFFu) << 2) | ((uint32_t)bf16_positive(q.y >> 16) << 3);
    } else {
      const float4 st = to_tf32 ? f4_tf32(v) : v;
      st_f4_hint(orow + c4, st, pol);
      nib = (uint32_t)(st.x > 0.0f) | ((uint32_t)(st.y > 0.0f) << 1) | ((uint32_t)(st.z > 0.0f) << 2) |
            ((uint32_t)(st.w > 0.0f) << 3);
    }
    if (SGN) reinterpret_cast<uint8_t*>(a.bits_out)[(int64_t)row * a.ld_bits + a.epi.c4_0 + c4] = (uint8_t)nib;
  }
}

// Accumulation budget for long rows (a hub row is summed in at least
// ⌈deg/256⌉ independent partial sums).  Each slot sums the edges of one block of kHubBlock
// consecutive CSR entries on its own (a pairwise tree per group of U, then a running sum of
// ≤ kHubBlock/(ES·U) groups), the finished blocks are added in block order, and the ES slot
// totals meet in the fixed xor tree: a degree-9,477 Reddit hub (2 slots, U = 8) takes
// ≈ 16 + 3 + 38 + 1 sequential FP32 additions instead of ≈ 590.  Rows of at most kHubBlock
// edges keep the plain single-block sum.  Alg. 3 P:373-384 (the per-row sum), P:357 (skew).
constexpr int64_t kHubBlock = 256;

// Sum of the gathered rows of CSR entries [s, e) (one row, or one chunk of a long row): on return
// every lane holds the total of its columns sub + j·LPR (slot partials met in the xor tree).
template <int LPR, int VPL, bool HAS_VAL, int UOV, bool PK, bool CARRY = false>
__device__ __forceinline__ void spmm_sum(const SpmmArgs& a, int64_t s, int64_t e, int lane, float4 (&acc)[VPL],
                                         int& carry, bool have) {
  constexpr int ES = 32 / LPR;
  // U gathers per slot in flight; U*VPL float4 loads per lane before the first use
  constexpr int U0 = (32 / ES) < 8 ? (32 / ES) : 8;
  constexpr int U = UOV > 0 ? UOV : ((U0 * VPL > 8) ? ((8 / VPL) < 2 ? 2 : (8 / VPL)) : U0);
  const int slot = lane / LPR, sub = lane % LPR;
  // acc sums the current block of kHubBlock edges; tot the finished blocks, in block order
  float4 tot[VPL];
#pragma unroll
  for (int j = 0; j < VPL; ++j) acc[j] = tot[j] = f4_zero();
  const uint64_t pol = l2_policy_evict_first();
  const int* vbits = reinterpret_cast<const int*>(a.val);
  // the row's first 32 ids: carried over from the previous row of a contiguous run (its last block
  // prefetched them), else loaded now
  int nxt = (CARRY && have) ? carry : ((s + lane < e) ? ldg_stream_i32_hint(a.col + s + lane, pol) : 0);
  int nxv = (HAS_VAL && s + lane < e) ? ldg_stream_i32_hint(vbits + s + lane, pol) : 0;
  int64_t blk_end = s + kHubBlock;
  for (int64_t base = s; base < e; base += 32) {
    if (base == blk_end) {  // close a block (rows longer than kHubBlock edges only)
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        tot[j] = f4_add(tot[j], acc[j]);
        acc[j] = f4_zero();
      }
      blk_end += kHubBlock;
    }
    const int nb = (int)min((int64_t)32, e - base);
    const int my_c = nxt;
    const float my_v = __int_as_float(nxv);
    // prefetch the next 32 ids: the rest of this row, or (last block) the next row's first ids when
    // rows run contiguously through col_idx (whole-row launches: a run of rows, or the chunked CSR)
    if constexpr (CARRY) {
      const int64_t pb = base + 32 < e ? base + 32 : e;
      nxt = (pb + lane < a.col_len) ? ldg_stream_i32_hint(a.col + pb + lane, pol) : 0;
    } else {
      nxt = (base + 32 + lane < e) ? ldg_stream_i32_hint(a.col + base + 32 + lane, pol) : 0;
    }
    if (HAS_VAL) nxv = (base + 32 + lane < e) ? ldg_stream_i32_hint(vbits + base + 32 + lane, pol) : 0;
    for (int k0 = 0; k0 < nb; k0 += ES * U) {
      float4 x[U][VPL];
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        const int k = k0 + uu * ES + slot;
        const int c = __shfl_sync(0xffffffffu, my_c, k & 31);
        const float4* p = reinterpret_cast<const float4*>(a.in + (int64_t)c * a.ld_in) + sub;
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          x[uu][j] = (k < nb && sub + j * LPR < a.nv4) ? ldg_f4(p + j * LPR) : f4_zero();
        if (HAS_VAL) {
          const float xv = __shfl_sync(0xffffffffu, my_v, k & 31);
#pragma unroll
          for (int j = 0; j < VPL; ++j) {
            x[uu][j].x *= xv;
            x[uu][j].y *= xv;
            x[uu][j].z *= xv;
            x[uu][j].w *= xv;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
#pragma unroll
        for (int w = 1; w < U; w <<= 1)
#pragma unroll
          for (int uu = 0; uu + w < U; uu += 2 * w) x[uu][j] = PK ? f4_add2(x[uu][j], x[uu + w][j]) : f4_add(x[uu][j], x[uu + w][j]);
        acc[j] = PK ? f4_add2(acc[j], x[0][j]) : f4_add(acc[j], x[0][j]);
      }
    }
  }
  if (CARRY) carry = nxt;  // the ids from position e on (the next row's first block in a contiguous run)
  if (e - s > kHubBlock) {
#pragma unroll
    for (int j = 0; j < VPL; ++j) acc[j] = f4_add(tot[j], acc[j]);
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
}

// One (virtual) row: its sum, then the fused epilogue by the slot-0 lanes.  Over the chunked
// virtual CSR of a whole-row launch (vmap != nullptr) a virtual row is either a whole row of the
// graph or chunk c of a long row (vmap = -1 - c: the sum of ≤ S consecutive CSR entries of it),
// whose partial row goes to chunk_part[c]; k_spmm_combine adds a row's chunk partials in chunk
// order after the launch and runs the epilogue, so every row's sum is fixed whatever order the
// chunks ran in (deterministic, no atomics, no fences).  Walking rows in row order with long rows
// cut this way keeps the rows gathered at any moment a narrow window of the graph;
// the per-row code is the same for both (a second copy of the gather loop costs its registers).
template <int LPR, int VPL, bool HAS_VAL, int UOV, bool SGN = false, bool PK = true, bool CARRY = false>
__device__ __forceinline__ void spmm_row(const SpmmArgs& a, int row, int lane, int& carry, bool have) {
  int64_t s = a.row_ptr[row], e = a.row_end[row];
  if (!a.vmap) {  // (a virtual CSR has its part's ranges built in)
    if (a.part == 0) e = a.split[row];
    if (a.part == 1) s = a.split[row];
  }
  float4 acc[VPL];
  spmm_sum<LPR, VPL, HAS_VAL, UOV, PK, CARRY>(a, s, e, lane, acc, carry, have);
  if (lane >= LPR) return;
  const int orow = (!HAS_VAL && a.vmap) ? a.vmap[row] : row;
  if (!HAS_VAL && orow < 0) {
    float4* part = a.chunk_part + (int64_t)(-1 - orow) * kChunkPartF4;
#pragma unroll
    for (int j = 0; j < VPL; ++j)
      if (lane + j * LPR < a.nv4) part[lane + j * LPR] = acc[j];
    return;
  }
  const float du = (a.part != 0 && a.dinv) ? a.dinv[orow] : 1.0f;
  const float rs = (a.part != 0 && (a.epi.flags & MPH_EPI_ROWSCALE)) ? a.epi.row_scale[orow] : 1.0f;
  store_row<LPR, VPL, SGN>(a, orow, lane, acc, du, rs, l2_policy_evict_first());
}

// 4 blocks (32 warps) per SM within the 64-register budget for the one-float4-per-lane shapes
// (the hub-block partials would otherwise cost a block per SM); 3 for the wider register tiles
template <int LPR, int VPL, bool HAS_VAL, int UOV, bool SGN = false, bool CARRY = false>
__global__ void __launch_bounds__(256, ((VPL == 1 || LPR == 4) ? 4 : 3)) k_spmm(SpmmArgs a) {
  const int lane = threadIdx.x & 31;
  while (true) {
    int it = 0;
    if (lane == 0) it = atomicAdd(a.counter, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= a.n_items) break;
    const int2 rr = a.items[it];
    int carry = 0;  // CARRY: row r + 1's entries start where row r's end (whole-row launch)
    for (int row = rr.x; row < rr.y; ++row)
      spmm_row<LPR, VPL, HAS_VAL, UOV, SGN, true, CARRY>(a, row, lane, carry, row > rr.x);
  }
}

// Row-slot variant for narrow rows on low-degree graphs (arxiv; products at w <= 64): the
// warp-per-row kernel spends its 32/LPR edge slots on ONE row, so a row of ~8-26 edges costs a
// row_ptr, an id and one or two gather latencies with most slots idle.  Here each slot of LPR
// lanes owns whole rows and the ES = 32/LPR slots of a warp work on ES different rows of the item
// at once.  A slot about to finish its row (last step) claims the item's next unclaimed row in the
// same step (claims in slot order through a ballot; the item's row bounds come from one coalesced
// load per 32 rows held across the warp's lanes), and loads that row's first neighbour ids, so
// its next step gathers immediately.  Per step a slot gathers U neighbours (U·VPL independent
// 16-byte loads per lane) whose ids were loaded one step earlier.  Every row is summed by one
// slot in edge order (pairwise tree per group of U): deterministic whatever the claim order.
template <int LPR, int VPL, int U, bool SGN = false>
__global__ void __launch_bounds__(256, 3) k_spmm_rows(SpmmArgs a) {
  constexpr int ES = 32 / LPR;
  constexpr int NID = (U + LPR - 1) / LPR;  // id registers per lane
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, slot = lane / LPR, sub = lane % LPR;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint64_t pol = l2_policy_evict_first();
  const bool scaled = a.part != 0;
  while (true) {
    int it = 0;
    if (lane == 0) it = atomicAdd(a.counter, 1);
    it = __shfl_sync(FULL, it, 0);
    if (it >= a.n_items) break;
    const int2 rr = a.items[it];
    if (rr.y - rr.x == 1) {  // a long row (> E edges) is an item of its own: all slots on it
      int carry = 0;
      spmm_row<LPR, VPL, false, 0, SGN, false>(a, rr.x, lane, carry, false);  // scalar adds: packed ones spill here
      continue;
    }
    int w0 = rr.x;  // row bounds window: lane i holds [ws, we) of row w0 + i
    int64_t ws = 0, we = 0;
    {
      const int r = w0 + lane;
      if (r < rr.y) {
        ws = __ldg(a.row_ptr + r);
        we = __ldg(a.row_ptr + r + 1);
        if (a.part == 0) we = __ldg(a.split + r);
        if (a.part == 1) ws = __ldg(a.split + r);
      }
    }
    int next = rr.x;
    int row = -1;  // this slot's current row (identical across the slot's lanes)
    int64_t s = 0, e = 0;
    float du = 1.0f, rs = 1.0f;
    int ids[NID];
#pragma unroll
    for (int k = 0; k < NID; ++k) ids[k] = 0;
    float4 acc[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) acc[j] = f4_zero();
    while (true) {
      // ---- claims: slots that are idle or on their last step take the next rows
      const bool want = row < 0 || s + U >= e;
      const unsigned need = __ballot_sync(FULL, want && sub == 0);
      const int n_need = __popc(need);
      if (next < rr.y && next + n_need > w0 + 32) {  // refill the bounds window (warp-uniform)
        w0 = next;
        const int r = w0 + lane;
        ws = we = 0;
        if (r < rr.y) {
          ws = __ldg(a.row_ptr + r);
          we = __ldg(a.row_ptr + r + 1);
          if (a.part == 0) we = __ldg(a.split + r);
          if (a.part == 1) ws = __ldg(a.split + r);
        }
      }
      const int avail = min(n_need, rr.y - next);
      int claim = (want && sub == 0 && __popc(need & lt_mask) < avail) ? next + __popc(need & lt_mask) : -1;
      claim = __shfl_sync(FULL, claim, slot * LPR);
      next += avail;
      const int src = claim >= 0 ? claim - w0 : 0;
      const int64_t ns = __shfl_sync(FULL, ws, src), ne = __shfl_sync(FULL, we, src);
      if (!__any_sync(FULL, row >= 0 || claim >= 0)) break;  // item done
      // ---- ids for the next step: the rest of this row, or the claimed row's first edges
      const bool cont = row >= 0 && !want;
      const int64_t nb = cont ? s + U : ns;
      const int64_t nend = cont ? e : ne;
      const bool nvalid = cont || claim >= 0;
      int nids[NID];
#pragma unroll
      for (int k = 0; k < NID; ++k) {
        const int64_t ei = nb + sub + (int64_t)k * LPR;
        nids[k] = (nvalid && ei < nend && sub + k * LPR < U) ? ldg_stream_i32_hint(a.col + ei, pol) : 0;
      }
      const float ndu = (claim >= 0 && scaled && a.dinv) ? __ldg(a.dinv + claim) : 1.0f;
      const float nrs = (claim >= 0 && scaled && (a.epi.flags & MPH_EPI_ROWSCALE)) ? __ldg(a.epi.row_scale + claim)
                                                                                   : 1.0f;
      // ---- this step's gathers: U neighbours of the current row
      float4 x[U][VPL];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = __shfl_sync(FULL, ids[u / LPR], slot * LPR + (u % LPR));
        const bool valid = row >= 0 && s + u < e;
        const float4* p = reinterpret_cast<const float4*>(a.in + (int64_t)c * a.ld_in) + sub;
#pragma unroll
        for (int j = 0; j < VPL; ++j) x[u][j] = (valid && sub + j * LPR < a.nv4) ? ldg_f4(p + j * LPR) : f4_zero();
      }
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
#pragma unroll
        for (int w = 1; w < U; w <<= 1)
#pragma unroll
          for (int uu = 0; uu + w < U; uu += 2 * w) x[uu][j] = f4_add(x[uu][j], x[uu + w][j]);
        acc[j] = f4_add(acc[j], x[0][j]);
      }
      // ---- a finished row is stored by its slot
      if (row >= 0 && want) {
        store_row<LPR, VPL, SGN>(a, row, sub, acc, du, rs, pol);
#pragma unroll
        for (int j = 0; j < VPL; ++j) acc[j] = f4_zero();
      }
      // ---- advance
      if (want) {
        row = claim;
        s = ns;
        e = ne;
        du = ndu;
        rs = nrs;
      } else {
        s += U;
      }
#pragma unroll
      for (int k = 0; k < NID; ++k) ids[k] = nids[k];
    }
  }
}

// The rows cut into chunks: one warp per row adds the row's chunk partials in chunk order (float4
// columns lane + 32·j) and runs the fused epilogue (store_row) exactly as an unsplit row would.
template <bool SGN>
__global__ void __launch_bounds__(256) k_spmm_combine(SpmmArgs a, const int4* srows, int n_srows) {
  const int lane = threadIdx.x & 31;
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  for (int r = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); r < n_srows; r += nwarps) {
    const int4 sr = srows[r];  // {row, first chunk, n chunks, -}
    float4 acc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j] = f4_zero();
    const float4* p = a.chunk_part + (int64_t)sr.y * kChunkPartF4;
    if (a.nv4 <= 32) {  // one float4 per lane: eight chunks' loads in flight, added in chunk order
      float4 v = f4_zero();
      int q = 0;
      for (; q + 8 <= sr.z; q += 8) {
        float4 x[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) x[t] = lane < a.nv4 ? p[(int64_t)(q + t) * kChunkPartF4 + lane] : f4_zero();
#pragma unroll
        for (int t = 0; t < 8; ++t) v = f4_add(v, x[t]);
      }
      if (q + 4 <= sr.z) {
        float4 x[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) x[t] = lane < a.nv4 ? p[(int64_t)(q + t) * kChunkPartF4 + lane] : f4_zero();
#pragma unroll
        for (int t = 0; t < 4; ++t) v = f4_add(v, x[t]);
        q += 4;
      }
      for (; q < sr.z; ++q) v = f4_add(v, lane < a.nv4 ? p[(int64_t)q * kChunkPartF4 + lane] : f4_zero());
      acc[0] = v;
    } else {
      for (int q = 0; q < sr.z; ++q, p += kChunkPartF4)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (lane + 32 * j < a.nv4) acc[j] = f4_add(acc[j], p[lane + 32 * j]);
    }
    const float du = a.dinv ? a.dinv[sr.x] : 1.0f;
    const float rs = (a.epi.flags & MPH_EPI_ROWSCALE) ? a.epi.row_scale[sr.x] : 1.0f;
    store_row<32, 4, SGN>(a, sr.x, lane, acc, du, rs, l2_policy_evict_first());
  }
}

Dropout make_dropout(const mph_epilogue* e) {
  Dropout d{};
  if (!e || !(e->flags & MPH_EPI_DROPOUT) || e->dropout_p <= 0.0f) {
    d.threshold = 0;
    d.scale = 1.0f;
    return d;
  }
  const double p = (double)e->dropout_p;
  d.threshold = (uint32_t)floor(p * 4294967296.0);
  d.scale = (float)(1.0 / (1.0 - p));
  d.key0 = (uint32_t)(e->dropout_seed & 0xffffffffull);
  d.key1 = (uint32_t)(e->dropout_seed >> 32);
  d.layer = (uint32_t)e->dropout_layer;
  d.epoch = (uint32_t)e->dropout_epoch;
  d.epoch_dev = e->dropout_epoch_d;
  return d;
}

// Work items (built once per graph, on the host from row_ptr): runs of consecutive rows of
// about E edges, E = nnz / (32 items per resident warp) clamped to [64, 512]; a row longer
// than E is an item of its own.  Items holding a row longer than 4E ("hubs") come first,
// longest first.
int build_work_items(const int64_t* row_ptr_d, int n_rows, int64_t nnz, int2** items_out, int* n_items,
                     cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // clamped to [64, 512]: reddit's E = 1010 -> 512 measured 0.8-2.3 % faster per call (a narrower
  // window of rows in flight; profiles/r02_experiments/spmm_item_edges_sweep.txt)
  int64_t kItemEdges = std::max<int64_t>(64, std::min<int64_t>(512, nnz / ((int64_t)sms * 24 * 32)));
  if (const char* ie = getenv("MPH_SPMM_ITEM_EDGES")) kItemEdges = std::max<int64_t>(8, atoll(ie));  // experiments
  std::vector<int64_t> rp((size_t)n_rows + 1);
  MPH_CUDA_TRY(cudaMemcpyAsync(rp.data(), row_ptr_d, rp.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  MPH_CUDA_TRY(cudaStreamSynchronize(s));
  std::vector<int2> hubs, rest;
  std::vector<int64_t> hub_len;
  int r0 = 0;
  int64_t acc = 0;
  for (int r = 0; r < n_rows; ++r) {
    const int64_t d = rp[r + 1] - rp[r];
    if (d > kItemEdges) {  // long row: flush the current run, then the row alone
      if (r > r0) rest.push_back(make_int2(r0, r));
      if (d > 4 * kItemEdges) {
        hubs.push_back(make_int2(r, r + 1));
        hub_len.push_back(d);
      } else {
        rest.push_back(make_int2(r, r + 1));
      }
      r0 = r + 1;
      acc = 0;
      continue;
    }
    acc += d;
    if (acc >= kItemEdges) {
      rest.push_back(make_int2(r0, r + 1));
      r0 = r + 1;
      acc = 0;
    }
  }
  if (r0 < n_rows) rest.push_back(make_int2(r0, n_rows));
  std::vector<size_t> order(hubs.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) { return hub_len[x] > hub_len[y]; });
  std::vector<int2> items;
  items.reserve(hubs.size() + rest.size());
  for (size_t i : order) items.push_back(hubs[i]);
  items.insert(items.end(), rest.begin(), rest.end());
  int2* d_items = nullptr;
  MPH_TRY(dev_alloc(&d_items, std::max<size_t>(items.size(), 1)));
  if (!items.empty()) {
    cudaError_t e = cudaMemcpyAsync(d_items, items.data(), items.size() * sizeof(int2), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      dev_free(d_items);
      return fail(MPH_ECUDA, "work items: %s", cudaGetErrorString(e));
    }
  }
  *items_out = d_items;
  *n_items = (int)items.size();
  return MPH_OK;
}

// The chunked virtual CSR of whole-row launches (part -1): every row longer than S edges is cut
// into ⌈deg/S⌉ virtual rows of ≤ S consecutive CSR entries (vrow_ptr indexes the graph's col_idx;
// vmap[v] = -1 - chunk), the other rows stay whole (vmap[v] = row), and the work items are runs of
// consecutive virtual rows of about S/2 edges, all in row order.  Walking the graph in row order
// keeps the rows gathered at any moment a narrow window (a community of the planted partition, the
// co-purchase clusters of products): with long rows as whole items, served first, the one warp on
// a hub keeps gathering long after the rest of the grid has moved on, and its hits become misses
// (LRU replay tools/sim/lru_items.c: 29 % of products' 128-wide gathers miss an 85 MB
// L2 with hub rows first, 16 % with chunks of 256; ncu: 10.8 -> 6.9 GB DRAM per launch).
// S = MPH_SPMM_CHUNK_EDGES, default min(E, 256) (E as in build_work_items).
static int build_split_items(mph_graph* g, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t E = std::max<int64_t>(64, std::min<int64_t>(2048, g->nnz / ((int64_t)sms * 24 * 32)));
  // graphs with fewer than 256 edges per item (E < 256: arxiv, 1.2 M edges) keep the hub-first
  // items: their SpMM measured 3 % slower on the chunked CSR
  if (E < 256 && g->split_mode != 2) return MPH_OK;
  int64_t S = std::min<int64_t>(E, 256);
  if (const char* ce = getenv("MPH_SPMM_CHUNK_EDGES")) S = std::max<int64_t>(32, atoll(ce));  // experiments
  std::vector<int64_t> rp((size_t)g->n_rows + 1), sp;
  MPH_CUDA_TRY(cudaMemcpyAsync(rp.data(), g->row_ptr, rp.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  if (g->local && g->split) {
    sp.resize((size_t)g->n_rows);
    MPH_CUDA_TRY(cudaMemcpyAsync(sp.data(), g->split, sp.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  }
  MPH_CUDA_TRY(cudaStreamSynchronize(s));
  int64_t max_chunks = 0;
  for (int part = -1; part <= (sp.empty() ? -1 : 1); ++part) {
    // the row range of this launch kind: whole rows, owned-column edges, ghost-column edges
    auto lo = [&](int r) { return part == 1 ? sp[r] : rp[r]; };
    auto hi = [&](int r) { return part == 0 ? sp[r] : rp[r + 1]; };
    std::vector<int64_t> vrp;
    std::vector<int> vmap;
    std::vector<int2> items;
    std::vector<int4> srows;  // {row, first chunk, n chunks, -}
    vrp.reserve((size_t)g->n_rows + 1);
    vmap.reserve((size_t)g->n_rows);
    int64_t n_chunks = 0;
    for (int r = 0; r < g->n_rows; ++r) {
      const int64_t d = hi(r) - lo(r);
      if (d > S) {
        const int nc = (int)((d + S - 1) / S);
        srows.push_back(make_int4(r, (int)n_chunks, nc, 0));
        for (int k = 0; k < nc; ++k) {
          vrp.push_back(lo(r) + (int64_t)k * S);
          vmap.push_back((int)(-1 - n_chunks));
          ++n_chunks;
        }
      } else {
        vrp.push_back(lo(r));
        vmap.push_back(r);
      }
    }
    // a virtual row ends where the next begins: the last one at the row range's end
    vrp.push_back(g->n_rows ? hi(g->n_rows - 1) : 0);
    if (vmap.size() > (size_t)INT32_MAX / 2) return fail(MPH_ENOTSUP, "spmm: %zu virtual rows", vmap.size());
    if (!n_chunks) continue;  // no row longer than S: the whole-row items serve as they are
    // part 0/1 ranges are not contiguous across rows (row r's range ends at split[r], row r+1's
    // starts at row_ptr[r+1]): their virtual rows keep explicit ends, so vrp holds begin/end pairs
    const int n_v = (int)vmap.size();
    std::vector<int64_t> vend((size_t)n_v);
    {
      int v = 0;
      for (int r = 0; r < g->n_rows; ++r) {
        const int64_t d = hi(r) - lo(r);
        if (d > S) {
          for (int64_t c = lo(r); c < hi(r); c += S) vend[v++] = std::min(c + S, hi(r));
        } else {
          vend[v++] = hi(r);
        }
      }
    }
    int v0 = 0;
    int64_t acc = 0;
    // edges per work item: half a chunk — a narrower window of rows in flight than items of S
    // (products per call: S/2 = 128 edges 4.62-4.64 ms vs 4.68-4.73 at 256, 5.0 at 512;
    // profiles/r02_experiments/spmm_chunked_csr.txt); MPH_SPMM_RUN_EDGES overrides (experiments)
    static const int64_t run_env = getenv("MPH_SPMM_RUN_EDGES") ? atoll(getenv("MPH_SPMM_RUN_EDGES")) : 0;
    const int64_t R = run_env > 0 ? run_env : std::max<int64_t>(32, S / 2);
    for (int v = 0; v < n_v; ++v) {
      acc += vend[v] - vrp[v];
      if (acc >= R) {
        items.push_back(make_int2(v0, v + 1));
        v0 = v + 1;
        acc = 0;
      }
    }
    if (v0 < n_v) items.push_back(make_int2(v0, n_v));
    // device layout: vrow_ptr = [begin_0 .. begin_{n_v-1}, end_0 .. end_{n_v-1}] for parts 0/1;
    // for whole rows (part -1) begin_{v+1} == end_v, so the plain n_v + 1 offsets suffice
    std::vector<int64_t> dev_vrp;
    if (part == -1) {
      dev_vrp = vrp;
    } else {
      dev_vrp.assign(vrp.begin(), vrp.begin() + n_v);
      dev_vrp.insert(dev_vrp.end(), vend.begin(), vend.end());
    }
    mph_graph::SplitCsr& c = g->scsr[part + 1];
    MPH_TRY(dev_alloc(&c.vrow_ptr, dev_vrp.size()));
    MPH_TRY(dev_alloc(&c.vmap, vmap.size()));
    MPH_TRY(dev_alloc(&c.items, std::max<size_t>(items.size(), 1)));
    MPH_TRY(dev_alloc(&c.srows, srows.size()));
    MPH_CUDA_TRY(cudaMemcpyAsync(c.vrow_ptr, dev_vrp.data(), dev_vrp.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    MPH_CUDA_TRY(cudaMemcpyAsync(c.vmap, vmap.data(), vmap.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    MPH_CUDA_TRY(cudaMemcpyAsync(c.items, items.data(), items.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
    MPH_CUDA_TRY(cudaMemcpyAsync(c.srows, srows.data(), srows.size() * sizeof(int4), cudaMemcpyHostToDevice, s));
    MPH_CUDA_TRY(cudaStreamSynchronize(s));
    c.n_items = (int)items.size();
    c.n_srows = (int)srows.size();
    c.n_chunks = n_chunks;
    c.n_vrows = n_v;
    max_chunks = std::max(max_chunks, n_chunks);
  }
  if (max_chunks) MPH_TRY(dev_alloc(&g->chunk_part, (size_t)max_chunks * kChunkPartF4));
  g->chunk_edges = (int)S;
  return MPH_OK;
}

// MPH_SPMM_SPLIT, read when a graph's items are built (setup): 0 off, 1 (default) when the gathered
// operand exceeds L2/2, 2 for every warp-per-row whole-row launch (tests)
static int split_mode_env() {
  const char* e = getenv("MPH_SPMM_SPLIT");
  return e ? atoi(e) : 1;
}

int ensure_graph_items(const mph_graph* gc, cudaStream_t s) {
  mph_graph* g = const_cast<mph_graph*>(gc);
  if (g->items) return MPH_OK;
  MPH_TRY(build_work_items(g->row_ptr, g->n_rows, g->nnz, &g->items, &g->n_items, s));
  g->split_mode = split_mode_env();
  if (g->split_mode) MPH_TRY(build_split_items(g, s));
  MPH_TRY(dev_alloc(&g->item_counter, 1));
  return MPH_OK;
}

template <int LPR, int VPL, bool HAS_VAL, int UOV = 0, bool SGN = false, bool CARRY = false>
static int launch_spmm(const SpmmArgs& a, cudaStream_t s) {
  static int blocks_per_sm = 0;
  static int sms = 0;
  if (!blocks_per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_spmm<LPR, VPL, HAS_VAL, UOV, SGN, CARRY>, 256, 0);
    blocks_per_sm = std::max(1, blocks_per_sm);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t grid = std::min<int64_t>((int64_t)sms * blocks_per_sm, ceil_div(a.n_items, 8));
  MPH_CUDA_TRY(cudaMemsetAsync(a.counter, 0, sizeof(int), s));
  k_spmm<LPR, VPL, HAS_VAL, UOV, SGN, CARRY><<<(unsigned)std::max<int64_t>(1, grid), 256, 0, s>>>(a);
  count_launch();
  return launch_check("spmm");
}


template <int LPR, int VPL, int U, bool SGN = false>
static int launch_spmm_rows(const SpmmArgs& a, cudaStream_t s) {
  static int blocks_per_sm = 0;
  static int sms = 0;
  if (!blocks_per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_spmm_rows<LPR, VPL, U, SGN>, 256, 0);
    blocks_per_sm = std::max(1, blocks_per_sm);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t grid = std::min<int64_t>((int64_t)sms * blocks_per_sm, ceil_div(a.n_items, 8));
  MPH_CUDA_TRY(cudaMemsetAsync(a.counter, 0, sizeof(int), s));
  k_spmm_rows<LPR, VPL, U, SGN><<<(unsigned)std::max<int64_t>(1, grid), 256, 0, s>>>(a);
  count_launch();
  return launch_check("spmm (row slots)");
}

static int env_int(const char* name) {
  const char* v = getenv(name);
  return v ? atoi(v) : 0;
}

// Per-shape unroll: 256-wide rows (32 lanes x 2 float4) gain from 8 gathers in flight per slot
// (measured with the round-1 unroll sweep, arxiv SpMM -8 %); every other shape is best at the
// default U.
template <int LPR, int VPL, bool HAS_VAL, bool SGN = false>
static int launch_spmm_u(const SpmmArgs& a, cudaStream_t s) {
  if constexpr (LPR == 32 && VPL == 2) return launch_spmm<LPR, VPL, HAS_VAL, 8, SGN>(a, s);
  else return launch_spmm<LPR, VPL, HAS_VAL, 0, SGN>(a, s);
}

template <bool HAS_VAL, bool SGN = false>
static int dispatch_spmm(const SpmmArgs& a, cudaStream_t s) {
  const int nv4 = a.nv4;
  if constexpr (!HAS_VAL && !SGN) {
    if (a.bits_out) return dispatch_spmm<false, true>(a, s);  // SIGNBITS: same maps, sign-byte store
  }
  if (!HAS_VAL && a.row_slots && nv4 <= 16) {  // narrow rows, low degree: several rows per warp
    if (nv4 <= 1) return launch_spmm_rows<1, 1, 4, SGN>(a, s);
    if (nv4 <= 2) return launch_spmm_rows<2, 1, 4, SGN>(a, s);
    if (nv4 <= 4) return launch_spmm_rows<4, 1, 4, SGN>(a, s);
    if (nv4 <= 8) return launch_spmm_rows<8, 1, 8, SGN>(a, s);
    if (nv4 <= 12) return launch_spmm_rows<4, 3, 4, SGN>(a, s);
    return launch_spmm_rows<16, 1, 8, SGN>(a, s);
  }
  if (nv4 <= 1) return launch_spmm<1, 1, HAS_VAL, 0, SGN>(a, s);
  if (nv4 <= 2) return launch_spmm<2, 1, HAS_VAL, 0, SGN>(a, s);
  if (nv4 <= 4) return launch_spmm<4, 1, HAS_VAL, 0, SGN>(a, s);
  if (nv4 <= 8) return launch_spmm<8, 1, HAS_VAL, 0, SGN>(a, s);
  if (nv4 <= 12) {
    // 48-wide rows: 4 lanes x 3 float4 (8 edge slots) where rows are long (reddit: the shuffle
    // reduction is amortised), 16 lanes x 1 float4 with 12 active (2 slots, a third of the
    // cross-slot reduction) at moderate degree (products, mean 26: -1.7 % epoch)
    if (a.mid_degree) {
      if constexpr (!HAS_VAL) {
        if (a.contig) return launch_spmm<16, 1, false, 0, SGN, true>(a, s);  // ids carried across rows
      }
      return launch_spmm_u<16, 1, HAS_VAL, SGN>(a, s);
    }
    return launch_spmm_u<4, 3, HAS_VAL, SGN>(a, s);
  }
  if (nv4 <= 16) return launch_spmm_u<16, 1, HAS_VAL, SGN>(a, s);
  if (nv4 <= 32) return launch_spmm_u<32, 1, HAS_VAL, SGN>(a, s);
  if (nv4 <= 64) return launch_spmm_u<32, 2, HAS_VAL, SGN>(a, s);
  if (nv4 <= 96) return launch_spmm<32, 3, HAS_VAL, 0, SGN>(a, s);
  return launch_spmm<32, 4, HAS_VAL, 0, SGN>(a, s);
}

// One whole-row launch: over the chunked virtual CSR when the gathered operand exceeds half of L2
// (what the window of concurrently walked rows buys is L2 hits; an L2-resident operand - reddit's
// 64-wide slabs, 60 MB - gains nothing and would pay for the chunk partials), its rows are at least
// 64 columns wide and the launch is a warp-per-row one, then the combine of the cut rows; otherwise
// over the hub-first whole-row items.
static int run_spmm(SpmmArgs a, const mph_graph* g, cudaStream_t s) {
  static int64_t l2_bytes = -1;
  if (l2_bytes < 0) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev);
    l2_bytes = v;
  }
  const bool rows_kernel = a.row_slots && a.nv4 <= 16;
  // rows narrower than 64 columns keep the hub-first items: products' 48-wide launch, issue-bound
  // rather than DRAM-bound, measured 2.6 % slower on the chunked CSR (1.489 vs 1.451 ms)
  const bool big = g->split_mode == 2 || ((int64_t)g->n_cols * a.nv4 * 16 > l2_bytes / 2 && a.nv4 >= 16);
  const mph_graph::SplitCsr& c = g->scsr[a.part + 1];
  const bool use_split = c.items && !rows_kernel && big;
  if (!use_split) {
    // carry each row's first ids over from the previous row's last block on graphs of moderate
    // degree (products' 48-wide rows, 26 edges each: 1.65 -> 1.52 ms); on reddit's long rows and
    // on the chunked CSR it measured 1-8 % slower
    a.contig = (a.part == -1 && a.mid_degree) ? 1 : 0;
    return dispatch_spmm<false>(a, s);
  }
  a.row_ptr = c.vrow_ptr;
  // whole rows: virtual row v ends where v + 1 begins; parts: explicit ends after the n_v begins
  a.row_end = a.part == -1 ? c.vrow_ptr + 1 : c.vrow_ptr + c.n_vrows;
  a.vmap = c.vmap;
  a.items = c.items;
  a.n_items = c.n_items;
  a.chunk_part = g->chunk_part;
  MPH_TRY(dispatch_spmm<false>(a, s));
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(c.n_srows, 8), 148 * 16);
  if (a.bits_out) k_spmm_combine<true><<<grid, 256, 0, s>>>(a, c.srows, c.n_srows);
  else k_spmm_combine<false><<<grid, 256, 0, s>>>(a, c.srows, c.n_srows);
  count_launch();
  return launch_check("spmm combine");
}

// MPH_EPI_SIGNBITS on mph_spmm: every lane map stores one sign byte per float4 column it owns.
bool spmm_signbits_ok(const mph_graph* g, int w) { return g && w > 0 && w % 4 == 0 && w <= 512; }

int spmm_launch(const mph_graph* g, int part, const float* in, int w, int ld_in, float* out, int ld_out,
                const mph_epilogue* epi, const float* post, cudaStream_t s, const float* partial) {
  if (!g || !in || !out) return fail(MPH_EINVAL, "spmm: null argument");
  if (w <= 0 || w % 4 || ld_in % 4 || ld_out % 4 || ld_in < w || ld_out < w)
    return fail(MPH_EINVAL, "spmm: w, ld_in, ld_out must be multiples of 4 with ld >= w (w=%d)", w);
  if (w > 512) return fail(MPH_ENOTSUP, "spmm: width %d > 512", w);
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(MPH_EINVAL, "spmm: operands must be 16-byte aligned");
  if (part != -1 && !g->local) return fail(MPH_EINVAL, "spmm: row parts need a localized graph");
  const uint32_t allowed = MPH_EPI_BIAS | MPH_EPI_RELU | MPH_EPI_DROPOUT | MPH_EPI_ROWSCALE | MPH_EPI_TF32 |
                           MPH_EPI_BF16 | MPH_EPI_SIGNBITS;
  if (epi && (epi->flags & ~allowed)) return fail(MPH_EINVAL, "spmm: unsupported epilogue flags 0x%x", epi->flags);
  if (epi && (epi->flags & MPH_EPI_BF16) && part != -1 && !(part == 1 && partial))
    return fail(MPH_ENOTSUP, "spmm: BF16 output needs whole rows (part -1), or part 1 over FP32 partial sums");
  if (epi && (epi->flags & MPH_EPI_BIAS) && (!epi->bias || (reinterpret_cast<uintptr_t>(epi->bias) & 15)))
    return fail(MPH_EINVAL, "spmm: bias must be non-null and 16-byte aligned");
  if (epi && (epi->flags & MPH_EPI_ROWSCALE) && !epi->row_scale) return fail(MPH_EINVAL, "spmm: null row_scale");
  if (epi && (epi->flags & MPH_EPI_SIGNBITS)) {
    if (!epi->bits_out || epi->ld_bits < w / 4) return fail(MPH_EINVAL, "spmm: SIGNBITS needs bits_out, ld_bits >= w/4");
    if (part == 0) return fail(MPH_EINVAL, "spmm: SIGNBITS on part 1 (or whole rows), not part 0");
  }
  if (g->n_rows == 0) return MPH_OK;
  MPH_TRY(ensure_graph_items(g, s));
  SpmmArgs a{};
  a.bits_out = (epi && (epi->flags & MPH_EPI_SIGNBITS)) ? epi->bits_out : nullptr;
  a.ld_bits = epi ? epi->ld_bits : 0;
  a.val = nullptr;
  a.row_ptr = g->row_ptr;
  a.row_end = g->row_ptr + 1;
  a.col_len = g->nnz;
  a.contig = 0;  // set per launch in run_spmm
  a.split = g->split;
  a.col = g->col_idx;
  a.dinv = post;
  a.in = in;
  a.out = out;
  a.items = g->items;
  a.counter = g->item_counter;
  a.n_items = g->n_items;
  a.ld_in = ld_in;
  a.ld_out = ld_out;
  a.n_rows = g->n_rows;
  a.nv4 = w / 4;
  a.part = part;
  a.partial = part == 1 ? partial : nullptr;
  a.epi.flags = epi ? (epi->flags & ~MPH_EPI_SIGNBITS) : 0u;
  a.epi.bias = epi ? epi->bias : nullptr;
  a.epi.row_scale = epi ? epi->row_scale : nullptr;
  a.epi.drop = make_dropout(epi);
  a.epi.row0 = epi ? epi->row0 : 0;
  if (a.epi.drop.threshold == 0) a.epi.flags &= ~MPH_EPI_DROPOUT;
  a.epi.c4_0 = 0;
  // Row slots (k_spmm_rows) for narrow rows when the mean degree is low; MPH_SPMM_ROWS=0/1 overrides.
  {
    const char* rs_env = getenv("MPH_SPMM_ROWS");
    const bool low_degree = g->nnz < kRowSlotMaxDegree * (int64_t)g->n_rows;
    a.row_slots = rs_env ? (atoi(rs_env) != 0) : low_degree;
    a.mid_degree = !low_degree && g->nnz < 64 * (int64_t)g->n_rows;
  }
  // Column slabs: on graphs with a mean degree >= 16, rows of w = 128 / 256 are aggregated as two
  // halves, one launch each, so the slab of the gathered operand that a community of rows
  // touches is half as large and stays in L2 (measured: products -1..4 %, reddit -2 %); on
  // sparse graphs the doubled per-row overhead costs more (arxiv, mean degree 7: +13 %).
  // MPH_SPMM_SLAB overrides (-1: off).
  static const int slab_env = env_int("MPH_SPMM_SLAB");
  const bool deep = g->nnz >= 16 * (int64_t)g->n_rows;
  const int slab = slab_env != 0 ? slab_env : ((deep && (w == 128 || w == 256)) ? w / 2 : 0);
  if (slab > 0 && part == -1 && w > slab && slab % 4 == 0) {
    for (int c0 = 0; c0 < w; c0 += slab) {
      SpmmArgs b = a;
      b.in = in + c0;
      b.out = (a.epi.flags & MPH_EPI_BF16) ? reinterpret_cast<float*>(reinterpret_cast<uint16_t*>(out) + c0) : out + c0;
      b.nv4 = std::min(slab, w - c0) / 4;
      if (b.epi.bias) b.epi.bias = a.epi.bias + c0;
      b.epi.c4_0 = c0 / 4;
      MPH_TRY(run_spmm(b, g, s));
    }
    return MPH_OK;
  }
  return run_spmm(a, g, s);
}

int spmm_csr_launch(const int64_t* row_ptr, const int32_t* col, const float* val, int n_rows, const int2* items,
                    int n_items, int* counter, const float* row_scale, const float* in, int w, int ld_in, float* out,
                    int ld_out, cudaStream_t s) {
  if (!row_ptr || !in || !out || (!items && n_items > 0) || !counter) return fail(MPH_EINVAL, "spmm_csr: null argument");
  if (w <= 0 || w % 4 || ld_in % 4 || ld_out % 4 || ld_in < w || ld_out < w || w > 512)
    return fail(MPH_EINVAL, "spmm_csr: bad width %d", w);
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(MPH_EINVAL, "spmm_csr: operands must be 16-byte aligned");
  if (n_rows == 0 || n_items == 0) return MPH_OK;
  SpmmArgs a{};
  a.row_ptr = row_ptr;
  a.row_end = row_ptr + 1;
  a.col_len = 0;
  a.contig = 0;  // (X_csr / X_csc-segment launches: no cross-row id prefetch)
  a.split = nullptr;
  a.col = col;
  a.val = val;
  a.dinv = row_scale;
  a.in = in;
  a.out = out;
  a.items = items;
  a.counter = counter;
  a.n_items = n_items;
  a.ld_in = ld_in;
  a.ld_out = ld_out;
  a.n_rows = n_rows;
  a.nv4 = w / 4;
  a.part = -1;
  a.epi.flags = 0u;
  a.epi.drop = make_dropout(nullptr);
  return val ? dispatch_spmm<true>(a, s) : dispatch_spmm<false>(a, s);
}

__global__ void k_pack_rows(const int32_t* ids, int64_t n, const float* buf, int ld, int nv4, float* out) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n; j += nwarps) {
    const float4* src = reinterpret_cast<const float4*>(buf + (int64_t)ids[j] * ld);
    float4* dst = reinterpret_cast<float4*>(out + j * (int64_t)nv4 * 4);
    for (int c = lane; c < nv4; c += 32) dst[c] = ldg_f4(src + c);
  }
}

int pack_rows(const int32_t* ids, int64_t n, const float* buf, int ld, int w, float* out, cudaStream_t s) {
  if (n == 0) return MPH_OK;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, 8), 148 * 64);
  k_pack_rows<<<grid, 256, 0, s>>>(ids, n, buf, ld, w / 4, out);
  count_launch();
  return launch_check("pack_rows");
}

}  // namespace mph

extern "C" int mph_spmm(const mph_graph* g, const float* in_d, int32_t w, int32_t ld_in, float* out_d, int32_t ld_out,
                        const mph_epilogue* epi, void* stream) {
  if (!g) return mph::fail(MPH_EINVAL, "spmm: null argument");
  return mph::spmm_launch(g, -1, in_d, w, ld_in, out_d, ld_out, epi, g->dinv, (cudaStream_t)stream);
}

extern "C" int mph_spmm_part(const mph_graph* g, int32_t part, const float* in_d, int32_t w, int32_t ld_in, float* out_d,
                             int32_t ld_out, const mph_epilogue* epi, void* stream) {
  if (part < -1 || part > 1) return mph::fail(MPH_EINVAL, "spmm_part: part must be -1, 0 or 1");
  if (!g) return mph::fail(MPH_EINVAL, "spmm: null argument");
  return mph::spmm_launch(g, part, in_d, w, ld_in, out_d, ld_out, epi, g->dinv, (cudaStream_t)stream);
}

extern "C" int mph_spmm_signbits_ok(const mph_graph* g, int32_t w, int32_t* ok_h) {
  if (!g || !ok_h) return mph::fail(MPH_EINVAL, "spmm_signbits_ok: null argument");
  *ok_h = mph::spmm_signbits_ok(g, w) ? 1 : 0;
  return MPH_OK;
}
