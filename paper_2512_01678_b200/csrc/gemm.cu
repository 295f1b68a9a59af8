// a2/a4/a7/a8 — dense transforms on 5th-gen tensor cores (tcgen05, TF32 in, FP32 accumulate
// in TMEM), TMA-fed through a multi-stage mbarrier pipeline ("dense, regular";
// P:221 vendor GEMM replaced by hand-written sm_100a kernels).
//
//   k_gemm_nt : C[M,N] = epi(A[M,K] · Bt[N,K]^T)   both operands K-major (activations x weights)
//               one CTA per 128-row stripe and the whole N <= 256 width, so A streams from HBM
//               exactly once; warp 0 = TMA producer, warp 1 = MMA issuer (one thread) and
//               TMEM owner, warps 2-5 = epilogue (tcgen05.ld -> fused epilogue -> global).
//   k_gemm_tn : P_s[M,N] = A[K_s,M]^T · B[K_s,N]   contraction over nodes (weight gradient),
//               both operands MN-major in shared memory; split-K over node ranges, FP32 partials
//               reduced afterwards in a fixed order (deterministic; "thread-local buffers
//               before a final reduction", without the paper's atomics P:361).
//
// These GEMMs are HBM-bound at GCN shapes (arithmetic intensity 15-64 flop/B < TF32 ridge,
// SURVEY §8(d) d.2): the design goal is streaming A at full bandwidth.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace mph {

Dropout make_dropout(const mph_epilogue* e);

namespace {

constexpr int kBM = 128;          // UMMA M (rows per CTA tile)
constexpr int kBK = 32;           // fp32 elements per 128 B swizzle row
constexpr int kThreads = 192;     // 6 warps
constexpr uint32_t kATileBytes = kBM * kBK * 4;  // 16 KB

struct EpiG {
  uint32_t flags;
  const float* row_scale;
  const float* bias;
  const float* mask_src;  // MASK_BITS: uint32 sign-bit words
  int ld_mask;
  uint32_t* bits_out;     // SIGNBITS
  int ld_bits;
  float mask_scale;
  float* colsum_out;
  Dropout drop;
  int64_t row0;
};

struct TnParams {
  int M, N, K, BN, stages, num_kb, kb_per_split;
  float* ws;
  uint32_t idesc, tmem_cols;
};

__device__ __forceinline__ void epi_bar_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

#include "gemm_nt.inc"

// BF: BF16 operands.  MN-major tiles: a chunk is 32 (tf32) or 64 (bf16) MN elements = one 128-byte
// row per node, kBK node rows per stage.  tf32 uses the SWIZZLE_128B_BASE32B layout (4-row atoms,
// UMMA_K = 8 nodes = 1 KB); bf16 the plain SWIZZLE_128B layout (8-row atoms, UMMA_K = 16 nodes =
// 2 KB).  In both, LBO = the stride between MN chunks, SBO = the stride between K atoms.
template <bool BF>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tn(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kMN = BF ? 64 : 32;            // MN elements per 128-byte row
  constexpr uint32_t kChunk = kBK * 128;       // one MN chunk of BK node rows: 4 KB
  const uint32_t a_bytes = (kBM / kMN) * kChunk;
  const uint32_t nchunk_b = (uint32_t)p.BN / kMN;
  const uint32_t b_bytes = nchunk_b * kChunk;
  uint8_t* sA = smem;
  uint8_t* sB = smem + (size_t)p.stages * a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + (size_t)p.stages * b_bytes);
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kBM;
  const int split = blockIdx.y;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(p.num_kb, kb0 + p.kb_per_split);
  const int nkb = max(0, kb1 - kb0);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(tfull, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch_desc(&tmA);
    tc::tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, p.tmem_cols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int kb = kb0 + i;
        const int s = i % p.stages;
        const uint32_t ph = (uint32_t)(i / p.stages) & 1u;
        tc::mbar_wait(&empty[s], ph ^ 1u);
        tc::mbar_arrive_expect_tx(&full[s], a_bytes + b_bytes);
        uint8_t* a_dst = sA + (size_t)s * a_bytes;
        uint8_t* b_dst = sB + (size_t)s * b_bytes;
#pragma unroll
        for (int c = 0; c < kBM / kMN; ++c)
          tc::tma_load_2d(a_dst + c * kChunk, &tmA, &full[s], m0 + kMN * c, kb * kBK);
        for (uint32_t c = 0; c < nchunk_b; ++c)
          tc::tma_load_2d(b_dst + c * kChunk, &tmB, &full[s], kMN * (int)c, kb * kBK);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % p.stages;
        const uint32_t ph = (uint32_t)(i / p.stages) & 1u;
        tc::mbar_wait(&full[s], ph);
        tc::fence_after_sync();
        const uint32_t a_base = tc::smem_u32(sA + (size_t)s * a_bytes);
        const uint32_t b_base = tc::smem_u32(sB + (size_t)s * b_bytes);
        if constexpr (BF) {
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {  // 16 node rows = two 1 KB SW128 atoms per chunk
            const uint64_t da = tc::smem_desc_sw128(a_base + k * 2048, kChunk, 1024, 2);
            const uint64_t db = tc::smem_desc_sw128(b_base + k * 2048, kChunk, 1024, 2);
            tc::mma_bf16(tmem, da, db, p.idesc, (i | k) != 0 ? 1u : 0u);
          }
        } else {
#pragma unroll
          for (int k = 0; k < kBK / 8; ++k) {  // 8 node rows = two 512 B SW128_32B atoms per chunk
            const uint64_t da = tc::smem_desc_sw128(a_base + k * 1024, kChunk, 512, 1);
            const uint64_t db = tc::smem_desc_sw128(b_base + k * 1024, kChunk, 512, 1);
            tc::mma_tf32(tmem, da, db, p.idesc, (i | k) != 0 ? 1u : 0u);
          }
        }
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(tfull);
    }
  } else {
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    if (nkb > 0) {
      tc::mbar_wait(tfull, 0);
      tc::fence_after_sync();
    }
    float* out = p.ws + ((int64_t)split * p.M + row) * p.N;
    const bool vec = (p.N & 3) == 0;  // partial rows 16-byte aligned: float4 stores
    for (int c0 = 0; c0 < p.BN; c0 += 16) {
      float v[16];
      if (nkb > 0)
        tc::tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
      else
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.0f;
      if (row < p.M) {
        if (vec) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (c0 + 4 * j < p.N)
              reinterpret_cast<float4*>(out + c0)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c0 + i < p.N) out[c0 + i] = v[i];
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 1) tc::tmem_dealloc(tmem, p.tmem_cols);
}

// Column sums in a fixed order: 8 row-groups per 32-column chunk (group g sums rows g, g+8, ...),
// then the 8 group sums in order.  Deterministic for a given shape.
__global__ void __launch_bounds__(256) k_reduce_rows(const float* in, int rows, int cols, int ld, float* out,
                                                     int accumulate) {
  __shared__ float part[8][33];
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int grp = threadIdx.x >> 5;
  float s = 0.0f;
  if (c < cols) {
#pragma unroll 4
    for (int r = grp; r < rows; r += 8) s += in[(int64_t)r * ld + c];
  }
  part[grp][threadIdx.x & 31] = s;
  __syncthreads();
  if (grp == 0 && c < cols) {
    float t = accumulate ? out[c] : 0.0f;
#pragma unroll
    for (int g2 = 0; g2 < 8; ++g2) t += part[g2][threadIdx.x];
    out[c] = t;
  }
}

// out[r*ldc + c] = sum_s ws[(s*M + r)*N + c] in a fixed order: a block owns 128 consecutive
// outputs (32 lanes x float4), warp w sums the splits s = w, w+8, w+16, ... (two accumulators,
// even and odd steps), then lane sums of the 8 warps are added in warp order.  Deterministic for
// a given (splits, M, N).  Needs M*N % 4 == 0 and 16-byte aligned ws.
__global__ void __launch_bounds__(256) k_reduce_splits4(const float* __restrict__ ws, int splits, int M, int N,
                                                        float* __restrict__ C, int ldc, const GradMirror mir) {
  __shared__ float4 part[8][32];
  const int64_t total4 = (int64_t)M * N / 4;
  const int64_t t4 = (int64_t)blockIdx.x * 32 + (threadIdx.x & 31);
  const int w = threadIdx.x >> 5;
  float4 a0 = f4_zero(), a1 = f4_zero();
  if (t4 < total4) {
    const float4* src = reinterpret_cast<const float4*>(ws) + t4;
    int k = w;
    for (; k + 8 < splits; k += 16) {
      a0 = f4_add(a0, __ldcs(src + (int64_t)k * total4));
      a1 = f4_add(a1, __ldcs(src + (int64_t)(k + 8) * total4));
    }
    if (k < splits) a0 = f4_add(a0, __ldcs(src + (int64_t)k * total4));
  }
  part[w][threadIdx.x & 31] = f4_add(a0, a1);
  __syncthreads();
  if (w == 0 && t4 < total4) {
    float4 s4 = part[0][threadIdx.x];
#pragma unroll
    for (int g = 1; g < 8; ++g) s4 = f4_add(s4, part[g][threadIdx.x]);
    const int64_t e = t4 * 4;
    const int64_t r = e / N;
    const int c = (int)(e - r * N);  // N % 4 == 0: the 4 outputs share a row
    if ((ldc & 3) == 0 && ((reinterpret_cast<uintptr_t>(C) & 15) == 0)) {
      *reinterpret_cast<float4*>(C + r * ldc + c) = s4;
    } else {
      C[r * ldc + c] = s4.x;
      C[r * ldc + c + 1] = s4.y;
      C[r * ldc + c + 2] = s4.z;
      C[r * ldc + c + 3] = s4.w;
    }
    if (mir.n) {  // NEXT-1: the finished dW also lands in every rank's gradient slab (P2P stores)
      const int64_t o = r * ldc + c + (*mir.gen_dev & 1) * mir.par_stride;
      for (int q = 0; q < mir.n; ++q) {
        mir.base[q][o] = s4.x;
        mir.base[q][o + 1] = s4.y;
        mir.base[q][o + 2] = s4.z;
        mir.base[q][o + 3] = s4.w;
      }
    }
  }
  if (mir.n) __threadfence_system();
}

// out[r*ldc + c] = sum_s ws[(s*M + r)*N + c]   (fixed order over splits; any N)
__global__ void k_reduce_splits(const float* ws, int splits, int M, int N, float* C, int ldc, const GradMirror mir) {
  const int64_t total = (int64_t)M * N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / N;
    const int c = (int)(t - r * N);
    float s = 0.0f;
    for (int k = 0; k < splits; ++k) s += ws[(int64_t)k * total + t];
    C[r * ldc + c] = s;
    if (mir.n) {
      const int64_t o = r * ldc + c + (*mir.gen_dev & 1) * mir.par_stride;
      for (int q = 0; q < mir.n; ++q) mir.base[q][o] = s;
    }
  }
  if (mir.n) __threadfence_system();
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int make_tmap(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
              uint32_t box_outer, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B, bool bf16 = false) {
  auto fn = encode_fn();
  if (!fn) return fail(MPH_ECUDA, "cuTensorMapEncodeTiled unavailable (driver too old or no device)");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * (bf16 ? 2 : 4)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(MPH_ECUDA, "cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu ld=%llu box=%ux%u", (int)r,
                (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)ld, box_inner, box_outer);
  return MPH_OK;
}

uint32_t tmem_cols_for(int n) {
  uint32_t c = 32;
  while ((int)c < n) c <<= 1;
  return c;
}

constexpr size_t kSmemBudget = 100 * 1024;  // ~2 CTAs per SM (one epilogue overlaps another's mainloop)

int gemm_tn_splits(int M, int N, int K) {
  const int mtiles = (int)ceil_div(M, kBM);
  const int num_kb = (int)ceil_div(K, kBK);
  const int want = std::max(1, (2 * 148 + mtiles - 1) / mtiles);
  return std::max(1, std::min(want, std::max(1, num_kb / 4)));
}

}  // namespace

static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// Rows of colsum partials a launch writes when not zero-filling: one per persistent CTA.
int gemm_nt_colsum_rows(int M) { return (int)std::min<int64_t>(ceil_div(M, kBM), sm_count()); }

int gemm_nt_launch(int M, int N, int K, const float* A, int lda, const float* Bt, int ldb, float* C, int ldc,
                   const mph_epilogue* epi, cudaStream_t s, int colsum_fill) {
  return gemm_nt_launch_ex(M, N, K, A, lda, Bt, ldb, C, ldc, epi, s, colsum_fill, false);
}

int gemm_nt_launch_ex(int M, int N, int K, const void* A, int lda, const void* Bt, int ldb, float* C, int ldc,
                      const mph_epilogue* epi, cudaStream_t s, int colsum_fill, bool bf16) {
  if (M < 0 || N <= 0 || K < 0 || !A || !Bt || !C) return fail(MPH_EINVAL, "gemm_nt: bad arguments");
  if (N > 256) return fail(MPH_ENOTSUP, "gemm_nt: N=%d > 256", N);
  const uint32_t f0 = epi ? epi->flags : 0u;
  if (lda % (bf16 ? 8 : 4) || ldb % (bf16 ? 8 : 4) || ldc % ((f0 & MPH_EPI_BF16) ? 8 : 4) || lda < K || ldb < K ||
      ldc < N)
    return fail(MPH_EINVAL, "gemm_nt: lda/ldb/ldc must be multiples of 16 bytes with lda, ldb >= K, ldc >= N");
  if ((f0 & MPH_EPI_MASK_BF16) && (!(f0 & MPH_EPI_MASK) || (epi->ld_mask % 8)))
    return fail(MPH_EINVAL, "gemm_nt: MASK_BF16 needs MASK and ld_mask %% 8 == 0");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(Bt) | reinterpret_cast<uintptr_t>(C)) & 15)
    return fail(MPH_EINVAL, "gemm_nt: A, Bt and C must be 16-byte aligned");
  const uint32_t flags = epi ? epi->flags : 0u;
  if ((flags & MPH_EPI_BIAS) && !epi->bias) return fail(MPH_EINVAL, "gemm_nt: null bias");
  if ((flags & MPH_EPI_ROWSCALE) && !epi->row_scale) return fail(MPH_EINVAL, "gemm_nt: null row_scale");
  if ((flags & MPH_EPI_MASK) && !(flags & MPH_EPI_MASK_BITS) && (!epi->mask_src || epi->ld_mask % 4 || epi->ld_mask < N ||
                                 (reinterpret_cast<uintptr_t>(epi->mask_src) & 15)))
    return fail(MPH_EINVAL, "gemm_nt: mask_src must be 16-byte aligned with ld_mask %% 4 == 0, >= N");
  if ((flags & MPH_EPI_COLSUM) && !epi->colsum_out) return fail(MPH_EINVAL, "gemm_nt: null colsum_out");
  if ((flags & MPH_EPI_MASK_BITS) && (!(flags & MPH_EPI_MASK) || (flags & MPH_EPI_MASK_BF16) ||
                                      epi->ld_mask < (N + 3) / 4 || epi->ld_mask % 8 ||
                                      (reinterpret_cast<uintptr_t>(epi->mask_src) & 7)))
    return fail(MPH_EINVAL, "gemm_nt: MASK_BITS needs MASK, 8-byte aligned sign bytes, ld_mask %% 8 == 0 and >= ceil(N/4)");
  if ((flags & MPH_EPI_SIGNBITS) && (!epi->bits_out || epi->ld_bits < (N + 3) / 4 || epi->ld_bits % 8 ||
                                     (reinterpret_cast<uintptr_t>(epi->bits_out) & 7)))
    return fail(MPH_EINVAL, "gemm_nt: SIGNBITS needs 8-byte aligned bits_out, ld_bits %% 8 == 0 and >= ceil(N/4)");
  if (M == 0) return MPH_OK;
  const int sms = sm_count();
  const int BN = round_up(N, 32);
  NtParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.BN = BN;
  const int kelems = bf16 ? 64 : kBK;  // K elements per 128-byte k-block
  p.num_kb = (int)ceil_div(K, kelems);
  p.n_tiles = (int)ceil_div(M, kBM);
  p.colsum_rows = colsum_fill ? p.n_tiles : 0;  // rows beyond the grid are zero-filled only for the ABI
  const size_t stage_bytes = kATileBytes + (size_t)BN * kBK * 4;
  // the epilogue (C tile out, mask tile in) is the long pole of these HBM-bound GEMMs: 8 warps
  // (two per TMEM lane quarter) whenever there are at least two 32-column chunks per quarter.
  // Measured on products: K <= 128 launches -10..-25 %, K = 256 launches -3 % even with the
  // operand ring cut to 2 stages.  MPH_GEMM_EPI=4 restores 4 warps (experiments).
  p.n_epi = BN >= 64 ? 8 : 4;
  if (const char* ev = getenv("MPH_GEMM_EPI")) p.n_epi = (atoi(ev) == 8 && BN >= 64) ? 8 : 4;
  // a mask tile streams in ahead of each chunk (3-buffer ring); without one, a chunk only needs its
  // staging buffer and the previous chunk's, still being stored: 2 buffers, and the 32 KB saved per
  // 8 warps buys the operand ring another stage (N = 256: 2 -> 3 stages of A + B in flight)
  p.nbufs = ((flags & MPH_EPI_MASK) && !(flags & MPH_EPI_MASK_BITS)) ? kEpiBufs : 2;
  const size_t epi_bytes = (size_t)p.n_epi * p.nbufs * kEpiChunkBytes;
  const size_t fixed = 1024 + epi_bytes + (size_t)BN * sizeof(float) +
                       (size_t)(2 * 8 + 4 + p.n_epi * p.nbufs) * 8 + 16 + 4 * (size_t)BN * sizeof(float);
  constexpr size_t kMaxSmem = 232448;  // 227 KB opt-in per block on sm_100
  p.stages = (int)std::max<size_t>(2, std::min<size_t>(8, (kMaxSmem - fixed) / stage_bytes));
  p.idesc = bf16 ? tc::idesc_bf16(kBM, BN, 0, 0) : tc::idesc_tf32(kBM, BN, 0, 0);
  p.tmem_cols = tmem_cols_for(2 * BN);
  p.epi.flags = flags;
  p.epi.row_scale = epi ? epi->row_scale : nullptr;
  p.epi.bias = epi ? epi->bias : nullptr;
  p.epi.mask_src = epi ? epi->mask_src : nullptr;
  p.epi.ld_mask = epi ? epi->ld_mask : 0;
  p.epi.bits_out = (epi && (flags & MPH_EPI_SIGNBITS)) ? epi->bits_out : nullptr;
  p.epi.ld_bits = epi ? epi->ld_bits : 0;
  p.epi.mask_scale = epi ? epi->mask_scale : 1.0f;
  p.epi.colsum_out = epi ? epi->colsum_out : nullptr;
  p.epi.drop = make_dropout(epi);
  p.epi.row0 = epi ? epi->row0 : 0;
  if (p.epi.drop.threshold == 0) p.epi.flags &= ~MPH_EPI_DROPOUT;
  CUtensorMap ta, tb, tcm, tm;
  MPH_TRY(make_tmap(&ta, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda, kelems, kBM, CU_TENSOR_MAP_SWIZZLE_128B, bf16));
  MPH_TRY(make_tmap(&tb, Bt, (uint64_t)K, (uint64_t)N, (uint64_t)ldb, kelems, (uint32_t)BN, CU_TENSOR_MAP_SWIZZLE_128B,
                    bf16));
  const bool out_bf = (flags & MPH_EPI_BF16) != 0, mask_bf = (flags & MPH_EPI_MASK_BF16) != 0;
  // BF16 output in 64-column units (full 128-byte smem rows, half the TMA stores), when the width
  // allows and a mask, if any, is BF16 too
  p.wide = (out_bf && BN % 64 == 0 && (!(flags & MPH_EPI_MASK) || mask_bf || (flags & MPH_EPI_MASK_BITS))) ? 1 : 0;
  const uint32_t cw = p.wide ? 64 : 32;
  MPH_TRY(make_tmap(&tcm, C, (uint64_t)N, (uint64_t)M, (uint64_t)ldc, cw, 32,
                    (out_bf && !p.wide) ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, out_bf));
  if ((flags & MPH_EPI_MASK) && !(flags & MPH_EPI_MASK_BITS))
    MPH_TRY(make_tmap(&tm, epi->mask_src, (uint64_t)N, (uint64_t)M, (uint64_t)epi->ld_mask, cw, 32,
                      (mask_bf && !p.wide) ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, mask_bf));
  else
    tm = tcm;
  const size_t smem = fixed + (size_t)p.stages * stage_bytes;
  if ((flags & MPH_EPI_SIGNBITS) && (flags & MPH_EPI_MASK_BITS))
    return fail(MPH_ENOTSUP, "gemm_nt: SIGNBITS and MASK_BITS in one launch");
  const int sb = (flags & MPH_EPI_SIGNBITS) ? 1 : (flags & MPH_EPI_MASK_BITS) ? 2 : 0;
  auto kern = bf16 ? (sb == 1 ? k_gemm_nt<true, 1> : sb == 2 ? k_gemm_nt<true, 2> : k_gemm_nt<true, 0>)
                   : (sb == 1 ? k_gemm_nt<false, 1> : sb == 2 ? k_gemm_nt<false, 2> : k_gemm_nt<false, 0>);
  static size_t configured[6] = {0, 0, 0, 0, 0, 0};
  const int ki = (bf16 ? 3 : 0) + sb;
  if (smem > configured[ki]) {
    MPH_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[ki] = smem;
  }
  const int grid = std::min(p.n_tiles, sms);
  kern<<<grid, 64 + 32 * p.n_epi, smem, s>>>(ta, tb, tcm, tm, p);
  count_launch();
  return launch_check("gemm_nt");
}

size_t gemm_tn_ws_bytes(int M, int N, int K) {
  if (M <= 0 || N <= 0) return 0;
  return (size_t)gemm_tn_splits(M, N, K) * M * N * sizeof(float);
}

int gemm_tn_launch(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C, int ldc, void* ws,
                   size_t ws_bytes, cudaStream_t s, const GradMirror* mirror) {
  return gemm_tn_launch_ex(M, N, K, A, lda, B, ldb, C, ldc, ws, ws_bytes, s, mirror, false);
}

int gemm_tn_launch_ex(int M, int N, int K, const void* A, int lda, const void* B, int ldb, float* C, int ldc,
                      void* ws, size_t ws_bytes, cudaStream_t s, const GradMirror* mirror, bool bf16) {
  if (M <= 0 || N <= 0 || K < 0 || !A || !B || !C) return fail(MPH_EINVAL, "gemm_tn: bad arguments");
  if (N > 256) return fail(MPH_ENOTSUP, "gemm_tn: N=%d > 256", N);
  if (lda % (bf16 ? 8 : 4) || ldb % (bf16 ? 8 : 4) || lda < M || ldb < N || ldc < N)
    return fail(MPH_EINVAL, "gemm_tn: lda/ldb (multiples of 16 bytes) >= M, N and ldc >= N");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15)
    return fail(MPH_EINVAL, "gemm_tn: A and B must be 16-byte aligned");
  const size_t need = gemm_tn_ws_bytes(M, N, K);
  if (!ws || ws_bytes < need) return fail(MPH_EINVAL, "gemm_tn: workspace %zu < %zu bytes", ws_bytes, need);
  if (reinterpret_cast<uintptr_t>(ws) & 15) return fail(MPH_EINVAL, "gemm_tn: workspace must be 16-byte aligned");
  const int BN = round_up(N, bf16 ? 64 : 32);
  TnParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.BN = BN;
  p.num_kb = (int)ceil_div(K, kBK);
  const int splits = gemm_tn_splits(M, N, K);
  p.kb_per_split = (int)ceil_div(std::max(p.num_kb, 1), splits);
  const int kmn = bf16 ? 64 : 32;
  const size_t stage_bytes = (size_t)(kBM / kmn) * kBK * 128 + (size_t)(BN / kmn) * kBK * 128;
  p.stages = (int)std::max<size_t>(2, std::min<size_t>(8, kSmemBudget / stage_bytes));
  p.ws = reinterpret_cast<float*>(ws);
  p.idesc = bf16 ? tc::idesc_bf16(kBM, BN, 1, 1) : tc::idesc_tf32(kBM, BN, 1, 1);
  p.tmem_cols = tmem_cols_for(BN);
  CUtensorMap ta, tb;
  const CUtensorMapSwizzle swz = bf16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
  MPH_TRY(make_tmap(&ta, A, (uint64_t)M, (uint64_t)std::max(K, 1), (uint64_t)lda, kmn, kBK, swz, bf16));
  MPH_TRY(make_tmap(&tb, B, (uint64_t)N, (uint64_t)std::max(K, 1), (uint64_t)ldb, kmn, kBK, swz, bf16));
  const size_t smem = 1024 + (size_t)p.stages * stage_bytes + (2 * p.stages + 1) * 8 + 16;
  static size_t configured[2] = {0, 0};
  if (smem > configured[bf16]) {
    MPH_CUDA_TRY(cudaFuncSetAttribute(bf16 ? k_gemm_tn<true> : k_gemm_tn<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[bf16] = smem;
  }
  dim3 grid((unsigned)ceil_div(M, kBM), (unsigned)splits);
  if (bf16)
    k_gemm_tn<true><<<grid, kThreads, smem, s>>>(ta, tb, p);
  else
    k_gemm_tn<false><<<grid, kThreads, smem, s>>>(ta, tb, p);
  count_launch();
  MPH_TRY(launch_check("gemm_tn"));
  const int64_t total = (int64_t)M * N;
  const GradMirror mir = mirror ? *mirror : GradMirror{};
  if (N % 4 == 0 && (ldc & 3) == 0)
    k_reduce_splits4<<<(unsigned)ceil_div(total / 4, 32), 256, 0, s>>>(p.ws, splits, M, N, C, ldc, mir);
  else
    k_reduce_splits<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 8), 256, 0, s>>>(p.ws, splits, M, N, C,
                                                                                              ldc, mir);
  count_launch();
  return launch_check("reduce_splits");
}

int reduce_rows_launch(const float* in, int rows, int cols, int ld, float* out, int accumulate, cudaStream_t s) {
  if (!in || !out || rows < 0 || cols <= 0 || ld < cols) return fail(MPH_EINVAL, "reduce_rows: bad arguments");
  k_reduce_rows<<<(unsigned)ceil_div(cols, 32), 256, 0, s>>>(in, rows, cols, ld, out, accumulate);
  count_launch();
  return launch_check("reduce_rows");
}

}  // namespace mph

extern "C" int mph_gemm_nt(int32_t M, int32_t N, int32_t K, const float* A_d, int32_t lda, const float* Bt_d,
                           int32_t ldb, float* C_d, int32_t ldc, const mph_epilogue* epi, void* stream) {
  return mph::gemm_nt_launch(M, N, K, A_d, lda, Bt_d, ldb, C_d, ldc, epi, (cudaStream_t)stream);
}

extern "C" int mph_gemm_tn_workspace(int32_t M, int32_t N, int32_t K, size_t* bytes_h) {
  if (!bytes_h) return mph::fail(MPH_EINVAL, "null bytes");
  *bytes_h = mph::gemm_tn_ws_bytes(M, N, K);
  return MPH_OK;
}

extern "C" int mph_gemm_tn(int32_t M, int32_t N, int32_t K, const float* A_d, int32_t lda, const float* B_d,
                           int32_t ldb, float* C_d, int32_t ldc, void* ws_d, size_t ws_bytes, void* stream) {
  return mph::gemm_tn_launch(M, N, K, A_d, lda, B_d, ldb, C_d, ldc, ws_d, ws_bytes, (cudaStream_t)stream);
}

extern "C" int mph_reduce_rows(const float* in_d, int32_t rows, int32_t cols, int32_t ld, float* out_d,
                               int32_t accumulate, void* stream) {
  return mph::reduce_rows_launch(in_d, rows, cols, ld, out_d, accumulate, (cudaStream_t)stream);
}

extern "C" int mph_gemm(int32_t M, int32_t N, int32_t K, const float* A_d, int32_t lda, int32_t transA,
                        const float* B_d, int32_t ldb, int32_t transB, float* C_d, int32_t ldc, int32_t precision,
                        uint32_t epilogue_flags, void* stream) {
  using namespace mph;
  if (precision != 0 && precision != 1) return fail(MPH_ENOTSUP, "mph_gemm: precision %d (0 TF32, 1 BF16)", precision);
  const bool bf16 = precision == 1;
  cudaStream_t s = (cudaStream_t)stream;
  if (transA == 0 && transB == 1) {
    if (epilogue_flags & ~(uint32_t)(MPH_EPI_RELU | MPH_EPI_TF32))
      return fail(MPH_EINVAL, "mph_gemm: flags 0x%x need operands (use mph_gemm_nt)", epilogue_flags);
    mph_epilogue e{};
    e.flags = epilogue_flags;
    e.mask_scale = 1.0f;
    return gemm_nt_launch_ex(M, N, K, A_d, lda, B_d, ldb, C_d, ldc, &e, s, 1, bf16);
  }
  if (transA == 1 && transB == 0) {
    if (epilogue_flags) return fail(MPH_EINVAL, "mph_gemm: no epilogue on the transposed-A shape");
    const size_t ws_bytes = gemm_tn_ws_bytes(M, N, K);
    void* ws = nullptr;
    if (ws_bytes) MPH_CUDA_TRY(cudaMallocAsync(&ws, ws_bytes, s));
    const int rc = gemm_tn_launch_ex(M, N, K, A_d, lda, B_d, ldb, C_d, ldc, ws, ws_bytes, s, nullptr, bf16);
    if (ws) cudaFreeAsync(ws, s);
    return rc;
  }
  return fail(MPH_ENOTSUP, "mph_gemm: (transA, transB) = (%d, %d); the GCN path uses (0, 1) and (1, 0)", transA,
              transB);
}
