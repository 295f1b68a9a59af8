// Library-internal handle layouts and kernel launchers shared between translation units.
#pragma once

#include <vector>

#include "common.cuh"

struct mph_graph {
  int32_t n_rows = 0;  // owned rows
  int32_t n_cols = 0;  // owned + ghost nodes (== n_rows for a global graph)
  int64_t nnz = 0;
  int32_t max_deg = 0;
  int64_t* row_ptr = nullptr;  // [n_rows+1]
  int32_t* col_idx = nullptr;  // [nnz] (local ids for a localized graph)
  int32_t* deg = nullptr;      // [n_cols] global degree d~
  float* dinv = nullptr;       // [n_cols] D̃^{-1/2} (G6)
  float* dinv1 = nullptr;      // [n_cols] D̃^{-1} (mean aggregation, R6)
  // localized graphs only (D2-D4)
  bool local = false;
  int32_t world = 1, rank = 0;
  int64_t row0 = 0;
  int64_t* split = nullptr;  // [n_rows] absolute edge index where ghost columns start
  std::vector<int64_t> recv_offset, n_recv, send_offset;  // host, per peer
  std::vector<int64_t> ghosts;                            // host, global ids of the ghost columns
  int32_t* send_ids = nullptr;                            // device, concatenated per peer
  int64_t n_send = 0;
  float* send_buf = nullptr;
  size_t send_cap = 0;  // floats
  // edge-balanced SpMM work items (spmm.cu): [first_row, end_row) runs, hubs first
  int2* items = nullptr;
  int n_items = 0;
  int* item_counter = nullptr;
  // launches over an operand larger than L2/2 walk a chunked virtual CSR (spmm.cu,
  // build_split_items), one per row range: whole rows (part -1), owned edges (part 0), ghost
  // edges (part 1) of a localized graph.  Rows longer than chunk_edges entries are cut into
  // virtual rows of <= chunk_edges; vrow_ptr [n_v + 1] indexes col_idx, vmap[v] = row or -1 -
  // chunk, items = runs of virtual rows; srows = {row, first chunk, n chunks} of every cut row for
  // the combine kernel.  chunk_part (kChunkPartF4 float4 per chunk) is shared by the three.
  struct SplitCsr {
    int64_t* vrow_ptr = nullptr;
    int* vmap = nullptr;
    int2* items = nullptr;
    int n_items = 0;
    int4* srows = nullptr;
    int n_srows = 0;
    int64_t n_chunks = 0;
    int n_vrows = 0;
  };
  int split_mode = 0;  // MPH_SPMM_SPLIT at item build: 0 off, 1 operand > L2/2, 2 always
  SplitCsr scsr[3];    // [part + 1]
  int chunk_edges = 0;
  float4* chunk_part = nullptr;
};

struct mph_features {
  int32_t N = 0, F = 0, P = 0;  // P = padded row stride of the dense copy
  int64_t nnz = 0;
  int32_t mode = 0, is_binary = 0;
  float* X = nullptr;  // dense mode: [N][P]
  int64_t* csr_ptr = nullptr;
  int32_t* csr_idx = nullptr;
  float* csr_val = nullptr;
  int64_t* csc_ptr = nullptr;
  int32_t* csc_idx = nullptr;
  float* csc_val = nullptr;
  // X_csc cut into segments of <= kSegNnz nonzeros per column (sparse-path dW, elementwise.cu)
  int64_t n_seg = 0;
  int32_t* seg_col = nullptr;
  int64_t* seg_begin = nullptr;
  int64_t* col_seg0 = nullptr;  // [F+1] first segment of each column
  int64_t* seg_ptr = nullptr;   // [n_seg+1] segments as the rows of a virtual CSR over X_csc
  float* part = nullptr;
  size_t part_cap = 0;
  // edge-balanced work items of the gather kernels (spmm.cu): rows of X_csr, segments of X_csc
  int2* xw_items = nullptr;
  int xw_n_items = 0;
  int2* xtg_items = nullptr;
  int xtg_n_items = 0;
  int* item_counter = nullptr;
};

constexpr int64_t kSegNnz = 128;

// NEXT-1: peer-memory (NVLink) communication state of a MPH_COMM_P2P model (p2p.cu).
// One cudaMalloc arena per rank, mapped by every peer through CUDA IPC:
//   [flags: uint64 [kP2PSlots][kP2PMaxWorld]] [loss: double [2][kP2PMaxWorld]]
//   [gsum: float [2][world][n_params]] [shared buffers: T'_l, dZ'_l, dinv ⊙ X ...]
// flags[slot][q] is the latest step counter rank q has signalled for that slot; the loss and
// gradient slabs are indexed by the parity of the generation (double buffered).
constexpr int kP2PMaxWorld = 16;
enum P2PSlot { kSlotHalo = 0, kSlotLoss = 1, kSlotGrad = 2, kSlotSetup = 3, kP2PSlots = 4 };
constexpr int kP2PHaloPerGen = 16;  // halo exchanges per epoch (2L <= 16)

struct P2PState {
  int world = 1, rank = 0;
  char* arena = nullptr;
  size_t arena_bytes = 0;
  int64_t off_flags = 0, off_loss = 0, off_gsum = 0;  // bytes into the arena
  int64_t n_params = 0;
  int64_t n_rows = 0, row0 = 0;
  std::vector<int64_t> off_buf;  // this rank's shared buffers (byte offsets, -1 = absent)
  uint32_t layout_sig = 0;       // feature mode + per-layer orders; every rank must agree
  // after mph_gcn_p2p_open
  bool opened = false;
  std::vector<char*> peer_base;                 // mapped arenas (own arena at [rank])
  std::vector<std::vector<int64_t>> peer_off;   // peers' off_buf
  std::vector<int64_t> peer_flags_off, peer_loss_off, peer_gsum_off;
  int32_t* ghost_ref = nullptr;  // device [n_ghost]: owner << 27 | owner-local row
  int64_t n_ghost = 0;
  int64_t* gen_dev = nullptr;    // device generation counter, advanced once per forward
  int* err_dev = nullptr;        // device timeout flag
  int64_t xgen = 0;              // host counter of setup exchanges (constant operands)
};

// A kernel that finalises gradient entries can also store them straight into every rank's
// receive slab (the all-reduce's "send" fused into the producer): element i of the producer's
// output also goes to base[q][i + (*gen_dev & 1) * par_stride] for q < n, then a system fence.
struct GradMirror {
  float* base[kP2PMaxWorld];
  int n;
  const int64_t* gen_dev;
  int64_t par_stride;
};

namespace mph {
int p2p_alloc_arena(P2PState* p, size_t bytes);
// Mirror of this rank's slab slot, starting at flat parameter offset `off`, in every rank.
int p2p_grad_mirror(const P2PState* p, int64_t off, GradMirror* out);
void p2p_free(P2PState* p);
int p2p_export(const P2PState* p, uint8_t* blob);
int p2p_open(P2PState* p, const mph_graph* g, const uint8_t* blobs, int world);
// flags[slot][rank] := gen·mult + add in every peer's arena (gen from the device counter when
// use_gen, else 0), after a system-scope fence: everything this stream wrote before is visible.
int p2p_signal(const P2PState* p, int slot, bool use_gen, int64_t mult, int64_t add, cudaStream_t s);
// Wait for every peer's flags[slot] >= gen·mult + add, then copy each ghost row of shared buffer
// `buf` from its owner into the local ghost slice [n_rows, n_cols) of `local` (stride ld = w).
int p2p_pull(const P2PState* p, int buf, float* local, int w, int slot, bool use_gen, int64_t mult, int64_t add,
             cudaStream_t s);
// grads[a, b) -> every rank's gradient slab [parity][rank] (a, b, multiples of 4).
int p2p_grad_push(const P2PState* p, const float* grads, int64_t a, int64_t b, cudaStream_t s);
// Global loss: push this rank's partial, signal, wait for all, sum in rank order into loss_d.
int p2p_loss_sum(const P2PState* p, double* loss_d, cudaStream_t s);
int p2p_gen_advance(const P2PState* p, cudaStream_t s);
// The gradient slabs of the current parity and the grad flag row, for the fused optimizer.
const float* p2p_gsum_local(const P2PState* p);
const uint64_t* p2p_flags_local(const P2PState* p, int slot);
}  // namespace mph

namespace mph {

// dinv[u] = (float)(1.0 / sqrt((double)deg[u]))  (G6)
int launch_dinv(const int32_t* deg, float* dinv, float* dinv1, int64_t n, cudaStream_t s);

// SpMM driver (spmm.cu). part: -1 whole row, 0 owned columns (raw sums, no epilogue),
// 1 ghost columns accumulated onto out + epilogue.
// post: the output row scale (D̃^{-1/2} for the GCN's Â, D̃^{-1} for mean, nullptr for sum).
// partial (part 1 only, nullable): where part 0 left its raw FP32 sums (row stride w) when the
// output itself is BF16; nullptr = they are in out.
int spmm_launch(const mph_graph* g, int part, const float* in, int w, int ld_in, float* out, int ld_out,
                const mph_epilogue* epi, const float* post, cudaStream_t s, const float* partial = nullptr);
int ensure_graph_items(const mph_graph* g, cudaStream_t s);
// MPH_EPI_SIGNBITS is available for whole-row aggregations of width w on g
bool spmm_signbits_ok(const mph_graph* g, int w);
// aggregate.cu (NEXT-4): scheme scales, max aggregation and its adjoint, chunked column sums
int agg_scales(const mph_graph* g, int scheme, int transpose, const float** pre, const float** post);
int aggregate_max_launch(const mph_graph* g, const float* in, int w, int ld_in, float* out, int ld_out, int32_t* arg,
                         int ld_arg, const mph_epilogue* epi, cudaStream_t s);
int aggregate_max_backward_launch(const mph_graph* g, const float* dY, int w, int ld_dy, const int32_t* arg, int ld_arg,
                                  float* dH, int ld_out, const mph_epilogue* epi, cudaStream_t s);
int colsum_chunks_launch(const float* in, int rows, int cols, int ld, float* part, cudaStream_t s);
// Edge-balanced work items over a CSR whose row_ptr lives on the device (synchronises; setup only).
int build_work_items(const int64_t* row_ptr_d, int n_rows, int64_t nnz, int2** items, int* n_items, cudaStream_t s);
// The same gather kernel on a general CSR: out[r,:] = row_scale[r] * sum_e val[e] * in[col[e],:]
// (val == nullptr: pattern / binary matrix; row_scale == nullptr: 1).  w, ld_in, ld_out multiples
// of 4, in/out 16-byte aligned, w <= 512.
int spmm_csr_launch(const int64_t* row_ptr, const int32_t* col, const float* val, int n_rows, const int2* items,
                    int n_items, int* counter, const float* row_scale, const float* in, int w, int ld_in, float* out,
                    int ld_out, cudaStream_t s);
// Halo exchange in two halves (comm.cu) so the model can overlap them with the local-edge SpMM.
int halo_reserve(const mph_graph* g, int w);
int halo_pack(const mph_graph* g, const float* buf, int w, int ld, cudaStream_t s);
int halo_sendrecv(const mph_graph* g, mph_comm* c, float* buf, int w, int ld, cudaStream_t s);
// Halo pack (spmm.cu): send_buf[j] = buf[send_ids[j]] for the whole send list.
int pack_rows(const int32_t* ids, int64_t n, const float* buf, int ld, int w, float* out, cudaStream_t s);

// colsum_fill: 1 = the ABI contract (colsum_out has ceil(M/128) rows, the ones no CTA owns are
// zero-filled); 0 = only the first gemm_nt_colsum_rows(M) rows are written (internal callers).
int gemm_nt_launch(int M, int N, int K, const float* A, int lda, const float* Bt, int ldb, float* C, int ldc,
                   const mph_epilogue* epi, cudaStream_t s, int colsum_fill = 1);
int gemm_nt_colsum_rows(int M);
// The same with BF16 operands when bf16 (A [M][lda], Bt [N][ldb] as uint16 bf16; lda, ldb % 8 == 0).
int gemm_nt_launch_ex(int M, int N, int K, const void* A, int lda, const void* Bt, int ldb, float* C, int ldc,
                      const mph_epilogue* epi, cudaStream_t s, int colsum_fill, bool bf16);
size_t gemm_tn_ws_bytes(int M, int N, int K);
int gemm_tn_launch(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C, int ldc,
                   void* ws, size_t ws_bytes, cudaStream_t s, const GradMirror* mirror = nullptr);
int gemm_tn_launch_ex(int M, int N, int K, const void* A, int lda, const void* B, int ldb, float* C, int ldc,
                      void* ws, size_t ws_bytes, cudaStream_t s, const GradMirror* mirror, bool bf16);
int reduce_rows_launch(const float* in, int rows, int cols, int ld, float* out, int accumulate, cudaStream_t s);

size_t softmax_ce_ws_bytes(int N, int C);
int softmax_ce_launch(const float* Z, int N, int C, int ld, const int32_t* labels, const uint8_t* mask, int64_t n_lab,
                      const float* row_scale, float* dZ, int ld_dz, float* db, double* loss, void* ws, size_t ws_bytes,
                      cudaStream_t s, int round_tf32 = 0);
int adam_launch(float* p, const float* g, float* m, float* v, int64_t n, const mph_adam_cfg* cfg, int t, cudaStream_t s,
                const int32_t* t_dev = nullptr);
int optim_launch(float* p, const float* g, float* m, float* v, int64_t n, const mph_optim_cfg* cfg, int t,
                 cudaStream_t s, const int32_t* t_dev = nullptr);
// NEXT-1 fused gradient sum + optimizer: waits until every rank's flags_grad >= *gen, takes
// g[i] = Σ_q gsum[(par·world + q)·n + i] in rank order (par = *gen & 1), writes it to grads[i]
// and applies the update of optim_launch in the same pass.
int optim_sum_launch(float* p, float* grads, float* m, float* v, int64_t n, const mph_optim_cfg* cfg, int t,
                     cudaStream_t s, const int32_t* t_dev, const float* gsum, int world, const uint64_t* flags_grad,
                     const int64_t* gen_dev, int* err);
int xavier_launch(float* W, int f_in, int f_out, int ld, uint64_t seed, int layer, cudaStream_t s);
// dst_t[j*ld_t + i] = tf32(src[i*ld_src + j]), dst_r[i*ld_r + j] = tf32(src[i*ld_src + j]) (dst_r nullable)
int weight_copies_launch(const float* src, int rows, int cols, int ld_src, float* dst_t, int ld_t, float* dst_r,
                         int ld_r, cudaStream_t s, bool bf16 = false);
int sparse_xw_launch(const mph_features* f, const float* W, int F_out, int ldw, const float* row_scale, float* T,
                     int ldt, cudaStream_t s);
int sparse_xtg_launch(const mph_features* f, const float* G, int F_out, int ldg, float* dW, int lddw, cudaStream_t s);
// out[i][c] = in[i][c] * scale[i] (scale nullable) for c < w, optionally rounded to TF32
int rowscale_launch(const float* in, int ld_in, const float* scale, int rows, int w, float* out, int ld_out, int round,
                    cudaStream_t s);

}  // namespace mph
