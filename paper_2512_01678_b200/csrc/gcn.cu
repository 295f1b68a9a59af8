// The L-layer GCN training step (Listing 1; layer update P:92 with readings Q1, Q6,
// Q7, Q8; loss Q9; Adam P:170/P:534-535).  This file only orders kernel launches and owns the
// buffers; every arithmetic step runs in the kernels of spmm.cu / gemm.cu / elementwise.cu.
//
// Data layout in HBM (row-major fp32, widths padded to pad_width(F), padding exactly zero):
//   params  [W_1 (P_0 x P_1) | b_1 (P_1) | ... ]   flat, one Adam launch
//   wt      [W_1^T (P_1 x P_0) | ...]              K-major B operands of the forward GEMMs
//   T_l     n_cols x P_l   dinv-prescaled transform output incl. ghost rows (halo target)
//   out_l   n_rows x P_l   H_l = ReLU(Z_l) (hidden, saved for backward) or logits Z_L
//   dZ_l    n_cols x P_l   dinv-prescaled loss/input gradient (halo target)
//   G_l     n_rows x P_l   backward aggregation Â·dZ_l
//   Y_1     n_rows x P_0   aggregate-first input Â·X (only when layer 1 is AF)
#include <algorithm>
#include <vector>

#include "internal.cuh"
#include "profile.cuh"

struct mph_comm;
extern "C" int mph_halo_exchange(const mph_graph* gc, mph_comm* c, float* buf_d, int32_t w, int32_t ld, void* stream);
extern "C" int mph_allreduce_sum(mph_comm* c, void* buf_d, int64_t n, int32_t is_double, void* stream);
extern "C" int mph_comm_info(const mph_comm* c, int32_t* world_h, int32_t* rank_h);

namespace {

struct Layer {
  int fin = 0, fout = 0, pin = 0, pout = 0;
  int order = 0;  // 0 transform-first, 1 aggregate-first
  int64_t off_w = 0, off_b = 0, off_wt = 0;
  float* T = nullptr;
  float* out = nullptr;
  float* dZ = nullptr;
  float* G = nullptr;
  float* Y = nullptr;     // aggregate-first input (AF layer 1; every layer under max)
  float* colsum = nullptr;
  int32_t* arg = nullptr;  // max aggregation: argmax of Y (layers > 1)
  float* dY = nullptr;     // max aggregation: dZ·Wᵀ, the gradient routed back through arg
  // hidden layers: the signs of out (= the ReLU + dropout mask of the backward dH GEMM) as sign
  // bytes, written by the producing SpMM / GEMM epilogue (MPH_EPI_SIGNBITS): the dH GEMM reads
  // 1/16 of out's bytes for the same decisions (MPH_EPI_MASK_BITS)
  uint8_t* sb = nullptr;
  int ld_sb = 0;
};

}  // namespace

struct mph_gcn {
  const mph_graph* g = nullptr;
  const mph_features* f = nullptr;
  mph_comm* comm = nullptr;
  P2PState* p2p = nullptr;  // MPH_COMM_P2P: NVLink peer-memory exchange (p2p.cu, NEXT-1)
  int world = 1;
  int L = 0;
  int agg = MPH_AGG_GCN;  // aggregation scheme (NEXT-4)
  // MPH_PREC_BF16: every tensor that only feeds tensor-core GEMMs (hidden H, backward G, Y_1, dZ_1,
  // the copies of X and W) is stored as bfloat16 and the GEMMs run kind::f16 (FP32 accumulate)
  bool bf16 = false;
  float* part0 = nullptr;  // BF16 with P > 1: FP32 owned-edge sums between the two SpMM parts
  // diagonal scales of a linear scheme: forward AGG = diag(fpost)·Ã·diag(fpre), adjoint
  // diag(bpost)·Ã·diag(bpre); nullptr = 1 (aggregate.cu)
  const float *fpre = nullptr, *fpost = nullptr, *bpre = nullptr, *bpost = nullptr;
  std::vector<Layer> layers;
  float *params = nullptr, *grads = nullptr, *m = nullptr, *v = nullptr, *wt = nullptr;
  bool own_params = true, own_grads = true, own_m = true, own_v = true, own_ws = true;  // mph_gcn_bind
  float* wr = nullptr;  // TF32-rounded copy of the W segments (B operand of the dH GEMM)
  float* Xr = nullptr;  // TF32-rounded copy of X (A operand of a dense transform-first layer 1)
  int64_t n_params = 0, n_wt = 0;
  const int32_t* labels = nullptr;
  const uint8_t* mask = nullptr;
  int64_t n_lab = 0;
  float* Xs = nullptr;  // dinv ⊙ X with ghost rows (AF layer 1)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  float dropout_p = 0.0f;
  uint64_t dropout_seed = 0;
  int epoch = 0;
  bool fwd_done = false, loss_done = false;
  // P > 1: NCCL runs on its own stream, ordered against the compute stream by events
  cudaStream_t cs = nullptr;
  // weight-gradient GEMMs run on a side stream: off the critical path G_l -> dH -> next SpMM, their
  // HBM traffic overlaps the (L2- or latency-bound) backward aggregations
  cudaStream_t ss = nullptr;
  cudaEvent_t ev_g = nullptr, ev_ss = nullptr;
  bool side_tn = false;  // set at create: only when the aggregation operands are small (see there)
  cudaEvent_t ev_pack = nullptr, ev_halo = nullptr, ev_grad = nullptr, ev_comm_done = nullptr, ev_loss = nullptr;
  cudaEvent_t ev_copied = nullptr, ev_derived = nullptr;  // mph_gcn_upload_features_async pipeline
  // CUDA-graph replay of one epoch: step counter and loss live in device memory
  int32_t* t_dev = nullptr;
  double* loss_dev = nullptr;
  bool graph_mode = false;  // set while capturing: kernels read t / epoch from t_dev
  bool warm = false;        // one eager epoch done (lazy setup finished)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  mph_optim_cfg graph_cfg{};
};

namespace mph {

static int64_t align16(int64_t x) { return (x + 15) / 16 * 16; }

static bool in_arena(const mph_gcn* m, const void* ptr) {
  if (!m->p2p || !m->p2p->arena || !ptr) return false;
  const char* c = (const char*)ptr;
  return c >= m->p2p->arena && c < m->p2p->arena + m->p2p->arena_bytes;
}

static void gcn_free(mph_gcn* m) {
  if (!m) return;
  for (auto& l : m->layers) {
    if (!in_arena(m, l.T)) dev_free(l.T);
    dev_free(l.out);
    dev_free(l.sb);
    if (!in_arena(m, l.dZ)) dev_free(l.dZ);
    dev_free(l.G);
    dev_free(l.Y);
    dev_free(l.colsum);
    dev_free(l.arg);
    dev_free(l.dY);
  }
  if (m->own_params) dev_free(m->params);
  if (m->own_grads) dev_free(m->grads);
  if (m->own_m) dev_free(m->m);
  if (m->own_v) dev_free(m->v);
  dev_free(m->wt);
  dev_free(m->wr);
  dev_free(m->Xr);
  dev_free(m->part0);
  if (!in_arena(m, m->Xs)) dev_free(m->Xs);
  if (m->own_ws) dev_free(m->ws);
  for (cudaEvent_t e : {m->ev_pack, m->ev_halo, m->ev_grad, m->ev_comm_done, m->ev_loss, m->ev_copied, m->ev_derived})
    if (e) cudaEventDestroy(e);
  if (m->cs) cudaStreamDestroy(m->cs);
  if (m->ss) cudaStreamDestroy(m->ss);
  for (cudaEvent_t e : {m->ev_g, m->ev_ss})
    if (e) cudaEventDestroy(e);
  if (m->graph_exec) cudaGraphExecDestroy(m->graph_exec);
  if (m->graph) cudaGraphDestroy(m->graph);
  dev_free(m->t_dev);
  dev_free(m->loss_dev);
  p2p_free(m->p2p);
  delete m;
}

// The feature mode and every layer's order (Q7) decide which buffers cross ranks and at which
// widths, so all ranks must take the same decisions (a rank-local dense/sparse switch would give
// mismatched exchanges).  Bit 0: mode; bit 1 + l: order of layer l.
static uint32_t layout_signature(const mph_features* f, const std::vector<Layer>& layers) {
  uint32_t sig = (uint32_t)(f->mode & 1);
  for (size_t i = 0; i < layers.size() && i < 20; ++i) sig |= (uint32_t)(layers[i].order & 1) << (i + 1);
  return sig;
}

// NCCL transport: Σ sig and Σ sig² over the ranks equal world·sig and world·sig² iff every rank
// has the same signature (exact in FP64: sig < 2^21).  Setup only (synchronises).
static int check_layout_agrees(mph_comm* c, uint32_t sig, cudaStream_t s) {
  int32_t world = 1, rank = 0;
  MPH_TRY(mph_comm_info(c, &world, &rank));
  if (world <= 1) return MPH_OK;
  double h[2] = {(double)sig, (double)sig * (double)sig};
  double* d = nullptr;
  MPH_TRY(dev_alloc(&d, 2));
  cudaError_t e = cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, s);
  int rc = e == cudaSuccess ? mph_allreduce_sum(c, d, 2, 1, s) : fail(MPH_ECUDA, "layout check: %s", cudaGetErrorString(e));
  if (rc == MPH_OK) e = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (rc == MPH_OK && e == cudaSuccess) e = cudaStreamSynchronize(s);
  dev_free(d);
  MPH_TRY(rc);
  if (e != cudaSuccess) return fail(MPH_ECUDA, "layout check: %s", cudaGetErrorString(e));
  if (h[0] != (double)world * sig || h[1] != (double)world * sig * (double)sig)
    return fail(MPH_EINVAL,
                "gcn_create: ranks decided different feature modes / layer orders (this rank 0x%x): the dense/sparse "
                "switch must be global (decide it from the global nnz, mph_features_decide, and pass force_mode)",
                sig);
  return MPH_OK;
}

// element `off` of a buffer that holds bf16 (BF16 mode) or float values
static float* elem(const mph_gcn* m, float* base, int64_t off) {
  return m->bf16 ? reinterpret_cast<float*>(reinterpret_cast<uint16_t*>(base) + off) : base + off;
}
// the bf16-or-tf32 stored-output epilogue flag for tensors that only feed GEMMs
static uint32_t gemm_operand_flag(const mph_gcn* m) { return m->bf16 ? MPH_EPI_BF16 : MPH_EPI_TF32; }

static int refresh_wt(mph_gcn* m, cudaStream_t s) {
  for (auto& l : m->layers)
    MPH_TRY(weight_copies_launch(m->params + l.off_w, l.pin, l.pout, l.pout, elem(m, m->wt, l.off_wt), l.pin,
                                 elem(m, m->wr, l.off_w), l.pout, s, m->bf16));
  return MPH_OK;
}

// SURVEY §8(d) d.3 algorithmic bytes: per edge 4 B col_idx + 4·w B gathered row (no reuse),
// per row 8 B row_ptr + 4 B dinv + 4·w B written.
static double spmm_bytes(const mph_graph* g, int w) {
  const double rows = g->n_rows, nnz = (double)g->nnz;
  return 8.0 * (rows + 1) + 4.0 * nnz + 4.0 * rows + 4.0 * nnz * w + 4.0 * rows * w;
}
static int spmm_p(const mph_graph* g, const float* in, int w, int ld_in, float* out, int ld_out, const mph_epilogue* e,
                  const float* post, cudaStream_t s) {
  prof::Scope sc(MPH_PROF_SPMM, s, spmm_bytes(g, w), 2.0 * (double)g->nnz * w);
  return spmm_launch(g, -1, in, w, ld_in, out, ld_out, e, post, s);
}

// a10 + a3/a6: aggregation whose input's ghost rows come from their owners.  With P > 1 the
// pack runs on the compute stream, the grouped send/recv on the comm stream, and the
// local-edge part of the SpMM overlaps the transfer; the ghost-edge part and the fused
// epilogue run once the halo has landed (overlap P:765).
// Shared-buffer indices of the P2P arena (P2PState::off_buf): T'_l, dZ'_l, dinv ⊙ X.
static int buf_T(int li) { return 2 * li; }
static int buf_dZ(int li) { return 2 * li + 1; }
static int buf_Xs(const mph_gcn* m) { return 2 * m->L; }

static int spmm_halo(mph_gcn* m, float* in, int w, float* out, const mph_epilogue* e, const float* post, int xchg,
                     int buf, cudaStream_t s) {
  const mph_graph* g = m->g;
  if (m->world == 1) return spmm_p(g, in, w, w, out, w, e, post, s);
  if (m->p2p) {
    // NEXT-1: publish "my rows of this buffer are final" (exchange xchg of this generation),
    // then the comm stream pulls the ghost rows from their owners over NVLink
    MPH_TRY(p2p_signal(m->p2p, kSlotHalo, true, kP2PHaloPerGen, xchg, s));
    MPH_CUDA_TRY(cudaEventRecord(m->ev_pack, s));
    MPH_CUDA_TRY(cudaStreamWaitEvent(m->cs, m->ev_pack, 0));
    prof::Scope sc(MPH_PROF_HALO, m->cs, 4.0 * (double)(g->n_cols - g->n_rows) * w, 0.0);
    MPH_TRY(p2p_pull(m->p2p, buf, in, w, kSlotHalo, true, kP2PHaloPerGen, xchg, m->cs));
  } else {
    MPH_TRY(halo_pack(g, in, w, w, s));
    MPH_CUDA_TRY(cudaEventRecord(m->ev_pack, s));
    MPH_CUDA_TRY(cudaStreamWaitEvent(m->cs, m->ev_pack, 0));
    prof::Scope sc(MPH_PROF_HALO, m->cs, 4.0 * (double)(g->n_cols - g->n_rows) * w, 0.0);
    MPH_TRY(halo_sendrecv(g, m->comm, in, w, w, m->cs));
  }
  MPH_CUDA_TRY(cudaEventRecord(m->ev_halo, m->cs));
  prof::Scope sc(MPH_PROF_SPMM, s, spmm_bytes(g, w), 2.0 * (double)g->nnz * w);
  // a BF16 output cannot hold part 0's raw sums: they go to an FP32 scratch (part0)
  const bool bf_out = e && (e->flags & MPH_EPI_BF16);
  MPH_TRY(spmm_launch(g, 0, in, w, w, bf_out ? m->part0 : out, w, nullptr, post, s));
  MPH_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_halo, 0));
  return spmm_launch(g, 1, in, w, w, out, w, e, post, s, bf_out ? m->part0 : nullptr);
}

// a11: all-reduce one layer's [dW_l | b_l] gradient segment on the comm stream as soon as it is
// complete, overlapping the rest of the backward pass (P:525-532 pipelined backward).
// P2P: the dW GEMM's final reduction stores dW_l into every rank's slab itself (GradMirror), so
// only the rest of the segment (b_l and padding) is pushed; `dw_mirrored` says which case.
static int grad_mirror(mph_gcn* m, int li, GradMirror* mir, const GradMirror** out) {
  *out = nullptr;
  if (!m->p2p) return MPH_OK;
  MPH_TRY(p2p_grad_mirror(m->p2p, m->layers[li].off_w, mir));
  *out = mir;
  return MPH_OK;
}

static int grad_allreduce_async(mph_gcn* m, int li, cudaStream_t s, bool dw_mirrored = false) {
  if (m->world == 1) return MPH_OK;
  const int64_t a = dw_mirrored ? m->layers[li].off_b : m->layers[li].off_w;
  const int64_t b = li + 1 < m->L ? m->layers[li + 1].off_w : m->n_params;
  MPH_CUDA_TRY(cudaEventRecord(m->ev_grad, s));
  MPH_CUDA_TRY(cudaStreamWaitEvent(m->cs, m->ev_grad, 0));
  if (m->p2p) return p2p_grad_push(m->p2p, m->grads, a, b, m->cs);  // NEXT-1: into every rank's slab
  return mph_allreduce_sum(m->comm, m->grads + a, b - a, 0, m->cs);
}
static int gemm_nt_p(int M, int N, int K, const float* A, int lda, const float* Bt, int ldb, float* C, int ldc,
                     const mph_epilogue* e, cudaStream_t s, int colsum_fill = 1, bool bf16 = false) {
  const uint32_t f = e ? e->flags : 0u;
  const double in_b = bf16 ? 2.0 : 4.0, out_b = (f & MPH_EPI_BF16) ? 2.0 : 4.0;
  // mask read (4 B / 2 B per element, a sign byte per 4 with MASK_BITS) + sign bytes written
  const double extra = ((f & MPH_EPI_MASK) ? ((f & MPH_EPI_MASK_BITS) ? 0.25 : (f & MPH_EPI_MASK_BF16) ? 2.0 : 4.0)
                                           : 0.0) * M * N +
                       ((f & MPH_EPI_SIGNBITS) ? 0.25 * M * N : 0.0);
  prof::Scope sc(MPH_PROF_GEMM_NT, s, in_b * ((double)M * K + (double)N * K) + out_b * M * N + extra,
                 2.0 * M * N * K);
  return gemm_nt_launch_ex(M, N, K, A, lda, Bt, ldb, C, ldc, e, s, colsum_fill, bf16);
}
static int gemm_tn_p(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C, int ldc,
                     void* ws, size_t wsb, cudaStream_t s, const GradMirror* mirror = nullptr, bool bf16 = false) {
  prof::Scope sc(MPH_PROF_GEMM_TN, s, (bf16 ? 2.0 : 4.0) * ((double)K * M + (double)K * N) + 4.0 * M * N,
                 2.0 * M * N * K);
  return gemm_tn_launch_ex(M, N, K, A, lda, B, ldb, C, ldc, ws, wsb, s, mirror, bf16);
}

static mph_epilogue epi_none() {
  mph_epilogue e{};
  e.mask_scale = 1.0f;
  return e;
}

static float dropout_scale(float p) { return p > 0.0f ? (float)(1.0 / (1.0 - (double)p)) : 1.0f; }

// max aggregation (aggregate.cu): per edge 4 B id + 4·w gathered, per row ptr + Y (+ arg) rows
static int aggmax_p(const mph_graph* g, const float* in, int w, int ld_in, float* Y, int32_t* arg, cudaStream_t s) {
  prof::Scope sc(MPH_PROF_SPMM, s, 8.0 * (g->n_rows + 1) + (4.0 + 4.0 * w) * g->nnz + (arg ? 8.0 : 4.0) * w * g->n_rows,
                 (double)g->nnz * w);
  mph_epilogue en = epi_none();
  en.flags = MPH_EPI_TF32;  // Y only feeds the GEMMs
  return aggregate_max_launch(g, in, w, ld_in, Y, w, arg, w, &en, s);
}
// ... and its adjoint: per edge 4 B id + 8·w (dY and arg rows), per row ptr + mask read + dH write
static int aggmax_bwd_p(const mph_graph* g, const float* dY, const int32_t* arg, int w, float* dH, const float* mask,
                        float mask_scale, cudaStream_t s) {
  prof::Scope sc(MPH_PROF_SPMM, s, 8.0 * (g->n_rows + 1) + (4.0 + 8.0 * w) * g->nnz + 8.0 * w * g->n_rows,
                 (double)g->nnz * w);
  mph_epilogue e = epi_none();
  e.flags = MPH_EPI_MASK | MPH_EPI_TF32;  // dZ_{l-1} feeds the dW and dY GEMMs
  e.mask_src = mask;
  e.ld_mask = w;
  e.mask_scale = mask_scale;
  return aggregate_max_backward_launch(g, dY, w, w, arg, w, dH, w, &e, s);
}

static int layer_forward(mph_gcn* m, int li, cudaStream_t s) {
  Layer& l = m->layers[li];
  const mph_graph* g = m->g;
  const int lnum = li + 1;
  const bool hidden = lnum < m->L;
  mph_epilogue eo = epi_none();
  // hidden outputs only feed tensor-core GEMMs (and the ReLU-mask sign test): store them as TF32
  eo.flags = MPH_EPI_BIAS | (hidden ? (MPH_EPI_RELU | gemm_operand_flag(m)) : 0u);
  eo.bias = m->params + l.off_b;
  if (hidden && l.sb) {
    eo.flags |= MPH_EPI_SIGNBITS;
    eo.bits_out = reinterpret_cast<uint32_t*>(l.sb);
    eo.ld_bits = l.ld_sb;
  }
  if (hidden && m->dropout_p > 0.0f) {
    eo.flags |= MPH_EPI_DROPOUT;
    eo.dropout_p = m->dropout_p;
    eo.dropout_seed = m->dropout_seed;
    eo.dropout_layer = lnum;
    eo.dropout_epoch = m->epoch;
    eo.dropout_epoch_d = m->graph_mode ? m->t_dev : nullptr;
    eo.row0 = g->row0;
  }
  if (m->agg == MPH_AGG_MAX) {
    // R7: Y_l = MAX(H_{l-1}) (with argmax; Y_1 = MAX(X) is prepared once), Z_l = Y_l·W_l + b
    if (li > 0) MPH_TRY(aggmax_p(g, m->layers[li - 1].out, l.pin, l.pin, l.Y, l.arg, s));
    return gemm_nt_p(g->n_rows, l.pout, l.pin, l.Y, l.pin, m->wt + l.off_wt, l.pin, l.out, l.pout, &eo, s);
  }
  if (l.order == 0) {
    // a2/a4: T' = pre ⊙ (H_{l-1} · W_l)   (pre = dinv for the GCN)
    if (li == 0 && m->f->mode == 1) {
      // no-reuse count (as for the SpMM): per nonzero 8 B (col, val) + a W row; per row ptr + T row
      prof::Scope sc(MPH_PROF_SPARSE, s, (8.0 + 4.0 * l.pout) * m->f->nnz + (8.0 + 4.0 * l.pout) * g->n_rows,
                     2.0 * m->f->nnz * l.pout);
      MPH_TRY(sparse_xw_launch(m->f, m->params + l.off_w, l.pout, l.pout, m->fpre, l.T, l.pout, s));
    } else {
      const float* A = li == 0 ? m->Xr : m->layers[li - 1].out;
      const int lda = li == 0 ? m->f->P : m->layers[li - 1].pout;
      mph_epilogue et = epi_none();
      et.flags = m->fpre ? MPH_EPI_ROWSCALE : 0u;
      et.row_scale = m->fpre;
      MPH_TRY(gemm_nt_p(g->n_rows, l.pout, l.pin, A, lda, elem(m, m->wt, l.off_wt), l.pin, l.T, l.pout, &et, s, 1,
                        m->bf16));
    }
    // a10 + a3: ghost rows of T' from their owners; Z = Â·T + b, ReLU (dropout) fused
    MPH_TRY(spmm_halo(m, l.T, l.pout, l.out, &eo, m->fpost, li, buf_T(li), s));
  } else {
    // aggregate-first layer 1: Y = Â·X (on dinv ⊙ X), Z = Y·W + b with the epilogue fused in the GEMM
    mph_epilogue en = epi_none();
    en.flags = gemm_operand_flag(m);  // Y only feeds the GEMMs
    MPH_TRY(spmm_p(g, m->Xs, l.pin, l.pin, l.Y, l.pin, &en, m->fpost, s));
    MPH_TRY(gemm_nt_p(g->n_rows, l.pout, l.pin, l.Y, l.pin, elem(m, m->wt, l.off_wt), l.pin, l.out, l.pout, &eo, s, 1,
                      m->bf16));
  }
  return MPH_OK;
}

static int do_forward(mph_gcn* m, int epoch, cudaStream_t s) {
  m->epoch = epoch;
  if (m->p2p) MPH_TRY(p2p_gen_advance(m->p2p, s));  // one generation of flags per epoch
  for (int li = 0; li < m->L; ++li) MPH_TRY(layer_forward(m, li, s));
  m->fwd_done = true;
  m->loss_done = false;
  return MPH_OK;
}

static int do_loss(mph_gcn* m, double* loss_d, cudaStream_t s) {
  if (!m->fwd_done) return fail(MPH_ESTATE, "loss before forward (S:353)");
  if (!m->labels) return fail(MPH_ESTATE, "labels not set");
  Layer& l = m->layers[m->L - 1];
  prof::Scope sc(MPH_PROF_LOSS, s, 8.0 * m->g->n_rows * l.pout + 4.0 * m->g->n_rows, 0.0);
  // TF: dZ' = bpre ⊙ dZ feeds the backward aggregation (FP32); max: dZ feeds the GEMMs (TF32)
  const bool max_agg = m->agg == MPH_AGG_MAX;
  MPH_TRY(softmax_ce_launch(l.out, m->g->n_rows, l.fout, l.pout, m->labels, m->mask, m->n_lab,
                            (l.order == 0 && !max_agg) ? m->bpre : nullptr, l.dZ, l.pout, m->grads + l.off_b, loss_d,
                            m->ws, m->ws_bytes, s, max_agg ? 1 : 0));
  m->loss_done = true;
  return MPH_OK;
}

static int do_backward(mph_gcn* m, cudaStream_t s) {
  if (!m->loss_done) return fail(MPH_ESTATE, "backward without a matching forward+loss (S:353)");
  bool forked = false;  // weight-gradient GEMMs sent to the side stream this pass
  const mph_graph* g = m->g;
  for (int li = m->L - 1; li >= 0 && m->agg == MPH_AGG_MAX; --li) {
    // R7: Z = Y·W + b:  dW = Yᵀ·dZ;  dY = dZ·Wᵀ;  dZ_{l-1} = route(dY, arg) ⊙ ReLU'(H_{l-1}) (/(1-p))
    Layer& l = m->layers[li];
    MPH_TRY(gemm_tn_p(l.pin, l.pout, g->n_rows, l.Y, l.pin, l.dZ, l.pout, m->grads + l.off_w, l.pout, m->ws,
                      m->ws_bytes, s));
    if (li > 0) {
      Layer& pl = m->layers[li - 1];
      MPH_TRY(gemm_nt_p(g->n_rows, l.pin, l.pout, l.dZ, l.pout, m->wr + l.off_w, l.pout, l.dY, l.pin, nullptr, s));
      MPH_TRY(aggmax_bwd_p(g, l.dY, l.arg, l.pin, pl.dZ, pl.out, dropout_scale(m->dropout_p), s));
      MPH_TRY(colsum_chunks_launch(pl.dZ, g->n_rows, pl.pout, pl.pout, pl.colsum, s));
      MPH_TRY(reduce_rows_launch(pl.colsum, (int)ceil_div(g->n_rows, 128), pl.pout, pl.pout, m->grads + pl.off_b, 0, s));
    }
  }
  for (int li = m->L - 1; li >= 0 && m->agg != MPH_AGG_MAX; --li) {
    Layer& l = m->layers[li];
    GradMirror mir{};
    const GradMirror* mirp = nullptr;  // set when this layer's dW GEMM writes every rank's slab itself
    cudaStream_t gs = s;               // the stream that finishes [dW_l | db_l]
    const float* Hin = li == 0 ? m->Xr : m->layers[li - 1].out;
    const int ld_in = li == 0 ? m->f->P : m->layers[li - 1].pout;
    const float* Gsrc;  // gradient w.r.t. the transform output (TF) or Z (AF)
    if (l.order == 0) {
      // a10 + a6: G = AGGᵀ·dZ = bpost ⊙ Ã·dZ' (Â symmetric: the forward kernel)
      mph_epilogue en = epi_none();
      // G only feeds the dW and dH GEMMs (sparse layer 1: the CUDA-core X_cscᵀ·G gather, FP32 input)
      const bool sparse_l1 = li == 0 && m->f->mode == 1;
      en.flags = sparse_l1 ? MPH_EPI_TF32 : gemm_operand_flag(m);
      // exchange indices must increase within a generation (the flags are monotone counters):
      // forward layers 0..L-1, then backward layers L-1..0
      MPH_TRY(spmm_halo(m, l.dZ, l.pout, l.G, &en, m->bpost, 2 * m->L - 1 - li, buf_dZ(li), s));
      Gsrc = l.G;
      // a7: dW = H^T·G  (sparse layer 1: X_csc^T·G)
      if (li == 0 && m->f->mode == 1) {
        // per nonzero 8 B + a G row; per column ptr + dW row (segment partials not counted)
        prof::Scope sc(MPH_PROF_SPARSE, s, (8.0 + 4.0 * l.pout) * m->f->nnz + (8.0 + 4.0 * l.pout) * m->f->F,
                       2.0 * m->f->nnz * l.pout);
        MPH_TRY(sparse_xtg_launch(m->f, l.G, l.pout, l.pout, m->grads + l.off_w, l.pout, s));
      } else {
        MPH_TRY(grad_mirror(m, li, &mir, &mirp));
        if (m->side_tn) {
          MPH_CUDA_TRY(cudaEventRecord(m->ev_g, s));  // G_l (and db_l) are final
          MPH_CUDA_TRY(cudaStreamWaitEvent(m->ss, m->ev_g, 0));
          gs = m->ss;
          forked = true;
        }
        MPH_TRY(gemm_tn_p(l.pin, l.pout, g->n_rows, Hin, ld_in, l.G, l.pout, m->grads + l.off_w, l.pout, m->ws,
                          m->ws_bytes, gs, mirp, m->bf16));
      }
    } else {
      // AF layer 1: dZ_1 (unscaled) is the gradient of Z = Y·W + b
      Gsrc = l.dZ;
      MPH_TRY(grad_mirror(m, li, &mir, &mirp));
      if (m->side_tn) {
        MPH_CUDA_TRY(cudaEventRecord(m->ev_g, s));
        MPH_CUDA_TRY(cudaStreamWaitEvent(m->ss, m->ev_g, 0));
        gs = m->ss;
        forked = true;
      }
      MPH_TRY(gemm_tn_p(l.pin, l.pout, g->n_rows, l.Y, l.pin, l.dZ, l.pout, m->grads + l.off_w, l.pout, m->ws,
                        m->ws_bytes, gs, mirp, m->bf16));
    }
    // [dW_l | db_l] complete (db_l came from the loss or the layer above): reduce it across ranks
    // while this layer's dH and the layers below proceed (a11)
    MPH_TRY(grad_allreduce_async(m, li, gs, mirp != nullptr));
    if (li > 0) {
      // a8: dZ_{l-1} = (G·W^T) ⊙ 1[H_{l-1} > 0] (/(1-p)), db_{l-1} as column sums, then the dinv
      // pre-scale for the next backward SpMM (TF) — all in one GEMM epilogue.
      Layer& pl = m->layers[li - 1];
      mph_epilogue ed = epi_none();
      // TF: dZ' feeds the FP32 SpMM (keep FP32); AF: dZ_1 feeds only the dW GEMM (TF32)
      ed.flags = MPH_EPI_MASK | MPH_EPI_COLSUM |
                 (pl.sb ? MPH_EPI_MASK_BITS : (m->bf16 ? MPH_EPI_MASK_BF16 : 0u)) |
                 (pl.order == 0 ? (m->bpre ? MPH_EPI_ROWSCALE : 0u) : gemm_operand_flag(m));
      ed.mask_src = pl.sb ? reinterpret_cast<const float*>(pl.sb) : pl.out;
      ed.ld_mask = pl.sb ? pl.ld_sb : pl.pout;
      ed.mask_scale = dropout_scale(m->dropout_p);
      ed.colsum_out = pl.colsum;
      ed.row_scale = m->bpre;
      MPH_TRY(gemm_nt_p(g->n_rows, pl.pout, l.pout, Gsrc, l.pout, elem(m, m->wr, l.off_w), l.pout, pl.dZ, pl.pout,
                        &ed, s, /*colsum_fill=*/0, m->bf16));
      // db_{l-1}: the GEMM wrote one column-sum row per persistent CTA
      MPH_TRY(reduce_rows_launch(pl.colsum, gemm_nt_colsum_rows(g->n_rows), pl.pout, pl.pout, m->grads + pl.off_b, 0,
                                 s));
    }
  }
  if (forked) {  // the optimizer needs every dW: join the side stream
    MPH_CUDA_TRY(cudaEventRecord(m->ev_ss, m->ss));
    MPH_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_ss, 0));
  }
  if (m->world > 1) {  // Adam needs every summed gradient segment
    if (m->p2p) MPH_TRY(p2p_signal(m->p2p, kSlotGrad, true, 1, 0, m->cs));  // all my slabs are pushed
    MPH_CUDA_TRY(cudaEventRecord(m->ev_comm_done, m->cs));
    MPH_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_comm_done, 0));
  }
  m->fwd_done = false;
  m->loss_done = false;
  return MPH_OK;
}

}  // namespace mph

using namespace mph;

extern "C" int mph_gcn_create(const mph_graph* g, const mph_features* f, const mph_gcn_desc* desc, mph_comm* comm,
                              void* stream, mph_gcn** out) {
  if (!g || !f || !desc || !out || !desc->dims_h || desc->num_layers < 1) return fail(MPH_EINVAL, "gcn_create arguments");
  *out = nullptr;
  if (f->N != g->n_rows) return fail(MPH_EINVAL, "features rows (%d) != graph rows (%d)", f->N, g->n_rows);
  if (desc->dims_h[0] != f->F) return fail(MPH_EINVAL, "dims[0]=%d != feature width %d", desc->dims_h[0], f->F);
  if (desc->dropout_p < 0.0f || desc->dropout_p >= 1.0f) return fail(MPH_EINVAL, "dropout_p must be in [0,1)");
  if (desc->aggregator < MPH_AGG_GCN || desc->aggregator > MPH_AGG_MAX)
    return fail(MPH_EINVAL, "unknown aggregator %d", desc->aggregator);
  if (desc->comm_mode != MPH_COMM_NCCL && desc->comm_mode != MPH_COMM_P2P)
    return fail(MPH_EINVAL, "unknown comm_mode %d", desc->comm_mode);
  if (desc->precision != MPH_PREC_TF32 && desc->precision != MPH_PREC_BF16)
    return fail(MPH_EINVAL, "unknown precision %d", desc->precision);
  if (desc->precision == MPH_PREC_BF16 && desc->aggregator == MPH_AGG_MAX)
    return fail(MPH_ENOTSUP, "BF16 GEMM operands: linear aggregators only");
  if (desc->precision == MPH_PREC_BF16 && f->mode == 0 && f->P % 8)
    return fail(MPH_ENOTSUP, "BF16 GEMM operands: dense features need a padded width multiple of 8 (F > 4)");
  const bool p2p = desc->comm_mode == MPH_COMM_P2P && g->local && g->world > 1;
  int world = 1;
  if (p2p) {
    if (comm) return fail(MPH_EINVAL, "MPH_COMM_P2P takes comm = NULL (the peers are mapped by mph_gcn_p2p_open)");
    if (g->world > kP2PMaxWorld) return fail(MPH_ENOTSUP, "MPH_COMM_P2P: world %d > %d", g->world, kP2PMaxWorld);
    if (2 * desc->num_layers > kP2PHaloPerGen) return fail(MPH_ENOTSUP, "MPH_COMM_P2P: more than 8 layers");
    world = g->world;
  } else if (comm) {
    MPH_TRY(mph_comm_info(comm, &world, nullptr));
  }
  if (world > 1 && !g->local) return fail(MPH_EINVAL, "distributed model needs a localized graph");
  if (g->local && g->world > 1 && world != g->world)
    return fail(MPH_EINVAL, "localized graph of world %d needs a comm (NCCL) or comm_mode = MPH_COMM_P2P", g->world);
  const bool max_agg = desc->aggregator == MPH_AGG_MAX;
  if (max_agg && (world > 1 || f->mode != 0))
    return fail(MPH_ENOTSUP, "max aggregation: single GPU, dense-mode features only");
  for (int i = 0; i <= desc->num_layers; ++i)
    if (desc->dims_h[i] <= 0 || pad_width(desc->dims_h[i]) > 256 + (i == 0 ? 1 << 20 : 0))
      return fail(MPH_ENOTSUP, "layer width %d outside (0, 256]", desc->dims_h[i]);
  cudaStream_t s = (cudaStream_t)stream;
  mph_gcn* m = new mph_gcn();
  m->g = g;
  m->f = f;
  m->comm = comm;
  m->world = world;
  m->L = desc->num_layers;
  m->dropout_p = desc->dropout_p;
  m->dropout_seed = desc->dropout_seed;
  m->agg = desc->aggregator;
  m->bf16 = desc->precision == MPH_PREC_BF16;
  if (!max_agg) {
    MPH_TRY(agg_scales(g, m->agg, 0, &m->fpre, &m->fpost));
    MPH_TRY(agg_scales(g, m->agg, 1, &m->bpre, &m->bpost));
  }
  m->layers.resize(m->L);
  int64_t off = 0, offt = 0;
  for (int li = 0; li < m->L; ++li) {
    Layer& l = m->layers[li];
    l.fin = desc->dims_h[li];
    l.fout = desc->dims_h[li + 1];
    // BF16 operands need 16-byte rows: widths padded to multiples of 8 (pad_width gives 4 for w <= 4)
    auto padw = [&](int w) { return m->bf16 ? round_up(w, 8) : pad_width(w); };
    l.pin = li == 0 ? (f->mode == 0 ? f->P : pad_width(f->F)) : padw(l.fin);
    l.pout = padw(l.fout);
    // reading Q7: TF iff F_out <= F_in, or layer 1 in Sparse mode; AF only ever needed on layer 1
    l.order = (desc->order_policy == 1 || l.fout <= l.fin || (li == 0 && f->mode == 1) || li > 0) ? 0 : 1;
    if (max_agg) l.order = 1;  // max is taken before the transform on every layer (R7)
    l.off_w = off;
    off = align16(off + (int64_t)l.pin * l.pout);
    l.off_b = off;
    off = align16(off + l.pout);
    l.off_wt = offt;
    offt = align16(offt + (int64_t)l.pout * l.pin);
  }
  m->n_params = off;
  m->n_wt = offt;
  if (m->bf16 && m->L == 1 && m->layers[0].order == 1) {
    gcn_free(m);
    return fail(MPH_ENOTSUP, "BF16: a one-layer aggregate-first model (its loss gradient feeds a GEMM directly)");
  }
  int rc = MPH_OK;
  auto bail = [&](int code) {
    gcn_free(m);
    return code;
  };
  if ((rc = dev_alloc(&m->params, off)) || (rc = dev_alloc(&m->grads, off)) || (rc = dev_alloc(&m->m, off)) ||
      (rc = dev_alloc(&m->v, off)) || (rc = dev_alloc(&m->wt, offt)) || (rc = dev_alloc(&m->wr, off)))
    return bail(rc);
  size_t ws = softmax_ce_ws_bytes(g->n_rows, m->layers.back().fout);
  const int64_t nr = g->n_rows, nc = g->n_cols;
  // NEXT-1: every buffer a peer reads (T'_l, dZ'_l of transform-first layers, dinv ⊙ X of an
  // aggregate-first layer 1) is carved from the rank's peer-mapped arena
  auto shared_bytes = [&](int64_t rows, int w) { return (rows * w * 4 + 255) / 256 * 256; };
  int64_t arena_next = 0;
  auto carve = [&](float** ptr, int64_t rows, int w, int buf) {
    m->p2p->off_buf[buf] = arena_next;
    *ptr = (float*)(m->p2p->arena + arena_next);
    arena_next += shared_bytes(rows, w);
  };
  if (p2p) {
    m->p2p = new P2PState();
    m->p2p->world = world;
    m->p2p->rank = g->rank;
    m->p2p->n_params = off;
    m->p2p->n_rows = nr;
    m->p2p->row0 = g->row0;
    m->p2p->off_buf.assign(2 * m->L + 1, -1);
    m->p2p->layout_sig = layout_signature(f, m->layers);
    int64_t bytes = 0;
    for (const auto& l : m->layers)
      if (l.order == 0) bytes += 2 * shared_bytes(nc, l.pout);
    if (m->layers[0].order == 1) bytes += shared_bytes(nc, m->layers[0].pin);
    if ((rc = p2p_alloc_arena(m->p2p, (size_t)bytes))) return bail(rc);
    arena_next = (int64_t)m->p2p->arena_bytes - bytes;
  }
  for (int li = 0; li < m->L; ++li) {
    Layer& l = m->layers[li];
    if ((rc = dev_alloc(&l.out, (size_t)nr * l.pout))) return bail(rc);
    if (p2p && l.order == 0)
      carve(&l.dZ, nc, l.pout, buf_dZ(li));
    else if ((rc = dev_alloc(&l.dZ, (size_t)(l.order == 0 ? nc : nr) * l.pout)))
      return bail(rc);
    if ((rc = dev_alloc(&l.colsum, (size_t)ceil_div(nr, 128) * l.pout))) return bail(rc);
#ifndef MPH_NO_SIGNBYTES
    if (!max_agg && li + 1 < m->L) {
      l.ld_sb = (int)round_up((int)ceil_div(l.pout, 4), 8);
      if ((rc = dev_alloc(&l.sb, (size_t)nr * l.ld_sb))) return bail(rc);
    }
#endif
    if (max_agg) {
      if ((rc = dev_alloc(&l.Y, (size_t)nr * l.pin))) return bail(rc);
      if (li > 0 && ((rc = dev_alloc(&l.arg, (size_t)nr * l.pin)) || (rc = dev_alloc(&l.dY, (size_t)nr * l.pin))))
        return bail(rc);
    } else if (l.order == 0) {
      if (p2p)
        carve(&l.T, nc, l.pout, buf_T(li));
      else if ((rc = dev_alloc(&l.T, (size_t)nc * l.pout)))
        return bail(rc);
      if ((rc = dev_alloc(&l.G, (size_t)nr * l.pout))) return bail(rc);
    } else {
      if ((rc = dev_alloc(&l.Y, (size_t)nr * l.pin))) return bail(rc);
    }
    if (!(li == 0 && f->mode == 1)) ws = std::max(ws, gemm_tn_ws_bytes(l.pin, l.pout, (int)nr));
  }
  m->ws_bytes = ws;
  if ((rc = dev_alloc((char**)&m->ws, ws))) return bail(rc);
  if ((rc = dev_alloc(&m->t_dev, 1)) || (rc = dev_alloc(&m->loss_dev, 1))) return bail(rc);
  cudaError_t e = cudaSuccess;
  for (auto& l : m->layers) {  // padding columns must start (and stay) zero
    if (e == cudaSuccess) e = cudaMemsetAsync(l.out, 0, (size_t)nr * l.pout * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(l.dZ, 0, (size_t)(l.order == 0 ? nc : nr) * l.pout * 4, s);
    if (e == cudaSuccess && l.T) e = cudaMemsetAsync(l.T, 0, (size_t)nc * l.pout * 4, s);
    if (e == cudaSuccess && l.G) e = cudaMemsetAsync(l.G, 0, (size_t)nr * l.pout * 4, s);
    if (e == cudaSuccess && l.Y) e = cudaMemsetAsync(l.Y, 0, (size_t)nr * l.pin * 4, s);
    if (e == cudaSuccess && l.dY) e = cudaMemsetAsync(l.dY, 0, (size_t)nr * l.pin * 4, s);
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(m->params, 0, off * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(m->grads, 0, off * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(m->m, 0, off * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(m->v, 0, off * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(m->wt, 0, offt * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(m->wr, 0, off * 4, s);
  if (e != cudaSuccess) return bail(fail(MPH_ECUDA, "gcn_create memset: %s", cudaGetErrorString(e)));
  if (max_agg) {
    // X is constant input data: Y_1 = MAX(X) is computed once (its argmax is never needed)
    const Layer& l = m->layers[0];
    mph_epilogue en = epi_none();
    en.flags = MPH_EPI_TF32;  // Y_1 only feeds the GEMMs
    if ((rc = aggregate_max_launch(g, f->X, l.pin, f->P, l.Y, l.pin, nullptr, 0, &en, s))) return bail(rc);
  } else if (m->layers[0].order == 1) {
    // X is constant input data: its pre-scale (and, distributed, its ghost rows) are set up once.
    const Layer& l = m->layers[0];
    if (p2p)
      carve(&m->Xs, nc, l.pin, buf_Xs(m));
    else if ((rc = dev_alloc(&m->Xs, (size_t)nc * l.pin)))
      return bail(rc);
    e = cudaMemsetAsync(m->Xs, 0, (size_t)nc * l.pin * 4, s);
    if (e != cudaSuccess) return bail(fail(MPH_ECUDA, "memset: %s", cudaGetErrorString(e)));
    if ((rc = rowscale_launch(f->X, f->P, m->fpre, (int)nr, l.pin, m->Xs, l.pin, 0, s))) return bail(rc);
    // P2P: the ghost rows of dinv ⊙ X arrive in mph_gcn_p2p_open, once the peers are mapped
    if (world > 1 && !p2p && (rc = mph_halo_exchange(g, comm, m->Xs, l.pin, l.pin, s))) return bail(rc);
  }
  // Side-stream weight gradients pay off when the backward aggregations leave HBM idle (operands
  // L2-resident or small: reddit -0.3 %, arxiv -4 %); next to HBM-bound aggregations (products,
  // 2.5 GB operands) the two compete and the epoch gets slower (+3 %), so they stay in line there.
  {
    int wmax2 = 0;
    for (const auto& l : m->layers) wmax2 = std::max(wmax2, l.pout);
    m->side_tn = (double)nc * wmax2 * 4.0 <= 512.0 * (1 << 20);
  }
  e = cudaStreamCreateWithFlags(&m->ss, cudaStreamNonBlocking);
  for (cudaEvent_t* ev : {&m->ev_g, &m->ev_ss})
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  if (e != cudaSuccess) return bail(fail(MPH_ECUDA, "gcn_create side stream: %s", cudaGetErrorString(e)));
  if (world > 1) {
    e = cudaStreamCreateWithFlags(&m->cs, cudaStreamNonBlocking);
    for (cudaEvent_t* ev : {&m->ev_pack, &m->ev_halo, &m->ev_grad, &m->ev_comm_done, &m->ev_loss})
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return bail(fail(MPH_ECUDA, "gcn_create streams: %s", cudaGetErrorString(e)));
    // widths that cross ranks / leave a split SpMM: T'_l and dZ'_l (pout) of transform-first
    // layers, and dinv ⊙ X (pin) of an aggregate-first layer 1 (its setup exchange and Y_1)
    int wmax = 0;
    for (const auto& l : m->layers) wmax = std::max(wmax, l.order == 0 ? l.pout : l.pin);
    if (!p2p && (rc = halo_reserve(g, wmax))) return bail(rc);  // no reallocation while sends are in flight
    if (m->bf16 && (rc = dev_alloc(&m->part0, (size_t)nr * wmax))) return bail(rc);
    if (!p2p && (rc = check_layout_agrees(m->comm, layout_signature(f, m->layers), s))) return bail(rc);
  }
  if (m->layers[0].order == 0 && f->mode == 0 && !max_agg) {
    // TF32-rounded copy of X: the A operand of the layer-1 transform and of its dW GEMM
    if ((rc = dev_alloc(&m->Xr, (size_t)nr * f->P))) return bail(rc);
    if ((rc = rowscale_launch(f->X, f->P, nullptr, (int)nr, f->P, m->Xr, f->P, m->bf16 ? 2 : 1, s))) return bail(rc);
  }
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return bail(fail(MPH_ECUDA, "gcn_create: %s", cudaGetErrorString(e)));
  *out = m;
  return MPH_OK;
}

extern "C" int mph_gcn_param_layout(const mph_gcn* m, int64_t* num_params_h, int64_t* offsets_h, int32_t* ld_w_h) {
  if (!m) return fail(MPH_EINVAL, "null model");
  if (num_params_h) *num_params_h = m->n_params;
  for (int li = 0; li < m->L; ++li) {
    if (offsets_h) {
      offsets_h[2 * li] = m->layers[li].off_w;
      offsets_h[2 * li + 1] = m->layers[li].off_b;
    }
    if (ld_w_h) ld_w_h[li] = m->layers[li].pout;
  }
  return MPH_OK;
}

extern "C" int mph_gcn_buffers(const mph_gcn* m, float** params_d, float** grads_d, float** adam_m_d, float** adam_v_d) {
  if (!m) return fail(MPH_EINVAL, "null model");
  if (params_d) *params_d = m->params;
  if (grads_d) *grads_d = m->grads;
  if (adam_m_d) *adam_m_d = m->m;
  if (adam_v_d) *adam_v_d = m->v;
  return MPH_OK;
}

extern "C" int mph_gcn_workspace_size(const mph_gcn* m, size_t* bytes_h) {
  if (!m || !bytes_h) return fail(MPH_EINVAL, "gcn_workspace_size arguments");
  *bytes_h = m->ws_bytes;
  return MPH_OK;
}

extern "C" int mph_gcn_bind(mph_gcn* m, float* params_d, float* grads_d, float* adam_m_d, float* adam_v_d,
                            void* workspace_d, size_t ws_bytes) {
  if (!m) return fail(MPH_EINVAL, "null model");
  if (workspace_d && ws_bytes < m->ws_bytes)
    return fail(MPH_EINVAL, "gcn_bind: workspace %zu B < mph_gcn_workspace_size %zu B", ws_bytes, m->ws_bytes);
  for (const void* p : {(const void*)params_d, (const void*)grads_d, (const void*)adam_m_d, (const void*)adam_v_d})
    if (p && (reinterpret_cast<uintptr_t>(p) & 15)) return fail(MPH_EINVAL, "gcn_bind: buffers must be 16-byte aligned");
  if (m->graph_exec) return fail(MPH_ESTATE, "gcn_bind: a captured CUDA graph holds the old buffers");
  MPH_CUDA_TRY(cudaDeviceSynchronize());  // nothing in flight still uses the buffers being replaced
  auto swap = [](float*& cur, bool& own, float* nw) {
    if (!nw) return;
    if (own) dev_free(cur);
    cur = nw;
    own = false;
  };
  swap(m->params, m->own_params, params_d);
  swap(m->grads, m->own_grads, grads_d);
  // gradient entries the kernels never write (padding) must read zero, as in the model's own buffer
  if (grads_d) MPH_CUDA_TRY(cudaMemset(grads_d, 0, (size_t)m->n_params * sizeof(float)));
  swap(m->m, m->own_m, adam_m_d);
  swap(m->v, m->own_v, adam_v_d);
  if (workspace_d) {
    if (m->own_ws) dev_free(m->ws);
    m->ws = workspace_d;
    m->own_ws = false;
  }
  return MPH_OK;
}

extern "C" int mph_gcn_init_xavier(mph_gcn* m, uint64_t seed, void* stream) {
  if (!m) return fail(MPH_EINVAL, "null model");
  cudaStream_t s = (cudaStream_t)stream;
  MPH_CUDA_TRY(cudaMemsetAsync(m->params, 0, m->n_params * 4, s));
  MPH_CUDA_TRY(cudaMemsetAsync(m->m, 0, m->n_params * 4, s));
  MPH_CUDA_TRY(cudaMemsetAsync(m->v, 0, m->n_params * 4, s));
  for (int li = 0; li < m->L; ++li) {
    const Layer& l = m->layers[li];
    MPH_TRY(xavier_launch(m->params + l.off_w, l.fin, l.fout, l.pout, seed, li + 1, s));
  }
  return refresh_wt(m, s);
}

extern "C" int mph_gcn_params_updated(mph_gcn* m, void* stream) {
  if (!m) return fail(MPH_EINVAL, "null model");
  return refresh_wt(m, (cudaStream_t)stream);
}

static int copy_features(const mph_features* f, const float* X_h, int32_t ld_h, cudaStream_t s) {
  if (ld_h == f->P)  // host rows already padded: one contiguous copy (the padding must be zero)
    MPH_CUDA_TRY(cudaMemcpyAsync(f->X, X_h, (size_t)f->N * f->P * 4, cudaMemcpyHostToDevice, s));
  else
    MPH_CUDA_TRY(cudaMemcpy2DAsync(f->X, (size_t)f->P * 4, X_h, (size_t)ld_h * 4, (size_t)f->F * 4, (size_t)f->N,
                                   cudaMemcpyHostToDevice, s));
  return MPH_OK;
}

// Ghost rows of the constant operand dinv ⊙ X (aggregate-first layer 1) over peer memory: a
// setup-slot signal with a host counter (create/upload are not captured in graphs), then a pull.
static int p2p_setup_exchange(mph_gcn* m, cudaStream_t s) {
  const int64_t seq = ++m->p2p->xgen;
  MPH_TRY(p2p_signal(m->p2p, kSlotSetup, false, 0, seq, s));
  return p2p_pull(m->p2p, buf_Xs(m), m->Xs, m->layers[0].pin, kSlotSetup, false, 0, seq, s);
}

// Everything the epoch reads is derived from X here (TF32 copy Xr, pre-scaled Xs, or MAX(X)); the
// epoch itself never reads f->X, so the next step's X may land in f->X while an epoch runs.
static int derive_from_features(mph_gcn* m, cudaStream_t s) {
  const mph_features* f = m->f;
  if (m->agg == MPH_AGG_MAX) {
    const Layer& l = m->layers[0];
    mph_epilogue en = epi_none();
    en.flags = MPH_EPI_TF32;
    MPH_TRY(aggregate_max_launch(m->g, f->X, l.pin, f->P, l.Y, l.pin, nullptr, 0, &en, s));
  } else if (m->layers[0].order == 1) {
    const Layer& l = m->layers[0];
    MPH_TRY(rowscale_launch(f->X, f->P, m->fpre, m->g->n_rows, l.pin, m->Xs, l.pin, 0, s));
    if (m->p2p) {
      MPH_TRY(p2p_setup_exchange(m, s));
    } else if (m->world > 1) {
      MPH_TRY(mph_halo_exchange(m->g, m->comm, m->Xs, l.pin, l.pin, s));
    }
  } else {
    MPH_TRY(rowscale_launch(f->X, f->P, nullptr, m->g->n_rows, f->P, m->Xr, f->P, m->bf16 ? 2 : 1, s));
  }
  return MPH_OK;
}

extern "C" int mph_gcn_upload_features(mph_gcn* m, const float* X_h, int32_t ld_h, void* stream) {
  if (!m || !X_h || ld_h < m->f->F) return fail(MPH_EINVAL, "upload_features arguments");
  if (m->f->mode != 0) return fail(MPH_ENOTSUP, "upload_features: sparse-mode features are fixed at creation");
  cudaStream_t s = (cudaStream_t)stream;
  MPH_TRY(copy_features(m->f, X_h, ld_h, s));
  return derive_from_features(m, s);
}

extern "C" int mph_gcn_upload_features_async(mph_gcn* m, const float* X_h, int32_t ld_h, void* copy_stream,
                                             void* stream) {
  if (!m || !X_h || ld_h < m->f->F) return fail(MPH_EINVAL, "upload_features arguments");
  if (m->f->mode != 0) return fail(MPH_ENOTSUP, "upload_features: sparse-mode features are fixed at creation");
  cudaStream_t cs = (cudaStream_t)copy_stream, s = (cudaStream_t)stream;
  if (!m->ev_copied) {
    MPH_CUDA_TRY(cudaEventCreateWithFlags(&m->ev_copied, cudaEventDisableTiming));
    MPH_CUDA_TRY(cudaEventCreateWithFlags(&m->ev_derived, cudaEventDisableTiming));
    MPH_CUDA_TRY(cudaEventRecord(m->ev_derived, s));
  }
  MPH_CUDA_TRY(cudaStreamWaitEvent(cs, m->ev_derived, 0));  // the previous upload has been consumed
  MPH_TRY(copy_features(m->f, X_h, ld_h, cs));
  MPH_CUDA_TRY(cudaEventRecord(m->ev_copied, cs));
  MPH_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_copied, 0));
  MPH_TRY(derive_from_features(m, s));
  MPH_CUDA_TRY(cudaEventRecord(m->ev_derived, s));
  return MPH_OK;
}

extern "C" int mph_gcn_set_labels(mph_gcn* m, const int32_t* labels_d, const uint8_t* mask_d, int64_t n_lab_global) {
  if (!m || !labels_d || n_lab_global <= 0) return fail(MPH_EINVAL, "set_labels arguments");
  m->labels = labels_d;
  m->mask = mask_d;
  m->n_lab = n_lab_global;
  return MPH_OK;
}

extern "C" int mph_gcn_forward(mph_gcn* m, int32_t epoch, void* stream) {
  if (!m) return fail(MPH_EINVAL, "null model");
  return do_forward(m, epoch, (cudaStream_t)stream);
}

// Loss of this rank's rows, then (P > 1) the global sum over ranks on the comm stream.
static int loss_global(mph_gcn* m, double* loss_d, cudaStream_t s) {
  MPH_TRY(do_loss(m, loss_d, s));
  if (m->world > 1) {  // global loss = sum of per-rank partial sums / global N_lab
    MPH_CUDA_TRY(cudaEventRecord(m->ev_loss, s));
    MPH_CUDA_TRY(cudaStreamWaitEvent(m->cs, m->ev_loss, 0));
    if (m->p2p)
      MPH_TRY(p2p_loss_sum(m->p2p, loss_d, m->cs));
    else
      MPH_TRY(mph_allreduce_sum(m->comm, loss_d, 1, 1, m->cs));
    MPH_CUDA_TRY(cudaEventRecord(m->ev_loss, m->cs));
    MPH_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_loss, 0));
  }
  return MPH_OK;
}

extern "C" int mph_gcn_loss(mph_gcn* m, double* loss_d, void* stream) {
  if (!m || !loss_d) return fail(MPH_EINVAL, "gcn_loss arguments");
  return loss_global(m, loss_d, (cudaStream_t)stream);
}

extern "C" int mph_gcn_backward(mph_gcn* m, void* stream) {
  if (!m) return fail(MPH_EINVAL, "null model");
  // a11 happens inside: per-layer gradient all-reduce pipelined on the comm stream
  return do_backward(m, (cudaStream_t)stream);
}

static mph_optim_cfg as_optim(const mph_adam_cfg* c) {
  return mph_optim_cfg{MPH_OPT_ADAM, c->lr, c->beta1, c->beta2, c->eps, 0.0f, 0.0f};
}

extern "C" int mph_gcn_optim_step(mph_gcn* m, const mph_optim_cfg* cfg, int32_t t, void* stream) {
  if (!m || !cfg) return fail(MPH_EINVAL, "gcn_optim_step arguments");
  cudaStream_t s = (cudaStream_t)stream;
  prof::Scope sc(MPH_PROF_ADAM, s, (cfg->kind == MPH_OPT_SGD ? 20.0 : 28.0) * m->n_params, 0.0);
  if (m->p2p) {  // NEXT-1: gradient all-reduce fused into the update (rank-order slab sum)
    MPH_TRY(optim_sum_launch(m->params, m->grads, m->m, m->v, m->n_params, cfg, t, s,
                             m->graph_mode ? m->t_dev : nullptr, p2p_gsum_local(m->p2p), m->world,
                             p2p_flags_local(m->p2p, kSlotGrad), m->p2p->gen_dev, m->p2p->err_dev));
  } else {
    MPH_TRY(optim_launch(m->params, m->grads, m->m, m->v, m->n_params, cfg, t, s, m->graph_mode ? m->t_dev : nullptr));
  }
  return refresh_wt(m, s);
}

extern "C" int mph_gcn_adam(mph_gcn* m, const mph_adam_cfg* cfg, int32_t t, void* stream) {
  if (!m || !cfg) return fail(MPH_EINVAL, "gcn_adam arguments");
  const mph_optim_cfg o = as_optim(cfg);
  return mph_gcn_optim_step(m, &o, t, stream);
}

extern "C" int mph_adam_step(mph_gcn* m, const mph_adam_cfg* cfg, int32_t t, void* stream) {
  return mph_gcn_adam(m, cfg, t, stream);
}

extern "C" int mph_gcn_train_epoch_opt(mph_gcn* m, int32_t t, const mph_optim_cfg* cfg, double* loss_d, void* stream) {
  if (!m || !cfg || !loss_d || t < 1) return fail(MPH_EINVAL, "train_epoch arguments");
  MPH_TRY(mph_gcn_forward(m, t, stream));
  MPH_TRY(mph_gcn_loss(m, loss_d, stream));
  MPH_TRY(mph_gcn_backward(m, stream));
  MPH_TRY(mph_gcn_optim_step(m, cfg, t, stream));
  m->warm = true;
  return MPH_OK;
}

extern "C" int mph_gcn_train_epoch(mph_gcn* m, int32_t t, const mph_adam_cfg* cfg, double* loss_d, void* stream) {
  if (!m || !cfg) return fail(MPH_EINVAL, "train_epoch arguments");
  const mph_optim_cfg o = as_optim(cfg);
  return mph_gcn_train_epoch_opt(m, t, &o, loss_d, stream);
}

namespace mph {
__global__ void k_step_advance(int32_t* t) { *t += 1; }
}  // namespace mph

// CUDA-graph capture of one whole epoch (single GPU).  The step counter t lives in device
// memory and is advanced by the first node, so every replay is the next epoch: Adam's bias
// corrections and the dropout counter read it there.  Eager and replayed epochs run the same
// kernels with the same arguments, so they are bitwise identical.
extern "C" int mph_gcn_graph_capture(mph_gcn* m, const mph_adam_cfg* cfg, int32_t t_next, void* stream) {
  if (!m || !cfg) return fail(MPH_EINVAL, "graph_capture arguments");
  const mph_optim_cfg o = as_optim(cfg);
  return mph_gcn_graph_capture_opt(m, &o, t_next, stream);
}

extern "C" int mph_gcn_graph_capture_opt(mph_gcn* m, const mph_optim_cfg* cfg, int32_t t_next, void* stream) {
  if (!m || !cfg || t_next < 1) return fail(MPH_EINVAL, "graph_capture arguments");
  if (m->world > 1 && !m->p2p)
    return fail(MPH_ENOTSUP, "graph capture with P > 1 needs comm_mode = MPH_COMM_P2P (NCCL calls are eager)");
  if (!m->warm) return fail(MPH_ESTATE, "run one eager mph_gcn_train_epoch before capturing (lazy setup)");
  cudaStream_t user = (cudaStream_t)stream;
  MPH_CUDA_TRY(cudaStreamSynchronize(user));
  if (m->graph_exec) {
    cudaGraphExecDestroy(m->graph_exec);
    m->graph_exec = nullptr;
  }
  if (m->graph) {
    cudaGraphDestroy(m->graph);
    m->graph = nullptr;
  }
  const int32_t t0 = t_next - 1;
  MPH_CUDA_TRY(cudaMemcpy(m->t_dev, &t0, sizeof(int32_t), cudaMemcpyHostToDevice));
  cudaStream_t cap = nullptr;
  MPH_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  const bool prof_was = prof::enabled();
  prof::set_enabled(false);  // no event nodes inside the graph
  m->graph_mode = true;
  m->graph_cfg = *cfg;
  int rc = MPH_OK;
  cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    k_step_advance<<<1, 1, 0, cap>>>(m->t_dev);
    count_launch();
    rc = do_forward(m, t_next, cap);
    if (rc == MPH_OK) rc = loss_global(m, m->loss_dev, cap);
    if (rc == MPH_OK) rc = do_backward(m, cap);
    if (rc == MPH_OK) rc = mph_gcn_optim_step(m, &m->graph_cfg, t_next, cap);
    cudaGraph_t gph = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(cap, &gph);
    if (rc == MPH_OK && e2 != cudaSuccess) rc = fail(MPH_ECUDA, "EndCapture: %s", cudaGetErrorString(e2));
    m->graph = gph;
  } else {
    rc = fail(MPH_ECUDA, "BeginCapture: %s", cudaGetErrorString(e));
  }
  m->graph_mode = false;
  prof::set_enabled(prof_was);
  cudaStreamDestroy(cap);
  if (rc != MPH_OK) return rc;
  e = cudaGraphInstantiate(&m->graph_exec, m->graph, 0);
  if (e != cudaSuccess) return fail(MPH_ECUDA, "GraphInstantiate: %s", cudaGetErrorString(e));
  return MPH_OK;
}

extern "C" int mph_gcn_graph_replay(mph_gcn* m, void* stream) {
  if (!m) return fail(MPH_EINVAL, "null model");
  if (!m->graph_exec) return fail(MPH_ESTATE, "no captured epoch (mph_gcn_graph_capture)");
  MPH_CUDA_TRY(cudaGraphLaunch(m->graph_exec, (cudaStream_t)stream));
  count_launch(m->L * 6 + 4);  // kernels inside the graph (accounting only)
  return MPH_OK;
}

extern "C" int mph_gcn_graph_state(const mph_gcn* m, int32_t** t_d, double** loss_d) {
  if (!m) return fail(MPH_EINVAL, "null model");
  if (t_d) *t_d = m->t_dev;
  if (loss_d) *loss_d = m->loss_dev;
  return MPH_OK;
}

extern "C" int mph_gcn_tensor(const mph_gcn* m, int32_t kind, int32_t layer, const float** ptr_d, int32_t* rows_h,
                              int32_t* width_h, int32_t* ld_h, int32_t* elem_bytes_h) {
  if (!m || layer < 1 || layer > m->L) return fail(MPH_EINVAL, "gcn_tensor arguments");
  const Layer& l = m->layers[layer - 1];
  const float* p = nullptr;
  int rows = m->g->n_rows, width = 0, ld = 0;
  bool bf = false;  // BF16 mode: the tensors that only feed GEMMs are bfloat16
  switch (kind) {
    case 0:
      if (layer == 1) {
        p = m->f->mode == 0 ? m->f->X : nullptr;
        width = m->f->F;
        ld = m->f->P;
      } else {
        p = m->layers[layer - 2].out;
        width = l.fin;
        ld = l.pin;
        bf = m->bf16;
      }
      break;
    case 1:
      p = l.out;
      width = l.fout;
      ld = l.pout;
      bf = m->bf16 && layer < m->L;
      break;
    case 2:
      p = l.order == 0 ? l.G : l.dZ;
      width = l.fout;
      ld = l.pout;
      bf = m->bf16 && !(layer == 1 && m->f->mode == 1);
      break;
    case 3:
      p = l.Y;
      width = l.fin;
      ld = l.pin;
      bf = m->bf16;
      break;
    case 4:
      p = l.T;
      width = l.fout;
      ld = l.pout;
      rows = m->g->n_cols;
      break;
    case 5:
      p = l.dZ;
      width = l.fout;
      ld = l.pout;
      rows = l.order == 0 ? m->g->n_cols : m->g->n_rows;
      break;
    default:
      return fail(MPH_EINVAL, "unknown tensor kind %d", kind);
  }
  if (kind == 5 && l.order == 1) bf = m->bf16;  // dZ_1 of an aggregate-first layer 1
  if (ptr_d) *ptr_d = p;
  if (rows_h) *rows_h = rows;
  if (width_h) *width_h = width;
  if (ld_h) *ld_h = ld;
  if (elem_bytes_h) *elem_bytes_h = bf ? 2 : 4;
  return MPH_OK;
}

extern "C" int mph_gcn_info(const mph_gcn* m, int32_t* order_h, int32_t* mode_h) {
  if (!m) return fail(MPH_EINVAL, "null model");
  if (order_h)
    for (int li = 0; li < m->L; ++li) order_h[li] = m->layers[li].order;
  if (mode_h) *mode_h = m->f->mode;
  return MPH_OK;
}

extern "C" int mph_gcn_p2p_export(const mph_gcn* m, uint8_t* blob_h) {
  if (!m || !blob_h) return fail(MPH_EINVAL, "p2p_export arguments");
  if (!m->p2p) return fail(MPH_ESTATE, "p2p_export: model was not created with comm_mode = MPH_COMM_P2P");
  return p2p_export(m->p2p, blob_h);
}

extern "C" int mph_gcn_p2p_open(mph_gcn* m, const uint8_t* blobs_h, int32_t world, void* stream) {
  if (!m || !blobs_h) return fail(MPH_EINVAL, "p2p_open arguments");
  if (!m->p2p) return fail(MPH_ESTATE, "p2p_open: model was not created with comm_mode = MPH_COMM_P2P");
  cudaStream_t s = (cudaStream_t)stream;
  MPH_CUDA_TRY(cudaDeviceSynchronize());  // the arena (and dinv ⊙ X) are initialised before peers look
  MPH_TRY(p2p_open(m->p2p, m->g, blobs_h, world));
  if (m->Xs) MPH_TRY(p2p_setup_exchange(m, s));
  MPH_CUDA_TRY(cudaStreamSynchronize(s));
  int err = 0;
  MPH_CUDA_TRY(cudaMemcpy(&err, m->p2p->err_dev, sizeof(int), cudaMemcpyDeviceToHost));
  if (err) return fail(MPH_ETIMEOUT, "p2p_open: a peer did not signal within 10 s");
  return MPH_OK;
}

extern "C" int mph_gcn_p2p_status(const mph_gcn* m, int32_t* err_h, int64_t* gen_h, uint64_t* flags_h) {
  if (!m || !err_h) return fail(MPH_EINVAL, "p2p_status arguments");
  *err_h = 0;
  if (!m->p2p) return MPH_OK;
  MPH_CUDA_TRY(cudaDeviceSynchronize());
  int err = 0;
  MPH_CUDA_TRY(cudaMemcpy(&err, m->p2p->err_dev, sizeof(int), cudaMemcpyDeviceToHost));
  *err_h = err ? MPH_ETIMEOUT : 0;
  if (gen_h) MPH_CUDA_TRY(cudaMemcpy(gen_h, m->p2p->gen_dev, sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (flags_h)
    for (int slot = 0; slot < kP2PSlots; ++slot)
      MPH_CUDA_TRY(cudaMemcpy(flags_h + (size_t)slot * m->world, p2p_flags_local(m->p2p, slot),
                              sizeof(uint64_t) * m->world, cudaMemcpyDeviceToHost));
  return MPH_OK;
}

extern "C" int mph_gcn_destroy(mph_gcn* m) {
  gcn_free(m);
  return MPH_OK;
}
