/*
 * morphling.h — C-ABI of the B200-native GCN training hot path of
 * "Morphling: Fast, Fused, and Flexible GNN Training at Scale" (arXiv 2512.01678).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (LaTeX source), S:n = SPEC.md line n,
 * SURVEY §x = /root/repo/SURVEY.md.  The calls follow the paper's statement of the problem,
 * Listing 1 and its semantics:
 *     load  ->  initializeLayers("xaviers")  ->  per epoch: forwardPass(l) for l = 1..L,
 *     backPropagation(l) for l = L..1, optimizer("adam", 0.01, 0.9, 0.999).
 *
 * Conventions (apply to every call below)
 *  - Every call returns an int status: MPH_OK (0) or a negative MPH_E* code; on error
 *    mph_last_error() returns a thread-local message valid until the next mph_* call on
 *    that thread.  No C++ exception crosses this boundary.
 *  - Pointers suffixed _h are HOST memory, borrowed for the duration of the call.
 *    Pointers suffixed _d (and every float/int tensor argument of a kernel-level entry
 *    point) are DEVICE memory owned by the caller; they must stay valid until the work
 *    enqueued on `stream` has finished.  `stream` is a cudaStream_t passed as void*
 *    (NULL = legacy default stream).
 *  - Opaque handles (mph_graph, mph_features, mph_plan, mph_comm, mph_gcn) are owned by the
 *    library; their device memory is allocated with cudaMalloc and released by the matching
 *    *_destroy, which accepts NULL.  Accessors that return device pointers return BORROWED
 *    views valid until the handle is destroyed.
 *  - Device calls only enqueue work on `stream`, except where "synchronises" is stated.
 *    An asynchronous kernel fault surfaces as MPH_ECUDA from the next synchronising call.
 *  - Floating-point results are deterministic: the same inputs and world size give
 *    bitwise-identical outputs (no floating-point atomics on any path).
 *  - Feature matrices are row-major float32 with a row stride `ld` (in elements).  Widths
 *    are padded to a multiple of 8 floats (4 when w <= 4); padded columns must be zero and
 *    stay zero.  Kernels reading a matrix through TMA need ld % 4 == 0 and a
 *    16-byte aligned base.
 *  - There is no CPU fallback: every compute call runs CUDA kernels compiled for sm_100a
 *    and fails with MPH_ECUDA when no such device is present.
 */
#ifndef MORPHLING_H_
#define MORPHLING_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPH_VERSION 1

/* ---- status codes (SURVEY §8(b) error table; SPEC error classes S:63) */
#define MPH_OK 0
#define MPH_EINVAL (-1)      /* null pointer, dimension mismatch, unsupported flag */
#define MPH_ERANGE (-2)      /* node id outside [0, N) */
#define MPH_EDEGENERATE (-3) /* N = 0 or N*F = 0 */
#define MPH_ESTATE (-4)      /* call order violated, e.g. backward before forward */
#define MPH_ENOMEM (-5)      /* device allocation failed */
#define MPH_ECUDA (-6)       /* CUDA error (includes "no sm_100a device") */
#define MPH_ENCCL (-7)       /* NCCL error */
#define MPH_EDIVERGED (-8)   /* replica parameter hashes differ across ranks */
#define MPH_ENOTSUP (-9)     /* shape outside what the kernels implement (e.g. width > 512) */
#define MPH_ETIMEOUT (-10)   /* a peer-memory wait saw no signal within 10 s (mph_gcn_p2p_status) */

int mph_version(void);
const char* mph_last_error(void);
/* library-internal device memory (CSR, plans, activations, workspaces) from a
 * caller allocator, e.g. torch's caching allocator; alloc(bytes, stream, ctx) returns a device
 * pointer or NULL, release(ptr, bytes, stream, ctx) takes it back (stream = the default stream).
 * NULL callbacks restore cudaMalloc / cudaFree.  Memory is released through whichever allocator
 * provided it.  The peer-mapped arena of a MPH_COMM_P2P model always comes from cudaMalloc
 * (CUDA IPC needs it).  Not thread-safe against concurrent mph_* calls. */
int mph_set_allocator(void* (*alloc)(size_t bytes, void* stream, void* ctx),
                      void (*release)(void* ptr, size_t bytes, void* stream, void* ctx), void* ctx);
/* Number of CUDA kernels this library has launched since it was loaded (bench accounting). */
int mph_launch_count(int64_t* count_h);
/* Resets the calling thread's error message; returns MPH_ECUDA unless an sm_100 device is present. */
int mph_device_check(int32_t* sm_count_h);

/* =====================================================================================
 * a0 — graph build (gnn.load, Listing 1; CSR "once during initialization" P:222).
 * Semantics fixed by SURVEY §8(c) G1-G6 (readings Q1-Q4):
 *   reject ids outside [0,N) (MPH_ERANGE); N = 0 -> MPH_EDEGENERATE;
 *   S  = {(u,v): u != v, (u,v) or (v,u) in the input}   (symmetrise, deduplicate, drop self loops)
 *   S' = S U {(u,u)}                                    (A + I)
 *   row_ptr int64[N+1], col_idx int32[nnz] ascending per row, deg int32[N] = row length (= d~),
 *   dinv float32[N] = (float)(1.0 / sqrt((double)deg))   (bit recipe G6).
 * Integer outputs are bit-exact with the oracle.  Synchronises.
 * ===================================================================================== */
typedef struct mph_graph mph_graph;
int mph_graph_build(const int32_t* src_h, const int32_t* dst_h, int64_t num_edges, int32_t num_nodes,
                    void* stream, mph_graph** out);
/* n_rows = owned rows; n_cols = n_rows + ghost rows (n_cols == n_rows for a global graph). */
int mph_graph_info(const mph_graph* g, int32_t* n_rows_h, int32_t* n_cols_h, int64_t* nnz_h, int32_t* max_deg_h);
/* Borrowed device views: row_ptr[n_rows+1], col_idx[nnz], deg[n_cols], dinv[n_cols]. */
int mph_graph_csr(const mph_graph* g, const int64_t** row_ptr_d, const int32_t** col_idx_d,
                  const int32_t** deg_d, const float** dinv_d);
int mph_graph_destroy(mph_graph* g);

/* =====================================================================================
 * a1 — feature analysis and the dense/sparse switch (Alg. 1 Initialize, P:256-266;
 * Eq. 1; tau ~ 0.80 P:216).  Readings Q11, Q12, Q28:
 *   nnz = #{X[i,k] != 0.0f};  mode = Sparse iff 10000*nnz <= (10000 - tau_bp)*N*F (int64);
 *   is_binary = every nonzero equals 1.0f.  force_mode: -1 auto, 0 Dense, 1 Sparse.
 * Sparse mode materialises X_csr (forward) and X_csc (backward, rows ascending per column).
 * Dense mode keeps a padded row-major copy of X (row stride pad_width(F)).
 * X_d [N][ld] is only read during the call.  Synchronises (the mode is a host decision).
 * ===================================================================================== */
typedef struct mph_features mph_features;
int mph_features_create(const float* X_d, int32_t N, int32_t F, int32_t ld, int32_t tau_bp,
                        int32_t force_mode, void* stream, mph_features** out);
/* tau_bp values: the paper's tau = 0.80 (gamma = 0.20 on its testbed), and the crossover
 * measured on B200 by the paper's own offline protocol (tools/calibrate_gamma.py, DESIGN §9.2:
 * s* = 0.910 / 0.952 / 0.972 on three shapes, median 0.95) — "tau is fully determined by the
 * hardware".  The Python binding defaults to the B200 value; the C calls take tau_bp
 * explicitly. */
#define MPH_TAU_PAPER_BP 8000
#define MPH_TAU_B200_BP 9500
/* Same switch from a HOST CSR matrix, for feature matrices too large to hold densely (NELL:
 * 65,755 x 61,278 at s = 99.21%).  ptr_h[N+1] (int64, ptr_h[0] = 0,
 * monotone), idx_h[ptr_h[N]] (int32 columns in [0,F), strictly ascending within each row: S3),
 * val_h[ptr_h[N]] (fp32).  Explicit zeros are dropped (S1 counts x != 0 only), so nnz and the
 * stored pattern equal what mph_features_create would give on the densified matrix.  Sparse mode
 * uploads X_csr and builds X_csc + segments on the device; dense mode scatters into the padded
 * copy.  Host arrays are only read during the call (pageable or pinned).  MPH_EINVAL on a
 * malformed CSR (nothing allocated).  Synchronises. */
int mph_features_create_csr(const int64_t* ptr_h, const int32_t* idx_h, const float* val_h, int32_t N,
                            int32_t F, int32_t tau_bp, int32_t force_mode, void* stream, mph_features** out);
int mph_features_info(const mph_features* f, int64_t* nnz_h, int32_t* mode_h, int32_t* is_binary_h);
/* The switch for a row-partitioned X (P > 1): every rank must take the SAME decision
 * (the mode and the layer orders it implies fix which buffers cross ranks), so the caller counts
 * its local rows' nonzeros with mph_features_count (device X_d [N][ld], synchronises), sums the
 * counts over the ranks (the process group is plumbing), and mph_features_decide applies Eq. 1 to
 * the GLOBAL count: *mode_h = 1 (Sparse) iff 10000*nnz <= (10000 - tau_bp)*N*F, N the global row
 * count.  Pass the result as force_mode on every rank.  mph_gcn_create checks that the ranks
 * agree (MPH_EINVAL otherwise).  MPH_EINVAL on nnz > N*F or a tau_bp outside [0, 10000]. */
int mph_features_count(const float* X_d, int32_t N, int32_t F, int32_t ld, void* stream, int64_t* nnz_h);
int mph_features_decide(int64_t nnz, int64_t N, int64_t F, int32_t tau_bp, int32_t* mode_h);
/* Borrowed device views (sparse mode only; MPH_ESTATE in dense mode). */
int mph_features_csr(const mph_features* f, const int64_t** ptr_d, const int32_t** idx_d, const float** val_d);
int mph_features_csc(const mph_features* f, const int64_t** ptr_d, const int32_t** idx_d, const float** val_d);
/* Dense copy [N][ld] (dense mode only). */
int mph_features_dense(const mph_features* f, const float** X_d, int32_t* ld_h);
int mph_features_destroy(mph_features* f);

/* =====================================================================================
 * Kernel-level entry points (raw pointers + shapes + stream), used by the model below and
 * by the per-kernel parity tests.
 * ===================================================================================== */

/* Fused epilogue flags. */
#define MPH_EPI_BIAS 1u      /* + bias[c]                                                    */
#define MPH_EPI_RELU 2u      /* max(x, 0); ReLU'(0) := 0 (Q8)                                */
#define MPH_EPI_ROWSCALE 4u  /* * row_scale[r], applied last (dinv pre-scale of the next SpMM) */
#define MPH_EPI_MASK 8u      /* * (mask_src[r,c] > 0 ? mask_scale : 0)  (ReLU'/dropout mask)  */
#define MPH_EPI_DROPOUT 16u  /* inverted dropout after ReLU, Philox4x32-10 (Q10)              */
#define MPH_EPI_COLSUM 32u   /* per-CTA column sums of the value before ROWSCALE -> colsum_out */
#define MPH_EPI_TF32 64u     /* round the stored value to TF32 (cvt.rna), for outputs that only feed
                                tensor-core GEMMs: unbiased operand rounding (reading R2) */
#define MPH_EPI_BF16 128u    /* store the output as bfloat16 (round to nearest even; the output pointer
                                holds bf16, ld in elements): outputs that only feed BF16 GEMMs.
                                mph_gemm_nt and mph_spmm (whole rows, part -1) */
#define MPH_EPI_MASK_BF16 256u /* mask_src holds bfloat16 values (ld_mask in elements); mph_gemm_nt */
#define MPH_EPI_SIGNBITS 1024u /* also write the signs of the stored output as "sign bytes": bit t of byte
                                  bits_out[r * ld_bits + c / 4] = (stored value at column c > 0), t = c % 4
                                  (ld_bits in bytes).  A ReLU (+ dropout) layer's mask in 1/16 of its
                                  FP32 bytes.  mph_gemm_nt (ld_bits % 8 == 0); mph_spmm (part -1 or 1) */
#define MPH_EPI_MASK_BITS 2048u /* MASK with mask_src holding such sign bytes (ld_mask in bytes, % 8 == 0,
                                   8-byte aligned): the same decisions as the value mask; mph_gemm_nt */

typedef struct {
  uint32_t flags;
  const float* row_scale;  /* [rows]            (ROWSCALE) */
  const float* bias;       /* [cols]            (BIAS)     */
  const float* mask_src;   /* [rows][ld_mask]   (MASK)     */
  int32_t ld_mask;
  float mask_scale;
  float* colsum_out;       /* [ceil(rows/128)][cols] partial sums (COLSUM); reduce with mph_reduce_rows */
  float dropout_p;         /* (DROPOUT) */
  uint64_t dropout_seed;
  int32_t dropout_layer, dropout_epoch;
  int64_t row0;            /* global id of row 0 (Philox counter; distributed ranks) */
  const int32_t* dropout_epoch_d; /* nullable: device epoch counter overriding dropout_epoch (graph replay) */
  uint32_t* bits_out;      /* [rows][ld_bits] sign bytes (SIGNBITS) */
  int32_t ld_bits;
} mph_epilogue;

/* a3/a6 — aggregation SpMM (Alg. 3, fused per P:361/P:735):
 *   out[u, c] = epi( dinv[u] * sum_{e in row u} in[col_idx[e], c] )   for u < n_rows, c < w
 * `in` holds rows already pre-scaled by dinv (in[v] = dinv[v]*T[v]), so out = epi(Â·T).
 * Supported epilogue flags: BIAS, RELU, DROPOUT (applied in that order).  w <= 512.
 * Deterministic, atomic-free; no O(|E|·F) buffer.  `in` has n_cols rows. */
int mph_spmm(const mph_graph* g, const float* in_d, int32_t w, int32_t ld_in, float* out_d, int32_t ld_out,
             const mph_epilogue* epi, void* stream);
/* *ok_h = 1 if mph_spmm of width w on g can write MPH_EPI_SIGNBITS (any width that is a multiple of
 * 4, <= 512), else 0.  Host only, no device work.  MPH_EINVAL on null arguments. */
int mph_spmm_signbits_ok(const mph_graph* g, int32_t w, int32_t* ok_h);
/* Same, restricted to one part of each row of a localized graph: part 0 = owned columns,
 * part 1 = ghost columns accumulated onto out (which must hold part 0's raw sums);
 * the epilogue runs with part 1 only.  part -1 = whole row (== mph_spmm). */
int mph_spmm_part(const mph_graph* g, int32_t part, const float* in_d, int32_t w, int32_t ld_in, float* out_d,
                  int32_t ld_out, const mph_epilogue* epi, void* stream);

/* Other aggregation schemes: "GCN uses normalized mean aggregation ...
 * GIN employs sum aggregation", "multiple aggregation schemes (mean, max, sum)",
 * Listing 1's SAGE "Max".  Reading R6: every scheme aggregates over Ñ(u) = N(u) ∪ {u}
 * (the graph's CSR, diagonal included).  A linear scheme is AGG = diag(post)·Ã·diag(pre):
 *   GCN  pre = post = D̃^{-1/2} (both directions)      SUM  none
 *   MEAN forward post = D̃^{-1}; adjoint (transpose = 1, Ã·D̃^{-1}) pre = D̃^{-1}
 * mph_graph_agg_scales returns the device arrays (n_cols floats; NULL = 1, borrowed).
 * mph_aggregate: out[u,:] = post[u] · Σ_{v∈Ñ(u)} in[v,:] then the epilogue (BIAS, RELU,
 * DROPOUT, ROWSCALE, TF32 as mph_spmm) — `in` must already carry the pre-scale (the producer
 * applies it, as for the GCN's dinv).  Constraints and errors as mph_spmm. */
#define MPH_AGG_GCN 0
#define MPH_AGG_SUM 1
#define MPH_AGG_MEAN 2
#define MPH_AGG_MAX 3
int mph_graph_agg_scales(const mph_graph* g, int32_t scheme, int32_t transpose, const float** pre_d,
                         const float** post_d);
int mph_aggregate(const mph_graph* g, int32_t scheme, int32_t transpose, const float* in_d, int32_t w, int32_t ld_in,
                  float* out_d, int32_t ld_out, const mph_epilogue* epi, void* stream);
/* Max aggregation (reading R7: applied before the transform; ties to the smallest
 * neighbour id):  out[u,c] = max_{v∈Ñ(u)} in[v,c],  arg[u,c] = smallest v attaining it
 * (arg_d nullable: not recorded).  Epilogue: TF32 only.  Values are compared exactly (no
 * rounding before the comparison), so out and arg are bit-exact given the same input.
 * w, ld_in, ld_out, ld_arg multiples of 4, 16-byte aligned, w <= 512.  Single GPU: MPH_ENOTSUP
 * on a localized graph with world > 1 (arg holds local ids). */
int mph_aggregate_max(const mph_graph* g, const float* in_d, int32_t w, int32_t ld_in, float* out_d, int32_t ld_out,
                      int32_t* arg_d, int32_t ld_arg, const mph_epilogue* epi, void* stream);
/* Its adjoint, the routing of every dY[u,c] to arg[u,c], computed as a gather over Ñ(v)
 * (Ã symmetric; deterministic, no atomics):  dH[v,c] = Σ_{u∈Ñ(v)} [arg[u,c] = v]·dY[u,c],
 * then the epilogue MASK (· (mask_src[v,c] > 0 ? mask_scale : 0): ReLU' and dropout of
 * H_{l-1}) and TF32.  Other flags: MPH_EINVAL. */
int mph_aggregate_max_backward(const mph_graph* g, const float* dY_d, int32_t w, int32_t ld_dy, const int32_t* arg_d,
                               int32_t ld_arg, float* dH_d, int32_t ld_out, const mph_epilogue* epi, void* stream);

/* a2/a4/a8 — dense transform on tcgen05 tensor cores (TF32 in, FP32 accumulate in TMEM):
 *   C[M, N] = epi( A[M, K] · Bt[N, K]^T )    A row-major (lda), Bt row-major (ldb)
 * TMA-fed, 128-row tiles, N <= 256 per tile.  Columns of C in [N, round_up(N,16)) are not
 * written.  Out-of-range K / N operand elements are read as zero. */
int mph_gemm_nt(int32_t M, int32_t N, int32_t K, const float* A_d, int32_t lda, const float* Bt_d, int32_t ldb,
                float* C_d, int32_t ldc, const mph_epilogue* epi, void* stream);
/* a7 — weight gradient (contraction over the node dimension, P:525-532 step (a)):
 *   C[M, N] = A[K, M]^T · B[K, N]    (A, B row-major; K = nodes)
 * Deterministic split-K: per-CTA FP32 partials in `ws_d` (16-byte aligned), reduced in a fixed order. */
int mph_gemm_tn_workspace(int32_t M, int32_t N, int32_t K, size_t* bytes_h);
/* SURVEY §8(b) generic form: C = op(A)·op(B) for the two shapes of the GCN path —
 * (transA, transB) = (0, 1): mph_gemm_nt with the epilogue flags RELU / TF32 (those needing no
 * operand pointer); (1, 0): mph_gemm_tn (workspace allocated and freed stream-ordered, flags
 * must be 0).  precision: 0 = TF32 (A_d, B_d float32), 1 = BF16 (A_d, B_d point to bfloat16
 * values; lda, ldb in elements, multiples of 8; tcgen05 kind::f16, FP32 accumulate).
 * Other transpose combinations or precisions: MPH_ENOTSUP. */
int mph_gemm(int32_t M, int32_t N, int32_t K, const float* A_d, int32_t lda, int32_t transA, const float* B_d,
             int32_t ldb, int32_t transB, float* C_d, int32_t ldc, int32_t precision, uint32_t epilogue_flags,
             void* stream);
int mph_gemm_tn(int32_t M, int32_t N, int32_t K, const float* A_d, int32_t lda, const float* B_d, int32_t ldb,
                float* C_d, int32_t ldc, void* ws_d, size_t ws_bytes, void* stream);

/* Fixed-order reduction over the leading axis: out[c] = sum_{r < rows} in[r*ld + c] (+= if accumulate). */
int mph_reduce_rows(const float* in_d, int32_t rows, int32_t cols, int32_t ld, float* out_d, int32_t accumulate,
                    void* stream);

/* a2 sparse path (Alg. 1 Forward, SpMM_Tiled(X_csr, W)):
 *   T[i, :] = row_scale[i] * sum_{k in row i of X} X[i,k] * W[k, :]     (row_scale nullable) */
int mph_sparse_xw(const mph_features* f, const float* W_d, int32_t F_out, int32_t ldw, const float* row_scale_d,
                  float* T_d, int32_t ldt, void* stream);
/* a7 sparse path (Alg. 1 Backward, SpMM_Col(X_csc, G), reading Q14):
 *   dW[k, :] = sum_{i in column k of X} X[i,k] * G[i, :]   (CSC gather, atomic-free) */
int mph_sparse_xtg(const mph_features* f, const float* G_d, int32_t F_out, int32_t ldg, float* dW_d, int32_t lddw,
                   void* stream);

/* a5 — fused softmax cross-entropy (reading Q9) over rows [0, N):
 *   lse_i = m_i + log sum_c exp(Z[i,c] - m_i),  c < C (padding ignored)
 *   loss_d[0] = (1/n_lab) * sum_{labelled i} (lse_i - Z[i, y_i])     (double)
 *   dZ[i, c] = row_scale[i] * (softmax - onehot)/n_lab   for labelled i, c < C; 0 otherwise
 *   db_d[c]  = sum_i (softmax - onehot)/n_lab             (unscaled; nullable)
 * mask_d nullable (= all rows labelled).  Workspace from mph_softmax_ce_workspace. */
int mph_softmax_ce_workspace(int32_t N, int32_t C, size_t* bytes_h);
int mph_softmax_ce(const float* Z_d, int32_t N, int32_t C, int32_t ld, const int32_t* labels_d, const uint8_t* mask_d,
                   int64_t n_lab, const float* row_scale_d, float* dZ_d, int32_t ld_dz, float* db_d, double* loss_d,
                   void* ws_d, size_t ws_bytes, void* stream);

/* a9 — Adam (Listing 1, "fused momentum and variance updates" P:535; reading Q15):
 *   m = b1*m + (1-b1)*g;  v = b2*v + (1-b2)*g^2;  p -= lr * (m/(1-b1^t)) / (sqrt(v/(1-b2^t)) + eps)
 * One launch over a flat buffer of n elements; t is 1-based. */
typedef struct {
  float lr, beta1, beta2, eps;
} mph_adam_cfg;
int mph_adam(float* params_d, const float* grads_d, float* m_d, float* v_d, int64_t n, const mph_adam_cfg* cfg,
             int32_t t, void* stream);
/* Optimizers of P:140 ("SGD, Adam, AdamW"; reading R8), one launch over a
 * flat buffer:
 *   ADAM   as mph_adam (weight_decay, momentum ignored)
 *   SGD    d = g + wd·p;  momentum μ > 0: m = μ·m + d, d = m  (m_d: velocity, starts at 0);
 *          p -= lr·d      (v_d unused, may be NULL)
 *   ADAMW  p -= lr·wd·p (decoupled, before the update), then the Adam update
 * t is 1-based (Adam / AdamW bias corrections). */
#define MPH_OPT_ADAM 0
#define MPH_OPT_SGD 1
#define MPH_OPT_ADAMW 2
typedef struct {
  int32_t kind;
  float lr, beta1, beta2, eps, weight_decay, momentum;
} mph_optim_cfg;
int mph_optim_step(float* params_d, const float* grads_d, float* m_d, float* v_d, int64_t n,
                   const mph_optim_cfg* cfg, int32_t t, void* stream);

/* Xavier-uniform fill ("xaviers", Listing 1; bound S:322; stream of reading Q16):
 *   W[i*ld + j] = (float)(a * (2*(x_{i*f_out+j} >> 40)/2^24 - 1)), a = sqrt(6/(f_in+f_out)),
 *   x_k = k-th output of splitmix64 seeded seed ^ (layer * 0x9E3779B97F4A7C15). */
int mph_xavier_fill(float* W_d, int32_t f_in, int32_t f_out, int32_t ld, uint64_t seed, int32_t layer, void* stream);

/* Optional kernel timing of the model runtime (bench.py): CUDA events on the launching stream
 * around every hot-path launch, with each launch's algorithmic bytes and flops (SURVEY §8(d)
 * d.3).  mph_profile_enable clears the records; mph_profile_read sums one kernel class
 * (call after synchronising the stream). */
#define MPH_PROF_SPMM 0
#define MPH_PROF_GEMM_NT 1
#define MPH_PROF_GEMM_TN 2
#define MPH_PROF_LOSS 3
#define MPH_PROF_ADAM 4
#define MPH_PROF_SPARSE 5
#define MPH_PROF_HALO 6
#define MPH_PROF_OTHER 7
int mph_profile_enable(int32_t on);
int mph_profile_read(int32_t kind, int64_t* count_h, double* total_ms_h, double* total_bytes_h, double* total_flops_h);
/* Gather-bandwidth probe: sums rows idx_d[0..n_idx) (w floats, w % 4 == 0,
 * w <= 128) of table_d [n_rows][w]; out_d needs 148*32*128 floats.  Used by bench.py to measure
 * the L2-resident and HBM-resident random-row gather peaks the SpMM is compared with. */
int mph_probe_gather(const float* table_d, int64_t n_rows, int32_t w, const int32_t* idx_d, int64_t n_idx,
                     float* out_d, void* stream);
/* L2 delivery ceiling: a coalesced streaming read (ld.global.cg, no L1) of an L2-resident buffer
 * buf_d [n_floats] repeated `passes` times by 2 x SMs blocks of 512 threads (n_floats a multiple
 * of 8 x SMs; out_d needs 2 x SMs x 2048 floats).  rate = passes * n_floats * 4 / time.  bench.py
 * reports the aggregation's gathered bytes per second against max(this, the gather probe). */
int mph_probe_l2_stream(const float* buf_d, int64_t n_floats, int32_t passes, float* out_d, void* stream);

/* =====================================================================================
 * a10/a11 — distributed runtime (MPI backend analogue).
 * ===================================================================================== */
/* D1: bounds[r] = min{u in [0,N] : world*row_ptr[u] >= r*nnz}; balances sum of deg(v)+1
 * (Alg. 4 Phase III weight; reading Q20).  Host only. */
int mph_partition_1d(const int64_t* row_ptr_h, int32_t N, int32_t world, int64_t* bounds_h);

/* Alg. 4 partitioners.  Host only; row_ptr_h / col_idx_h are the
 * GLOBAL Ã CSR (diagonal included, so a row's length is d̃_v = deg(v) + 1).  Reading R9: ties go
 * to the smaller node id / lower rank (bit-exact with the oracle).  Phase I (METIS) is out of
 * scope.
 *   mph_partition_greedy      Phase III: nodes by deg descending, each to the rank of least
 *                             weight, weight += deg(v) + 1.  load_h[world] nullable.
 *   mph_partition_components  Phase II: connected components by BFS, sorted by size descending,
 *                             each to the lightest rank, weight += |C|.  *n_comp_h =
 *                             component count; part_h is written only when it is > 1.
 *   mph_partition_hierarchical  Phase II when disconnected, else Phase III; *phase_h = 2 or 3.
 *   mph_relabel               new_id_h[v]: rank 0's nodes first, then rank 1's, ..., ascending old
 *                             id within a rank; bounds_h[world+1] so the relabelled graph's
 *                             contiguous ranges are exactly the partition (feed bounds_h to
 *                             mph_plan_create).  MPH_EINVAL if part_h[v] is outside [0, world).
 *   mph_partition_stats       stats_h[4*world]: per rank {owned nodes, Σ d̃ (SpMM work,
 *                             P:550-555), distinct ghost nodes (halo rows), cut
 *                             entries of A}. */
int mph_partition_greedy(const int64_t* row_ptr_h, int32_t N, int32_t world, int32_t* part_h, int64_t* load_h);
int mph_partition_components(const int64_t* row_ptr_h, const int32_t* col_idx_h, int32_t N, int32_t world,
                             int32_t* part_h, int32_t* n_comp_h);
int mph_partition_hierarchical(const int64_t* row_ptr_h, const int32_t* col_idx_h, int32_t N, int32_t world,
                               int32_t* part_h, int32_t* phase_h);
int mph_relabel(const int32_t* part_h, int32_t N, int32_t world, int64_t* new_id_h, int64_t* bounds_h);
int mph_partition_stats(const int64_t* row_ptr_h, const int32_t* col_idx_h, int32_t N, const int32_t* part_h,
                        int32_t world, int64_t* stats_h);

/* D2-D4: G2L local-then-ghost layout and halo lists.  Host only.
 * ghosts ascending by global id; local row = [owned cols | ghost cols], split[i] = #owned;
 * recv slice of peer q = ghost rows [recv_offset[q], recv_offset[q]+n_recv[q]);
 * send list to q = send_ids[send_offset[q] .. send_offset[q+1]) (ascending owned local ids);
 * deg_local[n_own + n_ghost] = global degrees of owned then ghost nodes. */
typedef struct mph_plan mph_plan;
int mph_plan_create(const int64_t* row_ptr_h, const int32_t* col_idx_h, int32_t N, const int64_t* bounds_h,
                    int32_t world, int32_t rank, mph_plan** out);
int mph_plan_info(const mph_plan* p, int32_t* n_own_h, int64_t* row0_h, int64_t* n_ghost_h, int64_t* nnz_h,
                  int64_t* n_send_h);
int mph_plan_arrays(const mph_plan* p, const int64_t** ghosts_h, const int64_t** row_ptr_h, const int32_t** col_idx_h,
                    const int64_t** split_h, const int32_t** deg_local_h, const int64_t** recv_offset_h,
                    const int64_t** n_recv_h, const int64_t** send_offset_h, const int32_t** send_ids_h);
int mph_plan_destroy(mph_plan* p);
/* SURVEY §8(b) mph_graph_localize: G2L + halo plan of `rank` straight from a global graph
 * (copies its CSR to the host, mph_plan_create, mph_graph_from_plan).  bounds_h: world+1 row
 * bounds (mph_partition_1d / mph_relabel).  Synchronises. */
int mph_graph_localize(const mph_graph* global, const int64_t* bounds_h, int32_t world, int32_t rank, void* stream,
                       mph_graph** local_out);
/* SURVEY §8(b) mph_halo_plan, for tests / inspection of a localized graph: the owned local row
 * ids this rank sends to `peer` (device, borrowed), their count, and where `peer`'s rows land
 * in the ghost slice (recv offset from n_rows, count). */
int mph_halo_plan(const mph_graph* local, int32_t peer, const int32_t** send_local_ids_d, int64_t* n_send_h,
                  int64_t* recv_offset_h, int64_t* n_recv_h);
/* Upload a plan as a localized graph (dinv by the G6 recipe from deg_local).  Synchronises. */
int mph_graph_from_plan(const mph_plan* p, void* stream, mph_graph** out);

/* NCCL communicator over the ranks of one box (NVLink 5 / NVSwitch).  The 128-byte unique id
 * is created on rank 0 and broadcast by the caller (torch.distributed is the plumbing). */
typedef struct mph_comm mph_comm;
int mph_comm_unique_id(uint8_t* id_h /*128 bytes*/);
int mph_comm_create(const uint8_t* id_h, int32_t world, int32_t rank, mph_comm** out);
int mph_comm_info(const mph_comm* c, int32_t* world_h, int32_t* rank_h);
int mph_comm_destroy(mph_comm* c);
/* a10: pack owned boundary rows per peer and ncclSend/ncclRecv them straight into the ghost
 * rows [n_rows, n_cols) of buf (grouped p2p; no unpack).  buf has n_cols rows of stride ld. */
int mph_halo_exchange(const mph_graph* local, mph_comm* c, float* buf_d, int32_t w, int32_t ld, void* stream);
/* a11: in-place sum all-reduce (ncclAllReduce, float32 or float64 when is_double). */
int mph_allreduce_sum(mph_comm* c, void* buf_d, int64_t n, int32_t is_double, void* stream);

/* =====================================================================================
 * The L-layer GCN training step (Listing 1): initializeLayers / forwardPass /
 * backPropagation / optimizer.  Layer l maps F_{l-1} -> F_l with bias, ReLU on hidden
 * layers, identity on the output, softmax cross-entropy loss, Adam.
 * Per-layer order (reading Q7): transform-first (T = H·W, Z = Â·T + b) iff F_l <= F_{l-1} or
 * l = 1 in Sparse mode; otherwise aggregate-first on layer 1 (Y = Â·X, Z = Y·W + b).
 * ===================================================================================== */
typedef struct mph_gcn mph_gcn;
typedef struct {
  int32_t num_layers;    /* L >= 1 */
  const int32_t* dims_h; /* L+1 unpadded widths F_0..F_L (F_0 = features, F_L = classes) */
  float dropout_p;       /* 0 disables (default); inverted dropout after hidden ReLU (Q10) */
  uint64_t dropout_seed;
  int32_t order_policy;  /* 0 auto (Q7), 1 force transform-first everywhere */
  int32_t aggregator;    /* MPH_AGG_GCN (default, the north star), _SUM, _MEAN (linear: the layer
                            order of Q7 applies) or _MAX (Z = MAX(H)·W + b on every layer, R7;
                            dense-mode features and a single GPU only, else MPH_ENOTSUP) */
  int32_t comm_mode;     /* P > 1 only: MPH_COMM_NCCL (0, default: pack + grouped ncclSend/Recv,
                            ncclAllReduce) or MPH_COMM_P2P (1: NVLink peer memory, see below) */
  int32_t precision;     /* GEMM operands: MPH_PREC_TF32 (0, default: FP32 storage, operands rounded
                            to TF32) or MPH_PREC_BF16 (1: the tensors that only feed tensor-core
                            GEMMs — hidden H, backward G, Y_1, dZ_1, the copies of X and W — are
                            stored as bfloat16 and the GEMMs run kind::f16; aggregation, loss and
                            optimizer stay FP32).  BF16: gcn/sum/mean aggregators, not a
                            one-layer aggregate-first model (else MPH_ENOTSUP); mph_gcn_tensor views
                            of those tensors hold bf16. */
} mph_gcn_desc;

#define MPH_PREC_TF32 0
#define MPH_PREC_BF16 1

#define MPH_COMM_NCCL 0
#define MPH_COMM_P2P 1

/* graph may be global (comm NULL) or localized (world > 1: comm non-NULL for MPH_COMM_NCCL,
 * NULL for MPH_COMM_P2P); features hold the owned rows.  Allocates parameters, gradients, Adam
 * state and activations. */
int mph_gcn_create(const mph_graph* g, const mph_features* f, const mph_gcn_desc* desc, mph_comm* comm,
                   void* stream, mph_gcn** out);
/* Flat parameter buffer: W_l at offsets[2(l-1)] as [F_{l-1}][ld_w[l-1]] row-major,
 * b_l at offsets[2(l-1)+1] (ld_w[l-1] entries).  Padding entries are zero. */
int mph_gcn_param_layout(const mph_gcn* m, int64_t* num_params_h, int64_t* offsets_h, int32_t* ld_w_h);
int mph_gcn_buffers(const mph_gcn* m, float** params_d, float** grads_d, float** adam_m_d, float** adam_v_d);
/* SURVEY §8(b) caller-owned state: mph_gcn_bind replaces the model's parameter / gradient /
 * Adam-moment buffers (num_params floats each, layout of mph_gcn_param_layout) and its
 * workspace (>= mph_gcn_workspace_size bytes) by caller-owned device memory; a NULL argument keeps
 * the model's own buffer.  The caller's params_d becomes the model's parameters: call
 * mph_gcn_params_updated (or mph_gcn_init_xavier) before the next epoch; its padding entries (and
 * those of adam_m_d / adam_v_d) must be zero.  grads_d is zeroed here.  Synchronises.  Caller
 * buffers must outlive the model; they are never freed by it. */
int mph_gcn_workspace_size(const mph_gcn* m, size_t* bytes_h);
int mph_gcn_bind(mph_gcn* m, float* params_d, float* grads_d, float* adam_m_d, float* adam_v_d, void* workspace_d,
                 size_t ws_bytes);
/* initializeLayers("xaviers"): W by mph_xavier_fill(seed, layer = l), b = 0, m = v = 0. */
int mph_gcn_init_xavier(mph_gcn* m, uint64_t seed, void* stream);
/* Call after editing params_d directly (refreshes the transposed weight copies). */
int mph_gcn_params_updated(mph_gcn* m, void* stream);
/* Replace the dense input features of the owned rows from HOST memory (pinned for async
 * copies): X_h [n_rows][ld_h], F columns.  Re-derives everything the model derives from X
 * (the dinv pre-scale of an aggregate-first layer 1 and its ghost rows).  Dense mode only. */
int mph_gcn_upload_features(mph_gcn* m, const float* X_h, int32_t ld_h, void* stream);
/* Pipelined variant (a data loader's prefetch): the H2D copy runs on copy_stream once the
 * previous upload has been consumed, and the derivation (TF32 copy / pre-scale / MAX of X) is
 * enqueued on `stream` behind it.  The epoch reads only the derived buffers, so the copy of the
 * next step's X overlaps the current epoch.  X_h must stay valid (pinned) until the copy is done. */
int mph_gcn_upload_features_async(mph_gcn* m, const float* X_h, int32_t ld_h, void* copy_stream, void* stream);
/* Labels (int32, owned rows), optional uint8 mask, and the GLOBAL labelled count. */
int mph_gcn_set_labels(mph_gcn* m, const int32_t* labels_d, const uint8_t* mask_d, int64_t n_lab_global);
int mph_gcn_forward(mph_gcn* m, int32_t epoch, void* stream);
int mph_gcn_loss(mph_gcn* m, double* loss_d, void* stream);
int mph_gcn_backward(mph_gcn* m, void* stream);
int mph_gcn_adam(mph_gcn* m, const mph_adam_cfg* cfg, int32_t t, void* stream);
/* SURVEY §8(b) name of the same step (optimizer("adam", ...)). */
int mph_adam_step(mph_gcn* m, const mph_adam_cfg* cfg, int32_t t, void* stream);
/* One epoch a2..a11: forward, loss (written to loss_d, global sum over ranks), backward,
 * gradient all-reduce (P > 1), Adam step t.  Capturable in a CUDA graph when comm == NULL. */
int mph_gcn_train_epoch(mph_gcn* m, int32_t t, const mph_adam_cfg* cfg, double* loss_d, void* stream);
/* The same with any optimizer of mph_optim_step (the Adam moments double as SGD velocity). */
int mph_gcn_optim_step(mph_gcn* m, const mph_optim_cfg* cfg, int32_t t, void* stream);
int mph_gcn_train_epoch_opt(mph_gcn* m, int32_t t, const mph_optim_cfg* cfg, double* loss_d, void* stream);
/* CUDA-graph replay of whole epochs (single GPU; launch-bound configs).  mph_gcn_graph_capture
 * records one epoch (step-counter advance, forward, loss, backward, Adam with cfg) after at
 * least one eager mph_gcn_train_epoch (MPH_ESTATE otherwise); the next replay runs epoch
 * t_next, each further replay the following one.  The step counter and the loss live in
 * device memory (mph_gcn_graph_state).  Replayed epochs are bitwise identical to eager ones.
 * Synchronises `stream` before capturing.  MPH_ENOTSUP for P > 1. */
int mph_gcn_graph_capture(mph_gcn* m, const mph_adam_cfg* cfg, int32_t t_next, void* stream);
int mph_gcn_graph_capture_opt(mph_gcn* m, const mph_optim_cfg* cfg, int32_t t_next, void* stream);
int mph_gcn_graph_replay(mph_gcn* m, void* stream);
int mph_gcn_graph_state(const mph_gcn* m, int32_t** t_d, double** loss_d);
/* Borrowed views of activations for tests: kind 0 = layer input H_{l-1} (l=1 is X),
 * 1 = layer output Z_l (hidden: post-ReLU H_l; last: logits), 2 = G_l (backward SpMM out
 * or dZ_1 for an AF layer 1), 3 = aggregate-first Y_1, 4 = transform output T'_l = dinv ⊙ (H·W)
 * (n_cols rows incl. ghosts), 5 = dZ'_l (dinv-prescaled gradient, n_cols rows; AF layer 1: dZ_1). */
int mph_gcn_tensor(const mph_gcn* m, int32_t kind, int32_t layer, const float** ptr_d, int32_t* rows_h,
                   int32_t* width_h, int32_t* ld_h, int32_t* elem_bytes_h /* nullable: 4 float32, 2 bfloat16 */);
/* ---- NEXT-1: NVLink peer-memory halo exchange and gradient sum (
 * halo P:517-523, gradient sum P:525-532, overlap P:765).
 * A model created with comm_mode = MPH_COMM_P2P on a localized graph keeps every buffer a peer
 * reads — the dinv-prescaled T'_l and dZ'_l (owned + ghost rows), dinv ⊙ X of an
 * aggregate-first layer 1, two parity-indexed gradient receive slabs [world][num_params], the
 * loss slots and the step flags — in ONE cudaMalloc arena that the peers map (CUDA IPC over
 * NVLink / NVSwitch).  Per SpMM, the owner signals "rows ready" with a system-scope release
 * store into every peer's flag row and the consumer's pull kernel (acquire-spin, then 16-byte
 * peer loads) copies each ghost row from its owner's buffer into the local ghost slice while
 * the local-edge SpMM runs — no pack, no send buffer, no NCCL.  Each layer's [dW | db] is
 * pushed into every peer's receive slab as soon as it is complete; the optimizer kernel waits
 * for all ranks, sums the P slabs in rank order (deterministic, identical on every rank) and
 * applies the update in the same pass (all-reduce fused into Adam/SGD/AdamW).  The loss is
 * summed the same way.  CUDA-graph capture is allowed in this mode (no host-side collective).
 *
 *   mph_gcn_p2p_export(m, blob_h)  writes this rank's MPH_P2P_BLOB_BYTES descriptor (IPC handle,
 *                                  buffer offsets, row0).  MPH_ESTATE unless comm_mode = P2P.
 *   mph_gcn_p2p_open(m, blobs_h, world, stream)  blobs_h = all ranks' descriptors in rank order
 *                                  (the caller all-gathers them, e.g. over torch.distributed).
 *                                  Maps the peers' arenas, builds the ghost-source table and
 *                                  exchanges the ghost rows of dinv ⊙ X.  Collective: every rank
 *                                  calls it once, before its first epoch.  Synchronises.
 *   mph_gcn_p2p_status(m, err_h, gen_h, flags_h)  *err_h = 0, or MPH_ETIMEOUT if a wait gave up (a
 *                                  peer stopped signalling): that epoch's results are undefined.
 *                                  Diagnostics (nullable): *gen_h = epochs run, flags_h[slot·world + q]
 *                                  = the last step counter rank q signalled here for slot 0 halo,
 *                                  1 loss, 2 gradient, 3 setup (4·world values).  Synchronises.
 * Constraints: world <= 16; every rank runs the same sequence of epochs. */
#define MPH_P2P_BLOB_BYTES 512
int mph_gcn_p2p_export(const mph_gcn* m, uint8_t* blob_h);
int mph_gcn_p2p_open(mph_gcn* m, const uint8_t* blobs_h, int32_t world, void* stream);
int mph_gcn_p2p_status(const mph_gcn* m, int32_t* err_h, int64_t* gen_h, uint64_t* flags_h);

/* order_h[l-1] = 0 transform-first, 1 aggregate-first; mode_h = feature mode. */
int mph_gcn_info(const mph_gcn* m, int32_t* order_h, int32_t* mode_h);
int mph_gcn_destroy(mph_gcn* m);

#ifdef __cplusplus
}
#endif
#endif /* MORPHLING_H_ */
