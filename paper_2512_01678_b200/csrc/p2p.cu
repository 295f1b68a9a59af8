// NEXT-1 — the halo exchange and the gradient sum over NVLink peer memory.
//
// The paper exchanges boundary rows with MPI Isend/Irecv after packing them and
// sums gradients with an all-reduce, overlapping both with local work.
// On one NVSwitch box every GPU can load from and store to every peer's HBM directly, so here
// the data path has no messages at all:
//   * halo: after the producer of T'_l (or dZ'_l) finishes, its rank publishes a step counter
//     into every peer's flag row (system-scope release store, k_p2p_signal); each consumer's
//     k_halo_pull waits for the owners' counters (acquire) and copies its ghost rows straight
//     out of the owners' buffers into its own ghost slice with 16-byte peer loads, while the
//     local-edge part of the SpMM runs on the compute stream.  No pack kernel, no send buffer.
//   * gradients: each layer's [dW | db] is stored into every rank's receive slab as soon as it is
//     complete (k_grad_push, overlapping the rest of the backward pass); the optimizer kernel
//     (elementwise.cu, optim_sum_launch) waits for all ranks and sums the slabs in rank order, so
//     every rank computes the same bits and the all-reduce is fused into the update.
//   * loss: one single-thread kernel pushes the partial sum, signals, waits and sums.
// Arena layout and slots: internal.cuh (P2PState).  Everything a peer touches lives in ONE
// cudaMalloc allocation per rank, exported once with cudaIpcGetMemHandle and mapped by the
// peers with cudaIpcOpenMemHandle (lazy peer access), so the per-step cost is kernels only.
#include <cstring>

#include "internal.cuh"

namespace mph {

namespace {

struct Blob {  // MPH_P2P_BLOB_BYTES descriptor exchanged by the caller
  cudaIpcMemHandle_t handle;
  uint64_t magic;
  int32_t world, rank;
  int64_t row0, n_rows, n_params;
  int64_t off_flags, off_loss, off_gsum;
  int32_t n_buf;
  uint32_t layout_sig;
  int64_t off_buf[40];
};
static_assert(sizeof(Blob) <= MPH_P2P_BLOB_BYTES, "blob too large");
constexpr uint64_t kMagic = 0x4d50483250325031ull;  // "MPH2P2P1"

struct PeerF4 {
  const float4* p[kP2PMaxWorld];
};
struct PeerMutF4 {
  float4* p[kP2PMaxWorld];
};
struct PeerU64 {
  uint64_t* p[kP2PMaxWorld];
};
struct PeerF64 {
  double* p[kP2PMaxWorld];
};

__device__ __forceinline__ uint64_t seq_of(const int64_t* gen_dev, int64_t mult, int64_t add) {
  return (uint64_t)((gen_dev ? *gen_dev : 0) * mult + add);
}

__global__ void k_gen_advance(int64_t* gen) { *gen += 1; }

__global__ void k_p2p_signal(const __grid_constant__ PeerU64 f, int world, int rank, const int64_t* gen_dev,
                             int64_t mult, int64_t add) {
  const uint64_t seq = seq_of(gen_dev, mult, add);
  __threadfence_system();  // this stream's earlier writes are visible system-wide first
  const int q = threadIdx.x;
  if (q < world) st_release_sys_u64(f.p[q] + rank, seq);
}

// 256 threads; each warp moves 4 ghost rows per step (4 x w/128 independent 16 B peer loads
// in flight per lane), L2-only loads (__ldcg: never a stale L1 line of a peer's buffer).
__global__ void __launch_bounds__(256) k_halo_pull(const __grid_constant__ PeerF4 src, int world,
                                                   const int32_t* __restrict__ ghost_ref, float4* __restrict__ dst,
                                                   int64_t n_ghost, int w4, const uint64_t* flags_row,
                                                   const int64_t* gen_dev, int64_t mult, int64_t add, int* err) {
  __shared__ int ok;
  if (threadIdx.x == 0) ok = p2p_wait_all(flags_row, world, seq_of(gen_dev, mult, add), err);
  __syncthreads();
  if (!ok) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j0 = warp * 4; j0 < n_ghost; j0 += nw * 4) {
    const float4* s[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t j = j0 + r;
      const int32_t ref = j < n_ghost ? __ldg(ghost_ref + j) : 0;
      s[r] = src.p[ref >> 27] + (int64_t)(ref & ((1 << 27) - 1)) * w4;
    }
    for (int c = lane; c < w4; c += 32) {
      float4 v[4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (j0 + r < n_ghost) v[r] = __ldcg(s[r] + c);
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (j0 + r < n_ghost) dst[(j0 + r) * w4 + c] = v[r];
    }
  }
}

__global__ void k_grad_push(const __grid_constant__ PeerMutF4 dst, int world, int rank, const float4* __restrict__ g,
                            int64_t a4, int64_t b4, int64_t n4, const int64_t* gen_dev) {
  const int64_t par = *gen_dev & 1;
  const int64_t base = (par * world + rank) * n4;
  for (int64_t i = a4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = g[i];
    for (int q = 0; q < world; ++q) dst.p[q][base + i] = v;
  }
  __threadfence_system();
}

__global__ void k_loss_sum(const __grid_constant__ PeerF64 slots, const __grid_constant__ PeerU64 flags, int world,
                           int rank, double* loss, const double* my_slots, const uint64_t* my_flags,
                           const int64_t* gen_dev, int* err) {
  const int64_t gen = *gen_dev;
  const int par = (int)(gen & 1);
  const double v = *loss;
  for (int q = 0; q < world; ++q) slots.p[q][par * kP2PMaxWorld + rank] = v;
  __threadfence_system();
  for (int q = 0; q < world; ++q) st_release_sys_u64(flags.p[q] + rank, (uint64_t)gen);
  if (!p2p_wait_all(my_flags, world, (uint64_t)gen, err)) return;
  double s = 0.0;
  for (int q = 0; q < world; ++q) s += *(volatile const double*)(my_slots + par * kP2PMaxWorld + q);
  *loss = s;
}

int64_t align256(int64_t x) { return (x + 255) / 256 * 256; }

}  // namespace

int p2p_alloc_arena(P2PState* p, size_t bytes) {
  p->off_flags = 0;
  p->off_loss = align256((int64_t)kP2PSlots * kP2PMaxWorld * 8);
  p->off_gsum = p->off_loss + align256(2 * kP2PMaxWorld * 8);
  const int64_t head = p->off_gsum + align256(2 * (int64_t)p->world * p->n_params * 4);
  p->arena_bytes = (size_t)head + bytes;
  cudaError_t e = cudaMalloc((void**)&p->arena, p->arena_bytes);
  if (e != cudaSuccess)
    return fail(e == cudaErrorMemoryAllocation ? MPH_ENOMEM : MPH_ECUDA, "p2p arena (%zu B): %s", p->arena_bytes,
                cudaGetErrorString(e));
  MPH_CUDA_TRY(cudaMemset(p->arena, 0, (size_t)head));  // flags start at 0 before any peer can signal
  MPH_TRY(dev_alloc(&p->gen_dev, 1));
  MPH_TRY(dev_alloc(&p->err_dev, 1));
  MPH_CUDA_TRY(cudaMemset(p->gen_dev, 0, sizeof(int64_t)));
  MPH_CUDA_TRY(cudaMemset(p->err_dev, 0, sizeof(int)));
  return MPH_OK;
}

void p2p_free(P2PState* p) {
  if (!p) return;
  for (int q = 0; q < (int)p->peer_base.size(); ++q)
    if (q != p->rank && p->peer_base[q]) cudaIpcCloseMemHandle(p->peer_base[q]);
  if (p->arena) cudaFree(p->arena);
  dev_free(p->ghost_ref);
  dev_free(p->gen_dev);
  dev_free(p->err_dev);
  delete p;
}

int p2p_export(const P2PState* p, uint8_t* blob_h) {
  Blob b;
  std::memset(&b, 0, sizeof(b));
  MPH_CUDA_TRY(cudaIpcGetMemHandle(&b.handle, p->arena));
  b.magic = kMagic;
  b.world = p->world;
  b.rank = p->rank;
  b.row0 = p->row0;
  b.n_rows = p->n_rows;
  b.n_params = p->n_params;
  b.off_flags = p->off_flags;
  b.off_loss = p->off_loss;
  b.off_gsum = p->off_gsum;
  if (p->off_buf.size() > 40) return fail(MPH_ENOTSUP, "p2p: too many shared buffers");
  b.n_buf = (int32_t)p->off_buf.size();
  b.layout_sig = p->layout_sig;
  for (size_t i = 0; i < p->off_buf.size(); ++i) b.off_buf[i] = p->off_buf[i];
  std::memset(blob_h, 0, MPH_P2P_BLOB_BYTES);
  std::memcpy(blob_h, &b, sizeof(b));
  return MPH_OK;
}

int p2p_open(P2PState* p, const mph_graph* g, const uint8_t* blobs, int world) {
  if (p->opened) return fail(MPH_ESTATE, "p2p_open: already open");
  if (world != p->world) return fail(MPH_EINVAL, "p2p_open: world %d != model world %d", world, p->world);
  std::vector<Blob> b(world);
  for (int q = 0; q < world; ++q) {
    std::memcpy(&b[q], blobs + (size_t)q * MPH_P2P_BLOB_BYTES, sizeof(Blob));
    if (b[q].magic != kMagic || b[q].world != world || b[q].rank != q)
      return fail(MPH_EINVAL, "p2p_open: blob %d is not rank %d's descriptor of a world-%d model", q, q, world);
    if (b[q].n_params != p->n_params || b[q].n_buf != (int32_t)p->off_buf.size())
      return fail(MPH_EINVAL, "p2p_open: rank %d's model has a different layout", q);
    if (b[q].layout_sig != p->layout_sig)
      return fail(MPH_EINVAL,
                  "p2p_open: rank %d decided feature mode / layer orders 0x%x, this rank 0x%x: the dense/sparse "
                  "switch must be global (decide it from the global nnz, mph_features_decide, and pass force_mode)",
                  q, b[q].layout_sig, p->layout_sig);
  }
  p->peer_base.assign(world, nullptr);
  p->peer_off.assign(world, {});
  p->peer_flags_off.assign(world, 0);
  p->peer_loss_off.assign(world, 0);
  p->peer_gsum_off.assign(world, 0);
  for (int q = 0; q < world; ++q) {
    if (q == p->rank) {
      p->peer_base[q] = p->arena;
    } else {
      void* ptr = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&ptr, b[q].handle, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return fail(MPH_ECUDA, "cudaIpcOpenMemHandle(rank %d): %s", q, cudaGetErrorString(e));
      p->peer_base[q] = (char*)ptr;
    }
    p->peer_off[q].assign(b[q].off_buf, b[q].off_buf + b[q].n_buf);
    p->peer_flags_off[q] = b[q].off_flags;
    p->peer_loss_off[q] = b[q].off_loss;
    p->peer_gsum_off[q] = b[q].off_gsum;
  }
  // ghost j of owner q (the receive slices are grouped by owner, D4) is row ghosts[j] - row0_q
  // of q's buffers: contiguous ranges, as D1 and mph_relabel produce.
  p->n_ghost = (int64_t)g->ghosts.size();
  std::vector<int32_t> ref(p->n_ghost);
  for (int q = 0; q < world; ++q) {
    const int64_t o = g->recv_offset[q], n = g->n_recv[q];
    for (int64_t j = o; j < o + n; ++j) {
      const int64_t r = g->ghosts[j] - b[q].row0;
      if (q == p->rank || r < 0 || r >= b[q].n_rows || r >= (1 << 27))
        return fail(MPH_EINVAL, "p2p_open: ghost %lld (global %lld) is not an owned row of rank %d", (long long)j,
                    (long long)g->ghosts[j], q);
      ref[j] = (int32_t)((q << 27) | r);
    }
  }
  if (p->n_ghost) {
    MPH_TRY(dev_alloc(&p->ghost_ref, (size_t)p->n_ghost));
    MPH_CUDA_TRY(cudaMemcpy(p->ghost_ref, ref.data(), ref.size() * 4, cudaMemcpyHostToDevice));
  }
  p->opened = true;
  return MPH_OK;
}

static PeerU64 flag_rows(const P2PState* p, int slot) {
  PeerU64 f{};
  for (int q = 0; q < p->world; ++q)
    f.p[q] = (uint64_t*)(p->peer_base[q] + p->peer_flags_off[q]) + (size_t)slot * kP2PMaxWorld;
  return f;
}

const uint64_t* p2p_flags_local(const P2PState* p, int slot) {
  return (const uint64_t*)(p->arena + p->off_flags) + (size_t)slot * kP2PMaxWorld;
}
const float* p2p_gsum_local(const P2PState* p) { return (const float*)(p->arena + p->off_gsum); }

int p2p_grad_mirror(const P2PState* p, int64_t off, GradMirror* out) {
  if (!p->opened) return fail(MPH_ESTATE, "p2p: mph_gcn_p2p_open has not been called");
  *out = GradMirror{};
  for (int q = 0; q < p->world; ++q)
    out->base[q] = (float*)(p->peer_base[q] + p->peer_gsum_off[q]) + (int64_t)p->rank * p->n_params + off;
  out->n = p->world;
  out->gen_dev = p->gen_dev;
  out->par_stride = (int64_t)p->world * p->n_params;
  return MPH_OK;
}

int p2p_gen_advance(const P2PState* p, cudaStream_t s) {
  k_gen_advance<<<1, 1, 0, s>>>(p->gen_dev);
  count_launch();
  return launch_check("p2p gen advance");
}

int p2p_signal(const P2PState* p, int slot, bool use_gen, int64_t mult, int64_t add, cudaStream_t s) {
  if (!p->opened) return fail(MPH_ESTATE, "p2p: mph_gcn_p2p_open has not been called");
  k_p2p_signal<<<1, 32, 0, s>>>(flag_rows(p, slot), p->world, p->rank, use_gen ? p->gen_dev : nullptr, mult, add);
  count_launch();
  return launch_check("p2p signal");
}

int p2p_pull(const P2PState* p, int buf, float* local, int w, int slot, bool use_gen, int64_t mult, int64_t add,
             cudaStream_t s) {
  if (!p->opened) return fail(MPH_ESTATE, "p2p: mph_gcn_p2p_open has not been called");
  if (w % 4) return fail(MPH_EINVAL, "p2p pull: width %d not a multiple of 4", w);
  PeerF4 src{};
  for (int q = 0; q < p->world; ++q) {
    const int64_t off = p->peer_off[q][buf];
    if (off < 0) return fail(MPH_EINVAL, "p2p pull: buffer %d is not shared", buf);
    src.p[q] = (const float4*)(p->peer_base[q] + off);
  }
  // launched even without ghosts: the wait alone keeps this rank in step with its peers
  const int w4 = w / 4;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(p->n_ghost, 32), 2 * 148));
  k_halo_pull<<<(unsigned)blocks, 256, 0, s>>>(src, p->world, p->ghost_ref, (float4*)(local + p->n_rows * (int64_t)w),
                                               p->n_ghost, w4, p2p_flags_local(p, slot), use_gen ? p->gen_dev : nullptr,
                                               mult, add, p->err_dev);
  count_launch();
  return launch_check("p2p halo pull");
}

int p2p_grad_push(const P2PState* p, const float* grads, int64_t a, int64_t b, cudaStream_t s) {
  if (!p->opened) return fail(MPH_ESTATE, "p2p: mph_gcn_p2p_open has not been called");
  if (a % 4 || b % 4 || p->n_params % 4) return fail(MPH_EINVAL, "p2p grad push: unaligned segment");
  if (b <= a) return MPH_OK;
  PeerMutF4 dst{};
  for (int q = 0; q < p->world; ++q) dst.p[q] = (float4*)(p->peer_base[q] + p->peer_gsum_off[q]);
  const int64_t n4 = (b - a) / 4;
  k_grad_push<<<(unsigned)std::min<int64_t>(ceil_div(n4, 256), 148), 256, 0, s>>>(
      dst, p->world, p->rank, (const float4*)grads, a / 4, b / 4, p->n_params / 4, p->gen_dev);
  count_launch();
  return launch_check("p2p grad push");
}

int p2p_loss_sum(const P2PState* p, double* loss_d, cudaStream_t s) {
  if (!p->opened) return fail(MPH_ESTATE, "p2p: mph_gcn_p2p_open has not been called");
  PeerF64 slots{};
  for (int q = 0; q < p->world; ++q) slots.p[q] = (double*)(p->peer_base[q] + p->peer_loss_off[q]);
  k_loss_sum<<<1, 1, 0, s>>>(slots, flag_rows(p, kSlotLoss), p->world, p->rank, loss_d,
                             (const double*)(p->arena + p->off_loss), p2p_flags_local(p, kSlotLoss), p->gen_dev,
                             p->err_dev);
  count_launch();
  return launch_check("p2p loss sum");
}

}  // namespace mph
