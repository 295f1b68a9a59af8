// a0 — graph build and the distributed plans D1-D4
// (partition P:440-445/P:488, G2L P:514-515, halo lists P:517-523).
//
// GPU build: 64-bit keys (u<<32 | v) for both directions of every non-loop input edge plus
// the diagonal, one radix sort, unique, then row pointers by binary search.  Every step is
// integer arithmetic, so the CSR is bit-exact with the oracle; dinv follows the G6 recipe
// (IEEE double sqrt and division, one rounding to float).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.cuh"

namespace mph {

static constexpr uint64_t kSentinel = ~0ull;

__global__ void k_check_range(const int32_t* src, const int32_t* dst, int64_t m, int32_t n, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t a = src[i], b = dst[i];
    if (a < 0 || a >= n || b < 0 || b >= n) atomicOr(bad, 1);
  }
}

__global__ void k_make_keys(const int32_t* src, const int32_t* dst, int64_t m, int32_t n, uint64_t* keys) {
  int64_t total = 2 * m + n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k;
    if (i < 2 * m) {
      int64_t e = i >> 1;
      uint64_t a = (uint32_t)src[e], b = (uint32_t)dst[e];
      if (a == b)
        k = kSentinel;  // G2: input self loops dropped (I is added below)
      else
        k = (i & 1) ? ((b << 32) | a) : ((a << 32) | b);  // G2: both directions
    } else {
      uint64_t u = (uint64_t)(i - 2 * m);
      k = (u << 32) | u;  // G3: diagonal
    }
    keys[i] = k;
  }
}

__global__ void k_split_keys(const uint64_t* keys, int64_t nnz, int32_t* col) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    col[i] = (int32_t)(keys[i] & 0xffffffffull);
}

// ptr[u] = first index i with (keys[i] >> 32) >= u, u in [0, n]  (G4)
__global__ void k_lower_bound_hi(const uint64_t* keys, int64_t nnz, int32_t n, int64_t* ptr) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u <= n; u += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nnz;
    uint64_t target = (uint64_t)u << 32;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target)
        lo = mid + 1;
      else
        hi = mid;
    }
    ptr[u] = lo;
  }
}

__global__ void k_degrees(const int64_t* row_ptr, int32_t n, int32_t* deg) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
    deg[u] = (int32_t)(row_ptr[u + 1] - row_ptr[u]);  // G5
}

__global__ void k_dinv(const int32_t* deg, float* dinv, float* dinv1, int64_t n) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    double d = (double)deg[u];
    dinv[u] = __double2float_rn(__ddiv_rn(1.0, __dsqrt_rn(d)));  // G6
    dinv1[u] = __double2float_rn(__ddiv_rn(1.0, d));             // mean aggregation (R6)
  }
}

int launch_dinv(const int32_t* deg, float* dinv, float* dinv1, int64_t n, cudaStream_t s) {
  if (n == 0) return MPH_OK;
  k_dinv<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 4096), 256, 0, s>>>(deg, dinv, dinv1, n);
  count_launch();
  return launch_check("dinv");
}

static unsigned grid_for(int64_t n, int threads = 256) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), 148 * 16));
}

static void graph_free(mph_graph* g) {
  if (!g) return;
  dev_free(g->row_ptr);
  dev_free(g->col_idx);
  dev_free(g->deg);
  dev_free(g->dinv);
  dev_free(g->dinv1);
  dev_free(g->split);
  dev_free(g->send_ids);
  dev_free(g->send_buf);
  dev_free(g->items);
  for (auto& c : g->scsr) {
    dev_free(c.vrow_ptr);
    dev_free(c.vmap);
    dev_free(c.items);
    dev_free(c.srows);
  }
  dev_free(g->chunk_part);
  dev_free(g->item_counter);
  delete g;
}

static int max_degree(const mph_graph* g, cudaStream_t s, int32_t* out) {
  int32_t* d_max = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int rc = MPH_OK;
  if (g->n_rows == 0) {
    *out = 0;
    return MPH_OK;
  }
  cub::DeviceReduce::Max(nullptr, tmp_bytes, g->deg, d_max, g->n_rows, s);
  if ((rc = dev_alloc(&d_max, 1)) != MPH_OK) return rc;
  if ((rc = dev_alloc((char**)&tmp, tmp_bytes)) != MPH_OK) {
    dev_free(d_max);
    return rc;
  }
  cub::DeviceReduce::Max(tmp, tmp_bytes, g->deg, d_max, g->n_rows, s);
  count_launch();
  cudaError_t e = cudaMemcpyAsync(out, d_max, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  dev_free(tmp);
  dev_free(d_max);
  if (e != cudaSuccess) return fail(MPH_ECUDA, "max degree: %s", cudaGetErrorString(e));
  return MPH_OK;
}

}  // namespace mph

using namespace mph;

extern "C" int mph_graph_build(const int32_t* src_h, const int32_t* dst_h, int64_t num_edges, int32_t num_nodes,
                               void* stream, mph_graph** out) {
  if (!out) return fail(MPH_EINVAL, "null out");
  *out = nullptr;
  if (num_nodes <= 0) return fail(MPH_EDEGENERATE, "N = 0 (G1)");
  if (num_edges < 0 || (num_edges > 0 && (!src_h || !dst_h))) return fail(MPH_EINVAL, "bad edge arrays");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t m = num_edges, n = num_nodes, total = 2 * m + n;

  int32_t *d_src = nullptr, *d_dst = nullptr;
  int* d_bad = nullptr;
  uint64_t *keys = nullptr, *keys2 = nullptr;
  int64_t* d_count = nullptr;
  void* tmp = nullptr;
  mph_graph* g = new mph_graph();
  int rc = MPH_OK;
  auto cleanup = [&]() {
    dev_free(d_src);
    dev_free(d_dst);
    dev_free(d_bad);
    dev_free(keys);
    dev_free(keys2);
    dev_free(d_count);
    dev_free(tmp);
  };
#define GB_TRY(x)          \
  do {                     \
    rc = (x);              \
    if (rc != MPH_OK) {    \
      cleanup();           \
      graph_free(g);       \
      return rc;           \
    }                      \
  } while (0)
#define GB_CUDA(x)                                                                             \
  do {                                                                                         \
    cudaError_t _e = (x);                                                                      \
    if (_e != cudaSuccess) {                                                                   \
      cleanup();                                                                               \
      graph_free(g);                                                                           \
      return fail(MPH_ECUDA, "graph_build %s: %s", #x, cudaGetErrorString(_e));                \
    }                                                                                          \
  } while (0)

  GB_TRY(dev_alloc(&d_src, (size_t)std::max<int64_t>(m, 1)));
  GB_TRY(dev_alloc(&d_dst, (size_t)std::max<int64_t>(m, 1)));
  GB_TRY(dev_alloc(&d_bad, 1));
  GB_TRY(dev_alloc(&keys, (size_t)total));
  GB_TRY(dev_alloc(&keys2, (size_t)total));
  GB_TRY(dev_alloc(&d_count, 1));
  if (m > 0) {
    GB_CUDA(cudaMemcpyAsync(d_src, src_h, m * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    GB_CUDA(cudaMemcpyAsync(d_dst, dst_h, m * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  }
  GB_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
  if (m > 0) {
    k_check_range<<<grid_for(m), 256, 0, s>>>(d_src, d_dst, m, (int32_t)n, d_bad);
    count_launch();
  }
  int bad = 0;
  GB_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  GB_CUDA(cudaStreamSynchronize(s));
  if (bad) {
    cleanup();
    graph_free(g);
    return fail(MPH_ERANGE, "node id outside [0, N) (G1)");
  }
  k_make_keys<<<grid_for(total), 256, 0, s>>>(d_src, d_dst, m, (int32_t)n, keys);
  count_launch();
  GB_CUDA(cudaGetLastError());

  // one radix sort over all keys, then unique (G2 dedup, G4 order)
  size_t sort_bytes = 0, uniq_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, keys, keys2, total, 0, 64, s);
  cub::DeviceSelect::Unique(nullptr, uniq_bytes, keys2, keys, d_count, total, s);
  GB_TRY(dev_alloc((char**)&tmp, std::max(sort_bytes, uniq_bytes)));
  GB_CUDA(cub::DeviceRadixSort::SortKeys(tmp, sort_bytes, keys, keys2, total, 0, 64, s));
  GB_CUDA(cub::DeviceSelect::Unique(tmp, uniq_bytes, keys2, keys, d_count, total, s));
  count_launch(2);
  int64_t n_unique = 0;
  GB_CUDA(cudaMemcpyAsync(&n_unique, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  uint64_t last = 0;
  GB_CUDA(cudaStreamSynchronize(s));
  GB_CUDA(cudaMemcpyAsync(&last, keys + (n_unique - 1), sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  GB_CUDA(cudaStreamSynchronize(s));
  const int64_t nnz = (last == kSentinel) ? n_unique - 1 : n_unique;

  g->n_rows = g->n_cols = (int32_t)n;
  g->nnz = nnz;
  GB_TRY(dev_alloc(&g->row_ptr, (size_t)n + 1));
  GB_TRY(dev_alloc(&g->col_idx, (size_t)nnz));
  GB_TRY(dev_alloc(&g->deg, (size_t)n));
  GB_TRY(dev_alloc(&g->dinv, (size_t)n));
  GB_TRY(dev_alloc(&g->dinv1, (size_t)n));
  k_split_keys<<<grid_for(nnz), 256, 0, s>>>(keys, nnz, g->col_idx);
  k_lower_bound_hi<<<grid_for(n + 1), 256, 0, s>>>(keys, nnz, (int32_t)n, g->row_ptr);
  k_degrees<<<grid_for(n), 256, 0, s>>>(g->row_ptr, (int32_t)n, g->deg);
  count_launch(3);
  GB_CUDA(cudaGetLastError());
  GB_TRY(launch_dinv(g->deg, g->dinv, g->dinv1, n, s));
  GB_TRY(max_degree(g, s, &g->max_deg));
  cleanup();
#undef GB_TRY
#undef GB_CUDA
  *out = g;
  return MPH_OK;
}

extern "C" int mph_graph_info(const mph_graph* g, int32_t* n_rows_h, int32_t* n_cols_h, int64_t* nnz_h,
                              int32_t* max_deg_h) {
  if (!g) return fail(MPH_EINVAL, "null graph");
  if (n_rows_h) *n_rows_h = g->n_rows;
  if (n_cols_h) *n_cols_h = g->n_cols;
  if (nnz_h) *nnz_h = g->nnz;
  if (max_deg_h) *max_deg_h = g->max_deg;
  return MPH_OK;
}

extern "C" int mph_graph_csr(const mph_graph* g, const int64_t** row_ptr_d, const int32_t** col_idx_d,
                             const int32_t** deg_d, const float** dinv_d) {
  if (!g) return fail(MPH_EINVAL, "null graph");
  if (row_ptr_d) *row_ptr_d = g->row_ptr;
  if (col_idx_d) *col_idx_d = g->col_idx;
  if (deg_d) *deg_d = g->deg;
  if (dinv_d) *dinv_d = g->dinv;
  return MPH_OK;
}

extern "C" int mph_graph_destroy(mph_graph* g) {
  graph_free(g);
  return MPH_OK;
}

// ------------------------------------------------------------------------------------------
// D1-D4 host plans
// ------------------------------------------------------------------------------------------
struct mph_plan {
  int32_t world = 1, rank = 0, n_own = 0;
  int64_t row0 = 0;
  std::vector<int64_t> ghosts, row_ptr, split, recv_offset, n_recv, send_offset;
  std::vector<int32_t> col_idx, deg_local, send_ids;
};

extern "C" int mph_partition_1d(const int64_t* row_ptr_h, int32_t N, int32_t world, int64_t* bounds_h) {
  if (!row_ptr_h || !bounds_h || world < 1 || N < 0) return fail(MPH_EINVAL, "partition_1d arguments");
  const int64_t nnz = row_ptr_h[N];
  // bounds[r] = min{u in [0,N] : world*row_ptr[u] >= r*nnz}  (D1); row_ptr is nondecreasing.
  int64_t u = 0;
  for (int32_t r = 0; r <= world; ++r) {
    const __int128 target = (__int128)r * nnz;
    int64_t lo = u, hi = N;  // answer in [u, N]
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if ((__int128)world * row_ptr_h[mid] >= target)
        hi = mid;
      else
        lo = mid + 1;
    }
    bounds_h[r] = lo;
    u = lo;
  }
  return MPH_OK;
}

extern "C" int mph_plan_create(const int64_t* row_ptr_h, const int32_t* col_idx_h, int32_t N, const int64_t* bounds_h,
                               int32_t world, int32_t rank, mph_plan** out) {
  if (!row_ptr_h || !col_idx_h || !bounds_h || !out || world < 1 || rank < 0 || rank >= world)
    return fail(MPH_EINVAL, "plan_create arguments");
  *out = nullptr;
  for (int32_t r = 0; r < world; ++r)
    if (bounds_h[r] > bounds_h[r + 1] || bounds_h[0] != 0 || bounds_h[world] != N)
      return fail(MPH_EINVAL, "bounds must be nondecreasing from 0 to N");
  mph_plan* p = new mph_plan();
  p->world = world;
  p->rank = rank;
  const int64_t b0 = bounds_h[rank], b1 = bounds_h[rank + 1];
  p->row0 = b0;
  p->n_own = (int32_t)(b1 - b0);
  const int64_t e0 = row_ptr_h[b0], e1 = row_ptr_h[b1];
  // D2: ghost set, ascending by global id
  std::vector<int64_t> gh;
  gh.reserve((size_t)std::min<int64_t>(e1 - e0, N));
  for (int64_t e = e0; e < e1; ++e) {
    int64_t v = col_idx_h[e];
    if (v < b0 || v >= b1) gh.push_back(v);
  }
  std::sort(gh.begin(), gh.end());
  gh.erase(std::unique(gh.begin(), gh.end()), gh.end());
  p->ghosts = gh;
  const int64_t n_own = p->n_own;
  // D3: local CSR; each row's global columns are ascending, so owned columns (ascending)
  // followed by ghost columns (ascending by global id == by local id) is the local order.
  p->row_ptr.resize(n_own + 1);
  p->split.resize(n_own);
  p->col_idx.resize((size_t)(e1 - e0));
  for (int64_t i = 0; i < n_own; ++i) {
    const int64_t s = row_ptr_h[b0 + i], e = row_ptr_h[b0 + i + 1];
    int64_t w = s - e0;
    p->row_ptr[i] = w;
    for (int64_t k = s; k < e; ++k) {
      int64_t v = col_idx_h[k];
      if (v >= b0 && v < b1) p->col_idx[w++] = (int32_t)(v - b0);
    }
    p->split[i] = w - (s - e0);
    for (int64_t k = s; k < e; ++k) {
      int64_t v = col_idx_h[k];
      if (v < b0 || v >= b1) {
        int64_t j = std::lower_bound(gh.begin(), gh.end(), v) - gh.begin();
        p->col_idx[w++] = (int32_t)(n_own + j);
      }
    }
  }
  p->row_ptr[n_own] = e1 - e0;
  // degrees of owned then ghost nodes
  p->deg_local.resize(n_own + gh.size());
  for (int64_t i = 0; i < n_own; ++i) p->deg_local[i] = (int32_t)(row_ptr_h[b0 + i + 1] - row_ptr_h[b0 + i]);
  for (size_t j = 0; j < gh.size(); ++j) p->deg_local[n_own + j] = (int32_t)(row_ptr_h[gh[j] + 1] - row_ptr_h[gh[j]]);
  // D4: receive slices (ghosts grouped by owner) and send lists
  p->recv_offset.assign(world, 0);
  p->n_recv.assign(world, 0);
  for (int64_t v : gh) {
    int32_t q = (int32_t)(std::upper_bound(bounds_h, bounds_h + world + 1, v) - bounds_h - 1);
    p->n_recv[q]++;
  }
  for (int32_t q = 1; q < world; ++q) p->recv_offset[q] = p->recv_offset[q - 1] + p->n_recv[q - 1];
  p->send_offset.assign(world + 1, 0);
  std::vector<uint8_t> mark((size_t)n_own);
  for (int32_t q = 0; q < world; ++q) {
    if (q != rank) {
      std::fill(mark.begin(), mark.end(), 0);
      const int64_t qs = row_ptr_h[bounds_h[q]], qe = row_ptr_h[bounds_h[q + 1]];
      for (int64_t k = qs; k < qe; ++k) {
        int64_t v = col_idx_h[k];
        if (v >= b0 && v < b1) mark[v - b0] = 1;
      }
      for (int64_t i = 0; i < n_own; ++i)
        if (mark[i]) p->send_ids.push_back((int32_t)i);
    }
    p->send_offset[q + 1] = (int64_t)p->send_ids.size();
  }
  *out = p;
  return MPH_OK;
}

extern "C" int mph_plan_info(const mph_plan* p, int32_t* n_own_h, int64_t* row0_h, int64_t* n_ghost_h, int64_t* nnz_h,
                             int64_t* n_send_h) {
  if (!p) return fail(MPH_EINVAL, "null plan");
  if (n_own_h) *n_own_h = p->n_own;
  if (row0_h) *row0_h = p->row0;
  if (n_ghost_h) *n_ghost_h = (int64_t)p->ghosts.size();
  if (nnz_h) *nnz_h = (int64_t)p->col_idx.size();
  if (n_send_h) *n_send_h = (int64_t)p->send_ids.size();
  return MPH_OK;
}

extern "C" int mph_plan_arrays(const mph_plan* p, const int64_t** ghosts_h, const int64_t** row_ptr_h,
                               const int32_t** col_idx_h, const int64_t** split_h, const int32_t** deg_local_h,
                               const int64_t** recv_offset_h, const int64_t** n_recv_h, const int64_t** send_offset_h,
                               const int32_t** send_ids_h) {
  if (!p) return fail(MPH_EINVAL, "null plan");
  if (ghosts_h) *ghosts_h = p->ghosts.data();
  if (row_ptr_h) *row_ptr_h = p->row_ptr.data();
  if (col_idx_h) *col_idx_h = p->col_idx.data();
  if (split_h) *split_h = p->split.data();
  if (deg_local_h) *deg_local_h = p->deg_local.data();
  if (recv_offset_h) *recv_offset_h = p->recv_offset.data();
  if (n_recv_h) *n_recv_h = p->n_recv.data();
  if (send_offset_h) *send_offset_h = p->send_offset.data();
  if (send_ids_h) *send_ids_h = p->send_ids.data();
  return MPH_OK;
}

extern "C" int mph_plan_destroy(mph_plan* p) {
  delete p;
  return MPH_OK;
}

__global__ void k_split_abs(const int64_t* row_ptr, const int64_t* split_count, int32_t n, int64_t* split) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    split[i] = row_ptr[i] + split_count[i];
}

extern "C" int mph_graph_from_plan(const mph_plan* p, void* stream, mph_graph** out) {
  if (!p || !out) return fail(MPH_EINVAL, "graph_from_plan arguments");
  *out = nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  mph_graph* g = new mph_graph();
  g->local = true;
  g->world = p->world;
  g->rank = p->rank;
  g->row0 = p->row0;
  g->n_rows = p->n_own;
  g->n_cols = (int32_t)(p->n_own + p->ghosts.size());
  g->nnz = (int64_t)p->col_idx.size();
  g->recv_offset = p->recv_offset;
  g->n_recv = p->n_recv;
  g->send_offset = p->send_offset;
  g->ghosts = p->ghosts;
  g->n_send = (int64_t)p->send_ids.size();
  int64_t* split_count = nullptr;
  int rc = MPH_OK;
  auto bail = [&](int code) {
    dev_free(split_count);
    graph_free(g);
    return code;
  };
  if ((rc = dev_alloc(&g->row_ptr, (size_t)g->n_rows + 1)) != MPH_OK) return bail(rc);
  if ((rc = dev_alloc(&g->col_idx, (size_t)g->nnz)) != MPH_OK) return bail(rc);
  if ((rc = dev_alloc(&g->deg, (size_t)g->n_cols)) != MPH_OK) return bail(rc);
  if ((rc = dev_alloc(&g->dinv, (size_t)g->n_cols)) != MPH_OK) return bail(rc);
  if ((rc = dev_alloc(&g->dinv1, (size_t)g->n_cols)) != MPH_OK) return bail(rc);
  if ((rc = dev_alloc(&g->split, (size_t)g->n_rows)) != MPH_OK) return bail(rc);
  if ((rc = dev_alloc(&split_count, (size_t)g->n_rows)) != MPH_OK) return bail(rc);
  if ((rc = dev_alloc(&g->send_ids, (size_t)g->n_send)) != MPH_OK) return bail(rc);
  cudaError_t e = cudaSuccess;
  e = cudaMemcpyAsync(g->row_ptr, p->row_ptr.data(), (g->n_rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && g->nnz)
    e = cudaMemcpyAsync(g->col_idx, p->col_idx.data(), g->nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && g->n_cols)
    e = cudaMemcpyAsync(g->deg, p->deg_local.data(), g->n_cols * sizeof(int32_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && g->n_rows)
    e = cudaMemcpyAsync(split_count, p->split.data(), g->n_rows * sizeof(int64_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && g->n_send)
    e = cudaMemcpyAsync(g->send_ids, p->send_ids.data(), g->n_send * sizeof(int32_t), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return bail(fail(MPH_ECUDA, "graph_from_plan upload: %s", cudaGetErrorString(e)));
  if (g->n_rows) {
    k_split_abs<<<grid_for(g->n_rows), 256, 0, s>>>(g->row_ptr, split_count, g->n_rows, g->split);
    count_launch();
  }
  if ((rc = launch_dinv(g->deg, g->dinv, g->dinv1, g->n_cols, s)) != MPH_OK) return bail(rc);
  if ((rc = max_degree(g, s, &g->max_deg)) != MPH_OK) return bail(rc);  // synchronises
  dev_free(split_count);
  *out = g;
  return MPH_OK;
}

extern "C" int mph_graph_localize(const mph_graph* global, const int64_t* bounds_h, int32_t world, int32_t rank,
                                  void* stream, mph_graph** local_out) {
  if (!global || !bounds_h || !local_out || world < 1 || rank < 0 || rank >= world)
    return fail(MPH_EINVAL, "graph_localize arguments");
  if (global->local) return fail(MPH_EINVAL, "graph_localize: the input is already a localized graph");
  *local_out = nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<int64_t> rp((size_t)global->n_rows + 1);
  std::vector<int32_t> ci((size_t)global->nnz);
  MPH_CUDA_TRY(cudaMemcpyAsync(rp.data(), global->row_ptr, rp.size() * 8, cudaMemcpyDeviceToHost, s));
  if (global->nnz)
    MPH_CUDA_TRY(cudaMemcpyAsync(ci.data(), global->col_idx, ci.size() * 4, cudaMemcpyDeviceToHost, s));
  MPH_CUDA_TRY(cudaStreamSynchronize(s));
  mph_plan* p = nullptr;
  MPH_TRY(mph_plan_create(rp.data(), ci.data(), global->n_rows, bounds_h, world, rank, &p));
  const int rc = mph_graph_from_plan(p, stream, local_out);
  mph_plan_destroy(p);
  return rc;
}

extern "C" int mph_halo_plan(const mph_graph* g, int32_t peer, const int32_t** send_local_ids_d, int64_t* n_send_h,
                             int64_t* recv_offset_h, int64_t* n_recv_h) {
  if (!g || !g->local) return fail(MPH_EINVAL, "halo_plan: needs a localized graph");
  if (peer < 0 || peer >= g->world) return fail(MPH_EINVAL, "halo_plan: peer %d outside [0, %d)", peer, g->world);
  const int64_t s0 = g->send_offset[peer], s1 = g->send_offset[peer + 1];
  if (send_local_ids_d) *send_local_ids_d = g->send_ids ? g->send_ids + s0 : nullptr;
  if (n_send_h) *n_send_h = s1 - s0;
  if (recv_offset_h) *recv_offset_h = g->recv_offset[peer];
  if (n_recv_h) *n_recv_h = g->n_recv[peer];
  return MPH_OK;
}
