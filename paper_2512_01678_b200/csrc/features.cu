// a1 — feature analysis and the dense/sparse switch (Alg. 1 Initialize; Eq. 1
// P:213-215; tau P:216; readings Q11/Q12/Q28).  All decisions are integer counts, so the mode
// and the X_csr / X_csc patterns are bit-exact with the oracle.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace mph {

// Warp per row: nonzero count and non-unit count of row i.
__global__ void k_row_counts(const float* X, int32_t N, int32_t F, int32_t ld, int64_t* row_nnz, int64_t* row_nonunit) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < N; i += nwarps) {
    const float* row = X + i * (int64_t)ld;
    int c = 0, nu = 0;
    for (int k = lane; k < F; k += 32) {
      float x = row[k];
      c += (x != 0.0f);                   // S1: IEEE compare (Q12)
      nu += (x != 0.0f) && (x != 1.0f);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      c += __shfl_xor_sync(0xffffffffu, c, o);
      nu += __shfl_xor_sync(0xffffffffu, nu, o);
    }
    if (lane == 0) {
      row_nnz[i] = c;
      row_nonunit[i] = nu;
    }
  }
}

// Warp per row: write the row's nonzeros in ascending column order at ptr[i] (S3).
__global__ void k_fill_csr(const float* X, int32_t N, int32_t F, int32_t ld, const int64_t* ptr, int32_t* idx,
                           float* val) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < N; i += nwarps) {
    const float* row = X + i * (int64_t)ld;
    int64_t pos = ptr[i];
    for (int k0 = 0; k0 < F; k0 += 32) {
      int k = k0 + lane;
      float x = k < F ? row[k] : 0.0f;
      unsigned bal = __ballot_sync(0xffffffffu, x != 0.0f);
      if (x != 0.0f) {
        int off = __popc(bal & ((1u << lane) - 1u));
        idx[pos + off] = k;
        val[pos + off] = x;
      }
      pos += __popc(bal);
    }
  }
}

// keys = (col << 32) | row for every CSR entry (CSC order after a sort).
__global__ void k_csc_keys(const int64_t* ptr, const int32_t* idx, int32_t N, uint64_t* keys) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < N; i += nwarps)
    for (int64_t e = ptr[i] + lane; e < ptr[i + 1]; e += 32) keys[e] = ((uint64_t)(uint32_t)idx[e] << 32) | (uint64_t)i;
}

__global__ void k_csc_split(const uint64_t* keys, int64_t nnz, int32_t* ridx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    ridx[e] = (int32_t)(keys[e] & 0xffffffffull);
}

__global__ void k_col_ptr(const uint64_t* keys, int64_t nnz, int32_t F, int64_t* cptr) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= F; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nnz;
    uint64_t t = (uint64_t)c << 32;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < t)
        lo = mid + 1;
      else
        hi = mid;
    }
    cptr[c] = lo;
  }
}

// Dense copy with zero padding: out[i][k] = k < F ? X[i][k] : 0, k < P.
__global__ void k_pad_copy(const float* X, int32_t N, int32_t F, int32_t ld, float* out, int32_t P) {
  int64_t total = (int64_t)N * P;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / P;
    int k = (int)(t - i * P);
    out[t] = k < F ? X[i * (int64_t)ld + k] : 0.0f;
  }
}

// X_csc from X_csr (sort of (col << 32 | row) keys, values carried along), then the per-column
// segments of <= kSegNnz nonzeros used by the sparse dW kernel.  Synchronises.
static int csc_from_csr(mph_features* f, cudaStream_t s) {
  const int64_t nnz = f->nnz;
  const int32_t N = f->N, F = f->F;
  uint64_t *keys = nullptr, *keys2 = nullptr;
  void* tmp = nullptr;
  int rc = MPH_OK;
  auto done = [&](int code) {
    dev_free(keys);
    dev_free(keys2);
    dev_free(tmp);
    return code;
  };
  cudaError_t e = cudaSuccess;
  if (nnz > 0) {
    if ((rc = dev_alloc(&keys, (size_t)nnz)) || (rc = dev_alloc(&keys2, (size_t)nnz))) return done(rc);
    const unsigned warps_grid = (unsigned)std::min<int64_t>(ceil_div((int64_t)N * 32, 256), 148 * 32);
    k_csc_keys<<<warps_grid, 256, 0, s>>>(f->csr_ptr, f->csr_idx, N, keys);
    count_launch();
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, f->csr_val, f->csc_val, nnz, 0, 64, s);
    if ((rc = dev_alloc((char**)&tmp, tb))) return done(rc);
    e = cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, f->csr_val, f->csc_val, nnz, 0, 64, s);
    count_launch();
    if (e != cudaSuccess) return done(fail(MPH_ECUDA, "csc sort: %s", cudaGetErrorString(e)));
    k_csc_split<<<(unsigned)std::min<int64_t>(ceil_div(nnz, 256), 4096), 256, 0, s>>>(keys2, nnz, f->csc_idx);
    count_launch();
  }
  k_col_ptr<<<(unsigned)ceil_div((int64_t)F + 1, 256), 256, 0, s>>>(keys2 ? keys2 : keys, nnz, F, f->csc_ptr);
  count_launch();
  e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return done(fail(MPH_ECUDA, "csc build: %s", cudaGetErrorString(e)));
  std::vector<int64_t> cptr((size_t)F + 1);
  e = cudaMemcpy(cptr.data(), f->csc_ptr, cptr.size() * sizeof(int64_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return done(fail(MPH_ECUDA, "segments: %s", cudaGetErrorString(e)));
  std::vector<int32_t> sc;
  std::vector<int64_t> sb, c0((size_t)F + 1);
  for (int32_t k = 0; k < F; ++k) {
    c0[k] = (int64_t)sc.size();
    for (int64_t b = cptr[k]; b < cptr[k + 1]; b += kSegNnz) {
      sc.push_back(k);
      sb.push_back(b);
    }
  }
  c0[F] = (int64_t)sc.size();
  f->n_seg = (int64_t)sc.size();
  if ((rc = dev_alloc(&f->col_seg0, (size_t)F + 1)) || (rc = dev_alloc(&f->seg_col, sc.size())) ||
      (rc = dev_alloc(&f->seg_begin, sb.size())))
    return done(rc);
  e = cudaMemcpy(f->col_seg0, c0.data(), c0.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !sc.empty())
    e = cudaMemcpy(f->seg_col, sc.data(), sc.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !sb.empty())
    e = cudaMemcpy(f->seg_begin, sb.data(), sb.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return done(fail(MPH_ECUDA, "segments upload: %s", cudaGetErrorString(e)));
  // segments are contiguous runs of X_csc in order, so their begins (+ nnz) form the row_ptr of a
  // virtual CSR whose rows are the segments: the dW gather runs on it like any SpMM
  sb.push_back(nnz);
  if ((rc = dev_alloc(&f->seg_ptr, sb.size()))) return done(rc);
  e = cudaMemcpy(f->seg_ptr, sb.data(), sb.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return done(fail(MPH_ECUDA, "segments upload: %s", cudaGetErrorString(e)));
  if ((rc = build_work_items(f->csr_ptr, N, nnz, &f->xw_items, &f->xw_n_items, s)) ||
      (rc = build_work_items(f->seg_ptr, (int)f->n_seg, nnz, &f->xtg_items, &f->xtg_n_items, s)) ||
      (rc = dev_alloc(&f->item_counter, 1)))
    return done(rc);
  return done(MPH_OK);
}

// Dense padded copy from CSR: warp per row scatters its entries.
__global__ void k_csr_scatter(const int64_t* ptr, const int32_t* idx, const float* val, int32_t N, float* X, int32_t P) {
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += nwarps)
    for (int64_t e = ptr[i] + lane; e < ptr[i + 1]; e += 32) X[i * P + idx[e]] = val[e];
}

static void features_free(mph_features* f) {
  if (!f) return;
  dev_free(f->X);
  dev_free(f->csr_ptr);
  dev_free(f->csr_idx);
  dev_free(f->csr_val);
  dev_free(f->csc_ptr);
  dev_free(f->csc_idx);
  dev_free(f->csc_val);
  dev_free(f->seg_col);
  dev_free(f->seg_begin);
  dev_free(f->col_seg0);
  dev_free(f->seg_ptr);
  dev_free(f->xw_items);
  dev_free(f->xtg_items);
  dev_free(f->item_counter);
  dev_free(f->part);
  delete f;
}

// S2 (Eq. 1, Alg. 1): Sparse iff s = 1 − nnz/(N·F) ≥ τ, decided in integers
// (Q11): 10000·nnz ≤ (10000 − τ_bp)·N·F.
static int32_t decide_mode(int64_t nnz, int64_t N, int64_t F, int32_t tau_bp) {
  const __int128 lhs = (__int128)10000 * nnz, rhs = (__int128)(10000 - tau_bp) * N * F;
  return lhs <= rhs ? 1 : 0;
}

}  // namespace mph

using namespace mph;

extern "C" int mph_features_decide(int64_t nnz, int64_t N, int64_t F, int32_t tau_bp, int32_t* mode_h) {
  if (!mode_h || nnz < 0 || N <= 0 || F <= 0 || tau_bp < 0 || tau_bp > 10000 || nnz > (__int128)N * F)
    return fail(MPH_EINVAL, "features_decide arguments");
  *mode_h = decide_mode(nnz, N, F, tau_bp);
  return MPH_OK;
}

extern "C" int mph_features_count(const float* X_d, int32_t N, int32_t F, int32_t ld, void* stream, int64_t* nnz_h) {
  if (!nnz_h || !X_d || N <= 0 || F <= 0 || ld < F) return fail(MPH_EINVAL, "features_count arguments");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t *row_nnz = nullptr, *row_nu = nullptr, *sums = nullptr;
  void* tmp = nullptr;
  auto done = [&](int code) {
    dev_free(row_nnz);
    dev_free(row_nu);
    dev_free(sums);
    dev_free(tmp);
    return code;
  };
  int rc = MPH_OK;
  if ((rc = dev_alloc(&row_nnz, (size_t)N)) || (rc = dev_alloc(&row_nu, (size_t)N)) || (rc = dev_alloc(&sums, 1)))
    return done(rc);
  const unsigned warps_grid = (unsigned)std::min<int64_t>(ceil_div((int64_t)N * 32, 256), 148 * 32);
  k_row_counts<<<warps_grid, 256, 0, s>>>(X_d, N, F, ld, row_nnz, row_nu);
  count_launch();
  size_t tb = 0;
  cub::DeviceReduce::Sum(nullptr, tb, row_nnz, sums, N, s);
  if ((rc = dev_alloc((char**)&tmp, std::max<size_t>(tb, 1)))) return done(rc);
  cudaError_t e = cub::DeviceReduce::Sum(tmp, tb, row_nnz, sums, N, s);
  count_launch();
  if (e == cudaSuccess) e = cudaMemcpyAsync(nnz_h, sums, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return done(fail(MPH_ECUDA, "features_count: %s", cudaGetErrorString(e)));
  return done(MPH_OK);
}

extern "C" int mph_features_create(const float* X_d, int32_t N, int32_t F, int32_t ld, int32_t tau_bp,
                                   int32_t force_mode, void* stream, mph_features** out) {
  if (!out) return fail(MPH_EINVAL, "null out");
  *out = nullptr;
  if (N <= 0 || F <= 0) return fail(MPH_EDEGENERATE, "N*F = 0");
  if (!X_d || ld < F || tau_bp < 0 || tau_bp > 10000 || force_mode < -1 || force_mode > 1)
    return fail(MPH_EINVAL, "features_create arguments");
  cudaStream_t s = (cudaStream_t)stream;
  mph_features* f = new mph_features();
  f->N = N;
  f->F = F;
  int64_t *row_nnz = nullptr, *row_nu = nullptr, *sums = nullptr;
  void* tmp = nullptr;
  int rc = MPH_OK;
  auto cleanup = [&]() {
    dev_free(row_nnz);
    dev_free(row_nu);
    dev_free(sums);
    dev_free(tmp);
  };
  auto bail = [&](int code) {
    cleanup();
    features_free(f);
    return code;
  };
  auto cuda_bail = [&](cudaError_t e, const char* what) {
    return bail(fail(MPH_ECUDA, "features_create %s: %s", what, cudaGetErrorString(e)));
  };
  if ((rc = dev_alloc(&row_nnz, (size_t)N)) || (rc = dev_alloc(&row_nu, (size_t)N)) || (rc = dev_alloc(&sums, 2)))
    return bail(rc);
  const unsigned warps_grid = (unsigned)std::min<int64_t>(ceil_div((int64_t)N * 32, 256), 148 * 32);
  k_row_counts<<<warps_grid, 256, 0, s>>>(X_d, N, F, ld, row_nnz, row_nu);
  count_launch();
  size_t tb = 0, tb2 = 0;
  cub::DeviceReduce::Sum(nullptr, tb, row_nnz, sums, N, s);
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, row_nnz, row_nnz, N, s);
  if ((rc = dev_alloc((char**)&tmp, std::max(tb, tb2)))) return bail(rc);
  cudaError_t e = cub::DeviceReduce::Sum(tmp, tb, row_nnz, sums, N, s);
  if (e == cudaSuccess) e = cub::DeviceReduce::Sum(tmp, tb, row_nu, sums + 1, N, s);
  count_launch(2);
  int64_t h_sums[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(h_sums, sums, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_bail(e, "count");
  f->nnz = h_sums[0];
  f->is_binary = (h_sums[1] == 0);
  f->mode = force_mode >= 0 ? force_mode : decide_mode(f->nnz, N, F, tau_bp);  // S2: s >= tau, in integers

  if (f->mode == 0) {
    f->P = pad_width(F);
    if ((rc = dev_alloc(&f->X, (size_t)N * f->P))) return bail(rc);
    k_pad_copy<<<(unsigned)std::min<int64_t>(ceil_div((int64_t)N * f->P, 256), 148 * 64), 256, 0, s>>>(X_d, N, F, ld,
                                                                                                       f->X, f->P);
    count_launch();
  } else {
    const int64_t nnz = f->nnz;
    if ((rc = dev_alloc(&f->csr_ptr, (size_t)N + 1)) || (rc = dev_alloc(&f->csr_idx, (size_t)nnz)) ||
        (rc = dev_alloc(&f->csr_val, (size_t)nnz)) || (rc = dev_alloc(&f->csc_ptr, (size_t)F + 1)) ||
        (rc = dev_alloc(&f->csc_idx, (size_t)nnz)) || (rc = dev_alloc(&f->csc_val, (size_t)nnz)))
      return bail(rc);
    e = cub::DeviceScan::ExclusiveSum(tmp, tb2, row_nnz, f->csr_ptr, N, s);
    count_launch();
    if (e == cudaSuccess) e = cudaMemcpyAsync(f->csr_ptr + N, &f->nnz, sizeof(int64_t), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_bail(e, "scan");
    k_fill_csr<<<warps_grid, 256, 0, s>>>(X_d, N, F, ld, f->csr_ptr, f->csr_idx, f->csr_val);
    count_launch();
    if ((rc = csc_from_csr(f, s))) return bail(rc);
  }
  e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_bail(e, "build");
  cleanup();
  *out = f;
  return MPH_OK;
}

extern "C" int mph_features_create_csr(const int64_t* ptr_h, const int32_t* idx_h, const float* val_h, int32_t N,
                                       int32_t F, int32_t tau_bp, int32_t force_mode, void* stream,
                                       mph_features** out) {
  if (!out) return fail(MPH_EINVAL, "null out");
  *out = nullptr;
  if (N <= 0 || F <= 0) return fail(MPH_EDEGENERATE, "N*F = 0");
  if (!ptr_h || tau_bp < 0 || tau_bp > 10000 || force_mode < -1 || force_mode > 1)
    return fail(MPH_EINVAL, "features_create_csr arguments");
  const int64_t m = ptr_h[N];
  if (ptr_h[0] != 0 || m < 0 || (m > 0 && (!idx_h || !val_h))) return fail(MPH_EINVAL, "features_create_csr: bad row_ptr");
  // Host validation (S3: columns strictly ascending within a row) and the S1 count of nonzeros:
  // explicit zeros in val are not entries of X_csr, so they are dropped.
  int64_t nnz = 0, nonunit = 0;
  bool has_zeros = false;
  for (int32_t i = 0; i < N; ++i) {
    if (ptr_h[i + 1] < ptr_h[i]) return fail(MPH_EINVAL, "features_create_csr: row_ptr not monotone at %d", i);
    for (int64_t e = ptr_h[i]; e < ptr_h[i + 1]; ++e) {
      if (idx_h[e] < 0 || idx_h[e] >= F || (e > ptr_h[i] && idx_h[e] <= idx_h[e - 1]))
        return fail(MPH_EINVAL, "features_create_csr: column index out of range or not ascending in row %d", i);
      const float x = val_h[e];
      if (x != 0.0f) {
        ++nnz;
        nonunit += (x != 1.0f);
      } else {
        has_zeros = true;
      }
    }
  }
  std::vector<int64_t> p2;
  std::vector<int32_t> i2;
  std::vector<float> v2;
  const int64_t* P_h = ptr_h;
  const int32_t* I_h = idx_h;
  const float* V_h = val_h;
  if (has_zeros) {
    p2.resize((size_t)N + 1);
    i2.reserve((size_t)nnz);
    v2.reserve((size_t)nnz);
    p2[0] = 0;
    for (int32_t i = 0; i < N; ++i) {
      for (int64_t e = ptr_h[i]; e < ptr_h[i + 1]; ++e)
        if (val_h[e] != 0.0f) {
          i2.push_back(idx_h[e]);
          v2.push_back(val_h[e]);
        }
      p2[(size_t)i + 1] = (int64_t)i2.size();
    }
    P_h = p2.data();
    I_h = i2.data();
    V_h = v2.data();
  }
  cudaStream_t s = (cudaStream_t)stream;
  mph_features* f = new mph_features();
  f->N = N;
  f->F = F;
  f->nnz = nnz;
  f->is_binary = (nonunit == 0);
  f->mode = force_mode >= 0 ? force_mode : decide_mode(nnz, N, F, tau_bp);  // S2, as in mph_features_create
  int rc = MPH_OK;
  int64_t* tptr = nullptr;
  int32_t* tidx = nullptr;
  float* tval = nullptr;
  auto bail = [&](int code) {
    dev_free(tptr);
    dev_free(tidx);
    dev_free(tval);
    features_free(f);
    return code;
  };
  if (f->mode == 1) {
    if ((rc = dev_alloc(&f->csr_ptr, (size_t)N + 1)) || (rc = dev_alloc(&f->csr_idx, (size_t)nnz)) ||
        (rc = dev_alloc(&f->csr_val, (size_t)nnz)) || (rc = dev_alloc(&f->csc_ptr, (size_t)F + 1)) ||
        (rc = dev_alloc(&f->csc_idx, (size_t)nnz)) || (rc = dev_alloc(&f->csc_val, (size_t)nnz)))
      return bail(rc);
    tptr = f->csr_ptr;
    tidx = f->csr_idx;
    tval = f->csr_val;
  } else {
    f->P = pad_width(F);
    if ((rc = dev_alloc(&f->X, (size_t)N * f->P)) || (rc = dev_alloc(&tptr, (size_t)N + 1)) ||
        (rc = dev_alloc(&tidx, (size_t)nnz)) || (rc = dev_alloc(&tval, (size_t)nnz)))
      return bail(rc);
  }
  cudaError_t e = cudaMemcpyAsync(tptr, P_h, ((size_t)N + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && nnz > 0) e = cudaMemcpyAsync(tidx, I_h, (size_t)nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && nnz > 0) e = cudaMemcpyAsync(tval, V_h, (size_t)nnz * sizeof(float), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) {
    if (f->mode == 1) tptr = nullptr, tidx = nullptr, tval = nullptr;
    return bail(fail(MPH_ECUDA, "features_create_csr upload: %s", cudaGetErrorString(e)));
  }
  if (f->mode == 1) {
    tptr = nullptr;  // owned by f from here on
    tidx = nullptr;
    tval = nullptr;
    if ((rc = csc_from_csr(f, s))) return bail(rc);
  } else {
    e = cudaMemsetAsync(f->X, 0, (size_t)N * f->P * sizeof(float), s);
    if (e != cudaSuccess) return bail(fail(MPH_ECUDA, "features_create_csr memset: %s", cudaGetErrorString(e)));
    const unsigned warps_grid = (unsigned)std::min<int64_t>(ceil_div((int64_t)N * 32, 256), 148 * 32);
    k_csr_scatter<<<warps_grid, 256, 0, s>>>(tptr, tidx, tval, N, f->X, f->P);
    count_launch();
  }
  e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return bail(fail(MPH_ECUDA, "features_create_csr build: %s", cudaGetErrorString(e)));
  dev_free(tptr);
  dev_free(tidx);
  dev_free(tval);
  *out = f;
  return MPH_OK;
}

extern "C" int mph_features_info(const mph_features* f, int64_t* nnz_h, int32_t* mode_h, int32_t* is_binary_h) {
  if (!f) return fail(MPH_EINVAL, "null features");
  if (nnz_h) *nnz_h = f->nnz;
  if (mode_h) *mode_h = f->mode;
  if (is_binary_h) *is_binary_h = f->is_binary;
  return MPH_OK;
}

extern "C" int mph_features_csr(const mph_features* f, const int64_t** ptr_d, const int32_t** idx_d, const float** val_d) {
  if (!f) return fail(MPH_EINVAL, "null features");
  if (f->mode != 1) return fail(MPH_ESTATE, "features are in dense mode");
  if (ptr_d) *ptr_d = f->csr_ptr;
  if (idx_d) *idx_d = f->csr_idx;
  if (val_d) *val_d = f->csr_val;
  return MPH_OK;
}

extern "C" int mph_features_csc(const mph_features* f, const int64_t** ptr_d, const int32_t** idx_d, const float** val_d) {
  if (!f) return fail(MPH_EINVAL, "null features");
  if (f->mode != 1) return fail(MPH_ESTATE, "features are in dense mode");
  if (ptr_d) *ptr_d = f->csc_ptr;
  if (idx_d) *idx_d = f->csc_idx;
  if (val_d) *val_d = f->csc_val;
  return MPH_OK;
}

extern "C" int mph_features_dense(const mph_features* f, const float** X_d, int32_t* ld_h) {
  if (!f) return fail(MPH_EINVAL, "null features");
  if (f->mode != 0) return fail(MPH_ESTATE, "features are in sparse mode");
  if (X_d) *X_d = f->X;
  if (ld_h) *ld_h = f->P;
  return MPH_OK;
}

extern "C" int mph_features_destroy(mph_features* f) {
  features_free(f);
  return MPH_OK;
}
