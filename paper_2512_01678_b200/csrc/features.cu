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
  dev_free(f->part);
  delete f;
}

}  // namespace mph

using namespace mph;

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
  uint64_t *keys = nullptr, *keys2 = nullptr;
  float* vals2 = nullptr;
  void* tmp = nullptr;
  int rc = MPH_OK;
  auto cleanup = [&]() {
    dev_free(row_nnz);
    dev_free(row_nu);
    dev_free(sums);
    dev_free(keys);
    dev_free(keys2);
    dev_free(vals2);
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
  size_t tb = 0, tb2 = 0, tb3 = 0;
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
  const __int128 lhs = (__int128)10000 * f->nnz, rhs = (__int128)(10000 - tau_bp) * N * F;
  f->mode = force_mode >= 0 ? force_mode : (lhs <= rhs ? 1 : 0);  // S2: s >= tau, decided in integers

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
    if (nnz > 0) {
      if ((rc = dev_alloc(&keys, (size_t)nnz)) || (rc = dev_alloc(&keys2, (size_t)nnz)) ||
          (rc = dev_alloc(&vals2, (size_t)nnz)))
        return bail(rc);
      k_csc_keys<<<warps_grid, 256, 0, s>>>(f->csr_ptr, f->csr_idx, N, keys);
      count_launch();
      cub::DeviceRadixSort::SortPairs(nullptr, tb3, keys, keys2, f->csr_val, f->csc_val, nnz, 0, 64, s);
      dev_free(tmp);
      tmp = nullptr;
      if ((rc = dev_alloc((char**)&tmp, tb3))) return bail(rc);
      e = cub::DeviceRadixSort::SortPairs(tmp, tb3, keys, keys2, f->csr_val, f->csc_val, nnz, 0, 64, s);
      count_launch();
      if (e != cudaSuccess) return cuda_bail(e, "csc sort");
      k_csc_split<<<(unsigned)std::min<int64_t>(ceil_div(nnz, 256), 4096), 256, 0, s>>>(keys2, nnz, f->csc_idx);
      count_launch();
    }
    k_col_ptr<<<(unsigned)ceil_div((int64_t)F + 1, 256), 256, 0, s>>>(keys2 ? keys2 : keys, nnz, F, f->csc_ptr);
    count_launch();
  }
  e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_bail(e, "build");
  if (f->mode == 1) {  // segments of <= kSegNnz nonzeros per CSC column (parallel, ordered dW reduction)
    std::vector<int64_t> cptr((size_t)F + 1);
    e = cudaMemcpy(cptr.data(), f->csc_ptr, cptr.size() * sizeof(int64_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_bail(e, "segments");
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
      return bail(rc);
    e = cudaMemcpy(f->col_seg0, c0.data(), c0.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !sc.empty())
      e = cudaMemcpy(f->seg_col, sc.data(), sc.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !sb.empty())
      e = cudaMemcpy(f->seg_begin, sb.data(), sb.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_bail(e, "segments upload");
  }
  cleanup();
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
