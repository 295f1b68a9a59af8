// a5 loss, a9 Adam, Xavier init, weight transposes, and the sparse-feature kernels of the
// density switch (a2 sparse X_csr·W, a7 sparse X_csc^T·G).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

#include "internal.cuh"

namespace mph {

// ------------------------------------------------------------------ a5 softmax cross-entropy
// Reading Q9: max-subtracted log-sum-exp over the first C columns, mean over the
// labelled rows (global count n_lab), dZ = (softmax - onehot)/n_lab.  Warp per row;
// each block accumulates its rows' loss (double) and column sums of dZ in a fixed order and
// writes one partial; a single-block pass reduces the partials in block order.
constexpr int kCeThreads = 256;
constexpr int kCeMaxC = 256;

static int ce_grid(int N) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(N, 64), 148 * 8)); }

// Warp per row, R rows per warp iteration with all their loads issued first (latency hiding);
// NJ = ceil(C/32) columns chunks per lane.
template <int NJ>
__global__ void __launch_bounds__(kCeThreads) k_softmax_ce(const float* Z, int N, int C, int ld, const int32_t* labels,
                                                           const uint8_t* mask, float inv_nlab, const float* row_scale,
                                                           float* dZ, int ld_dz, double* part_loss, float* part_db,
                                                           int round_tf32) {
  constexpr int R = NJ <= 2 ? 4 : (NJ <= 4 ? 2 : 1);
  __shared__ double s_loss[kCeThreads / 32];
  __shared__ float s_db[kCeThreads / 32][kCeMaxC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float dbacc[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) dbacc[j] = 0.0f;
  double lacc = 0.0;
  const int wpb = kCeThreads / 32;
  const int stride = gridDim.x * wpb;
  for (int i0 = blockIdx.x * wpb + warp; i0 < N; i0 += stride * R) {
    float zv[R][NJ];
    int yv[R];
    float rsv[R];
    bool labv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = i0 + r * stride;
      const bool ok = i < N;
      const float* z = Z + (int64_t)(ok ? i : 0) * ld;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int c = lane + 32 * j;
        zv[r][j] = (ok && c < C) ? __ldg(z + c) : -INFINITY;
      }
      yv[r] = ok ? __ldg(labels + i) : 0;
      rsv[r] = (ok && row_scale) ? __ldg(row_scale + i) : 1.0f;
      labv[r] = ok && (mask ? (mask[i] != 0) : true);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = i0 + r * stride;
      if (i >= N) continue;
      float* dz = dZ + (int64_t)i * ld_dz;
      if (!labv[r]) {
#pragma unroll
        for (int j = 0; j < NJ; ++j)
          if (lane + 32 * j < C) dz[lane + 32 * j] = 0.0f;
        continue;
      }
      float m = -INFINITY;
#pragma unroll
      for (int j = 0; j < NJ; ++j) m = fmaxf(m, zv[r][j]);
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      float se = 0.0f;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        if (lane + 32 * j < C) se += expf(zv[r][j] - m);
#pragma unroll
      for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
      const float lse = m + logf(se);
      const int y = yv[r];
      float zy = 0.0f;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int c = lane + 32 * j;
        if (c < C) {
          if (c == y) zy = zv[r][j];
          const float g = (expf(zv[r][j] - lse) - (c == y ? 1.0f : 0.0f)) * inv_nlab;
          dbacc[j] += g;
          dz[c] = round_tf32 ? tf32_rna(g * rsv[r]) : g * rsv[r];
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) zy += __shfl_xor_sync(0xffffffffu, zy, o);
      lacc += (double)lse - (double)zy;
    }
  }
  if (lane == 0) s_loss[warp] = lacc;
#pragma unroll
  for (int j = 0; j < NJ; ++j)
    if (lane + 32 * j < C) s_db[warp][lane + 32 * j] = dbacc[j];
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < wpb; ++w) t += s_loss[w];
    part_loss[blockIdx.x] = t;
  }
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float t = 0.0f;
    for (int w = 0; w < wpb; ++w) t += s_db[w][c];
    part_db[(int64_t)blockIdx.x * C + c] = t;
  }
}

// Vectorised variant (ld, ld_dz multiples of 4, 16-byte aligned rows): LPR lanes x VPL float4
// cover a row, 32/LPR rows per warp at once, so a 47-class row is 4 lanes x 3 float4 and no lane
// idles; exp is evaluated once per element (exp2 of the log2e-scaled shifted logit) and reused
// for the sum and the gradient.  Same partial layout as k_softmax_ce (fixed-order reductions).
template <int LPR, int VPL>
__global__ void __launch_bounds__(kCeThreads) k_softmax_ce4(const float* __restrict__ Z, int N, int C, int ld,
                                                            const int32_t* __restrict__ labels,
                                                            const uint8_t* __restrict__ mask, float inv_nlab,
                                                            const float* __restrict__ row_scale, float* __restrict__ dZ,
                                                            int ld_dz, double* part_loss, float* part_db,
                                                            int round_tf32) {
  constexpr int SPW = 32 / LPR;  // rows per warp step
  constexpr float kLog2e = 1.4426950408889634f;
  __shared__ double s_loss[kCeThreads / 32];
  __shared__ float s_db[kCeThreads / 32][kCeMaxC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = lane / LPR, sub = lane % LPR;
  const int nv4 = (C + 3) >> 2;
  float4 dbacc[VPL];
#pragma unroll
  for (int j = 0; j < VPL; ++j) dbacc[j] = f4_zero();
  double lacc = 0.0;
  const int64_t gw = (int64_t)blockIdx.x * (kCeThreads / 32) + warp;
  const int64_t nw = (int64_t)gridDim.x * (kCeThreads / 32);
  for (int64_t i = gw * SPW + slot; i - slot < N; i += nw * SPW) {
    const bool ok = i < N;
    const int64_t r = ok ? i : 0;
    float4 z[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c4 = sub + j * LPR;
      z[j] = (ok && c4 < nv4) ? __ldg(reinterpret_cast<const float4*>(Z + r * ld) + c4)
                              : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      if (4 * c4 + 3 >= C) {  // columns >= C of the last float4 are padding
        if (4 * c4 + 1 >= C) z[j].y = -INFINITY;
        if (4 * c4 + 2 >= C) z[j].z = -INFINITY;
        if (4 * c4 + 3 >= C) z[j].w = -INFINITY;
        if (4 * c4 >= C) z[j].x = -INFINITY;
      }
    }
    const int y = ok ? __ldg(labels + r) : -1;
    const float rsv = (ok && row_scale) ? __ldg(row_scale + r) : 1.0f;
    const bool lab = ok && (mask ? (__ldg(mask + r) != 0) : true);
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < VPL; ++j) m = fmaxf(m, fmaxf(fmaxf(z[j].x, z[j].y), fmaxf(z[j].z, z[j].w)));
#pragma unroll
    for (int o = 1; o < LPR; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float ms = ok ? m * kLog2e : 0.0f;
    float4 ex[VPL];
    float se = 0.0f, zy = 0.0f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      ex[j].x = exp2f(fmaf(z[j].x, kLog2e, -ms));
      ex[j].y = exp2f(fmaf(z[j].y, kLog2e, -ms));
      ex[j].z = exp2f(fmaf(z[j].z, kLog2e, -ms));
      ex[j].w = exp2f(fmaf(z[j].w, kLog2e, -ms));
      se += (ex[j].x + ex[j].y) + (ex[j].z + ex[j].w);
      const int c0 = 4 * (sub + j * LPR);
      if (y >= c0 && y < c0 + 4) zy = y == c0 ? z[j].x : (y == c0 + 1 ? z[j].y : (y == c0 + 2 ? z[j].z : z[j].w));
    }
#pragma unroll
    for (int o = 1; o < LPR; o <<= 1) {
      se += __shfl_xor_sync(0xffffffffu, se, o);
      zy += __shfl_xor_sync(0xffffffffu, zy, o);
    }
    if (!ok) continue;
    float4* dz = reinterpret_cast<float4*>(dZ + r * ld_dz);
    if (!lab) {
#pragma unroll
      for (int j = 0; j < VPL; ++j)
        if (sub + j * LPR < nv4) dz[sub + j * LPR] = f4_zero();
      continue;
    }
    const float inv_se = 1.0f / se;
    if (sub == 0) lacc += (double)(m + logf(se)) - (double)zy;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c4 = sub + j * LPR;
      if (c4 >= nv4) continue;
      const int c0 = 4 * c4;
      float4 g;
      g.x = (ex[j].x * inv_se - (y == c0 ? 1.0f : 0.0f)) * inv_nlab;
      g.y = (ex[j].y * inv_se - (y == c0 + 1 ? 1.0f : 0.0f)) * inv_nlab;
      g.z = (ex[j].z * inv_se - (y == c0 + 2 ? 1.0f : 0.0f)) * inv_nlab;
      g.w = (ex[j].w * inv_se - (y == c0 + 3 ? 1.0f : 0.0f)) * inv_nlab;
      dbacc[j] = f4_add(dbacc[j], g);
      g = make_float4(g.x * rsv, g.y * rsv, g.z * rsv, g.w * rsv);
      dz[c4] = round_tf32 ? f4_tf32(g) : g;
    }
  }
  // fixed-order reductions: slots of the warp by an xor tree, then warps in order
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) {
    lacc += __shfl_xor_sync(0xffffffffu, lacc, o);
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      dbacc[j].x += __shfl_xor_sync(0xffffffffu, dbacc[j].x, o);
      dbacc[j].y += __shfl_xor_sync(0xffffffffu, dbacc[j].y, o);
      dbacc[j].z += __shfl_xor_sync(0xffffffffu, dbacc[j].z, o);
      dbacc[j].w += __shfl_xor_sync(0xffffffffu, dbacc[j].w, o);
    }
  }
  if (lane == 0) s_loss[warp] = lacc;
  if (slot == 0) {
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c0 = 4 * (sub + j * LPR);
      if (c0 + 0 < C) s_db[warp][c0 + 0] = dbacc[j].x;
      if (c0 + 1 < C) s_db[warp][c0 + 1] = dbacc[j].y;
      if (c0 + 2 < C) s_db[warp][c0 + 2] = dbacc[j].z;
      if (c0 + 3 < C) s_db[warp][c0 + 3] = dbacc[j].w;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kCeThreads / 32; ++w) t += s_loss[w];
    part_loss[blockIdx.x] = t;
  }
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float t = 0.0f;
    for (int w = 0; w < kCeThreads / 32; ++w) t += s_db[w][c];
    part_db[(int64_t)blockIdx.x * C + c] = t;
  }
}

// Block c < C reduces column c of the block partials, block C the loss; strided per-thread sums
// then a fixed smem tree (deterministic).
__global__ void __launch_bounds__(256) k_ce_finish(const double* part_loss, const float* part_db, int parts, int C,
                                                   double inv_nlab, double* loss, float* db) {
  __shared__ double sd[256];
  const int t = threadIdx.x;
  double acc = 0.0;
  if ((int)blockIdx.x == C) {
    for (int b = t; b < parts; b += 256) acc += part_loss[b];
  } else {
    if (!db) return;
    float f = 0.0f;
    for (int b = t; b < parts; b += 256) f += part_db[(int64_t)b * C + blockIdx.x];
    acc = f;
  }
  sd[t] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (t < o) sd[t] += sd[t + o];
    __syncthreads();
  }
  if (t == 0) {
    if ((int)blockIdx.x == C)
      *loss = sd[0] * inv_nlab;
    else
      db[blockIdx.x] = (float)sd[0];
  }
}

size_t softmax_ce_ws_bytes(int N, int C) {
  const int g = ce_grid(std::max(N, 1));
  return (size_t)g * sizeof(double) + (size_t)g * std::max(C, 1) * sizeof(float) + 16;
}

int softmax_ce_launch(const float* Z, int N, int C, int ld, const int32_t* labels, const uint8_t* mask, int64_t n_lab,
                      const float* row_scale, float* dZ, int ld_dz, float* db, double* loss, void* ws, size_t ws_bytes,
                      cudaStream_t s, int round_tf32) {
  if (!Z || !labels || !dZ || !loss || N < 0 || C <= 0 || ld < C || ld_dz < C || n_lab <= 0)
    return fail(MPH_EINVAL, "softmax_ce: bad arguments");
  if (C > kCeMaxC) return fail(MPH_ENOTSUP, "softmax_ce: C=%d > %d", C, kCeMaxC);
  if (!ws || ws_bytes < softmax_ce_ws_bytes(N, C)) return fail(MPH_EINVAL, "softmax_ce: workspace too small");
  const int g = ce_grid(std::max(N, 1));
  double* part_loss = reinterpret_cast<double*>(ws);
  float* part_db = reinterpret_cast<float*>(part_loss + g);
  const float inv = (float)(1.0 / (double)n_lab);
  const bool vec = ld % 4 == 0 && ld_dz % 4 == 0 &&
                   ((reinterpret_cast<uintptr_t>(Z) | reinterpret_cast<uintptr_t>(dZ)) & 15) == 0;
  const int nv4 = (C + 3) / 4;
#define CE4(LPR, VPL) \
  k_softmax_ce4<LPR, VPL><<<g, kCeThreads, 0, s>>>(Z, N, C, ld, labels, mask, inv, row_scale, dZ, ld_dz, part_loss, \
                                                    part_db, round_tf32)
  if (vec && nv4 <= 1) CE4(1, 1);
  else if (vec && nv4 <= 2) CE4(2, 1);
  else if (vec && nv4 <= 4) CE4(4, 1);
  else if (vec && nv4 <= 8) CE4(8, 1);
  else if (vec && nv4 <= 12) CE4(4, 3);
  else if (vec && nv4 <= 16) CE4(16, 1);
  else if (vec && nv4 <= 32) CE4(32, 1);
  else if (vec && nv4 <= 64) CE4(32, 2);
#undef CE4
  else switch ((C + 31) / 32) {
#define CE_CASE(NJ)                                                                                              \
  case NJ:                                                                                                       \
    k_softmax_ce<NJ><<<g, kCeThreads, 0, s>>>(Z, N, C, ld, labels, mask, inv, row_scale, dZ, ld_dz, part_loss, \
                                              part_db, round_tf32);                                              \
    break;
    CE_CASE(1) CE_CASE(2) CE_CASE(3) CE_CASE(4) CE_CASE(5) CE_CASE(6) CE_CASE(7) CE_CASE(8)
#undef CE_CASE
  }
  k_ce_finish<<<C + 1, 256, 0, s>>>(part_loss, part_db, g, C, 1.0 / (double)n_lab, loss, db);
  count_launch(2);
  return launch_check("softmax_ce");
}

// ------------------------------------------------------------------ a9 Adam
// Bias corrections are computed on the device from t (host value, or device counter during a
// CUDA-graph replay), so eager and graph epochs are bitwise identical.
__global__ void k_optim(float* __restrict__ p, float* __restrict__ g, float* __restrict__ m,
                        float* __restrict__ v, int64_t n, int kind, float lr, float b1, float b2, float eps, float wd,
                        float mu, int t_host, const int32_t* t_dev, const float* __restrict__ gsum, int world,
                        const uint64_t* flags_grad, const int64_t* gen_dev, int* err) {
  const int t = t_dev ? *t_dev : t_host;
  float bc1 = 1.0f, bc2 = 1.0f;
  if (kind != MPH_OPT_SGD) {
    bc1 = (float)(1.0 - pow((double)b1, (double)t));
    bc2 = (float)(1.0 - pow((double)b2, (double)t));
  }
  if (gsum) {  // NEXT-1: every rank's slab of this generation has landed (p2p.cu)
    __shared__ int ok;
    if (threadIdx.x == 0) ok = p2p_wait_all(flags_grad, world, (uint64_t)*gen_dev, err);
    __syncthreads();
    if (!ok) return;
    gsum += (*gen_dev & 1) * world * n;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float gi;
    if (gsum) {  // the all-reduce: slabs summed in rank order, the same bits on every rank
      gi = __ldcg(gsum + i);
      for (int q = 1; q < world; ++q) gi += __ldcg(gsum + (int64_t)q * n + i);
      g[i] = gi;
    } else {
      gi = g[i];
    }
    if (kind == MPH_OPT_SGD) {  // d = g + wd·p; m = μ·m + d (μ > 0); p -= lr·d   (R8)
      float d = wd != 0.0f ? gi + wd * p[i] : gi;
      if (mu != 0.0f) {
        d = mu * m[i] + d;
        m[i] = d;
      }
      p[i] -= lr * d;
      continue;
    }
    float pi = p[i];
    if (kind == MPH_OPT_ADAMW) pi -= lr * wd * pi;  // decoupled weight decay before the update
    const float mi = b1 * m[i] + (1.0f - b1) * gi;
    const float vi = b2 * v[i] + (1.0f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] = pi - lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
  }
}

static int optim_check(const float* p, const float* g, const float* m, const float* v, int64_t n,
                       const mph_optim_cfg* cfg, int t, const int32_t* t_dev) {
  if (!p || !g || !cfg || n < 0 || (t < 1 && !t_dev) || cfg->kind < MPH_OPT_ADAM || cfg->kind > MPH_OPT_ADAMW)
    return fail(MPH_EINVAL, "optim: bad arguments");
  if (cfg->kind != MPH_OPT_SGD && (!m || !v)) return fail(MPH_EINVAL, "optim: Adam/AdamW need m and v");
  if (cfg->kind == MPH_OPT_SGD && cfg->momentum != 0.0f && !m) return fail(MPH_EINVAL, "optim: momentum needs m");
  return MPH_OK;
}

int optim_launch(float* p, const float* g, float* m, float* v, int64_t n, const mph_optim_cfg* cfg, int t,
                 cudaStream_t s, const int32_t* t_dev) {
  MPH_TRY(optim_check(p, g, m, v, n, cfg, t, t_dev));
  if (n == 0) return MPH_OK;
  const float wd = cfg->kind == MPH_OPT_ADAM ? 0.0f : cfg->weight_decay;
  const float mu = cfg->kind == MPH_OPT_SGD ? cfg->momentum : 0.0f;
  k_optim<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 8), 256, 0, s>>>(
      p, const_cast<float*>(g), m, v, n, cfg->kind, cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, wd, mu, t, t_dev,
      nullptr, 1, nullptr, nullptr, nullptr);
  count_launch();
  return launch_check("optim");
}

int optim_sum_launch(float* p, float* grads, float* m, float* v, int64_t n, const mph_optim_cfg* cfg, int t,
                     cudaStream_t s, const int32_t* t_dev, const float* gsum, int world, const uint64_t* flags_grad,
                     const int64_t* gen_dev, int* err) {
  MPH_TRY(optim_check(p, grads, m, v, n, cfg, t, t_dev));
  if (!gsum || !flags_grad || !gen_dev || !err || world < 1) return fail(MPH_EINVAL, "optim_sum: bad arguments");
  if (n == 0) return MPH_OK;
  const float wd = cfg->kind == MPH_OPT_ADAM ? 0.0f : cfg->weight_decay;
  const float mu = cfg->kind == MPH_OPT_SGD ? cfg->momentum : 0.0f;
  k_optim<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 4), 256, 0, s>>>(
      p, grads, m, v, n, cfg->kind, cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, wd, mu, t, t_dev, gsum, world,
      flags_grad, gen_dev, err);
  count_launch();
  return launch_check("optim (fused gradient sum)");
}

int adam_launch(float* p, const float* g, float* m, float* v, int64_t n, const mph_adam_cfg* cfg, int t, cudaStream_t s,
                const int32_t* t_dev) {
  if (!cfg) return fail(MPH_EINVAL, "adam: bad arguments");
  const mph_optim_cfg o{MPH_OPT_ADAM, cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, 0.0f, 0.0f};
  return optim_launch(p, g, m, v, n, &o, t, s, t_dev);
}

// ------------------------------------------------------------------ Xavier (Q16)
__global__ void k_xavier(float* W, int f_in, int f_out, int ld, uint64_t seed_l, double a) {
  const int64_t total = (int64_t)f_in * f_out;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed_l + (uint64_t)(k + 1) * 0x9E3779B97F4A7C15ull;  // k-th splitmix64 state
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    const double u24 = (double)(z >> 40);
    const double t = __dadd_rn(__ddiv_rn(__dmul_rn(2.0, u24), 16777216.0), -1.0);
    const int64_t i = k / f_out, j = k - i * f_out;
    W[i * ld + j] = __double2float_rn(__dmul_rn(a, t));
  }
}

int xavier_launch(float* W, int f_in, int f_out, int ld, uint64_t seed, int layer, cudaStream_t s) {
  if (!W || f_in <= 0 || f_out <= 0 || ld < f_out || layer < 1) return fail(MPH_EINVAL, "xavier: bad arguments");
  const uint64_t seed_l = seed ^ ((uint64_t)layer * 0x9E3779B97F4A7C15ull);
  const double a = std::sqrt(6.0 / (double)(f_in + f_out));
  const int64_t total = (int64_t)f_in * f_out;
  k_xavier<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 4096), 256, 0, s>>>(W, f_in, f_out, ld, seed_l, a);
  count_launch();
  return launch_check("xavier");
}

// ------------------------------------------------------------------ weight copies / row scale
// The tensor-core operand copies of W_l: dst_t = round_tf32(W^T) (K-major B of the forward
// GEMM) and dst_r = round_tf32(W) (B of the dH GEMM).  The FP32 master copy stays in params.
// BF: the copies are bfloat16 (dst_t / dst_r hold uint16, ld in elements) for BF16 GEMMs.
template <bool BF>
__global__ void k_weight_copies(const float* src, int rows, int cols, int ld_src, void* dst_t, int ld_t, void* dst_r,
                                int ld_r) {
  __shared__ float tile[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    const float x = (r < rows && c < cols) ? src[(int64_t)r * ld_src + c] : 0.0f;
    const float v = BF ? x : tf32_rna(x);
    tile[i][threadIdx.x] = v;
    if (dst_r && r < rows && c < cols) {
      if (BF)
        static_cast<uint16_t*>(dst_r)[(int64_t)r * ld_r + c] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
      else
        static_cast<float*>(dst_r)[(int64_t)r * ld_r + c] = v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows) {
      if (BF)
        static_cast<uint16_t*>(dst_t)[(int64_t)c * ld_t + r] = __bfloat16_as_ushort(__float2bfloat16_rn(tile[threadIdx.x][i]));
      else
        static_cast<float*>(dst_t)[(int64_t)c * ld_t + r] = tile[threadIdx.x][i];
    }
  }
}

int weight_copies_launch(const float* src, int rows, int cols, int ld_src, float* dst_t, int ld_t, float* dst_r,
                         int ld_r, cudaStream_t s, bool bf16) {
  if (rows <= 0 || cols <= 0) return MPH_OK;
  dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
  if (bf16)
    k_weight_copies<true><<<grid, dim3(32, 8), 0, s>>>(src, rows, cols, ld_src, dst_t, ld_t, dst_r, ld_r);
  else
    k_weight_copies<false><<<grid, dim3(32, 8), 0, s>>>(src, rows, cols, ld_src, dst_t, ld_t, dst_r, ld_r);
  count_launch();
  return launch_check("weight_copies");
}

// out[i][c] = in[i][c] * scale[i] (scale nullable), optionally rounded to TF32
__global__ void k_rowscale(const float* in, int ld_in, const float* scale, int rows, int w, float* out, int ld_out,
                           int round) {
  const int64_t total = (int64_t)rows * w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / w;
    const int c = (int)(t - i * w);
    float v = in[i * ld_in + c];
    if (scale) v *= scale[i];
    if (round == 2)  // bfloat16 output (BF16 GEMM operand copy)
      reinterpret_cast<uint16_t*>(out)[i * ld_out + c] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
    else
      out[i * ld_out + c] = round ? tf32_rna(v) : v;
  }
}

int rowscale_launch(const float* in, int ld_in, const float* scale, int rows, int w, float* out, int ld_out, int round,
                    cudaStream_t s) {
  if (rows <= 0 || w <= 0) return MPH_OK;
  const int64_t total = (int64_t)rows * w;
  k_rowscale<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 32), 256, 0, s>>>(in, ld_in, scale, rows, w,
                                                                                          out, ld_out, round);
  count_launch();
  return launch_check("rowscale");
}

// ------------------------------------------------------------------ sparse-feature path
// a2 (Alg. 1 Forward SpMM_Tiled(X_csr, W); CPU original keeps W blocks in L1,
// P:228): warp per row of X; the row's nonzeros are read 32 at a time and broadcast; lanes
// cover the output columns; W rows are re-read from L1/L2 (W is at most 128 KB here).
__global__ void k_sparse_xw(const int64_t* ptr, const int32_t* idx, const float* val, int N, const float* W, int F_out,
                            int ldw, const float* row_scale, float* T, int ldt) {
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += nwarps) {
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
    const int64_t s = ptr[i], e = ptr[i + 1];
    for (int64_t b = s; b < e; b += 32) {
      const int nb = (int)min((int64_t)32, e - b);
      const int kk = lane < nb ? idx[b + lane] : 0;
      const float xx = lane < nb ? val[b + lane] : 0.0f;
      for (int t = 0; t < nb; t += 4) {  // four independent W-row loads in flight
        float w[4][8];
        float x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = __shfl_sync(0xffffffffu, kk, (t + u) & 31);
          x[u] = t + u < nb ? __shfl_sync(0xffffffffu, xx, (t + u) & 31) : 0.0f;
          const float* wr = W + (int64_t)k * ldw;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = lane + 32 * j;
            w[u][j] = (c < F_out && t + u < nb) ? __ldg(wr + c) : 0.0f;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] = fmaf(x[u], w[u][j], acc[j]);
      }
    }
    const float rs = row_scale ? row_scale[i] : 1.0f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = lane + 32 * j;
      if (c < F_out) T[(int64_t)i * ldt + c] = acc[j] * rs;
    }
  }
}

// a7 (Alg. 1 Backward SpMM_Col(X_csc, G); "thread-local buffers before a final
// reduction" without atomics): each column of X is cut into segments of at most
// kSegNnz nonzeros (built once per feature set); a warp per segment gathers the G rows of its
// nonzeros into a partial row, then the partials of each column are summed in segment order.
__global__ void k_sparse_xtg_seg(const int32_t* seg_col, const int64_t* seg_begin, const int64_t* cptr,
                                 const int32_t* ridx, const float* cval, int64_t n_seg, const float* G, int F_out,
                                 int ldg, float* part) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t sg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sg < n_seg; sg += nwarps) {
    const int k = seg_col[sg];
    const int64_t s = seg_begin[sg], e = min(cptr[k + 1], s + kSegNnz);
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
    for (int64_t b = s; b < e; b += 32) {
      const int nb = (int)min((int64_t)32, e - b);
      const int ii = lane < nb ? ridx[b + lane] : 0;
      const float xx = lane < nb ? cval[b + lane] : 0.0f;
      for (int t = 0; t < nb; t += 4) {
        float g[4][8];
        float x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = __shfl_sync(0xffffffffu, ii, (t + u) & 31);
          x[u] = t + u < nb ? __shfl_sync(0xffffffffu, xx, (t + u) & 31) : 0.0f;
          const float* gr = G + (int64_t)i * ldg;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = lane + 32 * j;
            g[u][j] = (c < F_out && t + u < nb) ? __ldg(gr + c) : 0.0f;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] = fmaf(x[u], g[u][j], acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = lane + 32 * j;
      if (c < F_out) part[sg * F_out + c] = acc[j];
    }
  }
}

__global__ void k_sparse_xtg_sum(const int64_t* col_seg0, int F, const float* part, int F_out, float* dW, int lddw) {
  const int64_t total = (int64_t)F * F_out;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t / F_out;
    const int c = (int)(t - k * F_out);
    float acc = 0.0f;
    for (int64_t sg = col_seg0[k]; sg < col_seg0[k + 1]; ++sg) acc += part[sg * F_out + c];
    dW[k * lddw + c] = acc;
  }
}

int sparse_xw_launch(const mph_features* f, const float* W, int F_out, int ldw, const float* row_scale, float* T,
                     int ldt, cudaStream_t s) {
  if (!f || !W || !T || F_out <= 0 || ldw < F_out || ldt < F_out) return fail(MPH_EINVAL, "sparse_xw: bad arguments");
  if (f->mode != 1) return fail(MPH_ESTATE, "sparse_xw: features are in dense mode");
  if (F_out > 256) return fail(MPH_ENOTSUP, "sparse_xw: F_out > 256");
  if (F_out % 4 == 0 && ldw % 4 == 0 && ldt % 4 == 0 &&
      !((reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(T)) & 15))  // float4 gather kernel
    return spmm_csr_launch(f->csr_ptr, f->csr_idx, f->is_binary ? nullptr : f->csr_val, f->N, f->xw_items,
                           f->xw_n_items, f->item_counter, row_scale, W, F_out, ldw, T, ldt, s);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(f->N, 8), 148 * 16));
  k_sparse_xw<<<grid, 256, 0, s>>>(f->csr_ptr, f->csr_idx, f->csr_val, f->N, W, F_out, ldw, row_scale, T, ldt);
  count_launch();
  return launch_check("sparse_xw");
}

int sparse_xtg_launch(const mph_features* fc, const float* G, int F_out, int ldg, float* dW, int lddw, cudaStream_t s) {
  if (!fc || !G || !dW || F_out <= 0 || ldg < F_out || lddw < F_out) return fail(MPH_EINVAL, "sparse_xtg: bad arguments");
  if (fc->mode != 1) return fail(MPH_ESTATE, "sparse_xtg: features are in dense mode");
  if (F_out > 256) return fail(MPH_ENOTSUP, "sparse_xtg: F_out > 256");
  mph_features* f = const_cast<mph_features*>(fc);
  const size_t need = (size_t)std::max<int64_t>(f->n_seg, 1) * F_out;
  if (need > f->part_cap) {  // partial rows: grows once, outside the steady state
    dev_free(f->part);
    f->part = nullptr;
    f->part_cap = 0;
    MPH_TRY(dev_alloc(&f->part, need));
    f->part_cap = need;
  }
  if (f->n_seg > 0) {
    if (F_out % 4 == 0 && ldg % 4 == 0 && !(reinterpret_cast<uintptr_t>(G) & 15)) {  // float4 gather kernel
      MPH_TRY(spmm_csr_launch(f->seg_ptr, f->csc_idx, f->is_binary ? nullptr : f->csc_val, (int)f->n_seg,
                              f->xtg_items, f->xtg_n_items, f->item_counter, nullptr, G, F_out, ldg, f->part, F_out,
                              s));
    } else {
      const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(f->n_seg, 8), 148 * 16));
      k_sparse_xtg_seg<<<grid, 256, 0, s>>>(f->seg_col, f->seg_begin, f->csc_ptr, f->csc_idx, f->csc_val, f->n_seg,
                                            G, F_out, ldg, f->part);
      count_launch();
    }
  }
  const int64_t total = (int64_t)f->F * F_out;
  k_sparse_xtg_sum<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 148 * 16)), 256, 0, s>>>(
      f->col_seg0, f->F, f->part, F_out, dW, lddw);
  count_launch();
  return launch_check("sparse_xtg");
}

}  // namespace mph

using namespace mph;

extern "C" int mph_softmax_ce_workspace(int32_t N, int32_t C, size_t* bytes_h) {
  if (!bytes_h) return fail(MPH_EINVAL, "null bytes");
  *bytes_h = softmax_ce_ws_bytes(N, C);
  return MPH_OK;
}

extern "C" int mph_softmax_ce(const float* Z_d, int32_t N, int32_t C, int32_t ld, const int32_t* labels_d,
                              const uint8_t* mask_d, int64_t n_lab, const float* row_scale_d, float* dZ_d, int32_t ld_dz,
                              float* db_d, double* loss_d, void* ws_d, size_t ws_bytes, void* stream) {
  return softmax_ce_launch(Z_d, N, C, ld, labels_d, mask_d, n_lab, row_scale_d, dZ_d, ld_dz, db_d, loss_d, ws_d,
                           ws_bytes, (cudaStream_t)stream);
}

extern "C" int mph_adam(float* params_d, const float* grads_d, float* m_d, float* v_d, int64_t n, const mph_adam_cfg* cfg,
                        int32_t t, void* stream) {
  return adam_launch(params_d, grads_d, m_d, v_d, n, cfg, t, (cudaStream_t)stream);
}

extern "C" int mph_optim_step(float* params_d, const float* grads_d, float* m_d, float* v_d, int64_t n,
                              const mph_optim_cfg* cfg, int32_t t, void* stream) {
  return optim_launch(params_d, grads_d, m_d, v_d, n, cfg, t, (cudaStream_t)stream);
}

extern "C" int mph_xavier_fill(float* W_d, int32_t f_in, int32_t f_out, int32_t ld, uint64_t seed, int32_t layer,
                               void* stream) {
  return xavier_launch(W_d, f_in, f_out, ld, seed, layer, (cudaStream_t)stream);
}

extern "C" int mph_sparse_xw(const mph_features* f, const float* W_d, int32_t F_out, int32_t ldw,
                             const float* row_scale_d, float* T_d, int32_t ldt, void* stream) {
  return sparse_xw_launch(f, W_d, F_out, ldw, row_scale_d, T_d, ldt, (cudaStream_t)stream);
}

extern "C" int mph_sparse_xtg(const mph_features* f, const float* G_d, int32_t F_out, int32_t ldg, float* dW_d,
                              int32_t lddw, void* stream) {
  return sparse_xtg_launch(f, G_d, F_out, ldg, dW_d, lddw, (cudaStream_t)stream);
}
