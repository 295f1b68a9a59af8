// standalone TMA gather4 issue-rate probe: stages of G gathers share one mbarrier
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t by) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(by) : "memory"); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t par) { uint32_t ok; asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su(b)), "r"(par) : "memory"); return ok; }
__device__ __forceinline__ void g4(void* d, const CUtensorMap* m, uint64_t* b, int r0, int r1, int r2, int r3) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
    ::"r"(su(d)), "l"(reinterpret_cast<uint64_t>(m)), "r"(su(b)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory"); }
template <int W, int G, int S>
__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap tm, int nrows, int nstages, float* sink) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t full[S];
  if (threadIdx.x == 0) { for (int i = 0; i < S; ++i) mbar_init(&full[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  if (threadIdx.x != 0) return;
  uint32_t h = 2654435761u * (blockIdx.x + 1);
  for (int i = 0; i < nstages; ++i) {
    const int st = i % S;
    if (i >= S) while (!try_wait(&full[st], ((i / S) - 1) & 1)) {}
    expect(&full[st], G * 4 * W * 4);
    for (int q = 0; q < G; ++q) {
      int r[4];
      for (int k2 = 0; k2 < 4; ++k2) { h ^= h << 13; h ^= h >> 17; h ^= h << 5; r[k2] = (int)(((uint64_t)h * (uint32_t)nrows) >> 32); }
      g4(sm + ((size_t)st * G + q) * 4 * W, &tm, &full[st], r[0], r[1], r[2], r[3]);
    }
  }
  for (int i = nstages; i < nstages + S; ++i) if (i >= S) while (!try_wait(&full[i % S], ((i / S) - 1) & 1)) {}
  sink[blockIdx.x] = sm[0];
}
template <int W, int G, int S, int CTAS>
void run(PFN_cuTensorMapEncodeTiled_v12000 fn, float* t, long rows, float* sink, const char* tag) {
  CUtensorMap tm; cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)rows}; cuuint64_t str[1] = {(cuuint64_t)W * 4};
  cuuint32_t box[2] = {W, 1}, es[2] = {1, 1};
  fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, t, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  size_t smem = (size_t)S * G * 4 * W * 4;
  cudaFuncSetAttribute(k<W, G, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nst = 200000 / G;
  k<W, G, S><<<148 * CTAS, 32, smem>>>(tm, (int)rows, 100, sink); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<W, G, S><<<148 * CTAS, 32, smem>>>(tm, (int)rows, nst, sink); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double bytes = 148.0 * CTAS * nst * G * 4 * W * 4;
  printf("%s W=%d G=%d S=%d ctas/SM=%d: %.3f ms %.0f GB/s  %.1f ns per gather4 per CTA  (%s)\n", tag, W, G, S, CTAS, ms, bytes / ms / 1e6, ms * 1e6 / (nst * (double)G), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  float *small, *big, *sink; long rs = (64L << 20) / 512, rb = (2048L << 20) / 512;
  cudaMalloc(&small, 64L << 20); cudaMalloc(&big, 2048L << 20); cudaMalloc(&sink, 4096 * 4);
  cudaMemset(small, 0, 64L << 20); cudaMemset(big, 0, 2048L << 20);
  run<128, 1, 48, 1>(fn, small, rs, sink, "L2 64MB");
  run<128, 4, 12, 1>(fn, small, rs, sink, "L2 64MB");
  run<128, 8, 6, 1>(fn, small, rs, sink, "L2 64MB");
  run<128, 8, 12, 1>(fn, small, rs, sink, "L2 64MB");
  run<128, 8, 6, 2>(fn, small, rs, sink, "L2 64MB");
  run<128, 8, 3, 4>(fn, small, rs, sink, "L2 64MB");
  run<128, 8, 12, 1>(fn, big, rb, sink, "HBM 2GB");
  run<128, 8, 6, 2>(fn, big, rb, sink, "HBM 2GB");
  run<128, 8, 3, 4>(fn, big, rb, sink, "HBM 2GB");
  run<64, 8, 12, 1>(fn, small, rs * 2, sink, "L2 64MB");
  run<64, 8, 6, 4>(fn, small, rs * 2, sink, "L2 64MB");
  return 0;
}
