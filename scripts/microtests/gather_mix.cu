// Micro-benchmark: do the TMA gather and the LSU (cp.async) gather draw on
// separate limits?  Same workload as gather_rate.cu (random 64-B rows of a
// 480189-row L2-resident table into a 192 KB ring of 384-row tiles, 148
// persistent CTAs), but each tile's first L rows come by cp.async.cg from
// LW warps (one mbarrier arrival per thread when its copies land, .noinc)
// and the other 384 - L rows by TMA tile::gather4 from G warps.  If the two
// paths have separate ceilings, rows/s rises above the TMA-only ~60 G/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 gather_mix.cu -o gather_mix -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}"
               : "=r"(pred));
  return pred != 0;
}

constexpr int kRows = 384;
constexpr int W = 64;
constexpr int kSlotBytes = 196608;
constexpr int kS = kSlotBytes / (kRows * W);  // 8 slots

template <int G, int LW, int L>
__global__ void __launch_bounds__((G + LW) * 32, 1)
    mix_kernel(const __grid_constant__ CUtensorMap tm, const uint8_t* __restrict__ table,
               const int* rows, int64_t ntiles, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kSlotBytes);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kS; ++s) mbar_init(&full[s], (G > 0 ? G : 0) + LW * 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  constexpr int kTmaRows = kRows - L;
  constexpr int kPer = G > 0 ? kTmaRows / 4 / G : 0;
  static_assert(G == 0 || kTmaRows % (4 * G) == 0, "whole gather4 groups per warp");
  int acc = 0;
  int64_t k = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = (int)(k % kS);
    if (k >= kS) {
      mbar_wait(&full[s], (uint32_t)(((k - kS) / kS) & 1));
      acc += *reinterpret_cast<const int*>(sm + s * kRows * W + threadIdx.x * 4);
      __syncthreads();
    }
    uint8_t* slot = sm + s * kRows * W;
    if (warp < G) {
      const int* r = rows + t * kRows + L + warp * kPer * 4;
      if (elect_one()) {
        expect_tx(&full[s], kPer * 4 * W);
        for (int g = 0; g < kPer; ++g) {
          const int4 q = *reinterpret_cast<const int4*>(r + g * 4);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::"
              "bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
                  su32(slot + (L + (warp * kPer + g) * 4) * W)),
              "l"(&tm), "r"(0), "r"(q.x), "r"(q.y), "r"(q.z), "r"(q.w), "r"(su32(&full[s]))
              : "memory");
        }
      }
      __syncwarp();
    } else {
      const int lt = threadIdx.x - G * 32;
      for (int c = lt; c < L * 4; c += LW * 32) {
        const int rr = c >> 2, ch = c & 3;
        const int g = __ldg(rows + t * kRows + rr);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         su32(slot + rr * W + ((ch ^ ((rr >> 1) & 3)) * 16))),
                     "l"(table + (size_t)g * W + ch * 16)
                     : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s]))
                   : "memory");
    }
  }
  for (int64_t j = k > kS ? k - kS : 0; j < k; ++j)
    mbar_wait(&full[j % kS], (uint32_t)((j / kS) & 1));
  if (acc == 0x7fffffff) sink[0] = acc;
}

template <class F>
float time_it(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault,
                          &q);
  const int nrows = 480189;
  const int64_t n = 99072000;
  std::vector<int> h(n);
  std::mt19937_64 rng(1);
  for (auto& x : h) x = (int)(rng() % nrows);
  const int64_t ntiles = n / kRows;
  uint8_t* table;
  int *rows, *sink;
  cudaMalloc(&table, (size_t)nrows * W);
  cudaMemset(table, 1, (size_t)nrows * W);
  cudaMalloc(&rows, n * 4);
  cudaMalloc(&sink, 4);
  cudaMemcpy(rows, h.data(), n * 4, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[2] = {32, (cuuint64_t)nrows};
  cuuint64_t strides[1] = {W};
  cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, table, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = kSlotBytes + 128;
  auto report = [&](const char* what, float ms) {
    printf("%-34s %8.3f ms  %6.2f Grows/s\n", what, ms, n / ms / 1e6);
  };
#define MIX(G, LW, L)                                                                            \
  {                                                                                              \
    cudaFuncSetAttribute(mix_kernel<G, LW, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    report("tma G=" #G " + lsu warps=" #LW " rows=" #L,                                          \
           time_it([&] { mix_kernel<G, LW, L><<<148, (G + LW) * 32, smem>>>(tm, table, rows, ntiles, sink); })); \
  }
  MIX(2, 0, 0) MIX(4, 0, 0)
  MIX(2, 1, 128) MIX(2, 2, 128) MIX(4, 2, 128) MIX(2, 4, 128)
  MIX(2, 2, 192) MIX(4, 4, 192)
  MIX(2, 1, 64) MIX(2, 2, 64)
  MIX(0, 4, 384) MIX(0, 8, 384)
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
