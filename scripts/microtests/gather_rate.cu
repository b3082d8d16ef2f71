// Micro-benchmark: random-row gather throughput into shared memory, the
// operand path of the sweeps.  Rows of W bytes (64: the core sweep's fp16
// rows, 128: the factor sweep's fp32 rows) from an L2-resident table
// (480189 rows, the Netflix mode-1 shape), 148 persistent CTAs.
//   tma   : TMA tile::gather4 (4 rows per instruction), G issuing warps per
//           CTA (one elected lane each), into a ring of S slots of 128 rows
//   lsu   : cp.async.cg 16 B per thread (W / 16 threads per row), all warps
// Prints rows/s and GB/s; the data is checked on the last slot.  A second
// pass draws each tile's rows from the three Netflix mode sizes (the sweeps'
// actual mix: the two small modes are cache-friendlier).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 gather_rate.cu -o gather_rate -lcuda
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

constexpr int kRows = 384;  // one sweep tile: 3 modes x 128 nonzeros
constexpr int kSlotBytes = 196608;  // ring bytes (192 KB): kS = kSlotBytes / (kRows * W)

// TMA: warps 0..G-1 issue, every warp waits the slot then the whole CTA
// "consumes" it (a __syncthreads) before it is refilled.
template <int W, int G, int kS = kSlotBytes / (kRows * W)>
__global__ void __launch_bounds__(G * 32, 1)
    tma_kernel(const __grid_constant__ CUtensorMap tm, const int* rows, int64_t ntiles, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kSlotBytes);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kS; ++s) mbar_init(&full[s], G);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  constexpr int kPer = kRows / 4 / G;  // gather4 ops per warp per tile
  int acc = 0;
  int64_t k = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = (int)(k % kS);
    if (k >= kS) {  // the slot's previous fill: wait for it, read a word, free it
      mbar_wait(&full[s], (uint32_t)(((k - kS) / kS) & 1));
      acc += *reinterpret_cast<const int*>(sm + s * kRows * W + threadIdx.x * 4);
      __syncthreads();
    }
    const int* r = rows + t * kRows + warp * kPer * 4;
    if (elect_one()) {
      expect_tx(&full[s], kPer * 4 * W);
      for (int g = 0; g < kPer; ++g) {
        const int4 q = *reinterpret_cast<const int4*>(r + g * 4);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::"
            "bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
                su32(sm + s * kRows * W + (warp * kPer + g) * 4 * W)),
            "l"(&tm), "r"(0), "r"(q.x), "r"(q.y), "r"(q.z), "r"(q.w), "r"(su32(&full[s]))
            : "memory");
      }
    }
    __syncwarp();
  }
  for (int64_t j = k > kS ? k - kS : 0; j < k; ++j)
    mbar_wait(&full[j % kS], (uint32_t)((j / kS) & 1));
  if (acc == 0x7fffffff) sink[0] = acc;
}

// LSU: cp.async.cg 16 B per thread, T threads per CTA, kS-deep ring with
// cp.async groups.
template <int W, int T, int kS = kSlotBytes / (kRows * W)>
__global__ void __launch_bounds__(T, 1)
    lsu_kernel(const uint8_t* __restrict__ table, const int* rows, int64_t ntiles, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int kChunks = W / 16, kPerTile = kRows * kChunks;  // 16-B chunks per tile
  int acc = 0;
  int64_t k = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = (int)(k % kS);
    for (int c = threadIdx.x; c < kPerTile; c += T) {
      const int rr = c / kChunks, ch = c - rr * kChunks;
      const int g = __ldg(rows + t * kRows + rr);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                       su32(sm + s * kRows * W + rr * W + ((ch ^ (rr & (kChunks - 1))) * 16))),
                   "l"(table + (size_t)g * W + ch * 16)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(kS - 1) : "memory");
    __syncthreads();
    acc += *reinterpret_cast<const int*>(sm + ((k + 1) % kS) * kRows * W + threadIdx.x * 4);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
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

template <int W>
void run(PFN_cuTensorMapEncodeTiled_v12000 enc, int nrows, const std::vector<int>& h_rows) {
  const int64_t n = (int64_t)h_rows.size(), ntiles = n / kRows;
  uint8_t* table;
  int *rows, *sink;
  cudaMalloc(&table, (size_t)nrows * W);
  cudaMemset(table, 1, (size_t)nrows * W);
  cudaMalloc(&rows, n * 4);
  cudaMalloc(&sink, 4);
  cudaMemcpy(rows, h_rows.data(), n * 4, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  const int elems = W / 2;  // fp16 elements per row
  cuuint64_t dims[2] = {(cuuint64_t)elems, (cuuint64_t)nrows};
  cuuint64_t strides[1] = {(cuuint64_t)W};
  cuuint32_t box[2] = {(cuuint32_t)elems, 1}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, table, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, W == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = kSlotBytes + 64;
  auto report = [&](const char* what, float ms) {
    printf("W=%3d %-18s %8.3f ms  %6.2f Grows/s  %7.1f GB/s\n", W, what, ms, n / ms / 1e6,
           n * (double)W / ms / 1e6);
  };
#define TMA(G)                                                                              \
  {                                                                                         \
    cudaFuncSetAttribute(tma_kernel<W, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    report("tma gather4 G=" #G, time_it([&] { tma_kernel<W, G><<<148, G * 32, smem>>>(tm, rows, ntiles, sink); })); \
  }
  TMA(1) TMA(2) TMA(4) TMA(8)
#define LSU(T)                                                                              \
  {                                                                                         \
    cudaFuncSetAttribute(lsu_kernel<W, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    report("lsu cp.async T=" #T, time_it([&] { lsu_kernel<W, T><<<148, T, smem>>>(table, rows, ntiles, sink); })); \
  }
  LSU(256) LSU(512) LSU(1024)
  printf("  err: %s\n", cudaGetErrorString(cudaGetLastError()));
  cudaFree(table);
  cudaFree(rows);
  cudaFree(sink);
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault,
                          &q);
  const int nrows = 480189;
  const int64_t n = 99072000;  // one mode's rows per sweep
  std::vector<int> h(n);
  std::mt19937_64 rng(1);
  for (auto& x : h) x = (int)(rng() % nrows);
  run<64>(enc, nrows, h);
  run<128>(enc, nrows, h);
  // The sweeps' own mix: each 384-row tile takes 128 rows of each Netflix
  // mode (480189 / 17770 / 2182 rows), laid out as one table of three ranges.
  const int d0 = 480189, d1 = 17770, d2 = 2182;
  for (int64_t t = 0; t < n; t += 384)
    for (int r = 0; r < 384 && t + r < n; ++r)
      h[t + r] = r < 128 ? (int)(rng() % d0)
                         : (r < 256 ? d0 + (int)(rng() % d1) : d0 + d1 + (int)(rng() % d2));
  printf("# Netflix mode mix (128 rows of each mode per tile)\n");
  run<64>(enc, d0 + d1 + d2, h);
  run<128>(enc, d0 + d1 + d2, h);
  return 0;
}
