// Micro-test: scattered fp32 row updates (the factor sweep's write-back)
// through RED.v4 with 64-B row segments (the production scheme) versus
// 1-D bulk reductions (cp.reduce.async.bulk .add.f32, one per row, issued
// by the row's lane from shared memory).  Rows of 32 fp32 (J = 32), random
// row indices, every element += 1: the result must equal the per-row count.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#ifndef WIDTH
#define WIDTH 32
#endif
constexpr int W = WIDTH;
constexpr int kBW = W <= 32 ? 4 : 1;  // bulk kernel warps per block (static smem)

__device__ __forceinline__ void red_v4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w) : "memory");
}

__global__ void __launch_bounds__(256) red_kernel(float* a, const int* rows, int64_t n) {
  __shared__ __align__(16) float stage[8][32 * 16];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = ((int64_t)blockIdx.x * 8 + w) * 32; base < n; base += (int64_t)gridDim.x * 256) {
    const int my = base + lane < n ? rows[base + lane] : -1;
    for (int c = 0; c < W / 16; ++c) {
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(&stage[w][lane * 16 + ((q ^ ((lane >> 1) & 3)) * 4)]) =
            make_float4(1.f, 1.f, 1.f, 1.f);
      __syncwarp();
      for (int i = 0; i < 4; ++i) {
        const int rl = i * 8 + (lane >> 2), ch = lane & 3;
        const int g = __shfl_sync(0xffffffffu, my, rl);
        const float4 v = *reinterpret_cast<const float4*>(&stage[w][rl * 16 + ((ch ^ ((rl >> 1) & 3)) * 4)]);
        if (g >= 0) red_v4(a + (size_t)g * W + c * 16 + ch * 4, v);
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kBW * 32) bulk_kernel(float* a, const int* rows, int64_t n) {
  __shared__ __align__(128) float stage[kBW][2][32 * W];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int buf = 0;
  for (int64_t base = ((int64_t)blockIdx.x * kBW + w) * 32; base < n; base += (int64_t)gridDim.x * kBW * 32) {
    // the buffer written two rounds ago must have been read by its bulk ops
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    float* row = &stage[w][buf][lane * W];
    for (int q = 0; q < W / 4; ++q) reinterpret_cast<float4*>(row)[q] = make_float4(1.f, 1.f, 1.f, 1.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int g = base + lane < n ? rows[base + lane] : -1;
    if (g >= 0) {
      const uint32_t s = (uint32_t)__cvta_generic_to_shared(row);
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                   :: "l"(a + (size_t)g * W), "r"(s), "r"(W * 4) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    buf ^= 1;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const int nrows = 480189;
  const int64_t n = 99072112;  // one mode's updates per factor sweep
  std::vector<int> h(n);
  std::mt19937_64 rng(1);
  std::vector<int> cnt(nrows, 0);
  for (int64_t i = 0; i < n; ++i) { h[i] = (int)(rng() % nrows); cnt[h[i]]++; }
  int* d_rows; float* a;
  cudaMalloc(&d_rows, n * 4);
  cudaMalloc(&a, (size_t)nrows * W * 4);
  cudaMemcpy(d_rows, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int k = 0; k < 2; ++k) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(a, 0, (size_t)nrows * W * 4);
      cudaEventRecord(e0);
      if (k == 0) red_kernel<<<148 * 8, 256>>>(a, d_rows, n);
      else bulk_kernel<<<148 * 32 / kBW, kBW * 32>>>(a, d_rows, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      std::vector<float> out((size_t)nrows * W);
      cudaMemcpy(out.data(), a, out.size() * 4, cudaMemcpyDeviceToHost);
      int64_t bad = 0;
      for (int r = 0; r < nrows; ++r)
        for (int j = 0; j < W; ++j) bad += out[(size_t)r * W + j] != (float)cnt[r];
      printf("%s: %.3f ms (%.1f GB/s of updates), mismatches %lld, err %s\n",
             k == 0 ? "RED.v4 64-B segments" : "bulk reduce per row", ms,
             n * W * 4 / ms / 1e6, (long long)bad, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // both paths at once, half of the updates each (two streams)
  {
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(a, 0, (size_t)nrows * W * 4);
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      cudaStreamWaitEvent(s1, e0, 0);
      cudaStreamWaitEvent(s2, e0, 0);
      red_kernel<<<148 * 4, 256, 0, s1>>>(a, d_rows, n / 2);
      bulk_kernel<<<148 * 16 / kBW, kBW * 32, 0, s2>>>(a, d_rows + n / 2, n - n / 2);
      cudaEvent_t d1, d2;
      cudaEventCreate(&d1); cudaEventCreate(&d2);
      cudaEventRecord(d1, s1); cudaEventRecord(d2, s2);
      cudaStreamWaitEvent(0, d1, 0); cudaStreamWaitEvent(0, d2, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      std::vector<float> out((size_t)nrows * W);
      cudaMemcpy(out.data(), a, out.size() * 4, cudaMemcpyDeviceToHost);
      int64_t bad = 0;
      for (int r = 0; r < nrows; ++r)
        for (int j = 0; j < W; ++j) bad += out[(size_t)r * W + j] != (float)cnt[r];
      printf("RED + bulk concurrently: %.3f ms (%.1f GB/s of updates), mismatches %lld\n", ms,
             n * W * 4 / ms / 1e6, (long long)bad);
    }
  }
  return 0;
}
