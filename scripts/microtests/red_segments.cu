// Micro-test: scattered fp32 row updates (the factor sweep's write-back) by
// RED.v4 (red.global.add.v4.f32, 16 B per lane), with S lanes per row in
// one instruction: S = 2 (32-B segments, 16 rows / instr), 4 (64-B segments,
// 8 rows / instr, the production scheme) and 8 (whole 128-B rows, 4 rows /
// instr).  Same bytes, different numbers of L1 wavefronts / L2 requests per
// instruction.  Rows of 32 fp32 (J = 32) drawn uniformly from tables of the
// three Netflix mode sizes and two DSGD block sizes; 99,072,000 row updates per launch, every element
// += 1 (checked against the per-row counts).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 red_segments.cu -o red_segments
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

constexpr int W = 32;

__device__ __forceinline__ void red_v4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

// A warp owns 32 rows at a time; lane l of an instruction covers row
// i * (32 / S) + l / S, 16-B chunk (l % S) + c * S of that row, c over the
// W / 4 / S chunk rounds.
template <int S>
__global__ void __launch_bounds__(256) red_kernel(float* a, const int* rows, int64_t n) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int kRowsPer = 32 / S, kRounds = W / 4 / S;
  const float4 one = make_float4(1.f, 1.f, 1.f, 1.f);
  for (int64_t base = ((int64_t)blockIdx.x * 8 + w) * 32; base < n;
       base += (int64_t)gridDim.x * 256) {
    const int my = base + lane < n ? rows[base + lane] : -1;
#pragma unroll
    for (int i = 0; i < 32 / kRowsPer; ++i) {
      const int g = __shfl_sync(0xffffffffu, my, i * kRowsPer + lane / S);
#pragma unroll
      for (int c = 0; c < kRounds; ++c)
        if (g >= 0) red_v4(a + (size_t)g * W + (c * S + lane % S) * 4, one);
    }
  }
}

int main() {
  const int64_t n = 99072000;
  // the three Netflix mode sizes, then DSGD mode-3 blocks at P = 8
  // (strata: 2182 / 8 rows; ring: 2182 / 16)
  const int dims[5] = {480189, 17770, 2182, 273, 136};
  std::vector<int> h(n);
  int *rows;
  float* a;
  cudaMalloc(&rows, n * 4);
  cudaMalloc(&a, (size_t)dims[0] * W * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int m = 0; m < 5; ++m) {
    std::mt19937_64 rng(m + 1);
    std::vector<int64_t> cnt(dims[m], 0);
    for (auto& x : h) {
      x = (int)(rng() % dims[m]);
      ++cnt[x];
    }
    cudaMemcpy(rows, h.data(), n * 4, cudaMemcpyHostToDevice);
    auto run = [&](auto kern, const char* what) {
      cudaMemset(a, 0, (size_t)dims[m] * W * 4);
      kern<<<148 * 8, 256>>>(a, rows, n);  // warm-up pass (then checked below)
      cudaEventRecord(e0);
      const int reps = 3;
      for (int r = 0; r < reps; ++r) kern<<<148 * 8, 256>>>(a, rows, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= reps;
      std::vector<float> out((size_t)dims[m] * W);
      cudaMemcpy(out.data(), a, out.size() * 4, cudaMemcpyDeviceToHost);
      int64_t bad = 0;
      for (int r = 0; r < dims[m]; ++r)
        for (int j = 0; j < W; ++j)
          if (out[(size_t)r * W + j] != (float)(cnt[r] * (reps + 1))) ++bad;
      printf("rows=%6d %-22s %7.3f ms  %7.1f GB/s of updates  mismatches %lld  %s\n", dims[m],
             what, ms, n * (double)W * 4 / ms / 1e6, (long long)bad,
             cudaGetErrorString(cudaGetLastError()));
    };
    run(red_kernel<2>, "S=2 (32-B segments)");
    run(red_kernel<4>, "S=4 (64-B segments)");
    run(red_kernel<8>, "S=8 (128-B rows)");
  }
  return 0;
}
