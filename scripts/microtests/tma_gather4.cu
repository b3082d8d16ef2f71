// Micro-test: TMA tile::gather4 of 4 arbitrary rows of a [rows x 32] fp32
// matrix into smem with SWIZZLE_128B; tries boxDim[1] = 1 and 4.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void kern(const __grid_constant__ CUtensorMap tm, float* out, int r0, int r1, int r2, int r3) {
  __shared__ __align__(1024) float s[4 * 32 * 2];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 256; ++i) s[i] = -1.0f;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar)), "r"(512));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 :: "r"(smem_u32(s)), "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" :: "r"(smem_u32(&bar)) : "memory");
    for (int i = 0; i < 256; ++i) out[i] = s[i];
  }
}
int main() {
  const int rows = 1000, cols = 32;
  float* g; cudaMalloc(&g, rows * cols * 4);
  float* h = new float[rows * cols];
  for (int i = 0; i < rows * cols; ++i) h[i] = (float)i;  // value = row*32 + col
  cudaMemcpy(g, h, rows * cols * 4, cudaMemcpyHostToDevice);
  float* out; cudaMallocManaged(&out, 256 * 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no entry point\n"); return 1; }
  for (int boxh : {1, 4}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)boxh};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("boxh=%d encode=%d\n", boxh, (int)r);
    if (r) continue;
    kern<<<1, 32>>>(tm, out, 5, 9, 100, 7);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  kernel: %s\n", cudaGetErrorString(e));
    if (e) { cudaGetLastError(); return 0; }
    int rowsel[4] = {5, 9, 100, 7}; int ok = 1;
    for (int rr = 0; rr < 4; ++rr) for (int c = 0; c < 32; ++c) {
      int phys = rr * 32 + (((c / 4) ^ (rr % 8)) * 4) + c % 4;
      if (out[phys] != rowsel[rr] * 32 + c) ok = 0; }
    printf("  swizzled content ok=%d  first row: %g %g %g %g | row1 %g\n", ok, out[0], out[1], out[2], out[3], out[32]);
  }
  return 0;
}
