// Micro-test: does cp.reduce.async.bulk.tensor.2d...add.tile::scatter4 add?
// 4 rows x 32 fp32 of ones reduced twice into rows {1, 5, 9, 13} of a zero
// 16 x 32 matrix: expect 2 there, 0 elsewhere (a plain scatter would give 1).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
__global__ void kern(const __grid_constant__ CUtensorMap tm, int mode) {
  __shared__ __align__(1024) float buf[4 * 32];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) buf[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(buf);
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0)
        asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                     :: "l"(&tm), "r"(0), "r"(1), "r"(5), "r"(9), "r"(13), "r"(s) : "memory");
      else
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                     :: "l"(&tm), "r"(0), "r"(1), "r"(5), "r"(9), "r"(13), "r"(s) : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }
}
int main() {
  float* g;
  cudaMalloc(&g, 16 * 32 * 4);
  PFN_cuTensorMapEncodeTiled_v12000 fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {32, 16};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
  CUresult r = fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(g, 0, 16 * 32 * 4);
    kern<<<1, 128>>>(tm, mode);
    cudaError_t e = cudaDeviceSynchronize();
    float h[16 * 32];
    cudaMemcpy(h, g, sizeof h, cudaMemcpyDeviceToHost);
    printf("mode %s err=%s row1=%g row5=%g row0=%g row13=%g\n", mode ? "store" : "reduce",
           cudaGetErrorString(e), h[1 * 32 + 3], h[5 * 32], h[0], h[13 * 32 + 31]);
  }
  return 0;
}
