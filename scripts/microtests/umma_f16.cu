// Micro-test: one fp16 row tile (128 rows t x 32 cols j, K-major SWIZZLE_64B,
// 64-B rows -- what a TMA gather of fp16 rows writes) read by tcgen05.mma
// kind::f16 both as the K-major A operand of C = A B (M = t, K = j) and as
// the MN-major A operand of G = A^T D (M = j, K = t).  Compares with a CPU
// reference.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ constexpr uint32_t swz64(uint32_t row, uint32_t byte) {
  return row * 64 + ((((byte >> 4) ^ ((row >> 1) & 3))) << 4) + (byte & 15);
}
__device__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
constexpr int T = 128, J = 32, R = 32, NB = 4;  // NB M-blocks of 32 for the G GEMM (1 real)
__device__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
               :: "r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
// a: T x J, b: J x R, dm: T x R.  out_c: T x R (C = a b), out_g: J x R (G = a^T dm)
__global__ void kern(const float* a, const float* b, const float* dm, float* out_c, float* out_g,
                     int lbo_sel) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw;
  uint8_t* sA = sm;              // NB x 8 KB (block 0 real, rest zero)
  uint8_t* sB = sm + NB * 8192;  // B^T: rows r, K = j: 32 x 64 B
  uint8_t* sD = sB + 2048;       // D: rows t, 32 cols (N = r), MN-major for G
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int t = threadIdx.x;
  for (int e = t; e < NB * 8192 / 4; e += 128) ((uint32_t*)sA)[e] = 0;
  __syncthreads();
  for (int e = t; e < T * J; e += 128) { int r = e / J, j = e % J;
    *(__half*)(sA + swz64(r, j * 2)) = __float2half_rn(a[e]); }
  for (int e = t; e < J * R; e += 128) { int j = e / R, r = e % R;
    *(__half*)(sB + swz64(r, j * 2)) = __float2half_rn(b[e]); }
  for (int e = t; e < T * R; e += 128) { int r = e / R, c = e % R;
    *(__half*)(sD + swz64(r, c * 2)) = __float2half_rn(dm[e]); }
  if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" :: "r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tm = tslot;
  if (t == 0) {
    // C = A B: M = 128 (t), N = 32 (r), K = 32 (j) in 2 steps of 16 (32 B)
    for (int ks = 0; ks < 2; ++ks)
      mma(tm, sdesc(smem_u32(sA) + ks * 32, 16, 512, 4), sdesc(smem_u32(sB) + ks * 32, 16, 512, 4),
          idesc_f16(128, R, 0, 0), ks > 0);
    // G = A^T D: M = 128 (j blocks of 32, LBO = 8 KB), N = 32 (r), K = 128 (t) in steps of 16 rows
    uint32_t lbo = lbo_sel ? 512 : 8192, sbo = lbo_sel ? 8192 : 512;
    for (int ks = 0; ks < T / 16; ++ks)
      mma(tm + 32, sdesc(smem_u32(sA) + ks * 1024, lbo, sbo, 4),
          sdesc(smem_u32(sD) + ks * 1024, lbo, sbo, 4), idesc_f16(128, R, 1, 1), ks > 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" :: "r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  int w = t / 32;
  uint32_t v[32];
#define LD32(addr) asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" \
    : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31]) : "r"(addr))
  LD32(tm + ((uint32_t)(w * 32) << 16));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int n = 0; n < R; ++n) out_c[t * R + n] = __uint_as_float(v[n]);
  LD32(tm + 32 + ((uint32_t)(w * 32) << 16));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (t < J) for (int n = 0; n < R; ++n) out_g[t * R + n] = __uint_as_float(v[n]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(tm));
}
int main() {
  float *a, *b, *d, *oc, *og;
  cudaMallocManaged(&a, T * J * 4); cudaMallocManaged(&b, J * R * 4); cudaMallocManaged(&d, T * R * 4);
  cudaMallocManaged(&oc, T * R * 4); cudaMallocManaged(&og, J * R * 4);
  srand(1);
  for (int i = 0; i < T * J; ++i) a[i] = (rand() % 17) / 8.0f - 1.0f;
  for (int i = 0; i < J * R; ++i) b[i] = (rand() % 13) / 4.0f - 1.5f;
  for (int i = 0; i < T * R; ++i) d[i] = (rand() % 11) / 4.0f - 1.25f;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int sel = 0; sel < 2; ++sel) {
    kern<<<1, 128, 64 * 1024>>>(a, b, d, oc, og, sel);
    cudaError_t e = cudaDeviceSynchronize();
    double ec = 0, eg = 0;
    for (int t = 0; t < T; ++t) for (int r = 0; r < R; ++r) {
      double s = 0; for (int j = 0; j < J; ++j) s += (double)a[t * J + j] * b[j * R + r];
      ec = fmax(ec, fabs(s - oc[t * R + r])); }
    for (int j = 0; j < J; ++j) for (int r = 0; r < R; ++r) {
      double s = 0; for (int t = 0; t < T; ++t) s += (double)a[t * J + j] * d[t * R + r];
      eg = fmax(eg, fabs(s - og[j * R + r])); }
    printf("lbo_sel=%d err=%s C maxerr=%.3g G maxerr=%.3g  c00=%g g00=%g\n", sel, cudaGetErrorString(e), ec, eg, oc[0], og[0]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
