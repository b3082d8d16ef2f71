// Micro-test: D[128 x 32] = A[128 x K] * B[K x 32] with tcgen05.mma kind::tf32,
// operands in smem with 128B swizzle, A and B each either K-major or MN-major.
// Compares with a CPU reference.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ constexpr uint32_t swz(uint32_t row, uint32_t byte, uint32_t P) {
  return row * P + ((((byte >> 4) ^ (P == 128 ? (row & 7) : ((row >> 1) & 3)))) << 4) + (byte & 15);
}
__device__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
constexpr int M = 128, NN = 32, K = 32;
// a: M x K row-major (a[m*K+k]), b: K x NN row-major.
__global__ void kern(const float* a, const float* b, float* out, int a_mn, int b_mn, int lbo_sel) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;            // 64 KB max
  uint8_t* sB = sm + 65536;    // 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int t = threadIdx.x;
  // A operand
  if (!a_mn) {  // K-major: rows m, K contiguous (K=32 -> 128 B rows)
    for (int e = t; e < M * K; e += 128) { int m = e / K, k = e % K;
      uint32_t off = lbo_sel >= 3 && lbo_sel != 8 ? m * 128 + ((((k * 4) >> 5) ^ (m & 3)) << 5) + ((k * 4) & 31)
                                  : swz(m, k * 4, 128);
      *(float*)(sA + off) = a[e]; }
  } else {      // MN-major: rows k, M contiguous; M blocks of 32 at stride K*128
    for (int e = t; e < M * K; e += 128) { int m = e / K, k = e % K;
      int blk = m / 32, mm = m % 32;
      uint32_t off = lbo_sel == 2 ? k * 128 + ((((mm * 4) >> 5) ^ (k & 3)) << 5) + ((mm * 4) & 31)
                                  : swz(k, mm * 4, 128);
      *(float*)(sA + blk * (K * 128) + off) = a[e]; }
  }
  if (!b_mn) {  // K-major: rows n, K contiguous
    for (int e = t; e < K * NN; e += 128) { int k = e / NN, n = e % NN;
      *(float*)(sB + swz(n, k * 4, 128)) = b[e]; }
  } else {      // MN-major: rows k, N contiguous (32 -> 128 B)
    for (int e = t; e < K * NN; e += 128) { int k = e / NN, n = e % NN;
      uint32_t off = lbo_sel == 2 ? k * 128 + ((((n * 4) >> 5) ^ (k & 3)) << 5) + ((n * 4) & 31)
                                  : swz(k, n * 4, 128);
      *(float*)(sB + off) = b[e]; }
  }
  if (t == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar))); }
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
    uint32_t id = idesc_tf32(M, NN, a_mn, b_mn);
    for (int ks = 0; ks < K / 8; ++ks) {
      uint64_t da, db;
      if (!a_mn && lbo_sel == 3) da = sdesc(smem_u32(sA) + ks * 32, 16, 1024, 1);
      else if (!a_mn && lbo_sel == 4) da = sdesc(smem_u32(sA) + ks * 32, 16, 512, 1);
      else if (!a_mn && lbo_sel == 5) da = sdesc(smem_u32(sA) + ks * 32, 128, 1024, 1);
      else if (!a_mn && lbo_sel == 6) da = sdesc(smem_u32(sA), 16, 1024, 1) + ((uint64_t)ks << 49);
      else if (!a_mn && lbo_sel == 7) da = sdesc(smem_u32(sA) + ks * 16, 16, 1024, 1);
      else if (!a_mn) da = sdesc(smem_u32(sA) + ks * 32, 16, 1024, 2);
      else if (lbo_sel == 2) da = sdesc(smem_u32(sA) + ks * 1024, K * 128, 512, 1);
      else {
        uint32_t l = K * 128, s = 1024;  // block stride, k-group stride
        if (lbo_sel) { uint32_t x = l; l = s; s = x; }
        da = sdesc(smem_u32(sA) + ks * 1024, l, s, 2);
      }
      if (!b_mn) db = sdesc(smem_u32(sB) + ks * 32, 16, 1024, 2);
      else if (lbo_sel == 2) db = sdesc(smem_u32(sB) + ks * 1024, 4096, 512, 1);
      else {
        uint32_t l = 4096, s = 1024;
        if (lbo_sel) { uint32_t x = l; l = s; s = x; }
        db = sdesc(smem_u32(sB) + ks * 1024, l, s, 2);
      }
      uint32_t acc = ks > 0;
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                   :: "r"(tm), "l"(da), "l"(db), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" :: "r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  int w = t / 32;
  uint32_t v[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
    : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
    : "r"(tm + ((uint32_t)(w * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int n = 0; n < NN; ++n) out[t * NN + n] = __uint_as_float(v[n]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(tm));
}
int main(int argc, char** argv) {
  int only = argc > 1 ? atoi(argv[1]) : -1;
  float *a, *b, *o;
  cudaMallocManaged(&a, M * K * 4); cudaMallocManaged(&b, K * NN * 4); cudaMallocManaged(&o, M * NN * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) a[i] = (rand() % 17) / 8.0f - 1.0f;
  for (int i = 0; i < K * NN; ++i) b[i] = (rand() % 13) / 4.0f - 1.5f;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int am = 0; am < 2; ++am) for (int bm = 0; bm < 2; ++bm) for (int sel = 0; sel < 8; ++sel) {
    if (!am && !bm && sel && sel < 3) continue;
    if (sel >= 3 && (am || bm)) continue;
    if (only >= 0 && sel != only) continue;
    for (int i = 0; i < M * NN; ++i) o[i] = -777.0f;
    kern<<<1, 128, 100 * 1024>>>(a, b, o, am, bm, sel);
    cudaError_t e = cudaDeviceSynchronize();
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < NN; ++n) {
      double r = 0; for (int k = 0; k < K; ++k) r += (double)a[m * K + k] * b[k * NN + n];
      maxerr = fmax(maxerr, fabs(r - o[m * NN + n])); maxref = fmax(maxref, fabs(r)); }
    printf("a_mn=%d b_mn=%d lbo_swap=%d err=%s maxerr=%.3g maxref=%.3g o[0]=%g o[1]=%g\n", am, bm, sel,
           cudaGetErrorString(e), maxerr, maxref, o[0], o[1]);
  }
  return 0;
}
