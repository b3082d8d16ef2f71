// Micro-test: register layout of tcgen05.ld.16x256b (.x1, .x2): TMEM cell
// (lane, col) holds 1000 * lane + col; each thread prints what it received.
#include <cstdio>
#include <cstdint>
__global__ void kern(int* out) {
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, w = t / 32, l = t % 32;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"((uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;
  const uint32_t base = tm + ((uint32_t)(w * 32) << 16);
  uint32_t v[16];
  for (int c = 0; c < 16; ++c) v[c] = 1000 * (w * 32 + l) + c;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               :: "r"(base), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                  "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(base));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (w == 0) for (int i = 0; i < 8; ++i) out[l * 8 + i] = (int)r[i];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(tm));
}
int main() {
  int* o;
  cudaMallocManaged(&o, 32 * 8 * 4);
  kern<<<1, 128>>>(o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err=%s\n", cudaGetErrorString(e));
  for (int l = 0; l < 32; l += 1) {
    printf("t%2d:", l);
    for (int i = 0; i < 8; ++i) printf(" %5d", o[l * 8 + i]);
    printf("\n");
  }
  return 0;
}
