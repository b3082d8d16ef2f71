// FasterTucker (the paper's second convex baseline) on
// the device: ftk::epoch_fastertucker (decomposition.cpp:772-843).
//
// Buckets are keyed by the complement of mode n (all other indices), so a
// batch shares one d = prod_{k != n} C_cache^(k) row, and C_cache^(n) /
// B^(n) enter only through that batch's vectors:
//
// * Factor block (update_factor_fastertucker_impl, :451-489): an entry's step
//   reads and writes only its own mode-n row, given t = B^(n) d, and every
//   other input (cache rows of the other modes, B^(n)) is fixed in the
//   block.  So the rows are independent chains.  The host regroups the plan
//   by mode-n row (plan order inside a row) and one warp walks one row's
//   entries: bit-identical to the reference's sequential block at any
//   parallelism.
// * Core block (update_core_fastertucker_impl, :491-533): a batch's residuals
//   come from the block-entry cache of mode n, and its gradient is the outer
//   product g d^T with g = A_psi^T r.  Neither depends on B^(n), so each B
//   element's per-batch recurrence b <- b + lr (g_j d_c / M - reg b) runs on
//   its own thread over the batch sequence, after one parallel pass forms
//   every batch's (g, d, 1/M).  For workers > 1 the recurrence, being
//   linear, is instead summed in closed form over all batches in parallel.
//
// Arithmetic: the reference's fp32 sequence, each product and sum rounded on
// its own (__fmul_rn / __fadd_rn), sums in the reference's order; these
// loops have no padded extents.
#include "engine.cuh"

namespace ftkcu {
namespace {

__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }

constexpr int kFstWarps = 8;

// d[col] = C^(first)[i_first][col] * prod_{k > first, k != mode} C^(k)[i_k][col]
// (compute_d_row_impl, :420-449), lanes over col.
__device__ __forceinline__ void d_row(const KView& v, int mode, int64_t pos, float* d, int lane,
                                      int stride) {
  const int r = v.r, first = (mode == 0) ? 1 : 0;
  for (int c = lane; c < r; c += stride) {
    float acc = v.cc[first][(size_t)v.idx[first][pos] * r + c];
    for (int k = first + 1; k < v.order; ++k) {
      if (k == mode) continue;
      acc = fmul(acc, v.cc[k][(size_t)v.idx[k][pos] * r + c]);
    }
    d[c] = acc;
  }
}

__global__ void __launch_bounds__(kFstWarps * 32)
fst_factor_kernel(KView v, int mode, const int64_t* __restrict__ perm,
                  const int64_t* __restrict__ goff, int64_t ngroups, float lr, float reg) {
  extern __shared__ float smem[];
  const int r = v.r, jn = v.j[mode];
  const int per = (r + 2 * jn + 3) / 4 * 4;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* d = smem + (size_t)wib * per;
  float* t = d + r;
  float* a = t + jn;
  const float* __restrict__ bm = v.b[mode];
  float* amode = v.a[mode];
  for (int64_t g = (int64_t)blockIdx.x * kFstWarps + wib; g < ngroups;
       g += (int64_t)gridDim.x * kFstWarps) {
    const int64_t beg = goff[g], end = goff[g + 1];
    const int row = v.idx[mode][perm[beg]];
    for (int k = lane; k < jn; k += 32) a[k] = amode[(size_t)row * jn + k];
    for (int64_t e = beg; e < end; ++e) {
      const int64_t pos = perm[e];
      d_row(v, mode, pos, d, lane, 32);
      __syncwarp();
      // t = B^(n) d (:463-470), col ascending
      for (int k = lane; k < jn; k += 32) {
        float acc = 0.0f;
        for (int c = 0; c < r; ++c) acc = fadd(acc, fmul(__ldg(bm + (size_t)k * r + c), d[c]));
        t[k] = acc;
      }
      __syncwarp();
      // r = x - a . t (:474-479), j ascending
      float res = 0.0f;
      if (lane == 0) {
        float acc = 0.0f;
        for (int k = 0; k < jn; ++k) acc = fadd(acc, fmul(a[k], t[k]));
        res = fsub(v.vals[pos], acc);
      }
      res = __shfl_sync(0xffffffffu, res, 0);
      // single-sample step from the row's snapshot (:482-488)
      for (int k = lane; k < jn; k += 32) {
        const float s = a[k];
        a[k] = fadd(s, fmul(lr, fsub(fmul(res, t[k]), fmul(reg, s))));
      }
      __syncwarp();
    }
    for (int k = lane; k < jn; k += 32) amode[(size_t)row * jn + k] = a[k];
    __syncwarp();
  }
}

// Per batch: d, residuals from the block-entry cache of mode n
// (:506-512), g = A_psi^T r rows ascending (:515-522), and the step input
// x[j][c] = (g_j d_c) (1/M) of every element of B^(n) (:529).  One warp per
// batch; out row b holds the J x R values of x.
__global__ void __launch_bounds__(kFstWarps * 32)
fst_core_prep_kernel(KView v, int mode, const int64_t* __restrict__ perm,
                     const int64_t* __restrict__ boff, int64_t b0, int64_t nb,
                     float* __restrict__ out) {
  extern __shared__ float smem[];
  const int r = v.r, jn = v.j[mode];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* d = smem + (size_t)wib * (r + jn + 32);
  float* g = d + r;
  float* res = g + jn;  // 32 residuals at a time
  for (int64_t b = (int64_t)blockIdx.x * kFstWarps + wib; b < nb;
       b += (int64_t)gridDim.x * kFstWarps) {
    const int64_t beg = boff[b0 + b], end = boff[b0 + b + 1];
    const int m_eff = (int)(end - beg);
    if (m_eff <= 0) continue;  // the C-ABI rejects empty batches; never read perm[end]
    d_row(v, mode, perm[beg], d, lane, 32);
    __syncwarp();
    // g accumulates over rows ascending; lanes own j, rows come 32 at a time
    float gacc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int m0 = 0; m0 < m_eff; m0 += 32) {
      const int m = m0 + lane;
      if (m < m_eff) {
        const int64_t pos = perm[beg + m];
        const float* crow = v.cc[mode] + (size_t)v.idx[mode][pos] * r;
        float acc = 0.0f;
        for (int c = 0; c < r; ++c) acc = fadd(acc, fmul(crow[c], d[c]));
        res[lane] = fsub(v.vals[pos], acc);
      }
      __syncwarp();
      const int mm = (m_eff - m0) < 32 ? (m_eff - m0) : 32;
      for (int q = 0; q < 4; ++q) {
        const int k = lane + 32 * q;
        if (k >= jn) break;
        for (int i = 0; i < mm; ++i) {
          const int64_t pos = perm[beg + m0 + i];
          gacc[q] = fadd(gacc[q], fmul(res[i], v.a[mode][(size_t)v.idx[mode][pos] * jn + k]));
        }
      }
      __syncwarp();
    }
    for (int q = 0; q < 4; ++q) {
      const int k = lane + 32 * q;
      if (k < jn) g[k] = gacc[q];
    }
    __syncwarp();
    const float inv = __fdiv_rn(1.0f, (float)m_eff);
    float* o = out + (size_t)b * jn * r;
    for (int e = lane; e < jn * r; e += 32) {
      const int k = e / r, c = e - k * r;
      o[e] = fmul(fmul(g[k], d[c]), inv);
    }
    __syncwarp();
  }
}

// b <- b + lr (x - reg b) over the batches in order (:525-532), one thread
// per element of B^(n).  The x stream is triple-buffered in registers, two
// 32-step rounds ahead (one block reads 1 KB per step at J = R = 16: the
// loads, not the 4-op dependent chain, would otherwise set the pace).
constexpr int kAhead = 32;

__global__ void __launch_bounds__(256)
fst_core_chain_kernel(float* __restrict__ bm, int elems, const float* __restrict__ xs, int64_t nb,
                      float lr, float reg) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= elems) return;
  float b = bm[e];
  float cur[kAhead], nx1[kAhead], nx2[kAhead];
  const float* p = xs + e;
  // unpredicated: the scratch holds 2 kAhead steps of slack past any chunk
  // (steps past nb are loaded but never used)
  auto load = [&](float (&dst)[kAhead], int64_t t0) {
    const float* q = p + (size_t)t0 * elems;
#pragma unroll
    for (int i = 0; i < kAhead; ++i) dst[i] = __ldcs(q + i * elems);
  };
  load(cur, 0);
  load(nx1, kAhead);
  for (int64_t t0 = 0; t0 < nb; t0 += kAhead) {
    load(nx2, t0 + 2 * kAhead);  // two rounds ahead: covers the L2 latency
    const int n = (nb - t0) < kAhead ? (int)(nb - t0) : kAhead;
#pragma unroll
    for (int i = 0; i < kAhead; ++i)
      if (i < n) b = fadd(b, fmul(lr, fsub(cur[i], fmul(reg, b))));
#pragma unroll
    for (int i = 0; i < kAhead; ++i) {
      cur[i] = nx1[i];
      nx1[i] = nx2[i];
    }
  }
  bm[e] = b;
}

// Parallel schedule of the core block (workers > 1).  The recurrence is
// linear, b_T = a^T b_0 + lr sum_t a^(T-1-t) (g_t d_t^T) / M_t with
// a = 1 - lr reg, so every batch contributes an outer product with a known
// weight: warps take batches in any order and accumulate w g d^T into
// private shared-memory sums, one partial per CTA; fst_scan_apply adds them.
// Same mathematics as the chain, fp32 sums in a different order.
__global__ void __launch_bounds__(kFstWarps * 32)
fst_core_scan_kernel(KView v, int mode, const int64_t* __restrict__ perm,
                     const int64_t* __restrict__ boff, int64_t nb, double a,
                     float* __restrict__ partials) {
  extern __shared__ float smem[];
  const int r = v.r, jn = v.j[mode], elems = jn * r;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* acc = smem + (size_t)wib * elems;
  float* d = smem + (size_t)kFstWarps * elems + (size_t)wib * (r + jn + 32);
  float* g = d + r;
  float* res = g + jn;
  for (int e = lane; e < elems; e += 32) acc[e] = 0.0f;
  for (int64_t b = (int64_t)blockIdx.x * kFstWarps + wib; b < nb;
       b += (int64_t)gridDim.x * kFstWarps) {
    const int64_t beg = boff[b], end = boff[b + 1];
    const int m_eff = (int)(end - beg);
    if (m_eff <= 0) continue;  // the C-ABI rejects empty batches; never read perm[end]
    d_row(v, mode, perm[beg], d, lane, 32);
    __syncwarp();
    float gacc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int m0 = 0; m0 < m_eff; m0 += 32) {
      const int m = m0 + lane;
      if (m < m_eff) {
        const int64_t pos = perm[beg + m];
        const float* crow = v.cc[mode] + (size_t)v.idx[mode][pos] * r;
        float s = 0.0f;
        for (int c = 0; c < r; ++c) s = fmaf(crow[c], d[c], s);
        res[lane] = v.vals[pos] - s;
      }
      __syncwarp();
      const int mm = (m_eff - m0) < 32 ? (m_eff - m0) : 32;
      for (int q = 0; q < 4; ++q) {
        const int k = lane + 32 * q;
        if (k >= jn) break;
        for (int i = 0; i < mm; ++i) {
          const int64_t pos = perm[beg + m0 + i];
          gacc[q] = fmaf(res[i], v.a[mode][(size_t)v.idx[mode][pos] * jn + k], gacc[q]);
        }
      }
      __syncwarp();
    }
    const float w = (float)(pow(a, (double)(nb - 1 - b)) / (double)m_eff);
    for (int q = 0; q < 4; ++q) {
      const int k = lane + 32 * q;
      if (k < jn) g[k] = w * gacc[q];
    }
    __syncwarp();
    for (int e = lane; e < elems; e += 32) {
      const int k = e / r, c = e - k * r;
      acc[e] = fmaf(g[k], d[c], acc[e]);
    }
    __syncwarp();
  }
  __syncthreads();
  for (int e = threadIdx.x; e < elems; e += blockDim.x) {
    float t = 0.0f;
    for (int w = 0; w < kFstWarps; ++w) t += smem[(size_t)w * elems + e];
    partials[(size_t)blockIdx.x * elems + e] = t;
  }
}

// b <- a^T b + lr sum_ctas partial
__global__ void fst_scan_apply_kernel(float* __restrict__ bm, int elems,
                                      const float* __restrict__ partials, int nparts, float aT,
                                      float lr) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= elems) return;
  float t = 0.0f;
  for (int p = 0; p < nparts; ++p) t += partials[(size_t)p * elems + e];
  bm[e] = fmaf(lr, t, aT * bm[e]);
}

constexpr size_t kScratchFloats = (size_t)16 << 20;  // 64 MB of step inputs per round (L2-resident)

}  // namespace

cudaError_t launch_fst_factor(const KView& v, int mode, const int64_t* perm, const int64_t* goff,
                              int64_t ngroups, float lr_a, float reg_a, cudaStream_t st) {
  if (ngroups == 0) return cudaSuccess;
  const int per = (v.r + 2 * v.j[mode] + 3) / 4 * 4;
  const size_t bytes = sizeof(float) * per * kFstWarps;
  if (bytes > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(fst_factor_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  int64_t blocks = (ngroups + kFstWarps - 1) / kFstWarps;
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  fst_factor_kernel<<<(int)blocks, kFstWarps * 32, bytes, st>>>(v, mode, perm, goff, ngroups,
                                                                 lr_a, reg_a);
  return cudaGetLastError();
}

size_t fst_core_scratch_floats(const KView& v, int mode) {
  return kScratchFloats + (size_t)3 * kAhead * v.j[mode] * v.r;
}

bool fst_scan_supported(const KView& v, int mode) {
  const size_t elems = (size_t)v.j[mode] * v.r;
  return sizeof(float) * (kFstWarps * elems + kFstWarps * (v.r + v.j[mode] + 32)) <= 200 * 1024 &&
         v.j[mode] <= 128;
}

cudaError_t launch_fst_core_scan(const KView& v, int mode, const int64_t* perm,
                                 const int64_t* boff, int64_t nbatches, float lr_b, float reg_b,
                                 float* scratch, cudaStream_t st) {
  if (!fst_scan_supported(v, mode)) return cudaErrorInvalidValue;
  if (nbatches == 0) return cudaSuccess;
  const int elems = v.j[mode] * v.r;
  const size_t bytes = sizeof(float) * (kFstWarps * (size_t)elems + kFstWarps * (v.r + v.j[mode] + 32));
  cudaError_t e = cudaFuncSetAttribute(fst_core_scan_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  int64_t blocks = (nbatches + kFstWarps - 1) / kFstWarps;
  if (blocks > (int64_t)num_sms() * 2) blocks = (int64_t)num_sms() * 2;
  const float lr = lr_b;
  const double a = 1.0 - (double)lr_b * (double)reg_b;
  fst_core_scan_kernel<<<(int)blocks, kFstWarps * 32, bytes, st>>>(v, mode, perm, boff, nbatches,
                                                                    a, scratch);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const float aT = (float)pow(a, (double)nbatches);
  fst_scan_apply_kernel<<<(elems + 255) / 256, 256, 0, st>>>(const_cast<float*>(v.b[mode]), elems,
                                                              scratch, (int)blocks, aT, lr);
  return cudaGetLastError();
}

cudaError_t launch_fst_core(const KView& v, int mode, const int64_t* perm, const int64_t* boff,
                            int64_t nbatches, float lr_b, float reg_b, float* scratch,
                            cudaStream_t st) {
  if (v.j[mode] > 128) return cudaErrorInvalidValue;
  const size_t bytes = sizeof(float) * (v.r + v.j[mode] + 32) * kFstWarps;
  cudaError_t e = cudaFuncSetAttribute(fst_core_prep_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  float* bm = const_cast<float*>(v.b[mode]);
  const int elems = v.j[mode] * v.r;
  const int64_t chunk = (int64_t)(kScratchFloats / (size_t)elems);
  for (int64_t b0 = 0; b0 < nbatches; b0 += chunk) {
    const int64_t nb = (nbatches - b0) < chunk ? (nbatches - b0) : chunk;
    int64_t blocks = (nb + kFstWarps - 1) / kFstWarps;
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    fst_core_prep_kernel<<<(int)blocks, kFstWarps * 32, bytes, st>>>(v, mode, perm, boff, b0, nb,
                                                                      scratch);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    fst_core_chain_kernel<<<(elems + 255) / 256, 256, 0, st>>>(bm, elems, scratch, nb, lr_b,
                                                                reg_b);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ftkcu
