// FastTucker (the paper's convex baseline) on the
// device: ftk::epoch_fasttucker (decomposition.cpp:707-770).
//
// Factor block of mode n: the plan is EpochPlan::per_bucket over the
// fixed-mode index, so every batch lives in one bucket, i.e. shares one
// mode-n row, and moves only that row (update_factor_fasttucker_impl,
// decomposition.cpp:316-371).  Rows of the other modes and every B are
// read-only inside the block.  Buckets are therefore independent: one warp
// walks one bucket's batches in plan order, and the result is bit-identical
// to the reference's sequential (workers == 1) block in any bucket schedule.
//
// Core block of mode n: a global plan, and B^(n) moves after every batch
// (update_core_fasttucker_impl, :373-417), so the batches form one chain.
// Deterministic schedule: one CTA walks it and spreads each batch's C, D, x̂,
// G and B update over its threads.  Hogwild schedule (the reference's
// workers > 1): CTAs share the chain and add their B steps atomically.
//
// Arithmetic: the reference's fp32 sequence, each
// product and sum rounded on its own (__fmul_rn / __fadd_rn: the reference
// Release build has no FMA), sums in the reference's index order, one
// trailing `+ 0.0f` where the reference sums over a 16-padded tile extent.
#include "engine.cuh"

namespace ftkcu {
namespace {

__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }

constexpr int kFtWarps = 8;
constexpr int kFtCoreThreads = 512;

// Per-warp scratch of the factor block (floats): rows of every mode
// [n][cap][J_n] (mode n's slot unused), C [n][cap][R], D and U of mode n,
// the shared row and its c = a B^(n), residuals, values, indices.
struct FtLayout {
  int cap, aoff[kMaxOrder];
  int o_a, o_c, o_d, o_u, o_snap, o_cs, o_res, o_x, o_idx, per_warp;
};

__host__ __device__ inline FtLayout ft_layout(const KView& v, int cap, int mode) {
  FtLayout L{};
  L.cap = cap;
  int o = 0;
  for (int n = 0; n < v.order; ++n) {
    L.aoff[n] = o;
    o += cap * v.j[n];
  }
  L.o_a = 0;
  L.o_c = o; o += v.order * cap * v.r;
  L.o_d = o; o += cap * v.r;
  L.o_u = o; o += cap * v.j[mode];
  L.o_snap = o; o += v.j[mode];
  L.o_cs = o; o += v.r;
  L.o_res = o; o += cap;
  L.o_x = o; o += cap;
  L.o_idx = o; o += v.order * cap;
  L.per_warp = (o + 3) / 4 * 4;
  return L;
}

__global__ void __launch_bounds__(kFtWarps * 32)
ft_factor_kernel(KView v, int mode, const int64_t* __restrict__ perm,
                 const int64_t* __restrict__ boff, int64_t nbuckets, int cap, float lr,
                 float reg) {
  extern __shared__ float smem[];
  const FtLayout L = ft_layout(v, cap, mode);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* sm = smem + (size_t)wib * L.per_warp;
  int* s_idx = reinterpret_cast<int*>(sm + L.o_idx);
  const int r = v.r, jn = v.j[mode];
  const bool rpad = (r % kTile) != 0;
  float* amode = v.a[mode];
  for (int64_t bk = (int64_t)blockIdx.x * kFtWarps + wib; bk < nbuckets;
       bk += (int64_t)gridDim.x * kFtWarps) {
    const int64_t beg = boff[bk], end = boff[bk + 1];
    for (int64_t off = beg; off < end; off += cap) {
      const int m_eff = (int)((end - off) < cap ? (end - off) : cap);
      // Batch::stage (sparse_tensor.cpp:251-269)
      for (int m = lane; m < m_eff; m += 32) {
        const int64_t pos = perm[off + m];
        sm[L.o_x + m] = v.vals[pos];
        for (int n = 0; n < v.order; ++n) s_idx[n * cap + m] = v.idx[n][pos];
      }
      __syncwarp();
      const int row = s_idx[mode * cap];  // the bucket's shared i_n
      // stage_factor_rows_impl(skip = mode) (decomposition.cpp:170-184) and
      // the shared row's snapshot (:333-335); mode-n rows are written by this
      // warp only, and by the same lane that reads them back here
      for (int n = 0; n < v.order; ++n) {
        if (n == mode) continue;
        const int j = v.j[n];
        const float* src = v.a[n];
        float* dst = sm + L.aoff[n];
        for (int e = lane; e < m_eff * j; e += 32) {
          const int m = e / j, k = e - m * j;
          dst[e] = __ldg(src + (size_t)s_idx[n * cap + m] * j + k);
        }
      }
      for (int k = lane; k < jn; k += 32) sm[L.o_snap + k] = amode[(size_t)row * jn + k];
      __syncwarp();
      // compute_c_batch_impl(skip = mode): C^(k) = A_psi^(k) B^(k), padded J
      for (int n = 0; n < v.order; ++n) {
        if (n == mode) continue;
        const int j = v.j[n];
        const bool jpad = (j % kTile) != 0;
        const float* a = sm + L.aoff[n];
        const float* __restrict__ b = v.b[n];
        for (int e = lane; e < m_eff * r; e += 32) {
          const int m = e / r, c = e - m * r;
          float acc = 0.0f;
          for (int k = 0; k < j; ++k) acc = fadd(acc, fmul(a[m * j + k], __ldg(b + (size_t)k * r + c)));
          if (jpad) acc = fadd(acc, 0.0f);
          sm[L.o_c + (n * cap + m) * r + c] = acc;
        }
      }
      __syncwarp();
      // compute_d_single_impl (:214-224): D = C^(first) * prod_{n>first, n!=mode}
      const int first = (mode == 0) ? 1 : 0;
      for (int e = lane; e < m_eff * r; e += 32) {
        float acc = sm[L.o_c + first * cap * r + e];
        for (int n = first + 1; n < v.order; ++n) {
          if (n == mode) continue;
          acc = fmul(acc, sm[L.o_c + n * cap * r + e]);
        }
        sm[L.o_d + e] = acc;
      }
      __syncwarp();
      // compute_u_single_impl (:226-232): U = D B^(n)T, padded R; and the
      // shared row's c = a B^(n) (:336-345, unpadded j)
      const float* __restrict__ bm = v.b[mode];
      for (int e = lane; e < m_eff * jn; e += 32) {
        const int m = e / jn, k = e - m * jn;
        float acc = 0.0f;
        for (int c = 0; c < r; ++c) acc = fadd(acc, fmul(sm[L.o_d + m * r + c], __ldg(bm + (size_t)k * r + c)));
        if (rpad) acc = fadd(acc, 0.0f);
        sm[L.o_u + e] = acc;
      }
      for (int c = lane; c < r; c += 32) {
        float acc = 0.0f;
        for (int k = 0; k < jn; ++k) acc = fadd(acc, fmul(sm[L.o_snap + k], __ldg(bm + (size_t)k * r + c)));
        sm[L.o_cs + c] = acc;
      }
      __syncwarp();
      // x̂_m = c . d_m (:347-354, unpadded R), residual_from_xhat (:234-238)
      for (int m = lane; m < m_eff; m += 32) {
        float acc = 0.0f;
        for (int c = 0; c < r; ++c) acc = fadd(acc, fmul(sm[L.o_cs + c], sm[L.o_d + m * r + c]));
        sm[L.o_res + m] = fsub(sm[L.o_x + m], acc);
      }
      __syncwarp();
      // the row moves by the 1/M-mean gradient (:357-368)
      const float inv = __fdiv_rn(1.0f, (float)m_eff);
      for (int k = lane; k < jn; k += 32) {
        float g = 0.0f;
        for (int m = 0; m < m_eff; ++m) g = fadd(g, fmul(sm[L.o_res + m], sm[L.o_u + m * jn + k]));
        const float s = sm[L.o_snap + k];
        amode[(size_t)row * jn + k] = fadd(s, fmul(lr, fsub(fmul(g, inv), fmul(reg, s))));
      }
      __syncwarp();
    }
  }
}

// Core block: one CTA, batches in plan order.  Shared memory (floats): rows
// [n][cap][J_n], C [n][cap][R], D [cap][R], residuals, values, indices.
struct FtcLayout {
  int cap, aoff[kMaxOrder];
  int o_c, o_d, o_res, o_x, o_idx, end;
};

__host__ __device__ inline FtcLayout ftc_layout(const KView& v, int cap) {
  FtcLayout L{};
  L.cap = cap;
  int o = 0;
  for (int n = 0; n < v.order; ++n) {
    L.aoff[n] = o;
    o += cap * v.j[n];
  }
  L.o_c = o; o += v.order * cap * v.r;
  L.o_d = o; o += cap * v.r;
  L.o_res = o; o += cap;
  L.o_x = o; o += cap;
  L.o_idx = o; o += v.order * cap;
  L.end = o;
  return L;
}

__global__ void __launch_bounds__(kFtCoreThreads)
ft_core_kernel(KView v, int mode, const int64_t* __restrict__ perm, int cap, float lr,
               float reg) {
  extern __shared__ float sm[];
  const FtcLayout L = ftc_layout(v, cap);
  int* s_idx = reinterpret_cast<int*>(sm + L.o_idx);
  const int r = v.r, jn = v.j[mode];
  const bool rpad = (r % kTile) != 0;
  const int capp = (cap + kTile - 1) / kTile * kTile;
  float* bm = const_cast<float*>(v.b[mode]);
  for (int64_t off = 0; off < v.nnz; off += cap) {
    const int m_eff = (int)((v.nnz - off) < cap ? (v.nnz - off) : cap);
    for (int m = threadIdx.x; m < m_eff; m += blockDim.x) {
      const int64_t pos = perm[off + m];
      sm[L.o_x + m] = v.vals[pos];
      for (int n = 0; n < v.order; ++n) s_idx[n * cap + m] = v.idx[n][pos];
    }
    __syncthreads();
    // stage_factor_rows_impl(skip = -1): every mode's rows
    for (int n = 0; n < v.order; ++n) {
      const int j = v.j[n];
      for (int e = threadIdx.x; e < m_eff * j; e += blockDim.x) {
        const int m = e / j, k = e - m * j;
        sm[L.aoff[n] + e] = __ldg(v.a[n] + (size_t)s_idx[n * cap + m] * j + k);
      }
    }
    __syncthreads();
    // C^(k) for every mode: the block snapshot for k != mode (unchanged in
    // this block) and the current B^(n), which moved with the last batch
    // (:380-392); padded J
    for (int e = threadIdx.x; e < v.order * m_eff * r; e += blockDim.x) {
      const int n = e / (m_eff * r), rem = e - n * m_eff * r;
      const int m = rem / r, c = rem - m * r;
      const int j = v.j[n];
      const float* a = sm + L.aoff[n] + m * j;
      const float* b = v.b[n];
      float acc = 0.0f;
      if (n == mode)
        for (int k = 0; k < j; ++k) acc = fadd(acc, fmul(a[k], b[(size_t)k * r + c]));
      else
        for (int k = 0; k < j; ++k) acc = fadd(acc, fmul(a[k], __ldg(b + (size_t)k * r + c)));
      if (j % kTile) acc = fadd(acc, 0.0f);
      sm[L.o_c + (n * cap + m) * r + c] = acc;
    }
    __syncthreads();
    const int first = (mode == 0) ? 1 : 0;
    for (int e = threadIdx.x; e < m_eff * r; e += blockDim.x) {
      float acc = sm[L.o_c + first * cap * r + e];
      for (int n = first + 1; n < v.order; ++n) {
        if (n == mode) continue;
        acc = fmul(acc, sm[L.o_c + n * cap * r + e]);
      }
      sm[L.o_d + e] = acc;
    }
    __syncthreads();
    // predict_c_side_impl (:247-252): row_dot over padded R, residual
    for (int m = threadIdx.x; m < m_eff; m += blockDim.x) {
      float acc = 0.0f;
      for (int c = 0; c < r; ++c) acc = fadd(acc, fmul(sm[L.o_c + (mode * cap + m) * r + c], sm[L.o_d + m * r + c]));
      if (rpad) acc = fadd(acc, 0.0f);
      sm[L.o_res + m] = fsub(sm[L.o_x + m], acc);
    }
    __syncthreads();
    // E = r (x) A_psi^(n); G = E^T D over the padded batch; B^(n) moves by
    // the 1/M-mean gradient (:398-416)
    const float inv = __fdiv_rn(1.0f, (float)m_eff);
    const float* a = sm + L.aoff[mode];
    for (int e = threadIdx.x; e < jn * r; e += blockDim.x) {
      const int k = e / r, c = e - k * r;
      float g = 0.0f;
      for (int m = 0; m < m_eff; ++m)
        g = fadd(g, fmul(fmul(sm[L.o_res + m], a[m * jn + k]), sm[L.o_d + m * r + c]));
      if (capp > m_eff) g = fadd(g, 0.0f);
      const float bb = bm[e];
      bm[e] = fadd(bb, fmul(lr, fsub(fmul(g, inv), fmul(reg, bb))));
    }
    __syncthreads();
  }
}

// Hogwild core block (the reference's workers > 1 schedule, where the
// parallel_for workers update B^(n) concurrently, decomposition.cpp:752-766):
// CTAs take interleaved batches of the plan, read B^(n) through L2 and add
// their step lr (g / M - reg b) atomically.
__global__ void __launch_bounds__(256)
ft_core_hog_kernel(KView v, int mode, const int64_t* __restrict__ perm, int cap, float lr,
                   float reg) {
  extern __shared__ float sm[];
  const FtcLayout L = ftc_layout(v, cap);
  int* s_idx = reinterpret_cast<int*>(sm + L.o_idx);
  const int r = v.r, jn = v.j[mode];
  float* bm = const_cast<float*>(v.b[mode]);
  const int64_t nb = (v.nnz + cap - 1) / cap;
  for (int64_t bi = blockIdx.x; bi < nb; bi += gridDim.x) {
    const int64_t off = bi * cap;
    const int m_eff = (int)((v.nnz - off) < cap ? (v.nnz - off) : cap);
    for (int m = threadIdx.x; m < m_eff; m += blockDim.x) {
      const int64_t pos = perm[off + m];
      sm[L.o_x + m] = v.vals[pos];
      for (int n = 0; n < v.order; ++n) s_idx[n * cap + m] = v.idx[n][pos];
    }
    __syncthreads();
    for (int n = 0; n < v.order; ++n) {
      const int j = v.j[n];
      for (int e = threadIdx.x; e < m_eff * j; e += blockDim.x) {
        const int m = e / j, k = e - m * j;
        sm[L.aoff[n] + e] = __ldg(v.a[n] + (size_t)s_idx[n * cap + m] * j + k);
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < v.order * m_eff * r; e += blockDim.x) {
      const int n = e / (m_eff * r), rem = e - n * m_eff * r;
      const int m = rem / r, c = rem - m * r;
      const int j = v.j[n];
      const float* a = sm + L.aoff[n] + m * j;
      float acc = 0.0f;
      if (n == mode)
        for (int k = 0; k < j; ++k) acc = fmaf(a[k], __ldcg(v.b[n] + (size_t)k * r + c), acc);
      else
        for (int k = 0; k < j; ++k) acc = fmaf(a[k], __ldg(v.b[n] + (size_t)k * r + c), acc);
      sm[L.o_c + (n * cap + m) * r + c] = acc;
    }
    __syncthreads();
    const int first = (mode == 0) ? 1 : 0;
    for (int e = threadIdx.x; e < m_eff * r; e += blockDim.x) {
      float acc = sm[L.o_c + first * cap * r + e];
      for (int n = first + 1; n < v.order; ++n)
        if (n != mode) acc *= sm[L.o_c + n * cap * r + e];
      sm[L.o_d + e] = acc;
    }
    __syncthreads();
    for (int m = threadIdx.x; m < m_eff; m += blockDim.x) {
      float acc = 0.0f;
      for (int c = 0; c < r; ++c) acc = fmaf(sm[L.o_c + (mode * cap + m) * r + c], sm[L.o_d + m * r + c], acc);
      sm[L.o_res + m] = sm[L.o_x + m] - acc;
    }
    __syncthreads();
    const float inv = 1.0f / (float)m_eff;
    const float* a = sm + L.aoff[mode];
    for (int e = threadIdx.x; e < jn * r; e += blockDim.x) {
      const int k = e / r, c = e - k * r;
      float g = 0.0f;
      for (int m = 0; m < m_eff; ++m) g = fmaf(sm[L.o_res + m] * a[m * jn + k], sm[L.o_d + m * r + c], g);
      atomicAdd(bm + e, lr * (g * inv - reg * __ldcg(bm + e)));
    }
    __syncthreads();
  }
}

}  // namespace

size_t ft_factor_smem(const KView& v, int cap, int mode) {
  return (size_t)ft_layout(v, cap, mode).per_warp * kFtWarps * sizeof(float);
}

cudaError_t launch_ft_factor(const KView& v, int mode, const int64_t* perm, const int64_t* boff,
                             int64_t nbuckets, int cap, float lr_a, float reg_a, cudaStream_t st) {
  if (nbuckets == 0) return cudaSuccess;
  const size_t bytes = ft_factor_smem(v, cap, mode);
  if (bytes > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(ft_factor_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  int64_t blocks = (nbuckets + kFtWarps - 1) / kFtWarps;
  if (blocks > (int64_t)num_sms() * 4) blocks = (int64_t)num_sms() * 4;
  ft_factor_kernel<<<(int)blocks, kFtWarps * 32, bytes, st>>>(v, mode, perm, boff, nbuckets, cap,
                                                               lr_a, reg_a);
  return cudaGetLastError();
}

size_t ft_core_smem(const KView& v, int cap) {
  return (size_t)ftc_layout(v, cap).end * sizeof(float);
}

cudaError_t launch_ft_core(const KView& v, int mode, const int64_t* perm, int cap, float lr_b,
                           float reg_b, bool hogwild, cudaStream_t st) {
  if (v.nnz == 0) return cudaSuccess;
  const size_t bytes = ft_core_smem(v, cap);
  if (bytes > 227 * 1024) return cudaErrorInvalidValue;
  if (hogwild) {
    cudaError_t e = cudaFuncSetAttribute(ft_core_hog_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    const int64_t nb = (v.nnz + cap - 1) / cap;
    int64_t grid = (int64_t)num_sms() * 4;
    if (grid > nb) grid = nb;
    ft_core_hog_kernel<<<(int)grid, 256, bytes, st>>>(v, mode, perm, cap, lr_b, reg_b);
    return cudaGetLastError();
  }
  cudaError_t e = cudaFuncSetAttribute(ft_core_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  ft_core_kernel<<<1, kFtCoreThreads, bytes, st>>>(v, mode, perm, cap, lr_b, reg_b);
  return cudaGetLastError();
}

}  // namespace ftkcu
