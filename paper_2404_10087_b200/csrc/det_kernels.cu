// Deterministic FastTuckerPlus sweeps: one CTA walks the EpochPlan batches in
// order, so every batch sees every earlier batch's factor writes exactly as
// ftk::epoch_plus does with workers == 1 (decomposition.cpp:623-705).
//
// Arithmetic follows the reference's fp32 rounding sequence (SURVEY.md
// Appendix A): __fmul_rn / __fadd_rn keep every product and sum separately
// rounded (the reference's Release build has no FMA), sums run in the
// reference's index order, and the +0 contributions of the 16-padded tile
// extents are reproduced by one trailing `+ 0.0f` (it only matters when the
// partial sum is -0).  Result: bit-identical factor rows and core matrices.
//
// This is the parity path, not the throughput path (hog_kernels.cu,
// tc_kernels.cu).  It parallelises inside a batch: C, D, U and the update
// of all N x M x {R,J} outputs are spread over the CTA's threads.
#include "engine.cuh"

namespace ftkcu {
namespace {

constexpr int kDetThreads = 512;

__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__host__ __device__ __forceinline__ int pad16d(int x) { return (x + 15) / 16 * 16; }

// Shared-memory carve-up for one batch (all float-sized slots).
struct DetLayout {
  int cap, sum_j;
  int aoff[kMaxOrder];  // per-mode offset of the [cap][J_n] row blocks
  size_t o_x, o_xhat, o_res, o_a, o_u, o_c, o_d, o_idx, o_win, o_acc, end;
};

__host__ __device__ inline DetLayout make_layout(const KView& v, int cap,
                                                 bool with_acc) {
  DetLayout L{};
  L.cap = cap;
  int s = 0;
  for (int n = 0; n < v.order; ++n) {
    L.aoff[n] = s * cap;
    s += v.j[n];
  }
  L.sum_j = s;
  const size_t ncr = (size_t)v.order * cap * v.r;
  size_t o = 0;
  L.o_x = o; o += cap;
  L.o_xhat = o; o += cap;
  L.o_res = o; o += cap;
  L.o_a = o; o += (size_t)cap * s;
  L.o_u = o; o += (size_t)cap * s;
  L.o_c = o; o += ncr;
  L.o_d = o; o += ncr;
  L.o_idx = o; o += (size_t)v.order * cap;
  L.o_win = o; o += (size_t)v.order * cap;
  L.o_acc = o;
  if (with_acc) o += (size_t)s * v.r;
  L.end = o;
  return L;
}

// Positions, values and index columns of batch [off, off + m_eff)
// (EpochPlan::gather + Batch::stage, sparse_tensor.cpp:251-269, 319-323).
__device__ void load_batch(const KView& v, const DetLayout& L, float* sm,
                           const int64_t* perm, int64_t off, int m_eff) {
  int* s_idx = reinterpret_cast<int*>(sm + L.o_idx);
  float* s_x = sm + L.o_x;
  for (int t = threadIdx.x; t < L.cap; t += blockDim.x) {
    float x = 0.0f;
    if (t < m_eff) {
      const int64_t pos = perm[off + t];
      x = v.vals[pos];
      for (int n = 0; n < v.order; ++n) s_idx[n * L.cap + t] = v.idx[n][pos];
    } else {
      for (int n = 0; n < v.order; ++n) s_idx[n * L.cap + t] = 0;
    }
    s_x[t] = x;
  }
}

// stage_factor_rows (decomposition.cpp:170-184): A_psi^(n) rows.  Plain
// (coherent) loads: the previous batch of this CTA may just have written
// these rows.
__device__ void stage_rows(const KView& v, const DetLayout& L, float* sm,
                           int m_eff) {
  const int* s_idx = reinterpret_cast<const int*>(sm + L.o_idx);
  for (int n = 0; n < v.order; ++n) {
    const int jn = v.j[n];
    float* dst = sm + L.o_a + L.aoff[n];
    const float* src = v.a[n];
    for (int e = threadIdx.x; e < m_eff * jn; e += blockDim.x) {
      const int m = e / jn, j = e - m * jn;
      dst[e] = src[(size_t)s_idx[n * L.cap + m] * jn + j];
    }
  }
}

// C^(n) = A_psi^(n) B^(n), k ascending over padded J (tiles.cpp:21-47,
// compute_c_batch_impl decomposition.cpp:186-196).
__device__ void compute_c(const KView& v, const DetLayout& L, float* sm,
                          int m_eff) {
  const int r = v.r;
  float* s_c = sm + L.o_c;
  const int* s_idx = reinterpret_cast<const int*>(sm + L.o_idx);
  for (int n = 0; n < v.order; ++n) {
    const int jn = v.j[n];
    const bool pad = (jn % kTile) != 0;
    const float* a = sm + L.o_a + L.aoff[n];
    const float* __restrict__ b = v.b[n];
    if (v.cc[n]) {  // storage scheme: copy the cached row (decomposition.cpp:299-314)
      for (int e = threadIdx.x; e < m_eff * r; e += blockDim.x) {
        const int m = e / r, c = e - m * r;
        s_c[(n * L.cap + m) * r + c] = v.cc[n][(size_t)s_idx[n * L.cap + m] * r + c];
      }
      continue;
    }
    for (int e = threadIdx.x; e < m_eff * r; e += blockDim.x) {
      const int m = e / r, c = e - m * r;
      const float* arow = a + m * jn;
      float acc = 0.0f;
#pragma unroll 8
      for (int k = 0; k < jn; ++k) acc = fadd(acc, fmul(arow[k], __ldg(b + (size_t)k * r + c)));
      if (pad) acc = fadd(acc, 0.0f);
      s_c[(n * L.cap + m) * r + c] = acc;
    }
  }
}

// D^(k) = C^(first) * prod_{n>first, n!=k} C^(n), modes ascending
// (compute_d_batch_impl, decomposition.cpp:200-212).
__device__ void compute_d(const KView& v, const DetLayout& L, float* sm,
                          int m_eff) {
  const int r = v.r;
  const float* s_c = sm + L.o_c;
  float* s_d = sm + L.o_d;
  const int per = m_eff * r;
  for (int e = threadIdx.x; e < v.order * per; e += blockDim.x) {
    const int k = e / per, rem = e - k * per;
    const int first = (k == 0) ? 1 : 0;
    float acc = s_c[first * L.cap * r + rem];
    for (int n = first + 1; n < v.order; ++n) {
      if (n == k) continue;
      acc = fmul(acc, s_c[n * L.cap * r + rem]);
    }
    s_d[k * L.cap * r + rem] = acc;
  }
}

// U^(n) = D^(n) B^(n)T, r ascending over padded R (compute_u_single_impl,
// decomposition.cpp:226-232).
__device__ void compute_u(const KView& v, const DetLayout& L, float* sm,
                          int m_eff) {
  const int r = v.r;
  const bool pad = (r % kTile) != 0;
  const float* s_d = sm + L.o_d;
  for (int n = 0; n < v.order; ++n) {
    const int jn = v.j[n];
    float* u = sm + L.o_u + L.aoff[n];
    const float* __restrict__ b = v.b[n];
    for (int e = threadIdx.x; e < m_eff * jn; e += blockDim.x) {
      const int m = e / jn, j = e - m * jn;
      const float* drow = s_d + (n * L.cap + m) * r;
      const float* brow = b + (size_t)j * r;
      float acc = 0.0f;
#pragma unroll 8
      for (int c = 0; c < r; ++c) acc = fadd(acc, fmul(drow[c], __ldg(brow + c)));
      if (pad) acc = fadd(acc, 0.0f);
      u[e] = acc;
    }
  }
}

// row_dot over the padded extent + residual_from_xhat (tiles.cpp:86-99,
// decomposition.cpp:234-252).  p and q are [m][len] row blocks.
__device__ void predict_rows(const DetLayout& L, float* sm, const float* p,
                             const float* q, int len, int m_eff) {
  const bool pad = (len % kTile) != 0;
  for (int m = threadIdx.x; m < m_eff; m += blockDim.x) {
    float acc = 0.0f;
    for (int k = 0; k < len; ++k) acc = fadd(acc, fmul(p[m * len + k], q[m * len + k]));
    if (pad) acc = fadd(acc, 0.0f);
    sm[L.o_xhat + m] = acc;
    sm[L.o_res + m] = fsub(sm[L.o_x + m], acc);
  }
}

// Single-batch probe outputs (zero padding rows, like the reference tiles).
__device__ void publish_debug(const KView& v, const DetLayout& L, float* sm,
                              int m_eff, const DetDebug& dbg, bool factor) {
  const int cap = L.cap, r = v.r;
  if (factor) {
    for (int e = threadIdx.x; e < v.order * cap * r; e += blockDim.x) {
      const int m = (e % (cap * r)) / r;
      if (dbg.c) dbg.c[e] = m < m_eff ? sm[L.o_c + e] : 0.0f;
      if (dbg.d) dbg.d[e] = m < m_eff ? sm[L.o_d + e] : 0.0f;
    }
    if (dbg.u) {
      for (int e = threadIdx.x; e < v.order * cap * dbg.jmax; e += blockDim.x) {
        const int n = e / (cap * dbg.jmax), rem = e - n * cap * dbg.jmax;
        const int m = rem / dbg.jmax, j = rem - m * dbg.jmax;
        dbg.u[e] = (m < m_eff && j < v.j[n]) ? sm[L.o_u + L.aoff[n] + m * v.j[n] + j] : 0.0f;
      }
    }
  }
  for (int m = threadIdx.x; m < cap; m += blockDim.x) {
    if (dbg.xhat) dbg.xhat[m] = m < m_eff ? sm[L.o_xhat + m] : 0.0f;
    if (dbg.resid) dbg.resid[m] = m < m_eff ? sm[L.o_res + m] : 0.0f;
  }
}

// HOT LOOP 1, deterministic: decomposition.cpp:644-658 with workers == 1.
__global__ void __launch_bounds__(kDetThreads)
det_factor_kernel(KView v, const int64_t* __restrict__ perm, int cap, float lr,
                  float reg, DetDebug dbg) {
  extern __shared__ float sm[];
  const DetLayout L = make_layout(v, cap, false);
  int* s_idx = reinterpret_cast<int*>(sm + L.o_idx);
  int* s_win = reinterpret_cast<int*>(sm + L.o_win);
  for (int64_t off = 0; off < v.nnz; off += cap) {
    const int m_eff = (int)((v.nnz - off) < cap ? (v.nnz - off) : cap);
    load_batch(v, L, sm, perm, off, m_eff);
    __syncthreads();
    stage_rows(v, L, sm, m_eff);
    // Last-writer-wins mask for rows repeated inside the batch: the
    // reference scatters rows in ascending m (decomposition.cpp:257-272).
    for (int e = threadIdx.x; e < v.order * m_eff; e += blockDim.x) {
      const int n = e / m_eff, m = e - n * m_eff;
      const int me = s_idx[n * cap + m];
      int w = 1;
      for (int q = m + 1; q < m_eff; ++q) w &= (s_idx[n * cap + q] != me);
      s_win[n * cap + m] = w;
    }
    __syncthreads();
    compute_c(v, L, sm, m_eff);
    __syncthreads();
    compute_d(v, L, sm, m_eff);
    __syncthreads();
    compute_u(v, L, sm, m_eff);
    __syncthreads();
    predict_rows(L, sm, sm + L.o_a + L.aoff[0], sm + L.o_u + L.aoff[0], v.j[0], m_eff);
    __syncthreads();
    if (dbg.c || dbg.d || dbg.u || dbg.xhat || dbg.resid) publish_debug(v, L, sm, m_eff, dbg, true);
    // Eq. (14): A <- snap + lr (r u - reg snap) from the staged snapshot
    // (update_factors_plus_impl, decomposition.cpp:254-275).
    for (int n = 0; n < v.order; ++n) {
      const int jn = v.j[n];
      const float* snap = sm + L.o_a + L.aoff[n];
      const float* u = sm + L.o_u + L.aoff[n];
      float* dst = v.a[n];
      for (int e = threadIdx.x; e < m_eff * jn; e += blockDim.x) {
        const int m = e / jn, j = e - m * jn;
        if (!s_win[n * cap + m]) continue;
        const float s = snap[e];
        const float g = fmul(sm[L.o_res + m], u[e]);
        const float rg = fmul(reg, s);
        dst[(size_t)s_idx[n * cap + m] * jn + j] = fadd(s, fmul(lr, fsub(g, rg)));
      }
    }
    __syncthreads();
  }
}

// HOT LOOP 2, deterministic: decomposition.cpp:678-698 with workers == 1.
// The per-batch G = E^T D (m ascending over the padded batch) is added into
// the running accumulator in batch order (accumulate_core_grads_plus_impl,
// decomposition.cpp:277-296).  The accumulator lives in shared memory when it
// fits, otherwise in `grad` (each element owned by one thread either way).
__global__ void __launch_bounds__(kDetThreads)
det_core_kernel(KView v, const int64_t* __restrict__ perm, int cap,
                float* __restrict__ grad, int acc_in_smem, DetDebug dbg) {
  extern __shared__ float sm[];
  const DetLayout L = make_layout(v, cap, acc_in_smem != 0);
  const int r = v.r;
  const int capp = pad16d(cap);
  float* acc = acc_in_smem ? sm + L.o_acc : grad;
  const int total = L.sum_j * r;
  if (acc_in_smem)
    for (int e = threadIdx.x; e < total; e += blockDim.x) acc[e] = grad[e];
  __syncthreads();
  for (int64_t off = 0; off < v.nnz; off += cap) {
    const int m_eff = (int)((v.nnz - off) < cap ? (v.nnz - off) : cap);
    load_batch(v, L, sm, perm, off, m_eff);
    __syncthreads();
    stage_rows(v, L, sm, m_eff);
    __syncthreads();
    compute_c(v, L, sm, m_eff);
    __syncthreads();
    compute_d(v, L, sm, m_eff);
    __syncthreads();
    // C-side prediction (predict_c_side_impl, decomposition.cpp:247-252).
    predict_rows(L, sm, sm + L.o_c, sm + L.o_d, r, m_eff);
    __syncthreads();
    if (dbg.xhat || dbg.resid) publish_debug(v, L, sm, m_eff, dbg, false);
    // E = resid (x) A_psi; G[j][c] = sum_m E[m][j] D[m][c]; acc += G.
    const bool mpad = capp > m_eff;
    int base = 0;
    for (int n = 0; n < v.order; ++n) {
      const int jn = v.j[n];
      const float* a = sm + L.o_a + L.aoff[n];
      const float* d = sm + L.o_d + n * cap * r;
      for (int e = threadIdx.x; e < jn * r; e += blockDim.x) {
        const int j = e / r, c = e - j * r;
        float g = 0.0f;
        for (int m = 0; m < m_eff; ++m) {
          const float ee = fmul(sm[L.o_res + m], a[m * jn + j]);
          g = fadd(g, fmul(ee, d[m * r + c]));
        }
        if (mpad) g = fadd(g, 0.0f);
        acc[base + e] = fadd(acc[base + e], g);
      }
      base += jn * r;
    }
    __syncthreads();
  }
  if (acc_in_smem)
    for (int e = threadIdx.x; e < total; e += blockDim.x) grad[e] = acc[e];
}

// CoreGradAccumulator::merge into a zero total, then apply_core_update
// (decomposition.cpp:154-162, 576-589).
__global__ void apply_core_kernel(KView v, float* __restrict__ grad, float lr,
                                  float reg) {
  const float inv = __fdiv_rn(1.0f, (float)v.nnz);
  int base = 0;
  for (int n = 0; n < v.order; ++n) {
    const int len = v.j[n] * v.r;
    float* b = const_cast<float*>(v.b[n]);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < len;
         e += gridDim.x * blockDim.x) {
      const float total = fadd(0.0f, grad[base + e]);
      grad[base + e] = total;
      const float bb = b[e];
      b[e] = fadd(bb, fmul(lr, fsub(fmul(total, inv), fmul(reg, bb))));
    }
    base += len;
  }
}

// One thread per (row, column) of the cache; B_n staged in shared memory.
__global__ void ccache_kernel(const float* __restrict__ a, const float* __restrict__ b, int64_t rows,
                              int jn, int r, float* __restrict__ out) {
  extern __shared__ float sb[];
  for (int e = threadIdx.x; e < jn * r; e += blockDim.x) sb[e] = b[e];
  __syncthreads();
  const int64_t total = rows * r;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / r;
    const int c = (int)(e - i * r);
    const float* arow = a + i * jn;
    float acc = 0.0f;
    for (int j = 0; j < jn; ++j) acc = fadd(acc, fmul(__ldg(arow + j), sb[j * r + c]));
    out[e] = acc;
  }
}

}  // namespace

cudaError_t launch_ccache(const KView& v, const int32_t* dims, float* const* out,
                          cudaStream_t st, int only_mode) {
  for (int n = 0; n < v.order; ++n) {
    if (only_mode >= 0 && n != only_mode) continue;
    const int64_t total = (int64_t)dims[n] * v.r;
    if (total == 0) continue;
    const size_t bytes = sizeof(float) * v.j[n] * v.r;
    cudaError_t e = cudaFuncSetAttribute(ccache_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    int64_t blocks = (total + 255) / 256;
    if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
    ccache_kernel<<<(int)blocks, 256, bytes, st>>>(v.a[n], v.b[n], dims[n], v.j[n], v.r, out[n]);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_det_factor(const KView& v, const int64_t* perm, int cap,
                              float lr_a, float reg_a, const DetDebug& dbg,
                              cudaStream_t st) {
  const DetLayout L = make_layout(v, cap, false);
  const size_t bytes = L.end * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(det_factor_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)bytes);
  if (e != cudaSuccess) return e;
  det_factor_kernel<<<1, kDetThreads, bytes, st>>>(v, perm, cap, lr_a, reg_a, dbg);
  return cudaGetLastError();
}

cudaError_t launch_det_core(const KView& v, const int64_t* perm, int cap,
                            float* grad, const DetDebug& dbg, cudaStream_t st) {
  DetLayout L = make_layout(v, cap, true);
  int acc_in_smem = 1;
  if (L.end * sizeof(float) > 200 * 1024) {
    acc_in_smem = 0;
    L = make_layout(v, cap, false);
  }
  const size_t bytes = L.end * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(det_core_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)bytes);
  if (e != cudaSuccess) return e;
  det_core_kernel<<<1, kDetThreads, bytes, st>>>(v, perm, cap, grad, acc_in_smem, dbg);
  return cudaGetLastError();
}

cudaError_t launch_apply_core(const KView& v, float* grad, float lr_b,
                              float reg_b, cudaStream_t st) {
  int len = 0;
  for (int n = 0; n < v.order; ++n) len = len > v.j[n] * v.r ? len : v.j[n] * v.r;
  const int threads = 256;
  int blocks = (len + threads - 1) / threads;
  blocks = blocks < 1 ? 1 : (blocks > 1024 ? 1024 : blocks);
  apply_core_kernel<<<blocks, threads, 0, st>>>(v, grad, lr_b, reg_b);
  return cudaGetLastError();
}

}  // namespace ftkcu
