// fp64 evaluation: ftk::loss / ftk::evaluate (evaluation.cpp:36-72) over the
// resident model.
//
// predict_element (model.cpp:70-92) costs N*J*R fp64 MACs per entry as
// written.  The engine first materialises C64_n = A_n B_n in fp64 (I_n x R,
// j ascending -- the very sums predict_element forms), after which one entry
// costs N*R multiplies: x_hat = sum_r prod_n C64_n[i_n][r].  Every operation
// is the reference's (separately rounded __dmul_rn / __dadd_rn, same order),
// so per-entry residuals are bit-identical.
//
// Reductions: EXACT reproduces the reference's slab order for `workers`
// (ceil(n/w) contiguous entries per slab summed in order, slabs combined in
// order, evaluation.cpp:13-32) -- inherently sequential per slab, used for
// parity.  FAST is a deterministic two-level tree (block partials, then one
// ordered pass), used for throughput runs.
#include <vector>

#include "engine.cuh"

namespace ftkcu {
namespace {

constexpr int kEvalThreads = 256;

__global__ void c64_kernel(const float* __restrict__ a, const float* __restrict__ b,
                           int64_t rows, int jn, int r, double* __restrict__ out) {
  const int64_t total = rows * r;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / r;
    const int c = (int)(e - i * r);
    const float* arow = a + i * jn;
    double s = 0.0;
    for (int j = 0; j < jn; ++j)
      s = __dadd_rn(s, __dmul_rn((double)arow[j], (double)__ldg(b + (size_t)j * r + c)));
    out[e] = s;
  }
}

struct EntryView {
  int order, r;
  const int32_t* idx[kMaxOrder];
  const double* c64[kMaxOrder];
  const float* vals;
  int64_t nnz;
};

__device__ __forceinline__ double residual(const EntryView& v, int64_t e) {
  int32_t ii[kMaxOrder];
  for (int n = 0; n < v.order; ++n) ii[n] = v.idx[n][e];
  double acc = 0.0;
  for (int c = 0; c < v.r; ++c) {
    double prod = 1.0;
    for (int n = 0; n < v.order; ++n)
      prod = __dmul_rn(prod, v.c64[n][(int64_t)ii[n] * v.r + c]);
    acc = __dadd_rn(acc, prod);
  }
  return __dsub_rn((double)v.vals[e], acc);
}

// EXACT: per-entry squared and absolute residuals, reduced later in order.
__global__ void entry_exact_kernel(EntryView v, double* __restrict__ sq,
                                   double* __restrict__ ab) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < v.nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double res = residual(v, e);
    sq[e] = __dmul_rn(res, res);
    ab[e] = fabs(res);
  }
}

// FAST: per-block partial sums (fixed grid => deterministic).
__global__ void entry_fast_kernel(EntryView v, double* __restrict__ part) {
  __shared__ double s_sq[kEvalThreads], s_ab[kEvalThreads];
  double q = 0.0, a = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < v.nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double res = residual(v, e);
    q += res * res;
    a += fabs(res);
  }
  s_sq[threadIdx.x] = q;
  s_ab[threadIdx.x] = a;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s_sq[threadIdx.x] += s_sq[threadIdx.x + w];
      s_ab[threadIdx.x] += s_ab[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s_sq[0];
    part[2 * blockIdx.x + 1] = s_ab[0];
  }
}

// Ordered fold of buf[lo, hi) for each slab (one warp per slab): lane 0 adds
// the values one by one in index order; the warp only prefetches.
template <typename T, bool kSquare>
__global__ void slab_fold_kernel(const T* __restrict__ buf, int64_t n, int64_t chunk,
                                 double* __restrict__ out) {
  const int lane = threadIdx.x;
  const int64_t lo = blockIdx.x * chunk;
  const int64_t hi = lo + chunk < n ? lo + chunk : n;
  double acc = 0.0;
  for (int64_t base = lo; base < hi; base += 32) {
    double val = 0.0;
    if (base + lane < hi) {
      double x = (double)buf[base + lane];
      val = kSquare ? __dmul_rn(x, x) : x;
    }
    const int cnt = (int)((hi - base) < 32 ? (hi - base) : 32);
    for (int k = 0; k < cnt; ++k) {
      const double t = __shfl_sync(0xffffffffu, val, k);
      acc = __dadd_rn(acc, t);
    }
  }
  if (lane == 0) out[blockIdx.x] = acc;
}

// FAST sum of squares of a float matrix: block partials.
__global__ void sq_fast_kernel(const float* __restrict__ x, int64_t n,
                               double* __restrict__ part) {
  __shared__ double s[kEvalThreads];
  double q = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[e];
    q += v * v;
  }
  s[threadIdx.x] = q;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

int grid_for(int64_t n) {
  int64_t g = (n + kEvalThreads - 1) / kEvalThreads;
  const int cap = num_sms() * 8;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

size_t eval_scratch_bytes(const DevModel& m, const DevTensor& t, int workers) {
  size_t s = 0;
  for (int n = 0; n < m.order; ++n) s += align256((size_t)m.dims[n] * m.r * sizeof(double));
  s += 2 * align256((size_t)t.nnz * sizeof(double));  // exact per-entry buffers
  s += align256((size_t)(workers < 1 ? 1 : workers) * 2 * sizeof(double));
  s += align256((size_t)(num_sms() * 8) * (2 + 2 * kMaxOrder) * sizeof(double));
  s += align256((size_t)2 * kMaxOrder * sizeof(double));
  return s;
}

cudaError_t run_eval(const DevModel& m, const DevTensor& t, int workers,
                     double reg_a, double reg_b, bool exact, double* out3,
                     void* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (workers < 1) workers = 1;
  if (scratch_bytes < eval_scratch_bytes(m, t, workers)) return cudaErrorInvalidValue;
  char* p = static_cast<char*>(scratch);
  EntryView ev{};
  ev.order = m.order;
  ev.r = m.r;
  ev.vals = t.vals;
  ev.nnz = t.nnz;
  for (int n = 0; n < m.order; ++n) {
    double* c = reinterpret_cast<double*>(p);
    p += align256((size_t)m.dims[n] * m.r * sizeof(double));
    const int64_t cells = (int64_t)m.dims[n] * m.r;
    c64_kernel<<<grid_for(cells), kEvalThreads, 0, st>>>(m.a[n], m.b[n], m.dims[n],
                                                         m.ranks[n], m.r, c);
    ev.c64[n] = c;
    ev.idx[n] = t.idx[n];
  }
  double* sq = reinterpret_cast<double*>(p);
  p += align256((size_t)t.nnz * sizeof(double));
  double* ab = reinterpret_cast<double*>(p);
  p += align256((size_t)t.nnz * sizeof(double));
  double* slabs = reinterpret_cast<double*>(p);
  p += align256((size_t)workers * 2 * sizeof(double));
  double* part = reinterpret_cast<double*>(p);
  p += align256((size_t)(num_sms() * 8) * (2 + 2 * kMaxOrder) * sizeof(double));
  double* mats = reinterpret_cast<double*>(p);

  std::vector<double> h_mats(2 * m.order, 0.0);
  double sum_sq = 0.0, sum_ab = 0.0;
  if (exact) {
    if (t.nnz > 0) {
      entry_exact_kernel<<<grid_for(t.nnz), kEvalThreads, 0, st>>>(ev, sq, ab);
      const int64_t chunk = (t.nnz + workers - 1) / workers;
      slab_fold_kernel<double, false><<<workers, 32, 0, st>>>(sq, t.nnz, chunk, slabs);
      slab_fold_kernel<double, false><<<workers, 32, 0, st>>>(ab, t.nnz, chunk, slabs + workers);
    }
    // Regulariser: one sequential sum of squares per matrix (evaluation.cpp:40-52).
    for (int n = 0; n < m.order; ++n) {
      const int64_t la = (int64_t)m.dims[n] * m.ranks[n];
      const int64_t lb = (int64_t)m.ranks[n] * m.r;
      slab_fold_kernel<float, true><<<1, 32, 0, st>>>(m.a[n], la, la, mats + n);
      slab_fold_kernel<float, true><<<1, 32, 0, st>>>(m.b[n], lb, lb, mats + m.order + n);
    }
    std::vector<double> h_slabs(2 * workers, 0.0);
    cudaError_t e;
    if (t.nnz > 0) {
      e = cudaMemcpyAsync(h_slabs.data(), slabs, sizeof(double) * 2 * workers,
                          cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return e;
    }
    e = cudaMemcpyAsync(h_mats.data(), mats, sizeof(double) * 2 * m.order,
                        cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    // combine() in worker order (evaluation.cpp:25-29).  Slabs past the end
    // of a short tensor are empty and contribute +0.
    for (int w = 0; w < workers; ++w) sum_sq = sum_sq + h_slabs[w];
    for (int w = 0; w < workers; ++w) sum_ab = sum_ab + h_slabs[workers + w];
  } else {
    // part layout: [2 g] entry partials, then one [g_mat] block per matrix.
    const int g = grid_for(t.nnz);
    const int gm = num_sms() * 8;
    if (t.nnz > 0) entry_fast_kernel<<<g, kEvalThreads, 0, st>>>(ev, part);
    for (int n = 0; n < 2 * m.order; ++n) {
      const bool isa = n < m.order;
      const int k = isa ? n : n - m.order;
      const float* x = isa ? m.a[k] : m.b[k];
      const int64_t len = isa ? (int64_t)m.dims[k] * m.ranks[k] : (int64_t)m.ranks[k] * m.r;
      cudaMemsetAsync(part + 2 * gm + (size_t)n * gm, 0, sizeof(double) * gm, st);
      sq_fast_kernel<<<grid_for(len), kEvalThreads, 0, st>>>(x, len, part + 2 * gm + (size_t)n * gm);
    }
    const size_t nparts = 2 * (size_t)gm + 2 * (size_t)m.order * gm;
    std::vector<double> h_part(nparts, 0.0);
    cudaError_t e = cudaSuccess;
    if (t.nnz == 0) e = cudaMemsetAsync(part, 0, sizeof(double) * 2 * gm, st);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(h_part.data(), part, sizeof(double) * nparts, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    for (int i = 0; i < g; ++i) {
      sum_sq += h_part[2 * i];
      sum_ab += h_part[2 * i + 1];
    }
    for (int n = 0; n < 2 * m.order; ++n) {
      double acc = 0.0;
      for (int i = 0; i < gm; ++i) acc += h_part[2 * gm + (size_t)n * gm + i];
      h_mats[n] = acc;
    }
  }
  double reg = 0.0;
  for (int n = 0; n < m.order; ++n) reg = reg + reg_a * h_mats[n];
  for (int n = 0; n < m.order; ++n) reg = reg + reg_b * h_mats[m.order + n];
  out3[0] = sum_sq;
  out3[1] = sum_ab;
  out3[2] = reg;
  return cudaGetLastError();
}

}  // namespace ftkcu
