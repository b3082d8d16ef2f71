// Hogwild FastTuckerPlus sweeps on CUDA cores (FTKCU_PREC_FP32), plus the
// tiler that lays the COO stream out for them.
//
// Reference semantics: ftk::epoch_plus with workers > 1 -- batches are
// processed concurrently and factor rows are written without locks
// (Hogwild contract, model.hpp:27-30; decomposition.cpp:644-658).  Here every
// warp is a "worker": it walks whole tiles of kHogTile nonzeros of the
// shuffled stream, G nonzeros at a time, with
//   stage a rows -> C = a B -> D = hadamard -> xhat, r -> U = D B^T ->
//   a += lr (r u - reg a)      (Eq. 14 / Alg. 4)
// and, in the core sweep, grad += r a^T D accumulated per warp in shared
// memory, reduced per CTA and then across CTAs in a fixed order (Eq. 15 /
// Alg. 5) -- so the core sweep is deterministic run to run.
//
// Tile order: tile t of the epoch is physical tile (t * mul + add) mod T with
// gcd(mul, T) = 1, keyed per epoch by the host.  The shuffled stream itself is
// built once per session by a Feistel bijection (no scratch, no sort).
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "engine.cuh"

namespace ftkcu {
namespace {

constexpr int kHogThreads = 256;
constexpr int kG = 4;  // nonzeros per warp step (share every B load)

// ---- tiler -------------------------------------------------------------------

__device__ __forceinline__ uint32_t mix32(uint32_t x, uint32_t k) {
  x ^= k;
  x *= 0x9e3779b1u;
  x ^= x >> 15;
  x *= 0x85ebca77u;
  x ^= x >> 13;
  return x;
}

// Bijection on [0, 2^bits) (balanced Feistel, 4 rounds), cycle-walked to
// [0, n).
__device__ int64_t feistel_perm(int64_t i, int64_t n, int bits, uint64_t seed) {
  const int hb = bits / 2;
  const uint64_t mask = (1ull << hb) - 1;
  uint64_t x = (uint64_t)i;
  do {
    uint64_t lo = x & mask, hi = x >> hb;
    for (int r = 0; r < 4; ++r) {
      uint64_t f = mix32((uint32_t)lo, (uint32_t)(seed >> (r * 8)) ^ (uint32_t)(seed >> 32) * (r + 1)) & mask;
      uint64_t nl = hi ^ f;
      hi = lo;
      lo = nl;
    }
    x = (hi << hb) | lo;
  } while ((int64_t)x >= n);
  return (int64_t)x;
}

// Inverse of feistel_perm (the rounds backwards; cycle walking inverts too).
__device__ int64_t feistel_inv(int64_t i, int64_t n, int bits, uint64_t seed) {
  const int hb = bits / 2;
  const uint64_t mask = (1ull << hb) - 1;
  uint64_t x = (uint64_t)i;
  do {
    uint64_t lo = x & mask, hi = x >> hb;
    for (int r = 3; r >= 0; --r) {
      const uint64_t plo = hi;
      hi = lo ^ (mix32((uint32_t)plo, (uint32_t)(seed >> (r * 8)) ^ (uint32_t)(seed >> 32) * (r + 1)) & mask);
      lo = plo;
    }
    x = (hi << hb) | lo;
  } while ((int64_t)x >= n);
  return (int64_t)x;
}

struct ShuffleView {
  int order;
  const int32_t* src_idx[kMaxOrder];
  int32_t* dst_idx[kMaxOrder];
  const float* src_vals;
  float* dst_vals;
  int64_t nnz;
};

__global__ void shuffle_kernel(ShuffleView v, const int64_t* __restrict__ perm,
                               int bits, uint64_t seed) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < v.nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = perm ? perm[k] : feistel_perm(k, v.nnz, bits, seed);
    for (int n = 0; n < v.order; ++n) v.dst_idx[n][k] = v.src_idx[n][p];
    v.dst_vals[k] = v.src_vals[p];
  }
}

// Order 3: the storage-order columns as 16-B records, then one random
// aligned 16-B gather per nonzero (one sector instead of four).
__global__ void pack16_kernel(const int32_t* __restrict__ i0, const int32_t* __restrict__ i1,
                              const int32_t* __restrict__ i2, const float* __restrict__ vals,
                              int4* __restrict__ rec, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    rec[k] = make_int4(__ldcs(i0 + k), __ldcs(i1 + k), __ldcs(i2 + k), __float_as_int(__ldcs(vals + k)));
}
__global__ void shuffle16_kernel(const int4* __restrict__ rec, ShuffleView v,
                                 const int64_t* __restrict__ perm, int bits, uint64_t seed) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < v.nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    // bits < 0: keep the order (cells the caller arranged)
    const int64_t p = perm ? perm[k] : (bits < 0 ? k : feistel_perm(k, v.nnz, bits, seed));
    const int4 r = __ldcs(rec + p);
    __stcs(v.dst_idx[0] + k, r.x);
    __stcs(v.dst_idx[1] + k, r.y);
    __stcs(v.dst_idx[2] + k, r.z);
    __stcs(v.dst_vals + k, __int_as_float(r.w));
  }
}

// ---- delta-coded uploads (ftkcu_tensor_upload_delta_async) -------------------
//
// One block per chunk of kDeltaChunk entries, 16 consecutive entries per
// thread, one block scan: entry e = restart[chunk] + the chunk's deltas up to
// e.  Writes the storage-order SoA columns and, for order 3 with `rec` set,
// scatters the 16-B record to its tile-stream position feistel_inv(e) -- the
// position build_shuffled's gather would give it -- so the stream is built
// chunk by chunk while the rest of the upload is still on the PCIe link.
constexpr int kDeltaThreads = 256;
constexpr int kDeltaPer = kDeltaChunk / kDeltaThreads;

struct DeltaDecode {
  const uint8_t* deltas;
  const uint64_t* restarts;
  const float* vals;
  int32_t* col[kMaxOrder];
  int32_t dims[kMaxOrder];
  double inv[kMaxOrder];
  int order, width, bits;
  uint64_t seed;
  int64_t nnz;
  int4* rec;
  int* bad;
};

// <= 85 registers (3 blocks per SM): a block must fit beside the factor
// sweep's persistent CTA (384 threads x 112 registers), or the decode of the
// next upload waits for the epoch to end
//
// kW > 0: the delta width at compile time.  A thread's kDeltaPer deltas are
// kDeltaPer * kW contiguous, 16-B aligned bytes (chunk and thread offsets are
// multiples of 16 entries), read as kW 16-B loads instead of kDeltaPer * kW
// byte loads; the bytes are then picked out of registers.  kW = 0: any width,
// byte loads (also the ragged last thread of a tensor).
template <int kW>
__global__ void __launch_bounds__(kDeltaThreads, 3)
    delta_decode_kernel(DeltaDecode d, int64_t c0, int64_t c1) {
  using Scan = cub::BlockScan<uint64_t, kDeltaThreads>;
  __shared__ typename Scan::TempStorage scan;
  for (int64_t c = c0 + blockIdx.x; c < c1; c += gridDim.x) {
  __syncthreads();  // the scan storage of the previous chunk
  const int64_t e0 = c * kDeltaChunk + (int64_t)threadIdx.x * kDeltaPer;
  const int w = kW > 0 ? kW : d.width;
  uint64_t run[kDeltaPer];
  uint64_t sum = 0;
  if (kW > 0 && e0 + kDeltaPer <= d.nnz) {
    uint32_t wd[4 * (kW > 0 ? kW : 1)];
    const uint4* q = reinterpret_cast<const uint4*>(d.deltas + e0 * kW);
#pragma unroll
    for (int v = 0; v < (kW > 0 ? kW : 1); ++v) {
      const uint4 x = __ldcs(q + v);
      wd[4 * v] = x.x;
      wd[4 * v + 1] = x.y;
      wd[4 * v + 2] = x.z;
      wd[4 * v + 3] = x.w;
    }
#pragma unroll
    for (int i = 0; i < kDeltaPer; ++i) {
      uint64_t x = 0;
#pragma unroll
      for (int b = 0; b < (kW > 0 ? kW : 1); ++b) {
        const int at = i * kW + b;
        x |= (uint64_t)((wd[at >> 2] >> (8 * (at & 3))) & 0xffu) << (8 * b);
      }
      if (!(threadIdx.x | i)) x = 0;  // the chunk's first entry is its restart
      sum += x;
      run[i] = sum;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kDeltaPer; ++i) {
      const int64_t e = e0 + i;
      uint64_t x = 0;
      if (e < d.nnz && (threadIdx.x | i)) {  // the chunk's first entry is its restart
        const uint8_t* q = d.deltas + e * w;
        for (int b = 0; b < w; ++b) x |= (uint64_t)__ldcs(q + b) << (8 * b);
      }
      sum += x;
      run[i] = sum;
    }
  }
  uint64_t before;
  Scan(scan).ExclusiveSum(sum, before);
  const uint64_t base = d.restarts[c] + before;
  int flag = 0;
#pragma unroll
  for (int i = 0; i < kDeltaPer; ++i) {
    const int64_t e = e0 + i;
    if (e >= d.nnz) break;
    uint64_t k = base + run[i];
    int32_t ix[kMaxOrder];
    for (int n = d.order - 1; n > 0; --n) {
      // k < 2^53 (checked by the caller): the double quotient is off by at most one
      const uint64_t dn = (uint64_t)d.dims[n];
      uint64_t q = (uint64_t)((double)k * d.inv[n]);
      if (q * dn > k) --q;
      else if ((q + 1) * dn <= k) ++q;
      ix[n] = (int32_t)(k - q * dn);
      k = q;
    }
    flag |= k >= (uint64_t)d.dims[0];
    ix[0] = (int32_t)k;
    // streaming (evict-first) stores: this runs beside an epoch whose factor
    // rows live in L2
    for (int n = 0; n < d.order; ++n) __stcs(d.col[n] + e, ix[n]);
    if (d.rec)
      __stcs(d.rec + feistel_inv(e, d.nnz, d.bits, d.seed),
             make_int4(ix[0], ix[1], ix[2], __float_as_int(__ldcs(d.vals + e))));
  }
  if (flag) atomicExch(d.bad, 1);
  }
}

// ---- stream in last-mode runs -------------------------------------------------
//
// Order 3, option "runs": the cell's nonzeros are laid out in aligned chunks
// of kRun that share their last-mode index, the chunks in random order, so
// each epilogue warp of the J = R = 32 factor sweep (16 rows per mode) sums
// its rows' updates of that row and sends one RED instead of 16.  A
// 128-nonzero tile still spans 8 random rows (each row sees at most 16
// updates computed from one read per tile).  Built as: a Feistel shuffle
// (random order within a row), a stable radix sort by last-mode index (the
// index bits only), per-row chunk counts and two scans, then one scatter of
// whole records through a second Feistel bijection over the chunks.  A row's
// last < kRun nonzeros are pooled (by row) into mixed chunks; the one
// partial chunk of the cell stays last, so every chunk stays kRun-aligned.
constexpr int kRun = 16;

__global__ void runs_keys_kernel(const int4* __restrict__ rec, int64_t n, int bits, uint64_t seed,
                                 int32_t rows, uint32_t* __restrict__ keys,
                                 uint32_t* __restrict__ pos) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = feistel_perm(k, n, bits, seed);
    keys[k] = min((uint32_t)__ldg(&rec[p].z), (uint32_t)(rows - 1));  // range-checked later
    pos[k] = (uint32_t)p;
  }
}

// row start / end in the sorted keys (rows absent from the cell stay 0, 0)
__global__ void runs_bounds_kernel(const uint32_t* __restrict__ keys, int64_t n,
                                   uint32_t* __restrict__ rs, uint32_t* __restrict__ re) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = keys[k];
    if (k == 0 || keys[k - 1] != r) rs[r] = (uint32_t)k;
    if (k == n - 1 || keys[k + 1] != r) re[r] = (uint32_t)(k + 1);
  }
}

__global__ void runs_counts_kernel(const uint32_t* __restrict__ rs, const uint32_t* __restrict__ re,
                                   int32_t rows, uint32_t* __restrict__ full,
                                   uint32_t* __restrict__ left) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) {
    const uint32_t c = re[r] - rs[r];
    full[r] = c / kRun;
    left[r] = c % kRun;
  }
}

__global__ void runs_place_kernel(const int4* __restrict__ rec, const uint32_t* __restrict__ keys,
                                  const uint32_t* __restrict__ pos, const uint32_t* __restrict__ rs,
                                  const uint32_t* __restrict__ re, const uint32_t* __restrict__ fb,
                                  const uint32_t* __restrict__ lb, int32_t rows, ShuffleView v,
                                  int cbits, uint64_t seed) {
  const int64_t n = v.nnz, nc = n / kRun;  // whole chunks (permuted)
  const int64_t F = (int64_t)fb[rows - 1] + (re[rows - 1] - rs[rows - 1]) / kRun;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = keys[k];
    const int64_t o = k - rs[r], fl = (int64_t)(re[r] - rs[r]) / kRun * kRun;
    int64_t c, w;
    if (o < fl) {
      c = fb[r] + o / kRun;
      w = o % kRun;
    } else {
      const int64_t l = lb[r] + (o - fl);
      c = F + l / kRun;
      w = l % kRun;
    }
    const int64_t d = (c < nc ? feistel_perm(c, nc, cbits, seed) : c) * kRun + w;
    const int4 x = __ldg(rec + pos[k]);
    v.dst_idx[0][d] = x.x;
    v.dst_idx[1][d] = x.y;
    v.dst_idx[2][d] = x.z;
    v.dst_vals[d] = __int_as_float(x.w);
  }
}

// Scratch bytes of the runs build for n nonzeros and `rows` last-mode rows.
struct RunsScratch {
  size_t keys, keys2, pos, pos2, rs, re, full, left, fb, lb, temp, end;
};

RunsScratch runs_scratch_layout(int64_t n, int32_t rows, size_t temp) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  RunsScratch L{};
  size_t o = 0;
  L.keys = o; o += al(4 * (size_t)n);
  L.keys2 = o; o += al(4 * (size_t)n);
  L.pos = o; o += al(4 * (size_t)n);
  L.pos2 = o; o += al(4 * (size_t)n);
  L.rs = o; o += al(4 * (size_t)rows);
  L.re = o; o += al(4 * (size_t)rows);
  L.full = o; o += al(4 * (size_t)rows);
  L.left = o; o += al(4 * (size_t)rows);
  L.fb = o; o += al(4 * (size_t)rows);
  L.lb = o; o += al(4 * (size_t)rows);
  L.temp = o; o += al(temp);
  L.end = o;
  return L;
}

cudaError_t build_runs(DevTensor& t, const int4* rec, const ShuffleView& v, uint64_t seed,
                       cudaStream_t st) {
  const int64_t n = v.nnz;
  const int32_t rows = t.dims[2];
  int kb = 1;
  while ((1ll << kb) < rows) ++kb;
  size_t sort_temp = 0, s1 = 0, s2 = 0;
  cub::DoubleBuffer<uint32_t> dk(nullptr, nullptr), dp(nullptr, nullptr);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, sort_temp, dk, dp, (int)n, 0, kb, st);
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(nullptr, s1, (uint32_t*)nullptr, (uint32_t*)nullptr, rows, st);
  if (e != cudaSuccess) return e;
  s2 = s1 > sort_temp ? s1 : sort_temp;
  const RunsScratch L = runs_scratch_layout(n, rows, s2);
  if (L.end > t.runs_cap) {
    if (t.runs_scratch) cudaFree(t.runs_scratch);
    t.runs_scratch = nullptr;
    t.runs_cap = 0;
    e = cudaMalloc(&t.runs_scratch, L.end);
    if (e != cudaSuccess) return e;
    t.runs_cap = L.end;
  }
  uint8_t* b = static_cast<uint8_t*>(t.runs_scratch);
  auto u32 = [&](size_t off) { return reinterpret_cast<uint32_t*>(b + off); };
  int bits = 2;
  while ((1ll << bits) < n) bits += 2;
  int64_t blocks = (n + 255) / 256;
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  runs_keys_kernel<<<(int)blocks, 256, 0, st>>>(rec, n, bits, seed, rows, u32(L.keys),
                                                u32(L.pos));
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  cub::DoubleBuffer<uint32_t> keys(u32(L.keys), u32(L.keys2)), pos(u32(L.pos), u32(L.pos2));
  size_t tb = s2;
  e = cub::DeviceRadixSort::SortPairs(b + L.temp, tb, keys, pos, (int)n, 0, kb, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(b + L.rs, 0, L.full - L.rs, st);  // rs and re
  if (e != cudaSuccess) return e;
  runs_bounds_kernel<<<(int)blocks, 256, 0, st>>>(keys.Current(), n, u32(L.rs), u32(L.re));
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  runs_counts_kernel<<<(rows + 255) / 256, 256, 0, st>>>(u32(L.rs), u32(L.re), rows, u32(L.full),
                                                          u32(L.left));
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  tb = s2;
  e = cub::DeviceScan::ExclusiveSum(b + L.temp, tb, u32(L.full), u32(L.fb), rows, st);
  if (e != cudaSuccess) return e;
  tb = s2;
  e = cub::DeviceScan::ExclusiveSum(b + L.temp, tb, u32(L.left), u32(L.lb), rows, st);
  if (e != cudaSuccess) return e;
  const int64_t nc = n / kRun;
  int cbits = 2;
  while ((1ll << cbits) < nc) cbits += 2;
  runs_place_kernel<<<(int)blocks, 256, 0, st>>>(rec, keys.Current(), pos.Current(), u32(L.rs),
                                                 u32(L.re), u32(L.fb), u32(L.lb), rows, v, cbits,
                                                 seed * 0x2545f4914f6cdd1dull + 1);
  return cudaGetLastError();
}

// ---- shared-memory layout of the sweep kernels --------------------------------

struct HogLayout {
  int sum_j, b_in_smem;
  int aoff[kMaxOrder];  // offsets of mode blocks inside one G-row of a
  size_t o_b[kMaxOrder], o_bt[kMaxOrder];
  size_t o_warp, warp_floats, o_acc, acc_floats, end;  // floats
  int acc_global;  // per-warp gradient accumulators in global scratch (large J R)
};

constexpr size_t kHogSmemCap = 200 * 1024;

__host__ __device__ inline HogLayout hog_layout(const KView& v, bool core, int warps) {
  HogLayout L{};
  int s = 0;
  for (int n = 0; n < v.order; ++n) {
    L.aoff[n] = s;
    s += v.j[n];
  }
  L.sum_j = s;
  size_t o = 0;
  size_t bfloats = 0;
  for (int n = 0; n < v.order; ++n) bfloats += 2 * (size_t)v.j[n] * v.r;
  L.b_in_smem = bfloats * 4 <= 96 * 1024;
  if (L.b_in_smem) {
    for (int n = 0; n < v.order; ++n) {
      L.o_b[n] = o; o += (size_t)v.j[n] * v.r;
      L.o_bt[n] = o; o += (size_t)v.j[n] * v.r;
    }
  }
  // per warp: a[G][sum_j], c[G][N*R], d[G][N*R], x/res[G]
  L.o_warp = o;
  L.warp_floats = (size_t)kG * (s + 2 * v.order * v.r) + 2 * kG;
  o += L.warp_floats * warps;
  L.o_acc = o;
  L.acc_floats = core ? (size_t)s * v.r : 0;
  // J = R = 64 / 128: a warp's gradient (sum J x R floats) no longer fits
  // next to its siblings' in shared memory; it then lives in global scratch
  // (still one private accumulator per warp, so the sum stays deterministic).
  L.acc_global = (o + L.acc_floats * warps) * sizeof(float) > kHogSmemCap;
  if (!L.acc_global) o += L.acc_floats * warps;
  L.end = o;
  return L;
}

__device__ void load_b(const KView& v, const HogLayout& L, float* sm) {
  if (!L.b_in_smem) return;
  for (int n = 0; n < v.order; ++n) {
    const int jn = v.j[n], r = v.r;
    for (int e = threadIdx.x; e < jn * r; e += blockDim.x) {
      const int j = e / r, c = e - j * r;
      const float x = v.b[n][e];
      sm[L.o_b[n] + e] = x;
      sm[L.o_bt[n] + (size_t)c * jn + j] = x;
    }
  }
}

__device__ __forceinline__ float bval(const KView& v, const HogLayout& L, const float* sm,
                                      int n, int j, int c) {  // B_n[j][c]
  return L.b_in_smem ? sm[L.o_b[n] + (size_t)j * v.r + c] : __ldg(v.b[n] + (size_t)j * v.r + c);
}
__device__ __forceinline__ float btval(const KView& v, const HogLayout& L, const float* sm,
                                       int n, int c, int j) {  // B_n[j][c] via B^T
  return L.b_in_smem ? sm[L.o_bt[n] + (size_t)c * v.j[n] + j] : __ldg(v.b[n] + (size_t)j * v.r + c);
}

// Shared front half of both sweeps for G nonzeros starting at stream
// position e0: stage a rows, C, D, xhat and residual.  Returns through the
// per-warp scratch `w`: a rows at w[g*sum_j + aoff[n] + j], C at wc, D at wd,
// residuals at wres.
__device__ void front(const KView& v, const HogLayout& L, const float* sm, float* w,
                      int64_t e0, int nvalid, int32_t (&rows)[kG][kMaxOrder]) {
  const int lane = threadIdx.x & 31;
  const int N = v.order, r = v.r, sj = L.sum_j;
  float* wa = w;
  float* wc = w + kG * sj;
  float* wd = wc + kG * N * r;
  float* wx = wd + kG * N * r;
  float* wres = wx + kG;
  // indices + values: lane g*N+n loads idx[n][e0+g]
  {
    int32_t my = 0;
    float xv = 0.0f;
    const int g = lane / N, n = lane - g * N;
    if (g < kG && g < nvalid) my = v.idx[n][e0 + g];
    if (lane < kG && lane < nvalid) xv = v.vals[e0 + lane];
#pragma unroll
    for (int gg = 0; gg < kG; ++gg)
#pragma unroll
      for (int nn = 0; nn < kMaxOrder; ++nn)
        if (nn < N) rows[gg][nn] = __shfl_sync(0xffffffffu, my, gg * N + nn);
    if (lane < kG) wx[lane] = xv;
  }
  // stage a rows (coalesced: one warp reads whole rows)
#pragma unroll
  for (int g = 0; g < kG; ++g) {
    const bool ok = g < nvalid;
    for (int n = 0; n < N; ++n) {
      const int jn = v.j[n];
      const float* src = v.a[n] + (size_t)rows[g][n] * jn;
      for (int j = lane; j < jn; j += 32) wa[g * sj + L.aoff[n] + j] = ok ? src[j] : 0.0f;
    }
  }
  __syncwarp();
  // C^(n)[g][c] = sum_j a[g][n][j] B_n[j][c] (or the cached row, storage scheme)
  for (int n = 0; n < N; ++n) {
    const int jn = v.j[n];
    if (v.cc[n]) {
      for (int c = lane; c < r; c += 32)
#pragma unroll
        for (int g = 0; g < kG; ++g)
          wc[(g * N + n) * r + c] = g < nvalid ? v.cc[n][(size_t)rows[g][n] * r + c] : 0.0f;
      continue;
    }
    for (int c = lane; c < r; c += 32) {
      float acc[kG];
#pragma unroll
      for (int g = 0; g < kG; ++g) acc[g] = 0.0f;
      for (int j = 0; j < jn; ++j) {
        const float b = bval(v, L, sm, n, j, c);
#pragma unroll
        for (int g = 0; g < kG; ++g) acc[g] = fmaf(wa[g * sj + L.aoff[n] + j], b, acc[g]);
      }
#pragma unroll
      for (int g = 0; g < kG; ++g) wc[(g * N + n) * r + c] = acc[g];
    }
  }
  __syncwarp();
  // D and the C-side prediction xhat = sum_c C1 D1 (== A1 . U1, PAPER Eq. 14)
  float part[kG];
#pragma unroll
  for (int g = 0; g < kG; ++g) part[g] = 0.0f;
  for (int c = lane; c < r; c += 32) {
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      for (int n = 0; n < N; ++n) {
        float p = 1.0f;
        for (int k = 0; k < N; ++k)
          if (k != n) p *= wc[(g * N + k) * r + c];
        wd[(g * N + n) * r + c] = p;
        if (n == 0) part[g] = fmaf(wc[(g * N) * r + c], p, part[g]);
      }
    }
  }
#pragma unroll
  for (int g = 0; g < kG; ++g) {
    float s = part[g];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) wres[g] = (g < nvalid) ? wx[g] - s : 0.0f;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kHogThreads)
hog_factor_kernel(KView v, int64_t tmul, int64_t tadd, float lr, float reg,
                  int atomic_update) {
  extern __shared__ float sm[];
  if (v.tperm) {
    tmul = v.tperm[0];
    tadd = v.tperm[1];
  }
  const int warps = blockDim.x / 32;
  const HogLayout L = hog_layout(v, false, warps);
  load_b(v, L, sm);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* w = sm + L.o_warp + L.warp_floats * wid;
  const int N = v.order, r = v.r, sj = L.sum_j;
  const float* wa = w;
  const float* wd = w + kG * sj + kG * N * r;
  const float* wres = wd + kG * N * r + kG;
  const int64_t gw = (int64_t)blockIdx.x * warps + wid, nw = (int64_t)gridDim.x * warps;
  int32_t rows[kG][kMaxOrder];
  for (int64_t t = gw; t < v.ntiles; t += nw) {
    const int64_t tile = stream_tile(v, t, tmul, tadd);
    const int64_t base = tile * kHogTile;
    const int valid = v.tile_rows[tile];
    for (int g0 = 0; g0 < valid; g0 += kG) {
      front(v, L, sm, w, base + g0, valid - g0, rows);
      // U^(n)[g][j] = sum_c D[g][n][c] B_n[j][c]; a += lr (r u - reg a)
      for (int n = 0; n < N; ++n) {
        const int jn = v.j[n];
        for (int j = lane; j < jn; j += 32) {
          float u[kG];
#pragma unroll
          for (int g = 0; g < kG; ++g) u[g] = 0.0f;
          for (int c = 0; c < r; ++c) {
            const float b = btval(v, L, sm, n, c, j);
#pragma unroll
            for (int g = 0; g < kG; ++g) u[g] = fmaf(wd[(g * N + n) * r + c], b, u[g]);
          }
#pragma unroll
          for (int g = 0; g < kG; ++g) {
            if (g0 + g < valid) {
              const float a = wa[g * sj + L.aoff[n] + j];
              const float step = lr * (wres[g] * u[g] - reg * a);
              float* dst = v.a[n] + (size_t)rows[g][n] * jn + j;
              // Overwrite = the reference's rule (snapshot + step, last writer
              // wins); accumulate = lock-free RED.ADD, no update is lost when
              // thousands of warps hit the same short-mode row.
              if (atomic_update) atomicAdd(dst, step);
              else *dst = a + step;
            }
          }
        }
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kHogThreads)
hog_core_kernel(KView v, int64_t tmul, int64_t tadd, float* __restrict__ partials,
                float* __restrict__ gacc) {
  extern __shared__ float sm[];
  const int warps = blockDim.x / 32;
  const HogLayout L = hog_layout(v, true, warps);
  load_b(v, L, sm);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* acc = L.acc_global ? gacc + ((size_t)blockIdx.x * warps + wid) * L.acc_floats
                            : sm + L.o_acc + L.acc_floats * wid;
  for (size_t e = lane; e < L.acc_floats; e += 32) acc[e] = 0.0f;
  __syncthreads();
  float* w = sm + L.o_warp + L.warp_floats * wid;
  const int N = v.order, r = v.r, sj = L.sum_j;
  const float* wa = w;
  const float* wd = w + kG * sj + kG * N * r;
  const float* wres = wd + kG * N * r + kG;
  const int64_t gw = (int64_t)blockIdx.x * warps + wid, nw = (int64_t)gridDim.x * warps;
  int32_t rows[kG][kMaxOrder];
  for (int64_t t = gw; t < v.ntiles; t += nw) {
    const int64_t tile = stream_tile(v, t, tmul, tadd);
    const int64_t base = tile * kHogTile;
    const int valid = v.tile_rows[tile];
    for (int g0 = 0; g0 < valid; g0 += kG) {
      front(v, L, sm, w, base + g0, valid - g0, rows);
      // grad_n[j][c] += sum_g r_g a_g[j] D_g[c]
      int off = 0;
      for (int n = 0; n < N; ++n) {
        const int jn = v.j[n];
        for (int c = lane; c < r; c += 32) {
          float dd[kG];
#pragma unroll
          for (int g = 0; g < kG; ++g) dd[g] = wres[g] * wd[(g * N + n) * r + c];
          for (int j = 0; j < jn; ++j) {
            float s = acc[off + j * r + c];
#pragma unroll
            for (int g = 0; g < kG; ++g) s = fmaf(wa[g * sj + L.aoff[n] + j], dd[g], s);
            acc[off + j * r + c] = s;
          }
        }
        off += jn * r;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  // CTA reduction in warp order, then one partial per CTA.
  const float* accs = L.acc_global ? gacc + (size_t)blockIdx.x * warps * L.acc_floats : sm + L.o_acc;
  for (size_t e = threadIdx.x; e < L.acc_floats; e += blockDim.x) {
    float s = 0.0f;
    for (int k = 0; k < warps; ++k) s += accs[L.acc_floats * k + e];
    partials[(size_t)blockIdx.x * L.acc_floats + e] = s;
  }
}

// grad[e] = sum over CTAs in index order (deterministic).
__global__ void reduce_partials_kernel(const float* __restrict__ partials, int nparts,
                                       int len, float* __restrict__ grad) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < len; e += gridDim.x * blockDim.x) {
    float s = 0.0f;
    for (int k = 0; k < nparts; ++k) s += partials[(size_t)k * len + e];
    grad[e] = s;
  }
}

int hog_grid(int blocks_per_sm) { return num_sms() * (blocks_per_sm < 1 ? 1 : blocks_per_sm); }

}  // namespace

size_t shuffle_scratch_bytes(int64_t) { return 0; }

size_t hog_core_scratch_bytes(const KView& v, int blocks_per_sm) {
  const int warps = kHogThreads / 32;
  const HogLayout L = hog_layout(v, true, warps);
  const size_t grid = (size_t)hog_grid(blocks_per_sm);
  return grid * L.acc_floats * sizeof(float) * (1 + (L.acc_global ? warps : 0));
}

// Rows of each tile of a cell of n nonzeros: kHogTile, the last one the rest.
// Feistel parameters of a cell of n entries (as build_shuffled draws them).
static void cell_shuffle_params(int64_t n, uint64_t seed, int c, int* bits, uint64_t* cseed) {
  int b = 2;
  while ((1ll << b) < n) b += 2;
  *bits = b;
  *cseed = seed ^ (0x9e3779b97f4a7c15ull * (uint64_t)(c + 1));
}

__global__ void tile_rows_kernel(int32_t* __restrict__ rows, int64_t nt, int64_t n) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < nt) {
    const int64_t left = n - k * kHogTile;
    rows[k] = (int32_t)(left < kHogTile ? left : kHogTile);
  }
}

cudaError_t build_shuffled(DevTensor& t, const int64_t* d_perm, uint64_t seed,
                           void*, size_t, cudaStream_t st) {
  // Cells: every cell is shuffled on its own and padded to whole tiles
  // (index 0, value 0, masked by tile_rows), so a DSGD stratum is a
  // contiguous physical tile range.
  std::vector<int64_t> off = t.cell_off;
  if (off.empty() || d_perm) off = {0, t.nnz};
  const int ncell = (int)off.size() - 1;
  std::vector<int64_t> ctile(ncell + 1, 0);
  for (int c = 0; c < ncell; ++c)
    ctile[c + 1] = ctile[c] + (off[c + 1] - off[c] + kHogTile - 1) / kHogTile;
  const int64_t tiles = ctile[ncell];
  cudaError_t e;
  if (tiles > t.stream_cap || !t.svals) {
    for (int n = 0; n < t.order; ++n) {
      if (t.sidx[n]) cudaFree(t.sidx[n]);
      e = cudaMalloc(&t.sidx[n], sizeof(int32_t) * kHogTile * (tiles > 0 ? tiles : 1));
      if (e != cudaSuccess) return e;
    }
    if (t.svals) cudaFree(t.svals);
    if (t.tile_rows) cudaFree(t.tile_rows);
    e = cudaMalloc(&t.svals, sizeof(float) * kHogTile * (tiles > 0 ? tiles : 1));
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&t.tile_rows, sizeof(int32_t) * (tiles > 0 ? tiles : 1));
    if (e != cudaSuccess) return e;
    t.stream_cap = tiles;
  }
  if (t.order == 3 && t.rec16_cap < t.nnz) {
    if (t.rec16) cudaFree(t.rec16);
    t.rec16 = nullptr;
    e = cudaMalloc(&t.rec16, sizeof(int4) * (size_t)t.nnz);
    if (e != cudaSuccess) return e;
    t.rec16_cap = t.nnz;
  }
  for (int c = 0; c < ncell; ++c) {
    // the shuffle writes every valid entry: zero only the cell's padding
    // (index 0, value 0) instead of the whole stream
    const int64_t used = off[c + 1] - off[c], pad = (ctile[c + 1] - ctile[c]) * kHogTile - used;
    if (pad > 0) {
      const size_t p0 = (size_t)ctile[c] * kHogTile + used;
      for (int n = 0; n < t.order; ++n) {
        e = cudaMemsetAsync(t.sidx[n] + p0, 0, sizeof(int32_t) * pad, st);
        if (e != cudaSuccess) return e;
      }
      e = cudaMemsetAsync(t.svals + p0, 0, sizeof(float) * pad, st);
      if (e != cudaSuccess) return e;
    }
  }
  for (int c = 0; c < ncell; ++c) {
    const int64_t n = off[c + 1] - off[c];
    if (n == 0) continue;
    // rows per tile, written on the device: a host copy would queue behind
    // any bulk upload in flight on the copy engine
    const int64_t nt = ctile[c + 1] - ctile[c];
    tile_rows_kernel<<<(int)((nt + 255) / 256), 256, 0, st>>>(t.tile_rows + ctile[c], nt, n);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ShuffleView v{};
    v.order = t.order;
    for (int i = 0; i < t.order; ++i) {
      v.src_idx[i] = t.idx[i] + off[c];
      v.dst_idx[i] = t.sidx[i] + ctile[c] * kHogTile;
    }
    v.src_vals = t.vals + off[c];
    v.dst_vals = t.svals + ctile[c] * kHogTile;
    v.nnz = n;
    int bits;
    uint64_t cseed;
    cell_shuffle_params(n, seed, c, &bits, &cseed);
    int64_t blocks = (n + 255) / 256;
    if (blocks > num_sms() * 8) blocks = num_sms() * 8;
    if (t.order == 3) {
      pack16_kernel<<<(int)blocks, 256, 0, st>>>(v.src_idx[0], v.src_idx[1], v.src_idx[2],
                                                  v.src_vals, t.rec16 + off[c], n);
      if (t.runs && !t.keep_order && !d_perm && n >= 2 * kRun && n < (1ll << 31)) {
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        e = build_runs(t, t.rec16 + off[c], v, cseed, st);
        if (e != cudaSuccess) return e;
      } else {
        shuffle16_kernel<<<(int)blocks, 256, 0, st>>>(t.rec16 + off[c], v, d_perm,
                                                       (t.keep_order && !d_perm) ? -1 : bits, cseed);
      }
    } else {
      shuffle_kernel<<<(int)blocks, 256, 0, st>>>(v, d_perm, bits, cseed);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  t.cell_tile = ctile;
  t.stream_tiles = tiles;
  t.shuffled = true;
  return cudaSuccess;
}

cudaError_t prepare_scatter_stream(DevTensor& t) {
  const int64_t tiles = (t.nnz + kHogTile - 1) / kHogTile;
  cudaError_t e;
  if (tiles > t.stream_cap || !t.svals) {
    for (int n = 0; n < t.order; ++n) {
      if (t.sidx[n]) cudaFree(t.sidx[n]);
      e = cudaMalloc(&t.sidx[n], sizeof(int32_t) * kHogTile * tiles);
      if (e != cudaSuccess) return e;
    }
    if (t.svals) cudaFree(t.svals);
    if (t.tile_rows) cudaFree(t.tile_rows);
    e = cudaMalloc(&t.svals, sizeof(float) * kHogTile * tiles);
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&t.tile_rows, sizeof(int32_t) * tiles);
    if (e != cudaSuccess) return e;
    t.stream_cap = tiles;
  }
  if (t.rec16_cap < t.nnz) {
    if (t.rec16) cudaFree(t.rec16);
    t.rec16 = nullptr;
    e = cudaMalloc(&t.rec16, sizeof(int4) * (size_t)t.nnz);
    if (e != cudaSuccess) return e;
    t.rec16_cap = t.nnz;
  }
  return cudaSuccess;
}

cudaError_t launch_delta_decode(DevTensor& t, const uint8_t* deltas, const uint64_t* restarts,
                                int width, int64_t c0, int64_t c1, bool scatter, uint64_t seed,
                                int* bad, cudaStream_t st) {
  if (c1 <= c0) return cudaSuccess;
  DeltaDecode d{};
  d.deltas = deltas;
  d.restarts = restarts;
  d.vals = t.vals;
  d.order = t.order;
  d.width = width;
  d.nnz = t.nnz;
  d.bad = bad;
  for (int n = 0; n < t.order; ++n) {
    d.col[n] = t.idx[n];
    d.dims[n] = t.dims[n];
    d.inv[n] = 1.0 / (double)t.dims[n];
  }
  if (scatter && t.order == 3) {
    d.rec = t.rec16;
    cell_shuffle_params(t.nnz, seed, 0, &d.bits, &d.seed);
  }
  // a capped grid (a few blocks per SM) when the decode runs beside an
  // epoch: fewer resident blocks take fewer issue slots from its sweeps
  static const int64_t cap = [] {
    const char* e = getenv("FTKCU_DECODE_GRID");
    return e ? atoll(e) : 0ll;
  }();
  int64_t grid = c1 - c0;
  if (cap > 0 && grid > cap) grid = cap;
  switch (width) {
    case 3: delta_decode_kernel<3><<<(unsigned)grid, kDeltaThreads, 0, st>>>(d, c0, c1); break;
    case 4: delta_decode_kernel<4><<<(unsigned)grid, kDeltaThreads, 0, st>>>(d, c0, c1); break;
    case 2: delta_decode_kernel<2><<<(unsigned)grid, kDeltaThreads, 0, st>>>(d, c0, c1); break;
    default: delta_decode_kernel<0><<<(unsigned)grid, kDeltaThreads, 0, st>>>(d, c0, c1); break;
  }
  return cudaGetLastError();
}

// The scattered records (prepare_scatter_stream, launch_delta_decode with
// scatter) -> the single-cell tile stream build_shuffled(seed) would build.
cudaError_t finish_scatter_stream(DevTensor& t, cudaStream_t st) {
  const int64_t n = t.nnz, tiles = (n + kHogTile - 1) / kHogTile, pad = tiles * kHogTile - n;
  cudaError_t e;
  if (pad > 0) {
    for (int i = 0; i < t.order; ++i) {
      e = cudaMemsetAsync(t.sidx[i] + n, 0, sizeof(int32_t) * pad, st);
      if (e != cudaSuccess) return e;
    }
    e = cudaMemsetAsync(t.svals + n, 0, sizeof(float) * pad, st);
    if (e != cudaSuccess) return e;
  }
  tile_rows_kernel<<<(int)((tiles + 255) / 256), 256, 0, st>>>(t.tile_rows, tiles, n);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ShuffleView v{};
  v.order = t.order;
  for (int i = 0; i < t.order; ++i) v.dst_idx[i] = t.sidx[i];
  v.dst_vals = t.svals;
  v.nnz = n;
  int64_t blocks = (n + 255) / 256;
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  shuffle16_kernel<<<(int)blocks, 256, 0, st>>>(t.rec16, v, nullptr, -1, 0);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  t.cell_tile = {0, tiles};
  t.stream_tiles = tiles;
  t.runs = false;
  t.shuffled = true;
  return cudaSuccess;
}

cudaError_t launch_hog_factor(const KView& v, int64_t tile_mul, int64_t tile_add,
                              float lr_a, float reg_a, int blocks_per_sm, int atomic_update,
                              cudaStream_t st) {
  const int warps = kHogThreads / 32;
  const HogLayout L = hog_layout(v, false, warps);
  const size_t bytes = L.end * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(hog_factor_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  if (v.ntiles == 0) return cudaSuccess;
  hog_factor_kernel<<<(int)sweep_grid(v, blocks_per_sm < 1 ? 1 : blocks_per_sm), kHogThreads,
                      bytes, st>>>(
      v, tile_mul, tile_add, lr_a, reg_a, atomic_update);
  return cudaGetLastError();
}

cudaError_t launch_hog_core(const KView& v, int64_t tile_mul, int64_t tile_add,
                            float* grad, int blocks_per_sm, float* scratch,
                            size_t scratch_bytes, cudaStream_t st) {
  const int warps = kHogThreads / 32;
  const HogLayout L = hog_layout(v, true, warps);
  const size_t bytes = L.end * sizeof(float);
  const int grid = hog_grid(blocks_per_sm);
  if (scratch_bytes < hog_core_scratch_bytes(v, blocks_per_sm)) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(hog_core_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  float* gacc = scratch + (size_t)grid * L.acc_floats;
  hog_core_kernel<<<grid, kHogThreads, bytes, st>>>(v, tile_mul, tile_add, scratch, gacc);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int len = (int)L.acc_floats;
  reduce_partials_kernel<<<(len + 255) / 256, 256, 0, st>>>(scratch, grid, len, grad);
  return cudaGetLastError();
}

}  // namespace ftkcu
