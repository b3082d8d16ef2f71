// Tensor-core (tcgen05, kind::tf32) Hogwild sweeps for sm_100a.
//
// One persistent CTA per SM (4 warps = 128 threads; thread t owns nonzero t
// of a 128-nonzero tile and TMEM lane t).  Per tile:
//
//   gather   cp.async (LDGSTS) 16-B chunks of the N factor rows of every
//            nonzero straight into the UMMA K-major swizzled layout
//            (8 lanes per 128-B row: fully coalesced), S-stage ring,
//            completion on an mbarrier (cp.async.mbarrier.arrive);
//   C = A B  tcgen05.mma 128 x R x J per mode into TMEM (Alg. 4 line 4);
//   D, r     tcgen05.ld C rows -> thread-local Hadamard products, x_hat =
//            C1 . D1, residual r = x - x_hat (Eq. 14);
// factor sweep:
//   U = D B^T  D stored to TMEM (tcgen05.st), tcgen05.mma with A from TMEM;
//   update   a' = a + lr (r u - reg a) per row, then warp-cooperative
//            128-B vector RED.ADD (or STG) of whole rows back to HBM;
// core sweep:
//   G += A^T (r D)  tcgen05.mma with MN-major operands straight from the
//            gathered tile (rows = nonzeros) and the r-scaled D rows:
//            M = stacked modes (sum J <= 128), N = R, K = 128 nonzeros,
//            accumulated in TMEM over every tile the CTA visits (Eq. 15);
//            CTA partials reduced in a fixed order afterwards.
//
// Algorithm reference: decomposition.cpp:644-658 / :678-698 (the per-batch
// pipeline) and PAPER.md Alg. 4/5; SURVEY.md §7 step 4 for this design.
#include <cstdio>
#include <cstdlib>

#include "engine.cuh"
#include "tc_common.cuh"

namespace ftkcu {
namespace {
using namespace tc;

constexpr int kThreads = 128;
constexpr int kTileRows = 128;  // == kHogTile
constexpr int kStages = 3;

static_assert(kTileRows == kHogTile, "tile size shared with the CUDA-core path");

// Ranks below 16 (J or R = 8) run padded to 16: the padding columns of the
// operand tiles are zero (set once, never written), so they add exact zeros
// to every contraction; the C GEMM skips the all-zero K steps.
template <int N, int J, int R, bool kCore>
struct TcLayout {
  static constexpr int JP = J < 16 ? 16 : J, RP = R < 16 ? 16 : R;
  static constexpr uint32_t PJ = JP * 4, PR = RP * 4;
  // factor sweep: per-mode K-major tiles of 128 rows x PJ bytes (SW128/SW64)
  static constexpr uint32_t kA = kTileRows * PJ;
  // core sweep: stacked rows j' = n J + j in 128-B segments (BASE32B layout)
  static constexpr uint32_t kSeg = kTileRows * 128;
  static constexpr uint32_t NS = (N * JP + 31) / 32;   // A segments per row
  static constexpr uint32_t NSD = (N * RP + 31) / 32;  // D segments per row
  static constexpr uint32_t kSlot = kCore ? NS * kSeg : N * kA;
  static constexpr uint32_t kBt = RP * PJ;               // B^T per mode (C GEMM operand)
  static constexpr uint32_t kB = kCore ? 0 : JP * PR;    // B per mode (U GEMM operand)
  // The core G GEMM reads M = 128 stacked rows = 4 segments: the (4 - NS)
  // garbage segments past a slot must still be inside shared memory.
  static constexpr uint32_t kOverrun = kCore ? (4 - NS) * kSeg : 0;
  static constexpr uint32_t o_a = 0;
  static constexpr uint32_t o_d = o_a + kStages * kSlot;
  static constexpr uint32_t d_bytes = kCore ? NSD * kSeg : 0;
  static constexpr uint32_t pad = kOverrun > d_bytes ? kOverrun - d_bytes : 0;
  static constexpr uint32_t o_bt = o_d + d_bytes + pad;
  static constexpr uint32_t o_btlo = o_bt + N * kBt;     // low tf32 half of B^T
  static constexpr uint32_t o_b = o_btlo + N * kBt;
  static constexpr uint32_t o_idx = o_b + N * kB;
  static constexpr uint32_t o_val = o_idx + kStages * N * kTileRows * 4;
  static constexpr uint32_t o_bar = (o_val + kStages * kTileRows * 4 + 7) / 8 * 8;
  static constexpr uint32_t o_tmem = o_bar + (kStages + 1) * 8;
  static constexpr uint32_t bytes = o_tmem + 16 + 1024;  // + alignment slack
  // TMEM columns: C (then U in the factor sweep); D (factor) or G (core);
  // the core sweep's copy of the gathered rows (A operand of its C GEMM).
  static constexpr uint32_t t_c = 0;
  static constexpr uint32_t t_x = kCore ? N * RP : N * (RP > JP ? RP : JP);
  static constexpr uint32_t t_a = t_x + N * RP;                      // core: A rows (hi)
  static constexpr uint32_t t_alo = t_a + (kCore ? NS * 32 : 0);     // A rows, low part
  static constexpr uint32_t cols_used = t_alo + (kCore ? NS * 32 : N * JP);
  static constexpr uint32_t cols = cols_used <= 32 ? 32 : cols_used <= 64 ? 64
                                   : cols_used <= 128 ? 128 : cols_used <= 256 ? 256 : 512;
  static_assert(bytes <= 227 * 1024, "shared-memory budget");
  static_assert(cols_used <= 512, "TMEM budget");
  static_assert(!kCore || N * JP <= 128, "stacked core-gradient rows exceed M = 128");
};

struct TcParams {
  const int32_t* idx[kMaxOrder];
  const float* vals;
  float* a[kMaxOrder];
  const float* b[kMaxOrder];
  int64_t nnz, ntiles, tmul, tadd, tile_base;
  const int32_t* tile_rows;
  const int64_t* tperm;  // device {mul, add} or null (KView::tperm)
  int max_ctas;  // factor sweeps: grid cap (KView::max_ctas)
  float lr, reg;
  int atomic_update;
  int prec3;  // split-tf32 (hi*hi + hi*lo + lo*hi) for the C = A B contraction
  float* partials;
  float* dbg;  // optional per-row debug dump of CTA 0's first tile
};

// Loads B^(n) into the swizzled operand tiles (once per CTA).
template <int N, int J, int R, bool kCore>
__device__ void load_b_tiles(const TcParams& p, uint8_t* sm) {
  using L = TcLayout<N, J, R, kCore>;
  for (int n = 0; n < N; ++n) {
    const float* b = p.b[n];
    for (int e = threadIdx.x; e < L::JP * L::RP; e += kThreads) {
      const int j = e / L::RP, r = e - j * L::RP;
      const float x = (j < J && r < R) ? b[j * R + r] : 0.0f;
      const float hi = tf32_rna(x), lo = tf32_rna(x - hi);
      // C GEMM B operand: rows r, K = j (hi and lo tf32 halves).
      *reinterpret_cast<float*>(sm + L::o_bt + n * L::kBt + swz(r, j * 4, L::PJ)) = hi;
      *reinterpret_cast<float*>(sm + L::o_btlo + n * L::kBt + swz(r, j * 4, L::PJ)) = lo;
      if constexpr (!kCore)  // U GEMM B operand: rows j, K = r.
        *reinterpret_cast<float*>(sm + L::o_b + n * L::kB + swz(j, r * 4, L::PR)) = hi;
    }
  }
}

// Register prefetch of one tile's COO record for this thread's row.
template <int N>
struct Rec {
  int32_t idx[N];
  float x;
  bool ok;
};

template <int N>
__device__ __forceinline__ Rec<N> load_rec(const TcParams& p, int64_t tile) {
  Rec<N> r;
  const int64_t e = tile * kTileRows + threadIdx.x;
  r.ok = (int)threadIdx.x < p.tile_rows[tile];
#pragma unroll
  for (int n = 0; n < N; ++n) r.idx[n] = r.ok ? __ldcs(p.idx[n] + e) : 0;
  r.x = r.ok ? __ldcs(p.vals + e) : 0.0f;
  return r;
}

__device__ __forceinline__ int64_t phys_tile(const TcParams& p, int64_t k) {
  const int64_t t = (int64_t)blockIdx.x + k * gridDim.x;
  const int64_t mul = p.tperm ? __ldg(p.tperm) : p.tmul;
  const int64_t add = p.tperm ? __ldg(p.tperm + 1) : p.tadd;
  return p.tile_base + (t * mul + add) % p.ntiles;
}

// Stages one tile into `slot`: COO record to smem, factor rows by cp.async
// into the swizzled K-major tiles, completion counted on full_bar.
template <int N, int J, int R, bool kCore>
__device__ void stage_tile(const TcParams& p, uint8_t* sm, int slot, const Rec<N>& rec,
                           uint64_t* full_bar) {
  using L = TcLayout<N, J, R, kCore>;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int32_t* s_idx = reinterpret_cast<int32_t*>(sm + L::o_idx) + slot * N * kTileRows;
  float* s_val = reinterpret_cast<float*>(sm + L::o_val) + slot * kTileRows;
#pragma unroll
  for (int n = 0; n < N; ++n) s_idx[n * kTileRows + t] = rec.ok ? rec.idx[n] : -1;
  s_val[t] = rec.x;
  // 8-lane (J=32) or 4-lane (J=16) groups copy whole rows of this warp.
  constexpr int kChunks = J / 4;           // 16-B chunks per row
  constexpr int kRowsPer = 32 / kChunks;   // rows per warp instruction
  const uint32_t a_base = smem_u32(sm + L::o_a + slot * L::kSlot);
#pragma unroll
  for (int n = 0; n < N; ++n) {
    const float* src = p.a[n];
#pragma unroll
    for (int i = 0; i < 32 / kRowsPer; ++i) {
      const int rl = i * kRowsPer + lane / kChunks;  // row within this warp
      const int ch = lane % kChunks;
      const int32_t g = __shfl_sync(0xffffffffu, rec.idx[n], rl);
      const int row = warp * 32 + rl;
      uint32_t dst;
      if constexpr (kCore) {  // stacked row byte n J 4 + 16 ch, BASE32B segments
        const uint32_t byte = n * L::JP * 4 + ch * 16;
        dst = (byte >> 7) * L::kSeg + swz32(row, byte & 127);
      } else {
        dst = n * L::kA + swz(row, ch * 16, L::PJ);
      }
      cp_async16(a_base + dst, src + (size_t)g * J + ch * 4);
    }
  }
  cp_async_arrive(full_bar);
}

template <int N, int J, int R, bool kCore>
__device__ void cta_setup(const TcParams& p, uint8_t* sm, uint64_t* bars, uint32_t* tmem_slot) {
  using L = TcLayout<N, J, R, kCore>;
  load_b_tiles<N, J, R, kCore>(p, sm);
  if constexpr (J < 16)  // padding columns of the gathered rows stay zero
    for (uint32_t o = threadIdx.x * 16; o < kStages * L::kSlot; o += kThreads * 16)
      *reinterpret_cast<int4*>(sm + L::o_a + o) = make_int4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], kThreads);
    mbar_init(&bars[kStages], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(L::cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_before();
  __syncthreads();
  tc_after();
}

template <int N, int J, int R, bool kCore>
__device__ void cta_teardown(uint32_t tmem) {
  using L = TcLayout<N, J, R, kCore>;
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(L::cols));
}

// C^(n) = A_psi^(n) B^(n) for all modes into TMEM columns [t_c + n R).
template <int N, int J, int R, bool kCore>
__device__ __forceinline__ void issue_c(uint8_t* sm, int slot, uint32_t tmem, int prec3) {
  using L = TcLayout<N, J, R, kCore>;
  constexpr uint32_t id = idesc_tf32(128, L::RP, 0, 0);
  const uint32_t a0 = smem_u32(sm + L::o_a + slot * L::kSlot);
  const uint32_t b0 = smem_u32(sm + L::o_bt);
  const uint32_t bl = smem_u32(sm + L::o_btlo);
#pragma unroll
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int ks = 0; ks < J / 8; ++ks) {
      const uint64_t da = sdesc(a0 + n * L::kA + ks * 32, 16, 8 * L::PJ, L::PJ);
      mma_ss(tmem + L::t_c + n * L::RP, da, sdesc(b0 + n * L::kBt + ks * 32, 16, 8 * L::PJ, L::PJ),
             id, ks > 0);
      if (prec3) {
        mma_ss(tmem + L::t_c + n * L::RP, da,
               sdesc(bl + n * L::kBt + ks * 32, 16, 8 * L::PJ, L::PJ), id, 1);
        mma_ts(tmem + L::t_c + n * L::RP, tmem + L::t_alo + n * L::JP + ks * 8,
               sdesc(b0 + n * L::kBt + ks * 32, 16, 8 * L::PJ, L::PJ), id, 1);
      }
    }
}

// Split-tf32 support: this thread's factor rows minus their truncated tf32
// part, into TMEM (A operand of the lo*hi MMA).
template <int N, int J, int R>
__device__ __forceinline__ void stage_alo_factor(const uint8_t* tile, uint32_t tlane) {
  using L = TcLayout<N, J, R, false>;
  const int t = threadIdx.x;
#pragma unroll
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int h = 0; h < L::JP / 16; ++h) {
      uint32_t v[16];
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const float4 x = *reinterpret_cast<const float4*>(
            tile + n * L::kA + swz(t, (h * 16 + q4 * 4) * 4, L::PJ));
        v[q4 * 4 + 0] = __float_as_uint(x.x - tf32_trunc(x.x));
        v[q4 * 4 + 1] = __float_as_uint(x.y - tf32_trunc(x.y));
        v[q4 * 4 + 2] = __float_as_uint(x.z - tf32_trunc(x.z));
        v[q4 * 4 + 3] = __float_as_uint(x.w - tf32_trunc(x.w));
      }
      tmem_st16(tlane + L::t_alo + n * L::JP + h * 16, v);
    }
  tmem_wait_st();
}

// Reads C rows, forms D (thread-local) and the C-side prediction.
template <int N, int R>
__device__ __forceinline__ void load_c_form_d(uint32_t tcol, float (&c)[N][R], float& xhat) {
#pragma unroll
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int h = 0; h < R / 16; ++h) {
      uint32_t v[16];
      tmem_ld16(tcol + n * R + h * 16, v);
      tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 16; ++q) c[n][h * 16 + q] = __uint_as_float(v[q]);
    }
  xhat = 0.0f;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float d0 = 1.0f;
#pragma unroll
    for (int k = 1; k < N; ++k) d0 *= c[k][r];
    xhat = fmaf(c[0][r], d0, xhat);
  }
}

template <int N, int R>
__device__ __forceinline__ float d_of(const float (&c)[N][R], int n, int r) {
  float d = 1.0f;
#pragma unroll
  for (int k = 0; k < N; ++k)
    if (k != n) d *= c[k][r];
  return d;
}

// ---- factor sweep ---------------------------------------------------------------

template <int N, int J, int R>
__global__ void __launch_bounds__(kThreads, 1) tc_factor_kernel(TcParams p) {
  using L = TcLayout<N, J, R, false>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::o_bar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::o_tmem);
  cta_setup<N, J, R, false>(p, sm, bars, tmem_slot);
  const uint32_t tmem = *tmem_slot;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t tlane = tmem + ((uint32_t)(warp * 32) << 16);
  const int64_t nk = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  uint32_t mma_phase = 0;

  Rec<N> rec;
  if (nk > 0) rec = load_rec<N>(p, phys_tile(p, 0));
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) {
      stage_tile<N, J, R, false>(p, sm, s, rec, &bars[s]);
      if (s + 1 < nk) rec = load_rec<N>(p, phys_tile(p, s + 1));
    }
  }
  for (int64_t k = 0; k < nk; ++k) {
    const int64_t kk = k + kStages - 1;
    if (kk < nk) {
      stage_tile<N, J, R, false>(p, sm, (int)(kk % kStages), rec, &bars[kk % kStages]);
      if (kk + 1 < nk) rec = load_rec<N>(p, phys_tile(p, kk + 1));
    }
    const int slot = (int)(k % kStages);
    mbar_wait(&bars[slot], (uint32_t)((k / kStages) & 1));
    if (p.prec3) stage_alo_factor<N, J, R>(sm + L::o_a + slot * L::kSlot, tlane);
    fence_proxy_async();
    tc_before();
    __syncthreads();
    if (t == 0) {
      tc_after();
      issue_c<N, J, R, false>(sm, slot, tmem, p.prec3);
      mma_commit(&bars[kStages]);
    }
    mbar_wait(&bars[kStages], mma_phase);
    mma_phase ^= 1;
    tc_after();

    const float* s_val = reinterpret_cast<const float*>(sm + L::o_val) + slot * kTileRows;
    const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx) + slot * N * kTileRows;
    const bool ok = s_idx[t] >= 0;
    constexpr int RP = L::RP, JP = L::JP;
    float c[N][RP], xhat;
    load_c_form_d<N, RP>(tlane + L::t_c, c, xhat);
    const float resid = ok ? s_val[t] - xhat : 0.0f;
    // D^(n) -> TMEM (A operand of the U GEMM).
#pragma unroll
    for (int n = 0; n < N; ++n)
#pragma unroll
      for (int h = 0; h < RP / 16; ++h) {
        uint32_t v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = __float_as_uint(d_of<N, RP>(c, n, h * 16 + q)) + 0x1000u;
        tmem_st16(tlane + L::t_x + n * RP + h * 16, v);
      }
    tmem_wait_st();
    tc_before();
    __syncthreads();
    if (t == 0) {
      tc_after();
      constexpr uint32_t id = idesc_tf32(128, JP, 0, 0);
      const uint32_t b0 = smem_u32(sm + L::o_b);
#pragma unroll
      for (int n = 0; n < N; ++n)
#pragma unroll
        for (int ks = 0; ks < R / 8; ++ks)
          mma_ts(tmem + L::t_c + n * JP, tmem + L::t_x + n * RP + ks * 8,
                 sdesc(b0 + n * L::kB + ks * 32, 16, 8 * L::PR, L::PR), id, ks > 0);
      mma_commit(&bars[kStages]);
    }
    mbar_wait(&bars[kStages], mma_phase);
    mma_phase ^= 1;
    tc_after();

    // a' = a + lr (r u - reg a): this thread's row, in place in the tile.
    uint8_t* a_tile = sm + L::o_a + slot * L::kSlot;
#pragma unroll
    for (int n = 0; n < N; ++n) {
#pragma unroll
      for (int h = 0; h < JP / 16; ++h) {
        uint32_t v[16];
        tmem_ld16(tlane + L::t_c + n * JP + h * 16, v);
        tmem_wait_ld();
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          float4* cell = reinterpret_cast<float4*>(a_tile + n * L::kA +
                                                   swz(t, (h * 16 + q4 * 4) * 4, L::PJ));
          float4 a = *cell;
          float4 s;
          s.x = p.lr * (resid * __uint_as_float(v[q4 * 4 + 0]) - p.reg * a.x);
          s.y = p.lr * (resid * __uint_as_float(v[q4 * 4 + 1]) - p.reg * a.y);
          s.z = p.lr * (resid * __uint_as_float(v[q4 * 4 + 2]) - p.reg * a.z);
          s.w = p.lr * (resid * __uint_as_float(v[q4 * 4 + 3]) - p.reg * a.w);
          if (!p.atomic_update) {
            s.x += a.x;
            s.y += a.y;
            s.z += a.z;
            s.w += a.w;
          }
          *cell = s;
        }
      }
    }
    __syncwarp();
    // Warp-cooperative write-back of this warp's 32 rows: whole 128-B (64-B)
    // rows per 8 (4) lanes, vector RED.ADD (Hogwild accumulate) or STG.
    constexpr int kChunks = J / 4, kRowsPer = 32 / kChunks;
#pragma unroll
    for (int n = 0; n < N; ++n) {
      float* dst = p.a[n];
#pragma unroll
      for (int i = 0; i < 32 / kRowsPer; ++i) {
        const int row = warp * 32 + i * kRowsPer + lane / kChunks;
        const int ch = lane % kChunks;
        const int32_t g = s_idx[n * kTileRows + row];
        if (g >= 0) {
          const float4 v =
              *reinterpret_cast<const float4*>(a_tile + n * L::kA + swz(row, ch * 16, L::PJ));
          float* gp = dst + (size_t)g * J + ch * 4;
          if (p.atomic_update)
            red_add_v4(gp, v);
          else
            *reinterpret_cast<float4*>(gp) = v;
        }
      }
    }
    tc_before();
    __syncthreads();  // slot and TMEM free for the next tile
    tc_after();
  }
  cta_teardown<N, J, R, false>(tmem);
}

// ---- core sweep -------------------------------------------------------------------

template <int N, int J, int R>
__global__ void __launch_bounds__(kThreads, 1) tc_core_kernel(TcParams p) {
  using L = TcLayout<N, J, R, true>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::o_bar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::o_tmem);
  cta_setup<N, J, R, true>(p, sm, bars, tmem_slot);
  const uint32_t tmem = *tmem_slot;
  const int t = threadIdx.x, warp = t >> 5;
  const uint32_t tlane = tmem + ((uint32_t)(warp * 32) << 16);
  const int64_t nk = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  uint32_t mma_phase = 0;

  Rec<N> rec;
  if (nk > 0) rec = load_rec<N>(p, phys_tile(p, 0));
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) {
      stage_tile<N, J, R, true>(p, sm, s, rec, &bars[s]);
      if (s + 1 < nk) rec = load_rec<N>(p, phys_tile(p, s + 1));
    }
  }
  for (int64_t k = 0; k < nk; ++k) {
    const int64_t kk = k + kStages - 1;
    if (kk < nk) {
      stage_tile<N, J, R, true>(p, sm, (int)(kk % kStages), rec, &bars[kk % kStages]);
      if (kk + 1 < nk) rec = load_rec<N>(p, phys_tile(p, kk + 1));
    }
    const int slot = (int)(k % kStages);
    mbar_wait(&bars[slot], (uint32_t)((k / kStages) & 1));
    // Own stacked row -> TMEM (A operand of the C GEMM): the smem tile is in
    // the MN-major layout the G GEMM needs, which K-major reads cannot use.
    {
      const uint8_t* tile = sm + L::o_a + slot * L::kSlot;
#pragma unroll
      for (int sg = 0; sg < (int)L::NS; ++sg)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t v[16];
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const float4 x = *reinterpret_cast<const float4*>(
                tile + sg * L::kSeg + swz32(t, (h * 16 + q4 * 4) * 4));
            v[q4 * 4 + 0] = __float_as_uint(x.x);
            v[q4 * 4 + 1] = __float_as_uint(x.y);
            v[q4 * 4 + 2] = __float_as_uint(x.z);
            v[q4 * 4 + 3] = __float_as_uint(x.w);
          }
          if (!p.prec3)
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] += 0x1000u;  // round, don't truncate
          tmem_st16(tlane + L::t_a + sg * 32 + h * 16, v);
          if (p.prec3) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const float x = __uint_as_float(v[q]);
              v[q] = __float_as_uint(x - tf32_trunc(x));
            }
            tmem_st16(tlane + L::t_alo + sg * 32 + h * 16, v);
          }
        }
      tmem_wait_st();
    }
    fence_proxy_async();
    tc_before();
    __syncthreads();
    if (t == 0) {
      tc_after();
      constexpr uint32_t id = idesc_tf32(128, L::RP, 0, 0);
      const uint32_t b0 = smem_u32(sm + L::o_bt);
      const uint32_t bl = smem_u32(sm + L::o_btlo);
#pragma unroll
      for (int n = 0; n < N; ++n)
#pragma unroll
        for (int ks = 0; ks < J / 8; ++ks)
        {
          const uint64_t db = sdesc(b0 + n * L::kBt + ks * 32, 16, 8 * L::PJ, L::PJ);
          mma_ts(tmem + L::t_c + n * L::RP, tmem + L::t_a + n * L::JP + ks * 8, db, id, ks > 0);
          if (p.prec3) {
            mma_ts(tmem + L::t_c + n * L::RP, tmem + L::t_a + n * L::JP + ks * 8,
                   sdesc(bl + n * L::kBt + ks * 32, 16, 8 * L::PJ, L::PJ), id, 1);
            mma_ts(tmem + L::t_c + n * L::RP, tmem + L::t_alo + n * L::JP + ks * 8, db, id, 1);
          }
        }
      mma_commit(&bars[kStages]);
    }
    mbar_wait(&bars[kStages], mma_phase);
    mma_phase ^= 1;
    tc_after();

    const float* s_val = reinterpret_cast<const float*>(sm + L::o_val) + slot * kTileRows;
    const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx) + slot * N * kTileRows;
    const bool ok = s_idx[t] >= 0;
    constexpr int RP = L::RP, JP = L::JP;
    float c[N][RP], xhat;
    load_c_form_d<N, RP>(tlane + L::t_c, c, xhat);
    const float resid = ok ? s_val[t] - xhat : 0.0f;
    if (p.dbg && blockIdx.x == 0 && k == 0) {
      p.dbg[t * 8 + 0] = resid;
      p.dbg[t * 8 + 1] = xhat;
      p.dbg[t * 8 + 2] = c[0][0];
      p.dbg[t * 8 + 3] = c[1][0];
      p.dbg[t * 8 + 4] = s_val[t];
      p.dbg[t * 8 + 5] = (float)s_idx[t];
    }
    // r-scaled D rows -> smem (N-major B operand of the G GEMM).
#pragma unroll
    for (int n = 0; n < N; ++n)
#pragma unroll
      for (int q4 = 0; q4 < RP / 4; ++q4) {
        float4 d;
        // + half a tf32 ulp: the tensor core's truncation becomes rounding
        d.x = __uint_as_float(__float_as_uint(resid * d_of<N, RP>(c, n, q4 * 4 + 0)) + 0x1000u);
        d.y = __uint_as_float(__float_as_uint(resid * d_of<N, RP>(c, n, q4 * 4 + 1)) + 0x1000u);
        d.z = __uint_as_float(__float_as_uint(resid * d_of<N, RP>(c, n, q4 * 4 + 2)) + 0x1000u);
        d.w = __uint_as_float(__float_as_uint(resid * d_of<N, RP>(c, n, q4 * 4 + 3)) + 0x1000u);
        const uint32_t byte = (n * RP + q4 * 4) * 4;
        *reinterpret_cast<float4*>(sm + L::o_d + (byte >> 7) * L::kSeg + swz32(t, byte & 127)) = d;
      }
    fence_proxy_async();
    tc_before();
    __syncthreads();
    if (t == 0) {
      tc_after();
      // G[j'][r] += sum_t A[t][j'] (r_t D_n[t][r]): A = the gathered tile read
      // MN-major (M-blocks = modes, LBO = one mode tile), K = 8 nonzeros per
      // instruction (one swizzle atom of rows, SBO).
      constexpr uint32_t id = idesc_tf32(128, RP, 1, 1);
      const uint32_t a0 = smem_u32(sm + L::o_a + slot * L::kSlot);
      const uint32_t d0 = smem_u32(sm + L::o_d);
#pragma unroll
      for (int n = 0; n < N; ++n) {
        const uint32_t dbyte = n * RP * 4;
        const uint32_t dn = d0 + (dbyte >> 7) * L::kSeg + (dbyte & 127);
#pragma unroll 4
        for (int ks = 0; ks < kTileRows / 8; ++ks)
          mma_ss(tmem + L::t_x + n * RP, sdesc_l(a0 + ks * 1024, L::kSeg, 512, 1),
                 sdesc_l(dn + ks * 1024, L::kSeg, 512, 1), id, (k > 0 || ks > 0) ? 1u : 0u);
      }
      mma_commit(&bars[kStages]);
    }
    mbar_wait(&bars[kStages], mma_phase);
    mma_phase ^= 1;
    tc_after();
    __syncthreads();  // slot, D tiles and C columns free for the next tile
  }
  // Publish this CTA's gradient: TMEM lane j' (stacked mode rows) holds
  // G_{mode(j')}[j' mod J][:] in column block mode(j').
  constexpr int JP = L::JP, RP = L::RP;
  const int jrow = t;  // lane
  const int mode = jrow / JP, jj = jrow - mode * JP;
  float* out = p.partials + (size_t)blockIdx.x * (N * J * R);
#pragma unroll
  for (int n = 0; n < N; ++n) {
    if (n * JP >= (warp + 1) * 32 || (n + 1) * JP <= warp * 32) continue;  // warp-uniform
#pragma unroll
    for (int h = 0; h < RP / 16; ++h) {
      uint32_t v[16];
      tmem_ld16(tlane + L::t_x + n * RP + h * 16, v);
      tmem_wait_ld();
      if (p.dbg && blockIdx.x == 0 && h == 0) p.dbg[t * 8 + 6 + (n & 1)] = __uint_as_float(v[0]);
      if (mode == n && jj < J) {
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (h * 16 + q < R)
            out[((size_t)n * J + jj) * R + h * 16 + q] = nk > 0 ? __uint_as_float(v[q]) : 0.0f;
      }
    }
  }
  cta_teardown<N, J, R, true>(tmem);
}

__global__ void tc_reduce_kernel(const float* __restrict__ partials, int nparts, int len,
                                 float* __restrict__ grad) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < len; e += gridDim.x * blockDim.x) {
    float s = 0.0f;
    for (int k = 0; k < nparts; ++k) s += partials[(size_t)k * len + e];
    grad[e] = s;
  }
}

TcParams make_params(const KView& v, int64_t mul, int64_t add) {
  TcParams p{};
  for (int n = 0; n < v.order; ++n) {
    p.idx[n] = v.idx[n];
    p.a[n] = v.a[n];
    p.b[n] = v.b[n];
  }
  p.vals = v.vals;
  p.nnz = v.nnz;
  p.ntiles = v.ntiles;
  p.tile_base = v.tile_base;
  p.tile_rows = v.tile_rows;
  p.tperm = v.tperm;
  p.max_ctas = v.max_ctas;
  p.tmul = mul;
  p.tadd = add;
  return p;
}

template <int N, int J, int R>
cudaError_t run_factor(const TcParams& p, cudaStream_t st) {
  using L = TcLayout<N, J, R, false>;
  auto kern = tc_factor_kernel<N, J, R>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)L::bytes);
  if (e != cudaSuccess) return e;
  int grid = (int)(p.ntiles < num_sms() ? p.ntiles : num_sms());
  if (p.max_ctas > 0 && grid > p.max_ctas) grid = p.max_ctas;
  kern<<<grid, kThreads, L::bytes, st>>>(p);
  return cudaGetLastError();
}

template <int N, int J, int R>
cudaError_t run_core(TcParams p, float* grad, float* scratch, size_t scratch_bytes,
                     cudaStream_t st) {
  using L = TcLayout<N, J, R, true>;
  auto kern = tc_core_kernel<N, J, R>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)L::bytes);
  if (e != cudaSuccess) return e;
  const int grid = (int)(p.ntiles < num_sms() ? p.ntiles : num_sms());
  const int len = N * J * R;
  if (scratch_bytes < (size_t)grid * len * sizeof(float)) return cudaErrorInvalidValue;
  p.partials = scratch;
  static const bool debug = std::getenv("FTKCU_TC_DEBUG") != nullptr;
  float* dbg = nullptr;
  if (debug) {
    cudaMalloc(&dbg, 128 * 8 * sizeof(float));
    cudaMemsetAsync(dbg, 0, 128 * 8 * sizeof(float), st);
    p.dbg = dbg;
  }
  kern<<<grid, kThreads, L::bytes, st>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (debug) {
    float h[128 * 8];
    cudaMemcpyAsync(h, dbg, sizeof h, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    for (int t = 0; t < 128; t += 9)
      std::printf("dbg row %3d resid %.5g xhat %.5g c0 %.5g c1 %.5g x %.5g idx %.0f g0 %.5g g1 %.5g\n",
                  t, h[t * 8], h[t * 8 + 1], h[t * 8 + 2], h[t * 8 + 3], h[t * 8 + 4],
                  h[t * 8 + 5], h[t * 8 + 6], h[t * 8 + 7]);
    cudaFree(dbg);
  }
  tc_reduce_kernel<<<(len + 255) / 256, 256, 0, st>>>(scratch, grid, len, grad);
  return cudaGetLastError();
}

// Shape dispatch: uniform ranks J_n = J; (J, R) in {16, 32}^2 at N = 3,
// J = R = 16 at N = 4..6, J = R = 8 (padded to 16) at N = 3..6; sum of the
// padded J <= 128 (the core sweep's stacked M).
template <bool kCore, typename F>
cudaError_t dispatch(const KView& v, F&& f) {
  const int j = v.j[0], r = v.r, n = v.order;
#define FTK_CASE(NN, JJ, RR) \
  if (n == NN && j == JJ && r == RR) return f.template operator()<NN, JJ, RR>();
  FTK_CASE(3, 32, 32) FTK_CASE(3, 16, 16) FTK_CASE(4, 16, 16) FTK_CASE(5, 16, 16)
  FTK_CASE(6, 16, 16) FTK_CASE(3, 16, 32) FTK_CASE(3, 32, 16) FTK_CASE(3, 8, 8)
  FTK_CASE(4, 8, 8) FTK_CASE(5, 8, 8) FTK_CASE(6, 8, 8)
#undef FTK_CASE
  return cudaErrorNotSupported;
}

}  // namespace

bool tc_supported(const KView& v) {
  for (int n = 1; n < v.order; ++n)
    if (v.j[n] != v.j[0]) return false;
  const int n = v.order, j = v.j[0], r = v.r;
  return (n == 3 && (j == 16 || j == 32) && (r == 16 || r == 32)) ||
         (n >= 4 && n <= 6 && j == 16 && r == 16) || (n >= 3 && n <= 6 && j == 8 && r == 8);
}

struct FactorLaunch {
  const TcParams& p;
  cudaStream_t st;
  template <int N, int J, int R>
  cudaError_t operator()() { return run_factor<N, J, R>(p, st); }
};

struct CoreLaunch {
  const TcParams& p;
  float* grad;
  float* scratch;
  size_t bytes;
  cudaStream_t st;
  template <int N, int J, int R>
  cudaError_t operator()() { return run_core<N, J, R>(p, grad, scratch, bytes, st); }
};

cudaError_t launch_tc_factor(const KView& v, int64_t tile_mul, int64_t tile_add, float lr_a,
                             float reg_a, int precision, int atomic_update, cudaStream_t st) {
  TcParams p = make_params(v, tile_mul, tile_add);
  p.prec3 = precision == FTKCU_PREC_3XTF32;
  p.lr = lr_a;
  p.reg = reg_a;
  p.atomic_update = atomic_update;
  if (p.ntiles == 0) return cudaSuccess;
  FactorLaunch f{p, st};
  return dispatch<false>(v, f);
}

cudaError_t launch_tc_core(const KView& v, int64_t tile_mul, int64_t tile_add, float* grad,
                           int precision, float* scratch, size_t scratch_bytes,
                           cudaStream_t st) {
  TcParams p = make_params(v, tile_mul, tile_add);
  p.prec3 = precision == FTKCU_PREC_3XTF32;
  CoreLaunch f{p, grad, scratch, scratch_bytes, st};
  return dispatch<true>(v, f);
}

}  // namespace ftkcu
