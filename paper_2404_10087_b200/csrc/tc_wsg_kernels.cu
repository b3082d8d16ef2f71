// Warp-specialised tcgen05 sweeps for J = R = 16 at order N = 3..6 (BASELINE
// C1, C4 order 6, C5 rank 16): the design of tc_ws_kernels.cu (the N = 3,
// J = R = 32 headline sweeps) generalised over the order, at 16 columns.
//
//   warp 0      COO columns by 1-D bulk copies into a kI-deep ring
//   warps 10-11 TMA gather4 of the tile's factor rows (one elected lane
//               each, half of the 4-row groups each)
//   warp 1      MMA issuer (one thread)
//   warps 2-9   epilogue: two warps per TMEM lane quarter, 8 columns each
//
// Factor (tf32, rows 64 B, SWIZZLE_64B K-major): [C_n | A_n] = A_n [B_n | I]
// (N = 32) per mode into TMEM buffer k & 1; the epilogue exchanges x_hat
// halves through shared memory and writes D'_n = lr r prod_{m != n} C_m
// (prefix x suffix products) in place over C; U'_n = D'_n B_n^T +
// A_n (-lr reg I) is the Hogwild step, sent as vector RED of 32-B row
// segments from per-warp staging tiles.
//
// Core (fp16 copy of A, rows 32 B, SWIZZLE_32B): one gathered tile is the
// K-major A of C = A B and the MN-major A of G += A^T (r D) (kind::f16, fp32
// accumulate); G stacks the N modes' 16-row blocks in M (N <= 8) and is
// accumulated in TMEM over the CTA's tiles.
//
// J = R = 8 (C5 rank 8) runs padded to 16: the row-gather maps have 8
// columns and a 16-column box, so TMA zero-fills columns 8..15 of every
// gathered row (out of bounds); the padding rows / columns of the B operands
// are zero, so every padded C, D', U and G entry is exactly zero, and only
// the 8 real columns are written back.
//
// Reference: decomposition.cpp:644-658 / :678-698 (per-batch pipeline),
// PAPER.md Alg. 4 / Alg. 5.
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "engine.cuh"
#include "tc_common.cuh"

namespace ftkcu {
namespace {
using namespace tc;

constexpr int kW = 16;     // J = R
constexpr int kRows = 128;
constexpr int kEpiWarps = 8;
constexpr int kGW = 2;
constexpr int kGatherWarp = 2 + kEpiWarps;
constexpr int kThreads = (2 + kEpiWarps + kGW) * 32;
constexpr int kMaxN = 6;

struct __align__(64) WsgParams {
  CUtensorMap tmap[kMaxN];
  const int32_t* idx[kMaxN];
  const float* vals;
  float* a[kMaxN];
  const float* b[kMaxN];
  int64_t ntiles, tmul, tadd, tile_base;
  const int32_t* tile_rows;
  const int64_t* tperm;
  float lr, reg;
  float* partials;
  int jr;  // real J = R (16, or 8 padded to 16)
};

__device__ __forceinline__ int64_t wsg_tile(const WsgParams& p, int64_t k) {
  const int64_t t = (int64_t)blockIdx.x + k * gridDim.x;
  const int64_t mul = p.tperm ? __ldg(p.tperm) : p.tmul;
  const int64_t add = p.tperm ? __ldg(p.tperm + 1) : p.tadd;
  return p.tile_base + (t * mul + add) % p.ntiles;
}

__device__ __forceinline__ uint32_t rn_bits(float x) { return __float_as_uint(x) + 0x1000u; }

// 32-B-row swizzle (Swizzle<1,4,3>: 16-B chunk XOR bit 2 of the row).
__host__ __device__ constexpr uint32_t swz32b(uint32_t row, uint32_t byte) {
  return row * 32 + ((((byte >> 4) ^ ((row >> 2) & 1))) << 4) + (byte & 15);
}



// Layout per (order, sweep).  Row tiles: 128 rows x (64 B fp32 | 32 B fp16).
template <int N, bool kCore>
struct WsgLayout {
  static constexpr uint32_t kRowB = kCore ? 32 : 64;
  static constexpr uint32_t kModeTile = kRows * kRowB;
  static constexpr uint32_t kSlot = N * kModeTile;
  static constexpr int kS = kCore ? 6 : (N <= 4 ? 4 : 3);
  static constexpr uint32_t o_a = 0;
  // core: double-buffered r D tiles (fp16, N blocks of 16 r); the G GEMM's M
  // stack reads 8 blocks of 16 rows, past a slot into the next / these tiles
  static constexpr uint32_t o_d = o_a + kS * kSlot;
  static constexpr uint32_t d_bytes = kCore ? 2 * kSlot + (8 - N) * kModeTile : 0;
  // C GEMM B operand per mode: factor [B^T ; I] (32 rows x 64 B), core B^T fp16
  static constexpr uint32_t o_bt = o_d + d_bytes;
  static constexpr uint32_t bt_mode = kCore ? kW * 32 : 2 * kW * 64;
  static constexpr uint32_t o_b = o_bt + N * bt_mode;              // factor: B (rows j, K = r)
  static constexpr uint32_t o_diag = o_b + (kCore ? 0 : N * kW * 64);  // factor: -lr reg I
  static constexpr uint32_t o_idx = o_diag + (kCore ? 0 : kW * 64);
  static constexpr uint32_t kIdxSlot = (N + 1) * kRows * 4;
  static constexpr int kI = 6;
  static constexpr uint32_t o_stage = o_idx + kI * kIdxSlot;  // factor: per-warp write-back
  static constexpr uint32_t stage_bytes = kCore ? 0 : kEpiWarps * 32 * 32;
  static constexpr uint32_t o_xp = o_stage + stage_bytes;    // x_hat halves [2][2][128]
  static constexpr uint32_t o_rows = o_xp + 2 * 2 * kRows * 4;
  static constexpr uint32_t o_bar = o_rows + 64;
  static constexpr uint32_t o_tmem = o_bar + 32 * 8;
  static constexpr uint32_t bytes = (o_tmem + 16 + 1023) / 1024 * 1024;
  // TMEM: factor buffers 2 x N x 2W ([C|A] per mode) + U (N W); core C[2]
  // (N W each) + G (N R)
  static constexpr uint32_t t_u = 2 * N * 2 * kW;
  static constexpr uint32_t t_g = 2 * N * kW;
  static constexpr uint32_t tcols_used = kCore ? t_g + N * kW : t_u + N * kW;
  static constexpr uint32_t tcols = tcols_used <= 256 ? 256 : 512;
  static_assert(bytes <= 227 * 1024, "shared-memory budget");
  static_assert(tcols_used <= 512, "TMEM budget");
  static_assert(N * kW <= 128, "stacked G rows exceed M = 128");
};

enum : int {
  G_FULL = 0,     // [6] slot landed (one expect_tx arrival per gather warp)
  G_EMPTY = 6,    // [6] slot free
  G_IFULL = 12,   // [6] COO columns landed
  G_IEMPTY = 18,  // [6] COO columns consumed (epilogue warps + gather warps)
  G_CFULL = 24,   // [2] C ready
  G_DFULL = 26,   // [2] D' (factor, TMEM) / r D (core, smem) ready
  G_UFULL = 28,   // factor: U ready
  G_UEMPTY = 29,  // factor: U read
  G_DEMPTY = 30,  // [2] core: G GEMM done with r D tile b
};

template <int N, bool kCore>
__device__ void wsg_setup(const WsgParams& p, uint8_t* sm, uint64_t* bars, uint32_t* tslot) {
  using L = WsgLayout<N, kCore>;
  for (int n = 0; n < N; ++n) {
    const float* b = p.b[n];
    for (int e = threadIdx.x; e < kW * kW; e += blockDim.x) {
      const int j = e / kW, r = e - j * kW;
      const float x = (j < p.jr && r < p.jr) ? b[j * p.jr + r] : 0.0f;
      if constexpr (kCore) {
        *reinterpret_cast<__half*>(sm + L::o_bt + n * L::bt_mode + swz32b(r, j * 2)) =
            __float2half_rn(x);
      } else {
        const float hi = __uint_as_float(rn_bits(x));
        *reinterpret_cast<float*>(sm + L::o_bt + n * L::bt_mode + swz(r, j * 4, 64)) = hi;
        *reinterpret_cast<float*>(sm + L::o_bt + n * L::bt_mode + swz(kW + r, j * 4, 64)) =
            (r == j && j < p.jr) ? 1.0f : 0.0f;
        *reinterpret_cast<float*>(sm + L::o_b + n * kW * 64 + swz(j, r * 4, 64)) = hi;
      }
    }
  }
  if constexpr (!kCore)
    for (int e = threadIdx.x; e < kW * kW; e += blockDim.x) {
      const int j = e / kW, jj = e - j * kW;
      *reinterpret_cast<float*>(sm + L::o_diag + swz(j, jj * 4, 64)) =
          (j == jj && j < p.jr) ? __uint_as_float(rn_bits(-p.lr * p.reg)) : 0.0f;
    }
  if constexpr (kCore)  // the G GEMM's garbage M blocks read zeros
    for (uint32_t o = threadIdx.x * 16; o < L::d_bytes; o += blockDim.x * 16)
      *reinterpret_cast<int4*>(sm + L::o_d + o) = make_int4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kS; ++s) {
      mbar_init(&bars[G_FULL + s], kGW);
      mbar_init(&bars[G_EMPTY + s], 1);
    }
    for (int i = 0; i < L::kI; ++i) {
      mbar_init(&bars[G_IFULL + i], 1);
      mbar_init(&bars[G_IEMPTY + i], kEpiWarps + kGW);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars[G_CFULL + b], 1);
      mbar_init(&bars[G_DFULL + b], kEpiWarps);
      mbar_init(&bars[G_DEMPTY + b], 1);
    }
    mbar_init(&bars[G_UFULL], 1);
    mbar_init(&bars[G_UEMPTY], kEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int n = 0; n < N; ++n) prefetch_tmap(&p.tmap[n]);
  }
  if (threadIdx.x / 32 == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(L::tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_before();
  __syncthreads();
  tc_after();
}

template <int N, bool kCore>
__device__ void wsg_teardown(uint32_t tmem) {
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x / 32 == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(WsgLayout<N, kCore>::tcols));
}

template <int N, bool kCore>
__device__ void wsg_idx_producer(const WsgParams& p, uint8_t* sm, uint64_t* bars, int64_t nk) {
  using L = WsgLayout<N, kCore>;
  if ((threadIdx.x & 31) != 0) return;
  auto ahead = tile_ahead<4>([&](int64_t kk) { return wsg_tile(p, kk); }, p.tile_rows, nk);
  for (int64_t k = 0; k < nk; ++k) {
    const int i = (int)(k % L::kI);
    int64_t tile;
    int32_t valid;
    ahead.pop(k, tile, valid);
    mbar_wait(&bars[G_IEMPTY + i], (uint32_t)(((k / L::kI) & 1) ^ 1));
    int32_t* s_idx = reinterpret_cast<int32_t*>(sm + L::o_idx + i * L::kIdxSlot);
    reinterpret_cast<int32_t*>(sm + L::o_rows)[i] = valid;
    mbar_expect_tx(&bars[G_IFULL + i], L::kIdxSlot);
    for (int n = 0; n < N; ++n)
      bulk_g2s(s_idx + n * kRows, p.idx[n] + tile * kRows, kRows * 4, &bars[G_IFULL + i]);
    bulk_g2s(s_idx + N * kRows, p.vals + tile * kRows, kRows * 4, &bars[G_IFULL + i]);
  }
}

// Gather warps: groups of 4 rows, N x 32 per tile, half per warp.
template <int N, bool kCore>
__device__ void wsg_gather(const WsgParams& p, uint8_t* sm, uint64_t* bars, int64_t nk) {
  using L = WsgLayout<N, kCore>;
  const int gw = (int)(threadIdx.x >> 5) - kGatherWarp;
  constexpr int kGroups = N * kRows / 4, kPer = kGroups / kGW;
  static_assert(kPer % 4 == 0, "whole batches of 4 groups per gather warp");
  for (int64_t k = 0; k < nk; ++k) {
    const int s = (int)(k % L::kS), i = (int)(k % L::kI);
    mbar_wait(&bars[G_EMPTY + s], (uint32_t)(((k / L::kS) & 1) ^ 1));
    mbar_wait(&bars[G_IFULL + i], (uint32_t)((k / L::kI) & 1));
    const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + i * L::kIdxSlot);
    uint8_t* slot = sm + L::o_a + s * L::kSlot;
    __syncwarp();
    if (elect_one()) {
      mbar_expect_tx(&bars[G_FULL + s], kPer * 4 * L::kRowB);
#pragma unroll 1
      for (int g0 = gw * kPer; g0 < (gw + 1) * kPer; g0 += 4) {
        int4 r[4];  // 4 index loads in flight (batches never straddle modes)
#pragma unroll
        for (int g = 0; g < 4; ++g) r[g] = *reinterpret_cast<const int4*>(s_idx + (g0 + g) * 4);
        const int n = g0 / (kRows / 4), gm = g0 - n * (kRows / 4);
#pragma unroll
        for (int g = 0; g < 4; ++g)
          tma_gather4(slot + n * L::kModeTile + (gm + g) * 4 * L::kRowB, &p.tmap[n], 0, r[g].x,
                      r[g].y, r[g].z, r[g].w, &bars[G_FULL + s]);
      }
      mbar_arrive(&bars[G_IEMPTY + i]);
    }
    __syncwarp();
  }
}

// D_n = prod_{m != n} C_m for 8 columns (prefix x suffix products), x_hat
// partial = sum_i prod_n C_n.
template <int N>
__device__ __forceinline__ float prods(const float (&c)[N][8], float (&d)[N][8]) {
  float part = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float pre[N], suf[N];
    pre[0] = 1.0f;
#pragma unroll
    for (int n = 1; n < N; ++n) pre[n] = pre[n - 1] * c[n - 1][i];
    suf[N - 1] = 1.0f;
#pragma unroll
    for (int n = N - 2; n >= 0; --n) suf[n] = suf[n + 1] * c[n + 1][i];
#pragma unroll
    for (int n = 0; n < N; ++n) d[n][i] = pre[n] * suf[n];
    part = fmaf(c[0][i], d[0][i], part);
  }
  return part;
}

// ---- factor sweep ---------------------------------------------------------------
//
// Templated over the column count W (16, or 32 for the headline shape): the
// epilogue has W / 8 warps per TMEM lane quarter, each owning 8 columns, so
// W = 32 runs 16 epilogue warps (4 per scheduler) -- the latency hiding the
// 8-warp tc_ws_kernels.cu factor sweep lacks.

template <int W>
struct FW {
  static constexpr int E = 4 * (W / 8);         // epilogue warps
  static constexpr int GWarp = 2 + E;           // first gather warp
  static constexpr int Threads = (2 + E + kGW) * 32;
  static constexpr uint32_t RowB = W * 4;       // fp32 row bytes (64 | 128)
  static constexpr uint32_t Sbo = 8 * RowB;     // 8-row group stride
  static constexpr uint64_t Lay = W == 16 ? 4 : 2;  // SWIZZLE_64B | SWIZZLE_128B
};

template <int N, int W>
struct WsfLayout {
  using F = FW<W>;
  static constexpr uint32_t kModeTile = kRows * F::RowB;
  static constexpr uint32_t kSlot = N * kModeTile;
  static constexpr int kS = W == 32 ? 3 : (N <= 4 ? 4 : 3);
  static constexpr uint32_t o_a = 0;
  static constexpr uint32_t o_bt = o_a + kS * kSlot;  // [B^T ; I] per mode: 2W rows
  static constexpr uint32_t bt_mode = 2 * W * F::RowB;
  static constexpr uint32_t o_b = o_bt + N * bt_mode;  // B (rows j, K = r): W rows
  static constexpr uint32_t o_diag = o_b + N * W * F::RowB;
  static constexpr uint32_t o_idx = o_diag + W * F::RowB;
  static constexpr uint32_t kIdxSlot = (N + 1) * kRows * 4;
  static constexpr int kI = 6;
  static constexpr uint32_t o_stage = o_idx + kI * kIdxSlot;  // per-warp 32 rows x 32 B
  static constexpr uint32_t o_xp = o_stage + F::E * 1024;     // [2][W/8][128] x_hat parts
  static constexpr uint32_t o_rows = o_xp + 2 * (W / 8) * kRows * 4;
  static constexpr uint32_t o_bar = o_rows + 64;
  static constexpr uint32_t o_tmem = o_bar + 32 * 8;
  static constexpr uint32_t bytes = (o_tmem + 16 + 1023) / 1024 * 1024;
  static constexpr uint32_t t_u = 2 * N * 2 * W;  // buffers [C|A] x 2, then U
  static constexpr uint32_t tcols_used = t_u + N * W;
  static constexpr uint32_t tcols = tcols_used <= 256 ? 256 : 512;
  static_assert(bytes <= 227 * 1024, "shared-memory budget");
  static_assert(tcols_used <= 512, "TMEM budget");
};

template <int N, int W>
__device__ void wsf_setup(const WsgParams& p, uint8_t* sm, uint64_t* bars, uint32_t* tslot) {
  using L = WsfLayout<N, W>;
  using F = FW<W>;
  for (int n = 0; n < N; ++n) {
    const float* b = p.b[n];
    for (int e = threadIdx.x; e < W * W; e += blockDim.x) {
      const int j = e / W, r = e - j * W;
      const float x = (j < p.jr && r < p.jr) ? b[j * p.jr + r] : 0.0f;
      const float hi = __uint_as_float(rn_bits(x));
      *reinterpret_cast<float*>(sm + L::o_bt + n * L::bt_mode + swz(r, j * 4, F::RowB)) = hi;
      *reinterpret_cast<float*>(sm + L::o_bt + n * L::bt_mode + swz(W + r, j * 4, F::RowB)) =
          (r == j && j < p.jr) ? 1.0f : 0.0f;
      *reinterpret_cast<float*>(sm + L::o_b + n * W * F::RowB + swz(j, r * 4, F::RowB)) = hi;
    }
  }
  for (int e = threadIdx.x; e < W * W; e += blockDim.x) {
    const int j = e / W, jj = e - j * W;
    *reinterpret_cast<float*>(sm + L::o_diag + swz(j, jj * 4, F::RowB)) =
        (j == jj && j < p.jr) ? __uint_as_float(rn_bits(-p.lr * p.reg)) : 0.0f;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kS; ++s) {
      mbar_init(&bars[G_FULL + s], kGW);
      mbar_init(&bars[G_EMPTY + s], 1);
    }
    for (int i = 0; i < L::kI; ++i) {
      mbar_init(&bars[G_IFULL + i], 1);
      mbar_init(&bars[G_IEMPTY + i], F::E + kGW);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars[G_CFULL + b], 1);
      mbar_init(&bars[G_DFULL + b], F::E);
    }
    mbar_init(&bars[G_UFULL], 1);
    mbar_init(&bars[G_UEMPTY], F::E);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int n = 0; n < N; ++n) prefetch_tmap(&p.tmap[n]);
  }
  if (threadIdx.x / 32 == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(L::tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_before();
  __syncthreads();
  tc_after();
}

template <int N, int W>
__global__ void __launch_bounds__(FW<W>::Threads, 1)
    wsf_factor_kernel(const __grid_constant__ WsgParams p) {
  using L = WsfLayout<N, W>;
  using F = FW<W>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::o_bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + L::o_tmem);
  wsf_setup<N, W>(p, sm, bars, tslot);
  const uint32_t tmem = *tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nk = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  constexpr uint32_t kBuf = N * 2 * W, kMs = 2 * W;
  constexpr int kH = W / 8;  // epilogue warps per lane quarter

  if (warp == 0) {
    if (lane == 0) {
      auto ahead = tile_ahead<4>([&](int64_t kk) { return wsg_tile(p, kk); }, p.tile_rows, nk);
      for (int64_t k = 0; k < nk; ++k) {
        const int i = (int)(k % L::kI);
        int64_t tile;
        int32_t valid;
        ahead.pop(k, tile, valid);
        mbar_wait(&bars[G_IEMPTY + i], (uint32_t)(((k / L::kI) & 1) ^ 1));
        int32_t* s_idx = reinterpret_cast<int32_t*>(sm + L::o_idx + i * L::kIdxSlot);
        reinterpret_cast<int32_t*>(sm + L::o_rows)[i] = valid;
        mbar_expect_tx(&bars[G_IFULL + i], L::kIdxSlot);
        for (int n = 0; n < N; ++n)
          bulk_g2s(s_idx + n * kRows, p.idx[n] + tile * kRows, kRows * 4, &bars[G_IFULL + i]);
        bulk_g2s(s_idx + N * kRows, p.vals + tile * kRows, kRows * 4, &bars[G_IFULL + i]);
      }
    }
  } else if (warp >= F::GWarp) {
    const int gw = warp - F::GWarp;
    constexpr int kGroups = N * kRows / 4, kPer = kGroups / kGW;
    static_assert(kPer % 4 == 0, "whole batches of 4 groups per gather warp");
    for (int64_t k = 0; k < nk; ++k) {
      const int s = (int)(k % L::kS), i = (int)(k % L::kI);
      mbar_wait(&bars[G_EMPTY + s], (uint32_t)(((k / L::kS) & 1) ^ 1));
      mbar_wait(&bars[G_IFULL + i], (uint32_t)((k / L::kI) & 1));
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + i * L::kIdxSlot);
      uint8_t* slot = sm + L::o_a + s * L::kSlot;
      __syncwarp();
      if (elect_one()) {
        mbar_expect_tx(&bars[G_FULL + s], kPer * 4 * F::RowB);
#pragma unroll 1
        for (int g0 = gw * kPer; g0 < (gw + 1) * kPer; g0 += 4) {
          int4 r[4];
#pragma unroll
          for (int g = 0; g < 4; ++g) r[g] = *reinterpret_cast<const int4*>(s_idx + (g0 + g) * 4);
          const int n = g0 / (kRows / 4), gm = g0 - n * (kRows / 4);
#pragma unroll
          for (int g = 0; g < 4; ++g)
            tma_gather4(slot + n * L::kModeTile + (gm + g) * 4 * F::RowB, &p.tmap[n], 0, r[g].x,
                        r[g].y, r[g].z, r[g].w, &bars[G_FULL + s]);
        }
        mbar_arrive(&bars[G_IEMPTY + i]);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idc = idesc_tf32(128, 2 * W, 0, 0), idu = idesc_tf32(128, W, 0, 0);
      const uint32_t bt = smem_u32(sm + L::o_bt), bb = smem_u32(sm + L::o_b);
      const uint32_t dg = smem_u32(sm + L::o_diag);
      auto kadr = [](uint32_t base, int ks) { return base + ks * 32; };  // 8 fp32 per K step
      auto issue_u = [&](int64_t j) {
        const int b = (int)(j & 1);
        mbar_wait(&bars[G_DFULL + b], (uint32_t)((j >> 1) & 1));
        mbar_wait(&bars[G_UEMPTY], (uint32_t)((j & 1) ^ 1));
        tc_after();
        const uint32_t tb = tmem + b * kBuf;
#pragma unroll
        for (int n = 0; n < N; ++n) {
#pragma unroll
          for (int ks = 0; ks < W / 8; ++ks)
            mma_ts(tmem + L::t_u + n * W, tb + n * kMs + ks * 8,
                   sdesc_l(kadr(bb + n * W * F::RowB, ks), 16, F::Sbo, F::Lay), idu, ks > 0);
#pragma unroll
          for (int ks = 0; ks < W / 8; ++ks)
            mma_ts(tmem + L::t_u + n * W, tb + n * kMs + W + ks * 8,
                   sdesc_l(kadr(dg, ks), 16, F::Sbo, F::Lay), idu, 1);
        }
        mma_commit(&bars[G_UFULL]);
      };
      for (int64_t k = 0; k < nk; ++k) {
        const int s = (int)(k % L::kS), b = (int)(k & 1);
        mbar_wait(&bars[G_FULL + s], (uint32_t)((k / L::kS) & 1));
        // C(k) overwrites buffer b, whose D'(k - 2) is U(k - 2)'s A operand:
        // wait for U(k - 2) to complete (PTX orders MMAs only per accumulator)
        if (k >= 2) mbar_wait(&bars[G_UFULL], (uint32_t)((k - 2) & 1));
        tc_after();
        const uint32_t a0 = smem_u32(sm + L::o_a + s * L::kSlot);
#pragma unroll
        for (int n = 0; n < N; ++n)
#pragma unroll
          for (int ks = 0; ks < W / 8; ++ks)
            mma_ss(tmem + b * kBuf + n * kMs,
                   sdesc_l(kadr(a0 + n * L::kModeTile, ks), 16, F::Sbo, F::Lay),
                   sdesc_l(kadr(bt + n * L::bt_mode, ks), 16, F::Sbo, F::Lay), idc, ks > 0);
        mma_commit(&bars[G_CFULL + b]);
        mma_commit(&bars[G_EMPTY + s]);
        if (k >= 1) issue_u(k - 1);
      }
      if (nk >= 1) issue_u(nk - 1);
    }
  } else {
    const int ew = warp - 2, q = warp & 3, h = ew >> 2;  // h: 8-column block
    const int row = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    float* xp = reinterpret_cast<float*>(sm + L::o_xp);
    uint8_t* stage = sm + L::o_stage + ew * 1024;
    struct Tile {
      int32_t g[N];
      bool ok;
    };
    Tile cur, nxt;
    auto epi1 = [&](int64_t k, Tile& t) {
      const int b = (int)(k & 1), ii = (int)(k % L::kI);
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + ii * L::kIdxSlot);
      mbar_wait(&bars[G_IFULL + ii], (uint32_t)((k / L::kI) & 1));
      mbar_wait(&bars[G_CFULL + b], (uint32_t)((k >> 1) & 1));
      tc_after();
      const uint32_t tb = tl + b * kBuf;
      float c[N][8];
#pragma unroll
      for (int n = 0; n < N; ++n) {
        uint32_t v[8];
        tmem_ld8(tb + n * kMs + h * 8, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) c[n][i] = __uint_as_float(v[i]);
      }
      tmem_wait_ld();
      float d[N][8];
      const float part = prods<N>(c, d);
      // x_hat: the kH column blocks of this row are summed through shared memory
      xp[(b * kH + h) * kRows + row] = part;
      named_bar(1 + q, 32 * kH);
      float xhat = 0.0f;
#pragma unroll
      for (int hh = 0; hh < kH; ++hh) xhat += xp[(b * kH + hh) * kRows + row];
#pragma unroll
      for (int n = 0; n < N; ++n) t.g[n] = s_idx[n * kRows + row];
      const float xv = reinterpret_cast<const float*>(s_idx + N * kRows)[row];
      t.ok = row < reinterpret_cast<const int32_t*>(sm + L::o_rows)[ii];
#pragma unroll
      for (int n = 0; n < N; ++n) t.g[n] = t.ok ? t.g[n] : -1;  // one shuffle per row in epi2
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[G_IEMPTY + ii]);
      const float sc = t.ok ? p.lr * (xv - xhat) : 0.0f;
#pragma unroll
      for (int n = 0; n < N; ++n) {
        uint32_t v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = rn_bits(sc * d[n][i]);
        tmem_st8(tb + n * kMs + h * 8, v);
      }
      tmem_wait_st();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[G_DFULL + b]);
    };
    auto epi2 = [&](int64_t k, const Tile& t) {
      mbar_wait(&bars[G_UFULL], (uint32_t)(k & 1));
      tc_after();
      uint32_t u[N][8];
#pragma unroll
      for (int n = 0; n < N; ++n) tmem_ld8(tl + L::t_u + n * W + h * 8, u[n]);
      tmem_wait_ld();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[G_UEMPTY]);
      // per mode: this warp's 32 rows x 8 columns (32 B) through a 1 KB
      // staging tile, then 16 rows per RED instruction (2 lanes per row)
#pragma unroll
      for (int n = 0; n < N; ++n) {
#pragma unroll
        for (int q4 = 0; q4 < 2; ++q4)
          *reinterpret_cast<float4*>(stage + swz32b(lane, q4 * 16)) =
              make_float4(__uint_as_float(u[n][q4 * 4 + 0]), __uint_as_float(u[n][q4 * 4 + 1]),
                          __uint_as_float(u[n][q4 * 4 + 2]), __uint_as_float(u[n][q4 * 4 + 3]));
        __syncwarp();
        float* dst = p.a[n];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int rl = i * 16 + (lane >> 1), ch = lane & 1;
          const int32_t g = __shfl_sync(0xffffffffu, t.g[n], rl);
          const float4 v = *reinterpret_cast<const float4*>(stage + swz32b(rl, ch * 16));
          if (g >= 0 && h * 8 < p.jr) red_add_v4(dst + (size_t)g * p.jr + h * 8 + ch * 4, v);
        }
        __syncwarp();
      }
    };
    if (nk > 0) epi1(0, cur);
    for (int64_t k = 0; k < nk; ++k) {
      if (k + 1 < nk) epi1(k + 1, nxt);
      epi2(k, cur);
      cur = nxt;
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x / 32 == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::tcols));
}

// ---- core sweep (fp16 copy of A) ------------------------------------------------

template <int N>
__global__ void __launch_bounds__(kThreads, 1) wsg_core_kernel(const __grid_constant__ WsgParams p) {
  using L = WsgLayout<N, true>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::o_bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + L::o_tmem);
  wsg_setup<N, true>(p, sm, bars, tslot);
  const uint32_t tmem = *tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nk = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  constexpr uint32_t kC = N * kW;  // C buffer stride

  if (warp == 0) {
    wsg_idx_producer<N, true>(p, sm, bars, nk);
  } else if (warp >= kGatherWarp) {
    wsg_gather<N, true>(p, sm, bars, nk);
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idc = idesc_f16(128, kW, 0, 0);
      constexpr uint32_t idg = idesc_f16(128, N * kW, 1, 1);
      const uint32_t bt = smem_u32(sm + L::o_bt), d0 = smem_u32(sm + L::o_d);
      auto issue_g = [&](int64_t k) {
        const int s = (int)(k % L::kS), db = (int)(k & 1);
        mbar_wait(&bars[G_DFULL + db], (uint32_t)((k >> 1) & 1));
        tc_after();
        // G[j'][n R + r] += sum_t A[t][j'] (r D_n)[t][r]: M = 8 stacked blocks
        // of 16 (N real), N = N R, K = 16 nonzeros per instruction
        const uint32_t a0 = smem_u32(sm + L::o_a + s * L::kSlot), dd = d0 + db * L::kSlot;
#pragma unroll
        for (int ks = 0; ks < kRows / 16; ++ks)
          mma_f16(tmem + L::t_g, sdesc_l(a0 + ks * 512, L::kModeTile, 256, 6),
                  sdesc_l(dd + ks * 512, L::kModeTile, 256, 6), idg, (k > 0 || ks > 0) ? 1u : 0u);
        mma_commit(&bars[G_DEMPTY + db]);
        mma_commit(&bars[G_EMPTY + s]);
      };
      for (int64_t k = 0; k < nk; ++k) {
        const int s = (int)(k % L::kS), b = (int)(k & 1);
        mbar_wait(&bars[G_FULL + s], (uint32_t)((k / L::kS) & 1));
        // C(k) reuses buffer b after epilogue(k - 2) read it: that epilogue
        // wrote r D(k - 2), so G(k - 2)'s DFULL wait (issued above) covers it
        tc_after();
        const uint32_t a0 = smem_u32(sm + L::o_a + s * L::kSlot);
#pragma unroll
        for (int n = 0; n < N; ++n)
          mma_f16(tmem + b * kC + n * kW, sdesc_l(a0 + n * L::kModeTile, 16, 256, 6),
                  sdesc_l(bt + n * L::bt_mode, 16, 256, 6), idc, 0);
        mma_commit(&bars[G_CFULL + b]);
        if (k >= 1) issue_g(k - 1);
      }
      if (nk >= 1) issue_g(nk - 1);
    }
  } else {
    const int ew = warp - 2, q = warp & 3, h = ew >> 2;
    const int row = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    float* xp = reinterpret_cast<float*>(sm + L::o_xp);
    for (int64_t k = 0; k < nk; ++k) {
      const int b = (int)(k & 1), ii = (int)(k % L::kI);
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + ii * L::kIdxSlot);
      mbar_wait(&bars[G_IFULL + ii], (uint32_t)((k / L::kI) & 1));
      mbar_wait(&bars[G_CFULL + b], (uint32_t)((k >> 1) & 1));
      tc_after();
      float c[N][8];
#pragma unroll
      for (int n = 0; n < N; ++n) {
        uint32_t v[8];
        tmem_ld8(tl + b * kC + n * kW + h * 8, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) c[n][i] = __uint_as_float(v[i]);
      }
      tmem_wait_ld();
      float d[N][8];
      const float part = prods<N>(c, d);
      xp[(b * 2 + h) * kRows + row] = part;
      named_bar(1 + q, 64);
      const float xhat = part + xp[(b * 2 + (h ^ 1)) * kRows + row];
      const bool ok = row < reinterpret_cast<const int32_t*>(sm + L::o_rows)[ii];
      const float resid = ok ? reinterpret_cast<const float*>(s_idx + N * kRows)[row] - xhat : 0.0f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[G_IEMPTY + ii]);
      mbar_wait(&bars[G_DEMPTY + b], (uint32_t)(((k >> 1) & 1) ^ 1));  // G(k - 2) done with D[b]
      uint8_t* dt = sm + L::o_d + b * L::kSlot;
#pragma unroll
      for (int n = 0; n < N; ++n) {
        uint4 w;
        w.x = f16x2_sat(resid * d[n][0], resid * d[n][1]);
        w.y = f16x2_sat(resid * d[n][2], resid * d[n][3]);
        w.z = f16x2_sat(resid * d[n][4], resid * d[n][5]);
        w.w = f16x2_sat(resid * d[n][6], resid * d[n][7]);
        *reinterpret_cast<uint4*>(dt + n * L::kModeTile + swz32b(row, h * 16)) = w;
      }
      fence_proxy_async();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[G_DFULL + b]);
    }
    if (nk > 0) mbar_wait(&bars[G_DEMPTY + (int)((nk - 1) & 1)], (uint32_t)(((nk - 1) >> 1) & 1));
    tc_after();
    // TMEM lane j' = 16 n + j holds G_n[j][:] in columns [t_g + 16 n, +16)
    if (q * 2 < N) {
      const int n = q * 2 + (lane >> 4), j = lane & 15;
      uint32_t v[8];
      tmem_ld8(tl + L::t_g + (q * 2) * kW + h * 8, v);  // lanes of mode q*2 ...
      uint32_t v2[8];
      tmem_ld8(tl + L::t_g + (q * 2 + 1) * kW + h * 8, v2);  // ... and mode q*2+1
      tmem_wait_ld();
      const int jr = p.jr;
      if (n < N && j < jr && h * 8 < jr) {
        float* out = p.partials + (size_t)blockIdx.x * (N * jr * jr) + ((size_t)n * jr + j) * jr + h * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          out[i] = nk > 0 ? __uint_as_float((lane >> 4) ? v2[i] : v[i]) : 0.0f;
      }
    }
  }
  wsg_teardown<N, true>(tmem);
}

__global__ void wsg_half_kernel(const float* __restrict__ src, __half* __restrict__ dst, int64_t n2) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n2;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float2 x = reinterpret_cast<const float2*>(src)[e];
    reinterpret_cast<uint32_t*>(dst)[e] = f16x2_sat(x.x, x.y);
  }
}

__global__ void wsg_reduce_kernel(const float* __restrict__ partials, int nparts, int len,
                                  float* __restrict__ grad) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < len; e += gridDim.x * blockDim.x) {
    float s = 0.0f;
    for (int k = 0; k < nparts; ++k) s += partials[(size_t)k * len + e];
    grad[e] = s;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 wsg_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn),
                            cudaEnableDefault, &q);
  }
  return fn;
}

// Row-gather map: rows x jr elements, box of one row of `box` elements
// (fp32 16: 64-B rows, SWIZZLE_64B; fp32 32: 128-B rows, SWIZZLE_128B; fp16
// 16: 32-B rows, SWIZZLE_32B); at jr = 8 the box's upper half is out of
// bounds and arrives zero-filled.
bool wsg_row_map(CUtensorMap* tm, const void* a, int64_t rows, bool half, int jr, int box_cols = kW) {
  auto fn = wsg_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)jr, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)jr * (half ? 2 : 4)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, 1};
  cuuint32_t es[2] = {1, 1};
  return fn(tm, half ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
            const_cast<void*>(a), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            half ? CU_TENSOR_MAP_SWIZZLE_32B
                 : (box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B),
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

WsgParams base_params(const KView& v, int64_t mul, int64_t add) {
  WsgParams p{};
  for (int n = 0; n < v.order; ++n) {
    p.idx[n] = v.idx[n];
    p.a[n] = v.a[n];
    p.b[n] = v.b[n];
  }
  p.vals = v.vals;
  p.ntiles = v.ntiles;
  p.tile_base = v.tile_base;
  p.tile_rows = v.tile_rows;
  p.tperm = v.tperm;
  p.tmul = mul;
  p.tadd = add;
  p.jr = v.r;
  return p;
}

template <int N, int W>
cudaError_t run_factor(const KView& v, const int32_t* dims, int64_t mul, int64_t add, float lr,
                       float reg, cudaStream_t st) {
  WsgParams p = base_params(v, mul, add);
  for (int n = 0; n < N; ++n)
    if (!wsg_row_map(&p.tmap[n], v.a[n], dims[n], false, p.jr, W)) return cudaErrorNotSupported;
  p.lr = lr;
  p.reg = reg;
  const int bytes = (int)WsfLayout<N, W>::bytes;
  cudaError_t e = cudaFuncSetAttribute(wsf_factor_kernel<N, W>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  wsf_factor_kernel<N, W><<<(int)sweep_grid(v), FW<W>::Threads, bytes, st>>>(p);
  return cudaGetLastError();
}

template <int N>
cudaError_t run_core(const KView& v, const int32_t* dims, int64_t mul, int64_t add, float* grad,
                     float* scratch, size_t scratch_bytes, cudaStream_t st) {
  const int grid = (int)(v.ntiles < num_sms() ? v.ntiles : num_sms());
  const int len = N * v.r * v.r;
  if (grid < 1) return cudaErrorInvalidValue;
  if (scratch_bytes < wsg_core_scratch_bytes(v, dims)) return cudaErrorInvalidValue;
  WsgParams p = base_params(v, mul, add);
  p.partials = scratch;
  __half* a16 = reinterpret_cast<__half*>(scratch + (size_t)num_sms() * N * kW * kW);
  for (int n = 0; n < N; ++n) {
    const int64_t cnt2 = (int64_t)dims[n] * p.jr / 2;
    int64_t blocks = (cnt2 + 255) / 256;
    if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
    wsg_half_kernel<<<(int)(blocks > 0 ? blocks : 1), 256, 0, st>>>(v.a[n], a16, cnt2);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (!wsg_row_map(&p.tmap[n], a16, dims[n], true, p.jr)) return cudaErrorNotSupported;
    a16 += ((int64_t)dims[n] * p.jr + 7) / 8 * 8;  // keep every copy 16-B aligned
  }
  const int bytes = (int)WsgLayout<N, true>::bytes;
  cudaError_t e = cudaFuncSetAttribute(wsg_core_kernel<N>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  wsg_core_kernel<N><<<grid, kThreads, bytes, st>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  wsg_reduce_kernel<<<(len + 255) / 256, 256, 0, st>>>(scratch, grid, len, grad);
  return cudaGetLastError();
}

}  // namespace

// N = 3, J = R = 32 on the 16-epilogue-warp factor sweep (wsf_factor_kernel)
bool wsf32_supported(const KView& v) {
  return v.order == 3 && v.r == 32 && v.j[0] == 32 && v.j[1] == 32 && v.j[2] == 32 &&
         wsg_encode_fn() != nullptr;
}

bool wsg_supported(const KView& v) {
  if (v.order < 3 || v.order > kMaxN || (v.r != 16 && v.r != 8)) return false;
  for (int n = 0; n < v.order; ++n)
    if (v.j[n] != v.r) return false;
  return wsg_encode_fn() != nullptr;
}

size_t wsg_core_scratch_bytes(const KView& v, const int32_t* dims) {
  size_t f = (size_t)num_sms() * v.order * kW * kW;  // per-CTA gradients
  size_t h = 0;
  for (int n = 0; n < v.order; ++n) h += ((size_t)dims[n] * kW + 7) / 8 * 8;  // fp16 copy of A
  return (f + (h + 1) / 2 + 64) * sizeof(float);
}

cudaError_t launch_wsg_factor(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                              float lr, float reg, cudaStream_t st) {
  if (v.ntiles == 0) return cudaSuccess;
  if (v.r == 32) return run_factor<3, 32>(v, dims, mul, add, lr, reg, st);
  switch (v.order) {
    case 3: return run_factor<3, 16>(v, dims, mul, add, lr, reg, st);
    case 4: return run_factor<4, 16>(v, dims, mul, add, lr, reg, st);
    case 5: return run_factor<5, 16>(v, dims, mul, add, lr, reg, st);
    case 6: return run_factor<6, 16>(v, dims, mul, add, lr, reg, st);
  }
  return cudaErrorNotSupported;
}

cudaError_t launch_wsg_core(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                            float* grad, float* scratch, size_t scratch_bytes, cudaStream_t st) {
  switch (v.order) {
    case 3: return run_core<3>(v, dims, mul, add, grad, scratch, scratch_bytes, st);
    case 4: return run_core<4>(v, dims, mul, add, grad, scratch, scratch_bytes, st);
    case 5: return run_core<5>(v, dims, mul, add, grad, scratch, scratch_bytes, st);
    case 6: return run_core<6>(v, dims, mul, add, grad, scratch, scratch_bytes, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace ftkcu
