// Warp-specialized tcgen05 sweeps for the headline shape N = 3, J = R = 32
// (Netflix- / Yahoo!Music-shaped configs).  One persistent CTA per SM:
//
//   warp 0      producer: per tile, one 1-D bulk copy per COO column into an
//               index slot, then TMA tile::gather4 of the factor rows straight
//               into the UMMA operand layout (K-major SWIZZLE_128B for the
//               factor sweep, MN-major SWIZZLE_128B_ATOM_32B for the core
//               sweep's gradient GEMM), 3-slot ring, mbarrier transactions;
//   warp 1      MMA issuer (one thread): C = A B per tile into a double-
//               buffered TMEM accumulator, then U = D B^T (factor) or
//               G += A^T (r D) (core) one tile behind, so tensor-core latency
//               overlaps the epilogue of the previous tile;
//   warps 2-9   epilogue: two warps per TMEM lane quarter (128 rows), each
//               owning half of the R (D) and J (update) columns; x_hat halves
//               are exchanged through shared memory with a 64-thread named
//               barrier; Hogwild row updates leave as 128-B-coalesced vector
//               RED.ADD (or STG).
//
// Same algebra as tc_kernels.cu (the synchronous 4-warp sweeps that serve
// every other shape); reference: decomposition.cpp:644-658 / :678-698,
// PAPER.md Alg. 4 / Alg. 5.
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "engine.cuh"
#include "tc_common.cuh"

namespace ftkcu {
namespace {
using namespace tc;

constexpr int kN = 3;            // modes
constexpr int kW = 32;           // J = R
constexpr int kRows = 128;       // nonzeros per tile == TMEM lanes
constexpr int kS = 3;            // A-slot ring depth
constexpr int kEpiWarps = 8;
// warp 0 COO-column producer, warp 1 MMA, warps 2-9 epilogue, warp 10 gather producer
// Gather producers: the tile's 96 TMA gather4 issues are split over kGW
// warps (one elected lane each) -- a single issuing thread serialises them.
constexpr int kGW = 2;
constexpr int kThreadsWs = (2 + kEpiWarps + kGW) * 32;
// ring epochs: one more warp, the round-end mode-2 block copier (ring_agent)
constexpr int kRingWarp = 2 + kEpiWarps + kGW;
constexpr int kThreadsRing = kThreadsWs + 32;
constexpr int kGatherWarp = 2 + kEpiWarps;  // first of the kGW gather warps
constexpr uint32_t kModeTile = kRows * 128;  // 128 rows x 32 fp32 = 16 KB

struct __align__(64) WsParams {
  CUtensorMap tmap[kN];
  const int32_t* idx[kN];
  const float* vals;
  float* a[kN];
  const float* b[kN];
  int64_t nnz, ntiles, tmul, tadd, tile_base;
  const int32_t* tile_rows;
  const int64_t* tperm;  // device {mul, add} or null (KView::tperm)
  float lr, reg;
  int atomic_update, prec3;
  float* partials;
  const float* cc[kN];  // core sweep, storage scheme: C-row cache (KView::cc)
  int exp;  // timing experiments (FTKCU_WS_EXP), never set in production
  int window;  // ws_factor_kernel<true>: KView::window (0, 2 or 3)
  RingDev ring;  // ws_factor_kernel<true>: DSGD ring epoch (ring.ncell > 0)
};

// Timing-experiment bits: a compile-time 0 in the production build, so the
// experiment branches (and the stand-in values some of them would need,
// re-materialised every tile) vanish from the kernels.
__device__ __forceinline__ int ws_exp(const WsParams& p) {
#ifdef FTKCU_EXPERIMENTS
  return p.exp;
#else
  return 0;
#endif
}

// k3: the 3xtf32 factor sweep (ws_factor3_kernel): the C GEMM operand holds
// [B^T hi ; B^T lo] instead of [B^T ; I], and the -lr reg I region holds the
// U GEMM's B lo.
template <bool kCore, bool k3 = false>
struct WsLayout {
  static constexpr uint32_t kSlot = kN * kModeTile;
  static constexpr uint32_t o_a = 0;
  // core: the r-scaled D tile directly after the slots -- the G GEMM's fourth
  // (garbage) M segment of the last slot then still reads shared memory.
  static constexpr uint32_t o_d = o_a + kS * kSlot;
  static constexpr uint32_t d_bytes = kCore ? kN * kModeTile : 0;
  // C GEMM operand per mode: core B^T (hi, then lo); factor [B^T ; I], the
  // identity rows copying the A rows into TMEM for the regulariser GEMM
  static constexpr uint32_t o_bt = o_d + d_bytes;
  static constexpr uint32_t o_btlo = o_bt + kN * (kCore ? 4096 : 8192);
  static constexpr uint32_t o_b = o_btlo + (kCore ? kN * 4096 : 0);  // B (U GEMM operand, factor)
  // factor: -lr reg I (K-major), the regulariser as a second U GEMM operand;
  // 3xtf32 factor: B lo, the U GEMM's second B operand
  static constexpr uint32_t o_diag = o_b + (kCore ? 0 : kN * 4096);
  static constexpr uint32_t o_idx = o_diag + (kCore ? 0 : (k3 ? kN * 4096 : 4096));
  static constexpr uint32_t kIdxSlot = (kN + 1) * kRows * 4;
  static constexpr int kI = kCore ? 4 : 6;  // COO-column ring depth (decoupled from A slots)
  static constexpr uint32_t o_stage = o_idx + kI * kIdxSlot;  // factor: per-quarter write-back rows
  static constexpr uint32_t stage_bytes = kCore ? 0 : 4 * 32 * 128;
  // x_hat partial sums [2 tiles][column groups: 2 core, <= 4 factor][128]
  static constexpr uint32_t o_xp = o_stage + stage_bytes;
  static constexpr uint32_t o_rows = o_xp + 2 * (kCore ? 2 : 4) * kRows * 4;  // [kI] valid rows per COO slot
  static constexpr uint32_t o_bar = o_rows + 64;
  static constexpr int kBars = 32;
  static constexpr uint32_t o_tmem = o_bar + kBars * 8;
  static constexpr uint32_t bytes = o_tmem + 16;
  static_assert(bytes <= 227 * 1024, "shared-memory budget");
  static_assert(!kCore || 4 * kModeTile - kSlot <= d_bytes, "G GEMM overrun");
};

// barrier ids
enum : int {
  B_FULL = 0,        // [kS] gathered rows landed (TMA tx)
  B_EMPTY = 3,       // [kS] A slot free
  B_IFULL = 6,       // [kI <= 6] COO columns landed (bulk tx)
  B_IEMPTY = 12,     // [kI <= 6] COO slot free
  B_CFULL = 18,      // [2]  C accumulator ready
  B_DFULL = 20,      // factor [2]: D in TMEM; core [1]: D tile in smem
  B_UFULL = 22,      // factor [1]: U ready
  B_UEMPTY = 23,     // factor [1]: U read by the epilogue
  B_CEMPTY = 24,     // factor [2]: C read by the epilogue
  B_AFULL = 27,      // core: A rows copied to TMEM
  B_DEMPTY = 28,     // core [1]: G GEMM done with the D tile; factor [2]: U done with D[b]
  B_LOFULL = 30,     // 3xtf32 factor [2]: A lo rows of tile k staged in TMEM buffer k & 1
};

// Round-to-nearest for an operand the tensor core will read as tf32: it
// ignores the low 13 mantissa bits, so adding half an ulp of tf32 to the bit
// pattern turns its truncation into rounding (ties away from zero).
__device__ __forceinline__ uint32_t tf32_rn_bits(float x) { return __float_as_uint(x) + 0x1000u; }

// x_hat = sum_r C0 C1 C2 over all 32 columns of this row: the warp's own
// column half c[][] plus the other half, loaded and consumed here (modes
// `stride` TMEM columns apart).
__device__ __forceinline__ float xhat_full(uint32_t tcol_other, const float (&c)[kN][16],
                                           uint32_t stride = kW) {
  uint32_t o0[16], o1[16], o2[16];
  tmem_ld16(tcol_other, o0);
  tmem_ld16(tcol_other + stride, o1);
  tmem_ld16(tcol_other + 2 * stride, o2);
  tmem_wait_ld();
  float x = 0.0f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    x = fmaf(c[0][i], c[1][i] * c[2][i], x);
    x = fmaf(__uint_as_float(o0[i]), __uint_as_float(o1[i]) * __uint_as_float(o2[i]), x);
  }
  return x;
}

__device__ __forceinline__ int64_t ws_tile(const WsParams& p, int64_t k) {
  const int64_t t = (int64_t)blockIdx.x + k * gridDim.x;
  // tperm (a captured graph's per-epoch permutation) is read through the
  // read-only path once per warp and cached in L1 after the first tile
  const int64_t mul = p.tperm ? __ldg(p.tperm) : p.tmul;
  const int64_t add = p.tperm ? __ldg(p.tperm + 1) : p.tadd;
  return p.tile_base + (t * mul + add) % p.ntiles;
}

// ---- DSGD ring epoch (RingDev, engine.cuh) -----------------------------------
// The cells' tiles, concatenated in cell order, are dealt round-robin over
// the CTAs (CTA b takes tiles b, b + G, ... of the concatenation), so each
// CTA's total is balanced to one tile even when every cell leaves a
// remainder (a fixed start per cell gave CTAs 0..35 an extra tile in all 64
// cells at P = 8); each role keeps its own cursor over (cell, tile of the cell).
__device__ __forceinline__ uint32_t ring_cell_cta(const RingDev& r, int c) {
  // this CTA's position in cell c's deal
  const uint32_t off = (uint32_t)((__ldg(r.cell_tile + c) - __ldg(r.cell_tile)) % gridDim.x);
  return (blockIdx.x + gridDim.x - off) % gridDim.x;
}
__device__ __forceinline__ int64_t ring_cell_nk(const RingDev& r, int c) {
  const uint32_t T = (uint32_t)(__ldg(r.cell_tile + c + 1) - __ldg(r.cell_tile + c));
  const uint32_t b = ring_cell_cta(r, c);
  return T > b ? (T - 1 - b) / gridDim.x + 1 : 0;  // 32-bit: < 2^32 tiles
}
struct RingCursor {
  int c = 0;
  int64_t j = 0, nk = 0;
  int64_t base = 0, T = 1, mul = 1, add = 0, b = 0;  // the current cell's tiles, permutation, deal
  __device__ void enter(const RingDev& r, int c0) {
    j = 0;
    nk = 0;
    for (c = c0; c < r.ncell; ++c)
      if ((nk = ring_cell_nk(r, c)) > 0) break;
    if (c < r.ncell) {
      base = __ldg(r.cell_tile + c);
      T = __ldg(r.cell_tile + c + 1) - base;
      mul = __ldg(r.cell_perm + 2 * c);
      add = __ldg(r.cell_perm + 2 * c + 1);
      b = ring_cell_cta(r, c);
    }
  }
  __device__ int64_t tile(const RingDev&) const {
    const int64_t t = b + j * gridDim.x;
    return base + (t * mul + add) % T;
  }
  __device__ void next(const RingDev& r) {
    if (++j == nk) enter(r, c + 1);
  }
};
__device__ __forceinline__ int64_t ring_tiles(const RingDev& r) {
  int64_t n = 0;
  for (int c = 0; c < r.ncell; ++c) n += ring_cell_nk(r, c);
  return n;
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Waits until arrival flag f carries this epoch (the block it stands for has
// landed in this rank's factor matrices), then orders the TMA reads behind
// it.  A wait that outlives ~2 s raises r.err and gives up instead of
// hanging the device (the host reports the error after the epoch).
__device__ void ring_wait(const RingDev& r, int f) {
  if (f < 0 || r.emulate) return;
  const long long t0 = clock64();
  while (ld_acquire_sys(r.flags + f) < r.epoch) {
    if (clock64() - t0 > r.timeout_cycles) {
      atomicCAS(r.err, 0u, 0x10000u | (unsigned)f);  // the first wait that gave up
      break;
    }
    __nanosleep(128);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <bool kCore, bool k3 = false, int kEW = kEpiWarps>
__device__ void ws_setup(const WsParams& p, uint8_t* sm, uint64_t* bars, uint32_t* tslot) {
  using L = WsLayout<kCore, k3>;
  for (int n = 0; n < kN; ++n) {
    const float* b = p.b[n];
    for (int e = threadIdx.x; e < kW * kW; e += blockDim.x) {
      const int j = e / kW, r = e - j * kW;
      const float x = b[e];
      const float hi = tf32_rna(x), lo = tf32_rna(x - hi);
      if constexpr (kCore) {
        *reinterpret_cast<float*>(sm + L::o_bt + n * 4096 + swz(r, j * 4, 128)) = hi;
        *reinterpret_cast<float*>(sm + L::o_btlo + n * 4096 + swz(r, j * 4, 128)) = lo;
      } else {
        *reinterpret_cast<float*>(sm + L::o_bt + n * 8192 + swz(r, j * 4, 128)) = hi;
        // identity row r: copies a[j = r]; 3xtf32: B^T lo
        *reinterpret_cast<float*>(sm + L::o_bt + n * 8192 + swz(kW + r, j * 4, 128)) =
            k3 ? lo : (r == j ? 1.0f : 0.0f);
        *reinterpret_cast<float*>(sm + L::o_b + n * 4096 + swz(j, r * 4, 128)) = hi;
        if constexpr (k3)
          *reinterpret_cast<float*>(sm + L::o_diag + n * 4096 + swz(j, r * 4, 128)) = lo;
      }
    }
  }
  if constexpr (!kCore && !k3)
    for (int e = threadIdx.x; e < kW * kW; e += blockDim.x) {
      const int j = e / kW, jj = e - j * kW;
      *reinterpret_cast<float*>(sm + L::o_diag + swz(j, jj * 4, 128)) =
          j == jj ? tf32_rna(-p.lr * p.reg) : 0.0f;
    }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kS; ++s) {
      mbar_init(&bars[B_FULL + s], kGW);  // one expect_tx arrival per gather warp
      // core, and factor with atomic rows: released by the MMA that last
      // reads the slot; factor overwrite mode: by the epilogue (reads a)
      // (3xtf32 factor: by the epilogue, whose fp32 step reads a)
      // (window: by the epilogue once the tile's write-back is issued)
      mbar_init(&bars[B_EMPTY + s],
                (kCore || (p.atomic_update && !k3 && !p.window)) ? 1 : kEW);
    }
    for (int i = 0; i < L::kI; ++i) {
      mbar_init(&bars[B_IFULL + i], 1);
      mbar_init(&bars[B_IEMPTY + i], kEW);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars[B_CFULL + b], 1);
      mbar_init(&bars[B_DFULL + b], kEW);
      mbar_init(&bars[B_CEMPTY + b], kEW);
      mbar_init(&bars[B_DEMPTY + b], 1);
    }
    mbar_init(&bars[B_UFULL], 1);
    mbar_init(&bars[B_UEMPTY], kEW);
    mbar_init(&bars[B_AFULL], kEW);
    for (int b = 0; b < 2; ++b) mbar_init(&bars[B_LOFULL + b], kEW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x / 32 == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0)
    for (int n = 0; n < kN; ++n) prefetch_tmap(&p.tmap[n]);
  fence_proxy_async();
  tc_before();
  __syncthreads();
  tc_after();
}

__device__ void ws_teardown(uint32_t tmem) {
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x / 32 == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Warp 0: the tile's COO columns (N index columns + values, 512 B each) by
// 1-D bulk copies into a kI-deep ring, running ahead of the gathers.
template <bool kCore, bool k3 = false, bool kRing = false>
__device__ void ws_idx_producer(const WsParams& p, uint8_t* sm, uint64_t* bars, int64_t nk) {
  using L = WsLayout<kCore, k3>;
  if ((threadIdx.x & 31) != 0) return;
  constexpr bool ring = kRing;
  RingCursor cur;
  if (ring) cur.enter(p.ring, 0);
  // tile ids and valid-row counts kPf tiles ahead: the dependent global
  // loads (tile permutation -> tile_rows) overlap the waits for COO slots
  auto tile_of = [&](int64_t k) -> int64_t {
    if constexpr (ring) {
      const int64_t t = cur.tile(p.ring);
      cur.next(p.ring);
      return t;
    } else {
      return ws_tile(p, k);
    }
  };
  auto ahead = tile_ahead<4>(tile_of, p.tile_rows, nk);
  for (int64_t k = 0; k < nk; ++k) {
    const int i = (int)(k % L::kI);
    int64_t tile;
    int32_t rows;
    ahead.pop(k, tile, rows);
    mbar_wait(&bars[B_IEMPTY + i], (uint32_t)(((k / L::kI) & 1) ^ 1));
    int32_t* s_idx = reinterpret_cast<int32_t*>(sm + L::o_idx + i * L::kIdxSlot);
    // valid-row count of the tile rides with its COO slot (published by the
    // arrive below), keeping the global load off the epilogue's critical path
    reinterpret_cast<int32_t*>(sm + L::o_rows)[i] = rows;
    mbar_expect_tx(&bars[B_IFULL + i], L::kIdxSlot);
    for (int n = 0; n < kN; ++n)
      bulk_g2s(s_idx + n * kRows, p.idx[n] + tile * kRows, kRows * 4, &bars[B_IFULL + i]);
    bulk_g2s(s_idx + kN * kRows, p.vals + tile * kRows, kRows * 4, &bars[B_IFULL + i]);
  }
}

// Gather warps: as soon as an A slot is free, TMA gather4 of the tile's
// factor rows (N modes x 32 groups of 4 rows) into it; gather warp w issues
// groups [w * 96 / kGW, (w + 1) * 96 / kGW) and arrives with its own bytes.
template <bool kCore, bool k3 = false, bool kRing = false, int kEW = kEpiWarps>
__device__ void ws_gather_producer(const WsParams& p, uint8_t* sm, uint64_t* bars, int64_t nk) {
  using L = WsLayout<kCore, k3>;
  const int lane = threadIdx.x & 31, gw = (int)(threadIdx.x >> 5) - (2 + kEW);
  constexpr int kGroups = kN * kRows / 4, kPer = kGroups / kGW;
  static_assert(kGroups % (kGW * 8) == 0, "whole batches of 8 groups per gather warp");
  constexpr bool ring = kRing;
  RingCursor cur;
  if (ring) cur.enter(p.ring, 0);
  for (int64_t k = 0; k < nk; ++k) {
    // ring: the first tile of a cell waits for the cell's blocks to arrive
    int4 io = make_int4(-1, -1, -1, -1);
    if (ring) {
      if (cur.j == 0) io = __ldg(p.ring.cell_io + cur.c);
      cur.next(p.ring);
    }
    const int s = (int)(k % kS), i = (int)(k % L::kI);
    mbar_wait(&bars[B_EMPTY + s], (uint32_t)(((k / kS) & 1) ^ 1));
    // window 2: tile k - 2 retired as well (its slot's completion (k - 2) / kS;
    // the slot's next completion needs tile k + 1's gathers, so no aliasing)
    if (!kCore && !k3 && p.window == 2 && k >= 2)
      mbar_wait(&bars[B_EMPTY + (int)((k - 2) % kS)], (uint32_t)(((k - 2) / kS) & 1));
    mbar_wait(&bars[B_IFULL + i], (uint32_t)((k / L::kI) & 1));
    const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + i * L::kIdxSlot);
    if (ws_exp(p) & 2) {  // exp: no gathers (timing only)
      if (lane == 0) mbar_arrive(&bars[B_FULL + s]);
      continue;
    }
    __syncwarp();
    uint8_t* slot = sm + L::o_a + s * L::kSlot;
    // One elected thread per warp issues: per-lane operands would make the
    // compiler serialise every TMA issue over the 32 lanes (R2UR waterfall).
    if (elect_one()) {
      if (ring && (io.x >= 0 || io.y >= 0)) {
        ring_wait(p.ring, io.x);
        ring_wait(p.ring, io.y);
      }
      mbar_expect_tx(&bars[B_FULL + s], kPer * 512);
#pragma unroll 1
      for (int g0 = gw * kPer; g0 < (gw + 1) * kPer; g0 += 8) {
        int4 r[8];  // 8 index loads in flight before the issues
#pragma unroll
        for (int g = 0; g < 8; ++g)
          r[g] = *reinterpret_cast<const int4*>(s_idx + (g0 + g) * 4);
        const int n = g0 / (kRows / 4);  // a batch of 8 never straddles modes
        const int gm = g0 - n * (kRows / 4);
#pragma unroll
        for (int g = 0; g < 8; ++g)
          tma_gather4(slot + n * kModeTile + (gm + g) * 512, &p.tmap[n], 0, r[g].x, r[g].y,
                      r[g].z, r[g].w, &bars[B_FULL + s]);
      }
    }
    __syncwarp();
  }
}

// Ring epoch: this epilogue warp's write-backs of cell c are issued (and,
// when the count is deferred by a tile, long since performed).  Each warp
// counts itself in (G x kEpiWarps per cell) after a per-thread fence; the
// block copies to the left neighbour are ring_agent's.
__device__ void ring_done(const WsParams& p, int c, int lane) {
  const RingDev& r = p.ring;
  if (!(ws_exp(p) & 64)) __threadfence();  // this thread's REDs of the cell before the count (exp 64: timing only)
  __syncwarp();
  if (lane == 0) atomicAdd(r.done + c, 1u);
}

// One post, spread over the grid: this CTA's slice of the block's rows goes
// to the left neighbour's factor matrix; the CTA that completes the copy
// count raises the neighbour's flag.
__device__ void ring_post_slice(const RingDev& r, const WsParams& p, int post, unsigned* count,
                                int lane) {
  const int4 pd = __ldg(r.posts + post);  // {mode, row0, nrows, peer flag}
  const int64_t n4 = (int64_t)pd.z * (kW / 4);
  const int64_t lo = n4 * blockIdx.x / gridDim.x, hi = n4 * (blockIdx.x + 1) / gridDim.x;
  const float4* src = reinterpret_cast<const float4*>(p.a[pd.x] + (size_t)pd.y * kW);
  float4* dst = reinterpret_cast<float4*>(r.peer_a[pd.x] + (size_t)pd.y * kW);
#pragma unroll 4
  for (int64_t i = lo + lane; i < hi; i += 32) dst[i] = __ldcg(src + i);
  __threadfence_system();
  __syncwarp();
  if (lane == 0 && atomicAdd(count, 1u) == gridDim.x - 1) {
    __threadfence_system();
    st_release_sys(r.peer_flags + pd.w, r.epoch);
  }
}

// Ring epoch, warp kRingWarp of every CTA: walks the cells in order; once a
// cell with a post has been counted in by every epilogue warp of the grid,
// copies this CTA's slice of the cell's mode-3 block (and, at a round's end,
// of the round's mode-2 block) to the left neighbour (ring_post_slice).
// Spreading a post over all CTAs keeps it off the epilogue warps: copied by
// the one warp that completed the count, a 273-row block took ~10 us and
// stalled that CTA's sweep at every cell.  Polls with an exponential
// back-off (32 ns .. 1 us): 148 agents polling one counter every 64 ns put
// a hot line in L2 beside the sweep's REDs for the whole of a long cell.
__device__ void ring_agent(const WsParams& p, int lane) {
  const RingDev& r = p.ring;
  const int Q = r.ncell / r.parts;
  const unsigned want = gridDim.x * kEpiWarps;
  for (int c = 0; c < r.ncell; ++c) {
    const int4 io = __ldg(r.cell_io + c);
    if (io.z < 0 && io.w < 0) continue;
    if (lane == 0) {
      const long long t0 = clock64();
      unsigned v, ns = 32;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(r.done + c) : "memory");
        if (v >= want) break;
        if (clock64() - t0 > r.timeout_cycles) {
          atomicCAS(r.err, 0u, 0x20000u | (unsigned)(c / Q));
          break;
        }
        __nanosleep(ns);
        if (ns < 1024) ns *= 2;
      }
    }
    __syncwarp();
    if (io.z >= 0) ring_post_slice(r, p, io.z, r.copied + r.parts + c, lane);
    if (io.w >= 0) ring_post_slice(r, p, io.w, r.copied + c / Q, lane);
  }
}

// TMEM <-> registers, 16 or 8 consecutive columns of this thread's lane.
template <int kCols>
__device__ __forceinline__ void tmem_ldc(uint32_t a, uint32_t (&v)[kCols]) {
  if constexpr (kCols == 16) tmem_ld16(a, v);
  else tmem_ld8(a, v);
}
template <int kCols>
__device__ __forceinline__ void tmem_stc(uint32_t a, const uint32_t (&v)[kCols]) {
  if constexpr (kCols == 16) tmem_st16(a, v);
  else tmem_st8(a, v);
}

// ---- factor sweep --------------------------------------------------------------

// kEW epilogue warps: 8 (two per TMEM lane quarter, 16 columns each) or 16
// (four per quarter, 8 columns each: twice the warps to hide the epilogue's
// instruction latencies, half the registers per thread).
template <bool kAtomic, bool kRing = false, int kEW = kEpiWarps>
__global__ void __launch_bounds__((2 + kEW + kGW + (kRing ? 1 : 0)) * 32, 1)
    ws_factor_kernel(const __grid_constant__ WsParams p) {
  static_assert(kEW == 8 || kEW == 16, "two or four epilogue warps per lane quarter");
  static_assert(!kRing || kEW == kEpiWarps, "ring epochs count kEpiWarps epilogue warps");
  constexpr int kH = kEW / 4;      // epilogue warps per lane quarter
  constexpr int kCc = kW / kH;     // columns per epilogue warp
  constexpr int kRi = kCc / 4;     // 4-row RED groups per warp and mode (rows 32 / kH)
  constexpr int kGWarp = 2 + kEW;  // first gather warp
  using L = WsLayout<false>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::o_bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + L::o_tmem);
  ws_setup<false, false, kEW>(p, sm, bars, tslot);
  const uint32_t tmem = *tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool ring = kRing;
  static_assert(!kRing || kAtomic, "ring epochs run the accumulate rule");
  const int64_t nk = ring ? ring_tiles(p.ring)
                          : (p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0);
  // TMEM: tile k in buffer b = k & 1 at 192 b; mode n at +64 n holds C_n
  // (overwritten in place by D'_n) and, with atomic rows, a copy of the A
  // rows (+32, from the identity half of the C GEMM's B operand) for the
  // regulariser GEMM; U at 384.  C(k + 2) reuses buffer b only after U(k)
  // has completed (the MMA thread waits for its commit).
  constexpr uint32_t kC = 0, kU = 384, kBuf = 192, kMs = 64;

  if (warp == 0) {
    ws_idx_producer<false, false, kRing>(p, sm, bars, nk);
  } else if (kRing && warp == kRingWarp) {
    ring_agent(p, lane);
  } else if (warp >= kGWarp) {
    ws_gather_producer<false, false, kRing, kEW>(p, sm, bars, nk);
  } else if (warp == 1) {
    // The whole warp runs the MMA loop (barrier waits converged) and one
    // elected lane issues each GEMM: issued from a lane-0-only branch, ptxas
    // wrapped every tcgen05.mma in its own ELECT / PLOP3 / BRA loop, ~50
    // dependent cycles per MMA that kept this warp ~93% busy (36 per tile).
    {
      constexpr uint32_t id = idesc_tf32(128, kW, 0, 0);
      // atomic rows: N = 64, [C | A] = A [B | I]
      constexpr uint32_t idc = idesc_tf32(128, kAtomic ? 2 * kW : kW, 0, 0);
      const uint32_t bt = smem_u32(sm + L::o_bt), bb = smem_u32(sm + L::o_b);
      const uint32_t dg = smem_u32(sm + L::o_diag);
      // U(j) = (lr r D_j) B^T [+ A_j (-lr reg I)]: the step itself (atomic
      // rows) or U for the overwrite rule (scaled in the epilogue).
      auto issue_u = [&](int64_t j) {
        const int b = (int)(j & 1);
        mbar_wait(&bars[B_DFULL + b], (uint32_t)((j >> 1) & 1));
        mbar_wait(&bars[B_UEMPTY], (uint32_t)((j & 1) ^ 1));
        tc_after();
        const uint32_t tb = tmem + kC + b * kBuf;
        if (elect_one()) {
#pragma unroll
          for (int n = 0; n < kN; ++n) {
#pragma unroll
            for (int ks = 0; ks < kW / 8; ++ks)
              mma_ts(tmem + kU + n * kW, tb + n * kMs + ks * 8,
                     sdesc(bb + n * 4096 + ks * 32, 16, 1024, 128), id, ks > 0);
            if constexpr (kAtomic)
              if (!(ws_exp(p) & 256))  // exp 256: no regulariser GEMM (timing only)
#pragma unroll
                for (int ks = 0; ks < kW / 8; ++ks)
                  mma_ts(tmem + kU + n * kW, tb + n * kMs + kW + ks * 8,
                         sdesc(dg + ks * 32, 16, 1024, 128), id, 1);
          }
          mma_commit(&bars[B_UFULL]);
        }
        __syncwarp();
      };
      // ring: at a cell boundary U(k - 1) goes out BEFORE the wait for tile
      // k's rows, so a cell's write-back (and the block posts behind it)
      // never waits for the next cell's blocks to arrive
      RingCursor mc;
      if constexpr (kRing) mc.enter(p.ring, 0);
      for (int64_t k = 0; k < nk; ++k) {
        const int s = (int)(k % kS), b = (int)(k & 1);
        bool early_u = false;
        if constexpr (kRing) {
          early_u = k >= 1 && mc.j == 0;
          mc.next(p.ring);
          if (early_u) {
            if (k >= 2) mbar_wait(&bars[B_UFULL], (uint32_t)((k - 2) & 1));
            issue_u(k - 1);
          }
        }
        mbar_wait(&bars[B_FULL + s], (uint32_t)((k / kS) & 1));
        // C(k) overwrites buffer b, whose D'(k - 2) is U(k - 2)'s A operand:
        // issue it once U(k - 2) has completed (PTX orders MMAs only per
        // accumulator; U(k - 1) is not issued yet, so the phase is exact)
        // (exp 512: no wait -- timing only, corrupts D')
        if (k >= 2 && !early_u && !(ws_exp(p) & 512)) mbar_wait(&bars[B_UFULL], (uint32_t)((k - 2) & 1));
        tc_after();
        const uint32_t a0 = smem_u32(sm + L::o_a + s * L::kSlot);
        if (elect_one()) {
#pragma unroll
          for (int n = 0; n < kN; ++n)
#pragma unroll
            for (int ks = 0; ks < kW / 8; ++ks)
              mma_ss(tmem + kC + b * kBuf + n * kMs,
                     sdesc(a0 + n * kModeTile + ks * 32, 16, 1024, 128),
                     sdesc(bt + n * 8192 + ks * 32, 16, 1024, 128), idc, ks > 0);
          mma_commit(&bars[B_CFULL + b]);
          // the only read of the A slot (window: held until the write-back)
          if (kAtomic && !p.window) mma_commit(&bars[B_EMPTY + s]);
        }
        __syncwarp();
        if (k >= 1 && !early_u) issue_u(k - 1);
      }
      if (nk >= 1) issue_u(nk - 1);
    }
  } else {
    const int ew = warp - 2, q = warp & 3, h = ew >> 2;  // h: column group of the quarter
    const int row = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    // Software pipeline: epi1(k + 1) runs while U(k) is on the tensor core.
    // epi1: C -> residual -> D' = (lr r) D into TMEM, global row indices into
    // registers.  epi2: U -> step -> coalesced vector RED (or STG) of whole
    // rows.
    struct Tile {
      int32_t g[kN];
      float resid;
      bool ok;
      int slot;
    };
    Tile cur, nxt;
    auto epi1 = [&](int64_t k, Tile& t) {
      const int s = (int)(k % kS), b = (int)(k & 1), ii = (int)(k % L::kI);
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + ii * L::kIdxSlot);
      const float* s_val = reinterpret_cast<const float*>(s_idx + kN * kRows);
      mbar_wait(&bars[B_CFULL + b], (uint32_t)((k >> 1) & 1));
      tc_after();
      const uint32_t tb = tl + kC + b * kBuf;
      float c[kN][kCc];
      {  // the three modes' columns in flight before one wait
        uint32_t v[kN][kCc];
#pragma unroll
        for (int n = 0; n < kN; ++n) tmem_ldc(tb + n * kMs + h * kCc, v[n]);
        tmem_wait_ld();
#pragma unroll
        for (int n = 0; n < kN; ++n)
#pragma unroll
          for (int i = 0; i < kCc; ++i) c[n][i] = __uint_as_float(v[n][i]);
      }
      // x_hat partial sums exchanged among the quarter's kH warps (each warp
      // reads only its columns of C, so D' can go over them in place)
      f2 acc = {0.0f, 0.0f};
#pragma unroll
      for (int i = 0; i < kCc / 2; ++i)
        acc = fma2(f2{c[0][2 * i], c[0][2 * i + 1]},
                   mul2(f2{c[1][2 * i], c[1][2 * i + 1]}, f2{c[2][2 * i], c[2][2 * i + 1]}), acc);
      float* xp = reinterpret_cast<float*>(sm + L::o_xp);  // [2 tiles][kH][128]
      xp[(b * kH + h) * kRows + row] = acc.x + acc.y;
      named_bar(1 + q, 32 * kH);
      float xhat = 0.0f;
#pragma unroll
      for (int g = 0; g < kH; ++g) xhat += xp[(b * kH + g) * kRows + row];
      t.slot = s;
#pragma unroll
      for (int n = 0; n < kN; ++n) t.g[n] = s_idx[n * kRows + row];
      const float xv = s_val[row];
      const int nvalid = reinterpret_cast<const int32_t*>(sm + L::o_rows)[ii];
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_IEMPTY + ii]);  // COO slot may be refilled
      t.ok = row < nvalid;
      t.resid = t.ok ? xv - xhat : 0.0f;
      // padding rows carry row index -1: epi2 then needs one shuffle per row
#pragma unroll
      for (int n = 0; n < kN; ++n) t.g[n] = t.ok ? t.g[n] : -1;
      // kAtomic: D' = lr r D, so the U GEMM (plus A x (-lr reg I)) yields the
      // step itself; overwrite mode scales in epi2.
      const float sc = kAtomic ? p.lr * t.resid : 1.0f;
      const f2 s2 = {sc, sc};
      f2 c0[kCc / 2], c1[kCc / 2], c2[kCc / 2];
#pragma unroll
      for (int i = 0; i < kCc / 2; ++i) {
        c0[i] = mul2(f2{c[0][2 * i], c[0][2 * i + 1]}, s2);  // D'_1 = (sc c0) c2, D'_2 = (sc c0) c1
        c1[i] = f2{c[1][2 * i], c[1][2 * i + 1]};
        c2[i] = f2{c[2][2 * i], c[2][2 * i + 1]};
      }
#pragma unroll
      for (int n = 0; n < kN; ++n) {
        uint32_t v[kCc];
#pragma unroll
        for (int i = 0; i < kCc / 2; ++i) {
          const f2 d = n == 0 ? mul2(mul2(c1[i], s2), c2[i])
                              : (n == 1 ? mul2(c0[i], c2[i]) : mul2(c0[i], c1[i]));
          v[2 * i] = tf32_rn_bits(d.x);
          v[2 * i + 1] = tf32_rn_bits(d.y);
        }
        tmem_stc(tb + n * kMs + h * kCc, v);
      }
      tmem_wait_st();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_DFULL + b]);
    };
    auto epi2 = [&](int64_t k, const Tile& t) {
      // the row indices of the 4-row RED groups, shuffled before the wait:
      // this warp sends rows kCc h + 4 i + lane / 8 of its lane quarter
      int32_t gq[kN][kRi];
#pragma unroll
      for (int n = 0; n < kN; ++n)
#pragma unroll
        for (int i = 0; i < kRi; ++i)
          gq[n][i] = __shfl_sync(0xffffffffu, t.g[n], h * kCc + i * 4 + (lane >> 3));
      mbar_wait(&bars[B_UFULL], (uint32_t)(k & 1));
      tc_after();
      uint32_t u[kN][kCc];
#pragma unroll
      for (int n = 0; n < kN; ++n) tmem_ldc(tl + kU + n * kW + h * kCc, u[n]);
      tmem_wait_ld();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_UEMPTY]);
      const float lr_r = p.lr * t.resid, lr_reg = p.lr * p.reg;
      const uint8_t* slot = sm + L::o_a + t.slot * L::kSlot;
      // Per mode: the lane quarter's kH warps write their columns of the
      // quarter's 32 step rows into a shared 4 KB staging tile (128-B rows,
      // SWIZZLE_128B chunks: conflict-free both ways), then each sends 32 / kH
      // whole rows, 4 rows of 128 B per RED (or STG) instruction: half the L1
      // wavefronts / L2 requests of 64-B segments for the same bytes
      // (scripts/microtests/red_segments.cu: 6.3 vs 5.3 TB/s).  Two named
      // barriers per mode (columns written / tile read).
      uint8_t* stage = sm + L::o_stage + q * 4096;
#pragma unroll
      for (int n = 0; n < kN; ++n) {
#pragma unroll
        for (int q4 = 0; q4 < kCc / 4; ++q4) {
          float4 st;
          if constexpr (kAtomic) {  // the accumulator already holds the step
            st = make_float4(__uint_as_float(u[n][q4 * 4 + 0]), __uint_as_float(u[n][q4 * 4 + 1]),
                             __uint_as_float(u[n][q4 * 4 + 2]), __uint_as_float(u[n][q4 * 4 + 3]));
          } else {
            const float4 a = *reinterpret_cast<const float4*>(
                slot + n * kModeTile + swz(row, (h * kCc + q4 * 4) * 4, 128));
            st.x = a.x + fmaf(lr_r, __uint_as_float(u[n][q4 * 4 + 0]), -lr_reg * a.x);
            st.y = a.y + fmaf(lr_r, __uint_as_float(u[n][q4 * 4 + 1]), -lr_reg * a.y);
            st.z = a.z + fmaf(lr_r, __uint_as_float(u[n][q4 * 4 + 2]), -lr_reg * a.z);
            st.w = a.w + fmaf(lr_r, __uint_as_float(u[n][q4 * 4 + 3]), -lr_reg * a.w);
          }
          *reinterpret_cast<float4*>(stage + swz(lane, h * kCc * 4 + q4 * 16, 128)) = st;
        }
        named_bar(5 + q, 32 * kH);  // every column of the quarter's rows staged
        float* dst = p.a[n];
        // The last mode, accumulate rule: when all of this warp's rows update
        // one row (DSGD cells laid out in mode-3 runs), sum them and send one
        // row -- the updates of a small block's rows otherwise queue on the
        // same L2 lines (red_segments: 1.9 TB/s on 273 rows vs 6.3 spread).
        bool merged = false;
        if constexpr (kAtomic) {
          if (n == kN - 1) {
            const int32_t g0 = __shfl_sync(0xffffffffu, t.g[n], h * kCc);
            bool same = g0 >= 0;
#pragma unroll
            for (int i = 0; i < kRi; ++i) same = same && gq[n][i] == g0;
            if (__all_sync(0xffffffffu, same)) {
              const int ch = lane & 7;
              float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int i = 0; i < kRi; ++i) {
                const int rl = h * kCc + i * 4 + (lane >> 3);
                const float4 v = *reinterpret_cast<const float4*>(stage + swz(rl, ch * 16, 128));
                acc.x += v.x;
                acc.y += v.y;
                acc.z += v.z;
                acc.w += v.w;
              }
#pragma unroll
              for (int o = 8; o < 32; o <<= 1) {
                acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
                acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
              }
              if (lane < 8 && !(ws_exp(p) & 16)) red_add_v4(dst + (size_t)g0 * kW + ch * 4, acc);
              merged = true;
            }
          }
        }
        if (!merged) {
#pragma unroll
          for (int i = 0; i < kRi; ++i) {
            const int rl = h * kCc + i * 4 + (lane >> 3), ch = lane & 7;
            const int32_t g = gq[n][i];
            const float4 v = *reinterpret_cast<const float4*>(stage + swz(rl, ch * 16, 128));
            if (g >= 0 && !(ws_exp(p) & 16)) {  // exp 16: no write-back (timing only)
              float* gp = dst + (size_t)g * kW + ch * 4;
              if constexpr (kAtomic)
                red_add_v4(gp, v);
              else
                *reinterpret_cast<float4*>(gp) = v;
            }
          }
        }
        named_bar(5 + q, 32 * kH);  // the quarter is done reading before the next mode's stores
      }
      if (!kAtomic || p.window) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_EMPTY + t.slot]);
      }
    };
    // ring: a cell's count goes in one tile late (its REDs have landed by
    // then, so the fence is cheap) when the next tile is in the next cell and
    // the neighbour needs the block only K >= 2 cells later; otherwise (a
    // round's end, skipped cells, K = 1) right away -- a deferred count that
    // waited on a block the neighbour posts from the same cell index would
    // close a cycle around the ring
    RingCursor rc;
    int pending = -1;
    const int rq = p.ring.parts > 0 ? p.ring.ncell / p.ring.parts : 1;
    const bool can_defer = rq >= 2 * p.ring.parts;
    if constexpr (ring) {
      rc.enter(p.ring, 0);
      for (int c = 0; c < rc.c; ++c) ring_done(p, c, lane);  // no tiles here
    }
    if (nk > 0) epi1(0, cur);
    for (int64_t k = 0; k < nk; ++k) {
      if constexpr (ring) {
        // the last tile of a cell: write-back first, the next cell's epilogue
        // after (its rows may still be on their way)
        const int c0 = rc.c;
        rc.next(p.ring);
        if (rc.c != c0) {
          epi2(k, cur);
          if (pending >= 0) ring_done(p, pending, lane);
          pending = -1;
          const bool round_end = rc.c >= p.ring.ncell || rc.c / rq != c0 / rq;
          if (round_end || !can_defer || rc.c != c0 + 1) ring_done(p, c0, lane);
          else pending = c0;
          for (int c = c0 + 1; c < rc.c; ++c) ring_done(p, c, lane);  // no tiles here
          if (k + 1 < nk) epi1(k + 1, nxt);
        } else {
          if (k + 1 < nk) epi1(k + 1, nxt);
          epi2(k, cur);
          if (pending >= 0) ring_done(p, pending, lane);
          pending = -1;
        }
      } else {
        if (k + 1 < nk) epi1(k + 1, nxt);
        epi2(k, cur);
      }
      cur = nxt;
    }
  }
  // ring: the blocks this rank holds at the epoch's end have landed
  if (kRing && blockIdx.x == 0 && threadIdx.x == 0)
    for (int f = 0; f < p.ring.nfinal; ++f) ring_wait(p.ring, __ldg(p.ring.final_waits + f));
  ws_teardown(tmem);
}

// ---- factor sweep, 3xtf32 ----------------------------------------------------------
//
// fp32-equivalent products on the tf32 tensor cores (hi*hi + hi*lo + lo*hi,
// the split of ws_core_kernel / tc_factor_kernel) for the headline shape:
//   C_n = A B_n:    A straight from the slot (the tensor core reads its tf32
//                   truncation A_hi); A_lo = A - A_hi staged into TMEM by the
//                   epilogue; B hi / lo in shared memory;
//   U_n = D_n B_n^T with D_n = prod_{m != n} C_m split hi / lo by the
//                   epilogue into TMEM (hi over C_n, lo over A_lo_n);
//   step           = lr (r u - reg a) in fp32 in the epilogue with a from the
//                   slot -- the reference's own expression
//                   (decomposition.cpp:257-270) -- then RED.ADD (the Hogwild
//                   accumulate rule).
// TMEM: buffer b = k & 1 at 192 b; mode n at +64 n: C_n / D_hi_n (32
// columns), then A_lo_n / D_lo_n (32); U at 384.  The epilogue releases the
// slot after the step (it reads a there), and stages A_lo(k + 2) only after
// epi2(k) has seen U(k) complete, so C(k + 2) is never issued into buffer
// k & 1 before U(k) has read D(k) from it: no reliance on execution order
// between MMAs of different accumulators.
__global__ void __launch_bounds__(kThreadsWs, 1) ws_factor3_kernel(const __grid_constant__ WsParams p) {
  using L = WsLayout<false, true>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::o_bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + L::o_tmem);
  ws_setup<false, true>(p, sm, bars, tslot);
  const uint32_t tmem = *tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nk = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  constexpr uint32_t kU = 384, kBuf = 192, kMs = 64;

  if (warp == 0) {
    ws_idx_producer<false, true>(p, sm, bars, nk);
  } else if (warp >= kGatherWarp) {
    ws_gather_producer<false, true>(p, sm, bars, nk);
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id = idesc_tf32(128, kW, 0, 0);
      const uint32_t bt = smem_u32(sm + L::o_bt), bb = smem_u32(sm + L::o_b);
      const uint32_t bl = smem_u32(sm + L::o_diag);
      auto issue_u = [&](int64_t j) {
        const int b = (int)(j & 1);
        mbar_wait(&bars[B_DFULL + b], (uint32_t)((j >> 1) & 1));
        mbar_wait(&bars[B_UEMPTY], (uint32_t)((j & 1) ^ 1));
        tc_after();
        const uint32_t tb = tmem + b * kBuf;
#pragma unroll
        for (int n = 0; n < kN; ++n)
#pragma unroll
          for (int ks = 0; ks < kW / 8; ++ks) {
            const uint64_t dh = sdesc(bb + n * 4096 + ks * 32, 16, 1024, 128);
            mma_ts(tmem + kU + n * kW, tb + n * kMs + ks * 8, dh, id, ks > 0);
            mma_ts(tmem + kU + n * kW, tb + n * kMs + ks * 8,
                   sdesc(bl + n * 4096 + ks * 32, 16, 1024, 128), id, 1);
            mma_ts(tmem + kU + n * kW, tb + n * kMs + kW + ks * 8, dh, id, 1);
          }
        mma_commit(&bars[B_UFULL]);
      };
      for (int64_t k = 0; k < nk; ++k) {
        const int s = (int)(k % kS), b = (int)(k & 1);
        mbar_wait(&bars[B_FULL + s], (uint32_t)((k / kS) & 1));
        mbar_wait(&bars[B_LOFULL + b], (uint32_t)((k >> 1) & 1));
        tc_after();
        const uint32_t a0 = smem_u32(sm + L::o_a + s * L::kSlot);
        const uint32_t tb = tmem + b * kBuf;
#pragma unroll
        for (int n = 0; n < kN; ++n)
#pragma unroll
          for (int ks = 0; ks < kW / 8; ++ks) {
            const uint64_t da = sdesc(a0 + n * kModeTile + ks * 32, 16, 1024, 128);
            const uint64_t dh = sdesc(bt + n * 8192 + ks * 32, 16, 1024, 128);
            mma_ss(tb + n * kMs, da, dh, id, ks > 0);
            mma_ss(tb + n * kMs, da, sdesc(bt + n * 8192 + 4096 + ks * 32, 16, 1024, 128), id, 1);
            mma_ts(tb + n * kMs, tb + n * kMs + kW + ks * 8, dh, id, 1);
          }
        mma_commit(&bars[B_CFULL + b]);
        if (k >= 1) issue_u(k - 1);
      }
      if (nk >= 1) issue_u(nk - 1);
    }
  } else {
    const int ew = warp - 2, q = warp & 3, h = ew >> 2;
    const int row = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    struct Tile {
      int32_t g[kN];
      float resid;
      int slot;
    };
    Tile cur, nxt;
    // A_lo of this thread's row (column half h) -> TMEM buffer k & 1
    auto stage_lo = [&](int64_t k) {
      const int s = (int)(k % kS), b = (int)(k & 1);
      mbar_wait(&bars[B_FULL + s], (uint32_t)((k / kS) & 1));
      const uint8_t* slot = sm + L::o_a + s * L::kSlot;
#pragma unroll
      for (int n = 0; n < kN; ++n) {
        uint32_t v[16];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 x = *reinterpret_cast<const float4*>(
              slot + n * kModeTile + swz(row, (h * 16 + q4 * 4) * 4, 128));
          v[q4 * 4 + 0] = tf32_rn_bits(x.x - tf32_trunc(x.x));
          v[q4 * 4 + 1] = tf32_rn_bits(x.y - tf32_trunc(x.y));
          v[q4 * 4 + 2] = tf32_rn_bits(x.z - tf32_trunc(x.z));
          v[q4 * 4 + 3] = tf32_rn_bits(x.w - tf32_trunc(x.w));
        }
        tmem_st16(tl + b * kBuf + n * kMs + kW + h * 16, v);
      }
      tmem_wait_st();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_LOFULL + b]);
    };
    auto epi1 = [&](int64_t k, Tile& t) {
      const int s = (int)(k % kS), b = (int)(k & 1), ii = (int)(k % L::kI);
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + ii * L::kIdxSlot);
      const float* s_val = reinterpret_cast<const float*>(s_idx + kN * kRows);
      mbar_wait(&bars[B_CFULL + b], (uint32_t)((k >> 1) & 1));
      tc_after();
      const uint32_t tb = tl + b * kBuf;
      float c[kN][16];
      {
        uint32_t v[kN][16];
#pragma unroll
        for (int n = 0; n < kN; ++n) tmem_ld16(tb + n * kMs + h * 16, v[n]);
        tmem_wait_ld();
#pragma unroll
        for (int n = 0; n < kN; ++n)
#pragma unroll
          for (int i = 0; i < 16; ++i) c[n][i] = __uint_as_float(v[n][i]);
      }
      float part = 0.0f;
#pragma unroll
      for (int i = 0; i < 16; ++i) part = fmaf(c[0][i], c[1][i] * c[2][i], part);
      float* xp = reinterpret_cast<float*>(sm + L::o_xp);
      xp[(b * 2 + h) * kRows + row] = part;
      named_bar(1 + q, 64);
      const float xhat = part + xp[(b * 2 + (h ^ 1)) * kRows + row];
      t.slot = s;
#pragma unroll
      for (int n = 0; n < kN; ++n) t.g[n] = s_idx[n * kRows + row];
      const float xv = s_val[row];
      const int nvalid = reinterpret_cast<const int32_t*>(sm + L::o_rows)[ii];
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_IEMPTY + ii]);
      const bool ok = row < nvalid;
      t.resid = ok ? xv - xhat : 0.0f;
#pragma unroll
      for (int n = 0; n < kN; ++n) t.g[n] = ok ? t.g[n] : -1;
      // D_n split: hi = the tf32 the tensor core reads (round to nearest),
      // lo = the exact remainder (rounded to tf32 in turn)
#pragma unroll
      for (int n = 0; n < kN; ++n) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float d = n == 0 ? c[1][i] * c[2][i] : (n == 1 ? c[0][i] * c[2][i] : c[0][i] * c[1][i]);
          hi[i] = tf32_rn_bits(d) & 0xFFFFE000u;
          lo[i] = tf32_rn_bits(d - __uint_as_float(hi[i]));
        }
        tmem_st16(tb + n * kMs + h * 16, hi);
        tmem_st16(tb + n * kMs + kW + h * 16, lo);
      }
      tmem_wait_st();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_DFULL + b]);
    };
    auto epi2 = [&](int64_t k, const Tile& t) {
      int32_t gq[kN][4];  // rows 16 h + 4 i + lane / 8 of the quarter (as ws_factor_kernel)
#pragma unroll
      for (int n = 0; n < kN; ++n)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          gq[n][i] = __shfl_sync(0xffffffffu, t.g[n], h * 16 + i * 4 + (lane >> 3));
      mbar_wait(&bars[B_UFULL], (uint32_t)(k & 1));
      tc_after();
      uint32_t u[kN][16];
#pragma unroll
      for (int n = 0; n < kN; ++n) tmem_ld16(tl + kU + n * kW + h * 16, u[n]);
      tmem_wait_ld();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_UEMPTY]);
      const float r = t.resid, lr = p.lr, reg = p.reg;
      const uint8_t* slot = sm + L::o_a + t.slot * L::kSlot;
      uint8_t* stage = sm + L::o_stage + q * 4096;  // the quarter's whole 128-B rows
#pragma unroll
      for (int n = 0; n < kN; ++n) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 a = *reinterpret_cast<const float4*>(
              slot + n * kModeTile + swz(row, (h * 16 + q4 * 4) * 4, 128));
          float4 st;
          st.x = lr * (r * __uint_as_float(u[n][q4 * 4 + 0]) - reg * a.x);
          st.y = lr * (r * __uint_as_float(u[n][q4 * 4 + 1]) - reg * a.y);
          st.z = lr * (r * __uint_as_float(u[n][q4 * 4 + 2]) - reg * a.z);
          st.w = lr * (r * __uint_as_float(u[n][q4 * 4 + 3]) - reg * a.w);
          *reinterpret_cast<float4*>(stage + swz(lane, h * 64 + q4 * 16, 128)) = st;
        }
        named_bar(5 + q, 64);
        float* dst = p.a[n];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int rl = h * 16 + i * 4 + (lane >> 3), ch = lane & 7;
          const int32_t g = gq[n][i];
          const float4 v = *reinterpret_cast<const float4*>(stage + swz(rl, ch * 16, 128));
          if (g >= 0) red_add_v4(dst + (size_t)g * kW + ch * 4, v);
        }
        named_bar(5 + q, 64);
      }
      if (lane == 0) mbar_arrive(&bars[B_EMPTY + t.slot]);  // a read: the slot is free
    };
    if (nk > 0) stage_lo(0);
    if (nk > 1) stage_lo(1);
    if (nk > 0) epi1(0, cur);
    for (int64_t k = 0; k < nk; ++k) {
      if (k + 1 < nk) epi1(k + 1, nxt);
      epi2(k, cur);
      if (k + 2 < nk) stage_lo(k + 2);  // U(k) has completed: buffer k & 1 is free
      cur = nxt;
    }
  }
  ws_teardown(tmem);
}

// ---- core sweep ------------------------------------------------------------------

__global__ void __launch_bounds__(kThreadsWs, 1) ws_core_kernel(const __grid_constant__ WsParams p) {
  using L = WsLayout<true>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::o_bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + L::o_tmem);
  ws_setup<true>(p, sm, bars, tslot);
  const uint32_t tmem = *tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nk = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // TMEM: C[b] at 96 b; G at 192; A rows hi at 288, lo at 384.
  constexpr uint32_t kG = 192, kAhi = 288, kAlo = 384;

  if (warp == 0) {
    ws_idx_producer<true>(p, sm, bars, nk);
  } else if (warp >= kGatherWarp) {
    ws_gather_producer<true>(p, sm, bars, nk);
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idc = idesc_tf32(128, kW, 0, 0);
      constexpr uint32_t idg = idesc_tf32(128, kN * kW, 1, 1);  // all modes' D at once
      const uint32_t bt = smem_u32(sm + L::o_bt), btl = smem_u32(sm + L::o_btlo);
      const uint32_t d0 = smem_u32(sm + L::o_d);
      auto issue_g = [&](int64_t k) {
        const int s = (int)(k % kS);
        mbar_wait(&bars[B_DFULL], (uint32_t)(k & 1));
        tc_after();
        // G[j'][n' R + r] += sum_t A[t][j'] (r D_n')[t][r]: one N = 96 MMA per
        // 8 nonzeros; only the diagonal blocks n' = mode(j') are read back.
        const uint32_t a0 = smem_u32(sm + L::o_a + s * L::kSlot);
        const uint64_t da = sdesc_l(a0, kModeTile, 512, 1);
        const uint64_t dd = sdesc_l(d0, kModeTile, 512, 1);
        if (!(ws_exp(p) & 4))  // exp 4: no G GEMM (timing only)
#pragma unroll 4
          for (int ks = 0; ks < kRows / 8; ++ks)
            mma_ss(tmem + kG, da + (uint64_t)(ks * 64), dd + (uint64_t)(ks * 64), idg,
                   (k > 0 || ks > 0) ? 1u : 0u);
        mma_commit(&bars[B_DEMPTY]);
        if (!(ws_exp(p) & 1)) mma_commit(&bars[B_EMPTY + s]);
      };
      for (int64_t k = 0; k < nk; ++k) {
        const int b = (int)(k & 1);
        mbar_wait(&bars[B_AFULL], (uint32_t)(k & 1));
        tc_after();
#pragma unroll
        for (int n = 0; n < kN; ++n)
#pragma unroll
          for (int ks = 0; ks < kW / 8; ++ks) {
            const uint64_t db = sdesc(bt + n * 4096 + ks * 32, 16, 1024, 128);
            mma_ts(tmem + b * 96 + n * kW, tmem + kAhi + n * kW + ks * 8, db, idc, ks > 0);
            if (p.prec3) {
              mma_ts(tmem + b * 96 + n * kW, tmem + kAhi + n * kW + ks * 8,
                     sdesc(btl + n * 4096 + ks * 32, 16, 1024, 128), idc, 1);
              mma_ts(tmem + b * 96 + n * kW, tmem + kAlo + n * kW + ks * 8, db, idc, 1);
            }
          }
        mma_commit(&bars[B_CFULL + b]);
        if (ws_exp(p) & 1) mma_commit(&bars[B_EMPTY + (int)(k % kS)]);  // exp: slot freed after C
        if (k >= 1) issue_g(k - 1);
      }
      if (nk >= 1) issue_g(nk - 1);
    }
  } else {
    const int ew = warp - 2, q = warp & 3, h = ew >> 2;
    const int row = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    // Own row (half h of each mode) -> TMEM: the smem tile is in the MN-major
    // layout of the G GEMM, which the K-major C GEMM cannot read.
    auto stage_a = [&](int64_t k) {
      const int s = (int)(k % kS);
      mbar_wait(&bars[B_FULL + s], (uint32_t)((k / kS) & 1));
      const uint8_t* slot = sm + L::o_a + s * L::kSlot;
#pragma unroll
      for (int n = 0; n < kN; ++n) {
        uint32_t v[16];
        if (ws_exp(p) & 8) {  // exp 8: no smem reads of the rows (timing only)
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0x3f800000u;
        } else
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 x = *reinterpret_cast<const float4*>(slot + n * kModeTile +
                                                            swz32(row, (h * 16 + q4 * 4) * 4));
          v[q4 * 4 + 0] = __float_as_uint(x.x);
          v[q4 * 4 + 1] = __float_as_uint(x.y);
          v[q4 * 4 + 2] = __float_as_uint(x.z);
          v[q4 * 4 + 3] = __float_as_uint(x.w);
        }
        if (p.prec3) {  // exact split: hi = what the tensor core reads, lo = rest
          tmem_st16(tl + kAhi + n * kW + h * 16, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float x = __uint_as_float(v[i]);
            v[i] = __float_as_uint(x - tf32_trunc(x));
          }
          tmem_st16(tl + kAlo + n * kW + h * 16, v);
        } else {  // single pass: round to nearest instead of truncating
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += 0x1000u;
          tmem_st16(tl + kAhi + n * kW + h * 16, v);
        }
      }
      tmem_wait_st();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_AFULL]);
    };
    if (nk > 0) stage_a(0);
    for (int64_t k = 0; k < nk; ++k) {
      const int b = (int)(k & 1), ii = (int)(k % L::kI);
      const int64_t tile = ws_tile(p, k);
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + ii * L::kIdxSlot);
      const float* s_val = reinterpret_cast<const float*>(s_idx + kN * kRows);
      mbar_wait(&bars[B_CFULL + b], (uint32_t)((k >> 1) & 1));
      tc_after();
      float c[kN][16];
#pragma unroll
      for (int n = 0; n < kN; ++n) {
        uint32_t v[16];
        tmem_ld16(tl + b * 96 + n * kW + h * 16, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) c[n][i] = __uint_as_float(v[i]);
      }
      const float xhat = xhat_full(tl + b * 96 + (h ^ 1) * 16, c);
      if (k + 1 < nk) stage_a(k + 1);  // C(k) is complete: A rows TMEM is free
      const bool ok = row < reinterpret_cast<const int32_t*>(sm + L::o_rows)[ii];
      const float resid = ok ? s_val[row] - xhat : 0.0f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_IEMPTY + ii]);
      mbar_wait(&bars[B_DEMPTY], (uint32_t)((k & 1) ^ 1));  // G(k-1) done with the D tile
#pragma unroll
      for (int n = 0; n < kN; ++n)
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          float4 d;
          const int i = q4 * 4;
#define FTK_D(ii) (n == 0 ? c[1][ii] * c[2][ii] : (n == 1 ? c[0][ii] * c[2][ii] : c[0][ii] * c[1][ii]))
          d.x = __uint_as_float(tf32_rn_bits(resid * FTK_D(i + 0)));
          d.y = __uint_as_float(tf32_rn_bits(resid * FTK_D(i + 1)));
          d.z = __uint_as_float(tf32_rn_bits(resid * FTK_D(i + 2)));
          d.w = __uint_as_float(tf32_rn_bits(resid * FTK_D(i + 3)));
#undef FTK_D
          *reinterpret_cast<float4*>(sm + L::o_d + n * kModeTile +
                                     swz32(row, (h * 16 + i) * 4)) = d;
        }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_DFULL]);
    }
    // Publish this CTA's gradient once the last G GEMM has landed: TMEM lane
    // j' = 32 n + j (quarter q = mode n) holds G_n[j][:], half h = columns.
    if (nk > 0) mbar_wait(&bars[B_DEMPTY], (uint32_t)((nk - 1) & 1));
    tc_after();
    if (q < kN) {
      uint32_t v[16];
      tmem_ld16(tl + kG + q * kW + h * 16, v);
      tmem_wait_ld();
      float* out = p.partials + (size_t)blockIdx.x * (kN * kW * kW) + ((size_t)q * kW + lane) * kW + h * 16;
#pragma unroll
      for (int i = 0; i < 16; ++i) out[i] = nk > 0 ? __uint_as_float(v[i]) : 0.0f;
    }
  }
  ws_teardown(tmem);
}

// ---- core sweep, storage scheme -------------------------------------------------
//
// Same sweep with C rows read from the C cache (CCache, decomposition.cpp:
// 299-314) instead of computed: no C GEMM and no TMEM copy of the rows.  The
// epilogue loads its half of every C row straight from the (L2-resident)
// cache one tile ahead, exchanges the x_hat halves through shared memory,
// and writes r D for the G GEMM, the MMA warp's only work.

__global__ void __launch_bounds__(kThreadsWs, 1) ws_core_cc_kernel(const __grid_constant__ WsParams p) {
  using L = WsLayout<true>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::o_bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + L::o_tmem);
  ws_setup<true>(p, sm, bars, tslot);
  const uint32_t tmem = *tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nk = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  constexpr uint32_t kG = 0;  // TMEM: G only

  if (warp == 0) {
    ws_idx_producer<true>(p, sm, bars, nk);
  } else if (warp >= kGatherWarp) {
    ws_gather_producer<true>(p, sm, bars, nk);
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idg = idesc_tf32(128, kN * kW, 1, 1);
      const uint32_t d0 = smem_u32(sm + L::o_d);
      for (int64_t k = 0; k < nk; ++k) {
        const int s = (int)(k % kS);
        mbar_wait(&bars[B_FULL + s], (uint32_t)((k / kS) & 1));
        mbar_wait(&bars[B_DFULL], (uint32_t)(k & 1));
        tc_after();
        const uint64_t da = sdesc_l(smem_u32(sm + L::o_a + s * L::kSlot), kModeTile, 512, 1);
        const uint64_t dd = sdesc_l(d0, kModeTile, 512, 1);
#pragma unroll 4
        for (int ks = 0; ks < kRows / 8; ++ks)
          mma_ss(tmem + kG, da + (uint64_t)(ks * 64), dd + (uint64_t)(ks * 64), idg,
                 (k > 0 || ks > 0) ? 1u : 0u);
        mma_commit(&bars[B_DEMPTY]);
        mma_commit(&bars[B_EMPTY + s]);
      }
    }
  } else {
    const int ew = warp - 2, q = warp & 3, h = ew >> 2;
    const int row = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    float* xp = reinterpret_cast<float*>(sm + L::o_xp);  // [2 tiles][2 halves][128]
    // This thread's column half of the tile's C rows, from the cache.
    auto fetch = [&](int64_t k, float (&c)[kN][16]) {
      const int ii = (int)(k % L::kI);
      mbar_wait(&bars[B_IFULL + ii], (uint32_t)((k / L::kI) & 1));
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + ii * L::kIdxSlot);
#pragma unroll
      for (int n = 0; n < kN; ++n) {
        const float4* src =
            reinterpret_cast<const float4*>(p.cc[n] + (size_t)s_idx[n * kRows + row] * kW + h * 16);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 x = __ldg(src + q4);
          c[n][q4 * 4 + 0] = x.x;
          c[n][q4 * 4 + 1] = x.y;
          c[n][q4 * 4 + 2] = x.z;
          c[n][q4 * 4 + 3] = x.w;
        }
      }
    };
    float cur[kN][16], nxt[kN][16];
    if (nk > 0) fetch(0, cur);
    for (int64_t k = 0; k < nk; ++k) {
      const int b = (int)(k & 1), ii = (int)(k % L::kI), s = (int)(k % kS);
      if (k + 1 < nk) fetch(k + 1, nxt);
      float part = 0.0f;
#pragma unroll
      for (int i = 0; i < 16; ++i) part = fmaf(cur[0][i], cur[1][i] * cur[2][i], part);
      xp[(b * 2 + h) * kRows + row] = part;
      named_bar(1 + q, 64);
      const float xhat = part + xp[(b * 2 + (h ^ 1)) * kRows + row];
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + ii * L::kIdxSlot);
      const float* s_val = reinterpret_cast<const float*>(s_idx + kN * kRows);
      const bool ok = row < reinterpret_cast<const int32_t*>(sm + L::o_rows)[ii];
      const float resid = ok ? s_val[row] - xhat : 0.0f;
      // The gather warp reads this COO slot's indices: hold it until the
      // tile's rows have landed.
      mbar_wait(&bars[B_FULL + s], (uint32_t)((k / kS) & 1));
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_IEMPTY + ii]);
      mbar_wait(&bars[B_DEMPTY], (uint32_t)((k & 1) ^ 1));  // G(k-1) done with the D tile
#pragma unroll
      for (int n = 0; n < kN; ++n)
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          float4 d;
          const int i = q4 * 4;
#define FTK_D(ii) (n == 0 ? cur[1][ii] * cur[2][ii] : (n == 1 ? cur[0][ii] * cur[2][ii] : cur[0][ii] * cur[1][ii]))
          d.x = __uint_as_float(tf32_rn_bits(resid * FTK_D(i + 0)));
          d.y = __uint_as_float(tf32_rn_bits(resid * FTK_D(i + 1)));
          d.z = __uint_as_float(tf32_rn_bits(resid * FTK_D(i + 2)));
          d.w = __uint_as_float(tf32_rn_bits(resid * FTK_D(i + 3)));
#undef FTK_D
          *reinterpret_cast<float4*>(sm + L::o_d + n * kModeTile +
                                     swz32(row, (h * 16 + i) * 4)) = d;
        }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_DFULL]);
      if (k + 1 < nk) {
#pragma unroll
        for (int n = 0; n < kN; ++n)
#pragma unroll
          for (int i = 0; i < 16; ++i) cur[n][i] = nxt[n][i];
      }
    }
    if (nk > 0) mbar_wait(&bars[B_DEMPTY], (uint32_t)((nk - 1) & 1));
    tc_after();
    if (q < kN) {
      uint32_t v[16];
      tmem_ld16(tl + kG + q * kW + h * 16, v);
      tmem_wait_ld();
      float* out = p.partials + (size_t)blockIdx.x * (kN * kW * kW) + ((size_t)q * kW + lane) * kW + h * 16;
#pragma unroll
      for (int i = 0; i < 16; ++i) out[i] = nk > 0 ? __uint_as_float(v[i]) : 0.0f;
    }
  }
  ws_teardown(tmem);
}

// ---- core sweep, fp16 operand tile ------------------------------------------------
//
// The gathered rows feed two GEMMs that contract over different indices:
// C = A B over j (A K-major) and G += A^T (r D) over the nonzeros (A
// MN-major).  For tf32 tcgen05 reads MN-major operands only in the
// 128B_BASE32B swizzle, which ws_core_kernel gathers into and then copies row
// by row into TMEM for the C GEMM (the epilogue on the C GEMM's critical
// path).  For 16-bit operands any swizzle serves both majors, so this sweep
// gathers the rows of an fp16 copy of A (round-to-nearest, 10-bit mantissa
// like tf32; rebuilt per core phase, A is read-only here) ONCE into a
// 64-B-row SWIZZLE_64B tile that the C GEMM reads K-major and the G GEMM
// reads MN-major (scripts/microtests/umma_f16.cu), both kind::f16 with fp32
// accumulation.  Half the bytes per slot buys a 6-deep slot ring.
//
//   warp 0     COO columns (ring of kI)       warps 10-11  gathers (half each)
//   warp 1     MMA: C(k), then G(k - 1)       warps 2-9    epilogue: C -> r D (fp16)

constexpr uint32_t kModeTile16 = kRows * 64;  // 128 rows x 32 fp16
// C accumulators in TMEM (96 columns each): the C GEMM -> epilogue hand-off
// is latency-bound, so four tiles are in flight (two: 4.9 ms at C2)
constexpr int kCB = 4;

struct Ws16Layout {
  static constexpr uint32_t kSlot = kN * kModeTile16;  // 24 KB
  static constexpr int kS = 6;
  static constexpr uint32_t o_a = 0;
  // r D tiles (double-buffered); the G GEMM's 4th M segment of the last slot
  // reads into them
  static constexpr uint32_t o_d = o_a + kS * kSlot;
  static constexpr uint32_t o_bt = o_d + 2 * kSlot;  // B^T fp16, C GEMM operand
  static constexpr uint32_t o_idx = o_bt + kN * 2048;
  static constexpr uint32_t kIdxSlot = (kN + 1) * kRows * 4;
  static constexpr int kI = 6;
  static constexpr uint32_t o_rows = o_idx + kI * kIdxSlot;
  static constexpr uint32_t o_xp = o_rows + 64;  // x_hat halves [2 tiles][2 halves][128]
  static constexpr uint32_t o_bar = o_xp + 2 * 2 * kRows * 4;
  static constexpr uint32_t o_tmem = o_bar + 40 * 8;
  static constexpr uint32_t bytes = o_tmem + 16;
  static_assert(bytes <= 227 * 1024, "shared-memory budget");
};

enum : int {
  H_FULL = 0,     // [6] slot landed (one expect_tx arrival per gather warp)
  H_EMPTY = 6,    // [6] slot read by the G GEMM
  H_IFULL = 12,   // [6] COO columns landed
  H_IEMPTY = 18,  // [6] COO columns consumed (8 epilogue warps + 2 gather warps)
  H_CFULL = 24,   // [kCB] C accumulator ready
  H_CEMPTY = 28,  // [kCB] C accumulator read
  H_DFULL = 32,   // [2] r D tile written
  H_DEMPTY = 34,  // [2] G GEMM done with the r D tile
  H_GDONE = 36,   // [1] the CTA's last G GEMM completed (G may be read)
};



__global__ void ws_half_kernel(const float* __restrict__ src, __half* __restrict__ dst, int64_t n,
                               int* __restrict__ range) {
  const int64_t n2 = n / 2;  // n = rows x 32: even
  bool out = false;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n2;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float2 x = reinterpret_cast<const float2*>(src)[e];
    out |= !(fabsf(x.x) <= 65504.f) || !(fabsf(x.y) <= 65504.f);  // NaN too
    reinterpret_cast<uint32_t*>(dst)[e] = f16x2_sat(x.x, x.y);
  }
  if (out && range) atomicExch(range, 1);
}

// kEG epilogue groups of 8 warps: group g takes the tiles k = g (mod kEG), so
// two tiles' epilogues run concurrently (the TMEM C buffer, r D tile and x_hat
// exchange are already double-buffered by k & 1); gather warps follow them.
template <int kEG>
__global__ void __launch_bounds__((2 + kEG * kEpiWarps + kGW) * 32, 1)
    ws_core16_kernel(const __grid_constant__ WsParams p) {
  static_assert(kEG == 1 || kEG == 2, "one or two epilogue groups (two C buffers)");
  constexpr int kGather16 = 2 + kEG * kEpiWarps;
  using L = Ws16Layout;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::o_bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + L::o_tmem);
  for (int n = 0; n < kN; ++n)
    for (int e = threadIdx.x; e < kW * kW; e += blockDim.x) {
      const int j = e / kW, r = e - j * kW;
      *reinterpret_cast<__half*>(sm + L::o_bt + n * 2048 + swz(r, j * 2, 64)) =
          __float2half_rn(p.b[n][e]);
    }
  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kS; ++s) {
      mbar_init(&bars[H_FULL + s], kGW);
      mbar_init(&bars[H_EMPTY + s], 1);
    }
    for (int i = 0; i < L::kI; ++i) {
      mbar_init(&bars[H_IFULL + i], 1);
      mbar_init(&bars[H_IEMPTY + i], kEpiWarps + kGW);
    }
    for (int b = 0; b < kCB; ++b) {
      mbar_init(&bars[H_CFULL + b], 1);
      mbar_init(&bars[H_CEMPTY + b], kEpiWarps);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars[H_DFULL + b], kEpiWarps);
      mbar_init(&bars[H_DEMPTY + b], 1);
    }
    mbar_init(&bars[H_GDONE], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int n = 0; n < kN; ++n) prefetch_tmap(&p.tmap[n]);
  }
  if (threadIdx.x / 32 == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nk = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  constexpr uint32_t kG = 96 * kCB;  // TMEM: C[b] at 96 b, G after them

  if (warp == 0) {
    if (lane == 0) {
      auto ahead = tile_ahead<4>([&](int64_t kk) { return ws_tile(p, kk); }, p.tile_rows, nk);
      for (int64_t k = 0; k < nk; ++k) {
        const int i = (int)(k % L::kI);
        int64_t tile;
        int32_t rows;
        ahead.pop(k, tile, rows);
        mbar_wait(&bars[H_IEMPTY + i], (uint32_t)(((k / L::kI) & 1) ^ 1));
        int32_t* s_idx = reinterpret_cast<int32_t*>(sm + L::o_idx + i * L::kIdxSlot);
        reinterpret_cast<int32_t*>(sm + L::o_rows)[i] = rows;
        mbar_expect_tx(&bars[H_IFULL + i], L::kIdxSlot);
        for (int n = 0; n < kN; ++n)
          bulk_g2s(s_idx + n * kRows, p.idx[n] + tile * kRows, kRows * 4, &bars[H_IFULL + i]);
        bulk_g2s(s_idx + kN * kRows, p.vals + tile * kRows, kRows * 4, &bars[H_IFULL + i]);
      }
    }
  } else if (warp >= kGather16) {
    const int gw = warp - kGather16;
    constexpr int kGroups = kN * kRows / 4, kPer = kGroups / kGW;
    for (int64_t k = 0; k < nk; ++k) {
      const int s = (int)(k % L::kS), i = (int)(k % L::kI);
      mbar_wait(&bars[H_EMPTY + s], (uint32_t)(((k / L::kS) & 1) ^ 1));
      mbar_wait(&bars[H_IFULL + i], (uint32_t)((k / L::kI) & 1));
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + i * L::kIdxSlot);
      uint8_t* slot = sm + L::o_a + s * L::kSlot;
      if (ws_exp(p) & 2) {  // exp 2: no gathers (timing only)
        if (lane == 0) {
          mbar_arrive(&bars[H_IEMPTY + i]);
          mbar_arrive(&bars[H_FULL + s]);
        }
        continue;
      }
      __syncwarp();
      if (elect_one()) {
        mbar_expect_tx(&bars[H_FULL + s], kPer * 256);
#pragma unroll 1
        for (int g0 = gw * kPer; g0 < (gw + 1) * kPer; g0 += 8) {
          int4 r[8];
#pragma unroll
          for (int g = 0; g < 8; ++g) r[g] = *reinterpret_cast<const int4*>(s_idx + (g0 + g) * 4);
          const int n = g0 / (kRows / 4), gm = g0 - n * (kRows / 4);
#pragma unroll
          for (int g = 0; g < 8; ++g)
            tma_gather4(slot + n * kModeTile16 + (gm + g) * 256, &p.tmap[n], 0, r[g].x, r[g].y,
                        r[g].z, r[g].w, &bars[H_FULL + s]);
        }
        mbar_arrive(&bars[H_IEMPTY + i]);  // indices read before the issues
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    {  // whole warp; one elected lane issues each GEMM (see ws_factor_kernel)
      constexpr uint32_t idc = idesc_f16(128, kW, 0, 0);
      constexpr uint32_t idg = idesc_f16(128, kN * kW, 1, 1);
      const uint32_t bt = smem_u32(sm + L::o_bt), d0 = smem_u32(sm + L::o_d);
      auto issue_g = [&](int64_t k) {
        const int s = (int)(k % L::kS), db = (int)(k & 1);
        mbar_wait(&bars[H_DFULL + db], (uint32_t)((k >> 1) & 1));
        tc_after();
        // G[j'][n R + r] += sum_t A[t][j'] (r D_n)[t][r]: M = 3 stacked modes
        // (+ one garbage block), N = 96, K = 16 nonzeros per instruction
        const uint32_t a0 = smem_u32(sm + L::o_a + s * L::kSlot), dd = d0 + db * L::kSlot;
        if (elect_one()) {
          if (!(ws_exp(p) & 4))  // exp 4: no G GEMM (timing only)
#pragma unroll
            for (int ks = 0; ks < kRows / 16; ++ks)
              mma_f16(tmem + kG, sdesc_l(a0 + ks * 1024, kModeTile16, 512, 4),
                      sdesc_l(dd + ks * 1024, kModeTile16, 512, 4), idg,
                      (k > 0 || ks > 0) ? 1u : 0u);
          mma_commit(&bars[H_DEMPTY + db]);
          mma_commit(&bars[H_EMPTY + s]);
        }
        __syncwarp();
      };
      for (int64_t k = 0; k < nk; ++k) {
        const int s = (int)(k % L::kS), b = (int)(k % kCB);
        mbar_wait(&bars[H_FULL + s], (uint32_t)((k / L::kS) & 1));
        mbar_wait(&bars[H_CEMPTY + b], (uint32_t)(((k / kCB) & 1) ^ 1));
        tc_after();
        const uint32_t a0 = smem_u32(sm + L::o_a + s * L::kSlot);
        if (elect_one()) {
#pragma unroll
          for (int n = 0; n < kN; ++n)
#pragma unroll
            for (int ks = 0; ks < kW / 16; ++ks)
              mma_f16(tmem + b * 96 + n * kW,
                      sdesc_l(a0 + n * kModeTile16 + ks * 32, 16, 512, 4),
                      sdesc_l(bt + n * 2048 + ks * 32, 16, 512, 4), idc, ks > 0);
          mma_commit(&bars[H_CFULL + b]);
        }
        __syncwarp();
        if (k >= 1) issue_g(k - 1);
      }
      if (nk >= 1) issue_g(nk - 1);
      // after every G GEMM: tcgen05.commit tracks all prior MMAs of the thread,
      // and elect.sync picks the same lane every time (the lowest active one)
      if (elect_one()) mma_commit(&bars[H_GDONE]);
      __syncwarp();
    }
  } else {
    const int ew = warp - 2, q = warp & 3, eg = ew / kEpiWarps, h = (ew >> 2) & 1;
    const int row = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    for (int64_t k = eg; k < nk; k += kEG) {
      const int b = (int)(k & 1), cb = (int)(k % kCB), ii = (int)(k % L::kI);
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + ii * L::kIdxSlot);
      const float* s_val = reinterpret_cast<const float*>(s_idx + kN * kRows);
      mbar_wait(&bars[H_IFULL + ii], (uint32_t)((k / L::kI) & 1));
      mbar_wait(&bars[H_CFULL + cb], (uint32_t)((k / kCB) & 1));
      tc_after();
      float c[kN][16];
      {  // the three modes' columns in flight before one wait
        uint32_t v[kN][16];
#pragma unroll
        for (int n = 0; n < kN; ++n) tmem_ld16(tl + cb * 96 + n * kW + h * 16, v[n]);
        tmem_wait_ld();
#pragma unroll
        for (int n = 0; n < kN; ++n)
#pragma unroll
          for (int i = 0; i < 16; ++i) c[n][i] = __uint_as_float(v[n][i]);
      }
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[H_CEMPTY + cb]);  // C(k + kCB) may land
      // column pairs in packed fp32 (FMUL2 / FFMA2): C_1 C_2 (shared by
      // x_hat and D'_0), x_hat as an even / odd pair of partial sums
      f2 c0[8], c1[8], c2[8], p12[8], acc = {0.0f, 0.0f};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        c0[i] = f2{c[0][2 * i], c[0][2 * i + 1]};
        c1[i] = f2{c[1][2 * i], c[1][2 * i + 1]};
        c2[i] = f2{c[2][2 * i], c[2][2 * i + 1]};
        p12[i] = mul2(c1[i], c2[i]);
        acc = fma2(c0[i], p12[i], acc);
      }
      // x_hat halves exchanged with the sibling warp of this lane quarter
      const float part = acc.x + acc.y;
      float* xp = reinterpret_cast<float*>(sm + L::o_xp);
      xp[(b * 2 + h) * kRows + row] = part;
      named_bar(1 + q + 4 * eg, 64);
      const float xhat = part + xp[(b * 2 + (h ^ 1)) * kRows + row];
      const bool ok = row < reinterpret_cast<const int32_t*>(sm + L::o_rows)[ii];
      const float resid = ok ? s_val[row] - xhat : 0.0f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[H_IEMPTY + ii]);
      mbar_wait(&bars[H_DEMPTY + b], (uint32_t)(((k >> 1) & 1) ^ 1));  // G(k - 2) done with D[b]
      uint8_t* dt = sm + L::o_d + b * L::kSlot;
      if (ws_exp(p) & 32) {  // exp 32: no r D tile (timing only)
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[H_DFULL + b]);
        continue;
      }
      // r D'_n: r (C_1 C_2), (r C_0) C_2, (r C_0) C_1 -- four packed products
      // per column pair after x_hat's two
      const f2 rr = {resid, resid};
      f2 rc0[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) rc0[i] = mul2(rr, c0[i]);
#pragma unroll
      for (int n = 0; n < kN; ++n)
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {  // 8 fp16 = one 16-B chunk
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = q2 * 4 + e;
            w[e] = f16x2_sat(n == 0 ? mul2(rr, p12[i])
                                    : (n == 1 ? mul2(rc0[i], c2[i]) : mul2(rc0[i], c1[i])));
          }
          *reinterpret_cast<uint4*>(dt + n * kModeTile16 + swz(row, (h * 16 + q2 * 8) * 2, 64)) =
              make_uint4(w[0], w[1], w[2], w[3]);
        }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[H_DFULL + b]);
    }
    // the last G GEMM: a dedicated barrier -- with two epilogue groups one
    // group can finish while the other's D barrier is still two phases
    // behind, which a parity wait on it would mistake for done
    mbar_wait(&bars[H_GDONE], 0u);
    tc_after();
    if (eg == 0 && q < kN) {
      uint32_t v[16];
      tmem_ld16(tl + kG + q * kW + h * 16, v);
      tmem_wait_ld();
      float* out = p.partials + (size_t)blockIdx.x * (kN * kW * kW) + ((size_t)q * kW + lane) * kW + h * 16;
#pragma unroll
      for (int i = 0; i < 16; ++i) out[i] = nk > 0 ? __uint_as_float(v[i]) : 0.0f;
    }
  }
  ws_teardown(tmem);
}

// ---- write-back ceiling (measurement) ------------------------------------------
//
// The factor sweep's write-back alone, for the roofline that binds at
// L2-resident shapes: same tile stream, thread -> (row, column half) map,
// per-quarter 4 KB staging tiles and 4-row x 128-B RED.v4 groups as epi2 of
// ws_factor_kernel<true> -- no gathers, no MMA, no TMEM -- at full occupancy
// (8 CTAs per SM, so index-load latency is hidden), adding 1.0f to
// every element of each nonzero's three rows of `dst` (a scratch copy of the
// factor shapes).  Its time is the floor the full sweep's RED stream sets.
__global__ void __launch_bounds__(kEpiWarps * 32, 8)
    ws_writeback_kernel(const __grid_constant__ WsParams p, float* const* dst) {
  __shared__ __align__(1024) uint8_t stage_all[4 * 4096];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = (warp + 2) & 3, h = warp >> 2;  // the epilogue warps' map (warp 2 + w)
  const int row = q * 32 + lane;
  uint8_t* stage = stage_all + q * 4096;
  const int64_t nk = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  for (int64_t k = 0; k < nk; ++k) {
    const int64_t tile = ws_tile(p, k);
    const bool ok = row < __ldg(p.tile_rows + tile);
    int32_t g[kN];
#pragma unroll
    for (int n = 0; n < kN; ++n) g[n] = ok ? __ldg(p.idx[n] + tile * kRows + row) : -1;
    int32_t gq[kN][4];
#pragma unroll
    for (int n = 0; n < kN; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        gq[n][i] = __shfl_sync(0xffffffffu, g[n], h * 16 + i * 4 + (lane >> 3));
#pragma unroll
    for (int n = 0; n < kN; ++n) {
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4)
        *reinterpret_cast<float4*>(stage + swz(lane, h * 64 + q4 * 16, 128)) =
            make_float4(1.f, 1.f, 1.f, 1.f);
      named_bar(1 + q, 64);
      float* d = dst[n];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int rl = h * 16 + i * 4 + (lane >> 3), ch = lane & 7;
        const float4 v = *reinterpret_cast<const float4*>(stage + swz(rl, ch * 16, 128));
        if (gq[n][i] >= 0) red_add_v4(d + (size_t)gq[n][i] * kW + ch * 4, v);
      }
      named_bar(1 + q, 64);
    }
  }
}

__global__ void ws_reduce_kernel(const float* __restrict__ partials, int nparts, int len,
                                 float* __restrict__ grad) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < len; e += gridDim.x * blockDim.x) {
    float s = 0.0f;
    for (int k = 0; k < nparts; ++k) s += partials[(size_t)k * len + e];
    grad[e] = s;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn),
                            cudaEnableDefault, &q);
  }
  return fn;
}

// Row-gather tensor map of A_n (I_n x 32 fp32): box of one 128-B row.
bool make_row_map(CUtensorMap* tm, const float* a, int64_t rows, bool atom32) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)kW, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kW * 4};
  cuuint32_t box[2] = {(cuuint32_t)kW, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Row-gather map of an fp16 copy of A_n (rows x 32 fp16): box of one 64-B row.
bool make_row_map16(CUtensorMap* tm, const __half* a, int64_t rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)kW, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kW * 2};
  cuuint32_t box[2] = {(cuuint32_t)kW, 1};
  cuuint32_t es[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(a), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Timing experiments only: FTKCU_WS_EXP bits 1 / 2 / 4 / 8 / 16 drop the
// core slot hold / gathers / G GEMM / row copy / factor write-back
// (scripts/ws_exp.sh).  Read only in an experiments build
// (make EXPERIMENTS=1); the production library ignores the variable.
int ws_exp_bits() {
#ifdef FTKCU_EXPERIMENTS
  static const int bits = [] {
    const char* e = std::getenv("FTKCU_WS_EXP");
    return e ? std::atoi(e) : 0;
  }();
  return bits;
#else
  return 0;
#endif
}

bool make_params(WsParams& p, const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                 bool core) {
  for (int n = 0; n < kN; ++n) {
    if (!make_row_map(&p.tmap[n], v.a[n], dims[n], core)) return false;
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
  p.tmul = mul;
  p.tadd = add;
  return true;
}

}  // namespace

size_t ws_core_scratch_bytes(const KView& v, const int32_t* dims) {
  size_t f = (size_t)num_sms() * kN * kW * kW;  // per-CTA gradients
  size_t h = 0;
  for (int n = 0; n < v.order && n < kN; ++n) h += (size_t)dims[n] * kW;  // fp16 copy of A
  f += (h + 1) / 2;
  return f * sizeof(float);
}

bool ws_supported(const KView& v) {
  return v.order == kN && v.r == kW && v.j[0] == kW && v.j[1] == kW && v.j[2] == kW &&
         encode_fn() != nullptr;
}

cudaError_t launch_ws_factor(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                             float lr, float reg, int precision, int atomic_update,
                             int epi_warps, cudaStream_t st) {
  WsParams p{};
  if (!make_params(p, v, dims, mul, add, false)) return cudaErrorNotSupported;
  p.lr = lr;
  p.reg = reg;
  p.atomic_update = atomic_update;
  p.prec3 = precision == FTKCU_PREC_3XTF32;
  p.exp = ws_exp_bits();
  if (p.ntiles == 0) return cudaSuccess;
  const bool k3 = p.prec3 && atomic_update;
  p.window = (atomic_update && !k3) ? v.window : 0;
  const int bytes = (int)(k3 ? WsLayout<false, true>::bytes : WsLayout<false>::bytes);
  // 16 epilogue warps (ws_factor_kernel<., ., 16>) measured no faster than 8
  // at C2 (8.53 vs 8.48 ms): the sweep is not short of warps to hide latency
  (void)epi_warps;
  auto kern = k3 ? ws_factor3_kernel
                 : (atomic_update ? ws_factor_kernel<true> : ws_factor_kernel<false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  const int grid = (int)sweep_grid(v);
  kern<<<grid, kThreadsWs, bytes, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_ws_factor_ring(const KView& v, const int32_t* dims, const RingDev& ring,
                                  float lr, float reg, cudaStream_t st) {
  WsParams p{};
  if (!make_params(p, v, dims, 1, 0, false)) return cudaErrorNotSupported;
  p.lr = lr;
  p.reg = reg;
  p.atomic_update = 1;
  p.exp = ws_exp_bits();
  p.ring = ring;
  const int bytes = (int)WsLayout<false>::bytes;
  cudaError_t e = cudaFuncSetAttribute(ws_factor_kernel<true, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  // every CTA must be resident at once (cells end in cross-CTA counts)
  int grid = num_sms();
  if (v.max_ctas > 0 && v.max_ctas < grid) grid = v.max_ctas;
  ws_factor_kernel<true, true><<<grid, kThreadsRing, bytes, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_ws_core(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                           float* grad, int precision, int core16, float* scratch,
                           size_t scratch_bytes, cudaStream_t st) {
  WsParams p{};
  if (!make_params(p, v, dims, mul, add, true)) return cudaErrorNotSupported;
  p.prec3 = precision == FTKCU_PREC_3XTF32;
  p.exp = ws_exp_bits();
  const int grid = (int)sweep_grid(v);
  const int len = kN * kW * kW;
  if (grid < 1) return cudaErrorInvalidValue;
  if (scratch_bytes < (size_t)grid * len * sizeof(float)) return cudaErrorInvalidValue;
  p.partials = scratch;
  for (int n = 0; n < kN; ++n) p.cc[n] = v.cc[n];
  cudaError_t e;
  if (!v.cc[0] && !p.prec3 && core16) {
    // fp16 copy of A (after the partials), gathered once per tile
    if (scratch_bytes < ws_core_scratch_bytes(v, dims)) return cudaErrorInvalidValue;
    __half* a16 = reinterpret_cast<__half*>(scratch + (size_t)num_sms() * len);
    for (int n = 0; n < kN; ++n) {
      const int64_t cnt = (int64_t)dims[n] * kW;
      int64_t blocks = (cnt + 255) / 256;
      if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
      ws_half_kernel<<<(int)blocks, 256, 0, st>>>(v.a[n], a16, cnt, v.f16_range);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      if (!make_row_map16(&p.tmap[n], a16, dims[n])) return cudaErrorNotSupported;
      a16 += cnt;
    }
    const int bytes = (int)Ws16Layout::bytes;
    const int groups = core16 >= 2 ? 2 : 1;
    auto kern = groups == 2 ? ws_core16_kernel<2> : ws_core16_kernel<1>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    kern<<<grid, (2 + groups * kEpiWarps + kGW) * 32, bytes, st>>>(p);
  } else {
    const int bytes = (int)WsLayout<true>::bytes;
    auto kern = v.cc[0] ? ws_core_cc_kernel : ws_core_kernel;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreadsWs, bytes, st>>>(p);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ws_reduce_kernel<<<(len + 255) / 256, 256, 0, st>>>(scratch, grid, len, grad);
  return cudaGetLastError();
}

// Write-back ceiling of the N = 3, J = R = 32 factor sweep on this tile
// stream (see ws_writeback_kernel); dst[n] = I_n x 32 fp32 scratch.
cudaError_t launch_ws_writeback(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                                float* const* dst_dev, cudaStream_t st) {
  WsParams p{};
  if (!make_params(p, v, dims, mul, add, false)) return cudaErrorNotSupported;
  if (p.ntiles == 0) return cudaSuccess;
  // full occupancy (8 CTAs of 8 warps per SM): the ceiling is the RED rate
  // of this address stream, not the latency of the probe's own index loads
  ws_writeback_kernel<<<(int)sweep_grid(v, 8), kEpiWarps * 32, 0, st>>>(p, dst_dev);
  return cudaGetLastError();
}

}  // namespace ftkcu
