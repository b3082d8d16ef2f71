// tcgen05 Hogwild sweeps for the large ranks of the rank sweep (BASELINE C5:
// N = 3, J = R = W in {64, 128}).  At these ranks one tile's factor rows no
// longer fit next to B in shared memory (W = 128: A rows 3 x 64 KB, B and B^T
// 6 x 64 KB), so the sweeps run MODE-SERIAL over a ring of stages, each stage
// = one mode's gathered rows (128 x W) + one pre-swizzled B operand image
// (W x W), with the per-tile accumulators in TMEM:
//
//   factor   C_n = A_n B_n        n = 0..2 -> TMEM [nW, (n+1)W)  (3 stages)
//            epilogue: x_hat, r, D'_n = lr r prod_{m!=n} C_m, in place
//            U_n = D'_n B_n^T     n = 0..2 -> TMEM [3W, 4W)     (3 stages of
//            B images only); a += U - lr reg a, a re-read through L2, as
//            vector RED (Hogwild accumulate) or STG (overwrite rule)
//   core     one launch per mode p (TMEM holds C for all modes plus G_p):
//            C_n as above, D'_p = r prod_{m!=p} C_m into shared memory,
//            G_p += A_p^T D'_p    (A_p gathered again in the MN-major layout)
//
// Warp roles: warp 0 producer (COO record by bulk copy, rows by TMA gather4,
// B images by bulk copy), warp 1 MMA issuer, warps 2-5 epilogue (thread =
// nonzero = TMEM lane).  Algebra as tc_ws_kernels.cu (decomposition.cpp:
// 644-658 / :678-698); B operands and D' are rounded to nearest tf32.
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "engine.cuh"
#include "tc_common.cuh"

namespace ftkcu {
namespace {
using namespace tc;

constexpr int kN = 3;
constexpr int kRows = 128;
constexpr int kThreads = 6 * 32;   // core: producer, MMA, 4 epilogue warps
// factor: producer, MMA, 8 epilogue warps (column halves), second producer
// (warp 10) issuing half of every tile's row gathers
constexpr int kThreadsF = 11 * 32;
constexpr uint32_t kBlk = kRows * 128;  // one 32-column block of a row tile: 16 KB

template <int W, bool kCore>
struct BigLayout {
  static constexpr uint32_t kA = kRows * W * 4;  // row tile: W / 32 blocks of 16 KB
  static constexpr uint32_t kB = W * W * 4;      // B image: W / 32 blocks of W x 128 B
  static constexpr uint32_t kStage = kA + kB;
  static constexpr int kStages = W == 64 ? 3 : 1;
  static constexpr uint32_t o_st = 0;
  // core: D' tile (MN-major).  factor at W = 64: I (a second C GEMM per
  // mode copies the gathered rows into TMEM) and -lr reg I (the regulariser
  // as a second U GEMM operand, A from that TMEM copy), so a stage is free as
  // soon as its C GEMM has run
  static constexpr bool kACopy = !kCore && W == 64;
  static constexpr uint32_t o_d = o_st + kStages * kStage;
  static constexpr uint32_t d_bytes = kCore ? kA : (kACopy ? 2 * kB : 0);
  // the G GEMM reads M = 128 rows = 4 blocks of the A part: past a W = 64
  // tile it runs into the stage's B image / the next stage / the D' tile
  static constexpr uint32_t o_idx = o_d + d_bytes;
  static constexpr uint32_t kIdx = (kN + 1) * kRows * 4;
  static constexpr int kI = 4;  // COO-record ring depth
  static constexpr uint32_t o_rows = o_idx + kI * kIdx;
  static constexpr uint32_t o_xp = o_rows + 16;  // factor: x_hat halves [2][128]
  // factor: per epilogue warp a 2 KB staging tile for the 64-B write-back
  static constexpr uint32_t o_stage = o_xp + 2 * kRows * 4;
  static constexpr uint32_t o_bar = o_stage + (kCore ? 0 : 8 * 2048);
  static constexpr uint32_t o_tmem = o_bar + 32 * 8;
  static constexpr uint32_t bytes = o_tmem + 16;
  // TMEM: factor C/D [0, 3W) + U regions (one per mode at W = 64, so U_0..2
  // issue back to back; one shared at W = 128); core: C buffers (two at
  // W = 64, so C(k+1) overlaps the epilogue of k) + G_pass.
  // W = 64: two U regions (TMEM 3 x 2W + 2W = 512), so U(n + 1) runs while
  // the epilogue writes U(n) back
  static constexpr int kUN = kACopy ? 2 : 1;
  static constexpr int kCB = W == 64 ? 2 : 1;
  static constexpr uint32_t kMS = kACopy ? 2 * W : W;  // factor TMEM per mode: C [| A copy]
  static constexpr uint32_t t_u = 3 * kMS;
  static constexpr uint32_t t_g = kCB * 3 * W;
  static constexpr uint32_t tcols = 512;
  static_assert(bytes <= 227 * 1024, "shared-memory budget");
  static_assert((kCore ? t_g + W : t_u + kUN * W) <= tcols, "TMEM budget");
};

enum : int {
  B_FULL = 0,    // [4] stage loaded
  B_EMPTY = 4,   // [4] stage free (released by the MMA that read it)
  B_IFULL = 8,   // [4] COO record landed
  B_IEMPTY = 12, // [4] COO record consumed
  B_CFULL = 16,  // [2] C for all modes in TMEM buffer b
  B_DFULL = 18,  // D' ready (TMEM in place: factor; smem: core)
  B_UFULL = 19,  // [3] factor: U_n in TMEM
  B_UEMPTY = 22, // factor, one U region: U read
  B_DEMPTY = 23, // core: G GEMM done with the D' tile
  B_CEMPTY = 24, // [2] core: C buffer b read by the epilogue
  B_UEMPTY2 = 26, // factor, second U region
};

struct BigParams {
  CUtensorMap tmap[kN];  // K-major rows (SW128); core: [pass] MN-major (ATOM_32B) in tmap_mn
  CUtensorMap tmap_mn;
  const int32_t* idx[kN];
  const float* vals;
  float* a[kN];
  const float* bt_img[kN];  // C GEMM operand images (rows r, K = j)
  const float* b_img[kN];   // U GEMM operand images (rows j, K = r)
  const int32_t* tile_rows;
  const int64_t* tperm;
  int64_t ntiles, tmul, tadd, tile_base;
  float lr, reg;
  int atomic_update, pass;
  float* partials;
};

__device__ __forceinline__ int64_t big_tile(const BigParams& p, int64_t k) {
  const int64_t t = (int64_t)blockIdx.x + k * gridDim.x;
  const int64_t mul = p.tperm ? __ldg(p.tperm) : p.tmul;
  const int64_t add = p.tperm ? __ldg(p.tperm + 1) : p.tadd;
  return p.tile_base + (t * mul + add) % p.ntiles;
}

__device__ __forceinline__ uint32_t rn_bits(float x) { return __float_as_uint(x) + 0x1000u; }

// Producer (one elected lane of a converged warp, so every TMA operand is
// warp-uniform): gathers the W / 32 column blocks of a mode's 128 rows, eight
// index loads in flight ahead of their issues.
template <int W>
__device__ __forceinline__ void gather_rows(uint8_t* dst, const CUtensorMap* tm,
                                            const int32_t* s_idx, uint64_t* bar, int part = 0,
                                            int nparts = 1) {
  const int per = kRows / 4 / nparts;  // 4-row groups of this producer
#pragma unroll 1
  for (int g0 = part * per; g0 < (part + 1) * per; g0 += 8) {
    int4 r[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) r[g] = *reinterpret_cast<const int4*>(s_idx + (g0 + g) * 4);
#pragma unroll
    for (int g = 0; g < 8; ++g)
#pragma unroll
      for (int cb = 0; cb < W / 32; ++cb)
        tma_gather4(dst + cb * kBlk + (g0 + g) * 512, tm, cb * 32, r[g].x, r[g].y, r[g].z,
                    r[g].w, bar);
  }
}

template <int W, bool kCore, int kP = 1>
__device__ void big_setup(uint8_t* sm, uint64_t* bars, uint32_t* tslot, const BigParams& p) {
  using L = BigLayout<W, kCore>;
  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&bars[B_FULL + s], kP);
      mbar_init(&bars[B_EMPTY + s], 1);
    }
    for (int i = 0; i < L::kI; ++i) {
      mbar_init(&bars[B_IFULL + i], 1);
      mbar_init(&bars[B_IEMPTY + i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars[B_CFULL + b], 1);
      mbar_init(&bars[B_CEMPTY + b], 1);
    }
    for (int n = 0; n < kN; ++n) mbar_init(&bars[B_UFULL + n], 1);
    mbar_init(&bars[B_DFULL], 1);
    mbar_init(&bars[B_UEMPTY], 8);  // one arrival per epilogue warp
    mbar_init(&bars[B_UEMPTY2], 8);
    mbar_init(&bars[B_DEMPTY], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int n = 0; n < kN; ++n) prefetch_tmap(&p.tmap[n]);
    if (kCore) prefetch_tmap(&p.tmap_mn);
  }
  if (threadIdx.x / 32 == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(L::tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
}

template <int W, bool kCore>
__device__ void big_teardown(uint32_t tmem) {
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x / 32 == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(BigLayout<W, kCore>::tcols));
}

// Warp 0 (all lanes wait, one elected lane issues): per tile the COO
// record, then one stage per job.  Job order = the MMA warp's: factor
// C(0) [U(k) C(k+1)]...; core C(0) [C(k+1) G(k)]...
// kP producers walk the same job sequence: part 0 also fetches the COO
// records and issues the bulk copies, every part gathers 1 / kP of the rows
// and arrives once per job (FULL barriers count kP arrivals).
template <int W, bool kCore, int kP = 1>
__device__ void big_producer(const BigParams& p, uint8_t* sm, uint64_t* bars, int64_t nk,
                             int part = 0) {
  using L = BigLayout<W, kCore>;
  int64_t job = 0;
  constexpr uint32_t kHalfA = L::kA / kP;
  // COO records are requested kAhead tiles before their rows are gathered
  // (the stream comes from HBM: ~1 us per request)
  constexpr int kAhead = 2;
  auto request = [&](int64_t k) {  // tile k's COO record -> ring slot
    if (k >= nk || part != 0) return;
    const int i = (int)(k % L::kI);
    const int64_t tile = big_tile(p, k);
    mbar_wait(&bars[B_IEMPTY + i], (uint32_t)(((k / L::kI) & 1) ^ 1));
    int32_t* s_idx = reinterpret_cast<int32_t*>(sm + L::o_idx + i * L::kIdx);
    if (elect_one()) {
      reinterpret_cast<int32_t*>(sm + L::o_rows)[i] = __ldg(p.tile_rows + tile);
      mbar_expect_tx(&bars[B_IFULL + i], L::kIdx);
      for (int n = 0; n < kN; ++n)
        bulk_g2s(s_idx + n * kRows, p.idx[n] + tile * kRows, kRows * 4, &bars[B_IFULL + i]);
      bulk_g2s(s_idx + kN * kRows, p.vals + tile * kRows, kRows * 4, &bars[B_IFULL + i]);
    }
    __syncwarp();
  };
  auto record = [&](int64_t k) {  // request k + kAhead, wait for k
    request(k + kAhead);
    mbar_wait(&bars[B_IFULL + (int)(k % L::kI)], (uint32_t)((k / L::kI) & 1));
  };
  auto stage = [&]() {
    const int s = (int)(job % L::kStages);
    mbar_wait(&bars[B_EMPTY + s], (uint32_t)(((job / L::kStages) & 1) ^ 1));
    ++job;
    return s;
  };
  auto idx_of = [&](int64_t k) {
    return reinterpret_cast<const int32_t*>(sm + L::o_idx + (k % L::kI) * L::kIdx);
  };
  auto c_jobs = [&](int64_t k) {  // rows of every mode + the C GEMM's B images
    for (int n = 0; n < kN; ++n) {
      const int s = stage();
      uint8_t* st = sm + L::o_st + s * L::kStage;
      if (elect_one()) {
        mbar_expect_tx(&bars[B_FULL + s], kHalfA + (part == 0 ? L::kB : 0));
        gather_rows<W>(st, &p.tmap[n], idx_of(k) + n * kRows, &bars[B_FULL + s], part, kP);
        if (part == 0) bulk_g2s(st + L::kA, p.bt_img[n], L::kB, &bars[B_FULL + s]);
      }
      __syncwarp();
    }
  };
  if (nk == 0) return;
  for (int64_t k = 0; k < kAhead; ++k) request(k);
  record(0);
  c_jobs(0);
  for (int64_t k = 0; k < nk; ++k) {
    if constexpr (kCore) {  // C(k + 1) ahead of G(k), the MMA warp's order
      if (k + 1 < nk) {
        record(k + 1);
        c_jobs(k + 1);
      }
      const int s = stage();  // G operand: A_pass rows, MN-major
      if (elect_one()) {
        mbar_expect_tx(&bars[B_FULL + s], L::kA);
        gather_rows<W>(sm + L::o_st + s * L::kStage, &p.tmap_mn, idx_of(k) + p.pass * kRows,
                       &bars[B_FULL + s]);
      }
      __syncwarp();
    } else {
      for (int n = 0; n < kN; ++n) {  // U jobs: the B images only
        const int s = stage();
        if (elect_one()) {
          if (part == 0) {
            mbar_expect_tx(&bars[B_FULL + s], L::kB);
            bulk_g2s(sm + L::o_st + s * L::kStage + L::kA, p.b_img[n], L::kB, &bars[B_FULL + s]);
          } else {
            mbar_arrive(&bars[B_FULL + s]);
          }
        }
        __syncwarp();
      }
      if (k + 1 < nk) {
        record(k + 1);
        c_jobs(k + 1);
      }
    }
  }
}

// C_n = A_n B_n for the three modes of one tile (stages job..job+2).
template <int W, bool kCore>
__device__ __forceinline__ void issue_c(uint8_t* sm, uint64_t* bars, uint32_t tmem, int64_t& job,
                                        int cb, bool release = true, int* cs = nullptr) {
  using L = BigLayout<W, kCore>;
  constexpr uint32_t id = idesc_tf32(128, W, 0, 0);
  for (int n = 0; n < kN; ++n, ++job) {
    const int s = (int)(job % L::kStages);
    if (cs) cs[n] = s;
    mbar_wait(&bars[B_FULL + s], (uint32_t)((job / L::kStages) & 1));
    tc_after();
    const uint32_t a0 = smem_u32(sm + L::o_st + s * L::kStage);
    const uint32_t b0 = a0 + L::kA;
#pragma unroll
    for (int ks = 0; ks < W / 8; ++ks) {
      const uint64_t da = sdesc(a0 + (ks / 4) * kBlk + (ks % 4) * 32, 16, 1024, 128);
      mma_ss(tmem + n * L::kMS, da,
             sdesc(b0 + (ks / 4) * (W * 128) + (ks % 4) * 32, 16, 1024, 128), id, ks > 0);
      if constexpr (L::kACopy)  // A_n I: the rows into TMEM for the regulariser GEMM
        mma_ss(tmem + n * L::kMS + W, da,
               sdesc(smem_u32(sm + L::o_d) + (ks / 4) * (W * 128) + (ks % 4) * 32, 16, 1024, 128),
               id, ks > 0);
    }
    if (release) mma_commit(&bars[B_EMPTY + s]);
  }
  mma_commit(&bars[B_CFULL + cb]);
}

// Epilogue: x_hat = sum_r prod_n C_n and the residual of this thread's row.
template <int W>
__device__ __forceinline__ float big_xhat(uint32_t tl) {
  float x = 0.0f;
#pragma unroll 1
  for (int c = 0; c < W / 16; ++c) {
    uint32_t v0[16], v1[16], v2[16];
    tmem_ld16(tl + 0 * W + c * 16, v0);
    tmem_ld16(tl + 1 * W + c * 16, v1);
    tmem_ld16(tl + 2 * W + c * 16, v2);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; ++i)
      x = fmaf(__uint_as_float(v0[i]), __uint_as_float(v1[i]) * __uint_as_float(v2[i]), x);
  }
  return x;
}

// W = 64 (L::kACopy): U_n' = D'_n B_n^T + A_n (-lr reg I) with A_n from its
// TMEM copy is the whole Hogwild step, so the epilogue only issues REDs;
// W = 128 (and the overwrite rule) re-reads the row through L2 for the
// regulariser.
template <int W>
__global__ void __launch_bounds__(kThreadsF, 1) big_factor_kernel(const __grid_constant__ BigParams p) {
  using L = BigLayout<W, false>;
  constexpr bool kFold = L::kACopy;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::o_bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + L::o_tmem);
  if constexpr (L::kACopy) {  // I, then -lr reg I (rows j, K = j', K-major SW128 blocks)
    const float dv = __uint_as_float(rn_bits(-p.lr * p.reg));
    for (int e = threadIdx.x; e < W * W; e += blockDim.x) {
      const int j = e / W, jj = e - j * W;
      const uint32_t off = (jj / 32) * (W * 128) + swz(j, (jj % 32) * 4, 128);
      *reinterpret_cast<float*>(sm + L::o_d + off) = j == jj ? 1.0f : 0.0f;
      *reinterpret_cast<float*>(sm + L::o_d + L::kB + off) = j == jj ? dv : 0.0f;
    }
    fence_proxy_async();
  }
  big_setup<W, false, 2>(sm, bars, tslot, p);
  const uint32_t tmem = *tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nk = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (warp == 0 || warp == 10) {
    big_producer<W, false, 2>(p, sm, bars, nk, warp == 0 ? 0 : 1);
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id = idesc_tf32(128, W, 0, 0);
      int64_t job = 0;
      const uint32_t dg = smem_u32(sm + L::o_d) + L::kB;
      for (int64_t k = 0; k < nk; ++k) {
        // C(k) overwrites D'(k - 1), the A operand of tile k - 1's U GEMMs:
        // issue it only once the last of them has completed (its commit
        // covers all earlier MMAs of this thread).  PTX orders MMAs only per
        // accumulator, so issue order alone would not protect D'(k - 1).
        if (k >= 1) {
          const int64_t u = k * kN - 1;
          mbar_wait(&bars[B_UFULL + (int)(u % L::kUN)], (uint32_t)((u / L::kUN) & 1));
          tc_after();
        }
        issue_c<W, false>(sm, bars, tmem, job, 0);
        mbar_wait(&bars[B_DFULL], (uint32_t)(k & 1));
        for (int n = 0; n < kN; ++n, ++job) {
          const int s = (int)(job % L::kStages);
          const int64_t u = k * kN + n;
          const int uq = (int)(u % L::kUN);  // U region of this job
          mbar_wait(&bars[B_FULL + s], (uint32_t)((job / L::kStages) & 1));
          mbar_wait(&bars[uq ? B_UEMPTY2 : B_UEMPTY], (uint32_t)(((u / L::kUN) & 1) ^ 1));
          tc_after();
          const uint32_t b0 = smem_u32(sm + L::o_st + s * L::kStage) + L::kA;
          const uint32_t tu = tmem + L::t_u + uq * W;
#pragma unroll
          for (int ks = 0; ks < W / 8; ++ks)
            mma_ts(tu, tmem + n * L::kMS + ks * 8,
                   sdesc(b0 + (ks / 4) * (W * 128) + (ks % 4) * 32, 16, 1024, 128), id, ks > 0);
          if constexpr (kFold)  // + A_n (-lr reg I), A_n from its TMEM copy
#pragma unroll
            for (int ks = 0; ks < W / 8; ++ks)
              mma_ts(tu, tmem + n * L::kMS + W + ks * 8,
                     sdesc(dg + (ks / 4) * (W * 128) + (ks % 4) * 32, 16, 1024, 128), id, 1);
          mma_commit(&bars[B_EMPTY + s]);
          mma_commit(&bars[B_UFULL + uq]);
        }
      }
    }
  } else {
    // two warps per TMEM lane quarter, each owning half of the W columns
    const int q = warp & 3, h = (warp - 2) >> 2, row = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const float lr_reg = p.lr * p.reg;
    constexpr int kHalf = W / 2;
    float* xp = reinterpret_cast<float*>(sm + L::o_xp);  // x_hat halves [2][128]
    for (int64_t k = 0; k < nk; ++k) {
      const int i = (int)(k % L::kI);
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + L::o_idx + i * L::kIdx);
      mbar_wait(&bars[B_IFULL + i], (uint32_t)((k / L::kI) & 1));
      mbar_wait(&bars[B_CFULL], (uint32_t)(k & 1));
      tc_after();
      float part = 0.0f;
#pragma unroll 1
      for (int c = h * kHalf / 16; c < (h + 1) * kHalf / 16; ++c) {
        uint32_t v0[16], v1[16], v2[16];
        tmem_ld16(tl + 0 * L::kMS + c * 16, v0);
        tmem_ld16(tl + 1 * L::kMS + c * 16, v1);
        tmem_ld16(tl + 2 * L::kMS + c * 16, v2);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e)
          part = fmaf(__uint_as_float(v0[e]), __uint_as_float(v1[e]) * __uint_as_float(v2[e]), part);
      }
      xp[h * kRows + row] = part;
      named_bar(2 + q, 64);
      const float xhat = part + xp[(h ^ 1) * kRows + row];
      named_bar(2 + q, 64);  // both halves read before the next tile's writes
      const bool ok = row < reinterpret_cast<const int32_t*>(sm + L::o_rows)[i];
      const float resid = ok ? reinterpret_cast<const float*>(s_idx + kN * kRows)[row] - xhat : 0.0f;
      const float sc = p.lr * resid;
      // D'_n = lr r prod_{m != n} C_m, in place over this warp's half of C
      // (A operand of U_n)
#pragma unroll 1
      for (int c = h * kHalf / 16; c < (h + 1) * kHalf / 16; ++c) {
        uint32_t v0[16], v1[16], v2[16];
        tmem_ld16(tl + 0 * L::kMS + c * 16, v0);
        tmem_ld16(tl + 1 * L::kMS + c * 16, v1);
        tmem_ld16(tl + 2 * L::kMS + c * 16, v2);
        tmem_wait_ld();
        uint32_t d0[16], d1[16], d2[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float c0 = __uint_as_float(v0[e]) * sc, c1 = __uint_as_float(v1[e]),
                      c2 = __uint_as_float(v2[e]);
          d0[e] = rn_bits(c1 * sc * c2);
          d1[e] = rn_bits(c0 * c2);
          d2[e] = rn_bits(c0 * c1);
        }
        tmem_st16(tl + 0 * L::kMS + c * 16, d0);
        tmem_st16(tl + 1 * L::kMS + c * 16, d1);
        tmem_st16(tl + 2 * L::kMS + c * 16, d2);
      }
      int32_t g[kN];  // read before the barrier: the COO record is then free
#pragma unroll
      for (int n = 0; n < kN; ++n) g[n] = s_idx[n * kRows + row];
      tmem_wait_st();
      tc_before();
      named_bar(1, 256);
      if (warp == 2 && lane == 0) {
        mbar_arrive(&bars[B_DFULL]);
        mbar_arrive(&bars[B_IEMPTY + i]);
      }
      for (int n = 0; n < kN; ++n) {
        const int64_t u = k * kN + n;
        const int uq = (int)(u % L::kUN);
        float* dst = p.a[n] + (size_t)g[n] * W + h * kHalf;
        // the live half-row (through L2) for the regulariser term, loaded
        // ahead of the U wait so its latency overlaps the U GEMM
        float4 a4[kHalf / 4];
#pragma unroll
        for (int qq = 0; qq < kHalf / 4; ++qq)
          a4[qq] = (ok && (!kFold || !p.atomic_update))
                       ? __ldcg(reinterpret_cast<const float4*>(dst + qq * 4))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
        int32_t gr[4];  // row indices of the 8-row RED groups, shuffled before the wait
#pragma unroll
        for (int i = 0; i < 4; ++i) gr[i] = __shfl_sync(0xffffffffu, ok ? g[n] : -1, i * 8 + (lane >> 2));
        mbar_wait(&bars[B_UFULL + uq], (uint32_t)((u / L::kUN) & 1));
        tc_after();
        // U into registers, then the region is free for U(n + 2)
        uint32_t v[kHalf];
#pragma unroll
        for (int c = 0; c < kHalf / 16; ++c)
          tmem_ld16(tl + L::t_u + uq * W + h * kHalf + c * 16,
                    *reinterpret_cast<uint32_t(*)[16]>(v + c * 16));
        tmem_wait_ld();
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[uq ? B_UEMPTY2 : B_UEMPTY]);
        // write-back through a private 2 KB staging tile per warp: 16 columns
        // of its 32 rows at a time, sent as 64-B row segments (8 rows per RED)
        uint8_t* stage = sm + L::o_stage + (warp - 2) * 2048;
        float* dsw = p.a[n] + h * kHalf + (lane & 3) * 4;
#pragma unroll
        for (int c = 0; c < kHalf / 16; ++c) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const float4 a = a4[c * 4 + q4];
            float4 st;  // kFold: U' already holds the regulariser
            const float rg = kFold ? 0.0f : lr_reg;
            st.x = __uint_as_float(v[c * 16 + q4 * 4 + 0]) - rg * a.x;
            st.y = __uint_as_float(v[c * 16 + q4 * 4 + 1]) - rg * a.y;
            st.z = __uint_as_float(v[c * 16 + q4 * 4 + 2]) - rg * a.z;
            st.w = __uint_as_float(v[c * 16 + q4 * 4 + 3]) - rg * a.w;
            if (!p.atomic_update) {
              st.x += a.x;
              st.y += a.y;
              st.z += a.z;
              st.w += a.w;
            }
            *reinterpret_cast<float4*>(stage + swz(lane, q4 * 16, 64)) = st;
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 sv =
                *reinterpret_cast<const float4*>(stage + swz(i * 8 + (lane >> 2), (lane & 3) * 16, 64));
            if (gr[i] >= 0) {
              float* gp = dsw + (size_t)gr[i] * W + c * 16;
              if (p.atomic_update)
                red_add_v4(gp, sv);
              else
                *reinterpret_cast<float4*>(gp) = sv;
            }
          }
          __syncwarp();
        }
      }
    }
  }
  big_teardown<W, false>(tmem);
}

// ---- J = R = 128 factor sweep: K-split half jobs -------------------------------
//
// A whole-mode job (128 rows + a 64 KB B image) leaves room for one stage, so
// every TMA, MMA and epilogue step would serialise.  Here each GEMM is split
// along K into two half jobs of 64 KB (32 KB of rows or D' columns + 32 KB of
// the B image), three in flight.  A U half job also re-gathers the live rows
// of its column half, so the regulariser / overwrite term is read from shared
// memory instead of through L2 in the epilogue; its stage is released by the
// epilogue warps that read it, not by the MMA.

namespace f128 {
constexpr int W = 128;
constexpr uint32_t kHalfX = kRows * 64 * 4;  // rows of a 64-column half: 32 KB
constexpr uint32_t kHalfY = W * 64 * 4;      // B image half: 32 KB
constexpr uint32_t kStage = kHalfX + kHalfY;
constexpr int kS = 3, kI = 4;
constexpr uint32_t o_st = 0;
constexpr uint32_t kIdx = (kN + 1) * kRows * 4;
constexpr uint32_t o_idx = o_st + kS * kStage;
constexpr uint32_t o_rows = o_idx + kI * kIdx;
constexpr uint32_t o_xp = o_rows + 16;
constexpr uint32_t o_stage = o_xp + 2 * kRows * 4;  // per epilogue warp: 32 rows x 64 B
constexpr uint32_t o_bar = o_stage + 8 * 2048;
constexpr uint32_t o_tmem = o_bar + 24 * 8;
constexpr uint32_t bytes = o_tmem + 16;
static_assert(bytes <= 227 * 1024, "shared-memory budget");
constexpr int kJobs = 4 * kN;  // per tile: C and U, two halves per mode
// UFULL[n]: U_n in TMEM; U0READ: the epilogue has read U_0 (its region
// takes the next U_0); UREAD: it has read U_1 and U_2 (their regions, C
// regions 0 and 1, take the next tile's C)
enum : int { FULL = 0, EMPTY = 3, IFULL = 6, IEMPTY = 10, CFULL = 14, DFULL = 15, UFULL = 16, U0READ = 19, UREAD = 20 };
constexpr uint32_t t_u = kN * W;
// U_0 goes to the spare region, U_n (n > 0) over C region n - 1, whose D'
// U_{n-1} has consumed (the MMA thread waits for U_{n-1} to complete before
// it issues U_n)
__device__ __forceinline__ uint32_t u_col(int n) { return n == 0 ? t_u : (uint32_t)(n - 1) * W; }
// job index of the first job of tile k's U phase (C(0) comes first)
__device__ __forceinline__ int64_t u_job(int64_t k) { return 2 * kN + k * kJobs; }
}  // namespace f128

__global__ void __launch_bounds__(kThreadsF, 1) big128_factor_kernel(const __grid_constant__ BigParams p) {
  using namespace f128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + o_bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + o_tmem);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kS; ++s) {
      mbar_init(&bars[FULL + s], 2);
      // C half jobs: released by the MMA commit (1 arrival); U half jobs: by
      // the 4 epilogue warps that read the rows -- both count as 4
      mbar_init(&bars[EMPTY + s], 4);
    }
    for (int i = 0; i < kI; ++i) {
      mbar_init(&bars[IFULL + i], 1);
      mbar_init(&bars[IEMPTY + i], 1);
    }
    mbar_init(&bars[CFULL], 1);
    mbar_init(&bars[DFULL], 1);
    for (int n = 0; n < kN; ++n) mbar_init(&bars[UFULL + n], 1);
    mbar_init(&bars[U0READ], 8);  // one arrival per epilogue warp
    mbar_init(&bars[UREAD], 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int n = 0; n < kN; ++n) prefetch_tmap(&p.tmap[n]);
  }
  if (threadIdx.x / 32 == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nk = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto idx_of = [&](int64_t k) {
    return reinterpret_cast<const int32_t*>(sm + o_idx + (k % kI) * kIdx);
  };

  if (warp == 0 || warp == 10) {
    // two producers walk the same job sequence, each gathering half the rows;
    // part 0 also fetches the COO records and the B image halves
    const int part = warp == 0 ? 0 : 1;
    int64_t job = 0;
    constexpr int kAhead = 2;
    auto request = [&](int64_t k) {
      if (k >= nk || part != 0) return;
      const int i = (int)(k % kI);
      const int64_t tile = big_tile(p, k);
      mbar_wait(&bars[IEMPTY + i], (uint32_t)(((k / kI) & 1) ^ 1));
      int32_t* s_idx = reinterpret_cast<int32_t*>(sm + o_idx + i * kIdx);
      if (elect_one()) {
        reinterpret_cast<int32_t*>(sm + o_rows)[i] = __ldg(p.tile_rows + tile);
        mbar_expect_tx(&bars[IFULL + i], kIdx);
        for (int n = 0; n < kN; ++n)
          bulk_g2s(s_idx + n * kRows, p.idx[n] + tile * kRows, kRows * 4, &bars[IFULL + i]);
        bulk_g2s(s_idx + kN * kRows, p.vals + tile * kRows, kRows * 4, &bars[IFULL + i]);
      }
      __syncwarp();
    };
    // one half job: rows n, columns [64 hh, 64 hh + 64) + half hh of image img
    auto half_job = [&](int64_t k, int n, int hh, const float* img) {
      const int s = (int)(job % kS);
      mbar_wait(&bars[EMPTY + s], (uint32_t)(((job / kS) & 1) ^ 1));
      ++job;
      uint8_t* st = sm + o_st + s * kStage;
      if (elect_one()) {
        mbar_expect_tx(&bars[FULL + s], kHalfX / 2 + (part == 0 ? kHalfY : 0));
        const int32_t* s_idx = idx_of(k) + n * kRows;
        constexpr int per = kRows / 4 / 2;
#pragma unroll 1
        for (int g0 = part * per; g0 < (part + 1) * per; g0 += 8) {
          int4 r[8];
#pragma unroll
          for (int g = 0; g < 8; ++g) r[g] = *reinterpret_cast<const int4*>(s_idx + (g0 + g) * 4);
#pragma unroll
          for (int g = 0; g < 8; ++g)
#pragma unroll
            for (int cb = 0; cb < 2; ++cb)
              tma_gather4(st + cb * kBlk + (g0 + g) * 512, &p.tmap[n], (hh * 2 + cb) * 32, r[g].x,
                          r[g].y, r[g].z, r[g].w, &bars[FULL + s]);
        }
        if (part == 0) bulk_g2s(st + kHalfX, img + hh * (kHalfY / 4), kHalfY, &bars[FULL + s]);
      }
      __syncwarp();
    };
    if (nk > 0) {
      for (int64_t k = 0; k < kAhead; ++k) request(k);
      auto c_jobs = [&](int64_t k) {
        request(k + kAhead);
        mbar_wait(&bars[IFULL + (int)(k % kI)], (uint32_t)((k / kI) & 1));
        for (int n = 0; n < kN; ++n)
          for (int hh = 0; hh < 2; ++hh) half_job(k, n, hh, p.bt_img[n]);
      };
      c_jobs(0);
      for (int64_t k = 0; k < nk; ++k) {
        for (int n = 0; n < kN; ++n)
          for (int hh = 0; hh < 2; ++hh) half_job(k, n, hh, p.b_img[n]);
        if (k + 1 < nk) c_jobs(k + 1);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id = idesc_tf32(128, W, 0, 0);
      int64_t job = 0;
      auto wait_full = [&]() {
        const int s = (int)(job % kS);
        mbar_wait(&bars[FULL + s], (uint32_t)((job / kS) & 1));
        tc_after();
        ++job;
        return s;
      };
      auto issue_c = [&]() {
        for (int n = 0; n < kN; ++n)
          for (int hh = 0; hh < 2; ++hh) {
            const int s = wait_full();
            const uint32_t a0 = smem_u32(sm + o_st + s * kStage), b0 = a0 + kHalfX;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
              mma_ss(tmem + n * W, sdesc(a0 + (ks / 4) * kBlk + (ks % 4) * 32, 16, 1024, 128),
                     sdesc(b0 + (ks / 4) * (W * 128) + (ks % 4) * 32, 16, 1024, 128), id,
                     (hh > 0 || ks > 0) ? 1u : 0u);
#pragma unroll
            for (int a4 = 0; a4 < 4; ++a4) mma_commit(&bars[EMPTY + s]);
          }
        mma_commit(&bars[CFULL]);
      };
      if (nk > 0) issue_c();
      for (int64_t k = 0; k < nk; ++k) {
        mbar_wait(&bars[DFULL], (uint32_t)(k & 1));
        for (int n = 0; n < kN; ++n) {
          if (n == 0) mbar_wait(&bars[U0READ], (uint32_t)((k & 1) ^ 1));
          // U_n (n > 0) accumulates over C region n - 1, whose D'_{n-1} is
          // U_{n-1}'s A operand: wait for U_{n-1} to complete first (PTX
          // orders MMAs only per accumulator)
          if (n > 0) {
            mbar_wait(&bars[UFULL + n - 1], (uint32_t)(k & 1));
            tc_after();
          }
          for (int hh = 0; hh < 2; ++hh) {
            const int s = wait_full();
            const uint32_t b0 = smem_u32(sm + o_st + s * kStage) + kHalfX;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
              mma_ts(tmem + u_col(n), tmem + n * W + (hh * 8 + ks) * 8,
                     sdesc(b0 + (ks / 4) * (W * 128) + (ks % 4) * 32, 16, 1024, 128), id,
                     (hh > 0 || ks > 0) ? 1u : 0u);
            // the stage is released by the epilogue (it reads the rows)
          }
          mma_commit(&bars[UFULL + n]);
        }
        if (k + 1 < nk) {  // C(k + 1) overwrites U_1(k), U_2(k): after the epilogue read them
          mbar_wait(&bars[UREAD], (uint32_t)(k & 1));
          issue_c();
        }
      }
    }
  } else {
    const int q = warp & 3, h = (warp - 2) >> 2, row = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const float lr_reg = p.lr * p.reg;
    constexpr int kHalf = W / 2;
    float* xp = reinterpret_cast<float*>(sm + o_xp);
    for (int64_t k = 0; k < nk; ++k) {
      const int i = (int)(k % kI);
      const int32_t* s_idx = idx_of(k);
      mbar_wait(&bars[IFULL + i], (uint32_t)((k / kI) & 1));
      mbar_wait(&bars[CFULL], (uint32_t)(k & 1));
      tc_after();
      float part = 0.0f;
#pragma unroll 1
      for (int c = h * kHalf / 16; c < (h + 1) * kHalf / 16; ++c) {
        uint32_t v0[16], v1[16], v2[16];
        tmem_ld16(tl + 0 * W + c * 16, v0);
        tmem_ld16(tl + 1 * W + c * 16, v1);
        tmem_ld16(tl + 2 * W + c * 16, v2);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e)
          part = fmaf(__uint_as_float(v0[e]), __uint_as_float(v1[e]) * __uint_as_float(v2[e]), part);
      }
      xp[h * kRows + row] = part;
      named_bar(2 + q, 64);
      const float xhat = part + xp[(h ^ 1) * kRows + row];
      named_bar(2 + q, 64);
      const bool ok = row < reinterpret_cast<const int32_t*>(sm + o_rows)[i];
      const float resid = ok ? reinterpret_cast<const float*>(s_idx + kN * kRows)[row] - xhat : 0.0f;
      const float sc = p.lr * resid;
#pragma unroll 1
      for (int c = h * kHalf / 16; c < (h + 1) * kHalf / 16; ++c) {
        uint32_t v0[16], v1[16], v2[16];
        tmem_ld16(tl + 0 * W + c * 16, v0);
        tmem_ld16(tl + 1 * W + c * 16, v1);
        tmem_ld16(tl + 2 * W + c * 16, v2);
        tmem_wait_ld();
        uint32_t d0[16], d1[16], d2[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float c0 = __uint_as_float(v0[e]) * sc, c1 = __uint_as_float(v1[e]),
                      c2 = __uint_as_float(v2[e]);
          d0[e] = rn_bits(c1 * sc * c2);
          d1[e] = rn_bits(c0 * c2);
          d2[e] = rn_bits(c0 * c1);
        }
        tmem_st16(tl + 0 * W + c * 16, d0);
        tmem_st16(tl + 1 * W + c * 16, d1);
        tmem_st16(tl + 2 * W + c * 16, d2);
      }
      int32_t g[kN];  // read before the barrier: the COO record is then free
#pragma unroll
      for (int n = 0; n < kN; ++n) g[n] = s_idx[n * kRows + row];
      tmem_wait_st();
      tc_before();
      named_bar(1, 256);
      if (warp == 2 && lane == 0) {
        mbar_arrive(&bars[DFULL]);
        mbar_arrive(&bars[IEMPTY + i]);
      }
      for (int n = 0; n < kN; ++n) {
        const int64_t u = k * kN + n;
        // this warp's column half h came with U half job h of mode n
        const int64_t job = u_job(k) + 2 * n + h;
        const int s = (int)(job % kS);
        (void)u;
        mbar_wait(&bars[UFULL + n], (uint32_t)(k & 1));
        mbar_wait(&bars[FULL + s], (uint32_t)((job / kS) & 1));  // rows visible to this thread
        tc_after();
        uint32_t v[kHalf];
#pragma unroll
        for (int c = 0; c < kHalf / 16; ++c) tmem_ld16(tl + u_col(n) + h * kHalf + c * 16, *reinterpret_cast<uint32_t(*)[16]>(v + c * 16));
        tmem_wait_ld();
        const uint8_t* xs = sm + o_st + s * kStage;
        float4 a4[kHalf / 4];
#pragma unroll
        for (int qq = 0; qq < kHalf / 4; ++qq)  // column 4 qq of the half: block qq / 8
          a4[qq] = *reinterpret_cast<const float4*>(xs + (qq / 8) * kBlk + swz(row, (qq % 8) * 16, 128));
        tc_before();
        __syncwarp();
        if (lane == 0) {  // this warp has read its U columns and its rows
          mbar_arrive(&bars[EMPTY + s]);
          if (n == 0) mbar_arrive(&bars[U0READ]);
          if (n == kN - 1) mbar_arrive(&bars[UREAD]);
        }
        // write-back through a private 2 KB staging tile per warp: 16 columns
        // of its 32 rows at a time, sent as 64-B row segments (8 rows per RED)
        uint8_t* stage = sm + o_stage + (warp - 2) * 2048;
        int32_t gr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) gr[i] = __shfl_sync(0xffffffffu, ok ? g[n] : -1, i * 8 + (lane >> 2));
        float* dst = p.a[n] + h * kHalf + (lane & 3) * 4;
#pragma unroll
        for (int c = 0; c < kHalf / 16; ++c) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int qq = c * 4 + q4;
            const float4 a = a4[qq];
            float4 st;
            st.x = __uint_as_float(v[qq * 4 + 0]) - lr_reg * a.x;
            st.y = __uint_as_float(v[qq * 4 + 1]) - lr_reg * a.y;
            st.z = __uint_as_float(v[qq * 4 + 2]) - lr_reg * a.z;
            st.w = __uint_as_float(v[qq * 4 + 3]) - lr_reg * a.w;
            if (!p.atomic_update) {
              st.x += a.x;
              st.y += a.y;
              st.z += a.z;
              st.w += a.w;
            }
            *reinterpret_cast<float4*>(stage + swz(lane, q4 * 16, 64)) = st;
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 sv =
                *reinterpret_cast<const float4*>(stage + swz(i * 8 + (lane >> 2), (lane & 3) * 16, 64));
            if (gr[i] >= 0) {
              float* gp = dst + (size_t)gr[i] * W + c * 16;
              if (p.atomic_update)
                red_add_v4(gp, sv);
              else
                *reinterpret_cast<float4*>(gp) = sv;
            }
          }
          __syncwarp();
        }
      }
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x / 32 == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}


// B operand images, rounded to nearest tf32: bt (C GEMM: rows r, K = j) and
// b (U GEMM: rows j, K = r), K-major SW128 in 32-column blocks.
template <int W>
__global__ void big_images_kernel(const float* __restrict__ b, float* __restrict__ bt_img,
                                  float* __restrict__ b_img) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < W * W; e += gridDim.x * blockDim.x) {
    const int j = e / W, r = e - j * W;
    const float x = __uint_as_float(rn_bits(b[e]));
    *reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bt_img) + (j / 32) * (W * 128) +
                              swz(r, (j % 32) * 4, 128)) = x;
    *reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(b_img) + (r / 32) * (W * 128) +
                              swz(j, (r % 32) * 4, 128)) = x;
  }
}

__global__ void big_reduce_kernel(const float* __restrict__ partials, int nparts, int len,
                                  float* __restrict__ grad) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < len; e += gridDim.x * blockDim.x) {
    float s = 0.0f;
    for (int k = 0; k < nparts; ++k) s += partials[(size_t)k * len + e];
    grad[e] = s;
  }
}

// ---- J = R = 64 core sweep in one pass, fp16 copy of A ---------------------------
//
// With fp16 rows (128 B at W = 64) one SWIZZLE_128B tile per mode serves the
// K-major C GEMM and the MN-major G GEMM (16-bit operands take any swizzle in
// both majors), and TMEM holds C for all modes (192 columns) next to G for
// all modes (192): G stacks modes {0, 1} in M against [D'_0 | D'_1] (N = 128)
// and mode 2 (plus 64 ignored rows) against D'_2 (N = 64); only the diagonal
// blocks are read back.  One gather of 48 KB per tile replaces the three
// passes x four gathers of the tf32 sweep above.
//
//   warp 0  COO columns      warps 10-11  gathers (fp16 rows, half each)
//   warp 1  MMA issuer       warps 2-9    epilogue, two warps per lane quarter

namespace b16 {
constexpr int W = 64;
constexpr int kEpi = 8, kGW = 2, kGWarp = 2 + kEpi;
constexpr int kThreads = (2 + kEpi + kGW) * 32;
constexpr uint32_t kModeTile = kRows * 128;  // 128 rows x 64 fp16
constexpr uint32_t kSlot = kN * kModeTile;   // 48 KB
constexpr int kS = 3, kI = 3;
constexpr uint32_t o_a = 0;
constexpr uint32_t o_d = o_a + kS * kSlot;            // r D tiles (fp16, MN-major)
constexpr uint32_t o_bt = o_d + kSlot;                // B^T fp16 images, 8 KB per mode
constexpr uint32_t o_idx = o_bt + kN * W * 128;
constexpr uint32_t kIdxSlot = (kN + 1) * kRows * 4;
constexpr uint32_t o_rows = o_idx + kI * kIdxSlot;
constexpr uint32_t o_xp = o_rows + 64;                // x_hat halves [2][128]
constexpr uint32_t o_bar = o_xp + 2 * kRows * 4;
constexpr uint32_t o_tmem = o_bar + 16 * 8;
constexpr uint32_t bytes = o_tmem + 16;
static_assert(bytes <= 227 * 1024, "shared-memory budget");
enum : int { FULL = 0, EMPTY = 3, IFULL = 6, IEMPTY = 9, CFULL = 12, CEMPTY = 13, DFULL = 14, DEMPTY = 15 };
constexpr uint32_t t_c = 0, t_g = 3 * W;  // C: 192 columns; G: [stack01: 128][stack2: 64]

}  // namespace b16

__global__ void __launch_bounds__(b16::kThreads, 1) big16_core_kernel(const __grid_constant__ BigParams p) {
  using namespace b16;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + o_bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + o_tmem);
  for (int n = 0; n < kN; ++n)
    for (int e = threadIdx.x; e < W * W; e += blockDim.x) {
      const int j = e / W, r = e - j * W;  // B^T: rows r, K = j
      *reinterpret_cast<__half*>(sm + o_bt + n * W * 128 + swz(r, j * 2, 128)) =
          __float2half_rn(p.bt_img[n][e]);
    }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kS; ++s) {
      mbar_init(&bars[FULL + s], kGW);
      mbar_init(&bars[EMPTY + s], 1);
    }
    for (int i = 0; i < kI; ++i) {
      mbar_init(&bars[IFULL + i], 1);
      mbar_init(&bars[IEMPTY + i], kEpi + kGW);
    }
    mbar_init(&bars[CFULL], 1);
    mbar_init(&bars[CEMPTY], kEpi);
    mbar_init(&bars[DFULL], kEpi);
    mbar_init(&bars[DEMPTY], 1);
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

  if (warp == 0) {
    if (lane == 0) {
      auto ahead = tile_ahead<4>([&](int64_t kk) { return big_tile(p, kk); }, p.tile_rows, nk);
      for (int64_t k = 0; k < nk; ++k) {
        const int i = (int)(k % kI);
        int64_t tile;
        int32_t valid;
        ahead.pop(k, tile, valid);
        mbar_wait(&bars[IEMPTY + i], (uint32_t)(((k / kI) & 1) ^ 1));
        int32_t* s_idx = reinterpret_cast<int32_t*>(sm + o_idx + i * kIdxSlot);
        reinterpret_cast<int32_t*>(sm + o_rows)[i] = valid;
        mbar_expect_tx(&bars[IFULL + i], kIdxSlot);
        for (int n = 0; n < kN; ++n)
          bulk_g2s(s_idx + n * kRows, p.idx[n] + tile * kRows, kRows * 4, &bars[IFULL + i]);
        bulk_g2s(s_idx + kN * kRows, p.vals + tile * kRows, kRows * 4, &bars[IFULL + i]);
      }
    }
  } else if (warp >= kGWarp) {
    const int gw = warp - kGWarp;
    constexpr int kPer = kN * kRows / 4 / kGW;  // 48 groups of 4 rows
    for (int64_t k = 0; k < nk; ++k) {
      const int s = (int)(k % kS), i = (int)(k % kI);
      mbar_wait(&bars[EMPTY + s], (uint32_t)(((k / kS) & 1) ^ 1));
      mbar_wait(&bars[IFULL + i], (uint32_t)((k / kI) & 1));
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + o_idx + i * kIdxSlot);
      uint8_t* slot = sm + o_a + s * kSlot;
      __syncwarp();
      if (elect_one()) {
        mbar_expect_tx(&bars[FULL + s], kPer * 512);
#pragma unroll 1
        for (int g0 = gw * kPer; g0 < (gw + 1) * kPer; g0 += 8) {
          int4 r[8];
#pragma unroll
          for (int g = 0; g < 8; ++g) r[g] = *reinterpret_cast<const int4*>(s_idx + (g0 + g) * 4);
          const int n = g0 / (kRows / 4), gm = g0 - n * (kRows / 4);
#pragma unroll
          for (int g = 0; g < 8; ++g)
            tma_gather4(slot + n * kModeTile + (gm + g) * 512, &p.tmap[n], 0, r[g].x, r[g].y,
                        r[g].z, r[g].w, &bars[FULL + s]);
        }
        mbar_arrive(&bars[IEMPTY + i]);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idc = idesc_f16(128, W, 0, 0);
      const uint32_t bt = smem_u32(sm + o_bt), d0 = smem_u32(sm + o_d);
      auto issue_g = [&](int64_t k) {
        const int s = (int)(k % kS);
        mbar_wait(&bars[DFULL], (uint32_t)(k & 1));
        tc_after();
        const uint32_t a0 = smem_u32(sm + o_a + s * kSlot);
#pragma unroll
        for (int ks = 0; ks < kRows / 16; ++ks) {
          // stack {0, 1}: M = A_0^T ; A_1^T, N = D'_0 | D'_1
          mma_f16(tmem + t_g, sdesc_l(a0 + ks * 2048, kModeTile, 1024, 2),
                  sdesc_l(d0 + ks * 2048, kModeTile, 1024, 2), idesc_f16(128, 2 * W, 1, 1),
                  (k > 0 || ks > 0) ? 1u : 0u);
          // stack {2, -}: M = A_2^T (+ 64 ignored rows), N = D'_2
          mma_f16(tmem + t_g + 2 * W, sdesc_l(a0 + 2 * kModeTile + ks * 2048, kModeTile, 1024, 2),
                  sdesc_l(d0 + 2 * kModeTile + ks * 2048, kModeTile, 1024, 2),
                  idesc_f16(128, W, 1, 1), (k > 0 || ks > 0) ? 1u : 0u);
        }
        mma_commit(&bars[DEMPTY]);
        mma_commit(&bars[EMPTY + s]);
      };
      for (int64_t k = 0; k < nk; ++k) {
        const int s = (int)(k % kS);
        mbar_wait(&bars[FULL + s], (uint32_t)((k / kS) & 1));
        mbar_wait(&bars[CEMPTY], (uint32_t)((k & 1) ^ 1));
        tc_after();
        const uint32_t a0 = smem_u32(sm + o_a + s * kSlot);
#pragma unroll
        for (int n = 0; n < kN; ++n)
#pragma unroll
          for (int ks = 0; ks < W / 16; ++ks)
            mma_f16(tmem + t_c + n * W, sdesc_l(a0 + n * kModeTile + ks * 32, 16, 1024, 2),
                    sdesc_l(bt + n * W * 128 + ks * 32, 16, 1024, 2), idc, ks > 0);
        mma_commit(&bars[CFULL]);
        if (k >= 1) issue_g(k - 1);
      }
      if (nk >= 1) issue_g(nk - 1);
    }
  } else {
    const int ew = warp - 2, q = warp & 3, h = ew >> 2;  // h: 32-column half
    const int row = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    float* xp = reinterpret_cast<float*>(sm + o_xp);
    for (int64_t k = 0; k < nk; ++k) {
      const int ii = (int)(k % kI);
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + o_idx + ii * kIdxSlot);
      mbar_wait(&bars[IFULL + ii], (uint32_t)((k / kI) & 1));
      mbar_wait(&bars[CFULL], (uint32_t)(k & 1));
      tc_after();
      float c[kN][32];
#pragma unroll
      for (int n = 0; n < kN; ++n)
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
          uint32_t v[16];
          tmem_ld16(tl + t_c + n * W + h * 32 + c2 * 16, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) c[n][c2 * 16 + i] = __uint_as_float(v[i]);
        }
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[CEMPTY]);  // C(k + 1) may land
      float part = 0.0f;
#pragma unroll
      for (int i = 0; i < 32; ++i) part = fmaf(c[0][i], c[1][i] * c[2][i], part);
      xp[h * kRows + row] = part;
      named_bar(1 + q, 64);
      const float xhat = part + xp[(h ^ 1) * kRows + row];
      named_bar(1 + q, 64);  // both halves read before the next tile's writes
      const bool ok = row < reinterpret_cast<const int32_t*>(sm + o_rows)[ii];
      const float resid = ok ? reinterpret_cast<const float*>(s_idx + kN * kRows)[row] - xhat : 0.0f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[IEMPTY + ii]);
      mbar_wait(&bars[DEMPTY], (uint32_t)((k & 1) ^ 1));  // G(k - 1) done with D'
#pragma unroll
      for (int n = 0; n < kN; ++n)
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {  // 8 columns = one 16-B chunk of fp16
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i0 = q8 * 8 + e * 2;
#define FTK_D(ii) (n == 0 ? c[1][ii] * c[2][ii] : (n == 1 ? c[0][ii] * c[2][ii] : c[0][ii] * c[1][ii]))
            w[e] = f16x2_sat(resid * FTK_D(i0), resid * FTK_D(i0 + 1));
#undef FTK_D
          }
          *reinterpret_cast<uint4*>(sm + o_d + n * kModeTile + swz(row, (h * 32 + q8 * 8) * 2, 128)) =
              make_uint4(w[0], w[1], w[2], w[3]);
        }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[DFULL]);
    }
    if (nk > 0) mbar_wait(&bars[DEMPTY], (uint32_t)((nk - 1) & 1));
    tc_after();
    // diagonal blocks: lanes 0..63 -> G_0 (cols t_g) and G_2 (t_g + 128);
    // lanes 64..127 -> G_1 (t_g + 64); this warp: its 32 lanes, columns h*32..
    float* outb = p.partials + (size_t)blockIdx.x * (kN * W * W);
    const int modes[2] = {q < 2 ? 0 : 1, q < 2 ? 2 : -1};
    const uint32_t cols[2] = {q < 2 ? t_g : t_g + W, t_g + 2 * W};
    const int j = (q & 1) * 32 + lane;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      if (modes[mi] < 0) continue;  // warp-uniform
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        uint32_t v[16];
        tmem_ld16(tl + cols[mi] + h * 32 + c2 * 16, v);
        tmem_wait_ld();
        float* out = outb + ((size_t)modes[mi] * W + j) * W + h * 32 + c2 * 16;
#pragma unroll
        for (int i = 0; i < 16; ++i) out[i] = nk > 0 ? __uint_as_float(v[i]) : 0.0f;
      }
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x / 32 == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ---- J = R = 128 core sweep: one pass per mode on the fp16 copy of A -----------
//
// TMEM fits C for all modes (384 columns) next to one mode's G (128), so the
// core runs one launch per mode p.  Per tile the three C jobs gather each
// mode's fp16 rows (32 KB, two 128-B column blocks per row) into a 2-stage
// ring, mode p last; its stage is then also the MN-major A of G_p += A_p^T
// D'_p (kind::f16), so no second gather.  The B^T images stay resident.

namespace b16p {
constexpr int W = 128;
constexpr int kEpi = 8, kGW = 2, kGWarp = 2 + kEpi;
constexpr int kThreads = (2 + kEpi + kGW) * 32;
constexpr uint32_t kBlk16 = kRows * 128;          // 64 fp16 columns of 128 rows
constexpr uint32_t kStage = 2 * kBlk16;           // one mode's rows: 32 KB
constexpr int kS = 2, kI = 3;
constexpr uint32_t o_a = 0;
constexpr uint32_t o_d = o_a + kS * kStage;       // D'_p (fp16, MN-major, 2 blocks)
constexpr uint32_t o_bt = o_d + kStage;           // B^T fp16 images: 32 KB per mode
constexpr uint32_t o_idx = o_bt + kN * W * 256;
constexpr uint32_t kIdxSlot = (kN + 1) * kRows * 4;
constexpr uint32_t o_rows = o_idx + kI * kIdxSlot;
constexpr uint32_t o_xp = o_rows + 64;
constexpr uint32_t o_bar = o_xp + 2 * kRows * 4;
constexpr uint32_t o_tmem = o_bar + 16 * 8;
constexpr uint32_t bytes = o_tmem + 16;
static_assert(bytes <= 227 * 1024, "shared-memory budget");
enum : int { FULL = 0, EMPTY = 2, IFULL = 4, IEMPTY = 7, CFULL = 10, CEMPTY = 11, DFULL = 12, DEMPTY = 13 };
constexpr uint32_t t_c = 0, t_g = 3 * W;  // C: 384 columns; G_p: 128
}  // namespace b16p

__global__ void __launch_bounds__(b16p::kThreads, 1) big16p_core_kernel(const __grid_constant__ BigParams p) {
  using namespace b16p;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + o_bar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + o_tmem);
  const int pm = p.pass;
  for (int n = 0; n < kN; ++n)
    for (int e = threadIdx.x; e < W * W; e += blockDim.x) {
      const int j = e / W, r = e - j * W;  // B^T: rows r, K = j (two 64-column blocks)
      *reinterpret_cast<__half*>(sm + o_bt + n * W * 256 + (j / 64) * (W * 128) +
                                 swz(r, (j % 64) * 2, 128)) = __float2half_rn(p.bt_img[n][e]);
    }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kS; ++s) {
      mbar_init(&bars[FULL + s], kGW);
      mbar_init(&bars[EMPTY + s], 1);
    }
    for (int i = 0; i < kI; ++i) {
      mbar_init(&bars[IFULL + i], 1);
      mbar_init(&bars[IEMPTY + i], kEpi + kGW);
    }
    mbar_init(&bars[CFULL], 1);
    mbar_init(&bars[CEMPTY], kEpi);
    mbar_init(&bars[DFULL], kEpi);
    mbar_init(&bars[DEMPTY], 1);
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
  // per tile the modes are gathered in the order m0, m1, pm (pm last)
  const int m0 = pm == 0 ? 1 : 0, m1 = pm == 2 ? 1 : 2;
  auto mode_of = [&](int j) { return j == 0 ? m0 : (j == 1 ? m1 : pm); };

  if (warp == 0) {
    if (lane == 0) {
      auto ahead = tile_ahead<4>([&](int64_t kk) { return big_tile(p, kk); }, p.tile_rows, nk);
      for (int64_t k = 0; k < nk; ++k) {
        const int i = (int)(k % kI);
        int64_t tile;
        int32_t valid;
        ahead.pop(k, tile, valid);
        mbar_wait(&bars[IEMPTY + i], (uint32_t)(((k / kI) & 1) ^ 1));
        int32_t* s_idx = reinterpret_cast<int32_t*>(sm + o_idx + i * kIdxSlot);
        reinterpret_cast<int32_t*>(sm + o_rows)[i] = valid;
        mbar_expect_tx(&bars[IFULL + i], kIdxSlot);
        for (int n = 0; n < kN; ++n)
          bulk_g2s(s_idx + n * kRows, p.idx[n] + tile * kRows, kRows * 4, &bars[IFULL + i]);
        bulk_g2s(s_idx + kN * kRows, p.vals + tile * kRows, kRows * 4, &bars[IFULL + i]);
      }
    }
  } else if (warp >= kGWarp) {
    const int gw = warp - kGWarp;
    constexpr int kPer = kRows / 4 / kGW;  // 16 groups of 4 rows per warp per mode
    int64_t job = 0;
    for (int64_t k = 0; k < nk; ++k) {
      const int i = (int)(k % kI);
      mbar_wait(&bars[IFULL + i], (uint32_t)((k / kI) & 1));
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + o_idx + i * kIdxSlot);
      for (int j = 0; j < kN; ++j, ++job) {
        const int s = (int)(job % kS), n = mode_of(j);
        mbar_wait(&bars[EMPTY + s], (uint32_t)(((job / kS) & 1) ^ 1));
        uint8_t* st = sm + o_a + s * kStage;
        __syncwarp();
        if (elect_one()) {
          mbar_expect_tx(&bars[FULL + s], kPer * 4 * 256);
#pragma unroll 1
          for (int g0 = gw * kPer; g0 < (gw + 1) * kPer; g0 += 8) {
            int4 r[8];
#pragma unroll
            for (int g = 0; g < 8; ++g)
              r[g] = *reinterpret_cast<const int4*>(s_idx + n * kRows + (g0 + g) * 4);
#pragma unroll
            for (int g = 0; g < 8; ++g)
#pragma unroll
              for (int cb = 0; cb < 2; ++cb)
                tma_gather4(st + cb * kBlk16 + (g0 + g) * 512, &p.tmap[n], cb * 64, r[g].x,
                            r[g].y, r[g].z, r[g].w, &bars[FULL + s]);
          }
          if (j == kN - 1) mbar_arrive(&bars[IEMPTY + i]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idc = idesc_f16(128, W, 0, 0), idg = idesc_f16(128, W, 1, 1);
      const uint32_t bt = smem_u32(sm + o_bt), d0 = smem_u32(sm + o_d);
      int64_t job = 0;
      int sp_prev = 0;
      // G(k - 1) holds the previous pm stage, which is also job 1's stage of tile k:
      // issue it between jobs 0 and 1 (D'(k - 1) is written before C(k) may land)
      auto issue_g = [&](int64_t kg, int sg) {
        mbar_wait(&bars[DFULL], (uint32_t)(kg & 1));
        tc_after();
        const uint32_t a0 = smem_u32(sm + o_a + sg * kStage);
#pragma unroll
        for (int ks = 0; ks < kRows / 16; ++ks)
          mma_f16(tmem + t_g, sdesc_l(a0 + ks * 2048, kBlk16, 1024, 2),
                  sdesc_l(d0 + ks * 2048, kBlk16, 1024, 2), idg, (kg > 0 || ks > 0) ? 1u : 0u);
        mma_commit(&bars[DEMPTY]);
        mma_commit(&bars[EMPTY + sg]);
      };
      for (int64_t k = 0; k < nk; ++k) {
        mbar_wait(&bars[CEMPTY], (uint32_t)((k & 1) ^ 1));
        int sp = 0;
        for (int j = 0; j < kN; ++j, ++job) {
          const int s = (int)(job % kS), n = mode_of(j);
          mbar_wait(&bars[FULL + s], (uint32_t)((job / kS) & 1));
          tc_after();
          const uint32_t a0 = smem_u32(sm + o_a + s * kStage);
#pragma unroll
          for (int ks = 0; ks < W / 16; ++ks)
            mma_f16(tmem + t_c + n * W,
                    sdesc_l(a0 + (ks / 4) * kBlk16 + (ks % 4) * 32, 16, 1024, 2),
                    sdesc_l(bt + n * W * 256 + (ks / 4) * (W * 128) + (ks % 4) * 32, 16, 1024, 2),
                    idc, ks > 0);
          if (j < kN - 1) mma_commit(&bars[EMPTY + s]);  // pm's stage waits for G
          else sp = s;
          if (j == 0 && k >= 1) issue_g(k - 1, sp_prev);
        }
        mma_commit(&bars[CFULL]);
        sp_prev = sp;
      }
      if (nk >= 1) issue_g(nk - 1, sp_prev);
    }
  } else {
    const int ew = warp - 2, q = warp & 3, h = ew >> 2;  // h: 64-column half
    const int row = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    float* xp = reinterpret_cast<float*>(sm + o_xp);
    for (int64_t k = 0; k < nk; ++k) {
      const int ii = (int)(k % kI);
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(sm + o_idx + ii * kIdxSlot);
      mbar_wait(&bars[IFULL + ii], (uint32_t)((k / kI) & 1));
      mbar_wait(&bars[CFULL], (uint32_t)(k & 1));
      tc_after();
      float part = 0.0f;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v0[16], v1[16], v2[16];
        tmem_ld16(tl + t_c + 0 * W + h * 64 + c * 16, v0);
        tmem_ld16(tl + t_c + 1 * W + h * 64 + c * 16, v1);
        tmem_ld16(tl + t_c + 2 * W + h * 64 + c * 16, v2);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e)
          part = fmaf(__uint_as_float(v0[e]), __uint_as_float(v1[e]) * __uint_as_float(v2[e]), part);
      }
      xp[h * kRows + row] = part;
      named_bar(1 + q, 64);
      const float xhat = part + xp[(h ^ 1) * kRows + row];
      named_bar(1 + q, 64);
      const bool ok = row < reinterpret_cast<const int32_t*>(sm + o_rows)[ii];
      const float resid = ok ? reinterpret_cast<const float*>(s_idx + kN * kRows)[row] - xhat : 0.0f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[IEMPTY + ii]);
      mbar_wait(&bars[DEMPTY], (uint32_t)((k & 1) ^ 1));  // G(k - 1) done with D'
      // D'_pm = r C_m0 C_m1 over this warp's 64 columns, fp16, MN-major
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v0[16], v1[16];
        tmem_ld16(tl + t_c + m0 * W + h * 64 + c * 16, v0);
        tmem_ld16(tl + t_c + m1 * W + h * 64 + c * 16, v1);
        tmem_wait_ld();
#pragma unroll
        for (int q8 = 0; q8 < 2; ++q8) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i0 = q8 * 8 + e * 2;
            w[e] = f16x2_sat(resid * __uint_as_float(v0[i0]) * __uint_as_float(v1[i0]),
                             resid * __uint_as_float(v0[i0 + 1]) * __uint_as_float(v1[i0 + 1]));
          }
          *reinterpret_cast<uint4*>(sm + o_d + h * kBlk16 + swz(row, (c * 16 + q8 * 8) * 2, 128)) =
              make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[CEMPTY]);  // C(k + 1) may land
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[DFULL]);
    }
    if (nk > 0) mbar_wait(&bars[DEMPTY], (uint32_t)((nk - 1) & 1));
    tc_after();
    // G_pm: TMEM lane j (all 128), columns t_g + r; this warp: its lanes, half h
    float* out = p.partials + (size_t)blockIdx.x * (kN * W * W) + (size_t)pm * W * W +
                 (size_t)row * W + h * 64;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t v[16];
      tmem_ld16(tl + t_g + h * 64 + c * 16, v);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 16; ++e) out[c * 16 + e] = nk > 0 ? __uint_as_float(v[e]) : 0.0f;
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (threadIdx.x / 32 == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

__global__ void big_half_kernel(const float* __restrict__ src, __half* __restrict__ dst, int64_t n2,
                                int* __restrict__ range) {
  bool out = false;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n2;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float2 x = reinterpret_cast<const float2*>(src)[e];
    out |= !(fabsf(x.x) <= 65504.f) || !(fabsf(x.y) <= 65504.f);  // NaN too
    reinterpret_cast<uint32_t*>(dst)[e] = f16x2_sat(x.x, x.y);
  }
  if (out && range) atomicExch(range, 1);  // clamped: reported by the session (KView::f16_range)
}

PFN_cuTensorMapEncodeTiled_v12000 big_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn),
                            cudaEnableDefault, &q);
  }
  return fn;
}

// Row-gather map of A_n (rows x W fp32): box of 32 columns x 1 row.
bool big_row_map(CUtensorMap* tm, const float* a, int64_t rows, int w, bool atom32) {
  auto fn = big_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)w * 4};
  cuuint32_t box[2] = {32, 1};
  cuuint32_t es[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Row-gather map of an fp16 copy of A_n (rows x w fp16): box of 64 columns
// (one 128-B row block).
bool big_row_map16(CUtensorMap* tm, const __half* a, int64_t rows, int w = 64) {
  auto fn = big_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)w * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(a), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t run_core16(const KView& v, const int32_t* dims, int64_t mul, int64_t add, float* grad,
                       float* scratch, size_t scratch_bytes, cudaStream_t st) {
  constexpr int W = 64;
  const int grid = (int)(v.ntiles < num_sms() ? v.ntiles : num_sms());
  const size_t len = (size_t)kN * W * W;
  if (grid < 1) return cudaErrorInvalidValue;
  if (scratch_bytes < big_scratch_bytes(v, dims, true)) return cudaErrorInvalidValue;
  BigParams p{};
  __half* a16 = reinterpret_cast<__half*>(scratch + (size_t)num_sms() * len);
  for (int n = 0; n < kN; ++n) {
    const int64_t n2 = (int64_t)dims[n] * W / 2;
    int64_t blocks = (n2 + 255) / 256;
    if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
    big_half_kernel<<<(int)blocks, 256, 0, st>>>(v.a[n], a16, n2, v.f16_range);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (!big_row_map16(&p.tmap[n], a16, dims[n])) return cudaErrorNotSupported;
    p.idx[n] = v.idx[n];
    p.bt_img[n] = v.b[n];  // raw B (J x R), rounded to fp16 in the kernel
    a16 += (int64_t)dims[n] * W;
  }
  p.vals = v.vals;
  p.ntiles = v.ntiles;
  p.tile_base = v.tile_base;
  p.tile_rows = v.tile_rows;
  p.tperm = v.tperm;
  p.tmul = mul;
  p.tadd = add;
  p.partials = scratch;
  cudaError_t e = cudaFuncSetAttribute(big16_core_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b16::bytes);
  if (e != cudaSuccess) return e;
  big16_core_kernel<<<grid, b16::kThreads, b16::bytes, st>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  big_reduce_kernel<<<(int)((len + 255) / 256), 256, 0, st>>>(scratch, grid, (int)len, grad);
  return cudaGetLastError();
}

cudaError_t run_core16p(const KView& v, const int32_t* dims, int64_t mul, int64_t add, float* grad,
                        float* scratch, size_t scratch_bytes, cudaStream_t st) {
  constexpr int W = 128;
  const int grid = (int)(v.ntiles < num_sms() ? v.ntiles : num_sms());
  const size_t len = (size_t)kN * W * W;
  if (grid < 1) return cudaErrorInvalidValue;
  if (scratch_bytes < big_scratch_bytes(v, dims, true)) return cudaErrorInvalidValue;
  BigParams p{};
  __half* a16 = reinterpret_cast<__half*>(scratch + (size_t)num_sms() * len);
  for (int n = 0; n < kN; ++n) {
    const int64_t n2 = (int64_t)dims[n] * W / 2;
    int64_t blocks = (n2 + 255) / 256;
    if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
    big_half_kernel<<<(int)blocks, 256, 0, st>>>(v.a[n], a16, n2, v.f16_range);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (!big_row_map16(&p.tmap[n], a16, dims[n], W)) return cudaErrorNotSupported;
    p.idx[n] = v.idx[n];
    p.bt_img[n] = v.b[n];
    a16 += (int64_t)dims[n] * W;
  }
  p.vals = v.vals;
  p.ntiles = v.ntiles;
  p.tile_base = v.tile_base;
  p.tile_rows = v.tile_rows;
  p.tperm = v.tperm;
  p.tmul = mul;
  p.tadd = add;
  p.partials = scratch;
  cudaError_t e = cudaFuncSetAttribute(big16p_core_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b16p::bytes);
  if (e != cudaSuccess) return e;
  for (int pass = 0; pass < kN; ++pass) {
    p.pass = pass;
    big16p_core_kernel<<<grid, b16p::kThreads, b16p::bytes, st>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  big_reduce_kernel<<<(int)((len + 255) / 256), 256, 0, st>>>(scratch, grid, (int)len, grad);
  return cudaGetLastError();
}

template <int W>
cudaError_t prepare(BigParams& p, const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                    float* img, cudaStream_t st) {
  for (int n = 0; n < kN; ++n) {
    if (!big_row_map(&p.tmap[n], v.a[n], dims[n], W, false)) return cudaErrorNotSupported;
    p.idx[n] = v.idx[n];
    p.a[n] = v.a[n];
    float* bt = img + (size_t)(2 * n) * W * W;
    float* bb = img + (size_t)(2 * n + 1) * W * W;
    p.bt_img[n] = bt;
    p.b_img[n] = bb;
    big_images_kernel<W><<<(W * W + 255) / 256, 256, 0, st>>>(v.b[n], bt, bb);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  p.vals = v.vals;
  p.ntiles = v.ntiles;
  p.tile_base = v.tile_base;
  p.tile_rows = v.tile_rows;
  p.tperm = v.tperm;
  p.tmul = mul;
  p.tadd = add;
  return cudaSuccess;
}

template <int W>
cudaError_t run_factor(const KView& v, const int32_t* dims, int64_t mul, int64_t add, float lr,
                       float reg, int atomic_update, float* img, cudaStream_t st) {
  BigParams p{};
  cudaError_t e = prepare<W>(p, v, dims, mul, add, img, st);
  if (e != cudaSuccess) return e;
  p.lr = lr;
  p.reg = reg;
  p.atomic_update = atomic_update;
  // W = 128: the K-split half-job sweep
  int bytes;
  void (*kern)(BigParams);
  if constexpr (W == 128) {
    bytes = (int)f128::bytes;
    kern = big128_factor_kernel;
  } else {
    bytes = (int)BigLayout<W, false>::bytes;
    kern = big_factor_kernel<W>;
  }
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  kern<<<(int)sweep_grid(v), kThreadsF, bytes, st>>>(p);
  return cudaGetLastError();
}


}  // namespace

bool big_supported(const KView& v) {
  return v.order == kN && (v.r == 64 || v.r == 128) && v.j[0] == v.r && v.j[1] == v.r &&
         v.j[2] == v.r && big_encode_fn() != nullptr;
}

size_t big_scratch_bytes(const KView& v, const int32_t* dims, bool core) {
  const size_t w = (size_t)v.r;
  size_t f = 2 * kN * w * w;  // B operand images
  if (core) {
    f += (size_t)num_sms() * kN * w * w;  // per-CTA gradients
    for (int n = 0; n < kN; ++n) f += (size_t)dims[n] * w;  // rounded A copies
  }
  return f * sizeof(float);
}

cudaError_t launch_big_factor(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                              float lr, float reg, int atomic_update, float* scratch,
                              size_t scratch_bytes, cudaStream_t st) {
  if (v.ntiles == 0) return cudaSuccess;
  if (scratch_bytes < 2 * kN * (size_t)v.r * v.r * sizeof(float)) return cudaErrorInvalidValue;
  return v.r == 64 ? run_factor<64>(v, dims, mul, add, lr, reg, atomic_update, scratch, st)
                   : run_factor<128>(v, dims, mul, add, lr, reg, atomic_update, scratch, st);
}

cudaError_t launch_big_core(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                            float* grad, float* scratch, size_t scratch_bytes, cudaStream_t st) {
  // fp16 copy of A: W = 64 in one pass, W = 128 in one pass per mode
  return v.r == 64 ? run_core16(v, dims, mul, add, grad, scratch, scratch_bytes, st)
                   : run_core16p(v, dims, mul, add, grad, scratch, scratch_bytes, st);
}

}  // namespace ftkcu
