// Internal declarations shared by the engine's translation units.
//
// Device data layout:
//   * COO tensor, storage order: SoA, one int32 column per mode + fp32 values
//     (the reference's AoS `indices[nnz*N]`, sparse_tensor.hpp:14-33, is
//     transposed once at upload so a warp reads 128 B per mode per 32 nnz).
//   * COO tensor, Hogwild order: the same SoA shuffled once per session
//     (cub radix sort on hashed keys) and visited tile by tile in a per-epoch
//     affine tile permutation.
//   * Model: A_n (I_n x J_n) and B_n (J_n x R) fp32 row-major, one cudaMalloc
//     each (256-B aligned rows when J_n % 64 == 0).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ftkcu.h"

namespace ftkcu {

constexpr int kMaxOrder = 8;
constexpr int kTile = 16;  // reference tile edge (tiles.hpp:12-14)

inline int pad16(int x) { return (x + kTile - 1) / kTile * kTile; }

struct DevTensor {
  int order = 0;
  int32_t dims[kMaxOrder] = {};
  int64_t nnz = 0;
  int32_t* idx[kMaxOrder] = {};  // storage order SoA
  float* vals = nullptr;
  // Cells (DSGD strata blocks): entries [cell_off[c], cell_off[c+1]) in
  // storage order.  Empty = one cell holding everything.
  std::vector<int64_t> cell_off;
  // Hogwild stream, built lazily by the tiler: every cell shuffled and padded
  // to whole tiles; cell c owns physical tiles [cell_tile[c], cell_tile[c+1]).
  bool shuffled = false;
  int32_t* sidx[kMaxOrder] = {};
  float* svals = nullptr;
  int32_t* tile_rows = nullptr;      // valid rows per physical tile
  std::vector<int64_t> cell_tile;
  int64_t stream_tiles = 0;
  int64_t stream_cap = 0;            // allocated tiles
  // order 3: storage-order records (i0, i1, i2, value) of 16 B, so the
  // shuffle gathers one aligned record per nonzero instead of four words
  int4* rec16 = nullptr;
  int64_t rec16_cap = 0;
  // cells keep their uploaded order (no shuffle inside a cell; the caller
  // arranged it, e.g. DSGD cells in mode-3 runs); tiles are still permuted
  bool keep_order = false;
  // order 3: lay the stream out in aligned 16-nonzero chunks that share
  // their last-mode index, chunks in random order (build_shuffled); scratch
  // for the sort kept across re-uploads
  bool runs = false;
  void* runs_scratch = nullptr;
  size_t runs_cap = 0;
  // Asynchronous upload (ftkcu_tensor_upload_async): AoS staging on the
  // copy stream, completion event, index-range flag checked at first use.
  int32_t* staging = nullptr;
  size_t staging_cap = 0;
  int* d_bad = nullptr;
  cudaEvent_t ready = nullptr;
  bool pending = false;
  // delta-coded upload decoded at first use on the session stream (option
  // delta_decode = 1): the staging holds the deltas, then the restarts
  bool delta_pending = false, delta_scatter = false;
  int delta_width = 0;
  size_t delta_roff = 0;
  uint64_t delta_seed = 0;
  // Recorded on the session stream when another slot's work begins: every
  // kernel that read this slot precedes it, so an asynchronous re-upload
  // waits for exactly that (and not for work on other slots).
  cudaEvent_t used = nullptr;
  bool used_rec = false;
};

struct DevModel {
  int order = 0;
  int32_t dims[kMaxOrder] = {};
  int32_t ranks[kMaxOrder] = {};
  int32_t r = 0;
  float* a[kMaxOrder] = {};
  float* b[kMaxOrder] = {};
  // Storage scheme (EpochOptions.store_c): C_n = A_n B_n per mode, I_n x R,
  // rebuilt at the start of every core phase (CCache, decomposition.cpp:74-107).
  float* cc[kMaxOrder] = {};
  int sum_j() const {
    int s = 0;
    for (int n = 0; n < order; ++n) s += ranks[n];
    return s;
  }
  int max_j() const {
    int s = 0;
    for (int n = 0; n < order; ++n) s = ranks[n] > s ? ranks[n] : s;
    return s;
  }
};

// Kernel-side view of model + tensor, passed by value.
struct KView {
  int order;
  int r;
  int32_t j[kMaxOrder];
  float* a[kMaxOrder];
  const float* b[kMaxOrder];
  const int32_t* idx[kMaxOrder];
  const float* vals;
  int64_t nnz;
  // Hogwild stream range: physical tiles [tile_base, tile_base + ntiles),
  // tile_rows[p] valid rows of physical tile p (the rest is padding).
  const int32_t* tile_rows;
  int64_t tile_base, ntiles;
  // Factor sweeps: cap on resident CTAs (0 = one per SM), bounds how many
  // nonzeros are in flight against the same A rows (Hogwild staleness).
  int max_ctas;
  // Headline factor sweep (ws_factor_kernel): 0 = a tile's row slot is freed
  // when its C GEMM completes (gathers run up to kS tiles ahead of the
  // write-back); W in {2, 3} = freed only after the tile's write-back is
  // issued and a gather waits for tile k - W to retire, so at most W tiles
  // per CTA are between reading and writing their rows (Hogwild staleness).
  int window;
  // Optional device {mul, add} of the tile permutation (overrides the launch
  // arguments; lets a captured CUDA graph take a new permutation per epoch).
  const int64_t* tperm;
  // Core sweeps, storage scheme: C rows gathered from the cache instead of
  // computed (stage_c_rows_from_cache, decomposition.cpp:299-314); null =
  // calculation scheme.
  const float* cc[kMaxOrder];
  // fp16 operand copies of A (core16 sweeps): set to 1 when an entry is
  // outside the fp16 range (|a| > 65504 or not finite) and was clamped by
  // the satfinite conversion; mapped host memory, reported by the session
  int* f16_range;
};

int num_sms();

// Persistent grid for a tile range: one CTA per SM, at most one per tile,
// at most v.max_ctas when set.
inline int64_t sweep_grid(const KView& v, int64_t per_sm_ctas = 1) {
  int64_t g = (int64_t)num_sms() * per_sm_ctas;
  if (v.max_ctas > 0 && g > v.max_ctas) g = v.max_ctas;
  if (g > v.ntiles) g = v.ntiles;
  return g;
}

// Optional per-batch debug outputs of the deterministic kernels (device
// pointers, any may be null).  Layouts match ftkcu_batch_probe.
struct DetDebug {
  float* c = nullptr;       // [order][cap][R]
  float* d = nullptr;       // [order][cap][R]
  float* u = nullptr;       // [order][cap][Jmax]
  float* xhat = nullptr;    // [cap]
  float* resid = nullptr;   // [cap]
  int jmax = 0;
};

// ---- deterministic sweeps (det_kernels.cu) ---------------------------------
cudaError_t launch_det_factor(const KView& v, const int64_t* perm, int cap,
                              float lr_a, float reg_a, const DetDebug& dbg,
                              cudaStream_t st);
// Accumulates the ordered core gradient into grad (sum_n J_n*R floats,
// zeroed by the caller).
cudaError_t launch_det_core(const KView& v, const int64_t* perm, int cap,
                            float* grad, const DetDebug& dbg, cudaStream_t st);
// total = 0 + grad; B += lr_b (total * (1/nnz) - reg_b B)
cudaError_t launch_apply_core(const KView& v, float* grad, float lr_b,
                              float reg_b, cudaStream_t st);

// ---- FastTucker baseline (ft_kernels.cu) -----------
// Factor block of `mode`: perm holds the per-bucket plan's positions, boff
// the nbuckets + 1 bucket offsets into it (plan order); one warp per bucket.
size_t ft_factor_smem(const KView& v, int cap, int mode);
cudaError_t launch_ft_factor(const KView& v, int mode, const int64_t* perm, const int64_t* boff,
                             int64_t nbuckets, int cap, float lr_a, float reg_a, cudaStream_t st);
// Core block of `mode`: the global plan's batches in order, B^(mode) updated
// after every batch (hogwild: by many CTAs at once, atomically).
size_t ft_core_smem(const KView& v, int cap);
cudaError_t launch_ft_core(const KView& v, int mode, const int64_t* perm, int cap, float lr_b,
                           float reg_b, bool hogwild, cudaStream_t st);

// ---- FasterTucker baseline (fst_kernels.cu) -------
// Factor block of `mode`: perm = the complement-keyed per-bucket plan's
// positions regrouped by mode-n row (plan order inside a row), goff the
// ngroups + 1 group offsets.  v.cc: the C cache of every mode.
cudaError_t launch_fst_factor(const KView& v, int mode, const int64_t* perm, const int64_t* goff,
                              int64_t ngroups, float lr_a, float reg_a, cudaStream_t st);
// Core block of `mode`: batches [boff[b], boff[b+1]) of perm in order.
// scratch: at least fst_core_scratch_floats(v, mode) floats.
size_t fst_core_scratch_floats(const KView& v, int mode);
cudaError_t launch_fst_core(const KView& v, int mode, const int64_t* perm, const int64_t* boff,
                            int64_t nbatches, float lr_b, float reg_b, float* scratch,
                            cudaStream_t st);
// workers > 1: the block's linear B recurrence summed in closed form, batches
// in parallel (scratch: 2 x num_sms() x J x R floats).
bool fst_scan_supported(const KView& v, int mode);
cudaError_t launch_fst_core_scan(const KView& v, int mode, const int64_t* perm,
                                 const int64_t* boff, int64_t nbatches, float lr_b, float reg_b,
                                 float* scratch, cudaStream_t st);

// ---- Hogwild sweeps (hog_kernels.cu) -----------------------------------------
cudaError_t launch_hog_factor(const KView& v, int64_t tile_mul, int64_t tile_add,
                              float lr_a, float reg_a, int blocks_per_sm, int atomic_update,
                              cudaStream_t st);
size_t hog_core_scratch_bytes(const KView& v, int blocks_per_sm);
// Large ranks (N = 3, J = R in {64, 128}): mode-serial tcgen05 sweeps
// (tc_big_kernels.cu).  Scratch: B operand images (+ core partials).
bool big_supported(const KView& v);
size_t big_scratch_bytes(const KView& v, const int32_t* dims, bool core);
cudaError_t launch_big_factor(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                              float lr, float reg, int atomic_update, float* scratch,
                              size_t scratch_bytes, cudaStream_t st);
cudaError_t launch_big_core(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                            float* grad, float* scratch, size_t scratch_bytes, cudaStream_t st);
// CCache::refresh for every mode (decomposition.cpp:89-107): out[n][i][r] =
// sum_j A_n[i][j] B_n[j][r], j ascending, fp32 multiply then add (no FMA).
cudaError_t launch_ccache(const KView& v, const int32_t* dims, float* const* out,
                          cudaStream_t st, int only_mode = -1);
cudaError_t launch_hog_core(const KView& v, int64_t tile_mul, int64_t tile_add,
                            float* grad, int blocks_per_sm, float* scratch,
                            size_t scratch_bytes, cudaStream_t st);
// Builds the shuffled SoA copy (the tiler).  perm == nullptr: random order
// from `seed`; otherwise entries are laid out in perm order.
// Delta-coded uploads (ftkcu_tensor_upload_delta_async): chunks [c0, c1) of
// kDeltaChunk entries decoded into the SoA columns; with `scatter` (order 3)
// each record also goes straight to its single-cell tile-stream position
// (the build_shuffled(seed) layout), finished by finish_scatter_stream.
constexpr int kDeltaChunk = 4096;
cudaError_t prepare_scatter_stream(DevTensor& t);
cudaError_t launch_delta_decode(DevTensor& t, const uint8_t* deltas, const uint64_t* restarts,
                                int width, int64_t c0, int64_t c1, bool scatter, uint64_t seed,
                                int* bad, cudaStream_t st);
cudaError_t finish_scatter_stream(DevTensor& t, cudaStream_t st);
cudaError_t build_shuffled(DevTensor& t, const int64_t* d_perm, uint64_t seed,
                           void* scratch, size_t scratch_bytes,
                           cudaStream_t st);
// physical tile of range position t under the per-epoch affine permutation
__host__ __device__ inline int64_t stream_tile(const KView& v, int64_t t, int64_t mul,
                                               int64_t add) {
  return v.tile_base + (t * mul + add) % v.ntiles;
}
size_t shuffle_scratch_bytes(int64_t nnz);
constexpr int kHogTile = 128;  // nonzeros per Hogwild tile

// ---- tensor-core sweeps (tc_kernels.cu) -------------------------------------
bool tc_supported(const KView& v);
cudaError_t launch_tc_factor(const KView& v, int64_t tile_mul, int64_t tile_add,
                             float lr_a, float reg_a, int precision, int atomic_update,
                             cudaStream_t st);
cudaError_t launch_tc_core(const KView& v, int64_t tile_mul, int64_t tile_add,
                           float* grad, int precision, float* scratch,
                           size_t scratch_bytes, cudaStream_t st);

// ---- warp-specialized tensor-core sweeps, N = 3, J = R = 32 (tc_ws_kernels.cu)
bool ws_supported(const KView& v);
// J = R = 16 at order 3..6 (tc_wsg_kernels.cu): warp-specialised factor
// (tf32, Hogwild accumulate) and core (fp16 copy of A) sweeps.
bool wsg_supported(const KView& v);
bool wsf32_supported(const KView& v);  // N = 3, J = R = 32 on 16 epilogue warps
size_t wsg_core_scratch_bytes(const KView& v, const int32_t* dims);
cudaError_t launch_wsg_factor(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                              float lr, float reg, cudaStream_t st);
cudaError_t launch_wsg_core(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                            float* grad, float* scratch, size_t scratch_bytes, cudaStream_t st);
// Core sweep scratch: per-CTA gradients + the RN-rounded tf32 copy of A.
size_t ws_core_scratch_bytes(const KView& v, const int32_t* dims);
// epi_warps: 8 or 16 epilogue warps (tf32 single pass only)
cudaError_t launch_ws_factor(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                             float lr, float reg, int precision, int atomic_update,
                             int epi_warps, cudaStream_t st);
// core16: the single-pass sweep gathers an fp16 copy of A (ws_core16_kernel);
// 2 = the same with two epilogue warp groups taking alternate tiles; 0 = tf32
// rows copied into TMEM (ws_core_kernel).  3xtf32 and the storage
// scheme have their own kernels.
cudaError_t launch_ws_core(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                           float* grad, int precision, int core16, float* scratch,
                           size_t scratch_bytes, cudaStream_t st);

// DSGD ring epoch (dsgd.py, ring schedule): one persistent factor sweep over
// all of this rank's cells in order.  Mode-3 blocks circulate as tokens (2P
// blocks, each rank holds two): the epilogue warp that completes a cell's
// count copies the cell's mode-3 block into the left neighbour's factor
// matrices and raises the neighbour's arrival flag; at a round's end every
// CTA copies a slice of the round's mode-2 block the same way.  A cell's
// gathers start once its own arrival flags carry this epoch.
struct RingDev {
  int ncell = 0;             // 0: not a ring epoch
  int parts = 0;             // P (cells per round: 2P)
  int emulate = 0;           // no peers: posts go to local scratch, no waits
  unsigned epoch = 0;        // flag generation of this epoch (>= 1)
  const int64_t* cell_tile = nullptr;  // [ncell + 1] physical tile offsets
  const int64_t* cell_perm = nullptr;  // [ncell][2] affine tile permutation
  const int4* cell_io = nullptr;       // [ncell] {wait flag, wait flag, post, post}, -1 = none
  const int4* posts = nullptr;         // {mode, row0, nrows, peer flag}
  const int* final_waits = nullptr;    // flags CTA 0 waits for before it exits
  int nfinal = 0;
  unsigned* done = nullptr;            // [ncell] warp completion counts (zeroed per epoch)
  unsigned* copied = nullptr;          // [P] round-end mode-2 copy counts (zeroed per epoch)
  unsigned* flags = nullptr;           // this rank's arrival flags
  unsigned* peer_flags = nullptr;      // the left neighbour's
  float* peer_a[kMaxOrder] = {};       // the left neighbour's factor matrices
  unsigned* err = nullptr;             // the first wait that timed out (0: none)
  long long timeout_cycles = 4ll << 30;  // ~2 s
};
cudaError_t launch_ws_factor_ring(const KView& v, const int32_t* dims, const RingDev& ring,
                                  float lr, float reg, cudaStream_t st);

// Measurement: the headline factor sweep's RED write-back alone (roofline
// ceiling at L2-resident shapes); dst_dev: device array of order pointers.
cudaError_t launch_ws_writeback(const KView& v, const int32_t* dims, int64_t mul, int64_t add,
                                float* const* dst_dev, cudaStream_t st);

// ---- evaluation (eval_kernels.cu) ---------------------------------------------
// out3 = {sum sq, sum abs, reg}; exact = reference slab order.
cudaError_t run_eval(const DevModel& m, const DevTensor& t, int workers,
                     double reg_a, double reg_b, bool exact, double* out3,
                     void* scratch, size_t scratch_bytes, cudaStream_t st);
size_t eval_scratch_bytes(const DevModel& m, const DevTensor& t, int workers);

int num_sms();

}  // namespace ftkcu
