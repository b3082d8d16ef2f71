/*
 * ftkcu.h — the C-ABI of the B200-native FastTuckerPlus engine.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (/root/reference/proj) has no FFI: its boundary is the C++ header API
 * the proj/include/ftk headers, linked statically as ftkcore.  The engine keeps
 * that C++ API (the include/ftk headers, implemented in
 * paper_2404_10087_b200/host/ on top of this header) and moves the device
 * boundary *inside* ftk::epoch_plus / ftk::train / ftk::loss /
 * ftk::evaluate.  Every entry point below names the reference interface it
 * replaces.
 *
 * Conventions (mirroring the reference's):
 *   - Every call returns FTKCU_OK (0) or a non-zero status; the message is
 *     ftkcu_last_error(session).  The C++ shim turns non-zero into
 *     ftk::Error(message), which is how the reference reports every failure
 *     (common.hpp:23-32).
 *   - Host buffers are caller-owned and only read/written during the call.
 *     Device buffers are owned by the session.
 *   - A session is bound to one CUDA device and must be driven by one host
 *     thread at a time (the reference's Model& is likewise not to be touched
 *     concurrently, decomposition.hpp Hogwild contract).
 *   - Plain pointers and sizes only; no torch or CUDA types cross the ABI.
 */
#ifndef FTKCU_H_
#define FTKCU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FTKCU_ABI_VERSION 1

/* status codes */
#define FTKCU_OK 0
#define FTKCU_ERR_ARG 1      /* invalid argument (ftk::require failure)     */
#define FTKCU_ERR_CUDA 2     /* CUDA runtime / driver error                 */
#define FTKCU_ERR_STATE 3    /* call out of order (no tensor / no model)    */
#define FTKCU_ERR_NCCL 4     /* collective failure                          */
#define FTKCU_ERR_EMPTY 5    /* apply_core_update: empty tensor             */

/* execution modes for the two SGD sweeps */
#define FTKCU_MODE_DETERMINISTIC 0 /* single stream, reference fp32 order,
                                      bit-identical to workers == 1        */
#define FTKCU_MODE_HOGWILD 1       /* all SMs, lock-free row updates        */

/* contraction precision for FTKCU_MODE_HOGWILD (ftkcu_set_option) */
#define FTKCU_PREC_FP32 0   /* FFMA, no tensor cores                        */
#define FTKCU_PREC_TF32 1   /* single-pass tensor cores, fp32 accumulate:   */
                            /* 10-bit-mantissa operands rounded to nearest; */
                            /* kind::tf32, except the N=3 J=R=32 core sweep */
                            /* (kind::f16 on an fp16 copy of A, "core16")   */
#define FTKCU_PREC_3XTF32 2 /* tcgen05 split-tf32 (hi*hi + hi*lo + lo*hi)   */

/* evaluation reduction order */
#define FTKCU_EVAL_EXACT 0 /* reference slab order, bit-identical fp64     */
#define FTKCU_EVAL_FAST 1  /* tree reduction, fp64                          */

/* sweep kernels, as reported by get_option "last_factor_kernel" /
 * "last_core_kernel" (which kernel the last factor / core phase ran) */
#define FTKCU_K_NONE 0
#define FTKCU_K_DET 1    /* det_factor_kernel / det_core_kernel (parity mode)  */
#define FTKCU_K_WS 2     /* ws_factor_kernel / ws_core_kernel (N=3, J=R=32)    */
#define FTKCU_K_WS16 3   /* ws_core16_kernel (fp16 operand tile)               */
#define FTKCU_K_WS_CC 4  /* ws_core_cc_kernel (storage scheme)                 */
#define FTKCU_K_WSF 5    /* wsf_factor_kernel (16 epilogue warps)              */
#define FTKCU_K_WSG 6    /* wsg_factor_kernel / wsg_core_kernel (J=R<=16)      */
#define FTKCU_K_BIG 7    /* big*_factor / big16*_core (J=R in {64,128})        */
#define FTKCU_K_TC 8     /* tc_factor_kernel / tc_core_kernel (synchronous)    */
#define FTKCU_K_HOG 9    /* hog_factor_kernel / hog_core_kernel (fp32 FFMA)    */
#define FTKCU_K_WS3 10   /* ws_factor3_kernel (N=3, J=R=32, 3xtf32)            */

typedef struct ftkcu_session ftkcu_session;

/* ---- session --------------------------------------------------------- */

/* Creates a session on CUDA device `device`.  No reference counterpart
 * (the reference's "session" is the calling thread). */
int ftkcu_session_create(int device, ftkcu_session** out);
void ftkcu_session_destroy(ftkcu_session* s);
/* Last error message of `s`, or of the calling thread's last failed
 * ftkcu_session_create when s == NULL.  Never NULL. */
const char* ftkcu_last_error(const ftkcu_session* s);
int ftkcu_abi_version(void);

/* Tunables: "precision" (FTKCU_PREC_*), "eval" (FTKCU_EVAL_*),
 * "hog_blocks_per_sm", "hog_update" (1 = atomic row accumulate, 0 = overwrite),
 * "tc_ws" (warp-specialised tcgen05 sweeps), "max_ctas" (factor-sweep grid
 * cap, 0 = one CTA per SM), "graphs" (CUDA-graph replay of the DSGD
 * stratum loop, default 1), "staleness" (whole-tensor factor sweeps cap the
 * grid so at most this many nonzeros per row of the smallest mode are in
 * flight; default 32, 0 = off), "global_nnz" (|Omega|
 * over all ranks for the multi-GPU core update), "store_c" (core phase:
 * storage scheme, C rows from a C cache), "core16" (default 1; 0 keeps the
 * N=3 J=R=32 tf32 core sweep on kind::tf32), "shuffle_seed", "verbose".
 * get_option also reads "launches", "stream" (cudaStream_t), "num_sms",
 * "last_factor_kernel" and "last_core_kernel" (FTKCU_K_*).
 * Unknown keys are FTKCU_ERR_ARG. */
int ftkcu_set_option(ftkcu_session* s, const char* key, int64_t value);
int ftkcu_get_option(ftkcu_session* s, const char* key, int64_t* value);

/* ---- data ------------------------------------------------------------ */

/* Uploads a COO tensor into slot `slot` (0 = train, 1 = test, ...).
 * idx_rowmajor is nnz x order int32, 0-based; values fp32.  Replaces the
 * device-side role of ftk::SparseTensor (sparse_tensor.hpp:14-33); the host
 * loader ftk::load_coo (sparse_tensor.hpp:38) stays on the host.  The engine
 * keeps the entries in storage order (SoA, one int32 column per mode) for
 * the deterministic sweeps and builds a shuffled, tiled copy lazily for the
 * Hogwild sweeps. */
int ftkcu_tensor_upload(ftkcu_session* s, int slot, int order,
                        const int32_t* dims, int64_t nnz,
                        const int32_t* idx_rowmajor, const float* values);
/* Same as ftkcu_tensor_upload, asynchronous: the host-to-device copy and
 * the layout transpose run on the session's copy stream and overlap work
 * already enqueued on other slots.  `idx_rowmajor` / `values` (pinned host
 * memory for a true overlap) must stay valid until the slot's next use,
 * which waits for the copy and reports an out-of-range index then.  No
 * reference counterpart (engine addition for pipelined epochs). */
int ftkcu_tensor_upload_async(ftkcu_session* s, int slot, int order, const int32_t* dims,
                              int64_t nnz, const int32_t* idx_rowmajor, const float* values);
/* Packed-key COO for host-to-device streaming: nonzero e's mode-n index sits
 * in bits [off_n, off_n + w_n) of its key, w_n = bit width of dims[n] - 1
 * (at least 1), off_0 = 0, off_n = off_{n-1} + w_{n-1}; needs sum w_n <= 64.
 * A key is stored as its low 32 bits (`lo`, uint32 per nonzero) and its high
 * bits (`hi`: none if sum w_n <= 32, uint16 if <= 48, else uint32; see
 * ftkcu_key_layout).  Netflix shape: 19 + 15 + 12 = 46 bits, 6 bytes per
 * nonzero on the link (10 with the value) instead of 16.  ftkcu_pack_keys
 * builds the keys on the host (once, e.g. when the tensor is loaded) and
 * returns FTKCU_ERR_ARG if the widths do not fit or an index is out of
 * range.  ftkcu_tensor_upload_packed_async is ftkcu_tensor_upload_async for
 * packed keys (unpacked on the copy stream).  No reference counterpart
 * (engine addition for pipelined epochs). */
int ftkcu_key_layout(int order, const int32_t* dims, int* hi_bytes);
int ftkcu_pack_keys(int order, const int32_t* dims, int64_t nnz, const int32_t* idx_rowmajor,
                    uint32_t* lo, void* hi);
int ftkcu_tensor_upload_packed_async(ftkcu_session* s, int slot, int order, const int32_t* dims,
                                     int64_t nnz, const uint32_t* lo, const void* hi,
                                     const float* values);
/* Delta-coded COO for host-to-device streaming: nonzeros sorted by their
 * mixed-radix key ((i0 d1 + i1) d2 + i2 ...), in chunks of 4096; chunk c
 * stores its first key in restarts[c] and every later entry the difference
 * to its predecessor in `width` little-endian bytes (the chunk's first delta
 * slot holds 0).  Netflix shape: 3 bytes per nonzero (7 with the value)
 * instead of 6 for packed keys.  ftkcu_pack_delta sorts and encodes on the
 * host (once per tensor, like a file format): values_out receives the values
 * in the sorted order, *width the byte width; it fails with FTKCU_ERR_ARG if
 * deltas_cap < width * nnz (call again with a larger buffer), an index is
 * out of range or prod(dims) > 2^53.  ftkcu_tensor_upload_delta_async is
 * ftkcu_tensor_upload_async for this format (one block scan per chunk on the
 * copy stream).  No reference counterpart (engine addition). */
int ftkcu_pack_delta(int order, const int32_t* dims, int64_t nnz, const int32_t* idx_rowmajor,
                     const float* values, uint8_t* deltas, int64_t deltas_cap,
                     uint64_t* restarts, float* values_out, int* width);
int ftkcu_tensor_upload_delta_async(ftkcu_session* s, int slot, int order, const int32_t* dims,
                                    int64_t nnz, const uint8_t* deltas, int width,
                                    const uint64_t* restarts, const float* values);
int ftkcu_tensor_release(ftkcu_session* s, int slot);
int64_t ftkcu_tensor_nnz(ftkcu_session* s, int slot);

/* Uploads / downloads the model: A[n] is dims[n] x ranks[n], B[n] is
 * ranks[n] x R, fp32 row-major (ftk::Model, model.hpp:31-48). */
int ftkcu_model_upload(ftkcu_session* s, int order, const int32_t* dims,
                       const int32_t* ranks, int32_t R,
                       const float* const* A, const float* const* B);
int ftkcu_model_download(ftkcu_session* s, float* const* A, float* const* B);
/* The same copies enqueued without a host synchronisation (to_device = 1:
 * upload into the resident model of the same shape, on the session stream;
 * 0: download -- a device snapshot on the session stream, then the
 * device-to-host copy on a read-back stream, so later epochs do not wait for
 * the PCIe transfer).  Host buffers must be pinned and stay valid until
 * ftkcu_stream_sync returns.  No reference counterpart. */
int ftkcu_model_copy_async(ftkcu_session* s, int to_device, float* const* A, float* const* B);

/* ---- the hot path ------------------------------------------------------ */

/* Factor phase of ftk::epoch_plus (decomposition.cpp:637-661, Eq. 14,
 * Alg. 4).  perm: the EpochPlan::global permutation (nnz int64 entry
 * positions, batches of M in order) or NULL in Hogwild mode to use the
 * engine's device tile order keyed by `seed`.  In deterministic mode perm is
 * required and the result is bit-identical to the reference with
 * workers == 1.  ms (optional) receives the device time of the sweep. */
int ftkcu_factor_phase(ftkcu_session* s, int slot, const int64_t* perm,
                       int32_t M, float lr_a, float reg_a, int mode,
                       uint64_t seed, double* ms);

/* Core phase of ftk::epoch_plus (decomposition.cpp:663-703, Eq. 15,
 * Alg. 5): accumulate Grad(B) = sum (x - xhat) A_psi^T D over the tensor,
 * then B += lr_b (Grad/|Omega| - reg_b B) (apply_core_update,
 * decomposition.cpp:576-589).  Same perm / mode / seed rules as above.
 * grad_out (optional, sum_n J_n*R floats) receives the merged gradient. */
int ftkcu_core_phase(ftkcu_session* s, int slot, const int64_t* perm,
                     int32_t M, float lr_b, float reg_b, int mode,
                     uint64_t seed, float* grad_out, double* ms);

/* ---- FastTucker baseline --------------------------
 * ftk::epoch_fasttucker (decomposition.cpp:707-770) one block at a time, in
 * the reference's workers == 1 arithmetic (bit-identical models).
 *
 * Factor block of `mode`: perm = EpochPlan::per_bucket(fixed-mode index)
 * positions (nnz entries, plan order), bucket_off = the nbuckets + 1 offsets
 * of its buckets in perm (bucket_off[0] = 0, bucket_off[nbuckets] = nnz);
 * batches are cut from each bucket in M-entry chunks.  Replaces the
 * parallel_for over update_factor_fasttucker_impl (decomposition.cpp:729-742,
 * 316-371).  Core block of `mode`: perm = the global plan;
 * update_core_fasttucker_impl per batch (:752-766, 373-417), B^(mode)
 * updated in place after every batch.  schedule FTKCU_MODE_DETERMINISTIC:
 * the workers == 1 chain (bit-identical); FTKCU_MODE_HOGWILD: the workers > 1
 * schedule (batches spread over CTAs, B steps added atomically).  The
 * factor block has no such choice: its buckets are independent, so it is
 * parallel and bit-identical at once.  ms: device time of the block. */
int ftkcu_fasttucker_factor(ftkcu_session* s, int slot, int mode, const int64_t* perm,
                            const int64_t* bucket_off, int64_t nbuckets, int32_t M, float lr_a,
                            float reg_a, double* ms);
int ftkcu_fasttucker_core(ftkcu_session* s, int slot, int mode, const int64_t* perm, int32_t M,
                          float lr_b, float reg_b, int schedule, double* ms);

/* ---- FasterTucker baseline ------------------------
 * ftk::epoch_fastertucker (decomposition.cpp:772-843) one block at a time,
 * bit-identical to the reference's workers == 1 epoch.  The C cache
 * (CCache, decomposition.cpp:74-107: C_n = A_n B_n, dims[n] x R fp32) lives
 * on the device next to the model: upload it before the first block (the
 * reference requires cache.ready()), download it to keep a host copy.  Each
 * block ends with the refresh of its mode's cache rows (the block barrier,
 * :810, :837), inside the timed region as in the reference.
 *
 * Factor block: perm = EpochPlan::per_bucket(complement index of `mode`)
 * positions regrouped by mode-`mode` row, plan order kept inside a row;
 * row_off = the nrows + 1 group offsets.  (A step touches only its own row,
 * so rows are independent chains.)  Core block: perm = that plan for the
 * core seed, batch_off = its nbatches + 1 batch offsets (batches never cross
 * a bucket).  Core block supports J <= 128.  schedule
 * FTKCU_MODE_DETERMINISTIC: the workers == 1 recurrence, bit-identical;
 * FTKCU_MODE_HOGWILD (workers > 1): the block's linear B recurrence summed in
 * closed form over all batches in parallel (same mathematics, fp32 sums in
 * another order; falls back to the recurrence when J x R is too large). */
int ftkcu_ccache_upload(ftkcu_session* s, const float* const* C);
int ftkcu_ccache_download(ftkcu_session* s, float* const* C);
int ftkcu_fastertucker_factor(ftkcu_session* s, int slot, int mode, const int64_t* perm,
                              const int64_t* row_off, int64_t nrows, float lr_a, float reg_a,
                              double* ms);
int ftkcu_fastertucker_core(ftkcu_session* s, int slot, int mode, const int64_t* perm,
                            const int64_t* batch_off, int64_t nbatches, float lr_b, float reg_b,
                            int schedule, double* ms);

/* DSGD strata support.  Declares that the uploaded entries are sorted into
 * cells: entries [cell_offsets[c], cell_offsets[c+1]) form cell c.  The
 * Hogwild stream then shuffles and tiles every cell separately. */
int ftkcu_tensor_set_cells(ftkcu_session* s, int slot, const int64_t* cell_offsets,
                           int ncells);
/* Hogwild factor sweep over one cell only (one DSGD stratum on this rank). */
int ftkcu_factor_phase_cell(ftkcu_session* s, int slot, int cell, float lr_a,
                            float reg_a, uint64_t seed, double* ms);

/* fp64 metrics of the resident model on tensor `slot`
 * (ftk::loss / ftk::evaluate, evaluation.cpp:36-72, predict_element
 * model.cpp:70-92).  out[0] = sum (x - xhat)^2, out[1] = sum |x - xhat|,
 * out[2] = reg_a sum_n |A_n|^2 + reg_b sum_n |B_n|^2, each reduced in the
 * reference's slab order for `workers` when the "eval" option is EXACT. */
int ftkcu_eval(ftkcu_session* s, int slot, int workers, double reg_a,
               double reg_b, double* out3);

/* One batch through the device pipeline (parity probe for the reference's
 * per-batch API decomposition.hpp:86-124).  rows: m_eff entry positions,
 * batch capacity cap.  Outputs (all optional): C, D [order][cap][R];
 * U, A_new [order][cap][Jmax]; xhat/resid factor side and C side [cap];
 * G [order][Jmax][R].  Mutates the resident A exactly like
 * update_factors_plus. */
int ftkcu_batch_probe(ftkcu_session* s, int slot, const int64_t* rows,
                      int m_eff, int cap, float lr_a, float reg_a, float* C,
                      float* D, float* U, float* xhat_f, float* resid_f,
                      float* xhat_c, float* resid_c, float* A_new, float* G);

/* ---- multi-GPU (DSGD) --------------------------------------------------- */

/* 128-byte NCCL unique id for rank 0 to broadcast out of band. */
int ftkcu_comm_unique_id(uint8_t* id128);
/* Joins an NCCL communicator (one rank per session / GPU). */
int ftkcu_comm_init(ftkcu_session* s, const uint8_t* id128, int rank,
                    int world);
/* In-place sum all-reduce of a device-resident core gradient, exposed for
 * tests; ftkcu_core_phase calls it internally once a communicator is set. */
int ftkcu_comm_allreduce_grad(ftkcu_session* s);
/* DSGD block rotation: send factor rows [send_row0, +send_nrows) of mode
 * `mode` to rank dst while receiving rows [recv_row0, +recv_nrows) from src
 * (one NCCL group on the session stream, no host round trip). */
int ftkcu_comm_sendrecv_rows(ftkcu_session* s, int mode, int64_t send_row0,
                             int64_t send_nrows, int dst, int64_t recv_row0,
                             int64_t recv_nrows, int src);
/* Every rank r broadcasts its rows [row_off[r], row_off[r+1]) of `mode`
 * (all-gather of the owned blocks after a DSGD factor sweep). */
int ftkcu_comm_bcast_rows(ftkcu_session* s, int mode, const int64_t* row_off,
                          int nblocks);
/* One DSGD factor phase of this rank (dsgd.DsgdTrainer.factor_phase): for
 * stratum (s, t), s, t < parts, sweep local cell s*parts+t with tile
 * permutation seed cell_seeds[s*parts+t], then ring-shift the mode-3 block
 * (row_off3, parts+1 offsets) to rank-1 / from rank+1; after each s-round
 * the mode-2 block (row_off2); finally all-gather the mode-2/3 blocks.  The
 * whole loop is enqueued on the session stream without a host sync and, with
 * option "graphs" (default 1), captured once as a CUDA graph and replayed.
 * Needs ftkcu_tensor_set_cells with parts*parts cells and, for parts > 1, a
 * communicator (world 1 = one rank emulating `parts`, shifts to itself).
 * No reference counterpart: the reference is single-host. */
int ftkcu_dsgd_factor_epoch(ftkcu_session* s, int slot, int parts, const int64_t* row_off2,
                            const int64_t* row_off3, const uint64_t* cell_seeds, float lr_a,
                            float reg_a, double* ms);
/* DSGD ring epochs (dsgd.py ring schedule; no reference counterpart: the
 * reference is single-host).  Mode 3 is cut into 2*parts blocks that
 * circulate as tokens (rank g starts an epoch holding blocks 2g, 2g+1 and
 * mode-2 block g); cell s*2*parts+i of rank g holds its nonzeros of mode-2
 * block (g+s)%parts and mode-3 block (2g+i)%(2*parts).  One persistent
 * factor sweep (ws_factor_kernel) walks all cells: after the last CTA
 * finishes a cell it copies the cell's mode-3 block (and at a round's end
 * the mode-2 block) into the left neighbour's (rank g-1) factor matrices
 * over peer memory and raises the neighbour's arrival flag; a cell's gathers
 * wait only for its own flags.  No stratum barrier, no host sync.
 *
 * ftkcu_ring_export writes this session's peer descriptor (factor matrices
 * and flag array: device pointers + CUDA IPC handles) into blob
 * (FTKCU_RING_BLOB_BYTES); ftkcu_ring_connect maps the LEFT neighbour's
 * (same process: its pointers; another process: cudaIpcOpenMemHandle) and
 * clears this rank's flags -- every rank connects before any ring epoch.
 * ftkcu_ring_emulate instead points the posts at local scratch and skips the
 * waits (one GPU timing one rank's share).  Both take the training slot
 * (uploaded, cells set) and allocate everything an epoch uses, so no
 * allocation falls between two ranks' launches; model and tensor must stay
 * as uploaded between connect and the epochs.  N = 3, J = R = 32, tf32. */
#define FTKCU_RING_BLOB_BYTES 512
int ftkcu_ring_export(ftkcu_session* s, uint8_t* blob, int cap);
int ftkcu_ring_connect(ftkcu_session* s, int slot, const uint8_t* left_blob, int len);
int ftkcu_ring_emulate(ftkcu_session* s, int slot);
/* One ring factor phase of rank `rank` over `parts` ranks: row_off2 has
 * parts+1 offsets, row_off3 2*parts+1, cell_seeds 2*parts*parts tile
 * permutation seeds.  With a communicator of size parts the epoch ends with
 * the all-gather of the mode-2/3 blocks (as ftkcu_dsgd_factor_epoch). */
int ftkcu_ring_factor_epoch(ftkcu_session* s, int slot, int parts, int rank,
                            const int64_t* row_off2, const int64_t* row_off3,
                            const uint64_t* cell_seeds, float lr_a, float reg_a, double* ms);
/* Synchronises the session stream; *timed_out != 0 if a ring wait gave up
 * (a neighbour never posted: the epoch's result is invalid): 0x10000 | the
 * flag id of the first block wait that gave up, 0x20000 | the round of a
 * round-end copy that did.  Option "ring_timeout_ms" sets the limit. */
int ftkcu_ring_status(ftkcu_session* s, int* timed_out);
/* Test introspection: the first n arrival flags and cell counters
 * (flag ids: mode-3 block x in round r = r*2P + x; mode-2 block y in round
 * r = (P+1)*2P + r*P + y; rounds 0..P). */
int ftkcu_ring_debug(ftkcu_session* s, uint32_t* flags, uint32_t* done, int n);
/* Sum all-reduce of host fp64 values (metrics partials). */
int ftkcu_comm_allreduce_f64(ftkcu_session* s, double* host_inout, int n);
/* Waits for all work queued on the session stream. */
// Measurement only (no reference counterpart): the J = R = 32 factor
// sweep's RED.v4 write-back alone over slot's Hogwild tile stream, into
// scratch rows (the model is untouched); *ms = device time.  bench.py uses it
// as the roofline ceiling of the factor sweep at L2-resident shapes.
int ftkcu_writeback_ceiling(ftkcu_session* s, int slot, uint64_t seed, double* ms);
int ftkcu_stream_sync(ftkcu_session* s);

#ifdef __cplusplus
}
#endif

#endif /* FTKCU_H_ */
