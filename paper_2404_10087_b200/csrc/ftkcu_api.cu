// The C-ABI (include/ftkcu.h): session, data movement and dispatch of the
// device sweeps.  Host-side C++ only; kernels live in *_kernels.cu.
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "engine.cuh"

using namespace ftkcu;

struct ftkcu_session {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // asynchronous tensor uploads
  cudaStream_t dec_stream = nullptr;   // delta-coded uploads: decode + stream scatter
  cudaEvent_t dec_ev[8] = {};
  // enqueued model read-back (ftkcu_model_copy_async to host): a device
  // snapshot on the session stream, the device-to-host copy on its own stream
  cudaStream_t rb_stream = nullptr;
  cudaEvent_t rb_snap = nullptr, rb_done = nullptr;
  bool rb_pending = false;
  std::vector<float*> rb_buf;
  size_t rb_floats = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // fp16 range flag of the core16 operand copies (KView::f16_range): mapped
  // pinned memory, so the host reads it without a synchronisation
  volatile int* f16_range_h = nullptr;
  int* f16_range_d = nullptr;
  std::string err;
  DevTensor slots[8];
  int last_slot = -1;  // slot of the most recent phase / evaluation
  DevModel model;
  bool have_model = false;
  float* grad = nullptr;
  size_t grad_len = 0;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  int64_t* d_perm = nullptr;
  size_t perm_cap = 0;
  int64_t* d_boff = nullptr;  // FastTucker bucket offsets
  size_t boff_cap = 0;
  int64_t opt_precision = FTKCU_PREC_FP32;
  int64_t opt_eval = FTKCU_EVAL_EXACT;
  int64_t opt_hog_bps = 2;
  int64_t opt_hog_update = 1;  // 1: atomic accumulate, 0: overwrite (reference rule)
  int64_t opt_tc_ws = 1;  // warp-specialized tcgen05 sweeps where supported
  int64_t opt_store_c = 0;  // core sweeps: storage scheme (C-row cache) instead of calculation
  int64_t opt_core16 = 2;   // WS core sweep (tf32 precision): fp16 copy of A; 2 = two epilogue groups (default), 1 = one, 0 = tf32 rows
  int64_t opt_factor_warps = 8;  // N=3 J=R=32 factor sweep (ws_factor_kernel): 8 or 16 epilogue warps
  int64_t opt_verbose = 0;
  int64_t opt_shuffle_seed = 0x5eed5eedLL;
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  int64_t global_nnz = 0;  // |Omega| across ranks for the core update (DSGD)
  int64_t opt_max_ctas = 0;  // sweep grid cap (0 = one CTA per SM)
  int64_t opt_ring_timeout_ms = 0;  // ring waits give up after this (0: ~2 s)
  // Hogwild stream in last-mode runs: 0 off (default), 1 on, -1 auto (when
  // the factor sweep is the merging J = R = 32 one).  Off by default: on the
  // Netflix-shaped uniform workload it buys 6% of the factor sweep (8.8 ->
  // 8.3 ms) but moves the test RMSE 1.5e-3 further from the reference's
  // (16 updates of a row computed from one read per chunk), and the per-upload
  // sort costs the e2e loop ~5 ms per epoch
  int64_t opt_runs = 0;
  int64_t opt_cell_order = 0;
  int64_t opt_eager_stream = 1;  // delta-coded uploads scatter the tile stream while decoding
  // delta-coded uploads: 0 decode beside the running epochs (decode stream,
  // part by part as the bytes land), 1 decode at first use on the session
  // stream (serial with the epochs; measured slower in the e2e loop, 4.4e9 vs
  // 5.1e9 nnz/s)
  int64_t opt_delta_decode = 0;  // 1: ftkcu_tensor_set_cells keeps each cell's uploaded order
  int64_t opt_window = 0;  // headline factor sweep read-to-write window in tiles (0 = ring depth)
  // Whole-tensor factor sweeps: cap the grid so that at most this many
  // nonzeros per row of the smallest mode are in flight (0 = off).  See
  // dsgd.grid_cap for the measurement behind the default.
  int64_t opt_staleness = 32;
  int64_t opt_graphs = 1;  // capture the DSGD stratum loop in a CUDA graph
  int64_t opt_dsgd_shift = 1;  // 0: skip the DSGD ring shifts (cost breakdown only)
  // DSGD epoch: per-cell tile permutations (device + pinned host staging)
  // and the captured stratum loop, re-captured when its key changes.
  int64_t* d_cellperm = nullptr;
  int64_t* h_cellperm = nullptr;
  size_t cellperm_cap = 0;
  cudaGraphExec_t dsgd_exec = nullptr;
  std::vector<int64_t> dsgd_key;
  int64_t dsgd_launches = 0;
  // DSGD ring (ftkcu_ring_*): arrival flags, cell counters, the left
  // neighbour's buffers (or local scratch when emulating), per-epoch tables
  unsigned* ring_flags = nullptr;  // [kRingFlags]
  unsigned* ring_done = nullptr;   // [kRingFlags] cell counters, then [kRingFlags] copy counts
  unsigned* ring_err = nullptr;
  float* ring_peer_a[3] = {};
  unsigned* ring_peer_flags = nullptr;
  void* ring_ipc[4] = {};          // peers opened through CUDA IPC (closed on destroy)
  float* ring_emu_a[3] = {};
  unsigned* ring_emu_flags = nullptr;
  bool ring_ready = false, ring_emulate = false;
  float* ring_model_a[3] = {};     // factor matrices when connected (must not move)
  unsigned ring_epoch = 0;
  uint8_t* ring_tab = nullptr;     // device tables of the current epoch (kRingTabBytes)
  uint8_t* ring_tab_h = nullptr;   // pinned staging of the tables
  int64_t launches = 0;  // kernels launched by this session (for benches)
  // Which sweep kernel the last factor / core phase ran (FTKCU_K_*), so that
  // tests can assert the dispatch they mean to cover.
  int64_t last_factor_kernel = 0, last_core_kernel = 0;
};

namespace {

thread_local std::string g_create_err;

int fail(ftkcu_session* s, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (s)
    s->err = buf;
  else
    g_create_err = buf;
  return code;
}

#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      (void)cudaGetLastError(); /* clear a non-sticky launch error */         \
      return fail(s, FTKCU_ERR_CUDA, "%s: %s (%s:%d)", #call,                 \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                \
    }                                                                         \
  } while (0)

#define NK(call)                                                              \
  do {                                                                        \
    ncclResult_t r_ = (call);                                                 \
    if (r_ != ncclSuccess)                                                    \
      return fail(s, FTKCU_ERR_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

int bind(ftkcu_session* s) {
  if (!s) return fail(nullptr, FTKCU_ERR_ARG, "null session");
  CK(cudaSetDevice(s->device));
  return FTKCU_OK;
}

// An fp16 operand copy of A clamped an entry in an earlier core phase
// (core16 sweeps convert A with cvt.rn.satfinite): that phase's core gradient
// is wrong, so the next core phase, evaluation, stream sync or model download
// fails loudly instead of training on.  Cleared once reported; core16 = 0 runs
// the core sweep on tf32 rows, which have the fp32 range.
int check_f16_range(ftkcu_session* s) {
  if (!s->f16_range_h || !*s->f16_range_h) return FTKCU_OK;
  *s->f16_range_h = 0;
  return fail(s, FTKCU_ERR_ARG,
              "a factor entry exceeded the fp16 range (|a| > 65504 or not finite) in a core16 "
              "sweep's operand copy and was clamped; set option core16 = 0 (tf32 rows)");
}

int ensure_scratch(ftkcu_session* s, size_t bytes) {
  if (bytes <= s->scratch_bytes) return FTKCU_OK;
  if (s->scratch) CK(cudaFree(s->scratch));
  s->scratch = nullptr;
  s->scratch_bytes = 0;
  CK(cudaMalloc(&s->scratch, bytes));
  s->scratch_bytes = bytes;
  return FTKCU_OK;
}

// n plan entries, each a nonzero position in [0, bound) (bound = nnz)
int upload_perm(ftkcu_session* s, const int64_t* perm, int64_t n, int64_t bound) {
  // every plan entry indexes the tensor: an out-of-range one would be an
  // unchecked device read (the reference's plans come from iota + shuffle)
  for (int64_t i = 0; i < n; ++i)
    if ((uint64_t)perm[i] >= (uint64_t)bound)
      return fail(s, FTKCU_ERR_ARG, "plan entry %lld = %lld out of range [0, %lld)", (long long)i,
                  (long long)perm[i], (long long)bound);
  if ((size_t)n > s->perm_cap) {
    if (s->d_perm) CK(cudaFree(s->d_perm));
    s->d_perm = nullptr;
    CK(cudaMalloc(&s->d_perm, sizeof(int64_t) * (n > 0 ? n : 1)));
    s->perm_cap = n;
  }
  if (n > 0)
    CK(cudaMemcpyAsync(s->d_perm, perm, sizeof(int64_t) * n, cudaMemcpyHostToDevice,
                       s->stream));
  return FTKCU_OK;
}

void free_tensor(DevTensor& t) {
  for (int n = 0; n < kMaxOrder; ++n) {
    if (t.idx[n]) cudaFree(t.idx[n]);
    if (t.sidx[n]) cudaFree(t.sidx[n]);
  }
  if (t.vals) cudaFree(t.vals);
  if (t.svals) cudaFree(t.svals);
  if (t.tile_rows) cudaFree(t.tile_rows);
  if (t.staging) cudaFree(t.staging);
  if (t.rec16) cudaFree(t.rec16);
  if (t.runs_scratch) cudaFree(t.runs_scratch);
  if (t.d_bad) cudaFree(t.d_bad);
  if (t.ready) cudaEventDestroy(t.ready);
  if (t.used) cudaEventDestroy(t.used);
  t = DevTensor{};
}

void free_model(DevModel& m) {
  for (int n = 0; n < kMaxOrder; ++n) {
    if (m.a[n]) cudaFree(m.a[n]);
    if (m.b[n]) cudaFree(m.b[n]);
    if (m.cc[n]) cudaFree(m.cc[n]);
  }
  m = DevModel{};
}

// AoS -> SoA transpose with range check (SparseTensor::validate's index
// check, sparse_tensor.cpp:40-50; the O(nnz log nnz) duplicate check stays
// with the host loader).
struct SoAView {
  int order;
  int32_t dims[kMaxOrder];
  int32_t* col[kMaxOrder];
};
__global__ void aos_to_soa_kernel(const int32_t* __restrict__ aos, int64_t nnz, SoAView v,
                                  int* __restrict__ bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    for (int n = 0; n < v.order; ++n) {
      const int32_t x = aos[e * v.order + n];
      if (x < 0 || x >= v.dims[n]) atomicExch(bad, 1);
      v.col[n][e] = x;
    }
  }
}

// Packed keys (ftkcu_pack_keys layout) -> SoA columns, with the range check.
struct KeyLayout {
  int order;
  int hi_bytes;  // 0, 2 or 4
  int off[kMaxOrder];
  uint64_t mask[kMaxOrder];
};
__global__ void keys_to_soa_kernel(const uint32_t* __restrict__ lo, const void* __restrict__ hi,
                                   int64_t nnz, SoAView v, KeyLayout kl, int* __restrict__ bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = __ldcs(lo + e);
    if (kl.hi_bytes == 2)
      k |= (uint64_t)__ldcs(static_cast<const uint16_t*>(hi) + e) << 32;
    else if (kl.hi_bytes == 4)
      k |= (uint64_t)__ldcs(static_cast<const uint32_t*>(hi) + e) << 32;
    for (int n = 0; n < kl.order; ++n) {
      const int32_t x = (int32_t)((k >> kl.off[n]) & kl.mask[n]);
      if (x >= v.dims[n]) atomicExch(bad, 1);
      v.col[n][e] = x;
    }
  }
}

// Device-to-device copy on the SMs (the read-back snapshot): a copy-engine
// memcpy of the 64 MB model takes ~0.8 ms beside a concurrent upload on the
// copy engines, this ~0.05 ms.
__global__ void copy16_kernel(const float4* __restrict__ src, float4* __restrict__ dst, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
}

// A rows of the probe batch after the update (ftkcu_batch_probe A_new).
__global__ void gather_rows_kernel(KView v, const int64_t* __restrict__ rows, int m_eff,
                                   int cap, int jmax, float* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < v.order * m_eff * jmax;
       e += gridDim.x * blockDim.x) {
    const int n = e / (m_eff * jmax), rem = e - n * m_eff * jmax;
    const int m = rem / jmax, j = rem - m * jmax;
    if (j >= v.j[n]) continue;
    const int32_t i = v.idx[n][rows[m]];
    out[((size_t)n * cap + m) * jmax + j] = v.a[n][(size_t)i * v.j[n] + j];
  }
}

KView make_view(const ftkcu_session* s, const DevTensor& t, bool shuffled) {
  KView v{};
  const DevModel& m = s->model;
  v.order = m.order;
  v.r = m.r;
  for (int n = 0; n < m.order; ++n) {
    v.j[n] = m.ranks[n];
    v.a[n] = m.a[n];
    v.b[n] = m.b[n];
    v.idx[n] = shuffled ? t.sidx[n] : t.idx[n];
  }
  v.f16_range = s->f16_range_d;
  v.vals = shuffled ? t.svals : t.vals;
  v.nnz = t.nnz;
  v.tile_rows = shuffled ? t.tile_rows : nullptr;
  v.tile_base = 0;
  v.ntiles = shuffled ? t.stream_tiles : 0;
  return v;
}

// Completes an asynchronous upload before the slot's first use: the session
// stream waits for it, and the deferred index-range check runs.
int finish_upload(ftkcu_session* s, DevTensor& t) {
  if (!t.pending) return FTKCU_OK;
  t.pending = false;
  CK(cudaStreamWaitEvent(s->stream, t.ready, 0));
  if (t.delta_pending) {
    // the decode (and the tile-stream scatter) of a delta-coded upload, on
    // the session stream behind the epochs already enqueued: serial with
    // them instead of contending for L2 and HBM beside them
    t.delta_pending = false;
    const int64_t chunks = (t.nnz + kDeltaChunk - 1) / kDeltaChunk;
    const uint8_t* st = reinterpret_cast<const uint8_t*>(t.staging);
    CK(launch_delta_decode(t, st, reinterpret_cast<const uint64_t*>(st + t.delta_roff),
                           t.delta_width, 0, chunks, t.delta_scatter, t.delta_seed, t.d_bad,
                           s->stream));
    if (t.delta_scatter) CK(finish_scatter_stream(t, s->stream));
    CK(cudaEventRecord(t.ready, s->stream));
  }
  CK(cudaEventSynchronize(t.ready));
  int h_bad = 0;
  CK(cudaMemcpy(&h_bad, t.d_bad, sizeof(int), cudaMemcpyDeviceToHost));
  if (h_bad) {
    free_tensor(t);
    return fail(s, FTKCU_ERR_ARG, "index out of range in tensor upload");
  }
  return FTKCU_OK;
}

int check_ready(ftkcu_session* s, int slot) {
  if (slot < 0 || slot >= 8) return fail(s, FTKCU_ERR_ARG, "tensor slot %d out of range", slot);
  if (int rc = finish_upload(s, s->slots[slot])) return rc;
  if (!s->have_model) return fail(s, FTKCU_ERR_STATE, "no model uploaded");
  const DevTensor& t = s->slots[slot];
  if (!t.vals && t.nnz == 0 && t.order == 0)
    return fail(s, FTKCU_ERR_STATE, "no tensor in slot %d", slot);
  if (t.order != s->model.order)
    return fail(s, FTKCU_ERR_ARG, "model/tensor order mismatch");
  for (int n = 0; n < t.order; ++n)
    if (s->model.dims[n] < t.dims[n])
      return fail(s, FTKCU_ERR_ARG, "model dims too small for tensor");
  if (s->last_slot >= 0 && s->last_slot != slot) {
    DevTensor& p = s->slots[s->last_slot];
    if (!p.used) CK(cudaEventCreateWithFlags(&p.used, cudaEventDisableTiming));
    CK(cudaEventRecord(p.used, s->stream));
    p.used_rec = true;
  }
  s->last_slot = slot;
  return FTKCU_OK;
}

uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// Per-epoch affine tile permutation t -> (t * mul + add) mod T.
void tile_perm(uint64_t seed, int64_t ntiles, int64_t* mul, int64_t* add) {
  if (ntiles <= 1) {
    *mul = 1;
    *add = 0;
    return;
  }
  uint64_t h = splitmix(seed ^ 0x7469ull);
  int64_t m = (int64_t)(h % (uint64_t)ntiles);
  if (m == 0) m = 1;
  while (gcd64(m, ntiles) != 1) m = (m + 1) % ntiles == 0 ? 1 : m + 1;
  *mul = m;
  *add = (int64_t)(splitmix(h) % (uint64_t)ntiles);
}

// Whether the Hogwild stream is laid out in last-mode runs (option "runs";
// auto: when the factor sweep is the J = R = 32 one, whose epilogue merges
// a warp's 16 same-row updates of the last mode into one RED -- other sweeps
// would only see more same-row collisions per tile).
static bool stream_runs(const ftkcu_session* s, const DevTensor& t) {
  if (t.order != 3 || s->opt_runs == 0) return false;
  if (s->opt_runs == 1) return true;
  if (!s->have_model || !s->opt_tc_ws || !s->opt_hog_update) return false;
  if (s->opt_precision == FTKCU_PREC_FP32 || s->opt_factor_warps == 16) return false;
  const DevModel& m = s->model;
  return m.order == 3 && m.r == 32 && m.ranks[0] == 32 && m.ranks[1] == 32 && m.ranks[2] == 32;
}

// Ends an asynchronous upload on the copy stream.  The tile stream is built
// lazily on the session stream (prepare_stream): built here, behind the
// transfer, it would serialise with it (measured: packed-key e2e 4.8e9 ->
// 4.0e9 nnz/s).  Delta-coded uploads scatter it chunk by chunk instead.
int enqueue_ready(ftkcu_session* s, DevTensor& t) {
  CK(cudaEventRecord(t.ready, s->copy_stream));
  t.pending = true;
  return FTKCU_OK;
}

// Ensures the Hogwild stream exists.  perm != null lays it out in perm
// order (one gather pass, plan-generation cost, outside the sweep timing).
int prepare_stream(ftkcu_session* s, DevTensor& t, const int64_t* perm) {
  if (perm) {
    int rc = upload_perm(s, perm, t.nnz, t.nnz);
    if (rc) return rc;
    CK(build_shuffled(t, s->d_perm, 0, nullptr, 0, s->stream));
    t.shuffled = false;  // stream is in a caller order, not the session shuffle
    return FTKCU_OK;
  }
  if (!t.shuffled) {
    t.runs = stream_runs(s, t);
    CK(build_shuffled(t, nullptr, (uint64_t)s->opt_shuffle_seed, nullptr, 0, s->stream));
  }
  return FTKCU_OK;
}

int finish_timing(ftkcu_session* s, double* ms) {
  CK(cudaEventRecord(s->ev1, s->stream));
  if (ms) {
    CK(cudaEventSynchronize(s->ev1));
    float f = 0.0f;
    CK(cudaEventElapsedTime(&f, s->ev0, s->ev1));
    *ms = f;
  }
  return FTKCU_OK;
}

}  // namespace

namespace ftkcu {
int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}
}  // namespace ftkcu

extern "C" {

int ftkcu_abi_version(void) { return FTKCU_ABI_VERSION; }

const char* ftkcu_last_error(const ftkcu_session* s) {
  return s ? s->err.c_str() : g_create_err.c_str();
}

int ftkcu_session_create(int device, ftkcu_session** out) {
  ftkcu_session* s = nullptr;
  if (!out) return fail(nullptr, FTKCU_ERR_ARG, "null out pointer");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(nullptr, FTKCU_ERR_CUDA, "no CUDA device available: %s",
                cudaGetErrorString(e));
  if (device < 0 || device >= count)
    return fail(nullptr, FTKCU_ERR_ARG, "device %d out of range (%d devices)", device, count);
  s = new ftkcu_session;
  s->device = device;
  int major = 0;
  cudaSetDevice(device);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (major != 10) {
    delete s;
    return fail(nullptr, FTKCU_ERR_CUDA, "device %d is sm_%d0, engine is built for sm_100a",
                device, major);
  }
  if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&s->rb_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&s->dec_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&s->rb_snap, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&s->rb_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreate(&s->ev0) != cudaSuccess || cudaEventCreate(&s->ev1) != cudaSuccess) {
    delete s;
    return fail(nullptr, FTKCU_ERR_CUDA, "stream/event creation failed");
  }
  for (auto& e : s->dec_ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return fail(nullptr, FTKCU_ERR_CUDA, "event creation failed");
  {
    void* h = nullptr;
    if (cudaHostAlloc(&h, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->f16_range_d), h, 0) != cudaSuccess)
      return fail(nullptr, FTKCU_ERR_CUDA, "mapped flag allocation failed");
    s->f16_range_h = static_cast<volatile int*>(h);
    *s->f16_range_h = 0;
  }
  *out = s;
  return FTKCU_OK;
}

void ftkcu_session_destroy(ftkcu_session* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  cudaStreamSynchronize(s->stream);
  cudaStreamSynchronize(s->copy_stream);
  cudaStreamSynchronize(s->rb_stream);
  cudaStreamSynchronize(s->dec_stream);
  for (auto& t : s->slots) free_tensor(t);
  if (!s->rb_buf.empty() && s->rb_buf[0]) cudaFree(s->rb_buf[0]);
  free_model(s->model);
  if (s->grad) cudaFree(s->grad);
  if (s->scratch) cudaFree(s->scratch);
  if (s->d_perm) cudaFree(s->d_perm);
  if (s->d_boff) cudaFree(s->d_boff);
  if (s->d_cellperm) cudaFree(s->d_cellperm);
  if (s->dsgd_exec) cudaGraphExecDestroy(s->dsgd_exec);
  for (void* p : s->ring_ipc)
    if (p) cudaIpcCloseMemHandle(p);
  for (float* p : s->ring_emu_a)
    if (p) cudaFree(p);
  if (s->ring_emu_flags) cudaFree(s->ring_emu_flags);
  if (s->ring_flags) cudaFree(s->ring_flags);
  if (s->ring_done) cudaFree(s->ring_done);
  if (s->ring_err) cudaFree(s->ring_err);
  if (s->ring_tab) cudaFree(s->ring_tab);
  if (s->ring_tab_h) cudaFreeHost(s->ring_tab_h);
  if (s->comm) ncclCommDestroy(s->comm);
  cudaEventDestroy(s->ev0);
  cudaEventDestroy(s->ev1);
  cudaStreamDestroy(s->stream);
  cudaStreamDestroy(s->copy_stream);
  cudaStreamDestroy(s->rb_stream);
  cudaStreamDestroy(s->dec_stream);
  if (s->f16_range_h) cudaFreeHost(const_cast<int*>(s->f16_range_h));
  for (auto e : s->dec_ev)
    if (e) cudaEventDestroy(e);
  cudaEventDestroy(s->rb_snap);
  cudaEventDestroy(s->rb_done);
  delete s;
}

int ftkcu_set_option(ftkcu_session* s, const char* key, int64_t value) {
  if (!s || !key) return fail(s, FTKCU_ERR_ARG, "null argument");
  std::string k(key);
  if (k == "precision") {
    if (value < FTKCU_PREC_FP32 || value > FTKCU_PREC_3XTF32)
      return fail(s, FTKCU_ERR_ARG, "bad precision %lld", (long long)value);
    s->opt_precision = value;
  } else if (k == "eval") {
    if (value != FTKCU_EVAL_EXACT && value != FTKCU_EVAL_FAST)
      return fail(s, FTKCU_ERR_ARG, "bad eval mode %lld", (long long)value);
    s->opt_eval = value;
  } else if (k == "hog_blocks_per_sm") {
    if (value < 1 || value > 16) return fail(s, FTKCU_ERR_ARG, "bad hog_blocks_per_sm");
    s->opt_hog_bps = value;
  } else if (k == "tc_ws") {
    s->opt_tc_ws = value != 0;
  } else if (k == "store_c") {
    s->opt_store_c = value != 0;
  } else if (k == "core16") {
    if (value < 0 || value > 2) return fail(s, FTKCU_ERR_ARG, "core16 must be 0, 1 or 2");
    s->opt_core16 = value;
  } else if (k == "factor_warps") {
    if (value != 8 && value != 16) return fail(s, FTKCU_ERR_ARG, "factor_warps must be 8 or 16");
    s->opt_factor_warps = value;
  } else if (k == "hog_update") {
    if (value != 0 && value != 1) return fail(s, FTKCU_ERR_ARG, "bad hog_update");
    s->opt_hog_update = value;
  } else if (k == "verbose") {
    s->opt_verbose = value;
  } else if (k == "global_nnz") {
    s->global_nnz = value;
  } else if (k == "graphs") {
    s->opt_graphs = value != 0;
  } else if (k == "dsgd_shift") {
    s->opt_dsgd_shift = value != 0;
  } else if (k == "staleness") {
    if (value < 0) return fail(s, FTKCU_ERR_ARG, "staleness must be >= 0");
    s->opt_staleness = value;
  } else if (k == "max_ctas") {
    if (value < 0) return fail(s, FTKCU_ERR_ARG, "max_ctas must be >= 0");
    s->opt_max_ctas = value;
  } else if (k == "runs") {
    if (value < -1 || value > 1) return fail(s, FTKCU_ERR_ARG, "runs must be -1, 0 or 1");
    s->opt_runs = value;
    for (auto& t : s->slots) t.shuffled = false;
  } else if (k == "eager_stream") {
    s->opt_eager_stream = value != 0;
  } else if (k == "delta_decode") {
    if (value != 0 && value != 1) return fail(s, FTKCU_ERR_ARG, "delta_decode must be 0 or 1");
    s->opt_delta_decode = value;
  } else if (k == "cell_order") {
    if (value != 0 && value != 1) return fail(s, FTKCU_ERR_ARG, "cell_order must be 0 or 1");
    s->opt_cell_order = value;
  } else if (k == "ring_timeout_ms") {
    if (value < 0) return fail(s, FTKCU_ERR_ARG, "ring_timeout_ms must be >= 0");
    s->opt_ring_timeout_ms = value;
  } else if (k == "window") {
    if (value != 0 && value != 2 && value != 3)
      return fail(s, FTKCU_ERR_ARG, "window must be 0, 2 or 3");
    s->opt_window = value;
  } else if (k == "shuffle_seed") {
    s->opt_shuffle_seed = value;
    for (auto& t : s->slots) t.shuffled = false;
  } else {
    return fail(s, FTKCU_ERR_ARG, "unknown option '%s'", key);
  }
  return FTKCU_OK;
}

int ftkcu_get_option(ftkcu_session* s, const char* key, int64_t* value) {
  if (!s || !key || !value) return fail(s, FTKCU_ERR_ARG, "null argument");
  std::string k(key);
  if (k == "precision") *value = s->opt_precision;
  else if (k == "eval") *value = s->opt_eval;
  else if (k == "hog_blocks_per_sm") *value = s->opt_hog_bps;
  else if (k == "verbose") *value = s->opt_verbose;
  else if (k == "hog_update") *value = s->opt_hog_update;
  else if (k == "tc_ws") *value = s->opt_tc_ws;
  else if (k == "store_c") *value = s->opt_store_c;
  else if (k == "core16") *value = s->opt_core16;
  else if (k == "factor_warps") *value = s->opt_factor_warps;
  else if (k == "shuffle_seed") *value = s->opt_shuffle_seed;
  else if (k == "max_ctas") *value = s->opt_max_ctas;
  else if (k == "window") *value = s->opt_window;
  else if (k == "cell_order") *value = s->opt_cell_order;
  else if (k == "runs") *value = s->opt_runs;
  else if (k == "eager_stream") *value = s->opt_eager_stream;
  else if (k == "delta_decode") *value = s->opt_delta_decode;
  else if (k == "staleness") *value = s->opt_staleness;
  else if (k == "graphs") *value = s->opt_graphs;
  else if (k == "global_nnz") *value = s->global_nnz;
  else if (k == "launches") *value = s->launches;
  else if (k == "last_factor_kernel") *value = s->last_factor_kernel;
  else if (k == "last_core_kernel") *value = s->last_core_kernel;
  else if (k == "stream") *value = (int64_t)(intptr_t)s->stream;
  else if (k == "copy_stream") *value = (int64_t)(intptr_t)s->copy_stream;
  else if (k == "dec_stream") *value = (int64_t)(intptr_t)s->dec_stream;
  else if (k == "num_sms") *value = num_sms();
  else return fail(s, FTKCU_ERR_ARG, "unknown option '%s'", key);
  return FTKCU_OK;
}

int ftkcu_tensor_upload(ftkcu_session* s, int slot, int order, const int32_t* dims,
                        int64_t nnz, const int32_t* idx_rowmajor, const float* values) {
  int rc = bind(s);
  if (rc) return rc;
  if (slot < 0 || slot >= 8) return fail(s, FTKCU_ERR_ARG, "tensor slot %d out of range", slot);
  if (order < 1 || order > kMaxOrder)
    return fail(s, FTKCU_ERR_ARG, "order %d unsupported (1..%d)", order, kMaxOrder);
  if (nnz < 0) return fail(s, FTKCU_ERR_ARG, "negative nnz");
  if (nnz > 0 && (!idx_rowmajor || !values)) return fail(s, FTKCU_ERR_ARG, "null data");
  for (int n = 0; n < order; ++n)
    if (dims[n] < 1) return fail(s, FTKCU_ERR_ARG, "dims must be positive");
  DevTensor& t = s->slots[slot];
  if ((rc = finish_upload(s, t))) return rc;
  const size_t cnt = nnz > 0 ? (size_t)nnz : 1;
  if (t.vals && t.order == order && t.nnz == nnz) {
    // same extent (e.g. a new epoch's data): keep every device buffer,
    // including the tiled stream, which is rebuilt lazily
    CK(cudaStreamSynchronize(s->stream));
    t.cell_off.clear();
    t.cell_tile.clear();
    t.shuffled = false;
    t.stream_tiles = 0;
  } else {
    free_tensor(t);
    t.order = order;
    t.nnz = nnz;
    for (int n = 0; n < order; ++n) CK(cudaMalloc(&t.idx[n], sizeof(int32_t) * cnt));
    CK(cudaMalloc(&t.vals, sizeof(float) * cnt));
  }
  for (int n = 0; n < order; ++n) t.dims[n] = dims[n];
  if (nnz > 0) {
    int rc2 = ensure_scratch(s, sizeof(int32_t) * (size_t)nnz * order + 256);
    if (rc2) return rc2;
    int32_t* aos = static_cast<int32_t*>(s->scratch);
    int* bad = reinterpret_cast<int*>(static_cast<char*>(s->scratch) +
                                      sizeof(int32_t) * (size_t)nnz * order);
    CK(cudaMemcpyAsync(aos, idx_rowmajor, sizeof(int32_t) * (size_t)nnz * order,
                       cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(t.vals, values, sizeof(float) * nnz, cudaMemcpyHostToDevice,
                       s->stream));
    CK(cudaMemsetAsync(bad, 0, sizeof(int), s->stream));
    SoAView v{};
    v.order = order;
    for (int n = 0; n < order; ++n) {
      v.dims[n] = dims[n];
      v.col[n] = t.idx[n];
    }
    aos_to_soa_kernel<<<num_sms() * 8, 256, 0, s->stream>>>(aos, nnz, v, bad);
    CK(cudaGetLastError());
    int h_bad = 0;
    CK(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    if (h_bad) {
      free_tensor(t);
      return fail(s, FTKCU_ERR_ARG, "index out of range in tensor upload");
    }
  }
  return FTKCU_OK;
}

int ftkcu_tensor_upload_async(ftkcu_session* s, int slot, int order, const int32_t* dims,
                              int64_t nnz, const int32_t* idx_rowmajor, const float* values) {
  int rc = bind(s);
  if (rc) return rc;
  if (slot < 0 || slot >= 8) return fail(s, FTKCU_ERR_ARG, "tensor slot %d out of range", slot);
  if (order < 1 || order > kMaxOrder)
    return fail(s, FTKCU_ERR_ARG, "order %d unsupported (1..%d)", order, kMaxOrder);
  if (nnz < 1 || !idx_rowmajor || !values)
    return fail(s, FTKCU_ERR_ARG, "asynchronous upload needs a non-empty tensor");
  for (int n = 0; n < order; ++n)
    if (dims[n] < 1) return fail(s, FTKCU_ERR_ARG, "dims must be positive");
  DevTensor& t = s->slots[slot];
  if ((rc = finish_upload(s, t))) return rc;
  // the copies overwrite the slot's buffers: order them after the kernels
  // enqueued on the session stream that read this slot -- all of them if it
  // is the slot in use, else those up to its last use (so a caller can
  // enqueue slot k's epoch first and the copy into slot k + 1 still overlaps it)
  if (slot == s->last_slot || (t.used_rec && !t.used)) {
    CK(cudaEventRecord(s->ev1, s->stream));
    CK(cudaStreamWaitEvent(s->copy_stream, s->ev1, 0));
  } else if (t.used_rec) {
    CK(cudaStreamWaitEvent(s->copy_stream, t.used, 0));
  }
  if (!(t.vals && t.order == order && t.nnz == nnz)) {
    CK(cudaStreamSynchronize(s->stream));
    free_tensor(t);
    t.order = order;
    t.nnz = nnz;
    for (int n = 0; n < order; ++n) CK(cudaMalloc(&t.idx[n], sizeof(int32_t) * (size_t)nnz));
    CK(cudaMalloc(&t.vals, sizeof(float) * (size_t)nnz));
  }
  for (int n = 0; n < order; ++n) t.dims[n] = dims[n];
  t.cell_off.clear();
  t.cell_tile.clear();
  t.shuffled = false;
  t.stream_tiles = 0;
  const size_t aos = sizeof(int32_t) * (size_t)nnz * order;
  if (t.staging_cap < aos) {
    if (t.staging) CK(cudaFree(t.staging));
    t.staging = nullptr;
    CK(cudaMalloc(&t.staging, aos));
    t.staging_cap = aos;
  }
  if (!t.d_bad) CK(cudaMalloc(&t.d_bad, sizeof(int)));
  if (!t.ready) CK(cudaEventCreateWithFlags(&t.ready, cudaEventDisableTiming));
  CK(cudaMemcpyAsync(t.staging, idx_rowmajor, aos, cudaMemcpyHostToDevice, s->copy_stream));
  CK(cudaMemcpyAsync(t.vals, values, sizeof(float) * nnz, cudaMemcpyHostToDevice, s->copy_stream));
  CK(cudaMemsetAsync(t.d_bad, 0, sizeof(int), s->copy_stream));
  SoAView v{};
  v.order = order;
  for (int n = 0; n < order; ++n) {
    v.dims[n] = dims[n];
    v.col[n] = t.idx[n];
  }
  aos_to_soa_kernel<<<num_sms() * 8, 256, 0, s->copy_stream>>>(t.staging, nnz, v, t.d_bad);
  CK(cudaGetLastError());
  // the tile stream is built lazily on the session stream (prepare_stream), so
  // the copy stream is free for the next upload as soon as this one is checked
  return enqueue_ready(s, t);
}

// Bit layout of packed keys: w_n = bit width of dims[n] - 1 (>= 1).
static bool key_layout(int order, const int32_t* dims, KeyLayout* kl) {
  int off = 0;
  kl->order = order;
  for (int n = 0; n < order; ++n) {
    int w = 1;
    while (w < 31 && (int64_t)(dims[n] - 1) >= ((int64_t)1 << w)) ++w;
    kl->off[n] = off;
    kl->mask[n] = (1ull << w) - 1;
    off += w;
  }
  kl->hi_bytes = off <= 32 ? 0 : (off <= 48 ? 2 : 4);
  return off <= 64;
}

int ftkcu_key_layout(int order, const int32_t* dims, int* hi_bytes) {
  if (order < 1 || order > kMaxOrder || !dims || !hi_bytes)
    return fail(nullptr, FTKCU_ERR_ARG, "bad key_layout arguments");
  for (int n = 0; n < order; ++n)
    if (dims[n] < 1) return fail(nullptr, FTKCU_ERR_ARG, "dims must be positive");
  KeyLayout kl;
  if (!key_layout(order, dims, &kl)) return fail(nullptr, FTKCU_ERR_ARG, "index widths exceed 64 bits");
  *hi_bytes = kl.hi_bytes;
  return FTKCU_OK;
}

int ftkcu_pack_keys(int order, const int32_t* dims, int64_t nnz, const int32_t* idx_rowmajor,
                    uint32_t* lo, void* hi) {
  if (order < 1 || order > kMaxOrder || nnz < 0 || !dims || (nnz && (!idx_rowmajor || !lo)))
    return fail(nullptr, FTKCU_ERR_ARG, "bad pack_keys arguments");
  KeyLayout kl;
  for (int n = 0; n < order; ++n)
    if (dims[n] < 1) return fail(nullptr, FTKCU_ERR_ARG, "dims must be positive");
  if (!key_layout(order, dims, &kl))
    return fail(nullptr, FTKCU_ERR_ARG, "index widths exceed 64 bits");
  if (kl.hi_bytes && nnz && !hi) return fail(nullptr, FTKCU_ERR_ARG, "keys need a high part");
  int bad = 0;
  for (int64_t e = 0; e < nnz; ++e) {
    uint64_t k = 0;
    for (int n = 0; n < order; ++n) {
      const int32_t x = idx_rowmajor[e * order + n];
      bad |= (x < 0 || x >= dims[n]);
      k |= (uint64_t)(uint32_t)x << kl.off[n];
    }
    lo[e] = (uint32_t)k;
    if (kl.hi_bytes == 2) static_cast<uint16_t*>(hi)[e] = (uint16_t)(k >> 32);
    else if (kl.hi_bytes == 4) static_cast<uint32_t*>(hi)[e] = (uint32_t)(k >> 32);
  }
  if (bad) return fail(nullptr, FTKCU_ERR_ARG, "index out of range");
  return FTKCU_OK;
}

int ftkcu_tensor_upload_packed_async(ftkcu_session* s, int slot, int order, const int32_t* dims,
                                     int64_t nnz, const uint32_t* lo, const void* hi,
                                     const float* values) {
  int rc = bind(s);
  if (rc) return rc;
  if (slot < 0 || slot >= 8) return fail(s, FTKCU_ERR_ARG, "tensor slot %d out of range", slot);
  if (order < 1 || order > kMaxOrder)
    return fail(s, FTKCU_ERR_ARG, "order %d unsupported (1..%d)", order, kMaxOrder);
  if (nnz < 1 || !lo || !values)
    return fail(s, FTKCU_ERR_ARG, "asynchronous upload needs a non-empty tensor");
  for (int n = 0; n < order; ++n)
    if (dims[n] < 1) return fail(s, FTKCU_ERR_ARG, "dims must be positive");
  KeyLayout kl;
  if (!key_layout(order, dims, &kl)) return fail(s, FTKCU_ERR_ARG, "index widths exceed 64 bits");
  if (kl.hi_bytes && !hi) return fail(s, FTKCU_ERR_ARG, "keys need a high part");
  DevTensor& t = s->slots[slot];
  if ((rc = finish_upload(s, t))) return rc;
  // ordering against the slot's readers: as ftkcu_tensor_upload_async
  if (slot == s->last_slot || (t.used_rec && !t.used)) {
    CK(cudaEventRecord(s->ev1, s->stream));
    CK(cudaStreamWaitEvent(s->copy_stream, s->ev1, 0));
  } else if (t.used_rec) {
    CK(cudaStreamWaitEvent(s->copy_stream, t.used, 0));
  }
  if (!(t.vals && t.order == order && t.nnz == nnz)) {
    CK(cudaStreamSynchronize(s->stream));
    free_tensor(t);
    t.order = order;
    t.nnz = nnz;
    for (int n = 0; n < order; ++n) CK(cudaMalloc(&t.idx[n], sizeof(int32_t) * (size_t)nnz));
    CK(cudaMalloc(&t.vals, sizeof(float) * (size_t)nnz));
  }
  for (int n = 0; n < order; ++n) t.dims[n] = dims[n];
  t.cell_off.clear();
  t.cell_tile.clear();
  t.shuffled = false;
  t.stream_tiles = 0;
  const size_t lb = sizeof(uint32_t) * (size_t)nnz, hb = (size_t)kl.hi_bytes * nnz;
  const size_t kb = lb + (hb + 15) / 16 * 16;
  if (t.staging_cap < kb) {
    if (t.staging) CK(cudaFree(t.staging));
    t.staging = nullptr;
    CK(cudaMalloc(&t.staging, kb));
    t.staging_cap = kb;
  }
  if (!t.d_bad) CK(cudaMalloc(&t.d_bad, sizeof(int)));
  if (!t.ready) CK(cudaEventCreateWithFlags(&t.ready, cudaEventDisableTiming));
  uint8_t* st = reinterpret_cast<uint8_t*>(t.staging);
  CK(cudaMemcpyAsync(st, lo, lb, cudaMemcpyHostToDevice, s->copy_stream));
  if (hb) CK(cudaMemcpyAsync(st + lb, hi, hb, cudaMemcpyHostToDevice, s->copy_stream));
  CK(cudaMemcpyAsync(t.vals, values, sizeof(float) * nnz, cudaMemcpyHostToDevice, s->copy_stream));
  CK(cudaMemsetAsync(t.d_bad, 0, sizeof(int), s->copy_stream));
  SoAView v{};
  v.order = order;
  for (int n = 0; n < order; ++n) {
    v.dims[n] = dims[n];
    v.col[n] = t.idx[n];
  }
  keys_to_soa_kernel<<<num_sms() * 8, 256, 0, s->copy_stream>>>(
      reinterpret_cast<const uint32_t*>(st), st + lb, nnz, v, kl, t.d_bad);
  CK(cudaGetLastError());
  return enqueue_ready(s, t);
}

// ---- delta-coded COO --------------------------------------------------------

// Mixed-radix key of every nonzero, sorted ascending (LSD radix sort, 16-bit
// digits, stable), then chunked deltas.  Host code, run once per tensor
// (like writing a file format); no reference counterpart.
constexpr int kDeltaParts = 8;  // H2D / decode pipeline depth of a delta-coded upload

int ftkcu_pack_delta(int order, const int32_t* dims, int64_t nnz, const int32_t* idx_rowmajor,
                     const float* values, uint8_t* deltas, int64_t deltas_cap,
                     uint64_t* restarts, float* values_out, int* width) {
  if (order < 1 || order > kMaxOrder || nnz < 1 || !dims || !idx_rowmajor || !values ||
      !restarts || !values_out || !width)
    return fail(nullptr, FTKCU_ERR_ARG, "bad pack_delta arguments");
  double cells = 1.0;
  for (int n = 0; n < order; ++n) {
    if (dims[n] < 1) return fail(nullptr, FTKCU_ERR_ARG, "dims must be positive");
    cells *= (double)dims[n];
  }
  if (cells > 9007199254740992.0)  // 2^53: the decoder divides in double precision
    return fail(nullptr, FTKCU_ERR_ARG, "delta keys need prod(dims) <= 2^53");
  std::vector<uint64_t> key((size_t)nnz), key2((size_t)nnz);
  std::vector<uint32_t> pos((size_t)nnz), pos2((size_t)nnz);
  if (nnz >= ((int64_t)1 << 32)) return fail(nullptr, FTKCU_ERR_ARG, "pack_delta: nnz >= 2^32");
  uint64_t kmax = 0;
  for (int64_t e = 0; e < nnz; ++e) {
    uint64_t k = 0;
    for (int n = 0; n < order; ++n) {
      const int32_t x = idx_rowmajor[e * order + n];
      if (x < 0 || x >= dims[n]) return fail(nullptr, FTKCU_ERR_ARG, "index out of range");
      k = k * (uint64_t)dims[n] + (uint64_t)x;
    }
    key[e] = k;
    pos[e] = (uint32_t)e;
    kmax = std::max(kmax, k);
  }
  std::vector<int64_t> cnt(1 << 16);
  for (int sh = 0; sh < 64 && (kmax >> sh); sh += 16) {
    std::fill(cnt.begin(), cnt.end(), 0);
    for (int64_t e = 0; e < nnz; ++e) ++cnt[(key[e] >> sh) & 0xffff];
    int64_t run = 0;
    for (auto& x : cnt) {
      const int64_t t = x;
      x = run;
      run += t;
    }
    for (int64_t e = 0; e < nnz; ++e) {
      const int64_t d = cnt[(key[e] >> sh) & 0xffff]++;
      key2[d] = key[e];
      pos2[d] = pos[e];
    }
    key.swap(key2);
    pos.swap(pos2);
  }
  uint64_t dmax = 0;
  for (int64_t e = 1; e < nnz; ++e)
    if (e % kDeltaChunk) dmax = std::max(dmax, key[e] - key[e - 1]);
  int w = 1;
  while (w < 8 && (dmax >> (8 * w))) ++w;
  *width = w;
  if (!deltas || deltas_cap < (int64_t)w * nnz)
    return fail(nullptr, FTKCU_ERR_ARG, "pack_delta: deltas need %d bytes per nonzero", w);
  for (int64_t e = 0; e < nnz; ++e) {
    const uint64_t d = e % kDeltaChunk ? key[e] - key[e - 1] : 0;
    if (e % kDeltaChunk == 0) restarts[e / kDeltaChunk] = key[e];
    for (int b = 0; b < w; ++b) deltas[e * w + b] = (uint8_t)(d >> (8 * b));
    values_out[e] = values[pos[e]];
  }
  return FTKCU_OK;
}

int ftkcu_tensor_upload_delta_async(ftkcu_session* s, int slot, int order, const int32_t* dims,
                                    int64_t nnz, const uint8_t* deltas, int width,
                                    const uint64_t* restarts, const float* values) {
  int rc = bind(s);
  if (rc) return rc;
  if (slot < 0 || slot >= 8) return fail(s, FTKCU_ERR_ARG, "tensor slot %d out of range", slot);
  if (order < 1 || order > kMaxOrder)
    return fail(s, FTKCU_ERR_ARG, "order %d unsupported (1..%d)", order, kMaxOrder);
  if (nnz < 1 || !deltas || !restarts || !values || width < 1 || width > 8)
    return fail(s, FTKCU_ERR_ARG, "asynchronous upload needs a non-empty tensor");
  double cells = 1.0;
  for (int n = 0; n < order; ++n) {
    if (dims[n] < 1) return fail(s, FTKCU_ERR_ARG, "dims must be positive");
    cells *= (double)dims[n];
  }
  if (cells > 9007199254740992.0) return fail(s, FTKCU_ERR_ARG, "delta keys need prod(dims) <= 2^53");
  DevTensor& t = s->slots[slot];
  if ((rc = finish_upload(s, t))) return rc;
  // ordering against the slot's readers: as ftkcu_tensor_upload_async
  if (slot == s->last_slot || (t.used_rec && !t.used)) {
    CK(cudaEventRecord(s->ev1, s->stream));
    CK(cudaStreamWaitEvent(s->copy_stream, s->ev1, 0));
  } else if (t.used_rec) {
    CK(cudaStreamWaitEvent(s->copy_stream, t.used, 0));
  }
  if (!(t.vals && t.order == order && t.nnz == nnz)) {
    CK(cudaStreamSynchronize(s->stream));
    free_tensor(t);
    t.order = order;
    t.nnz = nnz;
    for (int n = 0; n < order; ++n) CK(cudaMalloc(&t.idx[n], sizeof(int32_t) * (size_t)nnz));
    CK(cudaMalloc(&t.vals, sizeof(float) * (size_t)nnz));
  }
  for (int n = 0; n < order; ++n) t.dims[n] = dims[n];
  t.cell_off.clear();
  t.cell_tile.clear();
  t.shuffled = false;
  t.stream_tiles = 0;
  const int64_t chunks = (nnz + kDeltaChunk - 1) / kDeltaChunk;
  const size_t db = (size_t)width * nnz, rb = sizeof(uint64_t) * (size_t)chunks;
  const size_t dpad = (db + 15) / 16 * 16;
  if (t.staging_cap < dpad + rb) {
    if (t.staging) CK(cudaFree(t.staging));
    t.staging = nullptr;
    CK(cudaMalloc(&t.staging, dpad + rb));
    t.staging_cap = dpad + rb;
  }
  if (!t.d_bad) CK(cudaMalloc(&t.d_bad, sizeof(int)));
  if (!t.ready) CK(cudaEventCreateWithFlags(&t.ready, cudaEventDisableTiming));
  // Order 3 single cell (no runs layout): every decoded chunk scatters its
  // records straight into the tile stream, so decoding and the stream build
  // overlap the rest of the transfer (copy stream: the parts' H2D copies;
  // decode stream: each part's kernel once its bytes have landed).
  const bool scatter = s->opt_eager_stream && order == 3 && !stream_runs(s, t);
  if (scatter) CK(prepare_scatter_stream(t));
  uint8_t* st = reinterpret_cast<uint8_t*>(t.staging);
  const uint64_t* rs_dev = reinterpret_cast<const uint64_t*>(st + dpad);
  CK(cudaMemsetAsync(t.d_bad, 0, sizeof(int), s->copy_stream));
  CK(cudaMemcpyAsync(st + dpad, restarts, rb, cudaMemcpyHostToDevice, s->copy_stream));
  if (s->opt_delta_decode == 1) {
    // copies only; decoded at the slot's first use (finish_upload)
    CK(cudaMemcpyAsync(st, deltas, db, cudaMemcpyHostToDevice, s->copy_stream));
    CK(cudaMemcpyAsync(t.vals, values, sizeof(float) * nnz, cudaMemcpyHostToDevice,
                       s->copy_stream));
    CK(cudaEventRecord(t.ready, s->copy_stream));
    t.delta_pending = true;
    t.delta_scatter = scatter;
    t.delta_width = width;
    t.delta_roff = dpad;
    t.delta_seed = (uint64_t)s->opt_shuffle_seed;
    if (scatter) {
      t.shuffled = true;  // the stream is built with the decode
      t.runs = false;
    }
    t.pending = true;
    return FTKCU_OK;
  }
  const int64_t per = (chunks + kDeltaParts - 1) / kDeltaParts;
  for (int part = 0; part < kDeltaParts; ++part) {
    const int64_t c0 = std::min<int64_t>(chunks, part * per), c1 = std::min<int64_t>(chunks, c0 + per);
    if (c1 <= c0) break;
    const int64_t e0 = c0 * kDeltaChunk, e1 = std::min<int64_t>(nnz, c1 * kDeltaChunk);
    CK(cudaMemcpyAsync(st + e0 * width, deltas + e0 * width, (size_t)(e1 - e0) * width,
                       cudaMemcpyHostToDevice, s->copy_stream));
    CK(cudaMemcpyAsync(t.vals + e0, values + e0, sizeof(float) * (e1 - e0), cudaMemcpyHostToDevice,
                       s->copy_stream));
    CK(cudaEventRecord(s->dec_ev[part], s->copy_stream));
    CK(cudaStreamWaitEvent(s->dec_stream, s->dec_ev[part], 0));
    CK(launch_delta_decode(t, st, rs_dev, width, c0, c1, scatter, (uint64_t)s->opt_shuffle_seed,
                           t.d_bad, s->dec_stream));
  }
  if (scatter) {
    CK(finish_scatter_stream(t, s->dec_stream));
    CK(cudaEventRecord(t.ready, s->dec_stream));
    t.pending = true;
    return FTKCU_OK;
  }
  CK(cudaEventRecord(s->dec_ev[0], s->dec_stream));
  CK(cudaStreamWaitEvent(s->copy_stream, s->dec_ev[0], 0));
  return enqueue_ready(s, t);
}

int ftkcu_tensor_release(ftkcu_session* s, int slot) {
  int rc = bind(s);
  if (rc) return rc;
  if (slot < 0 || slot >= 8) return fail(s, FTKCU_ERR_ARG, "tensor slot %d out of range", slot);
  CK(cudaStreamSynchronize(s->copy_stream));
  s->slots[slot].pending = false;
  CK(cudaStreamSynchronize(s->stream));
  free_tensor(s->slots[slot]);
  return FTKCU_OK;
}

int64_t ftkcu_tensor_nnz(ftkcu_session* s, int slot) {
  if (!s || slot < 0 || slot >= 8) return -1;
  return s->slots[slot].nnz;
}

int ftkcu_model_upload(ftkcu_session* s, int order, const int32_t* dims, const int32_t* ranks,
                       int32_t R, const float* const* A, const float* const* B) {
  int rc = bind(s);
  if (rc) return rc;
  if (order < 1 || order > kMaxOrder)
    return fail(s, FTKCU_ERR_ARG, "order %d unsupported (1..%d)", order, kMaxOrder);
  if (R < 1) return fail(s, FTKCU_ERR_ARG, "low rank must be positive");
  for (int n = 0; n < order; ++n)
    if (dims[n] < 1 || ranks[n] < 1) return fail(s, FTKCU_ERR_ARG, "zero dim or rank");
  DevModel& m = s->model;
  bool same = s->have_model && m.order == order && m.r == R;
  for (int n = 0; same && n < order; ++n)
    same = m.dims[n] == dims[n] && m.ranks[n] == ranks[n];
  if (!same) {
    CK(cudaStreamSynchronize(s->stream));
    free_model(m);
    s->have_model = false;
    m.order = order;
    m.r = R;
    for (int n = 0; n < order; ++n) {
      m.dims[n] = dims[n];
      m.ranks[n] = ranks[n];
      CK(cudaMalloc(&m.a[n], sizeof(float) * (size_t)dims[n] * ranks[n]));
      CK(cudaMalloc(&m.b[n], sizeof(float) * (size_t)ranks[n] * R));
    }
    const size_t glen = (size_t)m.sum_j() * R;
    if (glen > s->grad_len) {
      if (s->grad) CK(cudaFree(s->grad));
      CK(cudaMalloc(&s->grad, sizeof(float) * glen));
      s->grad_len = glen;
    }
  }
  for (int n = 0; n < order; ++n) {
    CK(cudaMemcpyAsync(m.a[n], A[n], sizeof(float) * (size_t)dims[n] * ranks[n],
                       cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(m.b[n], B[n], sizeof(float) * (size_t)ranks[n] * R,
                       cudaMemcpyHostToDevice, s->stream));
  }
  CK(cudaStreamSynchronize(s->stream));
  s->have_model = true;
  // the automatic stream layout depends on the model's ranks
  for (auto& t : s->slots)
    if (t.shuffled && t.runs != stream_runs(s, t)) t.shuffled = false;
  return FTKCU_OK;
}

int ftkcu_model_download(ftkcu_session* s, float* const* A, float* const* B) {
  int rc = bind(s);
  if (rc) return rc;
  if (!s->have_model) return fail(s, FTKCU_ERR_STATE, "no model uploaded");
  const DevModel& m = s->model;
  for (int n = 0; n < m.order; ++n) {
    if (A && A[n])
      CK(cudaMemcpyAsync(A[n], m.a[n], sizeof(float) * (size_t)m.dims[n] * m.ranks[n],
                         cudaMemcpyDeviceToHost, s->stream));
    if (B && B[n])
      CK(cudaMemcpyAsync(B[n], m.b[n], sizeof(float) * (size_t)m.ranks[n] * m.r,
                         cudaMemcpyDeviceToHost, s->stream));
  }
  CK(cudaStreamSynchronize(s->stream));
  return check_f16_range(s);
}

// Enqueued model copies (pinned host buffers; no host synchronisation): the
// e2e loop's per-step model transfers stay in stream order without a host
// round trip between epochs.
int ftkcu_model_copy_async(ftkcu_session* s, int to_device, float* const* A, float* const* B) {
  int rc = bind(s);
  if (rc) return rc;
  if (!s->have_model) return fail(s, FTKCU_ERR_STATE, "no model uploaded");
  const DevModel& m = s->model;
  if (!to_device) {
    // Read-back: snapshot the model on the session stream (a device copy at
    // HBM speed), then copy the snapshot to the host on rb_stream, so the
    // next epoch does not wait for the PCIe transfer.  The next snapshot
    // waits for this transfer (it overwrites the buffer).
    size_t total = 0;
    for (int n = 0; n < m.order; ++n)
      total += (size_t)m.dims[n] * m.ranks[n] + (size_t)m.ranks[n] * m.r;
    if (s->rb_floats < total) {
      CK(cudaStreamSynchronize(s->rb_stream));
      if (!s->rb_buf.empty() && s->rb_buf[0]) CK(cudaFree(s->rb_buf[0]));
      s->rb_buf.assign(1, nullptr);
      CK(cudaMalloc(&s->rb_buf[0], sizeof(float) * total));
      s->rb_floats = total;
      s->rb_pending = false;
    }
    if (s->rb_pending) CK(cudaStreamWaitEvent(s->stream, s->rb_done, 0));
    float* snap = s->rb_buf[0];
    for (int n = 0; n < m.order; ++n) {
      const size_t an = (size_t)m.dims[n] * m.ranks[n], bn = (size_t)m.ranks[n] * m.r;
      auto dcopy = [&](float* dst, const float* src, size_t nf) -> cudaError_t {
        if (nf % 4 || (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
          return cudaMemcpyAsync(dst, src, sizeof(float) * nf, cudaMemcpyDeviceToDevice, s->stream);
        const int64_t n4 = (int64_t)(nf / 4);
        int64_t blocks = (n4 + 255) / 256;
        if (blocks > num_sms() * 4) blocks = num_sms() * 4;
        if (blocks < 1) return cudaSuccess;
        copy16_kernel<<<(int)blocks, 256, 0, s->stream>>>(reinterpret_cast<const float4*>(src),
                                                          reinterpret_cast<float4*>(dst), n4);
        return cudaGetLastError();
      };
      if (A && A[n]) CK(dcopy(snap, m.a[n], an));
      snap += an;
      if (B && B[n]) CK(dcopy(snap, m.b[n], bn));
      snap += bn;
    }
    CK(cudaEventRecord(s->rb_snap, s->stream));
    CK(cudaStreamWaitEvent(s->rb_stream, s->rb_snap, 0));
    snap = s->rb_buf[0];
    for (int n = 0; n < m.order; ++n) {
      const size_t an = (size_t)m.dims[n] * m.ranks[n], bn = (size_t)m.ranks[n] * m.r;
      if (A && A[n])
        CK(cudaMemcpyAsync(A[n], snap, sizeof(float) * an, cudaMemcpyDeviceToHost, s->rb_stream));
      snap += an;
      if (B && B[n])
        CK(cudaMemcpyAsync(B[n], snap, sizeof(float) * bn, cudaMemcpyDeviceToHost, s->rb_stream));
      snap += bn;
    }
    CK(cudaEventRecord(s->rb_done, s->rb_stream));
    s->rb_pending = true;
    return FTKCU_OK;
  }
  const cudaMemcpyKind kind = to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  for (int n = 0; n < m.order; ++n) {
    const size_t an = sizeof(float) * (size_t)m.dims[n] * m.ranks[n];
    const size_t bn = sizeof(float) * (size_t)m.ranks[n] * m.r;
    if (A && A[n]) CK(cudaMemcpyAsync(to_device ? (void*)m.a[n] : (void*)A[n],
                                      to_device ? (const void*)A[n] : (const void*)m.a[n], an,
                                      kind, s->stream));
    if (B && B[n]) CK(cudaMemcpyAsync(to_device ? (void*)m.b[n] : (void*)B[n],
                                      to_device ? (const void*)B[n] : (const void*)m.b[n], bn,
                                      kind, s->stream));
  }
  return FTKCU_OK;
}

// Hogwild factor sweep over v's tile range: WS tcgen05 -> tcgen05 -> FFMA.
static int launch_factor(ftkcu_session* s, const KView& v, int64_t mul, int64_t add,
                         float lr_a, float reg_a) {
  if (v.ntiles <= 0) return FTKCU_OK;
  // WS factor sweeps: single-pass tf32 (atomic or overwrite rows) and
  // 3xtf32 (atomic rows); everything else on the synchronous tc sweep
  if (s->opt_precision == FTKCU_PREC_TF32 && s->opt_tc_ws && s->opt_hog_update &&
      s->opt_factor_warps == 16 && wsf32_supported(v)) {
    CK(launch_wsg_factor(v, s->model.dims, mul, add, lr_a, reg_a, s->stream));
    s->last_factor_kernel = FTKCU_K_WSF;
  } else if (s->opt_precision == FTKCU_PREC_TF32 && s->opt_tc_ws && ws_supported(v)) {
    CK(launch_ws_factor(v, s->model.dims, mul, add, lr_a, reg_a, (int)s->opt_precision,
                        (int)s->opt_hog_update, 8, s->stream));
    s->last_factor_kernel = FTKCU_K_WS;
  } else if (s->opt_precision == FTKCU_PREC_3XTF32 && s->opt_tc_ws && s->opt_hog_update &&
             ws_supported(v)) {
    CK(launch_ws_factor(v, s->model.dims, mul, add, lr_a, reg_a, (int)s->opt_precision, 1, 8,
                        s->stream));
    s->last_factor_kernel = FTKCU_K_WS3;
  } else if (s->opt_precision == FTKCU_PREC_TF32 && s->opt_tc_ws && s->opt_hog_update &&
             wsg_supported(v)) {
    CK(launch_wsg_factor(v, s->model.dims, mul, add, lr_a, reg_a, s->stream));
    s->last_factor_kernel = FTKCU_K_WSG;
  } else if (s->opt_precision == FTKCU_PREC_TF32 && big_supported(v)) {
    // large ranks: B operand images in the session scratch (allocated
    // before any graph capture, see ftkcu_dsgd_factor_epoch)
    int rc = ensure_scratch(s, big_scratch_bytes(v, s->model.dims, false));
    if (rc) return rc;
    CK(launch_big_factor(v, s->model.dims, mul, add, lr_a, reg_a, (int)s->opt_hog_update,
                         static_cast<float*>(s->scratch), s->scratch_bytes, s->stream));
    s->last_factor_kernel = FTKCU_K_BIG;
  } else if (s->opt_precision != FTKCU_PREC_FP32 && tc_supported(v)) {
    CK(launch_tc_factor(v, mul, add, lr_a, reg_a, (int)s->opt_precision,
                        (int)s->opt_hog_update, s->stream));
    s->last_factor_kernel = FTKCU_K_TC;
  } else {
    CK(launch_hog_factor(v, mul, add, lr_a, reg_a, (int)s->opt_hog_bps,
                         (int)s->opt_hog_update, s->stream));
    s->last_factor_kernel = FTKCU_K_HOG;
  }
  s->launches += 1;
  return FTKCU_OK;
}

static int factor_phase_impl(ftkcu_session* s, int slot, const int64_t* perm, int32_t M,
                             float lr_a, float reg_a, int mode, uint64_t seed, int cell,
                             double* ms) {
  int rc = bind(s);
  if (rc) return rc;
  if ((rc = check_ready(s, slot))) return rc;
  if (M < 1) return fail(s, FTKCU_ERR_ARG, "batch size must be positive");
  DevTensor& t = s->slots[slot];
  if (mode == FTKCU_MODE_DETERMINISTIC) {
    if (!perm && t.nnz > 0) return fail(s, FTKCU_ERR_ARG, "deterministic mode needs a permutation");
    if ((rc = upload_perm(s, perm, t.nnz, t.nnz))) return rc;
    KView v = make_view(s, t, false);
    DetDebug dbg{};
    CK(cudaEventRecord(s->ev0, s->stream));
    if (t.nnz > 0) {
      CK(launch_det_factor(v, s->d_perm, M, lr_a, reg_a, dbg, s->stream));
      s->launches += 1;
      s->last_factor_kernel = FTKCU_K_DET;
    }
    return finish_timing(s, ms);
  }
  if (mode != FTKCU_MODE_HOGWILD) return fail(s, FTKCU_ERR_ARG, "unknown mode %d", mode);
  if ((rc = prepare_stream(s, t, perm))) return rc;
  KView v = make_view(s, t, true);
  v.max_ctas = (int)s->opt_max_ctas;
  v.window = (int)s->opt_window;
  if (cell < 0 && s->opt_staleness > 0) {
    int64_t rows = s->model.dims[0];
    for (int n = 1; n < s->model.order; ++n) rows = std::min<int64_t>(rows, s->model.dims[n]);
    const int64_t cap = std::max<int64_t>(1, rows * s->opt_staleness / (3 * kHogTile));
    if (cap < num_sms() && (v.max_ctas == 0 || cap < v.max_ctas)) v.max_ctas = (int)cap;
  }
  if (cell >= 0) {
    if (cell + 1 >= (int)t.cell_tile.size())
      return fail(s, FTKCU_ERR_ARG, "cell %d out of range", cell);
    v.tile_base = t.cell_tile[cell];
    v.ntiles = t.cell_tile[cell + 1] - t.cell_tile[cell];
  }
  int64_t mul = 1, add = 0;
  if (!perm) tile_perm(seed, v.ntiles, &mul, &add);
  CK(cudaEventRecord(s->ev0, s->stream));
  if ((rc = launch_factor(s, v, mul, add, lr_a, reg_a))) return rc;
  return finish_timing(s, ms);
}

int ftkcu_factor_phase(ftkcu_session* s, int slot, const int64_t* perm, int32_t M, float lr_a,
                       float reg_a, int mode, uint64_t seed, double* ms) {
  return factor_phase_impl(s, slot, perm, M, lr_a, reg_a, mode, seed, -1, ms);
}

int ftkcu_factor_phase_cell(ftkcu_session* s, int slot, int cell, float lr_a, float reg_a,
                            uint64_t seed, double* ms) {
  if (cell < 0) return fail(s, FTKCU_ERR_ARG, "cell must be >= 0");
  return factor_phase_impl(s, slot, nullptr, 16, lr_a, reg_a, FTKCU_MODE_HOGWILD, seed, cell, ms);
}

// Measurement only: the headline factor sweep's RED write-back alone over
// slot's Hogwild tile stream (same grid and tile order as
// ftkcu_factor_phase with this seed), into scratch rows -- the model is not
// touched.  *ms = its device time.
int ftkcu_writeback_ceiling(ftkcu_session* s, int slot, uint64_t seed, double* ms) {
  int rc = bind(s);
  if (rc) return rc;
  if ((rc = check_ready(s, slot))) return rc;
  DevTensor& t = s->slots[slot];
  if ((rc = prepare_stream(s, t, nullptr))) return rc;
  KView v = make_view(s, t, true);
  v.max_ctas = (int)s->opt_max_ctas;
  if (!ws_supported(v)) return fail(s, FTKCU_ERR_ARG, "write-back ceiling: N = 3, J = R = 32 only");
  int64_t mul = 1, add = 0;
  tile_perm(seed, v.ntiles, &mul, &add);
  const DevModel& m = s->model;
  size_t total = 0;
  for (int n = 0; n < m.order; ++n) total += (size_t)m.dims[n] * 32;
  float* buf = nullptr;
  float** ptrs = nullptr;
  CK(cudaMalloc(&buf, sizeof(float) * total));
  CK(cudaMalloc(&ptrs, sizeof(float*) * m.order));
  float* h[kMaxOrder];
  size_t off = 0;
  for (int n = 0; n < m.order; ++n) {
    h[n] = buf + off;
    off += (size_t)m.dims[n] * 32;
  }
  CK(cudaMemcpyAsync(ptrs, h, sizeof(float*) * m.order, cudaMemcpyHostToDevice, s->stream));
  CK(cudaMemsetAsync(buf, 0, sizeof(float) * total, s->stream));
  CK(cudaEventRecord(s->ev0, s->stream));
  CK(launch_ws_writeback(v, m.dims, mul, add, ptrs, s->stream));
  s->launches += 1;
  rc = finish_timing(s, ms);
  CK(cudaStreamSynchronize(s->stream));
  CK(cudaFree(ptrs));
  CK(cudaFree(buf));
  return rc;
}

// Bucket / row / batch offsets of the baselines' plans: span [0, nnz] and
// strictly increasing (an empty batch would divide by m_eff = 0 in the
// kernels and read perm[nnz]).
static int check_offsets(ftkcu_session* s, const int64_t* off, int64_t n, int64_t nnz,
                         const char* what) {
  if (n == 0) return nnz == 0 ? FTKCU_OK : fail(s, FTKCU_ERR_ARG, "%s: no batches", what);
  if (off[0] != 0 || off[n] != nnz) return fail(s, FTKCU_ERR_ARG, "%s must span [0, nnz]", what);
  for (int64_t i = 0; i < n; ++i)
    if (off[i + 1] <= off[i])
      return fail(s, FTKCU_ERR_ARG, "%s must be strictly increasing (entry %lld)", what,
                  (long long)i);
  return FTKCU_OK;
}

// ---- FastTucker baseline (epoch_fasttucker, decomposition.cpp:707-770) ----

int ftkcu_fasttucker_factor(ftkcu_session* s, int slot, int mode, const int64_t* perm,
                            const int64_t* bucket_off, int64_t nbuckets, int32_t M, float lr_a,
                            float reg_a, double* ms) {
  int rc = bind(s);
  if (rc) return rc;
  if ((rc = check_ready(s, slot))) return rc;
  DevTensor& t = s->slots[slot];
  if (M < 1) return fail(s, FTKCU_ERR_ARG, "batch size must be positive");
  if (mode < 0 || mode >= t.order) return fail(s, FTKCU_ERR_ARG, "mode %d out of range", mode);
  if (nbuckets < 0 || (t.nnz > 0 && (!perm || !bucket_off)))
    return fail(s, FTKCU_ERR_ARG, "per-bucket plan missing");
  if ((rc = check_offsets(s, bucket_off, nbuckets, t.nnz, "bucket offsets"))) return rc;
  KView v = make_view(s, t, false);
  if (ft_factor_smem(v, M, mode) > 227 * 1024)
    return fail(s, FTKCU_ERR_ARG, "batch too large for the FastTucker factor block");
  if ((rc = upload_perm(s, perm, t.nnz, t.nnz))) return rc;
  if ((size_t)(nbuckets + 1) > s->boff_cap) {
    if (s->d_boff) CK(cudaFree(s->d_boff));
    s->d_boff = nullptr;
    CK(cudaMalloc(&s->d_boff, sizeof(int64_t) * (nbuckets + 1)));
    s->boff_cap = nbuckets + 1;
  }
  CK(cudaMemcpyAsync(s->d_boff, bucket_off, sizeof(int64_t) * (nbuckets + 1),
                     cudaMemcpyHostToDevice, s->stream));
  CK(cudaEventRecord(s->ev0, s->stream));
  CK(launch_ft_factor(v, mode, s->d_perm, s->d_boff, nbuckets, M, lr_a, reg_a, s->stream));
  s->launches += 1;
  return finish_timing(s, ms);
}

int ftkcu_fasttucker_core(ftkcu_session* s, int slot, int mode, const int64_t* perm, int32_t M,
                          float lr_b, float reg_b, int schedule, double* ms) {
  int rc = bind(s);
  if (rc) return rc;
  if ((rc = check_ready(s, slot))) return rc;
  DevTensor& t = s->slots[slot];
  if (M < 1) return fail(s, FTKCU_ERR_ARG, "batch size must be positive");
  if (mode < 0 || mode >= t.order) return fail(s, FTKCU_ERR_ARG, "mode %d out of range", mode);
  if (t.nnz > 0 && !perm) return fail(s, FTKCU_ERR_ARG, "global plan missing");
  KView v = make_view(s, t, false);
  if (ft_core_smem(v, M) > 227 * 1024)
    return fail(s, FTKCU_ERR_ARG, "batch too large for the FastTucker core block");
  if ((rc = upload_perm(s, perm, t.nnz, t.nnz))) return rc;
  CK(cudaEventRecord(s->ev0, s->stream));
  if (schedule != FTKCU_MODE_DETERMINISTIC && schedule != FTKCU_MODE_HOGWILD)
    return fail(s, FTKCU_ERR_ARG, "unknown schedule %d", schedule);
  CK(launch_ft_core(v, mode, s->d_perm, M, lr_b, reg_b, schedule == FTKCU_MODE_HOGWILD,
                    s->stream));
  s->launches += 1;
  return finish_timing(s, ms);
}

// ---- FasterTucker baseline (epoch_fastertucker, decomposition.cpp:772-843) --

static int ensure_ccache(ftkcu_session* s) {
  DevModel& m = s->model;
  for (int n = 0; n < m.order; ++n)
    if (!m.cc[n]) CK(cudaMalloc(&m.cc[n], sizeof(float) * ((size_t)m.dims[n] * m.r + 1)));
  return FTKCU_OK;
}

int ftkcu_ccache_upload(ftkcu_session* s, const float* const* C) {
  int rc = bind(s);
  if (rc) return rc;
  if (!s->have_model) return fail(s, FTKCU_ERR_STATE, "no model uploaded");
  if (!C) return fail(s, FTKCU_ERR_ARG, "null cache");
  if ((rc = ensure_ccache(s))) return rc;
  const DevModel& m = s->model;
  for (int n = 0; n < m.order; ++n)
    CK(cudaMemcpyAsync(m.cc[n], C[n], sizeof(float) * (size_t)m.dims[n] * m.r,
                       cudaMemcpyHostToDevice, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return FTKCU_OK;
}

int ftkcu_ccache_download(ftkcu_session* s, float* const* C) {
  int rc = bind(s);
  if (rc) return rc;
  const DevModel& m = s->model;
  if (!s->have_model || !m.cc[0]) return fail(s, FTKCU_ERR_STATE, "no C cache on the device");
  if (!C) return fail(s, FTKCU_ERR_ARG, "null cache");
  for (int n = 0; n < m.order; ++n)
    CK(cudaMemcpyAsync(C[n], m.cc[n], sizeof(float) * (size_t)m.dims[n] * m.r,
                       cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return FTKCU_OK;
}

static int fst_view(ftkcu_session* s, int slot, int mode, KView* out) {
  int rc = check_ready(s, slot);
  if (rc) return rc;
  DevTensor& t = s->slots[slot];
  if (t.order < 2) return fail(s, FTKCU_ERR_ARG, "FasterTucker needs order >= 2");
  if (mode < 0 || mode >= t.order) return fail(s, FTKCU_ERR_ARG, "mode %d out of range", mode);
  if (!s->model.cc[0]) return fail(s, FTKCU_ERR_STATE, "C cache must be uploaded first");
  *out = make_view(s, t, false);
  for (int n = 0; n < t.order; ++n) out->cc[n] = s->model.cc[n];
  return FTKCU_OK;
}

int ftkcu_fastertucker_factor(ftkcu_session* s, int slot, int mode, const int64_t* perm,
                              const int64_t* row_off, int64_t nrows, float lr_a, float reg_a,
                              double* ms) {
  int rc = bind(s);
  if (rc) return rc;
  KView v;
  if ((rc = fst_view(s, slot, mode, &v))) return rc;
  if (nrows < 0 || (v.nnz > 0 && (!perm || !row_off)))
    return fail(s, FTKCU_ERR_ARG, "row-grouped plan missing");
  if ((rc = check_offsets(s, row_off, nrows, v.nnz, "row offsets"))) return rc;
  if ((rc = upload_perm(s, perm, v.nnz, v.nnz))) return rc;
  if ((size_t)(nrows + 1) > s->boff_cap) {
    if (s->d_boff) CK(cudaFree(s->d_boff));
    s->d_boff = nullptr;
    CK(cudaMalloc(&s->d_boff, sizeof(int64_t) * (nrows + 1)));
    s->boff_cap = nrows + 1;
  }
  CK(cudaMemcpyAsync(s->d_boff, row_off, sizeof(int64_t) * (nrows + 1), cudaMemcpyHostToDevice,
                     s->stream));
  CK(cudaEventRecord(s->ev0, s->stream));
  CK(launch_fst_factor(v, mode, s->d_perm, s->d_boff, nrows, lr_a, reg_a, s->stream));
  // the block barrier's cache refresh of this mode (decomposition.cpp:810)
  CK(launch_ccache(v, s->model.dims, s->model.cc, s->stream, mode));
  s->launches += 2;
  return finish_timing(s, ms);
}

int ftkcu_fastertucker_core(ftkcu_session* s, int slot, int mode, const int64_t* perm,
                            const int64_t* batch_off, int64_t nbatches, float lr_b, float reg_b,
                            int schedule, double* ms) {
  int rc = bind(s);
  if (rc) return rc;
  KView v;
  if ((rc = fst_view(s, slot, mode, &v))) return rc;
  if (nbatches < 0 || (v.nnz > 0 && (!perm || !batch_off)))
    return fail(s, FTKCU_ERR_ARG, "plan missing");
  if ((rc = check_offsets(s, batch_off, nbatches, v.nnz, "batch offsets"))) return rc;
  if (v.j[mode] > 128) return fail(s, FTKCU_ERR_ARG, "FasterTucker core block supports J <= 128");
  if ((rc = upload_perm(s, perm, v.nnz, v.nnz))) return rc;
  if ((size_t)(nbatches + 1) > s->boff_cap) {
    if (s->d_boff) CK(cudaFree(s->d_boff));
    s->d_boff = nullptr;
    CK(cudaMalloc(&s->d_boff, sizeof(int64_t) * (nbatches + 1)));
    s->boff_cap = nbatches + 1;
  }
  CK(cudaMemcpyAsync(s->d_boff, batch_off, sizeof(int64_t) * (nbatches + 1),
                     cudaMemcpyHostToDevice, s->stream));
  if (schedule != FTKCU_MODE_DETERMINISTIC && schedule != FTKCU_MODE_HOGWILD)
    return fail(s, FTKCU_ERR_ARG, "unknown schedule %d", schedule);
  const bool scan = schedule == FTKCU_MODE_HOGWILD && fst_scan_supported(v, mode);
  const size_t need = scan ? (size_t)2 * num_sms() * v.j[mode] * v.r
                           : fst_core_scratch_floats(v, mode);
  if ((rc = ensure_scratch(s, sizeof(float) * need))) return rc;
  CK(cudaEventRecord(s->ev0, s->stream));
  if (scan)
    CK(launch_fst_core_scan(v, mode, s->d_perm, s->d_boff, nbatches, lr_b, reg_b,
                            static_cast<float*>(s->scratch), s->stream));
  else
    CK(launch_fst_core(v, mode, s->d_perm, s->d_boff, nbatches, lr_b, reg_b,
                       static_cast<float*>(s->scratch), s->stream));
  CK(launch_ccache(v, s->model.dims, s->model.cc, s->stream, mode));
  s->launches += 2;
  return finish_timing(s, ms);
}

int ftkcu_tensor_set_cells(ftkcu_session* s, int slot, const int64_t* cell_offsets, int ncells) {
  int rc = bind(s);
  if (rc) return rc;
  if (slot < 0 || slot >= 8) return fail(s, FTKCU_ERR_ARG, "tensor slot %d out of range", slot);
  DevTensor& t = s->slots[slot];
  if ((rc = finish_upload(s, t))) return rc;
  if (ncells < 1 || !cell_offsets) return fail(s, FTKCU_ERR_ARG, "need at least one cell");
  if (cell_offsets[0] != 0 || cell_offsets[ncells] != t.nnz)
    return fail(s, FTKCU_ERR_ARG, "cell offsets must span [0, nnz]");
  for (int c = 0; c < ncells; ++c)
    if (cell_offsets[c + 1] < cell_offsets[c]) return fail(s, FTKCU_ERR_ARG, "cell offsets not sorted");
  t.cell_off.assign(cell_offsets, cell_offsets + ncells + 1);
  t.keep_order = s->opt_cell_order != 0 && t.order == 3;
  t.shuffled = false;
  return FTKCU_OK;
}

// Storage scheme: (re)builds C_n = A_n B_n for every mode from the current
// model, as the reference does at the start of each core phase (outside its
// timed region, decomposition.cpp:668-670), and points the view at it.
int prepare_ccache(ftkcu_session* s, KView& v) {
  DevModel& m = s->model;
  for (int n = 0; n < m.order; ++n)
    if (!m.cc[n]) CK(cudaMalloc(&m.cc[n], sizeof(float) * ((size_t)m.dims[n] * m.r + 1)));
  CK(launch_ccache(v, m.dims, m.cc, s->stream));
  s->launches += m.order;
  for (int n = 0; n < m.order; ++n) v.cc[n] = m.cc[n];
  return FTKCU_OK;
}

int ftkcu_core_phase(ftkcu_session* s, int slot, const int64_t* perm, int32_t M, float lr_b,
                     float reg_b, int mode, uint64_t seed, float* grad_out, double* ms) {
  int rc = bind(s);
  if (rc) return rc;
  if ((rc = check_f16_range(s))) return rc;
  if ((rc = check_ready(s, slot))) return rc;
  if (M < 1) return fail(s, FTKCU_ERR_ARG, "batch size must be positive");
  DevTensor& t = s->slots[slot];
  if (t.nnz <= 0) return fail(s, FTKCU_ERR_EMPTY, "apply_core_update: empty tensor");
  const size_t glen = (size_t)s->model.sum_j() * s->model.r;
  KView v;
  if (mode == FTKCU_MODE_DETERMINISTIC) {
    if (!perm) return fail(s, FTKCU_ERR_ARG, "deterministic mode needs a permutation");
    if ((rc = upload_perm(s, perm, t.nnz, t.nnz))) return rc;
    v = make_view(s, t, false);
    if (s->opt_store_c && (rc = prepare_ccache(s, v))) return rc;
    CK(cudaEventRecord(s->ev0, s->stream));
    CK(cudaMemsetAsync(s->grad, 0, sizeof(float) * glen, s->stream));
    CK(launch_det_core(v, s->d_perm, M, s->grad, DetDebug{}, s->stream));
    s->launches += 1;
    s->last_core_kernel = FTKCU_K_DET;
  } else if (mode == FTKCU_MODE_HOGWILD) {
    if ((rc = prepare_stream(s, t, perm))) return rc;
    v = make_view(s, t, true);
    v.max_ctas = (int)s->opt_max_ctas;  // grid cap (tests: many tiles per CTA)
    int64_t mul = 1, add = 0;
    if (!perm) tile_perm(seed ^ 0xc0e5ull, v.ntiles, &mul, &add);
    size_t need = (size_t)num_sms() * 16 * glen * sizeof(float);
    const size_t hog_need = hog_core_scratch_bytes(v, (int)s->opt_hog_bps);
    if (hog_need > need) need = hog_need;
    if (big_supported(v) && big_scratch_bytes(v, s->model.dims, true) > need)
      need = big_scratch_bytes(v, s->model.dims, true);
    if (ws_supported(v) && ws_core_scratch_bytes(v, s->model.dims) > need)
      need = ws_core_scratch_bytes(v, s->model.dims);
    if (wsg_supported(v) && wsg_core_scratch_bytes(v, s->model.dims) > need)
      need = wsg_core_scratch_bytes(v, s->model.dims);
    if ((rc = ensure_scratch(s, need))) return rc;
    if (s->opt_store_c && (rc = prepare_ccache(s, v))) return rc;
    CK(cudaEventRecord(s->ev0, s->stream));
    // Storage scheme: the WS sweep reads C rows from the cache (no C GEMM);
    // other tensor-core shapes take the CUDA-core sweep, which reads them too.
    if (s->opt_precision != FTKCU_PREC_FP32 && s->opt_tc_ws && ws_supported(v)) {
      CK(launch_ws_core(v, s->model.dims, mul, add, s->grad, (int)s->opt_precision,
                        (int)s->opt_core16, static_cast<float*>(s->scratch), s->scratch_bytes,
                        s->stream));
      s->last_core_kernel = s->opt_store_c ? FTKCU_K_WS_CC
                            : (s->opt_precision == FTKCU_PREC_TF32 && s->opt_core16) ? FTKCU_K_WS16
                                                                                     : FTKCU_K_WS;
    } else if (s->opt_precision == FTKCU_PREC_TF32 && !s->opt_store_c && s->opt_tc_ws &&
               s->opt_core16 && wsg_supported(v)) {
      CK(launch_wsg_core(v, s->model.dims, mul, add, s->grad, static_cast<float*>(s->scratch),
                         s->scratch_bytes, s->stream));
      s->last_core_kernel = FTKCU_K_WSG;
    } else if (s->opt_precision == FTKCU_PREC_TF32 && !s->opt_store_c && big_supported(v)) {
      CK(launch_big_core(v, s->model.dims, mul, add, s->grad, static_cast<float*>(s->scratch),
                         s->scratch_bytes, s->stream));
      s->last_core_kernel = FTKCU_K_BIG;
    } else if (s->opt_precision != FTKCU_PREC_FP32 && !s->opt_store_c && tc_supported(v)) {
      CK(launch_tc_core(v, mul, add, s->grad, (int)s->opt_precision,
                        static_cast<float*>(s->scratch), s->scratch_bytes, s->stream));
      s->last_core_kernel = FTKCU_K_TC;
    } else {
      CK(launch_hog_core(v, mul, add, s->grad, (int)s->opt_hog_bps,
                         static_cast<float*>(s->scratch), s->scratch_bytes, s->stream));
      s->last_core_kernel = FTKCU_K_HOG;
    }
    s->launches += 2;
  } else {
    return fail(s, FTKCU_ERR_ARG, "unknown mode %d", mode);
  }
  if (s->comm && s->world > 1) {
    NK(ncclAllReduce(s->grad, s->grad, glen, ncclFloat, ncclSum, s->comm, s->stream));
    v.nnz = s->global_nnz > 0 ? s->global_nnz : v.nnz;  // |Omega| over all ranks
  }
  CK(launch_apply_core(v, s->grad, lr_b, reg_b, s->stream));
  s->launches += 1;
  if ((rc = finish_timing(s, ms))) return rc;
  if (grad_out) {
    CK(cudaMemcpyAsync(grad_out, s->grad, sizeof(float) * glen, cudaMemcpyDeviceToHost,
                       s->stream));
    CK(cudaStreamSynchronize(s->stream));
  }
  return FTKCU_OK;
}

int ftkcu_eval(ftkcu_session* s, int slot, int workers, double reg_a, double reg_b,
               double* out3) {
  int rc = bind(s);
  if (rc) return rc;
  if ((rc = check_f16_range(s))) return rc;
  if ((rc = check_ready(s, slot))) return rc;
  if (!out3) return fail(s, FTKCU_ERR_ARG, "null output");
  const DevTensor& t = s->slots[slot];
  if ((rc = ensure_scratch(s, eval_scratch_bytes(s->model, t, workers)))) return rc;
  CK(run_eval(s->model, t, workers, reg_a, reg_b, s->opt_eval == FTKCU_EVAL_EXACT, out3,
              s->scratch, s->scratch_bytes, s->stream));
  s->launches += 2 + s->model.order;
  return FTKCU_OK;
}

int ftkcu_batch_probe(ftkcu_session* s, int slot, const int64_t* rows, int m_eff, int cap,
                      float lr_a, float reg_a, float* C, float* D, float* U, float* xhat_f,
                      float* resid_f, float* xhat_c, float* resid_c, float* A_new, float* G) {
  int rc = bind(s);
  if (rc) return rc;
  if ((rc = check_ready(s, slot))) return rc;
  if (cap < 1 || m_eff < 0 || m_eff > cap) return fail(s, FTKCU_ERR_ARG, "batch overflow");
  if ((rc = upload_perm(s, rows, m_eff, s->slots[slot].nnz))) return rc;
  const DevModel& m = s->model;
  const int order = m.order, r = m.r, jmax = m.max_j();
  const size_t n_cr = (size_t)order * cap * r, n_cj = (size_t)order * cap * jmax;
  const size_t n_g = (size_t)order * jmax * r;
  const size_t glen = (size_t)m.sum_j() * r;
  const size_t floats = 2 * n_cr + 2 * n_cj + 4 * (size_t)cap + glen;
  if ((rc = ensure_scratch(s, floats * sizeof(float)))) return rc;
  float* base = static_cast<float*>(s->scratch);
  float *dc = base, *dd = dc + n_cr, *du = dd + n_cr, *da = du + n_cj;
  float *dxf = da + n_cj, *drf = dxf + cap, *dxc = drf + cap, *drc = dxc + cap;
  float* dg = drc + cap;
  CK(cudaMemsetAsync(base, 0, floats * sizeof(float), s->stream));
  KView v = make_view(s, s->slots[slot], false);
  v.nnz = m_eff;  // the probe batch is the whole "epoch"
  DetDebug dbg_core{};
  dbg_core.xhat = dxc;
  dbg_core.resid = drc;
  dbg_core.jmax = jmax;
  if (m_eff > 0) CK(launch_det_core(v, s->d_perm, cap, dg, dbg_core, s->stream));
  DetDebug dbg{};
  dbg.c = dc;
  dbg.d = dd;
  dbg.u = du;
  dbg.xhat = dxf;
  dbg.resid = drf;
  dbg.jmax = jmax;
  if (m_eff > 0) CK(launch_det_factor(v, s->d_perm, cap, lr_a, reg_a, dbg, s->stream));
  if (m_eff > 0)
    gather_rows_kernel<<<32, 256, 0, s->stream>>>(v, s->d_perm, m_eff, cap, jmax, da);
  CK(cudaGetLastError());
  auto d2h = [&](float* dst, const float* src, size_t n) -> int {
    if (dst) CK(cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToHost, s->stream));
    return FTKCU_OK;
  };
  if ((rc = d2h(C, dc, n_cr)) || (rc = d2h(D, dd, n_cr)) || (rc = d2h(U, du, n_cj)) ||
      (rc = d2h(A_new, da, n_cj)) || (rc = d2h(xhat_f, dxf, cap)) || (rc = d2h(resid_f, drf, cap)) ||
      (rc = d2h(xhat_c, dxc, cap)) || (rc = d2h(resid_c, drc, cap)))
    return rc;
  std::vector<float> hg(glen);
  CK(cudaMemcpyAsync(hg.data(), dg, glen * sizeof(float), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  if (G) {
    std::memset(G, 0, n_g * sizeof(float));
    size_t off = 0;
    for (int n = 0; n < order; ++n) {
      for (int j = 0; j < m.ranks[n]; ++j)
        for (int c = 0; c < r; ++c) G[((size_t)n * jmax + j) * r + c] = hg[off + (size_t)j * r + c];
      off += (size_t)m.ranks[n] * r;
    }
  }
  return FTKCU_OK;
}

int ftkcu_comm_unique_id(uint8_t* id128) {
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, FTKCU_ERR_NCCL, "ncclGetUniqueId: %s",
                                    ncclGetErrorString(r));
  static_assert(sizeof(id) == 128, "nccl unique id size");
  std::memcpy(id128, &id, 128);
  return FTKCU_OK;
}

int ftkcu_comm_init(ftkcu_session* s, const uint8_t* id128, int rank, int world) {
  int rc = bind(s);
  if (rc) return rc;
  if (world < 1 || rank < 0 || rank >= world) return fail(s, FTKCU_ERR_ARG, "bad rank/world");
  if (s->comm) {
    ncclCommDestroy(s->comm);
    s->comm = nullptr;
  }
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  NK(ncclCommInitRank(&s->comm, world, id, rank));
  s->rank = rank;
  s->world = world;
  return FTKCU_OK;
}

static int rows_of(ftkcu_session* s, int mode, int64_t row0, int64_t nrows, float** ptr,
                   size_t* count) {
  if (!s->have_model) return fail(s, FTKCU_ERR_STATE, "no model uploaded");
  const DevModel& m = s->model;
  if (mode < 0 || mode >= m.order) return fail(s, FTKCU_ERR_ARG, "mode %d out of range", mode);
  if (row0 < 0 || nrows < 0 || row0 + nrows > m.dims[mode])
    return fail(s, FTKCU_ERR_ARG, "row range out of bounds");
  *ptr = m.a[mode] + row0 * m.ranks[mode];
  *count = (size_t)nrows * m.ranks[mode];
  return FTKCU_OK;
}

// Rank r broadcasts rows [off[r], off[r+1]) of `mode`, for every rank r.
static int bcast_blocks(ftkcu_session* s, int mode, const int64_t* off) {
  int rc;
  NK(ncclGroupStart());
  for (int r = 0; r < s->world; ++r) {
    float* p;
    size_t c;
    if ((rc = rows_of(s, mode, off[r], off[r + 1] - off[r], &p, &c))) {
      ncclGroupEnd();
      return rc;
    }
    if (c) NK(ncclBroadcast(p, p, c, ncclFloat, r, s->comm, s->stream));
  }
  NK(ncclGroupEnd());
  return FTKCU_OK;
}

// Ring shift of one block of `mode`: send block `held` to rank-1, receive
// block `held`+1 from rank+1 (DSGD, dsgd.DsgdTrainer._shift).
static int shift_block(ftkcu_session* s, int mode, const int64_t* off, int parts, int held) {
  const int b0 = held % parts, b1 = (held + 1) % parts;
  const int dst = (s->rank - 1 + s->world) % s->world, src = (s->rank + 1) % s->world;
  float *sp, *rp;
  size_t sc, rcn;
  int rc;
  if ((rc = rows_of(s, mode, off[b0], off[b0 + 1] - off[b0], &sp, &sc))) return rc;
  if ((rc = rows_of(s, mode, off[b1], off[b1 + 1] - off[b1], &rp, &rcn))) return rc;
  NK(ncclGroupStart());
  if (sc) NK(ncclSend(sp, sc, ncclFloat, dst, s->comm, s->stream));
  if (rcn) NK(ncclRecv(rp, rcn, ncclFloat, src, s->comm, s->stream));
  NK(ncclGroupEnd());
  return FTKCU_OK;
}

// One DSGD factor phase on the session stream: P*P cell sweeps, the A3 ring
// shift after every stratum, the A2 shift after every s-round, then the
// all-gather of A2/A3 (world > 1).  Tile permutations come from
// s->d_cellperm so the same enqueue can be captured once and replayed.
static int enqueue_dsgd(ftkcu_session* s, DevTensor& t, int parts, const int64_t* off2,
                        const int64_t* off3, float lr_a, float reg_a) {
  int rc;
  for (int si = 0; si < parts; ++si) {
    for (int ti = 0; ti < parts; ++ti) {
      const int cell = si * parts + ti;
      KView v = make_view(s, t, true);
      v.max_ctas = (int)s->opt_max_ctas;
      v.tile_base = t.cell_tile[cell];
      v.ntiles = t.cell_tile[cell + 1] - t.cell_tile[cell];
      v.tperm = s->d_cellperm + 2 * cell;
      if ((rc = launch_factor(s, v, 1, 0, lr_a, reg_a))) return rc;
      if (parts > 1 && s->opt_dsgd_shift &&
          (rc = shift_block(s, 2, off3, parts, s->rank + ti)))
        return rc;
    }
    if (parts > 1 && s->opt_dsgd_shift && (rc = shift_block(s, 1, off2, parts, s->rank + si)))
      return rc;
  }
  if (s->world > 1) {
    if ((rc = bcast_blocks(s, 1, off2))) return rc;
    if ((rc = bcast_blocks(s, 2, off3))) return rc;
  }
  return FTKCU_OK;
}

int ftkcu_comm_sendrecv_rows(ftkcu_session* s, int mode, int64_t send_row0, int64_t send_nrows,
                             int dst, int64_t recv_row0, int64_t recv_nrows, int src) {
  int rc = bind(s);
  if (rc) return rc;
  if (!s->comm) return fail(s, FTKCU_ERR_STATE, "no communicator");
  float *sp, *rp;
  size_t sc, rcn;
  if ((rc = rows_of(s, mode, send_row0, send_nrows, &sp, &sc))) return rc;
  if ((rc = rows_of(s, mode, recv_row0, recv_nrows, &rp, &rcn))) return rc;
  NK(ncclGroupStart());
  if (sc) NK(ncclSend(sp, sc, ncclFloat, dst, s->comm, s->stream));
  if (rcn) NK(ncclRecv(rp, rcn, ncclFloat, src, s->comm, s->stream));
  NK(ncclGroupEnd());
  return FTKCU_OK;
}

int ftkcu_comm_bcast_rows(ftkcu_session* s, int mode, const int64_t* row_off, int nblocks) {
  int rc = bind(s);
  if (rc) return rc;
  if (!s->comm) return fail(s, FTKCU_ERR_STATE, "no communicator");
  if (nblocks != s->world) return fail(s, FTKCU_ERR_ARG, "need one block per rank");
  return bcast_blocks(s, mode, row_off);
}

int ftkcu_comm_allreduce_f64(ftkcu_session* s, double* host_inout, int n) {
  int rc = bind(s);
  if (rc) return rc;
  if (!s->comm) return fail(s, FTKCU_ERR_STATE, "no communicator");
  if ((rc = ensure_scratch(s, sizeof(double) * (n > 0 ? n : 1)))) return rc;
  double* d = static_cast<double*>(s->scratch);
  CK(cudaMemcpyAsync(d, host_inout, sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
  NK(ncclAllReduce(d, d, n, ncclDouble, ncclSum, s->comm, s->stream));
  CK(cudaMemcpyAsync(host_inout, d, sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return FTKCU_OK;
}

int ftkcu_stream_sync(ftkcu_session* s) {
  int rc = bind(s);
  if (rc) return rc;
  CK(cudaStreamSynchronize(s->stream));
  CK(cudaStreamSynchronize(s->rb_stream));
  return check_f16_range(s);
}

int ftkcu_dsgd_factor_epoch(ftkcu_session* s, int slot, int parts, const int64_t* row_off2,
                            const int64_t* row_off3, const uint64_t* cell_seeds, float lr_a,
                            float reg_a, double* ms) {
  int rc = bind(s);
  if (rc) return rc;
  if ((rc = check_ready(s, slot))) return rc;
  DevTensor& t = s->slots[slot];
  if (t.order != 3) return fail(s, FTKCU_ERR_ARG, "DSGD strata need an order-3 tensor");
  if (parts < 1 || !row_off2 || !row_off3 || !cell_seeds)
    return fail(s, FTKCU_ERR_ARG, "bad DSGD arguments");
  const int ncell = parts * parts;
  if ((int)t.cell_off.size() != ncell + 1)
    return fail(s, FTKCU_ERR_ARG, "tensor has %d cells, DSGD over %d parts needs %d",
                (int)t.cell_off.size() - 1, parts, ncell);
  if (parts > 1 && !s->comm) return fail(s, FTKCU_ERR_STATE, "DSGD over > 1 part needs a communicator");
  if (s->world > 1 && parts != s->world)
    return fail(s, FTKCU_ERR_ARG, "parts (%d) must equal the communicator size (%d)", parts,
                s->world);
  const int64_t* offs[2] = {row_off2, row_off3};
  for (int m = 0; m < 2; ++m) {
    if (offs[m][0] != 0 || offs[m][parts] != s->model.dims[m + 1])
      return fail(s, FTKCU_ERR_ARG, "mode-%d block offsets must span [0, %d]", m + 2,
                  s->model.dims[m + 1]);
    for (int p = 0; p < parts; ++p)
      if (offs[m][p + 1] < offs[m][p]) return fail(s, FTKCU_ERR_ARG, "block offsets not sorted");
  }
  if ((rc = prepare_stream(s, t, nullptr))) return rc;
  {
    const KView v = make_view(s, t, true);
    if (big_supported(v) && (rc = ensure_scratch(s, big_scratch_bytes(v, s->model.dims, false))))
      return rc;
  }
  if ((size_t)ncell > s->cellperm_cap) {
    if (s->d_cellperm) CK(cudaFree(s->d_cellperm));
    s->d_cellperm = nullptr;
    CK(cudaMalloc(&s->d_cellperm, sizeof(int64_t) * 2 * ncell));
    s->cellperm_cap = ncell;
  }
  std::vector<int64_t> perm(2 * (size_t)ncell);
  for (int c = 0; c < ncell; ++c)
    tile_perm(cell_seeds[c], t.cell_tile[c + 1] - t.cell_tile[c], &perm[2 * c], &perm[2 * c + 1]);
  CK(cudaEventRecord(s->ev0, s->stream));
  // pageable source: staged before the call returns, so `perm` may go away
  CK(cudaMemcpyAsync(s->d_cellperm, perm.data(), sizeof(int64_t) * 2 * ncell,
                     cudaMemcpyHostToDevice, s->stream));
  if (!s->opt_graphs) {
    if ((rc = enqueue_dsgd(s, t, parts, row_off2, row_off3, lr_a, reg_a))) return rc;
    return finish_timing(s, ms);
  }
  uint32_t lr_bits, reg_bits;
  std::memcpy(&lr_bits, &lr_a, 4);
  std::memcpy(&reg_bits, &reg_a, 4);
  std::vector<int64_t> key = {slot, parts, s->rank, s->world, (int64_t)lr_bits,
                              (int64_t)reg_bits, s->opt_precision, s->opt_hog_update,
                              s->opt_tc_ws, s->opt_max_ctas, s->opt_hog_bps,
                              (int64_t)(intptr_t)s->comm, (int64_t)(intptr_t)s->d_cellperm,
                              (int64_t)(intptr_t)t.svals, (int64_t)(intptr_t)t.tile_rows};
  for (int n = 0; n < 3; ++n) {
    key.push_back((int64_t)(intptr_t)s->model.a[n]);
    key.push_back((int64_t)(intptr_t)s->model.b[n]);
    key.push_back((int64_t)(intptr_t)t.sidx[n]);
  }
  key.insert(key.end(), row_off2, row_off2 + parts + 1);
  key.insert(key.end(), row_off3, row_off3 + parts + 1);
  key.insert(key.end(), t.cell_tile.begin(), t.cell_tile.end());
  if (!s->dsgd_exec || key != s->dsgd_key) {
    if (s->dsgd_exec) CK(cudaGraphExecDestroy(s->dsgd_exec));
    s->dsgd_exec = nullptr;
    const int64_t before = s->launches;
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeRelaxed));
    rc = enqueue_dsgd(s, t, parts, row_off2, row_off3, lr_a, reg_a);
    const cudaError_t e = cudaStreamEndCapture(s->stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    CK(e);
    const cudaError_t ei = cudaGraphInstantiate(&s->dsgd_exec, g, 0);
    cudaGraphDestroy(g);
    CK(ei);
    s->dsgd_key = key;
    s->dsgd_launches = s->launches - before;
    s->launches = before;
  }
  CK(cudaGraphLaunch(s->dsgd_exec, s->stream));
  s->launches += s->dsgd_launches;
  return finish_timing(s, ms);
}

int ftkcu_comm_allreduce_grad(ftkcu_session* s) {
  int rc = bind(s);
  if (rc) return rc;
  if (!s->comm) return fail(s, FTKCU_ERR_STATE, "no communicator");
  if (!s->have_model) return fail(s, FTKCU_ERR_STATE, "no model uploaded");
  const size_t glen = (size_t)s->model.sum_j() * s->model.r;
  NK(ncclAllReduce(s->grad, s->grad, glen, ncclFloat, ncclSum, s->comm, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return FTKCU_OK;
}

}  // extern "C"

// ---- DSGD ring epochs ----------------------------------------------------------

namespace {
constexpr int kRingFlags = 4096;
// one epoch's tables at the largest ring (kRingFlags cells): tile offsets,
// permutations, cell io, posts (<= 2 per cell), final waits
constexpr size_t kRingTabBytes = 8 * (kRingFlags + 1) + 16 * kRingFlags + 16 * kRingFlags +
                                 32 * kRingFlags + 64;
constexpr uint32_t kRingMagic = 0x52494e47u;  // "RING"
struct RingBlob {
  uint32_t magic;
  int32_t pid;
  int32_t device;
  int32_t pad;
  uint64_t a[3];
  uint64_t flags;
  cudaIpcMemHandle_t ha[3];
  cudaIpcMemHandle_t hf;
};
static_assert(sizeof(RingBlob) <= FTKCU_RING_BLOB_BYTES, "ring blob size");
}  // namespace

#include <unistd.h>

// Everything a ring epoch touches is allocated here, before any rank's
// kernel runs: a device allocation between two ranks' launches would
// serialise virtual ranks sharing one GPU (implicit synchronisation) and
// deadlock their flag waits.
static int ring_buffers(ftkcu_session* s) {
  if (!s->ring_tab) {
    CK(cudaMalloc(&s->ring_tab, kRingTabBytes));
    CK(cudaMallocHost(&s->ring_tab_h, kRingTabBytes));
  }
  if (!s->ring_flags) {
    CK(cudaMalloc(&s->ring_flags, sizeof(unsigned) * kRingFlags));
    CK(cudaMalloc(&s->ring_done, sizeof(unsigned) * 2 * kRingFlags));
    CK(cudaMalloc(&s->ring_err, sizeof(unsigned)));
    CK(cudaMemset(s->ring_flags, 0, sizeof(unsigned) * kRingFlags));
    CK(cudaMemset(s->ring_done, 0, sizeof(unsigned) * 2 * kRingFlags));
    CK(cudaMemset(s->ring_err, 0, sizeof(unsigned)));
  }
  return FTKCU_OK;
}

static int ring_model_ok(ftkcu_session* s) {
  if (!s->have_model || s->model.order != 3)
    return fail(s, FTKCU_ERR_STATE, "ring epochs need an uploaded order-3 model");
  return FTKCU_OK;
}

int ftkcu_ring_export(ftkcu_session* s, uint8_t* blob, int cap) {
  int rc = bind(s);
  if (rc) return rc;
  if (!blob || cap < (int)sizeof(RingBlob)) return fail(s, FTKCU_ERR_ARG, "blob too small");
  if ((rc = ring_model_ok(s)) || (rc = ring_buffers(s))) return rc;
  RingBlob b{};
  b.magic = kRingMagic;
  b.pid = (int32_t)getpid();
  b.device = s->device;
  for (int n = 0; n < 3; ++n) {
    b.a[n] = (uint64_t)(uintptr_t)s->model.a[n];
    CK(cudaIpcGetMemHandle(&b.ha[n], s->model.a[n]));
  }
  b.flags = (uint64_t)(uintptr_t)s->ring_flags;
  CK(cudaIpcGetMemHandle(&b.hf, s->ring_flags));
  std::memset(blob, 0, cap);
  std::memcpy(blob, &b, sizeof(b));
  return FTKCU_OK;
}

// The slot's Hogwild tile stream is built here too (its first build allocates).
static int ring_prepare(ftkcu_session* s, int slot) {
  int rc;
  if ((rc = check_ready(s, slot)) || (rc = ring_model_ok(s)) || (rc = ring_buffers(s))) return rc;
  return prepare_stream(s, s->slots[slot], nullptr);
}

int ftkcu_ring_connect(ftkcu_session* s, int slot, const uint8_t* left_blob, int len) {
  int rc = bind(s);
  if (rc) return rc;
  if (!left_blob || len < (int)sizeof(RingBlob)) return fail(s, FTKCU_ERR_ARG, "bad ring blob");
  if ((rc = ring_prepare(s, slot))) return rc;
  RingBlob b;
  std::memcpy(&b, left_blob, sizeof(b));
  if (b.magic != kRingMagic) return fail(s, FTKCU_ERR_ARG, "not a ring blob");
  for (void*& p : s->ring_ipc)
    if (p) {
      CK(cudaIpcCloseMemHandle(p));
      p = nullptr;
    }
  if (b.pid == (int32_t)getpid()) {  // same process (virtual ranks): plain pointers
    for (int n = 0; n < 3; ++n) s->ring_peer_a[n] = (float*)(uintptr_t)b.a[n];
    s->ring_peer_flags = (unsigned*)(uintptr_t)b.flags;
  } else {
    for (int n = 0; n < 3; ++n) {
      CK(cudaIpcOpenMemHandle(&s->ring_ipc[n], b.ha[n], cudaIpcMemLazyEnablePeerAccess));
      s->ring_peer_a[n] = static_cast<float*>(s->ring_ipc[n]);
    }
    CK(cudaIpcOpenMemHandle(&s->ring_ipc[3], b.hf, cudaIpcMemLazyEnablePeerAccess));
    s->ring_peer_flags = static_cast<unsigned*>(s->ring_ipc[3]);
  }
  CK(cudaMemsetAsync(s->ring_flags, 0, sizeof(unsigned) * kRingFlags, s->stream));
  CK(cudaMemsetAsync(s->ring_err, 0, sizeof(unsigned), s->stream));
  CK(cudaStreamSynchronize(s->stream));
  for (int n = 0; n < 3; ++n) s->ring_model_a[n] = s->model.a[n];
  s->ring_epoch = 0;
  s->ring_emulate = false;
  s->ring_ready = true;
  return FTKCU_OK;
}

int ftkcu_ring_emulate(ftkcu_session* s, int slot) {
  int rc = bind(s);
  if (rc) return rc;
  if ((rc = ring_prepare(s, slot))) return rc;
  for (int n = 0; n < 3; ++n) {
    if (s->ring_emu_a[n]) CK(cudaFree(s->ring_emu_a[n]));
    CK(cudaMalloc(&s->ring_emu_a[n], sizeof(float) * (size_t)s->model.dims[n] * s->model.ranks[n]));
    s->ring_peer_a[n] = s->ring_emu_a[n];
  }
  if (!s->ring_emu_flags) CK(cudaMalloc(&s->ring_emu_flags, sizeof(unsigned) * kRingFlags));
  CK(cudaMemset(s->ring_emu_flags, 0, sizeof(unsigned) * kRingFlags));
  CK(cudaStreamSynchronize(s->stream));
  s->ring_peer_flags = s->ring_emu_flags;
  for (int n = 0; n < 3; ++n) s->ring_model_a[n] = s->model.a[n];
  s->ring_epoch = 0;
  s->ring_emulate = true;
  s->ring_ready = true;
  return FTKCU_OK;
}

int ftkcu_ring_status(ftkcu_session* s, int* timed_out) {
  int rc = bind(s);
  if (rc) return rc;
  if (!timed_out) return fail(s, FTKCU_ERR_ARG, "null argument");
  *timed_out = 0;
  unsigned* e = nullptr;
  if (s->ring_err && s->ring_tab_h) {
    e = reinterpret_cast<unsigned*>(s->ring_tab_h + kRingTabBytes - 16);
    CK(cudaMemcpyAsync(e, s->ring_err, sizeof(unsigned), cudaMemcpyDeviceToHost, s->stream));
  }
  // poll with a sleep instead of a spinning synchronise: ranks sharing one
  // host (virtual ranks, or few cores) must not starve a rank whose kernel
  // the others are waiting for of the CPU it needs to launch
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s->stream);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) CK(q);
    usleep(50);
  }
  if (e) *timed_out = (int)*e;
  return FTKCU_OK;
}

int ftkcu_ring_debug(ftkcu_session* s, uint32_t* flags, uint32_t* done, int n) {
  int rc = bind(s);
  if (rc) return rc;
  if (!s->ring_flags || n < 0 || n > kRingFlags) return fail(s, FTKCU_ERR_ARG, "no ring state");
  CK(cudaStreamSynchronize(s->stream));
  if (flags) CK(cudaMemcpy(flags, s->ring_flags, sizeof(unsigned) * n, cudaMemcpyDeviceToHost));
  if (done) CK(cudaMemcpy(done, s->ring_done, sizeof(unsigned) * n, cudaMemcpyDeviceToHost));
  return FTKCU_OK;
}

int ftkcu_ring_factor_epoch(ftkcu_session* s, int slot, int parts, int rank,
                            const int64_t* row_off2, const int64_t* row_off3,
                            const uint64_t* cell_seeds, float lr_a, float reg_a, double* ms) {
  int rc = bind(s);
  if (rc) return rc;
  if ((rc = check_ready(s, slot))) return rc;
  if (!s->ring_ready) return fail(s, FTKCU_ERR_STATE, "ring not connected (ftkcu_ring_connect / _emulate)");
  for (int n = 0; n < 3; ++n)
    if (s->model.a[n] != s->ring_model_a[n])
      return fail(s, FTKCU_ERR_STATE, "model reallocated since the ring was connected");
  DevTensor& t = s->slots[slot];
  const int P = parts;
  if (P < 2 || rank < 0 || rank >= P || !row_off2 || !row_off3 || !cell_seeds)
    return fail(s, FTKCU_ERR_ARG, "bad ring arguments (parts >= 2, 0 <= rank < parts)");
  // tokens K = mode-3 blocks per rank: the tensor has P * (K P) cells
  const int ncell = (int)t.cell_off.size() - 1, K = ncell / (P * P), Q = K * P;
  if (K < 1 || K > 4 || ncell != P * Q)
    return fail(s, FTKCU_ERR_ARG, "tensor has %d cells, a ring over %d parts needs K*%d (K = 1..4)",
                ncell, P, P * P);
  if ((P + 1) * (Q + P) > kRingFlags || ncell > kRingFlags)
    return fail(s, FTKCU_ERR_ARG, "too many ring parts");
  if (s->world > 1 && (P != s->world || rank != s->rank))
    return fail(s, FTKCU_ERR_ARG, "parts/rank disagree with the communicator");
  const int64_t* offs[2] = {row_off2, row_off3};
  const int nb[2] = {P, Q};
  for (int m = 0; m < 2; ++m) {
    if (offs[m][0] != 0 || offs[m][nb[m]] != s->model.dims[m + 1])
      return fail(s, FTKCU_ERR_ARG, "mode-%d block offsets must span [0, %d]", m + 2,
                  s->model.dims[m + 1]);
    for (int p = 0; p < nb[m]; ++p)
      if (offs[m][p + 1] < offs[m][p]) return fail(s, FTKCU_ERR_ARG, "block offsets not sorted");
  }
  if (s->opt_precision != FTKCU_PREC_TF32 || !s->opt_hog_update)
    return fail(s, FTKCU_ERR_ARG, "ring epochs run the tf32 accumulate sweep");
  // (re)build the tile stream if the tensor was re-uploaded since connect; on
  // a GPU shared by virtual ranks that must happen before any rank's epoch
  // (its first build allocates, which would serialise their kernels)
  if ((rc = prepare_stream(s, t, nullptr))) return rc;
  KView v = make_view(s, t, true);
  v.max_ctas = (int)s->opt_max_ctas;
  if (!ws_supported(v)) return fail(s, FTKCU_ERR_ARG, "ring epochs need N = 3, J = R = 32");
  // tables: flag ids F3(round, block) / F2(round, block), rounds 0..P
  auto F3 = [&](int r, int x) { return r * Q + x; };
  auto F2 = [&](int r, int y) { return (P + 1) * Q + r * P + y; };
  std::vector<int64_t> perm(2 * (size_t)ncell);
  std::vector<int4> io(ncell), posts;
  for (int c = 0; c < ncell; ++c)
    tile_perm(cell_seeds[c], t.cell_tile[c + 1] - t.cell_tile[c], &perm[2 * c], &perm[2 * c + 1]);
  const int g = rank;
  for (int sr = 0; sr < P; ++sr)
    for (int i = 0; i < Q; ++i) {
      const int c = sr * Q + i, x = (K * g + i) % Q, y = (g + sr) % P;
      int4 e = make_int4(-1, -1, -1, -1);
      if (sr > 0 || i >= K) e.x = F3(sr, x);  // blocks Kg .. Kg+K-1 are held at the start
      if (i == 0 && sr > 0) e.y = F2(sr, y);
      // the mode-3 block goes to rank g-1, which sweeps it K steps later
      e.z = (int)posts.size();
      posts.push_back(make_int4(2, (int)row_off3[x], (int)(row_off3[x + 1] - row_off3[x]),
                                F3(sr + (i + K >= Q ? 1 : 0), x)));
      if (i == Q - 1) {  // round end: the mode-2 block follows for round sr+1
        e.w = (int)posts.size();
        posts.push_back(make_int4(1, (int)row_off2[y], (int)(row_off2[y + 1] - row_off2[y]),
                                  F2(sr + 1, y)));
      }
      io[c] = e;
    }
  int finals[5] = {F2(P, g), -1, -1, -1, -1};
  for (int q = 0; q < K; ++q) finals[1 + q] = F3(P, (K * g + q) % Q);
  const size_t b_tile = sizeof(int64_t) * (ncell + 1), b_perm = sizeof(int64_t) * perm.size();
  const size_t b_io = sizeof(int4) * ncell, b_post = sizeof(int4) * posts.size();
  const size_t o_perm = (b_tile + 15) / 16 * 16, o_io = o_perm + (b_perm + 15) / 16 * 16;
  const size_t o_post = o_io + b_io, o_fin = o_post + b_post, total = o_fin + sizeof(finals);
  if (total + 16 > kRingTabBytes) return fail(s, FTKCU_ERR_ARG, "ring tables too large");
  // the pinned staging is reused: the previous epoch's copy must have run
  CK(cudaStreamSynchronize(s->stream));
  uint8_t* h = s->ring_tab_h;
  std::memcpy(h, t.cell_tile.data(), b_tile);
  std::memcpy(h + o_perm, perm.data(), b_perm);
  std::memcpy(h + o_io, io.data(), b_io);
  std::memcpy(h + o_post, posts.data(), b_post);
  std::memcpy(h + o_fin, finals, sizeof(finals));
  CK(cudaEventRecord(s->ev0, s->stream));
  CK(cudaMemcpyAsync(s->ring_tab, h, total, cudaMemcpyHostToDevice, s->stream));
  CK(cudaMemsetAsync(s->ring_done, 0, sizeof(unsigned) * ncell, s->stream));
  CK(cudaMemsetAsync(s->ring_done + kRingFlags, 0, sizeof(unsigned) * (P + ncell), s->stream));
  CK(cudaMemsetAsync(s->ring_err, 0, sizeof(unsigned), s->stream));
  RingDev r;
  r.ncell = ncell;
  r.parts = P;
  r.copied = s->ring_done + kRingFlags;
  r.emulate = s->ring_emulate ? 1 : 0;
  r.epoch = ++s->ring_epoch;
  r.cell_tile = reinterpret_cast<const int64_t*>(s->ring_tab);
  r.cell_perm = reinterpret_cast<const int64_t*>(s->ring_tab + o_perm);
  r.cell_io = reinterpret_cast<const int4*>(s->ring_tab + o_io);
  r.posts = reinterpret_cast<const int4*>(s->ring_tab + o_post);
  r.final_waits = reinterpret_cast<const int*>(s->ring_tab + o_fin);
  r.nfinal = 1 + K;
  r.done = s->ring_done;
  r.flags = s->ring_flags;
  r.peer_flags = s->ring_peer_flags;
  for (int n = 0; n < 3; ++n) r.peer_a[n] = s->ring_peer_a[n];
  r.err = s->ring_err;
  if (s->opt_ring_timeout_ms > 0) r.timeout_cycles = (long long)s->opt_ring_timeout_ms * 2000000ll;
  CK(launch_ws_factor_ring(v, s->model.dims, r, lr_a, reg_a, s->stream));
  s->launches += 1;
  s->last_factor_kernel = FTKCU_K_WS;
  if (s->world > 1 && s->comm) {
    std::vector<int64_t> held3(P + 1);
    for (int p = 0; p <= P; ++p) held3[p] = row_off3[K * p];
    if ((rc = bcast_blocks(s, 1, row_off2))) return rc;
    if ((rc = bcast_blocks(s, 2, held3.data()))) return rc;
  }
  return finish_timing(s, ms);
}
