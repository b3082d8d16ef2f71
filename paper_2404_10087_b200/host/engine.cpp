// The device bridge: ftk::epoch_plus, ftk::train, ftk::loss, ftk::evaluate
// implemented over the C-ABI (include/ftkcu.h), plus history I/O and the
// analytic cost billing.  Reference: decomposition.cpp:623-705 (epoch_plus),
// :849-948 (train, history), evaluation.cpp:36-72 (loss, evaluate).
//
// Device state: one process-wide ftkcu_session (device from DeviceOptions
// or $FTK_DEVICE), with up to 8 host tensors cached on the device keyed by
// their buffers and a content fingerprint (a SparseTensor is read-only after
// construction, sparse_tensor.hpp:11-13).  epoch_plus syncs the model
// H2D/D2H around each call; train keeps it resident for all epochs.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <charconv>
#include <fstream>
#include <limits>
#include <mutex>
#include <sstream>
#include <thread>
#include <vector>

#include "ftk/decomposition.hpp"
#include "ftkcu.h"

namespace ftk {

namespace {

struct SlotKey {
  const void* vals = nullptr;
  const void* idx = nullptr;
  size64 nnz = -1;
  int order = 0;
  std::uint64_t fp = 0;
  std::uint64_t used = 0;
};

struct Engine {
  ftkcu_session* s = nullptr;
  SlotKey slots[8];
  std::uint64_t tick = 0;
  const Model* model_owner = nullptr;
};

std::mutex g_mu;
Engine g_eng;
DeviceOptions g_opts;

void check(int rc) {
  if (rc != FTKCU_OK) fail(ftkcu_last_error(g_eng.s));
}

ftkcu_session* session() {
  if (g_eng.s) return g_eng.s;
  int dev = g_opts.device;
  if (dev < 0) {
    const char* e = std::getenv("FTK_DEVICE");
    dev = e ? std::atoi(e) : 0;
  }
  ftkcu_session* s = nullptr;
  if (ftkcu_session_create(dev, &s) != FTKCU_OK) fail(ftkcu_last_error(nullptr));
  g_eng.s = s;
  return s;
}

void apply_options(ftkcu_session* s) {
  const int prec = g_opts.precision == DevicePrecision::kFp32   ? FTKCU_PREC_FP32
                   : g_opts.precision == DevicePrecision::kTf32 ? FTKCU_PREC_TF32
                                                                : FTKCU_PREC_3XTF32;
  check(ftkcu_set_option(s, "precision", prec));
  check(ftkcu_set_option(s, "eval", g_opts.exact_eval ? FTKCU_EVAL_EXACT : FTKCU_EVAL_FAST));
  int64_t sms = 0;
  check(ftkcu_get_option(s, "num_sms", &sms));
  check(ftkcu_set_option(s, "window", g_opts.parity ? 3 : 0));
  check(ftkcu_set_option(s, "max_ctas", g_opts.parity ? std::max<int64_t>(1, sms / 2) : 0));
}

// Content hash of every index and value byte (a sampled
// fingerprint missed in-place edits at unsampled positions).  Chunks are
// hashed on parallel threads and combined in chunk order, so the result does
// not depend on the thread count; at 1.6 GB (Netflix shape) it is bound by
// host memory bandwidth, tens of ms, once per train() and per epoch_plus().
std::uint64_t hash_bytes(const void* data, std::size_t bytes) {
  const auto* p = static_cast<const unsigned char*>(data);
  constexpr std::size_t kChunk = std::size_t{1} << 24;
  const std::size_t chunks = (bytes + kChunk - 1) / kChunk;
  std::vector<std::uint64_t> part(chunks, 0);
  auto run = [&](std::size_t c) {
    const std::size_t beg = c * kChunk, end = std::min(bytes, beg + kChunk);
    std::uint64_t lanes[4] = {0x9e3779b97f4a7c15ull ^ c, 0xbf58476d1ce4e5b9ull, 0x94d049bb133111ebull,
                              0x2545f4914f6cdd1dull};
    std::size_t i = beg;
    for (; i + 32 <= end; i += 32)
      for (int l = 0; l < 4; ++l) {
        std::uint64_t w;
        std::memcpy(&w, p + i + 8 * l, 8);
        lanes[l] = (lanes[l] ^ w) * 0x100000001b3ull + (lanes[l] >> 29);
      }
    std::uint64_t h = mix64(lanes[0] ^ mix64(lanes[1] ^ mix64(lanes[2] ^ mix64(lanes[3]))));
    for (; i < end; ++i) h = mix64(h ^ p[i]);
    part[c] = h;
  };
  const std::size_t threads =
      std::min<std::size_t>(chunks, std::max(1u, std::thread::hardware_concurrency()));
  if (threads <= 1) {
    for (std::size_t c = 0; c < chunks; ++c) run(c);
  } else {
    std::vector<std::thread> pool;
    for (std::size_t w = 0; w < threads; ++w)
      pool.emplace_back([&, w] {
        for (std::size_t c = w; c < chunks; c += threads) run(c);
      });
    for (auto& th : pool) th.join();
  }
  std::uint64_t h = mix64(bytes);
  for (std::uint64_t x : part) h = mix64(h ^ x);
  return h;
}

std::uint64_t fingerprint(const SparseTensor& t) {
  std::uint64_t h = mix64(static_cast<std::uint64_t>(t.nnz()) ^ (static_cast<std::uint64_t>(t.order) << 56));
  for (index_t d : t.dims) h = mix64(h ^ static_cast<std::uint32_t>(d));
  h = mix64(h ^ hash_bytes(t.indices.data(), t.indices.size() * sizeof(index_t)));
  return mix64(h ^ hash_bytes(t.values.data(), t.values.size() * sizeof(real)));
}

// Returns the device slot holding t, uploading it if needed.
int ensure_tensor(const SparseTensor& t) {
  ftkcu_session* s = session();
  const std::uint64_t fp = fingerprint(t);
  int victim = 0;
  for (int i = 0; i < 8; ++i) {
    SlotKey& k = g_eng.slots[i];
    if (k.vals == t.values.data() && k.idx == t.indices.data() && k.nnz == t.nnz() &&
        k.order == t.order && k.fp == fp) {
      k.used = ++g_eng.tick;
      return i;
    }
    if (k.used < g_eng.slots[victim].used) victim = i;
  }
  require(static_cast<size64>(t.indices.size()) == t.nnz() * t.order, "index storage size mismatch");
  check(ftkcu_tensor_upload(s, victim, t.order, t.dims.data(), t.nnz(), t.indices.data(),
                            t.values.data()));
  g_eng.slots[victim] = {t.values.data(), t.indices.data(), t.nnz(), t.order, fp, ++g_eng.tick};
  return victim;
}

void upload_model(const Model& m) {
  std::vector<const float*> a(m.order()), b(m.order());
  for (int n = 0; n < m.order(); ++n) {
    a[n] = m.a[n].data();
    b[n] = m.b[n].data();
  }
  check(ftkcu_model_upload(session(), m.order(), m.dims.data(), m.ranks.data(), m.r, a.data(),
                           b.data()));
}

void download_model(Model& m) {
  std::vector<float*> a(m.order()), b(m.order());
  for (int n = 0; n < m.order(); ++n) {
    a[n] = m.a[n].data();
    b[n] = m.b[n].data();
  }
  check(ftkcu_model_download(session(), a.data(), b.data()));
}

int device_mode(int workers) {
  if (g_opts.mode == DeviceMode::kDeterministic) return FTKCU_MODE_DETERMINISTIC;
  if (g_opts.mode == DeviceMode::kHogwild) return FTKCU_MODE_HOGWILD;
  return workers == 1 ? FTKCU_MODE_DETERMINISTIC : FTKCU_MODE_HOGWILD;
}

// Analytic replay of the reference's per-batch billing for one phase
// (decomposition.cpp:644-658 factor, :678-703 core).
void bill_phase(CostCounters& cc, const Model& m, size64 nnz, index_t cap, bool factor,
                bool store_c) {
  const int N = m.order();
  const size64 R = m.r;
  const size64 combine = N >= 2 ? N - 2 : 0;
  auto bill = [&](size64 me, size64 k, bool full) {
    if (k == 0 || me == 0) return;
    for (int n = 0; n < N; ++n) cc.count_batches(n, full, k);
    for (int n = 0; n < N; ++n) {
      const size64 J = m.ranks[n];
      cc.add(n, kRead, me * J * k, full);  // staged factor rows
      cc.add(n, kDStage, combine * me * R * k, full);
      if (factor) {
        cc.add(n, kRead, J * R * k, full);  // B^(n)
        cc.add(n, kDStage, me * J * R * k, full);
        cc.add(n, kBdtStage, me * R * J * k, full);
        cc.add(n, kUpdate, me * J * k, full);
      } else {
        if (store_c) {
          cc.add(n, kRead, me * R * k, full);  // cached C rows
        } else {
          cc.add(n, kRead, J * R * k, full);
          cc.add(n, kDStage, me * J * R * k, full);
        }
        cc.add(n, kOther, me * J * k, full);
        cc.add(n, kBdtStage, me * J * R * k, full);
      }
    }
    cc.add(0, kOther, me * (factor ? m.ranks[0] : R) * k, full);
  };
  bill(cap, nnz / cap, true);
  bill(nnz % cap, 1, false);
  if (!factor) {
    if (store_c)
      for (int n = 0; n < N; ++n) cc.add_overhead(kOther, static_cast<size64>(m.dims[n]) * m.ranks[n] * R);
    for (int n = 0; n < N; ++n) cc.add_overhead(kUpdate, static_cast<size64>(m.ranks[n]) * R);
  }
}

// One FastTuckerPlus epoch on the resident model.
EpochStats run_epoch(const SparseTensor& t, int slot, const Model& m, const Hyperparams& h,
                     const EpochOptions& opts, std::uint64_t seed) {
  ftkcu_session* s = session();
  const int workers = resolve_workers(opts.workers);
  const index_t cap = opts.canonical_order ? 1 : h.batch_size;
  const int mode = device_mode(workers);
  EpochStats st;
  st.factor.reset(m.order());
  st.core.reset(m.order());
  const bool need_plan = mode == FTKCU_MODE_DETERMINISTIC || opts.canonical_order;
  double ms_f = 0.0, ms_c = 0.0;
  {
    Rng rng(derive_seed(seed, {1}));
    const int64_t* perm = nullptr;
    EpochPlan plan;
    if (need_plan) {
      plan = opts.canonical_order ? EpochPlan::canonical(t) : EpochPlan::global(t, cap, rng);
      perm = plan.positions().data();
    }
    check(ftkcu_factor_phase(s, slot, perm, cap, h.lr_a, h.reg_a, mode, derive_seed(seed, {1}),
                             &ms_f));
  }
  {
    Rng rng(derive_seed(seed, {2}));
    const int64_t* perm = nullptr;
    EpochPlan plan;
    if (need_plan) {
      plan = opts.canonical_order ? EpochPlan::canonical(t) : EpochPlan::global(t, cap, rng);
      perm = plan.positions().data();
    }
    // storage scheme (CCache) or calculation scheme, decomposition.cpp:668-691
    check(ftkcu_set_option(s, "store_c", opts.store_c ? 1 : 0));
    check(ftkcu_core_phase(s, slot, perm, cap, h.lr_b, h.reg_b, mode, derive_seed(seed, {2}),
                           nullptr, &ms_c));
  }
  st.seconds_factor = ms_f * 1e-3;
  st.seconds_core = ms_c * 1e-3;
  bill_phase(st.factor, m, t.nnz(), cap, true, opts.store_c);
  bill_phase(st.core, m, t.nnz(), cap, false, opts.store_c);
  return st;
}

// FastTucker's per-batch billing (update_factor_fasttucker_impl /
// update_core_fasttucker_impl, decomposition.cpp:316-417) summed over a
// plan's batches: every tally is a per-batch constant plus a multiple of
// m_eff, and all of it lands on the block's mode.
void bill_fasttucker(CostCounters& cc, const Model& m, int mode, const EpochPlan& plan,
                     bool factor) {
  const int N = m.order();
  const size64 R = m.r, Jn = m.ranks[mode];
  size64 sum_other_j = 0, sum_all_j = 0, other_jr = 0;
  for (int n = 0; n < N; ++n) {
    sum_all_j += m.ranks[n];
    if (n != mode) {
      sum_other_j += m.ranks[n];
      other_jr += static_cast<size64>(m.ranks[n]) * R;
    }
  }
  const size64 combine = N >= 2 ? N - 2 : 0;
  for (size64 b = 0; b < plan.batches(); ++b) {
    const size64 me = plan.desc(b).len;
    const bool full = me == static_cast<size64>(plan.batch_size());
    cc.count_batch(mode, full);
    if (factor) {
      cc.add(mode, kRead, Jn + Jn * R + me * sum_other_j, full);
      cc.add(mode, kDStage, me * other_jr + combine * me * R, full);
      cc.add(mode, kBdtStage, me * R * Jn, full);
      cc.add(mode, kOther, Jn * R + me * R + me * Jn, full);
      cc.add(mode, kUpdate, Jn, full);
    } else {
      cc.add(mode, kRead, me * sum_all_j + Jn * R, full);
      cc.add(mode, kDStage, me * other_jr + combine * me * R, full);
      cc.add(mode, kOther, me * Jn * R + me * R + me * Jn, full);
      cc.add(mode, kBdtStage, me * Jn * R, full);
      cc.add(mode, kUpdate, Jn * R, full);
    }
  }
}

// One FastTucker epoch on the resident model (epoch_fasttucker,
// decomposition.cpp:707-770): factor blocks over per-bucket plans of the
// fixed-mode indices, then core blocks over global plans, mode by mode.  The
// factor block is schedule-invariant (bit-identical at any parallelism); the
// core block runs the workers == 1 chain, or for workers > 1 the Hogwild
// schedule like the reference's parallel_for.
EpochStats run_epoch_fasttucker(const SparseTensor& t, int slot, const Model& m,
                                const std::vector<ModeIndex>& fixed_mode, const Hyperparams& h,
                                const EpochOptions& opts, std::uint64_t seed) {
  ftkcu_session* s = session();
  const int N = m.order();
  require(static_cast<int>(fixed_mode.size()) == N, "need one fixed-mode index per mode");
  const index_t cap = opts.canonical_order ? 1 : h.batch_size;
  const int workers = resolve_workers(opts.workers);
  EpochStats st;
  st.factor.reset(N);
  st.core.reset(N);
  double total_f = 0.0, total_c = 0.0;
  for (int mode = 0; mode < N; ++mode) {
    Rng rng(derive_seed(seed, {1, static_cast<std::uint64_t>(mode)}));
    double ms = 0.0;
    if (opts.canonical_order) {
      // storage order, one entry per batch: the fixed-mode index's buckets
      // hold each row's entries in storage order, and rows are independent
      EpochPlan plan = EpochPlan::canonical(t);
      const ModeIndex& mi = fixed_mode[mode];
      std::vector<int64_t> boff(mi.offsets.begin(), mi.offsets.end());
      check(ftkcu_fasttucker_factor(s, slot, mode,
                                    reinterpret_cast<const int64_t*>(mi.positions.data()),
                                    boff.data(), static_cast<int64_t>(mi.buckets()), 1, h.lr_a,
                                    h.reg_a, &ms));
      bill_fasttucker(st.factor, m, mode, plan, true);
    } else {
      EpochPlan plan = EpochPlan::per_bucket(t, fixed_mode[mode], cap, rng);
      const auto& bo = plan.bucket_offsets();
      check(ftkcu_fasttucker_factor(s, slot, mode, plan.positions().data(), bo.data(),
                                    static_cast<int64_t>(bo.size()) - 1, cap, h.lr_a, h.reg_a,
                                    &ms));
      bill_fasttucker(st.factor, m, mode, plan, true);
    }
    total_f += ms;
  }
  for (int mode = 0; mode < N; ++mode) {
    Rng rng(derive_seed(seed, {2, static_cast<std::uint64_t>(mode)}));
    EpochPlan plan = opts.canonical_order ? EpochPlan::canonical(t) : EpochPlan::global(t, cap, rng);
    double ms = 0.0;
    check(ftkcu_fasttucker_core(s, slot, mode, plan.positions().data(), cap, h.lr_b, h.reg_b,
                                device_mode(workers), &ms));
    bill_fasttucker(st.core, m, mode, plan, false);
    total_c += ms;
  }
  st.seconds_factor = total_f * 1e-3;
  st.seconds_core = total_c * 1e-3;
  return st;
}

// FasterTucker's per-batch billing (update_factor_fastertucker_impl /
// update_core_fastertucker_impl, decomposition.cpp:420-533) over the plan's
// batches, plus the block barrier's cache refresh as overhead (:810, :837).
void bill_fastertucker(CostCounters& cc, const Model& m, int mode, const EpochPlan& plan,
                       bool factor) {
  const int N = m.order();
  const size64 R = m.r, Jn = m.ranks[mode];
  const size64 combine = N >= 2 ? N - 2 : 0;
  for (size64 b = 0; b < plan.batches(); ++b) {
    const size64 me = plan.desc(b).len;
    const bool full = me == static_cast<size64>(plan.batch_size());
    cc.count_batch(mode, full);
    cc.add(mode, kDStage, combine * R, full);
    if (factor) {
      cc.add(mode, kRead, (N - 1) * R + me * Jn + Jn * R, full);
      cc.add(mode, kBdtStage, Jn * R, full);
      cc.add(mode, kOther, me * Jn, full);
      cc.add(mode, kUpdate, me * Jn, full);
    } else {
      cc.add(mode, kRead, (N - 1) * R + me * Jn + me * R + Jn * R, full);
      cc.add(mode, kOther, me * R + me * Jn, full);
      cc.add(mode, kBdtStage, Jn * R, full);
      cc.add(mode, kUpdate, Jn * R, full);
    }
  }
  cc.add_overhead(kOther, static_cast<size64>(m.dims[mode]) * Jn * R);
}

// Plan positions regrouped by mode-n row, plan order kept inside a row
// (stable counting sort); out_off gets the group offsets.
void group_by_row(const SparseTensor& t, const std::vector<size64>& plan, int mode,
                  std::vector<int64_t>& out, std::vector<int64_t>& out_off) {
  const index_t rows = t.dims[mode];
  std::vector<int64_t> count(static_cast<std::size_t>(rows) + 1, 0);
  for (size64 p : plan) ++count[t.entry(p)[mode] + 1];
  for (index_t i = 0; i < rows; ++i) count[i + 1] += count[i];
  out.assign(plan.size(), 0);
  std::vector<int64_t> at(count.begin(), count.end() - 1);
  for (size64 p : plan) out[at[t.entry(p)[mode]]++] = static_cast<int64_t>(p);
  out_off.clear();
  out_off.push_back(0);
  for (index_t i = 0; i < rows; ++i)
    if (count[i + 1] > count[i]) out_off.push_back(count[i + 1]);
}

std::vector<int64_t> batch_offsets(const EpochPlan& plan) {
  std::vector<int64_t> off;
  off.reserve(static_cast<std::size_t>(plan.batches()) + 1);
  for (size64 b = 0; b < plan.batches(); ++b) off.push_back(plan.desc(b).offset);
  off.push_back(static_cast<int64_t>(plan.positions().size()));
  return off;
}

// One FasterTucker epoch on the resident model and device C cache
// (epoch_fastertucker, decomposition.cpp:772-843).
EpochStats run_epoch_fastertucker(const SparseTensor& t, int slot, const Model& m,
                                  const std::vector<ModeIndex>& complement, const Hyperparams& h,
                                  const EpochOptions& opts, std::uint64_t seed) {
  ftkcu_session* s = session();
  const int N = m.order();
  require(static_cast<int>(complement.size()) == N, "need one complement index per mode");
  require(!opts.eager_refresh, "eager_refresh is not supported by the device FasterTucker");
  const index_t cap = opts.canonical_order ? 1 : h.batch_size;
  const int workers = resolve_workers(opts.workers);
  EpochStats st;
  st.factor.reset(N);
  st.core.reset(N);
  double total[2] = {0.0, 0.0};
  std::vector<int64_t> perm, off;
  for (int phase = 0; phase < 2; ++phase) {
    for (int mode = 0; mode < N; ++mode) {
      Rng rng(derive_seed(seed, {static_cast<std::uint64_t>(phase + 1),
                                 static_cast<std::uint64_t>(mode)}));
      EpochPlan plan = opts.canonical_order ? EpochPlan::canonical(t)
                                            : EpochPlan::per_bucket(t, complement[mode], cap, rng);
      double ms = 0.0;
      if (phase == 0) {
        group_by_row(t, plan.positions(), mode, perm, off);
        check(ftkcu_fastertucker_factor(s, slot, mode, perm.data(), off.data(),
                                        static_cast<int64_t>(off.size()) - 1, h.lr_a, h.reg_a,
                                        &ms));
        bill_fastertucker(st.factor, m, mode, plan, true);
      } else {
        off = batch_offsets(plan);
        check(ftkcu_fastertucker_core(s, slot, mode, plan.positions().data(), off.data(),
                                      static_cast<int64_t>(off.size()) - 1, h.lr_b, h.reg_b,
                                      device_mode(workers), &ms));
        bill_fastertucker(st.core, m, mode, plan, false);
      }
      total[phase] += ms;
    }
  }
  st.seconds_factor = total[0] * 1e-3;
  st.seconds_core = total[1] * 1e-3;
  return st;
}

void upload_cache(CCache& cache) {
  auto& c = cache.storage();
  std::vector<const float*> p(c.size());
  for (std::size_t n = 0; n < c.size(); ++n) p[n] = c[n].data();
  check(ftkcu_ccache_upload(session(), p.data()));
}

void download_cache(CCache& cache) {
  auto& c = cache.storage();
  std::vector<float*> p(c.size());
  for (std::size_t n = 0; n < c.size(); ++n) p[n] = c[n].data();
  check(ftkcu_ccache_download(session(), p.data()));
}

std::string num_json(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

}  // namespace

void set_device_options(const DeviceOptions& o) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_opts = o;
  if (g_eng.s) apply_options(g_eng.s);
}

DeviceOptions device_options() {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_opts;
}

DeviceKernels device_last_kernels() {
  std::lock_guard<std::mutex> lk(g_mu);
  DeviceKernels k;
  if (!g_eng.s) return k;
  int64_t f = 0, c = 0;
  check(ftkcu_get_option(g_eng.s, "last_factor_kernel", &f));
  check(ftkcu_get_option(g_eng.s, "last_core_kernel", &c));
  k.factor = static_cast<int>(f);
  k.core = static_cast<int>(c);
  return k;
}

EpochStats epoch_plus(const SparseTensor& t, Model& m, const Hyperparams& h,
                      const EpochOptions& opts, std::uint64_t seed) {
  std::lock_guard<std::mutex> lk(g_mu);
  apply_options(session());
  const int slot = ensure_tensor(t);
  upload_model(m);
  EpochStats st;
  try {
    st = run_epoch(t, slot, m, h, opts, seed);
  } catch (...) {
    download_model(m);  // the reference mutates m in place before throwing
    throw;
  }
  download_model(m);
  return st;
}

void CCache::init(const Model& m) {
  const int n = m.order();
  r_ = m.r;
  c_.assign(n, {});
  for (int k = 0; k < n; ++k) c_[k].assign(static_cast<std::size_t>(m.dims[k]) * m.r, 0.0f);
  fresh_.assign(n, 0);
}

void CCache::build(const Model& m, CostCounters* cc) {
  if (c_.empty()) init(m);
  for (int k = 0; k < m.order(); ++k) refresh(m, k, cc);
}

void CCache::refresh(const Model& m, int mode, CostCounters* cc) {
  require(!c_.empty(), "cache not initialized");
  const index_t jn = m.ranks[mode], r = m.r;
  const real* b = m.b[mode].data();
  for (index_t i = 0; i < m.dims[mode]; ++i) {
    const real* arow = m.a_row(mode, i);
    real* crow = c_[mode].data() + static_cast<std::size_t>(i) * r;
    for (index_t col = 0; col < r; ++col) {
      real acc = 0.0f;
      for (index_t j = 0; j < jn; ++j) acc += arow[j] * b[static_cast<std::size_t>(j) * r + col];
      crow[col] = acc;
    }
  }
  fresh_[mode] = 1;
  if (cc) cc->add_overhead(kOther, static_cast<size64>(m.dims[mode]) * jn * r);
}

EpochStats epoch_fastertucker(const SparseTensor& t, const std::vector<ModeIndex>& complement,
                              Model& m, CCache& cache, const Hyperparams& h,
                              const EpochOptions& opts, std::uint64_t seed) {
  require(static_cast<int>(complement.size()) == m.order(),
          "need one complement index per mode");
  require(cache.ready(), "C cache must be built before the first epoch");
  std::lock_guard<std::mutex> lk(g_mu);
  apply_options(session());
  const int slot = ensure_tensor(t);
  upload_model(m);
  upload_cache(cache);
  EpochStats st;
  try {
    st = run_epoch_fastertucker(t, slot, m, complement, h, opts, seed);
  } catch (...) {
    download_model(m);
    throw;
  }
  download_model(m);
  download_cache(cache);
  for (int n = 0; n < m.order(); ++n) cache.mark_fresh(n);  // each block refreshed its mode
  return st;
}

EpochStats epoch_fasttucker(const SparseTensor& t, const std::vector<ModeIndex>& fixed_mode,
                            Model& m, const Hyperparams& h, const EpochOptions& opts,
                            std::uint64_t seed) {
  require(static_cast<int>(fixed_mode.size()) == m.order(),
          "need one fixed-mode index per mode");
  std::lock_guard<std::mutex> lk(g_mu);
  apply_options(session());
  const int slot = ensure_tensor(t);
  upload_model(m);
  EpochStats st;
  try {
    st = run_epoch_fasttucker(t, slot, m, fixed_mode, h, opts, seed);
  } catch (...) {
    download_model(m);
    throw;
  }
  download_model(m);
  return st;
}

namespace {

// Device loss/metrics of the resident model.
double device_loss(int slot, double reg_a, double reg_b, int workers) {
  double out[3];
  check(ftkcu_eval(session(), slot, workers, reg_a, reg_b, out));
  return out[0] + out[2];
}

Metrics device_metrics(int slot, size64 n, int workers) {
  require(n > 0, "empty evaluation set");
  double out[3];
  check(ftkcu_eval(session(), slot, workers, 0.0, 0.0, out));
  Metrics mt;
  mt.samples = n;
  mt.rmse = std::sqrt(out[0] / static_cast<double>(n));
  mt.mae = out[1] / static_cast<double>(n);
  return mt;
}

}  // namespace

double loss(const Model& m, const SparseTensor& t, double reg_a, double reg_b, int workers) {
  std::lock_guard<std::mutex> lk(g_mu);
  apply_options(session());
  const int slot = ensure_tensor(t);
  upload_model(m);
  return device_loss(slot, reg_a, reg_b, std::max(1, workers));
}

Metrics evaluate(const Model& m, const SparseTensor& testset, int workers) {
  require(testset.nnz() > 0, "empty evaluation set");
  std::lock_guard<std::mutex> lk(g_mu);
  apply_options(session());
  const int slot = ensure_tensor(testset);
  upload_model(m);
  return device_metrics(slot, testset.nnz(), std::max(1, workers));
}

double rmse(const Model& m, const SparseTensor& testset, int workers) {
  return evaluate(m, testset, workers).rmse;
}

double mae(const Model& m, const SparseTensor& testset, int workers) {
  return evaluate(m, testset, workers).mae;
}

History train(const SparseTensor& train_set, const SparseTensor* test_set, Model& m,
              const Hyperparams& h, const TrainOptions& opts) {
  h.validate();
  m.validate();
  require(m.order() == train_set.order, "model/tensor order mismatch");
  for (int n = 0; n < m.order(); ++n)
    require(m.dims[n] >= train_set.dims[n], "model dims too small for tensor");

  const int workers = resolve_workers(opts.workers);
  EpochOptions eo;
  eo.workers = workers;
  eo.store_c = opts.store_c;
  History hist;
  if (h.epochs == 0) return hist;
  std::lock_guard<std::mutex> lk(g_mu);
  apply_options(session());
  const int slot = ensure_tensor(train_set);
  int test_slot = -1;
  if (test_set != nullptr && test_set->nnz() > 0) {
    test_slot = ensure_tensor(*test_set);
  }
  std::vector<ModeIndex> fixed;  // fixed-mode (FastTucker) / complement (FasterTucker)
  if (opts.variant != Variant::kPlus)
    for (int n = 0; n < m.order(); ++n)
      fixed.push_back(build_mode_index(train_set, n,
                                       opts.variant == Variant::kFastTucker
                                           ? Keying::kFixedMode
                                           : Keying::kFixedComplement));
  upload_model(m);
  if (opts.variant == Variant::kFasterTucker) {  // cache.build once (decomposition.cpp:873)
    CCache cache;
    cache.build(m, nullptr);
    upload_cache(cache);
  }
  for (int epoch = 1; epoch <= h.epochs; ++epoch) {
    const std::uint64_t es = derive_seed(opts.seed, {static_cast<std::uint64_t>(epoch)});
    EpochRecord rec;
    rec.epoch = epoch;
    rec.stats = opts.variant == Variant::kFastTucker
                    ? run_epoch_fasttucker(train_set, slot, m, fixed, h, eo, es)
                : opts.variant == Variant::kFasterTucker
                    ? run_epoch_fastertucker(train_set, slot, m, fixed, h, eo, es)
                    : run_epoch(train_set, slot, m, h, eo, es);
    rec.seconds = rec.stats.seconds_factor + rec.stats.seconds_core;
    rec.train_loss = device_loss(slot, h.reg_a, h.reg_b, workers);
    if (test_slot >= 0) {
      Metrics mt = device_metrics(test_slot, test_set->nnz(), workers);
      rec.test_rmse = mt.rmse;
      rec.test_mae = mt.mae;
    } else {
      rec.test_rmse = std::numeric_limits<double>::quiet_NaN();
      rec.test_mae = std::numeric_limits<double>::quiet_NaN();
    }
    const auto& f = rec.stats.factor;
    const auto& c = rec.stats.core;
    rec.reads = f.total(kRead) + c.total(kRead);
    rec.mults = f.total(kDStage) + f.total(kBdtStage) + f.total(kOther) + c.total(kDStage) +
                c.total(kBdtStage) + c.total(kOther);
    if (!std::isfinite(rec.train_loss)) {
      download_model(m);
      fail("training diverged: non-finite loss at epoch " + std::to_string(epoch));
    }
    hist.push_back(std::move(rec));
  }
  download_model(m);
  return hist;
}

std::string history_line_json(const EpochRecord& r) {
  // Keys in the order nlohmann::json (std::map) emits them.
  std::string s = "{\"epoch\":" + std::to_string(r.epoch);
  s += ",\"mults\":" + std::to_string(r.mults);
  s += ",\"reads\":" + std::to_string(r.reads);
  s += ",\"seconds\":" + num_json(r.seconds);
  s += ",\"test_mae\":" + num_json(r.test_mae);
  s += ",\"test_rmse\":" + num_json(r.test_rmse);
  s += ",\"train_loss\":" + num_json(r.train_loss) + "}";
  return s;
}

void write_history_jsonl(const History& h, const std::string& path) {
  std::ofstream out(path);
  require(out.good(), "cannot write " + path);
  for (const auto& r : h) out << history_line_json(r) << '\n';
  require(out.good(), "write failed: " + path);
}

void write_history_csv(const History& h, const std::string& path) {
  std::ofstream out(path);
  require(out.good(), "cannot write " + path);
  out << "epoch,train_loss,test_rmse,test_mae,seconds,reads,mults\n";
  for (const auto& r : h)
    out << r.epoch << ',' << r.train_loss << ',' << r.test_rmse << ',' << r.test_mae << ','
        << r.seconds << ',' << r.reads << ',' << r.mults << '\n';
  require(out.good(), "write failed: " + path);
}

}  // namespace ftk
