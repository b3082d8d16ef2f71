// extern "C" helpers over the ftk:: C++ API, for Python (ctypes) callers:
// tests and bench.py drive the very same ftk::epoch_plus / ftk::train /
// ftk::load_coo a C++ user links against.
#include <cstring>
#include <string>

#include "ftk/decomposition.hpp"

using namespace ftk;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

SparseTensor make_tensor(int order, const int32_t* dims, int64_t nnz, const int32_t* idx,
                         const float* vals) {
  SparseTensor t;
  t.order = order;
  t.dims.assign(dims, dims + order);
  t.indices.assign(idx, idx + nnz * order);
  t.values.assign(vals, vals + nnz);
  return t;
}

Model make_model(int order, const int32_t* dims, const int32_t* ranks, int32_t r,
                 float* const* a, float* const* b) {
  Model m;
  m.dims.assign(dims, dims + order);
  m.ranks.assign(ranks, ranks + order);
  m.r = r;
  m.a.resize(order);
  m.b.resize(order);
  for (int n = 0; n < order; ++n) {
    m.a[n].assign(a[n], a[n] + static_cast<std::size_t>(dims[n]) * ranks[n]);
    m.b[n].assign(b[n], b[n] + static_cast<std::size_t>(ranks[n]) * r);
  }
  return m;
}

void copy_back(const Model& m, float* const* a, float* const* b) {
  for (int n = 0; n < m.order(); ++n) {
    std::memcpy(a[n], m.a[n].data(), m.a[n].size() * sizeof(float));
    std::memcpy(b[n], m.b[n].data(), m.b[n].size() * sizeof(float));
  }
}

Hyperparams hyper(float lr_a, float lr_b, float reg_a, float reg_b, int epochs, int m) {
  Hyperparams h;
  h.lr_a = lr_a;
  h.lr_b = lr_b;
  h.reg_a = reg_a;
  h.reg_b = reg_b;
  h.epochs = epochs;
  h.batch_size = m;
  return h;
}

}  // namespace

extern "C" {

const char* ftkh_last_error() { return g_err.c_str(); }

uint64_t ftkh_derive_seed(uint64_t base, const uint64_t* path, int n) {
  uint64_t h = mix64(base);
  for (int i = 0; i < n; ++i) h = mix64(h ^ path[i]);
  return h;
}

int ftkh_global_plan(int64_t nnz, int m, uint64_t seed, int64_t* out) {
  return guarded([&] {
    SparseTensor t;
    t.order = 1;
    t.values.resize(static_cast<std::size_t>(nnz));
    Rng rng(seed);
    EpochPlan p = EpochPlan::global(t, m, rng);
    std::memcpy(out, p.positions().data(), sizeof(int64_t) * nnz);
  });
}

// EpochPlan::per_bucket positions and bucket offsets (plan order) of an
// AoS index set, for Rng(seed); nb_out receives the bucket count.
int ftkh_per_bucket_plan(int order, int64_t nnz, const int32_t* idx, int mode, int keying, int m,
                         uint64_t seed, int64_t* perm_out, int64_t* boff_out, int64_t* nb_out) {
  return guarded([&] {
    SparseTensor t;
    t.order = order;
    t.indices.assign(idx, idx + nnz * order);
    t.values.assign(static_cast<std::size_t>(nnz), 0.0f);
    const ModeIndex mi =
        build_mode_index(t, mode, keying ? Keying::kFixedComplement : Keying::kFixedMode);
    Rng rng(seed);
    const EpochPlan p = EpochPlan::per_bucket(t, mi, m, rng);
    std::memcpy(perm_out, p.positions().data(), sizeof(int64_t) * nnz);
    const auto& bo = p.bucket_offsets();
    std::memcpy(boff_out, bo.data(), sizeof(int64_t) * bo.size());
    *nb_out = static_cast<int64_t>(bo.size()) - 1;
  });
}

int ftkh_init_model(int order, const int32_t* dims, const int32_t* ranks, int32_t r,
                    uint64_t seed, float scale, float* const* a, float* const* b) {
  return guarded([&] {
    Model m = init_model({dims, static_cast<std::size_t>(order)},
                         {ranks, static_cast<std::size_t>(order)}, r, seed, scale);
    copy_back(m, a, b);
  });
}

float ftkh_default_init_scale(double mean_abs, int order, int32_t r, const int32_t* ranks) {
  return default_init_scale(mean_abs, order, r, {ranks, static_cast<std::size_t>(order)});
}

// out buffers sized for nnz entries each; *ntest receives the test count.
int ftkh_split(int order, const int32_t* dims, int64_t nnz, const int32_t* idx,
               const float* vals, double frac, uint64_t seed, int32_t* tr_idx, float* tr_vals,
               int32_t* te_idx, float* te_vals, int64_t* ntest) {
  return guarded([&] {
    SparseTensor t = make_tensor(order, dims, nnz, idx, vals);
    auto [tr, te] = split_train_test(t, frac, seed);
    std::memcpy(tr_idx, tr.indices.data(), tr.indices.size() * sizeof(int32_t));
    std::memcpy(tr_vals, tr.values.data(), tr.values.size() * sizeof(float));
    std::memcpy(te_idx, te.indices.data(), te.indices.size() * sizeof(int32_t));
    std::memcpy(te_vals, te.values.data(), te.values.size() * sizeof(float));
    *ntest = te.nnz();
  });
}

void* ftkh_load_coo(const char* path, int order) {
  SparseTensor* t = nullptr;
  int rc = guarded([&] { t = new SparseTensor(load_coo(path, order)); });
  return rc ? nullptr : t;
}

void* ftkh_load_coo_binary(const char* path) {
  SparseTensor* t = nullptr;
  int rc = guarded([&] { t = new SparseTensor(load_coo_binary(path)); });
  return rc ? nullptr : t;
}

int ftkh_tensor_order(void* h) { return static_cast<SparseTensor*>(h)->order; }

int ftkh_save_coo_binary(int order, const int32_t* dims, int64_t nnz, const int32_t* idx,
                         const float* vals, const char* path) {
  return guarded([&] { save_coo_binary(make_tensor(order, dims, nnz, idx, vals), path); });
}

int ftkh_infer_coo_order(const char* path) {
  int o = -1;
  guarded([&] { o = infer_coo_order(path); });
  return o;
}

int64_t ftkh_tensor_nnz(void* h) { return static_cast<SparseTensor*>(h)->nnz(); }

void ftkh_tensor_copy(void* h, int32_t* dims, int32_t* idx, float* vals) {
  auto* t = static_cast<SparseTensor*>(h);
  std::memcpy(dims, t->dims.data(), sizeof(int32_t) * t->order);
  std::memcpy(idx, t->indices.data(), sizeof(int32_t) * t->indices.size());
  std::memcpy(vals, t->values.data(), sizeof(float) * t->values.size());
}

void ftkh_tensor_free(void* h) { delete static_cast<SparseTensor*>(h); }

int ftkh_save_coo(int order, const int32_t* dims, int64_t nnz, const int32_t* idx,
                  const float* vals, const char* path) {
  return guarded([&] { save_coo(make_tensor(order, dims, nnz, idx, vals), path); });
}

int ftkh_set_device_options(int device, int mode, int precision, int exact_eval, int parity) {
  return guarded([&] {
    DeviceOptions o;
    o.device = device;
    o.mode = static_cast<DeviceMode>(mode);
    o.precision = static_cast<DevicePrecision>(precision);
    o.exact_eval = exact_eval != 0;
    o.parity = parity != 0;
    set_device_options(o);
  });
}

int ftkh_last_kernels(int* factor, int* core) {
  return guarded([&] {
    const DeviceKernels k = device_last_kernels();
    *factor = k.factor;
    *core = k.core;
  });
}

// ftk::epoch_fasttucker with fixed-mode indices of every mode built here.
int ftkh_epoch_fasttucker(int order, const int32_t* dims, const int32_t* ranks, int32_t r,
                          int64_t nnz, const int32_t* idx, const float* vals, float* const* a,
                          float* const* b, float lr_a, float lr_b, float reg_a, float reg_b,
                          int m, int workers, int canonical, uint64_t seed, double* seconds2,
                          int64_t* counters) {
  return guarded([&] {
    SparseTensor t = make_tensor(order, dims, nnz, idx, vals);
    Model md = make_model(order, dims, ranks, r, a, b);
    std::vector<ModeIndex> fixed;
    for (int n = 0; n < order; ++n) fixed.push_back(build_mode_index(t, n, Keying::kFixedMode));
    EpochOptions eo;
    eo.workers = workers;
    eo.canonical_order = canonical != 0;
    EpochStats st;
    try {
      st = epoch_fasttucker(t, fixed, md, hyper(lr_a, lr_b, reg_a, reg_b, 1, m), eo, seed);
    } catch (...) {
      copy_back(md, a, b);
      throw;
    }
    copy_back(md, a, b);
    if (seconds2) {
      seconds2[0] = st.seconds_factor;
      seconds2[1] = st.seconds_core;
    }
    if (counters)
      for (int s = 0; s < kStages; ++s) {
        counters[s] = st.factor.total(static_cast<Stage>(s));
        counters[kStages + s] = st.core.total(static_cast<Stage>(s));
      }
  });
}

// ftk::epoch_fastertucker with complement indices and a freshly built C cache.
int ftkh_epoch_fastertucker(int order, const int32_t* dims, const int32_t* ranks, int32_t r,
                            int64_t nnz, const int32_t* idx, const float* vals, float* const* a,
                            float* const* b, float lr_a, float lr_b, float reg_a, float reg_b,
                            int m, int workers, int canonical, uint64_t seed, double* seconds2,
                            int64_t* counters) {
  return guarded([&] {
    SparseTensor t = make_tensor(order, dims, nnz, idx, vals);
    Model md = make_model(order, dims, ranks, r, a, b);
    std::vector<ModeIndex> comp;
    for (int n = 0; n < order; ++n)
      comp.push_back(build_mode_index(t, n, Keying::kFixedComplement));
    CCache cache;
    cache.build(md, nullptr);
    EpochOptions eo;
    eo.workers = workers;
    eo.canonical_order = canonical != 0;
    EpochStats st;
    try {
      st = epoch_fastertucker(t, comp, md, cache, hyper(lr_a, lr_b, reg_a, reg_b, 1, m), eo,
                              seed);
    } catch (...) {
      copy_back(md, a, b);
      throw;
    }
    copy_back(md, a, b);
    if (seconds2) {
      seconds2[0] = st.seconds_factor;
      seconds2[1] = st.seconds_core;
    }
    if (counters)
      for (int s = 0; s < kStages; ++s) {
        counters[s] = st.factor.total(static_cast<Stage>(s));
        counters[kStages + s] = st.core.total(static_cast<Stage>(s));
      }
  });
}

int ftkh_epoch_plus(int order, const int32_t* dims, const int32_t* ranks, int32_t r,
                    int64_t nnz, const int32_t* idx, const float* vals, float* const* a,
                    float* const* b, float lr_a, float lr_b, float reg_a, float reg_b, int m,
                    int workers, int store_c, int canonical, uint64_t seed, double* seconds2,
                    int64_t* counters) {
  return guarded([&] {
    SparseTensor t = make_tensor(order, dims, nnz, idx, vals);
    Model md = make_model(order, dims, ranks, r, a, b);
    EpochOptions eo;
    eo.workers = workers;
    eo.store_c = store_c != 0;
    eo.canonical_order = canonical != 0;
    EpochStats st;
    try {
      st = epoch_plus(t, md, hyper(lr_a, lr_b, reg_a, reg_b, 1, m), eo, seed);
    } catch (...) {
      copy_back(md, a, b);
      throw;
    }
    copy_back(md, a, b);
    if (seconds2) {
      seconds2[0] = st.seconds_factor;
      seconds2[1] = st.seconds_core;
    }
    if (counters)
      for (int s = 0; s < kStages; ++s) {
        counters[s] = st.factor.total(static_cast<Stage>(s));
        counters[kStages + s] = st.core.total(static_cast<Stage>(s));
      }
  });
}

// ftk::train for a variant (0 plus, 1 fasttucker, 2 fastertucker).
int ftkh_train_variant(int order, const int32_t* dims, const int32_t* ranks, int32_t r,
                       int64_t nnz, const int32_t* idx, const float* vals, int64_t nnz_test,
                       const int32_t* idx_test, const float* vals_test, float* const* a,
                       float* const* b, float lr_a, float lr_b, float reg_a, float reg_b,
                       int epochs, int m, int workers, int store_c, uint64_t seed,
                       double* loss_out, double* rmse_out, double* mae_out, double* seconds_out,
                       int64_t* reads_out, int64_t* mults_out, char* jsonl, int jsonl_cap,
                       int variant) {
  return guarded([&] {
    SparseTensor t = make_tensor(order, dims, nnz, idx, vals);
    SparseTensor te;
    if (nnz_test > 0) te = make_tensor(order, dims, nnz_test, idx_test, vals_test);
    Model md = make_model(order, dims, ranks, r, a, b);
    TrainOptions to;
    to.workers = workers;
    to.store_c = store_c != 0;
    to.seed = seed;
    to.variant = variant == 1   ? Variant::kFastTucker
                 : variant == 2 ? Variant::kFasterTucker
                                : Variant::kPlus;
    History h;
    try {
      h = train(t, nnz_test > 0 ? &te : nullptr, md, hyper(lr_a, lr_b, reg_a, reg_b, epochs, m),
                to);
    } catch (...) {
      copy_back(md, a, b);
      throw;
    }
    copy_back(md, a, b);
    std::string lines;
    for (std::size_t e = 0; e < h.size(); ++e) {
      loss_out[e] = h[e].train_loss;
      rmse_out[e] = h[e].test_rmse;
      mae_out[e] = h[e].test_mae;
      if (seconds_out) seconds_out[e] = h[e].seconds;
      if (reads_out) reads_out[e] = h[e].reads;
      if (mults_out) mults_out[e] = h[e].mults;
      lines += history_line_json(h[e]) + "\n";
    }
    if (jsonl && jsonl_cap > 0) {
      std::strncpy(jsonl, lines.c_str(), static_cast<std::size_t>(jsonl_cap) - 1);
      jsonl[jsonl_cap - 1] = '\0';
    }
  });
}

int ftkh_train(int order, const int32_t* dims, const int32_t* ranks, int32_t r, int64_t nnz,
               const int32_t* idx, const float* vals, int64_t nnz_test, const int32_t* idx_test,
               const float* vals_test, float* const* a, float* const* b, float lr_a, float lr_b,
               float reg_a, float reg_b, int epochs, int m, int workers, int store_c,
               uint64_t seed, double* loss_out, double* rmse_out, double* mae_out,
               double* seconds_out, int64_t* reads_out, int64_t* mults_out, char* jsonl,
               int jsonl_cap) {
  return ftkh_train_variant(order, dims, ranks, r, nnz, idx, vals, nnz_test, idx_test, vals_test,
                            a, b, lr_a, lr_b, reg_a, reg_b, epochs, m, workers, store_c, seed,
                            loss_out, rmse_out, mae_out, seconds_out, reads_out, mults_out, jsonl,
                            jsonl_cap, 0);
}

int ftkh_loss(int order, const int32_t* dims, const int32_t* ranks, int32_t r, int64_t nnz,
              const int32_t* idx, const float* vals, float* const* a, float* const* b,
              double reg_a, double reg_b, int workers, double* out) {
  return guarded([&] {
    SparseTensor t = make_tensor(order, dims, nnz, idx, vals);
    Model md = make_model(order, dims, ranks, r, a, b);
    *out = loss(md, t, reg_a, reg_b, workers);
  });
}

int ftkh_evaluate(int order, const int32_t* dims, const int32_t* ranks, int32_t r, int64_t nnz,
                  const int32_t* idx, const float* vals, float* const* a, float* const* b,
                  int workers, double* rmse_out, double* mae_out) {
  return guarded([&] {
    SparseTensor t = make_tensor(order, dims, nnz, idx, vals);
    Model md = make_model(order, dims, ranks, r, a, b);
    Metrics mt = evaluate(md, t, workers);
    *rmse_out = mt.rmse;
    *mae_out = mt.mae;
  });
}

int ftkh_predicted_costs(int order, int m, int r, const int32_t* ranks, int64_t* out4) {
  return guarded([&] {
    PredictedCosts p = predicted_costs(order, m, r, {ranks, static_cast<std::size_t>(order)},
                                       Variant::kPlus);
    out4[0] = p.reads;
    out4[1] = p.d_stage;
    out4[2] = p.bdt_stage;
    out4[3] = p.update;
  });
}

}  // extern "C"
