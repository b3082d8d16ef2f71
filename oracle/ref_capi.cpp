// TEST INFRASTRUCTURE ONLY — never part of the shipped engine.
//
// A thin extern "C" shim over the *unmodified* reference library
// (/root/reference/proj/src/*.cpp compiled with its own Release flags and
// -Dftk=ftkref, see oracle/Makefile).  It lets Python (ctypes) drive the
// reference through its public C++ API so that
//   * the C restatement in oracle/ftk_oracle.c can be pinned bit-for-bit,
//   * golden fixtures under tests/golden/ can be (re)generated,
//   * bench.py --impl reference / cpu_baseline can time ftkref::epoch_plus.
// Nothing here re-implements arithmetic: every number comes out of the
// reference's own functions.  Only tests/, __graft_entry__.smoke() and the
// CPU legs of bench.py may load the resulting oracle/_ref/libftkref.so.
//
// Reference entry points used (all under /root/reference/proj):
//   include/ftk/decomposition.hpp:86-124  per-batch pipeline
//   include/ftk/decomposition.hpp:189-190 epoch_plus
//   include/ftk/decomposition.hpp:234-235 train
//   include/ftk/evaluation.hpp:17-25      loss / evaluate
//   include/ftk/model.hpp:51-58           init_model / default_init_scale
//   include/ftk/sparse_tensor.hpp:46-48   split_train_test
//   include/ftk/sparse_tensor.hpp:99-119  EpochPlan::global / gather

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "ftk/counters.hpp"
#include "ftk/decomposition.hpp"
#include "ftk/evaluation.hpp"
#include "ftk/model.hpp"
#include "ftk/sparse_tensor.hpp"

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
  } catch (...) {
    g_err = "unknown exception";
    return 1;
  }
}

ftkref::Hyperparams hyper(float lr_a, float lr_b, float reg_a, float reg_b,
                          int epochs, int m) {
  ftkref::Hyperparams h;
  h.lr_a = lr_a;
  h.lr_b = lr_b;
  h.reg_a = reg_a;
  h.reg_b = reg_b;
  h.epochs = epochs;
  h.batch_size = m;
  return h;
}

// Dense copy of a tiled matrix's logical extent, row-major.
void dense_copy(const ftkref::TiledMatrix& t, float* out, int rows, int cols,
                int ld) {
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) out[r * ld + c] = t.at(r, c);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// common.hpp:43-48 derive_seed over a path of n components.
uint64_t ref_derive_seed(uint64_t base, const uint64_t* path, int n) {
  std::uint64_t s = ftkref::mix64(base);
  for (int i = 0; i < n; ++i) s = ftkref::mix64(s ^ path[i]);
  return s;
}

// ---- tensors ---------------------------------------------------------------

void* ref_tensor_new(int order, const int32_t* dims, int64_t nnz,
                     const int32_t* idx, const float* vals) {
  auto* t = new ftkref::SparseTensor;
  t->order = order;
  t->dims.assign(dims, dims + order);
  t->indices.assign(idx, idx + nnz * order);
  t->values.assign(vals, vals + nnz);
  return t;
}

int64_t ref_tensor_nnz(void* t) {
  return static_cast<ftkref::SparseTensor*>(t)->nnz();
}

void ref_tensor_get(void* tp, int32_t* dims, int32_t* idx, float* vals) {
  auto* t = static_cast<ftkref::SparseTensor*>(tp);
  std::memcpy(dims, t->dims.data(), sizeof(int32_t) * t->order);
  std::memcpy(idx, t->indices.data(), sizeof(int32_t) * t->indices.size());
  std::memcpy(vals, t->values.data(), sizeof(float) * t->values.size());
}

void ref_tensor_free(void* t) { delete static_cast<ftkref::SparseTensor*>(t); }

int ref_tensor_validate(void* t) {
  return guarded([&] { static_cast<ftkref::SparseTensor*>(t)->validate(); });
}

int ref_split(void* t, double frac, uint64_t seed, void** train, void** test) {
  return guarded([&] {
    auto pr = ftkref::split_train_test(*static_cast<ftkref::SparseTensor*>(t),
                                       frac, seed);
    *train = new ftkref::SparseTensor(std::move(pr.first));
    *test = new ftkref::SparseTensor(std::move(pr.second));
  });
}

int ref_load_coo(const char* path, int order, void** out) {
  return guarded([&] {
    *out = new ftkref::SparseTensor(ftkref::load_coo(path, order));
  });
}

// Positions visited by EpochPlan::global(t, m, Rng(seed)), in batch order.
// Recovered through the public gather(): a 1-mode tensor whose single index
// column is the entry position (sparse_tensor.cpp:271-282, 319-323).
int ref_global_plan(int64_t nnz, int m, uint64_t seed, int64_t* perm_out) {
  return guarded([&] {
    ftkref::SparseTensor pos;
    pos.order = 1;
    pos.dims = {static_cast<int32_t>(nnz)};
    pos.indices.resize(nnz);
    pos.values.assign(nnz, 0.0f);
    for (int64_t i = 0; i < nnz; ++i) pos.indices[i] = static_cast<int32_t>(i);
    ftkref::Rng rng(seed);
    ftkref::EpochPlan plan = ftkref::EpochPlan::global(pos, m, rng);
    ftkref::Batch b;
    int64_t k = 0;
    for (int64_t bi = 0; bi < plan.batches(); ++bi) {
      plan.gather(pos, bi, b);
      for (int r = 0; r < b.m_eff; ++r) perm_out[k++] = b.idx[0][r];
    }
  });
}

// EpochPlan::per_bucket over build_mode_index(t, mode, keying) for Rng(seed)
// (sparse_tensor.cpp:200-240, 284-308): the visited positions in batch order
// and the offsets of the buckets in that order (a bucket's batches are
// consecutive; recovered from Batch::bucket), through a position tensor as
// in ref_global_plan.
int ref_per_bucket_plan(void* tp, int mode, int keying, int m, uint64_t seed, int64_t* perm_out,
                        int64_t* boff_out, int64_t* nb_out) {
  return guarded([&] {
    const auto& t = *static_cast<ftkref::SparseTensor*>(tp);
    const auto idx = ftkref::build_mode_index(
        t, mode, keying ? ftkref::Keying::kFixedComplement : ftkref::Keying::kFixedMode);
    ftkref::SparseTensor pos;
    pos.order = 1;
    pos.dims = {static_cast<int32_t>(t.nnz())};
    pos.indices.resize(t.nnz());
    pos.values.assign(t.nnz(), 0.0f);
    for (int64_t i = 0; i < t.nnz(); ++i) pos.indices[i] = static_cast<int32_t>(i);
    ftkref::Rng rng(seed);
    ftkref::EpochPlan plan = ftkref::EpochPlan::per_bucket(pos, idx, m, rng);
    ftkref::Batch b;
    int64_t k = 0, nb = 0, last = -1;
    for (int64_t bi = 0; bi < plan.batches(); ++bi) {
      plan.gather(pos, bi, b);
      if (static_cast<int64_t>(b.bucket) != last) {
        boff_out[nb++] = k;
        last = static_cast<int64_t>(b.bucket);
      }
      for (int r = 0; r < b.m_eff; ++r) perm_out[k++] = b.idx[0][r];
    }
    boff_out[nb] = k;
    *nb_out = nb;
  });
}

// ---- models ----------------------------------------------------------------

void* ref_model_new(int order, const int32_t* dims, const int32_t* ranks,
                    int32_t r, const float* const* a, const float* const* b) {
  auto* m = new ftkref::Model;
  m->dims.assign(dims, dims + order);
  m->ranks.assign(ranks, ranks + order);
  m->r = r;
  m->a.resize(order);
  m->b.resize(order);
  for (int k = 0; k < order; ++k) {
    m->a[k].assign(a[k], a[k] + static_cast<size_t>(dims[k]) * ranks[k]);
    m->b[k].assign(b[k], b[k] + static_cast<size_t>(ranks[k]) * r);
  }
  return m;
}

int ref_model_init(int order, const int32_t* dims, const int32_t* ranks,
                   int32_t r, uint64_t seed, float scale, void** out) {
  return guarded([&] {
    std::vector<int32_t> d(dims, dims + order), j(ranks, ranks + order);
    *out = new ftkref::Model(ftkref::init_model(d, j, r, seed, scale));
  });
}

void ref_model_get(void* mp, float* const* a, float* const* b) {
  auto* m = static_cast<ftkref::Model*>(mp);
  for (int k = 0; k < m->order(); ++k) {
    std::memcpy(a[k], m->a[k].data(), sizeof(float) * m->a[k].size());
    std::memcpy(b[k], m->b[k].data(), sizeof(float) * m->b[k].size());
  }
}

void ref_model_free(void* m) { delete static_cast<ftkref::Model*>(m); }

float ref_default_init_scale(double mean_abs, int order, int32_t r,
                             const int32_t* ranks) {
  std::vector<int32_t> j(ranks, ranks + order);
  return ftkref::default_init_scale(mean_abs, order, r, j);
}

double ref_predict(void* m, const int32_t* idx) {
  auto* mm = static_cast<ftkref::Model*>(m);
  return ftkref::predict_element(
      *mm, std::span<const int32_t>(idx, static_cast<size_t>(mm->order())));
}

// ---- epochs / training -----------------------------------------------------

// counters_out[0..4] factor reads, d_stage, bdt_stage, update, other;
// counters_out[5..9] the same for the core phase.
int ref_epoch_plus(void* t, void* m, float lr_a, float lr_b, float reg_a,
                   float reg_b, int batch, int workers, int store_c,
                   uint64_t seed, double* seconds2, int64_t* counters_out) {
  return guarded([&] {
    ftkref::EpochOptions eo;
    eo.workers = workers;
    eo.store_c = store_c != 0;
    auto st = ftkref::epoch_plus(*static_cast<ftkref::SparseTensor*>(t),
                                 *static_cast<ftkref::Model*>(m),
                                 hyper(lr_a, lr_b, reg_a, reg_b, 1, batch), eo,
                                 seed);
    if (seconds2) {
      seconds2[0] = st.seconds_factor;
      seconds2[1] = st.seconds_core;
    }
    if (counters_out) {
      const ftkref::CostCounters* cs[2] = {&st.factor, &st.core};
      for (int p = 0; p < 2; ++p)
        for (int s = 0; s < ftkref::kStages; ++s)
          counters_out[p * ftkref::kStages + s] =
              cs[p]->total(static_cast<ftkref::Stage>(s));
    }
  });
}

// ftkref::epoch_fasttucker with fixed-mode indices of every mode
// (decomposition.cpp:707-770).
int ref_epoch_fasttucker(void* t, void* m, float lr_a, float lr_b, float reg_a, float reg_b,
                         int batch, int workers, int canonical, uint64_t seed, double* seconds2,
                         int64_t* counters_out) {
  return guarded([&] {
    const auto& ts = *static_cast<ftkref::SparseTensor*>(t);
    std::vector<ftkref::ModeIndex> fixed;
    for (int n = 0; n < ts.order; ++n)
      fixed.push_back(ftkref::build_mode_index(ts, n, ftkref::Keying::kFixedMode));
    ftkref::EpochOptions eo;
    eo.workers = workers;
    eo.canonical_order = canonical != 0;
    auto st = ftkref::epoch_fasttucker(ts, fixed, *static_cast<ftkref::Model*>(m),
                                       hyper(lr_a, lr_b, reg_a, reg_b, 1, batch), eo, seed);
    if (seconds2) {
      seconds2[0] = st.seconds_factor;
      seconds2[1] = st.seconds_core;
    }
    if (counters_out) {
      const ftkref::CostCounters* cs[2] = {&st.factor, &st.core};
      for (int p = 0; p < 2; ++p)
        for (int s = 0; s < ftkref::kStages; ++s)
          counters_out[p * ftkref::kStages + s] = cs[p]->total(static_cast<ftkref::Stage>(s));
    }
  });
}

// ftkref::epoch_fastertucker with complement indices of every mode and a
// freshly built C cache (as train() sets it up, decomposition.cpp:869-874).
int ref_epoch_fastertucker(void* t, void* m, float lr_a, float lr_b, float reg_a, float reg_b,
                           int batch, int workers, int canonical, uint64_t seed,
                           int64_t* counters_out) {
  return guarded([&] {
    const auto& ts = *static_cast<ftkref::SparseTensor*>(t);
    auto& md = *static_cast<ftkref::Model*>(m);
    std::vector<ftkref::ModeIndex> comp;
    for (int n = 0; n < ts.order; ++n)
      comp.push_back(ftkref::build_mode_index(ts, n, ftkref::Keying::kFixedComplement));
    ftkref::CCache cache;
    cache.build(md, nullptr);
    ftkref::EpochOptions eo;
    eo.workers = workers;
    eo.canonical_order = canonical != 0;
    auto st = ftkref::epoch_fastertucker(ts, comp, md, cache,
                                         hyper(lr_a, lr_b, reg_a, reg_b, 1, batch), eo, seed);
    if (counters_out) {
      const ftkref::CostCounters* cs[2] = {&st.factor, &st.core};
      for (int p = 0; p < 2; ++p)
        for (int s = 0; s < ftkref::kStages; ++s)
          counters_out[p * ftkref::kStages + s] = cs[p]->total(static_cast<ftkref::Stage>(s));
    }
  });
}

// Per-epoch trajectory of ftkref::train (plus variant).
int ref_train_variant(void* train, void* test, void* m, float lr_a, float lr_b,
                      float reg_a, float reg_b, int epochs, int batch, int workers,
                      int store_c, uint64_t seed, double* loss, double* rmse,
                      double* mae, double* seconds, int64_t* reads, int64_t* mults,
                      int variant) {
  return guarded([&] {
    ftkref::TrainOptions to;
    to.variant = variant == 1   ? ftkref::Variant::kFastTucker
                 : variant == 2 ? ftkref::Variant::kFasterTucker
                                : ftkref::Variant::kPlus;
    to.workers = workers;
    to.store_c = store_c != 0;
    to.seed = seed;
    auto hist = ftkref::train(*static_cast<ftkref::SparseTensor*>(train),
                              static_cast<ftkref::SparseTensor*>(test),
                              *static_cast<ftkref::Model*>(m),
                              hyper(lr_a, lr_b, reg_a, reg_b, epochs, batch),
                              to);
    for (size_t e = 0; e < hist.size(); ++e) {
      loss[e] = hist[e].train_loss;
      rmse[e] = hist[e].test_rmse;
      mae[e] = hist[e].test_mae;
      if (seconds) seconds[e] = hist[e].seconds;
      if (reads) reads[e] = hist[e].reads;
      if (mults) mults[e] = hist[e].mults;
    }
  });
}

int ref_train(void* train, void* test, void* m, float lr_a, float lr_b,
              float reg_a, float reg_b, int epochs, int batch, int workers,
              int store_c, uint64_t seed, double* loss, double* rmse,
              double* mae, double* seconds, int64_t* reads, int64_t* mults) {
  return ref_train_variant(train, test, m, lr_a, lr_b, reg_a, reg_b, epochs, batch, workers,
                           store_c, seed, loss, rmse, mae, seconds, reads, mults, 0);
}

int ref_loss(void* m, void* t, double reg_a, double reg_b, int workers,
             double* out) {
  return guarded([&] {
    *out = ftkref::loss(*static_cast<ftkref::Model*>(m),
                        *static_cast<ftkref::SparseTensor*>(t), reg_a, reg_b,
                        workers);
  });
}

int ref_evaluate(void* m, void* t, int workers, double* rmse, double* mae) {
  return guarded([&] {
    auto mt = ftkref::evaluate(*static_cast<ftkref::Model*>(m),
                               *static_cast<ftkref::SparseTensor*>(t), workers);
    *rmse = mt.rmse;
    *mae = mt.mae;
  });
}

int ref_history_line(void* train, void* m, float lr_a, int epochs, char* buf,
                     int cap) {
  return guarded([&] {
    ftkref::TrainOptions to;
    ftkref::Hyperparams h = hyper(lr_a, lr_a, 1e-4f, 1e-4f, epochs, 16);
    auto hist = ftkref::train(*static_cast<ftkref::SparseTensor*>(train),
                              nullptr, *static_cast<ftkref::Model*>(m), h, to);
    std::string s = hist.empty() ? "" : ftkref::history_line_json(hist.back());
    std::snprintf(buf, cap, "%s", s.c_str());
  });
}

// ---- one batch through the public per-batch pipeline -----------------------
//
// rows: entry positions (m_eff of them), batch capacity `cap`.  Outputs are
// dense [order][cap][R] for C and D, [order][cap][Jmax] for U and the
// updated (scattered) A rows, [cap] for the two predictions/residuals and
// [order][Jmax][R] for the core gradient of this batch.  The model `m` is
// mutated by update_factors_plus exactly as in the factor phase.
int ref_batch_probe(void* tp, void* mp, const int64_t* rows, int m_eff, int cap,
                    float lr_a, float reg_a, float* c_out, float* d_out,
                    float* u_out, float* xhat_f, float* resid_f, float* xhat_c,
                    float* resid_c, float* a_new, float* g_out) {
  return guarded([&] {
    auto& t = *static_cast<ftkref::SparseTensor*>(tp);
    auto& m = *static_cast<ftkref::Model*>(mp);
    const int order = m.order();
    int jmax = 0;
    for (int n = 0; n < order; ++n) jmax = std::max(jmax, m.ranks[n]);
    const int r = m.r;
    ftkref::Batch b;
    b.stage(t, std::span<const int64_t>(rows, static_cast<size_t>(m_eff)), cap,
            -1);
    ftkref::Workspace ws;
    ws.prepare(m, cap);
    ws.batch = b;
    ftkref::CoreTiles bt = ftkref::snapshot_core_tiles(m);
    ftkref::stage_factor_rows(m, ws, -1, nullptr);
    ftkref::compute_c_batch(bt, ws, -1, nullptr);
    ftkref::compute_d_batch(ws, nullptr);
    ftkref::compute_u_batch(bt, ws, nullptr);
    ftkref::predict_batch_factor_side(ws, nullptr);
    for (int n = 0; n < order; ++n) {
      dense_copy(ws.c[n], c_out + static_cast<size_t>(n) * cap * r, cap, r, r);
      dense_copy(ws.d[n], d_out + static_cast<size_t>(n) * cap * r, cap, r, r);
      dense_copy(ws.u[n], u_out + static_cast<size_t>(n) * cap * jmax, cap,
                 m.ranks[n], jmax);
    }
    for (int i = 0; i < cap; ++i) {
      xhat_f[i] = ws.xhat[i];
      resid_f[i] = ws.resid[i];
    }
    ftkref::Hyperparams h = hyper(lr_a, 1e-3f, reg_a, 1e-4f, 1, cap);
    ftkref::update_factors_plus(m, h, ws, nullptr);
    for (int n = 0; n < order; ++n)
      for (int i = 0; i < m_eff; ++i)
        for (int j = 0; j < m.ranks[n]; ++j)
          a_new[(static_cast<size_t>(n) * cap + i) * jmax + j] =
              m.a_row(n, b.idx[n][i])[j];
    ftkref::predict_batch_c_side(ws, nullptr);
    for (int i = 0; i < cap; ++i) {
      xhat_c[i] = ws.xhat[i];
      resid_c[i] = ws.resid[i];
    }
    ftkref::CoreGradAccumulator acc;
    acc.reset(m);
    ftkref::accumulate_core_grads_plus(ws, acc, nullptr);
    for (int n = 0; n < order; ++n)
      for (int j = 0; j < m.ranks[n]; ++j)
        for (int c = 0; c < r; ++c)
          g_out[(static_cast<size_t>(n) * jmax + j) * r + c] =
              acc.grad[n][static_cast<size_t>(j) * r + c];
  });
}

void ref_predicted_costs(int order, int m, int r, const int32_t* ranks,
                         int64_t* out4) {
  std::vector<int32_t> j(ranks, ranks + order);
  auto p = ftkref::predicted_costs(order, m, r, j, ftkref::Variant::kPlus);
  out4[0] = p.reads;
  out4[1] = p.d_stage;
  out4[2] = p.bdt_stage;
  out4[3] = p.update;
}

}  // extern "C"
