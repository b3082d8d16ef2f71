// ftk/decomposition.hpp -- drop-in for the FastTuckerPlus drivers of
// /root/reference/proj/include/ftk/decomposition.hpp (EpochOptions,
// EpochStats, epoch_plus, TrainOptions, EpochRecord, train, history I/O:
// decomposition.hpp:166-242).
//
// Not declared (out of the engine's scope):
//   * the host per-batch pipeline and its 16x16 tile layer (Workspace,
//     CoreTiles, TiledMatrix; decomposition.hpp:14-124, tiles.hpp) -- the
//     reference's CPU stand-in for WMMA, replaced by the device kernels; the
//     device equivalent for parity probing is ftkcu_batch_probe (ftkcu.h);
//   * the convex FastTucker / FasterTucker variants (f4).
#pragma once

#include <string>
#include <vector>

#include "ftk/counters.hpp"
#include "ftk/evaluation.hpp"
#include "ftk/model.hpp"
#include "ftk/sparse_tensor.hpp"

namespace ftk {

// Cached C rows C_n = A_n B_n of every mode, for the FasterTucker baseline
// (decomposition.hpp:26-44 of the reference).  build / refresh compute on the
// host; epoch_fastertucker keeps the device copy in step and writes the
// refreshed rows back.
class CCache {
 public:
  void init(const Model& m);
  void build(const Model& m, CostCounters* cc);
  void refresh(const Model& m, int mode, CostCounters* cc);
  void mark_stale(int mode) { fresh_[mode] = 0; }
  bool fresh(int mode) const { return fresh_[mode] != 0; }
  bool ready() const { return !c_.empty(); }
  std::span<const real> row(int mode, index_t i) const {
    return {c_[mode].data() + static_cast<std::size_t>(i) * r_, static_cast<std::size_t>(r_)};
  }
  // Engine additions: the per-mode row storage (dims[n] x R, row-major), and
  // marking rows refreshed on the device.
  std::vector<std::vector<real>>& storage() { return c_; }
  void mark_fresh(int mode) { fresh_[mode] = 1; }

 private:
  std::vector<std::vector<real>> c_;
  std::vector<char> fresh_;
  index_t r_ = 0;
};

struct EpochOptions {
  int workers = 1;               // 1: deterministic sweeps; > 1: Hogwild
  bool canonical_order = false;  // storage order, single-entry batches
  bool eager_refresh = false;    // FasterTucker per-batch refresh hook (not supported)
  bool store_c = false;          // storage scheme: core phase reads C rows from a C cache
};

struct EpochStats {
  double seconds_factor = 0.0;  // device time of the factor sweep
  double seconds_core = 0.0;    // device time of the core sweep + apply
  CostCounters factor;
  CostCounters core;
};

EpochStats epoch_plus(const SparseTensor& t, Model& m, const Hyperparams& h,
                      const EpochOptions& opts, std::uint64_t seed);

// The FasterTucker baseline (decomposition.hpp:201-206 of the reference):
// complement-keyed buckets, d rows from the C cache (which must be built),
// the block's cache rows refreshed at each block barrier.  Bit-identical to
// the reference with workers = 1 (the device schedule is order-equivalent).
EpochStats epoch_fastertucker(const SparseTensor& t, const std::vector<ModeIndex>& complement,
                              Model& m, CCache& cache, const Hyperparams& h,
                              const EpochOptions& opts, std::uint64_t seed);

// The FastTucker baseline (decomposition.hpp:194-199 of the reference):
// factor blocks over per-bucket plans of the fixed-mode indices, then core
// blocks with B^(n) moving every batch.  Runs on the device in the
// workers == 1 arithmetic (bit-identical to the reference with workers = 1).
EpochStats epoch_fasttucker(const SparseTensor& t, const std::vector<ModeIndex>& fixed_mode,
                            Model& m, const Hyperparams& h, const EpochOptions& opts,
                            std::uint64_t seed);

struct TrainOptions {
  Variant variant = Variant::kPlus;  // kPlus, kFastTucker or kFasterTucker
  bool store_c = false;
  int workers = 1;
  std::uint64_t seed = 0;
};

struct EpochRecord {
  int epoch = 0;
  double train_loss = 0.0;
  double test_rmse = 0.0;
  double test_mae = 0.0;
  double seconds = 0.0;
  size64 reads = 0;
  size64 mults = 0;
  EpochStats stats;
};

using History = std::vector<EpochRecord>;

// h.epochs epochs with the model resident on the device; fp64 train loss and
// test metrics per epoch; throws on a non-finite loss.
History train(const SparseTensor& train_set, const SparseTensor* test_set,
              Model& m, const Hyperparams& h, const TrainOptions& opts);

void write_history_jsonl(const History& h, const std::string& path);
void write_history_csv(const History& h, const std::string& path);
std::string history_line_json(const EpochRecord& r);

// ---- engine additions (no reference counterpart) ---------------------------

enum class DeviceMode { kAuto, kDeterministic, kHogwild };
enum class DevicePrecision { kFp32, kTf32, k3xTf32 };

struct DeviceOptions {
  int device = -1;                 // -1: $FTK_DEVICE, else 0
  DeviceMode mode = DeviceMode::kAuto;  // kAuto: workers == 1 -> deterministic
  // Hogwild sweeps (workers > 1): tf32 factor / fp16-copy core operands with
  // fp32 accumulate on the tensor cores -- test-RMSE parity with the
  // reference is tests/test_accuracy_gpu.py and bench.py's
  // test_rmse_vs_reference; kFp32 runs the fp32 CUDA-core sweeps, k3xTf32
  // fp32-equivalent split products.  Deterministic mode (workers == 1) is
  // bit-exact fp32 whatever this says.
  DevicePrecision precision = DevicePrecision::kTf32;
  bool exact_eval = true;          // reference slab order in loss/evaluate
  // Hogwild at the reference's asynchrony noise floor: at most 3 tiles per
  // CTA between reading a row and writing it back (session option window =
  // 3) on half the SMs (max_ctas) -- on unlearnable (uniform) values the
  // full grid's ~57K nonzeros in flight raise the test RMSE by 3-4e-3, this
  // by < 1e-3, at about 2x the epoch time (bench.py's `parity` variant).
  bool parity = false;
};

void set_device_options(const DeviceOptions& o);
DeviceOptions device_options();

// Which sweep kernels the last factor / core phase ran (FTKCU_K_* ids of
// include/ftkcu.h), so callers and tests can see the dispatch.
struct DeviceKernels {
  int factor = 0;
  int core = 0;
};
DeviceKernels device_last_kernels();

}  // namespace ftk
