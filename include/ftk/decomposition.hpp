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

struct EpochOptions {
  int workers = 1;               // 1: deterministic sweeps; > 1: Hogwild
  bool canonical_order = false;  // storage order, single-entry batches
  bool eager_refresh = false;    // FasterTucker hook (ignored)
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

// The FastTucker baseline (decomposition.hpp:194-199 of the reference):
// factor blocks over per-bucket plans of the fixed-mode indices, then core
// blocks with B^(n) moving every batch.  Runs on the device in the
// workers == 1 arithmetic (bit-identical to the reference with workers = 1).
EpochStats epoch_fasttucker(const SparseTensor& t, const std::vector<ModeIndex>& fixed_mode,
                            Model& m, const Hyperparams& h, const EpochOptions& opts,
                            std::uint64_t seed);

struct TrainOptions {
  Variant variant = Variant::kPlus;  // kPlus or kFastTucker (kFasterTucker: not built)
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
  DevicePrecision precision = DevicePrecision::kFp32;
  bool exact_eval = true;          // reference slab order in loss/evaluate
};

void set_device_options(const DeviceOptions& o);
DeviceOptions device_options();

}  // namespace ftk
