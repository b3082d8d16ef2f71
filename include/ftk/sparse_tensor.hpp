// ftk/sparse_tensor.hpp -- drop-in for the reference's COO store, loader,
// split and global sampler (/root/reference/proj/include/ftk/
// sparse_tensor.hpp:14-121).
//
// The per-mode bucket samplers (Keying / ModeIndex / EpochPlan::per_bucket)
// serve the convex FastTucker baseline.
#pragma once

#include <span>
#include <string>
#include <utility>
#include <vector>

#include "ftk/common.hpp"

namespace ftk {

// Order-N COO tensor on the host: AoS indices (nnz x order, 0-based), fp32
// values.  The engine transposes it to SoA columns on upload.
struct SparseTensor {
  int order = 0;
  std::vector<index_t> dims;
  std::vector<index_t> indices;
  std::vector<real> values;

  size64 nnz() const { return static_cast<size64>(values.size()); }
  std::span<const index_t> entry(size64 p) const {
    return {indices.data() + p * order, static_cast<std::size_t>(order)};
  }
  void push(std::span<const index_t> idx, real v) {
    indices.insert(indices.end(), idx.begin(), idx.end());
    values.push_back(v);
  }
  // Index ranges, finite values, no repeated tuple.
  void validate() const;
};

// FROSTT text: "i_1 .. i_N value" per line, 1-based, '#' comments, optional
// "# dims: I_1 .. I_N" header; duplicates / out-of-range are errors.
SparseTensor load_coo(const std::string& path, int order);
void save_coo(const SparseTensor& t, const std::string& path);
int infer_coo_order(const std::string& path);

// Binary COO ("FTKC1", engine addition next to the FROSTT text format, which
// parses at ~10^6 lines/s): magic "FTKC1\0\0\0", int32 order, int64 nnz,
// int32 dims[order], int32 indices[nnz * order] (0-based, AoS, as in
// SparseTensor), float values[nnz]; little-endian.  load_coo_binary runs
// SparseTensor::validate like load_coo.
SparseTensor load_coo_binary(const std::string& path);
void save_coo_binary(const SparseTensor& t, const std::string& path);

// Seeded disjoint split; |test| = llround(fraction * nnz) clamped to
// [1, nnz-1]; test entries in permutation order.
std::pair<SparseTensor, SparseTensor> split_train_test(const SparseTensor& t,
                                                       double test_fraction,
                                                       std::uint64_t seed);

// One staged batch (columns); rows >= m_eff are padding (value 0, index 0).
struct Batch {
  index_t m = 0;
  index_t m_eff = 0;
  size64 bucket = -1;
  std::vector<real> values;
  std::vector<std::vector<index_t>> idx;

  bool full() const { return m_eff == m; }
  void stage(const SparseTensor& t, std::span<const size64> rows, index_t m_cap,
             size64 bucket_id);
};

struct BatchDesc {
  size64 offset = 0;
  size64 len = 0;
  size64 bucket = -1;
};

// Entry positions grouped into buckets for one mode (sparse_tensor.hpp:50-72
// of the reference): kFixedMode buckets share the mode-n index,
// kFixedComplement buckets share every other index.  Positions inside a
// bucket stay in storage order; buckets are in key order.
enum class Keying { kFixedMode, kFixedComplement };

struct ModeIndex {
  int mode = 0;
  Keying keying = Keying::kFixedMode;
  std::vector<size64> positions;
  std::vector<size64> offsets;  // bucket b spans [offsets[b], offsets[b+1])

  size64 buckets() const { return static_cast<size64>(offsets.size()) - 1; }
  std::span<const size64> bucket(size64 b) const {
    return {positions.data() + offsets[b], static_cast<std::size_t>(offsets[b + 1] - offsets[b])};
  }
  size64 representative(size64 b) const { return positions[offsets[b]]; }
};

ModeIndex build_mode_index(const SparseTensor& t, int mode, Keying keying);

// The FastTuckerPlus (global) sampler: a uniform permutation of all entries
// cut into batches of m, the last one short.  Bit-identical to the
// reference's plans for the same Rng state (same libstdc++ std::shuffle).
class EpochPlan {
 public:
  static EpochPlan global(const SparseTensor& t, index_t m, Rng& rng);
  static EpochPlan canonical(const SparseTensor& t);  // storage order, m = 1
  // Bucket order shuffled, then each bucket's entries, cut into batches of m
  // that never cross a bucket (the FastTucker / FasterTucker samplers).
  static EpochPlan per_bucket(const SparseTensor& t, const ModeIndex& idx, index_t m, Rng& rng);

  size64 batches() const { return static_cast<size64>(descs_.size()); }
  const BatchDesc& desc(size64 b) const { return descs_[b]; }
  void gather(const SparseTensor& t, size64 b, Batch& out) const;

  // Engine additions: the flat permutation handed to the device sweeps.
  const std::vector<size64>& positions() const { return perm_; }
  index_t batch_size() const { return m_; }
  // per_bucket plans: offsets of the buckets (in plan order) in positions(),
  // with a final nnz; empty for global / canonical plans.
  const std::vector<size64>& bucket_offsets() const { return boff_; }

 private:
  index_t m_ = 0;
  std::vector<size64> perm_;
  std::vector<BatchDesc> descs_;
  std::vector<size64> boff_;
};

}  // namespace ftk
