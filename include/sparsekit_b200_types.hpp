// sparsekit_b200_types.hpp -- stand-in value types for building the C++ facade WITHOUT the
// reference headers (this repository's own tests, the GPU box).
//
// When the reference tree is on the include path, sparsekit_b200.hpp includes the reference's
// own headers instead and this file is not used.  Field names and meanings follow
//   MoEConfig / MoELayerWeights   proj/include/sparsekit/model.hpp:15-43
//   Matrix / MacCounter           proj/include/sparsekit/linalg.hpp:17-70
//   RouteResult / DispatchPlan    proj/include/sparsekit/router.hpp:20-44
//   SparsityLevel                 proj/include/sparsekit/activation.hpp:15-23
//   ForwardReport / MaskSet       proj/include/sparsekit/engine.hpp:19-34
//   SwitchTable / Stopwatch       proj/include/sparsekit/engine.hpp:52-69
//   SweepMode                     proj/include/sparsekit/profiler.hpp:38
//   BudgetRatios / ExpertGroups   proj/include/sparsekit/budget.hpp:15-28
//   exception types               proj/include/sparsekit/errors.hpp:12-43
// so that code written against the reference compiles against either.
#pragma once

#include <cstddef>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace sparsekit {

struct ShapeError : std::invalid_argument {
  explicit ShapeError(const std::string& m) : std::invalid_argument(m) {}
};
struct IndexError : std::out_of_range {
  explicit IndexError(const std::string& m) : std::out_of_range(m) {}
};
struct ConfigError : std::invalid_argument {
  explicit ConfigError(const std::string& m) : std::invalid_argument(m) {}
};
struct InternalError : std::logic_error {
  explicit InternalError(const std::string& m) : std::logic_error(m) {}
};

struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct FormatError : std::runtime_error {  // errors.hpp:36-43: carries the byte offset
  FormatError(const std::string& m, std::uint64_t at) : std::runtime_error(m), offset(at) {}
  std::uint64_t offset;
};

struct Matrix {
  int rows = 0, cols = 0;
  std::vector<float> data;
  Matrix() = default;
  Matrix(int r, int c) : rows(r), cols(c), data(static_cast<std::size_t>(r) * c, 0.0f) {}
  float& at(int r, int c) { return data[static_cast<std::size_t>(r) * cols + c]; }
  float at(int r, int c) const { return data[static_cast<std::size_t>(r) * cols + c]; }
};

struct MacCounter {
  std::uint64_t gate_macs = 0, up_macs = 0, down_macs = 0, other_macs = 0;
  std::uint64_t total() const { return gate_macs + up_macs + down_macs + other_macs; }
};

struct MoEConfig {
  int n_experts = 1, top_k = 1, d_model = 1, d_ffn = 1;
  bool has_shared = false;
  int d_shared = 0;
  bool renormalize = true;
  int align_block = 64;
  static constexpr int kTile = 64;
};

struct MoELayerWeights {
  MoEConfig config;
  Matrix router;
  std::vector<Matrix> gate, up, down_t;
  Matrix shared_gate, shared_up, shared_down_t;
};

struct RouteResult {
  int batch = 0, top_k = 0;
  std::vector<std::int32_t> ids;
  std::vector<float> weights;
};

struct DispatchPlan {
  std::vector<std::int32_t> sorted_token_slots, expert_of_block;
  int block_size = 0, n_padded = 0;
};

struct SparsityLevel {
  double s = 0.0;
  explicit SparsityLevel(double v) : s(v) {
    if (!(v >= 0.0 && v <= 1.0)) throw ConfigError("sparsity must lie in [0, 1]");
  }
};

// activation.hpp:17, 53-57
constexpr std::int32_t kPadIndex = -1;
struct ActiveIndexRow {
  std::vector<std::int32_t> flat;             // capacity entries
  std::vector<std::int32_t> active_per_slot;  // one count per slot
  std::int32_t total_active = 0;
};

enum class ExecPath { kDense, kSparse };
enum class SweepMode { kRoutedOnly, kRoutedAndShared };

// profiler.hpp:49-61
struct SweepPoint {
  double target = 0.0;
  double achieved_total = 0.0;
  double achieved_routed = 0.0;
  double quality = 0.0;
  double rel_error = 0.0;
  std::string path;  // "R" or "R+S"
};
struct SweepResult {
  std::vector<SweepPoint> points;
  double cutoff = 0.0;
};

struct ForwardReport {
  Matrix outputs;
  MacCounter macs;
  std::uint64_t active_neurons_total = 0;
  double achieved_routed_sparsity = 0.0;
  std::uint64_t tiles_total = 0, tiles_skipped = 0;
  ExecPath path_used = ExecPath::kDense;
};

struct MaskSet {
  std::vector<std::uint8_t> routed, shared;
};

// batches of at least tipping_batch run dense; kSparseAlways = never
struct SwitchTable {
  static constexpr std::size_t kSparseAlways = std::numeric_limits<std::size_t>::max();
  std::size_t tipping_batch = kSparseAlways;
  bool use_dense(std::size_t batch) const { return batch >= tipping_batch; }
};

// distribution ratios of the three router-weight groups; slot indices by router weight
struct BudgetRatios {
  double r0 = 1.0, r1 = 1.0, r2 = 1.0;
};
struct ExpertGroups {
  std::vector<int> g0, g1, g2;
};

// injectable monotonic clock (milliseconds)
class Stopwatch {
 public:
  virtual ~Stopwatch() = default;
  virtual double now_ms() = 0;
};

}  // namespace sparsekit
