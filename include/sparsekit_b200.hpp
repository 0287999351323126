// sparsekit_b200.hpp -- C++ facade: the reference's layer API on top of the C ABI.
//
// Same names, signatures, value types and exception types as the reference
// (proj/include/sparsekit/{engine,router,activation,profiler}.hpp), in namespace
// sparsekit::b200, so a call site switches with one `using` / namespace change:
//
//     sparsekit::forward_dense(w, x, threads)        ->  sparsekit::b200::forward_dense(w, x, threads)
//     sparsekit::forward_masked_dense(w, x, masks)   ->  sparsekit::b200::forward_masked_dense(...)
//     sparsekit::build_topk_masks(w, x, s, mode)     ->  sparsekit::b200::build_topk_masks(...)
//     route / align_dispatch / combine / topk_mask / mask_smallest_magnitudes likewise
//
// plus forward_topk_sparse(w, x, s_routed, s_shared), the fused entry the reference lacks
// (== forward_masked_dense(w, x, build_topk_masks(w, x, s, mode)) with the selection done on
// the device and the masked W_down rows never read).
//
// Header-only; link libsparsekit_b200.so.  With the reference tree on the include path the
// reference's own headers provide the types, otherwise sparsekit_b200_types.hpp does.
//
// The device weight image is cached per MoELayerWeights instance (keyed on its address, shape
// and a content stamp) so repeated forwards upload nothing; release(w) or clear_cache() drops it.
#pragma once

#if __has_include("sparsekit/engine.hpp")
#include "sparsekit/activation.hpp"
#include "sparsekit/budget.hpp"
#include "sparsekit/engine.hpp"
#include "sparsekit/profiler.hpp"
#include "sparsekit/router.hpp"
#else
#include "sparsekit_b200_types.hpp"
#endif

#include <algorithm>
#include <chrono>
#include <cmath>
#include <numeric>
#include <cstdio>
#include <cstring>
#include <type_traits>
#include <initializer_list>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "sparsekit_b200.h"

namespace sparsekit {
namespace b200 {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {

// C status codes back to the reference exception types (errors.hpp:12-43)
inline void check(int rc) {
  if (rc == SKB_OK) return;
  const std::string msg = skb_last_error();
  switch (rc) {
    case SKB_ESHAPE: throw ShapeError(msg);
    case SKB_ECONFIG: throw ConfigError(msg);
    case SKB_EINDEX: throw IndexError(msg);
    case SKB_EINTERNAL: throw InternalError(msg);
    default: throw CudaError(msg);
  }
}

inline skb_config to_c(const MoEConfig& c) {
  return skb_config{c.n_experts, c.top_k,    c.d_model,          c.d_ffn,
                    c.has_shared ? 1 : 0, c.d_shared, c.renormalize ? 1 : 0, c.align_block};
}

struct Entry {
  skb_layer* layer = nullptr;
  std::uint64_t stamp = 0;
};

inline std::mutex& cache_mutex() {
  static std::mutex m;
  return m;
}
inline std::map<const MoELayerWeights*, Entry>& cache() {
  static std::map<const MoELayerWeights*, Entry> c;
  return c;
}

// cheap content stamp: shape + a few words of every matrix (weights are immutable after load,
// SPEC.md:124; the stamp only guards against an address being reused by another model)
inline std::uint64_t stamp_of(const MoELayerWeights& w) {
  std::uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* p, std::size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  const skb_config c = to_c(w.config);
  mix(&c, sizeof(c));
  auto sample = [&](const Matrix& m) {
    const std::size_t n = m.data.size();
    if (n == 0) return;
    const std::size_t k = n < 16 ? n : 16;
    mix(m.data.data(), k * sizeof(float));
    mix(m.data.data() + (n - k), k * sizeof(float));
    const void* addr = m.data.data();
    mix(&addr, sizeof(addr));
  };
  sample(w.router);
  for (const Matrix& m : w.gate) sample(m);
  for (const Matrix& m : w.up) sample(m);
  for (const Matrix& m : w.down_t) sample(m);
  sample(w.shared_gate);
  sample(w.shared_up);
  sample(w.shared_down_t);
  return h;
}

inline skb_layer* layer_for(const MoELayerWeights& w, int device = 0) {
  std::lock_guard<std::mutex> lk(cache_mutex());
  const std::uint64_t st = stamp_of(w);
  Entry& e = cache()[&w];
  if (e.layer != nullptr && e.stamp == st) return e.layer;
  if (e.layer != nullptr) {
    skb_layer_destroy(e.layer);
    e.layer = nullptr;
  }
  const MoEConfig& c = w.config;
  const skb_config cc = to_c(c);
  check(skb_config_validate(&cc));
  const std::size_t E = static_cast<std::size_t>(c.n_experts);
  auto want = [&](const Matrix& m, int r, const char* what) {
    if (m.rows != r || m.cols != c.d_model ||
        m.data.size() != static_cast<std::size_t>(r) * c.d_model)
      throw ShapeError(std::string("weights: ") + what + " has the wrong shape");
  };
  want(w.router, c.n_experts, "router");
  if (w.gate.size() != E || w.up.size() != E || w.down_t.size() != E)
    throw ShapeError("weights: expected one gate/up/down_t matrix per expert");
  std::vector<const float*> g(E), u(E), d(E);
  for (std::size_t i = 0; i < E; ++i) {
    want(w.gate[i], c.d_ffn, "gate");
    want(w.up[i], c.d_ffn, "up");
    want(w.down_t[i], c.d_ffn, "down_t");
    g[i] = w.gate[i].data.data();
    u[i] = w.up[i].data.data();
    d[i] = w.down_t[i].data.data();
  }
  const float *sg = nullptr, *su = nullptr, *sd = nullptr;
  if (c.has_shared) {
    want(w.shared_gate, c.d_shared, "shared_gate");
    want(w.shared_up, c.d_shared, "shared_up");
    want(w.shared_down_t, c.d_shared, "shared_down_t");
    sg = w.shared_gate.data.data();
    su = w.shared_up.data.data();
    sd = w.shared_down_t.data.data();
  }
  skb_layer* L = nullptr;
  check(skb_layer_create(&cc, w.router.data.data(), g.data(), u.data(), d.data(), sg, su, sd,
                         device, &L));
  e.layer = L;
  e.stamp = st;
  return L;
}

inline ForwardReport run(const MoELayerWeights& w, const Matrix& x, skb_forward_args a,
                         MaskSet* masks_out = nullptr) {
  const MoEConfig& c = w.config;
  if (x.cols != c.d_model)  // engine.cpp:98-101
    throw ShapeError("forward: token width does not match d_model");
  skb_layer* L = layer_for(w);
  ForwardReport rep;
  rep.outputs = Matrix(x.rows, c.d_model);
  a.batch = x.rows;
  a.x = x.data.data();
  a.y = rep.outputs.data.data();
  if (masks_out != nullptr) {
    masks_out->routed.assign(static_cast<std::size_t>(x.rows) * c.top_k * c.d_ffn, 0);
    a.routed_mask_out = masks_out->routed.data();
    if (c.has_shared) {
      masks_out->shared.assign(static_cast<std::size_t>(x.rows) * c.d_shared, 0);
      a.shared_mask_out = masks_out->shared.data();
    }
  }
  skb_report r{};
  check(skb_layer_forward(L, &a, &r));
  rep.macs.gate_macs = r.gate_macs;
  rep.macs.up_macs = r.up_macs;
  rep.macs.down_macs = r.down_macs;
  rep.macs.other_macs = r.other_macs;
  rep.active_neurons_total = r.active_neurons_total;
  rep.achieved_routed_sparsity = r.achieved_routed_sparsity;
  rep.tiles_total = r.tiles_total;
  rep.tiles_skipped = r.tiles_skipped;
  rep.path_used = r.path_used ? ExecPath::kSparse : ExecPath::kDense;
  return rep;
}

}  // namespace detail

// Drops the cached device image of `w` (call before destroying or mutating it).
inline void release(const MoELayerWeights& w) {
  std::lock_guard<std::mutex> lk(detail::cache_mutex());
  auto it = detail::cache().find(&w);
  if (it != detail::cache().end()) {
    skb_layer_destroy(it->second.layer);
    detail::cache().erase(it);
  }
}
inline void clear_cache() {
  std::lock_guard<std::mutex> lk(detail::cache_mutex());
  for (auto& kv : detail::cache()) skb_layer_destroy(kv.second.layer);
  detail::cache().clear();
}

// engine.hpp:38-39.  `threads` is accepted for signature parity and ignored.
inline ForwardReport forward_dense(const MoELayerWeights& w, const Matrix& x, int /*threads*/ = 1) {
  skb_forward_args a{};
  a.mode = SKB_MODE_DENSE;
  return detail::run(w, x, a);
}

// engine.hpp:43-44
inline ForwardReport forward_masked_dense(const MoELayerWeights& w, const Matrix& x,
                                          const MaskSet& masks, int /*threads*/ = 1) {
  skb_forward_args a{};
  a.mode = SKB_MODE_MASKED;
  a.routed_mask_in = masks.routed.data();
  a.routed_mask_len = masks.routed.size();
  a.shared_mask_in = masks.shared.empty() ? nullptr : masks.shared.data();
  a.shared_mask_len = masks.shared.size();
  return detail::run(w, x, a);
}

// engine.hpp:46-51: the threshold runtime path.  A routed neuron is kept iff
// |silu(gate)| >= threshold; the shared expert stays dense; the report carries the reference's
// tile accounting (tiles_total / tiles_skipped, padded up/down MACs, path_used = kSparse).
inline ForwardReport forward_sparse(const MoELayerWeights& w, const Matrix& x, float threshold,
                                    int /*threads*/ = 1) {
  skb_forward_args a{};
  a.mode = SKB_MODE_THRESHOLD;
  a.tau = threshold;
  return detail::run(w, x, a);
}

// The fused top-k path.  s_shared = 0 leaves the shared expert dense (SweepMode::kRoutedOnly);
// pass the same level as s_routed for kRoutedAndShared.
inline ForwardReport forward_topk_sparse(const MoELayerWeights& w, const Matrix& x,
                                         SparsityLevel s_routed,
                                         SparsityLevel s_shared = SparsityLevel(0.0),
                                         int /*threads*/ = 1, MaskSet* masks_out = nullptr) {
  skb_forward_args a{};
  a.mode = SKB_MODE_TOPK;
  a.s_routed = s_routed.s;
  a.s_shared = s_shared.s;
  return detail::run(w, x, a, masks_out);
}

// profiler.hpp:71-72
inline MaskSet build_topk_masks(const MoELayerWeights& w, const Matrix& tokens, SparsityLevel s,
                                SweepMode mode) {
  MaskSet m;
  const bool rs = mode == SweepMode::kRoutedAndShared && w.config.has_shared;
  forward_topk_sparse(w, tokens, s, rs ? s : SparsityLevel(0.0), 1, &m);
  if (!rs) m.shared.clear();
  return m;
}

// ---- quality sweep and its report file (profiler.hpp:38-83) ----
// profiler.cpp:76-99
inline double mean_relative_error(const Matrix& outputs, const Matrix& dense_outputs) {
  if (outputs.rows != dense_outputs.rows || outputs.cols != dense_outputs.cols)
    throw ShapeError("mean_relative_error: shape mismatch");
  double total = 0.0;
  int used = 0;
  for (int t = 0; t < outputs.rows; ++t) {
    const float* y = outputs.data.data() + static_cast<std::size_t>(t) * outputs.cols;
    const float* d = dense_outputs.data.data() + static_cast<std::size_t>(t) * outputs.cols;
    double err2 = 0.0, ref2 = 0.0;
    for (int c = 0; c < outputs.cols; ++c) {
      const double dv = d[c], e = static_cast<double>(y[c]) - dv;
      err2 += e * e;
      ref2 += dv * dv;
    }
    const double ref = std::sqrt(ref2);
    if (ref >= 1e-12) {
      total += std::sqrt(err2) / ref;
      ++used;
    }
  }
  return used ? total / used : 0.0;
}

// profiler.hpp:66-69: every point is one fused top-k forward on the device (the selection runs
// inside the layer; same masks and outputs as build_topk_masks + forward_masked_dense).
// Metric: any callable (outputs, dense outputs) -> double, or nullptr for 1 - rel_error.
template <class Metric = std::nullptr_t>
inline SweepResult sweep_cutoff(const MoELayerWeights& w, const Matrix& eval_tokens,
                                const double* targets, std::size_t n_targets, double retention,
                                SweepMode mode, Metric metric = nullptr) {
  if (n_targets == 0) throw ConfigError("sweep_cutoff: no targets");
  for (std::size_t i = 0; i < n_targets; ++i) {
    if (!(targets[i] >= 0.0 && targets[i] <= 1.0))
      throw ConfigError("sweep_cutoff: targets must lie in [0, 1]");
    if (i && !(targets[i] > targets[i - 1]))
      throw ConfigError("sweep_cutoff: targets must be strictly increasing");
  }
  if (!(retention > 0.0 && retention <= 1.0))
    throw ConfigError("sweep_cutoff: retention must lie in (0, 1]");
  const MoEConfig& cfg = w.config;
  const ForwardReport dense = b200::forward_dense(w, eval_tokens);
  const bool rs = mode == SweepMode::kRoutedAndShared && cfg.has_shared;
  const auto point_at = [&](double target) {
    MaskSet masks;
    const SparsityLevel lvl(target);
    const ForwardReport rep =
        forward_topk_sparse(w, eval_tokens, lvl, rs ? lvl : SparsityLevel(0.0), 1, &masks);
    SweepPoint p;
    p.target = target;
    p.rel_error = b200::mean_relative_error(rep.outputs, dense.outputs);
    if constexpr (std::is_same<Metric, std::nullptr_t>::value)
      p.quality = 1.0 - p.rel_error;
    else
      p.quality = metric(rep.outputs, dense.outputs);
    p.achieved_routed = rep.achieved_routed_sparsity;
    std::uint64_t shared_off = 0;
    if (rs)
      for (std::uint8_t m : masks.shared) shared_off += m ? 0 : 1;
    const std::uint64_t routed = static_cast<std::uint64_t>(eval_tokens.rows) * cfg.top_k * cfg.d_ffn;
    const std::uint64_t per_token = static_cast<std::uint64_t>(cfg.top_k) * cfg.d_ffn + cfg.d_shared;
    p.achieved_total = static_cast<double>(routed - rep.active_neurons_total + shared_off) /
                       static_cast<double>(static_cast<std::uint64_t>(eval_tokens.rows) * per_token);
    p.path = mode == SweepMode::kRoutedOnly ? "R" : "R+S";
    return p;
  };
  const SweepPoint zero = point_at(0.0);  // the floor always refers to the zero-sparsity point
  SweepResult out;
  for (std::size_t i = 0; i < n_targets; ++i)
    out.points.push_back(targets[i] == 0.0 ? zero : point_at(targets[i]));
  for (const SweepPoint& p : out.points)
    if (p.quality >= retention * zero.quality && p.target > out.cutoff) out.cutoff = p.target;
  return out;
}

// profiler.hpp:79-83 (C stdio instead of <filesystem>/<fstream>: the facade stays header-light)
inline void emit_report(const SweepResult& result, const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) throw IoError("cannot open for writing: " + path);
  bool ok = std::fputs("target,achieved_total,achieved_routed,quality,rel_error,path\n", f) >= 0;
  for (const SweepPoint& p : result.points)
    ok = ok && std::fprintf(f, "%.9g,%.9g,%.9g,%.9g,%.9g,%s\n", p.target, p.achieved_total,
                            p.achieved_routed, p.quality, p.rel_error, p.path.c_str()) > 0;
  if (!result.points.empty()) ok = ok && std::fprintf(f, "# cutoff=%.9g\n", result.cutoff) > 0;
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) throw IoError("write failed: " + path);
}

// model.cpp:168-178: the standard-normal token batch profile_tipping probes with (host libm,
// bit-identical to the reference's generate_tokens on the same host).
inline Matrix generate_tokens(int batch, int d_model, std::uint64_t seed) {
  if (batch < 1 || d_model < 1) throw ConfigError("token batch needs batch >= 1 and d_model >= 1");
  Matrix x(batch, d_model);
  detail::check(skb_generate_tokens(batch, d_model, seed, x.data.data()));
  return x;
}

// Wall clock around the synchronous host entry points (each returns after its device work and
// the copy back have completed, so host time IS layer time as a caller sees it).
class SteadyClock final : public Stopwatch {
 public:
  double now_ms() override {
    using clock = std::chrono::steady_clock;
    return std::chrono::duration<double, std::milli>(clock::now().time_since_epoch()).count();
  }
};

namespace detail {
inline double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  const std::size_t n = v.size();
  return n % 2 == 1 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}
}  // namespace detail

// engine.hpp:76-83, engine.cpp:371-412: smallest batch of the (ascending) grid whose dense median
// is at or below the sparse median, else kSparseAlways.  Per grid point: `repetitions` sparse
// runs, then `repetitions` dense runs, one now_ms() before and one after each; probe tokens are
// generate_tokens(batch, d_model, token_seed + grid index).  Grid: any contiguous int container
// (std::vector, std::array, std::span).
template <class Grid>
inline SwitchTable profile_tipping(const MoELayerWeights& w, float threshold, const Grid& batch_grid,
                                   int repetitions = 5, Stopwatch* clock = nullptr,
                                   std::uint64_t token_seed = 0) {
  const std::size_t n_grid = batch_grid.size();
  if (n_grid == 0) throw ConfigError("profile_tipping: empty batch grid");
  const int* grid = batch_grid.data();
  for (std::size_t i = 0; i < n_grid; ++i)
    if (grid[i] < 1 || (i > 0 && grid[i] <= grid[i - 1]))
      throw ConfigError("profile_tipping: grid must be ascending, >= 1");
  if (repetitions < 1) throw ConfigError("profile_tipping: repetitions must be >= 1");
  SteadyClock own;
  if (clock == nullptr) clock = &own;
  for (std::size_t gi = 0; gi < n_grid; ++gi) {
    const Matrix tokens = b200::generate_tokens(grid[gi], w.config.d_model, token_seed + gi);
    std::vector<double> sparse_ms, dense_ms;
    for (int r = 0; r < repetitions; ++r) {
      const double t0 = clock->now_ms();
      b200::forward_sparse(w, tokens, threshold);
      sparse_ms.push_back(clock->now_ms() - t0);
    }
    for (int r = 0; r < repetitions; ++r) {
      const double t0 = clock->now_ms();
      b200::forward_dense(w, tokens);
      dense_ms.push_back(clock->now_ms() - t0);
    }
    if (detail::median(dense_ms) <= detail::median(sparse_ms))
      return SwitchTable{static_cast<std::size_t>(grid[gi])};
  }
  return SwitchTable{SwitchTable::kSparseAlways};
}

inline SwitchTable profile_tipping(const MoELayerWeights& w, float threshold,
                                   std::initializer_list<int> batch_grid, int repetitions = 5,
                                   Stopwatch* clock = nullptr, std::uint64_t token_seed = 0) {
  return profile_tipping(w, threshold, std::vector<int>(batch_grid), repetitions, clock, token_seed);
}

// engine.hpp:85-89, engine.cpp:414-420
inline ForwardReport step(const MoELayerWeights& w, const Matrix& x, float threshold,
                          const SwitchTable& table, int threads = 1) {
  if (table.use_dense(static_cast<std::size_t>(x.rows))) return b200::forward_dense(w, x, threads);
  return b200::forward_sparse(w, x, threshold, threads);
}

// router.hpp:34
inline RouteResult route(const Matrix& logits, int top_k, bool renormalize) {
  RouteResult r;
  r.batch = logits.rows;
  r.top_k = top_k;
  const std::size_t n = static_cast<std::size_t>(logits.rows > 0 ? logits.rows : 0) *
                        static_cast<std::size_t>(top_k > 0 ? top_k : 0);
  r.ids.assign(n, 0);
  r.weights.assign(n, 0.0f);
  detail::check(skb_route(logits.data.data(), logits.rows, logits.cols, top_k, renormalize ? 1 : 0,
                          r.ids.data(), r.weights.data()));
  return r;
}

// router.hpp:46-47
inline DispatchPlan align_dispatch(const RouteResult& r, int n_experts, int block) {
  DispatchPlan p;
  p.block_size = block;
  const std::size_t cap = r.ids.size() + static_cast<std::size_t>(n_experts) *
                                             static_cast<std::size_t>(block > 1 ? block - 1 : 0) + 1;
  p.sorted_token_slots.assign(cap, 0);
  p.expert_of_block.assign(cap, 0);
  std::int32_t n_padded = 0, n_blocks = 0;
  detail::check(skb_align_dispatch(r.ids.data(), r.batch, r.top_k, n_experts, block,
                                   p.sorted_token_slots.data(), p.expert_of_block.data(),
                                   &n_padded, &n_blocks));
  p.sorted_token_slots.resize(static_cast<std::size_t>(n_padded));
  p.expert_of_block.resize(static_cast<std::size_t>(n_blocks));
  p.n_padded = n_padded;
  return p;
}

// router.hpp:52-53 (pointer + length instead of std::span so that C++17 callers compile too)
inline Matrix combine(const float* slot_outputs, std::size_t n, const RouteResult& r, int d_model) {
  if (n != static_cast<std::size_t>(r.batch) * r.top_k * d_model)
    throw InternalError("combine: slot output count does not match batch * top_k * d_model");
  Matrix y(r.batch, d_model);
  detail::check(skb_combine(slot_outputs, r.weights.data(), r.batch, r.top_k, d_model,
                            y.data.data()));
  return y;
}

// activation.hpp:35-39
inline std::vector<std::uint8_t> mask_smallest_magnitudes(const float* h, std::size_t n, int count) {
  std::vector<std::uint8_t> mask(n);
  const std::int32_t c = count;
  detail::check(skb_mask_smallest(h, 1, static_cast<int>(n), &c, mask.data(), nullptr, nullptr));
  return mask;
}
inline std::vector<std::uint8_t> topk_mask(const float* h, std::size_t n, SparsityLevel s) {
  std::vector<std::uint8_t> mask(n);
  detail::check(skb_topk_mask(h, 1, static_cast<int>(n), s.s, mask.data()));
  return mask;
}

// activation.hpp:42-64: the threshold variant's stage functions (pointer + length where the
// reference takes std::span, so that the facade compiles as C++17)
inline std::vector<std::uint8_t> threshold_mask(const float* gate_out, std::size_t n, float threshold) {
  std::vector<std::uint8_t> mask(n);
  detail::check(skb_threshold_mask(gate_out, 1, static_cast<int>(n), threshold, mask.data()));
  return mask;
}
inline int default_capacity(int top_k, int d_ffn) { return skb_default_capacity(top_k, d_ffn); }
inline ActiveIndexRow compact_active(const std::uint8_t* masks, std::size_t n_masks,
                                     const std::int32_t* topk_ids, std::size_t n_slots, int d_ffn,
                                     int capacity) {
  ActiveIndexRow row;
  row.flat.assign(static_cast<std::size_t>(capacity > 0 ? capacity : 0), kPadIndex);
  row.active_per_slot.assign(n_slots, 0);
  detail::check(skb_compact_active(masks, n_masks, topk_ids, 1, static_cast<int>(n_slots), d_ffn,
                                   capacity, row.flat.data(), row.active_per_slot.data(),
                                   &row.total_active));
  return row;
}

// ---- neuron budgets (budget.hpp:29-44, budget.cpp) ----
// Weights: any contiguous float container (std::vector, std::array, std::span).
template <class Weights>
inline ExpertGroups group_experts(const Weights& topk_weights) {
  const int k = static_cast<int>(topk_weights.size());
  if (k < 1) throw ConfigError("group_experts: need at least one slot");
  std::vector<int> order(static_cast<std::size_t>(k));
  std::iota(order.begin(), order.end(), 0);
  const float* wt = topk_weights.data();
  std::stable_sort(order.begin(), order.end(), [wt](int a, int b) { return wt[a] > wt[b]; });
  const int third = k / 3;
  ExpertGroups g;
  g.g0.assign(order.begin(), order.begin() + third);
  g.g1.assign(order.begin() + third, order.begin() + 2 * third);
  g.g2.assign(order.begin() + 2 * third, order.end());
  return g;
}

inline std::vector<int> allocate_budget(int top_k, int d_ffn, double s_active,
                                        const ExpertGroups& groups, const BudgetRatios& ratios) {
  if (!(s_active >= 0.0 && s_active <= 1.0))
    throw ConfigError("allocate_budget: s_active must lie in [0, 1]");
  if (ratios.r0 < 0.0 || ratios.r1 < 0.0 || ratios.r2 < 0.0)
    throw ConfigError("allocate_budget: ratios must be non-negative");
  const std::vector<int>* members[3] = {&groups.g0, &groups.g1, &groups.g2};
  const double ratio[3] = {ratios.r0, ratios.r1, ratios.r2};
  double denom = 0.0;
  for (int x = 0; x < 3; ++x) denom += ratio[x] * static_cast<double>(members[x]->size());
  if (!(denom > 0.0)) throw ConfigError("allocate_budget: no ratio mass on non-empty groups");
  const double budget = s_active * top_k * d_ffn;
  std::vector<int> counts(static_cast<std::size_t>(top_k), 0);
  int assigned = 0;
  for (int x = 0; x < 3; ++x) {
    long n_e = static_cast<long>(std::floor(budget * ratio[x] / denom + 0.5));
    n_e = n_e < 0 ? 0 : (n_e > d_ffn ? d_ffn : n_e);
    for (int slot : *members[x]) {
      if (slot < 0 || slot >= top_k)
        throw IndexError("allocate_budget: slot " + std::to_string(slot) + " outside [0, " +
                         std::to_string(top_k) + ")");
      counts[static_cast<std::size_t>(slot)] = static_cast<int>(n_e);
      ++assigned;
    }
  }
  if (assigned != top_k) throw ConfigError("allocate_budget: groups must partition the slots");
  return counts;
}

inline std::vector<std::uint8_t> apply_budget(const float* h, std::size_t n, int keep_count) {
  if (keep_count < 0 || static_cast<std::size_t>(keep_count) > n)
    throw ConfigError("apply_budget: keep_count outside [0, N]");
  return b200::mask_smallest_magnitudes(h, n, static_cast<int>(n) - keep_count);
}

// The budget analysis mode of the reference CLI (tools/main.cpp:271-345) as one device forward:
// slot s of every token keeps the count allocate_budget gives rank s (slots are in descending
// router weight); mask_shared: the shared expert gets a plain top-k mask at `sparsity`.
inline ForwardReport forward_budget_sparse(const MoELayerWeights& w, const Matrix& x,
                                           SparsityLevel sparsity, const BudgetRatios& ratios,
                                           bool mask_shared = false, MaskSet* masks_out = nullptr) {
  const int K = w.config.top_k, N = w.config.d_ffn;
  std::vector<float> rank_weights(static_cast<std::size_t>(K > 0 ? K : 0));
  for (int sl = 0; sl < K; ++sl) rank_weights[static_cast<std::size_t>(sl)] = static_cast<float>(K - sl);
  const std::vector<int> counts =
      b200::allocate_budget(K, N, 1.0 - sparsity.s, b200::group_experts(rank_weights), ratios);
  std::vector<std::int32_t> n_off(counts.size());
  for (std::size_t i = 0; i < counts.size(); ++i) n_off[i] = N - counts[i];
  skb_forward_args a{};
  a.mode = SKB_MODE_TOPK;
  a.s_routed = sparsity.s;
  a.s_shared = (mask_shared && w.config.has_shared) ? sparsity.s : 0.0;
  a.slot_n_off = n_off.data();
  return detail::run(w, x, a, masks_out);
}

}  // namespace b200
}  // namespace sparsekit
