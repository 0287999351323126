// ref_shim.cpp -- extern "C" doorway into the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  This file contains no reference code: it includes
// the reference's public headers from /root/reference/proj/include at build
// time and is linked against the reference's own .cpp files where they lie
// (see oracle/Makefile).  The result, oracle/_ref/libsparsekit_ref.so, is the
// real reference CPU layer: it pins oracle/moe_oracle.c, generates
// tests/golden/, and is the CPU arm bench.py times (cpu_baseline.kind
// "reference").  The product never links or loads it.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "moe_oracle.h"  // ork_config / ork_report PODs shared with the C restatement
#include "sparsekit/activation.hpp"
#include "sparsekit/budget.hpp"
#include "sparsekit/calibrate.hpp"
#include "sparsekit/engine.hpp"
#include "sparsekit/model.hpp"
#include "sparsekit/profiler.hpp"
#include "sparsekit/router.hpp"
#include "support.hpp"  // testsupport::scalar_forward (proj/tests/support.hpp)

namespace sk = sparsekit;

namespace {

thread_local std::string g_error;

template <typename Fn>
int guarded(const Fn& fn) {
  try {
    fn();
    return 0;
  } catch (const sk::ShapeError& e) {
    g_error = e.what();
    return 1;
  } catch (const sk::ConfigError& e) {
    g_error = e.what();
    return 2;
  } catch (const sk::IndexError& e) {
    g_error = e.what();
    return 3;
  } catch (const sk::InternalError& e) {
    g_error = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 9;
  }
}

sk::MoEConfig to_cfg(const ork_config& c) {
  sk::MoEConfig cfg;
  cfg.n_experts = c.n_experts;
  cfg.top_k = c.top_k;
  cfg.d_model = c.d_model;
  cfg.d_ffn = c.d_ffn;
  cfg.has_shared = c.has_shared != 0;
  cfg.d_shared = c.d_shared;
  cfg.renormalize = c.renormalize != 0;
  cfg.align_block = c.align_block;
  return cfg;
}

sk::Matrix to_matrix(const float* src, int rows, int cols) {
  sk::Matrix m(rows, cols);
  std::memcpy(m.data.data(), src, sizeof(float) * m.data.size());
  return m;
}

void fill_report(const sk::ForwardReport& r, float* y, ork_report* rep) {
  if (y) std::memcpy(y, r.outputs.data.data(), sizeof(float) * r.outputs.data.size());
  if (!rep) return;
  rep->gate_macs = r.macs.gate_macs;
  rep->up_macs = r.macs.up_macs;
  rep->down_macs = r.macs.down_macs;
  rep->other_macs = r.macs.other_macs;
  rep->active_neurons_total = r.active_neurons_total;
  rep->achieved_routed_sparsity = r.achieved_routed_sparsity;
  rep->tiles_total = r.tiles_total;
  rep->tiles_skipped = r.tiles_skipped;
  rep->path_used = r.path_used == sk::ExecPath::kDense ? 0 : 1;
}

void round_bf16_inplace(std::vector<float>& v) {
  for (float& f : v) {
    std::uint32_t bits;
    std::memcpy(&bits, &f, 4);
    if ((bits & 0x7f800000u) != 0x7f800000u) bits += 0x7fffu + ((bits >> 16) & 1u);
    bits &= 0xffff0000u;
    std::memcpy(&f, &bits, 4);
  }
}

sk::MaskSet to_masks(const sk::MoEConfig& cfg, int batch, const std::uint8_t* routed,
                     const std::uint8_t* shared) {
  sk::MaskSet m;
  const std::size_t nr = static_cast<std::size_t>(batch) * cfg.top_k * cfg.d_ffn;
  m.routed.assign(routed, routed + nr);
  if (shared != nullptr) {
    const std::size_t ns = static_cast<std::size_t>(batch) * cfg.d_shared;
    m.shared.assign(shared, shared + ns);
  }
  return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

// ---- weights -------------------------------------------------------------

void* ref_layer_synthetic(const ork_config* c, std::uint64_t seed, float scale) {
  sk::MoELayerWeights* w = nullptr;
  const int rc = guarded([&] { w = new sk::MoELayerWeights(sk::generate_synthetic(to_cfg(*c), seed, scale)); });
  return rc == 0 ? w : nullptr;
}

// Contiguous arrays: router [E][D]; gate/up/down_t [E][N][D]; shared_* [S][D].
void* ref_layer_from_arrays(const ork_config* c, const float* router, const float* gate,
                            const float* up, const float* down_t, const float* sg, const float* su,
                            const float* sd) {
  auto* w = new sk::MoELayerWeights;
  w->config = to_cfg(*c);
  const int E = c->n_experts, D = c->d_model, N = c->d_ffn, S = c->d_shared;
  w->router = to_matrix(router, E, D);
  const std::size_t nd = static_cast<std::size_t>(N) * D;
  for (int e = 0; e < E; ++e) {
    w->gate.push_back(to_matrix(gate + e * nd, N, D));
    w->up.push_back(to_matrix(up + e * nd, N, D));
    w->down_t.push_back(to_matrix(down_t + e * nd, N, D));
  }
  if (c->has_shared) {
    w->shared_gate = to_matrix(sg, S, D);
    w->shared_up = to_matrix(su, S, D);
    w->shared_down_t = to_matrix(sd, S, D);
  }
  return w;
}

void ref_layer_free(void* h) { delete static_cast<sk::MoELayerWeights*>(h); }

// Operand preparation (not a reference function): snap every weight to the
// nearest bf16 value so the CPU layer sees the operands the device image holds.
void ref_layer_round_bf16(void* h) {
  auto* w = static_cast<sk::MoELayerWeights*>(h);
  round_bf16_inplace(w->router.data);
  for (auto& m : w->gate) round_bf16_inplace(m.data);
  for (auto& m : w->up) round_bf16_inplace(m.data);
  for (auto& m : w->down_t) round_bf16_inplace(m.data);
  round_bf16_inplace(w->shared_gate.data);
  round_bf16_inplace(w->shared_up.data);
  round_bf16_inplace(w->shared_down_t.data);
}

// Borrowed pointers into the reference's own storage (valid until ref_layer_free).
const float* ref_layer_router(void* h) { return static_cast<sk::MoELayerWeights*>(h)->router.data.data(); }
const float* ref_layer_gate(void* h, int e) { return static_cast<sk::MoELayerWeights*>(h)->gate[e].data.data(); }
const float* ref_layer_up(void* h, int e) { return static_cast<sk::MoELayerWeights*>(h)->up[e].data.data(); }
const float* ref_layer_down_t(void* h, int e) { return static_cast<sk::MoELayerWeights*>(h)->down_t[e].data.data(); }
const float* ref_layer_shared(void* h, int which) {
  auto* w = static_cast<sk::MoELayerWeights*>(h);
  const sk::Matrix& m = which == 0 ? w->shared_gate : which == 1 ? w->shared_up : w->shared_down_t;
  return m.data.empty() ? nullptr : m.data.data();
}

int ref_generate_tokens(int batch, int d_model, std::uint64_t seed, float* out) {
  return guarded([&] {
    const sk::Matrix x = sk::generate_tokens(batch, d_model, seed);
    std::memcpy(out, x.data.data(), sizeof(float) * x.data.size());
  });
}

int ref_save_weights(void* h, const char* path) {
  return guarded([&] { sk::save_weights(*static_cast<sk::MoELayerWeights*>(h), path); });
}

// ---- layer ---------------------------------------------------------------

int ref_forward_dense(void* h, const float* x, int batch, int threads, float* y, ork_report* rep) {
  auto* w = static_cast<sk::MoELayerWeights*>(h);
  return guarded([&] {
    fill_report(sk::forward_dense(*w, to_matrix(x, batch, w->config.d_model), threads), y, rep);
  });
}

int ref_forward_masked_dense(void* h, const float* x, int batch, const std::uint8_t* routed,
                             const std::uint8_t* shared, int threads, float* y, ork_report* rep) {
  auto* w = static_cast<sk::MoELayerWeights*>(h);
  return guarded([&] {
    const sk::MaskSet masks = to_masks(w->config, batch, routed, shared);
    fill_report(sk::forward_masked_dense(*w, to_matrix(x, batch, w->config.d_model), masks, threads), y, rep);
  });
}

int ref_forward_sparse(void* h, const float* x, int batch, float threshold, int threads, float* y,
                       ork_report* rep) {
  auto* w = static_cast<sk::MoELayerWeights*>(h);
  return guarded([&] {
    fill_report(sk::forward_sparse(*w, to_matrix(x, batch, w->config.d_model), threshold, threads), y, rep);
  });
}

int ref_build_topk_masks(void* h, const float* x, int batch, double s, int mode,
                         std::uint8_t* routed, std::uint8_t* shared) {
  auto* w = static_cast<sk::MoELayerWeights*>(h);
  return guarded([&] {
    const sk::MaskSet m = sk::build_topk_masks(
        *w, to_matrix(x, batch, w->config.d_model), sk::SparsityLevel(s),
        mode == 1 ? sk::SweepMode::kRoutedAndShared : sk::SweepMode::kRoutedOnly);
    std::memcpy(routed, m.routed.data(), m.routed.size());
    if (shared != nullptr && !m.shared.empty()) std::memcpy(shared, m.shared.data(), m.shared.size());
  });
}

int ref_scalar_forward(void* h, const float* x, int batch, const std::uint8_t* routed,
                       const std::uint8_t* shared, float* y) {
  auto* w = static_cast<sk::MoELayerWeights*>(h);
  return guarded([&] {
    const sk::Matrix xm = to_matrix(x, batch, w->config.d_model);
    sk::Matrix out;
    if (routed != nullptr) {
      const sk::MaskSet masks = to_masks(w->config, batch, routed, shared);
      out = testsupport::scalar_forward(*w, xm, &masks);
    } else {
      out = testsupport::scalar_forward(*w, xm, nullptr);
    }
    std::memcpy(y, out.data.data(), sizeof(float) * out.data.size());
  });
}

// tau for a routed-sparsity target via the reference's own calibration
// (collect_magnitudes -> build_table -> lookup), as the survey probe did.
int ref_calibrate_tau(void* h, double target_total, int calib_batch, std::uint64_t token_seed,
                      std::uint64_t sample_cap, std::uint64_t seed, double* tau_out) {
  auto* w = static_cast<sk::MoELayerWeights*>(h);
  return guarded([&] {
    const sk::Matrix toks = sk::generate_tokens(calib_batch, w->config.d_model, token_seed);
    const std::vector<float> mags = sk::collect_magnitudes(*w, toks, sample_cap, seed);
    const double targets[1] = {target_total};
    const sk::CalibrationTable table =
        sk::build_table(mags, targets, w->config.top_k, w->config.d_ffn, 0);
    *tau_out = sk::lookup(table, target_total);
  });
}

// sweep_cutoff (profiler.cpp:152-219) with the default quality metric; points as rows of
// {target, achieved_total, achieved_routed, quality, rel_error}; optionally emit_report to a file.
int ref_sweep_cutoff(void* h, const float* x, int batch, const double* targets, int n_targets,
                     double retention, int mode, double* points, double* cutoff, const char* csv) {
  auto* w = static_cast<sk::MoELayerWeights*>(h);
  return guarded([&] {
    const sk::SweepResult r = sk::sweep_cutoff(
        *w, to_matrix(x, batch, w->config.d_model),
        std::span<const double>(targets, static_cast<std::size_t>(n_targets)), retention,
        mode == 1 ? sk::SweepMode::kRoutedAndShared : sk::SweepMode::kRoutedOnly);
    for (std::size_t i = 0; i < r.points.size(); ++i) {
      const sk::SweepPoint& p = r.points[i];
      double* o = points + 5 * i;
      o[0] = p.target, o[1] = p.achieved_total, o[2] = p.achieved_routed, o[3] = p.quality, o[4] = p.rel_error;
    }
    *cutoff = r.cutoff;
    if (csv != nullptr) sk::emit_report(r, csv);
  });
}

// emit_report (profiler.cpp:221-243) of caller-given points: pins the file format
int ref_emit_report(const double* points, int n, const char* label, double cutoff, const char* csv) {
  return guarded([&] {
    sk::SweepResult r;
    for (int i = 0; i < n; ++i) {
      sk::SweepPoint p;
      const double* o = points + 5 * i;
      p.target = o[0], p.achieved_total = o[1], p.achieved_routed = o[2], p.quality = o[3], p.rel_error = o[4];
      p.path = label;
      r.points.push_back(p);
    }
    r.cutoff = cutoff;
    sk::emit_report(r, csv);
  });
}

// ---- stage functions -----------------------------------------------------

int ref_route(const float* logits, int batch, int n_experts, int top_k, int renorm,
              std::int32_t* ids, float* weights) {
  return guarded([&] {
    const sk::RouteResult r = sk::route(to_matrix(logits, batch, n_experts), top_k, renorm != 0);
    std::memcpy(ids, r.ids.data(), sizeof(std::int32_t) * r.ids.size());
    std::memcpy(weights, r.weights.data(), sizeof(float) * r.weights.size());
  });
}

int ref_align_dispatch(const std::int32_t* ids, int batch, int top_k, int n_experts, int block,
                       std::int32_t* sorted_out, std::int32_t* expert_of_block,
                       std::int32_t* n_padded, std::int32_t* n_blocks) {
  return guarded([&] {
    sk::RouteResult r;
    r.batch = batch;
    r.top_k = top_k;
    r.ids.assign(ids, ids + static_cast<std::size_t>(batch) * top_k);
    r.weights.assign(r.ids.size(), 1.0f);
    const sk::DispatchPlan p = sk::align_dispatch(r, n_experts, block);
    std::memcpy(sorted_out, p.sorted_token_slots.data(), sizeof(std::int32_t) * p.sorted_token_slots.size());
    std::memcpy(expert_of_block, p.expert_of_block.data(), sizeof(std::int32_t) * p.expert_of_block.size());
    *n_padded = p.n_padded;
    *n_blocks = static_cast<std::int32_t>(p.expert_of_block.size());
  });
}

int ref_combine(const float* slot_outputs, const std::int32_t* ids, const float* weights, int batch,
                int top_k, int d_model, float* y) {
  return guarded([&] {
    sk::RouteResult r;
    r.batch = batch;
    r.top_k = top_k;
    const std::size_t n = static_cast<std::size_t>(batch) * top_k;
    r.ids.assign(ids, ids + n);
    r.weights.assign(weights, weights + n);
    const sk::Matrix out = sk::combine({slot_outputs, n * d_model}, r, d_model);
    std::memcpy(y, out.data.data(), sizeof(float) * out.data.size());
  });
}

float ref_silu(float x) { return sk::silu(x); }

int ref_swiglu_rows(const float* g, const float* u, int n, float* h) {
  return guarded([&] {
    const auto out = sk::swiglu_rows({g, static_cast<std::size_t>(n)}, {u, static_cast<std::size_t>(n)});
    std::memcpy(h, out.data(), sizeof(float) * out.size());
  });
}

int ref_mask_smallest(const float* h, int n, int count, std::uint8_t* mask) {
  return guarded([&] {
    const auto m = sk::mask_smallest_magnitudes({h, static_cast<std::size_t>(n)}, count);
    std::memcpy(mask, m.data(), m.size());
  });
}

int ref_topk_mask(const float* h, int n, double s, std::uint8_t* mask) {
  return guarded([&] {
    const auto m = sk::topk_mask({h, static_cast<std::size_t>(n)}, sk::SparsityLevel(s));
    std::memcpy(mask, m.data(), m.size());
  });
}

int ref_apply_budget(const float* h, int n, int keep, std::uint8_t* mask) {
  return guarded([&] {
    const auto m = sk::apply_budget({h, static_cast<std::size_t>(n)}, keep);
    std::memcpy(mask, m.data(), m.size());
  });
}

int ref_threshold_mask(const float* g, int n, float threshold, std::uint8_t* mask) {
  return guarded([&] {
    const auto m = sk::threshold_mask({g, static_cast<std::size_t>(n)}, threshold);
    std::memcpy(mask, m.data(), m.size());
  });
}

int ref_default_capacity(int top_k, int d_ffn) { return sk::default_capacity(top_k, d_ffn); }

int ref_compact_active(const std::uint8_t* masks, const std::int32_t* topk_ids, int n_slots,
                       int d_ffn, int capacity, std::int32_t* flat, std::int32_t* per_slot,
                       std::int32_t* total) {
  return guarded([&] {
    const sk::ActiveIndexRow row = sk::compact_active(
        {masks, static_cast<std::size_t>(n_slots) * d_ffn}, {topk_ids, static_cast<std::size_t>(n_slots)},
        d_ffn, capacity);
    std::memcpy(flat, row.flat.data(), sizeof(std::int32_t) * row.flat.size());
    std::memcpy(per_slot, row.active_per_slot.data(), sizeof(std::int32_t) * row.active_per_slot.size());
    *total = row.total_active;
  });
}

int ref_matvec(const float* w, int rows, int cols, const float* x, float* y) {
  return guarded([&] {
    std::uint64_t macs = 0;
    const auto out = sk::matvec(to_matrix(w, rows, cols), {x, static_cast<std::size_t>(cols)}, macs);
    std::memcpy(y, out.data(), sizeof(float) * out.size());
  });
}

int ref_gathered_matvec_t(const float* w_t, int rows, int cols, const std::int32_t* idx,
                          const float* h, int m, float* y) {
  return guarded([&] {
    std::uint64_t macs = 0;
    const auto out = sk::gathered_matvec_t(to_matrix(w_t, rows, cols), {idx, static_cast<std::size_t>(m)},
                                           {h, static_cast<std::size_t>(m)}, macs);
    std::memcpy(y, out.data(), sizeof(float) * out.size());
  });
}

}  // extern "C"
