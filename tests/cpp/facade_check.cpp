// Exercises the C++ facade (include/sparsekit_b200.hpp) the way reference client code would.
// Built against the stand-in types here and, when /root/reference exists, syntax-checked
// against the reference's own headers (tests/test_cabi_cpu.py).  On a GPU it prints
// "facade ok <checksum>"; the Python test compares the checksum with the ctypes path.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "sparsekit_b200.hpp"

using namespace sparsekit;

static float lcg(std::uint64_t& s) {  // same generator as tests/test_gpu_parity.py::_lcg_fill
  s = s * 6364136223846793005ull + 1442695040888963407ull;
  return (static_cast<float>((s >> 40) & 0xFFFF) / 65536.0f - 0.5f) * 0.25f;
}
static void fill(Matrix& m, int r, int c, std::uint64_t& s) {
  m = Matrix(r, c);
  for (float& v : m.data) v = lcg(s);
}

int main() {
  MoELayerWeights w;
  w.config.n_experts = 8;
  w.config.top_k = 2;
  w.config.d_model = 128;
  w.config.d_ffn = 192;
  w.config.has_shared = true;
  w.config.d_shared = 64;
  std::uint64_t s = 12345;
  fill(w.router, 8, 128, s);
  w.gate.resize(8);
  w.up.resize(8);
  w.down_t.resize(8);
  for (int e = 0; e < 8; ++e) {
    fill(w.gate[e], 192, 128, s);
    fill(w.up[e], 192, 128, s);
    fill(w.down_t[e], 192, 128, s);
  }
  fill(w.shared_gate, 64, 128, s);
  fill(w.shared_up, 64, 128, s);
  fill(w.shared_down_t, 64, 128, s);
  Matrix x;
  fill(x, 5, 128, s);

  if (skb_device_count() < 1) {
    std::printf("facade built; no CUDA device\n");
    return 0;
  }
  const ForwardReport dense = b200::forward_dense(w, x, 4);
  const ForwardReport zero = b200::forward_topk_sparse(w, x, SparsityLevel(0.0), SparsityLevel(0.0));
  if (std::memcmp(dense.outputs.data.data(), zero.outputs.data.data(),
                  dense.outputs.data.size() * sizeof(float)) != 0) {
    std::printf("FAIL: s=0 differs from forward_dense\n");
    return 1;
  }
  const MaskSet masks = b200::build_topk_masks(w, x, SparsityLevel(0.5), SweepMode::kRoutedAndShared);
  const ForwardReport fused = b200::forward_topk_sparse(w, x, SparsityLevel(0.5), SparsityLevel(0.5));
  const ForwardReport masked = b200::forward_masked_dense(w, x, masks);
  double diff = 0.0;
  for (std::size_t i = 0; i < fused.outputs.data.size(); ++i)
    diff = std::fmax(diff, std::fabs(fused.outputs.data[i] - masked.outputs.data[i]));
  if (diff > 1e-6) {
    std::printf("FAIL: fused top-k vs masked dense on its own masks: %g\n", diff);
    return 1;
  }
  std::uint64_t kept = 0;
  for (auto b : masks.routed) kept += b;
  if (kept != 5u * 2u * 96u || fused.active_neurons_total != kept) {
    std::printf("FAIL: survivor count %llu\n", static_cast<unsigned long long>(kept));
    return 1;
  }
  // the threshold runtime path: tau = 0 keeps every neuron, a huge tau keeps none, tau < 0 throws
  const ForwardReport thr0 = b200::forward_sparse(w, x, 0.0f);
  const ForwardReport thr1 = b200::forward_sparse(w, x, 1e9f);
  diff = 0.0;
  for (std::size_t i = 0; i < thr0.outputs.data.size(); ++i)
    diff = std::fmax(diff, std::fabs(thr0.outputs.data[i] - dense.outputs.data[i]));
  if (diff > 1e-5 || thr0.active_neurons_total != 5u * 2u * 192u || thr0.tiles_skipped != 0 ||
      thr1.active_neurons_total != 0 || thr1.tiles_skipped != thr1.tiles_total ||
      thr0.path_used != ExecPath::kSparse) {
    std::printf("FAIL: forward_sparse limits: %g\n", diff);
    return 1;
  }
  bool neg = false;
  try {
    b200::forward_sparse(w, x, -0.5f);
  } catch (const ConfigError&) {
    neg = true;
  }
  if (!neg) {
    std::printf("FAIL: forward_sparse accepted a negative threshold\n");
    return 1;
  }
  // the dense/sparse switch (engine_test.cpp:355-408): scripted clock, then step()
  struct Scripted final : Stopwatch {
    std::vector<double> durations;
    std::size_t calls = 0;
    double t = 0.0;
    explicit Scripted(std::vector<double> d) : durations(std::move(d)) {}
    double now_ms() override {
      if (calls % 2 == 1) t += durations[calls / 2];
      ++calls;
      return t;
    }
  };
  {
    const std::vector<int> grid = {1, 2};
    Scripted never({1.0, 2.0, 1.0, 2.0}), second({1.0, 2.0, 2.0, 2.0}), med({1.0, 9.0, 1.0, 0.5, 0.6, 20.0});
    const std::vector<int> single = {4};
    if (b200::profile_tipping(w, 0.01f, grid, 1, &never, 0).tipping_batch != SwitchTable::kSparseAlways ||
        b200::profile_tipping(w, 0.01f, grid, 1, &second, 0).tipping_batch != 2 ||
        b200::profile_tipping(w, 0.01f, single, 3, &med, 0).tipping_batch != 4 || med.calls != 12) {
      std::printf("FAIL: profile_tipping with scripted timings\n");
      return 1;
    }
    bool empty_thrown = false;
    try {
      b200::profile_tipping(w, 0.01f, {}, 1, nullptr, 0);
    } catch (const ConfigError&) {
      empty_thrown = true;
    }
    if (!empty_thrown || b200::step(w, x, 0.01f, SwitchTable{6}).path_used != ExecPath::kSparse ||
        b200::step(w, x, 0.01f, SwitchTable{5}).path_used != ExecPath::kDense ||
        b200::step(w, x, 0.01f, SwitchTable{}).path_used != ExecPath::kSparse) {
      std::printf("FAIL: step() / empty grid\n");
      return 1;
    }
  }
  // neuron budgets (budget_test.cpp:47-54): 3:2:1 over K=6, N=8, half active; the budgeted forward
  {
    const std::vector<float> wts = {0.3f, 0.25f, 0.2f, 0.15f, 0.07f, 0.03f};
    const std::vector<int> counts =
        b200::allocate_budget(6, 8, 0.5, b200::group_experts(wts), BudgetRatios{3.0, 2.0, 1.0});
    const float hrow[3] = {1.0f, -3.0f, 2.0f};
    MaskSet bm;
    const ForwardReport budgeted =
        b200::forward_budget_sparse(w, x, SparsityLevel(0.5), BudgetRatios{}, true, &bm);
    // equal ratios == the plain top-k forward (other kernels at this batch: compare to tolerance)
    double bdiff = 0.0;
    for (std::size_t i = 0; i < fused.outputs.data.size(); ++i)
      bdiff = std::fmax(bdiff, std::fabs(budgeted.outputs.data[i] - fused.outputs.data[i]));
    std::uint64_t bkept = 0;
    for (auto b : bm.routed) bkept += b;
    if (counts != std::vector<int>{6, 6, 4, 4, 2, 2} ||
        b200::apply_budget(hrow, 3, 2) != std::vector<std::uint8_t>{0, 1, 1} || bdiff > 1e-5 ||
        bkept != kept || budgeted.active_neurons_total != kept) {
      std::printf("FAIL: neuron budgets\n");
      return 1;
    }
  }
  {
    // threshold stage functions (activation_test.cpp:117-153) and the quality sweep + report file
    const std::uint8_t m4[] = {1, 1, 1, 1};
    const std::int32_t id2[] = {1, 0};
    const ActiveIndexRow row = b200::compact_active(m4, 4, id2, 2, 2, 3);
    const float gate3[] = {2.0f, -2.0f, 0.01f};
    const double targets[] = {0.0, 0.5, 0.9};
    const SweepResult sw = b200::sweep_cutoff(w, x, targets, 3, 0.5, SweepMode::kRoutedAndShared);
    b200::emit_report(sw, "facade_report.csv");
    if (row.flat != std::vector<std::int32_t>{2, 3, 0} || row.total_active != 3 ||
        row.active_per_slot != std::vector<std::int32_t>{2, 1} || b200::default_capacity(3, 8) != 32 ||
        b200::threshold_mask(gate3, 3, 0.5f) != std::vector<std::uint8_t>{1, 0, 0} ||
        sw.points.size() != 3 || sw.points[0].rel_error != 0.0 || sw.points[0].quality != 1.0 ||
        !(sw.points[1].rel_error > 0.0) || !(sw.points[2].rel_error >= sw.points[1].rel_error) ||
        sw.points[2].path != "R+S" || sw.points[1].achieved_routed != 0.5) {
      std::printf("FAIL: threshold stage functions / sweep_cutoff\n");
      return 1;
    }
  }
  bool threw = false;
  try {
    Matrix bad(2, 64);
    b200::forward_dense(w, bad);
  } catch (const ShapeError&) {
    threw = true;
  }
  if (!threw) {
    std::printf("FAIL: ShapeError not raised\n");
    return 1;
  }
  threw = false;
  try {
    Matrix logits(1, 4);
    b200::route(logits, 9, true);
  } catch (const ConfigError&) {
    threw = true;
  }
  if (!threw) {
    std::printf("FAIL: ConfigError not raised\n");
    return 1;
  }
  double sum = 0.0;
  for (float v : fused.outputs.data) sum += v;
  std::printf("facade ok %.9e\n", sum);
  b200::clear_cache();
  return 0;
}
