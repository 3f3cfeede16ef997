// kat_test.cpp — the reference's own known-answer tests, restated against the
// CUDA-backed drop-in API (namespace samo, include/samo_b200/samo.hpp).  Each block names the
// reference test it ports (proj/tests/*.cpp).  Built by tests/test_cpp_kat.py;
// prints one line per test and exits non-zero on the first failure group.
#include <bit>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "samo/samo.hpp"  // the reference header name -> the CUDA-backed mirror

using namespace samo;

static int g_fail = 0, g_pass = 0;

#define CHECK(cond)                                                              \
  do {                                                                           \
    if (!(cond)) {                                                               \
      std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);            \
      throw std::runtime_error("check failed");                                  \
    }                                                                            \
  } while (0)

template <typename E, typename F>
static bool throws(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static void run(const char* name, const std::function<void()>& body) {
  try {
    body();
    ++g_pass;
    std::printf("PASS %s\n", name);
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("FAIL %s (%s)\n", name, e.what());
  }
}

static std::shared_ptr<const PrunedIndexSet> make_ind(std::uint64_t dense_len,
                                                      std::vector<std::uint32_t> idx) {
  PrunedIndexSet s;
  s.layer_id = "w";
  s.dense_len = dense_len;
  s.indices = std::move(idx);
  return std::make_shared<const PrunedIndexSet>(std::move(s));
}

static LayerParams layer(std::string id, std::vector<float> values, bool prunable = true) {
  const std::size_t n = values.size();
  return {std::move(id), Tensor<float>({n}, std::move(values)), prunable};
}

int main() {
  // ---- half_test.cpp ------------------------------------------------------
  run("Half.SpecExamples (half_test.cpp:54-59)", [] {
    CHECK(static_cast<float>(Half(1.0f)) == 1.0f);
    CHECK(static_cast<float>(Half(2049.0f)) == 2048.0f);
    CHECK(static_cast<float>(Half(0.5f)) == 0.5f);
  });
  run("Half.ExhaustiveRoundTrip (half_test.cpp:61-68)", [] {
    std::vector<Half> all;
    for (std::uint32_t b = 0; b <= 0xFFFF; ++b) {
      const Half h = Half::from_bits(static_cast<std::uint16_t>(b));
      if (h.is_finite()) all.push_back(h);
    }
    const auto back = to_half(to_float(all));
    for (std::size_t i = 0; i < all.size(); ++i) CHECK(back[i].bits() == all[i].bits());
  });
  run("Half.OverflowAndUnderflowEdges (half_test.cpp:83-94)", [] {
    const std::vector<float> f = {65504.0f, 65519.996f, 65520.0f, 1.0e10f, -1.0e10f, 0x1.0p-24f,
                                  0x1.0p-25f, std::nextafterf(0x1.0p-25f, 1.0f), -0.0f};
    const std::vector<std::uint16_t> want = {0x7BFF, 0x7BFF, 0x7C00, 0x7C00, 0xFC00,
                                             0x0001, 0x0000, 0x0001, 0x8000};
    const auto got = to_half(f);
    for (std::size_t i = 0; i < f.size(); ++i) CHECK(got[i].bits() == want[i]);
  });
  run("Half.InfinityAndNanSurvive (half_test.cpp:70-81)", [] {
    CHECK(Half(static_cast<float>(Half::from_bits(0x7C00))).bits() == 0x7C00);
    CHECK(Half(static_cast<float>(Half::from_bits(0xFC00))).bits() == 0xFC00);
    CHECK(Half(std::numeric_limits<float>::quiet_NaN()).is_nan());
    CHECK(std::isnan(static_cast<float>(Half::from_bits(0x7E01))));
  });

  // ---- store_test.cpp -----------------------------------------------------
  run("Compress.GatherByDefinition (store_test.cpp:29-33)", [] {
    const Tensor<float> dense({4}, {1.0f, 2.0f, 3.0f, 4.0f});
    CHECK((compress(dense, *make_ind(4, {0, 3})) == std::vector<float>{1.0f, 4.0f}));
  });
  run("Compress.FullIndexSetIsIdentity (store_test.cpp:35-40)", [] {
    const Tensor<float> dense({2, 2}, {1.0f, 2.0f, 3.0f, 4.0f});
    CHECK((compress(dense, *make_ind(4, {0, 1, 2, 3})) == std::vector<float>{1, 2, 3, 4}));
  });
  run("Compress.MatchesGatherOracle (store_test.cpp:42-58)", [] {
    std::mt19937_64 eng(41);
    Tensor<float> dense({4, 4});
    for (auto& v : dense.flat()) v = static_cast<float>(eng() >> 40) * 0x1.0p-24f;
    std::vector<std::uint32_t> idx;
    for (std::uint32_t i = 0; i < 16; ++i)
      if (eng() % 2) idx.push_back(i);
    const auto got = compress(dense, *make_ind(16, idx));
    CHECK(got.size() == idx.size());
    for (std::size_t k = 0; k < idx.size(); ++k) CHECK(got[k] == dense.flat()[idx[k]]);
  });
  run("Compress.LengthMismatch (store_test.cpp:60-64)", [] {
    const Tensor<float> dense({3});
    CHECK(throws<DimensionError>([&] { compress(dense, *make_ind(4, {0})); }));
  });
  run("Expand.ScatterByDefinition (store_test.cpp:66-71)", [] {
    const std::vector<float> values = {1.0f, 4.0f};
    const Tensor<float> got = expand<float>(values, *make_ind(4, {0, 3}), {2, 2});
    CHECK((got == Tensor<float>({2, 2}, {1.0f, 0.0f, 0.0f, 4.0f})));
  });
  run("Expand.EmptyIndexSetGivesZeros (store_test.cpp:73-77)", [] {
    const Tensor<float> got = expand<float>(std::vector<float>{}, *make_ind(4, {}), {4});
    CHECK((got == Tensor<float>({4})));
  });
  run("Expand.RoundTripProperty (store_test.cpp:79-108, 1000 trials)", [] {
    std::mt19937_64 eng(43);
    for (int trial = 0; trial < 1000; ++trial) {
      std::vector<std::size_t> shape(1 + eng() % 3);
      for (auto& e : shape) e = 1 + eng() % 5;
      const std::size_t n = numel(shape);
      std::vector<std::uint32_t> idx;
      for (std::uint32_t i = 0; i < n; ++i)
        if (eng() % 3) idx.push_back(i);
      const auto ind = make_ind(n, idx);
      std::vector<float> xf(n);
      for (auto& v : xf) v = (static_cast<float>(eng() >> 40) * 0x1.0p-24f - 0.5f) * 8.0f;
      const Tensor<Half> x(shape, to_half(xf));
      const auto values = compress(x, *ind);
      const Tensor<Half> expanded = expand<Half>(values, *ind, shape);
      Tensor<Half> masked(shape);
      for (auto i : idx) masked.flat()[i] = x.flat()[i];
      CHECK(bit_equal(expanded, masked));
      const auto back = compress(expanded, *ind);
      CHECK(back.size() == values.size());
      for (std::size_t k = 0; k < back.size(); ++k) CHECK(back[k].bits() == values[k].bits());
    }
  });

  // ---- prune_test.cpp -----------------------------------------------------
  run("Linearize.PaperExample2x2 / RowMajorOracle / OutOfBounds (prune_test.cpp:24-47)", [] {
    const std::vector<std::vector<std::uint64_t>> c = {{0, 0}, {1, 1}};
    const std::vector<std::size_t> s22 = {2, 2};
    CHECK((linearize(c, s22) == std::vector<std::uint64_t>{0, 3}));
    const std::vector<std::vector<std::uint64_t>> c3 = {{1, 2, 3}};
    const std::vector<std::size_t> s234 = {2, 3, 4};
    CHECK((linearize(c3, s234) == std::vector<std::uint64_t>{23}));
    const std::vector<std::vector<std::uint64_t>> bad = {{2, 0}};
    CHECK(throws<IndexError>([&] { linearize(bad, s22); }));
  });
  run("MagnitudePrune.SortByMagnitudeOracle (prune_test.cpp:84-92)", [] {
    const std::vector<LayerParams> layers = {layer("w", {3.0f, -1.0f, 0.5f, -4.0f})};
    const auto sets = magnitude_prune(layers, 0.5);
    CHECK(sets.size() == 1u);
    CHECK((sets[0].indices == std::vector<std::uint32_t>{0, 3}));
    CHECK(sets[0].dense_len == 4u && sets[0].layer_id == "w");
  });
  run("MagnitudePrune.ZeroSparsity / Ties / BadSparsity / NonPrunable (prune_test.cpp:94-118)", [] {
    CHECK((magnitude_prune(std::vector<LayerParams>{layer("w", {0.1f, -0.2f, 0.0f})}, 0.0)[0].indices ==
           std::vector<std::uint32_t>{0, 1, 2}));
    CHECK((magnitude_prune(std::vector<LayerParams>{layer("w", {1.0f, 1.0f, 1.0f, 1.0f})}, 0.5)[0].indices ==
           std::vector<std::uint32_t>{0, 1}));
    const std::vector<LayerParams> one = {layer("w", {1.0f})};
    CHECK(throws<ParameterError>([&] { magnitude_prune(one, 1.0); }));
    CHECK(throws<ParameterError>([&] { magnitude_prune(one, -0.1); }));
    const std::vector<LayerParams> two = {layer("w", {5.0f, 1.0f, 2.0f, 3.0f}), layer("b", {0.0f, 0.0f}, false)};
    const auto sets = magnitude_prune(two, 0.75);
    CHECK(sets[0].indices.size() == 1u);
    CHECK((sets[1].indices == std::vector<std::uint32_t>{0, 1}));
  });
  run("MagnitudePrune.CountMatchesRoundingConvention (prune_test.cpp:127-147)", [] {
    std::mt19937_64 eng(23);
    for (int trial = 0; trial < 200; ++trial) {
      const std::uint64_t den = 20, num = eng() % den;
      const double p = static_cast<double>(num) / static_cast<double>(den);
      const std::size_t n = 1 + eng() % 50;
      std::vector<float> values(n);
      for (auto& v : values) v = (static_cast<float>(eng() >> 40) * 0x1.0p-24f - 0.5f) * 2.0f;
      const auto sets = magnitude_prune(std::vector<LayerParams>{layer("w", values)}, p);
      const std::uint64_t q = (den - num) * n;
      CHECK(sets[0].indices.size() == (2 * q + den) / (2 * den));
      for (std::size_t i = 1; i < sets[0].indices.size(); ++i) CHECK(sets[0].indices[i - 1] < sets[0].indices[i]);
      for (auto i : sets[0].indices) CHECK(i < n);
    }
  });
  run("MagnitudePrune.ScaleInvariance (prune_test.cpp:149-168)", [] {
    std::mt19937_64 eng(29);
    for (int trial = 0; trial < 50; ++trial) {
      const std::size_t n = 8 + eng() % 32;
      std::vector<float> values(n);
      for (auto& v : values) v = (static_cast<float>(eng() >> 40) * 0x1.0p-24f - 0.5f) * 2.0f;
      const double p = 0.05 * static_cast<double>(eng() % 20);
      const auto base = magnitude_prune(std::vector<LayerParams>{layer("w", values)}, p);
      for (float c : {0.5f, 2.0f, 8.0f}) {
        std::vector<float> scaled(values);
        for (auto& v : scaled) v *= c;
        CHECK(magnitude_prune(std::vector<LayerParams>{layer("w", scaled)}, p)[0].indices == base[0].indices);
      }
    }
  });
  run("MagnitudePrune.GlobalScope (prune_test.cpp:170-202)", [] {
    const std::vector<LayerParams> layers = {layer("big", {10.0f, 9.0f, 8.0f, 7.0f}),
                                             layer("small", {1.0f, 0.9f, 0.8f, 0.7f})};
    const auto g = magnitude_prune(layers, 0.5, PruneScope::global);
    CHECK((g[0].indices == std::vector<std::uint32_t>{0, 1, 2, 3}) && g[1].indices.empty());
    const auto pl = magnitude_prune(layers, 0.5, PruneScope::per_layer);
    CHECK(pl[0].indices.size() == 2u && pl[1].indices.size() == 2u);
    std::mt19937_64 eng(31);
    std::vector<LayerParams> ls;
    std::uint64_t total = 0;
    for (int l = 0; l < 3; ++l) {
      const std::size_t n = 5 + eng() % 20;
      total += n;
      std::vector<float> v(n);
      for (auto& x : v) x = (static_cast<float>(eng() >> 40) * 0x1.0p-24f - 0.5f) * 2.0f;
      ls.push_back(layer("l" + std::to_string(l), v));
    }
    const auto sets = magnitude_prune(ls, 0.45, PruneScope::global);
    std::uint64_t kept = 0;
    for (const auto& s : sets) kept += s.indices.size();
    CHECK(kept == (2 * 11 * total + 20) / 40);
  });

  // ---- train_test.cpp -----------------------------------------------------
  run("OptimizerStep.ScalarAdamOracle (train_test.cpp:156-180)", [] {
    std::vector<float> th = {0.5f}, m = {0.0f}, v = {0.0f};
    const std::vector<float> g = {1.0f};
    OptimizerConfig cfg;
    cfg.learning_rate = 0.1f;
    cfg.loss_scale = 1.0f;
    adam_update(th, m, v, g, cfg, 1.0f - 0.9f, 1.0f - 0.999f);
    CHECK(std::fabs(th[0] - 0.4f) <= 1e-6f);
  });
  run("Model.ScalarAdamOracle through the fused step (train_test.cpp:156-180)", [] {
    Model model({*make_ind(1, {0})});
    model.init_layer(0, Tensor<float>({1, 1}, {0.5f}));
    OptimizerConfig cfg;
    cfg.learning_rate = 0.1f;
    cfg.loss_scale = 1.0f;
    model.set_config(cfg);
    DeviceBuffer<std::uint16_t> grad(1);
    const std::uint16_t one = Half(1.0f).bits();
    grad.upload(&one, 1);
    model.set_grads({grad.get()});
    model.step();
    const auto rec = model.record();
    CHECK(rec.t == 1 && rec.skipped_steps == 0);
    CHECK(std::fabs(model.theta32(0)[0] - 0.4f) <= 1e-6f);
    model.check_state_invariants();
  });
  run("OptimizerStep.NonFiniteGradientSkipsAndCounts (train_test.cpp:182-199)", [] {
    Model model({*make_ind(1, {0})});
    model.init_layer(0, Tensor<float>({1, 1}, {0.5f}));
    OptimizerConfig cfg;
    cfg.learning_rate = 0.1f;
    cfg.loss_scale = 65536.0f;
    model.set_config(cfg);
    DeviceBuffer<std::uint16_t> grad(1);
    const std::uint16_t inf = 0x7C00;
    grad.upload(&inf, 1);
    model.set_grads({grad.get()});
    model.step();
    const auto rec = model.record();
    CHECK(rec.skipped_steps == 1 && rec.last_skipped && rec.t == 0);
    CHECK(model.theta32(0)[0] == 0.5f);
    CHECK(model.adam_m(0)[0] == 0.0f);
  });
  run("OptimizerStep.StateErrors (train_test.cpp: optimizer_step requires backward)", [] {
    Model model({*make_ind(4, {0, 3})});
    CHECK(throws<StateError>([&] { model.step(); }));
    OptimizerConfig bad;
    bad.loss_scale = 1000.0f;
    CHECK(throws<ParameterError>([&] { model.set_config(bad); }));
  });

  run("Matmul.TransposeTimes (train.hpp:304, tensor.hpp:88-105) on the tensor cores", [] {
    // small integers: every product and partial sum is exact in fp32 and fp16
    const std::size_t batch = 3, in = 8, out = 16;
    std::vector<Half> xv, dv;
    for (std::size_t i = 0; i < batch * in; ++i) xv.push_back(Half(static_cast<float>(static_cast<int>(i % 7) - 3)));
    for (std::size_t i = 0; i < batch * out; ++i) dv.push_back(Half(static_cast<float>(static_cast<int>(i % 5) - 2)));
    const Tensor<Half> x({batch, in}, xv), dy({batch, out}, dv);
    const auto w = dw_matmul(x, dy);
    CHECK(w.shape() == std::vector<std::size_t>({in, out}));
    bool ok = true;
    for (std::size_t i = 0; i < in; ++i)
      for (std::size_t j = 0; j < out; ++j) {
        float acc = 0.0f;
        for (std::size_t b = 0; b < batch; ++b) acc += float(xv[b * in + i]) * float(dv[b * out + j]);
        ok = ok && float(w[i * out + j]) == acc;
      }
    CHECK(ok);
    CHECK(throws<DimensionError>([&] { dw_matmul(x, Tensor<Half>({2, out})); }));
  });
  run("Sink.FusedDwEqualsDenseSink (train.hpp:596-611)", [] {
    const std::size_t batch = 5, in = 16, out = 24;
    std::vector<std::uint32_t> keep;
    for (std::uint32_t k = 0; k < in * out; k += 7) keep.push_back(k);
    std::vector<Half> xv, dv;
    for (std::size_t i = 0; i < batch * in; ++i) xv.push_back(Half(0.25f * static_cast<float>(static_cast<int>(i % 9) - 4)));
    for (std::size_t i = 0; i < batch * out; ++i) dv.push_back(Half(8.0f * static_cast<float>(static_cast<int>(i % 5) - 2)));
    const Tensor<Half> x({batch, in}, xv), dy({batch, out}, dv);
    const auto w = dw_matmul(x, dy);
    auto make = [&] {
      Model m({*make_ind(in * out, keep)});
      m.init_layer(0, Tensor<float>({in, out}, std::vector<float>(in * out, 0.1f)));
      return m;
    };
    Model fused = make(), dense = make();
    DeviceBuffer<std::uint16_t> dx(reinterpret_cast<const std::uint16_t*>(xv.data()), xv.size());
    DeviceBuffer<std::uint16_t> dd(reinterpret_cast<const std::uint16_t*>(dv.data()), dv.size());
    DeviceBuffer<std::uint16_t> dw(reinterpret_cast<const std::uint16_t*>(w.flat().data()), w.size());
    fused.sink_dw(0, dx.get(), dd.get(), batch, in, out);
    fused.update();
    dense.set_grads({dw.get()});
    dense.step();
    CHECK(fused.theta32(0) == dense.theta32(0));
    CHECK(fused.record().t == 1);
    CHECK(throws<DimensionError>([&] { fused.sink_dw(0, dx.get(), dd.get(), batch, in, out - 8); }));
  });

  // ---- train_test.cpp OptimizerStep KATs through SamoTrainer ---------------
  // The reference drives them with a one-layer MLP forward/backward; here the
  // dense gradient that backward would hand to the sink is sunk directly.
  auto one_layer_state = [](Tensor<float> w) {
    const std::vector<LayerParams> params = {{"w", w, true}};
    auto sets = magnitude_prune(params, 0.0);
    ModelState st;
    st.layers.push_back(make_layer_state(w, std::make_shared<const PrunedIndexSet>(std::move(sets[0]))));
    return st;
  };
  auto plain_adam = [](float loss_scale) {
    OptimizerConfig cfg;
    cfg.learning_rate = 0.1f;
    cfg.loss_scale = loss_scale;
    return cfg;
  };
  run("OptimizerStep.ZeroGradientLeavesStateUntouched (train_test.cpp:139-154)", [&] {
    SamoTrainer tr(plain_adam(1.0f), one_layer_state(Tensor<float>({2, 2}, {1.0f, 0.0f, 0.0f, 1.0f})));
    const auto before = tr.state().layers[0].comp.theta32;
    tr.sink(0, Tensor<Half>({2, 2}));  // identity weights, y == x: dL/dW == 0
    CHECK(tr.optimizer_step());
    CHECK(tr.state().layers[0].comp.theta32 == before);
    for (float m : tr.state().layers[0].comp.adam_m) CHECK(m == 0.0f);
  });
  run("OptimizerStep.ScalarAdamOracle (train_test.cpp:156-180)", [&] {
    SamoTrainer tr(plain_adam(1.0f), one_layer_state(Tensor<float>({1, 1}, {0.5f})));
    tr.sink(0, Tensor<Half>({1, 1}, {Half(1.0f)}));  // 2 * (0.5 - 0) * 1
    CHECK(static_cast<float>(tr.state().layers[0].comp.grad16[0]) == 1.0f);
    CHECK(tr.optimizer_step());
    const double g = 1.0, lr = 0.1, b1 = 0.9, b2 = 0.999, eps = 1e-8;
    const double m_hat = (1.0 - b1) * g / (1.0 - b1), v_hat = (1.0 - b2) * g * g / (1.0 - b2);
    const double want = 0.5 - lr * m_hat / (std::sqrt(v_hat) + eps);
    const float got = tr.state().layers[0].comp.theta32[0];
    CHECK(std::fabs(got - want) <= 1e-6);
    CHECK(std::fabs(got - 0.4) <= 1e-6);
    CHECK(tr.state().layers[0].comp.grad16[0].bits() == 0);  // reset after the step
    check_state_invariants(tr.state());
  });
  run("OptimizerStep.NonFiniteGradientSkipsAndCounts (train_test.cpp:182-199)", [&] {
    SamoTrainer tr(plain_adam(65536.0f), one_layer_state(Tensor<float>({1, 1}, {0.5f})));
    tr.sink(0, Tensor<Half>({1, 1}, {Half(2.0f * 40000.5f * 65536.0f)}));  // overflows binary16
    CHECK(!tr.state().layers[0].comp.grad16[0].is_finite());
    CHECK(!tr.optimizer_step());
    CHECK(tr.skipped_steps() == 1u);
    CHECK(tr.state().layers[0].comp.theta32[0] == 0.5f);
    CHECK(tr.state().layers[0].comp.grad16[0].bits() == 0);
    for (float m : tr.state().layers[0].comp.adam_m) CHECK(m == 0.0f);
  });
  run("OptimizerStep.RequiresBackward (train.hpp:618)", [&] {
    SamoTrainer tr(plain_adam(1.0f), one_layer_state(Tensor<float>({1, 1}, {0.5f})));
    CHECK(throws<StateError>([&] { tr.optimizer_step(); }));
    CHECK(throws<IndexError>([&] { tr.sink(3, Tensor<Half>({1, 1})); }));
    CHECK(throws<DimensionError>([&] { tr.sink(0, Tensor<Half>({2, 1})); }));
  });
  run("SamoTrainer.MultiLayerStepsMatchModel (train.hpp:617-656)", [&] {
    // three layers, p = 0.5, two steps: the trainer's state equals a Model
    // stepped on the same gradients, and the invariants hold.
    std::vector<LayerParams> params;
    for (int l = 0; l < 3; ++l) {
      std::vector<float> v(64 + 8 * l);
      for (std::size_t i = 0; i < v.size(); ++i) v[i] = 0.01f * static_cast<float>((i * 37 + l * 11) % 29) - 0.14f;
      params.push_back(layer("l" + std::to_string(l), v));
    }
    auto sets = magnitude_prune(params, 0.5);
    ModelState st;
    for (int l = 0; l < 3; ++l)
      st.layers.push_back(make_layer_state(params[l].values, std::make_shared<const PrunedIndexSet>(sets[l])));
    check_state_invariants(st);
    OptimizerConfig cfg;
    SamoTrainer tr(cfg, st);
    Model m(sets);
    for (int l = 0; l < 3; ++l) m.init_layer(l, params[l].values);
    m.set_config(cfg);
    for (int step = 0; step < 2; ++step) {
      std::vector<DeviceBuffer<std::uint16_t>> bufs;
      std::vector<const std::uint16_t*> ptrs;
      for (int l = 2; l >= 0; --l) {  // last layer first, as mlp_backward
        std::vector<Half> g(params[l].values.size());
        for (std::size_t i = 0; i < g.size(); ++i) g[i] = Half(static_cast<float>((i * 13 + step * 7 + l) % 17) - 8.0f);
        tr.sink(l, Tensor<Half>({g.size()}, g));
        bufs.emplace_back(reinterpret_cast<const std::uint16_t*>(g.data()), g.size());
      }
      for (int l = 0; l < 3; ++l) ptrs.push_back(bufs[2 - l].get());
      m.set_grads(ptrs);
      m.step();
      CHECK(tr.optimizer_step());
    }
    for (int l = 0; l < 3; ++l) {
      CHECK(tr.state().layers[l].comp.theta32 == m.theta32(l));
      CHECK(tr.state().layers[l].comp.adam_v == m.adam_v(l));
      CHECK(bit_equal(tr.state().layers[l].theta16, Tensor<Half>({params[l].values.size()}, m.theta16(l))));
    }
    check_state_invariants(tr.state());
    CHECK(measured_bytes(tr.state(), Accounting::steady_state) ==
          measured_bytes(tr.state(), Accounting::peak) - 2 * tr.state().total_unpruned());
  });

  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
