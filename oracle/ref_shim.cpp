// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference headers
// (/root/reference/proj/include/samo/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libsamo_ref.so with the reference's own flags (-O3 -DNDEBUG
// -std=gnu++20, no -march).  Used to (i) generate the golden vectors that pin
// oracle/samo_oracle.c and the CUDA path, and (ii) time the reference's CPU
// implementation of the step ("reference" CPU baseline of bench.py).
//
// Nothing here re-implements the algorithm: every call goes into the
// reference's own functions.  Exceptions are mapped to the status codes of
// include/samo_cuda.h.
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <vector>

#include "samo/train.hpp"

#define EXPORT extern "C" __attribute__((visibility("default")))

namespace {

int status_of(const std::exception& e) {
  if (dynamic_cast<const samo::DimensionError*>(&e)) return 1;
  if (dynamic_cast<const samo::ParameterError*>(&e)) return 2;
  if (dynamic_cast<const samo::IndexError*>(&e)) return 3;
  if (dynamic_cast<const samo::StateError*>(&e)) return 4;
  if (dynamic_cast<const samo::ConfigError*>(&e)) return 5;
  return 99;
}

samo::PrunedIndexSet make_set(const uint32_t* idx, uint64_t n, uint64_t dense_len) {
  samo::PrunedIndexSet s;
  s.layer_id = "w";
  s.dense_len = dense_len;
  s.indices.assign(idx, idx + n);
  return s;
}

std::vector<samo::Half> halves(const uint16_t* bits, uint64_t n) {
  std::vector<samo::Half> d(n);
  for (uint64_t i = 0; i < n; ++i) d[i] = samo::Half::from_bits(bits[i]);
  return d;
}

}  // namespace

// half.hpp
EXPORT void ref_f2h(const float* in, uint16_t* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = samo::Half(in[i]).bits();
}
EXPORT void ref_h2f(const uint16_t* in, float* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<float>(samo::Half::from_bits(in[i]));
}

// store.hpp compress / expand over Half and float.
EXPORT int ref_compress_u16(const uint16_t* dense, uint64_t dense_len, const uint32_t* idx,
                            uint64_t n, uint64_t ind_dense_len, uint16_t* out) {
  try {
    std::vector<samo::Half> d(dense_len);
    for (uint64_t i = 0; i < dense_len; ++i) d[i] = samo::Half::from_bits(dense[i]);
    const samo::Tensor<samo::Half> t({static_cast<std::size_t>(dense_len)}, std::move(d));
    const auto got = samo::compress(t, make_set(idx, n, ind_dense_len));
    for (uint64_t k = 0; k < got.size(); ++k) out[k] = got[k].bits();
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

EXPORT int ref_compress_f32(const float* dense, uint64_t dense_len, const uint32_t* idx, uint64_t n,
                            uint64_t ind_dense_len, float* out) {
  try {
    const samo::Tensor<float> t({static_cast<std::size_t>(dense_len)},
                                std::vector<float>(dense, dense + dense_len));
    const auto got = samo::compress(t, make_set(idx, n, ind_dense_len));
    std::memcpy(out, got.data(), got.size() * 4);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

EXPORT int ref_expand_u16(const uint16_t* values, uint64_t n_values, const uint32_t* idx, uint64_t n,
                          uint64_t ind_dense_len, uint64_t shape_numel, uint16_t* dense) {
  try {
    std::vector<samo::Half> v(n_values);
    for (uint64_t k = 0; k < n_values; ++k) v[k] = samo::Half::from_bits(values[k]);
    const auto t = samo::expand<samo::Half>(v, make_set(idx, n, ind_dense_len),
                                            {static_cast<std::size_t>(shape_numel)});
    for (uint64_t i = 0; i < t.size(); ++i) dense[i] = t.flat()[i].bits();
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

EXPORT int ref_expand_f32(const float* values, uint64_t n_values, const uint32_t* idx, uint64_t n,
                          uint64_t ind_dense_len, uint64_t shape_numel, float* dense) {
  try {
    std::vector<float> v(values, values + n_values);
    const auto t = samo::expand<float>(v, make_set(idx, n, ind_dense_len),
                                       {static_cast<std::size_t>(shape_numel)});
    std::memcpy(dense, t.flat().data(), t.size() * 4);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// train.hpp adam_update
struct RefCfg {
  float lr, beta1, beta2, eps, loss_scale, wd;
};

static samo::OptimizerConfig to_cfg(const RefCfg* c) {
  samo::OptimizerConfig cfg;
  cfg.learning_rate = c->lr;
  cfg.beta1 = c->beta1;
  cfg.beta2 = c->beta2;
  cfg.epsilon = c->eps;
  cfg.loss_scale = c->loss_scale;
  cfg.weight_decay = c->wd;
  return cfg;
}

EXPORT void ref_adam_update(float* theta, float* m, float* v, const float* g, uint64_t n,
                            const RefCfg* c, float bias1, float bias2) {
  samo::adam_update({theta, n}, {m, n}, {v, n}, {g, n}, to_cfg(c), bias1, bias2);
}

EXPORT int ref_config_validate(const RefCfg* c) {
  try {
    to_cfg(c).validate();
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// prune.hpp
EXPORT uint64_t ref_unpruned_count(double p, uint64_t n) { return samo::detail::unpruned_count(p, n); }

EXPORT int ref_magnitude_prune(const float* const* vals, const uint64_t* lens, const uint8_t* prunable,
                               int nlayers, double p, int scope, uint32_t* const* idx_out,
                               uint64_t* counts_out) {
  try {
    std::vector<samo::LayerParams> layers;
    for (int l = 0; l < nlayers; ++l) {
      samo::LayerParams lp;
      lp.layer_id = "l" + std::to_string(l);
      lp.values = samo::Tensor<float>({static_cast<std::size_t>(lens[l])},
                                      std::vector<float>(vals[l], vals[l] + lens[l]));
      lp.prunable = prunable[l] != 0;
      layers.push_back(std::move(lp));
    }
    const auto sets = samo::magnitude_prune(
        layers, p, scope == 1 ? samo::PruneScope::global : samo::PruneScope::per_layer);
    for (int l = 0; l < nlayers; ++l) {
      counts_out[l] = sets[l].indices.size();
      std::memcpy(idx_out[l], sets[l].indices.data(), sets[l].indices.size() * 4);
    }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// init_params-compatible stream: n draws of uniform_symmetric(mt19937_64(seed), bound).
EXPORT void ref_uniform_symmetric(uint64_t seed, float bound, float* out, uint64_t n) {
  std::mt19937_64 eng(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = samo::uniform_symmetric(eng, bound);
}

// ---------------------------------------------------------------------------
// The unmodified SamoTrainer::optimizer_step at any scale ("driver-layer
// trick"): state.layers[0] is a 1x1 bias-free layer that the
// ModelSpec trains (forward/backward on a zero input give it a zero gradient);
// every other layer carries real compressed state whose grad16 is filled by
// samo::compress of the dense gradient — exactly the backward sink
// (train.hpp:603-606) — before optimizer_step runs over all layers.

struct RefSession {
  samo::ModelSpec spec;
  std::unique_ptr<samo::SamoTrainer> trainer;
  std::vector<std::shared_ptr<const samo::PrunedIndexSet>> sets;
  std::vector<uint64_t> dense_len;
};

EXPORT void* ref_session_create(int nlayers, const uint64_t* dense_len, const uint64_t* nnz,
                                const uint32_t* const* idx, const float* const* theta32,
                                const RefCfg* c) {
  auto* s = new RefSession();
  s->spec.layers = {{1, 1, false, samo::Activation::identity}};
  s->spec.loss = samo::LossKind::mse;
  samo::ModelState st;
  {
    auto dummy = std::make_shared<const samo::PrunedIndexSet>(
        samo::PrunedIndexSet{"dummy", 1, {0u}});
    samo::Tensor<float> w({1, 1}, {0.5f});
    st.layers.push_back(samo::make_layer_state(w, dummy));
  }
  for (int l = 0; l < nlayers; ++l) {
    auto set = std::make_shared<const samo::PrunedIndexSet>(
        samo::PrunedIndexSet{"l" + std::to_string(l), dense_len[l],
                             std::vector<uint32_t>(idx[l], idx[l] + nnz[l])});
    samo::LayerState ls;
    ls.layer_id = set->layer_id;
    ls.shape = {static_cast<std::size_t>(dense_len[l])};
    ls.comp.ind = set;
    ls.comp.theta32.assign(theta32[l], theta32[l] + nnz[l]);
    ls.comp.grad16.assign(nnz[l], samo::Half{});
    ls.comp.grad32.assign(nnz[l], 0.0f);
    ls.comp.adam_m.assign(nnz[l], 0.0f);
    ls.comp.adam_v.assign(nnz[l], 0.0f);
    std::vector<samo::Half> c16(nnz[l]);
    for (uint64_t k = 0; k < nnz[l]; ++k) c16[k] = samo::Half(ls.comp.theta32[k]);
    ls.theta16 = samo::expand<samo::Half>(c16, *set, ls.shape);
    st.layers.push_back(std::move(ls));
    s->sets.push_back(set);
    s->dense_len.push_back(dense_len[l]);
  }
  s->trainer = std::make_unique<samo::SamoTrainer>(s->spec, to_cfg(c), std::move(st));
  return s;
}

EXPORT void ref_session_destroy(void* h) { delete static_cast<RefSession*>(h); }

// One step: gather every layer's dense binary16 gradient (the backward sink,
// via samo::compress) then SamoTrainer::optimizer_step.  Returns 1 when the
// step was applied, 0 when skipped.
EXPORT int ref_session_step(void* h, const uint16_t* const* dense_grads) {
  auto* s = static_cast<RefSession*>(h);
  const samo::Tensor<samo::Half> x({1, 1}, {samo::Half(0.0f)});
  const samo::Tensor<float> y({1, 1}, {0.0f});
  s->trainer->forward(x, y);
  s->trainer->backward();  // dummy layer's sink; grads_ready_ = true
  auto& layers = const_cast<samo::ModelState&>(s->trainer->state()).layers;
  for (size_t l = 0; l < s->sets.size(); ++l) {
    const auto& set = *s->sets[l];
    const uint64_t n = s->dense_len[l];
    // compress() wants a Tensor<Half>; wrap the dense gradient (one copy).
    const samo::Tensor<samo::Half> t({static_cast<std::size_t>(n)}, halves(dense_grads[l], n));
    layers[l + 1].comp.grad16 = samo::compress(t, set);
  }
  return s->trainer->optimizer_step() ? 1 : 0;
}

// Times only what the reference does per step on this path: the sink gather
// (compress from a Tensor the caller already owns) + optimizer_step.
EXPORT void* ref_session_wrap_grads(void* h, const uint16_t* const* dense_grads) {
  auto* s = static_cast<RefSession*>(h);
  auto* v = new std::vector<samo::Tensor<samo::Half>>();
  for (size_t l = 0; l < s->sets.size(); ++l) {
    const uint64_t n = s->dense_len[l];
    v->emplace_back(std::vector<std::size_t>{static_cast<std::size_t>(n)}, halves(dense_grads[l], n));
  }
  return v;
}

EXPORT void ref_grads_destroy(void* g) { delete static_cast<std::vector<samo::Tensor<samo::Half>>*>(g); }

EXPORT int ref_session_step_wrapped(void* h, void* g) {
  auto* s = static_cast<RefSession*>(h);
  auto& grads = *static_cast<std::vector<samo::Tensor<samo::Half>>*>(g);
  const samo::Tensor<samo::Half> x({1, 1}, {samo::Half(0.0f)});
  const samo::Tensor<float> y({1, 1}, {0.0f});
  s->trainer->forward(x, y);
  s->trainer->backward();
  auto& layers = const_cast<samo::ModelState&>(s->trainer->state()).layers;
  for (size_t l = 0; l < s->sets.size(); ++l)
    layers[l + 1].comp.grad16 = samo::compress(grads[l], *s->sets[l]);
  return s->trainer->optimizer_step() ? 1 : 0;
}

EXPORT void ref_session_read(void* h, int layer, float* theta32, float* m, float* v, float* g32,
                             uint16_t* theta16) {
  auto* s = static_cast<RefSession*>(h);
  const auto& ls = s->trainer->state().layers[layer + 1];
  if (theta32) std::memcpy(theta32, ls.comp.theta32.data(), ls.comp.theta32.size() * 4);
  if (m) std::memcpy(m, ls.comp.adam_m.data(), ls.comp.adam_m.size() * 4);
  if (v) std::memcpy(v, ls.comp.adam_v.data(), ls.comp.adam_v.size() * 4);
  if (g32) std::memcpy(g32, ls.comp.grad32.data(), ls.comp.grad32.size() * 4);
  if (theta16)
    for (size_t i = 0; i < ls.theta16.size(); ++i) theta16[i] = ls.theta16.flat()[i].bits();
}

EXPORT void ref_session_counters(void* h, uint64_t* skipped, float* grad_norm) {
  auto* s = static_cast<RefSession*>(h);
  if (skipped) *skipped = s->trainer->skipped_steps();
  if (grad_norm) *grad_norm = s->trainer->last_grad_norm();
}

EXPORT int ref_session_check_invariants(void* h) {
  try {
    samo::check_state_invariants(static_cast<RefSession*>(h)->trainer->state());
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

EXPORT uint64_t ref_session_measured_bytes(void* h, int peak) {
  return samo::measured_bytes(static_cast<RefSession*>(h)->trainer->state(),
                              peak ? samo::Accounting::peak : samo::Accounting::steady_state);
}

// mlp_backward's weight gradient (train.hpp:304): matmul(transpose(x), dy).
EXPORT int ref_dw_matmul(const uint16_t* x, const uint16_t* dy, uint64_t batch, uint64_t in,
                         uint64_t out, uint16_t* dw) {
  try {
    std::vector<samo::Half> xv(batch * in), dv(batch * out);
    for (uint64_t i = 0; i < batch * in; ++i) xv[i] = samo::Half::from_bits(x[i]);
    for (uint64_t i = 0; i < batch * out; ++i) dv[i] = samo::Half::from_bits(dy[i]);
    const samo::Tensor<samo::Half> tx({static_cast<std::size_t>(batch), static_cast<std::size_t>(in)},
                                      std::move(xv));
    const samo::Tensor<samo::Half> td({static_cast<std::size_t>(batch), static_cast<std::size_t>(out)},
                                      std::move(dv));
    const auto w = samo::matmul(samo::transpose(tx), td);
    const auto f = w.flat();
    for (uint64_t i = 0; i < in * out; ++i) dw[i] = f[i].bits();
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

#ifdef SAMO_REF_JSON
// JSON checkpoints (serialize.hpp:121-190), when nlohmann's json.hpp is on
// the include path: parse -> checkpoint_from_json -> checkpoint_to_json ->
// dump, all of it the reference's own code.  98: not JSON; 100: `out` too small.
#include "samo/serialize.hpp"

EXPORT int ref_checkpoint_json_roundtrip(const char* in, char* out, uint64_t cap, uint64_t* need) {
  try {
    const samo::ModelState st = samo::checkpoint_from_json(nlohmann::json::parse(in));
    const std::string s = samo::checkpoint_to_json(st).dump();
    *need = s.size() + 1;
    if (s.size() + 1 > cap) return 100;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
  } catch (const nlohmann::json::parse_error&) {
    return 98;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// Pruned index sets <-> JSON (serialize.hpp:84-119), the same way.
EXPORT int ref_index_sets_json_roundtrip(const char* in, char* out, uint64_t cap, uint64_t* need) {
  try {
    const auto sets = samo::index_sets_from_json(nlohmann::json::parse(in));
    const std::string s = samo::index_sets_to_json(sets).dump();
    *need = s.size() + 1;
    if (s.size() + 1 > cap) return 100;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
  } catch (const nlohmann::json::parse_error&) {
    return 98;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
#endif
