// samo_b200/samo.hpp — C++ mirror of the reference's `samo::` API for the
// per-step parameter-state path, backed by the CUDA library through the C ABI
// of samo_cuda.h.  Header-only; link with libsamo_cuda.so.
//
// Drop-in surface (same names, argument meaning and exceptions as the
// reference headers /root/reference/proj/include/samo/*.hpp):
//   Half, Tensor<T>, numel, bit_equal                 (half.hpp, tensor.hpp)
//   PrunedIndexSet, LayerParams, PruneScope,
//   linearize, delinearize, magnitude_prune           (prune.hpp:21-170)
//   compress, expand                                  (store.hpp:58-87)
//   OptimizerConfig, adam_update                      (train.hpp:70-87, 332-347)
//   DimensionError, ParameterError, IndexError,
//   StateError, ConfigError                           (error.hpp:9-36)
// Host-container overloads copy to and from the device around one call (for
// call sites and tests written against the reference); production code keeps
// its state on the device with samo_b200::Model (ModelState + the
// SamoTrainer::optimizer_step of train.hpp:617-656, fused into two kernels).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "samo_cuda.h"

namespace samo_b200 {

// ---------------------------------------------------------------------------
// error.hpp

class DimensionError : public std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
class ParameterError : public std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
class IndexError : public std::out_of_range {
  using std::out_of_range::out_of_range;
};
class StateError : public std::logic_error {
  using std::logic_error::logic_error;
};
class ConfigError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
class CudaError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Rethrows a C-ABI status as the reference's exception class.
inline void check(int status) {
  if (status == SAMO_OK) return;
  const std::string msg = samo_last_error();
  switch (status) {
    case SAMO_E_DIMENSION: throw DimensionError(msg);
    case SAMO_E_PARAMETER: throw ParameterError(msg);
    case SAMO_E_INDEX: throw IndexError(msg);
    case SAMO_E_STATE: throw StateError(msg);
    case SAMO_E_CONFIG: throw ConfigError(msg);
    default: throw CudaError(std::string(samo_status_string(status)) + ": " + msg);
  }
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// half.hpp: binary16 storage type.  Conversions run on the device (bit-exact
// with float_to_half_bits / half_bits_to_float); the type itself is storage.

class Half {
 public:
  constexpr Half() = default;
  explicit Half(float value);
  static constexpr Half from_bits(std::uint16_t bits) {
    Half h;
    h.bits_ = bits;
    return h;
  }
  explicit operator float() const;
  constexpr std::uint16_t bits() const { return bits_; }
  bool is_finite() const { return (bits_ & 0x7C00u) != 0x7C00u; }
  bool is_nan() const { return (bits_ & 0x7C00u) == 0x7C00u && (bits_ & 0x03FFu) != 0u; }
  friend constexpr bool operator==(Half a, Half b) { return a.bits_ == b.bits_; }
  friend constexpr bool operator!=(Half a, Half b) { return a.bits_ != b.bits_; }

 private:
  std::uint16_t bits_ = 0;
};
static_assert(sizeof(Half) == 2, "Half is a 16-bit storage type");

// ---------------------------------------------------------------------------
// Device buffer (RAII) used by the host-container overloads.

template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t n) : n_(n) {
    if (n_) cuda_check(cudaMalloc(&p_, n_ * sizeof(T)), "cudaMalloc");
  }
  DeviceBuffer(const T* host, std::size_t n) : DeviceBuffer(n) { upload(host, n); }
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  void upload(const T* host, std::size_t n) {
    if (n) cuda_check(cudaMemcpy(p_, host, n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  }
  void download(T* host, std::size_t n) const {
    if (n) cuda_check(cudaMemcpy(host, p_, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
  }
  std::vector<T> to_host() const {
    std::vector<T> v(n_);
    download(v.data(), n_);
    return v;
  }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

inline Half::Half(float value) {
  DeviceBuffer<float> in(&value, 1);
  DeviceBuffer<std::uint16_t> out(1);
  check(samo_float_to_half(in.get(), out.get(), 1, nullptr));
  out.download(&bits_, 1);
}

inline Half::operator float() const {
  DeviceBuffer<std::uint16_t> in(&bits_, 1);
  DeviceBuffer<float> out(1);
  check(samo_half_to_float(in.get(), out.get(), 1, nullptr));
  float f;
  out.download(&f, 1);
  return f;
}

inline float to_float(Half h) { return static_cast<float>(h); }

// Batch conversions (one launch): Half(float) / float(Half) of every element.
inline std::vector<Half> to_half(std::span<const float> v) {
  std::vector<Half> out(v.size());
  if (v.empty()) return out;
  DeviceBuffer<float> in(v.data(), v.size());
  DeviceBuffer<std::uint16_t> o(v.size());
  check(samo_float_to_half(in.get(), o.get(), v.size(), nullptr));
  o.download(reinterpret_cast<std::uint16_t*>(out.data()), v.size());
  return out;
}

inline std::vector<float> to_float(std::span<const Half> v) {
  std::vector<float> out(v.size());
  if (v.empty()) return out;
  DeviceBuffer<std::uint16_t> in(reinterpret_cast<const std::uint16_t*>(v.data()), v.size());
  DeviceBuffer<float> o(v.size());
  check(samo_half_to_float(in.get(), o.get(), v.size(), nullptr));
  o.download(out.data(), v.size());
  return out;
}

// ---------------------------------------------------------------------------
// tensor.hpp (container part)

inline std::size_t numel(std::span<const std::size_t> shape) {
  std::size_t n = 1;
  for (std::size_t e : shape) n *= e;
  return n;
}

template <typename T>
class Tensor {
 public:
  Tensor() = default;
  explicit Tensor(std::vector<std::size_t> shape) : shape_(std::move(shape)), data_(numel(shape_)) {
    check_shape();
  }
  Tensor(std::vector<std::size_t> shape, std::vector<T> data)
      : shape_(std::move(shape)), data_(std::move(data)) {
    check_shape();
    if (data_.size() != numel(shape_)) throw DimensionError("tensor data length does not match shape");
  }
  const std::vector<std::size_t>& shape() const { return shape_; }
  std::size_t size() const { return data_.size(); }
  std::size_t rank() const { return shape_.size(); }
  std::size_t rows() const { return shape_.at(0); }  // 2-D accessors (tensor.hpp:55-56)
  std::size_t cols() const { return shape_.at(1); }
  std::span<const T> flat() const { return data_; }
  std::span<T> flat() { return data_; }
  T operator[](std::size_t i) const { return data_[i]; }
  T& operator[](std::size_t i) { return data_[i]; }
  friend bool operator==(const Tensor& a, const Tensor& b) = default;

 private:
  void check_shape() const {
    for (std::size_t e : shape_)
      if (e == 0) throw DimensionError("tensor extents must be positive");
  }
  std::vector<std::size_t> shape_;
  std::vector<T> data_;
};

template <typename T>
bool bit_equal(const Tensor<T>& a, const Tensor<T>& b) {
  if (a.shape() != b.shape()) return false;
  return std::memcmp(a.flat().data(), b.flat().data(), a.size() * sizeof(T)) == 0;
}

// ---------------------------------------------------------------------------
// prune.hpp

struct PrunedIndexSet {
  std::string layer_id;
  std::uint64_t dense_len = 0;
  std::vector<std::uint32_t> indices;  // strictly ascending, < dense_len
  std::size_t count() const { return indices.size(); }
};

// Row-major linear index per coordinate; output sorted ascending (prune.hpp:30-48).
inline std::vector<std::uint64_t> linearize(std::span<const std::vector<std::uint64_t>> coords,
                                            std::span<const std::size_t> shape) {
  std::vector<std::uint64_t> out;
  out.reserve(coords.size());
  for (const auto& c : coords) {
    if (c.size() != shape.size()) throw IndexError("coordinate rank does not match shape");
    std::uint64_t idx = 0;
    for (std::size_t d = 0; d < shape.size(); ++d) {
      if (c[d] >= shape[d]) throw IndexError("coordinate out of bounds");
      idx = idx * shape[d] + c[d];
    }
    out.push_back(idx);
  }
  std::sort(out.begin(), out.end());
  return out;
}

inline std::vector<std::uint64_t> delinearize(std::uint64_t index, std::span<const std::size_t> shape) {
  if (index >= numel(shape)) throw IndexError("linear index out of bounds");
  std::vector<std::uint64_t> c(shape.size());
  for (std::size_t d = shape.size(); d-- > 0;) {
    c[d] = index % shape[d];
    index /= shape[d];
  }
  return c;
}

enum class PruneScope { per_layer = SAMO_PRUNE_PER_LAYER, global = SAMO_PRUNE_GLOBAL };

struct LayerParams {
  std::string layer_id;
  Tensor<float> values;
  bool prunable = true;
};

// magnitude_prune (prune.hpp:99-170) on the device (kernel K0).
inline std::vector<PrunedIndexSet> magnitude_prune(std::span<const LayerParams> layers, double p,
                                                   PruneScope scope = PruneScope::per_layer) {
  const int L = static_cast<int>(layers.size());
  std::vector<DeviceBuffer<float>> vals;
  std::vector<DeviceBuffer<std::uint32_t>> outs;
  std::vector<const float*> vp(L);
  std::vector<std::uint32_t*> op(L);
  std::vector<std::uint64_t> lens(L), counts(L);
  std::vector<std::uint8_t> pr(L);
  vals.reserve(L);
  outs.reserve(L);
  for (int l = 0; l < L; ++l) {
    const auto f = layers[l].values.flat();
    vals.emplace_back(f.data(), f.size());
    outs.emplace_back(std::max<std::size_t>(1, f.size()));
    vp[l] = vals.back().get();
    op[l] = outs.back().get();
    lens[l] = f.size();
    pr[l] = layers[l].prunable ? 1 : 0;
  }
  check(samo_magnitude_prune(vp.data(), lens.data(), pr.data(), L, p, static_cast<int>(scope), op.data(),
                             counts.data(), nullptr));
  std::vector<PrunedIndexSet> sets(L);
  for (int l = 0; l < L; ++l) {
    sets[l].layer_id = layers[l].layer_id;
    sets[l].dense_len = lens[l];
    sets[l].indices.resize(counts[l]);
    outs[l].download(sets[l].indices.data(), counts[l]);
  }
  return sets;
}

// ---------------------------------------------------------------------------
// store.hpp: compress / expand

template <typename T>
std::vector<T> compress(const Tensor<T>& dense, const PrunedIndexSet& ind) {
  static_assert(sizeof(T) == 2 || sizeof(T) == 4, "16- or 32-bit elements");
  std::vector<T> out(ind.count());
  // The length check (store.hpp:60-62) happens in the C ABI -> DimensionError.
  DeviceBuffer<T> d(dense.flat().data(), dense.size());
  DeviceBuffer<std::uint32_t> idx(ind.indices.data(), ind.count());
  DeviceBuffer<T> o(ind.count());
  if constexpr (sizeof(T) == 2) {
    check(samo_compress_u16(reinterpret_cast<const std::uint16_t*>(d.get()), dense.size(), idx.get(),
                            ind.count(), ind.dense_len, reinterpret_cast<std::uint16_t*>(o.get()), nullptr));
  } else {
    check(samo_compress_u32(reinterpret_cast<const std::uint32_t*>(d.get()), dense.size(), idx.get(),
                            ind.count(), ind.dense_len, reinterpret_cast<std::uint32_t*>(o.get()), nullptr));
  }
  o.download(out.data(), out.size());
  return out;
}

template <typename T>
Tensor<T> expand(std::span<const T> values, const PrunedIndexSet& ind, std::vector<std::size_t> shape) {
  static_assert(sizeof(T) == 2 || sizeof(T) == 4, "16- or 32-bit elements");
  const std::size_t n = numel(shape);
  DeviceBuffer<T> v(values.data(), values.size());
  DeviceBuffer<std::uint32_t> idx(ind.indices.data(), ind.count());
  DeviceBuffer<T> o(std::max<std::size_t>(1, n));
  if constexpr (sizeof(T) == 2) {
    check(samo_expand_u16(reinterpret_cast<const std::uint16_t*>(v.get()), values.size(), idx.get(),
                          ind.count(), ind.dense_len, n, reinterpret_cast<std::uint16_t*>(o.get()), nullptr));
  } else {
    check(samo_expand_u32(reinterpret_cast<const std::uint32_t*>(v.get()), values.size(), idx.get(),
                          ind.count(), ind.dense_len, n, reinterpret_cast<std::uint32_t*>(o.get()), nullptr));
  }
  Tensor<T> out(std::move(shape));
  o.download(out.flat().data(), n);
  return out;
}

// ---------------------------------------------------------------------------
// train.hpp: OptimizerConfig + adam_update

struct OptimizerConfig {
  float learning_rate = 1e-3f;
  float beta1 = 0.9f;
  float beta2 = 0.999f;
  float epsilon = 1e-8f;
  float loss_scale = 1024.0f;
  float weight_decay = 0.0f;

  samo_optimizer_config c() const {
    return {learning_rate, beta1, beta2, epsilon, loss_scale, weight_decay};
  }
  void validate() const {
    const samo_optimizer_config cc = c();
    check(samo_optimizer_config_validate(&cc));
  }
};

inline void adam_update(std::span<float> theta, std::span<float> m, std::span<float> v,
                        std::span<const float> g, const OptimizerConfig& cfg, float bias1, float bias2) {
  const std::size_t n = theta.size();
  if (m.size() != n || v.size() != n || g.size() != n) throw DimensionError("adam_update: span lengths differ");
  DeviceBuffer<float> t(theta.data(), n), mm(m.data(), n), vv(v.data(), n), gg(g.data(), n);
  const samo_optimizer_config cc = cfg.c();
  check(samo_adam_update(t.get(), mm.get(), vv.get(), gg.get(), n, &cc, bias1, bias2, nullptr));
  t.download(theta.data(), n);
  mm.download(m.data(), n);
  vv.download(v.data(), n);
}

// matmul(transpose(x), dy) (train.hpp:304, tensor.hpp:88-105) on the tensor
// cores: x [batch x in], dy [batch x out] -> [in x out] binary16.  Host
// containers in, host tensor out (the reference's value semantics).
inline Tensor<Half> dw_matmul(const Tensor<Half>& x, const Tensor<Half>& dy) {
  if (x.rank() != 2 || dy.rank() != 2 || x.rows() != dy.rows())
    throw DimensionError("matmul expects MxK and KxN operands");
  const std::uint64_t batch = x.rows(), in = x.cols(), out = dy.cols();
  DeviceBuffer<std::uint16_t> dx(reinterpret_cast<const std::uint16_t*>(x.flat().data()), x.size());
  DeviceBuffer<std::uint16_t> dd(reinterpret_cast<const std::uint16_t*>(dy.flat().data()), dy.size());
  DeviceBuffer<std::uint16_t> dw(in * out);
  check(samo_dw_gemm_f16(dx.get(), dd.get(), batch, in, out, dw.get(), nullptr));
  std::vector<Half> h(in * out);
  dw.download(reinterpret_cast<std::uint16_t*>(h.data()), in * out);
  return Tensor<Half>({static_cast<std::size_t>(in), static_cast<std::size_t>(out)}, std::move(h));
}

// ---------------------------------------------------------------------------
// Device-resident model state + step driver (ModelState / SamoTrainer).

struct StepRecord {
  std::uint64_t t = 0, skipped_steps = 0;
  float grad_norm = 0.0f;
  bool last_skipped = false;
};

class Model {
 public:
  // One index set per parameter tensor (the ModelState's shared index sets).
  Model(const std::vector<PrunedIndexSet>& sets, std::uint32_t tile_elems = 0) {
    std::vector<samo_layer_desc> d(sets.size());
    for (std::size_t l = 0; l < sets.size(); ++l) d[l] = {sets[l].dense_len, sets[l].count()};
    samo_model* m = nullptr;
    check(samo_model_create(d.data(), static_cast<int>(d.size()), tile_elems, &m));
    h_.reset(m);
    for (std::size_t l = 0; l < sets.size(); ++l)
      check(samo_model_set_indices(m, static_cast<int>(l), sets[l].indices.data(), sets[l].count(), 1, nullptr));
    check(samo_model_finalize(m, nullptr));
    dense_len_.resize(sets.size());
    for (std::size_t l = 0; l < sets.size(); ++l) dense_len_[l] = sets[l].dense_len;
  }
  samo_model* handle() const { return h_.get(); }
  int num_layers() const { return samo_model_num_layers(h_.get()); }

  // make_layer_state (store.hpp:150-168) from dense fp32 initial values.
  void init_layer(int l, const Tensor<float>& init) {
    DeviceBuffer<float> d(init.flat().data(), init.size());
    check(samo_model_init_layer(h_.get(), l, d.get(), init.size(), nullptr));
    cuda_check(cudaDeviceSynchronize(), "init_layer");
  }
  void set_config(const OptimizerConfig& cfg) {
    const samo_optimizer_config c = cfg.c();
    check(samo_model_set_config(h_.get(), &c));
  }
  // Dense binary16 gradients on the device (the backward sink's input).
  void set_grads(const std::vector<const std::uint16_t*>& dev_ptrs, cudaStream_t s = nullptr) {
    check(samo_model_set_grads(h_.get(), dev_ptrs.data(), s));
  }
  // The trainer's backward sink (train.hpp:596-611), one layer at a time, as
  // each dense gradient is produced (single-GPU models; then update()).
  void sink_dense(int l, const std::uint16_t* dev_grad, cudaStream_t s = nullptr) {
    check(samo_model_sink_dense(h_.get(), l, dev_grad, s));
  }
  // Fused sink: dW = X^T . dY (mlp_backward, train.hpp:304-305) on the tensor
  // cores with the gather in the GEMM epilogue; x [batch x in], dy [batch x out].
  void sink_dw(int l, const std::uint16_t* x, const std::uint16_t* dy, std::uint64_t batch, std::uint64_t in,
               std::uint64_t out, cudaStream_t s = nullptr) {
    check(samo_model_sink_dw(h_.get(), l, x, dy, batch, in, out, s));
  }
  // Skip decision, AdamScalars::advance, Adam, downcast + expand after the sinks.
  void update(cudaStream_t s = nullptr) { check(samo_model_update(h_.get(), s)); }
  // After the sinks on a data-parallel model: exchange + update.
  void step_sunk(cudaStream_t s = nullptr) { check(samo_model_step_sunk(h_.get(), s)); }
  // SamoTrainer::optimizer_step (train.hpp:617-656) without host sync.
  void step(cudaStream_t s = nullptr, bool graph = false) {
    check(graph ? samo_model_step_graph(h_.get(), s) : samo_model_step(h_.get(), s));
  }
  StepRecord record(cudaStream_t s = nullptr) const {
    samo_step_record r{};
    check(samo_model_step_record(h_.get(), &r, s));
    return {r.t, r.skipped_steps, r.grad_norm, r.last_skipped != 0};
  }
  void check_state_invariants(cudaStream_t s = nullptr) { check(samo_model_check_invariants(h_.get(), s)); }
  samo_layer_view view(int l) const {
    samo_layer_view v{};
    check(samo_model_layer_view(h_.get(), l, &v));
    return v;
  }
  std::vector<float> theta32(int l) const { return read<float>(view(l).theta32, view(l).nnz); }
  std::vector<float> adam_m(int l) const { return read<float>(view(l).adam_m, view(l).nnz); }
  std::vector<float> adam_v(int l) const { return read<float>(view(l).adam_v, view(l).nnz); }
  std::vector<Half> theta16(int l) const { return read<Half>(view(l).theta16, view(l).dense_len); }

 private:
  template <typename T, typename P>
  static std::vector<T> read(P* dev, std::size_t n) {
    std::vector<T> out(n);
    if (n) cuda_check(cudaMemcpy(out.data(), dev, n * sizeof(T), cudaMemcpyDeviceToHost), "read");
    return out;
  }
  struct Del {
    void operator()(samo_model* m) const { samo_model_destroy(m); }
  };
  std::unique_ptr<samo_model, Del> h_;
  std::vector<std::uint64_t> dense_len_;
};

}  // namespace samo_b200
