// samo_b200/samo.hpp — C++ mirror of the reference's `samo::` API for the
// per-step parameter-state path, backed by the CUDA library through the C ABI
// of samo_cuda.h.  Header-only; link with libsamo_cuda.so.  The reference's
// header names are forwarding headers under include/samo/ (samo/half.hpp,
// samo/store.hpp, samo/train.hpp, ...), so `#include "samo/store.hpp"` with
// -I include compiles a reference call site against this mirror.
//
// Drop-in surface (namespace samo; same names, argument meaning and
// exceptions as the reference headers proj/include/samo/*.hpp):
//   Half, to_float, from_float, to_half/to_float (batch)  (half.hpp:75-118)
//   Tensor<T>, numel, cast, bit_equal                      (tensor.hpp:15-71, 120-127, 180-192)
//   PrunedIndexSet, LayerParams, PruneScope,
//   linearize, delinearize, magnitude_prune                (prune.hpp:21-170)
//   CompressedState, LayerState, ModelState                (store.hpp:22-55)
//   compress, expand                                       (store.hpp:58-87)
//   Rational, MemoryReport, memory_model, to_double,
//   model_state_bytes, Accounting, measured_bytes          (store.hpp:89-147)
//   make_layer_state, check_state_invariants               (store.hpp:150-197)
//   OptimizerConfig, AdamScalars, adam_update              (train.hpp:70-87, 320-347)
//   SamoTrainer: the backward sink + optimizer_step()      (train.hpp:574-704)
//   DimensionError, ParameterError, IndexError,
//   StateError, ConfigError, InfeasibleError               (error.hpp:9-36)
// Scalar binary16 conversions run on the host (the reference's RNE contract,
// restated in integer arithmetic); every array operation runs on the device.
// Host-container overloads copy to and from the device around one call (for
// call sites and tests written against the reference); production code keeps
// its state on the device with samo::Model (the ModelState + the
// SamoTrainer::optimizer_step of train.hpp:617-656 as fused kernels) or
// samo::SamoTrainer over it.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <bit>
#include <cmath>
#include <numeric>
#include <cstdint>
#include <cstring>
#include <memory>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "samo_cuda.h"

namespace samo {

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
class InfeasibleError : public std::runtime_error {
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
// half.hpp: binary16 storage type.  Scalar conversions on the host (below);
// array conversions (to_half / to_float of a span) in one device launch.

namespace detail {

// binary32 -> binary16, round to nearest even (half.hpp:13-49 contract):
// NaN keeps its top payload bits with the quiet bit set, overflow goes to
// infinity, |x| < 2^-25 to signed zero.  One rounding path serves normal and
// subnormal results: the kept significand is sig >> shift, and a carry out of
// the mantissa moves into the exponent field.
inline std::uint16_t half_rne_bits(float value) {
  const std::uint32_t x = std::bit_cast<std::uint32_t>(value);
  const std::uint32_t sign = (x >> 16) & 0x8000u;
  const std::uint32_t e = (x >> 23) & 0xFFu;
  const std::uint32_t m = x & 0x007FFFFFu;
  if (e == 0xFFu) return static_cast<std::uint16_t>(sign | 0x7C00u | (m ? 0x0200u | (m >> 13) : 0u));
  if (e < 102u) return static_cast<std::uint16_t>(sign);  // below 2^-25
  std::uint32_t sig, shift, base;
  if (e >= 113u) {  // binary16 normal (or overflow): 10 of 23 mantissa bits
    sig = m;
    shift = 13u;
    base = (e - 112u) << 10;
  } else {          // binary16 subnormal: the 24-bit significand >> [14, 24]
    sig = m | 0x00800000u;
    shift = 126u - e;
    base = 0u;
  }
  std::uint32_t q = sig >> shift;
  const std::uint32_t rem = sig & ((1u << shift) - 1u), half = 1u << (shift - 1u);
  q += (rem > half) || (rem == half && (q & 1u));
  const std::uint32_t out = base + q;
  return static_cast<std::uint16_t>(sign | (out >= 0x7C00u ? 0x7C00u : out));
}

// binary16 -> binary32, exact (half.hpp:52-71 contract; NaN payloads kept).
inline float half_to_float_exact(std::uint16_t h) {
  const std::uint32_t sign = (static_cast<std::uint32_t>(h) & 0x8000u) << 16;
  const std::uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x03FFu;
  if (e == 0x1Fu) return std::bit_cast<float>(sign | 0x7F800000u | (m << 13));
  if (e == 0u) {  // zero or subnormal: m * 2^-24 is exact in binary32
    const float mag = static_cast<float>(m) * 0x1.0p-24f;
    return std::bit_cast<float>(sign | std::bit_cast<std::uint32_t>(mag));
  }
  return std::bit_cast<float>(sign | ((e + 112u) << 23) | (m << 13));
}

}  // namespace detail

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

inline Half::Half(float value) : bits_(detail::half_rne_bits(value)) {}
inline Half::operator float() const { return detail::half_to_float_exact(bits_); }

inline float to_float(Half h) { return static_cast<float>(h); }
inline constexpr float to_float(float f) { return f; }

template <typename T>
T from_float(float f);
template <>
inline Half from_float<Half>(float f) {
  return Half(f);
}
template <>
inline constexpr float from_float<float>(float f) {
  return f;
}

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
  bool empty() const { return data_.empty(); }
  std::size_t rows() const { return shape_.at(0); }  // 2-D accessors (tensor.hpp:55-56)
  std::size_t cols() const { return shape_.at(1); }
  std::span<const T> flat() const { return data_; }
  std::span<T> flat() { return data_; }
  T operator[](std::size_t i) const { return data_[i]; }
  T& operator[](std::size_t i) { return data_[i]; }
  T at(std::size_t r, std::size_t c) const { return data_[r * cols() + c]; }
  T& at(std::size_t r, std::size_t c) { return data_[r * cols() + c]; }
  friend bool operator==(const Tensor& a, const Tensor& b) = default;

 private:
  void check_shape() const {
    for (std::size_t e : shape_)
      if (e == 0) throw DimensionError("tensor extents must be positive");
  }
  std::vector<std::size_t> shape_;
  std::vector<T> data_;
};

// cast (tensor.hpp:120-127): float -> Half rounds to nearest even, Half ->
// float is exact; array conversions run on the device.
template <typename To, typename From>
Tensor<To> cast(const Tensor<From>& t) {
  if constexpr (std::is_same_v<To, From>) {
    return t;
  } else if constexpr (std::is_same_v<To, Half>) {
    return Tensor<To>(t.shape(), to_half(t.flat()));
  } else {
    return Tensor<To>(t.shape(), to_float(t.flat()));
  }
}

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
// store.hpp: state containers, memory accounting, make_layer_state,
// check_state_invariants.  Host containers with the reference's fields; the
// array work (gather, downcast + expand) runs on the device.

// Compressed model state of one layer (store.hpp:22-31): five value buffers
// of count() elements sharing one index set.
struct CompressedState {
  std::shared_ptr<const PrunedIndexSet> ind;
  std::vector<float> theta32;
  std::vector<Half> grad16;
  std::vector<float> grad32;
  std::vector<float> adam_m;
  std::vector<float> adam_v;

  std::size_t count() const { return ind ? ind->count() : 0; }
};

// One parameter tensor (store.hpp:35-40).
struct LayerState {
  std::string layer_id;
  std::vector<std::size_t> shape;
  Tensor<Half> theta16;  // dense, zeros at pruned slots
  CompressedState comp;
};

struct ModelState {  // store.hpp:42-55
  std::vector<LayerState> layers;

  std::uint64_t total_params() const {
    std::uint64_t n = 0;
    for (const auto& l : layers) n += l.theta16.size();
    return n;
  }
  std::uint64_t total_unpruned() const {
    std::uint64_t n = 0;
    for (const auto& l : layers) n += l.comp.count();
    return n;
  }
};

// Exact rational in lowest terms with a positive denominator — the value
// type the reference's memory model uses (boost::rational<long long>,
// store.hpp:17), restated so the mirror has no boost dependency.
class Rational {
 public:
  constexpr Rational() = default;
  constexpr Rational(long long n) : num_(n) {}  // NOLINT: implicit, as boost::rational
  Rational(long long n, long long d) : num_(n), den_(d) {
    if (den_ == 0) throw std::domain_error("Rational: zero denominator");
    normalize();
  }
  constexpr long long numerator() const { return num_; }
  constexpr long long denominator() const { return den_; }

  friend Rational operator+(const Rational& a, const Rational& b) {
    const long long g = std::gcd(a.den_, b.den_);
    return Rational(a.num_ * (b.den_ / g) + b.num_ * (a.den_ / g), (a.den_ / g) * b.den_);
  }
  friend Rational operator-(const Rational& a, const Rational& b) { return a + Rational(-b.num_, b.den_); }
  friend Rational operator*(const Rational& a, const Rational& b) {
    const long long g1 = std::gcd(a.num_, b.den_), g2 = std::gcd(b.num_, a.den_);
    const long long d1 = g1 ? g1 : 1, d2 = g2 ? g2 : 1;
    return Rational((a.num_ / d1) * (b.num_ / d2), (a.den_ / d2) * (b.den_ / d1));
  }
  friend Rational operator/(const Rational& a, const Rational& b) {
    if (b.num_ == 0) throw std::domain_error("Rational: division by zero");
    return a * Rational(b.den_, b.num_);
  }
  Rational operator-() const { return Rational(-num_, den_); }
  friend bool operator==(const Rational& a, const Rational& b) { return a.num_ == b.num_ && a.den_ == b.den_; }
  friend bool operator<(const Rational& a, const Rational& b) {
    // denominators are positive: compare a.n * b.d with b.n * a.d
    return static_cast<__int128>(a.num_) * b.den_ < static_cast<__int128>(b.num_) * a.den_;
  }
  friend bool operator>(const Rational& a, const Rational& b) { return b < a; }
  friend bool operator<=(const Rational& a, const Rational& b) { return !(b < a); }
  friend bool operator>=(const Rational& a, const Rational& b) { return !(a < b); }
  friend bool operator!=(const Rational& a, const Rational& b) { return !(a == b); }

 private:
  void normalize() {
    if (den_ < 0) num_ = -num_, den_ = -den_;
    const long long g = std::gcd(num_, den_);
    if (g > 1) num_ /= g, den_ /= g;
  }
  long long num_ = 0;
  long long den_ = 1;
};

// Analytical model-state bytes (store.hpp:89-120): 20 phi dense mixed
// precision against 24 (1 - p) phi + 2 phi compressed.
struct MemoryReport {
  long long phi = 0;
  Rational p;
  Rational bytes_default;
  Rational bytes_samo;
  Rational bytes_saved;
  Rational savings_fraction;
};

inline double to_double(const Rational& r) {
  return static_cast<double>(r.numerator()) / static_cast<double>(r.denominator());
}

inline MemoryReport memory_model(long long phi, Rational p) {
  if (phi < 0) throw ParameterError("phi must be non-negative");
  if (p < Rational(0) || p > Rational(1)) throw ParameterError("sparsity must lie in [0, 1]");
  MemoryReport r;
  r.phi = phi;
  r.p = p;
  r.bytes_default = Rational(20 * phi);
  r.bytes_samo = Rational(24) * (Rational(1) - p) * Rational(phi) + Rational(2 * phi);
  r.bytes_saved = r.bytes_default - r.bytes_samo;  // = (24 p - 6) phi
  r.savings_fraction = (Rational(24) * p - Rational(6)) / Rational(20);
  return r;
}

inline double model_state_bytes(double phi, double p, bool samo) {
  return samo ? 24.0 * (1.0 - p) * phi + 2.0 * phi : 20.0 * phi;
}

// peak adds the transient compressed half copy of the downcast
// (store.hpp:127-147); steady_state does not.
enum class Accounting { steady_state, peak };

inline std::uint64_t measured_bytes(const ModelState& state, Accounting mode = Accounting::peak) {
  // per layer: dense theta16 2 phi_l; grad16 2, theta32 4, grad32 4, m + v 8,
  // shared u32 index 4 bytes per kept element (+ 2 for the peak half copy)
  const std::uint64_t per_kept = mode == Accounting::peak ? 24u : 22u;
  std::uint64_t total = 0;
  for (const auto& layer : state.layers) total += 2u * layer.theta16.size() + per_kept * layer.comp.count();
  return total;
}

// make_layer_state (store.hpp:150-168): theta32 = compress(init) and
// theta16 = expand(half(theta32)) on the device; grads and moments zero.
inline LayerState make_layer_state(const Tensor<float>& init, std::shared_ptr<const PrunedIndexSet> ind) {
  if (!ind) throw StateError("make_layer_state: null index set");
  LayerState layer;
  layer.layer_id = ind->layer_id;
  layer.shape = init.shape();
  layer.comp.theta32 = compress(init, *ind);  // DimensionError on a length mismatch
  const std::size_t n = ind->count();
  layer.comp.grad16.assign(n, Half{});
  layer.comp.grad32.assign(n, 0.0f);
  layer.comp.adam_m.assign(n, 0.0f);
  layer.comp.adam_v.assign(n, 0.0f);
  const std::size_t dense = init.size();
  DeviceBuffer<float> th(layer.comp.theta32.data(), n);
  DeviceBuffer<std::uint32_t> idx(ind->indices.data(), n);
  DeviceBuffer<std::uint16_t> t16(std::max<std::size_t>(1, dense));
  check(samo_downcast_expand(th.get(), n, idx.get(), ind->dense_len, t16.get(), nullptr));
  layer.theta16 = Tensor<Half>(init.shape());
  t16.download(reinterpret_cast<std::uint16_t*>(layer.theta16.flat().data()), dense);
  layer.comp.ind = std::move(ind);
  return layer;
}

// check_state_invariants (store.hpp:171-197): buffer lengths on the host;
// theta16 == expand(half(theta32)) with exact zeros at pruned slots by
// rebuilding expand(half(theta32)) on the device and comparing bits.  The
// first differing position decides the message, as the reference's
// ascending scan does.
inline void check_state_invariants(const ModelState& state) {
  for (const auto& layer : state.layers) {
    const auto& c = layer.comp;
    if (!c.ind) throw StateError("layer has no index set: " + layer.layer_id);
    const std::size_t n = c.ind->count();
    if (c.theta32.size() != n || c.grad16.size() != n || c.grad32.size() != n || c.adam_m.size() != n ||
        c.adam_v.size() != n)
      throw StateError("compressed buffer length mismatch: " + layer.layer_id);
    if (layer.theta16.size() != c.ind->dense_len || numel(layer.shape) != c.ind->dense_len)
      throw StateError("dense length mismatch: " + layer.layer_id);
    const std::size_t dense = layer.theta16.size();
    if (dense == 0) continue;
    DeviceBuffer<float> th(c.theta32.data(), n);
    DeviceBuffer<std::uint32_t> idx(c.ind->indices.data(), n);
    DeviceBuffer<std::uint16_t> want(dense);
    check(samo_downcast_expand(th.get(), n, idx.get(), c.ind->dense_len, want.get(), nullptr));
    const std::vector<std::uint16_t> w = want.to_host();
    const auto* have = reinterpret_cast<const std::uint16_t*>(layer.theta16.flat().data());
    if (std::memcmp(have, w.data(), dense * sizeof(std::uint16_t)) == 0) continue;
    std::size_t i = 0;
    while (have[i] == w[i]) ++i;
    const auto& ix = c.ind->indices;
    if (std::binary_search(ix.begin(), ix.end(), static_cast<std::uint32_t>(i)))
      throw StateError("theta16 disagrees with theta32: " + layer.layer_id);
    throw StateError("nonzero theta16 at pruned slot: " + layer.layer_id);
  }
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

// AdamScalars (train.hpp:320-330): beta^t by repeated float products.
struct AdamScalars {
  std::uint64_t t = 0;
  float beta1_pow = 1.0f;
  float beta2_pow = 1.0f;

  void advance(const OptimizerConfig& cfg) {
    ++t;
    beta1_pow *= cfg.beta1;
    beta2_pow *= cfg.beta2;
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

// ---------------------------------------------------------------------------
// SamoTrainer (train.hpp:574-704): the compressed-state trainer's parameter
// path over a device Model.  The reference's trainer also owns the MLP
// forward/backward (ModelSpec, mlp_forward, mlp_backward — outside the hot
// path); here the caller's backward hands each dense gradient to
// sink() the moment it is produced, which is what mlp_backward's sink
// callback receives (train.hpp:287-313, 596-611).  Layer i is the i-th
// LayerState of the ModelState (the reference's param_index).
//
//   SamoTrainer tr(cfg, std::move(state));
//   for (each layer, last to first) tr.sink(i, dense_grad);   // backward()
//   bool applied = tr.optimizer_step();                         // train.hpp:617-656
//   const ModelState& st = tr.state();                          // host snapshot
class SamoTrainer {
 public:
  SamoTrainer(OptimizerConfig cfg, ModelState state, std::uint32_t tile_elems = 0)
      : cfg_(cfg), state_(std::move(state)) {
    cfg_.validate();
    std::vector<PrunedIndexSet> sets;
    sets.reserve(state_.layers.size());
    for (const auto& l : state_.layers) {
      if (!l.comp.ind) throw StateError("layer has no index set: " + l.layer_id);
      sets.push_back(*l.comp.ind);
    }
    model_ = std::make_unique<Model>(sets, tile_elems);
    model_->set_config(cfg_);
    for (std::size_t i = 0; i < state_.layers.size(); ++i) {
      const LayerState& l = state_.layers[i];
      const samo_layer_view v = model_->view(static_cast<int>(i));
      if (l.comp.theta32.size() != v.nnz || l.comp.adam_m.size() != v.nnz || l.comp.adam_v.size() != v.nnz)
        throw StateError("compressed buffer length mismatch: " + l.layer_id);
      if (l.theta16.size() != v.dense_len) throw StateError("dense length mismatch: " + l.layer_id);
      put(v.theta32, l.comp.theta32.data(), v.nnz * 4);
      put(v.adam_m, l.comp.adam_m.data(), v.nnz * 4);
      put(v.adam_v, l.comp.adam_v.data(), v.nnz * 4);
      put(v.theta16, l.theta16.flat().data(), v.dense_len * 2);
    }
    cuda_check(cudaDeviceSynchronize(), "SamoTrainer upload");
  }

  // The backward sink for layer i: gather the kept entries of the dense
  // binary16 gradient on the device (K1), raising the skip flag on a
  // non-finite one.  Host tensor (staged to the device) or device pointer.
  void sink(std::size_t i, const Tensor<Half>& dense_grad) {
    check_layer(i);
    if (dense_grad.size() != state_.layers[i].theta16.size())
      throw DimensionError("sink: gradient length does not match layer " + state_.layers[i].layer_id);
    stage_.emplace_back(reinterpret_cast<const std::uint16_t*>(dense_grad.flat().data()), dense_grad.size());
    sink_device(i, stage_.back().get());
  }
  void sink_device(std::size_t i, const std::uint16_t* dev_grad, cudaStream_t s = nullptr) {
    check_layer(i);
    model_->sink_dense(static_cast<int>(i), dev_grad, s);
    grads_ready_ = true;
    fresh_ = false;
  }

  // train.hpp:617-656: false when the step was skipped on a non-finite
  // gradient (then nothing but the counter changes).
  bool optimizer_step(cudaStream_t s = nullptr) {
    if (!grads_ready_) throw StateError("optimizer_step requires backward");
    model_->update(s);
    rec_ = model_->record(s);  // synchronises
    stage_.clear();
    grads_ready_ = false;
    fresh_ = false;
    return !rec_.last_skipped;
  }

  // Host snapshot of the device state (downloaded when stale).  Between the
  // sinks and optimizer_step, grad16 holds the gathered gradients; after a
  // step both gradient buffers read as zeros (train.hpp:634-637, 652-653).
  const ModelState& state() const {
    if (!fresh_) {
      for (std::size_t i = 0; i < state_.layers.size(); ++i) {
        LayerState& l = state_.layers[i];
        const samo_layer_view v = model_->view(static_cast<int>(i));
        get(l.comp.theta32.data(), v.theta32, v.nnz * 4);
        get(l.comp.adam_m.data(), v.adam_m, v.nnz * 4);
        get(l.comp.adam_v.data(), v.adam_v, v.nnz * 4);
        get(l.theta16.flat().data(), v.theta16, v.dense_len * 2);
        if (grads_ready_) get(l.comp.grad16.data(), v.grad16, v.nnz * 2);
        else std::fill(l.comp.grad16.begin(), l.comp.grad16.end(), Half{});
        std::fill(l.comp.grad32.begin(), l.comp.grad32.end(), 0.0f);
      }
      fresh_ = true;
    }
    return state_;
  }
  std::uint64_t skipped_steps() const { return rec_.skipped_steps; }
  float last_grad_norm() const { return rec_.grad_norm; }
  const OptimizerConfig& config() const { return cfg_; }
  Model& model() { return *model_; }

 private:
  void check_layer(std::size_t i) const {
    if (i >= state_.layers.size()) throw IndexError("sink: layer index out of range");
  }
  static void put(void* dev, const void* host, std::size_t bytes) {
    if (bytes) cuda_check(cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice), "H2D");
  }
  static void get(void* host, const void* dev, std::size_t bytes) {
    if (bytes) cuda_check(cudaMemcpy(host, dev, bytes, cudaMemcpyDeviceToHost), "D2H");
  }

  OptimizerConfig cfg_;
  mutable ModelState state_;
  std::unique_ptr<Model> model_;
  std::vector<DeviceBuffer<std::uint16_t>> stage_;  // host-sunk gradients until the step
  StepRecord rec_{};
  bool grads_ready_ = false;
  mutable bool fresh_ = true;
};

}  // namespace samo

// The name this header was first published under.
namespace samo_b200 = samo;
