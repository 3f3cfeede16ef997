// common.cuh — shared device helpers for the SAMO sm_100a kernels.
//
// PTX wrappers for the Blackwell async-copy path (mbarrier + cp.async.bulk,
// the 1-D TMA), IEEE binary16 conversions that reproduce the reference's
// software rounding bit for bit (half.hpp:13-71), and the status plumbing of
// the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <cstdio>

#include "samo_cuda_testing.h"

namespace samo_dev {

// ---------------------------------------------------------------------------
// Host-side status plumbing.

void set_error(const char* fmt, ...);
void clear_error();
int fail(int status, const char* fmt, ...);
int cuda_fail(cudaError_t err, const char* what);
void note_launch(uint64_t n = 1);
void unnote_launch(uint64_t n);  // captured into a graph, not launched
int device_ok();  // SAMO_OK when a CUDA device is usable, else SAMO_E_CUDA

#define SAMO_CUDA_TRY(expr)                                   \
  do {                                                        \
    cudaError_t e_ = (expr);                                  \
    if (e_ != cudaSuccess) return ::samo_dev::cuda_fail(e_, #expr); \
  } while (0)

#define SAMO_TRY(expr)              \
  do {                              \
    int rc_ = (expr);               \
    if (rc_ != SAMO_OK) return rc_; \
  } while (0)

#define SAMO_LAUNCH_CHECK(what)                                       \
  do {                                                                \
    cudaError_t e_ = cudaGetLastError();                              \
    if (e_ != cudaSuccess) return ::samo_dev::cuda_fail(e_, what);    \
    ::samo_dev::note_launch();                                        \
  } while (0)

inline cudaStream_t as_stream(samo_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms();

// ---------------------------------------------------------------------------
// Device: PTX wrappers.

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// Checked builds (python -m paper_2302_05045_b200.build --checked ->
// libsamo_cuda_checked.so, loaded with SAMO_LIB): device-side bounds checks
// on shared-memory and arena indices, and mbarrier waits that trap instead of
// hanging.  The stand-in for compute-sanitizer, which this pool does not run.
#ifdef SAMO_CHECKED
#define SAMO_DCHECK(cond)                                                               \
  do {                                                                                  \
    if (!(cond)) {                                                                      \
      printf("SAMO_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,  \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x), #cond);        \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#else
#define SAMO_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

#ifdef SAMO_CHECKED
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (uint64_t spin = 0;; ++spin) {
    uint32_t done;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    if (done) return;
    SAMO_DCHECK(spin < (1ull << 28));  // a lost arrival: fail instead of hanging
  }
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "SAMO_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra SAMO_WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
#endif

// 1-D bulk copy global -> shared, completion signalled on `bar` (UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

// 1-D bulk copy shared -> global, tracked by the bulk async-group.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Orders this thread's generic-proxy shared-memory writes before later
// async-proxy (bulk copy) accesses.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Cross-GPU signalling over NVLink peer memory (system scope).
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Streaming loads / stores (read-once data: do not keep in L1).
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream_f32(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint16_t ld_stream_u16(const uint16_t* p) {
  uint16_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream_f32(float* p, float v) {
  asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// Opaque register copies of kernel parameters.  ptxas otherwise re-reads hot
// parameters from the constant bank (LDC) inside loops when it trims register
// use, which put LDC latency into the Adam dependency chains (measured: +15%
// on the update kernel).
__device__ __forceinline__ float pin_f32(float x) {
  float r;
  asm volatile("mov.b32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ uint32_t pin_u32(uint32_t x) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
template <typename T>
__device__ __forceinline__ T* pin_ptr(T* p) {
  uint64_t r;
  asm volatile("mov.b64 %0, %1;" : "=l"(r) : "l"(reinterpret_cast<uint64_t>(p)));
  return reinterpret_cast<T*>(r);
}

// ---------------------------------------------------------------------------
// binary16 conversions, bit-exact with half.hpp.

// float_to_half_bits (half.hpp:13-49).  Hardware cvt.rn.f16.f32 is IEEE RNE
// with the same overflow/underflow behaviour for every non-NaN input; NaNs
// keep sign and top payload bits with the quiet bit forced (half.hpp:18-24).
__device__ __forceinline__ uint16_t f32_to_f16_bits(float x) {
  uint16_t h = __half_as_ushort(__float2half_rn(x));
  const uint32_t w = __float_as_uint(x);
  const uint32_t a = w & 0x7FFFFFFFu;
  if (a > 0x7F800000u) {
    h = static_cast<uint16_t>(((w >> 16) & 0x8000u) | 0x7C00u | 0x0200u | ((a >> 13) & 0x03FFu));
  }
  return h;
}

// Two at once (one cvt.rn.f16x2.f32): lo -> bits 0-15, hi -> bits 16-31;
// NaN inputs (rare) take the exact path above.
__device__ __forceinline__ uint32_t f32x2_to_f16x2_bits(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  if ((__float_as_uint(lo) & 0x7FFFFFFFu) > 0x7F800000u || (__float_as_uint(hi) & 0x7FFFFFFFu) > 0x7F800000u)
    r = static_cast<uint32_t>(f32_to_f16_bits(lo)) | (static_cast<uint32_t>(f32_to_f16_bits(hi)) << 16);
  return r;
}

// half_bits_to_float (half.hpp:52-71): exact widening; NaNs keep their
// payload (signalling NaNs stay signalling).
__device__ __forceinline__ float f16_bits_to_f32(uint16_t h) {
  float f = __half2float(__ushort_as_half(h));
  if ((h & 0x7C00u) == 0x7C00u && (h & 0x03FFu) != 0u) {
    f = __uint_as_float((static_cast<uint32_t>(h & 0x8000u) << 16) | 0x7F800000u |
                        (static_cast<uint32_t>(h & 0x03FFu) << 13));
  }
  return f;
}

// Dense gradient element of either 16-bit type: binary16 (the reference's
// Half, half_bits_to_float above) or bfloat16 (north_star's other gradient
// type; bf16 -> binary32 widening is exact: the bits shifted up by 16).
__device__ __forceinline__ float grad_to_f32(uint32_t h, bool bf16) {
  return bf16 ? __uint_as_float(h << 16) : f16_bits_to_f32(static_cast<uint16_t>(h));
}
// The same for a value only a finite step consumes (K23 / K123: a non-finite
// gradient skips the step, train.hpp:632-639, so its NaN payload is never
// observed): the plain conversion, exact for every finite input.
__device__ __forceinline__ float grad_to_f32_finite(uint32_t h, bool bf16) {
  return bf16 ? __uint_as_float(h << 16) : __half2float(__ushort_as_half(static_cast<uint16_t>(h)));
}
// Exponent field of the 16-bit gradient type: all ones <=> inf or NaN.
__device__ __forceinline__ uint32_t grad_exp_mask(bool bf16) { return bf16 ? 0x7F80u : 0x7C00u; }

// x86 SSE `mulss` semantics for one multiply whose second operand is a
// non-NaN number: a NaN first operand is returned quieted (payload kept).
__device__ __forceinline__ float mul_x86(float a, float b) {
  const uint32_t w = __float_as_uint(a);
  if ((w & 0x7FFFFFFFu) > 0x7F800000u) return __uint_as_float(w | 0x00400000u);
  return __fmul_rn(a, b);
}

// ---------------------------------------------------------------------------
// Counter-based synthetic data (bench inputs).  Mirrored in oracle/samo_oracle.c.
__host__ __device__ __forceinline__ uint64_t synth_mix64(uint64_t seed, uint64_t stream,
                                                         uint64_t i) {
  uint64_t x = i + stream * 0xD1B54A32D192ED03ull + seed * 0x9E3779B97F4A7C15ull;
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

}  // namespace samo_dev

// ---------------------------------------------------------------------------
// Shared tables (host + device view).

// One dense tile of one layer: dense elements [dense_begin, dense_begin +
// dense_count) of layer `layer`, whose kept indices occupy the compressed
// arena range [k_begin, k_end).  out_off is the element offset of the tile's
// first dense element in the output (theta16) buffer the kernels write.
struct SamoTile {
  uint32_t layer;
  uint32_t dense_begin;
  uint32_t dense_count;
  uint32_t pad_;
  uint64_t k_begin;
  uint64_t k_end;
  uint64_t out_off;
  uint64_t pad2_;
};
static_assert(sizeof(SamoTile) == 48, "tile descriptor is 48 bytes");

struct SamoLayerDev {
  const uint16_t* grad;  // dense binary16 gradient of the current step
  uint16_t* theta16;     // dense binary16 weights (output of expand)
  uint64_t dense_len;
  uint64_t k_off;        // offset of the layer in the compressed arenas
};

// Device-resident step scalars (AdamScalars, train.hpp:320-330, plus the
// trainer's counters).  Written only by the last CTA of the update kernel.
struct SamoStepState {
  uint64_t t;
  uint64_t skipped_steps;
  float beta1_pow;
  float beta2_pow;
  float grad_norm;
  uint32_t last_skipped;
  uint32_t done_ctas;  // arrival counter for the last-CTA finalisation
  uint32_t tile_next;  // K123's dynamic tile claims (rewound by its last CTA)
};

struct SamoAdamParams {
  float lr, beta1, beta2, eps, wd;
};

// The optimizer scalars of a model step in device memory, written by a
// one-thread kernel on the step's stream whenever samo_model_set_config
// changed them — so a captured CUDA graph keeps working under a learning-rate
// schedule.  Kernels read this when their `cfg` pointer is set, else their
// by-value arguments.
struct SamoStepConfig {
  SamoAdamParams prm;
  float inv_scale;   // K1 fp32 output / K23 binary16 input: 1/loss_scale (x 1/G for fp32 exchanges)
  float p2p_scale;   // (1/loss_scale) * (1/G), the P2P shard kernels
  float pad_;
};
