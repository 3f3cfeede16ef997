// kernels_step.cu — the API-parity kernels of the SAMO path (sm_100a):
// expand<T> (store.hpp:72-87), downcast+expand (train.hpp:647-651),
// compress<T> (store.hpp:58-69), adam_update (train.hpp:332-347),
// check_state_invariants (store.hpp:171-197), binary16 conversions
// (half.hpp:13-71), the tile-table builder and the synthetic-data generator.
//
// The expand family shares the dense-tile machinery of the step: a tile's
// kept indices are a contiguous range of the ascending index arena; each CTA
// zero-fills the dense tile in shared memory, scatters the kept values into
// it and writes it back with one cp.async.bulk store, double-buffered against
// the next tile.  The per-step kernels (K1 gather, K23 update) are in
// kernels_fused.cu.
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace samo_dev {

namespace {

constexpr int kUnroll = 4;

// ---------------------------------------------------------------------------
// Tile table: k range of each tile by binary search (lower_bound).

__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t* a, uint64_t n, uint32_t key) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_tiles_fill(SamoTile* tiles, uint32_t ntiles, const uint64_t* __restrict__ k_off,
                             const uint32_t* __restrict__ idx) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  SamoTile td = tiles[t];
  const uint64_t kb = k_off[td.layer], ke = k_off[td.layer + 1];
  const uint32_t* seg = idx + kb;
  const uint64_t n = ke - kb;
  td.k_begin = kb + lower_bound_u32(seg, n, td.dense_begin);
  const uint64_t end = static_cast<uint64_t>(td.dense_begin) + td.dense_count;
  td.k_end = (end >= 0xFFFFFFFFull + 1) ? ke : kb + lower_bound_u32(seg, n, static_cast<uint32_t>(end));
  tiles[t] = td;
}

// ---------------------------------------------------------------------------
// Tile expand kernels: per-tile shared-memory expand (downcast / values /
// invariant check).  The per-step update kernel lives in kernels_fused.cu.

template <int MODE, typename OutT>
__global__ void __launch_bounds__(kThreads) k_expand_tiles(ExpandArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  OutT* buf0 = reinterpret_cast<OutT*>(smem_raw);
  OutT* buf1 = buf0 + a.tile_elems;

  const uint32_t tid = threadIdx.x;
  uint32_t it = 0;
  for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++it) {
    const SamoTile td = a.tiles[t];
    OutT* buf = (it & 1u) ? buf1 : buf0;
    const uint32_t bytes = td.dense_count * static_cast<uint32_t>(sizeof(OutT));
    {
      if (MODE != kModeCheck && tid == 0 && it >= 2) bulk_wait_read<1>();
      __syncthreads();  // buffer free (bulk store of tile it-2 has read it)
      uint4* b4 = reinterpret_cast<uint4*>(buf);
      const uint32_t n16 = (bytes + 15u) >> 4;
      for (uint32_t i = tid; i < n16; i += kThreads) b4[i] = make_uint4(0u, 0u, 0u, 0u);
      __syncthreads();
    }

#pragma unroll 1
    for (uint64_t kb = td.k_begin + tid; kb < td.k_end; kb += kUnroll * kThreads) {
      {
        OutT val[kUnroll];
        uint32_t iv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint64_t k = kb + static_cast<uint64_t>(u) * kThreads;
          if (k < td.k_end) {
            iv[u] = ld_stream_u32(a.idx + k);
            if (MODE == kModeValues) {
              val[u] = reinterpret_cast<const OutT*>(a.values)[k];
            } else {
              val[u] = static_cast<OutT>(f32_to_f16_bits(a.theta[k]));
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint64_t k = kb + static_cast<uint64_t>(u) * kThreads;
          if (k < td.k_end) buf[iv[u] - td.dense_begin] = val[u];
        }
      }
    }

    {
      OutT* dst = reinterpret_cast<OutT*>(a.out_base) + td.out_off;
      if (MODE == kModeCheck) {
        __syncthreads();
        bool bad = false;
        for (uint32_t i = tid; i < td.dense_count; i += kThreads) bad |= (dst[i] != buf[i]);
        if (__syncthreads_or(bad) && tid == 0) atomicOr(a.mismatch, 1u);
      } else {
        fence_proxy_async_smem();
        __syncthreads();
        const uint32_t bulk_bytes = a.use_bulk ? (bytes & ~15u) : 0u;
        if (tid == 0) {
          if (bulk_bytes) bulk_s2g(dst, buf, bulk_bytes);
          bulk_commit();  // always one group per tile: keeps wait_read<1> exact
        }
        for (uint32_t i = bulk_bytes / sizeof(OutT) + tid; i < td.dense_count; i += kThreads)
          dst[i] = buf[i];
      }
    }
  }
  if (MODE != kModeCheck && tid == 0) bulk_wait<0>();
}

// ---------------------------------------------------------------------------
// Plain kernels.

template <typename T>
__global__ void __launch_bounds__(kThreads)
k_compress(const T* __restrict__ dense, const uint32_t* __restrict__ idx, uint64_t n,
           T* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t kb = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; kb < n;
       kb += kUnroll * stride) {
    uint32_t iv[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t k = kb + u * stride;
      iv[u] = k < n ? ld_stream_u32(idx + k) : 0u;
    }
    T vals[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t k = kb + u * stride;
      if (k < n) vals[u] = dense[iv[u]];
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t k = kb + u * stride;
      if (k < n) out[k] = vals[u];
    }
  }
}

__global__ void __launch_bounds__(kThreads)
k_adam(float* __restrict__ theta, float* __restrict__ m, float* __restrict__ v,
       const float* __restrict__ g, uint64_t n, SamoAdamParams prm, float bias1, float bias2) {
  const float omb1 = __fsub_rn(1.0f, prm.beta1), omb2 = __fsub_rn(1.0f, prm.beta2);
  const float lrwd = __fmul_rn(prm.lr, prm.wd);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; k < n; k += stride) {
    const float gk = g[k];
    const float mk = __fadd_rn(__fmul_rn(prm.beta1, m[k]), __fmul_rn(omb1, gk));
    const float vk = __fadd_rn(__fmul_rn(prm.beta2, v[k]), __fmul_rn(omb2, __fmul_rn(gk, gk)));
    const float mh = __fdiv_rn(mk, bias1);
    const float vh = __fdiv_rn(vk, bias2);
    float tk = __fsub_rn(theta[k],
                         __fmul_rn(prm.lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), prm.eps))));
    if (prm.wd != 0.0f) tk = __fsub_rn(tk, __fmul_rn(lrwd, tk));
    m[k] = mk;
    v[k] = vk;
    theta[k] = tk;
  }
}

__global__ void k_f2h(const float* __restrict__ in, uint16_t* __restrict__ out, uint64_t n) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    out[i] = f32_to_f16_bits(in[i]);
}

__global__ void k_h2f(const uint16_t* __restrict__ in, float* __restrict__ out, uint64_t n) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    out[i] = f16_bits_to_f32(in[i]);
}

__device__ __forceinline__ float synth_value(uint64_t seed, uint64_t sid, uint64_t i, float bound) {
  const uint64_t u = synth_mix64(seed, sid, i);
  const float c = __fmul_rn(static_cast<float>(u >> 40), 0x1.0p-24f);  // canonical_float
  return __fmul_rn(__fsub_rn(__fmul_rn(2.0f, c), 1.0f), bound);        // uniform_symmetric
}

__global__ void k_synth_f32(float* __restrict__ out, uint64_t n, uint64_t seed, uint64_t sid,
                            float bound) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    out[i] = synth_value(seed, sid, i, bound);
}

__global__ void k_synth_f16(uint16_t* __restrict__ out, uint64_t n, uint64_t seed, uint64_t sid,
                            float bound, float scale) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    out[i] = f32_to_f16_bits(__fmul_rn(synth_value(seed, sid, i, bound), scale));
}

__global__ void k_check_indices(const uint32_t* __restrict__ idx, uint64_t n, uint64_t dense_len,
                                uint32_t* bad) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  bool b = false;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const uint32_t x = idx[i];
    b |= (x >= dense_len);
    if (i + 1 < n) b |= (idx[i + 1] <= x);
  }
  if (b) atomicOr(bad, 1u);
}

int elementwise_grid(uint64_t n, int threads) {
  const uint64_t want = (n + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(num_sms()) * 16;
  return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

// ---------------------------------------------------------------------------
// Launchers.

int launch_tiles_fill(SamoTile* tiles, uint32_t ntiles, const uint64_t* k_off,
                      const uint32_t* idx, cudaStream_t s) {
  if (ntiles == 0) return SAMO_OK;
  k_tiles_fill<<<(ntiles + 255) / 256, 256, 0, s>>>(tiles, ntiles, k_off, idx);
  SAMO_LAUNCH_CHECK("k_tiles_fill");
  return SAMO_OK;
}

static int occupancy_grid(const void* fn, int threads, size_t smem) {
  const char* env = getenv("SAMO_CARVEOUT");  // tuning override (percent shared)
  if (env && *env)
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(env));
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  if (const char* env = getenv("SAMO_CTAS_PER_SM")) {  // tuning override
    const int want = atoi(env);
    if (want > 0 && want < per_sm) per_sm = want;
  }
  return per_sm * num_sms();
}

template <int MODE, typename OutT>
int expand_grid(uint32_t tile_elems) {
  const size_t smem = 2ull * tile_elems * sizeof(OutT);
  auto fn = k_expand_tiles<MODE, OutT>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  return occupancy_grid(reinterpret_cast<const void*>(fn), kThreads, smem);
}

template <int MODE, typename OutT>
int launch_expand(const ExpandArgs& a, int grid, cudaStream_t s) {
  if (a.ntiles == 0) return SAMO_OK;
  const size_t smem = 2ull * a.tile_elems * sizeof(OutT);
  auto fn = k_expand_tiles<MODE, OutT>;
  SAMO_CUDA_TRY(
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (grid <= 0) grid = expand_grid<MODE, OutT>(a.tile_elems);
  if (static_cast<uint32_t>(grid) > a.ntiles) grid = static_cast<int>(a.ntiles);
  fn<<<grid, kThreads, smem, s>>>(a);
  SAMO_LAUNCH_CHECK("k_expand_tiles");
  return SAMO_OK;
}

template int launch_expand<kModeDowncast, uint16_t>(const ExpandArgs&, int, cudaStream_t);
template int launch_expand<kModeValues, uint16_t>(const ExpandArgs&, int, cudaStream_t);
template int launch_expand<kModeValues, uint32_t>(const ExpandArgs&, int, cudaStream_t);
template int launch_expand<kModeCheck, uint16_t>(const ExpandArgs&, int, cudaStream_t);

template <typename T>
int launch_compress(const T* dense, const uint32_t* idx, uint64_t n, T* out, cudaStream_t s) {
  if (n == 0) return SAMO_OK;
  const int grid = elementwise_grid((n + kUnroll - 1) / kUnroll, kThreads);
  k_compress<T><<<grid, kThreads, 0, s>>>(dense, idx, n, out);
  SAMO_LAUNCH_CHECK("k_compress");
  return SAMO_OK;
}
template int launch_compress<uint16_t>(const uint16_t*, const uint32_t*, uint64_t, uint16_t*,
                                       cudaStream_t);
template int launch_compress<uint32_t>(const uint32_t*, const uint32_t*, uint64_t, uint32_t*,
                                       cudaStream_t);

int launch_adam(float* theta, float* m, float* v, const float* g, uint64_t n, SamoAdamParams prm,
                float bias1, float bias2, cudaStream_t s) {
  if (n == 0) return SAMO_OK;
  k_adam<<<elementwise_grid(n, kThreads), kThreads, 0, s>>>(theta, m, v, g, n, prm, bias1, bias2);
  SAMO_LAUNCH_CHECK("k_adam");
  return SAMO_OK;
}

int launch_f2h(const float* in, uint16_t* out, uint64_t n, cudaStream_t s) {
  if (n == 0) return SAMO_OK;
  k_f2h<<<elementwise_grid(n, 256), 256, 0, s>>>(in, out, n);
  SAMO_LAUNCH_CHECK("k_f2h");
  return SAMO_OK;
}

int launch_h2f(const uint16_t* in, float* out, uint64_t n, cudaStream_t s) {
  if (n == 0) return SAMO_OK;
  k_h2f<<<elementwise_grid(n, 256), 256, 0, s>>>(in, out, n);
  SAMO_LAUNCH_CHECK("k_h2f");
  return SAMO_OK;
}

int launch_synth_f32(float* out, uint64_t n, uint64_t seed, uint64_t sid, float bound,
                     cudaStream_t s) {
  if (n == 0) return SAMO_OK;
  k_synth_f32<<<elementwise_grid(n, 256), 256, 0, s>>>(out, n, seed, sid, bound);
  SAMO_LAUNCH_CHECK("k_synth_f32");
  return SAMO_OK;
}

int launch_synth_f16(uint16_t* out, uint64_t n, uint64_t seed, uint64_t sid, float bound,
                     float scale, cudaStream_t s) {
  if (n == 0) return SAMO_OK;
  k_synth_f16<<<elementwise_grid(n, 256), 256, 0, s>>>(out, n, seed, sid, bound, scale);
  SAMO_LAUNCH_CHECK("k_synth_f16");
  return SAMO_OK;
}

int launch_check_indices(const uint32_t* idx, uint64_t n, uint64_t dense_len, uint32_t* bad,
                         cudaStream_t s) {
  if (n == 0) return SAMO_OK;
  k_check_indices<<<elementwise_grid(n, 256), 256, 0, s>>>(idx, n, dense_len, bad);
  SAMO_LAUNCH_CHECK("k_check_indices");
  return SAMO_OK;
}

}  // namespace samo_dev
