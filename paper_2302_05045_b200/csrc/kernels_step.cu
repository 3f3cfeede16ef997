// kernels_step.cu — the per-step SAMO kernels for sm_100a.
//
//   K1  gather + unscale + cast + finite flag     (train.hpp:598-611, 619-629)
//   K23 skip check + Adam + downcast + expand     (train.hpp:632-654,
//                                                   320-347; store.hpp:72-87)
//   and the API-parity pieces built from the same machinery: expand<T>
//   (store.hpp:72-87), downcast+expand, compress<T> (store.hpp:58-69),
//   adam_update (train.hpp:332-347), check_state_invariants
//   (store.hpp:171-197).
//
// All of them are HBM-bound byte/elementwise work (no contraction, no tensor
// cores).  The dense side of every layer is cut into fixed tiles of
// `tile_elems` elements; a tile's kept indices are a contiguous range of the
// ascending index arena, so a tile is one contiguous dense block plus one
// contiguous compressed block.  Persistent CTAs (a multiple of the SM count)
// walk the tile table round-robin:
//   K1  streams each dense gradient tile into shared memory with the 1-D TMA
//       (cp.async.bulk + mbarrier ring), gathers the kept halves out of shared
//       memory and writes coalesced fp32;
//   K23 builds each dense theta16 tile in shared memory (zero fill + scatter
//       of the freshly updated weights) and writes it back with one bulk
//       store, double-buffered against the next tile's Adam work.
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace samo_dev {

namespace {

constexpr int kUnroll = 4;

__device__ __forceinline__ bool finite_f32(float x) {
  return (__float_as_uint(x) & 0x7F800000u) != 0x7F800000u;
}

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
// K1: gather + unscale + cast, TMA-staged dense tiles.

template <int STAGES>
__global__ void __launch_bounds__(kThreads)
k1_gather_unscale(const SamoTile* __restrict__ tiles, uint32_t ntiles, uint32_t tile_elems,
                  const SamoLayerDev* __restrict__ layers, const uint32_t* __restrict__ idx,
                  float* __restrict__ g32, float inv_scale, float* flag_slot) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint16_t* stage_base = reinterpret_cast<uint16_t*>(smem_raw);
  __shared__ __align__(8) uint64_t full[STAGES];

  const uint32_t tid = threadIdx.x;
  const uint64_t policy = policy_evict_first();
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](uint32_t t, int s) {
    const SamoTile td = tiles[t];
    const uint16_t* src = layers[td.layer].grad + td.dense_begin;
    const uint32_t bytes = (td.dense_count * 2u) & ~15u;
    if (bytes) {
      mbar_arrive_expect_tx(&full[s], bytes);
      bulk_g2s(stage_base + static_cast<size_t>(s) * tile_elems, src, bytes, &full[s], policy);
    } else {
      mbar_arrive(&full[s]);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      const uint64_t t = blockIdx.x + static_cast<uint64_t>(s) * gridDim.x;
      if (t < ntiles) issue(static_cast<uint32_t>(t), s);
    }
  }

  bool bad = false;
  uint32_t it = 0;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = static_cast<int>(it % STAGES);
    const uint32_t parity = (it / STAGES) & 1u;
    const SamoTile td = tiles[t];
    const uint16_t* grad = layers[td.layer].grad;
    const uint32_t staged = ((td.dense_count * 2u) & ~15u) >> 1;
    const uint16_t* sb = stage_base + static_cast<size_t>(s) * tile_elems;
    mbar_wait(&full[s], parity);

#pragma unroll 1
    for (uint64_t kb = td.k_begin + tid; kb < td.k_end; kb += kUnroll * kThreads) {
      uint32_t iv[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t k = kb + static_cast<uint64_t>(u) * kThreads;
        iv[u] = (k < td.k_end) ? ld_stream_u32(idx + k) : 0u;
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t k = kb + static_cast<uint64_t>(u) * kThreads;
        if (k < td.k_end) {
          const uint32_t off = iv[u] - td.dense_begin;
          const uint16_t h = (off < staged) ? sb[off] : grad[iv[u]];
          const float gk = mul_x86(f16_bits_to_f32(h), inv_scale);
          st_stream_f32(g32 + k, gk);
          bad |= !finite_f32(gk);
        }
      }
    }
    __syncthreads();  // every thread is done reading stage s
    if (tid == 0) {
      const uint64_t tn = t + static_cast<uint64_t>(STAGES) * gridDim.x;
      if (tn < ntiles) {
        fence_proxy_async_smem();
        issue(static_cast<uint32_t>(tn), s);
      }
    }
  }
  if (__syncthreads_or(bad) && tid == 0) atomicAdd(flag_slot, 1.0f);
}

// ---------------------------------------------------------------------------
// K23 and friends: per-tile shared-memory expand.

template <typename OutT>
__device__ __forceinline__ OutT* layer_out(const SamoLayerDev* layers, uint32_t l) {
  return reinterpret_cast<OutT*>(layers[l].theta16);
}

template <int MODE, typename OutT>
__global__ void __launch_bounds__(kThreads) k_expand_tiles(ExpandArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  OutT* buf0 = reinterpret_cast<OutT*>(smem_raw);
  OutT* buf1 = buf0 + a.tile_elems;
  __shared__ float red[kThreads / 32];
  __shared__ int last_cta;

  const uint32_t tid = threadIdx.x;

  // Step scalars (train.hpp:640-642): every CTA derives the advanced
  // beta powers with the same float ops; only the last CTA stores them.
  bool skip = false;
  float b1p = 0.f, b2p = 0.f, bias1 = 1.f, bias2 = 1.f, omb1 = 0.f, omb2 = 0.f, lrwd = 0.f;
  if (MODE == kModeAdam) {
    skip = *reinterpret_cast<volatile float*>(a.flag_slot) != 0.0f;
    b1p = __fmul_rn(a.st->beta1_pow, a.prm.beta1);
    b2p = __fmul_rn(a.st->beta2_pow, a.prm.beta2);
    bias1 = __fsub_rn(1.0f, b1p);
    bias2 = __fsub_rn(1.0f, b2p);
    omb1 = __fsub_rn(1.0f, a.prm.beta1);  // train.hpp:335
    omb2 = __fsub_rn(1.0f, a.prm.beta2);  // train.hpp:336
    lrwd = __fmul_rn(a.prm.lr, a.prm.wd);
  }
  const bool write = !(MODE == kModeAdam && skip);
  float nacc = 0.0f;

  uint32_t it = 0;
  for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++it) {
    const SamoTile td = a.tiles[t];
    OutT* buf = (it & 1u) ? buf1 : buf0;
    const uint32_t bytes = td.dense_count * static_cast<uint32_t>(sizeof(OutT));
    if (write) {
      if (MODE != kModeCheck && tid == 0 && it >= 2) bulk_wait_read<1>();
      __syncthreads();  // buffer free (bulk store of tile it-2 has read it)
      uint4* b4 = reinterpret_cast<uint4*>(buf);
      const uint32_t n16 = (bytes + 15u) >> 4;
      for (uint32_t i = tid; i < n16; i += kThreads) b4[i] = make_uint4(0u, 0u, 0u, 0u);
      __syncthreads();
    }

#pragma unroll 1
    for (uint64_t kb = td.k_begin + tid; kb < td.k_end; kb += kUnroll * kThreads) {
      if (MODE == kModeAdam) {
        float gv[kUnroll], mv[kUnroll], vv[kUnroll], tv[kUnroll];
        uint32_t iv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint64_t k = kb + static_cast<uint64_t>(u) * kThreads;
          if (k < td.k_end) {
            gv[u] = ld_stream_f32(a.g + k);
            if (write) {
              mv[u] = a.m[k];
              vv[u] = a.v[k];
              tv[u] = a.theta[k];
              iv[u] = ld_stream_u32(a.idx + k);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint64_t k = kb + static_cast<uint64_t>(u) * kThreads;
          if (k < td.k_end) {
            const float gk = gv[u];
            nacc = __fadd_rn(nacc, __fmul_rn(gk, gk));
            if (write) {
              // adam_update (train.hpp:338-345), IEEE per op, no contraction.
              const float mk = __fadd_rn(__fmul_rn(a.prm.beta1, mv[u]), __fmul_rn(omb1, gk));
              const float vk =
                  __fadd_rn(__fmul_rn(a.prm.beta2, vv[u]), __fmul_rn(omb2, __fmul_rn(gk, gk)));
              const float mh = __fdiv_rn(mk, bias1);
              const float vh = __fdiv_rn(vk, bias2);
              float tk = __fsub_rn(
                  tv[u], __fmul_rn(a.prm.lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), a.prm.eps))));
              if (a.prm.wd != 0.0f) tk = __fsub_rn(tk, __fmul_rn(lrwd, tk));
              a.m[k] = mk;
              a.v[k] = vk;
              a.theta[k] = tk;
              buf[iv[u] - td.dense_begin] = f32_to_f16_bits(tk);
            }
          }
        }
      } else {
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

    if (write) {
      OutT* dst = layer_out<OutT>(a.layers, td.layer) + td.dense_begin;
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

  if (MODE == kModeAdam) {
    // Deterministic grad-norm: per-CTA partial (fixed tile schedule, fixed
    // tree), combined in CTA order in double by the last CTA.
    float x = nacc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = __fadd_rn(x, __shfl_xor_sync(0xFFFFFFFFu, x, o));
    if ((tid & 31) == 0) red[tid >> 5] = x;
    __syncthreads();
    if (tid == 0) {
      float s = 0.f;
      for (int w = 0; w < kThreads / 32; ++w) s = __fadd_rn(s, red[w]);
      a.norm_partials[blockIdx.x] = s;
      __threadfence();
      const uint32_t ticket = atomicAdd(&a.st->done_ctas, 1u);
      last_cta = (ticket == gridDim.x - 1);
    }
    __syncthreads();
    if (last_cta && tid == 0) {
      __threadfence();
      double acc = 0.0;
      const volatile float* np = a.norm_partials;
      for (uint32_t b = 0; b < gridDim.x; ++b) acc += static_cast<double>(np[b]);
      SamoStepState* st = a.st;
      st->grad_norm = static_cast<float>(sqrt(acc));
      if (skip) {  // train.hpp:632-639
        st->skipped_steps += 1;
        st->last_skipped = 1u;
      } else {     // AdamScalars::advance, train.hpp:325-329
        st->t += 1;
        st->beta1_pow = b1p;
        st->beta2_pow = b2p;
        st->last_skipped = 0u;
      }
      st->done_ctas = 0u;
      *a.flag_slot = 0.0f;  // every CTA has read it; ready for the next gather
      __threadfence();
    }
  }
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

int gather_grid(uint32_t tile_elems) {
  const size_t smem = static_cast<size_t>(kGatherStages) * tile_elems * 2;
  auto fn = k1_gather_unscale<kGatherStages>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  return occupancy_grid(reinterpret_cast<const void*>(fn), kThreads, smem);
}

int launch_gather_unscale(const SamoTile* tiles, uint32_t ntiles, uint32_t tile_elems,
                          const SamoLayerDev* layers, const uint32_t* idx, float* g32,
                          float inv_scale, float* flag_slot, int grid, cudaStream_t s) {
  if (ntiles == 0) return SAMO_OK;
  const size_t smem = static_cast<size_t>(kGatherStages) * tile_elems * 2;
  auto fn = k1_gather_unscale<kGatherStages>;
  SAMO_CUDA_TRY(
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (grid <= 0) grid = gather_grid(tile_elems);
  if (static_cast<uint32_t>(grid) > ntiles) grid = static_cast<int>(ntiles);
  fn<<<grid, kThreads, smem, s>>>(tiles, ntiles, tile_elems, layers, idx, g32, inv_scale, flag_slot);
  SAMO_LAUNCH_CHECK("k1_gather_unscale");
  return SAMO_OK;
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

template int launch_expand<kModeAdam, uint16_t>(const ExpandArgs&, int, cudaStream_t);
template int launch_expand<kModeDowncast, uint16_t>(const ExpandArgs&, int, cudaStream_t);
template int launch_expand<kModeValues, uint16_t>(const ExpandArgs&, int, cudaStream_t);
template int launch_expand<kModeValues, uint32_t>(const ExpandArgs&, int, cudaStream_t);
template int launch_expand<kModeCheck, uint16_t>(const ExpandArgs&, int, cudaStream_t);
template int expand_grid<kModeAdam, uint16_t>(uint32_t);

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
