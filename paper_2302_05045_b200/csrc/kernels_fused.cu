// kernels_fused.cu — the two per-step kernels of the SAMO path (sm_100a).
//
// Data layout (per rank, HBM):
//   dense side : per-layer binary16 gradients (inputs) and theta16 (outputs),
//                cut into tiles of T dense elements (T = tile_elems, 8192 by
//                default); tile t also owns T/32 bitmap words at
//                bitmap[t * T/32] — bit (d & 31) of word (d >> 5) set iff
//                dense element dense_begin + d is kept.  The bitmap is derived
//                once from the reference's ascending u32 index set
//                (PrunedIndexSet, prune.hpp:21-27) and carries the same
//                information in T/8 bytes per tile instead of 4 bytes per kept
//                element.
//   compressed : flat arenas theta32 / adam_m / adam_v / grad (layer
//                segments concatenated in layer order); the kept elements of
//                tile t are the contiguous range [k_begin, k_end).
//
// K1 gather (train.hpp:598-611 sink + 619-629 unscale/finite):
//   TMA ring: each stage = one dense gradient tile + its bitmap (cp.async.bulk,
//   mbarrier complete_tx).  The consumer ranks the set bits with a block
//   exclusive scan, gathers the kept halves out of shared memory into a
//   compacted shared buffer (converted and unscaled when the exchange needs
//   fp32; raw binary16 — the reference's grad16 — otherwise) and writes it
//   with coalesced stores.  Non-finite gradients raise the step's skip flag.
//
// K23 update (train.hpp:632-654, adam_update 332-347, expand store.hpp:72-87):
//   TMA ring over chunks of <= kChunk kept elements: each stage holds the
//   16-byte aligned superset of theta32/m/v/grad for the chunk (+ the tile's
//   bitmap on a tile's first chunk).  Per tile the bitmap is decoded into a
//   u16 list of dense offsets, the dense theta16 tile is built in shared
//   memory (zero fill + scatter of half_rn(theta)) and written back with one
//   bulk store, double-buffered against the next tile.  theta/m/v are written
//   straight from registers with coalesced stores.  The last CTA to finish
//   reduces the per-CTA grad-norm partials in CTA order and advances the
//   device-resident Adam scalars.
//
// Both kernels are persistent (grid = resident CTAs x SMs) and HBM-bound.
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace samo_dev {
namespace {

constexpr int kChunk = 1024;  // kept elements per K23 stage
constexpr int kK1Stages = 3;
constexpr int kK23Stages = 3;

__device__ __forceinline__ bool finite_f32(float x) {
  return (__float_as_uint(x) & 0x7F800000u) != 0x7F800000u;
}

// Block-wide exclusive scan of one uint32 per thread.  `ws` must hold
// kThreads/32 words; callers separate consecutive scans by a __syncthreads.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* ws, uint32_t& total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += y;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t v = lane < kThreads / 32 ? ws[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, v, o);
      if (lane >= static_cast<uint32_t>(o)) v += y;
    }
    if (lane < kThreads / 32) ws[lane] = v;
  }
  __syncthreads();
  total = ws[kThreads / 32 - 1];
  return incl - x + (warp ? ws[warp - 1] : 0u);
}

__device__ __forceinline__ void st_na_f32(float* p, float v) {
  asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_na_u16(uint16_t* p, uint16_t v) {
  asm volatile("st.global.L1::no_allocate.u16 [%0], %1;" ::"l"(p), "h"(v) : "memory");
}

// ---------------------------------------------------------------------------
// Bitmap construction (one CTA per tile, once at finalize).

__global__ void __launch_bounds__(kThreads)
k_build_bitmap(const SamoTile* __restrict__ tiles, uint32_t ntiles, uint32_t tile_elems,
               const uint32_t* __restrict__ idx, uint32_t* __restrict__ bitmap) {
  extern __shared__ uint32_t words[];
  const uint32_t nw = tile_elems / 32;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const SamoTile td = tiles[t];
    for (uint32_t i = threadIdx.x; i < nw; i += kThreads) words[i] = 0u;
    __syncthreads();
    for (uint64_t k = td.k_begin + threadIdx.x; k < td.k_end; k += kThreads) {
      const uint32_t d = idx[k] - td.dense_begin;
      atomicOr(&words[d >> 5], 1u << (d & 31));
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nw; i += kThreads)
      bitmap[static_cast<uint64_t>(t) * nw + i] = words[i];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K1

template <bool OUT_F32>
__global__ void __launch_bounds__(kThreads) k1_gather(StepArgs a) {
  using OutT = typename std::conditional<OUT_F32, float, uint16_t>::type;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kK1Stages];
  __shared__ uint32_t ws[kThreads / 32];

  const uint32_t T = a.tile_elems, NW = T / 32;
  const uint32_t stage_bytes = T * 2 + NW * 4;
  OutT* cbuf = reinterpret_cast<OutT*>(smem + kK1Stages * stage_bytes);
  const uint32_t tid = threadIdx.x;
  const uint64_t policy = policy_evict_first();
  if (tid == 0) {
    for (int s = 0; s < kK1Stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](uint32_t t, int s) {
    const SamoTile td = a.tiles[t];
    uint8_t* st = smem + s * stage_bytes;
    const uint32_t gbytes = (td.dense_count * 2u) & ~15u;
    mbar_arrive_expect_tx(&full[s], gbytes + NW * 4);
    if (gbytes) bulk_g2s(st, a.layers[td.layer].grad + td.dense_begin, gbytes, &full[s], policy);
    bulk_g2s(st + T * 2, a.bitmap + static_cast<uint64_t>(t) * NW, NW * 4, &full[s], policy);
  };
  if (tid == 0) {
    for (int s = 0; s < kK1Stages; ++s) {
      const uint64_t t = blockIdx.x + static_cast<uint64_t>(s) * gridDim.x;
      if (t < a.ntiles) issue(static_cast<uint32_t>(t), s);
    }
  }

  const uint32_t W = (NW + kThreads - 1) / kThreads;  // bitmap words per thread
  bool bad = false;
  uint32_t it = 0;
  for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++it) {
    const int s = static_cast<int>(it % kK1Stages);
    const SamoTile td = a.tiles[t];
    const uint16_t* gsrc = a.layers[td.layer].grad + td.dense_begin;
    const uint32_t staged = ((td.dense_count * 2u) & ~15u) >> 1;
    const uint8_t* st = smem + s * stage_bytes;
    const uint16_t* sg = reinterpret_cast<const uint16_t*>(st);
    const uint32_t* bm = reinterpret_cast<const uint32_t*>(st + T * 2);
    mbar_wait(&full[s], (it / kK1Stages) & 1u);

    const uint32_t w0 = tid * W;
    uint32_t cnt = 0;
    for (uint32_t w = w0; w < w0 + W && w < NW; ++w) cnt += __popc(bm[w]);
    uint32_t total;
    uint32_t pos = block_excl_scan(cnt, ws, total);
    for (uint32_t w = w0; w < w0 + W && w < NW; ++w) {
      uint32_t bits = bm[w];
      while (bits) {
        const uint32_t j = __ffs(bits) - 1;
        bits &= bits - 1;
        const uint32_t d = w * 32 + j;
        const uint16_t h = d < staged ? sg[d] : gsrc[d];
        if constexpr (OUT_F32) {
          const float gk = mul_x86(f16_bits_to_f32(h), a.inv_scale);
          bad |= !finite_f32(gk);
          cbuf[pos++] = gk;
        } else {
          bad |= (h & 0x7C00u) == 0x7C00u;  // |h * 2^-k| is finite iff h is
          cbuf[pos++] = h;
        }
      }
    }
    __syncthreads();  // stage s fully read, cbuf complete
    if (tid == 0) {
      const uint64_t tn = t + static_cast<uint64_t>(kK1Stages) * gridDim.x;
      if (tn < a.ntiles) {
        fence_proxy_async_smem();
        issue(static_cast<uint32_t>(tn), s);
      }
    }
    OutT* dst = reinterpret_cast<OutT*>(a.g) + td.k_begin;
    for (uint32_t i = tid; i < total; i += kThreads) {
      if constexpr (OUT_F32) st_na_f32(dst + i, cbuf[i]);
      else st_na_u16(dst + i, cbuf[i]);
    }
    // the next tile's scan (which begins with a barrier) orders these reads of
    // cbuf before it is overwritten
  }
  if (__syncthreads_or(bad) && tid == 0) atomicAdd(a.flag_slot, 1.0f);
}

// ---------------------------------------------------------------------------
// K23

struct ChunkPlan {
  uint64_t kc0, kc1;  // kept-element range of the chunk
  uint32_t j, nch;    // chunk index within its tile, chunks in the tile
};

__device__ __forceinline__ uint32_t tile_chunks(const SamoTile& td) {
  const uint64_t n = td.k_end - td.k_begin;
  return n == 0 ? 1u : static_cast<uint32_t>((n + kChunk - 1) / kChunk);
}

template <bool G16>
struct K23Layout {
  static constexpr uint32_t kF32 = (kChunk + 8) * 4;                  // theta/m/v/g32 slot
  static constexpr uint32_t kG = G16 ? (kChunk + 16) * 2 : kF32;     // grad slot
};

template <bool G16>
__global__ void __launch_bounds__(kThreads) k23_update(StepArgs a) {
  using L = K23Layout<G16>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kK23Stages];
  __shared__ uint32_t ws[kThreads / 32];
  __shared__ float red[kThreads / 32];
  __shared__ int last_cta;

  const uint32_t T = a.tile_elems, NW = T / 32;
  const uint32_t stage_bytes = 3 * L::kF32 + L::kG + NW * 4;
  uint8_t* lst_raw = smem + kK23Stages * stage_bytes;
  uint16_t* lst = reinterpret_cast<uint16_t*>(lst_raw);               // T entries
  uint16_t* outb = reinterpret_cast<uint16_t*>(lst_raw + T * 2);      // 2 x T halves
  const uint32_t tid = threadIdx.x;

  // Step scalars (train.hpp:640-642), identical float ops in every CTA.
  const bool skip = *reinterpret_cast<volatile float*>(a.flag_slot) != 0.0f;
  const float b1p = __fmul_rn(a.st->beta1_pow, a.prm.beta1);
  const float b2p = __fmul_rn(a.st->beta2_pow, a.prm.beta2);
  const float bias1 = __fsub_rn(1.0f, b1p), bias2 = __fsub_rn(1.0f, b2p);
  const float omb1 = __fsub_rn(1.0f, a.prm.beta1);  // train.hpp:335
  const float omb2 = __fsub_rn(1.0f, a.prm.beta2);  // train.hpp:336
  const float lrwd = __fmul_rn(a.prm.lr, a.prm.wd);

  const uint64_t policy = policy_evict_first();
  if (tid == 0) {
    for (int s = 0; s < kK23Stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // Producer cursor (thread 0 only) — runs kK23Stages chunks ahead.
  uint32_t pt = blockIdx.x, pj = 0;
  auto issue = [&](int s) {
    const SamoTile td = a.tiles[pt];
    const uint64_t kc0 = td.k_begin + static_cast<uint64_t>(pj) * kChunk;
    const uint64_t kc1 = min(td.k_end, kc0 + kChunk);
    uint8_t* st = smem + s * stage_bytes;
    const uint64_t f0 = kc0 & ~3ull, f1 = (kc1 + 3) & ~3ull;
    const uint32_t fb = static_cast<uint32_t>((f1 - f0) * 4);
    uint32_t gb;
    uint64_t g0;
    if (G16) {
      g0 = kc0 & ~7ull;
      gb = static_cast<uint32_t>((((kc1 + 7) & ~7ull) - g0) * 2);
    } else {
      g0 = f0;
      gb = fb;
    }
    const uint32_t bmb = pj == 0 ? NW * 4 : 0u;
    mbar_arrive_expect_tx(&full[s], 3 * fb + gb + bmb);
    if (fb) {
      bulk_g2s(st, a.theta + f0, fb, &full[s], policy);
      bulk_g2s(st + L::kF32, a.m + f0, fb, &full[s], policy);
      bulk_g2s(st + 2 * L::kF32, a.v + f0, fb, &full[s], policy);
    }
    if (gb) {
      const uint8_t* gsrc = reinterpret_cast<const uint8_t*>(a.g) + g0 * (G16 ? 2 : 4);
      bulk_g2s(st + 3 * L::kF32, gsrc, gb, &full[s], policy);
    }
    if (bmb) bulk_g2s(st + 3 * L::kF32 + L::kG, a.bitmap + static_cast<uint64_t>(pt) * NW, bmb,
                      &full[s], policy);
    if (++pj >= tile_chunks(td)) {
      pj = 0;
      pt += gridDim.x;
    }
  };
  if (tid == 0) {
    for (int s = 0; s < kK23Stages && pt < a.ntiles; ++s) issue(s);
  }

  const uint32_t W = (NW + kThreads - 1) / kThreads;
  float nacc = 0.0f;
  uint32_t it = 0, tile_it = 0;
  for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++tile_it) {
    const SamoTile td = a.tiles[t];
    const uint32_t nch = tile_chunks(td);
    uint16_t* out = outb + (tile_it & 1u) * T;
    for (uint32_t j = 0; j < nch; ++j, ++it) {
      const int s = static_cast<int>(it % kK23Stages);
      const uint8_t* st = smem + s * stage_bytes;
      const uint64_t kc0 = td.k_begin + static_cast<uint64_t>(j) * kChunk;
      const uint64_t kc1 = min(td.k_end, kc0 + kChunk);
      mbar_wait(&full[s], (it / kK23Stages) & 1u);

      if (j == 0 && !skip) {
        // New tile: its out buffer was last bulk-stored two tiles ago.
        if (tid == 0 && tile_it >= 2) bulk_wait_read<1>();
        const uint32_t* bm = reinterpret_cast<const uint32_t*>(st + 3 * L::kF32 + L::kG);
        const uint32_t w0 = tid * W;
        uint32_t cnt = 0;
        for (uint32_t w = w0; w < w0 + W && w < NW; ++w) cnt += __popc(bm[w]);
        uint32_t total;
        uint32_t pos = block_excl_scan(cnt, ws, total);  // has barriers: bulk wait visible
        for (uint32_t w = w0; w < w0 + W && w < NW; ++w) {
          uint32_t bits = bm[w];
          while (bits) {
            const uint32_t b = __ffs(bits) - 1;
            bits &= bits - 1;
            lst[pos++] = static_cast<uint16_t>(w * 32 + b);
          }
        }
        uint4* o4 = reinterpret_cast<uint4*>(out);
        const uint32_t n16 = (td.dense_count * 2u + 15u) >> 4;
        for (uint32_t i = tid; i < n16; i += kThreads) o4[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
      }

      const float* sth = reinterpret_cast<const float*>(st);
      const float* smv = reinterpret_cast<const float*>(st + L::kF32);
      const float* svv = reinterpret_cast<const float*>(st + 2 * L::kF32);
      const uint64_t f0 = kc0 & ~3ull;
      const uint64_t g0 = G16 ? (kc0 & ~7ull) : f0;
      for (uint64_t k = kc0 + tid; k < kc1; k += kThreads) {
        const uint32_t i = static_cast<uint32_t>(k - f0);
        const uint32_t ig = static_cast<uint32_t>(k - g0);
        float gk;
        if constexpr (G16) {
          const uint16_t h = reinterpret_cast<const uint16_t*>(st + 3 * L::kF32)[ig];
          gk = mul_x86(f16_bits_to_f32(h), a.inv_scale);
        } else {
          gk = reinterpret_cast<const float*>(st + 3 * L::kF32)[ig];
        }
        nacc = __fadd_rn(nacc, __fmul_rn(gk, gk));
        if (!skip) {
          // adam_update (train.hpp:338-345): IEEE per op, no contraction.
          const float mk = __fadd_rn(__fmul_rn(a.prm.beta1, smv[i]), __fmul_rn(omb1, gk));
          const float vk =
              __fadd_rn(__fmul_rn(a.prm.beta2, svv[i]), __fmul_rn(omb2, __fmul_rn(gk, gk)));
          const float mh = __fdiv_rn(mk, bias1);
          const float vh = __fdiv_rn(vk, bias2);
          float tk = __fsub_rn(
              sth[i], __fmul_rn(a.prm.lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), a.prm.eps))));
          if (a.prm.wd != 0.0f) tk = __fsub_rn(tk, __fmul_rn(lrwd, tk));
          st_na_f32(a.m + k, mk);
          st_na_f32(a.v + k, vk);
          st_na_f32(a.theta + k, tk);
          out[lst[k - td.k_begin]] = f32_to_f16_bits(tk);
        }
      }
      const bool last = (j + 1 == nch);
      if (last && !skip) fence_proxy_async_smem();
      __syncthreads();  // stage s consumed; on the last chunk the tile is complete
      if (tid == 0) {
        if (pt < a.ntiles) {
          fence_proxy_async_smem();
          issue(s);
        }
        if (last && !skip) {
          const uint32_t bytes = td.dense_count * 2u;
          const uint32_t bulk = bytes & ~15u;
          uint16_t* dst = a.layers[td.layer].theta16 + td.dense_begin;
          if (bulk) bulk_s2g(dst, out, bulk);
          bulk_commit();
          for (uint32_t i = bulk / 2; i < td.dense_count; ++i) dst[i] = out[i];
        }
      }
    }
  }
  if (tid == 0) bulk_wait<0>();

  // Grad norm partial per CTA (fixed schedule -> deterministic), finalised by
  // the last CTA in CTA order (double).
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
    SamoStepState* stt = a.st;
    stt->grad_norm = static_cast<float>(sqrt(acc));
    if (skip) {  // train.hpp:632-639
      stt->skipped_steps += 1;
      stt->last_skipped = 1u;
    } else {     // AdamScalars::advance, train.hpp:325-329
      stt->t += 1;
      stt->beta1_pow = b1p;
      stt->beta2_pow = b2p;
      stt->last_skipped = 0u;
    }
    stt->done_ctas = 0u;
    *a.flag_slot = 0.0f;  // every CTA has read it; ready for the next gather
    __threadfence();
  }
}

template <typename F>
int grid_for(F fn, size_t smem) {
  SAMO_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const char* env = getenv("SAMO_CTAS_PER_SM");  // tuning override
  if (env && *env && atoi(env) > 0 && atoi(env) < per_sm) per_sm = atoi(env);
  return per_sm * num_sms();
}

}  // namespace

size_t gather_smem(uint32_t tile_elems, bool f32) {
  return kK1Stages * (tile_elems * 2u + tile_elems / 8u) + tile_elems * (f32 ? 4u : 2u);
}

size_t update_smem(uint32_t tile_elems, bool g16) {
  const uint32_t fs = (kChunk + 8) * 4, gs = g16 ? (kChunk + 16) * 2 : fs;
  return kK23Stages * (3 * fs + gs + tile_elems / 8u) + tile_elems * 2u /*lst*/ +
         tile_elems * 4u /*2 out tiles*/;
}

int step_grid(int which, bool wide, uint32_t tile_elems) {
  if (which == 0) {
    const size_t sm = gather_smem(tile_elems, wide);
    return wide ? grid_for(k1_gather<true>, sm) : grid_for(k1_gather<false>, sm);
  }
  const size_t sm = update_smem(tile_elems, !wide);
  return wide ? grid_for(k23_update<false>, sm) : grid_for(k23_update<true>, sm);
}

int launch_gather(const StepArgs& a, bool out_f32, int grid, cudaStream_t s) {
  if (a.ntiles == 0) return SAMO_OK;
  const size_t sm = gather_smem(a.tile_elems, out_f32);
  if (grid <= 0) grid = step_grid(0, out_f32, a.tile_elems);
  if (static_cast<uint32_t>(grid) > a.ntiles) grid = static_cast<int>(a.ntiles);
  if (out_f32) {
    SAMO_CUDA_TRY(cudaFuncSetAttribute(k1_gather<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sm)));
    k1_gather<true><<<grid, kThreads, sm, s>>>(a);
  } else {
    SAMO_CUDA_TRY(cudaFuncSetAttribute(k1_gather<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sm)));
    k1_gather<false><<<grid, kThreads, sm, s>>>(a);
  }
  SAMO_LAUNCH_CHECK("k1_gather");
  return SAMO_OK;
}

int launch_update(const StepArgs& a, bool g_f32, int grid, cudaStream_t s) {
  if (a.ntiles == 0) return SAMO_OK;
  const size_t sm = update_smem(a.tile_elems, !g_f32);
  if (grid <= 0) grid = step_grid(1, g_f32, a.tile_elems);
  if (static_cast<uint32_t>(grid) > a.ntiles) grid = static_cast<int>(a.ntiles);
  if (g_f32) {
    SAMO_CUDA_TRY(cudaFuncSetAttribute(k23_update<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    k23_update<false><<<grid, kThreads, sm, s>>>(a);
  } else {
    SAMO_CUDA_TRY(cudaFuncSetAttribute(k23_update<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    k23_update<true><<<grid, kThreads, sm, s>>>(a);
  }
  SAMO_LAUNCH_CHECK("k23_update");
  return SAMO_OK;
}

int launch_build_bitmap(const SamoTile* tiles, uint32_t ntiles, uint32_t tile_elems,
                        const uint32_t* idx, uint32_t* bitmap, cudaStream_t s) {
  if (ntiles == 0) return SAMO_OK;
  const int grid = static_cast<int>(ntiles < 4096u ? ntiles : 4096u);
  k_build_bitmap<<<grid, kThreads, tile_elems / 8, s>>>(tiles, ntiles, tile_elems, idx, bitmap);
  SAMO_LAUNCH_CHECK("k_build_bitmap");
  return SAMO_OK;
}

}  // namespace samo_dev
