// kernels_fused.cu — the per-step kernels of the SAMO path (sm_100a).
//
// Data layout (per rank, HBM):
//   dense side : per-layer binary16 gradients (inputs) and theta16 (outputs),
//                cut into tiles of T dense elements (T = tile_elems, 16384 by
//                default, <= 65536).
//   compressed : flat arenas theta32 / adam_m / adam_v / grad and the tile-
//                local index arena off16 (layer segments concatenated in layer
//                order).  The kept elements of tile t are the contiguous range
//                [k_begin, k_end); off16[k] = idx[k] - dense_begin is the
//                reference index (PrunedIndexSet, prune.hpp:21-27) relative to
//                its tile — derived once, 2 bytes per kept element instead of
//                the 4 of the u32 index set, and directly usable as a shared-
//                memory offset by both kernels.
//
// K1 gather (train.hpp:598-611 sink + 619-629 unscale/finite):
//   TMA ring of dense gradient tiles (cp.async.bulk + mbarrier complete_tx);
//   kept elements gathered out of shared memory through off16, 8 per thread,
//   written with 16/32-byte stores — unscaled fp32 for the NCCL exchanges,
//   the raw compressed binary16 (the reference's grad16) otherwise, or, in
//   the peer-to-peer step's push mode, straight into the owner rank's receive
//   buffer over NVLink.  Non-finite gradients raise the step's skip flag.
//
// K23 update (train.hpp:632-654, adam_update 332-347, expand store.hpp:72-87):
//   warp-specialised: one producer warp streams the 16-byte aligned supersets
//   of theta32/m/v/grad/off16 per <= 1024-element chunk through a TMA ring
//   (full/empty mbarriers); eight consumer warps run the IEEE Adam from
//   shared memory, write theta/m/v from registers, scatter half_rn(theta)
//   into a dense tile in shared memory and copy it out with 128-bit stores
//   that also clear it (one named barrier per tile).  The last CTA reduces
//   the per-CTA grad-norm partials (fixed order) and advances the device
//   Adam scalars.  EXPAND = true is the expand-only pass of the data-
//   parallel steps (binary16 weights in, no Adam).
//
// Data-parallel pieces: k_adam_shard (NCCL sharded exchange), k_shard_p2p
// (fused peer-to-peer exchange: rank-ordered sum of the G
// contributions, Adam, binary16 weights stored to every rank, bucket
// signals), the peer-signal kernels (flag exchange, bucket wait, epoch) and
// k_step_finalize.
//
// The step kernels are persistent (grid = resident CTAs x SMs) and HBM-bound.
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace samo_dev {
namespace {

constexpr int kU = 4;         // independent elements per thread and pass (ILP)
#ifndef SAMO_P2P_GRID
#define SAMO_P2P_GRID 8  // CTAs per SM launched for k_shard_p2p (tuning)
#endif

__device__ __forceinline__ bool finite_f32(float x) {
  return (__float_as_uint(x) & 0x7F800000u) != 0x7F800000u;
}

__device__ __forceinline__ void st_na_f32(float* p, float v) {
  asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_na_u16(uint16_t* p, uint16_t v) {
  asm volatile("st.global.L1::no_allocate.u16 [%0], %1;" ::"l"(p), "h"(v) : "memory");
}
__device__ __forceinline__ void st_na_v4f(float* p, float a, float b, float c, float d) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ void st_na_v4u(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b),
               "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ uint4 ld_stream_v4(const uint16_t* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// The step scalars: from the device copy when `cfg` is set, else the by-value
// kernel arguments.  Field-wise, so no struct address is ever selected (that
// forced a local-memory copy of the arguments and cost K23 3%).
__device__ __forceinline__ SamoAdamParams step_prm(const SamoStepConfig* cfg, const SamoAdamParams& arg) {
  SamoAdamParams p = arg;
  if (cfg) {
    p.lr = cfg->prm.lr;
    p.beta1 = cfg->prm.beta1;
    p.beta2 = cfg->prm.beta2;
    p.eps = cfg->prm.eps;
    p.wd = cfg->prm.wd;
  }
  return p;
}

// ---------------------------------------------------------------------------
// off16 construction (once, at finalize).

__global__ void __launch_bounds__(kThreads)
k_build_off16(const SamoTile* __restrict__ tiles, uint32_t ntiles, const uint32_t* __restrict__ idx,
              uint16_t* __restrict__ off16) {
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const SamoTile td = tiles[t];
    for (uint64_t k = td.k_begin + threadIdx.x; k < td.k_end; k += kThreads)
      off16[k] = static_cast<uint16_t>(idx[k] - td.dense_begin);
  }
}

// ---------------------------------------------------------------------------
// K1

template <bool OUT_F32, int NS>
__global__ void __launch_bounds__(kThreads) k1_gather(StepArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[NS];

  const uint32_t T = a.tile_elems;
  const uint32_t tid = threadIdx.x;
  const uint64_t policy = policy_evict_first();
  const float inv_scale = a.cfg ? a.cfg->inv_scale : a.inv_scale;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // a PDL-launched K23 may begin its own setup now (no effect otherwise)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  auto issue = [&](uint32_t t, int s) {
    const SamoTile td = a.tiles[t];
    const uint32_t bytes = (td.dense_count * 2u) & ~15u;
    if (bytes) {
      mbar_arrive_expect_tx(&full[s], bytes);
      bulk_g2s(smem + static_cast<size_t>(s) * T * 2, a.layers[td.layer].grad + td.dense_begin,
               bytes, &full[s], policy);
    } else {
      mbar_arrive(&full[s]);
    }
  };
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      const uint64_t t = blockIdx.x + static_cast<uint64_t>(s) * gridDim.x;
      if (t < a.ntiles) issue(static_cast<uint32_t>(t), s);
    }
  }

  bool bad = false;
  const bool bf16 = a.grad_bf16 != 0;
  const uint32_t xm = grad_exp_mask(bf16);
  uint32_t it = 0;
  for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++it) {
    const int s = static_cast<int>(it % NS);
    const SamoTile td = a.tiles[t];
    // binary16 destination of element k: the local arena, or (push) the
    // owner's receive buffer over NVLink (tile-constant shift, same k % 8)
    uint16_t* g16 = reinterpret_cast<uint16_t*>(a.g);
    SAMO_DCHECK(td.k_begin <= td.k_end && td.dense_count <= T);
    SAMO_DCHECK(!a.push || td.pad_ < static_cast<uint32_t>(kMaxP2PRanks));
    if (!OUT_F32 && a.push)
      g16 = reinterpret_cast<uint16_t*>(reinterpret_cast<uintptr_t>(a.push16[td.pad_]) +
                                        2 * (td.pad2_ - td.k_begin));
    const uint16_t* gsrc = a.layers[td.layer].grad + td.dense_begin;
    const uint32_t staged = ((td.dense_count * 2u) & ~15u) >> 1;
    const uint16_t* sg = reinterpret_cast<const uint16_t*>(smem + static_cast<size_t>(s) * T * 2);
    mbar_wait(&full[s], (it / NS) & 1u);

    // Kept elements: 8-wide vectors on the 16-byte aligned middle of the
    // tile's k range (one 16-byte off16 load and one 16/32-byte store per 8),
    // scalar head and tail.
    const uint64_t kb0 = td.k_begin, ke = td.k_end;
    const uint64_t ka_up = (kb0 + 7) & ~7ull;
    const uint64_t ka = ka_up < ke ? ka_up : ke;
    const uint64_t ke8 = ka + ((ke - ka) & ~7ull);
    auto gather_one = [&](uint64_t k) {
      const uint16_t off = a.off16[k];
      SAMO_DCHECK(off < td.dense_count && k >= td.k_begin && k < td.k_end);
      const uint16_t h = off < staged ? sg[off] : gsrc[off];
      if constexpr (OUT_F32) {
        const float gk = mul_x86(grad_to_f32(h, bf16), inv_scale);
        bad |= !finite_f32(gk);
        st_na_f32(reinterpret_cast<float*>(a.g) + k, gk);
      } else {
        bad |= (h & xm) == xm;  // |h * 2^-s| is finite iff h is
        st_na_u16(g16 + k, h);
      }
    };
    if (tid < ka - kb0) gather_one(kb0 + tid);
    if (tid < ke - ke8) gather_one(ke8 + tid);
    const uint32_t nv = static_cast<uint32_t>((ke8 - ka) >> 3);
#pragma unroll 2
    for (uint32_t q = tid; q < nv; q += kThreads) {
      const uint64_t k = ka + 8ull * q;
      const uint4 o = ld_stream_v4(a.off16 + k);
      const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
      uint32_t hw[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t o0 = ow[e] & 0xFFFFu, o1 = ow[e] >> 16;
        SAMO_DCHECK(o0 < td.dense_count && o1 < td.dense_count);
        const uint32_t h0 = o0 < staged ? sg[o0] : gsrc[o0];
        const uint32_t h1 = o1 < staged ? sg[o1] : gsrc[o1];
        hw[e] = h0 | (h1 << 16);
      }
      if constexpr (OUT_F32) {
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint16_t h = static_cast<uint16_t>((e & 1) ? (hw[e >> 1] >> 16) : (hw[e >> 1] & 0xFFFFu));
          f[e] = mul_x86(grad_to_f32(h, bf16), inv_scale);
          bad |= !finite_f32(f[e]);
        }
        float* dst = reinterpret_cast<float*>(a.g) + k;
        st_na_v4f(dst, f[0], f[1], f[2], f[3]);
        st_na_v4f(dst + 4, f[4], f[5], f[6], f[7]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          bad |= ((hw[e] & xm) == xm) | ((hw[e] & (xm << 16)) == (xm << 16));
        st_na_v4u(g16 + k, hw[0], hw[1], hw[2], hw[3]);
      }
    }
    __syncthreads();  // every thread is done reading stage s
    if (tid == 0) {
      const uint64_t tn = t + static_cast<uint64_t>(NS) * gridDim.x;
      if (tn < a.ntiles) {
        fence_proxy_async_smem();
        issue(static_cast<uint32_t>(tn), s);
      }
    }
  }
  if (!OUT_F32 && a.push) asm volatile("fence.acq_rel.sys;" ::: "memory");  // peer stores visible system-wide
  if (__syncthreads_or(bad) && tid == 0) atomicAdd(a.flag_slot, 1.0f);
}

// ---------------------------------------------------------------------------
// K23

template <int CH>
__device__ __forceinline__ uint32_t tile_chunks(uint64_t k_begin, uint64_t k_end) {
  const uint64_t n = k_end - k_begin;
  return n == 0 ? 1u : static_cast<uint32_t>((n + CH - 1) / CH);
}

// The fields of a tile descriptor the update kernel needs, loaded with three
// 16-byte read-only loads straight into registers.
struct TileRegs {
  uint64_t k_begin, k_end, out_off;
  uint32_t dense_count;
};

__device__ __forceinline__ TileRegs load_tile(const SamoTile* p) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  const uint4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  TileRegs r;
  r.dense_count = a.z;
  r.k_begin = (static_cast<uint64_t>(b.y) << 32) | b.x;
  r.k_end = (static_cast<uint64_t>(b.w) << 32) | b.z;
  r.out_off = (static_cast<uint64_t>(c.y) << 32) | c.x;
  return r;
}

// Sum of n per-CTA float partials in double by all NT threads of the last
// CTA: thread i takes partials i, i + NT, ... in order, then a fixed
// shuffle/warp tree.  Deterministic for a given grid, and n/NT round trips to
// L2 instead of n.  `red` holds NT/32 doubles; the result is valid in thread 0.
template <int NT>
__device__ __forceinline__ double sum_partials(const float* p, uint32_t n, double* red) {
  const uint32_t tid = threadIdx.x;
  double acc = 0.0;
  const volatile float* vp = p;
  for (uint32_t i = tid; i < n; i += NT) acc += static_cast<double>(vp[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  double s = 0.0;
  if (tid == 0)
    for (int w = 0; w < NT / 32; ++w) s += red[w];
  return s;
}

template <bool G16, int CH, bool EXPAND = false>
struct K23Layout {
  // expand-only stages carry just the 16-bit values and off16 (compact, so
  // NCCL kernels still fit on the SMs while the expand runs)
  static constexpr uint32_t kF32 = EXPAND ? 0u : (CH + 8) * 4;    // theta/m/v/g32 slot
  static constexpr uint32_t kG = G16 ? (CH + 16) * 2 : kF32;    // grad slot
  static constexpr uint32_t kOff = (CH + 16) * 2;               // off16 slot
  static constexpr uint32_t kStage = 3 * kF32 + kG + kOff;
};

// EXPAND = true: expand-only pass of the sharded data-parallel step — the
// grad slot carries the all-gathered compressed binary16 weights (theta16c),
// no Adam, no theta/m/v traffic.
// CFG: the optimizer scalars come from a.cfg (graph captures); the eager
// instantiation keeps them kernel parameters — at 96 registers (the per-SMSP
// cap at 2 CTAs/SM) values derived from a global load would spill (+3%).
template <bool G16, int CH, int NS, bool EXPAND = false, bool CFG = false>
__global__ void __launch_bounds__(kThreads + 32) k23_update(StepArgs a) {
  static_assert(!EXPAND || G16, "expand-only reads 16-bit values");
  using L = K23Layout<G16, CH, EXPAND>;
  constexpr uint32_t kConsumerWarps = kThreads / 32;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[NS];
  __shared__ __align__(8) uint64_t empty[NS];
  __shared__ float red[kConsumerWarps];
  __shared__ int last_cta;

  const uint32_t T = a.tile_elems;
  uint16_t* outb = reinterpret_cast<uint16_t*>(smem + NS * L::kStage);  // 2 x T halves
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // Both dense out tiles start zeroed; afterwards the copy-out clears each
  // tile as it reads it, so no separate zero-fill phase is needed.
  {
    uint4* o4 = reinterpret_cast<uint4*>(outb);
    for (uint32_t i = tid; i < T * 4u / 16u; i += blockDim.x) o4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();  // the only CTA-wide barrier
  // PDL: everything above is local setup; K1's gradients and skip flag are
  // read only after the previous grid has completed (no-op without PDL).
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == kConsumerWarps) {
    // ---- producer warp: one elected lane walks the CTA's chunks and keeps
    // the ring full (16-byte aligned supersets of theta/m/v/grad/off16).
    if (lane == 0) {
      const uint64_t policy = policy_evict_first();
      uint32_t it = 0;
      TileRegs nxt{};
      if (blockIdx.x < a.ntiles) nxt = load_tile(a.tiles + blockIdx.x);
      for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        const TileRegs td = nxt;
        if (t + gridDim.x < a.ntiles) nxt = load_tile(a.tiles + t + gridDim.x);
        const uint32_t nch = tile_chunks<CH>(td.k_begin, td.k_end);
        for (uint32_t j = 0; j < nch; ++j, ++it) {
          const int s = static_cast<int>(it % NS);
          if (it >= static_cast<uint32_t>(NS))
            mbar_wait(&empty[s], ((it / NS) - 1) & 1u);
          const uint64_t kc0 = td.k_begin + static_cast<uint64_t>(j) * CH;
          const uint64_t kc1 = min(td.k_end, kc0 + CH);
          uint8_t* st = smem + s * L::kStage;
          const uint64_t f0 = kc0 & ~3ull;
          const uint32_t fb = static_cast<uint32_t>((((kc1 + 3) & ~3ull) - f0) * 4);
          const uint64_t h0 = kc0 & ~7ull;
          const uint32_t hb = static_cast<uint32_t>((((kc1 + 7) & ~7ull) - h0) * 2);
          const uint32_t gb = G16 ? hb : fb;
          if (kc1 == kc0) {  // empty tile: nothing to move, just publish the slot
            mbar_arrive(&full[s]);
            continue;
          }
          const void* gsrc = G16 ? static_cast<const void*>(reinterpret_cast<const uint16_t*>(a.g) + h0)
                                 : static_cast<const void*>(reinterpret_cast<const float*>(a.g) + f0);
          if constexpr (EXPAND) {  // theta/m/v slots unused; hb > 0 here
            mbar_arrive_expect_tx(&full[s], 2 * hb);
            bulk_g2s(st + 3 * L::kF32, gsrc, hb, &full[s], policy);
            bulk_g2s(st + 3 * L::kF32 + L::kG, a.off16 + h0, hb, &full[s], policy);
          } else {
            // kc1 > kc0, so every range rounded out to 16 bytes is non-empty.
            mbar_arrive_expect_tx(&full[s], 3 * fb + gb + hb);
            bulk_g2s(st, a.theta + f0, fb, &full[s], policy);
            bulk_g2s(st + L::kF32, a.m + f0, fb, &full[s], policy);
            bulk_g2s(st + 2 * L::kF32, a.v + f0, fb, &full[s], policy);
            bulk_g2s(st + 3 * L::kF32, gsrc, gb, &full[s], policy);
            bulk_g2s(st + 3 * L::kF32 + L::kG, a.off16 + h0, hb, &full[s], policy);
          }
        }
      }
    }
    return;
  }

  // ---- consumer warps ------------------------------------------------------
  // Step scalars (train.hpp:640-642), identical float ops in every CTA.
  const bool skip = !EXPAND && *reinterpret_cast<volatile float*>(a.flag_slot) != 0.0f;
  SamoAdamParams cprm = a.prm;
  if constexpr (CFG) cprm = step_prm(a.cfg, a.prm);
  const float b1p = __fmul_rn(a.st->beta1_pow, cprm.beta1);
  const float b2p = __fmul_rn(a.st->beta2_pow, cprm.beta2);
  const float bias1 = __fsub_rn(1.0f, b1p), bias2 = __fsub_rn(1.0f, b2p);
  const float omb1 = __fsub_rn(1.0f, cprm.beta1);  // train.hpp:335
  const float omb2 = __fsub_rn(1.0f, cprm.beta2);  // train.hpp:336
  const float lrwd = __fmul_rn(cprm.lr, cprm.wd);

  // Hot-loop parameters in registers (see pin_f32).
  const float p_beta1 = pin_f32(cprm.beta1), p_beta2 = pin_f32(cprm.beta2);
  const float p_lr = pin_f32(cprm.lr), p_eps = pin_f32(cprm.eps), p_wd = pin_f32(cprm.wd);
  float inv_scale = a.inv_scale;
  if constexpr (CFG) inv_scale = a.cfg ? a.cfg->inv_scale : a.inv_scale;
  const float p_inv = pin_f32(inv_scale);
  const uint32_t p_T = pin_u32(T);
  float* const p_theta = pin_ptr(a.theta);
  float* const p_m = pin_ptr(a.m);
  float* const p_v = pin_ptr(a.v);
  uint16_t* const p_t16 = pin_ptr(a.theta16);

  float nacc = 0.0f;
  uint32_t it = 0, tile_it = 0;
  TileRegs nxt{};
  if (blockIdx.x < a.ntiles) nxt = load_tile(a.tiles + blockIdx.x);
  for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++tile_it) {
    const TileRegs td = nxt;
    if (t + gridDim.x < a.ntiles) nxt = load_tile(a.tiles + t + gridDim.x);  // prefetch
    const uint32_t nch = tile_chunks<CH>(td.k_begin, td.k_end);
    uint16_t* out = outb + (tile_it & 1u) * p_T;
    uint16_t* dst = p_t16 + td.out_off;
    for (uint32_t j = 0; j < nch; ++j, ++it) {
      const int s = static_cast<int>(it % NS);
      const uint8_t* st = smem + s * L::kStage;
      const uint64_t kc0 = td.k_begin + static_cast<uint64_t>(j) * CH;
      const uint64_t kc1 = min(td.k_end, kc0 + CH);
      const uint32_t n = static_cast<uint32_t>(kc1 - kc0);
      const uint32_t fo = static_cast<uint32_t>(kc0 & 3ull);  // chunk offset in the f32 slots
      const uint32_t ho = static_cast<uint32_t>(kc0 & 7ull);  // ... in the 16-bit slots
      const float* sth = reinterpret_cast<const float*>(st) + fo;
      const float* smv = reinterpret_cast<const float*>(st + L::kF32) + fo;
      const float* svv = reinterpret_cast<const float*>(st + 2 * L::kF32) + fo;
      const uint16_t* soff = reinterpret_cast<const uint16_t*>(st + 3 * L::kF32 + L::kG) + ho;
      mbar_wait(&full[s], (it / NS) & 1u);

      if constexpr (EXPAND) {
        const uint16_t* sval = reinterpret_cast<const uint16_t*>(st + 3 * L::kF32) + ho;
#pragma unroll 4
        for (uint32_t i = tid; i < n; i += kThreads) {
          SAMO_DCHECK(soff[i] < p_T);
          out[soff[i]] = sval[i];
        }
      } else {
#pragma unroll 1
      for (uint32_t ib = tid; ib < n; ib += kU * kThreads) {
        float gv[kU], tv[kU], mv[kU], vv[kU];
        uint16_t ov[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const uint32_t i = ib + u * kThreads;
          if (i < n) {
            if constexpr (G16) {
              const uint16_t h = reinterpret_cast<const uint16_t*>(st + 3 * L::kF32)[ho + i];
              gv[u] = mul_x86(grad_to_f32(h, a.grad_bf16 != 0), p_inv);
            } else {
              gv[u] = reinterpret_cast<const float*>(st + 3 * L::kF32)[fo + i];
            }
            tv[u] = sth[i];
            mv[u] = smv[i];
            vv[u] = svv[i];
            ov[u] = soff[i];
            SAMO_DCHECK(ov[u] < p_T);
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const uint32_t i = ib + u * kThreads;
          if (i < n) {
            const float gk = gv[u];
            nacc = __fadd_rn(nacc, __fmul_rn(gk, gk));
            if (!skip) {
              // adam_update (train.hpp:338-345): IEEE per op, no contraction.
              const float mk = __fadd_rn(__fmul_rn(p_beta1, mv[u]), __fmul_rn(omb1, gk));
              const float vk =
                  __fadd_rn(__fmul_rn(p_beta2, vv[u]), __fmul_rn(omb2, __fmul_rn(gk, gk)));
              const float mh = __fdiv_rn(mk, bias1);
              const float vh = __fdiv_rn(vk, bias2);
              float tk = __fsub_rn(
                  tv[u], __fmul_rn(p_lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), p_eps))));
              if (p_wd != 0.0f) tk = __fsub_rn(tk, __fmul_rn(lrwd, tk));
              const uint64_t k = kc0 + i;
              st_na_f32(p_m + k, mk);
              st_na_f32(p_v + k, vk);
              st_na_f32(p_theta + k, tk);
              out[ov[u]] = f32_to_f16_bits(tk);
            }
          }
        }
      }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
    }
    // All consumer warps have scattered into `out`.
    asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
    if (!skip) {
      // Copy the finished dense tile out with 128-bit stores (layer segments
      // are 256-byte aligned, tiles start at multiples of T) and clear it for
      // its next use two tiles later.
      uint4* o4 = reinterpret_cast<uint4*>(out);
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      const uint32_t full16 = td.dense_count >> 3;
      for (uint32_t i0 = tid; i0 < full16; i0 += 4 * kThreads) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t i = i0 + u * kThreads;
          if (i < full16) v[u] = o4[i];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t i = i0 + u * kThreads;
          if (i < full16) {
            o4[i] = make_uint4(0u, 0u, 0u, 0u);
            d4[i] = v[u];
          }
        }
      }
      for (uint32_t i = full16 * 8 + tid; i < td.dense_count; i += kThreads) {
        dst[i] = out[i];
        out[i] = 0;
      }
    }
  }

  if constexpr (EXPAND) return;

  // Grad norm partial per CTA (fixed schedule -> deterministic), finalised by
  // the last CTA in CTA order (double).
  float x = nacc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = __fadd_rn(x, __shfl_xor_sync(0xFFFFFFFFu, x, o));
  if (lane == 0) red[warp] = x;
  asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
  if (tid == 0) {
    float s = 0.f;
    for (uint32_t w = 0; w < kConsumerWarps; ++w) s = __fadd_rn(s, red[w]);
    a.norm_partials[blockIdx.x] = s;
    __threadfence();
    const uint32_t ticket = atomicAdd(&a.st->done_ctas, 1u);
    last_cta = (ticket == gridDim.x - 1);
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
  if (!last_cta) return;
  __shared__ double dred[kConsumerWarps];
  double acc = 0.0;
  if (a.finalize) {
    if (tid == 0) __threadfence();
    asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
    acc = sum_partials<kThreads>(a.norm_all, a.norm_count, dred);
  }
  if (tid == 0) {
    SamoStepState* stt = a.st;
    if (a.finalize) {  // the step's last update launch
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
      *a.flag_slot = 0.0f;  // every CTA of every launch has read it
    }
    stt->done_ctas = 0u;
    __threadfence();
  }
}

// ---------------------------------------------------------------------------
// K123: the whole single-GPU step in one pass per tile (train.hpp:598-654:
// sink gather, unscale + finite check, Adam, downcast + expand).
//
// The skip decision (train.hpp:632-639) depends on every gradient of the
// step, so the pass is speculative: it reads theta/m/v and writes the updated
// values to the model's other buffer set (theta_o/m_o/v_o), and writes the
// new binary16 weights straight into theta16.  The last CTA then either
// advances the Adam scalars (the host swaps the buffer sets) or records the
// skip, after which k123_repair copies theta/m/v into the other set and
// rebuilds theta16 from theta — theta16 == expand(half(theta32)) is the
// state invariant (store.hpp:171-197), so the repair restores it bit for bit.
//
// Scheduling: tiles are claimed dynamically (one atomic per tile by the
// producer lane), so SMs that run faster take more tiles; the producer hands
// each claimed tile's descriptor to the consumers through shared memory.
// Per tile: one 1-D TMA copy of the dense binary16 gradient tile into one of
// NSG slots, then theta/m/v/off16 of the tile's kept range in <= CH-element
// chunks (NS-stage ring).  Consumers gather g = half(grad[off]) * 2^-s
// through off16, run the IEEE Adam, store theta/m/v with streaming stores,
// and write half(theta) back into the gradient tile at the same offset (each
// offset belongs to one kept element), marking it in a per-slot bitmap.
// Each warp signals the slot's `done` barrier when its share of the tile is
// computed and copies the tile out one tile LATER (after computing the next
// one), so no warp waits for the slowest warp of a tile: 128-bit stores to
// theta16, pruned positions zeroed by the bitmap, bitmap cleared.
//
// Grad norm: one partial per tile (lanes in element order, warps in order)
// into tile_norm[t]; k123_repair sums them in tile order, so the norm does
// not depend on which CTA took which tile.
//
// HBM bytes per step: 2 phi (grad) + 2 n (off16) + 24 n (theta/m/v read +
// write) + 2 phi (theta16) = 4 phi + 26 n, against 4 phi + 32 n for K1 + K23
// (grad16 written and read back, off16 read twice).

struct TileFull {
  uint32_t layer, dense_begin, dense_count;
  uint64_t k_begin, k_end, out_off;
};

__device__ __forceinline__ TileFull load_tile_full(const SamoTile* p) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  const uint4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  TileFull r;
  r.layer = a.x;
  r.dense_begin = a.y;
  r.dense_count = a.z;
  r.k_begin = (static_cast<uint64_t>(b.y) << 32) | b.x;
  r.k_end = (static_cast<uint64_t>(b.w) << 32) | b.z;
  r.out_off = (static_cast<uint64_t>(c.y) << 32) | c.x;
  return r;
}

// Up to this many tiles K123's last CTA sums the per-tile norm partials
// itself; above, the repair kernel's CTAs share the sum.
constexpr uint32_t kK123SmallNorm = 4096;

// A claimed tile as the producer hands it to the consumers.
struct K123Slot {
  uint64_t k_begin, k_end, out_off;
  const uint16_t* grad;  // the layer's dense gradient at the tile's first element
  uint32_t t;            // tile id, kNoTile once the tiles are exhausted
  uint32_t dense_count;
};
constexpr uint32_t kNoTile = 0xFFFFFFFFu;

template <int CH>
struct K123Layout {
  static constexpr uint32_t kF32 = (CH + 8) * 4;   // theta / m / v slot
  static constexpr uint32_t kOff = (CH + 16) * 2;  // off16 slot
  static constexpr uint32_t kStage = 3 * kF32 + kOff;
  static_assert(kStage % 16 == 0, "stages stay 16-byte aligned");
};
// Dense gradient slots per CTA: one being computed and copied out, one being
// filled.  (A deferred copy-out — each warp copying tile j out after
// computing tile j + 1, no consumer barrier — needs a third slot; it measured
// 25% slower at 16384-element tiles (one CTA per SM) and level at 8192, both
// behind this form: tools/sweep_k123.sh, profiles/r02d_k123_sweep.jsonl.)
constexpr int kK123Slots = 2;

// Lane masks of 8 binary16 values from 8 bitmap bits (bit e -> lane e).
__device__ __forceinline__ uint32_t lane_mask2(uint32_t bits, int e) {
  return ((0u - ((bits >> (2 * e)) & 1u)) & 0x0000FFFFu) | ((0u - ((bits >> (2 * e + 1)) & 1u)) & 0xFFFF0000u);
}

template <int CH, int NS, int NT, bool CFG>
__global__ void __launch_bounds__(NT + 32, 512 / NT) k123_step(StepArgs a) {
  using L = K123Layout<CH>;
  constexpr uint32_t kConsumerWarps = NT / 32;
  constexpr int NSG = kK123Slots;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[NS];
  __shared__ __align__(8) uint64_t empty[NS];
  __shared__ __align__(8) uint64_t gfull[NSG];
  __shared__ __align__(8) uint64_t gempty[NSG];
  __shared__ __align__(16) K123Slot slot[NSG];
  __shared__ float red[NSG][kConsumerWarps];
  __shared__ int last_cta;
  __shared__ int cta_bad;

  const uint32_t T = a.tile_elems;
  uint8_t* const gst = smem + NS * L::kStage;                                 // NSG x T halves
  uint32_t* const bm0 = reinterpret_cast<uint32_t*>(gst + NSG * T * 2u);     // NSG x T bits
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (uint32_t i = tid; i < NSG * (T / 32u); i += blockDim.x) bm0[i] = 0u;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    for (int s = 0; s < NSG; ++s) {
      mbar_init(&gfull[s], 1);
      mbar_init(&gempty[s], kConsumerWarps);
    }
    cta_bad = 0;
    fence_mbar_init();
  }
  __syncthreads();  // the only CTA-wide barrier
  // PDL: the previous step's kernels may still be running until here.
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == kConsumerWarps) {
    // ---- producer warp (one elected lane): claim a tile, publish its
    // descriptor, bring its dense gradient tile, then theta/m/v/off16 of its
    // kept range chunk by chunk.  The next claim is issued a tile ahead.
    if (lane == 0) {
      const uint64_t policy = policy_evict_first();
      uint32_t it = 0;
      // the first tile of each CTA is its own index, the rest are claimed
      // (the counter runs from gridDim.x): one atomic less on the critical
      // path of short steps
      uint32_t t = blockIdx.x;
      for (uint32_t tt = 0;; ++tt) {
        const int sg = static_cast<int>(tt % NSG);
        if (tt >= static_cast<uint32_t>(NSG)) mbar_wait(&gempty[sg], ((tt / NSG) - 1) & 1u);
        K123Slot& sl = slot[sg];
        if (t >= a.ntiles) {
          sl.t = kNoTile;
          mbar_arrive(&gfull[sg]);
          break;
        }
        const TileFull td = load_tile_full(a.tiles + t);
        SAMO_DCHECK(td.dense_count <= T && td.k_begin <= td.k_end);
        const uint16_t* grad = a.layers[td.layer].grad + td.dense_begin;
        const uint32_t t_cur = t;
        t = gridDim.x + atomicAdd(&a.st->tile_next, 1u);
        sl.k_begin = td.k_begin;
        sl.k_end = td.k_end;
        sl.out_off = td.out_off;
        sl.grad = grad;
        sl.t = t_cur;
        sl.dense_count = td.dense_count;
        const uint32_t bytes = (td.dense_count * 2u) & ~15u;
        if (bytes) {
          mbar_arrive_expect_tx(&gfull[sg], bytes);
          bulk_g2s(gst + static_cast<size_t>(sg) * T * 2u, grad, bytes, &gfull[sg], policy);
        } else {
          mbar_arrive(&gfull[sg]);
        }
        const uint32_t nch = tile_chunks<CH>(td.k_begin, td.k_end);
        for (uint32_t j = 0; j < nch; ++j, ++it) {
          const int s = static_cast<int>(it % NS);
          if (it >= static_cast<uint32_t>(NS)) mbar_wait(&empty[s], ((it / NS) - 1) & 1u);
          const uint64_t kc0 = td.k_begin + static_cast<uint64_t>(j) * CH;
          const uint64_t kc1 = min(td.k_end, kc0 + CH);
          if (kc1 == kc0) {
            mbar_arrive(&full[s]);
            continue;
          }
          uint8_t* st = smem + s * L::kStage;
          const uint64_t f0 = kc0 & ~3ull;
          const uint32_t fb = static_cast<uint32_t>((((kc1 + 3) & ~3ull) - f0) * 4);
          const uint64_t h0 = kc0 & ~7ull;
          const uint32_t hb = static_cast<uint32_t>((((kc1 + 7) & ~7ull) - h0) * 2);
          mbar_arrive_expect_tx(&full[s], 3 * fb + hb);
          bulk_g2s(st, a.theta + f0, fb, &full[s], policy);
          bulk_g2s(st + L::kF32, a.m + f0, fb, &full[s], policy);
          bulk_g2s(st + 2 * L::kF32, a.v + f0, fb, &full[s], policy);
          bulk_g2s(st + 3 * L::kF32, a.off16 + h0, hb, &full[s], policy);
        }
      }
    }
    return;
  }

  // ---- consumer warps ------------------------------------------------------
  SamoAdamParams cprm = a.prm;
  if constexpr (CFG) cprm = step_prm(a.cfg, a.prm);
  const float b1p = __fmul_rn(a.st->beta1_pow, cprm.beta1);  // train.hpp:325-329, 640-642
  const float b2p = __fmul_rn(a.st->beta2_pow, cprm.beta2);
  const float bias1 = __fsub_rn(1.0f, b1p), bias2 = __fsub_rn(1.0f, b2p);
  const float omb1 = __fsub_rn(1.0f, cprm.beta1);  // train.hpp:335
  const float omb2 = __fsub_rn(1.0f, cprm.beta2);  // train.hpp:336
  const float lrwd = __fmul_rn(cprm.lr, cprm.wd);
  const float p_beta1 = pin_f32(cprm.beta1), p_beta2 = pin_f32(cprm.beta2);
  const float p_lr = pin_f32(cprm.lr), p_eps = pin_f32(cprm.eps), p_wd = pin_f32(cprm.wd);
  float inv_scale = a.inv_scale;
  if constexpr (CFG) inv_scale = a.cfg ? a.cfg->inv_scale : a.inv_scale;
  const float p_inv = pin_f32(inv_scale);
  float* const p_to = pin_ptr(a.theta_o);
  float* const p_mo = pin_ptr(a.m_o);
  float* const p_vo = pin_ptr(a.v_o);
  uint16_t* const p_t16 = pin_ptr(a.theta16);

  // Copy-out of this CTA's j-th claimed tile, once every warp has computed
  // its share.
  auto copy_out = [&](uint32_t j) {
    const int sg = static_cast<int>(j % NSG);
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    const K123Slot& sl = slot[sg];
    const uint32_t dense_count = sl.dense_count;
    const uint4* o4 = reinterpret_cast<const uint4*>(gst + static_cast<size_t>(sg) * T * 2u);
    const uint16_t* o2 = reinterpret_cast<const uint16_t*>(o4);
    uint8_t* b8 = reinterpret_cast<uint8_t*>(bm0 + sg * (T / 32u));
    uint16_t* dst = p_t16 + sl.out_off;
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    const uint32_t full16 = dense_count >> 3;
    // A 32-byte sector of theta16 (16 values, two lanes' 16-byte chunks)
    // with no kept element is not written: theta16 is already zero there
    // (the state invariant, store.hpp:171-197; every writer of theta16
    // keeps pruned positions zero), so only sectors holding a kept element
    // reach HBM — at p = 0.9, 1 - 0.9^16 = 81% of them.  The loop is
    // warp-uniform so the lane pairs can compare masks.
    for (uint32_t base = tid - lane; base < full16; base += 4 * NT) {
      const uint32_t i0 = base + lane;
      uint4 v[4];
      uint32_t bits[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = i0 + u * NT;
        bits[u] = 0u;
        if (i < full16) {
          v[u] = o4[i];
          bits[u] = b8[i];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = i0 + u * NT;
        const uint32_t sector = bits[u] | __shfl_xor_sync(0xFFFFFFFFu, bits[u], 1);
        if (i < full16) {
          uint4 w = v[u];
          w.x &= lane_mask2(bits[u], 0);
          w.y &= lane_mask2(bits[u], 1);
          w.z &= lane_mask2(bits[u], 2);
          w.w &= lane_mask2(bits[u], 3);
          if (bits[u]) b8[i] = 0;
          if (sector) st_na_v4u(d4 + i, w.x, w.y, w.z, w.w);
        }
      }
    }
    if (tid == 0) {
      if (dense_count & 7u) {
        const uint32_t base = full16 * 8u;
        const uint32_t bits = b8[full16];
        for (uint32_t e = 0; e < (dense_count & 7u); ++e) dst[base + e] = ((bits >> e) & 1u) ? o2[base + e] : 0;
        b8[full16] = 0;
      }
      float s = 0.f;  // the tile's grad-norm partial, warps in order
      for (uint32_t w = 0; w < kConsumerWarps; ++w) s = __fadd_rn(s, red[sg][w]);
      a.tile_norm[sl.t] = s;
    }
    // The next TMA copy into this slot follows generic-proxy writes.
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&gempty[sg]);
  };

  bool bad = false;
  const bool bf16 = a.grad_bf16 != 0;
  const uint32_t xm = grad_exp_mask(bf16);
  uint32_t it = 0, tt = 0;
  for (;; ++tt) {
    const int sg = static_cast<int>(tt % NSG);
    mbar_wait(&gfull[sg], (tt / NSG) & 1u);
    const K123Slot& sl = slot[sg];
    const uint32_t t = sl.t;
    if (t == kNoTile) break;
    const uint64_t k_begin = sl.k_begin, k_end = sl.k_end;
    uint16_t* const sgr = reinterpret_cast<uint16_t*>(gst + static_cast<size_t>(sg) * T * 2u);
    uint32_t* const bm = bm0 + sg * (T / 32u);
    const uint32_t staged = ((sl.dense_count * 2u) & ~15u) >> 1;
    const uint16_t* const gsrc = sl.grad;  // unstaged tail (< 8 elements)
    const uint32_t nch = tile_chunks<CH>(k_begin, k_end);
    float nacc = 0.0f;
    for (uint32_t j = 0; j < nch; ++j, ++it) {
      const int s = static_cast<int>(it % NS);
      const uint8_t* st = smem + s * L::kStage;
      const uint64_t kc0 = k_begin + static_cast<uint64_t>(j) * CH;
      const uint64_t kc1 = min(k_end, kc0 + CH);
      const uint32_t n = static_cast<uint32_t>(kc1 - kc0);
      const uint32_t fo = static_cast<uint32_t>(kc0 & 3ull);
      const uint32_t ho = static_cast<uint32_t>(kc0 & 7ull);
      const float* sth = reinterpret_cast<const float*>(st) + fo;
      const float* smv = reinterpret_cast<const float*>(st + L::kF32) + fo;
      const float* svv = reinterpret_cast<const float*>(st + 2 * L::kF32) + fo;
      const uint16_t* soff = reinterpret_cast<const uint16_t*>(st + 3 * L::kF32) + ho;
      mbar_wait(&full[s], (it / NS) & 1u);
#pragma unroll 1
      for (uint32_t ib = tid; ib < n; ib += kU * NT) {
        float gv[kU], tv[kU], mv[kU], vv[kU];
        uint32_t ov[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const uint32_t i = ib + u * NT;
          if (i < n) {
            ov[u] = soff[i];
            SAMO_DCHECK(ov[u] < sl.dense_count && n <= CH);
            const uint16_t h = ov[u] < staged ? sgr[ov[u]] : gsrc[ov[u]];
            bad |= (h & xm) == xm;  // |h * 2^-s| is finite iff h is
            gv[u] = __fmul_rn(grad_to_f32_finite(h, bf16), p_inv);  // finite steps only (5% faster K123)
            tv[u] = sth[i];
            mv[u] = smv[i];
            vv[u] = svv[i];
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const uint32_t i = ib + u * NT;
          if (i < n) {
            const float gk = gv[u];
            nacc = __fadd_rn(nacc, __fmul_rn(gk, gk));
            // adam_update (train.hpp:338-345): IEEE per op, no contraction.
            const float mk = __fadd_rn(__fmul_rn(p_beta1, mv[u]), __fmul_rn(omb1, gk));
            const float vk = __fadd_rn(__fmul_rn(p_beta2, vv[u]), __fmul_rn(omb2, __fmul_rn(gk, gk)));
            const float mh = __fdiv_rn(mk, bias1);
            const float vh = __fdiv_rn(vk, bias2);
            float tk = __fsub_rn(tv[u], __fmul_rn(p_lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), p_eps))));
            if (p_wd != 0.0f) tk = __fsub_rn(tk, __fmul_rn(lrwd, tk));
            const uint64_t k = kc0 + i;
            st_na_f32(p_mo + k, mk);
            st_na_f32(p_vo + k, vk);
            st_na_f32(p_to + k, tk);
            sgr[ov[u]] = f32_to_f16_bits(tk);
            atomicOr(&bm[ov[u] >> 5], 1u << (ov[u] & 31u));
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // This warp's share of the tile is computed: its norm partial, then the
    // slot's done barrier; the copy-out of the PREVIOUS tile follows.
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nacc = __fadd_rn(nacc, __shfl_xor_sync(0xFFFFFFFFu, nacc, o));
    if (lane == 0) red[sg][warp] = nacc;
    copy_out(tt);
  }
  // The repair kernel may start its (waiting) CTAs now.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // Skip indicator per CTA; the last CTA decides the step.
  if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(&cta_bad, 1);
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  if (tid == 0) {
    if (cta_bad) atomicAdd(a.flag_slot, 1.0f);
    __threadfence();
    const uint32_t ticket = atomicAdd(&a.st->done_ctas, 1u);
    last_cta = (ticket == gridDim.x - 1);
  }
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  if (!last_cta) return;
  SamoStepState* stt = a.st;
  if (a.ntiles <= kK123SmallNorm) {  // short steps: the grad norm here, tiles in order
    __shared__ double dsum[NT / 32];
    if (tid == 0) __threadfence();
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    double acc = 0.0;
    for (uint32_t t = tid; t < a.ntiles; t += NT) acc += static_cast<double>(__ldcg(a.tile_norm + t));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if (lane == 0) dsum[warp] = acc;
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    if (tid == 0) {
      double s2 = 0.0;
      for (uint32_t w = 0; w < kConsumerWarps; ++w) s2 += dsum[w];
      stt->grad_norm = static_cast<float>(sqrt(s2));
    }
  }
  if (tid != 0) return;
  __threadfence();
  if (*reinterpret_cast<volatile float*>(a.flag_slot) != 0.0f) {  // train.hpp:632-639
    stt->skipped_steps += 1;
    stt->last_skipped = 1u;
  } else {  // AdamScalars::advance, train.hpp:325-329
    stt->t += 1;
    stt->beta1_pow = b1p;
    stt->beta2_pow = b2p;
    stt->last_skipped = 0u;
  }
  *a.flag_slot = 0.0f;
  // Every producer has made its last claim (its consumers saw kNoTile before
  // their CTA took a ticket), so the claim counter can be rewound.
  stt->tile_next = 0u;
  stt->done_ctas = 0u;
  __threadfence();
}

// After K123: the grad norm from the per-tile partials (train.hpp:627-630;
// fixed order: tile ranges per CTA, CTAs in order), then — only if the step
// was skipped — theta/m/v are copied into the other buffer set (the host
// swaps the sets after every step) and theta16 is rebuilt as
// expand(half(theta)), the state before the step.
__global__ void __launch_bounds__(kThreads) k123_repair(StepArgs a) {
  __shared__ double dred[kThreads / 32];
  __shared__ int last_cta;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t tid = threadIdx.x;
  if (a.ntiles > kK123SmallNorm) {  // (short steps: K123's last CTA summed them)
    const uint32_t per = (a.ntiles + gridDim.x - 1) / gridDim.x;
    const uint32_t t0 = min(a.ntiles, blockIdx.x * per), t1 = min(a.ntiles, t0 + per);
    double acc = 0.0;
    for (uint32_t t = t0 + tid; t < t1; t += kThreads) acc += static_cast<double>(__ldcg(a.tile_norm + t));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if ((tid & 31) == 0) dred[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) s += dred[w];
      a.norm_dpartials[blockIdx.x] = s;
      __threadfence();
      last_cta = (atomicAdd(&a.st->done_ctas, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (last_cta) {  // uniform: all threads fetch the partials, one sums them in order
      __shared__ double part[1024];
      __threadfence();
      for (uint32_t b = tid; b < gridDim.x; b += kThreads) part[b] = __ldcg(a.norm_dpartials + b);
      __syncthreads();
      if (tid == 0) {
        double s = 0.0;
        for (uint32_t b = 0; b < gridDim.x; ++b) s += part[b];
        a.st->grad_norm = static_cast<float>(sqrt(s));
        a.st->done_ctas = 0u;
        __threadfence();
      }
    }
  }
  if (*reinterpret_cast<volatile uint32_t*>(&a.st->last_skipped) == 0u) return;
  for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const TileFull td = load_tile_full(a.tiles + t);
    uint16_t* dst = a.theta16 + td.out_off;
    for (uint32_t i = threadIdx.x; i < td.dense_count; i += blockDim.x) dst[i] = 0;
    __syncthreads();
    for (uint64_t k = td.k_begin + threadIdx.x; k < td.k_end; k += blockDim.x) {
      const float th = a.theta[k];
      a.theta_o[k] = th;
      a.m_o[k] = a.m[k];
      a.v_o[k] = a.v[k];
      dst[a.off16[k]] = f32_to_f16_bits(th);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Sharded data-parallel step (ZeRO-1 on the compressed state): Adam on this
// rank's shard of the reduce-scattered gradient, writing the updated weights
// both as fp32 master copy and as compressed binary16 (theta16c) for the
// all-gather; then the expand-only tile pass rebuilds every dense theta16.

__device__ __forceinline__ float adam_one(float g, float& m, float& v, float t, const SamoAdamParams& p,
                                          float omb1, float omb2, float bias1, float bias2,
                                          float lrwd) {
  m = __fadd_rn(__fmul_rn(p.beta1, m), __fmul_rn(omb1, g));
  v = __fadd_rn(__fmul_rn(p.beta2, v), __fmul_rn(omb2, __fmul_rn(g, g)));
  const float mh = __fdiv_rn(m, bias1);
  const float vh = __fdiv_rn(v, bias2);
  t = __fsub_rn(t, __fmul_rn(p.lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), p.eps))));
  if (p.wd != 0.0f) t = __fsub_rn(t, __fmul_rn(lrwd, t));
  return t;
}

__global__ void __launch_bounds__(kThreads) k_adam_shard(ShardArgs a) {
  __shared__ float red[kThreads / 32];
  __shared__ int last_cta;
  const bool skip = *reinterpret_cast<const volatile float*>(a.flag_slot) != 0.0f;
  const SamoAdamParams prm = step_prm(a.cfg, a.prm);
  const float b1p = __fmul_rn(a.st->beta1_pow, prm.beta1);
  const float b2p = __fmul_rn(a.st->beta2_pow, prm.beta2);
  const float bias1 = __fsub_rn(1.0f, b1p), bias2 = __fsub_rn(1.0f, b2p);
  const float omb1 = __fsub_rn(1.0f, prm.beta1), omb2 = __fsub_rn(1.0f, prm.beta2);
  const float lrwd = __fmul_rn(prm.lr, prm.wd);
  float nacc = 0.0f;
  // k0 is a multiple of 8 (shard size), so 4-element vectors stay aligned.
  const uint64_t nv = (a.k1 - a.k0) / 4;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; q < nv; q += stride) {
    const uint64_t k = a.k0 + 4 * q;
    const float4 g = *reinterpret_cast<const float4*>(a.g + k);
    float4 t = *reinterpret_cast<const float4*>(a.theta + k);
    float4 m = *reinterpret_cast<const float4*>(a.m + k);
    float4 v = *reinterpret_cast<const float4*>(a.v + k);
    nacc = __fadd_rn(nacc, __fmul_rn(g.x, g.x));
    nacc = __fadd_rn(nacc, __fmul_rn(g.y, g.y));
    nacc = __fadd_rn(nacc, __fmul_rn(g.z, g.z));
    nacc = __fadd_rn(nacc, __fmul_rn(g.w, g.w));
    if (!skip) {
      t.x = adam_one(g.x, m.x, v.x, t.x, prm, omb1, omb2, bias1, bias2, lrwd);
      t.y = adam_one(g.y, m.y, v.y, t.y, prm, omb1, omb2, bias1, bias2, lrwd);
      t.z = adam_one(g.z, m.z, v.z, t.z, prm, omb1, omb2, bias1, bias2, lrwd);
      t.w = adam_one(g.w, m.w, v.w, t.w, prm, omb1, omb2, bias1, bias2, lrwd);
      *reinterpret_cast<float4*>(a.theta + k) = t;
      *reinterpret_cast<float4*>(a.m + k) = m;
      *reinterpret_cast<float4*>(a.v + k) = v;
    }
    uint2 h;
    h.x = static_cast<uint32_t>(f32_to_f16_bits(t.x)) | (static_cast<uint32_t>(f32_to_f16_bits(t.y)) << 16);
    h.y = static_cast<uint32_t>(f32_to_f16_bits(t.z)) | (static_cast<uint32_t>(f32_to_f16_bits(t.w)) << 16);
    *reinterpret_cast<uint2*>(a.theta16c + k) = h;
  }
  // scalar tail (fewer than 4 elements)
  if (blockIdx.x == 0 && threadIdx.x < (a.k1 - a.k0) % 4) {
    const uint64_t k = a.k0 + 4 * nv + threadIdx.x;
    const float g = a.g[k];
    float t = a.theta[k], m = a.m[k], v = a.v[k];
    nacc = __fadd_rn(nacc, __fmul_rn(g, g));
    if (!skip) {
      t = adam_one(g, m, v, t, prm, omb1, omb2, bias1, bias2, lrwd);
      a.theta[k] = t;
      a.m[k] = m;
      a.v[k] = v;
    }
    a.theta16c[k] = f32_to_f16_bits(t);
  }
  float x = nacc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = __fadd_rn(x, __shfl_xor_sync(0xFFFFFFFFu, x, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < kThreads / 32; ++w) s = __fadd_rn(s, red[w]);
    a.norm_partials[blockIdx.x] = s;
    __threadfence();
    last_cta = atomicAdd(a.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last_cta) return;
  __shared__ double dred[kThreads / 32];
  if (threadIdx.x == 0) __threadfence();
  __syncthreads();
  const double acc = sum_partials<kThreads>(a.norm_partials, gridDim.x, dred);
  if (threadIdx.x == 0) {
    *a.norm2_out = acc;
    *a.done = 0u;
    __threadfence();
  }
}

// ---------------------------------------------------------------------------
// Fused peer-to-peer exchange + shard update.  The skip-flag exchange before
// this kernel is the cross-rank barrier.  For the owned range, each thread
// takes VE consecutive elements: it loads their binary16 gradient from every
// rank — from the local receive buffer the ranks' K1 pushed into (push mode),
// or from each rank's own arena over NVLink (pull mode) — sums fl32(h * scale)
// in rank order (the oracle's rank-ascending fp32 sum, so the result is
// bit-exact for any G), runs Adam on its own fp32 state and stores the VE new
// binary16 weights into every rank's theta16c (peer stores).  Link bytes per
// rank: 2n(G-1)/G in (gradients) + 2n(G-1)/G out (weights).


__device__ __forceinline__ uint16_t half_lane(const uint4& v, int e) {
  const uint32_t w = e < 2 ? v.x : e < 4 ? v.y : e < 6 ? v.z : v.w;
  return static_cast<uint16_t>((e & 1) ? (w >> 16) : (w & 0xFFFFu));
}

// Epilogue of the shard kernels (NT participating threads, named barrier 1):
// per-CTA norm^2 partial, last CTA reduces them in CTA order and, in the
// pipelined step, publishes bucket completion + norm^2 to every rank.
template <int G, int NT>
__device__ __forceinline__ void shard_finish(const P2PArgs& a, float nacc, float* red, int* last_cta) {
  // Make the peer stores visible system-wide before the kernel retires and
  // before the completion signals below.
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  float x = nacc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = __fadd_rn(x, __shfl_xor_sync(0xFFFFFFFFu, x, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < NT / 32; ++w) s = __fadd_rn(s, red[w]);
    a.norm_partials[blockIdx.x] = s;
    __threadfence();
    *last_cta = atomicAdd(a.done, 1u) == gridDim.x - 1;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  if (!*last_cta) return;
  __shared__ double dred[NT / 32];
  if (threadIdx.x == 0) __threadfence();
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  const double acc = sum_partials<NT>(a.norm_partials, gridDim.x, dred);
  if (threadIdx.x == 0) {
    *a.norm2_out = acc;
    *a.done = 0u;
    __threadfence();
    if (a.bucket >= 0) {  // pipelined step: publish norm^2 + completion to every rank
      const uint64_t e = a.slots[a.rank]->epoch + 1;
      const int slot = a.bucket * kMaxP2PRanks + a.rank;
#pragma unroll
      for (int r = 0; r < G; ++r) a.slots[r]->norm[slot] = acc;
      asm volatile("fence.sc.sys;" ::: "memory");
#pragma unroll
      for (int r = 0; r < G; ++r) st_release_sys(&a.slots[r]->bucket_epoch[slot], e);
    }
  }
}

// VE binary16 lanes (8 or 4) of a 16- or 8-byte vector.
template <int VE>
struct HalfVec;
template <>
struct HalfVec<8> {
  uint4 v;
  __device__ __forceinline__ void load(const uint16_t* p) { v = ld_stream_v4(p); }
  __device__ __forceinline__ uint16_t lane(int e) const { return half_lane(v, e); }
  __device__ __forceinline__ static void store(uint16_t* p, const uint32_t (&w)[4]) {
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <>
struct HalfVec<4> {
  uint2 v;
  __device__ __forceinline__ void load(const uint16_t* p) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  }
  __device__ __forceinline__ uint16_t lane(int e) const {
    const uint32_t w = e < 2 ? v.x : v.y;
    return static_cast<uint16_t>((e & 1) ? (w >> 16) : (w & 0xFFFFu));
  }
  __device__ __forceinline__ static void store(uint16_t* p, const uint32_t (&w)[2]) {
    *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
  }
};

// VE elements per thread and vector.  Alone (the serial step) the kernel is
// latency-bound by the IEEE Adam's instruction count: VE = 4 at 4 CTAs/SM
// (<= 64 registers) runs the G = 2 shard update in 0.72 ms against 0.87 ms
// for VE = 8 at 2 CTAs/SM.  Overlapped with the expand (the pipelined step)
// VE = 8 at 2 CTAs/SM is 1-2% faster: there it is NVLink-bound and more
// resident warps only take issue slots from the expand.
template <int G, bool PUSH, int VE>
__global__ void __launch_bounds__(kThreads, VE == 4 ? 4 : 1) k_shard_p2p(P2PArgs a) {
  __shared__ float red[kThreads / 32];
  __shared__ int last_cta;
  const bool skip = *reinterpret_cast<const volatile float*>(a.flag_slot) != 0.0f;
  const SamoAdamParams prm = step_prm(a.cfg, a.prm);
  const float b1p = __fmul_rn(a.st->beta1_pow, prm.beta1);
  const float b2p = __fmul_rn(a.st->beta2_pow, prm.beta2);
  const float bias1 = __fsub_rn(1.0f, b1p), bias2 = __fsub_rn(1.0f, b2p);
  const float omb1 = __fsub_rn(1.0f, prm.beta1), omb2 = __fsub_rn(1.0f, prm.beta2);
  const float lrwd = __fmul_rn(prm.lr, prm.wd);
  const float scale = pin_f32(a.cfg ? a.cfg->p2p_scale : a.scale);
  const bool bf16 = a.grad_bf16 != 0;
  float nacc = 0.0f;
  const uint64_t n = a.k1 - a.k0;
  const uint64_t nv = (n + VE - 1) / VE;  // VE-element vectors (the last one may be partial)
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; q < nv; q += stride) {
    const uint64_t k = a.k0 + VE * q;
    const uint64_t left = a.k1 - k;
    const int cnt = left < VE ? static_cast<int>(left) : VE;
    HalfVec<VE> h[G];
    if constexpr (PUSH) {  // every rank's contribution is already in the local receive buffer
      const uint16_t* src = a.recv + a.i0 + (k - a.k0);
#pragma unroll
      for (int r = 0; r < G; ++r) h[r].load(src + r * a.rstride);
    } else {
#pragma unroll
      for (int r = 0; r < G; ++r) h[r].load(a.g16[r] + k);  // peer loads; arenas are padded
    }
    float th[VE], mm[VE], vv[VE];
    if (cnt == VE) {
#pragma unroll
      for (int j = 0; j < VE / 4; ++j) {
        const float4 t4 = *reinterpret_cast<const float4*>(a.theta + k + 4 * j);
        const float4 m4 = *reinterpret_cast<const float4*>(a.m + k + 4 * j);
        const float4 v4 = *reinterpret_cast<const float4*>(a.v + k + 4 * j);
        th[4 * j] = t4.x; th[4 * j + 1] = t4.y; th[4 * j + 2] = t4.z; th[4 * j + 3] = t4.w;
        mm[4 * j] = m4.x; mm[4 * j + 1] = m4.y; mm[4 * j + 2] = m4.z; mm[4 * j + 3] = m4.w;
        vv[4 * j] = v4.x; vv[4 * j + 1] = v4.y; vv[4 * j + 2] = v4.z; vv[4 * j + 3] = v4.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < VE; ++e) {
        th[e] = e < cnt ? a.theta[k + e] : 0.0f;
        mm[e] = e < cnt ? a.m[k + e] : 0.0f;
        vv[e] = e < cnt ? a.v[k + e] : 0.0f;
      }
    }
    uint32_t packed[VE / 2];
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      float g = 0.0f;  // rank-ascending fp32 sum, as the oracle's dp_sum
#pragma unroll
      for (int r = 0; r < G; ++r) g = __fadd_rn(g, mul_x86(grad_to_f32(h[r].lane(e), bf16), scale));
      if (e < cnt) nacc = __fadd_rn(nacc, __fmul_rn(g, g));
      float t = th[e];
      if (!skip && e < cnt) t = adam_one(g, mm[e], vv[e], t, prm, omb1, omb2, bias1, bias2, lrwd);
      th[e] = t;
      const uint32_t hb = f32_to_f16_bits(t);
      packed[e >> 1] = (e & 1) ? (packed[e >> 1] | (hb << 16)) : hb;
    }
    if (!skip) {
      if (cnt == VE) {
#pragma unroll
        for (int j = 0; j < VE / 4; ++j) {
          *reinterpret_cast<float4*>(a.theta + k + 4 * j) = make_float4(th[4 * j], th[4 * j + 1], th[4 * j + 2], th[4 * j + 3]);
          *reinterpret_cast<float4*>(a.m + k + 4 * j) = make_float4(mm[4 * j], mm[4 * j + 1], mm[4 * j + 2], mm[4 * j + 3]);
          *reinterpret_cast<float4*>(a.v + k + 4 * j) = make_float4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]);
        }
      } else {
        for (int e = 0; e < cnt; ++e) {
          a.theta[k + e] = th[e];
          a.m[k + e] = mm[e];
          a.v[k + e] = vv[e];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < G; ++r) HalfVec<VE>::store(a.c16[r] + k, packed);  // arenas are padded
  }
  shard_finish<G, kThreads>(a, nacc, red, &last_cta);
}

// Spin on a local signal word written by a peer (acquire, system scope).  A
// peer that never arrives is a dead job: trap after ~30 s rather than hang.
// Limit of a peer wait before the kernel traps (a dead peer): 30 s, raised
// with SAMO_SPIN_TIMEOUT_S for runs that pause a rank (ncu replay on rank 0).
__device__ uint64_t g_spin_limit_ns = 30ull * 1000000000ull;


__device__ void spin_until(const uint64_t* p, uint64_t target) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint32_t ns = 32;
  while (ld_acquire_sys(p) < target) {
    __nanosleep(ns);
    ns = ns < 1024 ? ns * 2 : ns;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > g_spin_limit_ns) __trap();
  }
}

// phase bit 0: publish this rank's skip indicator (and, by the fence, K1's
// pushed gradients) to every rank; bit 1: wait for every rank's and sum them.
__global__ void k_p2p_flag(P2PArgs a, float* flag, int phase) {
  SamoPeerSlots* mine = a.slots[a.rank];
  const uint64_t e = mine->epoch + 1;
  const int q = threadIdx.x;
  if (q < a.G) {
    if (phase & 1) {
      a.slots[q]->flag_val[a.rank] = *flag;
      asm volatile("fence.sc.sys;" ::: "memory");  // K1's grad16 + the value before the signal
      st_release_sys(&a.slots[q]->flag_epoch[a.rank], e);
    }
    if (phase & 2) spin_until(&mine->flag_epoch[q], e);
  }
  __syncwarp();
  if ((phase & 2) && q == 0) {
    float f = 0.0f;  // rank order: every rank computes the same value
    const volatile float* fv = mine->flag_val;
    for (int r = 0; r < a.G; ++r) f = __fadd_rn(f, fv[r]);
    *flag = f;
    __threadfence();
  }
}

__global__ void k_p2p_wait(const SamoPeerSlots* mine, int G, int bucket) {
  const int q = threadIdx.x;
  if (q < G) spin_until(&mine->bucket_epoch[bucket * kMaxP2PRanks + q], mine->epoch + 1);
  __syncwarp();
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

__global__ void k_p2p_epoch(SamoPeerSlots* mine) { mine->epoch += 1; }

__global__ void k_set_step_config(SamoStepConfig* dst, SamoStepConfig v) { *dst = v; }

// One thread: the step's scalars once the global grad norm^2 and skip flag
// are known (AdamScalars::advance, train.hpp:325-329; skip, 632-639).
__global__ void k_step_finalize(SamoStepState* st, const double* norm2, int nslots, float* flag,
                                float beta1, float beta2, const SamoStepConfig* cfg) {
  if (cfg) {
    beta1 = cfg->prm.beta1;
    beta2 = cfg->prm.beta2;
  }
  const bool skip = *flag != 0.0f;
  double acc = 0.0;
  for (int i = 0; i < nslots; ++i) acc += norm2[i];  // fixed order: deterministic
  st->grad_norm = static_cast<float>(sqrt(acc));
  if (skip) {
    st->skipped_steps += 1;
    st->last_skipped = 1u;
  } else {
    st->t += 1;
    st->beta1_pow = __fmul_rn(st->beta1_pow, beta1);
    st->beta2_pow = __fmul_rn(st->beta2_pow, beta2);
    st->last_skipped = 0u;
  }
  *flag = 0.0f;
}

template <typename F>
int grid_for(F fn, size_t smem, int threads = kThreads) {
  SAMO_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
  const char* carve = getenv("SAMO_CARVEOUT");  // tuning override (percent shared)
  if (carve && *carve)
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(carve));
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const char* env = getenv("SAMO_CTAS_PER_SM");  // tuning override
  if (env && *env && atoi(env) > 0 && atoi(env) < per_sm) per_sm = atoi(env);
  return per_sm * num_sms();
}

}  // namespace

// K1 ring depth: three dense tiles up to T = 8192, two above (keeps three
// CTAs resident per SM at T = 16384).
static int k1_stages(uint32_t tile_elems) { return tile_elems <= 8192 ? 3 : 2; }

size_t gather_smem(uint32_t tile_elems, bool) { return k1_stages(tile_elems) * tile_elems * 2u; }

template <bool F32, typename F>
static int with_k1(uint32_t tile_elems, F f) {
  const size_t sm = gather_smem(tile_elems, F32);
  return k1_stages(tile_elems) == 3 ? f(k1_gather<F32, 3>, sm) : f(k1_gather<F32, 2>, sm);
}

// K23 variants (kept elements per stage, ring depth): trades stage depth for
// resident CTAs.  SAMO_K23_VARIANT selects one for tuning.
struct K23Variant {
  int chunk, stages;
};
constexpr K23Variant kK23Variants[] = {{1024, 3}, {1024, 2}, {512, 3}, {512, 4}, {2048, 2}};
constexpr int kK23Default = 0;

static int k23_variant() {
  const char* env = getenv("SAMO_K23_VARIANT");
  const int v = (env && *env) ? atoi(env) : kK23Default;
  return (v >= 0 && v < static_cast<int>(sizeof(kK23Variants) / sizeof(kK23Variants[0]))) ? v
                                                                                           : kK23Default;
}

template <bool G16, int CH, int NS, bool EXPAND = false>
static size_t k23_smem(uint32_t tile_elems) {
  return NS * K23Layout<G16, CH, EXPAND>::kStage + tile_elems * 4u /* two dense out tiles */;
}

// Calls f(kernel, smem) for the selected variant.
template <bool G16, bool CFG, typename F>
static int with_k23(uint32_t tile_elems, F f) {
  const char* env = getenv("SAMO_K23_VARIANT");
  if (!(env && *env)) {
    // Default: 1024-element chunks, three stages when two CTAs still fit per
    // SM (227 KB of shared memory), else two.
    if (k23_smem<G16, 1024, 3>(tile_elems) <= 113u * 1024u)
      return f(k23_update<G16, 1024, 3, false, CFG>, k23_smem<G16, 1024, 3>(tile_elems));
    return f(k23_update<G16, 1024, 2, false, CFG>, k23_smem<G16, 1024, 2>(tile_elems));
  }
  switch (k23_variant()) {
    case 1: return f(k23_update<G16, 1024, 2, false, CFG>, k23_smem<G16, 1024, 2>(tile_elems));
    case 2: return f(k23_update<G16, 512, 3, false, CFG>, k23_smem<G16, 512, 3>(tile_elems));
    case 3: return f(k23_update<G16, 512, 4, false, CFG>, k23_smem<G16, 512, 4>(tile_elems));
    case 4: return f(k23_update<G16, 2048, 2, false, CFG>, k23_smem<G16, 2048, 2>(tile_elems));
    default: return f(k23_update<G16, 1024, 3, false, CFG>, k23_smem<G16, 1024, 3>(tile_elems));
  }
}

int step_grid(int which, bool wide, uint32_t tile_elems) {
  if (which == 0) {
    auto g = [](auto fn, size_t sm) { return grid_for(fn, sm); };
    return wide ? with_k1<true>(tile_elems, g) : with_k1<false>(tile_elems, g);
  }
  auto g = [](auto fn, size_t sm) { return grid_for(fn, sm, kThreads + 32); };
  return wide ? with_k23<false, false>(tile_elems, g) : with_k23<true, false>(tile_elems, g);
}

template <typename F>
static int launch_persistent(F fn, const StepArgs& a, size_t sm, int grid, cudaStream_t s, int threads,
                             const char* what, bool pdl = false) {
  SAMO_CUDA_TRY(
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
  if (static_cast<uint32_t>(grid) > a.ntiles) grid = static_cast<int>(a.ntiles);
  if (pdl) {
    // Programmatic dependent launch: the kernel may start (set up its
    // barriers and shared memory) while the previous one drains; it waits
    // with griddepcontrol.wait before reading that kernel's results.
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SAMO_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, a));
  } else {
    fn<<<grid, threads, sm, s>>>(a);
  }
  SAMO_LAUNCH_CHECK(what);
  return SAMO_OK;
}

int launch_gather(const StepArgs& a, bool out_f32, int grid, cudaStream_t s) {
  if (a.ntiles == 0) return SAMO_OK;
  if (grid <= 0) grid = step_grid(0, out_f32, a.tile_elems);
  auto go = [&](auto fn, size_t sm) {
    return launch_persistent(fn, a, sm, grid, s, kThreads, "k1_gather");
  };
  return out_f32 ? with_k1<true>(a.tile_elems, go) : with_k1<false>(a.tile_elems, go);
}

int launch_update(const StepArgs& a, bool g_f32, int grid, cudaStream_t s) {
  if (a.ntiles == 0) return SAMO_OK;
  if (grid <= 0) grid = step_grid(1, g_f32, a.tile_elems);
  const char* e = getenv("SAMO_PDL");
  const bool pdl = !(e && *e && atoi(e) == 0);
  auto go = [&](auto fn, size_t sm) {
    return launch_persistent(fn, a, sm, grid, s, kThreads + 32, "k23_update", pdl);
  };
  if (a.cfg) return g_f32 ? with_k23<false, true>(a.tile_elems, go) : with_k23<true, true>(a.tile_elems, go);
  return g_f32 ? with_k23<false, false>(a.tile_elems, go) : with_k23<true, false>(a.tile_elems, go);
}

// K123: 1024-element chunks, three stages when two CTAs still fit per SM.
template <int CH, int NS>
static size_t k123_smem(uint32_t tile_elems) {
  return NS * K123Layout<CH>::kStage + kK123Slots * (tile_elems * 2u + tile_elems / 8u);
}
constexpr size_t kSmemTwoPerSM = 111u * 1024u, kSmemOnePerSM = 225u * 1024u;

// Two CTAs of 256 consumer threads per SM when the slots fit twice, else one
// CTA of 512; 0 when even two chunk stages do not fit (the split path runs).
template <bool CFG, typename F>
static int with_k123(uint32_t tile_elems, F f) {
  if (k123_smem<1024, 3>(tile_elems) <= kSmemTwoPerSM)
    return f(k123_step<1024, 3, kThreads, CFG>, k123_smem<1024, 3>(tile_elems), kThreads + 32);
  if (k123_smem<1024, 3>(tile_elems) <= kSmemOnePerSM)
    return f(k123_step<1024, 3, 2 * kThreads, CFG>, k123_smem<1024, 3>(tile_elems), 2 * kThreads + 32);
  if (k123_smem<1024, 2>(tile_elems) <= kSmemOnePerSM)
    return f(k123_step<1024, 2, 2 * kThreads, CFG>, k123_smem<1024, 2>(tile_elems), 2 * kThreads + 32);
  return 0;
}

int fused_grid(uint32_t tile_elems) {
  return with_k123<false>(tile_elems, [](auto fn, size_t sm, int nt) { return grid_for(fn, sm, nt); });
}

int launch_step_fused(const StepArgs& a, int grid, cudaStream_t s) {
  if (a.ntiles == 0) return SAMO_OK;
  if (grid <= 0) grid = fused_grid(a.tile_elems);
  if (grid <= 0) return fail(SAMO_E_PARAMETER, "fused step: tile of %u elements does not fit in shared memory", a.tile_elems);
  const char* e = getenv("SAMO_PDL");
  const bool pdl = !(e && *e && atoi(e) == 0);
  auto go = [&](auto fn, size_t sm, int nt) {
    return launch_persistent(fn, a, sm, grid, s, nt, "k123_step", pdl);
  };
  return a.cfg ? with_k123<true>(a.tile_elems, go) : with_k123<false>(a.tile_elems, go);
}

int launch_step_repair(const StepArgs& a, cudaStream_t s) {
  if (a.ntiles == 0) return SAMO_OK;
  const char* e = getenv("SAMO_PDL");
  const bool pdl = !(e && *e && atoi(e) == 0);
  return launch_persistent(k123_repair, a, 0, num_sms(), s, kThreads, "k123_repair", pdl);
}

int launch_shard_p2p(const P2PArgs& a, cudaStream_t s) {
  if (a.G < 2 || a.G > kMaxP2PRanks) return fail(SAMO_E_PARAMETER, "peer-to-peer exchange supports 2..8 ranks");
  const bool serial = a.bucket < 0;  // alone on the GPU (else overlapped with the expand)
  const uint64_t ve = serial ? 4 : 8;
  const uint64_t nv = (a.k1 > a.k0) ? (a.k1 - a.k0 + ve - 1) / ve : 0;
  const uint64_t cap = a.grid > 0 ? a.grid : static_cast<uint64_t>(num_sms()) * SAMO_P2P_GRID;
  const int grid = static_cast<int>(
      std::max<uint64_t>(1, std::min<uint64_t>(cap, (nv + kThreads - 1) / kThreads)));
#define SAMO_SHARD_CASE(GG)                                                                \
  case GG:                                                                                 \
    if (serial) {                                                                          \
      if (a.push) k_shard_p2p<GG, true, 4><<<grid, kThreads, 0, s>>>(a);                   \
      else k_shard_p2p<GG, false, 4><<<grid, kThreads, 0, s>>>(a);                         \
    } else {                                                                               \
      if (a.push) k_shard_p2p<GG, true, 8><<<grid, kThreads, 0, s>>>(a);                   \
      else k_shard_p2p<GG, false, 8><<<grid, kThreads, 0, s>>>(a);                         \
    }                                                                                      \
    break;
  switch (a.G) {
    SAMO_SHARD_CASE(2)
    SAMO_SHARD_CASE(3)
    SAMO_SHARD_CASE(4)
    SAMO_SHARD_CASE(5)
    SAMO_SHARD_CASE(6)
    SAMO_SHARD_CASE(7)
    SAMO_SHARD_CASE(8)
    default: return fail(SAMO_E_PARAMETER, "peer-to-peer exchange supports 2..8 ranks");
  }
#undef SAMO_SHARD_CASE
  SAMO_LAUNCH_CHECK("k_shard_p2p");
  return SAMO_OK;
}

int launch_p2p_flag(SamoPeerSlots* const* slots, int G, int rank, float* flag, int phase, cudaStream_t s) {
  if (G < 2 || G > kMaxP2PRanks) return fail(SAMO_E_PARAMETER, "peer-to-peer exchange supports 2..8 ranks");
  P2PArgs a{};
  for (int q = 0; q < G; ++q) a.slots[q] = slots[q];
  a.G = G;
  a.rank = rank;
  k_p2p_flag<<<1, 32, 0, s>>>(a, flag, phase);
  SAMO_LAUNCH_CHECK("k_p2p_flag");
  return SAMO_OK;
}

int launch_p2p_wait(const SamoPeerSlots* mine, int G, int bucket, cudaStream_t s) {
  k_p2p_wait<<<1, 32, 0, s>>>(mine, G, bucket);
  SAMO_LAUNCH_CHECK("k_p2p_wait");
  return SAMO_OK;
}

int launch_set_step_config(SamoStepConfig* dst, const SamoStepConfig& v, cudaStream_t s) {
  k_set_step_config<<<1, 1, 0, s>>>(dst, v);
  SAMO_LAUNCH_CHECK("k_set_step_config");
  return SAMO_OK;
}

// Push of compressed binary16 gradients already in `src` (indexed by k) to
// their owners' receive buffers: piece t of a.tiles carries owner pad_ and
// destination offset pad2_ (build_push_tiles), the layout K1's push mode
// writes.  Used after the fused dW sink, whose epilogue gathers locally.
__global__ void __launch_bounds__(kThreads) k_push_copy(StepArgs a, const uint16_t* __restrict__ src) {
  for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const SamoTile td = a.tiles[t];
    if (td.k_end <= td.k_begin) continue;
    SAMO_DCHECK(td.pad_ < static_cast<uint32_t>(kMaxP2PRanks));
    uint16_t* dst = a.push16[td.pad_] + td.pad2_;
    const uint64_t n = td.k_end - td.k_begin;
    for (uint64_t i = threadIdx.x; i < n; i += kThreads) dst[i] = src[td.k_begin + i];
  }
  asm volatile("fence.acq_rel.sys;" ::: "memory");  // peer stores visible system-wide
}

int set_spin_limit_from_env() {
  const char* e = getenv("SAMO_SPIN_TIMEOUT_S");
  if (!e || !*e) return SAMO_OK;
  const uint64_t ns = static_cast<uint64_t>(atof(e) * 1e9);
  SAMO_CUDA_TRY(cudaMemcpyToSymbol(g_spin_limit_ns, &ns, sizeof(ns)));
  return SAMO_OK;
}

int launch_push_copy(const StepArgs& a, const uint16_t* src, cudaStream_t s) {
  if (a.ntiles == 0) return SAMO_OK;
  const int grid = static_cast<int>(std::min<uint32_t>(a.ntiles, 4u * num_sms()));
  k_push_copy<<<grid, kThreads, 0, s>>>(a, src);
  SAMO_LAUNCH_CHECK("k_push_copy");
  return SAMO_OK;
}

int launch_p2p_epoch(SamoPeerSlots* mine, cudaStream_t s) {
  k_p2p_epoch<<<1, 1, 0, s>>>(mine);
  SAMO_LAUNCH_CHECK("k_p2p_epoch");
  return SAMO_OK;
}

int launch_adam_shard(const ShardArgs& a, int grid, cudaStream_t s) {
  if (a.k1 <= a.k0) return SAMO_OK;
  k_adam_shard<<<grid, kThreads, 0, s>>>(a);
  SAMO_LAUNCH_CHECK("k_adam_shard");
  return SAMO_OK;
}

int launch_step_finalize(SamoStepState* st, const double* norm2, int nslots, float* flag,
                         float beta1, float beta2, const SamoStepConfig* cfg, cudaStream_t s) {
  k_step_finalize<<<1, 1, 0, s>>>(st, norm2, nslots, flag, beta1, beta2, cfg);
  SAMO_LAUNCH_CHECK("k_step_finalize");
  return SAMO_OK;
}

int expand_grid(uint32_t tile_elems) {
  return grid_for(k23_update<true, 1024, 3, true>, k23_smem<true, 1024, 3, true>(tile_elems),
                  kThreads + 32);
}

int launch_expand_c16(const StepArgs& a, int grid, cudaStream_t s) {
  if (a.ntiles == 0) return SAMO_OK;
  if (grid <= 0) grid = expand_grid(a.tile_elems);
  return launch_persistent(k23_update<true, 1024, 3, true>, a, k23_smem<true, 1024, 3, true>(a.tile_elems),
                           grid, s, kThreads + 32, "k23_expand");
}

int launch_build_off16(const SamoTile* tiles, uint32_t ntiles, const uint32_t* idx,
                       uint16_t* off16, cudaStream_t s) {
  if (ntiles == 0) return SAMO_OK;
  const int grid = static_cast<int>(ntiles < 8192u ? ntiles : 8192u);
  k_build_off16<<<grid, kThreads, 0, s>>>(tiles, ntiles, idx, off16);
  SAMO_LAUNCH_CHECK("k_build_off16");
  return SAMO_OK;
}

}  // namespace samo_dev
