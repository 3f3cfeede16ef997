// Weight-gradient GEMM dW = X^T . dY on the 5th-generation tensor cores, with
// the SAMO gather fused into its epilogue (PAPER.md:883-888:
// "fusing the compression operation with the backward pass kernels").
//
// Reference: mlp_backward (train.hpp:304-305) computes
//   dw = matmul(transpose(acts[l]), d)     [in x out], binary16
// and hands it to the trainer's sink, which gathers the kept positions into
// grad16 (train.hpp:596-611).  matmul (tensor.hpp:88-105) accumulates exact
// half x half products in fp32 and rounds once to binary16.  Here the
// products are accumulated by tcgen05.mma (fp32 accumulator in TMEM, a
// different addition order: tolerance vs the reference) and
// the epilogue either stores the dense binary16 dW (EPI 0), or gathers only
// the kept elements into the model's compressed binary16 gradient arena and
// raises the skip flag (EPI 1): the 2*phi dense gradient never reaches HBM.
// EPI 1 is bit-identical to EPI 0 followed by the K1 gather.
//
// Operands: X [batch x in] and dY [batch x out], row-major binary16, so both
// are MN-major for a contraction over the batch.  Persistent CTA pairs
// (cta_group::2) on 256 x 256 x 64 tiles, a 5-stage TMA ring per SM
// (128-byte swizzle, 64-element boxes), the accumulator double-buffered in
// TMEM:
//   warp 0      TMA producer (one lane; both CTAs complete on the leader's barrier)
//   warp 1      TMEM allocation; MMA issue by one lane of the leader CTA
//   warps 2..5  epilogue: tcgen05.ld (32 lanes x 32 columns per load), in two
//               128-column halves; each thread owns one accumulator row
// Long K uses 512 x 256 pair tiles (MS = 2, both accumulators in TMEM) or
// 256 x 384 ones (BN = 384) where they fill the waves better; see
// launch_dw_gemm.  Measured (tools/bench_dw.py): 1.09-1.39
// PFLOP/s on the GPT-2.7B layer shapes at 4096-8192 tokens, 77-102% of
// cuBLAS; the fused sink is within +-5% of the dense GEMM followed by the K1
// gather.
#include "kernels.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

namespace samo_dev {
namespace {

// warps: producer, MMA, then EW groups of four epilogue warps
constexpr int gemm_threads(int ew) { return 64 + 128 * ew; }
constexpr uint32_t kBM = 128, kBK = 64;
constexpr uint32_t kBox = 64 * kBK * 2;  // one 64-element x kBK-row TMA box (LBO between MN chunks)

// 2-SM form: the completion may signal the mbarrier of the peer CTA (bar is a
// shared::cluster address, e.g. from mapa).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}

__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t ncluster_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}

// Shared-memory matrix descriptor, MN-major, 128-byte swizzle (canonical
// layout ((8,n),(8,k)) : ((1,LBO),(8,SBO)) in 16-byte units): LBO = bytes
// between 64-element MN chunks, SBO = bytes between 8-row K groups.
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // descriptor version (Blackwell)
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: fp32 accumulate, f16 A/B, both MN-major,
// M x N (M = 256: the CTA pair, 128 rows per SM).
template <int M, int N>
constexpr uint32_t umma_idesc() {
  return (1u << 4) | (1u << 15) | (1u << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void umma_f16_pair(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit_pair_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_addr(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 32 lanes x 32 consecutive fp32 columns of the accumulator, without the
// wait, so several loads are in flight at once;
// tmem_wait32 then waits and ties the registers to the wait ("+r"), so no use
// of them can be scheduled before it.
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait32(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                 "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
                 "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]),
                 "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]),
                 "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// Bounded mbarrier wait for the GEMM pipeline: a protocol bug traps (an
// error at the next sync) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint64_t spin = 0;; ++spin) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (spin > (1ull << 26)) __trap();
  }
}

// Work units of the persistent schedule: pair tiles [0, tail0) whole
// (256 x BN), then every remaining tile as two 256 x BN/2 halves, so that a
// last wave of r < #pairs / 2 tiles keeps 2r pairs busy for about half as
// long instead of r pairs for a whole tile (launch_dw_gemm picks tail0).
struct DwUnit {
  uint32_t mpair, n0, width;  // M-block pair, first column, columns (BN or BN / 2)
};
template <int BN>
__device__ __forceinline__ DwUnit dw_unit(uint32_t u, uint32_t tail0, uint32_t mp) {
  uint32_t pt = u, n0 = 0, width = BN;
  if (u >= tail0) {
    pt = tail0 + (u - tail0) / 2;
    n0 = ((u - tail0) & 1u) * (BN / 2);
    width = BN / 2;
  }
  return DwUnit{pt % mp, (pt / mp) * BN + n0, width};
}

// Shared memory: the epilogue staging half-tile (128 rows x 128 columns,
// padded rows) first, then the NS-stage operand ring (1024-byte aligned for
// the 128-byte swizzle atoms).
constexpr bool kStage_check(uint32_t a, uint32_t b) { return (a + b) % 1024 == 0; }

template <int BN, int NS, int EW, int MS = 1>
struct GemmSmem {
  static constexpr uint32_t kA = MS * kBM * kBK * 2;  // per M sub-tile two 64(M) x kBK(K) boxes
  static constexpr uint32_t kB = (BN / 2) * kBK * 2;  // this SM's half of B: BN/128 boxes
  static_assert(kStage_check(kA, kB), "stage sizes keep 1024-byte alignment");
  static constexpr uint32_t kStage = kA + kB;
  static constexpr uint32_t kHalf = 128;           // epilogue columns per pass (= kb table granularity)
  static constexpr uint32_t kTileLd = kHalf + 8;   // halves per staging row (16-byte multiple)
  static constexpr uint32_t kTile = kBM * kTileLd * 2;
  static_assert(kTile % 1024 == 0, "stages must stay 1024-byte aligned");
  static constexpr uint32_t kBytes = EW * kTile + NS * kStage;  // one staging half-tile per epilogue group
};

// Persistent CTA pairs (cluster of two, tcgen05 cta_group::2): pair c takes
// 256 x BN output tiles c, c + #pairs, ... (M fastest).  Each SM holds its
// 128 rows of X (A) and half of the dY (B) columns of every k-block; the
// leader CTA issues the 256 x BN x 16 MMAs for both, each SM accumulates its
// 128 rows in its own TMEM.  Per SM and k-block: 32 KB of shared-memory fill
// and half the operand reads of a one-SM 128 x BN tile (shared-memory
// bandwidth is what bounds the one-SM form).  Both CTAs' TMA loads complete
// on the leader's full barrier; the leader's commits free the stage in both
// CTAs and publish the accumulator to both epilogues, whose drain arrivals
// (4 * EW warps per CTA) gate the reuse of a TMEM buffer.  The accumulator is double
// buffered (2 x BN columns): the epilogue of tile i overlaps the mainloop of
// tile i + 1.
// EW = 2: two epilogue groups work on the two 128-column halves at once
// (short-K problems, where the epilogue would pace the mainloop).
// MS = 2: a pair tile is 512 x BN — two 256-row M sub-tiles that share every
// dY stage (per SM and k-block 48 KB of fill for twice the MMAs: 25% fewer
// operand bytes per flop, the bound of the MS = 1 form at 256 x 256, DESIGN
// §7c).  Both accumulators fill the 512 TMEM columns, so there is one
// buffer and the epilogue does not overlap the next tile's mainloop.
// BN = 384 (MS = 1): a 256 x 384 pair tile, issued as two MMAs per k-step
// that share the A operand — N = 128 (each SM holds 64 dY columns: one box)
// then N = 256 (128 columns: two boxes) — so each SM's B is three whole
// 64-column boxes and TMEM column c is output column n0 + c.  384 columns
// leave no room for a second buffer: like MS = 2 the epilogue does not
// overlap.  It fills the waves where neither 256-wide form does (2560 x 2560:
// 70 tiles on 74 pairs against 50 or 100), at 40 KB of fill per SM and
// k-block for 1.5x the MMAs of a 256 x 256 tile.
template <int EPI, int BN, int NS, int EW, int MS>
__global__ void __launch_bounds__(gemm_threads(EW), 1)
    k_dw_gemm(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tdy, DwArgs a) {
  using L = GemmSmem<BN, NS, EW, MS>;
  static_assert(MS == 1 || MS == 2, "one or two M sub-tiles");
  static_assert(BN == 256 || (BN == 384 && MS == 1), "256-wide tiles, or the 384-wide form with MS = 1");
  constexpr bool kWide = BN == 384;
  constexpr uint32_t NBUF = (MS == 1 && !kWide) ? 2 : 1;  // accumulator buffers
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[NS];
  __shared__ __align__(8) uint64_t empty[NS];
  __shared__ __align__(8) uint64_t accf[2];
  __shared__ __align__(8) uint64_t acce[2];
  __shared__ uint32_t tmem_slot;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nk = static_cast<uint32_t>((a.K + kBK - 1) / kBK);
  const uint32_t mt = static_cast<uint32_t>((a.M + kBM - 1) / kBM);
  const uint32_t mp = (mt + 2 * MS - 1) / (2 * MS);  // pair tiles along M
  const uint32_t ntiles = mp * static_cast<uint32_t>((a.N + BN - 1) / BN);
  const uint32_t tail0 = a.tail0 < ntiles ? a.tail0 : ntiles;
  const uint32_t nunits = tail0 + 2 * (ntiles - tail0);
  const uint32_t crank = cluster_ctarank(), cid = cluster_id_x(), ncl = ncluster_x();
  constexpr uint32_t kCols = NBUF * MS * BN <= 256 ? 256 : 512;  // a power of two
  static_assert(NBUF * MS * BN <= 512, "accumulators exceed TMEM");
  uint8_t* ring = smem + EW * L::kTile;
  if (threadIdx.x == 0 && (smem_addr(ring) & 1023u)) __trap();  // swizzle atoms need 1024-byte alignment

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);   // leader: its producer's arrive (+ both CTAs' bytes)
      mbar_init(&empty[s], 1);  // the leader's MMA commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 8 * EW);  // leader: the epilogue warps of both CTAs
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(&tmem_slot)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs), completing on the leader's full barrier
      uint32_t g = 0;
      for (uint32_t u = cid; u < nunits; u += ncl) {
        const DwUnit t = dw_unit<BN>(u, tail0, mp);
        const int n0 = static_cast<int>(t.n0 + crank * (t.width / 2));  // my half of the columns
        const uint32_t boxes = t.width / 128;                          // 64-column dY boxes per CTA
        // wide form: my 64 columns of the N = 128 MMA, then my 128 of the N = 256 one
        const int nb0 = static_cast<int>(t.n0 + crank * 64), nb1 = static_cast<int>(t.n0 + 128 + crank * 128);
        for (uint32_t kb = 0; kb < nk; ++kb, ++g) {
          const uint32_t s = g % NS;
          if (g >= static_cast<uint32_t>(NS)) mbar_wait_bounded(&empty[s], ((g / NS) - 1) & 1u);
          uint8_t* st = ring + s * L::kStage;
          const uint32_t fb = mapa_shared(smem_addr(&full[s]), 0);
          if (crank == 0) mbar_arrive_expect_tx(&full[s], 2 * (L::kA + boxes * kBox));  // both CTAs (OOB parts count)
          const int kc = static_cast<int>(kb * kBK);
#pragma unroll
          for (int j = 0; j < MS; ++j) {  // my 128 rows of each M sub-tile
            const int m0 = static_cast<int>((2 * (MS * t.mpair + j) + crank) * kBM);
            tma_load_2d_pair(st + 2 * j * kBox, &tx, m0, kc, fb);
            tma_load_2d_pair(st + (2 * j + 1) * kBox, &tx, m0 + 64, kc, fb);
          }
          if constexpr (kWide) {
            tma_load_2d_pair(st + L::kA, &tdy, nb0, kc, fb);
            tma_load_2d_pair(st + L::kA + kBox, &tdy, nb1, kc, fb);
            tma_load_2d_pair(st + L::kA + 2 * kBox, &tdy, nb1 + 64, kc, fb);
          } else {
            for (uint32_t c = 0; c < boxes; ++c) tma_load_2d_pair(st + L::kA + c * kBox, &tdy, n0 + 64 * c, kc, fb);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {  // ---- MMA issue (leader)
      constexpr uint32_t idesc_full = umma_idesc<2 * kBM, kWide ? 256 : BN>(),
                         idesc_half = umma_idesc<2 * kBM, kWide ? 128 : BN / 2>();
      uint32_t g = 0, i = 0;
      for (uint32_t u = cid; u < nunits; u += ncl, ++i) {
        const uint32_t idesc = u < tail0 ? idesc_full : idesc_half;
        const uint32_t buf = i % NBUF;
        if (i >= NBUF) mbar_wait_bounded(&acce[buf], ((i / NBUF) - 1) & 1u);  // both epilogues drained it
        tc_fence_after();
        const uint32_t acc = tmem + buf * MS * BN;
        for (uint32_t kb = 0; kb < nk; ++kb, ++g) {
          const uint32_t s = g % NS;
          mbar_wait_bounded(&full[s], (g / NS) & 1u);
          tc_fence_after();
          const uint32_t sa = smem_addr(ring + s * L::kStage), sb = sa + L::kA;
#pragma unroll
          for (uint32_t kk = 0; kk < kBK / 16; ++kk) {  // UMMA_K = 16: 16 K-rows of 128 bytes
            if constexpr (kWide) {  // columns [0, 128) from box 0, [128, 384) from boxes 1-2
              const uint64_t da = umma_desc_mn_sw128(sa + kk * 2048, kBox, 1024);
              umma_f16_pair(acc, da, umma_desc_mn_sw128(sb + kk * 2048, kBox, 1024), idesc_half,
                            (kb | kk) != 0u);
              umma_f16_pair(acc + 128, da, umma_desc_mn_sw128(sb + kBox + kk * 2048, kBox, 1024), idesc_full,
                            (kb | kk) != 0u);
            } else {
              const uint64_t db = umma_desc_mn_sw128(sb + kk * 2048, kBox, 1024);
#pragma unroll
              for (uint32_t j = 0; j < static_cast<uint32_t>(MS); ++j) {
                const uint64_t da = umma_desc_mn_sw128(sa + 2 * j * kBox + kk * 2048, kBox, 1024);
                umma_f16_pair(acc + j * BN, da, db, idesc, (kb | kk) != 0u);
              }
            }
          }
          umma_commit_pair_mc(&empty[s], 0x3);  // frees the stage in both CTAs
        }
        umma_commit_pair_mc(&accf[buf], 0x3);   // accumulator complete in both CTAs
      }
    }
  } else {
    // ---- epilogue (warps 2..): warp w reads TMEM lanes 32*(w % 4) .. +31;
    // group gx = (w - 2) / 4 takes the halves gx, gx + EW, ...
    const uint32_t q = warp & 3u;
    const uint32_t r = q * 32 + lane;  // tile row of this thread
    const uint32_t gx = (warp - 2) >> 2;
    uint16_t* tile = reinterpret_cast<uint16_t*>(smem + gx * L::kTile);
    uint32_t i = 0;
    for (uint32_t u = cid; u < nunits; u += ncl, ++i) {
      const uint32_t buf = i % NBUF;
      const DwUnit t = dw_unit<BN>(u, tail0, mp);
      const uint32_t nhalves = t.width / L::kHalf;
      mbar_wait_bounded(&accf[buf], (i / NBUF) & 1u);
      tc_fence_after();
      if (gx >= nhalves) {  // nothing of this unit for this group: release the buffer at once
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_addr(&acce[buf]), 0));
        continue;
      }
#pragma unroll 1
      for (uint32_t sub = 0; sub < static_cast<uint32_t>(MS); ++sub) {
      const uint64_t m0 = static_cast<uint64_t>(2 * (MS * t.mpair + sub) + crank) * kBM;
      const uint64_t row = m0 + r;
      const uint32_t tcol = (buf * MS + sub) * BN;  // this sub-tile's accumulator columns
#pragma unroll 1
      for (uint32_t h = gx; h < nhalves; h += EW) {
        const uint64_t nh = static_cast<uint64_t>(t.n0) + h * L::kHalf;  // first column of this half
        uint32_t ks = 0, cnt = 0;
        if constexpr (EPI == 1) {  // this row's kept range in the column half (kb: 128-column blocks)
          if (row < a.M && nh < a.N) {
            const uint64_t cb = nh / L::kHalf;
            ks = a.kb[cb * a.M + row];
            cnt = a.kb[(cb + 1) * a.M + row] - ks;
          }
        }
        // accumulator half -> binary16 -> staging row r: kLd 32-column loads
        // in flight together, one wait (4 = the whole half; 2 with three
        // epilogue groups, whose 448 threads get at most 128 registers)
        constexpr uint32_t kLd = EW >= 3 ? 2 : 4;
#pragma unroll
        for (uint32_t c0 = 0; c0 < L::kHalf / 32; c0 += kLd) {
          uint32_t v[kLd][32];
#pragma unroll
          for (uint32_t cc = 0; cc < kLd; ++cc)
            tmem_ld32_nowait(tmem + ((q * 32u) << 16) + tcol + h * L::kHalf + (c0 + cc) * 32, v[cc]);
#pragma unroll
          for (uint32_t cc = 0; cc < kLd; ++cc) {
            tmem_wait32(v[cc]);
            uint4* dst = reinterpret_cast<uint4*>(tile + r * L::kTileLd + (c0 + cc) * 32);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              uint32_t w[4];
#pragma unroll
              for (int z = 0; z < 4; ++z)
                w[z] = f32x2_to_f16x2_bits(__uint_as_float(v[cc][8 * e + 2 * z]),
                                           __uint_as_float(v[cc][8 * e + 2 * z + 1]));
              dst[e] = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
        if (sub + 1 == MS && h + EW >= nhalves) {  // this group's last half: TMEM drained for it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_addr(&acce[buf]), 0));
        }
        if constexpr (EPI == 1) {
          // Gather of this thread's own row (TMEM lane = tile row): its kept
          // elements in the half are the arena range [ks, ks + cnt), read
          // back from the row it just staged, so no barrier is needed.
          const uint16_t* mine = tile + r * L::kTileLd;
          const uint32_t colbase = static_cast<uint32_t>(row * a.N + nh);
          uint32_t bad = 0;
          for (uint32_t j = 0; j < cnt; j += 4) {
            uint32_t ix[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) ix[u] = j + u < cnt ? __ldg(a.idx + ks + j + u) : colbase;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (j + u < cnt) {
                SAMO_DCHECK(ix[u] >= colbase && ix[u] - colbase < L::kHalf);
                const uint16_t hv = mine[ix[u] - colbase];
                a.g16[ks + j + u] = hv;
                bad |= (hv & 0x7C00u) == 0x7C00u;
              }
            }
          }
          if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicAdd(a.flag, 1.0f);
        } else {
          asm volatile("bar.sync %0, 128;" ::"r"(1 + gx) : "memory");
          // coalesced copy-out of the staged half: warp q writes rows q, q + 4, ...
          for (uint32_t rr = q; rr < kBM; rr += 4) {
            const uint64_t grow = m0 + rr;
            const uint64_t col = nh + lane * 4;
            if (grow < a.M && col < a.N) {
              const uint2 v = *reinterpret_cast<const uint2*>(tile + rr * L::kTileLd + lane * 4);
              *reinterpret_cast<uint2*>(a.dw + grow * a.N + col) = v;
            }
          }
          asm volatile("bar.sync %0, 128;" ::"r"(1 + gx) : "memory");
        }
      }
      }  // M sub-tiles
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync_all();  // no CTA exits while its peer may still signal or multicast into it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols) : "memory");
  }
}

// kb[b * M + i] = first layer-local k with idx[k] >= i * N + min(b * BN, N).
__global__ void k_build_rowblocks(const uint32_t* idx, uint64_t n, uint64_t M, uint64_t N, uint32_t BN,
                                  uint32_t nb, uint32_t* kb) {
  const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (t >= (nb + 1ull) * M) return;
  const uint64_t b = t / M, i = t % M;
  const uint64_t key = i * N + (b * BN < N ? b * BN : N);
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (idx[mid] < key) lo = mid + 1; else hi = mid;
  }
  kb[t] = static_cast<uint32_t>(lo);
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {  // thread-safe one-time lookup
    cudaDriverEntryPointQueryResult q{};
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
  return fn;
}

// [rows x cols] row-major binary16, box 64 (cols, inner) x kBK (rows), 128-byte swizzle.
int make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SAMO_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, kBK};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SAMO_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return SAMO_OK;
}

constexpr int kGemmBN = 256;
constexpr int kGemmNS = 5;
constexpr uint32_t kKbCols = 128;  // column granularity of the row/column-block k table

}  // namespace

int dw_check(uint64_t batch, uint64_t in, uint64_t out, const void* x, const void* dy) {
  if (batch == 0 || in == 0 || out == 0) return fail(SAMO_E_DIMENSION, "dW GEMM: empty operand");
  if (in % 8 || out % 8)
    return fail(SAMO_E_DIMENSION, "dW GEMM: in (%llu) and out (%llu) must be multiples of 8",
                static_cast<unsigned long long>(in), static_cast<unsigned long long>(out));
  if (batch >= (1ull << 31) || in >= (1ull << 31) || out >= (1ull << 31) || in * out >= (1ull << 32))
    return fail(SAMO_E_DIMENSION, "dW GEMM: operand too large");
  if (!x || !dy) return fail(SAMO_E_PARAMETER, "dW GEMM: null operand");
  if (reinterpret_cast<uintptr_t>(x) % 16 || reinterpret_cast<uintptr_t>(dy) % 16)
    return fail(SAMO_E_PARAMETER, "dW GEMM: operands must be 16-byte aligned");
  return SAMO_OK;
}

uint32_t dw_col_blocks(uint64_t out) { return static_cast<uint32_t>((out + kKbCols - 1) / kKbCols); }

int launch_build_rowblocks(const uint32_t* idx, uint64_t n, uint64_t in, uint64_t out, uint32_t* kb,
                           cudaStream_t s) {
  const uint32_t nb = dw_col_blocks(out);
  const uint64_t total = (nb + 1ull) * in;
  const int grid = static_cast<int>((total + 255) / 256);
  k_build_rowblocks<<<grid, 256, 0, s>>>(idx, n, in, out, kKbCols, nb, kb);
  SAMO_LAUNCH_CHECK("k_build_rowblocks");
  return SAMO_OK;
}

// Tensor maps are encoded on the host (cuTensorMapEncodeTiled, ~µs each);
// a small cache keyed by (base, rows, cols) keeps repeated launches on the
// same operands — every training step — free of that host work.
static int cached_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols) {
  struct Entry {
    const void* base;
    uint64_t rows, cols;
    CUtensorMap map;
  };
  static thread_local Entry cache[16];
  static thread_local unsigned next = 0;
  for (const Entry& e : cache)
    if (e.base == base && e.rows == rows && e.cols == cols && base) {
      *m = e.map;
      return SAMO_OK;
    }
  SAMO_TRY(make_map(m, base, rows, cols));
  cache[next % 16] = Entry{base, rows, cols, *m};
  ++next;
  return SAMO_OK;
}

int launch_dw_gemm(const uint16_t* x, const uint16_t* dy, const DwArgs& a, int epi, cudaStream_t s) {
  CUtensorMap tx, tdy;
  SAMO_TRY(cached_map(&tx, x, a.K, a.M));
  SAMO_TRY(cached_map(&tdy, dy, a.K, a.N));
  // Variants: short K (<= 16 k-blocks per tile) -> two epilogue groups,
  // 256 x 256 pair tiles (one stage less); long K -> 512 x 256 pair tiles
  // (MS = 2, two epilogue groups, 3 stages of 48 KB; SAMO_DW_MS2_EW=1: one
  // group, 4 stages, 0.6-7% slower) or 256 x 256 (MS = 1, 5 stages).
  auto env_on = [](const char* name, int dflt) {
    const char* e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
  };
  const int ew = env_on("SAMO_DW_EW", 0);  // tuning override: 1 or 2 epilogue groups
  const bool short_k = ew ? ew == 2 : a.K <= 16 * kBK;
  // MS = 2 fills its waves worse (half as many tiles) and exposes its
  // epilogue, so it is taken when its last wave is >= 85% full and K spans
  // >= 48 k-blocks, or when it fits in one wave where MS = 1 needs two
  // (measured on 10 shapes; SAMO_DW_MS=1/2 forces a form).
  const uint64_t P = static_cast<uint64_t>(num_sms() / 2);
  const uint64_t ncol = (a.N + kGemmBN - 1) / kGemmBN, nkb = (a.K + kBK - 1) / kBK;
  const uint64_t t1 = ((a.M + 2 * kBM - 1) / (2 * kBM)) * ncol, t2 = ((a.M + 4 * kBM - 1) / (4 * kBM)) * ncol;
  const double fill2 = static_cast<double>(t2) / static_cast<double>(((t2 + P - 1) / P) * P);
  const bool auto2 = (fill2 >= 0.85 && nkb >= 48) || (t2 <= P && t1 > P);
  const int ms_env = env_on("SAMO_DW_MS", 0);
  // ms 3: the 256 x 384 pair tile.  Taken when its waves cost less than the
  // form picked above, in units of a 256 x 256 tile-time: MS = 2 tiles are 2
  // units, MS = 1 tiles 1 unit at 0.91 of MS = 2's rate (a split tail half
  // a wave), 384-wide tiles 1.5 units at 0.93 (measured rates).
  // Interleaved A/B: -10% on qkv (2560 x 7680), -9% on attn out (2560 x 2560),
  // never chosen where it lost (SAMO_DW_MS=3 forces it).
  const uint64_t t3 = ((a.M + 2 * kBM - 1) / (2 * kBM)) * ((a.N + 383) / 384);
  const bool tail_on = env_on("SAMO_DW_TAIL", 1) != 0;
  const uint64_t r1 = t1 % P;
  const double cost1 = (static_cast<double>(t1 / P) + (r1 ? (2 * r1 <= P && tail_on ? 0.5 : 1.0) : 0.0)) / 0.91;
  const double cost2 = static_cast<double>((t2 + P - 1) / P) * 2.0;
  const double cost3 = static_cast<double>((t3 + P - 1) / P) * 1.5 / 0.93;
  int ms = short_k ? 1 : (ms_env >= 1 && ms_env <= 3) ? ms_env : (auto2 ? 2 : 1);
  if (!short_k && ms_env == 0 && cost3 < (ms == 2 ? cost2 : cost1)) ms = 3;
  // Tail split (MS = 1): a last partial wave of r tiles with 2r <= #pairs
  // runs as 2r half tiles (SAMO_DW_TAIL=0 turns it off, for A/B).
  const uint64_t tiles = ms == 2 ? t2 : ms == 3 ? t3 : t1;
  const uint64_t r = tiles % P;
  DwArgs args = a;
  args.tail0 = static_cast<uint32_t>(tiles);
  if (ms == 1 && r > 0 && 2 * r <= P && tail_on) args.tail0 = static_cast<uint32_t>(tiles - r);
  const uint64_t units = args.tail0 + 2 * (tiles - args.tail0);
  const int grid = 2 * static_cast<int>(std::min<uint64_t>(units, P));
  using F = void (*)(CUtensorMap, CUtensorMap, DwArgs);
  F fn;
  uint32_t smem;
  int threads, variant;
  if (short_k) {
    fn = epi == 0 ? k_dw_gemm<0, kGemmBN, 4, 2, 1> : k_dw_gemm<1, kGemmBN, 4, 2, 1>;
    smem = GemmSmem<kGemmBN, 4, 2>::kBytes;
    threads = gemm_threads(2);
    variant = 0;
  } else if (ms == 1) {
    fn = epi == 0 ? k_dw_gemm<0, kGemmBN, kGemmNS, 1, 1> : k_dw_gemm<1, kGemmBN, kGemmNS, 1, 1>;
    smem = GemmSmem<kGemmBN, kGemmNS, 1>::kBytes;
    threads = gemm_threads(1);
    variant = 1;
  } else if (ms == 3 && env_on("SAMO_DW_W_EW", 3) == 3) {
    // three epilogue groups, one 128-column half each: the one-buffer
    // epilogue drains in a third of the time (interleaved A/B: +6% on qkv,
    // +10% on attn out over two groups; SAMO_DW_W_EW=1/2 for A/B)
    fn = epi == 0 ? k_dw_gemm<0, 384, 3, 3, 1> : k_dw_gemm<1, 384, 3, 3, 1>;
    smem = GemmSmem<384, 3, 3, 1>::kBytes;
    threads = gemm_threads(3);
    variant = 6;
  } else if (ms == 3 && env_on("SAMO_DW_W_EW", 3) == 1) {
    fn = epi == 0 ? k_dw_gemm<0, 384, 4, 1, 1> : k_dw_gemm<1, 384, 4, 1, 1>;
    smem = GemmSmem<384, 4, 1, 1>::kBytes;
    threads = gemm_threads(1);
    variant = 4;
  } else if (ms == 3) {
    fn = epi == 0 ? k_dw_gemm<0, 384, 3, 2, 1> : k_dw_gemm<1, 384, 3, 2, 1>;
    smem = GemmSmem<384, 3, 2, 1>::kBytes;
    threads = gemm_threads(2);
    variant = 5;
  } else if (env_on("SAMO_DW_MS2_EW", 2) != 2) {
    fn = epi == 0 ? k_dw_gemm<0, kGemmBN, 4, 1, 2> : k_dw_gemm<1, kGemmBN, 4, 1, 2>;
    smem = GemmSmem<kGemmBN, 4, 1, 2>::kBytes;
    threads = gemm_threads(1);
    variant = 2;
  } else {
    fn = epi == 0 ? k_dw_gemm<0, kGemmBN, 3, 2, 2> : k_dw_gemm<1, kGemmBN, 3, 2, 2>;
    smem = GemmSmem<kGemmBN, 3, 2, 2>::kBytes;
    threads = gemm_threads(2);
    variant = 3;
  }
  // The shared-memory opt-in is per device: remember it per (device, kernel).
  static bool attr_set[64][16] = {};
  int dev = 0;
  SAMO_CUDA_TRY(cudaGetDevice(&dev));
  const int slot = (epi != 0) + 2 * variant;
  if (dev < 0 || dev >= 64 || !attr_set[dev][slot]) {
    SAMO_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (dev >= 0 && dev < 64) attr_set[dev][slot] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SAMO_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, tx, tdy, args));
  SAMO_LAUNCH_CHECK("k_dw_gemm");
  return SAMO_OK;
}

}  // namespace samo_dev
