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
// are MN-major for a contraction over the batch.  Tile 128 x 256 x 64, 3-stage
// TMA ring (128-byte swizzle, 64-element boxes), persistent CTAs with the
// accumulator double-buffered in TMEM:
//   warp 0      TMA producer (one lane)
//   warp 1      TMEM allocation + MMA issue (one lane), tcgen05.commit
//   warps 2..5  epilogue: tcgen05.ld (32 lanes x 32 columns per load), in two
//               128-column halves staged through shared memory
#include "kernels.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

namespace samo_dev {
namespace {

constexpr int kGemmThreads = 192;
constexpr uint32_t kBM = 128, kBK = 64;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
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

// kind::f16 instruction descriptor: fp32 accumulate, f16 A/B, both MN-major.
template <int BN>
constexpr uint32_t umma_idesc() {
  return (1u << 4) | (1u << 15) | (1u << 16) | (static_cast<uint32_t>(BN >> 3) << 17) |
         (static_cast<uint32_t>(kBM >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 32 lanes x 32 consecutive fp32 columns of the accumulator.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
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
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
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

// OR over the 128 epilogue threads (named barrier 1); also orders the
// staging buffer's reads before the next pass overwrites it.
__device__ __forceinline__ int __syncthreads_or_named(uint32_t pred) {
  uint32_t out;
  asm volatile(
      "{\n.reg .pred p, q;\nsetp.ne.u32 p, %1, 0;\nbar.red.or.pred q, 1, 128, p;\nselp.u32 %0, 1, 0, q;\n}\n"
      : "=r"(out)
      : "r"(pred)
      : "memory");
  return static_cast<int>(out);
}

// Shared memory: the epilogue staging half-tile (128 rows x 128 columns,
// padded rows) first, then the NS-stage operand ring (1024-byte aligned for
// the 128-byte swizzle atoms).
template <int BN, int NS>
struct GemmSmem {
  static constexpr uint32_t kA = kBM * kBK * 2;    // two 64(M) x 64(K) boxes
  static constexpr uint32_t kB = BN * kBK * 2;     // BN/64 boxes
  static constexpr uint32_t kStage = kA + kB;
  static constexpr uint32_t kHalf = 128;           // epilogue columns per pass (= kb table granularity)
  static constexpr uint32_t kTileLd = kHalf + 8;   // halves per staging row (16-byte multiple)
  static constexpr uint32_t kTile = kBM * kTileLd * 2;
  static_assert(kTile % 1024 == 0, "stages must stay 1024-byte aligned");
  static constexpr uint32_t kBytes = kTile + NS * kStage;
};

// Persistent: CTA b takes output tiles b, b + grid, ... (M-block fastest, so
// concurrent CTAs share dY column blocks in L2).  The accumulator is double
// buffered in TMEM (2 x BN columns): the epilogue of tile i overlaps the
// mainloop of tile i + 1.
template <int EPI, int BN, int NS>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_dw_gemm(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tdy, DwArgs a) {
  using L = GemmSmem<BN, NS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[NS];
  __shared__ __align__(8) uint64_t empty[NS];
  __shared__ __align__(8) uint64_t accf[2];
  __shared__ __align__(8) uint64_t acce[2];
  __shared__ uint32_t tmem_slot;
  __shared__ uint32_t s_off[kBM + 1];  // epilogue: exclusive scan of kept counts per row
  __shared__ uint32_t s_ks[kBM];       // epilogue: first k of each row in the column half
  __shared__ uint32_t s_wsum[4];

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nk = static_cast<uint32_t>((a.K + kBK - 1) / kBK);
  const uint32_t mt = static_cast<uint32_t>((a.M + kBM - 1) / kBM);
  const uint32_t ntiles = mt * static_cast<uint32_t>((a.N + BN - 1) / BN);
  constexpr uint32_t kCols = 2 * BN;  // two accumulator buffers
  static_assert(kCols == 256 || kCols == 512, "TMEM allocation must be a power of two");
  uint8_t* ring = smem + L::kTile;
  if (threadIdx.x == 0 && (smem_addr(ring) & 1023u)) __trap();  // swizzle atoms need 1024-byte alignment

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 4);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(&tmem_slot)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      uint32_t g = 0;
      for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = static_cast<int>((t % mt) * kBM), n0 = static_cast<int>((t / mt) * BN);
        for (uint32_t kb = 0; kb < nk; ++kb, ++g) {
          const uint32_t s = g % NS;
          if (g >= static_cast<uint32_t>(NS)) mbar_wait_bounded(&empty[s], ((g / NS) - 1) & 1u);
          uint8_t* st = ring + s * L::kStage;
          mbar_arrive_expect_tx(&full[s], L::kStage);  // out-of-bounds box parts are zero-filled and counted
          const int kc = static_cast<int>(kb * kBK);
          tma_load_2d(st, &tx, m0, kc, &full[s]);
          tma_load_2d(st + 8192, &tx, m0 + 64, kc, &full[s]);
#pragma unroll
          for (int c = 0; c < BN / 64; ++c) tma_load_2d(st + L::kA + c * 8192, &tdy, n0 + 64 * c, kc, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issue
      constexpr uint32_t idesc = umma_idesc<BN>();
      uint32_t g = 0, i = 0;
      for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const uint32_t buf = i & 1u;
        if (i >= 2) mbar_wait_bounded(&acce[buf], ((i >> 1) - 1) & 1u);  // epilogue drained this buffer
        tc_fence_after();
        const uint32_t acc = tmem + buf * BN;
        for (uint32_t kb = 0; kb < nk; ++kb, ++g) {
          const uint32_t s = g % NS;
          mbar_wait_bounded(&full[s], (g / NS) & 1u);
          tc_fence_after();
          const uint32_t sa = smem_addr(ring + s * L::kStage), sb = sa + L::kA;
#pragma unroll
          for (uint32_t j = 0; j < kBK / 16; ++j) {  // UMMA_K = 16: 16 K-rows of 128 bytes
            const uint64_t da = umma_desc_mn_sw128(sa + j * 2048, 8192, 1024);
            const uint64_t db = umma_desc_mn_sw128(sb + j * 2048, 8192, 1024);
            umma_f16(acc, da, db, idesc, (kb | j) != 0u);
          }
          umma_commit(&empty[s]);  // frees the stage once these MMAs have read it
        }
        umma_commit(&accf[buf]);   // accumulator of this tile complete
      }
    }
  } else {
    // ---- epilogue (warps 2..5): warp w reads TMEM lanes 32*(w % 4) .. +31
    const uint32_t q = warp & 3u;
    const uint32_t r = q * 32 + lane;  // tile row of this thread
    const uint32_t tid = threadIdx.x - 64;
    uint16_t* tile = reinterpret_cast<uint16_t*>(smem);
    uint32_t i = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const uint32_t buf = i & 1u;
      const uint64_t m0 = static_cast<uint64_t>(t % mt) * kBM;
      const uint32_t nb = t / mt;
      const uint64_t row = m0 + r;
      mbar_wait_bounded(&accf[buf], (i >> 1) & 1u);
      tc_fence_after();
#pragma unroll 1
      for (uint32_t h = 0; h < BN / L::kHalf; ++h) {
        const uint64_t nh = static_cast<uint64_t>(nb) * BN + h * L::kHalf;  // first column of this half
        uint32_t ks = 0, cnt = 0;
        if constexpr (EPI == 1) {  // this row's kept range in the column half (kb: 128-column blocks)
          if (row < a.M && nh < a.N) {
            const uint64_t cb = nh / L::kHalf;
            ks = a.kb[cb * a.M + row];
            cnt = a.kb[(cb + 1) * a.M + row] - ks;
          }
        }
        // accumulator half -> binary16 -> staging row r
#pragma unroll 1
        for (uint32_t c = 0; c < L::kHalf; c += 32) {
          uint32_t v[32];
          tmem_ld32(tmem + ((q * 32u) << 16) + buf * BN + h * L::kHalf + c, v);
          uint4* dst = reinterpret_cast<uint4*>(tile + r * L::kTileLd + c);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint32_t w[4];
#pragma unroll
            for (int z = 0; z < 4; ++z)
              w[z] = f32_to_f16_bits(__uint_as_float(v[8 * e + 2 * z])) |
                     (static_cast<uint32_t>(f32_to_f16_bits(__uint_as_float(v[8 * e + 2 * z + 1]))) << 16);
            dst[e] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
        if (h + 1 == BN / L::kHalf) {  // TMEM buffer drained: the MMA warp may reuse it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acce[buf]);
        }
        if constexpr (EPI == 1) {
          // exclusive scan of the per-row counts over the 128 rows
          uint32_t x = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= static_cast<uint32_t>(o)) x += y;
          }
          if (lane == 31) s_wsum[q] = x;
          s_ks[r] = ks;
          asm volatile("bar.sync 1, 128;" ::: "memory");
          uint32_t base = 0;
          for (uint32_t w = 0; w < q; ++w) base += s_wsum[w];
          s_off[r] = base + x - cnt;
          if (r == kBM - 1) s_off[kBM] = base + x;
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const uint32_t total = s_off[kBM];
          const uint32_t colbase = static_cast<uint32_t>(nh);
          uint32_t bad = 0;
          for (uint32_t f0 = 0; f0 < total; f0 += 4 * 128) {
            uint32_t kk[4], rr[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint32_t f = f0 + u * 128 + tid;
              uint32_t lo = 0, hi = kBM;  // last row with s_off[row] <= f
              while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (s_off[mid] <= f) lo = mid; else hi = mid;
              }
              rr[u] = lo;
              kk[u] = f < total ? s_ks[lo] + (f - s_off[lo]) : 0xFFFFFFFFu;
            }
            uint32_t ix[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) ix[u] = kk[u] != 0xFFFFFFFFu ? __ldg(a.idx + kk[u]) : 0u;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (kk[u] == 0xFFFFFFFFu) continue;
              const uint32_t col = ix[u] - static_cast<uint32_t>((m0 + rr[u]) * a.N) - colbase;
              const uint16_t hv = tile[rr[u] * L::kTileLd + col];
              a.g16[kk[u]] = hv;
              bad |= (hv & 0x7C00u) == 0x7C00u;
            }
          }
          if (__syncthreads_or_named(bad)) {
            if (tid == 0) atomicAdd(a.flag, 1.0f);
          }
        } else {
          asm volatile("bar.sync 1, 128;" ::: "memory");
          // coalesced copy-out of the staged half: warp q writes rows q, q + 4, ...
          for (uint32_t rr = q; rr < kBM; rr += 4) {
            const uint64_t grow = m0 + rr;
            const uint64_t col = nh + lane * 4;
            if (grow < a.M && col < a.N) {
              const uint2 v = *reinterpret_cast<const uint2*>(tile + rr * L::kTileLd + lane * 4);
              *reinterpret_cast<uint2*>(a.dw + grow * a.N + col) = v;
            }
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols) : "memory");
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
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q{};
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// [rows x cols] row-major binary16, box 64 (cols, inner) x 64 (rows), 128-byte swizzle.
int make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SAMO_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, 64};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SAMO_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return SAMO_OK;
}

constexpr int kGemmBN = 256;
constexpr int kGemmNS = 3;
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

int launch_dw_gemm(const uint16_t* x, const uint16_t* dy, const DwArgs& a, int epi, cudaStream_t s) {
  CUtensorMap tx, tdy;
  SAMO_TRY(make_map(&tx, x, a.K, a.M));
  SAMO_TRY(make_map(&tdy, dy, a.K, a.N));
  const uint64_t tiles = ((a.M + kBM - 1) / kBM) * ((a.N + kGemmBN - 1) / kGemmBN);
  const int grid = static_cast<int>(std::min<uint64_t>(tiles, static_cast<uint64_t>(num_sms())));
  constexpr uint32_t smem = GemmSmem<kGemmBN, kGemmNS>::kBytes;
  if (epi == 0) {
    auto fn = k_dw_gemm<0, kGemmBN, kGemmNS>;
    SAMO_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    fn<<<grid, kGemmThreads, smem, s>>>(tx, tdy, a);
  } else {
    auto fn = k_dw_gemm<1, kGemmBN, kGemmNS>;
    SAMO_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    fn<<<grid, kGemmThreads, smem, s>>>(tx, tdy, a);
  }
  SAMO_LAUNCH_CHECK("k_dw_gemm");
  return SAMO_OK;
}

}  // namespace samo_dev
