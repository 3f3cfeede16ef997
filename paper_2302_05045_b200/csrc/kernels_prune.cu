// kernels_prune.cu — K0: magnitude_prune on the device (prune.hpp:99-170).
//
// The reference keeps, per problem (one prunable layer in per_layer scope,
// all prunable layers together in global scope), the `keep` elements that
// come first under the total order (|v| desc, layer asc, index asc)
// (prune.hpp:87-91, 132-138), then returns each layer's kept indices sorted
// ascending (prune.hpp:140, 166-168).  With key = bits(|v|) (monotone for
// non-NaN floats) that set is
//     { key > T }  ∪  { the first need_eq elements, in concatenation order,
//                       with key == T }
// where T is the keep-th largest key.  So instead of sorting:
//   1. radix-select T: three histogram passes over the 31-bit key (11/11/10
//      bit digits), each followed by a one-block digit selection;
//   2. count key>T and key==T per chunk;
//   3. one ordered scan over the chunks (equal-key ranks per problem, output
//      offsets per layer);
//   4. an order-preserving compaction that writes the layer-local indices —
//      already ascending, so no final sort is needed.
// Non-prunable layers are problems with keep == len (iota, prune.hpp:117-120).
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

#include <cub/block/block_scan.cuh>

namespace samo_dev {
namespace {

constexpr int kChunk = 16384;       // elements per chunk (chunks never span layers)
constexpr int kPT = 256;            // threads per CTA
constexpr int kBins = 2048;

struct PSeg {            // one layer inside a problem
  const float* values;
  uint32_t* out;
  uint64_t len;
  uint32_t problem;
  uint32_t pad_;
};

struct PChunk {
  uint32_t seg;
  uint32_t count;
  uint64_t begin;        // element offset inside the segment
};

struct PProblem {
  uint64_t keep;
  uint64_t remaining;    // rank still to place inside the current prefix
  uint32_t prefix;       // selected high bits of T so far
  uint32_t thresh;       // T (valid after the last pass); 0xFFFFFFFF = keep none
  uint64_t need_eq;      // how many key==T elements are kept
};

__device__ __forceinline__ uint32_t mag_key(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

__constant__ int c_shift[3] = {21, 10, 0};
__constant__ int c_width[3] = {11, 11, 10};

__global__ void __launch_bounds__(kPT)
k_prune_hist(const PChunk* __restrict__ chunks, const PSeg* __restrict__ segs,
             const PProblem* __restrict__ probs, uint32_t* __restrict__ hist, int pass) {
  __shared__ uint32_t h[kBins];
  for (int i = threadIdx.x; i < kBins; i += kPT) h[i] = 0;
  __syncthreads();
  const PChunk c = chunks[blockIdx.x];
  const PSeg sg = segs[c.seg];
  const PProblem pb = probs[sg.problem];
  if (pb.remaining == 0) return;  // keep none, or already resolved
  const int shift = c_shift[pass];
  const uint32_t dmask = (1u << c_width[pass]) - 1u;
  const int hi_shift = shift + c_width[pass];  // bits above this pass's digit must match
  const float* v = sg.values + c.begin;
  for (uint32_t i = threadIdx.x; i < c.count; i += kPT) {
    const uint32_t key = mag_key(v[i]);
    const bool match = (hi_shift >= 32) || ((key >> hi_shift) == (pb.prefix >> hi_shift));
    if (match) atomicAdd(&h[(key >> shift) & dmask], 1u);
  }
  __syncthreads();
  uint32_t* gh = hist + static_cast<size_t>(sg.problem) * kBins;
  for (int i = threadIdx.x; i < kBins; i += kPT)
    if (h[i]) atomicAdd(&gh[i], h[i]);
}

// One CTA per problem: pick the digit holding the remaining-th largest key.
__global__ void __launch_bounds__(1024)
k_prune_select(PProblem* probs, uint32_t* hist, int pass) {
  __shared__ unsigned long long warp_tot[32];
  PProblem& pb = probs[blockIdx.x];
  uint32_t* gh = hist + static_cast<size_t>(blockIdx.x) * kBins;
  const uint64_t r = pb.remaining;
  const int width = c_width[pass];
  const int nb = 1 << width;
  // Suffix sums over bins (from the top) — two bins per thread.
  const int t = threadIdx.x;
  const int b0 = nb - 1 - 2 * t, b1 = nb - 2 - 2 * t;  // descending digit order
  unsigned long long c0 = (b0 >= 0) ? gh[b0] : 0ull, c1 = (b1 >= 0) ? gh[b1] : 0ull;
  unsigned long long x = c0 + c1;
  // inclusive warp scan
  const int lane = t & 31, w = t >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned long long z = warp_tot[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, z, o);
      if (lane >= o) z += y;
    }
    warp_tot[lane] = z;
  }
  __syncthreads();
  const unsigned long long before = (x - (c0 + c1)) + (w > 0 ? warp_tot[w - 1] : 0ull);
  // above(b0) = before; above(b1) = before + c0
  if (r > 0) {
    if (b0 >= 0 && before < r && before + c0 >= r) {
      pb.prefix |= static_cast<uint32_t>(b0) << c_shift[pass];
      pb.remaining = r - before;
    }
    if (b1 >= 0 && before + c0 < r && before + c0 + c1 >= r) {
      pb.prefix |= static_cast<uint32_t>(b1) << c_shift[pass];
      pb.remaining = r - (before + c0);
    }
  }
  __syncthreads();
  if (pass == 2 && t == 0) {
    if (pb.keep == 0) {
      pb.thresh = 0xFFFFFFFFu;
      pb.need_eq = 0;
    } else {
      pb.thresh = pb.prefix;
      pb.need_eq = pb.remaining;
    }
  }
}

__global__ void __launch_bounds__(kPT)
k_prune_count(const PChunk* __restrict__ chunks, const PSeg* __restrict__ segs,
              const PProblem* __restrict__ probs, uint32_t* __restrict__ gt_cnt,
              uint32_t* __restrict__ eq_cnt) {
  __shared__ uint32_t sg_[2];
  if (threadIdx.x < 2) sg_[threadIdx.x] = 0;
  __syncthreads();
  const PChunk c = chunks[blockIdx.x];
  const PSeg sg = segs[c.seg];
  const uint32_t T = probs[sg.problem].thresh;
  const float* v = sg.values + c.begin;
  uint32_t gt = 0, eq = 0;
  for (uint32_t i = threadIdx.x; i < c.count; i += kPT) {
    const uint32_t key = mag_key(v[i]);
    gt += (T != 0xFFFFFFFFu) && key > T;
    eq += key == T;
  }
  for (int o = 16; o > 0; o >>= 1) {
    gt += __shfl_xor_sync(0xFFFFFFFFu, gt, o);
    eq += __shfl_xor_sync(0xFFFFFFFFu, eq, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&sg_[0], gt);
    atomicAdd(&sg_[1], eq);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    gt_cnt[blockIdx.x] = sg_[0];
    eq_cnt[blockIdx.x] = sg_[1];
  }
}

// Ordered scan over all chunks, one block of kScanT threads walking windows
// of kScanT chunks: two exclusive prefix sums with carries — the key==T
// counts (eq ranks restart per problem: subtract the prefix at the problem's
// first chunk) and the kept counts gt + take (output offsets restart per
// layer: subtract the prefix at the segment's first chunk).
constexpr int kScanT = 1024;
__global__ void __launch_bounds__(kScanT)
k_prune_scan(const PChunk* __restrict__ chunks, const PSeg* __restrict__ segs,
             const PProblem* __restrict__ probs, uint32_t nchunks,
             const uint32_t* __restrict__ gt_cnt, const uint32_t* __restrict__ eq_cnt,
             const uint32_t* __restrict__ seg_first, const uint32_t* __restrict__ prob_first,
             uint64_t* __restrict__ pre_e, uint64_t* __restrict__ pre_w,
             uint64_t* __restrict__ eq_before, uint64_t* __restrict__ out_pos,
             uint64_t* __restrict__ seg_count) {
  using Scan = cub::BlockScan<uint64_t, kScanT>;
  __shared__ typename Scan::TempStorage tmp;
  uint64_t carry_e = 0, carry_w = 0;
  for (uint32_t base = 0; base < nchunks; base += kScanT) {
    const uint32_t c = base + threadIdx.x;
    const bool on = c < nchunks;
    uint32_t sg = 0, pb = 0;
    uint64_t e = 0, gt = 0;
    if (on) {
      sg = chunks[c].seg;
      pb = segs[sg].problem;
      e = eq_cnt[c];
      gt = gt_cnt[c];
    }
    uint64_t ex, agg;
    Scan(tmp).ExclusiveSum(e, ex, agg);
    ex += carry_e;
    carry_e += agg;
    if (on) pre_e[c] = ex;
    __syncthreads();
    uint64_t w = 0;
    if (on) {
      const uint64_t eqb = ex - pre_e[prob_first[pb]];
      const uint64_t need = probs[pb].need_eq;
      const uint64_t rest = need > eqb ? need - eqb : 0;
      eq_before[c] = eqb;
      w = gt + (rest < e ? rest : e);
    }
    __syncthreads();  // tmp reuse
    uint64_t wx;
    Scan(tmp).ExclusiveSum(w, wx, agg);
    wx += carry_w;
    carry_w += agg;
    if (on) pre_w[c] = wx;
    __syncthreads();
    if (on) {
      const uint64_t pos = wx - pre_w[seg_first[sg]];
      out_pos[c] = pos;
      if (c + 1 == nchunks || chunks[c + 1].seg != sg) seg_count[sg] = pos + w;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kPT)
k_prune_write(const PChunk* __restrict__ chunks, const PSeg* __restrict__ segs,
              const PProblem* __restrict__ probs, const uint64_t* __restrict__ eq_before,
              const uint64_t* __restrict__ out_pos) {
  __shared__ uint32_t wk[kPT / 32], we[kPT / 32];
  const PChunk c = chunks[blockIdx.x];
  const PSeg sg = segs[c.seg];
  const PProblem pb = probs[sg.problem];
  const uint32_t T = pb.thresh;
  uint64_t eqb = eq_before[blockIdx.x];
  uint64_t pos = out_pos[blockIdx.x];
  const float* v = sg.values + c.begin;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  for (uint32_t base = 0; base < c.count; base += kPT) {
    const uint32_t i = base + threadIdx.x;
    const bool in = i < c.count;
    const uint32_t key = in ? mag_key(v[i]) : 0u;
    const bool is_gt = in && T != 0xFFFFFFFFu && key > T;
    const bool is_eq = in && key == T;
    // equal-key rank inside the chunk (block exclusive scan of is_eq)
    const uint32_t be = __ballot_sync(0xFFFFFFFFu, is_eq);
    if (lane == 0) we[w] = __popc(be);
    __syncthreads();
    uint32_t eoff = 0, etot = 0;
    for (int j = 0; j < kPT / 32; ++j) {
      if (j < w) eoff += we[j];
      etot += we[j];
    }
    const uint64_t erank = eqb + eoff + __popc(be & lt_mask);
    const bool keep = is_gt || (is_eq && erank < pb.need_eq);
    const uint32_t bk = __ballot_sync(0xFFFFFFFFu, keep);
    if (lane == 0) wk[w] = __popc(bk);
    __syncthreads();
    uint32_t koff = 0, ktot = 0;
    for (int j = 0; j < kPT / 32; ++j) {
      if (j < w) koff += wk[j];
      ktot += wk[j];
    }
    if (keep) sg.out[pos + koff + __popc(bk & lt_mask)] = static_cast<uint32_t>(c.begin + i);
    eqb += etot;
    pos += ktot;
    __syncthreads();
  }
}

}  // namespace
}  // namespace samo_dev

using namespace samo_dev;

extern "C" {

uint64_t samo_unpruned_count(double p, uint64_t n) {
  // prune.hpp:76-79
  const double exact = (1.0 - p) * static_cast<double>(n);
  return static_cast<uint64_t>(std::floor(exact + 0.5 + 1e-9));
}

int samo_magnitude_prune(const float* const* values, const uint64_t* lens, const uint8_t* prunable,
                         int nlayers, double p, int scope, uint32_t* const* idx_out,
                         uint64_t* counts_out, samo_stream_t stream) {
  if (int rc = device_ok(); rc != SAMO_OK) return rc;
  if (!(p >= 0.0 && p < 1.0)) return fail(SAMO_E_PARAMETER, "sparsity must lie in [0, 1)");
  if (nlayers < 0 || (nlayers > 0 && (!values || !lens || !prunable || !idx_out || !counts_out)))
    return fail(SAMO_E_PARAMETER, "magnitude_prune: null argument");
  if (scope != SAMO_PRUNE_PER_LAYER && scope != SAMO_PRUNE_GLOBAL)
    return fail(SAMO_E_PARAMETER, "unknown prune scope");
  for (int l = 0; l < nlayers; ++l) {
    if (lens[l] >= (1ull << 32))  // prune.hpp:105-109
      return fail(SAMO_E_PARAMETER, "layer too large for 32-bit indices: layer %d", l);
    if (lens[l] && (!values[l] || !idx_out[l]))
      return fail(SAMO_E_PARAMETER, "magnitude_prune: null pointer for layer %d", l);
  }
  if (nlayers == 0) return SAMO_OK;
  cudaStream_t s = as_stream(stream);

  // Problems: one per layer (per_layer scope, and every non-prunable layer
  // with keep = len), or one for all prunable layers (global scope).
  std::vector<PSeg> segs;
  std::vector<PProblem> probs;
  std::vector<int> seg_layer;
  int global_prob = -1;
  uint64_t prunable_total = 0;
  for (int l = 0; l < nlayers; ++l)
    if (prunable[l]) prunable_total += lens[l];
  for (int l = 0; l < nlayers; ++l) {
    counts_out[l] = 0;
    if (lens[l] == 0) continue;
    PSeg sg{};
    sg.values = values[l];
    sg.out = idx_out[l];
    sg.len = lens[l];
    if (!prunable[l]) {
      PProblem pb{};
      pb.keep = lens[l];
      probs.push_back(pb);
      sg.problem = static_cast<uint32_t>(probs.size() - 1);
    } else if (scope == SAMO_PRUNE_PER_LAYER) {
      PProblem pb{};
      pb.keep = samo_unpruned_count(p, lens[l]);
      probs.push_back(pb);
      sg.problem = static_cast<uint32_t>(probs.size() - 1);
    } else {
      if (global_prob < 0) {
        PProblem pb{};
        pb.keep = samo_unpruned_count(p, prunable_total);
        probs.push_back(pb);
        global_prob = static_cast<int>(probs.size() - 1);
      }
      sg.problem = static_cast<uint32_t>(global_prob);
    }
    segs.push_back(sg);
    seg_layer.push_back(l);
  }
  // Global scope orders ties by layer position: keep the prunable segments of
  // the global problem contiguous and in layer order for the scan.  Segments
  // of other problems may sit between them, so reorder: all non-global
  // segments first (each their own problem), then the global ones.
  std::vector<int> order(segs.size());
  for (size_t i = 0; i < segs.size(); ++i) order[i] = static_cast<int>(i);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    const bool ga = static_cast<int>(segs[a].problem) == global_prob;
    const bool gb = static_cast<int>(segs[b].problem) == global_prob;
    return ga < gb;
  });
  std::vector<PSeg> segs_o;
  std::vector<int> layer_o;
  for (int i : order) {
    segs_o.push_back(segs[i]);
    layer_o.push_back(seg_layer[i]);
  }
  for (auto& pb : probs) {
    pb.remaining = pb.keep;
    pb.prefix = 0;
    pb.thresh = 0xFFFFFFFFu;
    pb.need_eq = 0;
  }
  std::vector<PChunk> chunks;
  for (size_t si = 0; si < segs_o.size(); ++si) {
    for (uint64_t b = 0; b < segs_o[si].len; b += kChunk) {
      PChunk c{};
      c.seg = static_cast<uint32_t>(si);
      c.begin = b;
      c.count = static_cast<uint32_t>(std::min<uint64_t>(kChunk, segs_o[si].len - b));
      chunks.push_back(c);
    }
  }
  const uint32_t nchunks = static_cast<uint32_t>(chunks.size());
  const uint32_t nsegs = static_cast<uint32_t>(segs_o.size());
  const uint32_t nprobs = static_cast<uint32_t>(probs.size());
  if (nchunks == 0) return SAMO_OK;

  // Scratch layout.
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off = (off + bytes + 255) / 256 * 256;
    return o;
  };
  const size_t o_chunks = carve(nchunks * sizeof(PChunk)), o_segs = carve(nsegs * sizeof(PSeg));
  const size_t o_probs = carve(nprobs * sizeof(PProblem));
  const size_t o_hist = carve(3ull * nprobs * kBins * 4);
  const size_t o_gt = carve(nchunks * 4ull), o_eq = carve(nchunks * 4ull);
  const size_t o_eqb = carve(nchunks * 8ull), o_pos = carve(nchunks * 8ull);
  const size_t o_cnt = carve(nsegs * 8ull);
  const size_t o_pe = carve(nchunks * 8ull), o_pw = carve(nchunks * 8ull);
  const size_t o_sf = carve(nsegs * 4ull), o_pf = carve(nprobs * 4ull);
  void* block = nullptr;
  SAMO_CUDA_TRY(cudaMallocAsync(&block, off, s));
  char* b = static_cast<char*>(block);
  auto* d_chunks = reinterpret_cast<PChunk*>(b + o_chunks);
  auto* d_segs = reinterpret_cast<PSeg*>(b + o_segs);
  auto* d_probs = reinterpret_cast<PProblem*>(b + o_probs);
  auto* d_hist = reinterpret_cast<uint32_t*>(b + o_hist);
  auto* d_gt = reinterpret_cast<uint32_t*>(b + o_gt);
  auto* d_eq = reinterpret_cast<uint32_t*>(b + o_eq);
  auto* d_eqb = reinterpret_cast<uint64_t*>(b + o_eqb);
  auto* d_pos = reinterpret_cast<uint64_t*>(b + o_pos);
  auto* d_cnt = reinterpret_cast<uint64_t*>(b + o_cnt);
  auto* d_pe = reinterpret_cast<uint64_t*>(b + o_pe);
  auto* d_pw = reinterpret_cast<uint64_t*>(b + o_pw);
  auto* d_sf = reinterpret_cast<uint32_t*>(b + o_sf);
  auto* d_pf = reinterpret_cast<uint32_t*>(b + o_pf);
  // first chunk of every segment and of every problem (segments are ordered by problem)
  std::vector<uint32_t> seg_first(nsegs, 0), prob_first(nprobs, 0);
  {
    std::vector<uint8_t> seen_p(nprobs, 0);
    for (uint32_t c = nchunks; c-- > 0;) seg_first[chunks[c].seg] = c;
    for (uint32_t si = 0; si < nsegs; ++si) {
      const uint32_t pb = segs_o[si].problem;
      if (!seen_p[pb]) {
        seen_p[pb] = 1;
        prob_first[pb] = seg_first[si];
      }
    }
  }
  int rc = SAMO_OK;
  std::vector<uint64_t> seg_counts(nsegs);
  do {
    cudaError_t e;
    if ((e = cudaMemcpyAsync(d_chunks, chunks.data(), nchunks * sizeof(PChunk), cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemcpyAsync(d_segs, segs_o.data(), nsegs * sizeof(PSeg), cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemcpyAsync(d_probs, probs.data(), nprobs * sizeof(PProblem), cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemcpyAsync(d_sf, seg_first.data(), nsegs * 4ull, cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemcpyAsync(d_pf, prob_first.data(), nprobs * 4ull, cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemsetAsync(d_cnt, 0, nsegs * 8ull, s)) ||
        (e = cudaMemsetAsync(d_hist, 0, 3ull * nprobs * kBins * 4, s))) {
      rc = cuda_fail(e, "prune setup");
      break;
    }
    for (int pass = 0; pass < 3 && rc == SAMO_OK; ++pass) {
      uint32_t* h = d_hist + static_cast<size_t>(pass) * nprobs * kBins;
      k_prune_hist<<<nchunks, kPT, 0, s>>>(d_chunks, d_segs, d_probs, h, pass);
      if ((e = cudaGetLastError())) { rc = cuda_fail(e, "k_prune_hist"); break; }
      note_launch();
      k_prune_select<<<nprobs, 1024, 0, s>>>(d_probs, h, pass);
      if ((e = cudaGetLastError())) { rc = cuda_fail(e, "k_prune_select"); break; }
      note_launch();
    }
    if (rc != SAMO_OK) break;
    k_prune_count<<<nchunks, kPT, 0, s>>>(d_chunks, d_segs, d_probs, d_gt, d_eq);
    if ((e = cudaGetLastError())) { rc = cuda_fail(e, "k_prune_count"); break; }
    k_prune_scan<<<1, kScanT, 0, s>>>(d_chunks, d_segs, d_probs, nchunks, d_gt, d_eq, d_sf, d_pf, d_pe, d_pw,
                                      d_eqb, d_pos, d_cnt);
    if ((e = cudaGetLastError())) { rc = cuda_fail(e, "k_prune_scan"); break; }
    k_prune_write<<<nchunks, kPT, 0, s>>>(d_chunks, d_segs, d_probs, d_eqb, d_pos);
    if ((e = cudaGetLastError())) { rc = cuda_fail(e, "k_prune_write"); break; }
    note_launch(3);
    if ((e = cudaMemcpyAsync(seg_counts.data(), d_cnt, nsegs * 8ull, cudaMemcpyDeviceToHost, s)) ||
        (e = cudaStreamSynchronize(s))) {
      rc = cuda_fail(e, "prune readback");
      break;
    }
  } while (false);
  cudaFreeAsync(block, s);
  if (rc != SAMO_OK) return rc;
  for (uint32_t si = 0; si < nsegs; ++si) counts_out[layer_o[si]] = seg_counts[si];
  return SAMO_OK;
}

}  // extern "C"
