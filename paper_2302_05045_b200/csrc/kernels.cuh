// kernels.cuh — launch interfaces of the SAMO step kernels (kernels_step.cu).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace samo_dev {

constexpr int kThreads = 256;       // threads per CTA for the tile kernels

enum ExpandMode : int {
  kModeDowncast = 1,  // K3 : downcast + expand (train.hpp:647-651)
  kModeValues = 2,    // expand<T> of given values (store.hpp:72-87)
  kModeCheck = 3      // check_state_invariants (store.hpp:171-197)
};

struct ExpandArgs {
  const SamoTile* tiles;
  uint32_t ntiles;
  uint32_t tile_elems;
  void* out_base;              // dense output buffer; tile t writes at out_base + out_off
  const uint32_t* idx;         // index arena (layer-local indices)
  float* theta;                // compressed fp32 master weights
  const void* values;          // kModeValues: compressed values (u16/u32)
  uint32_t* mismatch;          // kModeCheck: set to nonzero on violation
  int use_bulk;                // 1 when every dense output is 16-byte aligned
};

// Fills k_begin/k_end of every tile (layer/dense fields preset) by binary
// search in the layer's ascending index segment.
int launch_tiles_fill(SamoTile* tiles, uint32_t ntiles, const uint64_t* k_off,
                      const uint32_t* idx, cudaStream_t s);

constexpr int kMaxP2PRanks = 8;

// Arguments of the two per-step kernels (kernels_fused.cu).
struct StepArgs {
  const SamoTile* tiles;
  uint32_t ntiles;
  uint32_t tile_elems;
  const SamoLayerDev* layers;  // dense gradient inputs (per layer)
  uint16_t* theta16;           // dense output arena; tile t writes at theta16 + out_off
  const uint16_t* off16;       // kept index relative to its tile's dense_begin
  void* g;                     // compressed gradient arena: fp32 or binary16
  float* theta;
  float* m;
  float* v;
  // K123 (fused single-GPU step): theta/m/v are read from the buffers above
  // and the updated values written to these (the model's other buffer set).
  float* theta_o;
  float* m_o;
  float* v_o;
  float inv_scale;             // 1/loss_scale (and 1/G when exchanging fp32)
  uint32_t grad_bf16;          // dense (and compressed 16-bit) gradients are bfloat16
  SamoAdamParams prm;
  SamoStepState* st;
  float* flag_slot;            // non-finite indicator (summed across ranks)
  float* norm_partials;        // this launch's per-CTA grad-norm partials
  float* tile_norm;            // K123: one grad-norm partial per tile
  double* norm_dpartials;      // k123_repair: one per CTA
  const float* norm_all;       // every partial of the step (read when finalize)
  uint32_t norm_count;
  uint32_t finalize;           // 1 on the step's last update launch
  const SamoStepConfig* cfg;   // device scalars (model steps); overrides prm / inv_scale
  // K1 push mode (peer-to-peer step): tile t's kept elements go to rank
  // tiles[t].pad_'s receive buffer push16[pad_] at element pad2_ + (k - k_begin)
  // instead of g + k (binary16 output only).
  uint32_t push;
  uint16_t* push16[kMaxP2PRanks];
};

// K1 gather: out_f32 -> unscaled fp32 for the exchange, else raw binary16.
int launch_gather(const StepArgs& a, bool out_f32, int grid, cudaStream_t s);
// K23 update: g_f32 selects the gradient arena type written by K1.
int launch_update(const StepArgs& a, bool g_f32, int grid, cudaStream_t s);
// K123, the fused single-GPU step (gather + unscale + Adam + downcast +
// expand in one pass per tile), speculative on the global skip flag: reads
// theta/m/v, writes theta_o/m_o/v_o and theta16 in place; the last CTA
// advances the scalars or records the skip.  k123_repair, launched after it,
// restores theta16 and copies theta/m/v -> theta_o/m_o/v_o when the step was
// skipped (a no-op otherwise).  The host then swaps the two buffer sets.
int launch_step_fused(const StepArgs& a, int grid, cudaStream_t s);
int launch_step_repair(const StepArgs& a, cudaStream_t s);
int fused_grid(uint32_t tile_elems);
// which: 0 = gather, 1 = update; wide = fp32 gradient arena.
int step_grid(int which, bool wide, uint32_t tile_elems);
// Fused peer-to-peer exchange + shard update (kernels_fused.cu, k_shard_p2p):
// rank `rank` owns [k0, k1) of the compressed arena; it reads that range of
// every rank's binary16 gradient over NVLink, sums in rank order, runs Adam
// and writes the binary16 weights into every rank's theta16c arena.
constexpr int kMaxP2PBuckets = 32;
// Signal area of the pipelined peer-to-peer step, one per rank inside its
// IPC-mapped model block.  Rank q writes only the [q] columns of its peers'
// areas (release stores at system scope); each rank spins only on its own.
// `epoch` (local) counts completed pipelined steps; every signal of step s
// carries epoch + 1 = s + 1, so no slot is ever reset.
struct SamoPeerSlots {
  uint64_t epoch;
  uint64_t flag_epoch[kMaxP2PRanks];
  float flag_val[kMaxP2PRanks];
  uint64_t bucket_epoch[kMaxP2PBuckets * kMaxP2PRanks];  // [bucket * 8 + rank]
  double norm[kMaxP2PBuckets * kMaxP2PRanks];             // [bucket * 8 + rank]
};
struct P2PArgs {
  const uint16_t* g16[kMaxP2PRanks];  // per-rank compressed binary16 gradients
  uint16_t* c16[kMaxP2PRanks];        // per-rank theta16c arenas
  int G;
  int rank;
  float* theta;
  float* m;
  float* v;
  uint64_t k0, k1;                    // k0 a multiple of 8
  float scale;                        // (1/loss_scale) * (1/G)
  int grad_bf16;                      // the 16-bit gradients are bfloat16
  SamoAdamParams prm;
  const SamoStepState* st;
  const float* flag_slot;             // global skip indicator (already reduced)
  float* norm_partials;
  double* norm2_out;
  uint32_t* done;
  // Pipelined step only (bucket >= 0): every rank's signal area; the last CTA
  // publishes this bucket's norm^2 and its completion to all of them.
  SamoPeerSlots* slots[kMaxP2PRanks];
  int bucket;
  int grid;                           // 0 = default
  // Push mode: every rank's K1 already wrote its contribution for [k0, k1)
  // into this rank's receive buffer: rank q's at recv[q * rstride + i0 + (k - k0)].
  int push;
  const uint16_t* recv;
  uint64_t rstride, i0;
  const SamoStepConfig* cfg;          // device scalars: override prm / scale
};
int launch_shard_p2p(const P2PArgs& a, cudaStream_t s);
// Skip-flag exchange over peer memory (one warp): publishes this rank's
// non-finite count to every peer, waits for all of theirs and writes the
// rank-ordered sum to *flag.  Also the step's first cross-rank barrier.
int launch_p2p_flag(SamoPeerSlots* const* slots, int G, int rank, float* flag, int phase, cudaStream_t s);
// Waits (one warp) until every rank has published bucket `bucket`.
int launch_p2p_wait(const SamoPeerSlots* mine, int G, int bucket, cudaStream_t s);
// Advances the local epoch (after the step's last read of the slots).
int launch_p2p_epoch(SamoPeerSlots* mine, cudaStream_t s);
// Peer-wait trap limit from SAMO_SPIN_TIMEOUT_S (seconds), on the current device.
int set_spin_limit_from_env();
// Copies compressed binary16 gradients src[k] to their owners' receive
// buffers along the push pieces a.tiles[0, a.ntiles) (a.push16 = peers).
int launch_push_copy(const StepArgs& a, const uint16_t* src, cudaStream_t s);

// Sharded data-parallel step pieces.
struct ShardArgs {
  const float* g;              // reduce-scattered gradient (this rank's shard in place)
  float* theta;
  float* m;
  float* v;
  uint16_t* theta16c;          // compressed binary16 weights (all-gathered afterwards)
  uint64_t k0, k1;             // this rank's shard, k0 a multiple of 8
  SamoAdamParams prm;
  const SamoStepState* st;
  const float* flag_slot;      // global skip indicator (already reduced)
  float* norm_partials;
  double* norm2_out;           // this rank's sum of g^2
  uint32_t* done;
  const SamoStepConfig* cfg;   // device scalars: override prm
};
int launch_adam_shard(const ShardArgs& a, int grid, cudaStream_t s);
int launch_step_finalize(SamoStepState* st, const double* norm2, int nslots, float* flag,
                         float beta1, float beta2, const SamoStepConfig* cfg, cudaStream_t s);
// Writes `v` to `dst` (one thread) on `s`: the stream-ordered update of the
// device step scalars.
int launch_set_step_config(SamoStepConfig* dst, const SamoStepConfig& v, cudaStream_t s);
// Expand-only tile pass: a.g holds theta16c.
int launch_expand_c16(const StepArgs& a, int grid, cudaStream_t s);
int expand_grid(uint32_t tile_elems);
int launch_build_off16(const SamoTile* tiles, uint32_t ntiles, const uint32_t* idx,
                       uint16_t* off16, cudaStream_t s);

// Weight-gradient GEMM dW[M x N] = X^T . dY, X [K x M], dY [K x N] binary16
// row-major (kernels_gemm.cu).  epi 0: dense binary16 dW; epi 1: gather of
// the kept elements into g16 (layer-local k) + skip flag.
struct DwArgs {
  uint64_t M, N, K;      // in, out, batch
  uint16_t* dw;          // epi 0
  const uint32_t* idx;   // epi 1: layer's ascending kept indices
  const uint32_t* kb;    // epi 1: [(col blocks + 1) x M] row/column-block k starts
  uint16_t* g16;         // epi 1: layer's compressed binary16 gradient
  float* flag;           // epi 1: skip indicator
  uint32_t tail0;        // set by launch_dw_gemm: pair tiles >= tail0 run as two 256 x BN/2 halves
};
int dw_check(uint64_t batch, uint64_t in, uint64_t out, const void* x, const void* dy);
uint32_t dw_col_blocks(uint64_t out);
int launch_build_rowblocks(const uint32_t* idx, uint64_t n, uint64_t in, uint64_t out, uint32_t* kb,
                           cudaStream_t s);
int launch_dw_gemm(const uint16_t* x, const uint16_t* dy, const DwArgs& a, int epi, cudaStream_t s);

template <int MODE, typename OutT>
int launch_expand(const ExpandArgs& a, int grid, cudaStream_t s);
template <int MODE, typename OutT>
int expand_grid(uint32_t tile_elems);

// Plain gather out[k] = dense[idx[k]] (compress<T>, store.hpp:58-69).
template <typename T>
int launch_compress(const T* dense, const uint32_t* idx, uint64_t n, T* out, cudaStream_t s);

int launch_adam(float* theta, float* m, float* v, const float* g, uint64_t n,
                SamoAdamParams prm, float bias1, float bias2, cudaStream_t s);

int launch_f2h(const float* in, uint16_t* out, uint64_t n, cudaStream_t s);
int launch_h2f(const uint16_t* in, float* out, uint64_t n, cudaStream_t s);
int launch_synth_f32(float* out, uint64_t n, uint64_t seed, uint64_t stream_id, float bound,
                     cudaStream_t s);
int launch_synth_f16(uint16_t* out, uint64_t n, uint64_t seed, uint64_t stream_id, float bound,
                     float scale, cudaStream_t s);
// Strictly-ascending and < dense_len check of one index segment.
int launch_check_indices(const uint32_t* idx, uint64_t n, uint64_t dense_len, uint32_t* bad,
                         cudaStream_t s);

}  // namespace samo_dev
