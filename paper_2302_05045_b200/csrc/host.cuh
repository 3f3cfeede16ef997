// host.cuh — private header of the library's host side (abi.cu, model.cu,
// dp.cu): the communicator, the model state and the helpers they share.
#pragma once

#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

using namespace samo_dev;

constexpr uint32_t kDefaultTile = 8192;   // single-layer API-parity plans
constexpr uint32_t kModelTile = 16384;    // model step (measured best)

struct samo_comm {
  ncclComm_t comm = nullptr;  // gradient buckets
  ncclComm_t flag = nullptr;  // the skip indicator, concurrently with the buckets
  int nranks = 1;
  int rank = 0;
  bool local_group = false;  // samo_model_attach_local_group: peers are models on this device, no NCCL
};

inline int nccl_fail(ncclResult_t r, const char* what) {
  return fail(SAMO_E_NCCL, "%s: %s", what, ncclGetErrorString(r));
}

inline int clear_ok() {
  clear_error();
  return SAMO_OK;
}

inline SamoAdamParams adam_params(const samo_optimizer_config* cfg) {
  SamoAdamParams p;
  p.lr = cfg->learning_rate;
  p.beta1 = cfg->beta1;
  p.beta2 = cfg->beta2;
  p.eps = cfg->epsilon;
  p.wd = cfg->weight_decay;
  return p;
}

// ---------------------------------------------------------------------------
// Model state + step driver

// Bucketing of the sharded (ZeRO-1) data-parallel step (step_sharded).
struct ShardPlan {
  int G = 0, B = 0;
  uint64_t c = 0, C = 0;
  std::vector<uint32_t> k1_t, ex_t;  // tile boundaries per bucket, B + 1 each
};

struct samo_model {
  int nlayers = 0;
  uint32_t tile_elems = kDefaultTile;
  std::vector<uint64_t> dense_len, nnz, k_off, d_off;
  std::vector<uint8_t> idx_set;
  uint64_t phi = 0, n_tot = 0, d_tot = 0;
  uint32_t ntiles = 0;
  // device arenas
  void* block = nullptr;  // one allocation for every arena/table
  uint64_t block_bytes = 0;
  float* theta = nullptr;
  float* m = nullptr;
  float* v = nullptr;
  float* g = nullptr;          // compressed gradient arena (+ skip-indicator slot)
  uint16_t* c16 = nullptr;     // compressed binary16 weights (sharded exchange)
  double* norm2 = nullptr;     // this rank's / the global sum of g^2 (sharded exchange)
  uint32_t* done = nullptr;    // arrival counter of k_adam_shard
  uint64_t n_al = 0;
  int exchange = -1;           // SAMO_EXCHANGE_*; -1 = environment default
  uint32_t* idx = nullptr;
  uint16_t* off16 = nullptr;   // idx[k] - dense_begin of k's tile (step kernels)
  uint16_t* theta16 = nullptr;
  SamoTile* tiles = nullptr;
  SamoLayerDev* layers_dev = nullptr;
  uint64_t* k_off_dev = nullptr;
  SamoStepState* st = nullptr;
  float* norm_partials = nullptr;
  int grad_bf16 = 0;                  // dense gradients are bfloat16 (else binary16)
  float* tile_norm = nullptr;         // K123: per-tile grad-norm partials
  double* norm_dpartials = nullptr;   // k123_repair: per-CTA sums of them
  std::vector<SamoLayerDev> layers_host;
  std::vector<SamoTile> tiles_host;
  samo_optimizer_config cfg{};
  samo_comm* comm = nullptr;
  bool finalized = false;
  bool grads_set = false;
  int grid_gather16 = 0, grid_gather32 = 0, grid_update16 = 0, grid_update32 = 0;
  // Fused single-GPU step (K123): the second set of theta/m/v buffers the
  // step writes; the host swaps the sets after every step (`parity` = which
  // set theta/m/v point at), so everything else always sees the live state.
  float* theta_alt = nullptr;
  float* m_alt = nullptr;
  float* v_alt = nullptr;
  int parity = 0;
  int grid_fused = 0;
  cudaGraphExec_t fgraph[2] = {nullptr, nullptr};  // captured fused steps, one per parity
  uint64_t fgraph_kernels = 0;
  // CUDA graph of one step
  cudaGraphExec_t graph = nullptr;
  samo_comm* graph_comm = nullptr;
  uint64_t graph_kernels = 0;
  cudaStream_t capture_stream = nullptr;
  // Overlapped data-parallel step: tile-range buckets whose allreduce runs on
  // a side stream while later buckets gather and earlier ones update.
  int nbuckets = 0;
  std::vector<uint32_t> bucket_t;       // tile boundaries, nbuckets + 1
  cudaStream_t s_comm = nullptr, s_flag = nullptr;
  std::vector<cudaEvent_t> ev_k1, ev_ar;
  cudaEvent_t ev_fork = nullptr, ev_flag = nullptr;
  int reserve_sms = 16;                 // SMs left to NCCL while our kernels run
  ShardPlan shard_plan;
  ShardPlan p2p_plan;                   // peer-to-peer step (serial: 1 bucket)
  // K1 tile table of the push-mode P2P step: tiles split at owner boundaries,
  // pad_ = owner rank, pad2_ = receive-buffer element of k_begin.
  SamoTile* push_tiles = nullptr;
  uint32_t push_ntiles = 0;
  int push_G = 0, push_B = 0;
  std::vector<uint32_t> push_layer_t;  // first push piece of each layer (+ end)
  bool sunk_push = false;              // this step's sinks pushed to the owners
  uint16_t* sink16 = nullptr;          // fused dW sink's gather target in push mode (n halves)
  int group_dev = -1;                  // local group across devices: this model's device
  cudaStream_t s_group = nullptr;      // ... and its stream for the group step
  SamoPeerSlots* slots = nullptr;       // this rank's signal area (in the block)
  // Device copy of the step scalars (SamoStepConfig), refreshed on the step's
  // stream before the next step whenever set_config / attach_comm changed them.
  SamoStepConfig* cfg_dev = nullptr;
  bool cfg_dirty = true;
  bool capturing = false;  // only captured steps read cfg_dev (eager steps pass the scalars by value)
  // Backward sinks: first tile of every layer; per-layer row/column-block k
  // tables of the fused dW sink (built on first use).
  std::vector<uint32_t> layer_t;
  std::vector<uint32_t*> dw_kb;
  std::vector<uint64_t> dw_kb_in;
  // Peer mappings of the other ranks' model blocks (CUDA IPC) for the fused
  // peer-to-peer exchange; p2p_ok is agreed by every rank.
  void* peer_base[kMaxP2PRanks] = {};
  bool p2p_ok = false;
  samo_comm* own_comm = nullptr;  // the virtual communicator of a local group (owned)
  std::vector<cudaEvent_t> ev_sh;       // sharded pipeline: K1 and all-gather events
  int grid_expand = 0;
  // Phase timing of the data-parallel step.
  bool phase_timing = false;
  cudaEvent_t phase_ev[16] = {};
  int phase_count = 0;
};

constexpr int kMaxBuckets = 32;
constexpr uint64_t kArenaSlack = 2048;  // elements: bucket x rank padding of the sharded exchange + flag
constexpr uint64_t kFlagOff = 2040;     // flag slot at g + n_al + kFlagOff

inline float* flag_ptr(const samo_model* md) { return md->g + md->n_al + kFlagOff; }

// Optional phase timing of the data-parallel step (samo_model_enable_phase_timing).
inline int phase_mark(samo_model* md, int i, cudaStream_t s) {
  if (!md->phase_timing) return SAMO_OK;
  if (!md->phase_ev[i]) SAMO_CUDA_TRY(cudaEventCreate(&md->phase_ev[i]));
  SAMO_CUDA_TRY(cudaEventRecord(md->phase_ev[i], s));
  return SAMO_OK;
}

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

inline int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

inline int comm_size(const samo_model* md) { return md->comm ? md->comm->nranks : 1; }

// Drops every captured step graph (the step plan changed).
inline void drop_graphs(samo_model* md) {
  if (md->graph) cudaGraphExecDestroy(md->graph);
  md->graph = nullptr;
  for (auto& g : md->fgraph) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
}

// The fused single-GPU step (K123) is the default without a communicator;
// SAMO_FUSED_STEP=0 selects the K1 | K23 pair.
inline bool fused_step(const samo_model* md) {
  return comm_size(md) <= 1 && md->grid_fused > 0 && env_int("SAMO_FUSED_STEP", 1) != 0;
}

inline int step_ready(samo_model* md) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  if (!md->finalized) return fail(SAMO_E_STATE, "model not finalized");
  return SAMO_OK;
}

// model.cu
// The gradient arena holds unscaled fp32 when it is exchanged between ranks,
// and the raw compressed binary16 gradient (the reference's grad16) otherwise.
bool wide_grads(const samo_model* md);
StepArgs step_args(samo_model* md);
int flush_cfg(samo_model* md, cudaStream_t s);  // stream-ordered update of cfg_dev if dirty

// dp.cu — data-parallel machinery
int open_peers(samo_model* md);   // collective: CUDA IPC peer mappings
void close_peers(samo_model* md);
int exchange_mode(const samo_model* md);
bool p2p_push();
int p2p_buckets(int G);
int plan_shards(samo_model* md, ShardPlan& p, int B);
int build_push_tiles(samo_model* md, const ShardPlan& p);
// Backward sinks of a peer-to-peer model (push mode): the step's plan and
// push pieces, then one layer's K1 push (sink_dense) or the copy of its
// locally gathered binary16 gradients (sink_dw) to the owners.
int push_sink_prepare(samo_model* md);
int push_sink_layer(samo_model* md, int layer, const uint16_t* local_src, cudaStream_t s);
bool p2p_push();
int step_p2p(samo_model* md, cudaStream_t S, bool gather = true);
int step_sharded(samo_model* md, cudaStream_t S);
int step_overlapped(samo_model* md, cudaStream_t S);
