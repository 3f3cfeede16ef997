// abi.cu — the C ABI (include/samo_cuda.h): argument checks with the
// reference's error taxonomy, the plain API-parity entry points, the model
// state (flat device arenas + tile table + device scalars), the step drivers
// (single GPU: K1 -> K23; data parallel: the peer-to-peer step over CUDA-IPC
// peer memory — push-mode K1, peer-signalled barriers, bucketed shard update
// || expand — or the NCCL sharded / allreduce steps; any of them as one CUDA
// graph), the backward sinks, checkpoints and the NCCL communicator.
#include <cuda.h>
#include <nccl.h>
#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"

// ---------------------------------------------------------------------------
// Status plumbing.

namespace samo_dev {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return status;
}

int cuda_fail(cudaError_t err, const char* what) {
  return fail(err == cudaErrorMemoryAllocation ? SAMO_E_NOMEM : SAMO_E_CUDA, "%s: %s (%s)", what,
              cudaGetErrorString(err), cudaGetErrorName(err));
}

void note_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int device_ok() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(SAMO_E_CUDA, "no CUDA device available (the SAMO path has no CPU fallback)");
  }
  return SAMO_OK;
}

int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

}  // namespace samo_dev

using namespace samo_dev;

static int clear_ok() {
  g_last_error.clear();
  return SAMO_OK;
}

extern "C" {

int samo_abi_version(void) { return SAMO_ABI_VERSION; }

const char* samo_status_string(int status) {
  switch (status) {
    case SAMO_OK: return "ok";
    case SAMO_E_DIMENSION: return "DimensionError";
    case SAMO_E_PARAMETER: return "ParameterError";
    case SAMO_E_INDEX: return "IndexError";
    case SAMO_E_STATE: return "StateError";
    case SAMO_E_CONFIG: return "ConfigError";
    case SAMO_E_CUDA: return "CudaError";
    case SAMO_E_NCCL: return "NcclError";
    case SAMO_E_NOMEM: return "OutOfDeviceMemory";
    default: return "unknown";
  }
}

const char* samo_last_error(void) { return g_last_error.c_str(); }

uint64_t samo_kernel_launch_count(void) { return g_launches.load(); }

// ---------------------------------------------------------------------------
// half.hpp

int samo_float_to_half(const float* in, uint16_t* out, uint64_t n, samo_stream_t stream) {
  SAMO_TRY(device_ok());
  if (n && (!in || !out)) return fail(SAMO_E_PARAMETER, "float_to_half: null pointer");
  SAMO_TRY(launch_f2h(in, out, n, as_stream(stream)));
  return clear_ok();
}

int samo_half_to_float(const uint16_t* in, float* out, uint64_t n, samo_stream_t stream) {
  SAMO_TRY(device_ok());
  if (n && (!in || !out)) return fail(SAMO_E_PARAMETER, "half_to_float: null pointer");
  SAMO_TRY(launch_h2f(in, out, n, as_stream(stream)));
  return clear_ok();
}

// ---------------------------------------------------------------------------
// store.hpp: compress / expand

}  // extern "C"

template <typename T>
static int compress_impl(const T* dense, uint64_t dense_len, const uint32_t* idx, uint64_t n,
                         uint64_t ind_dense_len, T* out, samo_stream_t stream) {
  SAMO_TRY(device_ok());
  if (dense_len != ind_dense_len)  // store.hpp:60-62
    return fail(SAMO_E_DIMENSION, "compress: dense length does not match index set");
  if (n && (!dense || !idx || !out)) return fail(SAMO_E_PARAMETER, "compress: null pointer");
  SAMO_TRY(launch_compress<T>(dense, idx, n, out, as_stream(stream)));
  return clear_ok();
}

extern "C" {

int samo_compress_u16(const uint16_t* dense, uint64_t dense_len, const uint32_t* idx, uint64_t n,
                      uint64_t ind_dense_len, uint16_t* out, samo_stream_t stream) {
  return compress_impl<uint16_t>(dense, dense_len, idx, n, ind_dense_len, out, stream);
}

int samo_compress_u32(const uint32_t* dense, uint64_t dense_len, const uint32_t* idx, uint64_t n,
                      uint64_t ind_dense_len, uint32_t* out, samo_stream_t stream) {
  return compress_impl<uint32_t>(dense, dense_len, idx, n, ind_dense_len, out, stream);
}

}  // extern "C"

// Single-layer tile plan in stream-ordered scratch: tile table + a one-entry
// layer table whose output pointer is `out`.
struct ScratchPlan {
  SamoTile* tiles = nullptr;
  SamoLayerDev* layer = nullptr;
  uint64_t* k_off = nullptr;
  uint32_t ntiles = 0;
  void* block = nullptr;
  cudaStream_t s = nullptr;
  ~ScratchPlan() {
    if (block) cudaFreeAsync(block, s);
  }
};

static int make_plan(ScratchPlan& p, const uint32_t* idx, uint64_t n, uint64_t dense_len, void* out,
                     uint32_t tile_elems, cudaStream_t s) {
  p.s = s;
  const uint64_t ntiles = (dense_len + tile_elems - 1) / tile_elems;
  if (ntiles > 0xFFFFFFFFull) return fail(SAMO_E_PARAMETER, "too many tiles");
  p.ntiles = static_cast<uint32_t>(ntiles);
  const size_t tiles_bytes = ntiles * sizeof(SamoTile);
  const size_t total = tiles_bytes + sizeof(SamoLayerDev) + 2 * sizeof(uint64_t);
  SAMO_CUDA_TRY(cudaMallocAsync(&p.block, total, s));
  p.tiles = static_cast<SamoTile*>(p.block);
  p.layer = reinterpret_cast<SamoLayerDev*>(static_cast<char*>(p.block) + tiles_bytes);
  p.k_off = reinterpret_cast<uint64_t*>(p.layer + 1);
  std::vector<SamoTile> host(ntiles);
  for (uint64_t t = 0; t < ntiles; ++t) {
    host[t].layer = 0;
    host[t].dense_begin = static_cast<uint32_t>(t * tile_elems);
    host[t].dense_count = static_cast<uint32_t>(std::min<uint64_t>(tile_elems, dense_len - t * tile_elems));
    host[t].pad_ = 0;
    host[t].k_begin = host[t].k_end = 0;
    host[t].out_off = t * tile_elems;  // relative to the caller's dense output
    host[t].pad2_ = 0;
  }
  SamoLayerDev ld{};
  ld.grad = nullptr;
  ld.theta16 = static_cast<uint16_t*>(out);
  ld.dense_len = dense_len;
  ld.k_off = 0;
  const uint64_t koff[2] = {0, n};
  SAMO_CUDA_TRY(cudaMemcpyAsync(p.tiles, host.data(), tiles_bytes, cudaMemcpyHostToDevice, s));
  SAMO_CUDA_TRY(cudaMemcpyAsync(p.layer, &ld, sizeof(ld), cudaMemcpyHostToDevice, s));
  SAMO_CUDA_TRY(cudaMemcpyAsync(p.k_off, koff, sizeof(koff), cudaMemcpyHostToDevice, s));
  SAMO_TRY(launch_tiles_fill(p.tiles, p.ntiles, p.k_off, idx, s));
  // Pageable sources: the copies above are staged before returning, but keep
  // the host vectors alive until the stream has consumed them.
  SAMO_CUDA_TRY(cudaStreamSynchronize(s));
  return SAMO_OK;
}

constexpr uint32_t kDefaultTile = 8192;   // single-layer API-parity plans
constexpr uint32_t kModelTile = 16384;    // model step (measured best)

template <typename T>
static int expand_impl(const T* values, uint64_t n_values, const uint32_t* idx, uint64_t n,
                       uint64_t ind_dense_len, uint64_t shape_numel, T* dense_out,
                       samo_stream_t stream) {
  SAMO_TRY(device_ok());
  if (n_values != n)  // store.hpp:75-77
    return fail(SAMO_E_DIMENSION, "expand: value count does not match index set");
  if (shape_numel != ind_dense_len)  // store.hpp:78-80
    return fail(SAMO_E_DIMENSION, "expand: shape does not match index set dense length");
  if (shape_numel == 0) return fail(SAMO_E_DIMENSION, "tensor extents must be positive");
  if (!dense_out || (n && (!values || !idx))) return fail(SAMO_E_PARAMETER, "expand: null pointer");
  if (ind_dense_len > 0xFFFFFFFFull)
    return fail(SAMO_E_PARAMETER, "layer too large for 32-bit indices");
  cudaStream_t s = as_stream(stream);
  ScratchPlan plan;
  SAMO_TRY(make_plan(plan, idx, n, ind_dense_len, dense_out, kDefaultTile, s));
  ExpandArgs a{};
  a.tiles = plan.tiles;
  a.ntiles = plan.ntiles;
  a.tile_elems = kDefaultTile;
  a.out_base = dense_out;
  a.idx = idx;
  a.values = values;
  a.use_bulk = (reinterpret_cast<uintptr_t>(dense_out) % 16) == 0;
  SAMO_TRY((launch_expand<kModeValues, T>(a, 0, s)));
  return clear_ok();
}

extern "C" {

int samo_expand_u16(const uint16_t* values, uint64_t n_values, const uint32_t* idx, uint64_t n,
                    uint64_t ind_dense_len, uint64_t shape_numel, uint16_t* dense_out,
                    samo_stream_t stream) {
  return expand_impl<uint16_t>(values, n_values, idx, n, ind_dense_len, shape_numel, dense_out,
                               stream);
}

int samo_expand_u32(const uint32_t* values, uint64_t n_values, const uint32_t* idx, uint64_t n,
                    uint64_t ind_dense_len, uint64_t shape_numel, uint32_t* dense_out,
                    samo_stream_t stream) {
  return expand_impl<uint32_t>(values, n_values, idx, n, ind_dense_len, shape_numel, dense_out,
                               stream);
}

int samo_downcast_expand(const float* theta32, uint64_t n, const uint32_t* idx, uint64_t dense_len,
                         uint16_t* theta16_dense, samo_stream_t stream) {
  SAMO_TRY(device_ok());
  if (dense_len == 0) return fail(SAMO_E_DIMENSION, "tensor extents must be positive");
  if (n > dense_len) return fail(SAMO_E_DIMENSION, "expand: more values than dense slots");
  if (!theta16_dense || (n && (!theta32 || !idx)))
    return fail(SAMO_E_PARAMETER, "downcast_expand: null pointer");
  if (dense_len > 0xFFFFFFFFull) return fail(SAMO_E_PARAMETER, "layer too large for 32-bit indices");
  cudaStream_t s = as_stream(stream);
  ScratchPlan plan;
  SAMO_TRY(make_plan(plan, idx, n, dense_len, theta16_dense, kDefaultTile, s));
  ExpandArgs a{};
  a.tiles = plan.tiles;
  a.ntiles = plan.ntiles;
  a.tile_elems = kDefaultTile;
  a.out_base = theta16_dense;
  a.idx = idx;
  a.theta = const_cast<float*>(theta32);
  a.use_bulk = (reinterpret_cast<uintptr_t>(theta16_dense) % 16) == 0;
  SAMO_TRY((launch_expand<kModeDowncast, uint16_t>(a, 0, s)));
  return clear_ok();
}

// ---------------------------------------------------------------------------
// train.hpp: OptimizerConfig + adam_update

void samo_optimizer_config_default(samo_optimizer_config* cfg) {
  if (!cfg) return;
  cfg->learning_rate = 1e-3f;
  cfg->beta1 = 0.9f;
  cfg->beta2 = 0.999f;
  cfg->epsilon = 1e-8f;
  cfg->loss_scale = 1024.0f;
  cfg->weight_decay = 0.0f;
}

int samo_optimizer_config_validate(const samo_optimizer_config* cfg) {
  if (!cfg) return fail(SAMO_E_PARAMETER, "null config");
  // train.hpp:78-86
  if (!(cfg->beta1 >= 0.0f && cfg->beta1 < 1.0f) || !(cfg->beta2 >= 0.0f && cfg->beta2 < 1.0f))
    return fail(SAMO_E_PARAMETER, "betas must lie in [0, 1)");
  uint32_t bits;
  std::memcpy(&bits, &cfg->loss_scale, 4);
  if (!(cfg->loss_scale >= 1.0f) || (bits & 0x007FFFFFu) != 0)
    return fail(SAMO_E_PARAMETER, "loss_scale must be a power of two >= 1");
  return clear_ok();
}

static SamoAdamParams adam_params(const samo_optimizer_config* cfg) {
  SamoAdamParams p;
  p.lr = cfg->learning_rate;
  p.beta1 = cfg->beta1;
  p.beta2 = cfg->beta2;
  p.eps = cfg->epsilon;
  p.wd = cfg->weight_decay;
  return p;
}

int samo_adam_update(float* theta, float* m, float* v, const float* g, uint64_t n,
                     const samo_optimizer_config* cfg, float bias1, float bias2,
                     samo_stream_t stream) {
  SAMO_TRY(device_ok());
  if (!cfg) return fail(SAMO_E_PARAMETER, "null config");
  if (n && (!theta || !m || !v || !g)) return fail(SAMO_E_PARAMETER, "adam_update: null pointer");
  SAMO_TRY(launch_adam(theta, m, v, g, n, adam_params(cfg), bias1, bias2, as_stream(stream)));
  return clear_ok();
}

int samo_copy_async(void* dst, const void* src, uint64_t bytes, samo_stream_t stream) {
  if (bytes == 0) return clear_ok();
  if (!dst || !src) return fail(SAMO_E_PARAMETER, "copy: null pointer");
  SAMO_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream)));
  return clear_ok();
}

int samo_stream_synchronize(samo_stream_t stream) {
  SAMO_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
  return clear_ok();
}

// ---------------------------------------------------------------------------
// Synthetic data

int samo_synth_uniform_f32(float* out, uint64_t n, uint64_t seed, uint64_t stream_id, float bound,
                           samo_stream_t stream) {
  SAMO_TRY(device_ok());
  if (n && !out) return fail(SAMO_E_PARAMETER, "synth: null pointer");
  SAMO_TRY(launch_synth_f32(out, n, seed, stream_id, bound, as_stream(stream)));
  return clear_ok();
}

int samo_synth_uniform_f16(uint16_t* out, uint64_t n, uint64_t seed, uint64_t stream_id, float bound,
                           float scale, samo_stream_t stream) {
  SAMO_TRY(device_ok());
  if (n && !out) return fail(SAMO_E_PARAMETER, "synth: null pointer");
  SAMO_TRY(launch_synth_f16(out, n, seed, stream_id, bound, scale, as_stream(stream)));
  return clear_ok();
}

// ---------------------------------------------------------------------------
// NCCL communicator

}  // extern "C"

struct samo_comm {
  ncclComm_t comm = nullptr;  // gradient buckets
  ncclComm_t flag = nullptr;  // the skip indicator, concurrently with the buckets
  int nranks = 1;
  int rank = 0;
  uint8_t uid[SAMO_UNIQUE_ID_BYTES] = {};  // names the local rendezvous socket of the NVLS setup
  int nvls_seq = 0;                        // one multicast object per attached model
};

static int nccl_fail(ncclResult_t r, const char* what) {
  return fail(SAMO_E_NCCL, "%s: %s", what, ncclGetErrorString(r));
}

extern "C" {

int samo_comm_unique_id(uint8_t id_out[SAMO_UNIQUE_ID_BYTES]) {
  static_assert(sizeof(ncclUniqueId) == SAMO_UNIQUE_ID_BYTES, "ncclUniqueId size");
  if (!id_out) return fail(SAMO_E_PARAMETER, "null id buffer");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id_out, &id, sizeof(id));
  return clear_ok();
}

int samo_comm_create(const uint8_t id[SAMO_UNIQUE_ID_BYTES], int nranks, int rank, samo_comm** out) {
  SAMO_TRY(device_ok());
  if (!id || !out) return fail(SAMO_E_PARAMETER, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SAMO_E_PARAMETER, "bad rank/size");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  auto* c = new samo_comm();
  c->nranks = nranks;
  c->rank = rank;
  std::memcpy(c->uid, id, SAMO_UNIQUE_ID_BYTES);
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  // A second communicator carries the one-float skip indicator, so that it can
  // be reduced while gradient buckets are still in flight on the first.
  r = ncclCommSplit(c->comm, 0, rank, &c->flag, nullptr);
  if (r != ncclSuccess) {
    ncclCommDestroy(c->comm);
    delete c;
    return nccl_fail(r, "ncclCommSplit");
  }
  *out = c;
  return clear_ok();
}

int samo_comm_destroy(samo_comm* comm) {
  if (!comm) return clear_ok();
  if (comm->flag) ncclCommDestroy(comm->flag);
  if (comm->comm) ncclCommDestroy(comm->comm);
  delete comm;
  return clear_ok();
}

int samo_comm_size(const samo_comm* comm) { return comm ? comm->nranks : 0; }

int samo_allreduce_sum_f32(samo_comm* comm, float* buf, uint64_t n, samo_stream_t stream) {
  if (!comm || (n && !buf)) return fail(SAMO_E_PARAMETER, "allreduce: null argument");
  if (n == 0) return clear_ok();
  ncclResult_t r = ncclAllReduce(buf, buf, n, ncclFloat32, ncclSum, comm->comm, as_stream(stream));
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  return clear_ok();
}

}  // extern "C"

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
  std::vector<SamoLayerDev> layers_host;
  std::vector<SamoTile> tiles_host;
  samo_optimizer_config cfg{};
  samo_comm* comm = nullptr;
  bool finalized = false;
  bool grads_set = false;
  int grid_gather16 = 0, grid_gather32 = 0, grid_update16 = 0, grid_update32 = 0;
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
  SamoPeerSlots* slots = nullptr;       // this rank's signal area (in the block)
  // Backward sinks: first tile of every layer; per-layer row/column-block k
  // tables of the fused dW sink (built on first use).
  std::vector<uint32_t> layer_t;
  std::vector<uint32_t*> dw_kb;
  std::vector<uint64_t> dw_kb_in;
  // Peer mappings of the other ranks' model blocks (CUDA IPC) for the fused
  // peer-to-peer exchange; p2p_ok is agreed by every rank.
  void* peer_base[kMaxP2PRanks] = {};
  bool p2p_ok = false;
  // NVLS multicast of the binary16 weights (P2P step): every rank's theta16c
  // lives in VMM memory bound to one multicast object; the shard kernel
  // stores each vector once through mc_c16 and the switch replicates it.
  uint16_t* mc_c16 = nullptr;        // multicast mapping
  uint16_t* uc_c16 = nullptr;        // this rank's unicast mapping of the bound memory
  uint64_t nvls_bytes = 0;
  CUmemGenericAllocationHandle nvls_mem = 0, nvls_mc = 0;
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

static float* flag_ptr(const samo_model* md) { return md->g + md->n_al + kFlagOff; }

// Optional phase timing of the data-parallel step (samo_model_enable_phase_timing).
static int phase_mark(samo_model* md, int i, cudaStream_t s) {
  if (!md->phase_timing) return SAMO_OK;
  if (!md->phase_ev[i]) SAMO_CUDA_TRY(cudaEventCreate(&md->phase_ev[i]));
  SAMO_CUDA_TRY(cudaEventRecord(md->phase_ev[i], s));
  return SAMO_OK;
}

static uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

static void close_nvls(samo_model* md);

static void close_peers(samo_model* md) {
  close_nvls(md);
  for (int q = 0; q < kMaxP2PRanks; ++q) {
    if (md->peer_base[q] && md->peer_base[q] != md->block) cudaIpcCloseMemHandle(md->peer_base[q]);
    md->peer_base[q] = nullptr;
  }
  md->p2p_ok = false;
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

// ---------------------------------------------------------------------------
// NVLS multicast for the P2P weight push (SAMO_P2P_NVLS=1; off by default:
// measured at G = 4 the shard update takes 0.82 ms with one multimem.st per
// vector against 0.63 ms with G peer stores).  Driver API through
// cudaGetDriverEntryPoint (the runtime is linked statically).

struct NvlsApi {
  decltype(&cuMulticastCreate) mc_create = nullptr;
  decltype(&cuMulticastAddDevice) mc_add = nullptr;
  decltype(&cuMulticastBindMem) mc_bind = nullptr;
  decltype(&cuMulticastUnbind) mc_unbind = nullptr;
  decltype(&cuMulticastGetGranularity) mc_gran = nullptr;
  decltype(&cuMemCreate) mem_create = nullptr;
  decltype(&cuMemRelease) mem_release = nullptr;
  decltype(&cuMemAddressReserve) va_reserve = nullptr;
  decltype(&cuMemAddressFree) va_free = nullptr;
  decltype(&cuMemMap) mem_map = nullptr;
  decltype(&cuMemUnmap) mem_unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemExportToShareableHandle) export_h = nullptr;
  decltype(&cuMemImportFromShareableHandle) import_h = nullptr;
  decltype(&cuMemGetAllocationGranularity) mem_gran = nullptr;
  decltype(&cuCtxGetDevice) ctx_device = nullptr;
  bool ok = false;
};

static const NvlsApi& nvls_api() {
  static NvlsApi api;
  static bool init = false;
  if (init) return api;
  init = true;
  auto get = [](const char* name, auto& fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      return false;
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
    return true;
  };
  api.ok = get("cuMulticastCreate", api.mc_create) && get("cuMulticastAddDevice", api.mc_add) &&
           get("cuMulticastBindMem", api.mc_bind) && get("cuMulticastUnbind", api.mc_unbind) &&
           get("cuMulticastGetGranularity", api.mc_gran) && get("cuMemCreate", api.mem_create) &&
           get("cuMemRelease", api.mem_release) && get("cuMemAddressReserve", api.va_reserve) &&
           get("cuMemAddressFree", api.va_free) && get("cuMemMap", api.mem_map) &&
           get("cuMemUnmap", api.mem_unmap) && get("cuMemSetAccess", api.set_access) &&
           get("cuMemExportToShareableHandle", api.export_h) &&
           get("cuMemImportFromShareableHandle", api.import_h) &&
           get("cuMemGetAllocationGranularity", api.mem_gran) && get("cuCtxGetDevice", api.ctx_device);
  cudaGetLastError();
  return api;
}

// min over ranks of `ok` (a barrier as well).
static int agree(samo_comm* c, int* ok) {
  int* d = nullptr;
  cudaStream_t s = nullptr;
  SAMO_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int rc = SAMO_OK;
  cudaError_t e = cudaMalloc(&d, sizeof(int));
  if (e == cudaSuccess) e = cudaMemcpyAsync(d, ok, sizeof(int), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    const ncclResult_t nr = ncclAllReduce(d, d, 1, ncclInt32, ncclMin, c->comm, s);
    if (nr != ncclSuccess) rc = nccl_fail(nr, "ncclAllReduce(agree)");
  }
  if (rc == SAMO_OK && e == cudaSuccess) e = cudaMemcpyAsync(ok, d, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (rc == SAMO_OK && e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (rc == SAMO_OK && e != cudaSuccess) rc = cuda_fail(e, "agree");
  if (d) cudaFree(d);
  cudaStreamDestroy(s);
  return rc;
}

// Rank 0 hands the multicast object's file descriptor to the other ranks of
// this node over an abstract Unix socket named after the communicator id.
static void nvls_sock_name(const samo_comm* c, int seq, sockaddr_un* a, socklen_t* len) {
  std::memset(a, 0, sizeof(*a));
  a->sun_family = AF_UNIX;
  char name[96];
  int n = std::snprintf(name, sizeof(name), "samo-nvls-");
  for (int i = 0; i < 12; ++i) n += std::snprintf(name + n, sizeof(name) - n, "%02x", c->uid[i]);
  n += std::snprintf(name + n, sizeof(name) - n, "-%d", seq);
  std::memcpy(a->sun_path + 1, name, n);  // leading NUL: abstract namespace
  *len = static_cast<socklen_t>(offsetof(sockaddr_un, sun_path) + 1 + n);
}

static bool send_fd(int sock, int fd) {
  char byte = 0;
  iovec iov{&byte, 1};
  char ctl[CMSG_SPACE(sizeof(int))] = {};
  msghdr msg{};
  msg.msg_iov = &iov;
  msg.msg_iovlen = 1;
  msg.msg_control = ctl;
  msg.msg_controllen = sizeof(ctl);
  cmsghdr* cm = CMSG_FIRSTHDR(&msg);
  cm->cmsg_level = SOL_SOCKET;
  cm->cmsg_type = SCM_RIGHTS;
  cm->cmsg_len = CMSG_LEN(sizeof(int));
  std::memcpy(CMSG_DATA(cm), &fd, sizeof(int));
  return sendmsg(sock, &msg, 0) == 1;
}

static int recv_fd(int sock) {
  char byte = 0;
  iovec iov{&byte, 1};
  char ctl[CMSG_SPACE(sizeof(int))] = {};
  msghdr msg{};
  msg.msg_iov = &iov;
  msg.msg_iovlen = 1;
  msg.msg_control = ctl;
  msg.msg_controllen = sizeof(ctl);
  if (recvmsg(sock, &msg, 0) != 1) return -1;
  cmsghdr* cm = CMSG_FIRSTHDR(&msg);
  if (!cm || cm->cmsg_type != SCM_RIGHTS) return -1;
  int fd = -1;
  std::memcpy(&fd, CMSG_DATA(cm), sizeof(int));
  return fd;
}

static void close_nvls(samo_model* md) {
  const NvlsApi& api = nvls_api();
  if (!api.ok) return;
  if (md->mc_c16) {
    api.mem_unmap(reinterpret_cast<CUdeviceptr>(md->mc_c16), md->nvls_bytes);
    api.va_free(reinterpret_cast<CUdeviceptr>(md->mc_c16), md->nvls_bytes);
  }
  if (md->uc_c16) {
    api.mem_unmap(reinterpret_cast<CUdeviceptr>(md->uc_c16), md->nvls_bytes);
    api.va_free(reinterpret_cast<CUdeviceptr>(md->uc_c16), md->nvls_bytes);
  }
  if (md->nvls_mem) api.mem_release(md->nvls_mem);
  if (md->nvls_mc) api.mem_release(md->nvls_mc);
  md->mc_c16 = md->uc_c16 = nullptr;
  md->nvls_mem = md->nvls_mc = 0;
  md->nvls_bytes = 0;
}

// Collective (after open_peers succeeded).  Any failure on any rank leaves
// every rank on the peer-store path.
static int open_nvls(samo_model* md) {
  samo_comm* c = md->comm;
  const int G = c->nranks, r = c->rank;
  const NvlsApi& api = nvls_api();
  const bool dbg = env_int("SAMO_NVLS_DEBUG", 0) != 0;
  auto chk = [&](const char* what, CUresult e) {
    if (e != CUDA_SUCCESS && dbg) std::fprintf(stderr, "[samo nvls] rank %d: %s failed (%d)\n", r, what, int(e));
    return e == CUDA_SUCCESS;
  };
  if (dbg && !api.ok) std::fprintf(stderr, "[samo nvls] rank %d: driver entry points missing\n", r);
  int ok = (api.ok && env_int("SAMO_P2P_NVLS", 0) != 0) ? 1 : 0;
  SAMO_TRY(agree(c, &ok));
  if (!ok) return SAMO_OK;
  const int seq = c->nvls_seq++;
  CUdevice dev = 0;
  CUmulticastObjectProp mp{};
  CUmemAllocationProp ap{};
  size_t gran = 0, g2 = 0;
  int fd = -1;
  ok = chk("cuCtxGetDevice", api.ctx_device(&dev));
  if (ok) {
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = static_cast<int>(dev);
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // bindable to the multicast object
    mp.numDevices = static_cast<unsigned>(G);
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = 2 * (md->n_al + kArenaSlack) * sizeof(uint16_t);
    ok = chk("cuMulticastGetGranularity", api.mc_gran(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED)) &&
         chk("cuMemGetAllocationGranularity", api.mem_gran(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    gran = std::max(gran, g2);
    if (ok) mp.size = (mp.size + gran - 1) / gran * gran;
  }
  if (ok && r == 0) {
    ok = chk("cuMulticastCreate", api.mc_create(&md->nvls_mc, &mp)) &&
         chk("cuMemExportToShareableHandle", api.export_h(&fd, md->nvls_mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  }
  SAMO_TRY(agree(c, &ok));
  // file descriptor hand-over (rank 0 serves G - 1 connections)
  if (ok) {
    sockaddr_un addr;
    socklen_t alen;
    nvls_sock_name(c, seq, &addr, &alen);
    if (r == 0) {
      const int ls = socket(AF_UNIX, SOCK_STREAM, 0);
      ok = ls >= 0 && bind(ls, reinterpret_cast<sockaddr*>(&addr), alen) == 0 && listen(ls, G) == 0;
      for (int i = 1; ok && i < G; ++i) {
        pollfd pf{ls, POLLIN, 0};
        if (poll(&pf, 1, 30000) != 1) { ok = 0; break; }
        const int cs = accept(ls, nullptr, nullptr);
        ok = cs >= 0 && send_fd(cs, fd);
        if (cs >= 0) close(cs);
      }
      if (ls >= 0) close(ls);
    } else {
      int got = -1;
      for (int attempt = 0; attempt < 3000 && got < 0; ++attempt) {  // up to ~30 s for rank 0 to listen
        const int cs = socket(AF_UNIX, SOCK_STREAM, 0);
        if (cs < 0) break;
        if (connect(cs, reinterpret_cast<sockaddr*>(&addr), alen) == 0) got = recv_fd(cs);
        close(cs);
        if (got < 0) usleep(10000);
      }
      if (got < 0 && dbg) std::fprintf(stderr, "[samo nvls] rank %d: no file descriptor from rank 0\n", r);
      ok = got >= 0 && chk("cuMemImportFromShareableHandle",
                           api.import_h(&md->nvls_mc, reinterpret_cast<void*>(static_cast<intptr_t>(got)),
                                        CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
      if (got >= 0) close(got);
    }
  }
  if (fd >= 0) close(fd);
  SAMO_TRY(agree(c, &ok));
  if (ok) ok = chk("cuMulticastAddDevice", api.mc_add(md->nvls_mc, dev));
  SAMO_TRY(agree(c, &ok));  // every device added before any bind
  if (ok) {
    md->nvls_bytes = mp.size;
    CUdeviceptr uc = 0, mc = 0;
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = static_cast<int>(dev);
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    ok = chk("cuMemCreate", api.mem_create(&md->nvls_mem, mp.size, &ap, 0)) &&
         chk("cuMulticastBindMem", api.mc_bind(md->nvls_mc, 0, md->nvls_mem, 0, mp.size, 0)) &&
         chk("cuMemAddressReserve", api.va_reserve(&uc, mp.size, gran, 0, 0));
    if (ok) {
      ok = chk("cuMemMap(uc)", api.mem_map(uc, mp.size, 0, md->nvls_mem, 0)) &&
           chk("cuMemSetAccess(uc)", api.set_access(uc, mp.size, &acc, 1));
      if (ok) md->uc_c16 = reinterpret_cast<uint16_t*>(uc);
      else api.va_free(uc, mp.size);
    }
    if (ok) ok = api.va_reserve(&mc, mp.size, gran, 0, 0) == CUDA_SUCCESS;
    if (ok) {
      ok = chk("cuMemMap(mc)", api.mem_map(mc, mp.size, 0, md->nvls_mc, 0)) &&
           chk("cuMemSetAccess(mc)", api.set_access(mc, mp.size, &acc, 1));
      if (ok) md->mc_c16 = reinterpret_cast<uint16_t*>(mc);
      else api.va_free(mc, mp.size);
    }
  }
  cudaGetLastError();
  SAMO_TRY(agree(c, &ok));
  if (!ok) close_nvls(md);
  if (dbg) std::fprintf(stderr, "[samo nvls] rank %d: multicast %s\n", r, ok ? "on" : "off");
  return SAMO_OK;
}

// Collective over the attached communicator: exchanges the CUDA IPC handles
// of every rank's model block (all ranks have the same arena layout) and maps
// the peers.  Every rank ends with the same p2p_ok (min over ranks).
static int open_peers(samo_model* md) {
  samo_comm* c = md->comm;
  const int G = c->nranks, r = c->rank;
  if (G > kMaxP2PRanks) return SAMO_OK;
  int ok = 1;
  cudaIpcMemHandle_t mine{};
  if (cudaIpcGetMemHandle(&mine, md->block) != cudaSuccess) {
    cudaGetLastError();
    ok = 0;
  }
  cudaStream_t s = nullptr;
  SAMO_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  uint8_t* d = nullptr;
  SAMO_CUDA_TRY(cudaMalloc(&d, G * sizeof(cudaIpcMemHandle_t) + 16));
  int* dok = reinterpret_cast<int*>(d + G * sizeof(cudaIpcMemHandle_t));
  std::vector<cudaIpcMemHandle_t> all(G);
  int rc = SAMO_OK;
  do {
    cudaError_t e;
    if ((e = cudaMemcpyAsync(d + r * sizeof(cudaIpcMemHandle_t), &mine, sizeof(mine), cudaMemcpyHostToDevice, s))) {
      rc = cuda_fail(e, "ipc handle upload");
      break;
    }
    ncclResult_t nr = ncclAllGather(d + r * sizeof(cudaIpcMemHandle_t), d, sizeof(cudaIpcMemHandle_t), ncclUint8,
                                    c->comm, s);
    if (nr != ncclSuccess) {
      rc = nccl_fail(nr, "ncclAllGather(ipc handles)");
      break;
    }
    if ((e = cudaMemcpyAsync(all.data(), d, G * sizeof(cudaIpcMemHandle_t), cudaMemcpyDeviceToHost, s)) ||
        (e = cudaStreamSynchronize(s))) {
      rc = cuda_fail(e, "ipc handle download");
      break;
    }
    for (int q = 0; q < G && ok; ++q) {
      if (q == r) {
        md->peer_base[q] = md->block;
        continue;
      }
      if (cudaIpcOpenMemHandle(&md->peer_base[q], all[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        md->peer_base[q] = nullptr;
        ok = 0;
      }
    }
    // every rank must take the same path
    if ((e = cudaMemcpyAsync(dok, &ok, sizeof(int), cudaMemcpyHostToDevice, s))) {
      rc = cuda_fail(e, "ok upload");
      break;
    }
    nr = ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, c->comm, s);
    if (nr != ncclSuccess) {
      rc = nccl_fail(nr, "ncclAllReduce(p2p ok)");
      break;
    }
    if ((e = cudaMemcpyAsync(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost, s)) || (e = cudaStreamSynchronize(s))) {
      rc = cuda_fail(e, "ok download");
      break;
    }
  } while (false);
  cudaFree(d);
  cudaStreamDestroy(s);
  if (rc != SAMO_OK || !ok) {
    close_peers(md);
    return rc;
  }
  md->p2p_ok = true;
  return open_nvls(md);
}

extern "C" {

int samo_model_create(const samo_layer_desc* layers, int nlayers, uint32_t tile_elems,
                      samo_model** out) {
  SAMO_TRY(device_ok());
  if (!out || (nlayers > 0 && !layers)) return fail(SAMO_E_PARAMETER, "null argument");
  if (nlayers < 0) return fail(SAMO_E_PARAMETER, "negative layer count");
  if (tile_elems == 0) tile_elems = kModelTile;
  if (tile_elems < 1024 || tile_elems > 65536 || (tile_elems & (tile_elems - 1)))
    return fail(SAMO_E_PARAMETER, "tile_elems must be a power of two in [1024, 65536]");
  auto* md = new samo_model();
  md->nlayers = nlayers;
  md->tile_elems = tile_elems;
  md->dense_len.resize(nlayers);
  md->nnz.resize(nlayers);
  md->k_off.resize(nlayers + 1);
  md->d_off.resize(nlayers);
  md->idx_set.assign(nlayers, 0);
  uint64_t ntiles = 0;
  for (int l = 0; l < nlayers; ++l) {
    const uint64_t dl = layers[l].dense_len, nz = layers[l].nnz;
    if (dl == 0) {
      delete md;
      return fail(SAMO_E_DIMENSION, "tensor extents must be positive (layer %d)", l);
    }
    if (dl >= (1ull << 32)) {
      delete md;
      return fail(SAMO_E_PARAMETER, "layer too large for 32-bit indices (layer %d)", l);
    }
    if (nz > dl) {
      delete md;
      return fail(SAMO_E_DIMENSION, "layer %d keeps more indices than it has elements", l);
    }
    md->dense_len[l] = dl;
    md->nnz[l] = nz;
    md->k_off[l] = md->n_tot;
    md->n_tot += nz;
    md->d_off[l] = md->d_tot;
    md->d_tot += align_up(dl, 128);  // 256-byte aligned dense segments
    md->phi += dl;
    ntiles += (dl + tile_elems - 1) / tile_elems;
  }
  md->k_off[nlayers] = md->n_tot;
  if (ntiles > 0xFFFFFFFFull) {
    delete md;
    return fail(SAMO_E_PARAMETER, "too many tiles");
  }
  md->ntiles = static_cast<uint32_t>(ntiles);

  if (tile_elems > 16384) {  // two dense out tiles + the stage ring must fit in shared memory
    delete md;
    return fail(SAMO_E_PARAMETER, "the step kernels support tile_elems <= 16384");
  }
  md->grid_gather16 = step_grid(0, false, tile_elems);
  md->grid_gather32 = step_grid(0, true, tile_elems);
  md->grid_update16 = step_grid(1, false, tile_elems);
  md->grid_update32 = step_grid(1, true, tile_elems);
  md->grid_expand = expand_grid(tile_elems);
  const int max_grid = std::max(md->grid_update16, md->grid_update32);

  // Carve one allocation.
  // +64 elements of slack: the update kernel's 16-byte aligned bulk loads may
  // read up to 7 elements past the last kept one.
  const uint64_t n_al = align_up(md->n_tot + 64, 64);
  md->n_al = n_al;
  uint64_t off = 0;
  auto carve = [&](uint64_t bytes) {
    const uint64_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const uint64_t o_theta = carve(n_al * 4), o_m = carve(n_al * 4), o_v = carve(n_al * 4);
  // grad arena: n_al floats (the sharded exchange pads it to G * shard size,
  // G <= 128) + the skip-indicator slot at n_al + kFlagOff.
  const uint64_t o_g = carve((n_al + kArenaSlack) * 4), o_idx = carve(n_al * 4);
  const uint64_t o_off = carve(n_al * 2);
  const uint64_t o_t16 = carve(md->d_tot * 2), o_tiles = carve(ntiles * sizeof(SamoTile));
  const uint64_t o_layers = carve(std::max(1, nlayers) * sizeof(SamoLayerDev));
  const uint64_t o_koff = carve((nlayers + 1) * sizeof(uint64_t));
  const uint64_t o_st = carve(sizeof(SamoStepState));
  const uint64_t o_np = carve(static_cast<uint64_t>(max_grid) * kMaxBuckets * sizeof(float));
  // Buffers of the sharded exchange last: the step kernels' streams keep the
  // relative placement measured best.
  const uint64_t o_c16 = carve((n_al + kArenaSlack) * 2);
  const uint64_t o_n2 = carve(256);  // 16 norm^2 slots + arrival counter
  const uint64_t o_slots = carve(sizeof(SamoPeerSlots));
  md->block_bytes = off;
  cudaError_t e = cudaMalloc(&md->block, off);
  if (e != cudaSuccess) {
    delete md;
    return cuda_fail(e, "cudaMalloc(model arenas)");
  }
  char* b = static_cast<char*>(md->block);
  md->theta = reinterpret_cast<float*>(b + o_theta);
  md->m = reinterpret_cast<float*>(b + o_m);
  md->v = reinterpret_cast<float*>(b + o_v);
  md->g = reinterpret_cast<float*>(b + o_g);
  md->idx = reinterpret_cast<uint32_t*>(b + o_idx);
  md->off16 = reinterpret_cast<uint16_t*>(b + o_off);
  md->c16 = reinterpret_cast<uint16_t*>(b + o_c16);
  md->norm2 = reinterpret_cast<double*>(b + o_n2);
  md->done = reinterpret_cast<uint32_t*>(b + o_n2 + 16 * sizeof(double));
  md->slots = reinterpret_cast<SamoPeerSlots*>(b + o_slots);
  md->theta16 = reinterpret_cast<uint16_t*>(b + o_t16);
  md->tiles = reinterpret_cast<SamoTile*>(b + o_tiles);
  md->layers_dev = reinterpret_cast<SamoLayerDev*>(b + o_layers);
  md->k_off_dev = reinterpret_cast<uint64_t*>(b + o_koff);
  md->st = reinterpret_cast<SamoStepState*>(b + o_st);
  md->norm_partials = reinterpret_cast<float*>(b + o_np);
  e = cudaMemset(md->block, 0, off);
  if (e != cudaSuccess) {
    cudaFree(md->block);
    delete md;
    return cuda_fail(e, "cudaMemset(model arenas)");
  }
  SamoStepState st0{};
  st0.beta1_pow = 1.0f;  // AdamScalars (train.hpp:320-323)
  st0.beta2_pow = 1.0f;
  cudaMemcpy(md->st, &st0, sizeof(st0), cudaMemcpyHostToDevice);

  md->layers_host.resize(nlayers);
  md->tiles_host.resize(ntiles);
  uint64_t t = 0;
  for (int l = 0; l < nlayers; ++l) {
    md->layers_host[l].grad = nullptr;
    md->layers_host[l].theta16 = md->theta16 + md->d_off[l];
    md->layers_host[l].dense_len = md->dense_len[l];
    md->layers_host[l].k_off = md->k_off[l];
    for (uint64_t d = 0; d < md->dense_len[l]; d += tile_elems, ++t) {
      SamoTile& td = md->tiles_host[t];
      td.layer = static_cast<uint32_t>(l);
      td.dense_begin = static_cast<uint32_t>(d);
      td.dense_count = static_cast<uint32_t>(std::min<uint64_t>(tile_elems, md->dense_len[l] - d));
      td.pad_ = 0;
      td.k_begin = td.k_end = 0;
      td.out_off = md->d_off[l] + d;  // into the model's theta16 arena
      td.pad2_ = 0;
    }
  }
  if (nlayers > 0) {
    cudaMemcpy(md->layers_dev, md->layers_host.data(), nlayers * sizeof(SamoLayerDev),
               cudaMemcpyHostToDevice);
  }
  cudaMemcpy(md->k_off_dev, md->k_off.data(), (nlayers + 1) * sizeof(uint64_t),
             cudaMemcpyHostToDevice);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFree(md->block);
    delete md;
    return cuda_fail(e, "model setup");
  }
  samo_optimizer_config_default(&md->cfg);
  *out = md;
  return clear_ok();
}

int samo_model_destroy(samo_model* md) {
  if (!md) return clear_ok();
  if (md->graph) cudaGraphExecDestroy(md->graph);
  close_peers(md);
  if (md->capture_stream) cudaStreamDestroy(md->capture_stream);
  if (md->s_comm) cudaStreamDestroy(md->s_comm);
  if (md->s_flag) cudaStreamDestroy(md->s_flag);
  for (auto e : md->ev_k1) cudaEventDestroy(e);
  for (auto e : md->ev_ar) cudaEventDestroy(e);
  if (md->ev_fork) cudaEventDestroy(md->ev_fork);
  if (md->ev_flag) cudaEventDestroy(md->ev_flag);
  for (auto e : md->ev_sh) cudaEventDestroy(e);
  for (auto e : md->phase_ev)
    if (e) cudaEventDestroy(e);
  for (auto p : md->dw_kb)
    if (p) cudaFree(p);
  if (md->push_tiles) cudaFree(md->push_tiles);
  if (md->block) cudaFree(md->block);
  delete md;
  return clear_ok();
}

int samo_model_num_layers(const samo_model* md) { return md ? md->nlayers : 0; }

int samo_model_layer_view(const samo_model* md, int l, samo_layer_view* out) {
  if (!md || !out) return fail(SAMO_E_PARAMETER, "null argument");
  if (l < 0 || l >= md->nlayers) return fail(SAMO_E_INDEX, "layer %d out of range", l);
  const uint64_t k = md->k_off[l];
  out->theta16 = md->theta16 + md->d_off[l];
  out->theta32 = md->theta + k;
  out->adam_m = md->m + k;
  out->adam_v = md->v + k;
  out->grad32 = md->g + k;
  out->grad16 = reinterpret_cast<uint16_t*>(md->g) + k;
  out->indices = md->idx + k;
  out->dense_len = md->dense_len[l];
  out->nnz = md->nnz[l];
  out->k_offset = k;
  return clear_ok();
}

int samo_model_totals(const samo_model* md, uint64_t* phi, uint64_t* nnz, uint64_t* ntiles) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  if (phi) *phi = md->phi;
  if (nnz) *nnz = md->n_tot;
  if (ntiles) *ntiles = md->ntiles;
  return clear_ok();
}

uint64_t samo_model_device_bytes(const samo_model* md) { return md ? md->block_bytes : 0; }

int samo_model_set_indices(samo_model* md, int l, const uint32_t* idx, uint64_t n, int src_on_host,
                           samo_stream_t stream) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  if (l < 0 || l >= md->nlayers) return fail(SAMO_E_INDEX, "layer %d out of range", l);
  if (n != md->nnz[l]) return fail(SAMO_E_DIMENSION, "layer %d: %llu indices, expected %llu", l,
                                   (unsigned long long)n, (unsigned long long)md->nnz[l]);
  if (n && !idx) return fail(SAMO_E_PARAMETER, "null index pointer");
  cudaStream_t s = as_stream(stream);
  uint32_t* dst = md->idx + md->k_off[l];
  if (n && idx != dst) {  // idx == dst: validate in place (checkpoint load)
    SAMO_CUDA_TRY(cudaMemcpyAsync(dst, idx, n * 4,
                                  src_on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
  }
  // Validate on the device: strictly ascending, < dense_len.
  uint32_t* bad = reinterpret_cast<uint32_t*>(md->norm_partials);  // scratch (idle outside a step)
  SAMO_CUDA_TRY(cudaMemsetAsync(bad, 0, 4, s));
  SAMO_TRY(launch_check_indices(dst, n, md->dense_len[l], bad, s));
  uint32_t hbad = 0;
  SAMO_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s));
  SAMO_CUDA_TRY(cudaStreamSynchronize(s));
  if (hbad) return fail(SAMO_E_INDEX, "layer %d: indices must be strictly ascending and < dense_len", l);
  md->idx_set[l] = 1;
  md->finalized = false;
  return clear_ok();
}

int samo_model_finalize(samo_model* md, samo_stream_t stream) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  for (int l = 0; l < md->nlayers; ++l)
    if (!md->idx_set[l] && md->nnz[l] > 0)
      return fail(SAMO_E_STATE, "layer %d has no index set", l);
  cudaStream_t s = as_stream(stream);
  if (md->ntiles) {
    SAMO_CUDA_TRY(cudaMemcpyAsync(md->tiles, md->tiles_host.data(), md->ntiles * sizeof(SamoTile),
                                  cudaMemcpyHostToDevice, s));
    SAMO_TRY(launch_tiles_fill(md->tiles, md->ntiles, md->k_off_dev, md->idx, s));
    SAMO_TRY(launch_build_off16(md->tiles, md->ntiles, md->idx, md->off16, s));
    // k ranges back on the host: bucket planning for the overlapped step.
    SAMO_CUDA_TRY(cudaMemcpyAsync(md->tiles_host.data(), md->tiles, md->ntiles * sizeof(SamoTile),
                                  cudaMemcpyDeviceToHost, s));
  }
  SAMO_CUDA_TRY(cudaStreamSynchronize(s));
  md->finalized = true;
  if (md->graph) {
    cudaGraphExecDestroy(md->graph);
    md->graph = nullptr;
  }
  return clear_ok();
}

int samo_model_init_layer(samo_model* md, int l, const float* init, uint64_t dense_len,
                          samo_stream_t stream) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  if (l < 0 || l >= md->nlayers) return fail(SAMO_E_INDEX, "layer %d out of range", l);
  if (!md->finalized) return fail(SAMO_E_STATE, "init_layer requires finalize()");
  if (dense_len != md->dense_len[l])  // compress() length check, store.hpp:60-62
    return fail(SAMO_E_DIMENSION, "compress: dense length does not match index set");
  if (!init) return fail(SAMO_E_PARAMETER, "null init");
  cudaStream_t s = as_stream(stream);
  const uint64_t k = md->k_off[l], n = md->nnz[l];
  // theta32 = compress(init) (store.hpp:156); moments and grad32 zero (157-160)
  SAMO_TRY(launch_compress<uint32_t>(reinterpret_cast<const uint32_t*>(init), md->idx + k, n,
                                     reinterpret_cast<uint32_t*>(md->theta + k), s));
  if (n) {
    SAMO_CUDA_TRY(cudaMemsetAsync(md->m + k, 0, n * 4, s));
    SAMO_CUDA_TRY(cudaMemsetAsync(md->v + k, 0, n * 4, s));
    SAMO_CUDA_TRY(cudaMemsetAsync(md->g + k, 0, n * 4, s));
  }
  // theta16 = expand(half(theta32)) (store.hpp:162-166): this layer's tiles only.
  uint64_t t0 = 0;
  for (int j = 0; j < l; ++j) t0 += (md->dense_len[j] + md->tile_elems - 1) / md->tile_elems;
  const uint64_t nt = (md->dense_len[l] + md->tile_elems - 1) / md->tile_elems;
  ExpandArgs a{};
  a.tiles = md->tiles + t0;
  a.ntiles = static_cast<uint32_t>(nt);
  a.tile_elems = md->tile_elems;
  a.out_base = md->theta16;
  a.idx = md->idx;
  a.theta = md->theta;
  a.use_bulk = 1;
  SAMO_TRY((launch_expand<kModeDowncast, uint16_t>(a, 0, s)));
  return clear_ok();
}

int samo_model_set_config(samo_model* md, const samo_optimizer_config* cfg) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  SAMO_TRY(samo_optimizer_config_validate(cfg));
  md->cfg = *cfg;
  if (md->graph) {  // scalars are baked into the graph's kernel nodes
    cudaGraphExecDestroy(md->graph);
    md->graph = nullptr;
  }
  return clear_ok();
}

int samo_model_attach_comm(samo_model* md, samo_comm* comm) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  close_peers(md);
  md->comm = comm;
  if (comm && comm->nranks > 1) SAMO_TRY(open_peers(md));
  return clear_ok();
}

int samo_model_set_grads(samo_model* md, const uint16_t* const* ptrs, samo_stream_t stream) {
  if (!md || (md->nlayers && !ptrs)) return fail(SAMO_E_PARAMETER, "null argument");
  for (int l = 0; l < md->nlayers; ++l) {
    if (!ptrs[l]) return fail(SAMO_E_PARAMETER, "layer %d: null gradient pointer", l);
    if (reinterpret_cast<uintptr_t>(ptrs[l]) % 16)
      return fail(SAMO_E_PARAMETER, "layer %d: gradient pointer must be 16-byte aligned", l);
    md->layers_host[l].grad = ptrs[l];
  }
  if (md->nlayers) {
    SAMO_CUDA_TRY(cudaMemcpyAsync(md->layers_dev, md->layers_host.data(),
                                  md->nlayers * sizeof(SamoLayerDev), cudaMemcpyHostToDevice,
                                  as_stream(stream)));
  }
  md->grads_set = true;
  return clear_ok();
}

static int comm_size(const samo_model* md) { return md->comm ? md->comm->nranks : 1; }

static int step_ready(samo_model* md) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  if (!md->finalized) return fail(SAMO_E_STATE, "model not finalized");
  return SAMO_OK;
}

}  // extern "C"

// The gradient arena holds unscaled fp32 when it is exchanged between ranks,
// and the raw compressed binary16 gradient (the reference's grad16) otherwise.
static bool wide_grads(const samo_model* md) { return comm_size(md) > 1; }

static StepArgs step_args(samo_model* md) {
  StepArgs a{};
  a.tiles = md->tiles;
  a.ntiles = md->ntiles;
  a.tile_elems = md->tile_elems;
  a.layers = md->layers_dev;
  a.theta16 = md->theta16;
  a.off16 = md->off16;
  a.g = md->g;
  a.theta = md->theta;
  a.m = md->m;
  a.v = md->v;
  // inv_scale = 1/loss_scale exactly as train.hpp:619; with an fp32 exchange
  // 1/G is folded in (exact for power-of-two G).
  float inv_scale = 1.0f / md->cfg.loss_scale;
  const int G = comm_size(md);
  if (G > 1) inv_scale = inv_scale * (1.0f / static_cast<float>(G));
  a.inv_scale = inv_scale;
  a.prm = adam_params(&md->cfg);
  a.st = md->st;
  a.flag_slot = flag_ptr(md);
  a.norm_partials = md->norm_partials;
  a.norm_all = md->norm_partials;
  a.norm_count = 0;
  a.finalize = 1;
  return a;
}

// Splits the tiles into contiguous buckets of about equal kept-element count.
static int plan_buckets(samo_model* md) {
  if (md->nbuckets > 0) return SAMO_OK;
  int B = env_int("SAMO_BUCKETS", 8);
  B = std::max(1, std::min({B, kMaxBuckets, static_cast<int>(md->ntiles)}));
  md->bucket_t.assign(1, 0);
  const uint64_t n = md->n_tot;
  uint64_t done = 0;
  for (uint32_t t = 0; t < md->ntiles && static_cast<int>(md->bucket_t.size()) < B; ++t) {
    done = md->tiles_host[t].k_end;
    const uint64_t target = n * md->bucket_t.size() / B;
    if (done >= target && t + 1 < md->ntiles) md->bucket_t.push_back(t + 1);
  }
  md->bucket_t.push_back(md->ntiles);
  md->nbuckets = static_cast<int>(md->bucket_t.size()) - 1;
  md->reserve_sms = std::max(0, std::min(env_int("SAMO_NCCL_SMS", 16), num_sms() - 8));
  SAMO_CUDA_TRY(cudaStreamCreateWithFlags(&md->s_comm, cudaStreamNonBlocking));
  SAMO_CUDA_TRY(cudaStreamCreateWithFlags(&md->s_flag, cudaStreamNonBlocking));
  md->ev_k1.resize(md->nbuckets);
  md->ev_ar.resize(md->nbuckets);
  for (int b = 0; b < md->nbuckets; ++b) {
    SAMO_CUDA_TRY(cudaEventCreateWithFlags(&md->ev_k1[b], cudaEventDisableTiming));
    SAMO_CUDA_TRY(cudaEventCreateWithFlags(&md->ev_ar[b], cudaEventDisableTiming));
  }
  SAMO_CUDA_TRY(cudaEventCreateWithFlags(&md->ev_fork, cudaEventDisableTiming));
  SAMO_CUDA_TRY(cudaEventCreateWithFlags(&md->ev_flag, cudaEventDisableTiming));
  return SAMO_OK;
}

// One data-parallel step with the exchange overlapped:
//   S (caller):  K1[0] K1[1] ... K1[B-1]  |wait flag|  wait AR[0] K23[0] ... wait AR[B-1] K23[B-1]
//   s_comm:          AR[0]  AR[1] ...  AR[B-1]          (bucket b after K1[b])
//   s_flag:                               AR(flag)      (after K1[B-1], second communicator)
// Persistent grids leave `reserve_sms` SMs free so the NCCL kernels run
// concurrently with ours.
static int step_overlapped(samo_model* md, cudaStream_t S) {
  SAMO_TRY(plan_buckets(md));
  const int B = md->nbuckets;
  const int sms = num_sms();
  const int per_g = std::max(1, md->grid_gather32 / sms), per_u = std::max(1, md->grid_update32 / sms);
  const int gg = per_g * (sms - md->reserve_sms), gu = per_u * (sms - md->reserve_sms);
  const StepArgs base = step_args(md);
  SAMO_CUDA_TRY(cudaEventRecord(md->ev_fork, S));
  SAMO_CUDA_TRY(cudaStreamWaitEvent(md->s_comm, md->ev_fork, 0));
  SAMO_CUDA_TRY(cudaStreamWaitEvent(md->s_flag, md->ev_fork, 0));
  uint32_t norm_total = 0;
  for (int b = 0; b < B; ++b) {
    const uint32_t t0 = md->bucket_t[b], t1 = md->bucket_t[b + 1];
    StepArgs a = base;
    a.tiles = md->tiles + t0;
    a.ntiles = t1 - t0;
    SAMO_TRY(launch_gather(a, true, std::min<int>(gg, a.ntiles), S));
    SAMO_CUDA_TRY(cudaEventRecord(md->ev_k1[b], S));
    SAMO_CUDA_TRY(cudaStreamWaitEvent(md->s_comm, md->ev_k1[b], 0));
    const uint64_t k0 = md->tiles_host[t0].k_begin, k1 = md->tiles_host[t1 - 1].k_end;
    if (k1 > k0) {
      const ncclResult_t r = ncclAllReduce(md->g + k0, md->g + k0, k1 - k0, ncclFloat32, ncclSum,
                                           md->comm->comm, md->s_comm);
      if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(bucket)");
    }
    SAMO_CUDA_TRY(cudaEventRecord(md->ev_ar[b], md->s_comm));
    norm_total += std::min<uint32_t>(gu, a.ntiles);
  }
  SAMO_CUDA_TRY(cudaStreamWaitEvent(md->s_flag, md->ev_k1[B - 1], 0));
  {
    float* flag = flag_ptr(md);
    const ncclResult_t r = ncclAllReduce(flag, flag, 1, ncclFloat32, ncclSum, md->comm->flag, md->s_flag);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(flag)");
  }
  SAMO_CUDA_TRY(cudaEventRecord(md->ev_flag, md->s_flag));
  SAMO_CUDA_TRY(cudaStreamWaitEvent(S, md->ev_flag, 0));
  uint32_t norm_off = 0;
  for (int b = 0; b < B; ++b) {
    const uint32_t t0 = md->bucket_t[b], t1 = md->bucket_t[b + 1];
    SAMO_CUDA_TRY(cudaStreamWaitEvent(S, md->ev_ar[b], 0));
    StepArgs a = base;
    a.tiles = md->tiles + t0;
    a.ntiles = t1 - t0;
    const int grid = std::min<int>(gu, a.ntiles);
    a.norm_partials = md->norm_partials + norm_off;
    a.norm_all = md->norm_partials;
    a.norm_count = norm_total;
    a.finalize = (b == B - 1) ? 1u : 0u;
    norm_off += grid;
    SAMO_TRY(launch_update(a, true, grid, S));
  }
  return SAMO_OK;
}

static int exchange_mode(const samo_model* md) {
  if (md->exchange >= 0) return md->exchange;
  const char* e = getenv("SAMO_EXCHANGE");
  if (e && std::strcmp(e, "allreduce") == 0) return SAMO_EXCHANGE_ALLREDUCE;
  if (e && std::strcmp(e, "sharded") == 0) return SAMO_EXCHANGE_SHARDED;
  return md->p2p_ok ? SAMO_EXCHANGE_P2P : SAMO_EXCHANGE_SHARDED;
}

// One data-parallel step with the fused peer-to-peer exchange (ZeRO-1 on the
// compressed state, no NCCL on the data path):
//   K1 (binary16 compressed grads, local)
//   -> allreduce(skip flag)            [NCCL, 4 bytes: also the barrier]
//   -> k_shard_p2p on the own shard    [peer loads of every rank's grad16,
//                                       rank-ordered fp32 sum, Adam, peer
//                                       stores of the binary16 weights]
//   -> allreduce(norm^2)               [NCCL, 8 bytes: also the barrier]
//   -> expand every tile from theta16c -> scalars.
static int p2p_buckets(int G);
static bool p2p_push();
static bool p2p_pull();
static void set_pull_args(samo_model* md, const ShardPlan& p, StepArgs& a);
static int plan_shards(samo_model* md, ShardPlan& p, int B);
static int build_push_tiles(samo_model* md, const ShardPlan& p);
static int launch_gather_push(samo_model* md, cudaStream_t S);
static int step_p2p_pipelined(samo_model* md, cudaStream_t S, int B, bool gather);

// gather = false: the backward sinks have already written grad16 (and the
// local skip count) — the step starts at the exchange.
static int step_p2p(samo_model* md, cudaStream_t S, bool gather = true) {
  const int G = md->comm->nranks, r = md->comm->rank;
  if (p2p_buckets(G) > 1) return step_p2p_pipelined(md, S, p2p_buckets(G), gather);
  const uint64_t c = align_up((md->n_tot + G - 1) / G, 8);
  if (static_cast<uint64_t>(G) * c + 8 > md->n_al + kFlagOff)
    return fail(SAMO_E_PARAMETER, "too many ranks for the arena padding");
  float* flag = flag_ptr(md);
  const bool push = gather && p2p_push();
  const bool pull = p2p_pull();
  SAMO_TRY(plan_shards(md, md->p2p_plan, 1));
  if (md->p2p_plan.c != c) return fail(SAMO_E_STATE, "P2P plan mismatch");
  if (push) SAMO_TRY(build_push_tiles(md, md->p2p_plan));
  SAMO_TRY(phase_mark(md, 0, S));
  if (push) {
    SAMO_TRY(launch_gather_push(md, S));
  } else if (gather) {
    SAMO_TRY(launch_gather(step_args(md), false, md->grid_gather16, S));
  }
  SAMO_TRY(phase_mark(md, 1, S));
  ncclResult_t rr = ncclAllReduce(flag, flag, 1, ncclFloat32, ncclSum, md->comm->flag, S);
  if (rr != ncclSuccess) return nccl_fail(rr, "ncclAllReduce(flag)");
  SAMO_TRY(phase_mark(md, 2, S));
  P2PArgs pa{};
  const char* base = static_cast<const char*>(md->block);
  const size_t g_off = reinterpret_cast<const char*>(md->g) - base;
  const size_t c_off = reinterpret_cast<const char*>(md->c16) - base;
  for (int q = 0; q < G; ++q) {
    pa.g16[q] = reinterpret_cast<const uint16_t*>(static_cast<const char*>(md->peer_base[q]) + g_off);
    pa.c16[q] = reinterpret_cast<uint16_t*>(static_cast<char*>(md->peer_base[q]) + c_off);
  }
  pa.G = G;
  pa.rank = r;
  pa.theta = md->theta;
  pa.m = md->m;
  pa.v = md->v;
  pa.k0 = std::min<uint64_t>(r * c, md->n_tot);
  pa.k1 = std::min<uint64_t>((r + 1) * c, md->n_tot);
  pa.scale = (1.0f / md->cfg.loss_scale) * (1.0f / static_cast<float>(G));
  pa.prm = adam_params(&md->cfg);
  pa.st = md->st;
  pa.flag_slot = flag;
  pa.norm_partials = md->norm_partials;
  pa.norm2_out = md->norm2;
  pa.done = md->done;
  pa.bucket = -1;
  pa.tma = env_int("SAMO_P2P_TMA", 0);
  pa.push = push ? 1 : 0;
  pa.recv = reinterpret_cast<const uint16_t*>(md->g);
  pa.rstride = c;  // one bucket: [G][c]
  pa.i0 = 0;
  pa.local_c16 = pull ? 1 : 0;
  const bool nvls = md->mc_c16 && !pull;
  pa.mc16 = nvls ? md->mc_c16 : nullptr;
  if (pa.k1 > pa.k0) {
    SAMO_TRY(launch_shard_p2p(pa, S));
  } else {
    SAMO_CUDA_TRY(cudaMemsetAsync(md->norm2, 0, sizeof(double), S));
  }
  SAMO_TRY(phase_mark(md, 3, S));
  rr = ncclAllReduce(md->norm2, md->norm2, 1, ncclFloat64, ncclSum, md->comm->flag, S);
  if (rr != ncclSuccess) return nccl_fail(rr, "ncclAllReduce(norm)");
  SAMO_TRY(phase_mark(md, 4, S));
  StepArgs a = step_args(md);
  a.g = nvls ? md->uc_c16 : md->c16;
  if (pull) set_pull_args(md, md->p2p_plan, a);
  SAMO_TRY(launch_expand_c16(a, std::min<int>(md->grid_expand, md->ntiles), S));
  SAMO_TRY(phase_mark(md, 5, S));
  SAMO_TRY(launch_step_finalize(md->st, md->norm2, 1, flag, md->cfg.beta1, md->cfg.beta2, S));
  SAMO_TRY(phase_mark(md, 6, S));
  md->phase_count = 6;
  return SAMO_OK;
}

static int shard_buckets() { return std::max(1, std::min(env_int("SAMO_SHARD_BUCKETS", 4), 16)); }
// Buckets of the P2P step (DESIGN §7 sweeps): 8 from G = 3 — the pipelined
// schedule's peer-signalled flag exchange also avoids the NCCL barrier that
// stalls behind K1's NVLink pushes; at G = 2 one bucket is as fast.
static int p2p_buckets(int G) {
  return std::max(1, std::min(env_int("SAMO_P2P_BUCKETS", G >= 3 ? 8 : 1), kMaxP2PBuckets));
}

// One data-parallel step, ZeRO-1 style on the compressed state, pipelined
// over B k-buckets (bucket b = arena range [b*C, (b+1)*C), C = G*c, rank r
// owns [b*C + r*c, b*C + (r+1)*c) of every bucket):
//
//   S (caller):  K1[0] .. K1[B-1]                      wait AG[b] -> expand[b] ...   finalize
//   s_comm:           RS[0] .. RS[B-1] | wait flag | Adam[b] AG[b] ...
//   s_flag:                    flag allreduce (after K1[B-1])        norm allreduce
//
// K1[b] covers the tiles whose first kept element lies in bucket b (so RS[b]
// only waits for K1[0..b]); expand[b] covers the tiles whose last kept element
// lies in bucket b (so it only waits for AG[0..b]).  The reduce-scatter hides
// behind the gather kernels and the all-gather behind the expand kernels.
// Link bytes per rank 6n(G-1)/G instead of 8n(G-1)/G; Adam HBM traffic / G.
static int plan_shards(samo_model* md, ShardPlan& p, int B) {
  const int G = comm_size(md);
  if (p.G == G && p.B == B) return SAMO_OK;
  p.G = G;
  p.B = B;
  p.c = align_up((md->n_tot + static_cast<uint64_t>(G) * B - 1) / (static_cast<uint64_t>(G) * B), 8);
  p.C = p.c * G;
  if (p.C * B > md->n_al + kFlagOff)
    return fail(SAMO_E_PARAMETER, "too many ranks x buckets for the arena padding");
  auto bucket_of = [&](uint64_t k) { return static_cast<int>(std::min<uint64_t>(k / p.C, B - 1)); };
  p.k1_t.assign(B + 1, md->ntiles);
  p.ex_t.assign(B + 1, md->ntiles);
  p.k1_t[0] = p.ex_t[0] = 0;
  // first tile of each bucket (keys are non-decreasing in tile order)
  std::vector<int> k1_first(B + 1, -1), ex_first(B + 1, -1);
  for (uint32_t t = 0; t < md->ntiles; ++t) {
    const SamoTile& td = md->tiles_host[t];
    const int b1 = bucket_of(td.k_begin);
    const int be = bucket_of(td.k_end > 0 ? td.k_end - 1 : 0);
    for (int b = 1; b <= b1; ++b)
      if (p.k1_t[b] == md->ntiles) p.k1_t[b] = t;
    for (int b = 1; b <= be; ++b)
      if (p.ex_t[b] == md->ntiles) p.ex_t[b] = t;
  }
  (void)k1_first;
  (void)ex_first;
  for (int b = 1; b <= B; ++b) {  // monotone
    p.k1_t[b] = std::max(p.k1_t[b], p.k1_t[b - 1]);
    p.ex_t[b] = std::max(p.ex_t[b], p.ex_t[b - 1]);
  }
  p.k1_t[B] = p.ex_t[B] = md->ntiles;
  return SAMO_OK;
}

static int step_sharded(samo_model* md, cudaStream_t S) {
  SAMO_TRY(plan_buckets(md));  // side streams + events
  ShardPlan& p = md->shard_plan;
  SAMO_TRY(plan_shards(md, p, shard_buckets()));
  const int r = md->comm->rank, B = p.B;
  if (static_cast<int>(md->ev_sh.size()) < 2 * B) {
    for (int i = static_cast<int>(md->ev_sh.size()); i < 2 * B; ++i) {
      cudaEvent_t e;
      SAMO_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      md->ev_sh.push_back(e);
    }
  }
  cudaEvent_t* ev_k1 = md->ev_sh.data();
  cudaEvent_t* ev_ag = md->ev_sh.data() + B;
  cudaStream_t C = md->s_comm, F = md->s_flag;
  float* flag = flag_ptr(md);
  const StepArgs base = step_args(md);
  // Persistent grids leave SAMO_SHARD_NCCL_SMS SMs to the concurrent NCCL
  // kernels (reduce-scatter behind K1, all-gather behind the expand).
  const int sms = num_sms();
  const int reserve = std::max(0, std::min(env_int("SAMO_SHARD_NCCL_SMS", 0), sms - 8));
  const int gg = std::max(1, md->grid_gather32 / sms) * (sms - reserve);
  const int ge = std::max(1, md->grid_expand / sms) * (sms - reserve);

  SAMO_TRY(phase_mark(md, 0, S));
  SAMO_CUDA_TRY(cudaEventRecord(md->ev_fork, S));
  SAMO_CUDA_TRY(cudaStreamWaitEvent(C, md->ev_fork, 0));
  SAMO_CUDA_TRY(cudaStreamWaitEvent(F, md->ev_fork, 0));
  for (int b = 0; b < B; ++b) {
    StepArgs a = base;
    a.tiles = md->tiles + p.k1_t[b];
    a.ntiles = p.k1_t[b + 1] - p.k1_t[b];
    if (a.ntiles) SAMO_TRY(launch_gather(a, true, std::min<int>(gg, a.ntiles), S));
    SAMO_CUDA_TRY(cudaEventRecord(ev_k1[b], S));
    SAMO_CUDA_TRY(cudaStreamWaitEvent(C, ev_k1[b], 0));
    float* gb = md->g + b * p.C;
    const ncclResult_t rr = ncclReduceScatter(gb, gb + r * p.c, p.c, ncclFloat32, ncclSum, md->comm->comm, C);
    if (rr != ncclSuccess) return nccl_fail(rr, "ncclReduceScatter");
  }
  SAMO_TRY(phase_mark(md, 1, S));
  SAMO_CUDA_TRY(cudaStreamWaitEvent(F, ev_k1[B - 1], 0));
  ncclResult_t rr = ncclAllReduce(flag, flag, 1, ncclFloat32, ncclSum, md->comm->flag, F);
  if (rr != ncclSuccess) return nccl_fail(rr, "ncclAllReduce(flag)");
  SAMO_CUDA_TRY(cudaEventRecord(md->ev_flag, F));
  SAMO_CUDA_TRY(cudaStreamWaitEvent(C, md->ev_flag, 0));
  for (int b = 0; b < B; ++b) {
    ShardArgs sa{};
    sa.g = md->g;
    sa.theta = md->theta;
    sa.m = md->m;
    sa.v = md->v;
    sa.theta16c = md->c16;
    sa.k0 = std::min<uint64_t>(b * p.C + r * p.c, md->n_tot);
    sa.k1 = std::min<uint64_t>(b * p.C + (r + 1) * p.c, md->n_tot);
    sa.prm = adam_params(&md->cfg);
    sa.st = md->st;
    sa.flag_slot = flag;
    sa.norm_partials = md->norm_partials;
    sa.norm2_out = md->norm2 + b;
    sa.done = md->done;
    const uint64_t nv = (sa.k1 - sa.k0 + 3) / 4;
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(num_sms() * 8, (nv + 255) / 256)));
    if (sa.k1 > sa.k0) {
      SAMO_TRY(launch_adam_shard(sa, grid, C));
    } else {
      SAMO_CUDA_TRY(cudaMemsetAsync(md->norm2 + b, 0, sizeof(double), C));
    }
    uint16_t* cb = md->c16 + b * p.C;
    rr = ncclAllGather(cb + r * p.c, cb, p.c, ncclFloat16, md->comm->comm, C);
    if (rr != ncclSuccess) return nccl_fail(rr, "ncclAllGather");
    SAMO_CUDA_TRY(cudaEventRecord(ev_ag[b], C));
  }
  SAMO_CUDA_TRY(cudaStreamWaitEvent(F, ev_ag[B - 1], 0));
  rr = ncclAllReduce(md->norm2, md->norm2, B, ncclFloat64, ncclSum, md->comm->flag, F);
  if (rr != ncclSuccess) return nccl_fail(rr, "ncclAllReduce(norm)");
  SAMO_CUDA_TRY(cudaEventRecord(md->ev_flag, F));
  for (int b = 0; b < B; ++b) {
    SAMO_CUDA_TRY(cudaStreamWaitEvent(S, ev_ag[b], 0));
    if (b == 0) SAMO_TRY(phase_mark(md, 2, S));
    StepArgs a = base;
    a.g = md->c16;
    a.tiles = md->tiles + p.ex_t[b];
    a.ntiles = p.ex_t[b + 1] - p.ex_t[b];
    if (a.ntiles) SAMO_TRY(launch_expand_c16(a, std::min<int>(ge, a.ntiles), S));
  }
  SAMO_TRY(phase_mark(md, 3, S));
  SAMO_CUDA_TRY(cudaStreamWaitEvent(S, md->ev_flag, 0));
  SAMO_TRY(launch_step_finalize(md->st, md->norm2, B, flag, md->cfg.beta1, md->cfg.beta2, S));
  SAMO_TRY(phase_mark(md, 4, S));
  md->phase_count = 4;
  return SAMO_OK;
}

// Push mode of the P2P step (SAMO_P2P_PUSH, default on): K1 writes every
// kept gradient straight into its owner's receive buffer over NVLink, so the
// reduce-scatter traffic rides under K1's HBM-bound gather and the shard
// update reads all G contributions locally.  Receive buffer of rank r = its
// gradient arena as binary16, [G][B * c]: source q's element k (bucket b,
// owner r) at q * B * c + b * c + (k - b * C - r * c).
static bool p2p_push() { return env_int("SAMO_P2P_PUSH", 1) != 0; }
// Pull mode of the expand (SAMO_P2P_PULL=1, off by default): each owner keeps
// its binary16 weights in its own theta16c arena and every rank's expand
// pulls them over NVLink with its TMA loads.  Measured: the shard
// update drops 0.62 -> 0.46 ms at G = 4 but the expand rises 1.03 -> 1.29 ms
// (any ring depth), so pushing the weights stays the default.
static bool p2p_pull() { return env_int("SAMO_P2P_PULL", 0) != 0; }

static void set_pull_args(samo_model* md, const ShardPlan& p, StepArgs& a) {
  a.pull = 1;
  a.pB = static_cast<uint32_t>(p.B);
  a.pc = p.c;
  a.pC = p.C;
  const char* base = static_cast<const char*>(md->block);
  const size_t c_off = reinterpret_cast<const char*>(md->c16) - base;
  for (int q = 0; q < md->comm->nranks; ++q)
    a.peer16c[q] = reinterpret_cast<const uint16_t*>(static_cast<const char*>(md->peer_base[q]) + c_off);
}

static int build_push_tiles(samo_model* md, const ShardPlan& p) {
  if (md->push_tiles && md->push_G == p.G && md->push_B == p.B) return SAMO_OK;
  const uint64_t q = static_cast<uint64_t>(md->comm->rank);
  std::vector<SamoTile> out;
  out.reserve(md->ntiles + 2ull * p.G * p.B);
  for (uint32_t t = 0; t < md->ntiles; ++t) {
    SamoTile td = md->tiles_host[t];
    if (td.k_end <= td.k_begin) {
      td.pad_ = 0;
      td.pad2_ = 0;
      out.push_back(td);
      continue;
    }
    for (uint64_t cur = td.k_begin; cur < td.k_end;) {
      const uint64_t b = std::min<uint64_t>(cur / p.C, p.B - 1);
      const uint64_t r = (cur - b * p.C) / p.c;
      const uint64_t end = std::min<uint64_t>(td.k_end, b * p.C + (r + 1) * p.c);
      SamoTile piece = td;
      piece.k_begin = cur;
      piece.k_end = end;
      piece.pad_ = static_cast<uint32_t>(r);
      piece.pad2_ = q * p.B * p.c + b * p.c + (cur - b * p.C - r * p.c);
      out.push_back(piece);
      cur = end;
    }
  }
  if (md->push_tiles) cudaFree(md->push_tiles);
  md->push_tiles = nullptr;
  SAMO_CUDA_TRY(cudaMalloc(&md->push_tiles, out.size() * sizeof(SamoTile)));
  SAMO_CUDA_TRY(cudaMemcpy(md->push_tiles, out.data(), out.size() * sizeof(SamoTile), cudaMemcpyHostToDevice));
  md->push_ntiles = static_cast<uint32_t>(out.size());
  md->push_G = p.G;
  md->push_B = p.B;
  return SAMO_OK;
}

// K1 of the P2P step in push mode.
static int launch_gather_push(samo_model* md, cudaStream_t S) {
  StepArgs a = step_args(md);
  a.tiles = md->push_tiles;
  a.ntiles = md->push_ntiles;
  a.push = 1;
  const char* base = static_cast<const char*>(md->block);
  const size_t g_off = reinterpret_cast<const char*>(md->g) - base;
  for (int q = 0; q < md->comm->nranks; ++q)
    a.push16[q] = reinterpret_cast<uint16_t*>(static_cast<char*>(md->peer_base[q]) + g_off);
  return launch_gather(a, false, std::min<int>(md->grid_gather16, std::max<uint32_t>(1, a.ntiles)), S);
}

// The fused peer-to-peer step, pipelined over B k-buckets with no NCCL on
// it at all: the barriers are release/acquire signals in the ranks' peer-
// mapped SamoPeerSlots (bucket b = arena range [b*C, (b+1)*C), rank r owns
// [b*C + r*c, b*C + (r+1)*c)).
//
//   S:   K1 -> flag exchange -> shard[0] -> shard[1] -> ... shard[B-1]   | join -> finalize
//   E:                      wait[0] expand[0] -> wait[1] expand[1] -> ...
//
// shard[b] (NVLink-bound: peer loads of every rank's grad16, peer stores of
// the binary16 weights) publishes bucket b's completion + norm^2 to every
// rank; expand[b] (HBM-bound) covers the tiles whose last kept element lies
// in bucket b, once every rank has published bucket b.  The global skip flag
// forces every K1 to finish before any shard update, so K1 stays serial.
// Grids: SAMO_P2P_SHARD_CTAS / SAMO_P2P_EXPAND_CTAS per SM (tuning).
static int step_p2p_pipelined(samo_model* md, cudaStream_t S, int B, bool gather) {
  const int G = md->comm->nranks, r = md->comm->rank;
  SAMO_TRY(plan_buckets(md));  // side streams + events
  ShardPlan& p = md->p2p_plan;
  SAMO_TRY(plan_shards(md, p, B));
  if (static_cast<int>(md->ev_sh.size()) < 2 * B) {
    for (int i = static_cast<int>(md->ev_sh.size()); i < 2 * B; ++i) {
      cudaEvent_t e;
      SAMO_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      md->ev_sh.push_back(e);
    }
  }
  cudaStream_t E = md->s_comm;
  float* flag = flag_ptr(md);
  const bool push = gather && p2p_push();
  const bool pull = p2p_pull();
  if (push) SAMO_TRY(build_push_tiles(md, p));
  const char* base = static_cast<const char*>(md->block);
  const size_t g_off = reinterpret_cast<const char*>(md->g) - base;
  const size_t c_off = reinterpret_cast<const char*>(md->c16) - base;
  const size_t s_off = reinterpret_cast<const char*>(md->slots) - base;
  P2PArgs pa{};
  for (int q = 0; q < G; ++q) {
    char* pb = static_cast<char*>(md->peer_base[q]);
    pa.g16[q] = reinterpret_cast<const uint16_t*>(pb + g_off);
    pa.c16[q] = reinterpret_cast<uint16_t*>(pb + c_off);
    pa.slots[q] = reinterpret_cast<SamoPeerSlots*>(pb + s_off);
  }
  pa.G = G;
  pa.rank = r;
  pa.theta = md->theta;
  pa.m = md->m;
  pa.v = md->v;
  pa.scale = (1.0f / md->cfg.loss_scale) * (1.0f / static_cast<float>(G));
  pa.prm = adam_params(&md->cfg);
  pa.st = md->st;
  pa.flag_slot = flag;
  pa.norm_partials = md->norm_partials;
  pa.norm2_out = md->norm2;  // scratch: the bucket totals travel in the slots
  pa.done = md->done;
  const int sms = num_sms();
  pa.tma = env_int("SAMO_P2P_TMA", 0);
  pa.grid = sms * std::max(1, env_int("SAMO_P2P_SHARD_CTAS", pa.tma ? 1 : 2));
  const int ge = std::min(md->grid_expand, sms * std::max(1, env_int("SAMO_P2P_EXPAND_CTAS", 2)));

  pa.push = push ? 1 : 0;
  pa.recv = reinterpret_cast<const uint16_t*>(md->g);
  pa.rstride = static_cast<uint64_t>(B) * p.c;
  pa.local_c16 = pull ? 1 : 0;
  const bool nvls = md->mc_c16 && !pull;
  pa.mc16 = nvls ? md->mc_c16 : nullptr;
  SAMO_TRY(phase_mark(md, 0, S));
  if (push) {
    SAMO_TRY(launch_gather_push(md, S));
  } else if (gather) {
    SAMO_TRY(launch_gather(step_args(md), false, md->grid_gather16, S));
  }
  SAMO_TRY(phase_mark(md, 1, S));
  SAMO_TRY(launch_p2p_flag(pa.slots, G, r, flag, S));
  SAMO_TRY(phase_mark(md, 2, S));
  SAMO_CUDA_TRY(cudaEventRecord(md->ev_fork, S));
  SAMO_CUDA_TRY(cudaStreamWaitEvent(E, md->ev_fork, 0));
  for (int b = 0; b < B; ++b) {
    pa.k0 = std::min<uint64_t>(b * p.C + r * p.c, md->n_tot);
    pa.k1 = std::min<uint64_t>(b * p.C + (r + 1) * p.c, md->n_tot);
    pa.i0 = static_cast<uint64_t>(b) * p.c;
    pa.bucket = b;
    SAMO_TRY(launch_shard_p2p(pa, S));  // also when empty: it signals
  }
  StepArgs sbase = step_args(md);
  if (pull) set_pull_args(md, p, sbase);
  for (int b = 0; b < B; ++b) {
    SAMO_TRY(launch_p2p_wait(md->slots, G, b, E));
    StepArgs a = sbase;
    a.g = nvls ? md->uc_c16 : md->c16;
    a.tiles = md->tiles + p.ex_t[b];
    a.ntiles = p.ex_t[b + 1] - p.ex_t[b];
    if (a.ntiles) SAMO_TRY(launch_expand_c16(a, std::min<int>(ge, a.ntiles), E));
  }
  SAMO_CUDA_TRY(cudaEventRecord(md->ev_flag, E));
  SAMO_CUDA_TRY(cudaStreamWaitEvent(S, md->ev_flag, 0));
  SAMO_TRY(phase_mark(md, 3, S));
  SAMO_TRY(launch_step_finalize(md->st, md->slots->norm, B * kMaxP2PRanks, flag, md->cfg.beta1,
                                md->cfg.beta2, S));
  SAMO_TRY(launch_p2p_epoch(md->slots, S));
  SAMO_TRY(phase_mark(md, 4, S));
  md->phase_count = 4;
  return SAMO_OK;
}

extern "C" {

int samo_model_set_exchange(samo_model* md, int mode) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  if (mode != -1 && mode != SAMO_EXCHANGE_ALLREDUCE && mode != SAMO_EXCHANGE_SHARDED &&
      mode != SAMO_EXCHANGE_P2P)
    return fail(SAMO_E_PARAMETER, "unknown exchange mode %d", mode);
  md->exchange = mode;
  if (md->graph) {
    cudaGraphExecDestroy(md->graph);
    md->graph = nullptr;
  }
  return clear_ok();
}

int samo_model_enable_phase_timing(samo_model* md, int on) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  md->phase_timing = on != 0;
  md->phase_count = 0;
  return clear_ok();
}

int samo_model_phase_times(samo_model* md, float* ms, int cap) {
  if (!md || (cap > 0 && !ms)) return -fail(SAMO_E_PARAMETER, "null argument");
  const int n = std::min(cap, md->phase_count);
  if (n <= 0) return 0;
  if (cudaEventSynchronize(md->phase_ev[n]) != cudaSuccess) return -fail(SAMO_E_CUDA, "event sync");
  for (int i = 0; i < n; ++i) cudaEventElapsedTime(&ms[i], md->phase_ev[i], md->phase_ev[i + 1]);
  return n;
}

int samo_model_p2p_features(const samo_model* md) {
  if (!md || comm_size(md) <= 1) return 0;
  int f = 0;
  if (md->p2p_ok) f |= SAMO_P2P_MAPPED;
  if (md->p2p_ok && p2p_push()) f |= SAMO_P2P_PUSH;
  if (md->p2p_ok && p2p_pull()) f |= SAMO_P2P_PULL;
  if (md->mc_c16 && !p2p_pull()) f |= SAMO_P2P_NVLS;
  return f;
}

int samo_model_exchange_mode(const samo_model* md) {
  return md ? (comm_size(md) > 1 ? exchange_mode(md) : SAMO_EXCHANGE_NONE) : -1;
}

int samo_model_shard_layout(samo_model* md, uint64_t* chunk, uint64_t* stride, int* buckets,
                            int* rank) {
  if (!md || !chunk || !stride || !buckets || !rank) return fail(SAMO_E_PARAMETER, "null argument");
  if (comm_size(md) <= 1 || exchange_mode(md) == SAMO_EXCHANGE_ALLREDUCE) {
    *chunk = *stride = md->n_tot;
    *buckets = 1;
    *rank = 0;
    return clear_ok();
  }
  if (exchange_mode(md) == SAMO_EXCHANGE_P2P && p2p_buckets(comm_size(md)) > 1) {
    if (!md->finalized) return fail(SAMO_E_STATE, "model not finalized");
    SAMO_TRY(plan_shards(md, md->p2p_plan, p2p_buckets(comm_size(md))));
    *chunk = md->p2p_plan.c;
    *stride = md->p2p_plan.C;
    *buckets = md->p2p_plan.B;
    *rank = md->comm->rank;
    return clear_ok();
  }
  if (exchange_mode(md) == SAMO_EXCHANGE_P2P) {
    const uint64_t G = comm_size(md);
    *chunk = align_up((md->n_tot + G - 1) / G, 8);
    *stride = *chunk * G;
    *buckets = 1;
    *rank = md->comm->rank;
    return clear_ok();
  }
  if (!md->finalized) return fail(SAMO_E_STATE, "model not finalized");
  SAMO_TRY(plan_shards(md, md->shard_plan, shard_buckets()));
  *chunk = md->shard_plan.c;
  *stride = md->shard_plan.C;
  *buckets = md->shard_plan.B;
  *rank = md->comm->rank;
  return clear_ok();
}

int samo_model_gather(samo_model* md, samo_stream_t stream) {
  SAMO_TRY(step_ready(md));
  if (!md->grads_set) return fail(SAMO_E_STATE, "optimizer_step requires backward (no gradients set)");
  const bool wide = wide_grads(md);
  SAMO_TRY(launch_gather(step_args(md), wide, wide ? md->grid_gather32 : md->grid_gather16,
                         as_stream(stream)));
  return clear_ok();
}

int samo_model_exchange(samo_model* md, samo_stream_t stream) {
  SAMO_TRY(step_ready(md));
  if (comm_size(md) > 1) {
    // grad32 arena through the non-finite indicator slot, one in-place sum
    // (the zero padding in between is noise-free and < 1024 elements).
    SAMO_TRY(samo_allreduce_sum_f32(md->comm, md->g, md->n_al + kFlagOff + 1, stream));
  }
  return clear_ok();
}

static int sink_ready(samo_model* md, int l) {
  SAMO_TRY(step_ready(md));
  if (l < 0 || l >= md->nlayers) return fail(SAMO_E_INDEX, "layer %d out of range", l);
  if (comm_size(md) > 1 && (exchange_mode(md) != SAMO_EXCHANGE_P2P || !md->p2p_ok))
    return fail(SAMO_E_STATE,
                "backward sinks need a single-GPU model or the peer-to-peer exchange (binary16 gradient arena)");
  if (md->layer_t.empty()) {
    md->layer_t.assign(md->nlayers + 1, md->ntiles);
    for (uint32_t t = md->ntiles; t-- > 0;) md->layer_t[md->tiles_host[t].layer] = t;
    for (int q = md->nlayers - 1; q >= 0; --q)  // layers without tiles
      md->layer_t[q] = std::min(md->layer_t[q], md->layer_t[q + 1]);
  }
  return SAMO_OK;
}

int samo_model_sink_dense(samo_model* md, int l, const uint16_t* grad, samo_stream_t stream) {
  SAMO_TRY(sink_ready(md, l));
  if (!grad) return fail(SAMO_E_PARAMETER, "layer %d: null gradient pointer", l);
  if (reinterpret_cast<uintptr_t>(grad) % 16)
    return fail(SAMO_E_PARAMETER, "layer %d: gradient pointer must be 16-byte aligned", l);
  md->layers_host[l].grad = grad;
  SAMO_CUDA_TRY(cudaMemcpyAsync(md->layers_dev + l, &md->layers_host[l], sizeof(SamoLayerDev),
                                cudaMemcpyHostToDevice, as_stream(stream)));
  StepArgs a = step_args(md);
  a.tiles = md->tiles + md->layer_t[l];
  a.ntiles = md->layer_t[l + 1] - md->layer_t[l];
  if (a.ntiles) SAMO_TRY(launch_gather(a, false, std::min<int>(md->grid_gather16, a.ntiles), as_stream(stream)));
  return clear_ok();
}

int samo_model_sink_dw(samo_model* md, int l, const uint16_t* x, const uint16_t* dy, uint64_t batch,
                       uint64_t in, uint64_t out, samo_stream_t stream) {
  SAMO_TRY(sink_ready(md, l));
  SAMO_TRY(dw_check(batch, in, out, x, dy));
  if (in * out != md->dense_len[l])
    return fail(SAMO_E_DIMENSION, "layer %d: in x out = %llu, dense_len = %llu", l,
                static_cast<unsigned long long>(in * out), static_cast<unsigned long long>(md->dense_len[l]));
  cudaStream_t s = as_stream(stream);
  if (md->dw_kb.empty()) {
    md->dw_kb.assign(md->nlayers, nullptr);
    md->dw_kb_in.assign(md->nlayers, 0);
  }
  if (!md->dw_kb[l] || md->dw_kb_in[l] != in) {
    if (md->dw_kb[l]) cudaFree(md->dw_kb[l]);
    md->dw_kb[l] = nullptr;
    const uint64_t entries = (dw_col_blocks(out) + 1ull) * in;
    SAMO_CUDA_TRY(cudaMalloc(&md->dw_kb[l], entries * sizeof(uint32_t)));
    md->dw_kb_in[l] = in;
    SAMO_TRY(launch_build_rowblocks(md->idx + md->k_off[l], md->nnz[l], in, out, md->dw_kb[l], s));
  }
  DwArgs a{};
  a.M = in;
  a.N = out;
  a.K = batch;
  a.idx = md->idx + md->k_off[l];
  a.kb = md->dw_kb[l];
  a.g16 = reinterpret_cast<uint16_t*>(md->g) + md->k_off[l];
  a.flag = flag_ptr(md);
  SAMO_TRY(launch_dw_gemm(x, dy, a, 1, s));
  return clear_ok();
}

int samo_dw_gemm_f16(const uint16_t* x, const uint16_t* dy, uint64_t batch, uint64_t in, uint64_t out,
                     uint16_t* dw, samo_stream_t stream) {
  SAMO_TRY(device_ok());
  SAMO_TRY(dw_check(batch, in, out, x, dy));
  if (!dw) return fail(SAMO_E_PARAMETER, "dW GEMM: null output");
  if (reinterpret_cast<uintptr_t>(dw) % 16) return fail(SAMO_E_PARAMETER, "dW GEMM: output must be 16-byte aligned");
  DwArgs a{};
  a.M = in;
  a.N = out;
  a.K = batch;
  a.dw = dw;
  SAMO_TRY(launch_dw_gemm(x, dy, a, 0, as_stream(stream)));
  return clear_ok();
}

int samo_model_update(samo_model* md, samo_stream_t stream) {
  SAMO_TRY(step_ready(md));
  const bool wide = wide_grads(md);
  StepArgs a = step_args(md);
  const int grid = std::min<int>(wide ? md->grid_update32 : md->grid_update16, md->ntiles);
  a.norm_count = static_cast<uint32_t>(grid);
  SAMO_TRY(launch_update(a, wide, grid, as_stream(stream)));
  return clear_ok();
}

int samo_model_step_sunk(samo_model* md, samo_stream_t stream) {
  SAMO_TRY(step_ready(md));
  if (comm_size(md) > 1) {
    if (exchange_mode(md) != SAMO_EXCHANGE_P2P || !md->p2p_ok)
      return fail(SAMO_E_STATE, "step after backward sinks needs the peer-to-peer exchange");
    SAMO_TRY(step_p2p(md, as_stream(stream), false));
    return clear_ok();
  }
  SAMO_TRY(samo_model_update(md, stream));
  return clear_ok();
}

int samo_model_step(samo_model* md, samo_stream_t stream) {
  SAMO_TRY(step_ready(md));
  if (!md->grads_set) return fail(SAMO_E_STATE, "optimizer_step requires backward (no gradients set)");
  if (comm_size(md) > 1 && exchange_mode(md) == SAMO_EXCHANGE_P2P) {
    if (!md->p2p_ok) return fail(SAMO_E_STATE, "peer-to-peer exchange unavailable (IPC mapping failed)");
    SAMO_TRY(step_p2p(md, as_stream(stream)));
    return clear_ok();
  }
  if (comm_size(md) > 1 && exchange_mode(md) == SAMO_EXCHANGE_SHARDED) {
    SAMO_TRY(step_sharded(md, as_stream(stream)));
    return clear_ok();
  }
  if (comm_size(md) > 1 && env_int("SAMO_OVERLAP", 1)) {
    SAMO_TRY(step_overlapped(md, as_stream(stream)));
    return clear_ok();
  }
  SAMO_TRY(samo_model_gather(md, stream));
  SAMO_TRY(samo_model_exchange(md, stream));
  SAMO_TRY(samo_model_update(md, stream));
  return clear_ok();
}

int samo_model_step_graph(samo_model* md, samo_stream_t stream) {
  SAMO_TRY(step_ready(md));
  if (!md->grads_set) return fail(SAMO_E_STATE, "optimizer_step requires backward (no gradients set)");
  cudaStream_t s = as_stream(stream);
  if (md->graph && md->graph_comm != md->comm) {
    cudaGraphExecDestroy(md->graph);
    md->graph = nullptr;
  }
  if (!md->graph) {
    // Capture on a private stream (the legacy default stream cannot be
    // captured); the instantiated graph is then launched on the caller's.
    if (!md->capture_stream)
      SAMO_CUDA_TRY(cudaStreamCreateWithFlags(&md->capture_stream, cudaStreamNonBlocking));
    // Host-side planning (allocations, synchronous uploads) before capture.
    if (comm_size(md) > 1 && exchange_mode(md) == SAMO_EXCHANGE_P2P && md->p2p_ok && p2p_push()) {
      SAMO_TRY(plan_shards(md, md->p2p_plan, p2p_buckets(comm_size(md))));
      SAMO_TRY(build_push_tiles(md, md->p2p_plan));
    }
    const uint64_t before = samo_kernel_launch_count();
    SAMO_CUDA_TRY(cudaStreamBeginCapture(md->capture_stream, cudaStreamCaptureModeThreadLocal));
    int rc = samo_model_step(md, md->capture_stream);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(md->capture_stream, &graph);
    if (rc != SAMO_OK) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&md->graph, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      md->graph = nullptr;
      return cuda_fail(e, "cudaGraphInstantiate");
    }
    md->graph_kernels = samo_kernel_launch_count() - before;
    g_launches.fetch_sub(md->graph_kernels);  // captured, not launched
    md->graph_comm = md->comm;
  }
  SAMO_CUDA_TRY(cudaGraphLaunch(md->graph, s));
  note_launch(md->graph_kernels);
  return clear_ok();
}

int samo_model_step_record(samo_model* md, samo_step_record* out, samo_stream_t stream) {
  if (!md || !out) return fail(SAMO_E_PARAMETER, "null argument");
  SamoStepState st{};
  cudaStream_t s = as_stream(stream);
  SAMO_CUDA_TRY(cudaMemcpyAsync(&st, md->st, sizeof(st), cudaMemcpyDeviceToHost, s));
  SAMO_CUDA_TRY(cudaStreamSynchronize(s));
  out->t = st.t;
  out->skipped_steps = st.skipped_steps;
  out->beta1_pow = st.beta1_pow;
  out->beta2_pow = st.beta2_pow;
  out->grad_norm = st.grad_norm;
  out->last_skipped = st.last_skipped;
  return clear_ok();
}

int samo_model_step_record_async(samo_model* md, samo_step_record* out, samo_stream_t stream) {
  static_assert(sizeof(samo_step_record) == 32, "record layout");
  static_assert(offsetof(SamoStepState, last_skipped) == offsetof(samo_step_record, last_skipped),
                "SamoStepState starts with a samo_step_record");
  if (!md || !out) return fail(SAMO_E_PARAMETER, "null argument");
  SAMO_CUDA_TRY(cudaMemcpyAsync(out, md->st, sizeof(samo_step_record), cudaMemcpyDeviceToHost,
                                as_stream(stream)));
  return clear_ok();
}

int samo_model_set_step_record(samo_model* md, const samo_step_record* rec, samo_stream_t stream) {
  if (!md || !rec) return fail(SAMO_E_PARAMETER, "null argument");
  SamoStepState st{};
  st.t = rec->t;
  st.skipped_steps = rec->skipped_steps;
  st.beta1_pow = rec->beta1_pow;
  st.beta2_pow = rec->beta2_pow;
  st.grad_norm = rec->grad_norm;
  st.last_skipped = rec->last_skipped;
  cudaStream_t s = as_stream(stream);
  SAMO_CUDA_TRY(cudaMemcpyAsync(md->st, &st, sizeof(st), cudaMemcpyHostToDevice, s));
  SAMO_CUDA_TRY(cudaStreamSynchronize(s));
  return clear_ok();
}

int samo_model_check_invariants(samo_model* md, samo_stream_t stream) {
  SAMO_TRY(step_ready(md));
  cudaStream_t s = as_stream(stream);
  uint32_t* bad = reinterpret_cast<uint32_t*>(md->norm_partials);
  SAMO_CUDA_TRY(cudaMemsetAsync(bad, 0, 4, s));
  ExpandArgs a{};
  a.tiles = md->tiles;
  a.ntiles = md->ntiles;
  a.tile_elems = md->tile_elems;
  a.out_base = md->theta16;
  a.idx = md->idx;
  a.theta = md->theta;
  a.mismatch = bad;
  SAMO_TRY((launch_expand<kModeCheck, uint16_t>(a, 0, s)));
  uint32_t hbad = 0;
  SAMO_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s));
  SAMO_CUDA_TRY(cudaStreamSynchronize(s));
  if (hbad) return fail(SAMO_E_STATE, "theta16 disagrees with expand(half(theta32))");
  return clear_ok();
}

}  // extern "C"

// ---------------------------------------------------------------------------
// State formats: binary checkpoint of the arenas (serialize.hpp:120-190
// equivalent: indices, theta32, adam_m, adam_v per layer; theta16 rebuilt by
// downcast+expand on load, gradients not saved) plus the Adam scalars, and
// the memory report (store.hpp:129-147 measured_bytes).

namespace {

constexpr char kCkptMagic[8] = {'S', 'A', 'M', 'O', 'C', 'K', 'P', 'T'};
constexpr uint32_t kCkptVersion = 1;

struct CkptHeader {
  char magic[8];
  uint32_t version;
  uint32_t nlayers;
  uint32_t tile_elems;
  uint32_t reserved;
  samo_step_record rec;
};

// Streams `bytes` between a device buffer and a FILE through a pinned
// staging buffer (64 MiB chunks).
int stream_file(FILE* f, void* dev, uint64_t bytes, bool to_file, cudaStream_t s) {
  constexpr uint64_t kChunk = 64ull << 20;
  if (bytes == 0) return SAMO_OK;
  void* host = nullptr;
  SAMO_CUDA_TRY(cudaMallocHost(&host, std::min(bytes, kChunk)));
  int rc = SAMO_OK;
  for (uint64_t off = 0; off < bytes && rc == SAMO_OK; off += kChunk) {
    const uint64_t n = std::min(kChunk, bytes - off);
    char* d = static_cast<char*>(dev) + off;
    if (to_file) {
      cudaError_t e = cudaMemcpyAsync(host, d, n, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) rc = cuda_fail(e, "checkpoint D2H");
      else if (fwrite(host, 1, n, f) != n) rc = fail(SAMO_E_CONFIG, "checkpoint write failed");
    } else {
      if (fread(host, 1, n, f) != n) {
        rc = fail(SAMO_E_CONFIG, "checkpoint truncated");
        break;
      }
      cudaError_t e = cudaMemcpyAsync(d, host, n, cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) rc = cuda_fail(e, "checkpoint H2D");
    }
  }
  cudaFreeHost(host);
  return rc;
}

}  // namespace

extern "C" {

int samo_model_save(samo_model* md, const char* path, samo_stream_t stream) {
  SAMO_TRY(step_ready(md));
  if (!path) return fail(SAMO_E_PARAMETER, "null path");
  if (comm_size(md) > 1 && exchange_mode(md) != SAMO_EXCHANGE_ALLREDUCE)
    return fail(SAMO_E_STATE, "sharded state: theta32/m/v are only authoritative on each rank's shard");
  cudaStream_t s = as_stream(stream);
  CkptHeader h{};
  std::memcpy(h.magic, kCkptMagic, 8);
  h.version = kCkptVersion;
  h.nlayers = static_cast<uint32_t>(md->nlayers);
  h.tile_elems = md->tile_elems;
  SAMO_TRY(samo_model_step_record(md, &h.rec, stream));
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(SAMO_E_CONFIG, "cannot open %s for writing", path);
  int rc = SAMO_OK;
  if (fwrite(&h, sizeof(h), 1, f) != 1) rc = fail(SAMO_E_CONFIG, "checkpoint write failed");
  for (int l = 0; l < md->nlayers && rc == SAMO_OK; ++l) {
    const uint64_t d[2] = {md->dense_len[l], md->nnz[l]};
    if (fwrite(d, sizeof(d), 1, f) != 1) rc = fail(SAMO_E_CONFIG, "checkpoint write failed");
  }
  const uint64_t n = md->n_tot;
  if (rc == SAMO_OK) rc = stream_file(f, md->idx, n * 4, true, s);
  if (rc == SAMO_OK) rc = stream_file(f, md->theta, n * 4, true, s);
  if (rc == SAMO_OK) rc = stream_file(f, md->m, n * 4, true, s);
  if (rc == SAMO_OK) rc = stream_file(f, md->v, n * 4, true, s);
  if (std::fclose(f) != 0 && rc == SAMO_OK) rc = fail(SAMO_E_CONFIG, "checkpoint close failed");
  return rc == SAMO_OK ? clear_ok() : rc;
}

int samo_model_load(const char* path, uint32_t tile_elems, samo_model** out, samo_stream_t stream) {
  if (!path || !out) return fail(SAMO_E_PARAMETER, "null argument");
  SAMO_TRY(device_ok());
  FILE* f = std::fopen(path, "rb");
  if (!f) return fail(SAMO_E_CONFIG, "cannot open %s", path);
  CkptHeader h{};
  std::vector<samo_layer_desc> descs;
  int rc = SAMO_OK;
  if (fread(&h, sizeof(h), 1, f) != 1 || std::memcmp(h.magic, kCkptMagic, 8) != 0 ||
      h.version != kCkptVersion) {
    rc = fail(SAMO_E_CONFIG, "%s is not a SAMO checkpoint", path);
  }
  for (uint32_t l = 0; l < h.nlayers && rc == SAMO_OK; ++l) {
    uint64_t d[2];
    if (fread(d, sizeof(d), 1, f) != 1) rc = fail(SAMO_E_CONFIG, "checkpoint truncated");
    else descs.push_back({d[0], d[1]});
  }
  samo_model* md = nullptr;
  if (rc == SAMO_OK) {
    rc = samo_model_create(descs.data(), static_cast<int>(descs.size()),
                           tile_elems ? tile_elems : h.tile_elems, &md);
    if (rc == SAMO_E_DIMENSION) rc = fail(SAMO_E_CONFIG, "checkpoint layer table: %s", samo_last_error());
  }
  cudaStream_t s = as_stream(stream);
  if (rc == SAMO_OK) rc = stream_file(f, md->idx, md->n_tot * 4, false, s);
  if (rc == SAMO_OK) {
    // serialize.hpp:156-163: indices strictly ascending and in range -> ConfigError
    for (int l = 0; l < md->nlayers && rc == SAMO_OK; ++l) {
      const int r2 = samo_model_set_indices(md, l, md->idx + md->k_off[l], md->nnz[l], 0, stream);
      if (r2 == SAMO_E_INDEX) rc = fail(SAMO_E_CONFIG, "checkpoint indices must be strictly ascending and in range (layer %d)", l);
      else rc = r2;
    }
  }
  if (rc == SAMO_OK) rc = samo_model_finalize(md, stream);
  if (rc == SAMO_OK) rc = stream_file(f, md->theta, md->n_tot * 4, false, s);
  if (rc == SAMO_OK) rc = stream_file(f, md->m, md->n_tot * 4, false, s);
  if (rc == SAMO_OK) rc = stream_file(f, md->v, md->n_tot * 4, false, s);
  std::fclose(f);
  if (rc == SAMO_OK) {  // theta16 = expand(half(theta32)) for every tile (serialize.hpp:184-186)
    ExpandArgs a{};
    a.tiles = md->tiles;
    a.ntiles = md->ntiles;
    a.tile_elems = md->tile_elems;
    a.out_base = md->theta16;
    a.idx = md->idx;
    a.theta = md->theta;
    a.use_bulk = 1;
    rc = launch_expand<kModeDowncast, uint16_t>(a, 0, s);
  }
  if (rc == SAMO_OK) rc = samo_model_set_step_record(md, &h.rec, stream);
  if (rc != SAMO_OK) {
    samo_model_destroy(md);
    return rc;
  }
  *out = md;
  return clear_ok();
}

int samo_model_memory(const samo_model* md, samo_memory_report* out) {
  if (!md || !out) return fail(SAMO_E_PARAMETER, "null argument");
  const uint64_t phi = md->phi, n = md->n_tot;
  out->dense_params = phi;
  out->kept = n;
  out->theta16_bytes = md->d_tot * 2;
  out->compressed_state_bytes = 4 * md->n_al * 4;          // theta32, m, v, grad
  out->index_bytes = md->n_al * (4 + 2);                    // u32 index set + off16
  out->table_bytes = static_cast<uint64_t>(md->ntiles) * sizeof(SamoTile);
  out->device_bytes = md->block_bytes;
  // store.hpp:129-147 (per layer 2*dense + (2+4+4+8+4)*nnz [+ 2*nnz peak])
  out->reference_steady_bytes = 2 * phi + 22 * n;
  out->reference_peak_bytes = 2 * phi + 24 * n;
  return clear_ok();
}

}  // extern "C"
