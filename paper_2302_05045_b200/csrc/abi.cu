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

#include "host.cuh"

// ---------------------------------------------------------------------------
// Status plumbing.

namespace samo_dev {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void clear_error() { g_last_error.clear(); }

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
void unnote_launch(uint64_t n) { g_launches.fetch_sub(n, std::memory_order_relaxed); }

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
