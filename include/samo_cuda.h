/*
 * samo_cuda.h — C ABI of the B200-native SAMO per-step parameter-state path.
 *
 * Drop-in boundary for the hot path of the reference library
 * (the headers proj/include/samo/<name>.hpp).  The reference is a header-only
 * C++20 library whose "interface" is a set of free functions in namespace
 * `samo`; every entry point below names the reference symbol it replaces
 * (file:line).  The C++ mirror of the reference signatures lives in
 * include/samo_b200/samo.hpp and is a thin layer over this ABI.
 *
 * Conventions
 *  - Every function returns an int status (SAMO_OK == 0).  The status codes map
 *    1:1 onto the reference's exception taxonomy (error.hpp:9-36); the C++
 *    wrapper rethrows them as the same exception classes.  A human-readable
 *    message for the last failure on the calling thread is available from
 *    samo_last_error().
 *  - Pointers documented as "device" are CUDA device pointers; all such work
 *    is enqueued asynchronously on the given stream (0 = legacy default
 *    stream).  Argument checks are synchronous; device faults surface at the
 *    next synchronisation.
 *  - binary16 values travel as uint16_t bit patterns, binary32 as float.
 *  - Index sets are uint32 linear indices, strictly ascending and
 *    < dense_len (prune.hpp:21-27).
 *  - No function allocates on the hot path (samo_model_step*).  The one-time
 *    and API-parity entry points may allocate stream-ordered scratch.
 *  - There is no CPU fallback: if no CUDA device is present every compute
 *    entry point returns SAMO_E_CUDA.
 */
#ifndef SAMO_CUDA_H_
#define SAMO_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAMO_ABI_VERSION 1

/* Status codes.  error.hpp:9-36 defines the reference's exception classes. */
enum samo_status {
  SAMO_OK = 0,
  SAMO_E_DIMENSION = 1, /* DimensionError  (error.hpp:9-12)  */
  SAMO_E_PARAMETER = 2, /* ParameterError  (error.hpp:14-17) */
  SAMO_E_INDEX = 3,     /* IndexError      (error.hpp:19-22) */
  SAMO_E_STATE = 4,     /* StateError      (error.hpp:24-27) */
  SAMO_E_CONFIG = 5,    /* ConfigError     (error.hpp:29-32) */
  SAMO_E_CUDA = 6,      /* CUDA runtime failure (no reference analogue) */
  SAMO_E_NCCL = 7,      /* NCCL failure (no reference analogue) */
  SAMO_E_NOMEM = 8      /* device allocation failure */
};

typedef void* samo_stream_t; /* a cudaStream_t */

int samo_abi_version(void);
const char* samo_status_string(int status);
/* Message of the last non-OK status returned on this thread ("" if none). */
const char* samo_last_error(void);
/* Number of kernels this library has launched in this process (all streams). */
uint64_t samo_kernel_launch_count(void);

/* ------------------------------------------------------------------------ */
/* binary16 numerics — half.hpp:13-71.  Bit-exact with float_to_half_bits /  */
/* half_bits_to_float, NaN payload rules included.                           */
int samo_float_to_half(const float* in, uint16_t* out, uint64_t n,
                       samo_stream_t stream);
int samo_half_to_float(const uint16_t* in, float* out, uint64_t n,
                       samo_stream_t stream);

/* ------------------------------------------------------------------------ */
/* compress / expand — store.hpp:58-87.                                      */
/*                                                                           */
/* samo_compress_u16/u32 replace `compress<T>(const Tensor<T>&, const        */
/* PrunedIndexSet&)` (store.hpp:58-69): out[k] = dense[idx[k]].  `dense_len` */
/* is the tensor's element count and `ind_dense_len` the index set's         */
/* dense_len; they must agree (store.hpp:60-62 -> SAMO_E_DIMENSION).         */
int samo_compress_u16(const uint16_t* dense, uint64_t dense_len,
                      const uint32_t* idx, uint64_t n, uint64_t ind_dense_len,
                      uint16_t* out, samo_stream_t stream);
int samo_compress_u32(const uint32_t* dense, uint64_t dense_len,
                      const uint32_t* idx, uint64_t n, uint64_t ind_dense_len,
                      uint32_t* out, samo_stream_t stream);

/* samo_expand_u16/u32 replace `expand<T>(span<const T>, const             */
/* PrunedIndexSet&, shape)` (store.hpp:72-87): dense = 0; dense[idx[k]] =    */
/* values[k].  `n_values` must equal the index count (store.hpp:75-77) and   */
/* `shape_numel` must equal ind_dense_len (store.hpp:78-80).                 */
int samo_expand_u16(const uint16_t* values, uint64_t n_values,
                    const uint32_t* idx, uint64_t n, uint64_t ind_dense_len,
                    uint64_t shape_numel, uint16_t* dense_out,
                    samo_stream_t stream);
int samo_expand_u32(const uint32_t* values, uint64_t n_values,
                    const uint32_t* idx, uint64_t n, uint64_t ind_dense_len,
                    uint64_t shape_numel, uint32_t* dense_out,
                    samo_stream_t stream);

/* Downcast + expand (train.hpp:647-651, store.hpp:72-87):                   */
/* dense = 0; dense[idx[k]] = half_rn(theta32[k]).                           */
int samo_downcast_expand(const float* theta32, uint64_t n, const uint32_t* idx,
                         uint64_t dense_len, uint16_t* theta16_dense,
                         samo_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Adam — train.hpp:70-87 (OptimizerConfig), 320-347 (AdamScalars,          */
/* adam_update).                                                             */
typedef struct samo_optimizer_config {
  float learning_rate; /* 1e-3  */
  float beta1;         /* 0.9   */
  float beta2;         /* 0.999 */
  float epsilon;       /* 1e-8  */
  float loss_scale;    /* 1024, power of two >= 1 */
  float weight_decay;  /* 0, decoupled */
} samo_optimizer_config;

/* Fills the reference defaults (train.hpp:70-76). */
void samo_optimizer_config_default(samo_optimizer_config* cfg);
/* OptimizerConfig::validate (train.hpp:78-86) -> SAMO_E_PARAMETER. */
int samo_optimizer_config_validate(const samo_optimizer_config* cfg);

/* adam_update(theta, m, v, g, cfg, bias1, bias2) (train.hpp:332-347), in
 * place on device spans of length n.  IEEE per-op rounding, no contraction:
 * bit-exact with the reference built without FMA. Does no config checks, as
 * the reference. */
int samo_adam_update(float* theta, float* m, float* v, const float* g,
                     uint64_t n, const samo_optimizer_config* cfg, float bias1,
                     float bias2, samo_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Mask & index construction — prune.hpp:61-170.                            */
enum samo_prune_scope { SAMO_PRUNE_PER_LAYER = 0, SAMO_PRUNE_GLOBAL = 1 };

/* detail::unpruned_count (prune.hpp:76-79), host arithmetic in double. */
uint64_t samo_unpruned_count(double p, uint64_t n);

/* magnitude_prune (prune.hpp:99-170) on device.  `values[l]` (device) holds
 * layer l's dense fp32 values (len lens[l]); prunable[l] != 0 marks a prunable
 * layer.  idx_out[l] (device) must have room for lens[l] indices.  On return
 * counts_out[l] (host) holds the number of kept indices of layer l; the index
 * sets are strictly ascending.  Synchronises the stream.  Errors: p outside
 * [0,1) or a layer >= 2^32 elements -> SAMO_E_PARAMETER (prune.hpp:102-109).
 * Bit-exact with the reference for NaN-free inputs. */
int samo_magnitude_prune(const float* const* values, const uint64_t* lens,
                         const uint8_t* prunable, int nlayers, double p,
                         int scope, uint32_t* const* idx_out,
                         uint64_t* counts_out, samo_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Gradient exchange communicator (NCCL).  The reference has no executable   */
/* exchange; its cost model is sim.hpp:110-117 with the compressed volume of */
/* sim.hpp:272-276.                                                          */
typedef struct samo_comm samo_comm;
#define SAMO_UNIQUE_ID_BYTES 128
int samo_comm_unique_id(uint8_t id_out[SAMO_UNIQUE_ID_BYTES]);
/* Collective over `nranks` processes; the current CUDA device is used. */
int samo_comm_create(const uint8_t id[SAMO_UNIQUE_ID_BYTES], int nranks,
                     int rank, samo_comm** out);
int samo_comm_destroy(samo_comm* comm);
int samo_comm_size(const samo_comm* comm);
/* In-place sum allreduce of n floats (device). */
int samo_allreduce_sum_f32(samo_comm* comm, float* buf, uint64_t n,
                           samo_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Model state + step driver — store.hpp:22-55 (CompressedState, LayerState, */
/* ModelState), store.hpp:150-197 (make_layer_state, check_state_invariants),*/
/* train.hpp:594-656 (SamoTrainer backward sink + optimizer_step).           */
/*                                                                           */
/* A samo_model owns flat device arenas: theta32, adam_m, adam_v, grad32 and */
/* the u32 index arena (layer segments concatenated in layer order), the     */
/* dense binary16 theta16 arena (one 256-byte aligned segment per layer),    */
/* the dense-tile table and the device-resident Adam scalars.                */
typedef struct samo_model samo_model;

typedef struct samo_layer_desc {
  uint64_t dense_len; /* numel(shape) of the layer, >= 1 and < 2^32 */
  uint64_t nnz;       /* kept count = index set size */
} samo_layer_desc;

typedef struct samo_layer_view { /* all device pointers */
  uint16_t* theta16;  /* dense, dense_len elements */
  float* theta32;     /* nnz */
  float* adam_m;      /* nnz */
  float* adam_v;      /* nnz */
  float* grad32;      /* nnz */
  uint32_t* indices;  /* nnz */
  uint64_t dense_len;
  uint64_t nnz;
  uint64_t k_offset;  /* offset of this layer in the compressed arenas */
  uint16_t* grad16;   /* nnz; the same arena viewed as binary16 (grad16 of the
                         single-GPU and peer-to-peer steps) */
} samo_layer_view;

typedef struct samo_step_record { /* train.hpp:538-544 StepRecord + trainer counters */
  uint64_t t;             /* AdamScalars::t (train.hpp:321) */
  uint64_t skipped_steps; /* SamoTrainer::skipped_steps_ (train.hpp:701) */
  float beta1_pow;        /* AdamScalars::beta1_pow */
  float beta2_pow;        /* AdamScalars::beta2_pow */
  float grad_norm;        /* sqrt(sum g^2) over the (exchanged) grad32 */
  uint32_t last_skipped;  /* 1 when the last step was skipped */
} samo_step_record;

/* tile_elems: dense elements per tile, a power of two in [1024, 16384]; 0 picks
 * the default 16384 (the measured optimum for the step kernels on B200). */
int samo_model_create(const samo_layer_desc* layers, int nlayers,
                      uint32_t tile_elems, samo_model** out);
int samo_model_destroy(samo_model* model);
int samo_model_num_layers(const samo_model* model);
int samo_model_layer_view(const samo_model* model, int layer,
                          samo_layer_view* out);
/* Totals: dense parameter count phi, kept count n, tile count. */
int samo_model_totals(const samo_model* model, uint64_t* phi, uint64_t* nnz,
                      uint64_t* ntiles);
/* Bytes of device memory the model holds (arenas + tables). */
uint64_t samo_model_device_bytes(const samo_model* model);

/* Copies layer `layer`'s index set in (device or host source).  Indices must
 * be strictly ascending and < dense_len -> else SAMO_E_INDEX (the check
 * serialize.hpp:156-163 applies on load).  Synchronises the stream. */
int samo_model_set_indices(samo_model* model, int layer, const uint32_t* idx,
                           uint64_t n, int src_on_host, samo_stream_t stream);
/* Builds the dense-tile table from the index arena; call once after all
 * set_indices.  Synchronises the stream. */
int samo_model_finalize(samo_model* model, samo_stream_t stream);

/* make_layer_state (store.hpp:150-168) for one layer from dense fp32 initial
 * values (device): theta32 = compress(init), m = v = grad32 = 0,
 * theta16 = expand(half(theta32)). */
int samo_model_init_layer(samo_model* model, int layer, const float* init,
                          uint64_t dense_len, samo_stream_t stream);

int samo_model_set_config(samo_model* model, const samo_optimizer_config* cfg);
/* Attaches a communicator; grad32 is sum-allreduced between the gather and
 * Adam, with 1/nranks folded into the unscale. NULL detaches. */
int samo_model_attach_comm(samo_model* model, samo_comm* comm);

/* Gradient exchange of a data-parallel step (communicator size > 1):
 *  SAMO_EXCHANGE_ALLREDUCE — every rank keeps the full compressed state; the
 *    fp32 gradient arena is sum-allreduced (bucketed, overlapped with the
 *    step kernels) and every rank runs the full update.
 *  SAMO_EXCHANGE_SHARDED — ZeRO-1 on the compressed state: reduce-scatter of
 *    the gradient arena, Adam on the rank's shard only, all-gather of the
 *    compressed binary16 weights, local expand.  theta32/m/v are
 *    authoritative only on the rank's shard (samo_model_shard_layout);
 *    theta16 everywhere.  The exchange is pipelined over k-buckets
 *    (SAMO_SHARD_BUCKETS, default 4) behind the gather and expand kernels.
 *  SAMO_EXCHANGE_P2P — the sharded update with the exchange fused into our
 *    own kernels over NVLink peer memory (CUDA IPC mappings made by
 *    samo_model_attach_comm, which is then collective).  Push mode (default):
 *    K1 writes every kept binary16 gradient straight into its owner rank's
 *    receive buffer; the shard kernel sums its shard's G contributions in
 *    rank order in fp32 (deterministic, bit-exact with a rank-ordered sum
 *    for any G), runs Adam and stores the binary16 weights into every rank.
 *    From G = 3 the step is pipelined over k-buckets (shard update || expand)
 *    with release/acquire signals in peer memory as its only barriers — no
 *    NCCL call at all; at G = 2 two 4/8-byte NCCL allreduces are the
 *    barriers.  Tuning: SAMO_P2P_BUCKETS, SAMO_P2P_PUSH.
 * The default is P2P when the peer mappings succeeded on every rank, else
 * SHARDED (environment SAMO_EXCHANGE=allreduce|sharded overrides); mode -1
 * restores the default. */
enum samo_exchange_mode {
  SAMO_EXCHANGE_NONE = 0,
  SAMO_EXCHANGE_ALLREDUCE = 1,
  SAMO_EXCHANGE_SHARDED = 2,
  SAMO_EXCHANGE_P2P = 3
};
int samo_model_set_exchange(samo_model* model, int mode);
/* SAMO_EXCHANGE_NONE without a communicator of size > 1. */
int samo_model_exchange_mode(const samo_model* model);
/* Which peer-to-peer mechanisms this model's step uses (bitmask): peer
 * mappings made (agreed by every rank at samo_model_attach_comm), K1 pushes
 * the gradients to their owners (else the shard update pulls them). */
enum samo_p2p_feature {
  SAMO_P2P_MAPPED = 1,
  SAMO_P2P_PUSH = 2
};
int samo_model_p2p_features(const samo_model* model);
/* (The one-GPU local-group test harness is declared in samo_cuda_testing.h.) */
/* Compressed-arena elements this rank updates: for b in [0, buckets) the
 * range [b*stride + rank*chunk, b*stride + (rank+1)*chunk) clipped to the
 * arena (chunk = stride = nnz, buckets = 1, rank = 0 unless sharded). */
int samo_model_shard_layout(samo_model* model, uint64_t* chunk, uint64_t* stride,
                            int* buckets, int* rank);

/* Phase timing of the data-parallel step (CUDA events between its stages;
 * off by default).  samo_model_phase_times writes the durations (ms) of the
 * last step's phases and returns their count; it synchronises on the last
 * phase.  Phases: P2P serial — gather, flag allreduce, shard update, norm
 * allreduce, expand, finalize; P2P pipelined — gather, flag exchange,
 * shard update || expand, finalize; sharded — gather (+ reduce-scatter),
 * flag + shard Adam + first all-gather, expand (+ all-gathers), norm +
 * finalize. */
int samo_model_enable_phase_timing(samo_model* model, int on);
int samo_model_phase_times(samo_model* model, float* ms, int cap);

/* Element type of the dense gradients the model consumes (set_grads, the
 * backward sinks): binary16 (SAMO_GRAD_F16, the default — the reference's
 * Half, half.hpp) or bfloat16 (SAMO_GRAD_BF16: widened exactly to binary32,
 * bits << 16; then the same unscale, finite check and Adam).  The fused dW
 * sink stays binary16-only (SAMO_E_STATE). */
#define SAMO_GRAD_F16 0
#define SAMO_GRAD_BF16 1
int samo_model_set_grad_dtype(samo_model* model, int dtype);
int samo_model_grad_dtype(const samo_model* model);

/* Per-layer dense binary16 gradients (device pointers, 16-byte aligned,
 * dense_len elements each) consumed by the next step. `ptrs` is a host array
 * of nlayers device pointers; it is copied to the device on `stream`. */
int samo_model_set_grads(samo_model* model, const uint16_t* const* ptrs,
                         samo_stream_t stream);

/* Stage K1 alone — backward-sink gather (train.hpp:598-611) fused with the
 * unscale/cast/finite check of optimizer_step (train.hpp:619-629). */
int samo_model_gather(samo_model* model, samo_stream_t stream);
/* Backward sinks (the trainer's per-layer gradient sink, train.hpp:596-611):
 * each writes one layer's compressed binary16 gradient (grad16) and raises
 * the skip flag on a non-finite kept element, the moment the layer's
 * gradient is produced.  Single-GPU models or the peer-to-peer exchange (the
 * NCCL exchanges gather fp32 inside their step); follow the layers' sinks
 * with samo_model_step_sunk (= samo_model_update on one GPU).
 *
 * samo_model_sink_dense: K1 on one layer's tiles from its dense binary16
 * gradient (dense_len elements, 16-byte aligned).
 *
 * samo_model_sink_dw: the layer's weight gradient dW = X^T . dY
 * (mlp_backward, train.hpp:304-305; X [batch x in], dY [batch x out],
 * binary16 row-major, 16-byte aligned, in and out multiples of 8,
 * in * out == dense_len) computed on the tensor cores with the gather fused
 * into the GEMM epilogue: the dense gradient never reaches HBM.  The result
 * is bit-identical to samo_dw_gemm_f16 followed by samo_model_sink_dense.
 *
 * Data-parallel models (peer-to-peer exchange only): each rank sinks its own
 * gradients, then samo_model_step_sunk runs the exchange and the update. */
int samo_model_sink_dense(samo_model* model, int layer, const uint16_t* dense_grad,
                          samo_stream_t stream);
int samo_model_sink_dw(samo_model* model, int layer, const uint16_t* x, const uint16_t* dy,
                       uint64_t batch, uint64_t in, uint64_t out, samo_stream_t stream);

/* The step after the backward sinks: exchange (peer-to-peer) + update — the
 * same as samo_model_step without its gather.  Single-GPU models: the same as
 * samo_model_update. */
int samo_model_step_sunk(samo_model* model, samo_stream_t stream);

/* Dense weight gradient dW[in x out] = X^T . dY as binary16 (tcgen05 tensor
 * cores, fp32 accumulation, one rounding; matmul(transpose(x), dy) of
 * tensor.hpp:88-105 up to the fp32 summation order). */
int samo_dw_gemm_f16(const uint16_t* x, const uint16_t* dy, uint64_t batch, uint64_t in,
                     uint64_t out, uint16_t* dw, samo_stream_t stream);

/* Stage exchange alone (no-op without a communicator of size > 1). */
int samo_model_exchange(samo_model* model, samo_stream_t stream);
/* Stage K23 alone — skip decision, AdamScalars::advance, adam_update and
 * downcast+expand (train.hpp:632-654). */
int samo_model_update(samo_model* model, samo_stream_t stream);

/* One full SAMO step = gather + exchange + update, fully device-resident
 * (no host synchronisation). */
int samo_model_step(samo_model* model, samo_stream_t stream);
/* Same step through a CUDA graph captured on first use.  The optimizer
 * scalars live in device memory and are refreshed on `stream` before the
 * graph launch whenever samo_model_set_config changed them, so a per-step
 * learning-rate schedule replays the same graph; samo_model_set_exchange and
 * a new communicator drop the graph and the next call re-captures it. */
int samo_model_step_graph(samo_model* model, samo_stream_t stream);

/* Reads the device-resident step scalars (synchronises the stream). */
int samo_model_step_record(samo_model* model, samo_step_record* out,
                           samo_stream_t stream);
/* Enqueues a copy of the step scalars into `out` (pinned host memory for a
 * truly asynchronous copy); valid once the stream has been synchronised. */
int samo_model_step_record_async(samo_model* model, samo_step_record* out,
                                 samo_stream_t stream);
/* Overwrites the device-resident Adam scalars (checkpoint resume). */
int samo_model_set_step_record(samo_model* model, const samo_step_record* rec,
                               samo_stream_t stream);

/* check_state_invariants (store.hpp:171-197) on the device: theta16 ==
 * expand(half(theta32)) with exact zeros at pruned slots -> else
 * SAMO_E_STATE.  Synchronises the stream. */
int samo_model_check_invariants(samo_model* model, samo_stream_t stream);

/* Stream-ordered copy between any two host/device buffers (cudaMemcpyDefault);
 * used to read/write arena views (not part of the reference API). */
int samo_copy_async(void* dst, const void* src, uint64_t bytes, samo_stream_t stream);
int samo_stream_synchronize(samo_stream_t stream);

/* ------------------------------------------------------------------------ */
/* State formats.  Binary checkpoint with the fields of the reference's JSON  */
/* checkpoint (serialize.hpp:120-190: per-layer indices, theta32, adam_m,     */
/* adam_v; theta16 rebuilt by downcast+expand on load; gradients not saved)   */
/* plus the device Adam scalars.  Load errors -> SAMO_E_CONFIG, as the        */
/* reference's checkpoint_from_json.  Synchronise the stream.                 */
int samo_model_save(samo_model* model, const char* path, samo_stream_t stream);
int samo_model_load(const char* path, uint32_t tile_elems, samo_model** out,
                    samo_stream_t stream);

/* Memory accounting of a model (store.hpp:129-147 measured_bytes beside the
 * real device footprint). */
typedef struct samo_memory_report {
  uint64_t dense_params;           /* phi */
  uint64_t kept;                   /* n */
  uint64_t theta16_bytes;          /* dense binary16 weights */
  uint64_t compressed_state_bytes; /* theta32, m, v (two sets), grad arenas */
  uint64_t index_bytes;            /* u32 index sets + off16 */
  uint64_t table_bytes;            /* tile table */
  uint64_t device_bytes;           /* everything the model allocated */
  uint64_t reference_steady_bytes; /* measured_bytes(steady_state) = 2phi + 22n */
  uint64_t reference_peak_bytes;   /* measured_bytes(peak) = 2phi + 24n */
} samo_memory_report;
int samo_model_memory(const samo_model* model, samo_memory_report* out);

/* ------------------------------------------------------------------------ */
/* Synthetic data (bench/test inputs; not part of the reference API).        */
/* Counter-based: element i of stream s under seed gets                      */
/*   u = mix64(seed, s, i); c = (u >> 40) * 2^-24;                           */
/*   v = (2c - 1) * bound          (uniform_symmetric, train.hpp:93-100)     */
/* fp16 variant stores half_rn(v * scale).                                   */
int samo_synth_uniform_f32(float* out, uint64_t n, uint64_t seed,
                           uint64_t stream_id, float bound,
                           samo_stream_t stream);
int samo_synth_uniform_f16(uint16_t* out, uint64_t n, uint64_t seed,
                           uint64_t stream_id, float bound, float scale,
                           samo_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* SAMO_CUDA_H_ */
