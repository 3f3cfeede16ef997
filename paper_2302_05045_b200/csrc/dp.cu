// dp.cu — the data-parallel machinery of the model: CUDA IPC peer mappings
// (set up by samo_model_attach_comm), the bucket / shard / push-tile plans,
// and the step drivers — the fused peer-to-peer step (serial and pipelined,
// push / pull of the gradients), the NCCL sharded and overlapped-allreduce
// steps — plus the exchange-related C entry points.
#include <cstdio>
#include <cstring>
#include <string>

#include "host.cuh"

void close_peers(samo_model* md) {
  const bool ipc = !(md->comm && md->comm->local_group);  // a local group maps its peers directly
  for (int q = 0; q < kMaxP2PRanks; ++q) {
    if (ipc && md->peer_base[q] && md->peer_base[q] != md->block) cudaIpcCloseMemHandle(md->peer_base[q]);
    md->peer_base[q] = nullptr;
  }
  md->p2p_ok = false;
}

// Collective over the attached communicator: exchanges the CUDA IPC handles
// of every rank's model block (all ranks have the same arena layout) and maps
// the peers.  Every rank ends with the same p2p_ok (min over ranks).
int open_peers(samo_model* md) {
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
  if (const cudaError_t e = cudaMalloc(&d, G * sizeof(cudaIpcMemHandle_t) + 16)) {
    cudaStreamDestroy(s);
    return cuda_fail(e, "ipc handle buffer");
  }
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
  return set_spin_limit_from_env();
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
int step_overlapped(samo_model* md, cudaStream_t S) {
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

int exchange_mode(const samo_model* md) {
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

// gather = false: the backward sinks have already written grad16 (and the
// local skip count) — the step starts at the exchange.
static int step_p2p_pipelined(samo_model* md, cudaStream_t S, int B, bool gather);
static int launch_gather_push(samo_model* md, cudaStream_t S);

int step_p2p(samo_model* md, cudaStream_t S, bool gather) {
  const int G = md->comm->nranks, r = md->comm->rank;
  // A local group's ranks share one host thread: stepped one at a time they
  // would wait for each other forever.
  if (md->comm->local_group)
    return fail(SAMO_E_STATE, "a local-group member steps through samo_local_group_step");
  if (p2p_buckets(G) > 1) return step_p2p_pipelined(md, S, p2p_buckets(G), gather);
  const uint64_t c = align_up((md->n_tot + G - 1) / G, 8);
  if (static_cast<uint64_t>(G) * c + 8 > md->n_al + kFlagOff)
    return fail(SAMO_E_PARAMETER, "too many ranks for the arena padding");
  float* flag = flag_ptr(md);
  const bool push = gather ? p2p_push() : md->sunk_push;  // sunk: the sinks pushed already
  md->sunk_push = false;
  SAMO_TRY(plan_shards(md, md->p2p_plan, 1));
  if (md->p2p_plan.c != c) return fail(SAMO_E_STATE, "P2P plan mismatch");
  if (push) SAMO_TRY(build_push_tiles(md, md->p2p_plan));
  SAMO_TRY(phase_mark(md, 0, S));
  if (push && gather) {
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
  pa.grad_bf16 = md->grad_bf16;
  pa.prm = adam_params(&md->cfg);
  pa.cfg = md->capturing ? md->cfg_dev : nullptr;
  pa.st = md->st;
  pa.flag_slot = flag;
  pa.norm_partials = md->norm_partials;
  pa.norm2_out = md->norm2;
  pa.done = md->done;
  pa.bucket = -1;
  pa.push = push ? 1 : 0;
  pa.recv = reinterpret_cast<const uint16_t*>(md->g);
  pa.rstride = c;  // one bucket: [G][c]
  pa.i0 = 0;
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
  a.g = md->c16;
  SAMO_TRY(launch_expand_c16(a, std::min<int>(md->grid_expand, md->ntiles), S));
  SAMO_TRY(phase_mark(md, 5, S));
  SAMO_TRY(launch_step_finalize(md->st, md->norm2, 1, flag, md->cfg.beta1, md->cfg.beta2, md->capturing ? md->cfg_dev : nullptr, S));
  SAMO_TRY(phase_mark(md, 6, S));
  md->phase_count = 6;
  return SAMO_OK;
}

static int shard_buckets() { return std::max(1, std::min(env_int("SAMO_SHARD_BUCKETS", 4), 16)); }
// Buckets of the P2P step (DESIGN §7 sweeps): 8 from G = 3 — the pipelined
// schedule's peer-signalled flag exchange also avoids the NCCL barrier that
// stalls behind K1's NVLink pushes; at G = 2 one bucket is as fast.
int p2p_buckets(int G) {
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
int plan_shards(samo_model* md, ShardPlan& p, int B) {
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
  for (uint32_t t = 0; t < md->ntiles; ++t) {
    const SamoTile& td = md->tiles_host[t];
    const int b1 = bucket_of(td.k_begin);
    const int be = bucket_of(td.k_end > 0 ? td.k_end - 1 : 0);
    for (int b = 1; b <= b1; ++b)
      if (p.k1_t[b] == md->ntiles) p.k1_t[b] = t;
    for (int b = 1; b <= be; ++b)
      if (p.ex_t[b] == md->ntiles) p.ex_t[b] = t;
  }
  for (int b = 1; b <= B; ++b) {  // monotone
    p.k1_t[b] = std::max(p.k1_t[b], p.k1_t[b - 1]);
    p.ex_t[b] = std::max(p.ex_t[b], p.ex_t[b - 1]);
  }
  p.k1_t[B] = p.ex_t[B] = md->ntiles;
  return SAMO_OK;
}

int step_sharded(samo_model* md, cudaStream_t S) {
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
    sa.cfg = md->capturing ? md->cfg_dev : nullptr;
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
  SAMO_TRY(launch_step_finalize(md->st, md->norm2, B, flag, md->cfg.beta1, md->cfg.beta2, md->capturing ? md->cfg_dev : nullptr, S));
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
bool p2p_push() { return env_int("SAMO_P2P_PUSH", 1) != 0; }
int build_push_tiles(samo_model* md, const ShardPlan& p) {
  if (md->push_tiles && md->push_G == p.G && md->push_B == p.B) return SAMO_OK;
  const uint64_t q = static_cast<uint64_t>(md->comm->rank);
  std::vector<SamoTile> out;
  out.reserve(md->ntiles + 2ull * p.G * p.B);
  md->push_layer_t.assign(md->nlayers + 1, 0);
  int cur_layer = -1;
  for (uint32_t t = 0; t < md->ntiles; ++t) {
    SamoTile td = md->tiles_host[t];
    while (cur_layer < static_cast<int>(td.layer)) md->push_layer_t[++cur_layer] = static_cast<uint32_t>(out.size());
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
  while (cur_layer < md->nlayers) md->push_layer_t[++cur_layer] = static_cast<uint32_t>(out.size());
  if (md->push_tiles) cudaFree(md->push_tiles);
  md->push_tiles = nullptr;
  SAMO_CUDA_TRY(cudaMalloc(&md->push_tiles, out.size() * sizeof(SamoTile)));
  SAMO_CUDA_TRY(cudaMemcpy(md->push_tiles, out.data(), out.size() * sizeof(SamoTile), cudaMemcpyHostToDevice));
  md->push_ntiles = static_cast<uint32_t>(out.size());
  md->push_G = p.G;
  md->push_B = p.B;
  return SAMO_OK;
}

int push_sink_prepare(samo_model* md) {
  const int B = p2p_buckets(md->comm->nranks);
  SAMO_TRY(plan_shards(md, md->p2p_plan, B));
  return build_push_tiles(md, md->p2p_plan);
}

// One layer's share of the exchange, sent during the backward (last layer
// first, train.hpp:287-313): K1 in push mode over the layer's push pieces
// (local_src == nullptr), or the push copy of its binary16 gradients that a
// fused dW sink gathered into local_src.
int push_sink_layer(samo_model* md, int l, const uint16_t* local_src, cudaStream_t s) {
  StepArgs a = step_args(md);
  a.tiles = md->push_tiles + md->push_layer_t[l];
  a.ntiles = md->push_layer_t[l + 1] - md->push_layer_t[l];
  a.push = 1;
  const char* base = static_cast<const char*>(md->block);
  const size_t g_off = reinterpret_cast<const char*>(md->g) - base;
  for (int q = 0; q < md->comm->nranks; ++q)
    a.push16[q] = reinterpret_cast<uint16_t*>(static_cast<char*>(md->peer_base[q]) + g_off);
  md->sunk_push = true;
  if (a.ntiles == 0) return SAMO_OK;
  if (local_src) return launch_push_copy(a, local_src, s);
  return launch_gather(a, false, std::min<int>(md->grid_gather16, a.ntiles), s);
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
// The pipelined step in phases, so that a local group (one device, no
// concurrency between its ranks' streams) can queue every rank's phase
// before any rank's next one: then each wait below is already satisfied.
struct P2PStep {
  P2PArgs pa{};
  StepArgs sbase{};
  int B = 1, ge = 0;
  bool push = false, gather = true;
};

static int p2p_prepare(samo_model* md, int B, bool gather, P2PStep& sp) {
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
  sp.B = B;
  sp.gather = gather;
  sp.push = gather ? p2p_push() : md->sunk_push;  // sunk: the sinks pushed already
  md->sunk_push = false;
  if (sp.push) SAMO_TRY(build_push_tiles(md, p));
  const char* base = static_cast<const char*>(md->block);
  const size_t g_off = reinterpret_cast<const char*>(md->g) - base;
  const size_t c_off = reinterpret_cast<const char*>(md->c16) - base;
  const size_t s_off = reinterpret_cast<const char*>(md->slots) - base;
  P2PArgs& pa = sp.pa;
  pa = P2PArgs{};
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
  pa.grad_bf16 = md->grad_bf16;
  pa.prm = adam_params(&md->cfg);
  pa.cfg = md->capturing ? md->cfg_dev : nullptr;
  pa.st = md->st;
  pa.flag_slot = flag_ptr(md);
  pa.norm_partials = md->norm_partials;
  pa.norm2_out = md->norm2;  // scratch: the bucket totals travel in the slots
  pa.done = md->done;
  const int sms = num_sms();
  pa.grid = sms * std::max(1, env_int("SAMO_P2P_SHARD_CTAS", 2));
  sp.ge = std::min(md->grid_expand, sms * std::max(1, env_int("SAMO_P2P_EXPAND_CTAS", 2)));
  pa.push = sp.push ? 1 : 0;
  pa.recv = reinterpret_cast<const uint16_t*>(md->g);
  pa.rstride = static_cast<uint64_t>(B) * p.c;
  sp.sbase = step_args(md);
  return SAMO_OK;
}

static int p2p_gather(samo_model* md, const P2PStep& sp, cudaStream_t S) {
  if (sp.push && sp.gather) return launch_gather_push(md, S);
  if (sp.gather) return launch_gather(step_args(md), false, md->grid_gather16, S);
  return SAMO_OK;
}

// phase 1: publish this rank's skip indicator; 2: wait for every rank's and
// sum them in rank order; 3: both (one kernel).
static int p2p_flag(samo_model* md, const P2PStep& sp, int phase, cudaStream_t S) {
  return launch_p2p_flag(sp.pa.slots, sp.pa.G, sp.pa.rank, flag_ptr(md), phase, S);
}

static int p2p_shards(samo_model* md, P2PStep& sp, cudaStream_t S) {
  const ShardPlan& p = md->p2p_plan;
  const int r = md->comm->rank;
  for (int b = 0; b < sp.B; ++b) {
    sp.pa.k0 = std::min<uint64_t>(b * p.C + r * p.c, md->n_tot);
    sp.pa.k1 = std::min<uint64_t>(b * p.C + (r + 1) * p.c, md->n_tot);
    sp.pa.i0 = static_cast<uint64_t>(b) * p.c;
    sp.pa.bucket = b;
    SAMO_TRY(launch_shard_p2p(sp.pa, S));  // also when empty: it signals
  }
  return SAMO_OK;
}

static int p2p_expand(samo_model* md, const P2PStep& sp, cudaStream_t E) {
  const ShardPlan& p = md->p2p_plan;
  for (int b = 0; b < sp.B; ++b) {
    SAMO_TRY(launch_p2p_wait(md->slots, sp.pa.G, b, E));
    StepArgs a = sp.sbase;
    a.g = md->c16;
    a.tiles = md->tiles + p.ex_t[b];
    a.ntiles = p.ex_t[b + 1] - p.ex_t[b];
    if (a.ntiles) SAMO_TRY(launch_expand_c16(a, std::min<int>(sp.ge, a.ntiles), E));
  }
  return SAMO_OK;
}

static int p2p_finish(samo_model* md, const P2PStep& sp, cudaStream_t S) {
  SAMO_TRY(launch_step_finalize(md->st, md->slots->norm, sp.B * kMaxP2PRanks, flag_ptr(md), md->cfg.beta1,
                                md->cfg.beta2, md->capturing ? md->cfg_dev : nullptr, S));
  return launch_p2p_epoch(md->slots, S);
}

static int step_p2p_pipelined(samo_model* md, cudaStream_t S, int B, bool gather) {
  P2PStep sp;
  SAMO_TRY(p2p_prepare(md, B, gather, sp));
  cudaStream_t E = md->s_comm;
  SAMO_TRY(phase_mark(md, 0, S));
  SAMO_TRY(p2p_gather(md, sp, S));
  SAMO_TRY(phase_mark(md, 1, S));
  SAMO_TRY(p2p_flag(md, sp, 3, S));
  SAMO_TRY(phase_mark(md, 2, S));
  SAMO_CUDA_TRY(cudaEventRecord(md->ev_fork, S));
  SAMO_CUDA_TRY(cudaStreamWaitEvent(E, md->ev_fork, 0));
  SAMO_TRY(p2p_shards(md, sp, S));
  SAMO_TRY(p2p_expand(md, sp, E));
  SAMO_CUDA_TRY(cudaEventRecord(md->ev_flag, E));
  SAMO_CUDA_TRY(cudaStreamWaitEvent(S, md->ev_flag, 0));
  SAMO_TRY(phase_mark(md, 3, S));
  SAMO_TRY(p2p_finish(md, sp, S));
  SAMO_TRY(phase_mark(md, 4, S));
  md->phase_count = 4;
  return SAMO_OK;
}

namespace {
// Sets the caller's device back on every return path (multi-device groups).
struct RestoreDevice {
  int dev;
  ~RestoreDevice() { cudaSetDevice(dev); }
};
}  // namespace

// One step of every rank of a local group, queued phase by phase on one
// stream: each rank's waits (flag, buckets) find their signals already
// written, so no kernel spins on another that is queued behind it.
// A group spread over several devices (one model per device, peers mapped
// directly: a single-process stand-in for G processes, e.g. to profile the
// NVLink traffic of the fused kernels with one ncu) runs each rank's phase
// on its own device and stream and waits for every device between phases.
static int step_local_group(samo_model* const* models, int G, bool gather, cudaStream_t S) {
  const int B = p2p_buckets(G);
  if (B < 2) return fail(SAMO_E_STATE, "a local group needs the pipelined exchange (SAMO_P2P_BUCKETS >= 2)");
  const bool multi = models[0]->group_dev >= 0;
  int dev0 = 0;
  SAMO_CUDA_TRY(cudaGetDevice(&dev0));
  const RestoreDevice restore{dev0};
  auto on = [&](int r) -> cudaStream_t {
    if (!multi) return S;
    cudaSetDevice(models[r]->group_dev);
    return models[r]->s_group;
  };
  auto phase_end = [&]() -> int {
    if (!multi) return SAMO_OK;
    for (int r = 0; r < G; ++r) {
      SAMO_CUDA_TRY(cudaSetDevice(models[r]->group_dev));
      SAMO_CUDA_TRY(cudaStreamSynchronize(models[r]->s_group));
    }
    return SAMO_OK;
  };
  std::vector<P2PStep> sp(G);
  for (int r = 0; r < G; ++r) {
    cudaStream_t s = on(r);
    SAMO_TRY(flush_cfg(models[r], s));
    SAMO_TRY(p2p_prepare(models[r], B, gather, sp[r]));
  }
  for (int r = 0; r < G; ++r) SAMO_TRY(p2p_gather(models[r], sp[r], on(r)));
  SAMO_TRY(phase_end());
  for (int r = 0; r < G; ++r) SAMO_TRY(p2p_flag(models[r], sp[r], 1, on(r)));
  SAMO_TRY(phase_end());
  for (int r = 0; r < G; ++r) SAMO_TRY(p2p_flag(models[r], sp[r], 2, on(r)));
  SAMO_TRY(phase_end());
  for (int r = 0; r < G; ++r) SAMO_TRY(p2p_shards(models[r], sp[r], on(r)));
  SAMO_TRY(phase_end());
  for (int r = 0; r < G; ++r) SAMO_TRY(p2p_expand(models[r], sp[r], on(r)));
  SAMO_TRY(phase_end());
  for (int r = 0; r < G; ++r) SAMO_TRY(p2p_finish(models[r], sp[r], on(r)));
  return phase_end();
}

extern "C" {

int samo_model_set_exchange(samo_model* md, int mode) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  if (mode != -1 && mode != SAMO_EXCHANGE_ALLREDUCE && mode != SAMO_EXCHANGE_SHARDED &&
      mode != SAMO_EXCHANGE_P2P)
    return fail(SAMO_E_PARAMETER, "unknown exchange mode %d", mode);
  md->exchange = mode;
  drop_graphs(md);
  return clear_ok();
}

// Test harness (samo_cuda.h): G models on this device become the ranks of
// one data-parallel group with directly mapped peers.  Everything the
// pipelined peer-to-peer step needs is planned here, before any rank's
// kernels are queued, because those kernels wait for each other.
int samo_model_attach_local_group(samo_model* const* models, int G) {
  if (!models || G < 2 || G > kMaxP2PRanks)
    return fail(SAMO_E_PARAMETER, "local group of %d models (2..%d)", G, kMaxP2PRanks);
  int dev = -1;
  SAMO_CUDA_TRY(cudaGetDevice(&dev));
  std::vector<int> devs(G);
  bool multi = false;
  for (int r = 0; r < G; ++r) {
    samo_model* md = models[r];
    if (!md) return fail(SAMO_E_PARAMETER, "null model %d", r);
    SAMO_TRY(step_ready(md));
    if (md->block_bytes != models[0]->block_bytes || md->n_tot != models[0]->n_tot ||
        md->ntiles != models[0]->ntiles || md->nlayers != models[0]->nlayers)
      return fail(SAMO_E_DIMENSION, "model %d: layout differs from model 0", r);
    cudaPointerAttributes pa{};
    SAMO_CUDA_TRY(cudaPointerGetAttributes(&pa, md->block));
    devs[r] = pa.device;
    multi = multi || pa.device != dev;
  }
  if (multi) {  // one model per device, every pair of devices peer-capable
    const RestoreDevice restore{dev};
    for (int r = 0; r < G; ++r)
      for (int q = 0; q < G; ++q) {
        if (q == r) continue;
        if (devs[q] == devs[r]) return fail(SAMO_E_PARAMETER, "a multi-device group takes one model per device");
        int ok = 0;
        SAMO_CUDA_TRY(cudaDeviceCanAccessPeer(&ok, devs[r], devs[q]));
        if (!ok) return fail(SAMO_E_PARAMETER, "device %d cannot access device %d", devs[r], devs[q]);
        SAMO_CUDA_TRY(cudaSetDevice(devs[r]));
        const cudaError_t e = cudaDeviceEnablePeerAccess(devs[q], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
        cudaGetLastError();
      }
    for (int r = 0; r < G; ++r) {
      SAMO_CUDA_TRY(cudaSetDevice(devs[r]));
      models[r]->group_dev = devs[r];
      if (!models[r]->s_group) SAMO_CUDA_TRY(cudaStreamCreateWithFlags(&models[r]->s_group, cudaStreamNonBlocking));
    }
  }
  for (int r = 0; r < G; ++r) {
    samo_model* md = models[r];
    close_peers(md);
    delete md->own_comm;
    md->own_comm = new samo_comm{};
    md->own_comm->nranks = G;
    md->own_comm->rank = r;
    md->own_comm->local_group = true;
    md->comm = md->own_comm;
    md->cfg_dirty = true;
    md->exchange = SAMO_EXCHANGE_P2P;
    for (int q = 0; q < G; ++q) md->peer_base[q] = models[q]->block;
    md->p2p_ok = true;
    drop_graphs(md);
  }
  const int B = p2p_buckets(G);
  for (int r = 0; r < G && B > 1; ++r) {
    if (multi) SAMO_CUDA_TRY(cudaSetDevice(devs[r]));
    SAMO_TRY(plan_shards(models[r], models[r]->p2p_plan, B));
    if (p2p_push()) SAMO_TRY(build_push_tiles(models[r], models[r]->p2p_plan));
  }
  if (multi) SAMO_CUDA_TRY(cudaSetDevice(dev));
  return clear_ok();
}

int samo_local_group_step(samo_model* const* models, int G, samo_stream_t stream) {
  if (!models || G < 2 || G > kMaxP2PRanks) return fail(SAMO_E_PARAMETER, "local group of %d models", G);
  for (int r = 0; r < G; ++r) {
    samo_model* md = models[r];
    SAMO_TRY(step_ready(md));
    if (!md->comm || !md->comm->local_group || md->comm->nranks != G || md->comm->rank != r)
      return fail(SAMO_E_STATE, "model %d is not rank %d of this local group", r, r);
    // every rank's peer map must be exactly this list, in this order: the
    // kernels address rank q's arena through peer_base[q]
    for (int q = 0; q < G; ++q)
      if (md->peer_base[q] != models[q]->block)
        return fail(SAMO_E_STATE, "model %d: rank %d of its local group is not models[%d]", r, q, q);
    if (!md->grads_set) return fail(SAMO_E_STATE, "optimizer_step requires backward (no gradients set)");
  }
  SAMO_TRY(step_local_group(models, G, true, as_stream(stream)));
  return clear_ok();
}

// The local group's step after every rank's backward sinks (exchange +
// update only; the sinks have pushed or written the gradients).
int samo_local_group_step_sunk(samo_model* const* models, int G, samo_stream_t stream) {
  if (!models || G < 2 || G > kMaxP2PRanks) return fail(SAMO_E_PARAMETER, "local group of %d models", G);
  for (int r = 0; r < G; ++r) {
    samo_model* md = models[r];
    SAMO_TRY(step_ready(md));
    if (!md->comm || !md->comm->local_group || md->comm->nranks != G || md->comm->rank != r)
      return fail(SAMO_E_STATE, "model %d is not rank %d of this local group", r, r);
    for (int q = 0; q < G; ++q)
      if (md->peer_base[q] != models[q]->block)
        return fail(SAMO_E_STATE, "model %d: rank %d of its local group is not models[%d]", r, q, q);
  }
  SAMO_TRY(step_local_group(models, G, false, as_stream(stream)));
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
  SAMO_TRY(flush_cfg(md, as_stream(stream)));
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

}  // extern "C"
