// model.cu — the model state behind samo_model_*: one device allocation for
// every arena and table, layer views, index sets, initialisation, the step
// entry points (single GPU K1 -> K23, dispatch to the data-parallel drivers in
// dp.cu, CUDA-graph capture), the backward sinks, step records, invariant
// checks, binary checkpoints and the memory report.
#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>

#include "host.cuh"

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
  md->grid_fused = fused_grid(tile_elems);
  const int max_grid = std::max(std::max(md->grid_update16, md->grid_update32), md->grid_fused);

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
  // the fused step's second theta/m/v set (K123)
  const uint64_t o_theta_b = carve(n_al * 4), o_m_b = carve(n_al * 4), o_v_b = carve(n_al * 4);
  // grad arena: n_al floats (the sharded exchange pads it to G * shard size,
  // G <= 128) + the skip-indicator slot at n_al + kFlagOff.
  const uint64_t o_g = carve((n_al + kArenaSlack) * 4), o_idx = carve(n_al * 4);
  const uint64_t o_off = carve(n_al * 2);
  const uint64_t o_t16 = carve(md->d_tot * 2), o_tiles = carve(ntiles * sizeof(SamoTile));
  const uint64_t o_layers = carve(std::max(1, nlayers) * sizeof(SamoLayerDev));
  const uint64_t o_koff = carve((nlayers + 1) * sizeof(uint64_t));
  const uint64_t o_st = carve(sizeof(SamoStepState));
  const uint64_t o_np = carve(static_cast<uint64_t>(max_grid) * kMaxBuckets * sizeof(float));
  const uint64_t o_tn = carve(static_cast<uint64_t>(ntiles) * sizeof(float) + 1024 * sizeof(double));
  // Buffers of the sharded exchange last: the step kernels' streams keep the
  // relative placement measured best.
  const uint64_t o_c16 = carve((n_al + kArenaSlack) * 2);
  const uint64_t o_n2 = carve(256);  // 16 norm^2 slots + arrival counter
  const uint64_t o_slots = carve(sizeof(SamoPeerSlots));
  const uint64_t o_cfg = carve(sizeof(SamoStepConfig));
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
  md->theta_alt = reinterpret_cast<float*>(b + o_theta_b);
  md->m_alt = reinterpret_cast<float*>(b + o_m_b);
  md->v_alt = reinterpret_cast<float*>(b + o_v_b);
  md->g = reinterpret_cast<float*>(b + o_g);
  md->idx = reinterpret_cast<uint32_t*>(b + o_idx);
  md->off16 = reinterpret_cast<uint16_t*>(b + o_off);
  md->c16 = reinterpret_cast<uint16_t*>(b + o_c16);
  md->norm2 = reinterpret_cast<double*>(b + o_n2);
  md->done = reinterpret_cast<uint32_t*>(b + o_n2 + 16 * sizeof(double));
  md->slots = reinterpret_cast<SamoPeerSlots*>(b + o_slots);
  md->cfg_dev = reinterpret_cast<SamoStepConfig*>(b + o_cfg);
  md->theta16 = reinterpret_cast<uint16_t*>(b + o_t16);
  md->tiles = reinterpret_cast<SamoTile*>(b + o_tiles);
  md->layers_dev = reinterpret_cast<SamoLayerDev*>(b + o_layers);
  md->k_off_dev = reinterpret_cast<uint64_t*>(b + o_koff);
  md->st = reinterpret_cast<SamoStepState*>(b + o_st);
  md->norm_partials = reinterpret_cast<float*>(b + o_np);
  md->norm_dpartials = reinterpret_cast<double*>(b + o_tn);  // <= 1024 repair CTAs
  md->tile_norm = reinterpret_cast<float*>(b + o_tn + 1024 * sizeof(double));
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
  drop_graphs(md);
  close_peers(md);
  delete md->own_comm;
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
  if (md->sink16) cudaFree(md->sink16);
  if (md->s_group) cudaStreamDestroy(md->s_group);
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
  drop_graphs(md);
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
  md->cfg_dirty = true;  // the step kernels read cfg_dev: a captured graph stays valid
  return clear_ok();
}

int samo_model_set_grad_dtype(samo_model* md, int dtype) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  if (dtype != SAMO_GRAD_F16 && dtype != SAMO_GRAD_BF16)
    return fail(SAMO_E_PARAMETER, "gradient dtype must be SAMO_GRAD_F16 or SAMO_GRAD_BF16");
  const int bf16 = dtype == SAMO_GRAD_BF16;
  if (bf16 != md->grad_bf16) drop_graphs(md);  // captured steps baked the decode in
  md->grad_bf16 = bf16;
  return clear_ok();
}

int samo_model_grad_dtype(const samo_model* md) { return md && md->grad_bf16 ? SAMO_GRAD_BF16 : SAMO_GRAD_F16; }

int samo_model_attach_comm(samo_model* md, samo_comm* comm) {
  if (!md) return fail(SAMO_E_PARAMETER, "null model");
  close_peers(md);
  delete md->own_comm;
  md->own_comm = nullptr;
  md->comm = comm;
  md->cfg_dirty = true;  // the scales fold in 1/G
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



}  // extern "C"

// The gradient arena holds unscaled fp32 when it is exchanged between ranks,
// and the raw compressed binary16 gradient (the reference's grad16) otherwise.
bool wide_grads(const samo_model* md) { return comm_size(md) > 1; }

StepArgs step_args(samo_model* md) {
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
  a.grad_bf16 = md->grad_bf16 ? 1u : 0u;
  a.prm = adam_params(&md->cfg);
  a.st = md->st;
  a.flag_slot = flag_ptr(md);
  a.norm_partials = md->norm_partials;
  a.norm_all = md->norm_partials;
  a.norm_count = 0;
  a.finalize = 1;
  a.cfg = md->capturing ? md->cfg_dev : nullptr;
  return a;
}


extern "C" {

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
  if (comm_size(md) > 1 && p2p_push()) {  // straight to the owners over NVLink
    SAMO_TRY(push_sink_prepare(md));
    SAMO_TRY(push_sink_layer(md, l, nullptr, as_stream(stream)));
    return clear_ok();
  }
  StepArgs a = step_args(md);
  a.tiles = md->tiles + md->layer_t[l];
  a.ntiles = md->layer_t[l + 1] - md->layer_t[l];
  if (a.ntiles) SAMO_TRY(launch_gather(a, false, std::min<int>(md->grid_gather16, a.ntiles), as_stream(stream)));
  return clear_ok();
}

int samo_model_sink_dw(samo_model* md, int l, const uint16_t* x, const uint16_t* dy, uint64_t batch,
                       uint64_t in, uint64_t out, samo_stream_t stream) {
  SAMO_TRY(sink_ready(md, l));
  if (md->grad_bf16)
    return fail(SAMO_E_STATE, "sink_dw: the fused dW GEMM produces binary16 gradients (model expects bfloat16)");
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
  // Push mode: this rank's gradient arena is its receive buffer, which peers
  // fill during their backward.  The epilogue gathers into a scratch arena
  // of its own (2 n bytes, allocated on first use) rather than borrowing
  // theta16c, so the sinks never touch the exchange's weight buffer, and a
  // copy pushes the layer to its owners.
  const bool push = comm_size(md) > 1 && p2p_push();
  if (push) {
    SAMO_TRY(push_sink_prepare(md));
    if (!md->sink16) SAMO_CUDA_TRY(cudaMalloc(&md->sink16, (md->n_tot + 8) * sizeof(uint16_t)));
  }
  uint16_t* g16 = push ? md->sink16 : reinterpret_cast<uint16_t*>(md->g);
  DwArgs a{};
  a.M = in;
  a.N = out;
  a.K = batch;
  a.idx = md->idx + md->k_off[l];
  a.kb = md->dw_kb[l];
  a.g16 = g16 + md->k_off[l];
  a.flag = flag_ptr(md);
  SAMO_TRY(launch_dw_gemm(x, dy, a, 1, s));
  if (push) SAMO_TRY(push_sink_layer(md, l, md->sink16, s));
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

extern "C++" int flush_cfg(samo_model* md, cudaStream_t s) {
  if (!md->cfg_dirty) return SAMO_OK;
  SamoStepConfig v{};
  v.prm = adam_params(&md->cfg);
  const int G = comm_size(md);
  float inv_scale = 1.0f / md->cfg.loss_scale;  // as step_args
  if (G > 1) inv_scale = inv_scale * (1.0f / static_cast<float>(G));
  v.inv_scale = inv_scale;
  v.p2p_scale = (1.0f / md->cfg.loss_scale) * (1.0f / static_cast<float>(G));
  SAMO_TRY(launch_set_step_config(md->cfg_dev, v, s));
  md->cfg_dirty = false;
  return SAMO_OK;
}

int samo_model_update(samo_model* md, samo_stream_t stream) {
  SAMO_TRY(step_ready(md));
  SAMO_TRY(flush_cfg(md, as_stream(stream)));
  const bool wide = wide_grads(md);
  StepArgs a = step_args(md);
  const int grid = std::min<int>(wide ? md->grid_update32 : md->grid_update16, md->ntiles);
  a.norm_count = static_cast<uint32_t>(grid);
  SAMO_TRY(launch_update(a, wide, grid, as_stream(stream)));
  return clear_ok();
}

int samo_model_step_sunk(samo_model* md, samo_stream_t stream) {
  SAMO_TRY(step_ready(md));
  SAMO_TRY(flush_cfg(md, as_stream(stream)));
  if (comm_size(md) > 1) {
    if (exchange_mode(md) != SAMO_EXCHANGE_P2P || !md->p2p_ok)
      return fail(SAMO_E_STATE, "step after backward sinks needs the peer-to-peer exchange");
    SAMO_TRY(step_p2p(md, as_stream(stream), false));
    return clear_ok();
  }
  SAMO_TRY(samo_model_update(md, stream));
  return clear_ok();
}

// The fused single-GPU step on `s`: K123 from the live theta/m/v set into the
// other one, then the skip repair.  The caller swaps the sets once the work
// is enqueued (not while capturing: a captured graph runs later).
static int enqueue_fused(samo_model* md, cudaStream_t s) {
  StepArgs a = step_args(md);
  a.theta_o = md->theta_alt;
  a.m_o = md->m_alt;
  a.v_o = md->v_alt;
  a.tile_norm = md->tile_norm;
  a.norm_dpartials = md->norm_dpartials;
  const int grid = std::min<int>(md->grid_fused, md->ntiles);
  a.norm_count = static_cast<uint32_t>(grid);
  SAMO_TRY(phase_mark(md, 0, s));
  SAMO_TRY(launch_step_fused(a, grid, s));
  SAMO_TRY(phase_mark(md, 1, s));
  SAMO_TRY(launch_step_repair(a, s));
  SAMO_TRY(phase_mark(md, 2, s));
  if (md->phase_timing) md->phase_count = 2;
  return SAMO_OK;
}

static void swap_sets(samo_model* md) {
  if (md->graph) {  // a K1 | K23 graph captured the other set's pointers
    cudaGraphExecDestroy(md->graph);
    md->graph = nullptr;
  }
  std::swap(md->theta, md->theta_alt);
  std::swap(md->m, md->m_alt);
  std::swap(md->v, md->v_alt);
  md->parity ^= 1;
}

int samo_model_step(samo_model* md, samo_stream_t stream) {
  SAMO_TRY(step_ready(md));
  if (!md->grads_set) return fail(SAMO_E_STATE, "optimizer_step requires backward (no gradients set)");
  SAMO_TRY(flush_cfg(md, as_stream(stream)));  // (never inside a capture: step_graph flushes first)
  if (fused_step(md)) {
    if (md->ntiles == 0) return clear_ok();
    SAMO_TRY(enqueue_fused(md, as_stream(stream)));
    if (!md->capturing) swap_sets(md);
    return clear_ok();
  }
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
  SAMO_TRY(flush_cfg(md, s));  // outside the graph: new scalars without a re-capture
  if (fused_step(md)) {
    // One graph per buffer parity: the step of parity p reads set p and
    // writes set 1 - p.
    if (md->ntiles == 0) return clear_ok();
    cudaGraphExec_t& ge = md->fgraph[md->parity];
    if (!ge) {
      if (!md->capture_stream)
        SAMO_CUDA_TRY(cudaStreamCreateWithFlags(&md->capture_stream, cudaStreamNonBlocking));
      const uint64_t before = samo_kernel_launch_count();
      SAMO_CUDA_TRY(cudaStreamBeginCapture(md->capture_stream, cudaStreamCaptureModeThreadLocal));
      md->capturing = true;
      int rc = enqueue_fused(md, md->capture_stream);
      md->capturing = false;
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamEndCapture(md->capture_stream, &graph);
      if (rc != SAMO_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
      }
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
      e = cudaGraphInstantiate(&ge, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) {
        ge = nullptr;
        return cuda_fail(e, "cudaGraphInstantiate");
      }
      md->fgraph_kernels = samo_kernel_launch_count() - before;
      unnote_launch(md->fgraph_kernels);  // captured, not launched
    }
    SAMO_CUDA_TRY(cudaGraphLaunch(ge, s));
    note_launch(md->fgraph_kernels);
    swap_sets(md);
    return clear_ok();
  }
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
    md->capturing = true;
    int rc = samo_model_step(md, md->capture_stream);
    md->capturing = false;
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
    unnote_launch(md->graph_kernels);  // captured, not launched
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
  out->compressed_state_bytes = 7 * md->n_al * 4;          // theta32, m, v (x2: the fused step's two sets), grad
  out->index_bytes = md->n_al * (4 + 2);                    // u32 index set + off16
  out->table_bytes = static_cast<uint64_t>(md->ntiles) * sizeof(SamoTile);
  out->device_bytes = md->block_bytes;
  // store.hpp:129-147 (per layer 2*dense + (2+4+4+8+4)*nnz [+ 2*nnz peak])
  out->reference_steady_bytes = 2 * phi + 22 * n;
  out->reference_peak_bytes = 2 * phi + 24 * n;
  return clear_ok();
}

}  // extern "C"
