/*
 * samo_cuda_testing.h — test-harness entry points of libsamo_cuda.so.
 *
 * Not part of the drop-in boundary (samo_cuda.h) and not part of the
 * reference's API: these let the GPU tests run the peer-to-peer exchange at
 * G = 5..8 on a single B200, which the pool's 2- and 4-GPU boxes cannot run
 * as processes.  Production code never calls them.
 */
#ifndef SAMO_CUDA_TESTING_H_
#define SAMO_CUDA_TESTING_H_

#include "samo_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Test harness for the peer-to-peer step at any G <= 8 on ONE device:
 * models[0..G) (same layout, all on the current device) become the ranks of
 * one data-parallel group whose peers are mapped directly, with no NCCL
 * communicator and no IPC.  samo_local_group_step then runs one pipelined
 * P2P step of every rank (G >= 3 by default, or SAMO_P2P_BUCKETS >= 2),
 * queued phase by phase on one stream — all gathers, all skip-flag signals,
 * all flag waits, all shard updates, all bucket waits + expands, all
 * finalizes — so every wait finds its signal already written.  The kernels,
 * peer stores and signals are those of the cross-process step; only the
 * cross-rank concurrency differs.  The members' own step calls fail with
 * SAMO_E_STATE.  Re-attach (samo_model_attach_comm) or destroy all members
 * together: each maps the others' memory.  Not part of the reference's API;
 * it lets tests/test_gpu_dp.py check G = 5..8 on a single GPU.  Models on
 * different devices (one per device, every pair peer-capable) form a group
 * across GPUs in one process: each rank's phase runs on its own device,
 * and the step waits for every device between phases (the harness
 * tools/nvlink_group_ncu.py profiles the NVLink bytes with). */
int samo_model_attach_local_group(samo_model* const* models, int G);
int samo_local_group_step(samo_model* const* models, int G, samo_stream_t stream);
/* The same after every member's backward sinks (samo_model_sink_dense /
 * samo_model_sink_dw on each rank): exchange + update only. */
int samo_local_group_step_sunk(samo_model* const* models, int G, samo_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif  /* SAMO_CUDA_TESTING_H_ */
