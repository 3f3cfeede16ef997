// bw_probe.cu — HBM bandwidth of streaming read/write mixes on one B200.
//
// Calibrates the roofline of the SAMO kernels, whose traffic is not the 1:1
// read:write of a copy: K1 is read-heavy (2phi+2n read : 2n write), K23 is
// write-heavy (~1 : 2).  Each kernel streams 16-byte vectors through a
// persistent grid; R read streams and W write streams of `bytes` each.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bw_probe tools/bw_probe.cu
//   tools/bw_probe [GiB per stream]
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                   \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

template <int R, int W>
__global__ void __launch_bounds__(256) stream(const uint4* __restrict__ in, uint4* __restrict__ out,
                                              size_t n) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += 4 * stride) {
    uint4 v[4][R > 0 ? R : 1];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (i + u * stride < n) v[u][r] = __ldcs(in + r * n + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint4 x = make_uint4(static_cast<unsigned>(i), 1u, 2u, 3u);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        x.x ^= v[u][r].x; x.y ^= v[u][r].y; x.z ^= v[u][r].z; x.w ^= v[u][r].w;
      }
      acc.x ^= x.x;
#pragma unroll
      for (int w = 0; w < W; ++w)
        if (i + u * stride < n) __stcs(out + w * n + i + u * stride, x);
    }
  }
  if (acc.x == 0xFFFFFFFFu && W == 0) out[0] = acc;  // keep reads alive
}

template <int R, int W>
void run(const char* name, uint4* in, uint4* out, size_t n, int grid) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) stream<R, W><<<grid, 256>>>(in, out, n);
  CK(cudaDeviceSynchronize());
  const int reps = 10;
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    CK(cudaEventRecord(a));
    stream<R, W><<<grid, 256>>>(in, out, n);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  const double bytes = static_cast<double>(n) * 16.0 * (R + W);
  printf("{\"mix\": \"%s\", \"read_streams\": %d, \"write_streams\": %d, \"bytes\": %.0f, "
         "\"ms\": %.4f, \"GBps\": %.1f}\n",
         name, R, W, bytes, best, bytes / (best * 1e-3) / 1e9);
}

// Copy through the TMA engines: per CTA an NS-stage ring of CH-byte chunks,
// one elected thread issues cp.async.bulk global->shared (mbarrier
// completion) and cp.async.bulk shared->global (bulk-group completion) — no
// data passes through registers.  The ceiling for kernels that stage through
// shared memory with TMA (the SAMO step kernels do for their reads).
template <int NS, int CH>
__global__ void __launch_bounds__(32) tma_copy(const char* __restrict__ in, char* __restrict__ out, size_t bytes) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long bar[NS];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NS; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t nch = bytes / CH;
  unsigned it = 0;
  for (size_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
    const int s = it % NS;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sm + s * CH);
    const unsigned ba = (unsigned)__cvta_generic_to_shared(&bar[s]);
    if (it >= NS)  // the store that last read this stage has finished reading it
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NS - 1) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa),
                 "l"(in + c * CH), "r"(CH), "r"(ba) : "memory");
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(ba),
                 "r"((it / NS) & 1u) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * CH), "r"(sa), "r"(CH)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int NS, int CH>
void run_tma(char* in, char* out, size_t bytes, int ctas_per_sm, int sms) {
  const int smem = NS * CH;
  CK(cudaFuncSetAttribute(tma_copy<NS, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = sms * ctas_per_sm;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) tma_copy<NS, CH><<<grid, 32, smem>>>(in, out, bytes);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int i = 0; i < 10; ++i) {
    CK(cudaEventRecord(a));
    tma_copy<NS, CH><<<grid, 32, smem>>>(in, out, bytes);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  const double moved = 2.0 * static_cast<double>(bytes / CH * CH);
  printf("{\"mix\": \"tma copy 1:1\", \"stages\": %d, \"chunk\": %d, \"ctas_per_sm\": %d, \"bytes\": %.0f, "
         "\"ms\": %.4f, \"GBps\": %.1f}\n", NS, CH, ctas_per_sm, moved, best, moved / (best * 1e-3) / 1e9);
}

int main(int argc, char** argv) {
  const double gib = argc > 1 ? atof(argv[1]) : 2.0;
  const size_t n = static_cast<size_t>(gib * (1ull << 30) / 16);
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  uint4 *in, *out;
  CK(cudaMalloc(&in, n * 16 * 3));
  CK(cudaMalloc(&out, n * 16 * 3));
  CK(cudaMemset(in, 1, n * 16 * 3));
  CK(cudaMemset(out, 0, n * 16 * 3));
  const int grid = sms * 8;
  run<1, 0>("read", in, out, n, grid);
  run<0, 1>("write", in, out, n, grid);
  run<1, 1>("copy 1:1", in, out, n, grid);
  run<2, 1>("2:1 (K1-like)", in, out, n, grid);
  run<1, 2>("1:2 (K23-like)", in, out, n, grid);
  run<3, 2>("3:2", in, out, n, grid);
  const size_t tb = n * 16 * 3;  // 6 GiB each way at the default size
  run_tma<4, 16384>(reinterpret_cast<char*>(in), reinterpret_cast<char*>(out), tb, 2, sms);
  run_tma<6, 16384>(reinterpret_cast<char*>(in), reinterpret_cast<char*>(out), tb, 2, sms);
  run_tma<8, 16384>(reinterpret_cast<char*>(in), reinterpret_cast<char*>(out), tb, 1, sms);
  run_tma<4, 32768>(reinterpret_cast<char*>(in), reinterpret_cast<char*>(out), tb, 1, sms);
  run_tma<3, 32768>(reinterpret_cast<char*>(in), reinterpret_cast<char*>(out), tb, 2, sms);
  CK(cudaFree(in));
  CK(cudaFree(out));
  return 0;
}
