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
  CK(cudaFree(in));
  CK(cudaFree(out));
  return 0;
}
