// sector_probe.cu — does a sector-sparse gather beat K1's streaming read?
//
// "at p >= 0.95 a sector-gather K1 can read fewer than 2*phi
// (touched-sector model 32 * #distinct(idx >> 4))".  K1 streams the whole
// dense binary16 gradient (2*phi bytes) at the copy peak; a gather that loads
// only the kept elements touches only their sectors, but issues scattered
// requests.  For a random (i.i.d.) keep mask of density 1 - p over phi
// elements this probe measures, per launch:
//   stream   read all 2*phi bytes (16-byte vectors, persistent grid) — K1's floor
//   gather   out[k] = dense[idx[k]] for the n kept elements (2-byte loads, k
//            warp-contiguous so a warp's loads share sectors)
// and prints time, effective GB/s and the touched-sector model for 32- and
// 64-byte granules.  Run it under ncu for the DRAM bytes (dram__bytes_read).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sector_probe tools/sector_probe.cu
//   tools/sector_probe [phi (default 2651553280)] [p ...]
// SECTOR_PROBE_L2_FETCH=<bytes> sets cudaLimitMaxL2FetchGranularity first.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <cuda_runtime.h>

#define CK(x)                                                 \
  do {                                                        \
    cudaError_t e = (x);                                      \
    if (e != cudaSuccess) {                                   \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); \
      exit(1);                                                \
    }                                                         \
  } while (0)

__host__ __device__ inline uint32_t mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return static_cast<uint32_t>(x);
}

struct Keep {
  uint32_t thr;
  __host__ __device__ bool operator()(uint32_t i) const { return mix(i) < thr; }
};

__global__ void fill(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    p[i] = make_uint4(mix(i), mix(i + 1), mix(i + 2), mix(i + 3));
}

__global__ void __launch_bounds__(256) stream(const uint4* __restrict__ in, size_t n, uint32_t* sink) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i + u * stride < n ? __ldcs(in + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;  // keeps the loads
}

template <int U>
__global__ void __launch_bounds__(256) gather(const uint16_t* __restrict__ dense, const uint32_t* __restrict__ idx,
                                              uint16_t* __restrict__ out, size_t n) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n; k += U * stride) {
    uint32_t ix[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ix[u] = k + u * stride < n ? __ldcs(idx + k + u * stride) : 0u;
    uint16_t h[U];
#pragma unroll
    for (int u = 0; u < U; ++u) h[u] = k + u * stride < n ? __ldcs(dense + ix[u]) : 0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + u * stride < n) __stcs(out + k + u * stride, h[u]);
  }
}

template <typename F>
static float timed(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  return best;
}

int main(int argc, char** argv) {
  const size_t phi = argc > 1 ? strtoull(argv[1], nullptr, 10) : 2651553280ull;
  std::vector<double> ps;
  for (int i = 2; i < argc; ++i) ps.push_back(atof(argv[i]));
  if (ps.empty()) ps = {0.9, 0.95, 0.99};
  if (const char* g = getenv("SECTOR_PROBE_L2_FETCH")) {
    CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(atoi(g))));
    size_t v = 0;
    CK(cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity));
    printf("{\"l2_fetch_granularity\": %zu}\n", v);
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint16_t* dense;
  uint32_t *idx, *nsel, *sink;
  uint16_t* out;
  const size_t nmax = static_cast<size_t>((1.0 - ps[0] + 0.01) * phi) + 1024;
  for (double p : ps) {
    const size_t need = static_cast<size_t>((1.0 - p + 0.01) * phi) + 1024;
    if (need > nmax) {
      fprintf(stderr, "list the sparsities in ascending order\n");
      return 1;
    }
  }
  CK(cudaMalloc(&dense, (phi + 64) * 2));
  CK(cudaMalloc(&idx, nmax * 4));
  CK(cudaMalloc(&out, nmax * 2));
  CK(cudaMalloc(&nsel, 4));
  CK(cudaMalloc(&sink, 4));
  fill<<<sms * 8, 256>>>(reinterpret_cast<uint4*>(dense), (phi + 64) * 2 / 16);
  CK(cudaGetLastError());
  const size_t nv = phi * 2 / 16;
  const float t_stream = timed([&] { stream<<<sms * 8, 256>>>(reinterpret_cast<const uint4*>(dense), nv, sink); }, 10);
  printf("{\"kernel\": \"stream\", \"phi\": %zu, \"ms\": %.4f, \"GBps\": %.1f}\n", phi, t_stream,
         2.0 * phi / t_stream / 1e6);
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  for (double p : ps) {
    const Keep keep{static_cast<uint32_t>((1.0 - p) * 4294967296.0)};
    thrust::counting_iterator<uint32_t> it(0);
    size_t want = 0;
    CK(cub::DeviceSelect::If(nullptr, want, it, idx, nsel, static_cast<int64_t>(phi), keep));
    if (want > tmp_bytes) {
      if (tmp) CK(cudaFree(tmp));
      CK(cudaMalloc(&tmp, want));
      tmp_bytes = want;
    }
    CK(cub::DeviceSelect::If(tmp, tmp_bytes, it, idx, nsel, static_cast<int64_t>(phi), keep));
    uint32_t n = 0;
    CK(cudaMemcpy(&n, nsel, 4, cudaMemcpyDeviceToHost));
    // touched-sector model on the host (exact for the mask just built)
    std::vector<uint32_t> h(n);
    CK(cudaMemcpy(h.data(), idx, n * 4ull, cudaMemcpyDeviceToHost));
    size_t s32 = 0, s64 = 0;
    uint64_t last32 = ~0ull, last64 = ~0ull;
    for (uint32_t x : h) {
      if ((x >> 4) != last32) ++s32, last32 = x >> 4;
      if ((x >> 5) != last64) ++s64, last64 = x >> 5;
    }
    const float t4 = timed([&] { gather<4><<<sms * 8, 256>>>(dense, idx, out, n); }, 10);
    const float t8 = timed([&] { gather<8><<<sms * 8, 256>>>(dense, idx, out, n); }, 10);
    const float t = t4 < t8 ? t4 : t8;
    printf("{\"kernel\": \"gather\", \"p\": %.3f, \"n\": %u, \"ms\": %.4f, \"ms_u4\": %.4f, \"ms_u8\": %.4f, "
           "\"vs_stream\": %.3f, \"sector32_bytes\": %zu, \"sector64_bytes\": %zu, "
           "\"sector32_frac_of_2phi\": %.3f, \"sector64_frac_of_2phi\": %.3f}\n",
           p, n, t, t4, t8, t / t_stream, 32 * s32, 64 * s64, 32.0 * s32 / (2.0 * phi), 64.0 * s64 / (2.0 * phi));
    fflush(stdout);
  }
  return 0;
}
