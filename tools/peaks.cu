// Microbenchmarks for the roofline denominators MEASURED_PEAKS.json lacks
// (SURVEY §6): L2-resident random-gather bandwidth (8 / 16 B per load, tables of
// 32 and 64 MiB, the size class of the hash tables), FP64 and FP32 FMA issue
// peaks. Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 peaks.cu
// Prints one JSON object. Timed with CUDA events, best of 5, after warm-up.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// every thread issues U independent random loads per iteration (a hash-grid
// level's 8 corners are 8 independent gathers); indices from a cheap hash
template <class T, int U>
__global__ void gather_kernel(const T* __restrict__ tab, uint32_t mask, int iters, float* out) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(tab + (mix(s * 2654435761u + (uint32_t)(i * U + u)) & mask));
#pragma unroll
    for (int u = 0; u < U; ++u) acc += reinterpret_cast<const float*>(&v[u])[0];
  }
  if (acc == 1234.5f) out[0] = acc;
}

template <class T>
__global__ void fma_kernel(T a, T b, int iters, T* out) {
  T x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = (T)(threadIdx.x + j);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = x[j] * a + b;
  T s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == (T)1234.5) out[0] = s;
}

template <class F>
float best_ms(F launch, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int sms = p.multiProcessorCount;
  float* out;
  CK(cudaMalloc(&out, 64));
  void* tab;
  CK(cudaMalloc(&tab, 64u << 20));
  CK(cudaMemset(tab, 0, 64u << 20));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"sm_max_mhz\": %.0f", p.name, sms, p.l2CacheSize,
         clk / 1e3);
  const int threads = 256, blocks = sms * 8, iters = 256;
  for (int mib : {32, 64}) {
    {
      const uint32_t n = (uint32_t)((mib << 20) / 8);
      auto L = [&] { gather_kernel<float2, 8><<<blocks, threads>>>((const float2*)tab, n - 1, iters, out); };
      const float ms = best_ms(L);
      const double bytes = (double)blocks * threads * iters * 8 * 8;
      printf(", \"l2_gather_8B_%dMiB_gbs\": %.1f", mib, bytes / (ms * 1e-3) / 1e9);
    }
    {
      const uint32_t n = (uint32_t)((mib << 20) / 16);
      auto L = [&] { gather_kernel<float4, 8><<<blocks, threads>>>((const float4*)tab, n - 1, iters, out); };
      const float ms = best_ms(L);
      const double bytes = (double)blocks * threads * iters * 8 * 16;
      printf(", \"l2_gather_16B_%dMiB_gbs\": %.1f", mib, bytes / (ms * 1e-3) / 1e9);
    }
  }
  {
    const int it = 4096;
    auto L = [&] { fma_kernel<double><<<sms * 16, 256>>>(1.0000001, 1e-9, it, (double*)out); };
    const float ms = best_ms(L);
    const double flop = 2.0 * sms * 16 * 256 * (double)it * 8;
    printf(", \"fp64_fma_tflops\": %.2f", flop / (ms * 1e-3) / 1e12);
  }
  {
    const int it = 8192;
    auto L = [&] { fma_kernel<float><<<sms * 16, 256>>>(1.0000001f, 1e-9f, it, (float*)out); };
    const float ms = best_ms(L);
    const double flop = 2.0 * sms * 16 * 256 * (double)it * 8;
    printf(", \"fp32_fma_tflops\": %.2f", flop / (ms * 1e-3) / 1e12);
  }
  printf(", \"how\": \"tools/peaks.cu: gathers = 8 independent random __ldg per thread per iteration, %d CTAs x %d "
         "threads; FMA = 8 independent chains per thread; best of 5, CUDA events\"}\n", blocks, threads);
  return 0;
}
