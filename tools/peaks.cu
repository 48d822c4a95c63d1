// Microbenchmarks for the roofline denominators MEASURED_PEAKS.json lacks
// (SURVEY §6): L2-resident random-gather bandwidth (8 / 16 B per load, tables of
// 32 and 64 MiB, the size class of the hash tables), FP64 and FP32 FMA issue
// peaks. Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 peaks.cu
// Prints one JSON object. Timed with CUDA events, best of 5, after warm-up.
#include <cstdio>
#include <cmath>
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

// The hash encoding's own access pattern with no interpolation math: consecutive
// lanes are consecutive samples along a ray (spacing `step` in unit coordinates, as
// the march emits them), each gathers the 8 corner entries of its cell on each of the
// L levels (N_l = floor(N_min b^l); dense index when (N_l + 1)^3 <= T, else the
// spatial hash). The ceiling for the hash stages: what the memory system delivers
// for exactly these gathers (L1 reuse between neighbouring samples included).
template <class T, int L>
__global__ void hash_gather_kernel(const T* __restrict__ tab, const uint32_t* __restrict__ res,
                                   const uint32_t* __restrict__ off, int log2T, float step, int samples,
                                   float* out) {
  const uint32_t mask = (1u << log2T) - 1u;
  float acc = 0.f;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < samples; s += gridDim.x * blockDim.x) {
    const uint32_t ray = (uint32_t)s / 128u, j = (uint32_t)s % 128u;
    const float ox = 0.2f + 0.6f * (mix(ray * 3u) & 0xffff) / 65536.f, oy = 0.2f + 0.6f * (mix(ray * 3u + 1u) & 0xffff) / 65536.f,
                oz = 0.2f + 0.6f * (mix(ray * 3u + 2u) & 0xffff) / 65536.f;
    float dx = (mix(ray * 7u) & 0xffff) / 32768.f - 1.f, dy = (mix(ray * 7u + 1u) & 0xffff) / 32768.f - 1.f,
          dz = (mix(ray * 7u + 2u) & 0xffff) / 32768.f - 1.f;
    const float inv = rsqrtf(dx * dx + dy * dy + dz * dz + 1e-12f);
    const float t = ((float)j - 64.f) * step;
    const float p[3] = {fminf(fmaxf(ox + t * dx * inv, 0.f), 1.f), fminf(fmaxf(oy + t * dy * inv, 0.f), 1.f),
                        fminf(fmaxf(oz + t * dz * inv, 0.f), 1.f)};
#pragma unroll 4
    for (int l = 0; l < L; ++l) {
      const uint32_t N = res[l];
      uint32_t g[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) g[a] = min((uint32_t)(p[a] * (float)N), N - 1u);
      const uint32_t stride = N + 1u;
      const bool dense = (uint64_t)stride * stride * stride <= (1ull << log2T);
      T v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t cx = g[0] + (k & 1), cy = g[1] + ((k >> 1) & 1), cz = g[2] + ((k >> 2) & 1);
        const uint32_t idx = dense ? cx + cy * stride + cz * stride * stride
                                   : ((cx ^ (cy * 2654435761u) ^ (cz * 805459861u)) & mask);
        v[k] = __ldg(tab + off[l] + idx);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += reinterpret_cast<const float*>(&v[k])[0];
    }
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
  // the two hash grids' access patterns (render.py CANON_GRID / DEFORM_GRID), 2^21 samples
  // on rays with the march's spacing in unit coordinates (4.7 m / 128 over a 2.2 m cube)
  for (int grid = 0; grid < 2; ++grid) {
    const int L = grid == 0 ? 16 : 8, log2T = grid == 0 ? 19 : 17, F = grid == 0 ? 2 : 4;
    const double nmin = 16, nmax = grid == 0 ? 2048 : 256;
    uint32_t hres[16], hoff[16], total = 0;
    const double b = exp((log(nmax) - log(nmin)) / (L - 1));
    for (int l = 0; l < L; ++l) {
      hres[l] = (uint32_t)floor(nmin * pow(b, l));
      const uint64_t dense = (uint64_t)(hres[l] + 1) * (hres[l] + 1) * (hres[l] + 1);
      hoff[l] = total;
      total += (uint32_t)(dense <= (1ull << log2T) ? dense : (1ull << log2T));
    }
    uint32_t *dres, *doff;
    CK(cudaMalloc(&dres, sizeof(hres)));
    CK(cudaMalloc(&doff, sizeof(hoff)));
    CK(cudaMemcpy(dres, hres, sizeof(hres), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(doff, hoff, sizeof(hoff), cudaMemcpyHostToDevice));
    const int samples = 1 << 21;
    const float step = (float)((4.7 / 128) / 2.2);
    float ms;
    if (F == 2) {
      auto K = [&] { hash_gather_kernel<float2, 16><<<sms * 8, 128>>>((const float2*)tab, dres, doff, log2T, step, samples, out); };
      ms = best_ms(K);
    } else {
      auto K = [&] { hash_gather_kernel<float4, 8><<<sms * 8, 128>>>((const float4*)tab, dres, doff, log2T, step, samples, out); };
      ms = best_ms(K);
    }
    const double bytes = (double)samples * L * 8 * F * 4;
    printf(", \"hash_gather_%s_gbs\": %.1f", grid == 0 ? "canonical_16x2p19xF2_f32" : "deform_8x2p17xF4_f32",
           bytes / (ms * 1e-3) / 1e9);
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
         "threads; hash_gather = the hash grids' 8-corner gathers on all levels for samples along rays at the march "
         "spacing, no interpolation math (all levels' bytes counted); FMA = 8 independent chains per thread; best of 5, "
         "CUDA events\"}\n", blocks, threads);
  return 0;
}
