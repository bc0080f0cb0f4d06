// FP64 peak microbenchmark for B200 (sm_100a): DFMA vs DMMA.8x8x4 vs mixed.
// Sets the roofline denominator for the Q(f,f) kernels.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double acc[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { acc[i][0] = i; acc[i][1] = threadIdx.x; }
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < CH; ++i) dmma884(acc[i][0], acc[i][1], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// half the warps do DFMA, half do DMMA: tests whether the pipes are separate
template <int CH>
__global__ void k_mixed(double* out, int iters, double a, double b) {
  int w = threadIdx.x / 32;
  if (w & 1) {
    double acc[CH][2];
#pragma unroll
    for (int i = 0; i < CH; ++i) { acc[i][0] = i; acc[i][1] = threadIdx.x; }
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int i = 0; i < CH; ++i) dmma884(acc[i][0], acc[i][1], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
  } else {
    double acc[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += acc[i];
    if (s == 12345.678) out[threadIdx.x] = s;
  }
}

// shared-memory LDS.64 bandwidth (conflict-free, per-lane distinct addresses)
__global__ void k_lds(double* out, int iters) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double s = 0;
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) s += sm[(idx + r * 256) & 4095];
    idx = (idx + 1) & 4095;
  }
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int nsm = p.multiProcessorCount;
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int smem_optin = 0; cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"smem_optin\": %d, \"l2\": %d}\n", p.name, nsm, clk, smem_optin, p.l2CacheSize);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  auto run = [&](const char* name, void (*kern)(double*, int, double, double), int threads, int blocks_per_sm, double flops_per_thread_iter) {
    int blocks = nsm * blocks_per_sm;
    for (int w = 0; w < 2; ++w) kern<<<blocks, threads>>>(out, iters / 4, 1.0000001, 1e-9);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double fl = flops_per_thread_iter * iters * (double)threads * blocks;
    printf("{\"kernel\": \"%s\", \"threads\": %d, \"blocks\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n", name, threads, blocks, best, fl / best / 1e9);
    cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  };
  // DFMA: 8*CH FMAs per thread-iter, 2 flops each
  run("dfma_ch4_256x4", k_dfma<4>, 256, 4, 8 * 4 * 2);
  run("dfma_ch8_256x4", k_dfma<8>, 256, 4, 8 * 8 * 2);
  run("dfma_ch8_512x2", k_dfma<8>, 512, 2, 8 * 8 * 2);
  run("dfma_ch16_256x2", k_dfma<16>, 256, 2, 8 * 16 * 2);
  // DMMA 8x8x4: 256 MAC per warp per instr = 8 MAC/thread = 16 flops/thread
  run("dmma_ch2_256x4", k_dmma<2>, 256, 4, 8 * 2 * 16);
  run("dmma_ch4_256x4", k_dmma<4>, 256, 4, 8 * 4 * 16);
  run("dmma_ch8_256x2", k_dmma<8>, 256, 2, 8 * 8 * 16);
  run("dmma_ch4_128x4", k_dmma<4>, 128, 4, 8 * 4 * 16);
  run("dmma_ch4_128x1", k_dmma<4>, 128, 1, 8 * 4 * 16);
  // mixed: half warps DFMA(8 chains:128 flops/iter), half DMMA(4 chains:512 flops/iter)
  run("mixed_ch4_256x4_avg", k_mixed<4>, 256, 4, 0.5 * (8 * 4 * 2) + 0.5 * (8 * 4 * 16));
  {
    int blocks = nsm * 4, threads = 256;
    k_lds<<<blocks, threads>>>(out, 256); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k_lds<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 16.0 * 8 * iters * threads * blocks;
    printf("{\"kernel\": \"lds64\", \"ms\": %.3f, \"TB/s\": %.3f, \"B_per_clk_per_sm_at_maxclk\": %.1f}\n", ms, bytes / ms / 1e9, bytes / (ms * 1e-3) / nsm / (clk * 1e3));
  }
  return 0;
}
