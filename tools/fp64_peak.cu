// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) vs DFMA.
// Used once to fix the FP64 roofline denominator (MEASURED_PEAKS.json has none).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out; CK(cudaMalloc(&out, 8));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int threads : {128, 256, 512, 1024}) {
    for (int bps : {1, 2, 4}) {
      int grid = sms * bps;
      dmma_loop<8><<<grid, threads>>>(out, 100); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_loop<8><<<grid, threads>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double warps = (double)grid * threads / 32;
      double flop = warps * iters * 8 * 512.0;
      printf("DMMA threads=%d blocks/SM=%d: %.2f TFLOP/s\n", threads, bps, flop / ms / 1e9);
    }
  }
  for (int threads : {256, 512, 1024}) {
    int grid = sms * 2;
    dfma_loop<8><<<grid, threads>>>(out, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_loop<8><<<grid, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flop = (double)grid * threads * iters * 8 * 2.0;
    printf("DFMA threads=%d: %.2f TFLOP/s\n", threads, flop / ms / 1e9);
  }
  // sustained: DMMA for ~3 s
  {
    int grid = sms * 2, threads = 256;
    cudaEventRecord(e0);
    for (int r = 0; r < 30; ++r) dmma_loop<8><<<grid, threads>>>(out, iters * 2);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flop = 30.0 * grid * threads / 32 * iters * 2 * 8 * 512.0;
    printf("DMMA sustained (%.0f ms): %.2f TFLOP/s\n", ms, flop / ms / 1e9);
  }
  return 0;
}
