// Dependent-chain latency (cycles per op) of fp64 sqrt, div, rsqrt-Newton and DFMA on one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0) {
  double x = x0 + threadIdx.x * 1e-9, y = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) x = sqrt(x) + 1.5;
  long long t1 = clock64();
  for (int i = 0; i < 1000; ++i) y = 1.0 / (y + 2.0);
  long long t2 = clock64();
  double z = x;
  for (int i = 0; i < 1000; ++i) { double r = rsqrt(z); r = r * (1.5 - 0.5 * z * r * r); z = r + 2.0; }
  long long t3 = clock64();
  double w = y;
  for (int i = 0; i < 1000; ++i) w = fma(w, 0.999999, 1e-7);
  long long t4 = clock64();
  out[threadIdx.x] = x + y + z + w;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 64);
  k<<<1, 32>>>(o, c, 3.0); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 3.0); cudaDeviceSynchronize();
  printf("cycles/op: sqrt %.1f  div %.1f  rsqrt+newton %.1f  dfma %.1f\n", c[0] / 1000.0, c[1] / 1000.0, c[2] / 1000.0, c[3] / 1000.0);
}
