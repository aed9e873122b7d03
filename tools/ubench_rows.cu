// Microbenchmark: u = sum_e sd_e A[coord_e][:] for tau random rows of a dense m x m A (the explicit
// update's gather), several access patterns.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// tools/ubench_rows.cu -o tools/ubench_rows && ./tools/ubench_rows 4096 1024
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

// V1: column block of CB doubles (each lane 2 per 64), NS splits; partial u per split
template <int CB>
__global__ void v_colblock(const double* __restrict__ A, long long lda, const int* __restrict__ coord,
                           const double* __restrict__ sd, int len, int m, double* __restrict__ part) {
  const int ns = gridDim.y, sp = blockIdx.y, per = (len + ns - 1) / ns;
  const int e0 = min(len, sp * per), e1 = min(len, e0 + per);
  constexpr int PL = CB / 32;   // doubles per lane
  double acc[PL] = {};
  const long long j0 = (long long)blockIdx.x * CB;
  for (int e = e0 + threadIdx.y; e < e1; e += blockDim.y) {
    const double* row = A + (long long)coord[e] * lda + j0;
    const double s = sd[e];
#pragma unroll
    for (int q = 0; q < PL / 2; ++q) {
      const long long j = 64 * q + 2 * threadIdx.x;
      if (j0 + j < m) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(row + j));
        acc[2 * q] += s * v.x;
        acc[2 * q + 1] += s * v.y;
      }
    }
  }
  __shared__ double red[8][CB];
#pragma unroll
  for (int q = 0; q < PL / 2; ++q) {
    red[threadIdx.y][64 * q + 2 * threadIdx.x] = acc[2 * q];
    red[threadIdx.y][64 * q + 2 * threadIdx.x + 1] = acc[2 * q + 1];
  }
  __syncthreads();
  for (int j = threadIdx.y * 32 + threadIdx.x; j < CB; j += 256) {
    double u = 0;
    for (int y = 0; y < 8; ++y) u += red[y][j];
    if (j0 + j < m) part[(long long)sp * m + j0 + j] = u;
  }
}

// V3: whole rows: block of 256 threads covers all m columns (m <= 4096: 8 double2 per thread),
// rows e strided over blocks; partial u per block
__global__ void __launch_bounds__(256) v_rows(const double* __restrict__ A, long long lda,
                                              const int* __restrict__ coord,
                                              const double* __restrict__ sd, int len, int m,
                                              double* __restrict__ part) {
  double acc[16] = {};
  for (int e = blockIdx.x; e < len; e += gridDim.x) {
    const double* row = A + (long long)coord[e] * lda;
    const double s = sd[e];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = 512 * q + 2 * threadIdx.x;
      if (j < m) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(row + j));
        acc[2 * q] += s * v.x;
        acc[2 * q + 1] += s * v.y;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int j = 512 * q + 2 * threadIdx.x;
    if (j < m) {
      part[(long long)blockIdx.x * m + j] = acc[2 * q];
      part[(long long)blockIdx.x * m + j + 1] = acc[2 * q + 1];
    }
  }
}

__global__ void v_copy(const double* __restrict__ a, double* __restrict__ b, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n / 2;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(a) + i);
    if (v.x == 12345.0) b[0] = v.y;
  }
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 4096, tau = argc > 2 ? atoi(argv[2]) : 1024;
  const long long lda = (m + 3) / 4 * 4;
  double *A, *sd, *part, *flush;
  int* coord;
  cudaMalloc(&A, (size_t)m * lda * 8);
  cudaMemset(A, 0, (size_t)m * lda * 8);
  cudaMalloc(&sd, tau * 8);
  cudaMemset(sd, 0, tau * 8);
  cudaMalloc(&coord, tau * 4);
  cudaMalloc(&part, (size_t)4096 * m * 8);
  const size_t FL = 512ull << 20;
  cudaMalloc(&flush, FL);
  std::vector<int> h(m);
  for (int i = 0; i < m; ++i) h[i] = i;
  srand(1);
  std::random_shuffle(h.begin(), h.end());
  std::sort(h.begin(), h.begin() + tau);
  cudaMemcpy(coord, h.data(), tau * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)tau * m * 8;
  auto run = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int it = 0; it < 20; ++it) {
      cudaMemsetAsync(flush, it, FL);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
    }
    printf("%-34s %8.2f us  %7.0f GB/s  (%s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int ns : {4, 8, 16, 32}) {
    char nm[64];
    snprintf(nm, 64, "colblock64 ns=%d", ns);
    run(nm, [&] { v_colblock<64><<<dim3((m + 63) / 64, ns), dim3(32, 8)>>>(A, lda, coord, sd, tau, m, part); });
    snprintf(nm, 64, "colblock128 ns=%d", ns);
    run(nm, [&] { v_colblock<128><<<dim3((m + 127) / 128, ns), dim3(32, 8)>>>(A, lda, coord, sd, tau, m, part); });
    snprintf(nm, 64, "colblock256 ns=%d", ns);
    run(nm, [&] { v_colblock<256><<<dim3((m + 255) / 256, ns), dim3(32, 8)>>>(A, lda, coord, sd, tau, m, part); });
  }
  if (m <= 4096)
    for (int g : {148, 296, 592, 1024}) {
      char nm[64];
      snprintf(nm, 64, "rows grid=%d", g);
      run(nm, [&] { v_rows<<<g, 256>>>(A, lda, coord, sd, tau, m, part); });
    }
  run("contiguous read of the same bytes", [&] { v_copy<<<148 * 8, 256>>>(A, part, (long long)tau * lda); });
  run("empty kernel", [&] { v_copy<<<1, 32>>>(A, part, 0); });
  return 0;
}
