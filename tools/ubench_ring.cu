// Microbenchmark: per-SM bandwidth of the group kernel's phase C access pattern -- u_j = sum_e
// coef_e A[row_e][j] over a CTA's column block (cw doubles) of nr random rows of a dense m x m A --
// with (a) register loads (16 rows per lane per batch, 16-byte loads, as k_iterate) and (b) a
// cp.async.bulk ring (one producer thread, row segments of cw doubles into shared memory, mbarrier
// transaction counts, 16 consumer warps).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/ubench_ring.cu -o tools/ubench_ring
//   ./tools/ubench_ring [m=4096] [nr=1024]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// (a) register loads
__global__ void __launch_bounds__(512, 1)
k_reg(const double* __restrict__ A, long long lda, const int* __restrict__ rows, const double* __restrict__ coef,
      int nr, long long m, double* __restrict__ u, int reps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long cw = ((m + gridDim.x - 1) / gridDim.x + 1) & ~1LL;
  const long long j0 = min(m, (long long)blockIdx.x * cw), j1 = min(m, j0 + cw);
  __shared__ double red[16][4][64];
  const double2* A2 = reinterpret_cast<const double2*>(A);
  for (int rep = 0; rep < reps; ++rep) {
    const int nch = (int)((j1 - j0 + 63) / 64);
    for (int c0 = 0; c0 < nch; c0 += 4) {
      double s[4][2] = {};
      for (int eb = warp; eb < nr; eb += 16 * 16) {
        int off[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int e = eb + 16 * q;
          off[q] = e < nr ? (int)(((long long)rows[e] * lda) >> 1) : -1;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c0 + c >= nch) break;
          const long long j = j0 + 64LL * (c0 + c) + 2 * lane;
          const bool jin = j < j1;
          double2 x[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) x[q] = (jin && off[q] >= 0) ? __ldg(A2 + off[q] + (j >> 1)) : make_double2(0, 0);
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (off[q] >= 0) {
              const double cf = coef[eb + 16 * q];
              s[c][0] += cf * x[q].x;
              s[c][1] += cf * x[q].y;
            }
        }
      }
      for (int c = 0; c < 4; ++c) { red[warp][c][2 * lane] = s[c][0]; red[warp][c][2 * lane + 1] = s[c][1]; }
      __syncthreads();
      if (warp < 4 && c0 + warp < nch) {
        const long long j = j0 + 64LL * (c0 + warp) + 2 * lane;
        double a0 = 0, a1 = 0;
        for (int w = 0; w < 16; ++w) { a0 += red[w][warp][2 * lane]; a1 += red[w][warp][2 * lane + 1]; }
        if (j < j1) u[j] = a0;
        if (j + 1 < j1) u[j + 1] = a1;
      }
      __syncthreads();
    }
  }
}

// (b) bulk ring: stage = RPS row segments of cw doubles (cw <= CWMAX); warp 16 is the producer
// (row offsets staged in shared memory, lane 0 issues), warps 0-15 consume
template <int NST, int RPS, int CWMAX>
__global__ void __launch_bounds__(544, 1)
k_ring(const double* __restrict__ A, long long lda, const int* __restrict__ rows, const double* __restrict__ coef,
       int nr, long long m, double* __restrict__ u, int reps) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)NST * RPS * CWMAX);
  uint64_t* empty = full + NST;
  double* red = reinterpret_cast<double*>(empty + NST);   // [16][CWMAX]
  int* s_row = reinterpret_cast<int*>(red + 16 * CWMAX);
  double* s_cf = reinterpret_cast<double*>(s_row + nr + (nr & 1));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long cw = ((m + gridDim.x - 1) / gridDim.x + 1) & ~1LL;
  const long long j0 = min(m, (long long)blockIdx.x * cw), j1 = min(m, j0 + cw);
  const int w = (int)(j1 - j0);
  const unsigned seg = (unsigned)w * 8u;
  for (int e = tid; e < nr; e += 544) { s_row[e] = rows[e]; s_cf[e] = coef[e]; }
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&empty[s])), "r"(16));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int nstage = (nr + RPS - 1) / RPS;
  const int total = nstage * reps;
  auto wait = [&](uint64_t* b, unsigned ph) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n"
                 ::"r"(su32(b)), "r"(ph) : "memory");
  };
  if (warp == 16) {   // producer warp: lane q issues row q of each stage (RPS <= 32)
    for (int t = 0; t < total; ++t) {
      const int s = t % NST, st = t % nstage;
      const int e0 = st * RPS, n = min(RPS, nr - e0);
      if (t >= NST) wait(&empty[s], (unsigned)(((t / NST) - 1) & 1));
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&full[s])), "r"(seg * n) : "memory");
      __syncwarp();
      if (lane < n)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     ::"r"(su32(sm + ((size_t)s * RPS + lane) * CWMAX)), "l"(A + (long long)s_row[e0 + lane] * lda + j0),
                     "r"(seg), "r"(su32(&full[s])) : "memory");
    }
    return;
  }
  double acc[CWMAX / 64][2];
  for (int t = 0; t < total; ++t) {
    const int s = t % NST, st = t % nstage;
    if (st == 0)
      for (int k = 0; k < CWMAX / 64; ++k) acc[k][0] = acc[k][1] = 0.0;
    wait(&full[s], (unsigned)((t / NST) & 1));
    const int e0 = st * RPS, n = min(RPS, nr - e0);
    const double* buf = sm + (size_t)s * RPS * CWMAX;
    for (int q = warp; q < n; q += 16) {
      const double cf = s_cf[e0 + q];
#pragma unroll
      for (int k = 0; k < CWMAX / 64; ++k) {
        const int c = 2 * (lane + 32 * k);
        if (c < w) {
          const double2 v = *reinterpret_cast<const double2*>(buf + (size_t)q * CWMAX + c);
          acc[k][0] += cf * v.x;
          acc[k][1] += cf * v.y;
        }
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&empty[s])) : "memory");
    if (st == nstage - 1) {   // end of a rep: reduce the 16 row groups (consumer warps only)
      for (int k = 0; k < CWMAX / 64; ++k) {
        const int c = 2 * (lane + 32 * k);
        if (c < w) { red[warp * CWMAX + c] = acc[k][0]; red[warp * CWMAX + c + 1] = acc[k][1]; }
      }
      asm volatile("bar.sync 1, 512;\n" ::: "memory");
      for (int c = tid; c < w; c += 512) {
        double a = 0;
        for (int g = 0; g < 16; ++g) a += red[g * CWMAX + c];
        u[j0 + c] = a;
      }
      asm volatile("bar.sync 1, 512;\n" ::: "memory");
    }
  }
}

int main(int argc, char** argv) {
  const long long m = argc > 1 ? atoll(argv[1]) : 4096;
  const int nr = argc > 2 ? atoi(argv[2]) : 1024;
  const long long lda = m;
  double* A; int* rows; double* coef; double* u;
  CK(cudaMalloc(&A, m * lda * 8));
  CK(cudaMemset(A, 0, m * lda * 8));
  CK(cudaMalloc(&rows, nr * 4));
  CK(cudaMalloc(&coef, nr * 8));
  CK(cudaMalloc(&u, m * 8));
  std::mt19937 g(1);
  std::vector<int> idx(m);
  for (int i = 0; i < m; ++i) idx[i] = i;
  std::shuffle(idx.begin(), idx.end(), g);
  idx.resize(nr);
  std::vector<double> cf(nr, 0.5);
  CK(cudaMemcpy(rows, idx.data(), nr * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(coef, cf.data(), nr * 8, cudaMemcpyHostToDevice));
  // flush buffer (> L2) between runs: A alone is 134 MB for m = 4096
  double* fl; const size_t FL = 256ull << 20;
  CK(cudaMalloc(&fl, FL));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 20;
  auto run = [&](const char* nm, auto launch, int S) {
    for (int it = 0; it < 3; ++it) {
      CK(cudaMemsetAsync(fl, it, FL));
      cudaEventRecord(e0);
      launch(S);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)reps * nr * m * 8.0;
    printf("%-22s S=%3d  %.3f ms/rep  %.1f GB/s total  %.1f GB/s per SM\n", nm, S, ms / reps, bytes / ms / 1e6,
           bytes / ms / 1e6 / S);
  };
  for (int S : {16, 32, 48, 64, 148}) {
    run("reg (k_iterate)", [&](int s) { k_reg<<<s, 512>>>(A, lda, rows, coef, nr, m, u, reps); }, S);
    {
      constexpr int NST = 5, RPS = 16, CW = 256;
      const size_t smem = (size_t)NST * RPS * CW * 8 + 2 * NST * 8 + 16 * CW * 8 + (size_t)nr * 12 + 8;
      CK(cudaFuncSetAttribute(k_ring<NST, RPS, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if ((m + S - 1) / S <= CW)
        run("ring 5x16 (cw<=256)", [&](int s) { k_ring<NST, RPS, CW><<<s, 544, smem>>>(A, lda, rows, coef, nr, m, u, reps); }, S);
    }
    {
      constexpr int NST = 10, RPS = 16, CW = 128;
      const size_t smem = (size_t)NST * RPS * CW * 8 + 2 * NST * 8 + 16 * CW * 8 + (size_t)nr * 12 + 8;
      CK(cudaFuncSetAttribute(k_ring<NST, RPS, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if ((m + S - 1) / S <= CW)
        run("ring 10x16 (cw<=128)", [&](int s) { k_ring<NST, RPS, CW><<<s, 544, smem>>>(A, lda, rows, coef, nr, m, u, reps); }, S);
    }
    {
      constexpr int NST = 5, RPS = 32, CW = 128;
      const size_t smem = (size_t)NST * RPS * CW * 8 + 2 * NST * 8 + 16 * CW * 8 + (size_t)nr * 12 + 8;
      CK(cudaFuncSetAttribute(k_ring<NST, RPS, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if ((m + S - 1) / S <= CW && smem <= 227 * 1024)
        run("ring 5x32 (cw<=128)", [&](int s) { k_ring<NST, RPS, CW><<<s, 544, smem>>>(A, lda, rows, coef, nr, m, u, reps); }, S);
    }
    {
      constexpr int NST = 10, RPS = 32, CW = 64;
      const size_t smem = (size_t)NST * RPS * CW * 8 + 2 * NST * 8 + 16 * CW * 8 + (size_t)nr * 12 + 8;
      CK(cudaFuncSetAttribute(k_ring<NST, RPS, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if ((m + S - 1) / S <= CW)
        run("ring 10x32 (cw<=64)", [&](int s) { k_ring<NST, RPS, CW><<<s, 544, smem>>>(A, lda, rows, coef, nr, m, u, reps); }, S);
    }
  }
  return 0;
}
