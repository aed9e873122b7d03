// Kernel ridge regression route (Section "Using a kernel").
//
// The dual of ridge regression on a feature map phi is the n x n system (Eq. kernelridge)
//     K (K + lambda I) alpha = K y,      K_ij = exp(-||x_i - x_j||^2 / (2 sigma^2))  (Eq. Gausskernel)
// i.e. A = K^T (K + lambda I), b = K^T y, solved by the unchanged EXPLICIT-mode hot
// path (sketch-ahead gathers of the rows of A, batched factorisation, fused update).  Setup:
//   k_rbf       K from the explicit differences x_i - x_j (32 x 32 tiles, rows of X in shared memory)
//   A           = K K on the lower-triangle tiles of the TMA DMMA GEMM (K symmetric: K^T K = K K),
//                 mirrored, then A += lambda K (k_axpy_mat)
//   b           = K y (the X^T y kernel applied to K, K symmetric)
// K is freed once A and b exist; the solution alpha (n) is the returned weight vector, and the
// predictor on the training inputs is K alpha.
#include <cmath>
#include <string>

#include "engine.h"
#include "rs_internal.cuh"

namespace rs {

namespace {

constexpr int RB = 32;

__global__ void __launch_bounds__(RB * 8)
k_rbf(const double* __restrict__ X, long long ldx, long long n, long long d, double inv2s2,
      double* __restrict__ K, long long ldk) {
  __shared__ double xi[RB][RB + 1], xj[RB][RB + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const long long i0 = (long long)blockIdx.y * RB, j0 = (long long)blockIdx.x * RB;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};   // rows i0 + ty + 8 q, column j0 + tx
  for (long long k0 = 0; k0 < d; k0 += RB) {
    for (int r = ty; r < RB; r += 8) {
      const long long k = k0 + tx;
      xi[r][tx] = (i0 + r < n && k < d) ? X[(i0 + r) * ldx + k] : 0.0;
      xj[r][tx] = (j0 + r < n && k < d) ? X[(j0 + r) * ldx + k] : 0.0;
    }
    __syncthreads();
    const int kk = (int)(d - k0 < RB ? d - k0 : RB);
    for (int k = 0; k < kk; ++k) {
      const double b = xj[tx][k];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double t = xi[ty + 8 * q][k] - b;
        acc[q] += t * t;
      }
    }
    __syncthreads();
  }
  const long long j = j0 + tx;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const long long i = i0 + ty + 8 * q;
    if (i < n && j < n) K[i * ldk + j] = exp(-acc[q] * inv2s2);
  }
}

// A += lambda K (m x m, shared leading dimension)
__global__ void k_axpy_mat(double* __restrict__ A, const double* __restrict__ K, long long ld,
                           long long m, double lambda) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < m * m;
       q += (long long)gridDim.x * blockDim.x) {
    const long long i = q / m, j = q % m;
    A[i * ld + j] += lambda * K[i * ld + j];
  }
}

}  // namespace

rs_status create_kernel(rs_problem* out, int64_t n, int64_t d, const double* X, int64_t ldx,
                        const double* y, double lambda, double sigma, rs_mem mem,
                        const rs_dist* dist) {
  if (!out) return fail(RS_EINVAL, "out is NULL");
  *out = nullptr;
  if (n < 1 || d < 1) return fail(RS_EINVAL, "need n >= 1 and d >= 1");
  if (!(lambda > 0.0) || !std::isfinite(lambda)) return fail(RS_EINVAL, "need finite lambda > 0 (P:L36)");
  if (!(sigma > 0.0) || !std::isfinite(sigma)) return fail(RS_EINVAL, "need finite sigma > 0 (P:L180)");
  if (!X || !y) return fail(RS_EINVAL, "X and y must be non-NULL");
  if (ldx < d) return fail(RS_EINVAL, "ldx < d");
  if (mem != RS_MEM_HOST && mem != RS_MEM_DEVICE_COPY && mem != RS_MEM_DEVICE_BORROW)
    return fail(RS_EINVAL, "bad rs_mem");
  if (dist && dist->world > 1) return fail(RS_EUNSUPPORTED, "kernel ridge route: one GPU (v1)");
  if (n > 0x7fffffffLL) return fail(RS_EUNSUPPORTED, "n >= 2^31");

  Problem* p = new Problem();
  auto guard = [&](rs_status s) {
    if (s != RS_OK) delete p;
    return s;
  };
  rs_status s = setup_common(p, dist);
  if (s != RS_OK) return guard(s);
  p->fmt = 0;
  p->route = 1;
  p->mode = RS_AS_EXPLICIT;
  p->n = n;
  p->d = n;   // the weight vector is alpha (n)
  p->m = n;
  p->rows_loc = 0;
  p->lambda = lambda;
  cudaStream_t st = p->st;
  const cudaMemcpyKind kd = kind_of(mem);

  double *Xd = nullptr, *yd = nullptr, *K = nullptr;
  unsigned long long* bad = nullptr;
  auto cleanup = [&]() {
    dfree(Xd);
    dfree(yd);
    dfree(K);
    dfree(bad);
  };
  s = dalloc(&Xd, (size_t)n * d);
  if (s == RS_OK) s = dalloc(&yd, n);
  if (s == RS_OK) s = dalloc(&bad, 1);
  if (s != RS_OK) { cleanup(); return guard(s); }
  if (cudaMemcpy2DAsync(Xd, d * 8, X, ldx * 8, d * 8, n, kd, st) != cudaSuccess ||
      cudaMemcpyAsync(yd, y, n * 8, kd, st) != cudaSuccess) {
    cleanup();
    return guard(fail(RS_ECUDA, "copy X / y"));
  }
  cudaMemsetAsync(bad, 0, 8, st);
  launch_count_nonfinite(Xd, d, n, d, bad, st);
  launch_count_nonfinite(yd, 1, n, 1, bad, st);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, bad, 8, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) { cleanup(); return guard(fail(RS_ECUDA, "copy")); }
  if (h) { cleanup(); return guard(fail(RS_EINVAL, "X or y has non-finite entries")); }

  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  p->lda = round_up(n, 4);
  s = dalloc(&K, (size_t)n * p->lda);
  if (s == RS_OK) s = dalloc(&p->A, (size_t)n * p->lda);
  if (s == RS_OK) s = dalloc(&p->b, n);
  if (s != RS_OK) { cleanup(); return guard(s); }
  // K (Eq. Gausskernel)
  {
    const unsigned T = (unsigned)((n + RB - 1) / RB);
    k_rbf<<<dim3(T, T), dim3(RB, 8), 0, st>>>(Xd, d, n, d, 1.0 / (2.0 * sigma * sigma), K, p->lda);
    if (cudaGetLastError() != cudaSuccess) { cleanup(); return guard(fail(RS_ECUDA, "k_rbf")); }
  }
  // b = K y
  {
    double* work = nullptr;
    s = dalloc(&work, dense_xty_work(n, n));
    if (s != RS_OK) { cleanup(); return guard(s); }
    cudaError_t ce = launch_dense_xty(K, p->lda, n, n, yd, p->b, work, st);
    cudaStreamSynchronize(st);
    dfree(work);
    if (ce != cudaSuccess) { cleanup(); return guard(fail(RS_ECUDA, "b = K y")); }
  }
  // A = K K + lambda K (lower tiles of the DMMA contraction, mirrored)
  {
    TmaGemm tg{};
    double* work = nullptr;
    cudaError_t ce = tma_gemm_plan(&tg, K, p->lda, K, p->lda, n, n, n, p->num_sms, 1);
    tg.lower = 1;
    if (ce == cudaSuccess && tg.work_elems) {
      s = dalloc(&work, tg.work_elems);
      if (s != RS_OK) { cleanup(); return guard(s); }
    }
    if (ce == cudaSuccess) ce = tma_gemm_launch(tg, p->A, p->lda, work, nullptr, st);
    if (ce == cudaSuccess) ce = launch_mirror_lower(p->A, p->lda, n, st);
    if (ce == cudaSuccess) {
      k_axpy_mat<<<p->num_sms * 8, 256, 0, st>>>(p->A, K, p->lda, n, lambda);
      ce = cudaGetLastError();
    }
    cudaStreamSynchronize(st);
    dfree(work);
    if (ce != cudaSuccess) { cleanup(); return guard(fail(RS_ECUDA, std::string("A = K(K + lambda I): ") + cudaGetErrorString(ce))); }
  }
  cudaEventRecord(e1, st);
  cleanup();
  s = finish_setup(p);
  if (s != RS_OK) return guard(s);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  p->setup_seconds = ms * 1e-3;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) return guard(fail(RS_ECUDA, cudaGetErrorString(ce)));
  *out = reinterpret_cast<rs_problem>(p);
  return RS_OK;
}

}  // namespace rs

extern "C" rs_status rs_create_kernel(rs_problem* out, int64_t n, int64_t d, const double* X,
                                      int64_t ldx, const double* y, double lambda, double sigma,
                                      rs_mem mem, const rs_dist* dist) {
  return rs::create_kernel(out, n, d, X, ldx, y, lambda, sigma, mem, dist);
}
