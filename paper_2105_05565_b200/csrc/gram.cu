// Gram ("matvec-chain") implicit mode for dense primal X -- SURVEY §8(f) NEXT-2.
//
// A S is never materialised.  With XS = X S (a2) and v = S delta (the dense m-vector `sdelta`):
//   G = S^T A S = (XS)^T (XS) + lambda S^T S                 (A = X^T X + lambda I)
//   u = A S delta = X^T (X v) + lambda v                      (the residual update needs only A S delta)
// identical to the materialised path in exact arithmetic; the iterates of Alg. 2 are unchanged.
// S^T S = diag(|bucket b|) for the disjoint-support sketches used here.
//   G: the TMA/DMMA contraction of gemm_tma.cu with A = B = XS (K = n, M = N = tau).
//   u: k_xpass streams X once: per row i, t_i = <X_i, v> (block reduction) then u += t_i X_i,
//      per-CTA partial u vectors reduced in a fixed order (deterministic).  HBM-bound: n d 8 bytes.
#include "rs_internal.cuh"

namespace rs {

namespace {

constexpr int XP_THREADS = 512;
constexpr int XP_Q = 8;          // columns per thread: d <= 4096
constexpr int XP_R = 4;          // rows per batch
constexpr int XP_WARPS = XP_THREADS / 32;

__global__ void __launch_bounds__(XP_THREADS, 1)
k_xpass(const double* __restrict__ X, long long ldx, long long rows, long long d,
        const double* __restrict__ v, double* __restrict__ partials, long long rows_per_cta,
        const Ctrl* ctrl) {
  if (ctrl->done) return;
  __shared__ double red[2][XP_R][XP_WARPS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double vr[XP_Q], acc[XP_Q];
#pragma unroll
  for (int q = 0; q < XP_Q; ++q) {
    const long long j = tid + (long long)XP_THREADS * q;
    vr[q] = j < d ? v[j] : 0.0;
    acc[q] = 0.0;
  }
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  const long long r1 = min(rows, r0 + rows_per_cta);
  int buf = 0;
  for (long long i = r0; i < r1; i += XP_R) {
    double x[XP_R][XP_Q];
#pragma unroll
    for (int r = 0; r < XP_R; ++r)
#pragma unroll
      for (int q = 0; q < XP_Q; ++q) {
        const long long j = tid + (long long)XP_THREADS * q;
        x[r][q] = (i + r < r1 && j < d) ? __ldcs(X + (i + r) * ldx + j) : 0.0;
      }
    double dot[XP_R];
#pragma unroll
    for (int r = 0; r < XP_R; ++r) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < XP_Q; ++q) s += x[r][q] * vr[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      dot[r] = s;
    }
    if (lane == 0)
#pragma unroll
      for (int r = 0; r < XP_R; ++r) red[buf][r][warp] = dot[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < XP_R; ++r) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < XP_WARPS; ++w) t += red[buf][r][w];
#pragma unroll
      for (int q = 0; q < XP_Q; ++q) acc[q] += t * x[r][q];
    }
    buf ^= 1;   // the next batch writes the other buffer: one barrier per batch suffices
  }
#pragma unroll
  for (int q = 0; q < XP_Q; ++q) {
    const long long j = tid + (long long)XP_THREADS * q;
    if (j < d) partials[(long long)blockIdx.x * d + j] = acc[q];
  }
}

// u[j] = sum_c partials[c][j]  (fixed order)
__global__ void k_xpass_reduce(const double* __restrict__ partials, int nparts, long long d,
                               double* __restrict__ u, const Ctrl* ctrl) {
  if (ctrl->done) return;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < nparts; ++c) s += partials[(long long)c * d + j];
    u[j] = s;
  }
}

}  // namespace

int xpass_ctas(int num_sms) { return num_sms; }
size_t xpass_partials(long long d, int num_sms) { return (size_t)num_sms * (size_t)d; }

cudaError_t launch_xpass(const double* X, long long ldx, long long rows, long long d,
                         const double* v, double* partials, double* u, int num_sms,
                         const Ctrl* ctrl, cudaStream_t st) {
  if (d > (long long)XP_THREADS * XP_Q) return cudaErrorInvalidValue;
  const int nc = xpass_ctas(num_sms);
  const long long rpc = std::max<long long>(1, (rows + nc - 1) / nc);
  k_xpass<<<nc, XP_THREADS, 0, st>>>(X, ldx, rows, d, v, partials, rpc, ctrl);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_xpass_reduce<<<(unsigned)((d + 255) / 256), 256, 0, st>>>(partials, nc, d, u, ctrl);
  return cudaGetLastError();
}

}  // namespace rs
