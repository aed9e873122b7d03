// a6 + a7 -- fused momentum update and stop rule.
//
//   u = (A S_k) delta_k                                       ("multiplying a m x tau matrix")
//   r^{k+1} = r^k - gamma u + beta (r^k - r^{k-1})            (Eq. res_update_mom)
//   w^{k+1} = w^k - gamma S_k delta_k + beta (w^k - w^{k-1})
// kept in the increment form (x, dx = x^k - x^{k-1}):  dx <- beta dx - gamma v;  x <- x + dx, which
// is algebraically the printed recurrence (R13).  S_k delta_k arrives as the dense vector
// `sdelta` (scattered by the solve kernel) and is cleared here for the next iteration.
//   ||r^{k+1}||^2 is reduced deterministically (per-block partials, then the last block sums them
// in a fixed order), and the last block applies the stop rule ||r^k|| <= tol ||r^0|| (P:L248-251,
// DESIGN.md R1), the divergence guard and the iteration counter.
#include <algorithm>

#include "rs_internal.cuh"

namespace rs {

namespace {

constexpr int UX = 32, UY = 8;   // block: 32 columns j x 8 slices of tau

// k += 1, record ||r||, apply the stop rule (last block of the update kernel only).
__device__ void finish_iteration(Ctrl* ctrl, double tot) {
  ctrl->arrive = 0;
  ctrl->rnorm2 = tot;
  const long long k = ctrl->k + 1;
  ctrl->k = k;
  const double rel = sqrt(tot) / sqrt(ctrl->bnorm2);
  if (ctrl->trace && k <= ctrl->trace_cap) ctrl->trace[k - 1] = rel;
  if (!isfinite(tot) || rel > 1e8) {
    ctrl->status = ST_DIVERGED;
    ctrl->done = 1;
  } else if (rel <= ctrl->tol) {
    ctrl->status = ST_CONVERGED;
    ctrl->done = 1;
  } else if (k >= ctrl->max_iter) {
    ctrl->status = ST_MAXITER;
    ctrl->done = 1;
  }
}

__global__ void __launch_bounds__(UX * UY)
k_update(const double* __restrict__ ASt, long long ld_as, int tau, const double* __restrict__ delta,
         double* __restrict__ sdelta, double* __restrict__ w, double* __restrict__ dw,
         double* __restrict__ r, double* __restrict__ dr, long long m, double gamma, double beta,
         double* __restrict__ partials, Ctrl* ctrl) {
  if (ctrl->done) return;
  if (ctrl->status >= ST_NOTSPD) {   // set by the solve / AS kernels of this iteration
    if (blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) ctrl->done = 1;
    return;
  }
  mom_at(ctrl, gamma, beta);   // schedule (gamma_k, beta_k), rs_momentum
  __shared__ double red[UY][UX + 1];
  __shared__ double s_delta[1024];
  __shared__ bool s_last;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * UX + tx;
  const long long j = (long long)blockIdx.x * UX + tx;
  const bool small = tau <= 1024;
  if (small)
    for (int b = tid; b < tau; b += UX * UY) s_delta[b] = delta[b];
  __syncthreads();
  double acc = 0.0;
  if (j < m) {
    for (int b = ty; b < tau; b += UY) {
      const double db = small ? s_delta[b] : delta[b];
      acc += ASt[(long long)b * ld_as + j] * db;
    }
  }
  red[ty][tx] = acc;
  __syncthreads();
  double r2 = 0.0;
  if (ty == 0) {
    if (j < m) {
      double u = 0.0;
#pragma unroll
      for (int q = 0; q < UY; ++q) u += red[q][tx];
      const double drj = beta * dr[j] - gamma * u;
      const double rj = r[j] + drj;
      dr[j] = drj;
      r[j] = rj;
      const double sd = sdelta[j];
      sdelta[j] = 0.0;
      const double dwj = beta * dw[j] - gamma * sd;
      dw[j] = dwj;
      w[j] += dwj;
      r2 = rj * rj;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r2 += __shfl_down_sync(0xffffffffu, r2, o);
    if (tx == 0) {
      partials[blockIdx.x] = r2;
      __threadfence();
      const unsigned prev = atomicAdd(&ctrl->arrive, 1u);
      s_last = (prev == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (!s_last) return;
  // last block: fixed-order reduction of the partials
  __threadfence();
  double s = 0.0;
  for (unsigned q = tid; q < gridDim.x; q += UX * UY) s += __ldcg(&partials[q]);
  red[ty][tx] = s;
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
    for (int q = 0; q < UY; ++q)
      for (int p = 0; p < UX; ++p) tot += red[q][p];
    finish_iteration(ctrl, tot);
  }
}

// Same for AS stored row-major (m x tau): one warp per coordinate j, lanes over the tau columns.
constexpr int RM_WARPS = 8;
__global__ void __launch_bounds__(RM_WARPS * 32)
k_update_rm(const double* __restrict__ AS, long long ld_as, int tau,
            const double* __restrict__ delta, double* __restrict__ sdelta, double* __restrict__ w,
            double* __restrict__ dw, double* __restrict__ r, double* __restrict__ dr, long long m,
            double gamma, double beta, double* __restrict__ partials, Ctrl* ctrl) {
  if (ctrl->done) return;
  if (ctrl->status >= ST_NOTSPD) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ctrl->done = 1;
    return;
  }
  mom_at(ctrl, gamma, beta);   // schedule (gamma_k, beta_k), rs_momentum
  __shared__ double s_delta[1024];
  __shared__ double red[RM_WARPS];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool small = tau <= 1024;
  if (small)
    for (int b = tid; b < tau; b += RM_WARPS * 32) s_delta[b] = delta[b];
  __syncthreads();
  double r2 = 0.0;
  // each block: RM_WARPS * 4 consecutive coordinates, one warp per coordinate at a time
  const long long jb = (long long)blockIdx.x * RM_WARPS * 4;
  for (int q = warp; q < RM_WARPS * 4; q += RM_WARPS) {
    const long long j = jb + q;
    if (j >= m) break;
    const double* row = AS + j * ld_as;
    double u = 0.0;
    for (int b = lane; b < tau; b += 32) u += row[b] * (small ? s_delta[b] : delta[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
    if (lane == 0) {
      const double drj = beta * dr[j] - gamma * u;
      const double rj = r[j] + drj;
      dr[j] = drj;
      r[j] = rj;
      const double sd = sdelta[j];
      sdelta[j] = 0.0;
      const double dwj = beta * dw[j] - gamma * sd;
      dw[j] = dwj;
      w[j] += dwj;
      r2 += rj * rj;
    }
  }
  if (lane == 0) red[warp] = r2;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int q = 0; q < RM_WARPS; ++q) s += red[q];
    partials[blockIdx.x] = s;
    __threadfence();
    const unsigned prev = atomicAdd(&ctrl->arrive, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) {
    double tot = 0.0;
    for (unsigned q = 0; q < gridDim.x; ++q) tot += __ldcg(&partials[q]);
    finish_iteration(ctrl, tot);
  }
}

// Gram mode: u given as a dense vector (X^T X S delta); A S delta = u + lambda S delta.
constexpr int VT = 256;
__global__ void __launch_bounds__(VT)
k_update_vec(const double* __restrict__ u, double lambda, double* __restrict__ sdelta,
             double* __restrict__ w, double* __restrict__ dw, double* __restrict__ r,
             double* __restrict__ dr, long long m, double gamma, double beta,
             double* __restrict__ partials, Ctrl* ctrl) {
  if (ctrl->done) return;
  if (ctrl->status >= ST_NOTSPD) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ctrl->done = 1;
    return;
  }
  mom_at(ctrl, gamma, beta);   // schedule (gamma_k, beta_k), rs_momentum
  __shared__ double red[VT / 32];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long j = (long long)blockIdx.x * VT + tid;
  double r2 = 0.0;
  if (j < m) {
    const double sd = sdelta[j];
    const double uj = u[j] + lambda * sd;
    const double drj = beta * dr[j] - gamma * uj;
    const double rj = r[j] + drj;
    dr[j] = drj;
    r[j] = rj;
    sdelta[j] = 0.0;
    const double dwj = beta * dw[j] - gamma * sd;
    dw[j] = dwj;
    w[j] += dwj;
    r2 = rj * rj;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
  if (lane == 0) red[warp] = r2;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int q = 0; q < VT / 32; ++q) s += red[q];
    partials[blockIdx.x] = s;
    __threadfence();
    const unsigned prev = atomicAdd(&ctrl->arrive, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) {
    double tot = 0.0;
    for (unsigned q = 0; q < gridDim.x; ++q) tot += __ldcg(&partials[q]);
    finish_iteration(ctrl, tot);
  }
}

// Explicit A, few sketch entries: block = 64 coordinates j (a warp reads 512 contiguous bytes of a
// row of A as double2) x RW_Y warps over the entries; u_j = sum_e sd_e A[coord_e][j] with
// sd_e = sign_e delta[bucket_e] (A symmetric: row coord_e = column coord_e).  Launched as the last
// kernel of the iteration's PDL chain (bfactor.cu): the first RW_PRE rows of each warp (A and the
// sketch are static) are loaded into registers BEFORE pdl_wait(), overlapping the solve kernels.
constexpr int RW_Y = 8;
constexpr int RW_PRE = 8;
constexpr int RW_COLS = 64;
constexpr int RW_MAXS = 16;
// u = A S delta over the rows e of slot `sk`, split over gridDim.y row ranges: block (cb, sp) sums
// rows e in its range for columns 64 cb .. 64 cb + 63 into upart[sp][j]; the last split of a column
// block (counter cnt[cb]) adds the splits in order (deterministic), applies the momentum update to
// its 64 coordinates and contributes ||r||^2; the last column block finishes the iteration.
__global__ void __launch_bounds__(32 * RW_Y)
k_update_rows(const double* __restrict__ A, long long lda, DevSketch sk,
              const double* __restrict__ delta, double* __restrict__ sdelta,
              double* __restrict__ w, double* __restrict__ dw, double* __restrict__ r,
              double* __restrict__ dr, long long m, double gamma, double beta,
              double* __restrict__ partials, double* __restrict__ upart, int* __restrict__ cnt,
              Ctrl* ctrl) {
  pdl_trigger();
  if (ctrl->done) return;   // previous iteration's stop rule (static for this chain)
  __shared__ double red[RW_Y][2][33];
  __shared__ bool s_last;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int len = sk.len;   // = bptr[tau] for subsample / SubCount / count
  const int ns = gridDim.y, sp = blockIdx.y;
  const int per = (len + ns - 1) / ns;
  const int e0 = min(len, sp * per), e1 = min(len, e0 + per), span = e1 - e0;
  // lane tx owns columns j0, j0 + 1 (lda is a multiple of 4 doubles, so the pair is 16-B aligned and
  // inside the row's padding when j0 + 1 == m)
  const long long j0 = (long long)blockIdx.x * RW_COLS + 2 * tx;
  const bool jin = j0 < m;
  double2 v[RW_PRE];
  int sb[RW_PRE];   // bucket, bit-complemented for a negative sign
#pragma unroll
  for (int u = 0; u < RW_PRE; ++u) {
    const int e = ty + RW_Y * u;
    v[u] = make_double2(0.0, 0.0);
    sb[u] = 0;
    if (e < span) {
      const int c = sk.coord[e0 + e];
      sb[u] = sk.sign[e0 + e] > 0 ? sk.bucket[e0 + e] : ~sk.bucket[e0 + e];
      if (jin) v[u] = __ldg(reinterpret_cast<const double2*>(A + (long long)c * lda + j0));
    }
  }
  pdl_wait();
  if (ctrl->status >= ST_NOTSPD) {   // set by the solve kernels of this iteration
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) ctrl->done = 1;
    return;
  }
  mom_at(ctrl, gamma, beta);   // schedule (gamma_k, beta_k), rs_momentum
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int u = 0; u < RW_PRE; ++u) {
    if (ty + RW_Y * u < span) {
      const double dv = delta[sb[u] >= 0 ? sb[u] : ~sb[u]];
      const double sd = sb[u] >= 0 ? dv : -dv;
      a0 += sd * v[u].x;
      a1 += sd * v[u].y;
    }
  }
  for (int e = ty + RW_Y * RW_PRE; e < span; e += RW_Y) {
    const int c = sk.coord[e0 + e];
    const double dv = delta[sk.bucket[e0 + e]];
    const double sd = sk.sign[e0 + e] > 0 ? dv : -dv;
    if (jin) {
      const double2 x = __ldg(reinterpret_cast<const double2*>(A + (long long)c * lda + j0));
      a0 += sd * x.x;
      a1 += sd * x.y;
    }
  }
  red[ty][0][tx] = a0;
  red[ty][1][tx] = a1;
  __syncthreads();
  if (ty == 0) {
    double u0 = 0.0, u1 = 0.0;
#pragma unroll
    for (int q = 0; q < RW_Y; ++q) {
      u0 += red[q][0][tx];
      u1 += red[q][1][tx];
    }
    if (j0 < m) upart[(long long)sp * m + j0] = u0;
    if (j0 + 1 < m) upart[(long long)sp * m + j0 + 1] = u1;
    __threadfence();
    __syncwarp();
    if (tx == 0) s_last = atomicAdd(&cnt[blockIdx.x], 1) == ns - 1;
    __syncwarp();
  }
  __syncthreads();
  if (!s_last) return;
  // last split of this column block: u_j = sum of the splits in order, then the update
  if (ty == 0) {
    __threadfence();
    double r2 = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long j = j0 + h;
      if (j < m) {
        double u = 0.0;
        for (int q = 0; q < ns; ++q) u += __ldcg(&upart[(long long)q * m + j]);
        const double drj = beta * dr[j] - gamma * u;
        const double rj = r[j] + drj;
        dr[j] = drj;
        r[j] = rj;
        const double sd = sdelta[j];
        sdelta[j] = 0.0;
        const double dwj = beta * dw[j] - gamma * sd;
        dw[j] = dwj;
        w[j] += dwj;
        r2 += rj * rj;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r2 += __shfl_down_sync(0xffffffffu, r2, o);
    if (tx == 0) {
      cnt[blockIdx.x] = 0;
      partials[blockIdx.x] = r2;
      __threadfence();
      const unsigned prev = atomicAdd(&ctrl->arrive, 1u);
      s_last = (prev == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double s2 = 0.0;
  for (unsigned q = tid; q < gridDim.x; q += 32 * RW_Y) s2 += __ldcg(&partials[q]);
  red[ty][0][tx] = s2;
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
    for (int q = 0; q < RW_Y; ++q)
      for (int p = 0; p < 32; ++p) tot += red[q][0][p];
    finish_iteration(ctrl, tot);
  }
}

}  // namespace

cudaError_t update_init() {
  return cudaSuccess;
}

size_t update_rows_scratch(long long m) { return (size_t)RW_MAXS * (size_t)m; }
size_t update_rows_counters(long long m) { return (size_t)((m + 31) / 32); }

cudaError_t launch_update_rows(const double* A, long long lda, const DevSketch& sk,
                               const double* delta, double* sdelta, double* w, double* dw,
                               double* r, double* dr, long long m, double gamma, double beta,
                               double* partials, double* upart, int* cnt, int num_sms, Ctrl* ctrl,
                               cudaStream_t st) {
  const long long cb = (m + RW_COLS - 1) / RW_COLS;
  // splits: every warp's rows fit its register preload when possible, and >= 2 blocks per SM
  long long ns = (sk.len + RW_Y * RW_PRE - 1) / (RW_Y * RW_PRE);
  ns = std::max(ns, (2LL * num_sms + cb - 1) / cb);
  ns = std::max(1LL, std::min<long long>({ns, (long long)RW_MAXS, (long long)sk.len / RW_Y}));
  return launch_pdl(k_update_rows, dim3((unsigned)cb, (unsigned)ns), dim3(32, RW_Y), 0, st, A, lda,
                    sk, delta, sdelta, w, dw, r, dr, m, gamma, beta, partials, upart, cnt, ctrl);
}

cudaError_t launch_update_vec(const double* u, double lambda, double* sdelta, double* w, double* dw,
                              double* r, double* dr, long long m, double gamma, double beta,
                              double* partials, Ctrl* ctrl, cudaStream_t st) {
  const unsigned g = (unsigned)((m + VT - 1) / VT);
  k_update_vec<<<g, VT, 0, st>>>(u, lambda, sdelta, w, dw, r, dr, m, gamma, beta, partials, ctrl);
  return cudaGetLastError();
}

size_t update_partials(long long m) { return (size_t)((m + UX - 1) / UX); }

cudaError_t launch_update(const double* ASt, long long ld_as, bool as_rowmajor, int tau,
                          const double* delta, double* sdelta, double* w, double* dw, double* r,
                          double* dr, long long m, double gamma, double beta, double* partials,
                          Ctrl* ctrl, cudaStream_t st) {
  if (as_rowmajor) {
    const unsigned g = (unsigned)((m + RM_WARPS * 4 - 1) / (RM_WARPS * 4));
    k_update_rm<<<g, RM_WARPS * 32, 0, st>>>(ASt, ld_as, tau, delta, sdelta, w, dw, r, dr, m, gamma,
                                             beta, partials, ctrl);
    return cudaGetLastError();
  }
  const unsigned grid = (unsigned)((m + UX - 1) / UX);
  k_update<<<grid, dim3(UX, UY), 0, st>>>(ASt, ld_as, tau, delta, sdelta, w, dw, r, dr, m, gamma,
                                          beta, partials, ctrl);
  return cudaGetLastError();
}

}  // namespace rs
