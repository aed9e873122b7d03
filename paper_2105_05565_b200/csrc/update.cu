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
#include <cstdlib>
#include <cooperative_groups.h>

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
// The gridDim.y row splits of a column block form one thread-block cluster: their partial sums
// are added in rank order through distributed shared memory by the rank-0 block, which applies
// the momentum update to its 64 coordinates and contributes ||r||^2 (the last column block to
// arrive finishes the iteration).
constexpr int RW_Y = 8;
constexpr int RW_PRE = 8;     // rows per warp loaded before pdl_wait()
constexpr int RW_B = 16;      // rows per warp per later batch (loads first)
constexpr int RW_COLS = 64;
constexpr int RW_MAXS = 8;    // portable cluster size
template <bool CLUSTER>
__global__ void __launch_bounds__(32 * RW_Y)
k_update_rows(const double* __restrict__ A, long long lda, DevSketch sk,
              const double* __restrict__ delta, double* __restrict__ sdelta,
              double* __restrict__ w, double* __restrict__ dw, double* __restrict__ r,
              double* __restrict__ dr, long long m, double gamma, double beta,
              double* __restrict__ partials, Ctrl* ctrl) {
  pdl_trigger();
  namespace cg = cooperative_groups;
  extern __shared__ double rw_sd[];   // [per] sd_e, then [per] coord_e
  __shared__ double red[RW_Y][2][33];
  __shared__ double part[2][32];
  __shared__ int s_flag;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int len = sk.len;   // = bptr[tau] for subsample / SubCount / count
  const int ns = gridDim.y, sp = blockIdx.y;
  const int per = (len + ns - 1) / ns;
  const int e0 = min(len, sp * per), e1 = min(len, e0 + per), span = e1 - e0;
  int* s_co = reinterpret_cast<int*>(rw_sd + per);
  // static: the block's sketch coordinates, then the first RW_PRE rows of each warp
  for (int e = tid; e < span; e += 32 * RW_Y) s_co[e] = sk.coord[e0 + e];
  __syncthreads();
  // lane tx owns columns j0, j0 + 1 (lda is a multiple of 4 doubles, so the pair is 16-B aligned and
  // inside the row's padding when j0 + 1 == m)
  const long long j0 = (long long)blockIdx.x * RW_COLS + 2 * tx;
  const bool jin = j0 < m;
  double2 v[RW_PRE];
#pragma unroll
  for (int u = 0; u < RW_PRE; ++u) {
    const int e = ty + RW_Y * u;
    v[u] = (jin && e < span)
               ? __ldg(reinterpret_cast<const double2*>(A + (long long)s_co[e] * lda + j0))
               : make_double2(0.0, 0.0);
  }
  pdl_wait();
  // block-uniform exits only: every block of a cluster reaches both cluster barriers or none does
  if (ctrl->done) return;
  if (ctrl->status >= ST_NOTSPD) {   // set by the solve kernels of this iteration
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) ctrl->done = 1;
    return;
  }
  mom_at(ctrl, gamma, beta);   // schedule (gamma_k, beta_k), rs_momentum
  for (int e = tid; e < span; e += 32 * RW_Y) {
    const double dv = delta[sk.bucket[e0 + e]];
    rw_sd[e] = sk.sign[e0 + e] > 0 ? dv : -dv;
  }
  __syncthreads();
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int u = 0; u < RW_PRE; ++u) {
    const int e = ty + RW_Y * u;
    if (e < span) {
      a0 += rw_sd[e] * v[u].x;
      a1 += rw_sd[e] * v[u].y;
    }
  }
  for (int eb = ty + RW_Y * RW_PRE; eb < span; eb += RW_Y * RW_B) {
    double2 x[RW_B];
#pragma unroll
    for (int u = 0; u < RW_B; ++u) {
      const int e = eb + RW_Y * u;
      x[u] = (jin && e < span)
                 ? __ldg(reinterpret_cast<const double2*>(A + (long long)s_co[e] * lda + j0))
                 : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < RW_B; ++u) {
      const int e = eb + RW_Y * u;
      if (e < span) {
        a0 += rw_sd[e] * x[u].x;
        a1 += rw_sd[e] * x[u].y;
      }
    }
  }
  red[ty][0][tx] = a0;
  red[ty][1][tx] = a1;
  __syncthreads();
  double u0 = 0.0, u1 = 0.0;
  if (ty == 0) {
#pragma unroll
    for (int q = 0; q < RW_Y; ++q) {
      u0 += red[q][0][tx];
      u1 += red[q][1][tx];
    }
  }
  bool leader = true;
  if constexpr (CLUSTER) {   // add the splits of the column block in rank order through DSMEM
    cg::cluster_group cl = cg::this_cluster();
    if (ty == 0) {
      part[0][tx] = u0;
      part[1][tx] = u1;
    }
    cl.sync();
    leader = cl.block_rank() == 0;
    if (leader && ty == 0) {
      u0 = u1 = 0.0;
      for (int q = 0; q < ns; ++q) {   // rank order = split order (the cluster spans gridDim.y)
        const double* pq = cl.map_shared_rank(&part[0][0], q);
        u0 += pq[tx];
        u1 += pq[32 + tx];
      }
    }
    cl.sync();   // the other splits' shared memory stays alive until rank 0 has read it
  }
  if (!leader) return;
  if (ty == 0) {
    double r2 = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long j = j0 + h;
      if (j < m) {
        const double u = h ? u1 : u0;
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
      partials[blockIdx.x] = r2;
      __threadfence();
      const unsigned prev = atomicAdd(&ctrl->arrive, 1u);
      s_flag = (prev == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (!s_flag) return;
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
  cudaError_t e = cudaFuncSetAttribute(k_update_rows<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_update_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              200 * 1024);
}


cudaError_t launch_update_rows(const double* A, long long lda, const DevSketch& sk,
                               const double* delta, double* sdelta, double* w, double* dw,
                               double* r, double* dr, long long m, double gamma, double beta,
                               double* partials, int num_sms, Ctrl* ctrl, cudaStream_t st) {
  const long long cb = (m + RW_COLS - 1) / RW_COLS;
  // splits (one cluster per column block): about two blocks per SM in total (128 registers per
  // thread), at least 4 rows per warp, at most the portable cluster size
  const long long bps = 4;   // blocks per SM targeted
  long long ns = (bps * num_sms + cb / 2) / cb;   // ~4 blocks per SM (8 / 16 / 32 measured slower
                                                  // on c4: 55 / 68 / 68 vs 54 us)
  ns = std::min<long long>(ns, (sk.len + 4 * RW_Y - 1) / (4 * RW_Y));   // >= 4 rows per warp
  ns = std::max(1LL, std::min<long long>(ns, RW_MAXS));
  const int per = (int)((sk.len + ns - 1) / ns);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)cb, (unsigned)ns);
  cfg.blockDim = dim3(32, RW_Y);
  cfg.dynamicSmemBytes = (size_t)per * 12;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (ns > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 1;
    attr[na].val.clusterDim.y = (unsigned)ns;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (cfg.dynamicSmemBytes > 200 * 1024) return cudaErrorInvalidValue;
  if (ns > 1)
    return cudaLaunchKernelEx(&cfg, k_update_rows<true>, A, lda, sk, delta, sdelta, w, dw, r, dr, m,
                              gamma, beta, partials, ctrl);
  return cudaLaunchKernelEx(&cfg, k_update_rows<false>, A, lda, sk, delta, sdelta, w, dw, r, dr, m,
                            gamma, beta, partials, ctrl);
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
