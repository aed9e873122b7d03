// a4 + a5 -- the sketched system.
//
//   G = S^T (A S) (lower triangle), g = S^T r^k
//   delta = least_norm_solution(G, g) = G^{-1} g                (R3)
//   by Cholesky G = L L^T (lower triangle read only, R12), L y = g, L^T delta = y.
//   Empty count bucket b (all-zero column of S): G_bb := 1, so delta_b = 0 exactly (R3).
//
// Layout: Gx is (tau + 1) x ldg row-major; rows 0..tau-1 hold the lower triangle of G and row tau
// holds g^T.  A blocked right-looking Cholesky of this bordered matrix (its last diagonal entry is
// never factored) leaves L in rows 0..tau-1 and y = L^{-1} g in row tau: the forward solve comes
// free with the trailing updates.  The factorisation is one cooperative kernel (grid.sync between
// the diagonal / panel / trailing phases of each 32-wide block column), so the whole solve is a
// single graph node; the backward solve and the scatter S delta run in the same kernel.
#include <cooperative_groups.h>

#include "rs_internal.cuh"

namespace cg = cooperative_groups;

namespace rs {

namespace {

constexpr int NB = 32;
constexpr int CT = 256;

// G (lower, incl. diagonal) and g.  Block b' handles column b of G (= row b of AS^T, gathered
// at the sketch coordinates of every bucket a >= b); block tau computes g.
__global__ void k_form_g(const double* __restrict__ ASt, long long ld_as,
                         const double* __restrict__ r, DevSketch sk, double* __restrict__ Gx,
                         long long ldg, const Ctrl* ctrl) {
  if (ctrl->done) return;
  const int b = blockIdx.x, tau = sk.tau;
  if (b == tau) {  // g = S^T r
    for (int a = threadIdx.x; a < tau; a += blockDim.x) {
      double s = 0.0;
      for (int e = sk.bptr[a]; e < sk.bptr[a + 1]; ++e) {
        const double v = r[sk.coord[e]];
        s += sk.sign[e] > 0 ? v : -v;
      }
      Gx[(long long)tau * ldg + a] = s;
    }
    return;
  }
  const double* row = ASt + (long long)b * ld_as;
  const bool b_empty = sk.bptr[b] == sk.bptr[b + 1];
  for (int a = b + threadIdx.x; a < tau; a += blockDim.x) {
    const int e0 = sk.bptr[a], e1 = sk.bptr[a + 1];
    double s = 0.0;
    for (int e = e0; e < e1; ++e) {
      const double v = row[sk.coord[e]];
      s += sk.sign[e] > 0 ? v : -v;
    }
    if (b_empty || e0 == e1) s = (a == b) ? 1.0 : 0.0;   // empty-bucket rule (R3)
    Gx[(long long)a * ldg + b] = s;
  }
}

// Same for AS stored row-major (m x tau, ld_as): block a computes row a of G from the rows
// coord_e (e in bucket a) of AS, coalesced over b <= a.
__global__ void k_form_g_rm(const double* __restrict__ AS, long long ld_as,
                            const double* __restrict__ r, DevSketch sk, double* __restrict__ Gx,
                            long long ldg, const Ctrl* ctrl) {
  if (ctrl->done) return;
  const int a = blockIdx.x, tau = sk.tau;
  if (a == tau) {  // g = S^T r
    for (int q = threadIdx.x; q < tau; q += blockDim.x) {
      double s = 0.0;
      for (int e = sk.bptr[q]; e < sk.bptr[q + 1]; ++e) {
        const double v = r[sk.coord[e]];
        s += sk.sign[e] > 0 ? v : -v;
      }
      Gx[(long long)tau * ldg + q] = s;
    }
    return;
  }
  const int e0 = sk.bptr[a], e1 = sk.bptr[a + 1];
  for (int b = threadIdx.x; b <= a; b += blockDim.x) {
    double s = 0.0;
    for (int e = e0; e < e1; ++e) {
      const double v = AS[(long long)sk.coord[e] * ld_as + b];
      s += sk.sign[e] > 0 ? v : -v;
    }
    const bool b_empty = sk.bptr[b] == sk.bptr[b + 1];
    if (b_empty || e0 == e1) s = (a == b) ? 1.0 : 0.0;   // empty-bucket rule (R3)
    Gx[(long long)a * ldg + b] = s;
  }
}

// Records a failed pivot.  `done` is NOT set here (a late-starting CTA of this cooperative grid
// must not see it and skip the grid barriers); the update kernel turns the status into `done`.
__device__ __forceinline__ void flag_notspd(Ctrl* ctrl) { ctrl->status = ST_NOTSPD; }

// Cooperative blocked Cholesky of the bordered Gx, backward solve, scatter of S delta.
__global__ void __launch_bounds__(CT)
k_chol(double* __restrict__ Gx, long long ldg, int tau, DevSketch sk, double* __restrict__ delta,
       double* __restrict__ sdelta, Ctrl* ctrl) {
  if (ctrl->done) return;   // uniform across the grid: set before this launch
  cg::grid_group grid = cg::this_grid();
  __shared__ double T0[NB][NB + 1];
  __shared__ double T1[NB][NB + 1];
  __shared__ double T2[NB][NB + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows = tau + 1;
  const int Tc = (tau + NB - 1) / NB;        // block columns
  const int Tr = (rows + NB - 1) / NB;       // block rows (incl. border row tau)
  bool bad = false;

  for (int p = 0; p < Tc; ++p) {
    const int c0 = p * NB, cp = min(NB, tau - c0);
    // ---- phase 1: factor the diagonal tile (rows c0.., incl. the border row if it is in it)
    if (blockIdx.x == 0) {
      const int rp = min(NB, rows - c0);
      for (int q = tid; q < NB * NB; q += CT) {
        const int i = q / NB, j = q % NB;
        T0[i][j] = (i < rp && j < cp && j <= i) ? __ldcg(&Gx[(long long)(c0 + i) * ldg + c0 + j]) : 0.0;
      }
      __syncthreads();
      if (warp == 0) {   // left-looking, lane i owns row i
        for (int j = 0; j < cp; ++j) {
          double s = 0.0;
          if (lane >= j && lane < rp) {
            s = T0[lane][j];
            for (int k = 0; k < j; ++k) s -= T0[lane][k] * T0[j][k];
          }
          double dj = __shfl_sync(0xffffffffu, s, j);
          if (!(dj > 0.0) || !isfinite(dj)) { bad = true; dj = 1.0; }
          dj = sqrt(dj);
          if (lane == j) T0[lane][j] = dj;
          else if (lane > j && lane < rp) T0[lane][j] = s / dj;
          __syncwarp();
        }
        if (bad && lane == 0) flag_notspd(ctrl);
      }
      __syncthreads();
      for (int q = tid; q < NB * NB; q += CT) {
        const int i = q / NB, j = q % NB;
        if (i < rp && j < cp && j <= i) Gx[(long long)(c0 + i) * ldg + c0 + j] = T0[i][j];
      }
    }
    grid.sync();
    // ---- phase 2: panel  L_ip = G_ip L_pp^{-T}  for block rows i > p
    {
      bool loaded = false;
      for (int i = p + 1 + blockIdx.x; i < Tr; i += gridDim.x) {
        if (!loaded) {
          for (int q = tid; q < NB * NB; q += CT) {
            const int a = q / NB, j = q % NB;
            T0[a][j] = (a < cp && j <= a) ? __ldcg(&Gx[(long long)(c0 + a) * ldg + c0 + j]) : 0.0;
          }
          loaded = true;
        }
        const int r0 = i * NB, ri = min(NB, rows - r0);
        for (int q = tid; q < NB * NB; q += CT) {
          const int a = q / NB, j = q % NB;
          T1[a][j] = (a < ri && j < cp) ? __ldcg(&Gx[(long long)(r0 + a) * ldg + c0 + j]) : 0.0;
        }
        __syncthreads();
        if (warp == 0 && lane < ri) {   // row `lane`: forward substitution x L^T = g
          for (int j = 0; j < cp; ++j) {
            double s = T1[lane][j];
            for (int k = 0; k < j; ++k) s -= T1[lane][k] * T0[j][k];
            T1[lane][j] = s / T0[j][j];
          }
        }
        __syncthreads();
        for (int q = tid; q < NB * NB; q += CT) {
          const int a = q / NB, j = q % NB;
          if (a < ri && j < cp) Gx[(long long)(r0 + a) * ldg + c0 + j] = T1[a][j];
        }
        __syncthreads();
      }
    }
    grid.sync();
    // ---- phase 3: trailing update  G_ij -= L_ip L_jp^T,  p < j <= i < Tr (j < Tc)
    {
      const int nj = Tc - (p + 1);
      // enumerate tiles (i, j), j in [p+1, Tc), i in [j, Tr)
      long long ntiles = 0;
      for (int j = p + 1; j < Tc; ++j) ntiles += Tr - j;
      (void)nj;
      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int j = p + 1;
        long long tt = t;
        while (tt >= Tr - j) { tt -= Tr - j; ++j; }
        const int i = j + (int)tt;
        const int ri = min(NB, rows - i * NB), rj = min(NB, tau - j * NB);
        for (int q = tid; q < NB * NB; q += CT) {
          const int a = q / NB, k = q % NB;
          T1[a][k] = (a < ri && k < cp) ? __ldcg(&Gx[(long long)(i * NB + a) * ldg + c0 + k]) : 0.0;
          T2[a][k] = (a < rj && k < cp) ? __ldcg(&Gx[(long long)(j * NB + a) * ldg + c0 + k]) : 0.0;
        }
        __syncthreads();
        for (int q = tid; q < NB * NB; q += CT) {
          const int a = q / NB, c = q % NB;
          const int gi = i * NB + a, gj = j * NB + c;
          if (a < ri && c < rj && (i != j || c <= a) && gj < tau) {
            double s = 0.0;
#pragma unroll 8
            for (int k = 0; k < NB; ++k) s += T1[a][k] * T2[c][k];
            { double* gp = &Gx[(long long)gi * ldg + gj]; __stcg(gp, __ldcg(gp) - s); }
          }
        }
        __syncthreads();
      }
    }
    grid.sync();
  }
  if (blockIdx.x != 0) return;
  if (ctrl->status == ST_NOTSPD) return;
  // ---- backward solve L^T delta = y (y = row tau of Gx), block columns from the last
  double* y = Gx + (long long)tau * ldg;   // overwritten by the running right-hand side z
  for (int p = Tc - 1; p >= 0; --p) {
    const int c0 = p * NB, cp = min(NB, tau - c0);
    for (int q = tid; q < NB * NB; q += CT) {
      const int a = q / NB, j = q % NB;
      T0[a][j] = (a < cp && j <= a) ? __ldcg(&Gx[(long long)(c0 + a) * ldg + c0 + j]) : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      double z = lane < cp ? __ldcg(&y[c0 + lane]) : 0.0;
      for (int a = cp - 1; a >= 0; --a) {
        const double da = __shfl_sync(0xffffffffu, z, a) / T0[a][a];
        if (lane == a) z = da;
        else if (lane < a) z -= T0[a][lane] * da;
      }
      if (lane < cp) { y[c0 + lane] = z; delta[c0 + lane] = z; }
    }
    __syncthreads();
    // z_a -= sum_{q in block p} L[q][a] delta_q  for a < c0
    for (int a = tid; a < c0; a += CT) {
      double s = 0.0;
      for (int q = 0; q < cp; ++q) s += __ldcg(&Gx[(long long)(c0 + q) * ldg + a]) * y[c0 + q];
      y[a] = __ldcg(&y[a]) - s;
    }
    __syncthreads();
  }
  // S delta scatter (coordinates are distinct across entries)
  for (int e = tid; e < sk.len; e += CT) {
    const double d = delta[sk.bucket[e]];
    sdelta[sk.coord[e]] = sk.sign[e] > 0 ? d : -d;
  }
}

}  // namespace

size_t solve_gx_elems(int tau) {
  const long long ldg = ((long long)tau + NB - 1) / NB * NB;
  return (size_t)(tau + 1) * (size_t)ldg;
}

SolveWork plan_solve(int tau, int num_sms) {
  SolveWork w{};
  w.ldg = ((long long)tau + NB - 1) / NB * NB;
  const int Tc = (tau + NB - 1) / NB, Tr = (tau + 1 + NB - 1) / NB;
  long long tiles0 = 0;
  for (int j = 1; j < Tc; ++j) tiles0 += Tr - j;
  long long g = std::max<long long>(1, std::max<long long>(tiles0, Tr - 1));
  w.grid = (int)std::min<long long>(g, num_sms);
  return w;
}

cudaError_t launch_sketched_solve(const double* ASt, long long ld_as, bool as_rowmajor,
                                  const double* r, const DevSketch& sk, SolveWork& sw,
                                  double* sdelta, Ctrl* ctrl, cudaStream_t st) {
  if (as_rowmajor)
    k_form_g_rm<<<sk.tau + 1, 256, 0, st>>>(ASt, ld_as, r, sk, sw.Gx, sw.ldg, ctrl);
  else
    k_form_g<<<sk.tau + 1, 256, 0, st>>>(ASt, ld_as, r, sk, sw.Gx, sw.ldg, ctrl);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int tau = sk.tau;
  DevSketch skc = sk;
  void* args[] = {&sw.Gx, &sw.ldg, &tau, &skc, &sw.delta, &sdelta, &ctrl};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)sw.grid);
  cfg.blockDim = dim3(CT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, (const void*)k_chol, args);
}

}  // namespace rs
