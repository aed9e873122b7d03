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

// Gram mode: Gx[a][b] = Gram[a][b] + lambda |bucket a| delta_ab (b <= a); row tau = g = S^T r.
__global__ void k_form_g_gram(const double* __restrict__ Gram, long long ld_gram, double lambda,
                              const double* __restrict__ r, DevSketch sk, double* __restrict__ Gx,
                              long long ldg, const Ctrl* ctrl) {
  if (ctrl->done) return;
  const int a = blockIdx.x, tau = sk.tau;
  if (a == tau) {
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
    double s = Gram[(long long)a * ld_gram + b];
    if (a == b) s += lambda * (double)(e1 - e0);
    if (e0 == e1 || sk.bptr[b] == sk.bptr[b + 1]) s = (a == b) ? 1.0 : 0.0;   // R3
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

// Single-CTA path for tau <= kSmallTau.  The bordered matrix (lower triangle of G plus the row
// g^T) lives in shared memory as 8 x 8 blocks, block-packed by block row (block (I, J), J <= I, at
// index I(I+1)/2 + J), each block row-major with an XOR swizzle (column c of row r stored at
// c ^ 4((r >> 1) & 1)) so that DMMA fragment loads are bank-conflict free.  Blocked right-looking
// Cholesky, block width 8:
//   panel p  : warp 0 factors the whole block column (diagonal block + every block below it,
//              including the border row = forward substitution), left-looking inside the panel;
//   trailing : all warps update blocks (I, J), p < J <= I, with two mma.sync.m8n8k4.f64 each
//              (C -= L_Ip L_Jp^T, SASS DMMA).
// Two block barriers per block column; then warp 0 runs the blocked backward substitution.
constexpr int kSmallTau = 224;
// phase timers (debug; read by rs_internal_chol_times): 0 gather, 1 diag, 2 panel, 3 trailing,
// 4 backward, 5 scatter, 6 calls
__device__ unsigned long long g_chol_t[8];
constexpr int kSmallThreads = 1024;
constexpr int NB8 = 8;

__device__ __forceinline__ int blk(int I, int J) { return I * (I + 1) / 2 + J; }
// shared index of element (row, col) of the bordered matrix (col <= row, block-lower)
__device__ __forceinline__ int sidx(int row, int col) {
  const int I = row >> 3, J = col >> 3, r = row & 7, c = col & 7;
  return blk(I, J) * 64 + r * 8 + (c ^ (((r >> 1) & 1) << 2));
}
__device__ __forceinline__ void dmma8(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kSmallThreads, 1)
k_chol_small(const double* __restrict__ ASt, long long ld_as, bool rowmajor,
             const double* __restrict__ Gram, long long ld_gram, double lambda,
             const double* __restrict__ r, DevSketch sk, double* __restrict__ delta,
             double* __restrict__ sdelta, Ctrl* ctrl) {
  if (ctrl->done) return;
  extern __shared__ double sL[];
  const int tau = sk.tau, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows = tau + 1;
  const int Tc = (tau + NB8 - 1) / NB8, Tr = (rows + NB8 - 1) / NB8;
  const int nblk = blk(Tr - 1, 0) + min(Tr, Tc);   // blocks of the last block row: J < min(Tr, Tc)
  __shared__ double s_inv[kSmallTau];
  __shared__ int s_bad;
  // trailing-tile list of step 0: (I, J) for 1 <= J < Tc, J <= I < Tr, ordered by J then I;
  // s_toff[J] = index of the first tile of column J
  constexpr int kMaxT = (kSmallTau + 1 + NB8 - 1) / NB8 + 1;
  __shared__ unsigned char s_tI[kMaxT * kMaxT / 2 + kMaxT], s_tJ[kMaxT * kMaxT / 2 + kMaxT];
  __shared__ int s_toff[kMaxT + 1];
  if (tid == 0) {
    s_bad = 0;
    int t = 0;
    s_toff[0] = 0;
    for (int J = 0; J < Tc; ++J) {
      s_toff[J] = t;
      if (J == 0) continue;
      for (int I = J; I < Tr; ++I, ++t) {
        s_tI[t] = (unsigned char)I;
        s_tJ[t] = (unsigned char)J;
      }
    }
    s_toff[Tc] = t;
  }
  long long tc0 = clock64(), tc1;
  unsigned long long acc_t[6] = {0, 0, 0, 0, 0, 0};
#define RS_STAMP(k)                       \
  if (tid == 0) {                         \
    tc1 = clock64();                      \
    acc_t[k] += (unsigned long long)(tc1 - tc0); \
    tc0 = tc1;                            \
  }
  // ---- a4: gather G (lower) and g into the blocked layout; padding entries = 0
  for (int q = tid; q < nblk * 64; q += kSmallThreads) sL[q] = 0.0;
  __syncthreads();
  for (int a = warp; a <= tau; a += kSmallThreads / 32) {   // one warp per row of G (row tau = g)
    if (a == tau) {
      for (int c = lane; c < tau; c += 32) {
        double v = 0.0;
        for (int t = sk.bptr[c]; t < sk.bptr[c + 1]; ++t) {
          const double x = r[sk.coord[t]];
          v += sk.sign[t] > 0 ? x : -x;
        }
        sL[sidx(tau, c)] = v;
      }
      continue;
    }
    const int e0 = sk.bptr[a], e1 = sk.bptr[a + 1];
    for (int c = lane; c <= a; c += 32) {
      double v = 0.0;
      if (Gram) {   // Gram mode: G = (XS)^T XS + lambda S^T S, S^T S = diag(|bucket|)
        v = Gram[(long long)a * ld_gram + c];
        if (a == c) v += lambda * (double)(e1 - e0);
      } else {
        for (int t = e0; t < e1; ++t) {
          const long long co = sk.coord[t];
          const double x = rowmajor ? ASt[co * ld_as + c] : ASt[(long long)c * ld_as + co];
          v += sk.sign[t] > 0 ? x : -x;
        }
      }
      if (e0 == e1 || sk.bptr[c] == sk.bptr[c + 1]) v = (a == c) ? 1.0 : 0.0;   // R3
      sL[sidx(a, c)] = v;
    }
  }
  __syncthreads();
  RS_STAMP(0)
  for (int p = 0; p < Tc; ++p) {
    const int c0 = p * NB8;
    const int ncol = min(NB8, tau - c0);
    // ---- diagonal block (warp 0, registers): lane r holds row c0 + r; left-looking, rsqrt pivots
    if (warp == 0) {
      const int rr = lane & 7;
      const int grow = c0 + rr;
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = (k <= rr && grow < rows) ? sL[sidx(grow, c0 + k)] : 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < ncol) {
          double sj = v[j];
#pragma unroll
          for (int k = 0; k < j; ++k) sj -= v[k] * __shfl_sync(0xffffffffu, v[k], j);
          double d = __shfl_sync(0xffffffffu, sj, j);
          if (!(d > 0.0) || !isfinite(d)) { if (lane == 0) s_bad = 1; d = 1.0; }
          const double inv = rsqrt(d);
          if (rr == j) v[j] = d * inv;
          else if (rr > j) v[j] = sj * inv;
          if (lane == j) s_inv[c0 + j] = inv;
        }
      }
      if (lane < 8 && grow < rows) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k <= rr && k < ncol) sL[sidx(grow, c0 + k)] = v[k];
      }
    }
    __syncthreads();
    RS_STAMP(1)
    // ---- panel below the diagonal block (all threads, one row each): x L_pp^T = g
    for (int row = c0 + NB8 + tid; row < rows; row += kSmallThreads) {
      double x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = k < ncol ? sL[sidx(row, c0 + k)] : 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < ncol) {
#pragma unroll
          for (int k = 0; k < j; ++k) x[j] -= x[k] * sL[sidx(c0 + j, c0 + k)];
          x[j] *= s_inv[c0 + j];
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < ncol) sL[sidx(row, c0 + k)] = x[k];
    }
    __syncthreads();
    RS_STAMP(2)
    // ---- trailing update of blocks (I, J), p < J <= I < Tr, J < Tc: C -= L_Ip L_Jp^T
    {
      const int ar = lane >> 2, ak = lane & 3;
      // tiles with J >= p + 1 are a suffix of the step-0 list (ordered by J, then I)
      const int t_end = s_toff[Tc];
      for (int t = s_toff[p + 1] + warp; t < t_end; t += kSmallThreads / 32) {
        const int I = s_tI[t], J = s_tJ[t];
        const double* Lip = sL + blk(I, p) * 64;
        const double* Ljp = sL + blk(J, p) * 64;
        double* Cb = sL + blk(I, J) * 64;
        const int sw = ((ar >> 1) & 1) << 2;
        const double a0 = -Lip[ar * 8 + (ak ^ sw)], a1 = -Lip[ar * 8 + ((ak + 4) ^ sw)];
        const double b0 = Ljp[ar * 8 + (ak ^ sw)], b1 = Ljp[ar * 8 + ((ak + 4) ^ sw)];
        const int cr = ar, cc = 2 * ak;
        const int csw = ((cr >> 1) & 1) << 2;
        double acc[2] = {Cb[cr * 8 + (cc ^ csw)], Cb[cr * 8 + ((cc + 1) ^ csw)]};
        dmma8(acc, a0, b0);
        dmma8(acc, a1, b1);
        Cb[cr * 8 + (cc ^ csw)] = acc[0];
        Cb[cr * 8 + ((cc + 1) ^ csw)] = acc[1];
      }
    }
    __syncthreads();
    RS_STAMP(3)
  }
  if (s_bad) {
    if (tid == 0) ctrl->status = ST_NOTSPD;
    return;
  }
  // ---- backward substitution L^T delta = y; y = border row, overwritten by delta.  Per block
  // column (from the last): warp 0 solves the 8 x 8 diagonal block in registers, then all threads
  // update y_k -= sum_{q in block} L[q][k] delta_q for k < c0.
  for (int p = Tc - 1; p >= 0; --p) {
    const int c0 = p * NB8, ncol = min(NB8, tau - c0);
    if (warp == 0) {
      const int q = lane & 7;
      double yq = q < ncol ? sL[sidx(tau, c0 + q)] : 0.0;
#pragma unroll
      for (int j = 7; j >= 0; --j) {
        if (j < ncol) {
          const double dj = __shfl_sync(0xffffffffu, yq, j) * s_inv[c0 + j];
          if (q == j) yq = dj;
          else if (q < j) yq -= sL[sidx(c0 + j, c0 + q)] * dj;
        }
      }
      if (lane < ncol) sL[sidx(tau, c0 + lane)] = yq;
    }
    __syncthreads();
    for (int k = tid; k < c0; k += kSmallThreads) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < ncol) s += sL[sidx(c0 + q, k)] * sL[sidx(tau, c0 + q)];
      sL[sidx(tau, k)] -= s;
    }
    __syncthreads();
  }
  RS_STAMP(4)
  for (int b = tid; b < tau; b += kSmallThreads) delta[b] = sL[sidx(tau, b)];
  for (int e = tid; e < sk.len; e += kSmallThreads) {
    const double dv = sL[sidx(tau, sk.bucket[e])];
    sdelta[sk.coord[e]] = sk.sign[e] > 0 ? dv : -dv;
  }
  RS_STAMP(5)
  if (tid == 0) {
    for (int k = 0; k < 6; ++k) atomicAdd(&g_chol_t[k], acc_t[k]);
    atomicAdd(&g_chol_t[6], 1ull);
  }
#undef RS_STAMP
}

size_t small_smem(int tau) {
  const int Tr = (tau + 1 + NB8 - 1) / NB8;
  return (size_t)(Tr * (Tr + 1) / 2) * 64 * sizeof(double);
}

}  // namespace

extern "C" int rs_internal_chol_times(unsigned long long* out) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_chol_t, sizeof(g_chol_t));
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(g_chol_t, z, sizeof(z));
  return (int)e;
}

cudaError_t chol_init() {
  return cudaFuncSetAttribute(k_chol_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)small_smem(kSmallTau));
}

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
                                  const double* Gram, long long ld_gram, double lambda,
                                  const double* r, const DevSketch& sk, SolveWork& sw,
                                  double* sdelta, Ctrl* ctrl, cudaStream_t st) {
  if (sk.tau <= kSmallTau) {
    k_chol_small<<<1, kSmallThreads, small_smem(sk.tau), st>>>(ASt, ld_as, as_rowmajor, Gram,
                                                                ld_gram, lambda, r, sk, sw.delta,
                                                                sdelta, ctrl);
    return cudaGetLastError();
  }
  if (Gram)
    k_form_g_gram<<<sk.tau + 1, 256, 0, st>>>(Gram, ld_gram, lambda, r, sk, sw.Gx, sw.ldg, ctrl);
  else if (as_rowmajor)
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
