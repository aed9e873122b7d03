// Sketch-ahead batched factorisation -- SURVEY §8(a) rows a4 + a5 ("the fused S^T A S gather plus
// batched tau x tau Cholesky", BASELINE.json north_star).
//
// Alg. 2 draws S_k ~ D independently of the iterate, so G_k = S_k^T A S_k
// is a function of (seed, k) and the data only.  For a group of P future iterations the
// engine draws the P sketches, forms the P matrices G_k and factors them here in ONE launch (one CTA
// per G_k, all SMs busy), off the iteration's critical path:
//
//   G = L L^T       right-looking blocked Cholesky, 8 x 8 blocks, DMMA trailing updates
//                   (lower triangle of G read only, R12; empty-bucket rule R3)
//   W = L^{-1}      blocked in-place triangular inversion (column blocks from the last):
//                   W_JJ = L_JJ^{-1},  W_IJ = -(sum_{K=J+1..I} W_IK L_KJ) W_JJ
//   Ginv = W^T W    = G^{-1}, written in full (tau x tau, row-major) to the slot (tau <= 224); for
//                   tau > 224 the slot holds W (lower) and W^T (upper) instead
//
// so the iteration needs only delta = Ginv (S^T r^k) = W^T (W g) (P:L217 least-norm solution =
// G^{-1} g for SPD G, R3/R21): parallel GEMVs instead of a latency-bound factorisation per
// iteration.
//
// Shared-memory layout (one CTA, tau <= 224): the lower block triangle of G as 8 x 8 blocks packed by
// block row (block (I, J), J <= I, at index I(I+1)/2 + J), each block row-major with an XOR swizzle
// (column c of row r at c ^ 4((r >> 1) & 1)) so DMMA fragment loads -- plain and transposed -- are
// bank-conflict free; then a panel temp of Tc blocks.
#include <algorithm>
#include <cstdlib>

#include "rs_internal.cuh"

namespace rs {

namespace {

constexpr int BF_THREADS = 1024;
constexpr int BF_WARPS = BF_THREADS / 32;
constexpr int BF_MAXTAU = 224;
constexpr int AG_WARPS = 8;
constexpr int AG_MAXTAU = 4096;

__device__ __forceinline__ int bblk(int I, int J) { return I * (I + 1) / 2 + J; }
__device__ __forceinline__ int bsw(int r, int c) { return r * 8 + (c ^ (((r >> 1) & 1) << 2)); }
__device__ __forceinline__ int bidx(int row, int col) {
  return bblk(row >> 3, col >> 3) * 64 + bsw(row & 7, col & 7);
}
// D = A B + D, A 8x4 row-major (lane: A[lane/4][lane%4]), B 4x8 (lane: B[lane%4][lane/4]),
// D 8x8 (lane: D[lane/4][2(lane%4)], D[lane/4][2(lane%4)+1]).  SASS DMMA.8x8x4.
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
// t -> (I, J), J <= I, t = I(I+1)/2 + J
__device__ __forceinline__ void tri_decode(int t, int& I, int& J) {
  int i = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  I = i;
  J = t - i * (i + 1) / 2;
}

size_t bf_smem(int tau) {
  const int Tc = (tau + 7) / 8;
  return (size_t)(Tc * (Tc + 1) / 2 + Tc) * 64 * sizeof(double);
}

__global__ void __launch_bounds__(BF_THREADS, 1)
k_bfactor_small(FactorSrc src, DevSketch skb, double* __restrict__ Ginv, long long ldgi,
                long long gi_stride, int* __restrict__ flags, const Ctrl* ctrl) {
  if (slot_unused(ctrl, blockIdx.x)) return;
  extern __shared__ double sL[];
  __shared__ double s_inv[BF_MAXTAU];
  __shared__ int s_bad;
  const int slot = blockIdx.x;
  const DevSketch sk = skb.at(slot);
  const int tau = sk.tau, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ar = lane >> 2, ak = lane & 3;
  const int Tc = (tau + 7) / 8;
  const int nblk = Tc * (Tc + 1) / 2;
  double* sT = sL + nblk * 64;
  for (int q = tid; q < (nblk + Tc) * 64; q += BF_THREADS) sL[q] = 0.0;
  for (int q = tid; q < BF_MAXTAU; q += BF_THREADS) s_inv[q] = 0.0;
  if (tid == 0) s_bad = 0;
  __syncthreads();

  // ---- a4: G = S^T A S (lower): from AS^T rows (G[a][c] = sum_{e in a} sign_e AS^T[c][coord_e])
  // or from the Gram slot (G = (XS)^T XS + lambda S^T S, S^T S = diag(|bucket|)); R3 rule.
  const double* ASt = src.ASt ? src.ASt + slot * src.as_stride : nullptr;
  const double* Gram = src.Gram ? src.Gram + slot * src.gram_stride : nullptr;
  for (int a = warp; a < tau; a += BF_WARPS) {
    const int e0 = sk.bptr[a], e1 = sk.bptr[a + 1];
    for (int c = lane; c <= a; c += 32) {
      double v = 0.0;
      if (Gram) {
        v = Gram[(long long)a * src.ld_gram + c];
        if (a == c) v += src.lambda * (double)(e1 - e0);
      } else if (!ASt) {   // straight from explicit A
        const int f0 = sk.bptr[c], f1 = sk.bptr[c + 1];
        for (int e = e0; e < e1; ++e) {
          const double* Ae = src.A + (long long)sk.coord[e] * src.lda;
          double t = 0.0;
          for (int f = f0; f < f1; ++f) {
            const double x = Ae[sk.coord[f]];
            t += sk.sign[f] > 0 ? x : -x;
          }
          v += sk.sign[e] > 0 ? t : -t;
        }
      } else {
        const double* col = ASt + (long long)c * src.ld_as;
        for (int e = e0; e < e1; ++e) {
          const double x = col[sk.coord[e]];
          v += sk.sign[e] > 0 ? x : -x;
        }
      }
      if (e0 == e1 || sk.bptr[c] == sk.bptr[c + 1]) v = (a == c) ? 1.0 : 0.0;
      sL[bidx(a, c)] = v;
    }
  }
  __syncthreads();

  // ---- a5: Cholesky G = L L^T, block columns p = 0 .. Tc-1
  for (int p = 0; p < Tc; ++p) {
    const int c0 = p * 8, ncol = min(8, tau - c0);
    if (warp == 0) {   // diagonal block in registers: lane (mod 8) = row, left-looking
      const int rr = lane & 7, grow = c0 + rr;
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = (k <= rr && rr < ncol) ? sL[bidx(grow, c0 + k)] : 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < ncol) {
          double sj = v[j];
#pragma unroll
          for (int k = 0; k < j; ++k) sj -= v[k] * __shfl_sync(0xffffffffu, v[k], j);
          double dd = __shfl_sync(0xffffffffu, sj, j);
          if (!(dd > 0.0) || !isfinite(dd)) {
            if (lane == 0) s_bad = 1;
            dd = 1.0;
          }
          const double inv = rsqrt(dd);
          if (rr == j) v[j] = dd * inv;
          else if (rr > j) v[j] = sj * inv;
          if (lane == j) s_inv[c0 + j] = inv;
        }
      }
      if (lane < 8 && rr < ncol) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k <= rr) sL[bidx(grow, c0 + k)] = v[k];
      }
    }
    __syncthreads();
    // panel: rows below the diagonal block, one thread per row:  x L_pp^T = g
    for (int row = c0 + 8 + tid; row < tau; row += BF_THREADS) {
      double x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = k < ncol ? sL[bidx(row, c0 + k)] : 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < ncol) {
#pragma unroll
          for (int k = 0; k < j; ++k) x[j] -= x[k] * sL[bidx(c0 + j, c0 + k)];
          x[j] *= s_inv[c0 + j];
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < ncol) sL[bidx(row, c0 + k)] = x[k];
    }
    __syncthreads();
    // trailing update C_IJ -= L_Ip L_Jp^T, p < J <= I < Tc (two DMMA per block)
    {
      const int nt = Tc - 1 - p;
      const int ntiles = nt * (nt + 1) / 2;
      for (int t = warp; t < ntiles; t += BF_WARPS) {
        int Ii, Jj;
        tri_decode(t, Ii, Jj);
        const int I = p + 1 + Ii, J = p + 1 + Jj;
        const double* Lip = sL + bblk(I, p) * 64;
        const double* Ljp = sL + bblk(J, p) * 64;
        double* Cb = sL + bblk(I, J) * 64;
        double acc[2] = {Cb[bsw(ar, 2 * ak)], Cb[bsw(ar, 2 * ak + 1)]};
        dmma(acc, -Lip[bsw(ar, ak)], Ljp[bsw(ar, ak)]);
        dmma(acc, -Lip[bsw(ar, ak + 4)], Ljp[bsw(ar, ak + 4)]);
        Cb[bsw(ar, 2 * ak)] = acc[0];
        Cb[bsw(ar, 2 * ak + 1)] = acc[1];
      }
    }
    __syncthreads();
  }
  if (s_bad) {
    if (tid == 0) flags[slot] = 1;
    return;
  }

  // ---- W = L^{-1} in place, block columns J = Tc-1 .. 0
  for (int J = Tc - 1; J >= 0; --J) {
    const int c0 = J * 8, ncol = min(8, tau - c0);
    if (warp == 0) {
      if (lane < 8) {   // lane j: column j of W_JJ = L_JJ^{-1} (forward substitution on e_j)
        const int j = lane;
        double x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          double xi = 0.0;
          if (j < ncol && i < ncol && i >= j) {
            if (i == j) {
              xi = s_inv[c0 + i];
            } else {
              double s = 0.0;
#pragma unroll
              for (int k = 0; k < i; ++k)
                if (k >= j) s += sL[bidx(c0 + i, c0 + k)] * x[k];
              xi = -s * s_inv[c0 + i];
            }
          }
          x[i] = xi;
        }
        double* Wjj = sL + bblk(J, J) * 64;
#pragma unroll
        for (int i = 0; i < 8; ++i) Wjj[bsw(i, j)] = x[i];   // zeros above the diagonal
      }
    } else {
      // T_I = sum_{K=J+1..I} W_IK L_KJ  (W_IK final for K > J; L_KJ still L)
      for (int I = J + warp; I < Tc; I += BF_WARPS - 1) {
        double acc[2] = {0.0, 0.0};
        for (int K = J + 1; K <= I; ++K) {
          const double* Wik = sL + bblk(I, K) * 64;
          const double* Lkj = sL + bblk(K, J) * 64;
          dmma(acc, Wik[bsw(ar, ak)], Lkj[bsw(ak, ar)]);
          dmma(acc, Wik[bsw(ar, ak + 4)], Lkj[bsw(ak + 4, ar)]);
        }
        sT[I * 64 + bsw(ar, 2 * ak)] = acc[0];
        sT[I * 64 + bsw(ar, 2 * ak + 1)] = acc[1];
      }
    }
    __syncthreads();
    // W_IJ = -T_I W_JJ, written over L_IJ
    for (int I = J + 1 + warp; I < Tc; I += BF_WARPS) {
      const double* Ti = sT + I * 64;
      const double* Wjj = sL + bblk(J, J) * 64;
      double acc[2] = {0.0, 0.0};
      dmma(acc, Ti[bsw(ar, ak)], Wjj[bsw(ak, ar)]);
      dmma(acc, Ti[bsw(ar, ak + 4)], Wjj[bsw(ak + 4, ar)]);
      double* Cb = sL + bblk(I, J) * 64;
      Cb[bsw(ar, 2 * ak)] = -acc[0];
      Cb[bsw(ar, 2 * ak + 1)] = -acc[1];
    }
    __syncthreads();
  }

  // ---- Ginv = W^T W: block (I, J), J <= I, = sum_{K >= I} W_KI^T W_KJ; mirrored above
  double* Gi = Ginv + slot * gi_stride;
  const int npairs = Tc * (Tc + 1) / 2;
  for (int t = warp; t < npairs; t += BF_WARPS) {
    int I, J;
    tri_decode(t, I, J);
    double acc[2] = {0.0, 0.0};
    for (int K = I; K < Tc; ++K) {
      const double* Wki = sL + bblk(K, I) * 64;
      const double* Wkj = sL + bblk(K, J) * 64;
      dmma(acc, Wki[bsw(ak, ar)], Wkj[bsw(ak, ar)]);
      dmma(acc, Wki[bsw(ak + 4, ar)], Wkj[bsw(ak + 4, ar)]);
    }
    const int row = I * 8 + ar;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int col = J * 8 + 2 * ak + q;
      if (row < tau && col < tau) {
        Gi[(long long)row * ldgi + col] = acc[q];
        if (I != J) Gi[(long long)col * ldgi + row] = acc[q];
      }
    }
  }
  if (tid == 0) flags[slot] = 0;
}

// g = S^T r: one warp per bucket (lanes over the bucket's entries, fixed-order reduction).
__global__ void __launch_bounds__(AG_WARPS * 32)
k_sketch_g(DevSketch sk, const int* __restrict__ flag, const double* __restrict__ r,
           double* __restrict__ g, const Ctrl* ctrl) {
  pdl_trigger();   // the iteration's GEMV / update kernels may start their static loads
  if (ctrl->done || *flag) return;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * AG_WARPS + (threadIdx.x >> 5);
  if (b >= sk.tau) return;
  double v = 0.0;
  for (int e = sk.bptr[b] + lane; e < sk.bptr[b + 1]; e += 32) {
    const double x = r[sk.coord[e]];
    v += sk.sign[e] > 0 ? x : -x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) g[b] = v;
}

// Row GEMVs of the iteration, out_a = sum_c M[a][c] x_c over the column range of row a:
//   AP_FULL   (tau <= 224)  the slot holds G^{-1} in full:        delta = G^{-1} g, c in [0, tau)
//   AP_LOWER  (tau > 224)   lower triangle of the slot = W = L^{-1}: t = W g,      c in [0, a]
//   AP_UPPER  (tau > 224)   upper triangle of the slot = W^T:       delta = W^T t, c in [a, tau)
// AP_FULL / AP_UPPER also scatter S delta.  A block of 8 warps owns 2 rows, 4 warps per row
// (32-column chunks interleaved over the 4 warps).  The kernels are launched as a PDL chain after
// k_sketch_g: the first AP_PRE chunks of each lane's part of the row (the slot is static) are
// loaded into registers BEFORE pdl_wait(), so the slot reads of all three kernels of the iteration
// overlap each other and the predecessor; only the x vector is read after the wait.
enum { AP_FULL = 0, AP_LOWER = 1, AP_UPPER = 2 };
constexpr int AP_WPR = 4;                      // warps per row
constexpr int AP_ROWS = AG_WARPS / AP_WPR;     // rows per block
constexpr int AP_PRE = 8;                      // register-preloaded values per lane (1024 columns)

constexpr int AP_MAXFUSE = 4096;               // sketch entries of a fused g = S^T r

// x = g (MODE AP_FULL / AP_LOWER) or t (AP_UPPER).  gv == null: g = S^T r is formed here for the
// buckets the block needs (few entries per bucket): the entries (static) are staged before
// pdl_wait(), the residual is gathered after it.
template <int MODE>
__global__ void __launch_bounds__(AG_WARPS * 32)
k_apply_rows(const double* __restrict__ Mx, long long ldm, DevSketch sk, const int* __restrict__ flag,
             const double* __restrict__ x, const double* __restrict__ r, double* __restrict__ out,
             double* __restrict__ sdelta, Ctrl* ctrl, const double* __restrict__ pfA, long long pf_lda,
             unsigned pf_bytes) {
  pdl_trigger();
  if (pfA && threadIdx.x < 32) {   // EXPLICIT: pull this iteration's sketched rows of A into L2 for
    // the update kernel at the end of the chain (static data; one bulk prefetch per row)
    for (int e = blockIdx.x * 32 + threadIdx.x; e < sk.len; e += gridDim.x * 32)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(pfA + (long long)sk.coord[e] * pf_lda),
                   "r"(pf_bytes) : "memory");
  }
  extern __shared__ double xs[];     // [tau] x, then (fused g) s_bp[tau + 1], s_ce[len]
  __shared__ double red[AG_WARPS];
  const int bad = *flag;    // factor slot not SPD (static)
  const int tau = sk.tau, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* s_bp = reinterpret_cast<int*>(xs + tau);
  int* s_ce = s_bp + tau + 1;         // coord_e, bit-complemented for a negative sign
  const int q = warp % AP_WPR, a = blockIdx.x * AP_ROWS + warp / AP_WPR;
  const int c0 = MODE == AP_UPPER ? a : 0, c1 = MODE == AP_LOWER ? a + 1 : tau;
  const double* row = Mx + (long long)min(a, tau - 1) * ldm;
  const int cb = c0 + 32 * q + lane;                 // chunk u: column cb + 128 u
  const int p1 = min(c1, c0 + 32 * AP_WPR * AP_PRE);   // end of the preloaded pass
  double v[AP_PRE];
#pragma unroll
  for (int u = 0; u < AP_PRE; ++u) {
    const int c = cb + 32 * AP_WPR * u;
    v[u] = (!bad && a < tau && c < p1) ? __ldg(row + c) : 0.0;
  }
  const int xlo = MODE == AP_UPPER ? min(tau, blockIdx.x * AP_ROWS) : 0;
  const int xhi = MODE == AP_LOWER ? min(tau, (blockIdx.x + 1) * AP_ROWS) : tau;
  const bool fuse = MODE != AP_UPPER && x == nullptr;
  int e_lo = 0;
  if (fuse) {   // static sketch entries of buckets [xlo, xhi)
    e_lo = sk.bptr[xlo];
    const int e_hi = sk.bptr[xhi];
    for (int b = xlo + tid; b <= xhi; b += AG_WARPS * 32) s_bp[b - xlo] = sk.bptr[b] - e_lo;
    for (int e = e_lo + tid; e < e_hi; e += AG_WARPS * 32)
      s_ce[e - e_lo] = sk.sign[e] > 0 ? sk.coord[e] : ~sk.coord[e];
  }
  pdl_wait();
  if (ctrl->done) return;   // the previous iteration's stop rule (written by the predecessor)
  if (bad) {   // the update kernel of this iteration turns the status into `done`
    if (MODE != AP_UPPER && blockIdx.x == 0 && tid == 0) ctrl->status = ST_NOTSPD;
    return;
  }
  if (fuse) {
    __syncthreads();
    for (int b = xlo + tid; b < xhi; b += AG_WARPS * 32) {
      double g = 0.0;
      for (int e = s_bp[b - xlo]; e < s_bp[b - xlo + 1]; ++e) {
        const int ce = s_ce[e];
        g += ce >= 0 ? __ldcg(r + ce) : -__ldcg(r + ~ce);
      }
      xs[b] = g;
    }
  } else {
    for (int c = xlo + tid; c < xhi; c += AG_WARPS * 32) xs[c] = x[c];
  }
  __syncthreads();
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int u = 0; u < AP_PRE; ++u) {
    const int c = cb + 32 * AP_WPR * u;
    if (c < p1) (u & 1 ? s1 : s0) += v[u] * xs[c];
  }
  for (int c = p1 + 32 * q + lane; c < c1; c += 32 * AP_WPR) s0 += __ldg(row + c) * xs[c];
  double t = s0 + s1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) red[warp] = t;
  __syncthreads();
  if (q != 0 || a >= tau) return;
  const int w0 = warp;   // first warp of the row
  const double sa = (red[w0] + red[w0 + 1]) + (red[w0 + 2] + red[w0 + 3]);
  if (lane == 0) out[a] = sa;
  if (MODE != AP_LOWER)
    for (int e = sk.bptr[a] + lane; e < sk.bptr[a + 1]; e += 32)
      sdelta[sk.coord[e]] = sk.sign[e] > 0 ? sa : -sa;
}

// =================================================================================================
// Large tau (BF_MAXTAU < tau <= BB_MAXTAU): the first two steps with G held in global memory (a
// per-slot work matrix, zero-padded to whole 32 x 32 tiles with an identity tail so that every tile
// is full), one CTA of 16 warps per slot, every tile product on DMMA (one warp per 32 x 32 tile):
//   Cholesky   right-looking over block columns p: warp 0 factors L_pp in registers and forms
//              L_pp^{-1}; panel L_ip = G_ip L_pp^{-T}; trailing G_ij -= L_ip L_jp^T (j <= i)
//   W = L^{-1} block columns J from the last: T_I = sum_{K=J+1..I} W_IK L_KJ, W_IJ = -T_I W_JJ
//   the slot receives W (lower) and W^T (upper); delta = W^T (W g) per iteration (k_apply_w, _wt)
constexpr int BB_THREADS = 512;
constexpr int BB_WARPS = BB_THREADS / 32;
constexpr int BB_MAXTAU = 4096;

// padded size: a whole number of 64-wide tile pairs (identity padding)
__host__ __device__ __forceinline__ int bb_tp(int tau) { return (tau + 63) / 64 * 64; }

// acc[R][C] (8 x 8 blocks of a 32 x 32 tile) += op(A) op(B) (op(A) scaled by `sign`), with
// op(A)[r][k] = TA ? A[k][r] : A[r][k] and op(B)[k][c] = TB ? B[c][k] : B[k][c]; A has leading
// dimension lda, B ldb (row-major).
template <bool TA, bool TB>
__device__ __forceinline__ void mma_tile(double (&acc)[4][4][2], const double* A, int lda,
                                         const double* B, int ldb, int lane, double sign,
                                         int R0 = 0, int nR = 4) {
  // only the 8-row blocks R0 .. R0+nR-1 of the tile (warp-uniform range)
  const int q = lane >> 2, k4 = lane & 3;
#pragma unroll 1
  for (int K = 0; K < 8; ++K) {
    double a[4], b[4];
#pragma unroll
    for (int R = 0; R < 4; ++R) {
      const int r = 8 * R + q, k = 4 * K + k4;
      a[R] = (R >= R0 && R < R0 + nR)
                 ? sign * (TA ? A[(long long)k * lda + r] : A[(long long)r * lda + k]) : 0.0;
    }
#pragma unroll
    for (int C = 0; C < 4; ++C) {
      const int c = 8 * C + q, k = 4 * K + k4;
      b[C] = TB ? B[(long long)c * ldb + k] : B[(long long)k * ldb + c];
    }
#pragma unroll
    for (int R = 0; R < 4; ++R)
      if (R >= R0 && R < R0 + nR)
#pragma unroll
        for (int C = 0; C < 4; ++C) dmma(acc[R][C], a[R], b[C]);
  }
}
__device__ __forceinline__ void acc_load(double (&acc)[4][4][2], const double* Ct, int ld, int lane) {
  const int q = lane >> 2, k4 = lane & 3;
#pragma unroll
  for (int R = 0; R < 4; ++R)
#pragma unroll
    for (int C = 0; C < 4; ++C) {
      const double2 v = *reinterpret_cast<const double2*>(Ct + (long long)(8 * R + q) * ld + 8 * C + 2 * k4);
      acc[R][C][0] = v.x;
      acc[R][C][1] = v.y;
    }
}
__device__ __forceinline__ void acc_zero(double (&acc)[4][4][2]) {
#pragma unroll
  for (int R = 0; R < 4; ++R)
#pragma unroll
    for (int C = 0; C < 4; ++C) acc[R][C][0] = acc[R][C][1] = 0.0;
}
__device__ __forceinline__ void acc_store(const double (&acc)[4][4][2], double* Ct, int ld, int lane,
                                          int R0 = 0, int nR = 4) {
  const int q = lane >> 2, k4 = lane & 3;
#pragma unroll
  for (int R = 0; R < 4; ++R)
    if (R >= R0 && R < R0 + nR)
#pragma unroll
    for (int C = 0; C < 4; ++C) {
      *reinterpret_cast<double2*>(Ct + (long long)(8 * R + q) * ld + 8 * C + 2 * k4) =
          make_double2(acc[R][C][0], acc[R][C][1]);
    }
}

// Diagonal tile (one warp), on chip and in compact loops (it runs twice per block-column pair, from
// a cold instruction cache: fully unrolled register code measured 5x slower): D (32 x 32 shared,
// leading dim ldd, lower triangle read) is factored in place, right-looking, lane r owning row r;
// L goes to Lg (global, zeros above the diagonal) and L^{-1} (lane j = column j, forward
// substitution against the rows of L) to Dig (global, 32 x 32) and Dis (shared, leading dim ldis).
// Returns true if a pivot was <= 0 or not finite.
__device__ __noinline__ bool diag_factor_s(double* D, int ldd, double* Lg, int ldl, double* Dig,
                                           double* Dis, int ldis, int lane) {
  bool bad = false;
#pragma unroll 1
  for (int j = 0; j < 32; ++j) {
    double d = D[j * ldd + j];
    if (!(d > 0.0) || !isfinite(d)) {
      bad = true;
      d = 1.0;
    }
    const double ljj = sqrt(d), inv = 1.0 / ljj;
    __syncwarp();
    double lrj = 0.0;
    if (lane > j) {
      lrj = D[lane * ldd + j] * inv;
      D[lane * ldd + j] = lrj;
    }
    if (lane == j) D[j * ldd + j] = ljj;
    __syncwarp();
#pragma unroll 4
    for (int k = j + 1; k <= lane; ++k) D[lane * ldd + k] -= lrj * D[k * ldd + j];
    __syncwarp();
  }
#pragma unroll 4
  for (int r = 0; r < 32; ++r) Lg[(long long)r * ldl + lane] = lane <= r ? D[r * ldd + lane] : 0.0;
  // x = column `lane` of L^{-1}: x_i = (delta_{i,lane} - sum_{k<i} L_ik x_k) / L_ii (zero for i < lane)
#pragma unroll 1
  for (int i = 0; i < 32; ++i) {
    double t = (i == lane) ? 1.0 : 0.0;
#pragma unroll 4
    for (int k = lane; k < i; ++k) t -= D[i * ldd + k] * Dis[k * ldis + lane];
    const double x = i < lane ? 0.0 : t / D[i * ldd + i];
    __syncwarp();   // row i of L (read above) may share storage with row i of L^{-1} (Dis == D)
    Dis[i * ldis + lane] = x;
    Dig[i * 32 + lane] = x;
    __syncwarp();
  }
  __syncwarp();
  return bad;
}

// -------------------------------------------------------------------------------------------------
// Left-looking variant (default for tau > 224): block columns are processed in PAIRS (64 wide).
// Each warp accumulates a 32 x 64 strip in registers (acc[4][8][2]) from its own row tiles (the A
// operand) and the rows every strip of a step shares -- rows p0, p0+1 of L (Cholesky) or block
// columns J0, J1 of L (inverse), the B operand.  BOTH operands stream through an LP_STAGES-deep
// cp.async ring in 16-wide k slices (per stage: B 64 x 16 or 16 x 64, and one 32 x 16 A slice per
// warp), so the DMMA loop reads shared memory only and the slot's work matrix -- which 148 slots
// in flight keep in HBM, not L2 -- is fetched LP_STAGES - 1 slices ahead.  Global traffic is about
// Tc^3/12 tiles per phase (the right-looking kernel above re-reads and rewrites the trailing matrix
// every 32 columns).
//   Cholesky, pair p0 = 2P:  [C_i,p0 C_i,p0+1] = [G_i,p0 G_i,p0+1] - sum_{k<p0} L_ik [L_p0,k L_p0+1,k]^T
//     diagonal pair (warp 0): L00 = chol(C00), L10 = C10 L00^-T, L11 = chol(C11 - L10 L10^T)
//     strips i > p0+1: L_i,p0 = C_i,p0 L00^-T, L_i,p0+1 = (C_i,p0+1 - L_i,p0 L10^T) L11^-T
//   Inverse W = L^-1, pair (J0, J1 = J0+1) from the last: strips I > J1 (highest first, so that a
//   round never stages a row an earlier round has overwritten):
//     [T_I,J0 T_I,J1] = sum_{K=J1+1..I} W_IK [L_K,J0 L_K,J1]
//     W_I,J1 = -T_I,J1 W_J1J1,  W_I,J0 = -(T_I,J0 + W_I,J1 L_J1,J0) W_J0J0
//     diagonal pair: W_J1,J0 = -W_J1J1 L_J1,J0 W_J0J0
//   Blocked inverse (sbt < Tc, the group kernel's slots): the inverse runs inside each diagonal
//   super-block of sbt tiles only (strips I < E, the super-block's end), so W_bb = L_bb^{-1} costs
//   1/nb^2 of the full inverse's flop; the L tiles below the super-blocks go to the slot as their
//   strips are finished, and the iteration substitutes block by block (iterate.cu).
// Two shapes of the same kernel (LpCfg<NW>): 8 warps with 32-deep slices, one CTA per SM (the
// pipeline-fill group, all SMs free), and 4 warps with 16-deep slices, two CTAs per SM, so that one
// slot's barriers, diagonal pairs and finishing steps run while the other slot's warps keep the DMMA
// pipe busy (one warp per SM sub-partition nearly saturates it: profiles/r01_fp64_peak.txt).
template <int NW>
struct LpCfg {
  static constexpr int WARPS = NW;
  static constexpr int THREADS = NW * 32;           // 255 registers: acc[4][8][2] per lane
  static constexpr int CTAS = NW == 8 ? 1 : 2;      // resident CTAs per SM
#ifndef RS_LP4_KS
#define RS_LP4_KS 16
#endif
#ifndef RS_LP4_ST
#define RS_LP4_ST 2
#endif
#ifndef RS_LP8_ST
#define RS_LP8_ST 2
#endif
  static constexpr int KS = NW == 8 ? 32 : RS_LP4_KS;   // k slice depth
  static constexpr int STAGES = NW == 8 ? RS_LP8_ST : RS_LP4_ST;   // k slices in flight + 1
  static constexpr int BLD = KS + 4;                // B [n][k] row stride (Cholesky) and A [r][k]:
  static constexpr int ALD = KS + 4;                //   36 / 20 / 12 = +-4 mod 16 -> conflict-free
  static constexpr int BTLD = 68;                   // B [k][n] row stride (inverse), 68 = 4 mod 16
  static constexpr int BSZ = 64 * BLD;              // >= KS * BTLD
  static constexpr int ASZ = 32 * ALD;
  static constexpr int STAGE = BSZ + NW * ASZ;      // doubles per stage
  static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  // the ring doubles as the diagonal pair's 64 x 65 M and Lm, the split-reduce buffers (2048 per
  // warp) and the per-warp 32 x 36 finishing tiles
  static constexpr int RING = cmax(cmax(STAGES * STAGE, 2 * 64 * 65), NW * 2048);
  static constexpr size_t SMEM = ((size_t)RING + 3 * 32 * 36) * sizeof(double);   // ring + pair tiles
  static_assert(KS * BTLD <= BSZ, "inverse B tile must fit the B region");
  static_assert(NW * 32 * 36 <= RING, "finishing scratch must fit the ring");
};
#ifdef RS_BF_PHASES
// development probe (build with RS_NVCC_EXTRA=-DRS_BF_PHASES): SM cycles per factor phase, summed
// over CTAs: 0 gather, 1 chol accumulate, 2 chol diag, 3 chol total, 4 inv accumulate, 5 inv total,
// 6 inv diag, 7 write-out
__device__ unsigned long long g_bf_phase[8];
#define BF_T(v) long long v = clock64()
#define BF_ADD(ph, a, b) if (threadIdx.x == 0) atomicAdd(&g_bf_phase[ph], (unsigned long long)((b) - (a)))
#else
#define BF_T(v)
#define BF_ADD(ph, a, b)
#endif

__device__ __forceinline__ void lp_cp16(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

// One k slice of a strip: acc[R][C] += A[8R+q][k] B(k, 8C+q) -- A [r][k] (ALD), B [n][k] (BLD,
// Cholesky) or [k][n] (BTLD, inverse).
template <bool CHOL, class CF>
__device__ __forceinline__ void lp_slice(double (&acc)[4][8][2], const double* xs, const double* ys,
                                         int q, int k4) {
#pragma unroll
  for (int K = 0; K < CF::KS / 4; ++K) {
    double a[4];
#pragma unroll
    for (int R = 0; R < 4; ++R) a[R] = xs[(8 * R + q) * CF::ALD + 4 * K + k4];
#pragma unroll
    for (int C = 0; C < 8; ++C) {
      const int n = 8 * C + q, kq = 4 * K + k4;
      const double b = CHOL ? ys[n * CF::BLD + kq] : ys[kq * CF::BTLD + n];
#pragma unroll
      for (int R = 0; R < 4; ++R) dmma(acc[R][C], a[R], b);
    }
  }
}

// a4 for the large-tau factorisation: the lower triangle of G = S^T A S (R3 empty-bucket rule,
// identity on the padding) into each slot's work matrix, one warp per row, blockIdx.y = slot.  A
// kernel of its own (many warps per SM, no shared-memory ring) so that the random gathers from A
// have full memory-level parallelism.  The slot's sketch is staged per block: coord_e (sign folded
// in as bit complement) and bptr, so each element costs one independent gather of A.
constexpr int GA_WARPS = 8;
constexpr size_t GA_SMEM = (size_t)(4096 + 1 + 8192) * 4;
__global__ void __launch_bounds__(GA_WARPS * 32)
k_bf_gather(FactorSrc src, DevSketch skb, double* work, long long work_stride, const Ctrl* ctrl) {
  const int slot = blockIdx.y;
  __shared__ int s_unused;   // one reading per block (ctrl moves under a concurrent group kernel)
  if (threadIdx.x == 0) s_unused = slot_unused(ctrl, slot) ? 1 : 0;
  __syncthreads();
  if (s_unused) return;
  extern __shared__ __align__(16) double ga_sm[];
  const DevSketch sk = skb.at(slot);
  const int tau = sk.tau, tp = bb_tp(tau);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Wm = work + slot * work_stride;

  const double* ASt = src.ASt ? src.ASt + slot * src.as_stride : nullptr;
  const double* Gram = src.Gram ? src.Gram + slot * src.gram_stride : nullptr;
  int* s_bp = reinterpret_cast<int*>(ga_sm);
  int* s_ce = s_bp + tau + 1;
  const bool staged = !Gram && !ASt && (size_t)(tau + 1 + sk.len) * 4 <= GA_SMEM;
  if (staged) {
    for (int b = tid; b <= tau; b += GA_WARPS * 32) s_bp[b] = sk.bptr[b];
    for (int e = tid; e < sk.len; e += GA_WARPS * 32) s_ce[e] = sk.sign[e] > 0 ? sk.coord[e] : ~sk.coord[e];
    __syncthreads();
  }
  for (int a = blockIdx.x * GA_WARPS + warp; a < tp; a += gridDim.x * GA_WARPS) {
    const int a32 = a & ~31;
    const int e0 = a < tau ? (staged ? s_bp[a] : sk.bptr[a]) : 0;
    const int e1 = a < tau ? (staged ? s_bp[a + 1] : sk.bptr[a + 1]) : 0;
    if (staged && a < tau && e1 - e0 == 1) {   // subsample row: one entry
      const int ca = s_ce[e0];
      const double* Ae = src.A + (long long)(ca >= 0 ? ca : ~ca) * src.lda;
      const double sa = ca >= 0 ? 1.0 : -1.0;
      double* dst = Wm + (long long)a * tp;
      const bool single = sk.len == tau;   // subsample: exactly one entry per bucket
      const int n = a + 1;                 // columns c <= a (< tau)
      if (single) {   // batches of 32 independent gathers per lane (one batch for n <= 1024)
        for (int c0 = lane; c0 < n; c0 += 32 * 32) {
          double x[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int c = c0 + 32 * u;
            const int cf = c < n ? s_ce[c] : 0;
            x[u] = c < n ? __ldg(Ae + (cf >= 0 ? cf : ~cf)) : 0.0;
            if (cf < 0) x[u] = -x[u];
          }
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int c = c0 + 32 * u;
            if (c < n) dst[c] = sa * x[u];
          }
        }
      } else {
        for (int c = lane; c < n; c += 32) {
          const int f0 = s_bp[c], f1 = s_bp[c + 1];
          double v = 0.0;
          for (int f = f0; f < f1; ++f) {
            const int cf = s_ce[f];
            const double x = __ldg(Ae + (cf >= 0 ? cf : ~cf));
            v += cf >= 0 ? x : -x;
          }
          v *= sa;
          if (f0 == f1) v = 0.0;   // empty bucket c != a (R3)
          dst[c] = v;
        }
      }
      for (int c = n + lane; c < a32 + 32; c += 32) dst[c] = 0.0;   // above the diagonal
      continue;
    }
    for (int c = lane; c < a32 + 32; c += 32) {   // every lower tile of row a
      double v = 0.0;
      if (a >= tau || c >= tau || c > a) {
        v = (a == c) ? 1.0 : 0.0;
      } else if (Gram) {
        v = Gram[(long long)a * src.ld_gram + c];
        if (a == c) v += src.lambda * (double)(e1 - e0);
      } else if (!ASt) {
        const int f0 = staged ? s_bp[c] : sk.bptr[c], f1 = staged ? s_bp[c + 1] : sk.bptr[c + 1];
        for (int e = e0; e < e1; ++e) {
          const double* Ae = src.A + (long long)sk.coord[e] * src.lda;
          double t = 0.0;
          for (int f = f0; f < f1; ++f) {
            const double x = Ae[sk.coord[f]];
            t += sk.sign[f] > 0 ? x : -x;
          }
          v += sk.sign[e] > 0 ? t : -t;
        }
        if (e0 == e1 || f0 == f1) v = (a == c) ? 1.0 : 0.0;
      } else {
        const double* col = ASt + (long long)c * src.ld_as;
        for (int e = e0; e < e1; ++e) {
          const double x = col[sk.coord[e]];
          v += sk.sign[e] > 0 ? x : -x;
        }
      }
      if (a < tau && c < tau && c <= a && (Gram || ASt) && (e0 == e1 || sk.bptr[c] == sk.bptr[c + 1]))
        v = (a == c) ? 1.0 : 0.0;
      Wm[(long long)a * tp + c] = v;
    }
  }
}

// One slot's factorisation by the whole CTA; false: the solve has stopped (abandon the launch).
template <int NW>
__device__ __forceinline__ bool lp_factor_slot(const FactorSrc& src, const DevSketch& skb,
                                               double* __restrict__ Ginv, long long ldgi,
                                               long long gi_stride, double* work,
                                               long long work_stride, int* __restrict__ flags,
                                               const Ctrl* ctrl, const int slot, int sbt,
                                               int& s_bad, int& s_stop) {
  using CF = LpCfg<NW>;
  constexpr int LP_WARPS = CF::WARPS, LP_THREADS = CF::THREADS, LP_STAGES = CF::STAGES;
  constexpr int LP_STAGE = CF::STAGE, LP_BSZ = CF::BSZ, LP_ASZ = CF::ASZ, KS = CF::KS;
  constexpr int SPT = 32 / KS;   // k slices per 32-wide tile
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // slot beyond max_iter or solve done: ctrl->k and done move under a concurrent group kernel, so
  // one reading, shared by the block
  if (tid == 0) s_stop = slot_unused(ctrl, slot) ? 1 : 0;
  __syncthreads();
  const int unused = s_stop;
  __syncthreads();
  if (unused) return true;
  BF_T(t_start);
  extern __shared__ __align__(16) double lp_sm[];   // slice ring, then the pair tiles
  const DevSketch sk = skb.at(slot);
  const int tau = sk.tau, tp = bb_tp(tau), Tc = tp / 32;
  const int q = lane >> 2, k4 = lane & 3;
  // the solve may finish while this group is factored ahead (overlapped pipeline): poll its flag
  // once per block-column pair, block-uniformly
  auto stopped = [&]() {
    if (tid == 0) s_stop = ctrl ? *reinterpret_cast<const volatile int*>(&ctrl->done) : 0;
    __syncthreads();
    return s_stop != 0;
  };
  double* Wm = work + slot * work_stride;           // tp x tp, row-major
  double* dinv = Wm + (long long)tp * tp;           // Tc tiles 32 x 32 (L_pp^{-1})
  double* scr = dinv + (long long)Tc * 1024;        // 2 tiles per warp
  auto T = [&](int I, int J) { return Wm + (long long)(32 * I) * tp + 32 * J; };
  if (tid == 0) s_bad = 0;

  // ---- a4: lower triangle of G in the work matrix (k_bf_gather, the preceding launch)


  // Work split of a round of m strips (m <= LP_WARPS): spw warps per strip, part `part` of them
  // accumulating the k tiles kt with (kt - kb) % spw == part; the partial accumulators are summed
  // into part 0 in part order (deterministic) -- short rounds (the last pairs of each phase) keep
  // every warp on the DMMA pipe.  Returns the strip slot j (-1: idle warp).
  auto split = [&](int m, int& spw, int& part) {
    spw = m <= LP_WARPS / 4 ? 4 : (m <= LP_WARPS / 2 ? 2 : 1);
    part = warp % spw;
    const int j = warp / spw;
    return j < m ? j : -1;
  };
  // k slice s of [kb, ke): columns co .. co + KS - 1 of tile kt = kb + s / SPT (co = KS (s % SPT)).
  // Stage buffer: B then one A slice per warp.  Every thread commits one group per slice (possibly
  // empty), so wait_group counts stay uniform.
  double acc[4][8][2];
  auto issue = [&](int s, bool chol, int p0, int kb, bool act_a, int i) {
    double* buf = lp_sm + (s % LP_STAGES) * LP_STAGE;
    const int kt = kb + s / SPT, co = KS * (s % SPT);
#pragma unroll
    for (int u = 0; u < 32 * KS / LP_THREADS; ++u) {   // B: 32 KS pieces of 16 bytes
      const int t = tid + LP_THREADS * u;
      if (chol) {   // rows n of L_{p0 + n/32, kt} -> [n][BLD]
        const int n = t / (KS / 2), c16 = t % (KS / 2);
        lp_cp16(buf + n * CF::BLD + 2 * c16, T(p0 + (n >> 5), kt) + (long long)(n & 31) * tp + co + 2 * c16);
      } else {      // rows co + kr of tiles (kt, p0 + h), all 64 columns -> [kr][BTLD]
        const int kr = t >> 5, n32 = t & 31;
        lp_cp16(buf + kr * CF::BTLD + 2 * n32,
                T(kt, p0 + (n32 >> 4)) + (long long)(co + kr) * tp + 2 * (n32 & 15));
      }
    }
    if (act_a) {   // A: columns co .. of the warp's tile T(i, kt), KS / 2 pieces per lane
      double* a = buf + LP_BSZ + warp * LP_ASZ;
      const double* srcA = T(i, kt) + co;
#pragma unroll
      for (int u = 0; u < KS / 2; ++u) {
        const int t = lane + 32 * u, r = t / (KS / 2), c16 = t % (KS / 2);
        lp_cp16(a + r * CF::ALD + 2 * c16, srcA + (long long)r * tp + 2 * c16);
      }
    }
    asm volatile("cp.async.commit_group;\n");
  };
  // strip accumulation over k tiles [kb, ke); strip row i (-1: idle warp) uses k <= klim only
  auto accumulate = [&](bool chol, int p0, int kb, int ke, int i, int klim, int spw, int part) {
#pragma unroll
    for (int R = 0; R < 4; ++R)
#pragma unroll
      for (int C = 0; C < 8; ++C) acc[R][C][0] = acc[R][C][1] = 0.0;
    const int ns = (ke - kb) * SPT;
    if (ns <= 0) return;
    __syncthreads();   // the ring doubles as the strips' finishing scratch
    BF_T(t_acc0);
    auto mine = [&](int s) { return i >= 0 && kb + s / SPT <= klim && (s % spw) == part; };
#pragma unroll 1
    for (int s = 0; s < LP_STAGES - 1; ++s) {
      if (s < ns) issue(s, chol, p0, kb, mine(s), i);
      else asm volatile("cp.async.commit_group;\n");
    }
#pragma unroll 1
    for (int s = 0; s < ns; ++s) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(LP_STAGES - 2));
      __syncthreads();   // slice s landed for every warp; slice s-1's buffer is free
      if (s + LP_STAGES - 1 < ns) issue(s + LP_STAGES - 1, chol, p0, kb, mine(s + LP_STAGES - 1), i);
      else asm volatile("cp.async.commit_group;\n");
      if (mine(s)) {
        const double* buf = lp_sm + (s % LP_STAGES) * LP_STAGE;
        const double* xs = buf + LP_BSZ + warp * LP_ASZ;
        if (chol) lp_slice<true, CF>(acc, xs, buf, q, k4);
        else lp_slice<false, CF>(acc, xs, buf, q, k4);
      }
    }
    asm volatile("cp.async.wait_group 0;\n");
    __syncthreads();   // the ring is free for the caller (and for the next accumulate)
    if (spw > 1) {     // sum the parts into part 0, in part order, through the ring
      double* red = lp_sm + warp * 2048;
      if (part > 0 && i >= 0)
#pragma unroll
        for (int R = 0; R < 4; ++R)
#pragma unroll
          for (int C = 0; C < 8; ++C) {
            red[((R * 8 + C) * 2 + 0) * 32 + lane] = acc[R][C][0];
            red[((R * 8 + C) * 2 + 1) * 32 + lane] = acc[R][C][1];
          }
      __syncthreads();
      if (part == 0 && i >= 0)
        for (int pp = 1; pp < spw; ++pp) {
          const double* rp = lp_sm + (warp + pp) * 2048;
#pragma unroll
          for (int R = 0; R < 4; ++R)
#pragma unroll
            for (int C = 0; C < 8; ++C) {
              acc[R][C][0] += rp[((R * 8 + C) * 2 + 0) * 32 + lane];
              acc[R][C][1] += rp[((R * 8 + C) * 2 + 1) * 32 + lane];
            }
        }
      __syncthreads();
    }
    BF_T(t_acc1);
    BF_ADD(chol ? 1 : 4, t_acc0, t_acc1);
  };
  // store half h of the strip accumulator (8 x 8 blocks C = 4h .. 4h+3) to a 32 x 32 tile,
  // optionally as base - acc (base may alias Ct: read in full before the stores)
  auto store_half = [&](int h, double* Ct, int ld, const double* base, int ldb) {
    double2 bv[4][4];
#pragma unroll
    for (int R = 0; R < 4; ++R)
#pragma unroll
      for (int C = 0; C < 4; ++C)
        bv[R][C] = base ? *reinterpret_cast<const double2*>(base + (long long)(8 * R + q) * ldb + 8 * C + 2 * k4)
                        : make_double2(0.0, 0.0);
#pragma unroll
    for (int R = 0; R < 4; ++R)
#pragma unroll
      for (int C = 0; C < 4; ++C) {
        const int r = 8 * R + q, c = 8 * C + 2 * k4;
        double v0 = acc[R][4 * h + C][0], v1 = acc[R][4 * h + C][1];
        if (base) {
          v0 = bv[R][C].x - v0;
          v1 = bv[R][C].y - v1;
        }
        *reinterpret_cast<double2*>(Ct + (long long)r * ld + c) = make_double2(v0, v1);
      }
  };
  double t32[4][4][2];   // 32 x 32 tile products (mma_tile)
  // the three tiles every strip of a pair step needs (row-major, LD 36):
  //   Cholesky: L_p0p0^{-1}, L_p0+1,p0, L_p0+1p0+1^{-1} (written by the diagonal-pair warp);
  //   inverse:  W_J0J0, L_J1,J0, W_J1J1 (staged once per pair)
  double* P3 = lp_sm + CF::RING;
  constexpr int PLD = 36, PT = 32 * PLD;
  auto stage3 = [&](const double* t0, int ld0, const double* t1, int ld1, const double* t2, int ld2) {
    // 3 x 1024 elements, 12 per thread per pass, all loads of a pass in flight before its stores
#pragma unroll 1
    for (int x0 = 0; x0 < 3072; x0 += 12 * LP_THREADS) {
      double v[12];
#pragma unroll
      for (int u = 0; u < 12; ++u) {
        const int x = x0 + tid + LP_THREADS * u, w = x >> 10, rr = (x >> 5) & 31, cc = x & 31;
        const double* src = w == 0 ? t0 + (long long)rr * ld0 : w == 1 ? t1 + (long long)rr * ld1
                                                                       : t2 + (long long)rr * ld2;
        v[u] = src[cc];
      }
#pragma unroll
      for (int u = 0; u < 12; ++u) {
        const int x = x0 + tid + LP_THREADS * u, w = x >> 10, rr = (x >> 5) & 31, cc = x & 31;
        P3[w * PT + rr * PLD + cc] = v[u];
      }
    }
  };
  // per-warp 32 x 32 scratch (LD 36) in the slice ring, free between accumulations
  double* S = lp_sm + warp * PT;
  // a finished tile (I, J) of the slot's blocked inverse (src: 32 x 32 row-major, ld lds, shared or
  // global) -- W_IJ inside a diagonal super-block, L_IJ below them -- into the slot: the tile in its
  // lower triangle, its transpose in its upper triangle, both row-contiguous (coalesced both ways)
  double* Gi = Ginv + slot * gi_stride;
  auto emit_w = [&](int I, int J, const double* src, int lds) {
#pragma unroll 4
    for (int rr = 0; rr < 32; ++rr) {
      const int row = 32 * I + rr, col = 32 * J + lane;
      if (row < tau && col <= row) Gi[(long long)row * ldgi + col] = src[rr * lds + lane];
    }
#pragma unroll 4
    for (int rr = 0; rr < 32; ++rr) {   // row 32 J + rr of the upper triangle: W[32 I + lane][32 J + rr]
      const int row = 32 * J + rr, col = 32 * I + lane;
      if (row < tau && col < tau && col > row) Gi[(long long)row * ldgi + col] = src[lane * lds + rr];
    }
  };
  // finish Cholesky strip i of pair p0 from its accumulator
  // acc = sum_{k<p0} L_ik [L_p0,k L_p0+1,k]^T:
  //   L_i,p0 = (G_i,p0 - acc_0) L00^{-T},  L_i,p0+1 = (G_i,p0+1 - acc_1 - L_i,p0 L10^T) L11^{-T}
  auto finish_chol = [&](int i, int p0) {
    store_half(0, S, PLD, T(i, p0), tp);                       // C0
    __syncwarp();
    acc_zero(t32);
    mma_tile<false, true>(t32, S, PLD, P3, PLD, lane, 1.0);    // L_i,p0
    __syncwarp();
    acc_store(t32, S, PLD, lane);
    acc_store(t32, T(i, p0), tp, lane);
    const bool offd = i / sbt != p0 / sbt;   // tile outside the diagonal super-blocks: the slot keeps L
    if (offd) {
      __syncwarp();
      emit_w(i, p0, S, PLD);
    }
    const double* base = T(i, p0 + 1);
#pragma unroll
    for (int R = 0; R < 4; ++R)
#pragma unroll
      for (int C = 0; C < 4; ++C) {
        double2 bv = make_double2(0.0, 0.0);
        bv = *reinterpret_cast<const double2*>(base + (long long)(8 * R + q) * tp + 8 * C + 2 * k4);
        t32[R][C][0] = bv.x - acc[R][4 + C][0];
        t32[R][C][1] = bv.y - acc[R][4 + C][1];
      }
    __syncwarp();
    mma_tile<false, true>(t32, S, PLD, P3 + PT, PLD, lane, -1.0);   // - L_i,p0 L10^T
    __syncwarp();
    acc_store(t32, S, PLD, lane);
    __syncwarp();
    acc_zero(t32);
    mma_tile<false, true>(t32, S, PLD, P3 + 2 * PT, PLD, lane, 1.0);   // L_i,p0+1
    acc_store(t32, T(i, p0 + 1), tp, lane);
    __syncwarp();
    if (offd) {   // (from shared memory: the transposed half reads down columns)
      acc_store(t32, S, PLD, lane);
      __syncwarp();
      emit_w(i, p0 + 1, S, PLD);
      __syncwarp();
    }
  };
  // finish inverse strip I of pair (J0, J1) from acc = [T_I,J0 T_I,J1]:
  //   W_I,J1 = -T_I,J1 W_J1J1,  W_I,J0 = -(T_I,J0 + W_I,J1 L_J1,J0) W_J0J0
  auto finish_inv = [&](int I, int J0) {
    store_half(1, S, PLD, nullptr, 0);                          // T_I,J1
    __syncwarp();
    acc_zero(t32);
    mma_tile<false, false>(t32, S, PLD, P3 + 2 * PT, PLD, lane, -1.0);   // W_I,J1
    __syncwarp();
    acc_store(t32, S, PLD, lane);
    acc_store(t32, T(I, J0 + 1), tp, lane);
    __syncwarp();
    emit_w(I, J0 + 1, S, PLD);
#pragma unroll
    for (int R = 0; R < 4; ++R)
#pragma unroll
      for (int C = 0; C < 4; ++C) {
        t32[R][C][0] = acc[R][C][0];
        t32[R][C][1] = acc[R][C][1];
      }
    __syncwarp();
    mma_tile<false, false>(t32, S, PLD, P3 + PT, PLD, lane, 1.0);   // T_I,J0 + W_I,J1 L_J1,J0
    __syncwarp();
    acc_store(t32, S, PLD, lane);
    __syncwarp();
    acc_zero(t32);
    mma_tile<false, false>(t32, S, PLD, P3, PLD, lane, -1.0);       // W_I,J0
    acc_store(t32, T(I, J0), tp, lane);
    __syncwarp();
    acc_store(t32, S, PLD, lane);
    __syncwarp();
    emit_w(I, J0, S, PLD);
    __syncwarp();
  };

  // ---- a5: Cholesky G = L L^T, block-column pairs.  Round 0 holds the diagonal pair's rows: their
  // strips are stored as C, warp 0 factors the pair on chip (C00, L10 and C11 in the pair-tile
  // buffer, which ends up holding L00^{-1}, L10, L11^{-1} for the panel), and every other strip is
  // finished from its register accumulator (no C round trip, no panel pass).
  BF_T(t_c0);
  for (int p0 = 0; p0 < Tc; p0 += 2) {
    if (stopped()) return false;
    const int nstrip = Tc - p0, rounds = (nstrip + LP_WARPS - 1) / LP_WARPS;
    for (int rd = 0; rd < rounds; ++rd) {
      int spw, part;
      const int j = split(min(LP_WARPS, nstrip - rd * LP_WARPS), spw, part);
      const int i = j < 0 ? -1 : p0 + rd * LP_WARPS + j;
      const bool own = i >= 0 && part == 0;   // holds the strip's summed accumulator
      accumulate(true, p0, 0, p0, i, Tc, spw, part);
      if (rd == 0) {
        if (own && i == p0) store_half(0, T(i, p0), tp, T(i, p0), tp);
        if (own && i == p0 + 1) {
          store_half(0, T(i, p0), tp, T(i, p0), tp);
          store_half(1, T(i, p0 + 1), tp, T(i, p0 + 1), tp);
        }
        __syncthreads();
        BF_T(t_d0);
        {   // diagonal pair (64 x 64), all warps, on chip: right-looking with the unscaled rank-1
            // update M_rc -= M_rj M_cj / M_jj, one barrier per column; column j of L to Lm
          double* M = lp_sm;                 // 64 x 65 (the ring is free here)
          double* Lm = lp_sm + 64 * 65;      // 64 x 65
#pragma unroll 1
          for (int x0 = 0; x0 < 4096; x0 += 16 * LP_THREADS) {
            double v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              const int x = x0 + tid + LP_THREADS * u, r = x >> 6, c = x & 63;
              v[u] = (c <= r) ? T(p0 + (r >> 5), p0 + (c >> 5))[(long long)(r & 31) * tp + (c & 31)] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              const int x = x0 + tid + LP_THREADS * u, r = x >> 6, c = x & 63;
              M[r * 65 + c] = v[u];
              Lm[r * 65 + c] = 0.0;
            }
          }
          __syncthreads();
          // update: row j + 1 + ur, columns j + 1 + uc + UC t
          constexpr int UC = LP_THREADS / 64;
          const int ur = tid / UC, uc = tid % UC;
#pragma unroll 1
          for (int j = 0; j < 64; ++j) {
            double d = M[j * 65 + j];
            if (!(d > 0.0) || !isfinite(d)) {
              if (tid == 0) s_bad = 1;
              d = 1.0;
            }
            if (tid < 64 && tid >= j) {
              const double rs = 1.0 / sqrt(d);
              Lm[tid * 65 + j] = tid == j ? d * rs : M[tid * 65 + j] * rs;
            }
            const int r = j + 1 + ur;
            if (r < 64) {
              const double f = M[r * 65 + j] / d;
#pragma unroll 4
              for (int c = j + 1 + uc; c <= r; c += UC) M[r * 65 + c] -= f * M[c * 65 + j];
            }
            __syncthreads();
          }
          // L00^{-1} -> P3[0], L11^{-1} -> P3[2]: column jc of block b by 4 threads (partial sums
          // over k = jc + part (mod 4), shuffle-reduced), rows in order
#pragma unroll 1
          for (int c0 = 0; c0 < 64; c0 += LP_THREADS / 4) {
            const int col = c0 + (tid >> 2), part = tid & 3, b = col >> 5, jc = col & 31;
            double* Di = P3 + (b ? 2 * PT : 0);
            const double* Lb = Lm + (32 * b) * 65 + 32 * b;
#pragma unroll 1
            for (int i = 0; i < 32; ++i) {
              double t = 0.0;
              for (int k = jc + part; k < i; k += 4) t += Lb[i * 65 + k] * Di[k * PLD + jc];
              t += __shfl_xor_sync(0xffffffffu, t, 1);
              t += __shfl_xor_sync(0xffffffffu, t, 2);
              const double x = i < jc ? 0.0 : ((i == jc ? 1.0 : 0.0) - t) / Lb[i * 65 + i];
              __syncwarp();
              if (part == 0) Di[i * PLD + jc] = x;
              __syncwarp();
            }
          }
          __syncthreads();
          // L tiles to the work matrix, L10 to P3[1], the inverses to dinv
#pragma unroll 4
          for (int x = tid; x < 64 * 64; x += LP_THREADS) {
            const int r = x >> 6, c = x & 63;
            if (c < 32 || r >= 32) {   // tiles (p0,p0), (p0+1,p0), (p0+1,p0+1)
              const double lv = c <= r ? Lm[r * 65 + c] : 0.0;
              T(p0 + (r >> 5), p0 + (c >> 5))[(long long)(r & 31) * tp + (c & 31)] = lv;
              if (r >= 32 && c < 32) P3[PT + (r - 32) * PLD + c] = lv;
            }
          }
          for (int x = tid; x < 2 * 1024; x += LP_THREADS) {
            const int b = x >> 10, rr = (x >> 5) & 31, cc = x & 31;
            dinv[(long long)(p0 + b) * 1024 + rr * 32 + cc] = P3[(b ? 2 * PT : 0) + rr * PLD + cc];
          }
        }
        __syncthreads();
        BF_T(t_d1);
        BF_ADD(2, t_d0, t_d1);
      }
      if (own && i >= p0 + 2) finish_chol(i, p0);
    }
  }
  __syncthreads();
  BF_T(t_c1);
  BF_ADD(3, t_c0, t_c1);
  if (s_bad) {
    __syncthreads();   // (every thread has read s_bad before the next slot resets it)
    if (tid == 0) {
      __threadfence();
      flags[slot] = 1;
    }
    return true;
  }
  // ---- W = L^{-1}, block-column pairs from the last
  for (int J0 = Tc - 2; J0 >= 0; J0 -= 2) {
    if (stopped()) return false;
    const int E = min(Tc, (J0 / sbt + 1) * sbt);   // end of J0's diagonal super-block (tiles)
    const int J1 = J0 + 1, nstrip = E - 1 - J1;
    const int rounds = (nstrip + LP_WARPS - 1) / LP_WARPS;
    if (rounds > 0) {
      __syncthreads();
      stage3(dinv + (long long)J0 * 1024, 32, T(J1, J0), tp, dinv + (long long)J1 * 1024, 32);
      __syncthreads();
    }
    for (int rd = 0; rd < rounds; ++rd) {   // highest strips first
      int spw, part;
      const int j = split(min(LP_WARPS, nstrip - rd * LP_WARPS), spw, part);
      const int I = j < 0 ? -1 : E - 1 - (rd * LP_WARPS + j);
      const int kend = E - rd * LP_WARPS;   // rows of this round are <= kend - 1
      accumulate(false, J0, J1 + 1, kend, I, I, spw, part);
      if (I > J1 && part == 0) finish_inv(I, J0);
    }
    __syncthreads();
    BF_T(t_i0);
    if (rounds == 0) {   // the pair tiles (staged above for pairs with strips)
      __syncthreads();
      stage3(dinv + (long long)J0 * 1024, 32, T(J1, J0), tp, dinv + (long long)J1 * 1024, 32);
      __syncthreads();
    }
    {   // diagonal pair: W_J1,J0 = -W_J1J1 L_J1,J0 W_J0J0, warp w < 4 owning rows 8w .. 8w+7
      double* X = lp_sm;   // 32 x 36 (the ring is free here)
      if (warp < 4) {
        acc_zero(t32);
        mma_tile<false, false>(t32, P3 + 2 * PT, PLD, P3 + PT, PLD, lane, 1.0, warp, 1);
        acc_store(t32, X, PLD, lane, warp, 1);
      }
      __syncthreads();
      if (warp < 4) {
        acc_zero(t32);
        mma_tile<false, false>(t32, X, PLD, P3, PLD, lane, -1.0, warp, 1);
        acc_store(t32, T(J1, J0), tp, lane, warp, 1);   // W_J1,J0
      }
      for (int qd = tid; qd < 1024; qd += LP_THREADS) {
        T(J0, J0)[(long long)(qd >> 5) * tp + (qd & 31)] = P3[(qd >> 5) * PLD + (qd & 31)];
        T(J1, J1)[(long long)(qd >> 5) * tp + (qd & 31)] = P3[2 * PT + (qd >> 5) * PLD + (qd & 31)];
      }
    }
    __syncthreads();
    if (warp == 0) emit_w(J1, J0, T(J1, J0), tp);                 // W_J1,J0
    else if (warp == 1) emit_w(J0, J0, P3, PLD);                  // W_J0J0
    else if (warp == 2) emit_w(J1, J1, P3 + 2 * PT, PLD);         // W_J1J1
    BF_T(t_i1);
    BF_ADD(6, t_i0, t_i1);
  }
  BF_T(t_w0);
  BF_ADD(5, t_c1, t_w0);
  BF_T(t_w1);
  BF_ADD(7, t_w0, t_w1);
  __syncthreads();   // every W tile of the slot written (emit_w) before the flag
  if (tid == 0) {
    __threadfence();
    flags[slot] = 0;
  }
  return true;
}

// The batched factorisation: one slot per CTA (claim == null: slot = blockIdx.x), or slots claimed
// from claim[0] by CTAs that run on at most max_sms distinct SMs, so that the overlapped
// pipeline's factorisation leaves num_sms - max_sms SMs to the concurrent iteration kernel even
// when the GPU dispatches the factorisation first (claim[1]: CTAs started, claim[2]: CTAs allowed,
// claim[3]: SMs taken, claim[4 + smid]: 0 unseen, 1 allowed, 2 refused, 3 deciding; a refused CTA
// that starts last while none was allowed works anyway, so every launch completes its slots).
template <int NW>
__global__ void __launch_bounds__(LpCfg<NW>::THREADS, LpCfg<NW>::CTAS)
k_bfactor_lp(FactorSrc src, DevSketch skb, double* __restrict__ Ginv, long long ldgi,
             long long gi_stride, double* work, long long work_stride, int* __restrict__ flags,
             const Ctrl* ctrl, int nslots, int* claim, int max_sms, int sbt) {
  __shared__ int s_bad, s_stop, s_slot;
  const int tid = threadIdx.x;
  if (!claim) {
    lp_factor_slot<NW>(src, skb, Ginv, ldgi, gi_stride, work, work_stride, flags, ctrl, blockIdx.x,
                       sbt, s_bad, s_stop);
    return;
  }
  if (tid == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    int* st = claim + 4 + (sm & 255);
    int v = atomicCAS(st, 0, 3);
    if (v == 0) {   // first CTA on this SM: take it if the budget allows
      v = atomicAdd(claim + 3, 1) < max_sms ? 1 : 2;
      atomicExch(st, v);
    }
    while (v == 3) v = *reinterpret_cast<volatile int*>(st);
    if (v == 1) atomicAdd(claim + 2, 1);
    __threadfence();
    const int started = atomicAdd(claim + 1, 1);
    if (v != 1 && started == (int)gridDim.x - 1 && atomicAdd(claim + 2, 0) == 0) v = 1;
    s_slot = v == 1 ? 0 : -1;
  }
  __syncthreads();
  if (s_slot < 0) return;
  for (;;) {
    __syncthreads();   // (s_slot read by every thread of the previous round)
    if (tid == 0) s_slot = atomicAdd(claim, 1);
    __syncthreads();
    const int slot = s_slot;
    if (slot >= nslots) return;
    if (!lp_factor_slot<NW>(src, skb, Ginv, ldgi, gi_stride, work, work_stride, flags, ctrl, slot,
                            sbt, s_bad, s_stop))
      return;
  }
}

}  // namespace

int bfactor_max_tau() { return BB_MAXTAU; }

#ifdef RS_BF_PHASES
extern "C" int rs_debug_bf_phases(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, g_bf_phase, sizeof(g_bf_phase)) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_bf_phase, z, sizeof(z));
  }
  return 0;
}
#endif

size_t bfactor_work_elems(int tau) {
  if (tau <= BF_MAXTAU) return 0;
  const long long tp = bb_tp(tau);
  // work matrix, Tc L_pp^{-1} tiles, then Tc tiles (right-looking T_I) or 2 per warp (left-looking)
  return (size_t)(tp * tp + (tp / 32) * 1024 + std::max<long long>(tp / 32, 16) * 1024);
}

cudaError_t bfactor_init() {
  const int ap_smem = AG_MAXTAU * 8 + (AG_MAXTAU + 1 + AP_MAXFUSE) * 4;
  cudaError_t e = cudaFuncSetAttribute(k_apply_rows<AP_FULL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, ap_smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_apply_rows<AP_LOWER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             ap_smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_apply_rows<AP_UPPER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             ap_smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_bf_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GA_SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_bfactor_lp<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)LpCfg<8>::SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_bfactor_lp<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)LpCfg<4>::SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_bfactor_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)bf_smem(BF_MAXTAU));
}

cudaError_t launch_bfactor(const FactorSrc& src, const DevSketch& skb, int nslots, double* Ginv,
                           long long ldgi, long long gi_stride, int* flags, double* work,
                           const Ctrl* ctrl, cudaStream_t st, bool dual, const BfClaim* claim,
                           int sb) {
  if (skb.tau > BB_MAXTAU || nslots < 1) return cudaErrorInvalidValue;
  if (skb.tau > BF_MAXTAU) {
    if (!work) return cudaErrorInvalidValue;
    const int tp = bb_tp(skb.tau);
    const long long ws = (long long)bfactor_work_elems(skb.tau);
    k_bf_gather<<<dim3((unsigned)((tp + GA_WARPS - 1) / GA_WARPS), (unsigned)nslots), GA_WARPS * 32,
                  std::min(GA_SMEM, (size_t)(skb.tau + 1 + skb.len) * 4), st>>>(src, skb, work, ws, ctrl);
    int* cw = claim ? claim->words : nullptr;
    const int max_sms = claim ? claim->max_sms : 0;
    const int cps = dual ? LpCfg<4>::CTAS : LpCfg<8>::CTAS;
    // super-block width in 32-wide tiles (a whole number of 64-wide pairs); >= tp: full inverse
    if (sb > 0 && sb % 64) return cudaErrorInvalidValue;
    const int sbt = sb > 0 && sb < tp ? sb / 32 : tp / 32;
    // (claimed slots: CTAs on every SM, so that those refused by the SM budget leave enough workers)
    const unsigned grid = (unsigned)(claim ? cps * claim->num_sms : nslots);
    if (cw) {
      const cudaError_t e = cudaMemsetAsync(cw, 0, BF_CLAIM_WORDS * sizeof(int), st);
      if (e != cudaSuccess) return e;
    }
    if (dual)
      k_bfactor_lp<4><<<grid, LpCfg<4>::THREADS, LpCfg<4>::SMEM, st>>>(
          src, skb, Ginv, ldgi, gi_stride, work, ws, flags, ctrl, nslots, cw, max_sms, sbt);
    else
      k_bfactor_lp<8><<<grid, LpCfg<8>::THREADS, LpCfg<8>::SMEM, st>>>(
          src, skb, Ginv, ldgi, gi_stride, work, ws, flags, ctrl, nslots, cw, max_sms, sbt);
    return cudaGetLastError();
  }
  k_bfactor_small<<<nslots, BF_THREADS, bf_smem(skb.tau), st>>>(src, skb, Ginv, ldgi, gi_stride,
                                                                 flags, ctrl);
  return cudaGetLastError();
}

cudaError_t launch_apply_ginv(const double* Ginv, long long ldgi, const DevSketch& sk,
                              const int* flag, const double* r, double* gbuf, double* delta,
                              double* sdelta, Ctrl* ctrl, cudaStream_t st, bool first,
                              const double* pfA, long long pf_lda, long long pf_m) {
  // L2 prefetch of the sketched rows of A only while they fit comfortably in the 126 MB L2
  if (!pfA || (double)sk.len * pf_m * 8.0 > 48e6) pfA = nullptr;
  const unsigned pf_bytes = (unsigned)(((pf_m * 8) + 15) / 16 * 16);
  if (sk.tau > AG_MAXTAU) return cudaErrorInvalidValue;
  // few entries per bucket (subsample, SubCount): g = S^T r is formed inside the first GEMV kernel
  const bool fuse = sk.len <= 8 * sk.tau && sk.len <= AP_MAXFUSE;
  const double* gv = nullptr;
  if (!fuse) {
    k_sketch_g<<<(unsigned)((sk.tau + AG_WARPS - 1) / AG_WARPS), AG_WARPS * 32, 0, st>>>(
        sk, flag, r, gbuf, ctrl);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    gv = gbuf;
    first = false;   // k_sketch_g is the ordinary launch of the chain
  }
  // the first kernel of a group follows the factorisation that wrote the slot: ordinary launch
  auto launch = [&](auto kern, const double* xin, double* out, const double* pf) {
    const dim3 grid((unsigned)((sk.tau + AP_ROWS - 1) / AP_ROWS)), blk(AG_WARPS * 32);
    const size_t smem = (size_t)sk.tau * 8 + (xin ? 0 : (size_t)(sk.tau + 1 + sk.len) * 4);
    if (first) {
      kern<<<grid, blk, smem, st>>>(Ginv, ldgi, sk, flag, xin, r, out, sdelta, ctrl, pf, pf_lda, pf_bytes);
      return cudaGetLastError();
    }
    return launch_pdl(kern, grid, blk, smem, st, Ginv, ldgi, sk, flag, xin, r, out, sdelta, ctrl, pf,
                      pf_lda, pf_bytes);
  };
  if (sk.tau > BF_MAXTAU) {   // slot holds W = L^{-1} (lower) and W^T (upper): delta = W^T (W g)
    double* tv = gbuf + sk.tau;
    const cudaError_t e = launch(k_apply_rows<AP_LOWER>, gv, tv, pfA);
    if (e != cudaSuccess) return e;
    first = false;
    return launch(k_apply_rows<AP_UPPER>, (const double*)tv, delta, (const double*)nullptr);
  }
  return launch(k_apply_rows<AP_FULL>, gv, delta, pfA);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("RS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace rs
