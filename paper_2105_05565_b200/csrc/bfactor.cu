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
                                         const double* B, int ldb, int lane, double sign) {
  const int q = lane >> 2, k4 = lane & 3;
#pragma unroll 4
  for (int K = 0; K < 8; ++K) {
    double a[4], b[4];
#pragma unroll
    for (int R = 0; R < 4; ++R) {
      const int r = 8 * R + q, k = 4 * K + k4;
      a[R] = sign * (TA ? A[(long long)k * lda + r] : A[(long long)r * lda + k]);
    }
#pragma unroll
    for (int C = 0; C < 4; ++C) {
      const int c = 8 * C + q, k = 4 * K + k4;
      b[C] = TB ? B[(long long)c * ldb + k] : B[(long long)k * ldb + c];
    }
#pragma unroll
    for (int R = 0; R < 4; ++R)
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
__device__ __forceinline__ void acc_store(const double (&acc)[4][4][2], double* Ct, int ld, int lane) {
  const int q = lane >> 2, k4 = lane & 3;
#pragma unroll
  for (int R = 0; R < 4; ++R)
#pragma unroll
    for (int C = 0; C < 4; ++C) {
      *reinterpret_cast<double2*>(Ct + (long long)(8 * R + q) * ld + 8 * C + 2 * k4) =
          make_double2(acc[R][C][0], acc[R][C][1]);
    }
}

// Diagonal tile p (warp 0): L_pp in registers (lane i = row i, right-looking), written back over
// the tile; L_pp^{-1} (lane j = column j, forward substitution) written to Di (32 x 32 row-major,
// zeros above the diagonal).  Returns false if a pivot was <= 0 or non-finite.
__device__ __noinline__ bool diag_factor(double* D, int ld, double* Di, double (*sL)[33], int lane) {
  bool bad = false;
  double v[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = k <= lane ? D[(long long)lane * ld + k] : 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    double d = __shfl_sync(0xffffffffu, v[j], j);
    if (!(d > 0.0) || !isfinite(d)) {
      bad = true;
      d = 1.0;
    }
    const double ljj = sqrt(d), inv = 1.0 / ljj;
    if (lane == j) v[j] = ljj;
    else if (lane > j) v[j] *= inv;
    const double lij = lane > j ? v[j] : 0.0;
#pragma unroll
    for (int k = j + 1; k < 32; ++k) v[k] -= lij * __shfl_sync(0xffffffffu, lij, k);
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double x = k <= lane ? v[k] : 0.0;
    D[(long long)lane * ld + k] = x;
    sL[lane][k] = x;
  }
  __syncwarp();
#pragma unroll 1
  for (int i = 0; i < 32; ++i) {   // column `lane` of L^{-1}: x_i, reusing v as x
    double s = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k)
      if (k < i) s -= sL[i][k] * Di[k * 32 + lane];
    Di[i * 32 + lane] = i < lane ? 0.0 : s / sL[i][i];
    __syncwarp();
  }
  return bad;
}

__global__ void __launch_bounds__(BB_THREADS, 1)
k_bfactor_big(FactorSrc src, DevSketch skb, double* __restrict__ Ginv, long long ldgi,
              long long gi_stride, double* work, long long work_stride, int* __restrict__ flags,
              const Ctrl* ctrl) {
  if (slot_unused(ctrl, blockIdx.x)) return;
  __shared__ double sL[32][33];
  __shared__ int s_bad;
  const int slot = blockIdx.x;
  const DevSketch sk = skb.at(slot);
  const int tau = sk.tau, tp = bb_tp(tau), Tc = tp / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Wm = work + slot * work_stride;           // tp x tp, row-major
  double* dinv = Wm + (long long)tp * tp;           // Tc tiles 32 x 32 (L_pp^{-1})
  double* tmp = dinv + (long long)Tc * 1024;        // Tc tiles (T_I)
  auto T = [&](int I, int J) { return Wm + (long long)(32 * I) * tp + 32 * J; };
  if (tid == 0) s_bad = 0;

  // ---- a4: lower triangle of G (R3 empty-bucket rule), identity on the padding
  const double* ASt = src.ASt ? src.ASt + slot * src.as_stride : nullptr;
  const double* Gram = src.Gram ? src.Gram + slot * src.gram_stride : nullptr;
  for (int a = warp; a < tp; a += BB_WARPS) {
    const int a32 = a & ~31;
    const int e0 = a < tau ? sk.bptr[a] : 0, e1 = a < tau ? sk.bptr[a + 1] : 0;
    for (int c = lane; c < a32 + 32; c += 32) {   // every lower tile of row a
      double v = 0.0;
      if (a >= tau || c >= tau || c > a) {
        v = (a == c) ? 1.0 : 0.0;
      } else if (Gram) {
        v = Gram[(long long)a * src.ld_gram + c];
        if (a == c) v += src.lambda * (double)(e1 - e0);
      } else if (!ASt) {
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
      if (a < tau && c < tau && c <= a && (e0 == e1 || sk.bptr[c] == sk.bptr[c + 1]))
        v = (a == c) ? 1.0 : 0.0;
      Wm[(long long)a * tp + c] = v;
    }
  }
  __syncthreads();

  double acc[4][4][2];
  // ---- a5: Cholesky G = L L^T
  for (int p = 0; p < Tc; ++p) {
    if (warp == 0) {
      const bool bad = diag_factor(T(p, p), tp, dinv + (long long)p * 1024, sL, lane);
      if (bad && lane == 0) s_bad = 1;
    }
    __syncthreads();
    // panel: L_ip = G_ip (L_pp^{-1})^T, in place (the warp reads its whole tile before storing)
    for (int i = p + 1 + warp; i < Tc; i += BB_WARPS) {
      acc_zero(acc);
      mma_tile<false, true>(acc, T(i, p), tp, dinv + (long long)p * 1024, 32, lane, 1.0);
      acc_store(acc, T(i, p), tp, lane);
    }
    __syncthreads();
    // trailing: G_ij -= L_ip L_jp^T, p < j <= i
    {
      const int nt = Tc - 1 - p, ntiles = nt * (nt + 1) / 2;
      for (int t = warp; t < ntiles; t += BB_WARPS) {
        int Ii, Jj;
        tri_decode(t, Ii, Jj);
        const int i = p + 1 + Ii, j = p + 1 + Jj;
        acc_load(acc, T(i, j), tp, lane);
        mma_tile<false, true>(acc, T(i, p), tp, T(j, p), tp, lane, -1.0);
        acc_store(acc, T(i, j), tp, lane);
      }
    }
    __syncthreads();
  }
  if (s_bad) {
    if (tid == 0) flags[slot] = 1;
    return;
  }
  // ---- W = L^{-1}, block columns J = Tc-1 .. 0 (W_IK final for K > J; L_KJ still L)
  for (int J = Tc - 1; J >= 0; --J) {
    for (int I = J + 1 + warp; I < Tc; I += BB_WARPS) {
      acc_zero(acc);
      for (int K = J + 1; K <= I; ++K) mma_tile<false, false>(acc, T(I, K), tp, T(K, J), tp, lane, 1.0);
      acc_store(acc, tmp + (long long)I * 1024, 32, lane);
    }
    __syncthreads();
    // W_IJ = -T_I W_JJ over L_IJ;  W_JJ = L_JJ^{-1} over L_JJ
    for (int I = J + 1 + warp; I < Tc; I += BB_WARPS) {
      acc_zero(acc);
      mma_tile<false, false>(acc, tmp + (long long)I * 1024, 32, dinv + (long long)J * 1024, 32, lane,
                             -1.0);
      acc_store(acc, T(I, J), tp, lane);
    }
    if (warp == BB_WARPS - 1) {
      const double* Wjj = dinv + (long long)J * 1024;
      double* D = T(J, J);
      for (int q = lane; q < 1024; q += 32) D[(long long)(q >> 5) * tp + (q & 31)] = Wjj[q];
    }
    __syncthreads();
  }
  // ---- the slot receives W = L^{-1} in its lower triangle and W^T in its upper triangle (both
  // row-contiguous): G^{-1} = W^T W is applied as two triangular GEMVs per iteration (k_apply_w,
  // k_apply_wt), which saves the W^T W product (a third of the factorisation's flops)
  double* Gi = Ginv + slot * gi_stride;
  for (int row = warp; row < tau; row += BB_WARPS)
    for (int col = lane; col <= row; col += 32) {
      const double x = Wm[(long long)row * tp + col];
      Gi[(long long)row * ldgi + col] = x;
      if (col < row) Gi[(long long)col * ldgi + row] = x;
    }
  if (tid == 0) flags[slot] = 0;
}

// -------------------------------------------------------------------------------------------------
// Left-looking variant (default for tau > 224): block columns are processed in PAIRS (64 wide), and
// the operand every strip of a step shares -- rows p0, p0+1 of L (Cholesky) or block columns J0, J1
// of L (inverse) -- is staged in shared memory in chunks of LP_KC tile pairs (cp.async, double
// buffered).  Each warp accumulates a 32 x 64 strip in registers (acc[4][8][2]) from its own row
// tiles read once per PAIR of block columns, so global traffic is about Tc^3/12 tiles per phase
// (the right-looking kernel above re-reads and rewrites the trailing matrix every 32 columns).
//   Cholesky, pair p0 = 2P:  [C_i,p0 C_i,p0+1] = [G_i,p0 G_i,p0+1] - sum_{k<p0} L_ik [L_p0,k L_p0+1,k]^T
//     diagonal pair (warp 0): L00 = chol(C00), L10 = C10 L00^-T, L11 = chol(C11 - L10 L10^T)
//     strips i > p0+1: L_i,p0 = C_i,p0 L00^-T, L_i,p0+1 = (C_i,p0+1 - L_i,p0 L10^T) L11^-T
//   Inverse W = L^-1, pair (J0, J1 = J0+1) from the last: strips I > J1 (highest first, so that a
//   round never stages a row an earlier round has overwritten):
//     [T_I,J0 T_I,J1] = sum_{K=J1+1..I} W_IK [L_K,J0 L_K,J1]
//     W_I,J1 = -T_I,J1 W_J1J1,  W_I,J0 = -(T_I,J0 + W_I,J1 L_J1,J0) W_J0J0
//     diagonal pair: W_J1,J0 = -W_J1J1 L_J1,J0 W_J0J0
constexpr int LP_WARPS = 8;                     // 255 registers: acc[4][8][2] per lane
constexpr int LP_THREADS = LP_WARPS * 32;
constexpr int LP_KC = 4;                        // k tiles per staged chunk
constexpr int LP_LD = 36;                       // staged tile row stride (conflict-free fragments)
constexpr int LP_TILE = 32 * LP_LD;
constexpr int LP_CHUNK = 2 * LP_KC * LP_TILE;   // doubles per chunk buffer
constexpr size_t LP_SMEM = 2 * LP_CHUNK * sizeof(double);

__device__ __forceinline__ void lp_cp16(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

__global__ void __launch_bounds__(LP_THREADS, 1)
k_bfactor_lp(FactorSrc src, DevSketch skb, double* __restrict__ Ginv, long long ldgi,
             long long gi_stride, double* work, long long work_stride, int* __restrict__ flags,
             const Ctrl* ctrl) {
  if (slot_unused(ctrl, blockIdx.x)) return;
  extern __shared__ __align__(16) double lp_sm[];   // 2 chunk buffers (the a4 gather: sketch)
  __shared__ double sL[32][33];
  __shared__ int s_bad;
  const int slot = blockIdx.x;
  const DevSketch sk = skb.at(slot);
  const int tau = sk.tau, tp = bb_tp(tau), Tc = tp / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane >> 2, k4 = lane & 3;
  double* Wm = work + slot * work_stride;           // tp x tp, row-major
  double* dinv = Wm + (long long)tp * tp;           // Tc tiles 32 x 32 (L_pp^{-1})
  double* scr = dinv + (long long)Tc * 1024;        // 2 tiles per warp
  auto T = [&](int I, int J) { return Wm + (long long)(32 * I) * tp + 32 * J; };
  if (tid == 0) s_bad = 0;

  // ---- a4: lower triangle of G (R3 empty-bucket rule), identity on the padding.  From explicit A
  // with the slot's sketch staged in the (not yet used) chunk buffers: coord_e (sign folded in as
  // bit complement) and bptr, so each element costs one independent gather of A.
  const double* ASt = src.ASt ? src.ASt + slot * src.as_stride : nullptr;
  const double* Gram = src.Gram ? src.Gram + slot * src.gram_stride : nullptr;
  int* s_bp = reinterpret_cast<int*>(lp_sm);
  int* s_ce = s_bp + tau + 1;
  const bool staged = !Gram && !ASt && (size_t)(tau + 1 + sk.len) * 4 <= LP_SMEM;
  if (staged) {
    for (int b = tid; b <= tau; b += LP_THREADS) s_bp[b] = sk.bptr[b];
    for (int e = tid; e < sk.len; e += LP_THREADS) s_ce[e] = sk.sign[e] > 0 ? sk.coord[e] : ~sk.coord[e];
    __syncthreads();
  }
  for (int a = warp; a < tp; a += LP_WARPS) {
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
  __syncthreads();

  // chunk staging: tiles (h, kk), h = 0, 1, kk < LP_KC; Cholesky: T(p0 + h, k), inverse: T(k, p0 + h)
  auto stage = [&](int buf, bool chol, int p0, int k0, int kend) {
    double* dst = lp_sm + buf * LP_CHUNK;
    for (int t = tid; t < 2 * LP_KC * 32 * 16; t += LP_THREADS) {   // 16-byte pieces
      const int tile = t >> 9, rr = (t >> 4) & 31, c16 = t & 15;
      const int h = tile / LP_KC, kk = tile % LP_KC, k = k0 + kk;
      if (k >= kend) continue;
      const double* srcp = chol ? T(p0 + h, k) : T(k, p0 + h);
      lp_cp16(dst + tile * LP_TILE + rr * LP_LD + 2 * c16, srcp + (long long)rr * tp + 2 * c16);
    }
    asm volatile("cp.async.commit_group;\n");
  };
  // strip accumulation over staged chunks [kb, ke); strip row i uses k <= klim only
  double acc[4][8][2];
  auto accumulate = [&](bool chol, int p0, int kb, int ke, int i, int klim) {
#pragma unroll
    for (int R = 0; R < 4; ++R)
#pragma unroll
      for (int C = 0; C < 8; ++C) acc[R][C][0] = acc[R][C][1] = 0.0;
    const int nch = (ke - kb + LP_KC - 1) / LP_KC;
    if (nch > 0) stage(0, chol, p0, kb, ke);
    for (int c = 0; c < nch; ++c) {
      if (c + 1 < nch) stage((c + 1) & 1, chol, p0, kb + (c + 1) * LP_KC, ke);
      else asm volatile("cp.async.commit_group;\n");
      asm volatile("cp.async.wait_group 1;\n");
      __syncthreads();
      const double* ys = lp_sm + (c & 1) * LP_CHUNK;
      if (i >= 0) {
        for (int kk = 0; kk < LP_KC; ++kk) {
          const int k = kb + c * LP_KC + kk;
          if (k >= ke || k > klim) break;
          const double* X = T(i, k);
          if (k + 1 < ke && k + 1 <= klim) {   // next tile of the strip row into L1 (2 lines per row)
            const double* nx = X + 32 + (long long)lane * tp;
            asm volatile("prefetch.global.L1 [%0];\n" ::"l"(nx));
            asm volatile("prefetch.global.L1 [%0];\n" ::"l"(nx + 16));
          }
          const double* y0 = ys + kk * LP_TILE;
          const double* y1 = ys + (LP_KC + kk) * LP_TILE;
#pragma unroll 2
          for (int K = 0; K < 8; ++K) {
            double a[4];
#pragma unroll
            for (int R = 0; R < 4; ++R) a[R] = X[(long long)(8 * R + q) * tp + 4 * K + k4];
#pragma unroll
            for (int C = 0; C < 8; ++C) {
              const double* y = C < 4 ? y0 : y1;
              const int n = 8 * (C & 3) + q, kq = 4 * K + k4;
              const double b = chol ? y[n * LP_LD + kq] : y[kq * LP_LD + n];
#pragma unroll
              for (int R = 0; R < 4; ++R) dmma(acc[R][C], a[R], b);
            }
          }
        }
      }
      __syncthreads();
    }
  };
  // store half h of the strip accumulator (8 x 8 blocks C = 4h .. 4h+3) to a 32 x 32 tile,
  // optionally as base - acc
  auto store_half = [&](int h, double* Ct, int ld, const double* base, int ldb) {
    // base (may alias Ct) is read in full before the first store: one batch of 16 double2 loads
    // instead of 16 load -> store round trips
    double2 bv[4][4];
#pragma unroll
    for (int R = 0; R < 4; ++R)
#pragma unroll
      for (int C = 0; C < 4; ++C)
        bv[R][C] = base ? *reinterpret_cast<const double2*>(base + (long long)(8 * R + q) * ldb +
                                                            8 * C + 2 * k4)
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

  // ---- a5: Cholesky G = L L^T, block-column pairs
  for (int p0 = 0; p0 < Tc; p0 += 2) {
    const int nstrip = Tc - p0, rounds = (nstrip + LP_WARPS - 1) / LP_WARPS;
    for (int rd = 0; rd < rounds; ++rd) {
      const int i = p0 + rd * LP_WARPS + warp;
      accumulate(true, p0, 0, p0, i < Tc ? i : -1, Tc);
      if (i < Tc) {
        store_half(0, T(i, p0), tp, T(i, p0), tp);
        if (i > p0) store_half(1, T(i, p0 + 1), tp, T(i, p0 + 1), tp);
      }
    }
    __syncthreads();
    if (warp == 0) {   // diagonal pair
      bool bad = diag_factor(T(p0, p0), tp, dinv + (long long)p0 * 1024, sL, lane);
      __syncwarp();
      acc_zero(t32);
      mma_tile<false, true>(t32, T(p0 + 1, p0), tp, dinv + (long long)p0 * 1024, 32, lane, 1.0);
      __syncwarp();
      acc_store(t32, T(p0 + 1, p0), tp, lane);   // L10
      __syncwarp();
      acc_load(t32, T(p0 + 1, p0 + 1), tp, lane);
      mma_tile<false, true>(t32, T(p0 + 1, p0), tp, T(p0 + 1, p0), tp, lane, -1.0);
      __syncwarp();
      acc_store(t32, T(p0 + 1, p0 + 1), tp, lane);
      __syncwarp();
      bad |= diag_factor(T(p0 + 1, p0 + 1), tp, dinv + (long long)(p0 + 1) * 1024, sL, lane);
      if (bad && lane == 0) s_bad = 1;
    }
    __syncthreads();
    for (int i = p0 + 2 + warp; i < Tc; i += LP_WARPS) {   // panel strips
      acc_zero(t32);
      mma_tile<false, true>(t32, T(i, p0), tp, dinv + (long long)p0 * 1024, 32, lane, 1.0);
      __syncwarp();
      acc_store(t32, T(i, p0), tp, lane);                  // L_i,p0
      __syncwarp();
      acc_load(t32, T(i, p0 + 1), tp, lane);
      mma_tile<false, true>(t32, T(i, p0), tp, T(p0 + 1, p0), tp, lane, -1.0);
      __syncwarp();
      acc_store(t32, T(i, p0 + 1), tp, lane);
      __syncwarp();
      acc_zero(t32);
      mma_tile<false, true>(t32, T(i, p0 + 1), tp, dinv + (long long)(p0 + 1) * 1024, 32, lane, 1.0);
      __syncwarp();
      acc_store(t32, T(i, p0 + 1), tp, lane);              // L_i,p0+1
    }
    __syncthreads();
  }
  if (s_bad) {
    if (tid == 0) flags[slot] = 1;
    return;
  }
  // ---- W = L^{-1}, block-column pairs from the last
  double* S0 = scr + (long long)warp * 2048;
  double* S1 = S0 + 1024;
  for (int J0 = Tc - 2; J0 >= 0; J0 -= 2) {
    const int J1 = J0 + 1, nstrip = Tc - 1 - J1;
    const int rounds = (nstrip + LP_WARPS - 1) / LP_WARPS;
    for (int rd = 0; rd < rounds; ++rd) {   // highest strips first
      const int I = Tc - 1 - (rd * LP_WARPS + warp);
      const bool act = I > J1;
      const int kend = Tc - rd * LP_WARPS;   // rows of this round are <= kend - 1
      accumulate(false, J0, J1 + 1, kend, act ? I : -1, act ? I : -1);
      if (act) {
        store_half(0, S0, 32, nullptr, 0);
        store_half(1, S1, 32, nullptr, 0);
        __syncwarp();
        acc_zero(t32);
        mma_tile<false, false>(t32, S1, 32, dinv + (long long)J1 * 1024, 32, lane, -1.0);
        __syncwarp();
        acc_store(t32, T(I, J1), tp, lane);               // W_I,J1
        __syncwarp();
        acc_load(t32, S0, 32, lane);
        mma_tile<false, false>(t32, T(I, J1), tp, T(J1, J0), tp, lane, 1.0);
        __syncwarp();
        acc_store(t32, S0, 32, lane);
        __syncwarp();
        acc_zero(t32);
        mma_tile<false, false>(t32, S0, 32, dinv + (long long)J0 * 1024, 32, lane, -1.0);
        __syncwarp();
        acc_store(t32, T(I, J0), tp, lane);               // W_I,J0
      }
    }
    __syncthreads();
    if (warp == 0) {   // diagonal pair
      acc_zero(t32);
      mma_tile<false, false>(t32, dinv + (long long)J1 * 1024, 32, T(J1, J0), tp, lane, 1.0);
      __syncwarp();
      acc_store(t32, S0, 32, lane);
      __syncwarp();
      acc_zero(t32);
      mma_tile<false, false>(t32, S0, 32, dinv + (long long)J0 * 1024, 32, lane, -1.0);
      __syncwarp();
      acc_store(t32, T(J1, J0), tp, lane);                // W_J1,J0
      for (int qd = lane; qd < 1024; qd += 32) {
        T(J0, J0)[(long long)(qd >> 5) * tp + (qd & 31)] = dinv[(long long)J0 * 1024 + qd];
        T(J1, J1)[(long long)(qd >> 5) * tp + (qd & 31)] = dinv[(long long)J1 * 1024 + qd];
      }
    }
    __syncthreads();
  }
  // ---- the slot receives W (lower triangle) and W^T (upper triangle), both row-contiguous:
  // tile (I, J), J <= I, goes to Gi[I][J] and, transposed through a per-warp shared tile, to
  // Gi[J][I] (coalesced both ways)
  double* Gi = Ginv + slot * gi_stride;
  double* tt = lp_sm + warp * (32 * 33);
  const int ntile = Tc * (Tc + 1) / 2;
  for (int t = warp; t < ntile; t += LP_WARPS) {
    int I, J;
    tri_decode(t, I, J);
    if (32 * J >= tau) continue;
    double xr[32];   // the whole tile in flight first: 32 independent loads per lane
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) xr[rr] = T(I, J)[(long long)rr * tp + lane];
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) {
      const int row = 32 * I + rr, col = 32 * J + lane;
      const double x = (row < tau && col <= row) ? xr[rr] : 0.0;
      tt[rr * 33 + lane] = x;
      if (row < tau && col <= row) Gi[(long long)row * ldgi + col] = x;
    }
    __syncwarp();
    for (int rr = 0; rr < 32; ++rr) {   // row 32 J + rr of the upper triangle: W[32 I + lane][32 J + rr]
      const int row = 32 * J + rr, col = 32 * I + lane;
      if (row < tau && col < tau && col > row) Gi[(long long)row * ldgi + col] = tt[lane * 33 + rr];
    }
    __syncwarp();
  }
  if (tid == 0) flags[slot] = 0;
}

}  // namespace

int bfactor_max_tau() { return BB_MAXTAU; }

size_t bfactor_work_elems(int tau) {
  if (tau <= BF_MAXTAU) return 0;
  const long long tp = bb_tp(tau);
  // work matrix, Tc L_pp^{-1} tiles, then Tc tiles (right-looking T_I) or 2 per warp (left-looking)
  return (size_t)(tp * tp + (tp / 32) * 1024 + std::max<long long>(tp / 32, 2 * LP_WARPS) * 1024);
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
  e = cudaFuncSetAttribute(k_bfactor_lp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LP_SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_bfactor_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)bf_smem(BF_MAXTAU));
}

cudaError_t launch_bfactor(const FactorSrc& src, const DevSketch& skb, int nslots, double* Ginv,
                           long long ldgi, long long gi_stride, int* flags, double* work,
                           const Ctrl* ctrl, cudaStream_t st) {
  if (skb.tau > BB_MAXTAU || nslots < 1) return cudaErrorInvalidValue;
  if (skb.tau > BF_MAXTAU) {
    if (!work) return cudaErrorInvalidValue;
    static const bool rl = std::getenv("RS_BF_RIGHT") != nullptr;   // A/B: right-looking kernel
    if (rl)
      k_bfactor_big<<<nslots, BB_THREADS, 0, st>>>(src, skb, Ginv, ldgi, gi_stride, work,
                                                   (long long)bfactor_work_elems(skb.tau), flags, ctrl);
    else
      k_bfactor_lp<<<nslots, LP_THREADS, LP_SMEM, st>>>(src, skb, Ginv, ldgi, gi_stride, work,
                                                        (long long)bfactor_work_elems(skb.tau), flags,
                                                        ctrl);
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
  static const bool no_pf = std::getenv("RS_NO_L2PF") != nullptr;
  if (no_pf || !pfA || (double)sk.len * pf_m * 8.0 > 48e6) pfA = nullptr;
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
