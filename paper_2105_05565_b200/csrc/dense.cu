// Dense-X kernels of the hot path (explicit-A build).
//
//  a2  XS = X S  ("fetching the rows/columns indexed by a random subset"; count/SubCount:
//      signed segmented sums).  Row-major XS[n x ld_xs].
//  a3  AS^T = (XS)^T X, i.e. (X^T (X S))^T  ("multiplying a m x tau matrix A S_k"), the
//      tall-skinny TN contraction on FP64 tensor cores: mma.sync.m8n8k4.f64 (SASS DMMA) fed by a
//      4-stage cp.async shared-memory pipeline, deterministic split-K (partials reduced in a fixed
//      order by a second kernel).  FP64 has no tcgen05/UMMA kind on sm_100a; DMMA is the
//      FP64 tensor path and measures 37.1 TFLOP/s on this B200 (profiles/r01_fp64_peak.txt).
//  explicit A = X^T X + lambda I is the same TN contraction with Bop = X, built once.
//  explicit a2: AS^T[b,:] = sum_{e in b} sign_e A[coord_e, :] (A symmetric, rows are columns).
#include <cmath>
#include <algorithm>

#include "rs_internal.cuh"

namespace rs {

namespace {

// ------------------------------------------------------------------------------ a2 gathers
__global__ void k_dense_xs(const double* __restrict__ X, long long ldx, long long rows,
                           DevSketch sk, double* __restrict__ XS, long long ld_xs, int rows_per_blk,
                           const Ctrl* ctrl, int slot) {
  if (slot_unused(ctrl, slot)) return;
  const long long r0 = (long long)blockIdx.x * rows_per_blk;
  const int per_blk = rows_per_blk * (int)ld_xs;
  for (int q = threadIdx.x; q < per_blk; q += blockDim.x) {
    const long long i = r0 + q / ld_xs;
    const int b = q % ld_xs;
    if (i >= rows) break;
    double v = 0.0;
    if (b < sk.tau) {
      const double* xr = X + i * ldx;
      const int e0 = sk.bptr[b], e1 = sk.bptr[b + 1];
      for (int e = e0; e < e1; ++e) {
        const double x = __ldg(xr + sk.coord[e]);
        v += sk.sign[e] > 0 ? x : -x;
      }
    }
    XS[i * ld_xs + b] = v;
  }
}

// a2 with the sketch staged in shared memory (coord with the sign folded in as bit complement, and
// the bucket pointers): one warp per row (XW_ROWS rows per warp in flight), lane b takes buckets
// b, b + 32, ...; a subsample bucket is one independent gather, so a row of tau = 1024 is 32
// gathers per lane in flight instead of a bptr -> coord -> X chain per element.  Rows are written
// whole (lanes on consecutive buckets: coalesced), the padding columns tau .. ld_xs zeroed.
constexpr int XW_WARPS = 8, XW_ROWS = 2;
constexpr size_t XW_SMEM = 48 * 1024;
__global__ void __launch_bounds__(XW_WARPS * 32)
k_dense_xs_warp(const double* __restrict__ X, long long ldx, long long rows, DevSketch sk,
                double* __restrict__ XS, long long ld_xs, const Ctrl* ctrl, int slot) {
  if (slot_unused(ctrl, slot)) return;
  extern __shared__ int xw_sm[];
  int* s_bp = xw_sm;
  int* s_ce = xw_sm + sk.tau + 1;
  const int tau = sk.tau, len = sk.len;
  for (int b = threadIdx.x; b <= tau; b += blockDim.x) s_bp[b] = sk.bptr[b];
  for (int e = threadIdx.x; e < len; e += blockDim.x) s_ce[e] = sk.sign[e] > 0 ? sk.coord[e] : ~sk.coord[e];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool single = len == tau;   // subsample: one entry per bucket
  for (long long i0 = ((long long)blockIdx.x * XW_WARPS + warp) * XW_ROWS; i0 < rows;
       i0 += (long long)gridDim.x * XW_WARPS * XW_ROWS) {
    for (int b0 = 0; b0 < ld_xs; b0 += 32 * 16) {   // 16 buckets per lane per pass
      double v[XW_ROWS][16];
#pragma unroll
      for (int r = 0; r < XW_ROWS; ++r) {
        const long long i = i0 + r;
        const double* xr = X + (i < rows ? i : 0) * ldx;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int b = b0 + lane + 32 * u;
          double x = 0.0;
          if (i < rows && b < tau) {
            if (single) {
              const int ce = s_ce[b];
              x = __ldg(xr + (ce >= 0 ? ce : ~ce));
              if (ce < 0) x = -x;
            } else {
              for (int e = s_bp[b]; e < s_bp[b + 1]; ++e) {
                const int ce = s_ce[e];
                const double y = __ldg(xr + (ce >= 0 ? ce : ~ce));
                x += ce >= 0 ? y : -y;
              }
            }
          }
          v[r][u] = x;
        }
      }
#pragma unroll
      for (int r = 0; r < XW_ROWS; ++r) {
        const long long i = i0 + r;
        if (i >= rows) break;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int b = b0 + lane + 32 * u;
          if (b < ld_xs) XS[i * ld_xs + b] = v[r][u];
        }
      }
    }
  }
}

// a2 when the sketch touches most 128-byte lines of a row (1 - (1 - len/d)^16 >= 0.7, e.g. c5's
// tau = 1024 of d = 4096): each row is streamed whole into shared memory by one cp.async.bulk (two
// rows in flight per CTA, mbarrier transaction counts) and gathered there, so X is read exactly
// once; the per-lane gathers of k_dense_xs_warp re-fetch lines between passes (ncu: 115 GB of DRAM
// reads per c5 XS for the 65.5 GB X).  Needs 16-byte aligned rows (X, ldx even, d even).
constexpr int XR_THREADS = 256;
__device__ __forceinline__ unsigned xr_su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(XR_THREADS)
k_dense_xs_rows(const double* __restrict__ X, long long ldx, long long rows, DevSketch sk,
                double* __restrict__ XS, long long ld_xs, const Ctrl* ctrl, int slot) {
  if (slot_unused(ctrl, slot)) return;
  extern __shared__ __align__(16) double xr_sm[];
  const int d = sk.m, tau = sk.tau, len = sk.len, tid = threadIdx.x;
  double* buf0 = xr_sm;                                            // [2][d]
  uint64_t* bar = reinterpret_cast<uint64_t*>(xr_sm + 2 * (long long)d);
  int* s_bp = reinterpret_cast<int*>(bar + 2);
  int* s_ce = s_bp + tau + 1;
  for (int b = tid; b <= tau; b += XR_THREADS) s_bp[b] = sk.bptr[b];
  for (int e = tid; e < len; e += XR_THREADS) s_ce[e] = sk.sign[e] > 0 ? sk.coord[e] : ~sk.coord[e];
  const unsigned bytes = (unsigned)d * 8u;
  auto issue = [&](int s, long long i) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(xr_su32(&bar[s])),
                 "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
        ::"r"(xr_su32(buf0 + (long long)s * d)), "l"(X + i * ldx), "r"(bytes), "r"(xr_su32(&bar[s]))
        : "memory");
  };
  const long long i0 = blockIdx.x, di = gridDim.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(xr_su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(xr_su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (i0 < rows) issue(0, i0);
    if (i0 + di < rows) issue(1, i0 + di);
  }
  __syncthreads();
  const bool single = len == tau;
  int k = 0;
  for (long long i = i0; i < rows; i += di, ++k) {
    const int s = k & 1;
    asm volatile(
        "{\n.reg .pred P;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra W_%=;\n}\n" ::"r"(xr_su32(&bar[s])), "r"((unsigned)((k >> 1) & 1)) : "memory");
    const double* xr = buf0 + (long long)s * d;
    for (int b = tid; b < ld_xs; b += XR_THREADS) {
      double x = 0.0;
      if (b < tau) {
        if (single) {
          const int ce = s_ce[b];
          x = ce >= 0 ? xr[ce] : -xr[~ce];
        } else {
          for (int e = s_bp[b]; e < s_bp[b + 1]; ++e) {
            const int ce = s_ce[e];
            x += ce >= 0 ? xr[ce] : -xr[~ce];
          }
        }
      }
      XS[i * ld_xs + b] = x;
    }
    __syncthreads();   // every thread is done with buffer s before it is refilled
    if (tid == 0 && i + 2 * di < rows) issue(s, i + 2 * di);
  }
}

__global__ void k_explicit_rows(const double* __restrict__ A, long long lda, long long m,
                                DevSketch sk, double* __restrict__ ASt, long long ld_as,
                                long long as_stride, const Ctrl* ctrl) {
  if (slot_unused(ctrl, blockIdx.z)) return;
  const int b = blockIdx.y;
  sk = sk.at(blockIdx.z);          // batched: slot blockIdx.z
  ASt += blockIdx.z * as_stride;
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int e0 = sk.bptr[b], e1 = sk.bptr[b + 1];
  double v = 0.0;
  for (int e = e0; e < e1; ++e) {
    const double a = A[(long long)sk.coord[e] * lda + j];
    v += sk.sign[e] > 0 ? a : -a;
  }
  ASt[(long long)b * ld_as + j] = v;
}

__global__ void k_add_lambda_s(double lambda, DevSketch sk, double* ASt, long long ld_as,
                               bool rowmajor, const Ctrl* ctrl) {
  if (ctrl && ctrl->done) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= sk.len) return;
  const double s = sk.sign[e] > 0 ? lambda : -lambda;
  if (rowmajor) ASt[(long long)sk.coord[e] * ld_as + sk.bucket[e]] += s;
  else ASt[(long long)sk.bucket[e] * ld_as + sk.coord[e]] += s;
}

__global__ void k_add_diag(double* A, long long lda, long long m, double lambda) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) A[i * lda + i] += lambda;
}

// ------------------------------------------------------------------------------ a3 DMMA GEMM
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// C'[M x N] (+)= sum_k A[k, m] * B[k, n]  over this CTA's K range.
//   A: row-major K x M (lda), B: row-major K x N (ldb).  CTA tile BM x BN x BK with WM x WN warps,
//   each warp TM x TN DMMA 8x8 tiles (BM = 8 TM WM, BN = 8 TN WN).
template <int TM, int TN, int WM, int WN, int STAGES, int MINB>
__global__ void __launch_bounds__(WM * WN * 32, MINB)
k_tn_gemm(const double* __restrict__ A, long long lda, const double* __restrict__ B, long long ldb,
          long long M, long long N, long long K, long long k_per_split, double* __restrict__ C,
          long long ldc, long long split_stride, const Ctrl* ctrl) {
  if (ctrl && ctrl->done) return;
  constexpr int BM = 8 * TM * WM, BN = 8 * TN * WN, BK = 16;
  constexpr int NT = WM * WN * 32;
  // +4 doubles: BM + 4 = 4 or 12 mod 16, so the 16 lanes of a half-warp fragment load hit
  // distinct 8-byte bank pairs; rows stay 16-byte aligned for cp.async
  constexpr int LDA_S = BM + 4, LDB_S = BN + 4;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                               // [STAGES][BK][LDA_S]
  double* Bs = smem + STAGES * BK * LDA_S;         // [STAGES][BK][LDB_S]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const long long m0 = (long long)blockIdx.x * BM, n0 = (long long)blockIdx.y * BN;
  const long long kbeg = (long long)blockIdx.z * k_per_split;
  const long long kend = min(K, kbeg + k_per_split);
  const int nkb = kbeg < kend ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  auto load_stage = [&](int stage, int kb) {
    const long long k0 = kbeg + (long long)kb * BK;
    double* as = As + stage * BK * LDA_S;
    double* bs = Bs + stage * BK * LDB_S;
    constexpr int ACH = BK * BM / 2, BCH = BK * BN / 2;
#pragma unroll
    for (int c = tid; c < ACH; c += NT) {
      const int r = c / (BM / 2), cc = (c % (BM / 2)) * 2;
      const long long k = k0 + r, mm = m0 + cc;
      int bytes = 0;
      if (k < kend) bytes = mm + 1 < M ? 16 : (mm < M ? 8 : 0);
      const double* src = bytes ? A + k * lda + mm : A;
      cp_async16(as + r * LDA_S + cc, src, bytes);
    }
#pragma unroll
    for (int c = tid; c < BCH; c += NT) {
      const int r = c / (BN / 2), cc = (c % (BN / 2)) * 2;
      const long long k = k0 + r, nn = n0 + cc;
      int bytes = 0;
      if (k < kend) bytes = nn + 1 < N ? 16 : (nn < N ? 8 : 0);
      const double* src = bytes ? B + k * ldb + nn : B;
      cp_async16(bs + r * LDB_S + cc, src, bytes);
    }
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkb) load_stage(s, s);
    cp_async_commit();
  }
  const int arow = lane & 3, acol = lane >> 2;
  for (int kb = 0; kb < nkb; ++kb) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = kb + STAGES - 1;
    if (nxt < nkb) load_stage(nxt % STAGES, nxt);
    cp_async_commit();
    const double* as = As + (kb % STAGES) * BK * LDA_S + wm * (TM * 8) + acol;
    const double* bs = Bs + (kb % STAGES) * BK * LDB_S + wn * (TN * 8) + acol;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[TM], bf[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) af[i] = as[(kk + arow) * LDA_S + i * 8];
#pragma unroll
      for (int j = 0; j < TN; ++j) bf[j] = bs[(kk + arow) * LDB_S + j * 8];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  double* Cz = C + (long long)blockIdx.z * split_stride;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const long long row = m0 + wm * (TM * 8) + i * 8 + (lane >> 2);
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const long long col = n0 + wn * (TN * 8) + j * 8 + 2 * (lane & 3);
      double* dst = Cz + row * ldc + col;
      if (col + 1 < N) {
        *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else if (col < N) {
        dst[0] = acc[i][j][0];
      }
    }
  }
}

__global__ void k_splitk_reduce(const double* __restrict__ work, int splits, long long split_stride,
                                long long M, long long N, long long ldw, double* __restrict__ C,
                                long long ldc, const Ctrl* ctrl) {
  if (ctrl && ctrl->done) return;
  const long long row = blockIdx.y;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < N;
       j += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += work[z * split_stride + row * ldw + j];
    C[row * ldc + j] = s;
  }
}

// Tile variants: the plan picks the one whose padded work / wave quantisation is smallest.
struct Variant {
  int tm, tn, wm, wn, stages;
  int bm() const { return 8 * tm * wm; }
  int bn() const { return 8 * tn * wn; }
  int threads() const { return 32 * wm * wn; }
  size_t smem() const { return (size_t)stages * 16 * ((bm() + 4) + (bn() + 4)) * sizeof(double); }
};
constexpr int kNumVariants = 3;
const Variant kVariants[kNumVariants] = {
    {4, 4, 2, 4, 4},   //  64 x 128, 8 warps
    {5, 4, 5, 2, 4},   // 200 x  64, 10 warps (tau = 200: no M padding)
    {4, 4, 4, 2, 4},   // 128 x  64, 8 warps
};
#define RS_GEMM_KERNELS(X)              \
  X(0, k_tn_gemm<4, 4, 2, 4, 4, 2>)     \
  X(1, k_tn_gemm<5, 4, 5, 2, 4, 1>)     \
  X(2, k_tn_gemm<4, 4, 4, 2, 4, 1>)
int g_ctas_per_sm[kNumVariants] = {1, 1, 1};

const void* variant_fn(int v) {
#define RS_CASE(i, ...) if (v == i) return (const void*)__VA_ARGS__;
  RS_GEMM_KERNELS(RS_CASE)
#undef RS_CASE
  return nullptr;
}

// ------------------------------------------------------------------------------ misc
__global__ void k_fill(double* p, long long n, double v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void k_neg(const double* b, double* r, long long m) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x)
    r[i] = -b[i];
}
// deterministic sum of squares: one block, fixed-order strided partials then a tree
__global__ void k_dot_self(const double* x, long long n, double* out) {
  __shared__ double s[1024];
  double acc = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) acc += x[i] * x[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}
// X^T y: pass 1, each block sums a row range into work[blk][cols]; pass 2 sums blocks in order.
constexpr int XTY_ROWS = 1024;
__global__ void k_xty_partial(const double* __restrict__ X, long long ldx, long long rows,
                              long long cols, const double* __restrict__ y, double* work) {
  const long long r0 = (long long)blockIdx.y * XTY_ROWS, r1 = min(rows, r0 + XTY_ROWS);
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < cols;
       j += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (long long i = r0; i < r1; ++i) s += X[i * ldx + j] * y[i];
    work[(long long)blockIdx.y * cols + j] = s;
  }
}
__global__ void k_xty_final(const double* work, long long nblk, long long cols, double* out) {
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < cols;
       j += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (long long z = 0; z < nblk; ++z) s += work[z * cols + j];
    out[j] = s;
  }
}

__global__ void k_count_nonfinite(const double* X, long long ldx, long long rows, long long cols,
                                  unsigned long long* out) {
  unsigned long long bad = 0;
  const long long total = rows * cols;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long i = q / cols, j = q % cols;
    bad += !isfinite(X[i * ldx + j]);
  }
  if (bad) atomicAdd(out, bad);
}

}  // namespace

cudaError_t launch_count_nonfinite(const double* X, long long ldx, long long rows, long long cols,
                                   unsigned long long* out, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  k_count_nonfinite<<<1184, 256, 0, st>>>(X, ldx, rows, cols, out);
  return cudaGetLastError();
}

cudaError_t launch_dense_xs(const double* X, long long ldx, long long rows, const DevSketch& sk,
                            double* XS, long long ld_xs, const Ctrl* ctrl, cudaStream_t st,
                            int slot) {
  if (rows <= 0) return cudaSuccess;
  const size_t smem = (size_t)(sk.len + sk.tau + 1) * 4;
  // whole rows through shared memory when most of each row's 128-byte lines are touched anyway
  const double touched = 1.0 - std::pow(1.0 - std::min(1.0, (double)sk.len / std::max(1, sk.m)), 16.0);
  const size_t rsmem = (size_t)2 * sk.m * 8 + 16 + smem;
  if (touched >= 0.7 && sk.m % 2 == 0 && ldx % 2 == 0 && ((uintptr_t)X & 15) == 0 && rsmem <= 200 * 1024) {
    int dev = 0, sms = 148, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaFuncSetAttribute(k_dense_xs_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)rsmem);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_xs_rows, XR_THREADS, rsmem);
    if (e != cudaSuccess) return e;
    const long long blocks = std::min<long long>(rows, (long long)sms * std::max(1, per_sm));
    k_dense_xs_rows<<<(unsigned)blocks, XR_THREADS, rsmem, st>>>(X, ldx, rows, sk, XS, ld_xs, ctrl, slot);
    return cudaGetLastError();
  }
  if (smem <= XW_SMEM) {   // sketch staged per block, warp-owned rows, independent gathers
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long blocks = std::min<long long>((rows + XW_WARPS * XW_ROWS - 1) / (XW_WARPS * XW_ROWS),
                                                 (long long)sms * 8);
    k_dense_xs_warp<<<(unsigned)std::max(1LL, blocks), XW_WARPS * 32, smem, st>>>(X, ldx, rows, sk, XS,
                                                                                  ld_xs, ctrl, slot);
    return cudaGetLastError();
  }
  const int rpb = (int)std::max<long long>(1, 2048 / ld_xs);
  const long long grid = (rows + rpb - 1) / rpb;
  k_dense_xs<<<(unsigned)grid, 256, 0, st>>>(X, ldx, rows, sk, XS, ld_xs, rpb, ctrl, slot);
  return cudaGetLastError();
}

cudaError_t launch_explicit_rows(const double* A, long long lda, long long m, const DevSketch& sk,
                                 double* ASt, long long ld_as, const Ctrl* ctrl, cudaStream_t st) {
  return launch_explicit_rows_batch(A, lda, m, sk, 1, ASt, ld_as, 0, ctrl, st);
}

cudaError_t launch_explicit_rows_batch(const double* A, long long lda, long long m,
                                       const DevSketch& skb, int nslots, double* ASt,
                                       long long ld_as, long long as_stride, const Ctrl* ctrl,
                                       cudaStream_t st) {
  dim3 grid((unsigned)((m + 255) / 256), (unsigned)skb.tau, (unsigned)nslots);
  k_explicit_rows<<<grid, 256, 0, st>>>(A, lda, m, skb, ASt, ld_as, as_stride, ctrl);
  return cudaGetLastError();
}

cudaError_t launch_add_lambda_s(double lambda, const DevSketch& sk, double* ASt, long long ld_as,
                                bool as_rowmajor, const Ctrl* ctrl, cudaStream_t st) {
  k_add_lambda_s<<<(sk.len + 255) / 256, 256, 0, st>>>(lambda, sk, ASt, ld_as, as_rowmajor, ctrl);
  return cudaGetLastError();
}

namespace {
__global__ void k_add_lower(double* __restrict__ A, const double* __restrict__ T, long long lda,
                            long long m) {
  const long long r = blockIdx.y;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c <= r && c < m;
       c += (long long)gridDim.x * blockDim.x)
    A[r * lda + c] += T[r * lda + c];
}
}  // namespace

cudaError_t launch_add_lower(double* A, const double* T, long long lda, long long m, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_add_lower<<<dim3((unsigned)std::min<long long>((m + 255) / 256, 16), (unsigned)m), 256, 0, st>>>(A, T, lda, m);
  return cudaGetLastError();
}

cudaError_t launch_add_diag(double* A, long long lda, long long m, double lambda, cudaStream_t st) {
  k_add_diag<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(A, lda, m, lambda);
  return cudaGetLastError();
}

cudaError_t gemm_init() {
  for (int v = 0; v < kNumVariants; ++v) {
    const void* f = variant_fn(v);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kVariants[v].smem());
    if (e != cudaSuccess) return e;
    int nb = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kVariants[v].threads(),
                                                      kVariants[v].smem());
    if (e != cudaSuccess) return e;
    g_ctas_per_sm[v] = nb > 0 ? nb : 1;
  }
  return cudaSuccess;
}

// Cost model: time ~ waves x (per-CTA tile work), waves = ceil(CTAs / resident slots); the
// padded tile work counts the DMMA spent on ragged M / N edges; split-K adds a partial write.
GemmPlan plan_tn_gemm(long long M, long long N, long long K, int num_sms) {
  GemmPlan best{};
  double best_cost = 1e300;
  for (int v = 0; v < kNumVariants; ++v) {
    const Variant& V = kVariants[v];
    const long long tm = (M + V.bm() - 1) / V.bm(), tn = (N + V.bn() - 1) / V.bn();
    const long long tiles = tm * tn;
    const long long slots = (long long)g_ctas_per_sm[v] * num_sms;
    for (int s = 1; s <= 32; ++s) {
      if (s > 1 && K / s < 256) break;
      const long long ctas = tiles * s;
      const long long waves = (ctas + slots - 1) / slots;
      // per-SM work of one wave: g_ctas_per_sm CTAs of (bm x bn x K/s)
      const double wave_work = (double)g_ctas_per_sm[v] * V.bm() * V.bn() * ((double)K / s);
      double cost = waves * wave_work;
      if (s > 1) cost += (double)s * M * N * 40.0 / num_sms;   // partial write + reduce
      if (cost < best_cost * 0.98) {
        best_cost = cost;
        best.variant = v;
        best.bm = V.bm();
        best.bn = V.bn();
        best.splits = s;
      }
    }
  }
  long long kps = (K + best.splits - 1) / best.splits;
  kps = (kps + 15) / 16 * 16;
  best.k_per_split = kps;
  best.work_elems = best.splits > 1 ? (size_t)best.splits * (size_t)M * (size_t)((N + 1) / 2 * 2) : 0;
  return best;
}

cudaError_t launch_tn_gemm(const double* Aop, long long lda, const double* Bop, long long ldb,
                           long long M, long long N, long long K, double* C, long long ldc,
                           const GemmPlan& plan, double* work, const Ctrl* ctrl, cudaStream_t st) {
  const Variant& V = kVariants[plan.variant];
  dim3 grid((unsigned)((M + V.bm() - 1) / V.bm()), (unsigned)((N + V.bn() - 1) / V.bn()),
            (unsigned)plan.splits);
  const bool direct = plan.splits == 1;
  const long long ldw = (N + 1) / 2 * 2;   // even: 16-byte double2 stores in the epilogue
  const long long stride = M * ldw;
  double* out = direct ? C : work;
  const long long ldo = direct ? ldc : ldw;
  const long long so = direct ? 0 : stride;
#define RS_LAUNCH(i, ...)                                                                   \
  if (plan.variant == i)                                                                    \
    __VA_ARGS__<<<grid, V.threads(), V.smem(), st>>>(Aop, lda, Bop, ldb, M, N, K,             \
                                                     plan.k_per_split, out, ldo, so, ctrl);
  RS_GEMM_KERNELS(RS_LAUNCH)
#undef RS_LAUNCH
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || direct) return e;
  dim3 rg((unsigned)std::min<long long>((N + 255) / 256, 64), (unsigned)M);
  k_splitk_reduce<<<rg, 256, 0, st>>>(work, plan.splits, stride, M, N, ldw, C, ldc, ctrl);
  return cudaGetLastError();
}

cudaError_t launch_fill(double* p, long long n, double v, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_fill<<<(unsigned)std::min<long long>((n + 255) / 256, 4096), 256, 0, st>>>(p, n, v);
  return cudaGetLastError();
}
cudaError_t launch_axpby_neg(const double* b, double* r, long long m, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_neg<<<(unsigned)std::min<long long>((m + 255) / 256, 4096), 256, 0, st>>>(b, r, m);
  return cudaGetLastError();
}
cudaError_t launch_dot_self(const double* x, long long n, double* out, cudaStream_t st) {
  k_dot_self<<<1, 1024, 0, st>>>(x, n, out);
  return cudaGetLastError();
}
size_t dense_xty_work(long long rows, long long cols) {
  return (size_t)((rows + XTY_ROWS - 1) / XTY_ROWS) * (size_t)cols;
}
cudaError_t launch_dense_xty(const double* X, long long ldx, long long rows, long long cols,
                             const double* y, double* out, double* work, cudaStream_t st) {
  const long long nblk = (rows + XTY_ROWS - 1) / XTY_ROWS;
  if (nblk == 0) return launch_fill(out, cols, 0.0, st);
  dim3 g1((unsigned)((cols + 127) / 128), (unsigned)nblk);
  k_xty_partial<<<g1, 128, 0, st>>>(X, ldx, rows, cols, y, work);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_xty_final<<<(unsigned)((cols + 255) / 256), 256, 0, st>>>(work, nblk, cols, out);
  return cudaGetLastError();
}

}  // namespace rs
