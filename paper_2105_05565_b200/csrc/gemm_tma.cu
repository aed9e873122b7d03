// a3 -- the A S contraction on FP64 tensor cores, Blackwell-style pipeline.
//
//   C'[M x N] = sum_{k < K} A[k, 0:M]^T (x) B[k, 0:N]      (dense primal: C' = (XS)^T X = (A S)^T - lambda S^T)
//
// Warp-specialised: one producer warp issues TMA tile loads (cp.async.bulk.tensor.2d, SASS
// UTMALDG) into a STAGES-deep shared-memory ring, completion tracked by mbarrier transaction
// counts; WM x WN consumer warps wait on the "full" barrier of a stage, run TM x TN
// mma.sync.m8n8k4.f64 (SASS DMMA -- FP64 has no tcgen05/UMMA kind on sm_100a) per k-step of 4, and
// release the stage with one arrive per warp on its "empty" barrier.  No CTA-wide barrier in the
// main loop.  TMA boxes are BM+4 / BN+4 wide so that shared rows are padded by 4 doubles (the 16
// lanes of a half-warp fragment load then hit distinct bank pairs); out-of-bounds elements of a box
// are zero-filled by TMA, which also handles the ragged M / N / K edges.  Split-K partials are
// reduced deterministically by k_splitk_reduce2.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "rs_internal.cuh"

namespace rs {

namespace {

constexpr int BK = 16;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int TM, int TN, int WM, int WN, int STAGES>
__global__ void __launch_bounds__((WM * WN + 1) * 32, 1)
k_tn_gemm_tma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              long long M, long long N, long long K, long long k_per_split, double* __restrict__ C,
              long long ldc, long long split_stride, int lower, const Ctrl* ctrl) {
  if (ctrl && ctrl->done) return;
  constexpr int BM = 8 * TM * WM, BN = 8 * TN * WN;
  constexpr int LDA_S = BM + 4, LDB_S = BN + 4;
  constexpr int A_STAGE = BK * LDA_S, B_STAGE = BK * LDB_S;   // doubles
  constexpr unsigned STAGE_BYTES = (unsigned)(A_STAGE + B_STAGE) * 8u;
  constexpr int NCONS = WM * WN;
  extern __shared__ __align__(128) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_STAGE;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long m0 = (long long)blockIdx.x * BM, n0 = (long long)blockIdx.y * BN;
  if (lower && m0 + BM <= n0) return;   // tile strictly above the diagonal (SYRK-shaped use)
  const long long kbeg = (long long)blockIdx.z * k_per_split;
  const long long kend = min(K, kbeg + k_per_split);
  const int nkb = kbeg < kend ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == NCONS) {   // ------------------------------------------------ producer warp
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        mbar_expect_tx(&full[s], STAGE_BYTES);
        const int k0 = (int)(kbeg + (long long)kb * BK);
        tma_load_2d(As + s * A_STAGE, &tmA, (int)m0, k0, &full[s]);
        tma_load_2d(Bs + s * B_STAGE, &tmB, (int)n0, k0, &full[s]);
      }
    }
    return;
  }
  // ------------------------------------------------------------------- consumer warps
  const int wm = warp / WN, wn = warp % WN;
  const int arow = lane & 3, acol = lane >> 2;
  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb % STAGES;
    mbar_wait(&full[s], (kb / STAGES) & 1);
    const double* as = As + s * A_STAGE + wm * (TM * 8) + acol;
    const double* bs = Bs + s * B_STAGE + wn * (TN * 8) + acol;
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

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

__global__ void k_splitk_reduce2(const double* __restrict__ work, int splits, long long split_stride,
                                 long long M, long long N, long long ldw, double* __restrict__ C,
                                 long long ldc, const Ctrl* ctrl, int lbm, int lbn) {
  // lbm > 0 (lower use, tiles lbm x lbn): columns in tiles strictly above the diagonal are never
  // written by the contraction (left to the mirror / never read) and skipped here
  if (ctrl && ctrl->done) return;
  const long long row = blockIdx.y;
  long long jmax = N;
  if (lbm > 0) {
    const long long mend = (row / lbm) * lbm + lbm;   // a tile works iff n0 < m0 + bm
    jmax = min(N, (mend + lbn - 1) / lbn * lbn);
  }
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < N && j < jmax;
       j += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += work[z * split_stride + row * ldw + j];
    C[row * ldc + j] = s;
  }
}

struct TVariant {
  int tm, tn, wm, wn, stages;
  int bm() const { return 8 * tm * wm; }
  int bn() const { return 8 * tn * wn; }
  int threads() const { return 32 * (wm * wn + 1); }
  size_t smem() const { return (size_t)stages * BK * ((bm() + 4) + (bn() + 4)) * sizeof(double); }
};
constexpr int kNumT = 4;
const TVariant kT[kNumT] = {
    {4, 4, 2, 4, 6},   //  64 x 128, 8 consumer warps
    {5, 4, 5, 2, 6},   // 200 x  64, 10 consumer warps (tau = 200: no M padding)
    {4, 4, 4, 2, 6},   // 128 x  64, 8 consumer warps
    {8, 4, 2, 4, 6},   // 128 x 128, 8 consumer warps (large tau)
};
#define RS_TGEMM(X)                        \
  X(0, k_tn_gemm_tma<4, 4, 2, 4, 6>)       \
  X(1, k_tn_gemm_tma<5, 4, 5, 2, 6>)       \
  X(2, k_tn_gemm_tma<4, 4, 4, 2, 6>)       \
  X(3, k_tn_gemm_tma<8, 4, 2, 4, 6>)
int g_tctas[kNumT] = {1, 1, 1, 1};

const void* tvariant_fn(int v) {
#define RS_CASE(i, ...) \
  if (v == i) return (const void*)__VA_ARGS__;
  RS_TGEMM(RS_CASE)
#undef RS_CASE
  return nullptr;
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool encode_2d(CUtensorMap* map, const double* base, long long inner, long long outer, long long ld,
               int box_inner, int box_outer) {
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

cudaError_t tma_gemm_init() {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess) return e;
    if (q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  for (int v = 0; v < kNumT; ++v) {
    const void* f = tvariant_fn(v);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kT[v].smem());
    if (e != cudaSuccess) return e;
    int nb = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kT[v].threads(), kT[v].smem());
    if (e != cudaSuccess) return e;
    g_tctas[v] = nb > 0 ? nb : 1;
  }
  return cudaSuccess;
}

// Plan (variant, split-K) by the same wave / padded-work cost model as plan_tn_gemm, and encode
// the two TMA descriptors (the operand pointers are fixed for the life of the workspace).
cudaError_t tma_gemm_plan(TmaGemm* g, const double* Aop, long long lda, const double* Bop,
                          long long ldb, long long M, long long N, long long K, int num_sms,
                          int lower) {
  double best_cost = 1e300;
  for (int v = 0; v < kNumT; ++v) {
    const TVariant& V = kT[v];
    // lower: only the tiles on or below the diagonal work (the others return at entry), so the
    // waves are counted over those (c5's A build: 528 of 1024 128 x 128 tiles)
    long long tiles = 0;
    const long long tmn = (M + V.bm() - 1) / V.bm(), tnn = (N + V.bn() - 1) / V.bn();
    if (lower) {
      for (long long i = 0; i < tmn; ++i)
        for (long long j = 0; j < tnn; ++j)
          if (i * V.bm() + V.bm() > j * V.bn()) ++tiles;
    } else {
      tiles = tmn * tnn;
    }
    const long long slots = (long long)g_tctas[v] * num_sms;
    for (int s = 1; s <= 32; ++s) {
      if (s > 1 && K / s < 256) break;
      // split-K partials are s full M x N fp64 buffers: at most ~1 GB of them (an m = 2e4 system's
      // output is 3.2 GB per split -- its allocation and reduce would cost more than the waves)
      if (s > 1 && (double)s * M * N * 8.0 > 1.0e9) break;
      const long long ctas = tiles * s;
      const long long waves = (ctas + slots - 1) / slots;
      const double wave_work = (double)g_tctas[v] * V.bm() * V.bn() * ((double)K / s);
      double cost = waves * wave_work;
      if (s > 1) cost += (double)s * M * N * 40.0 / num_sms;
      if (cost < best_cost * 0.98) {
        best_cost = cost;
        g->variant = v;
        g->splits = s;
      }
    }
  }
  const TVariant& V = kT[g->variant];
  g->lower = lower;
  long long kps = (K + g->splits - 1) / g->splits;
  g->k_per_split = (kps + BK - 1) / BK * BK;
  g->M = M;
  g->N = N;
  g->K = K;
  g->bm = V.bm();
  g->bn = V.bn();
  g->ldw = (N + 1) / 2 * 2;
  g->work_elems = g->splits > 1 ? (size_t)g->splits * (size_t)M * (size_t)g->ldw : 0;
  if (M > 0x7fffffff || N > 0x7fffffff || K > 0x7fffffff) return cudaErrorInvalidValue;
  if (!encode_2d(reinterpret_cast<CUtensorMap*>(g->tmA), Aop, M, K, lda, V.bm() + 4, BK))
    return cudaErrorInvalidValue;
  if (!encode_2d(reinterpret_cast<CUtensorMap*>(g->tmB), Bop, N, K, ldb, V.bn() + 4, BK))
    return cudaErrorInvalidValue;
  return cudaSuccess;
}

cudaError_t tma_gemm_launch(const TmaGemm& g, double* C, long long ldc, double* work,
                            const Ctrl* ctrl, cudaStream_t st) {
  const TVariant& V = kT[g.variant];
  dim3 grid((unsigned)((g.M + V.bm() - 1) / V.bm()), (unsigned)((g.N + V.bn() - 1) / V.bn()),
            (unsigned)g.splits);
  const bool direct = g.splits == 1;
  double* out = direct ? C : work;
  const long long ldo = direct ? ldc : g.ldw;
  const long long so = direct ? 0 : g.M * g.ldw;
  const CUtensorMap& ta = *reinterpret_cast<const CUtensorMap*>(g.tmA);
  const CUtensorMap& tb = *reinterpret_cast<const CUtensorMap*>(g.tmB);
#define RS_LAUNCH(i, ...)                                                                     \
  if (g.variant == i)                                                                         \
    __VA_ARGS__<<<grid, V.threads(), V.smem(), st>>>(ta, tb, g.M, g.N, g.K, g.k_per_split, out, \
                                                     ldo, so, g.lower, ctrl);
  RS_TGEMM(RS_LAUNCH)
#undef RS_LAUNCH
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || direct) return e;
  dim3 rg((unsigned)std::min<long long>((g.N + 255) / 256, 64), (unsigned)g.M);
  k_splitk_reduce2<<<rg, 256, 0, st>>>(work, g.splits, so, g.M, g.N, g.ldw, C, ldc, ctrl,
                                       g.lower ? V.bm() : 0, V.bn());
  return cudaGetLastError();
}

__global__ void k_mirror_lower(double* A, long long lda, long long m) {
  // 32 x 32 tiles (I, J), I > J: A[J-tile]^T <- A[I-tile]; diagonal tiles: upper from lower
  __shared__ double t[32][33];
  const int I = blockIdx.y, J = blockIdx.x;
  if (J > I) return;
  const long long r0 = (long long)I * 32, c0 = (long long)J * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const long long r = r0 + y, c = c0 + threadIdx.x;
    t[y][threadIdx.x] = (r < m && c < m) ? A[r * lda + c] : 0.0;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const long long r = c0 + y, c = r0 + threadIdx.x;   // element (c, r) of the source tile
    if (r < m && c < m && c > r) A[r * lda + c] = t[threadIdx.x][y];
  }
}

cudaError_t launch_mirror_lower(double* A, long long lda, long long m, cudaStream_t st) {
  const unsigned T = (unsigned)((m + 31) / 32);
  k_mirror_lower<<<dim3(T, T), dim3(32, 8), 0, st>>>(A, lda, m);
  return cudaGetLastError();
}

}  // namespace rs
