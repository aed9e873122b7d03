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
#include <cstdlib>

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

// TMA variant: one producer warp streams blocks of XT_R consecutive rows (one cp.async.bulk each,
// the rows are contiguous in memory) into a XT_ST-deep shared-memory ring tracked by mbarriers; 8
// consumer warps compute the row dots <X_i, v> (warp shuffles + a named barrier among consumers)
// and the axpy u += t_i X_i from shared memory.  Deep enough in flight to stream X at HBM rate.
constexpr int XT_CONS = 8;                  // consumer warps
constexpr int XT_THREADS = (XT_CONS + 1) * 32;
constexpr int XT_Q = 16;                    // columns per consumer thread: d <= 4096
constexpr int XT_MAXR = 8;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void xt_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra W_%=;\n}\n" ::"r"(su32(bar)), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(XT_THREADS, 1)
k_xpass_tma(const double* __restrict__ X, long long ldx, long long rows, long long d,
            const double* __restrict__ v, double* __restrict__ partials, long long rows_per_cta,
            int R, int stages, const Ctrl* ctrl) {
  if (ctrl->done) return;
  extern __shared__ __align__(128) double xs_ring[];   // [stages][R * ldx]
  __shared__ __align__(8) uint64_t full[8], empty[8];
  __shared__ double red[2][XT_MAXR][XT_CONS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  const long long r1 = min(rows, r0 + rows_per_cta);
  const int nblk = r0 < r1 ? (int)((r1 - r0 + R - 1) / R) : 0;
  const long long stage_elems = (long long)R * ldx;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&empty[s])), "r"(XT_CONS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == XT_CONS) {   // producer
    if (lane == 0) {
      for (int b = 0; b < nblk; ++b) {
        const int s = b % stages;
        if (b >= stages) xt_wait(&empty[s], ((b / stages) - 1) & 1);
        const long long i0 = r0 + (long long)b * R;
        const int nr = (int)min((long long)R, r1 - i0);
        const unsigned bytes = (unsigned)(nr * ldx * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&full[s])),
                     "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
            ::"r"(su32(xs_ring + s * stage_elems)), "l"(X + i0 * ldx), "r"(bytes), "r"(su32(&full[s]))
            : "memory");
      }
    }
    return;
  }
  // consumers
  double vr[XT_Q], acc[XT_Q];
#pragma unroll
  for (int q = 0; q < XT_Q; ++q) {
    const long long j = tid + (long long)(XT_CONS * 32) * q;
    vr[q] = j < d ? v[j] : 0.0;
    acc[q] = 0.0;
  }
  int buf = 0;
  for (int b = 0; b < nblk; ++b) {
    const int s = b % stages;
    xt_wait(&full[s], (b / stages) & 1);
    const double* xs = xs_ring + s * stage_elems;
    const long long i0 = r0 + (long long)b * R;
    const int nr = (int)min((long long)R, r1 - i0);
    for (int r = 0; r < nr; ++r) {
      const double* row = xs + r * ldx;
      double sdot = 0.0;
#pragma unroll
      for (int q = 0; q < XT_Q; ++q) {
        const long long j = tid + (long long)(XT_CONS * 32) * q;
        if (j < d) sdot += row[j] * vr[q];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
      if (lane == 0) red[buf][r][warp] = sdot;
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(XT_CONS * 32) : "memory");
    for (int r = 0; r < nr; ++r) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < XT_CONS; ++w) t += red[buf][r][w];
      const double* row = xs + r * ldx;
#pragma unroll
      for (int q = 0; q < XT_Q; ++q) {
        const long long j = tid + (long long)(XT_CONS * 32) * q;
        if (j < d) acc[q] += t * row[j];
      }
    }
    buf ^= 1;
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&empty[s])) : "memory");
  }
#pragma unroll
  for (int q = 0; q < XT_Q; ++q) {
    const long long j = tid + (long long)(XT_CONS * 32) * q;
    if (j < d) partials[(long long)blockIdx.x * d + j] = acc[q];
  }
}

// u[j] = sum_c partials[c][j]  (fixed order: 8 interleaved slices c = ty (mod 8) summed in
// ascending c, then the slices in ascending ty).  Block: 32 coordinates x 8 slices.
constexpr int XR_Y = 8;
__global__ void __launch_bounds__(32 * XR_Y)
k_xpass_reduce(const double* __restrict__ partials, int nparts, long long d,
               double* __restrict__ u, const Ctrl* ctrl) {
  if (ctrl->done) return;
  __shared__ double red[XR_Y][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const long long j = (long long)blockIdx.x * 32 + tx;
  double s = 0.0;
  if (j < d) {
#pragma unroll 4
    for (int c = ty; c < nparts; c += XR_Y) s += __ldcs(partials + (long long)c * d + j);
  }
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && j < d) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < XR_Y; ++q) t += red[q][tx];
    u[j] = t;
  }
}

// ---------------------------------------------------------------------------------------------
// Fused gather + Gram for tau <= 200 (subsample sketch): G_partial[cta] = sum_{i in slice} x_i x_i^T
// with x_i = X[i, C] gathered straight from X into shared memory (cp.async 8-byte copies, 4-stage
// ring), so X S is never written.  15 consumer warps each own a 40 x 40 region (I >= J) of the lower
// triangle of G in 5 x 5 DMMA tiles; the CTA's 16th warp only helps loading.  Partials per K-slice
// are reduced in a fixed order by k_gram_reduce (deterministic).
constexpr int GF_THREADS = 512;
constexpr int GF_BK = 16;
constexpr int GF_STAGES = 4;
constexpr int GF_MAXTAU = 200;
constexpr int GF_LD = 204;        // row stride (doubles): 204 = 12 mod 16 -> conflict-free fragments

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void dmma_g(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(GF_THREADS, 1)
k_gram_fused(const double* __restrict__ X, long long ldx, long long rows, DevSketch sk,
             long long rows_per_cta, double* __restrict__ partials, const Ctrl* ctrl) {
  if (ctrl->done) return;
  extern __shared__ __align__(16) double gsm[];   // [GF_STAGES][GF_BK][GF_LD]
  __shared__ int s_col[GF_MAXTAU];
  const int tau = sk.tau, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = tid; b < tau; b += GF_THREADS) s_col[b] = sk.coord[sk.bptr[b]];
  __syncthreads();
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  const long long r1 = min(rows, r0 + rows_per_cta);
  const int nkb = r0 < r1 ? (int)((r1 - r0 + GF_BK - 1) / GF_BK) : 0;
  const int tau8 = (tau + 7) & ~7;   // columns >= tau are loaded as zeros
  auto load = [&](int stage, int kb) {
    double* dst = gsm + stage * GF_BK * GF_LD;
    const long long i0 = r0 + (long long)kb * GF_BK;
    for (int q = tid; q < GF_BK * tau8; q += GF_THREADS) {
      const int rr = q / tau8, b = q % tau8;
      const long long i = i0 + rr;
      const bool ok = i < r1 && b < tau;
      cp_async8(dst + rr * GF_LD + b, ok ? X + i * ldx + s_col[b] : X, ok);
    }
  };
#pragma unroll
  for (int s = 0; s < GF_STAGES - 1; ++s) {
    if (s < nkb) load(s, s);
    asm volatile("cp.async.commit_group;\n");
  }
  // region of this warp: (I, J) with I >= J over ceil(tau / 40) groups
  const int ng = (tau + 39) / 40;
  int I = -1, J = -1;
  {
    int t = 0;
    for (int a = 0; a < ng; ++a)
      for (int b = 0; b <= a; ++b, ++t)
        if (t == warp) { I = a; J = b; }
  }
  const bool active = I >= 0;
  double acc[5][5][2];
#pragma unroll
  for (int x = 0; x < 5; ++x)
#pragma unroll
    for (int y = 0; y < 5; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const int arow = lane & 3, acol = lane >> 2;
  for (int kb = 0; kb < nkb; ++kb) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(GF_STAGES - 2));
    __syncthreads();
    const int nxt = kb + GF_STAGES - 1;
    if (nxt < nkb) load(nxt % GF_STAGES, nxt);
    asm volatile("cp.async.commit_group;\n");
    if (active) {
      const double* st = gsm + (kb % GF_STAGES) * GF_BK * GF_LD + acol;
#pragma unroll
      for (int kk = 0; kk < GF_BK; kk += 4) {
        double bf[5];
        const double* rowp = st + (kk + arow) * GF_LD;
#pragma unroll
        for (int y = 0; y < 5; ++y) bf[y] = rowp[J * 40 + y * 8];
#pragma unroll
        for (int x = 0; x < 5; ++x) {   // one A fragment live at a time (register budget 128)
          const double af = rowp[I * 40 + x * 8];
#pragma unroll
          for (int y = 0; y < 5; ++y) dmma_g(acc[x][y], af, bf[y]);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n");
  if (!active) return;
  double* out = partials + (long long)blockIdx.x * GF_MAXTAU * GF_MAXTAU;
#pragma unroll
  for (int x = 0; x < 5; ++x) {
    const int a = I * 40 + x * 8 + (lane >> 2);
#pragma unroll
    for (int y = 0; y < 5; ++y) {
      const int b = J * 40 + y * 8 + 2 * (lane & 3);
      if (a < tau) {
        if (b < tau) out[a * GF_MAXTAU + b] = acc[x][y][0];
        if (b + 1 < tau) out[a * GF_MAXTAU + b + 1] = acc[x][y][1];
      }
    }
  }
}

// G[a][b] = sum_c partials[c][a][b] for b <= a (fixed order: c ascending)
__global__ void k_gram_reduce(const double* __restrict__ partials, int nparts, int tau,
                              double* __restrict__ G, long long ldg, const Ctrl* ctrl) {
  if (ctrl->done) return;
  const int a = blockIdx.x;
  for (int b = threadIdx.x; b <= a; b += blockDim.x) {
    const double* p = partials + a * GF_MAXTAU + b;
    double s = 0.0;
#pragma unroll 8
    for (int c = 0; c < nparts; ++c) s += __ldcs(p + (long long)c * GF_MAXTAU * GF_MAXTAU);
    G[(long long)a * ldg + b] = s;
  }
}

}  // namespace

bool gram_fused_ok(int kind, int tau) { return kind == SK_SUBSAMPLE && tau <= GF_MAXTAU; }
size_t gram_fused_partials(int num_sms) { return (size_t)num_sms * GF_MAXTAU * GF_MAXTAU; }

cudaError_t gram_init() {
  cudaError_t e = cudaFuncSetAttribute(k_xpass_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       210 * 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_gram_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              GF_STAGES * GF_BK * GF_LD * (int)sizeof(double));
}

cudaError_t launch_gram_fused(const double* X, long long ldx, long long rows, const DevSketch& sk,
                              double* partials, double* G, long long ldg, int num_sms,
                              const Ctrl* ctrl, cudaStream_t st) {
  const int nc = num_sms;
  const long long rpc = std::max<long long>(GF_BK, ((rows + nc - 1) / nc + GF_BK - 1) / GF_BK * GF_BK);
  const size_t smem = (size_t)GF_STAGES * GF_BK * GF_LD * sizeof(double);
  k_gram_fused<<<nc, GF_THREADS, smem, st>>>(X, ldx, rows, sk, rpc, partials, ctrl);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_gram_reduce<<<sk.tau, 256, 0, st>>>(partials, nc, sk.tau, G, ldg, ctrl);
  return cudaGetLastError();
}

int xpass_ctas(int num_sms) { return num_sms; }
size_t xpass_partials(long long d, int num_sms) { return (size_t)num_sms * (size_t)d; }

cudaError_t launch_xpass(const double* X, long long ldx, long long rows, long long d,
                         const double* v, double* partials, double* u, int num_sms,
                         const Ctrl* ctrl, cudaStream_t st) {
  if (d > (long long)XP_THREADS * XP_Q) return cudaErrorInvalidValue;
  const int nc = xpass_ctas(num_sms);
  const long long rpc = std::max<long long>(1, (rows + nc - 1) / nc);
  static const bool no_tma = std::getenv("RS_NO_TMA_XPASS") != nullptr;
  // ring: R rows per stage (~64 KB), as many stages as fit in ~200 KB (>= 2)
  const long long row_bytes = ldx * 8;
  int R = (int)std::max<long long>(1, std::min<long long>(XT_MAXR, 65536 / row_bytes));
  int stages = (int)std::min<long long>(8, (200 * 1024) / (R * row_bytes));
  if (!no_tma && stages >= 2 && d <= (long long)XT_CONS * 32 * XT_Q) {
    const size_t smem = (size_t)stages * R * row_bytes;
    k_xpass_tma<<<nc, XT_THREADS, smem, st>>>(X, ldx, rows, d, v, partials, rpc, R, stages, ctrl);
  } else {
    k_xpass<<<nc, XP_THREADS, 0, st>>>(X, ldx, rows, d, v, partials, rpc, ctrl);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_xpass_reduce<<<(unsigned)((d + 31) / 32), dim3(32, XR_Y), 0, st>>>(partials, nc, d, u, ctrl);
  return cudaGetLastError();
}

}  // namespace rs
