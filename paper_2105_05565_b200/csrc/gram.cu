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

// Row-owner variant (d <= 2048, v = S delta sparse): the same TMA ring, but each consumer warp owns
// whole rows (local row i -> warp i mod 8), so no CTA barrier or cross-warp reduction per row:
//   t_i = <X_i, v> over the len sketch entries only (v = S delta has len nonzeros: coord_e, and
//         sd_e = sign_e delta_{bucket_e}, staged once in shared memory behind the ring),
//   acc += t_i X_i (the warp's own d-vector accumulator in registers, XR_NQ values per lane).
// Every warp waits on every block's "full" barrier in order (also blocks without a row of its own),
// so no warp can run two phases ahead of a stage; "empty" counts the R row releases of a stage.  At
// the end the 8 warp accumulators are summed in warp order through shared memory (deterministic).
constexpr int XR_NQ = 64;                     // d <= 2048
constexpr int XR_MAXLEN = 4096;               // sketch entries

template <int XR_CONS>
__global__ void __launch_bounds__((XR_CONS + 1) * 32)
k_xpass_rows(const double* __restrict__ X, long long ldx, long long rows, long long d, DevSketch sk,
             const double* __restrict__ delta, double* __restrict__ partials,
             long long rows_per_cta, int R, int stages, const Ctrl* ctrl) {
  if (ctrl->done) return;
  extern __shared__ __align__(128) double xs_ring[];   // [stages][R * ldx], then sd[len], coord[len]
  __shared__ __align__(8) uint64_t full[8], empty[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  const long long r1 = min(rows, r0 + rows_per_cta);
  const long long nrows = r0 < r1 ? r1 - r0 : 0;
  const int nblk = (int)((nrows + R - 1) / R);
  const long long stage_elems = (long long)R * ldx;
  const int len = sk.len;
  double* s_sd = xs_ring + stages * stage_elems;
  int* s_co = reinterpret_cast<int*>(s_sd + len);
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&empty[s])), "r"(R));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int e = tid; e < len; e += (XR_CONS + 1) * 32) {
    const double dv = delta[sk.bucket[e]];
    s_sd[e] = sk.sign[e] > 0 ? dv : -dv;
    s_co[e] = sk.coord[e];
  }
  __syncthreads();
  if (warp == XR_CONS) {   // producer
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
  double acc[XR_NQ];
#pragma unroll
  for (int q = 0; q < XR_NQ; ++q) acc[q] = 0.0;
  for (int b = 0; b < nblk; ++b) {
    const int s = b % stages;
    xt_wait(&full[s], (b / stages) & 1);
    const long long i0 = (long long)b * R;
    const int nr = (int)min((long long)R, nrows - i0);
    // rows i0 + r of this block owned by this warp: (i0 + r) mod 8 == warp
    for (int r = (int)((warp - i0 % XR_CONS + XR_CONS) % XR_CONS); r < nr; r += XR_CONS) {
      const double* row = xs_ring + s * stage_elems + (long long)r * ldx;
      double t0 = 0.0, t1 = 0.0;
      int e = lane;
      for (; e + 32 < len; e += 64) {
        t0 += s_sd[e] * row[s_co[e]];
        t1 += s_sd[e + 32] * row[s_co[e + 32]];
      }
      if (e < len) t0 += s_sd[e] * row[s_co[e]];
      double t = t0 + t1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
#pragma unroll
      for (int q = 0; q < XR_NQ; ++q) {
        const int j = lane + 32 * q;
        if (j < d) acc[q] += t * row[j];
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&empty[s])) : "memory");
    }
  }
  // every block's data has been consumed: the ring is free for the 8 warp accumulators
  asm volatile("bar.sync 1, %0;\n" ::"n"(XR_CONS * 32) : "memory");
  double* wacc = xs_ring + (long long)warp * d;
#pragma unroll
  for (int q = 0; q < XR_NQ; ++q) {
    const int j = lane + 32 * q;
    if (j < d) wacc[j] = acc[q];
  }
  asm volatile("bar.sync 1, %0;\n" ::"n"(XR_CONS * 32) : "memory");
  for (long long j = tid; j < d; j += XR_CONS * 32) {
    double u = 0.0;
#pragma unroll
    for (int w = 0; w < XR_CONS; ++w) u += xs_ring[(long long)w * d + j];
    partials[(long long)blockIdx.x * d + j] = u;
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
             long long rows_per_cta, double* __restrict__ partials, int slot, const Ctrl* ctrl) {
  if (slot_unused(ctrl, slot)) return;
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
  const bool active = I >= 0, diag = I == J;
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
          for (int y = 0; y < 5; ++y)
            if (!diag || y <= x) dmma_g(acc[x][y], af, bf[y]);   // diagonal region: lower tiles
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

// Gram from the transposed copy XT (d x n, row-major, built once per problem): the tau sketched
// columns of X are tau contiguous rows of XT, so a K-slice of the Gram reads tau coalesced
// 256-byte segments (the algorithmic tau n 8 bytes) instead of gathering 8-byte elements that
// touch ~0.8 of X's lines.  Stage layout [region rows][GW_LDK] (k contiguous, conflict-free DMMA
// fragments); the same 15-warp 40 x 40 region split and per-CTA partials as k_gram_fused, reduced
// in order by k_gram_reduce.  Warp-specialised: warp 15 is a producer that
// streams each stage's tau row segments (32 k-values = 256 B each, one cp.async.bulk per row,
// completion on the stage's "full" mbarrier by transaction count) into a 3-deep ring; the 15
// consumer warps wait on "full", run their region's DMMA k-steps and release the stage with one
// arrive each on "empty" -- no CTA-wide barrier in the main loop.  X^T's rows are zero-padded to a
// multiple of 64, and interior K slices are whole 32-row chunks, so every copy is a full segment.
constexpr int GW_BK = 32, GW_LDK = 36, GW_STAGES = 3, GW_CONS = 15;
constexpr int GW_THREADS = (GW_CONS + 1) * 32;
size_t gram_xtw_smem(int tau) { return (size_t)GW_STAGES * ((tau + 39) / 40 * 40) * GW_LDK * 8; }

__global__ void __launch_bounds__(GW_THREADS, 1)
k_gram_xtw(const double* __restrict__ XT, long long ldxt, long long rows, DevSketch sk,
           long long rows_per_cta, double* __restrict__ partials, int slot, const Ctrl* ctrl) {
  if (slot_unused(ctrl, slot)) return;
  extern __shared__ __align__(16) double gsm[];   // [GW_STAGES][ng * 40][GW_LDK]
  __shared__ __align__(8) uint64_t full[GW_STAGES], empty[GW_STAGES];
  __shared__ int s_col[GF_MAXTAU];
  const int tau = sk.tau, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = tid; b < tau; b += GW_THREADS) s_col[b] = sk.coord[sk.bptr[b]];
  if (tid == 0) {
    for (int s = 0; s < GW_STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&empty[s])), "r"(GW_CONS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const long long r0 = (long long)blockIdx.x * rows_per_cta;
  const long long r1 = min(rows, r0 + rows_per_cta);
  const int nkb = r0 < r1 ? (int)((r1 - r0 + GW_BK - 1) / GW_BK) : 0;
  const int ng = (tau + 39) / 40, srows = ng * 40;
  const int stage_elems = srows * GW_LDK;
  if (warp == GW_CONS) {   // producer warp
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % GW_STAGES;
      if (kb >= GW_STAGES) xt_wait(&empty[s], ((kb / GW_STAGES) - 1) & 1);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&full[s])),
                     "r"((unsigned)(tau * GW_BK * 8)) : "memory");
      __syncwarp();
      const long long k0 = r0 + (long long)kb * GW_BK;
      double* dst = gsm + s * stage_elems;
      for (int b = lane; b < tau; b += 32)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
            ::"r"(su32(dst + b * GW_LDK)), "l"(XT + (long long)s_col[b] * ldxt + k0),
            "r"(GW_BK * 8), "r"(su32(&full[s]))
            : "memory");
    }
    return;
  }
  // consumers: region of this warp (I, J), I >= J
  int I = -1, J = -1;
  {
    int t = 0;
    for (int a = 0; a < ng; ++a)
      for (int b = 0; b <= a; ++b, ++t)
        if (t == warp) { I = a; J = b; }
  }
  const bool active = I >= 0, diag = I == J;
  double acc[5][5][2];
#pragma unroll
  for (int x = 0; x < 5; ++x)
#pragma unroll
    for (int y = 0; y < 5; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const int kq = lane & 3, mq = lane >> 2;
  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb % GW_STAGES;
    xt_wait(&full[s], (kb / GW_STAGES) & 1);
    if (active) {
      const double* st = gsm + s * stage_elems + mq * GW_LDK + kq;
      const double* sa = st + (I * 40) * GW_LDK;
      const double* sb = st + (J * 40) * GW_LDK;
#pragma unroll
      for (int kk = 0; kk < GW_BK; kk += 4) {
        double bf[5];
#pragma unroll
        for (int y = 0; y < 5; ++y) bf[y] = sb[y * 8 * GW_LDK + kk];
#pragma unroll
        for (int x = 0; x < 5; ++x) {
          const double af = sa[x * 8 * GW_LDK + kk];
#pragma unroll
          for (int y = 0; y < 5; ++y)
            if (!diag || y <= x) dmma_g(acc[x][y], af, bf[y]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&empty[s])) : "memory");
  }
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

// XT[j][i] = X[i][j] (32 x 32 tiles through shared memory)
__global__ void k_transpose(const double* __restrict__ X, long long ldx, long long rows, long long d,
                            double* __restrict__ XT, long long ldxt) {
  __shared__ double t[32][33];
  const long long i0 = (long long)blockIdx.y * 32, j0 = (long long)blockIdx.x * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const long long i = i0 + y, j = j0 + threadIdx.x;
    t[y][threadIdx.x] = (i < rows && j < d) ? X[i * ldx + j] : 0.0;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const long long j = j0 + y, i = i0 + threadIdx.x;
    if (j < d && i < ldxt) XT[j * ldxt + i] = t[threadIdx.x][y];
  }
}

// G[a][b] = sum_c partials[c][a][b] for b <= a (fixed order: 8 interleaved slices c = ty (mod 8)
// summed in ascending c, then the slices in ascending ty).  Block: 32 consecutive entries of the
// square GF_MAXTAU x GF_MAXTAU partial layout x 8 slices; entries above the diagonal are skipped.
__global__ void __launch_bounds__(256)
k_gram_reduce(const double* __restrict__ partials, int nparts, int tau, double* __restrict__ G,
              long long ldg, const Ctrl* ctrl, int slot = 0, const long long* kbase = nullptr) {
  if (ctrl->done || (kbase ? *kbase : ctrl->k) + slot >= ctrl->max_iter) return;
  __shared__ double red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int q = blockIdx.x * 32 + tx, a = q / GF_MAXTAU, b = q % GF_MAXTAU;
  const bool in = a < tau && b <= a;
  double s = 0.0;
  if (in) {
#pragma unroll 4
    for (int c = ty; c < nparts; c += 8) s += __ldcs(partials + (long long)c * GF_MAXTAU * GF_MAXTAU + q);
  }
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && in) {
    double t = 0.0;
#pragma unroll
    for (int y = 0; y < 8; ++y) t += red[y][tx];
    G[(long long)a * ldg + b] = t;
  }
}
inline unsigned gram_reduce_grid(int tau) { return (unsigned)((tau * GF_MAXTAU + 31) / 32); }


}  // namespace

bool gram_fused_ok(int kind, int tau) { return kind == SK_SUBSAMPLE && tau <= GF_MAXTAU; }
size_t gram_fused_partials(int num_sms) { return (size_t)num_sms * GF_MAXTAU * GF_MAXTAU; }

cudaError_t gram_init() {
  cudaError_t e = cudaFuncSetAttribute(k_xpass_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       210 * 1024);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_xpass_rows<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e != cudaSuccess) return e;

  e = cudaFuncSetAttribute(k_gram_xtw, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)gram_xtw_smem(GF_MAXTAU));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_gram_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              GF_STAGES * GF_BK * GF_LD * (int)sizeof(double));
}

cudaError_t launch_gram_fused(const double* X, long long ldx, long long rows, const DevSketch& sk,
                              double* partials, double* G, long long ldg, int num_sms,
                              const Ctrl* ctrl, cudaStream_t st, int slot) {
  const int nc = num_sms;
  const long long rpc = std::max<long long>(GF_BK, ((rows + nc - 1) / nc + GF_BK - 1) / GF_BK * GF_BK);
  const size_t smem = (size_t)GF_STAGES * GF_BK * GF_LD * sizeof(double);
  k_gram_fused<<<nc, GF_THREADS, smem, st>>>(X, ldx, rows, sk, rpc, partials, slot, ctrl);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_gram_reduce<<<gram_reduce_grid(sk.tau), 256, 0, st>>>(partials, nc, sk.tau, G, ldg, ctrl, slot);
  return cudaGetLastError();
}

cudaError_t launch_transpose(const double* X, long long ldx, long long rows, long long d, double* XT,
                             long long ldxt, cudaStream_t st) {
  const dim3 grid((unsigned)((d + 31) / 32), (unsigned)((ldxt + 31) / 32));
  k_transpose<<<grid, dim3(32, 8), 0, st>>>(X, ldx, rows, d, XT, ldxt);
  return cudaGetLastError();
}

cudaError_t launch_gram_xt(const double* XT, long long ldxt, long long rows, const DevSketch& sk,
                           double* partials, double* G, long long ldg, int num_sms,
                           const Ctrl* ctrl, cudaStream_t st, int slot) {
  const int nc = num_sms;
  if (ldxt % 64 != 0) return cudaErrorInvalidValue;   // rows of X^T are zero-padded to 64
  const long long rpw = std::max<long long>(GW_BK, ((rows + nc - 1) / nc + GW_BK - 1) / GW_BK * GW_BK);
  k_gram_xtw<<<nc, GW_THREADS, gram_xtw_smem(sk.tau), st>>>(XT, ldxt, rows, sk, rpw, partials, slot,
                                                           ctrl);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_gram_reduce<<<gram_reduce_grid(sk.tau), 256, 0, st>>>(partials, nc, sk.tau, G, ldg, ctrl, slot,
                                                          nullptr);
  return cudaGetLastError();
}

int xpass_ctas(int num_sms) { return num_sms; }
size_t xpass_partials(long long d, int num_sms) { return (size_t)num_sms * (size_t)d; }

cudaError_t launch_xpass(const double* X, long long ldx, long long rows, long long d,
                         const double* v, double* partials, double* u, int num_sms,
                         const Ctrl* ctrl, cudaStream_t st, const DevSketch* sk,
                         const double* delta) {
  if (d > (long long)XP_THREADS * XP_Q) return cudaErrorInvalidValue;
  const int nc = xpass_ctas(num_sms);
  const long long rpc = std::max<long long>(1, (rows + nc - 1) / nc);
  // ring: R rows per stage (~64 KB), as many stages as fit in ~200 KB (>= 2)
  const long long row_bytes = ldx * 8;
  const int R = (int)std::max<long long>(1, std::min<long long>(XT_MAXR, 65536 / row_bytes));
  const int stages = (int)std::min<long long>(8, (200 * 1024) / (R * row_bytes));
  const size_t ring = (size_t)stages * R * row_bytes;
  if (sk && delta && d <= 32LL * XR_NQ && sk->len <= XR_MAXLEN && stages >= 2 &&
      ring >= (size_t)8 * d * 8 && ring + (size_t)sk->len * 12 <= 220 * 1024) {
    // warp-owned rows, <X_i, S delta> from the sketch entries only
    k_xpass_rows<8><<<nc, 9 * 32, ring + (size_t)sk->len * 12, st>>>(X, ldx, rows, d, *sk, delta, partials,
                                                                   rpc, R, stages, ctrl);
  } else if (stages >= 2 && d <= (long long)XT_CONS * 32 * XT_Q) {
    k_xpass_tma<<<nc, XT_THREADS, ring, st>>>(X, ldx, rows, d, v, partials, rpc, R, stages, ctrl);
  } else {
    k_xpass<<<nc, XP_THREADS, 0, st>>>(X, ldx, rows, d, v, partials, rpc, ctrl);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_xpass_reduce<<<(unsigned)((d + 31) / 32), dim3(32, XR_Y), 0, st>>>(partials, nc, d, u, ctrl);
  return cudaGetLastError();
}
}  // namespace rs
