// The EXPLICIT-mode iterations of a sketch-ahead group as ONE persistent cooperative kernel
// (SURVEY §8(a) rows a4-a7 on precomputed factor slots; DESIGN.md §1 "Sketch-ahead pipeline").
//
// After the group's batched factorisation (bfactor.cu) every G_k^{-1} of the group is known, so one
// iteration of Alg. 2 on slot q is three data-parallel phases separated by grid-wide
// barriers:
//   A  g = S_k^T r^k (each CTA, into shared memory);  tau <= 224: delta = G_k^{-1} g (rows of the
//      slot, one warp per row) and S delta scattered;  tau > 224: t = W g (W = L^{-1}, lower rows)
//   B  (tau > 224)  delta = W^T t (upper rows of the slot), S delta scattered
//   C  u = A S delta over a column block per CTA (the sketched rows of A, or the slot's rows of
//      A S^T for the count sketch), then the heavy-ball update of w and r and ||r||^2 partials
//                                                                            (R13)
// and after the last barrier every CTA sums the partials in the same order and takes the same
// stop decision; CTA 0 writes the control block.  A kernel boundary of the
// launch-per-phase chain it replaces costs more than a grid barrier here, and the chain's per-kernel
// prologues (g gather, preloads, cluster reductions) disappear.  The next phase's rows are pulled
// into L2 (cp.async.bulk.prefetch) before each barrier.
#include <cooperative_groups.h>

#include <algorithm>

#include "rs_internal.cuh"

namespace rs {

namespace {

namespace cg = cooperative_groups;

constexpr int IT_WARPS = 16;
constexpr int IT_NG = 4;   // 64-column chunks per pass of phase C
constexpr int IT_THREADS = IT_WARPS * 32;
constexpr int IT_MAXTAU = 4096;
constexpr int IT_MAXLEN = 8192;

#ifdef RS_IT_PHASES
// development probe (build with RS_NVCC_EXTRA=-DRS_IT_PHASES): SM cycles of CTA 0 per phase:
// 0 A, 1 sync1, 2 B, 3 sync2, 4 C, 5 next-slot staging, 6 sync3, 7 stop rule
__device__ unsigned long long g_it_phase[12];   // 8: A g gather, 9: A prefetch issue, 10: A rows
#define IT_T(v) long long v = clock64()
#define IT_ADD(ph, t0_, t1_) if (blockIdx.x == 0 && threadIdx.x == 0) g_it_phase[ph] += (unsigned long long)((t1_) - (t0_))
#else
#define IT_T(v)
#define IT_ADD(ph, x, y)
#endif

__device__ __forceinline__ void pf_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// (gamma_k, beta_k) at iteration k (rs_momentum; the same formulas as mom_at)
__device__ __forceinline__ void mom_k(const Ctrl& c, long long k, double& gamma, double& beta) {
  if (c.mom_kind == 0) return;
  if (c.mom_kind == 2) {
    const long long i = k < c.mom_ntab ? k : c.mom_ntab - 1;
    gamma = c.mom_tab[2 * i];
    beta = c.mom_tab[2 * i + 1];
    return;
  }
  const double den = (double)(k + 1) * (1.0 - c.mom_eta) + 1.0;
  beta = 1.0 - (2.0 - c.mom_eta) / den;
  gamma = c.mom_kind == 3 ? c.mom_eta / den : 1.0;
}

// row a of the slot times x (shared): sum_{c in [c0, c1)} M[a][c] x[c], warp-wide (fixed order);
// up to 32 loads per lane in flight (a whole row of 1024)
__device__ __forceinline__ double row_dot(const double* __restrict__ row, const double* x, int c0, int c1,
                                          int lane) {
  double s = 0.0;
  for (int cb = c0; cb < c1; cb += 1024) {
    double v[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int c = cb + lane + 32 * u;
      v[u] = c < c1 ? __ldcg(row + c) : 0.0;   // (L2: the slot may be written during this launch)
    }
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int c = cb + lane + 32 * u;
      if (c < c1) s += v[u] * x[c];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// slot q's sketch into shared memory (coord with the sign folded in as bit complement, bucket, bptr)
__device__ __forceinline__ void stage_sketch(const DevSketch& sk, int* s_ce, int* s_bk, int* s_bp, int tid) {
  const int len = sk.bptr[sk.tau];
  for (int e = tid; e < len; e += IT_THREADS) {
    const int c = sk.coord[e];
    s_ce[e] = sk.sign[e] > 0 ? c : ~c;
    s_bk[e] = sk.bucket[e];
  }
  for (int b = tid; b <= sk.tau; b += IT_THREADS) s_bp[b] = sk.bptr[b];
}

__global__ void __launch_bounds__(IT_THREADS, 1)
k_iterate(IterArgs a, Ctrl* ctrl) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double it_sm[];
  __shared__ double s_wp[IT_WARPS];   // per-warp partials of the block reductions
  __shared__ double s_r2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, gw = blockIdx.x * IT_WARPS + warp, GW = G * IT_WARPS;
  const long long m = a.m;
  const Ctrl c0 = *ctrl;   // static for the launch except k / done, which this kernel owns
  if (c0.done) return;
  long long k = c0.k;
  // this CTA's column block of u, w, r (even width: 16-byte aligned prefetches)
  const long long cw = ((m + G - 1) / G + 1) & ~1LL;
  const long long j0 = min(m, (long long)blockIdx.x * cw), j1 = min(m, j0 + cw);
  const int tau_c = a.skb.tau, len_c = a.skb.len;      // len_c: slot stride of the sketch entries
  double* xs = it_sm;                                   // [tau]: g / h / delta (phases A, B)
  double* ys = xs + tau_c;                              // [tau]: y = L^{-1} g (tau > 224)
  double* coef = ys + tau_c;                            // [rows]: coefficient of each row of u
  int* s_ce = reinterpret_cast<int*>(coef + len_c);     // [len] coord (sign as complement)
  int* s_bk = s_ce + len_c;                             // [len] bucket
  int* s_bp = s_bk + len_c;                             // [tau + 1]
  int* s_ro = s_bp + tau_c + 1;                         // [len] row offsets of u's rows (16 B units)
  double* red = reinterpret_cast<double*>(                               // [IT_WARPS][IT_NG][64]
      (reinterpret_cast<uintptr_t>(s_ro + len_c) + 15) & ~(uintptr_t)15);
  const double rsb = 1.0 / sqrt(c0.bnorm2);
  if (a.nslots > 0) stage_sketch(a.skb.at(0), s_ce, s_bk, s_bp, tid);
  __syncthreads();
  // g = S^T r of the staged sketch into xs, by threads t0, t0 + nt, ..
  auto gather_g = [&](int t0, int nt) {
    for (int b = t0; b < tau_c; b += nt) {
      double g = 0.0;
      for (int e = s_bp[b]; e < s_bp[b + 1]; ++e) {
        const int ce = s_ce[e];
        g += ce >= 0 ? __ldcg(a.r + ce) : -__ldcg(a.r + ~ce);
      }
      xs[b] = g;
    }
  };
  for (int q = 0; q < a.nslots; ++q) {
    const int tau = a.skb.tau;
    const int len = s_bp[tau];
    const double* Gi = a.Ginv + (long long)q * a.gi_stride;
    if (a.wait) {   // the slot may still be in a concurrent factorisation kernel (flag -1)
      if (tid == 0) {
        const volatile int* f = a.flags + q;
        while (*f < 0 && !*reinterpret_cast<const volatile int*>(&ctrl->done)) __nanosleep(500);
        __threadfence();
      }
      __syncthreads();
    }
    const int fq = __ldcg(a.flags + q);
    if (fq < 0) return;   // (only if the solve stopped meanwhile)
    if (fq) {   // the group's factorisation found S^T A S not SPD (uniform)
      if (blockIdx.x == 0 && tid == 0) {
        ctrl->status = ST_NOTSPD;
        ctrl->done = 1;
      }
      return;
    }
    double gamma = a.gamma, beta = a.beta;
    mom_k(c0, k, gamma, beta);
    const int nr = a.ASt ? tau : len;   // rows of u's sum
    const double* X = a.ASt ? a.ASt + (long long)q * a.as_stride : a.A;
    const long long ldx = a.ASt ? a.ld_as : a.lda;
    // ---- phase A: g = S^T r in shared memory (for q > 0 gathered right after the previous
    // iteration's last barrier, beside the stop rule's reads); delta (tau <= 224) or t = W g
    IT_T(ta0);
    if (q == 0) {
      gather_g(tid, IT_THREADS);
      __syncthreads();
    }
    IT_T(ta_g);
    IT_ADD(8, ta0, ta_g);
    // (no L2 prefetch of phase C's row segments: ~1000 cp.async.bulk.prefetch per CTA cost 7 us of
    // issue per iteration on c5, more than the loads they would cover)
    auto scatter = [&](int row, double d) {
      for (int e = s_bp[row] + lane; e < s_bp[row + 1]; e += 32) {
        const int ce = s_ce[e];
        a.sdelta[ce >= 0 ? ce : ~ce] = ce >= 0 ? d : -d;
      }
    };
    if (!a.big) {   // delta = G^{-1} g, full rows
      for (int row = gw; row < tau; row += GW) {
        const double d = row_dot(Gi + (long long)row * a.ld_gi, xs, 0, tau, lane);
        if (lane == 0) a.dvec[row] = d;
        scatter(row, d);
      }
      IT_T(ta1);
      IT_ADD(0, ta0, ta1);
      grid.sync();
    } else {
      // tau > 224: the slot holds, in its lower triangle, W_bb = L_bb^{-1} on the diagonal
      // super-blocks b (width sbw) and L_bc (b > c) below them, and the transpose in its upper
      // triangle (bfactor.cu).  delta = G^{-1} g = L^{-T} (L^{-1} g) by block substitution:
      //   forward   y_b = W_bb (g_b - sum_{c<b} L_bc y_c)             b = 0 .. nb-1
      //   backward  delta_b = W_bb^T (y_b - sum_{c>b} L_cb^T delta_c)   b = nb-1 .. 0
      // one grid barrier after every block step; nb = 1 is t = W g, delta = W^T t (W = L^{-1}).
      // Vectors between CTAs: forward h in dvec, y in tvec; backward h in tvec, delta in dvec (each
      // buffer is rewritten only after a barrier that follows every CTA's read of it).
      const int sbw = a.sb > 0 && a.sb < tau ? a.sb : tau;
      const int nb = (tau + sbw - 1) / sbw;
      for (int b = 0; b < nb; ++b) {
        const int r0 = b * sbw, r1 = min(tau, r0 + sbw);
        if (b > 0) {   // h_b = g_b - L_{b,<b} y_{<b}  (lower rows, columns [0, r0))
          for (int row = r0 + gw; row < r1; row += GW) {
            const double h = row_dot(Gi + (long long)row * a.ld_gi, ys, 0, r0, lane);
            if (lane == 0) a.dvec[row] = xs[row] - h;
          }
          grid.sync();
          for (int x = r0 + tid; x < r1; x += IT_THREADS) xs[x] = __ldcg(a.dvec + x);
          __syncthreads();
        }
        for (int row = r0 + gw; row < r1; row += GW) {   // y_b = W_bb h_b (columns [r0, row])
          const double t = row_dot(Gi + (long long)row * a.ld_gi, xs, r0, row + 1, lane);
          if (lane == 0) a.tvec[row] = t;
        }
        if (b == 0)   // this CTA's upper rows (the transposed factors), into L2 for the backward steps
          for (int row = gw; row < tau; row += GW)
            if (lane == 0)
              pf_l2(Gi + (long long)row * a.ld_gi + (row & ~1), (unsigned)(((tau - (row & ~1)) * 8 + 15) & ~15));
        grid.sync();
        for (int x = r0 + tid; x < r1; x += IT_THREADS) ys[x] = __ldcg(a.tvec + x);
        __syncthreads();
      }
      IT_T(tb0);
      IT_ADD(0, ta0, tb0);
      for (int b = nb - 1; b >= 0; --b) {
        const int r0 = b * sbw, r1 = min(tau, r0 + sbw);
        const double* hv = ys;
        if (b < nb - 1) {   // h_b = y_b - L_{>b,b}^T delta_{>b}  (upper rows, columns [r1, tau))
          for (int row = r0 + gw; row < r1; row += GW) {
            const double h = row_dot(Gi + (long long)row * a.ld_gi, xs, r1, tau, lane);
            if (lane == 0) a.tvec[row] = ys[row] - h;
          }
          grid.sync();
          for (int x = r0 + tid; x < r1; x += IT_THREADS) xs[x] = __ldcg(a.tvec + x);
          __syncthreads();
          hv = xs;
        }
        for (int row = r0 + gw; row < r1; row += GW) {   // delta_b = W_bb^T h_b (columns [row, r1))
          const double d = row_dot(Gi + (long long)row * a.ld_gi, hv, row, r1, lane);
          if (lane == 0) a.dvec[row] = d;
          scatter(row, d);
        }
        grid.sync();
        if (b > 0) {   // delta_b for the next blocks' h (xs[r0, r1): h_b is consumed)
          for (int x = r0 + tid; x < r1; x += IT_THREADS) xs[x] = __ldcg(a.dvec + x);
          __syncthreads();
        }
      }
      IT_T(tb1);
      IT_ADD(2, tb0, tb1);
    }
    IT_T(tc0);
    // ---- phase C: u_j = sum_rows coef_row X[row][j] over this CTA's columns; heavy-ball update.
    // Coefficients and row offsets once per iteration; then per batch of 16 rows per lane the
    // offsets are read once and reused by up to IT_NG 64-column chunks (lane = a column pair,
    // 16-byte loads: lda and ld_as are multiples of 4, so the pair's second element is inside the
    // row even at an odd m), the chunks' warp partials reduced in one barrier round
    for (int e = tid; e < nr; e += IT_THREADS) {
      int row;
      if (a.ASt) {
        coef[e] = __ldcg(a.dvec + e);
        row = e;
      } else {
        const double d = __ldcg(a.dvec + s_bk[e]);
        const int ce = s_ce[e];
        coef[e] = ce >= 0 ? d : -d;
        row = ce >= 0 ? ce : ~ce;
      }
      s_ro[e] = (int)(((long long)row * ldx) >> 1);
    }
    __syncthreads();
    const double2* X2 = reinterpret_cast<const double2*>(X);
    double r2 = 0.0;
    const int nch = (int)((j1 - j0 + 63) / 64);
    for (int c0 = 0; c0 < nch; c0 += IT_NG) {
      double s[IT_NG][2];
#pragma unroll
      for (int c = 0; c < IT_NG; ++c) s[c][0] = s[c][1] = 0.0;
      for (int eb = warp; eb < nr; eb += 16 * IT_WARPS) {
        int off[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int e = eb + IT_WARPS * u;
          off[u] = e < nr ? s_ro[e] : -1;
        }
#pragma unroll
        for (int c = 0; c < IT_NG; ++c) {
          if (c0 + c >= nch) break;   // (warp-uniform)
          const long long j = j0 + 64LL * (c0 + c) + 2 * lane;
          const bool jin = j < j1;
          const long long jh = j >> 1;
          double2 x[16];
#pragma unroll
          for (int u = 0; u < 16; ++u)
            x[u] = (jin && off[u] >= 0) ? __ldg(X2 + off[u] + jh) : make_double2(0.0, 0.0);
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            if (off[u] >= 0) {
              const double cf = coef[eb + IT_WARPS * u];
              s[c][0] += cf * x[u].x;
              s[c][1] += cf * x[u].y;
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < IT_NG; ++c) {
        red[(warp * IT_NG + c) * 64 + 2 * lane] = s[c][0];
        red[(warp * IT_NG + c) * 64 + 2 * lane + 1] = s[c][1];
      }
      __syncthreads();
      const int c = warp;   // warp c < IT_NG updates chunk c0 + c (fixed warp order in the sum)
      if (c < IT_NG && c0 + c < nch) {
        const long long j = j0 + 64LL * (c0 + c) + 2 * lane;
        double u0 = 0.0, u1 = 0.0;
#pragma unroll
        for (int w = 0; w < IT_WARPS; ++w) {
          u0 += red[(w * IT_NG + c) * 64 + 2 * lane];
          u1 += red[(w * IT_NG + c) * 64 + 2 * lane + 1];
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const long long jj = j + h;
          if (jj >= j1) break;
          const double u = h ? u1 : u0;
          const double drj = beta * a.dr[jj] - gamma * u;
          const double rj = a.r[jj] + drj;
          a.dr[jj] = drj;
          a.r[jj] = rj;
          const double sd = a.sdelta[jj];
          a.sdelta[jj] = 0.0;
          const double dwj = beta * a.dw[jj] - gamma * sd;
          a.dw[jj] = dwj;
          a.w[jj] += dwj;
          r2 += rj * rj;
        }
      }
      __syncthreads();
    }
    // r2: block reduction into warp 0 (fixed order)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    if (lane == 0) s_wp[warp] = r2;
    __syncthreads();
    if (warp == 0) {
      r2 = lane < IT_WARPS ? s_wp[lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
      if (lane == 0) a.partials[blockIdx.x] = r2;
    }
    IT_T(tc1);
    IT_ADD(4, tc0, tc1);
    // the next slot: its sketch into shared memory and its rows (phase A) into L2 while the grid meets
    if (q + 1 < a.nslots) {
      const DevSketch sn = a.skb.at(q + 1);
      stage_sketch(sn, s_ce, s_bk, s_bp, tid);
      const double* Gn = a.Ginv + (long long)(q + 1) * a.gi_stride;
      for (int row = gw; row < tau; row += GW)
        if (lane == 0) pf_l2(Gn + (long long)row * a.ld_gi, (unsigned)(((a.big ? row + 1 : tau) * 8 + 15) & ~15));
    }
    IT_T(tc2);
    IT_ADD(5, tc1, tc2);
    grid.sync();
    IT_T(tc3);
    IT_ADD(6, tc2, tc3);
    // ---- stop rule: every CTA sums the partials in the same order (warp 0), while
    // the other warps gather the next slot's g = S^T r from the final r (discarded if the rule
    // stops the solve)
    if (warp == 0) {
      double t = 0.0;
      for (int p = lane; p < G; p += 32) t += __ldcg(a.partials + p);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) s_r2 = t;
    } else if (q + 1 < a.nslots) {
      gather_g(tid - 32, IT_THREADS - 32);
    }
    __syncthreads();
    const double tot = s_r2;
    ++k;
    const double rel = sqrt(tot) * rsb;
    int status = ST_RUNNING;
    if (!isfinite(tot) || rel > 1e8) status = ST_DIVERGED;
    else if (rel <= c0.tol) status = ST_CONVERGED;
    else if (k >= c0.max_iter) status = ST_MAXITER;
    if (blockIdx.x == 0 && tid == 0) {
      ctrl->rnorm2 = tot;
      ctrl->k = k;
#ifdef RS_IT_TIMES
      // development probe (RS_NVCC_EXTRA=-DRS_IT_TIMES): the trace holds each iteration's
      // completion time (globaltimer, ns) instead of its relative residual
      if (c0.trace && k <= c0.trace_cap) {
        unsigned long long tns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
        c0.trace[k - 1] = (double)tns;
      }
#else
      if (c0.trace && k <= c0.trace_cap) c0.trace[k - 1] = rel;
#endif
      if (status != ST_RUNNING) {
        ctrl->status = status;
        ctrl->done = 1;
      }
    }
    IT_T(tc4);
    IT_ADD(7, tc3, tc4);
    if (status != ST_RUNNING) return;
  }
}

}  // namespace

size_t iterate_smem() { return 218 * 1024; }   // + the small static arrays <= the 227 KB opt-in

// dynamic shared memory: g / t and the coefficients (doubles), sketch entries, buckets, bucket
// pointers and row offsets (ints), phase C's reduction buffer
static size_t it_smem_bytes(int tau, int len) {
  return (size_t)(2 * tau + len) * 8 + (size_t)(2 * len + tau + 1) * 4 + (size_t)len * 4 + 16 +
         (size_t)IT_WARPS * IT_NG * 64 * 8;
}

bool iterate_ok(const DevSketch& sk, long long m, int grid) {
  (void)grid;
  // phase C's row offsets are 32-bit in 16-byte units: m x round_up(m, 4) / 2 < 2^31
  return sk.tau <= IT_MAXTAU && sk.len <= IT_MAXLEN && it_smem_bytes(sk.tau, sk.len) <= iterate_smem() &&
         m * ((m + 3) / 4 * 4) / 2 < (1LL << 31);
}

#ifdef RS_IT_PHASES
extern "C" int rs_debug_it_phases(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, g_it_phase, sizeof(g_it_phase)) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[12] = {0};
    cudaMemcpyToSymbol(g_it_phase, z, sizeof(z));
  }
  return 0;
}
#endif

cudaError_t iterate_init() {
  return cudaFuncSetAttribute(k_iterate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)iterate_smem());
}

cudaError_t launch_iterate(const IterArgs& args, int grid, Ctrl* ctrl, cudaStream_t st) {
  IterArgs a = args;
  // shared memory: the sketch staging of one slot (g / t, coefficients, entries, bucket pointers)
  const size_t smem = it_smem_bytes(a.skb.tau, a.skb.len);
  if (smem > iterate_smem()) return cudaErrorInvalidValue;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_iterate, IT_THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  Ctrl* c = ctrl;
  void* kargs[] = {&a, &c};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(IT_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  // top priority: in the overlapped pipeline the group's CTAs must take their SMs before the
  // concurrent factorisation's CTAs (two per SM) fill every SM
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = greatest;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelExC(&cfg, (const void*)k_iterate, kargs);
}

}  // namespace rs
