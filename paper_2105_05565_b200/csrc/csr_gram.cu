// GRAM mode for CSR X (SURVEY §8(f) NEXT-2 applied to the sparse configs c3 / c4): A S is never
// formed.  With R = X (primal, m = d) or R = X^T (dual, m = n), A = R^T R +
// lambda I and one iteration of Alg. 2 needs only
//
//   G      = S^T A S = (R S)^T (R S) + lambda S^T S
//   A S d  = R^T (R (S d)) + lambda S d
//
// (same iterates as IMPLICIT in exact arithmetic).  Three kernels:
//
//   k_hash_rows   stage 1, one warp per row of R: the row's sketched entries R_ij, j in supp(S),
//                 are mapped to (bucket h(j), sign_j R_ij), equal buckets merged (fixed lane order,
//                 deterministic) in a per-warp shared accumulator, and written back compacted and
//                 sorted by bucket -- row i of R S as a sparse vector ("O(nnz)").
//   k_gram_bands  stage 2: G_lower = sum_i v_i v_i^T, v_i = row i of R S.  The packed lower triangle
//                 is cut into bands of G rows that fit one CTA's shared memory; CTA (band, chunk)
//                 accumulates, for the rows of its nnz-balanced chunk, every pair (s, t), t <= s, of
//                 merged entries whose row bucket b_s lies in the band (int64 fixed-point shared
//                 atomics, fx_add: exact sums), then writes its band to a per-chunk partial; k_gram_band_reduce sums the partials in
//                 chunk order into the row-major Gram.
//   k_spmv        t = R (S d), u = R^T t through the CSR and CSC copies (sub-warp per row).
//
// Cost per iteration: nnz(R) lookups + sum_i |v_i|^2 / 2 pair updates (c3: ~5.8e8, c4: Zipf rows
// ~1e7) instead of the sum_j nnz(col j) * nnz(row) MACs of the materialised A S (c3 1.2e9 + a 200 MB
// A S written and read three times).
#include <algorithm>
#include <climits>
#include <string>
#include <vector>

#include "csr.h"
#include "engine.h"
#include "rs_internal.cuh"

namespace rs {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int HR_WARPS = 8;
constexpr int HR_MAXTAU = 1536;
constexpr int GB_THREADS = 1024;
constexpr int GB_BUDGET = 25856;   // doubles of one band (202 KB of shared memory + 24 KB of
                                   // per-warp row staging, 1 CTA / SM)

__host__ __device__ __forceinline__ long long tri(long long a) { return a * (a + 1) / 2; }

// ------------------------------------------------------------------------------------ stage 1
// Per-warp merge state in shared memory: acc[tau] (values), stage[32], bits[ceil(tau/32)] (touched).
struct WarpMerge {
  double* acc;
  double* stage;
  unsigned* bits;
  int nw;
  const double* fsc;   // per-bucket fixed-point scale 2^e_b of the slot (k_bucket_scale)
  __device__ WarpMerge(double* hsm, int tau, int w, const double* f) : fsc(f) {
    nw = (tau + 31) >> 5;
    acc = hsm + (size_t)w * tau;
    stage = hsm + (size_t)HR_WARPS * tau + w * 32;
    bits = reinterpret_cast<unsigned*>(hsm + (size_t)HR_WARPS * (tau + 32)) + w * nw;
  }
  // one entry per lane (cm < 0: none); equal buckets summed by the group leader in lane order
  __device__ __forceinline__ void add(int cm, double x, int lane) {
    if (!__ballot_sync(FULL, cm >= 0)) return;
    const int b = cm >> 1;
    const unsigned grp = __match_any_sync(FULL, cm >= 0 ? b : -1);
    stage[lane] = x;
    __syncwarp();
    if (cm >= 0 && lane == __ffs(grp) - 1) {
      double s = 0.0;
      for (unsigned g = grp; g; g &= g - 1) s += stage[__ffs(g) - 1];
      const unsigned bit = 1u << (b & 31);
      const unsigned old = atomicOr(&bits[b >> 5], bit);
      if (old & bit) acc[b] += s;
      else acc[b] = s;
    }
    __syncwarp();
  }
  // write the touched buckets in ascending order to hb/hv at `a` (values pre-scaled by the bucket's
  // 2^e_b: exact), clear; returns the count
  __device__ __forceinline__ int flush(long long a, int* hb, double* hv, int lane) {
    int total = 0;
    for (int w0 = 0; w0 < nw; w0 += 32) {
      const int wi = w0 + lane;
      unsigned word = wi < nw ? bits[wi] : 0u;
      const int c = __popc(word);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      long long pos = a + total + incl - c;
      for (; word; word &= word - 1) {
        const int bucket = wi * 32 + __ffs(word) - 1;
        hb[pos] = bucket;
        hv[pos] = acc[bucket] * fsc[bucket];
        ++pos;
      }
      if (wi < nw) bits[wi] = 0u;
      total += __shfl_sync(FULL, incl, 31);
    }
    __syncwarp();
    return total;
  }
};

// Fixed-point accumulation of the CSR Gram bands (sm_100a has no native shared fp64 add; 32-bit
// shared atomics are native): an entry is an int64 in units of 2^-E, added as two 32-bit words
// with the carry of the low word taken from the value the low-word atomic returns.  Two's
// complement addition is exact modulo 2^64, so the result is exact whenever the final value fits,
// which the per-bucket scales of k_bucket_scale guarantee (|G_ab| 2^(e_a + e_b) < 2^61).  Each
// product is rounded once; the sum itself is exact and order independent.
__device__ __forceinline__ void fx_add(unsigned* w, long long x) {
  const unsigned lo = (unsigned)x;
  const unsigned old = atomicAdd(w, lo);
  const int h = (int)(x >> 32) + (old + lo < old ? 1 : 0);
  if (h) atomicAdd(reinterpret_cast<int*>(w) + 1, h);
}

__device__ __forceinline__ int cm_of(const int* __restrict__ cmap, const int* __restrict__ idx,
                                     long long t, long long e) {
  return t < e ? __ldg(cmap + __ldg(idx + t)) : -1;
}

// light rows (<= heavy threshold): one warp per row, 32-row blocks of row pointers per warp,
// 64 entries loaded per step.  ALL (count sketch: every coordinate mapped): the first 64 entries
// of the NEXT row (codes and values, loaded unconditionally) are in flight while the current row
// merges, so the idx -> cmap -> val chain of one row overlaps the merge of the previous one.
template <bool ALL>
__global__ void __launch_bounds__(HR_WARPS * 32)
k_hash_rows(const long long* __restrict__ ptr, const int* __restrict__ idx,
            const double* __restrict__ val, long long rows, long long heavy, const int* __restrict__ cmap,
            int tau, int* __restrict__ hb, double* __restrict__ hv, int* __restrict__ hcnt,
            int slot, const Ctrl* ctrl, const double* __restrict__ fsc) {
  if (slot_unused(ctrl, slot)) return;
  extern __shared__ double hsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpMerge M(hsm, tau, warp, fsc);
  for (int q = lane; q < M.nw; q += 32) M.bits[q] = 0u;
  __syncwarp();
  const long long nwarps = (long long)gridDim.x * HR_WARPS;
  for (long long i0 = ((long long)blockIdx.x * HR_WARPS + warp) * 32; i0 < rows; i0 += nwarps * 32) {
    const long long il = i0 + lane;
    const long long pa = il < rows ? ptr[il] : 0, pe = il < rows ? ptr[il + 1] : 0;
    const int nr = (int)min(32LL, rows - i0);
    if (ALL) {
      // prefetched head (first 64 entries) of row j
      auto head = [&](int j, int& c0, int& c1, double& v0, double& v1) {
        const long long a = __shfl_sync(FULL, pa, j), e = __shfl_sync(FULL, pe, j);
        const long long t0 = a + lane, t1 = a + 32 + lane;
        const bool in = e - a <= heavy;
        c0 = in ? cm_of(cmap, idx, t0, e) : -1;
        c1 = in ? cm_of(cmap, idx, t1, e) : -1;
        v0 = in && t0 < e ? val[t0] : 0.0;
        v1 = in && t1 < e ? val[t1] : 0.0;
      };
      int nc0, nc1;
      double nv0, nv1;
      head(0, nc0, nc1, nv0, nv1);
      for (int j = 0; j < nr; ++j) {
        const int cm0 = nc0, cm1 = nc1;
        const double v0 = nv0, v1 = nv1;
        if (j + 1 < nr) head(j + 1, nc0, nc1, nv0, nv1);
        const long long a = __shfl_sync(FULL, pa, j), e = __shfl_sync(FULL, pe, j);
        if (e - a > heavy) continue;   // k_hash_rows_heavy
        bool touched = false;
        if (__ballot_sync(FULL, cm0 >= 0 || cm1 >= 0)) {
          touched = true;
          M.add(cm0, (cm0 & 1) ? -v0 : v0, lane);
          M.add(cm1, (cm1 & 1) ? -v1 : v1, lane);
        }
        for (long long base = a + 64; base < e; base += 64) {   // rows longer than 64
          const long long t0 = base + lane, t1 = base + 32 + lane;
          const int c0 = cm_of(cmap, idx, t0, e), c1 = cm_of(cmap, idx, t1, e);
          if (!__ballot_sync(FULL, c0 >= 0 || c1 >= 0)) continue;
          touched = true;
          const double w0 = c0 >= 0 ? val[t0] : 0.0, w1 = c1 >= 0 ? val[t1] : 0.0;
          M.add(c0, (c0 & 1) ? -w0 : w0, lane);
          M.add(c1, (c1 & 1) ? -w1 : w1, lane);
        }
        const int total = touched ? M.flush(a, hb, hv, lane) : 0;
        if (lane == 0) hcnt[i0 + j] = total;
      }
      continue;
    }
    for (int j = 0; j < nr; ++j) {
      const long long a = __shfl_sync(FULL, pa, j), e = __shfl_sync(FULL, pe, j);
      if (e - a > heavy) continue;   // k_hash_rows_heavy
      bool touched = false;   // rows with no sketched entry (most of a dual R under SubCount) skip
      for (long long base = a; base < e; base += 64) {   // the merge and its flush
        const long long t0 = base + lane, t1 = base + 32 + lane;
        const int cm0 = cm_of(cmap, idx, t0, e), cm1 = cm_of(cmap, idx, t1, e);
        if (!__ballot_sync(FULL, cm0 >= 0 || cm1 >= 0)) continue;
        touched = true;
        const double v0 = cm0 >= 0 ? val[t0] : 0.0, v1 = cm1 >= 0 ? val[t1] : 0.0;
        M.add(cm0, (cm0 & 1) ? -v0 : v0, lane);
        M.add(cm1, (cm1 & 1) ? -v1 : v1, lane);
      }
      const int total = touched ? M.flush(a, hb, hv, lane) : 0;
      if (lane == 0) hcnt[i0 + j] = total;
    }
  }
}

// heavy rows: one CTA per row; warp w merges chunks w, w + 8, ... into its own accumulator, then the
// eight accumulators are summed in warp order (deterministic) and warp 0 writes the merged row
__global__ void __launch_bounds__(HR_WARPS * 32)
k_hash_rows_heavy(const long long* __restrict__ ptr, const int* __restrict__ idx,
                  const double* __restrict__ val, const int* __restrict__ heavy_rows,
                  const int* __restrict__ cmap, int tau, int* __restrict__ hb,
                  double* __restrict__ hv, int* __restrict__ hcnt, int slot, const Ctrl* ctrl,
                  const double* __restrict__ fsc) {
  if (slot_unused(ctrl, slot)) return;
  extern __shared__ double hsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpMerge M(hsm, tau, warp, fsc);
  for (int q = lane; q < M.nw; q += 32) M.bits[q] = 0u;
  __syncwarp();
  const long long i = heavy_rows[blockIdx.x];
  const long long a = ptr[i], e = ptr[i + 1];
  for (long long base = a + 32LL * warp; base < e; base += 32LL * HR_WARPS) {
    const long long t = base + lane;
    const int cm = cm_of(cmap, idx, t, e);
    const double v = cm >= 0 ? val[t] : 0.0;
    M.add(cm, (cm & 1) ? -v : v, lane);
  }
  __syncthreads();
  // sum the warps' accumulators into warp 0's (thread owns bucket b; other threads only set
  // other bits of warp 0's words, so the read of bit b is race free)
  WarpMerge M0(hsm, tau, 0, fsc);
  for (int b = threadIdx.x; b < tau; b += HR_WARPS * 32) {
    double s = 0.0;
    bool any = false;
    for (int w = 0; w < HR_WARPS; ++w) {
      WarpMerge Mw(hsm, tau, w, fsc);
      if (Mw.bits[b >> 5] & (1u << (b & 31))) {
        s += Mw.acc[b];
        any = true;
      }
    }
    M0.acc[b] = s;
    if (any) atomicOr(&M0.bits[b >> 5], 1u << (b & 31));
  }
  __syncthreads();
  if (warp == 0) {
    const int total = M.flush(a, hb, hv, lane);
    if (lane == 0) hcnt[i] = total;
  }
}

// ---------------------------------------------------------------- stage 1, selected samples (dual)
// Dual route with a subsample / SubCount sketch: only the s selected samples (rows of X) carry
// sketched entries.  k_sel_emit walks their X rows (s x ~nnz/row entries instead of all of R) and
// marks each entry's position in R = X^T with its (bucket << 1 | neg) code, collecting the touched
// R rows; k_sel_merge then merges every touched light row exactly like k_hash_rows (same R order,
// same lane order) reading the codes contiguously, and resets them; entries of heavy (Zipf-popular)
// rows go straight into a dense tau-vector per heavy row (fp64 atomics) whose Gram contribution is
// one lower-tile DMMA GEMM H^T H -- no scan of those long rows, no pair loop over them.
// One warp per selected sample, 4 warps per block (the s = 1024 samples of c4 spread over every
// SM); each lane walks 4 entries per step with independent load chains (colidx -> hidx / cscpos /
// tflag), and first touches are appended with one warp-aggregated atomic on the list counter.
constexpr int SE_WARPS = 4, SE_U = 4;
__global__ void __launch_bounds__(SE_WARPS * 32)
k_sel_emit(DevSketch sk, const long long* __restrict__ rowptr, const int* __restrict__ colidx,
           const double* __restrict__ vals, const int* __restrict__ cscpos, int* __restrict__ cmR,
           int* __restrict__ tflag, int* __restrict__ tlist, int* __restrict__ tcount,
           const int* __restrict__ hidx, double* __restrict__ hacc, long long ldh, int slot,
           const Ctrl* ctrl) {
  if (slot_unused(ctrl, slot)) return;
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * SE_WARPS + (threadIdx.x >> 5);
  if (e >= sk.len) return;
  const int i = sk.coord[e];
  const int b = sk.bucket[e];
  const bool neg = sk.sign[e] <= 0;
  const int code = (b << 1) | (neg ? 1 : 0);
  const long long p1 = rowptr[i + 1];
  for (long long pb = rowptr[i]; pb < p1; pb += 32 * SE_U) {   // warp-uniform trip count
    int f[SE_U], h[SE_U];
#pragma unroll
    for (int u = 0; u < SE_U; ++u) {
      const long long p = pb + 32 * u + lane;
      f[u] = p < p1 ? colidx[p] : -1;
    }
#pragma unroll
    for (int u = 0; u < SE_U; ++u) h[u] = f[u] >= 0 ? hidx[f[u]] : -1;
    bool need[SE_U];
#pragma unroll
    for (int u = 0; u < SE_U; ++u) {
      const long long p = pb + 32 * u + lane;
      need[u] = false;
      if (f[u] < 0) continue;
      if (h[u] >= 0) {   // heavy (Zipf-popular) feature: straight into its dense tau-vector
        const double x = vals[p];
        atomicAdd(&hacc[(long long)h[u] * ldh + b], neg ? -x : x);
        continue;
      }
      cmR[cscpos[p]] = code;
      need[u] = tflag[f[u]] == 0 && atomicExch(&tflag[f[u]], 1) == 0;
    }
#pragma unroll
    for (int u = 0; u < SE_U; ++u) {
      const unsigned m = __ballot_sync(FULL, need[u]);
      if (!m) continue;
      const int leader = __ffs(m) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(tcount, __popc(m));
      base = __shfl_sync(FULL, base, leader);
      if (need[u]) tlist[base + __popc(m & ((1u << lane) - 1u))] = f[u];
    }
  }
}

__global__ void __launch_bounds__(HR_WARPS * 32)
k_sel_merge(const long long* __restrict__ ptr, const double* __restrict__ val, long long heavy,
            int* __restrict__ cmR, int* __restrict__ tflag, const int* __restrict__ tlist,
            const int* __restrict__ tcount, int tau, int* __restrict__ hb, double* __restrict__ hv,
            int* __restrict__ hcnt, int slot, const Ctrl* ctrl, const double* __restrict__ fsc) {
  if (slot_unused(ctrl, slot)) return;
  extern __shared__ double hsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpMerge M(hsm, tau, warp, fsc);
  for (int q = lane; q < M.nw; q += 32) M.bits[q] = 0u;
  __syncwarp();
  const int nt = *tcount;
  for (int k = blockIdx.x * HR_WARPS + warp; k < nt; k += gridDim.x * HR_WARPS) {
    const int f = tlist[k];
    if (lane == 0) tflag[f] = 0;
    const long long a = ptr[f], e = ptr[f + 1];
    if (e - a > heavy) continue;   // heavy rows: dense H^T H (csr_gram_into)
    for (long long base = a; base < e; base += 64) {
      const long long t0 = base + lane, t1 = base + 32 + lane;
      const int cm0 = t0 < e ? cmR[t0] : -1, cm1 = t1 < e ? cmR[t1] : -1;
      if (!__ballot_sync(FULL, cm0 >= 0 || cm1 >= 0)) continue;
      const double v0 = cm0 >= 0 ? val[t0] : 0.0, v1 = cm1 >= 0 ? val[t1] : 0.0;
      M.add(cm0, (cm0 & 1) ? -v0 : v0, lane);
      M.add(cm1, (cm1 & 1) ? -v1 : v1, lane);
      if (cm0 >= 0) cmR[t0] = -1;
      if (cm1 >= 0) cmR[t1] = -1;
    }
    const int total = M.flush(a, hb, hv, lane);
    if (lane == 0) hcnt[f] = total;
  }
}

// t = R v = X^T v for the dual with v = S delta nonzero on the s selected samples only: each
// selected sample's X row is scattered into t (fp64 atomics at L2: t's summation order is not
// fixed; t feeds u = X t, which every rank allreduces)
__global__ void __launch_bounds__(SE_WARPS * 32)
k_sel_scatter(DevSketch sk, const double* __restrict__ v, const long long* __restrict__ rowptr,
              const int* __restrict__ colidx, const double* __restrict__ vals,
              double* __restrict__ t, const Ctrl* ctrl) {
  if (ctrl->done) return;
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * SE_WARPS + (threadIdx.x >> 5);
  if (e >= sk.len) return;
  const int i = sk.coord[e];
  const double sd = v[i];
  for (long long p = rowptr[i] + lane; p < rowptr[i + 1]; p += 32) atomicAdd(&t[colidx[p]], sd * vals[p]);
}

// ------------------------------------------------------------------------------------ stage 2
constexpr int GB_STAGE = 64;   // entries of a light row staged per warp (shared memory)
constexpr size_t GB_STAGE_BYTES = (size_t)(GB_THREADS / 32) * GB_STAGE * 12;
template <bool STAGE>
__global__ void __launch_bounds__(GB_THREADS, 1)
k_gram_bands(const long long* __restrict__ ptr, const int* __restrict__ hcnt,
             const int* __restrict__ hb, const double* __restrict__ hv,
             const int* __restrict__ band_a0, const long long* __restrict__ chunk_r0,
             long long heavy, const int* __restrict__ heavy_rows, const int* __restrict__ chunk_h0,
             double* __restrict__ part, long long part_stride, int slot, const Ctrl* ctrl,
             const int* __restrict__ rlist, const int* __restrict__ rcount, int sz_cap) {
  // rlist (optional): visit only the listed rows (the touched rows of the selected-row path),
  // chunk y taking list entries [y n / nchunks, (y + 1) n / nchunks)
  if (slot_unused(ctrl, slot)) return;
  extern __shared__ double band[];   // [sz_cap] band, then (STAGE) per-warp V[64], B[64]
  const int a0 = band_a0[blockIdx.x], a1 = band_a0[blockIdx.x + 1];
  const long long base = tri(a0);
  const int sz = (int)(tri(a1) - base);
  // the band holds int64 fixed-point entries (fx_add); the merged values carry their bucket's scale
  // 2^e_b (k_bucket_scale), so a product is already in units of 2^-(e_a + e_b)
  const double sc = 1.0;
  unsigned* bw = reinterpret_cast<unsigned*>(band);
  long long* bl = reinterpret_cast<long long*>(band);
  for (int q = threadIdx.x; q < sz; q += GB_THREADS) bl[q] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long r0 = chunk_r0[blockIdx.y], r1 = chunk_r0[blockIdx.y + 1];
  if (rlist) {
    const long long n = *rcount;
    r0 = n * blockIdx.y / gridDim.y;
    r1 = n * (blockIdx.y + 1) / gridDim.y;
  }
  for (long long rb = r0 + 32LL * warp; rb < r1; rb += 32LL * (GB_THREADS / 32)) {
    const long long rk = rb + lane;
    const long long rl = rk < r1 ? (rlist ? (long long)rlist[rk] : rk) : 0;
    int Ll = rk < r1 ? hcnt[rl] : 0;
    const long long offl = Ll ? ptr[rl] : 0;
    if (Ll && ptr[rl + 1] - offl > heavy) Ll = 0;   // heavy phase below
    // STAGE: the first 64 entries of the NEXT row of the ballot order are loaded into registers
    // while the current row's pairs run (its band bounds and staging then need no global loads)
    const unsigned nz0 = __ballot_sync(FULL, Ll > 0);
    int pb0 = INT_MAX, pb1 = INT_MAX;
    double pv0 = 0.0, pv1 = 0.0;
    auto fetch = [&](unsigned m) {   // warp-uniform m
      if (!m) return;
      const int jj = __ffs(m) - 1;
      const int LL = __shfl_sync(FULL, Ll, jj);
      const long long oo = __shfl_sync(FULL, offl, jj);
      pb0 = lane < LL ? hb[oo + lane] : INT_MAX;
      pb1 = lane + 32 < LL ? hb[oo + 32 + lane] : INT_MAX;
      pv0 = lane < LL ? hv[oo + lane] : 0.0;
      pv1 = lane + 32 < LL ? hv[oo + 32 + lane] : 0.0;
    };
    if (STAGE) fetch(nz0);
    for (unsigned nz = nz0; nz; nz &= nz - 1) {
      const int cb0 = pb0, cb1 = pb1;
      const double cv0 = pv0, cv1 = pv1;
      if (STAGE) fetch(nz & (nz - 1));
      const int j = __ffs(nz) - 1;
      const int L = __shfl_sync(FULL, Ll, j);
      const long long off = __shfl_sync(FULL, offl, j);
      const int* B = hb + off;
      const double* V = hv + off;
      int s0 = 0, s1 = 0;   // entries with bucket < a0, < a1 (B ascending)
      if (STAGE && L <= GB_STAGE) {
        s0 = __popc(__ballot_sync(FULL, cb0 < a0)) + __popc(__ballot_sync(FULL, cb1 < a0));
        s1 = __popc(__ballot_sync(FULL, cb0 < a1)) + __popc(__ballot_sync(FULL, cb1 < a1));
      } else {
        for (int q = 0; q < L; q += 32) {
          const int bq = q + lane < L ? B[q + lane] : INT_MAX;
          s0 += __popc(__ballot_sync(FULL, bq < a0));
          s1 += __popc(__ballot_sync(FULL, bq < a1));
          if (__shfl_sync(FULL, bq, 31) >= a1) break;
        }
      }
      if (s1 == s0) continue;
      // pairs (s, t), s0 <= s < s1, t <= s, enumerated q = tri(s) + t: every lane busy, its
      // cursor advancing by 32 pairs per step
      const int np = (int)(tri(s1) - tri(s0));
      if (STAGE && s1 <= GB_STAGE && np >= 96) {   // (short rows: the copy does not pay)
        // the row's first s1 entries staged in the warp's shared buffer: the pair loop reads
        // shared memory only and forms the packed offset in 32-bit arithmetic
        double* wV = reinterpret_cast<double*>(band + sz_cap) + warp * GB_STAGE;
        int* wB = reinterpret_cast<int*>(band + sz_cap + (GB_THREADS / 32) * GB_STAGE) + warp * GB_STAGE;
        __syncwarp();
        if (L <= GB_STAGE) {
          if (lane < s1) { wB[lane] = cb0; wV[lane] = cv0; }
          if (lane + 32 < s1) { wB[lane + 32] = cb1; wV[lane + 32] = cv1; }
        } else {
          for (int q = lane; q < s1; q += 32) {
            wB[q] = B[q];
            wV[q] = V[q];
          }
        }
        __syncwarp();
        const int ib = (int)base;
        int ss = s0, tt = lane;
        while (tt > ss) { tt -= ss + 1; ++ss; }
        // two pairs per lane per step: both low-word atomics are in flight before either carry
        int p = lane;
        for (; p + 32 < np; p += 64) {
          int s2 = ss, t2 = tt + 32;
          while (t2 > s2) { t2 -= s2 + 1; ++s2; }
          const int b1 = wB[ss], b2 = wB[s2];
          unsigned* w1 = bw + 2 * (b1 * (b1 + 1) / 2 - ib + wB[tt]);
          unsigned* w2 = bw + 2 * (b2 * (b2 + 1) / 2 - ib + wB[t2]);
          const long long x1 = __double2ll_rn(wV[ss] * wV[tt] * sc);
          const long long x2 = __double2ll_rn(wV[s2] * wV[t2] * sc);
          const unsigned o1 = atomicAdd(w1, (unsigned)x1);
          const unsigned o2 = atomicAdd(w2, (unsigned)x2);
          const int h1 = (int)(x1 >> 32) + (o1 + (unsigned)x1 < o1 ? 1 : 0);
          const int h2 = (int)(x2 >> 32) + (o2 + (unsigned)x2 < o2 ? 1 : 0);
          if (h1) atomicAdd(reinterpret_cast<int*>(w1) + 1, h1);
          if (h2) atomicAdd(reinterpret_cast<int*>(w2) + 1, h2);
          ss = s2;
          tt = t2 + 32;
          while (tt > ss) { tt -= ss + 1; ++ss; }
        }
        if (p < np) {
          const int bs = wB[ss];
          fx_add(bw + 2 * (bs * (bs + 1) / 2 - ib + wB[tt]), __double2ll_rn(wV[ss] * wV[tt] * sc));
        }
        continue;
      }
      int s = s0, t = lane;
      while (t > s) { t -= s + 1; ++s; }
      for (int p = lane; p < np; p += 32) {
        fx_add(bw + 2 * (tri(B[s]) - base + B[t]), __double2ll_rn(V[s] * V[t] * sc));
        t += 32;
        while (t > s) { t -= s + 1; ++s; }
      }
    }
  }
  // heavy rows of the chunk (Zipf-popular features): all warps on one row at a time, warp w owns
  // the G rows b = w (mod 32) of the band, so the updates need no atomics and no barrier
  __syncthreads();
  for (int h = chunk_h0[blockIdx.y]; h < chunk_h0[blockIdx.y + 1]; ++h) {
    const long long r = heavy_rows[h];
    const int L = hcnt[r];
    const long long off = ptr[r];
    const int* B = hb + off;
    const double* V = hv + off;
    for (int q = 0; q < L; q += 32) {
      const int bq = q + lane < L ? B[q + lane] : INT_MAX;
      if (__shfl_sync(FULL, bq, 0) >= a1) break;
      for (unsigned mine = __ballot_sync(FULL, bq >= a0 && bq < a1 && (bq & 31) == warp); mine;
           mine &= mine - 1) {
        const int s = q + __ffs(mine) - 1;
        const int bs = B[s];
        const double vs = V[s];
        long long* rowp = bl + (tri(bs) - base);
        for (int t = lane; t <= s; t += 32) rowp[B[t]] += __double2ll_rn(vs * V[t] * sc);
      }
    }
  }
  __syncthreads();
  double* out = part + blockIdx.y * part_stride + base;   // scaled units (k_gram_band_reduce)
  for (int q = threadIdx.x; q < sz; q += GB_THREADS) out[q] = (double)bl[q];
}

__global__ void k_gram_band_reduce(const double* __restrict__ part, int nchunks,
                                   long long part_stride, double* __restrict__ G, long long ldg,
                                   int slot, const Ctrl* ctrl, const double* __restrict__ gh,
                                   const double* __restrict__ fsc) {
  if (slot_unused(ctrl, slot)) return;
  const int a = blockIdx.x;
  const long long base = tri(a);
  const double ia = 1.0 / fsc[a];   // powers of two: exact
  for (int c = threadIdx.x; c <= a; c += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nchunks; ++k) s += part[k * part_stride + base + c];
    s *= ia * (1.0 / fsc[c]);
    if (gh) s += gh[(long long)a * ldg + c];   // heavy rows' H^T H (true units, same ld as G)
    G[(long long)a * ldg + c] = s;
  }
}

// Column norms of R (rows of R^T), one warp per row in lane order: the static input of the
// per-bucket fixed-point scales.  With rptr (the CSR row pointer of R) the entries of heavy rows of
// R (longer than `heavy`) are left out: on the dual selected-row path those rows go to dense
// tau-vectors in fp64 (H^T H on DMMA), not into the fixed-point bands.
__global__ void k_row_norms(const long long* __restrict__ ptr, const int* __restrict__ idx,
                            const double* __restrict__ val, long long rows,
                            const long long* __restrict__ rptr, long long heavy,
                            double* __restrict__ out) {
  const long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  double s = 0.0;
  for (long long q = ptr[r] + lane; q < ptr[r + 1]; q += 32) {
    if (rptr) {
      const long long i = idx[q];
      if (rptr[i + 1] - rptr[i] > heavy) continue;
    }
    s += val[q] * val[q];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
  if (lane == 0) out[r] = sqrt(s);
}

// Per-bucket fixed-point scale of the slot's Gram: column b of R S is sum_{e in b} sign_e R[:, c_e],
// so G_bb <= B_b = (sum_{e in b} ||R[:, c_e]||)^2 (triangle inequality), and with
// e_b = floor((60 - ilogb(B_b)) / 2), |G_ab| 2^(e_a + e_b) <= sqrt(B_a B_b) 2^(e_a + e_b) < 2^61
// (Cauchy-Schwarz): every band entry fits the int64 with two bits to spare, and a product is
// rounded to 2^-(e_a + e_b), about 2^-59 of sqrt(B_a B_b) -- relative to its own buckets, not to
// trace(G) (one column scaled by 1e6 no longer costs the other buckets their precision).  The
// bound depends on the sketch and on static norms only: deterministic, no pass over the data.
__global__ void k_bucket_scale(DevSketch sk, const double* __restrict__ cn, double* __restrict__ fsc,
                               int slot, const Ctrl* ctrl) {
  if (slot_unused(ctrl, slot)) return;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= sk.tau) return;
  double s = 0.0;
  for (int e = sk.bptr[b] + lane; e < sk.bptr[b + 1]; e += 32) s += cn[sk.coord[e]];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
  const double B = s * s;
  int e = 0;
  if (B > 0.0 && isfinite(B)) {
    const int t = 60 - ilogb(B);
    e = max(-480, min(480, t >= 0 ? t / 2 : -((1 - t) / 2)));   // floor(t / 2)
  }
  if (lane == 0) fsc[b] = ldexp(1.0, e);
}

// chunk boundaries: first row r with ptr[r] >= c * nnz / nchunks (nnz-balanced)
__global__ void k_chunk_bounds(const long long* __restrict__ ptr, long long rows, int nchunks,
                               long long* __restrict__ r0) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > nchunks) return;
  if (c == nchunks) { r0[c] = rows; return; }
  const long long target = (long long)((double)ptr[rows] * c / nchunks);
  long long lo = 0, hi = rows;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (ptr[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  r0[c] = c == 0 ? 0 : lo;
}

// ------------------------------------------------------------------------------------ SpMV
// out[i] = sum_q val[q] v[idx[q]] over row i; rows longer than `heavy` are left to k_spmv_heavy
template <int VW>
__global__ void __launch_bounds__(256)
k_spmv(const long long* __restrict__ ptr, const int* __restrict__ idx,
       const double* __restrict__ val, long long rows, long long heavy,
       const double* __restrict__ v, double* __restrict__ out, const Ctrl* ctrl) {
  if (ctrl->done) return;
  const int sub = threadIdx.x & (VW - 1);
  const long long g = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / VW;
  const long long ng = ((long long)gridDim.x * blockDim.x) / VW;
  const long long rows_pad = (rows + ng - 1) / ng * ng;   // whole sub-warps iterate together
  for (long long i = g; i < rows_pad; i += ng) {
    double s = 0.0;
    long long a = 0, e = 0;
    if (i < rows) {
      a = ptr[i];
      e = ptr[i + 1];
      if (e - a <= heavy)
        for (long long q = a + sub; q < e; q += VW) s += val[q] * __ldg(v + idx[q]);
    }
#pragma unroll
    for (int o = VW / 2; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o, VW);
    if (sub == 0 && i < rows && e - a <= heavy) out[i] = s;
  }
}

constexpr int SH_THREADS = 256;
__global__ void __launch_bounds__(SH_THREADS)
k_spmv_heavy(const long long* __restrict__ ptr, const int* __restrict__ idx,
             const double* __restrict__ val, const int* __restrict__ heavy_rows,
             const double* __restrict__ v, double* __restrict__ out, const Ctrl* ctrl) {
  if (ctrl->done) return;
  __shared__ double red[SH_THREADS / 32];
  const long long i = heavy_rows[blockIdx.x];
  double s = 0.0;
  for (long long q = ptr[i] + threadIdx.x; q < ptr[i + 1]; q += SH_THREADS) s += val[q] * __ldg(v + idx[q]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < SH_THREADS / 32; ++w) t += red[w];
    out[i] = t;
  }
}

__global__ void k_heavy_list(const long long* __restrict__ ptr, long long rows, long long heavy,
                             int* __restrict__ list, int* __restrict__ count) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (long long)gridDim.x * blockDim.x)
    if (ptr[i + 1] - ptr[i] > heavy) list[atomicAdd(count, 1)] = (int)i;
}

cudaError_t launch_spmv(const long long* ptr, const int* idx, const double* val, long long rows,
                        long long nnz, long long heavy, const int* heavy_rows, int nheavy,
                        const double* v, double* out, int num_sms, const Ctrl* ctrl,
                        cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const double avg = (double)nnz / (double)rows;
  const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((rows * 32 + 255) / 256,
                                                                             (long long)num_sms * 16));
  // lanes per row: about four entries per lane or more (latency: the index -> gather chain)
  if (avg >= 64) k_spmv<32><<<grid, 256, 0, st>>>(ptr, idx, val, rows, heavy, v, out, ctrl);
  else if (avg >= 12) k_spmv<16><<<grid, 256, 0, st>>>(ptr, idx, val, rows, heavy, v, out, ctrl);
  else if (avg >= 6) k_spmv<8><<<grid, 256, 0, st>>>(ptr, idx, val, rows, heavy, v, out, ctrl);
  else k_spmv<4><<<grid, 256, 0, st>>>(ptr, idx, val, rows, heavy, v, out, ctrl);
  if (nheavy > 0) k_spmv_heavy<<<nheavy, SH_THREADS, 0, st>>>(ptr, idx, val, heavy_rows, v, out, ctrl);
  return cudaGetLastError();
}

// heavy threshold: max(256, 8 x mean row length)
long long heavy_threshold(long long nnz, long long rows) {
  const long long avg = rows > 0 ? (nnz + rows - 1) / rows : 0;
  return std::max<long long>(256, 8 * avg);
}

}  // namespace

// R = X (primal) or X^T (dual) as (ptr, idx, val, rows); R^T likewise
struct RView {
  const long long* ptr;
  const int* idx;
  const double* val;
  long long rows;
};

void Problem::csr_gram_free() {
  if (!csr) return;
  dfree(csr->hb);
  dfree(csr->hv);
  dfree(csr->hcnt);
  dfree(csr->band_a0);
  dfree(csr->chunk_r0);
  dfree(csr->gpart);
  dfree(csr->fsc);
  dfree(csr->cnorm);
  csr->fsc = nullptr;
  csr->cnorm = nullptr;
  dfree(csr->tvec);
  dfree(csr->heavy_rowsR);
  dfree(csr->heavy_rowsRt);
  dfree(csr->chunk_h0);
  csr->chunk_h0 = nullptr;
  dfree(csr->cmR);
  dfree(csr->hidx);
  dfree(csr->hacc);
  dfree(csr->gh);
  dfree(csr->gh_work);
  dfree(csr->chunk_h0_none);
  csr->hidx = nullptr;
  csr->hacc = nullptr;
  csr->gh = csr->gh_work = nullptr;
  csr->chunk_h0_none = nullptr;
  dfree(csr->tflag);
  dfree(csr->tlist);
  dfree(csr->tcount);
  csr->cmR = csr->tflag = csr->tlist = csr->tcount = nullptr;
  csr->heavy_rowsR = csr->heavy_rowsRt = nullptr;
  csr->nheavyR = csr->nheavyRt = 0;
  csr->hb = nullptr;
  csr->hv = nullptr;
  csr->hcnt = nullptr;
  csr->band_a0 = nullptr;
  csr->chunk_r0 = nullptr;
  csr->gpart = nullptr;
  csr->tvec = nullptr;
  csr->nbands = csr->nchunks = 0;
}

rs_status Problem::csr_gram_workspace(int kind, int tau) {
  CsrData* c = csr;
  if (tau > HR_MAXTAU) return fail(RS_EUNSUPPORTED, "CSR GRAM mode: tau > 1536");
  const RView R = route == 1 ? RView{c->rowptr, c->colidx, c->vals, c->rows}
                             : RView{c->colptr, c->rowidx, c->cvals, c->cols};
  if (kind != SK_COUNT) RS_TRY(dalloc(&c->cmap_all, m));
  if (route == 2 && kind != SK_COUNT && c->cscpos && !std::getenv("RS_NO_SELROWS")) {
    RS_TRY(dalloc(&c->cmR, std::max<long long>(1, c->nnz)));
    RS_TRY(dalloc(&c->tflag, std::max<long long>(1, R.rows)));
    RS_TRY(dalloc(&c->tlist, std::max<long long>(1, R.rows)));
    RS_TRY(dalloc(&c->tcount, 1));
    RS_CUDA(cudaMemsetAsync(c->cmR, 0xFF, std::max<long long>(1, c->nnz) * sizeof(int), st));
    RS_CUDA(cudaMemsetAsync(c->tflag, 0, std::max<long long>(1, R.rows) * sizeof(int), st));
    RS_CUDA(cudaMemsetAsync(c->tcount, 0, sizeof(int), st));
  }
  RS_TRY(dalloc(&c->hb, c->nnz));
  RS_TRY(dalloc(&c->hv, c->nnz));
  RS_TRY(dalloc(&c->hcnt, R.rows));
  RS_TRY(dalloc(&c->tvec, R.rows));
  ld_gram = round_up(tau, 4);
  RS_TRY(dalloc(&Gram, (size_t)tau * ld_gram));
  RS_TRY(dalloc(&uvec, m));
  // bands of equal area of the packed lower triangle, each <= GB_BUDGET doubles
  const long long total = tri(tau);
  int nb = (int)((total + GB_BUDGET - 1) / GB_BUDGET);
  std::vector<int> a0;
  for (;;) {
    a0.assign(1, 0);
    const double target = (double)total / nb;
    bool ok = true;
    int a = 0;
    for (int k = 1; k < nb; ++k) {
      while (a < tau && (double)tri(a + 1) <= target * k) ++a;
      if (tri(a) - tri(a0.back()) > GB_BUDGET) { ok = false; break; }
      a0.push_back(a);
    }
    a0.push_back(tau);
    if (ok && tri(tau) - tri(a0[a0.size() - 2]) <= GB_BUDGET) break;
    ++nb;
  }
  a0.erase(std::unique(a0.begin(), a0.end()), a0.end());
  c->nbands = (int)a0.size() - 1;
  long long maxband = 0;
  for (int k = 0; k < c->nbands; ++k) maxband = std::max(maxband, tri(a0[k + 1]) - tri(a0[k]));
  c->nchunks = (int)std::max<long long>(1, std::min<long long>(num_sms / std::max(1, c->nbands),
                                                               std::max<long long>(1, R.rows)));
  RS_TRY(dalloc(&c->band_a0, a0.size()));
  RS_CUDA(cudaMemcpyAsync(c->band_a0, a0.data(), a0.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  RS_TRY(dalloc(&c->chunk_r0, c->nchunks + 1));
  k_chunk_bounds<<<(c->nchunks + 1 + 127) / 128, 128, 0, st>>>(R.ptr, R.rows, c->nchunks, c->chunk_r0);
  RS_CUDA(cudaGetLastError());
  c->gpart_stride = round_up(total, 4);
  RS_TRY(dalloc(&c->gpart, (size_t)c->gpart_stride * c->nchunks));
  // heavy-row lists of R and R^T
  {
    const RView Rt = route == 1 ? RView{c->colptr, c->rowidx, c->cvals, c->cols}
                                : RView{c->rowptr, c->colidx, c->vals, c->rows};
    int* cnt = nullptr;
    RS_TRY(dalloc(&cnt, 2));
    RS_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(int), st));
    c->heavyR = heavy_threshold(c->nnz, R.rows);
    c->heavyRt = heavy_threshold(c->nnz, Rt.rows);
    RS_TRY(dalloc(&c->heavy_rowsR, std::max<long long>(1, c->nnz / (c->heavyR + 1) + 1)));
    RS_TRY(dalloc(&c->heavy_rowsRt, std::max<long long>(1, c->nnz / (c->heavyRt + 1) + 1)));
    if (R.rows > 0)
      k_heavy_list<<<(unsigned)std::min<long long>((R.rows + 255) / 256, 4096), 256, 0, st>>>(
          R.ptr, R.rows, c->heavyR, c->heavy_rowsR, cnt);
    if (Rt.rows > 0)
      k_heavy_list<<<(unsigned)std::min<long long>((Rt.rows + 255) / 256, 4096), 256, 0, st>>>(
          Rt.ptr, Rt.rows, c->heavyRt, c->heavy_rowsRt, cnt + 1);
    int h[2] = {0, 0};
    RS_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaStreamSynchronize(st));
    dfree(cnt);
    c->nheavyR = h[0];
    c->nheavyRt = h[1];
    // sorted heavy rows of R and their range per stage-2 chunk
    std::vector<int> hl(c->nheavyR);
    std::vector<long long> cr(c->nchunks + 1);
    if (c->nheavyR)
      RS_CUDA(cudaMemcpy(hl.data(), c->heavy_rowsR, hl.size() * sizeof(int), cudaMemcpyDeviceToHost));
    RS_CUDA(cudaMemcpy(cr.data(), c->chunk_r0, cr.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    std::sort(hl.begin(), hl.end());
    std::vector<int> h0(c->nchunks + 1);
    for (int k = 0; k <= c->nchunks; ++k)
      h0[k] = (int)(std::lower_bound(hl.begin(), hl.end(), cr[k]) - hl.begin());
    if (c->nheavyR)
      RS_CUDA(cudaMemcpy(c->heavy_rowsR, hl.data(), hl.size() * sizeof(int), cudaMemcpyHostToDevice));
    RS_TRY(dalloc(&c->chunk_h0, h0.size()));
    RS_CUDA(cudaMemcpy(c->chunk_h0, h0.data(), h0.size() * sizeof(int), cudaMemcpyHostToDevice));
    if (c->cmR) {   // selected-row path: heavy rows accumulate into dense tau-vectors
      std::vector<int> hx(std::max<long long>(1, R.rows), -1);
      for (int k = 0; k < c->nheavyR; ++k) hx[hl[k]] = k;
      RS_TRY(dalloc(&c->hidx, hx.size()));
      RS_CUDA(cudaMemcpy(c->hidx, hx.data(), hx.size() * sizeof(int), cudaMemcpyHostToDevice));
      const long long nh = std::max(1, c->nheavyR);
      c->ldh = round_up(tau, 4);
      RS_TRY(dalloc(&c->hacc, (size_t)nh * c->ldh));
      RS_CUDA(cudaMemsetAsync(c->hacc, 0, (size_t)nh * c->ldh * sizeof(double), st));
      RS_TRY(dalloc(&c->chunk_h0_none, h0.size()));
      RS_CUDA(cudaMemsetAsync(c->chunk_h0_none, 0, h0.size() * sizeof(int), st));
      if (c->nheavyR > 0) {
        RS_CUDA(tma_gemm_plan(&c->tg_heavy, c->hacc, c->ldh, c->hacc, c->ldh, tau, tau, c->nheavyR,
                              num_sms, 1));
        c->tg_heavy.lower = 1;
        if (c->tg_heavy.work_elems) RS_TRY(dalloc(&c->gh_work, c->tg_heavy.work_elems));
        RS_TRY(dalloc(&c->gh, (size_t)tau * round_up(tau, 4)));
      }
    }
  }
  // per-bucket fixed-point scales (k_bucket_scale) from the column norms of R = rows of R^T
  RS_TRY(dalloc(&c->fsc, tau));
  RS_TRY(dalloc(&c->cnorm, std::max<long long>(1, m)));
  {
    const RView Rt = route == 1 ? RView{c->colptr, c->rowidx, c->cvals, c->cols}
                                : RView{c->rowptr, c->colidx, c->vals, c->rows};
    const bool light_only = route == 2 && c->cmR != nullptr;   // selected-row path (heavy: fp64)
    if (Rt.rows > 0)
      k_row_norms<<<(unsigned)((Rt.rows + 7) / 8), 256, 0, st>>>(
          Rt.ptr, Rt.idx, Rt.val, Rt.rows, light_only ? R.ptr : nullptr, c->heavyR, c->cnorm);
    RS_CUDA(cudaGetLastError());
  }
  c->gb_smem = (size_t)maxband * sizeof(double);
  c->hr_smem = (size_t)HR_WARPS * (tau + 32) * sizeof(double) + (size_t)HR_WARPS * ((tau + 31) / 32) * 4;
  c->gb_cap = (int)round_up(maxband, 2);
  // staged light rows pay on long rows (c3: 50 entries, Gram 2.06 -> 1.85 ms); on short Zipf rows
  // (c4: 10) the unstaged loop is 2 % faster
  c->gb_stage = c->nnz >= 32 * std::max(1LL, R.rows) &&
                (size_t)c->gb_cap * 8 + GB_STAGE_BYTES <= 227 * 1024;
  if (c->gb_stage) c->gb_smem = (size_t)c->gb_cap * 8 + GB_STAGE_BYTES;
  RS_CUDA(cudaFuncSetAttribute(k_gram_bands<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)std::max<size_t>(c->gb_smem, 48 * 1024)));
  RS_CUDA(cudaFuncSetAttribute(k_gram_bands<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)std::max<size_t>(c->gb_smem, 48 * 1024)));
  RS_CUDA(cudaFuncSetAttribute(k_hash_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)std::max<size_t>(c->hr_smem, 48 * 1024)));
  RS_CUDA(cudaFuncSetAttribute(k_hash_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)std::max<size_t>(c->hr_smem, 48 * 1024)));
  RS_CUDA(cudaFuncSetAttribute(k_hash_rows_heavy, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)std::max<size_t>(c->hr_smem, 48 * 1024)));
  RS_CUDA(cudaStreamSynchronize(st));
  if (std::getenv("RS_VERBOSE"))
    fprintf(stderr, "[rs] csr gram: tau %d, %d bands (max %lld doubles), %d chunks, heavy rows "
            "%d (> %lld) / %d (> %lld)\n", tau, c->nbands, maxband, c->nchunks, c->nheavyR,
            c->heavyR, c->nheavyRt, c->heavyRt);
  return RS_OK;
}

static cudaError_t launch_bucket_scale(const DevSketch& s, const double* cn, double* fsc, int slot,
                                       const Ctrl* ctrl, cudaStream_t st) {
  k_bucket_scale<<<(unsigned)((s.tau + 7) / 8), 256, 0, st>>>(s, cn, fsc, slot, ctrl);
  return cudaGetLastError();
}

rs_status Problem::csr_gram_into(const DevSketch& s, double* G, cudaEvent_t* ev, int slot,
                                  bool reduce) {
  auto mark = [&](int cls, int edge) {
    if (ev) cudaEventRecordWithFlags(ev[2 * cls + edge], st, cudaEventRecordExternal);
  };
  CsrData* c = csr;
  const RView R = route == 1 ? RView{c->rowptr, c->colidx, c->vals, c->rows}
                             : RView{c->colptr, c->rowidx, c->cvals, c->cols};
  const int tau = s.tau;
  const int* cmap = s.cmap;
  mark(RS_K_XS, 0);
  RS_CUDA(launch_bucket_scale(s, c->cnorm, c->fsc, slot, ctrl, st));
  const bool sel = s.kind != SK_COUNT && c->cmR != nullptr;   // dual: from the selected samples
  if (s.kind != SK_COUNT && !sel) {
    RS_CUDA(launch_cmap_build(s, c->cmap_all, m, ctrl, st, slot));
    cmap = c->cmap_all;
  }
  if (R.rows > 0 && sel) {   // a2: rows of R S from the s selected rows of X
    RS_CUDA(cudaMemsetAsync(c->hcnt, 0, R.rows * sizeof(int), st));
    k_sel_emit<<<(unsigned)std::max(1, (s.len + SE_WARPS - 1) / SE_WARPS), SE_WARPS * 32, 0, st>>>(
        s, c->rowptr, c->colidx, c->vals, c->cscpos, c->cmR, c->tflag, c->tlist, c->tcount, c->hidx,
        c->hacc, c->ldh, slot, ctrl);
    const unsigned grid = (unsigned)((long long)num_sms * 8);
    k_sel_merge<<<grid, HR_WARPS * 32, c->hr_smem, st>>>(R.ptr, R.val, c->heavyR, c->cmR, c->tflag,
                                                         c->tlist, c->tcount, tau, c->hb, c->hv,
                                                         c->hcnt, slot, ctrl, c->fsc);
    if (c->nheavyR > 0) {   // heavy rows: H^T H on the lower DMMA tiles, then H cleared
      RS_CUDA(tma_gemm_launch(c->tg_heavy, c->gh, ld_gram, c->gh_work, ctrl, st));
      RS_CUDA(cudaMemsetAsync(c->hacc, 0, (size_t)c->nheavyR * c->ldh * sizeof(double), st));
    }
    RS_CUDA(cudaGetLastError());
  } else if (R.rows > 0) {   // a2: rows of R S, merged and bucket-sorted
    const unsigned grid = (unsigned)std::max<long long>(
        1, std::min<long long>((R.rows + HR_WARPS - 1) / HR_WARPS, (long long)num_sms * 8));
    (s.kind == SK_COUNT ? k_hash_rows<true> : k_hash_rows<false>)
        <<<grid, HR_WARPS * 32, c->hr_smem, st>>>(R.ptr, R.idx, R.val, R.rows, c->heavyR, cmap, tau,
                                                  c->hb, c->hv, c->hcnt, slot, ctrl, c->fsc);
    if (c->nheavyR > 0)
      k_hash_rows_heavy<<<c->nheavyR, HR_WARPS * 32, c->hr_smem, st>>>(
          R.ptr, R.idx, R.val, c->heavy_rowsR, cmap, tau, c->hb, c->hv, c->hcnt, slot, ctrl, c->fsc);
    RS_CUDA(cudaGetLastError());
  }
  if (R.rows > 0) {
    mark(RS_K_XS, 1);
    mark(RS_K_GRAM, 0);
    // a3/a4: (R S)^T (R S), lower triangle
    const bool hgemm = sel && c->nheavyR > 0;   // heavy rows already in gh
    (c->gb_stage ? k_gram_bands<true> : k_gram_bands<false>)
        <<<dim3((unsigned)c->nbands, (unsigned)c->nchunks), GB_THREADS, c->gb_smem, st>>>(
        R.ptr, c->hcnt, c->hb, c->hv, c->band_a0, c->chunk_r0, c->heavyR, c->heavy_rowsR,
        hgemm ? c->chunk_h0_none : c->chunk_h0, c->gpart, c->gpart_stride, slot, ctrl,
        sel ? c->tlist : nullptr, sel ? c->tcount : nullptr, c->gb_cap);
    RS_CUDA(cudaGetLastError());
    if (sel) RS_CUDA(cudaMemsetAsync(c->tcount, 0, sizeof(int), st));   // touched list consumed
    k_gram_band_reduce<<<tau, 256, 0, st>>>(c->gpart, c->nchunks, c->gpart_stride, G, ld_gram, slot,
                                            ctrl, hgemm ? c->gh : nullptr, c->fsc);
    RS_CUDA(cudaGetLastError());
  } else {
    mark(RS_K_XS, 1);
    mark(RS_K_GRAM, 0);
    RS_CUDA(launch_fill(G, (long long)tau * ld_gram, 0.0, st));
  }
  if (reduce) RS_TRY(allreduce(G, (size_t)tau * ld_gram));   // else the caller sums a batch
  mark(RS_K_GRAM, 1);
  return RS_OK;
}

rs_status Problem::csr_gram_apply(const double* v, double* u, const DevSketch* s) {
  CsrData* c = csr;
  const RView R = route == 1 ? RView{c->rowptr, c->colidx, c->vals, c->rows}
                             : RView{c->colptr, c->rowidx, c->cvals, c->cols};
  const RView Rt = route == 1 ? RView{c->colptr, c->rowidx, c->cvals, c->cols}
                              : RView{c->rowptr, c->colidx, c->vals, c->rows};
  if (s && c->cmR && s->kind != SK_COUNT) {   // dual, selected samples: t = R v from their X rows
    RS_CUDA(cudaMemsetAsync(c->tvec, 0, std::max<long long>(1, R.rows) * sizeof(double), st));
    k_sel_scatter<<<(unsigned)std::max(1, (s->len + SE_WARPS - 1) / SE_WARPS), SE_WARPS * 32, 0, st>>>(
        *s, v, c->rowptr, c->colidx, c->vals, c->tvec, ctrl);
    RS_CUDA(cudaGetLastError());
  } else {
    RS_CUDA(launch_spmv(R.ptr, R.idx, R.val, R.rows, c->nnz, c->heavyR, c->heavy_rowsR, c->nheavyR,
                        v, c->tvec, num_sms, ctrl, st));
  }
  RS_CUDA(launch_spmv(Rt.ptr, Rt.idx, Rt.val, Rt.rows, c->nnz, c->heavyRt, c->heavy_rowsRt,
                      c->nheavyRt, c->tvec, u, num_sms, ctrl, st));
  return RS_OK;
}

// One iteration of Alg. 2 in CSR GRAM mode (sketch already drawn by the caller).
rs_status Problem::csr_enqueue_gram(const rs_solve_opts* o, cudaEvent_t* ev) {
  auto mark = [&](int cls, int edge) {
    if (ev) cudaEventRecordWithFlags(ev[2 * cls + edge], st, cudaEventRecordExternal);
  };
  RS_TRY(csr_gram_into(sk, Gram, ev));                                            // a2 - a4
  mark(RS_K_SOLVE, 0);
  RS_CUDA(launch_sketched_solve(nullptr, 0, false, Gram, ld_gram, lambda, r, sk, sw, sdelta, ctrl,
                                st));                                              // a4 + a5
  mark(RS_K_SOLVE, 1);
  mark(RS_K_AS, 0);   // u = R^T (R (S delta)), summed over ranks
  RS_TRY(csr_gram_apply(sdelta, uvec, &sk));
  RS_TRY(allreduce(uvec, (size_t)m));
  mark(RS_K_AS, 1);
  mark(RS_K_UPDATE, 0);
  RS_CUDA(launch_update_vec(uvec, lambda, sdelta, w, dw, r, dr, m, o->gamma, o->beta, partials,
                            ctrl, st));                                          // a6 + a7
  mark(RS_K_UPDATE, 1);
  return RS_OK;
}

}  // namespace rs
