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
//                 merged entries whose row bucket b_s lies in the band (shared fp64 atomics), then
//                 writes its band to a per-chunk partial; k_gram_band_reduce sums the partials in
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
constexpr int GB_BUDGET = 26624;   // doubles of one band (208 KB of shared memory, 1 CTA / SM)

__host__ __device__ __forceinline__ long long tri(long long a) { return a * (a + 1) / 2; }

// ------------------------------------------------------------------------------------ stage 1
__global__ void __launch_bounds__(HR_WARPS * 32)
k_hash_rows(const long long* __restrict__ ptr, const int* __restrict__ idx,
            const double* __restrict__ val, long long rows, const int* __restrict__ cmap, int tau,
            int* __restrict__ hb, double* __restrict__ hv, int* __restrict__ hcnt,
            const Ctrl* ctrl) {
  if (ctrl->done) return;
  extern __shared__ double hsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (tau + 31) >> 5;
  double* acc = hsm + (size_t)warp * tau;
  double* stage = hsm + (size_t)HR_WARPS * tau + warp * 32;
  unsigned* bits = reinterpret_cast<unsigned*>(hsm + (size_t)HR_WARPS * (tau + 32)) + warp * nw;
  for (int q = lane; q < nw; q += 32) bits[q] = 0u;
  __syncwarp();
  const long long nwarps = (long long)gridDim.x * HR_WARPS;
  for (long long i = (long long)blockIdx.x * HR_WARPS + warp; i < rows; i += nwarps) {
    const long long a = ptr[i], e = ptr[i + 1];
    bool any = false;
    for (long long base = a; base < e; base += 32) {
      const long long t = base + lane;
      int cm = -1;
      double x = 0.0;
      if (t < e) {
        cm = __ldg(cmap + idx[t]);
        if (cm >= 0) x = (cm & 1) ? -val[t] : val[t];
      }
      if (!__ballot_sync(FULL, cm >= 0)) continue;
      any = true;
      const int b = cm >> 1;
      const unsigned grp = __match_any_sync(FULL, cm >= 0 ? b : -1);
      stage[lane] = x;
      __syncwarp();
      if (cm >= 0 && lane == __ffs(grp) - 1) {   // leader: sum of the group in lane order
        double s = 0.0;
        for (unsigned g = grp; g; g &= g - 1) s += stage[__ffs(g) - 1];
        const unsigned bit = 1u << (b & 31);
        const unsigned old = atomicOr(&bits[b >> 5], bit);
        if (old & bit) acc[b] += s;
        else acc[b] = s;
      }
      __syncwarp();
    }
    int total = 0;
    if (any) {   // compaction in ascending bucket order
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
          hv[pos] = acc[bucket];
          ++pos;
        }
        if (wi < nw) bits[wi] = 0u;
        total += __shfl_sync(FULL, incl, 31);
      }
    }
    if (lane == 0) hcnt[i] = total;
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------ stage 2
__device__ __forceinline__ void pair_decode(long long q, int& s, int& t) {
  // q = tri(s) + t, 0 <= t <= s
  int i = (int)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
  while (tri(i + 1) <= q) ++i;
  while (tri(i) > q) --i;
  s = i;
  t = (int)(q - tri(i));
}

__global__ void __launch_bounds__(GB_THREADS, 1)
k_gram_bands(const long long* __restrict__ ptr, const int* __restrict__ hcnt,
             const int* __restrict__ hb, const double* __restrict__ hv,
             const int* __restrict__ band_a0, const long long* __restrict__ chunk_r0,
             double* __restrict__ part, long long part_stride, const Ctrl* ctrl) {
  if (ctrl->done) return;
  extern __shared__ double band[];
  const int a0 = band_a0[blockIdx.x], a1 = band_a0[blockIdx.x + 1];
  const long long base = tri(a0);
  const int sz = (int)(tri(a1) - base);
  for (int q = threadIdx.x; q < sz; q += GB_THREADS) band[q] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long r0 = chunk_r0[blockIdx.y], r1 = chunk_r0[blockIdx.y + 1];
  for (long long r = r0 + warp; r < r1; r += GB_THREADS / 32) {
    const int L = hcnt[r];
    if (L == 0) continue;
    const long long off = ptr[r];
    const int* B = hb + off;
    const double* V = hv + off;
    int s0 = 0, s1 = 0;   // entries with bucket < a0, < a1 (B ascending)
    for (int q = 0; q < L; q += 32) {
      const int bq = q + lane < L ? B[q + lane] : INT_MAX;
      s0 += __popc(__ballot_sync(FULL, bq < a0));
      s1 += __popc(__ballot_sync(FULL, bq < a1));
    }
    if (s1 == s0) continue;
    const long long p0 = tri(s0), np = tri(s1) - p0;   // pairs (s, t), s0 <= s < s1, t <= s
    for (long long p = lane; p < np; p += 32) {
      int s, t;
      pair_decode(p0 + p, s, t);
      const int bs = B[s];
      atomicAdd(&band[tri(bs) - base + B[t]], V[s] * V[t]);
    }
  }
  __syncthreads();
  double* out = part + blockIdx.y * part_stride + base;
  for (int q = threadIdx.x; q < sz; q += GB_THREADS) out[q] = band[q];
}

__global__ void k_gram_band_reduce(const double* __restrict__ part, int nchunks,
                                   long long part_stride, double* __restrict__ G, long long ldg,
                                   const Ctrl* ctrl) {
  if (ctrl->done) return;
  const int a = blockIdx.x;
  const long long base = tri(a);
  for (int c = threadIdx.x; c <= a; c += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nchunks; ++k) s += part[k * part_stride + base + c];
    G[(long long)a * ldg + c] = s;
  }
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
template <int VW>
__global__ void __launch_bounds__(256)
k_spmv(const long long* __restrict__ ptr, const int* __restrict__ idx,
       const double* __restrict__ val, long long rows, const double* __restrict__ v,
       double* __restrict__ out, const Ctrl* ctrl) {
  if (ctrl->done) return;
  const int sub = threadIdx.x & (VW - 1);
  const long long g = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / VW;
  const long long ng = ((long long)gridDim.x * blockDim.x) / VW;
  const long long rows_pad = (rows + ng - 1) / ng * ng;   // whole sub-warps iterate together
  for (long long i = g; i < rows_pad; i += ng) {
    double s = 0.0;
    if (i < rows)
      for (long long q = ptr[i] + sub; q < ptr[i + 1]; q += VW) s += val[q] * __ldg(v + idx[q]);
#pragma unroll
    for (int o = VW / 2; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o, VW);
    if (sub == 0 && i < rows) out[i] = s;
  }
}

cudaError_t launch_spmv(const long long* ptr, const int* idx, const double* val, long long rows,
                        long long nnz, const double* v, double* out, int num_sms, const Ctrl* ctrl,
                        cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const double avg = (double)nnz / (double)rows;
  const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((rows * 32 + 255) / 256,
                                                                             (long long)num_sms * 16));
  if (avg >= 24) k_spmv<32><<<grid, 256, 0, st>>>(ptr, idx, val, rows, v, out, ctrl);
  else if (avg >= 12) k_spmv<16><<<grid, 256, 0, st>>>(ptr, idx, val, rows, v, out, ctrl);
  else if (avg >= 6) k_spmv<8><<<grid, 256, 0, st>>>(ptr, idx, val, rows, v, out, ctrl);
  else k_spmv<4><<<grid, 256, 0, st>>>(ptr, idx, val, rows, v, out, ctrl);
  return cudaGetLastError();
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
  dfree(csr->tvec);
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
  c->gb_smem = (size_t)maxband * sizeof(double);
  c->hr_smem = (size_t)HR_WARPS * (tau + 32) * sizeof(double) + (size_t)HR_WARPS * ((tau + 31) / 32) * 4;
  RS_CUDA(cudaFuncSetAttribute(k_gram_bands, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)std::max<size_t>(c->gb_smem, 48 * 1024)));
  RS_CUDA(cudaFuncSetAttribute(k_hash_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)std::max<size_t>(c->hr_smem, 48 * 1024)));
  RS_CUDA(cudaStreamSynchronize(st));
  if (std::getenv("RS_VERBOSE"))
    fprintf(stderr, "[rs] csr gram: tau %d, %d bands (max %lld doubles), %d chunks\n", tau,
            c->nbands, maxband, c->nchunks);
  return RS_OK;
}

// One iteration of Alg. 2 in CSR GRAM mode (sketch already drawn by the caller).
rs_status Problem::csr_enqueue_gram(const rs_solve_opts* o, cudaEvent_t* ev) {
  auto mark = [&](int cls, int edge) {
    if (ev) cudaEventRecordWithFlags(ev[2 * cls + edge], st, cudaEventRecordExternal);
  };
  CsrData* c = csr;
  const RView R = route == 1 ? RView{c->rowptr, c->colidx, c->vals, c->rows}
                             : RView{c->colptr, c->rowidx, c->cvals, c->cols};
  const RView Rt = route == 1 ? RView{c->colptr, c->rowidx, c->cvals, c->cols}
                              : RView{c->rowptr, c->colidx, c->vals, c->rows};
  const int tau = sk.tau;
  mark(RS_K_XS, 0);
  const int* cmap = sk.cmap;
  if (sk.kind != SK_COUNT) {
    RS_CUDA(launch_cmap_build(sk, c->cmap_all, m, ctrl, st));
    cmap = c->cmap_all;
  }
  if (R.rows > 0) {   // a2: rows of R S, merged and bucket-sorted
    const unsigned grid = (unsigned)std::max<long long>(
        1, std::min<long long>((R.rows + HR_WARPS - 1) / HR_WARPS, (long long)num_sms * 8));
    k_hash_rows<<<grid, HR_WARPS * 32, c->hr_smem, st>>>(R.ptr, R.idx, R.val, R.rows, cmap, tau,
                                                          c->hb, c->hv, c->hcnt, ctrl);
    RS_CUDA(cudaGetLastError());
  }
  mark(RS_K_XS, 1);
  mark(RS_K_GRAM, 0);
  if (R.rows > 0) {   // a3/a4: (R S)^T (R S), lower triangle
    k_gram_bands<<<dim3((unsigned)c->nbands, (unsigned)c->nchunks), GB_THREADS, c->gb_smem, st>>>(
        R.ptr, c->hcnt, c->hb, c->hv, c->band_a0, c->chunk_r0, c->gpart, c->gpart_stride, ctrl);
    RS_CUDA(cudaGetLastError());
    k_gram_band_reduce<<<tau, 256, 0, st>>>(c->gpart, c->nchunks, c->gpart_stride, Gram, ld_gram, ctrl);
    RS_CUDA(cudaGetLastError());
  } else {
    RS_CUDA(launch_fill(Gram, (long long)tau * ld_gram, 0.0, st));
  }
  RS_TRY(allreduce(Gram, (size_t)tau * ld_gram));
  mark(RS_K_GRAM, 1);
  mark(RS_K_SOLVE, 0);
  RS_CUDA(launch_sketched_solve(nullptr, 0, false, Gram, ld_gram, lambda, r, sk, sw, sdelta, ctrl,
                                st));                                              // a4 + a5
  mark(RS_K_SOLVE, 1);
  mark(RS_K_AS, 0);   // u = R^T (R (S delta)), summed over ranks
  RS_CUDA(launch_spmv(R.ptr, R.idx, R.val, R.rows, c->nnz, sdelta, c->tvec, num_sms, ctrl, st));
  RS_CUDA(launch_spmv(Rt.ptr, Rt.idx, Rt.val, Rt.rows, c->nnz, c->tvec, uvec, num_sms, ctrl, st));
  RS_TRY(allreduce(uvec, (size_t)m));
  mark(RS_K_AS, 1);
  mark(RS_K_UPDATE, 0);
  RS_CUDA(launch_update_vec(uvec, lambda, sdelta, w, dw, r, dr, m, o->gamma, o->beta, partials,
                            ctrl, st));                                          // a6 + a7
  mark(RS_K_UPDATE, 1);
  return RS_OK;
}

}  // namespace rs
