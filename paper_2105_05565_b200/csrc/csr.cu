// CSR-X kernels of the hot path (SURVEY §8(a) rows a2 + a3 for sparse X; BASELINE.json c3, c4).
//
// Primal (c3): m = d, AS = X^T (X S) + lambda S stored row-major (m x tau).
//   One warp owns one output coordinate j (a row of AS): it walks column j of X (CSC), and for every
//   row i of that column walks row i (CSR), adding X_ij * sign(j') * X_ij' into acc[bucket(j')] for
//   every sketched coordinate j' of the row -- X S is never formed (its rows share X's pattern,
//   P:L341 "cost O(nnz(A))").  acc lives in shared memory.
// Dual (c4): m = n, AS = X (X^T S) + lambda S stored row-major (n x tau).
//   A CTA owns a group of B buckets and a chunk of rows.  For each bucket b it builds, in shared
//   memory, the sparse vector z_b = X^T S[:, b] = sum_{e in b} sign_e X_{coord_e,:} as an
//   open-addressing hash table (entries of a bucket are inserted one row after another, so every
//   value is a fixed-order sum); then every row i of the chunk is dotted with the B tables by one
//   warp: AS[i, b] = <X_i, z_b> (lanes over the row's non-zeros, warp-shuffle reduction).
//   Row-owned outputs: no atomics on the result, deterministic.
// Setup: the CSC copy of X is built on the device with a stable CUB radix sort of the column
// indices (a library sort primitive), so every column lists its rows in ascending order.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <string>

#include "csr.h"
#include "engine.h"
#include "nccl_dl.h"
#include "rs_internal.cuh"

namespace rs {



namespace {

// --------------------------------------------------------------------------------- setup kernels
__global__ void k_csr_validate(const long long* rowptr, const int* colidx, long long rows,
                               long long cols, long long nnz, unsigned long long* bad) {
  unsigned long long b = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (long long)gridDim.x * blockDim.x) {
    const long long a = rowptr[i], e = rowptr[i + 1];
    if (a > e || a < 0 || e > nnz) { ++b; continue; }
    for (long long q = a; q < e; ++q) {
      const int c = colidx[q];
      if (c < 0 || c >= cols) ++b;
      if (q > a && colidx[q - 1] >= c) ++b;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (rowptr[0] != 0 || rowptr[rows] != nnz)) ++b;
  if (b) atomicAdd(bad, b);
}

__global__ void k_row_of(const long long* rowptr, long long rows, int* row_of, long long* maxnnz) {
  long long mx = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (long long)gridDim.x * blockDim.x) {
    const long long a = rowptr[i], e = rowptr[i + 1];
    for (long long q = a; q < e; ++q) row_of[q] = (int)i;
    mx = max(mx, e - a);
  }
  atomicMax(reinterpret_cast<unsigned long long*>(maxnnz), (unsigned long long)mx);
}

__global__ void k_iota(int* p, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = (int)i;
}

// after the stable sort by column: perm[q] = original nnz index of the q-th CSC entry
__global__ void k_csc_fill(const int* perm, const int* row_of, const double* vals, int* rowidx,
                           double* cvals, long long nnz) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < nnz;
       q += (long long)gridDim.x * blockDim.x) {
    const int e = perm[q];
    rowidx[q] = row_of[e];
    cvals[q] = vals[e];
  }
}

// inv[perm[q]] = q
__global__ void k_inv_perm(const int* perm, int* inv, long long n) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x)
    inv[perm[q]] = (int)q;
}

// colptr[c] = first q with sorted_col[q] >= c  (binary search), c in [0, cols]
__global__ void k_colptr(const int* sorted_col, long long nnz, long long cols, long long* colptr) {
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c <= cols;
       c += (long long)gridDim.x * blockDim.x) {
    long long lo = 0, hi = nnz;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (sorted_col[mid] < c) lo = mid + 1;
      else hi = mid;
    }
    colptr[c] = lo;
  }
}

// out[c] = sum_{q in column c} cvals[q] * v[rowidx[q]]   (X^T v via CSC, deterministic)
__global__ void k_csc_spmv_t(const long long* colptr, const int* rowidx, const double* cvals,
                             long long cols, const double* v, double* out) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long c = warp; c < cols; c += nw) {
    double s = 0.0;
    for (long long q = colptr[c] + lane; q < colptr[c + 1]; q += 32) s += cvals[q] * v[rowidx[q]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[c] = s;
  }
}

// ------------------------------------------------------------------------------ per-iteration
// primal: per-coordinate sketch map for subsample / SubCount (count uses its own cmap)
__global__ void k_cmap_clear(int* cmap, long long m, const Ctrl* ctrl, int slot = 0) {
  if (slot_unused(ctrl, slot)) return;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x)
    cmap[i] = -1;
}
__global__ void k_cmap_scatter(DevSketch sk, int* cmap, const Ctrl* ctrl, int slot = 0) {
  if (slot_unused(ctrl, slot)) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < sk.len) cmap[sk.coord[e]] = (sk.bucket[e] << 1) | (sk.sign[e] < 0 ? 1 : 0);
}

// primal AS rows: warp per coordinate j; acc[tau] per warp in shared memory.
constexpr int P_WARPS = 8;
__global__ void __launch_bounds__(P_WARPS * 32)
k_csr_primal_as(const long long* __restrict__ colptr, const int* __restrict__ rowidx,
                const double* __restrict__ cvals, const long long* __restrict__ rowptr,
                const int* __restrict__ colidx, const double* __restrict__ vals,
                const int* __restrict__ cmap, long long m, int tau, double* __restrict__ AS,
                long long ld_as, const Ctrl* ctrl) {
  if (ctrl->done) return;
  extern __shared__ double pacc[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* acc = pacc + (size_t)warp * tau;
  for (int b = lane; b < tau; b += 32) acc[b] = 0.0;
  __syncwarp();
  const long long nw = (long long)gridDim.x * P_WARPS;
  for (long long j = (long long)blockIdx.x * P_WARPS + warp; j < m; j += nw) {
    const long long c0 = colptr[j], c1 = colptr[j + 1];
    for (long long q = c0; q < c1; ++q) {
      const int i = rowidx[q];
      const double xij = cvals[q];
      const long long r0 = rowptr[i], r1 = rowptr[i + 1];
      for (long long t = r0 + lane; t < r1; t += 32) {
        const int cm = __ldg(cmap + colidx[t]);
        if (cm >= 0) {
          const double v = xij * vals[t];
          atomicAdd(&acc[cm >> 1], (cm & 1) ? -v : v);
        }
      }
    }
    __syncwarp();
    double* out = AS + j * ld_as;
    for (int b = lane; b < tau; b += 32) {
      out[b] = acc[b];
      acc[b] = 0.0;
    }
    __syncwarp();
  }
}

// dual AS: CTA per (bucket group, row chunk).  Hash tables: keys int (-1 empty), vals double.
constexpr int D_THREADS = 512;
__device__ __forceinline__ unsigned hslot(int key, int log2) {
  return ((unsigned)key * 0x9E3779B1u) >> (32 - log2);
}
__global__ void __launch_bounds__(D_THREADS)
k_csr_dual_as(const long long* __restrict__ rowptr, const int* __restrict__ colidx,
              const double* __restrict__ vals, long long rows, DevSketch sk, int group,
              int chunk_rows, int log2slots, double* __restrict__ AS, long long ld_as,
              Ctrl* ctrl) {
  if (ctrl->done) return;
  Ctrl* ctrl_err = ctrl;
  extern __shared__ double dsm_d[];
  const int slots = 1 << log2slots;
  const int tau = sk.tau;
  const int b0 = blockIdx.x * group;
  const int nb = min(group, tau - b0);
  double* hv = dsm_d;                                          // [group][slots]
  int* hk = reinterpret_cast<int*>(dsm_d + (size_t)group * slots);   // [group][slots]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int q = tid; q < group * slots; q += D_THREADS) {
    hk[q] = -1;
    hv[q] = 0.0;
  }
  __syncthreads();
  // build z_b for each bucket of the group, entries in order (fixed-order sums)
  for (int g = 0; g < nb; ++g) {
    const int b = b0 + g;
    int* keys = hk + g * slots;
    double* hvals = hv + g * slots;
    for (int e = sk.bptr[b]; e < sk.bptr[b + 1]; ++e) {
      const int c = sk.coord[e];
      const double sg = sk.sign[e] > 0 ? 1.0 : -1.0;
      for (long long t = rowptr[c] + tid; t < rowptr[c + 1]; t += D_THREADS) {
        const int key = colidx[t];
        unsigned s = hslot(key, log2slots);
        int probes = 0;
        for (; probes < slots - 1; ++probes) {   // keep >= 1 empty slot: lookups terminate
          const int prev = atomicCAS(&keys[s], -1, key);
          if (prev == -1 || prev == key) break;
          s = (s + 1) & (slots - 1);
        }
        if (probes == slots - 1) {
          ctrl_err->status = ST_OVERFLOW;   // table full: reported as RS_EUNSUPPORTED
        } else {
          hvals[s] += sg * vals[t];   // keys are distinct within one row: no race
        }
      }
      __syncthreads();
    }
  }
  // probe: warp per row
  const long long i0 = (long long)blockIdx.y * chunk_rows;
  const long long i1 = min(rows, i0 + chunk_rows);
  for (long long i = i0 + warp; i < i1; i += D_THREADS / 32) {
    double acc[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) acc[g] = 0.0;
    for (long long t = rowptr[i] + lane; t < rowptr[i + 1]; t += 32) {
      const int key = colidx[t];
      const double x = vals[t];
      const unsigned s0 = hslot(key, log2slots);
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        if (g < nb) {
          const int* keys = hk + g * slots;
          unsigned s = s0;
          int k;
          while ((k = keys[s]) != key && k != -1) s = (s + 1) & (slots - 1);
          if (k == key) acc[g] += x * hv[g * slots + s];
        }
      }
    }
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      if (g < nb) {
        double v = acc[g];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[g] = v;
      }
    }
    if (lane < nb) {
      double v = 0.0;
#pragma unroll
      for (int g = 0; g < 8; ++g)
        if (g == lane) v = acc[g];
      AS[i * ld_as + b0 + lane] = v;
    }
  }
}

}  // namespace

cudaError_t launch_cmap_build(const DevSketch& sk, int* cmap_all, long long m, const Ctrl* ctrl,
                              cudaStream_t st, int slot) {
  k_cmap_clear<<<(unsigned)std::min<long long>((m + 255) / 256, 1024), 256, 0, st>>>(cmap_all, m, ctrl,
                                                                                     slot);
  k_cmap_scatter<<<(sk.len + 255) / 256, 256, 0, st>>>(sk, cmap_all, ctrl, slot);
  return cudaGetLastError();
}

// ================================================================================================
void Problem::csr_free() {
  if (!csr) return;
  dfree(csr->rowptr);
  dfree(csr->colidx);
  dfree(csr->vals);
  dfree(csr->colptr);
  dfree(csr->rowidx);
  dfree(csr->cvals);
  dfree(csr->cmap_all);
  dfree(csr->cscpos);
  delete csr;
  csr = nullptr;
}

void Problem::csr_free_workspace() {
  if (!csr) return;
  dfree(csr->cmap_all);
  csr->cmap_all = nullptr;
  csr_gram_free();
}

rs_status Problem::csr_ensure_workspace(int kind, int tau, int ksum) {
  (void)ksum;
  if (mode == RS_AS_GRAM) return csr_gram_workspace(kind, tau);
  if (route == 1) {
    if (kind != SK_COUNT) RS_TRY(dalloc(&csr->cmap_all, m));
    const size_t smem = (size_t)P_WARPS * tau * sizeof(double);
    if (smem > 200 * 1024) return fail(RS_EUNSUPPORTED, "CSR primal: tau too large for shared accumulators");
    RS_CUDA(cudaFuncSetAttribute(k_csr_primal_as, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(smem, 48 * 1024)));
  } else {
    // hash capacity: >= 2 x (entries per bucket) x (max row nnz), power of two (count: twice the
    // mean bucket size as the cap; a fuller bucket is reported as ST_OVERFLOW, never a hang)
    const long long per_bucket = kind == SK_COUNT ? 2 * ((m + tau - 1) / tau) + 8
                                                  : (long long)sk.len / tau;
    long long need = std::max<long long>(64, 2 * per_bucket * std::max<long long>(1, csr->max_row_nnz));
    int lg = 6;
    while ((1LL << lg) < need) ++lg;
    const size_t per_table = (size_t)(1LL << lg) * (sizeof(double) + sizeof(int));
    const size_t budget = 200 * 1024;
    if (per_table > budget)
      return fail(RS_EUNSUPPORTED, "CSR dual: sketched rows too dense for shared-memory hash tables");
    int group = (int)std::min<size_t>(8, budget / per_table);
    group = std::max(1, std::min(group, tau));
    csr->hash_log2 = lg;
    csr->hash_slots = 1 << lg;
    csr->group = group;
    const long long ngroups = (tau + group - 1) / group;
    long long chunks = std::max<long long>(1, (2LL * num_sms + ngroups - 1) / ngroups);
    chunks = std::min<long long>(chunks, std::max<long long>(1, csr->rows / 64));
    csr->chunks = (int)chunks;
    csr->dual_smem = (size_t)group * per_table;
    RS_CUDA(cudaFuncSetAttribute(k_csr_dual_as, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(csr->dual_smem, 48 * 1024)));
  }
  return RS_OK;
}

rs_status Problem::csr_enqueue_as(const rs_solve_opts* o, cudaEvent_t* ev) {
  (void)o;
  auto mark = [&](int cls, int edge) {
    if (ev) cudaEventRecordWithFlags(ev[2 * cls + edge], st, cudaEventRecordExternal);
  };
  const int tau = sk.tau;
  if (route == 1) {
    const int* cmap = sk.cmap;
    mark(RS_K_XS, 0);
    if (sk.kind != SK_COUNT) {
      k_cmap_clear<<<(unsigned)std::min<long long>((m + 255) / 256, 1024), 256, 0, st>>>(csr->cmap_all, m, ctrl);
      k_cmap_scatter<<<(sk.len + 255) / 256, 256, 0, st>>>(sk, csr->cmap_all, ctrl);
      cmap = csr->cmap_all;
    }
    RS_CUDA(cudaGetLastError());
    mark(RS_K_XS, 1);
    mark(RS_K_AS, 0);
    const size_t smem = (size_t)P_WARPS * tau * sizeof(double);
    const unsigned grid = (unsigned)std::min<long long>((m + P_WARPS - 1) / P_WARPS, (long long)num_sms * 8);
    k_csr_primal_as<<<grid, P_WARPS * 32, smem, st>>>(csr->colptr, csr->rowidx, csr->cvals,
                                                       csr->rowptr, csr->colidx, csr->vals, cmap,
                                                       m, tau, ASt, ld_as, ctrl);
    RS_CUDA(cudaGetLastError());
  } else {
    mark(RS_K_AS, 0);
    const int ngroups = (tau + csr->group - 1) / csr->group;
    const int chunk_rows = (int)((csr->rows + csr->chunks - 1) / csr->chunks);
    dim3 grid((unsigned)ngroups, (unsigned)csr->chunks);
    k_csr_dual_as<<<grid, D_THREADS, csr->dual_smem, st>>>(csr->rowptr, csr->colidx, csr->vals,
                                                           csr->rows, sk, csr->group, chunk_rows,
                                                           csr->hash_log2, ASt, ld_as, ctrl);
    RS_CUDA(cudaGetLastError());
  }
  RS_TRY(allreduce(ASt, (size_t)m * ld_as));
  RS_CUDA(launch_add_lambda_s(lambda, sk, ASt, ld_as, true, ctrl, st));
  mark(RS_K_AS, 1);
  return RS_OK;
}

rs_status Problem::csr_dual_weights(double* w_out, cudaMemcpyKind kd) {
  // w = X^T alpha: local column block, then summed into the full d-vector over ranks
  double* wfull = nullptr;
  RS_TRY(dalloc(&wfull, d));
  rs_status s = RS_OK;
  if (launch_fill(wfull, d, 0.0, st) != cudaSuccess) s = fail(RS_ECUDA, "fill");
  if (s == RS_OK) {
    k_csc_spmv_t<<<(unsigned)std::min<long long>((csr->cols * 32 + 255) / 256, 65535), 256, 0, st>>>(
        csr->colptr, csr->rowidx, csr->cvals, csr->cols, w, wfull + csr->col_offset);
    if (cudaGetLastError() != cudaSuccess) s = fail(RS_ECUDA, "dual weights kernel");
  }
  if (s == RS_OK) s = allreduce(wfull, d);
  if (s == RS_OK && cudaMemcpyAsync(w_out, wfull, d * 8, kd, st) != cudaSuccess)
    s = fail(RS_ECUDA, "copy w");
  cudaStreamSynchronize(st);
  dfree(wfull);
  return s;
}

// ------------------------------------------------------------------------------------------------
rs_status create_csr(rs_problem* out, int64_t n, int64_t d, int64_t nnz_local, const int64_t* rowptr,
                     const int32_t* colidx, const double* vals, const double* y, double lambda,
                     rs_route route, rs_as_mode mode, rs_mem mem, const rs_dist* dist) {
  if (!out) return fail(RS_EINVAL, "out is NULL");
  *out = nullptr;
  if (n < 1 || d < 1) return fail(RS_EINVAL, "need n >= 1 and d >= 1");
  if (!(lambda > 0.0) || !std::isfinite(lambda)) return fail(RS_EINVAL, "need finite lambda > 0 (P:L36)");
  if (nnz_local < 0 || nnz_local > 0x7fffffffLL) return fail(RS_EINVAL, "need 0 <= nnz_local < 2^31");
  if (!rowptr || !y || (nnz_local > 0 && (!colidx || !vals))) return fail(RS_EINVAL, "NULL input");
  if (mem != RS_MEM_HOST && mem != RS_MEM_DEVICE_COPY && mem != RS_MEM_DEVICE_BORROW)
    return fail(RS_EINVAL, "bad rs_mem");
  if (route != RS_ROUTE_AUTO && route != RS_ROUTE_PRIMAL && route != RS_ROUTE_DUAL)
    return fail(RS_EINVAL, "bad route");
  if (mode != RS_AS_IMPLICIT && mode != RS_AS_GRAM && mode != RS_AS_EXPLICIT)
    return fail(RS_EINVAL, "bad as_mode");
  const int rt = route == RS_ROUTE_AUTO ? (d <= n ? 1 : 2) : (route == RS_ROUTE_PRIMAL ? 1 : 2);
  RS_TRY(validate_dist(dist, rt == 1 ? n : d));
  const long long rows = rt == 1 ? (dist ? dist->shard_len : n) : n;
  const long long cols = rt == 1 ? d : (dist ? dist->shard_len : d);
  if (rows > 0x7fffffffLL || cols > 0x7fffffffLL) return fail(RS_EUNSUPPORTED, "dimension >= 2^31");

  Problem* p = new Problem();
  auto guard = [&](rs_status s) {
    if (s != RS_OK) delete p;
    return s;
  };
  rs_status s = setup_common(p, dist);
  if (s != RS_OK) return guard(s);
  p->fmt = 1;
  p->route = rt;
  p->mode = mode;
  p->n = n;
  p->d = d;
  p->m = rt == 1 ? d : n;
  p->lambda = lambda;
  p->csr = new CsrData();
  CsrData* c = p->csr;
  c->rows = rows;
  c->cols = cols;
  c->nnz = nnz_local;
  c->col_offset = (rt == 2 && dist) ? dist->shard_begin : 0;
  cudaStream_t st = p->st;
  // copies (the CSR arrays are always library-owned: the CSC build needs scratch anyway)
  s = dalloc(&c->rowptr, rows + 1);
  if (s == RS_OK) s = dalloc(&c->colidx, nnz_local);
  if (s == RS_OK) s = dalloc(&c->vals, nnz_local);
  if (s != RS_OK) return guard(s);
  const cudaMemcpyKind kd = kind_of(mem);
  if (cudaMemcpyAsync(c->rowptr, rowptr, (rows + 1) * 8, kd, st) != cudaSuccess ||
      (nnz_local && cudaMemcpyAsync(c->colidx, colidx, nnz_local * 4, kd, st) != cudaSuccess) ||
      (nnz_local && cudaMemcpyAsync(c->vals, vals, nnz_local * 8, kd, st) != cudaSuccess))
    return guard(fail(RS_ECUDA, "copy CSR"));
  const long long ylen = rt == 1 ? rows : n;
  s = dalloc(&p->y, ylen);
  if (s != RS_OK) return guard(s);
  if (cudaMemcpyAsync(p->y, y, ylen * 8, kd, st) != cudaSuccess) return guard(fail(RS_ECUDA, "copy y"));
  // validation
  {
    unsigned long long* bad = nullptr;
    s = dalloc(&bad, 1);
    if (s != RS_OK) return guard(s);
    cudaMemsetAsync(bad, 0, 8, st);
    k_csr_validate<<<(unsigned)std::min<long long>((rows + 255) / 256, 4096), 256, 0, st>>>(
        c->rowptr, c->colidx, rows, cols, nnz_local, bad);
    launch_count_nonfinite(c->vals, 1, nnz_local, 1, bad, st);
    launch_count_nonfinite(p->y, 1, ylen, 1, bad, st);
    unsigned long long h = 0;
    cudaMemcpyAsync(&h, bad, 8, cudaMemcpyDeviceToHost, st);
    cudaError_t ce = cudaStreamSynchronize(st);
    dfree(bad);
    if (ce != cudaSuccess) return guard(fail(RS_ECUDA, cudaGetErrorString(ce)));
    if (h) return guard(fail(RS_EINVAL, "CSR invariants violated or non-finite values"));
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  // CSC via stable radix sort of the column indices
  {
    int *row_of = nullptr, *perm_in = nullptr, *perm_out = nullptr, *keys_out = nullptr;
    long long* mx = nullptr;
    s = dalloc(&row_of, nnz_local);
    if (s == RS_OK) s = dalloc(&perm_in, nnz_local);
    if (s == RS_OK) s = dalloc(&perm_out, nnz_local);
    if (s == RS_OK) s = dalloc(&keys_out, nnz_local);
    if (s == RS_OK) s = dalloc(&mx, 1);
    if (s == RS_OK) s = dalloc(&c->colptr, cols + 1);
    if (s == RS_OK) s = dalloc(&c->rowidx, nnz_local);
    if (s == RS_OK) s = dalloc(&c->cvals, nnz_local);
    if (s != RS_OK) return guard(s);
    cudaMemsetAsync(mx, 0, 8, st);
    k_row_of<<<(unsigned)std::min<long long>((rows + 255) / 256, 4096), 256, 0, st>>>(c->rowptr, rows, row_of, mx);
    k_iota<<<4096, 256, 0, st>>>(perm_in, nnz_local);
    size_t tmp_bytes = 0;
    int end_bit = 1;
    while (end_bit < 31 && (1LL << end_bit) <= cols) ++end_bit;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, c->colidx, keys_out, perm_in, perm_out,
                                    (int)nnz_local, 0, end_bit, st);
    void* tmp = nullptr;
    s = dalloc(reinterpret_cast<char**>(&tmp), tmp_bytes);
    if (s != RS_OK) return guard(s);
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, c->colidx, keys_out, perm_in, perm_out,
                                    (int)nnz_local, 0, end_bit, st);
    k_csc_fill<<<4096, 256, 0, st>>>(perm_out, row_of, c->vals, c->rowidx, c->cvals, nnz_local);
    if (rt == 2 && mode == RS_AS_GRAM && nnz_local > 0) {   // R entry of every X entry (csr_gram.cu)
      s = dalloc(&c->cscpos, nnz_local);
      if (s != RS_OK) return guard(s);
      k_inv_perm<<<4096, 256, 0, st>>>(perm_out, c->cscpos, nnz_local);
    }
    k_colptr<<<(unsigned)std::min<long long>((cols + 256) / 256, 65535), 256, 0, st>>>(keys_out, nnz_local, cols, c->colptr);
    cudaMemcpyAsync(&c->max_row_nnz, mx, 8, cudaMemcpyDeviceToHost, st);
    cudaError_t ce = cudaStreamSynchronize(st);
    dfree(row_of);
    dfree(perm_in);
    dfree(perm_out);
    dfree(keys_out);
    dfree(mx);
    dfree(tmp);
    if (ce != cudaSuccess) return guard(fail(RS_ECUDA, std::string("CSC build: ") + cudaGetErrorString(ce)));
  }
  // b: primal b = X^T y summed over row shards; dual b = y
  s = dalloc(&p->b, p->m);
  if (s != RS_OK) return guard(s);
  if (rt == 1) {
    k_csc_spmv_t<<<(unsigned)std::min<long long>((cols * 32 + 255) / 256, 65535), 256, 0, st>>>(
        c->colptr, c->rowidx, c->cvals, cols, p->y, p->b);
    s = p->allreduce(p->b, p->m);
    if (s != RS_OK) return guard(s);
  } else {
    cudaMemcpyAsync(p->b, p->y, n * 8, cudaMemcpyDeviceToDevice, st);
  }
  if (mode == RS_AS_EXPLICIT) {   // dense A = R^T R + lambda I from the sparse X
    s = p->csr_build_explicit();
    if (s != RS_OK) return guard(s);
  }
  cudaEventRecord(e1, st);
  s = finish_setup(p);
  if (s != RS_OK) return guard(s);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  p->setup_seconds = ms * 1e-3;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) return guard(fail(RS_ECUDA, cudaGetErrorString(ce)));
  *out = reinterpret_cast<rs_problem>(p);
  return RS_OK;
}

}  // namespace rs
