// EXPLICIT mode for CSR X ("sparse explicit A"): the dense m x m matrix
//   A = R^T R + lambda I,   R = X (primal, m = d) or X^T (dual, m = n)        (Eq. Axb)
// is built once in rs_create_csr, after which the EXPLICIT iteration (sketch-ahead gathers of the
// sketched rows of A, batched factorisation, split-row update) runs unchanged.  R^T R is the sum
// of the outer products r_i r_i^T of R's rows ("O(nnz)" per row pair):
//   heavy rows (nnz > RX_HEAVY; c4: the Zipf-popular features) are scattered into a dense
//     |H| x m block R_H and contracted on the FP64 tensor cores, R_H^T R_H on the lower-triangle
//     tiles of the TMA DMMA GEMM (their outer products are dense: ~(2e4)^2 entries each);
//   light rows add their lower-triangle pairs (col_s >= col_t) with fp64 reductions to global
//     memory (RED.ADD.F64 in L2; summation order not fixed, rounding varies in the last bits);
// then the upper triangle is mirrored and lambda added on the diagonal.  Multi-rank: each rank
// builds its shard's R_p^T R_p and the partials are summed with one allreduce.
#include <algorithm>
#include <string>
#include <vector>

#include "csr.h"
#include "engine.h"
#include "rs_internal.cuh"

namespace rs {

namespace {

constexpr long long RX_HEAVY = 64;

__global__ void k_heavy_dense(const long long* __restrict__ ptr, const int* __restrict__ idx,
                              const double* __restrict__ val, const int* __restrict__ hrows,
                              double* __restrict__ RH, long long ld) {
  const long long i = hrows[blockIdx.x];
  double* out = RH + (long long)blockIdx.x * ld;
  for (long long q = ptr[i] + threadIdx.x; q < ptr[i + 1]; q += blockDim.x) out[idx[q]] = val[q];
}

// light rows: warp per row, lanes over the pairs (s, t), t <= s (columns ascending within a row)
__global__ void k_light_outer(const long long* __restrict__ ptr, const int* __restrict__ idx,
                              const double* __restrict__ val, long long rows, long long heavy,
                              double* __restrict__ A, long long lda) {
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < rows; i += nw) {
    const long long a = ptr[i], L = ptr[i + 1] - a;
    if (L == 0 || L > heavy) continue;
    const long long np = L * (L + 1) / 2;
    int s = 0, t = lane;
    while (t > s) { t -= s + 1; ++s; }
    for (long long p = lane; p < np; p += 32) {
      const long long cs = idx[a + s], ct = idx[a + t];
      atomicAdd(&A[cs * lda + ct], val[a + s] * val[a + t]);
      t += 32;
      while (t > s) { t -= s + 1; ++s; }
    }
  }
}

__global__ void k_heavy_rows_list(const long long* __restrict__ ptr, long long rows, long long heavy,
                                  int* __restrict__ list, int* __restrict__ count) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (long long)gridDim.x * blockDim.x)
    if (ptr[i + 1] - ptr[i] > heavy) list[atomicAdd(count, 1)] = (int)i;
}

}  // namespace

rs_status Problem::csr_build_explicit() {
  CsrData* c = csr;
  struct { const long long* ptr; const int* idx; const double* val; long long rows; } R;
  if (route == 1) R = {c->rowptr, c->colidx, c->vals, c->rows};
  else R = {c->colptr, c->rowidx, c->cvals, c->cols};
  lda = round_up(m, 4);
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  if ((double)m * lda * 8.0 > 0.8 * (double)free_b)
    return fail(RS_ENOMEM, "CSR explicit A: m x m doubles exceed the free device memory");
  RS_TRY(dalloc(&A, (size_t)m * lda));
  RS_CUDA(cudaMemsetAsync(A, 0, (size_t)m * lda * sizeof(double), st));
  // heavy rows -> dense block -> lower tiles of R_H^T R_H
  int* list = nullptr;
  int* cnt = nullptr;
  RS_TRY(dalloc(&list, std::max<long long>(1, R.rows)));
  RS_TRY(dalloc(&cnt, 1));
  RS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), st));
  if (R.rows > 0)
    k_heavy_rows_list<<<(unsigned)std::min<long long>((R.rows + 255) / 256, 4096), 256, 0, st>>>(
        R.ptr, R.rows, RX_HEAVY, list, cnt);
  int nh = 0;
  RS_CUDA(cudaMemcpyAsync(&nh, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
  RS_CUDA(cudaStreamSynchronize(st));
  rs_status s = RS_OK;
  if (nh > 0) {
    std::vector<int> hl(nh);   // ascending heavy rows: a deterministic K order for the GEMM
    RS_CUDA(cudaMemcpy(hl.data(), list, nh * sizeof(int), cudaMemcpyDeviceToHost));
    std::sort(hl.begin(), hl.end());
    RS_CUDA(cudaMemcpy(list, hl.data(), nh * sizeof(int), cudaMemcpyHostToDevice));
    double* RH = nullptr;
    s = dalloc(&RH, (size_t)nh * lda);
    if (s == RS_OK) {
      cudaMemsetAsync(RH, 0, (size_t)nh * lda * sizeof(double), st);
      k_heavy_dense<<<nh, 256, 0, st>>>(R.ptr, R.idx, R.val, list, RH, lda);
      TmaGemm tg{};
      double* work = nullptr;
      cudaError_t ce = tma_gemm_plan(&tg, RH, lda, RH, lda, m, m, nh, num_sms, 1);
      tg.lower = 1;
      if (std::getenv("RS_VERBOSE"))
        fprintf(stderr, "[rs] csr explicit heavy GEMM: M %lld K %d, variant %d (%dx%d), splits %d\n", m, nh,
                tg.variant, tg.bm, tg.bn, tg.splits);
      if (ce == cudaSuccess && tg.work_elems) s = dalloc(&work, tg.work_elems);
      if (s == RS_OK && ce == cudaSuccess) ce = tma_gemm_launch(tg, A, lda, work, nullptr, st);
      cudaStreamSynchronize(st);
      dfree(work);
      if (s == RS_OK && ce != cudaSuccess) s = fail(RS_ECUDA, std::string("R_H^T R_H: ") + cudaGetErrorString(ce));
    }
    dfree(RH);
  }
  dfree(list);
  dfree(cnt);
  if (s != RS_OK) return s;
  if (std::getenv("RS_VERBOSE"))
    fprintf(stderr, "[rs] csr explicit A: m %lld, heavy rows %d (> %lld nnz) on DMMA\n", m, nh, RX_HEAVY);
  // light rows: lower-triangle pairs by fp64 reductions
  if (R.rows > 0) {
    const unsigned grid = (unsigned)std::min<long long>((R.rows * 32 + 255) / 256, (long long)num_sms * 32);
    k_light_outer<<<grid, 256, 0, st>>>(R.ptr, R.idx, R.val, R.rows, RX_HEAVY, A, lda);
    RS_CUDA(cudaGetLastError());
  }
  RS_CUDA(launch_mirror_lower(A, lda, m, st));
  RS_TRY(allreduce(A, (size_t)m * lda));
  RS_CUDA(launch_add_diag(A, lda, m, lambda, st));
  RS_CUDA(cudaStreamSynchronize(st));
  return RS_OK;
}

}  // namespace rs
