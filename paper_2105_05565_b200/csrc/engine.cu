// Host engine behind the C ABI (include/ridgesketch.h): argument validation, the problem object,
// device memory, the per-iteration launch sequence captured in a CUDA graph, the device stop flag,
// NCCL for world > 1.  No arithmetic of the method runs on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ridgesketch.h"
#include "engine.h"
#include "nccl_dl.h"
#include "rs_internal.cuh"

namespace rs {

thread_local std::string g_last_error;

rs_status fail(rs_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}



// ------------------------------------------------------------------------------------------------
Problem::~Problem() {
  if (device >= 0) cudaSetDevice(device);
  if (st) cudaStreamSynchronize(st);
  free_workspace();
  dfree(XT);
  if (st2) cudaStreamDestroy(st2);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (ev_pro) cudaEventDestroy(ev_pro);
  if (ev_pro_tail) cudaEventDestroy(ev_pro_tail);
  if (own_X) dfree(X);
  if (own_Xo) dfree(Xo);
  dfree(y);
  dfree(b);
  dfree(A);
  dfree(w);
  dfree(dw);
  dfree(r);
  dfree(dr);
  dfree(sdelta);
  dfree(ctrl);
  dfree(trace_dev);
  dfree(mom_tab_dev);
  dfree(scratch);
  csr_free();
  if (ctrl_host) cudaFreeHost(ctrl_host);
  if (comm) {
    std::string err;
    if (const NcclApi* api = nccl_api(&err)) api->ncclCommDestroy(comm);
  }
  hostcoll_destroy(hcoll);
  if (own_stream && st) cudaStreamDestroy(st);
}

void Problem::free_workspace() {
  if (graph_exec) cudaGraphExecDestroy(graph_exec);
  graph_exec = nullptr;
  for (auto ev : prof_events) cudaEventDestroy(ev);
  prof_events.clear();
  dfree(sk.coord);
  dfree(sk.sign);
  dfree(sk.bucket);
  dfree(sk.bptr);
  dfree(sk.cmap);
  sk = DevSketch{};
  dfree(XS);
  XS = nullptr;
  dfree(Gram);
  Gram = nullptr;
  dfree(xp_part);
  xp_part = nullptr;
  dfree(uvec);
  uvec = nullptr;
  dfree(ASt);
  ASt = nullptr;
  dfree(gemm_work);
  gemm_work = nullptr;
  dfree(sw.Gx);
  dfree(sw.delta);
  sw = SolveWork{};
  dfree(partials);
  partials = nullptr;
  dfree(skb.coord);
  dfree(skb.sign);
  dfree(skb.bucket);
  dfree(skb.bptr);
  dfree(skb.cmap);
  skb = DevSketch{};
  dfree(ASt_slots);
  ASt_slots = nullptr;
  dfree(Gram_slots);
  Gram_slots = nullptr;
  dfree(Ginv_slots);
  Ginv_slots = nullptr;
  dfree(slot_flags);
  slot_flags = nullptr;
  dfree(bf_work);
  bf_work = nullptr;
  dfree(bf_claim);
  bf_claim = nullptr;
  dfree(it_scratch);
  it_scratch = nullptr;
  use_iterate = false;
  pipe_xg = false;
  ws_xg = -1;
  pipe = false;
  P = 0;
  ws_depth = -1;
  ws_kind = -1;
  ws_tau = -1;
  ws_ksum = -1;
  csr_free_workspace();
}

rs_status Problem::allreduce(double* buf, size_t count) {
  if (world <= 1) return RS_OK;
  if (coll == RS_COLL_HOST) {
    if (!hcoll) return fail(RS_ENCCL, "host collective not attached");
    RS_CUDA(hostcoll_allreduce(hcoll, buf, count, st));
    return RS_OK;
  }
  std::string err;
  const NcclApi* api = nccl_api(&err);
  if (!api) return fail(RS_ENCCL, err);
  ncclResult_t e = api->ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, comm, st);
  if (e != ncclSuccess) {
    api->ncclCommAbort(comm);
    comm = nullptr;
    return fail(RS_ENCCL, std::string("ncclAllReduce: ") + api->ncclGetErrorString(e));
  }
  return RS_OK;
}

// ------------------------------------------------------------------------------------------------
rs_status setup_common(Problem* p, const rs_dist* dist) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(RS_ECUDA, std::string("no usable CUDA device: ") +
                              (e != cudaSuccess ? cudaGetErrorString(e) : "count = 0"));
  p->device = dist ? dist->device : 0;
  if (p->device < 0 || p->device >= ndev) return fail(RS_EINVAL, "dist->device out of range");
  RS_CUDA(cudaSetDevice(p->device));
  RS_CUDA(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, p->device));
  RS_CUDA(sketch_init());
  RS_CUDA(gemm_init());
  RS_CUDA(chol_init());
  RS_CUDA(tma_gemm_init());
  RS_CUDA(gram_init());
  RS_CUDA(bfactor_init());
  RS_CUDA(update_init());
  RS_CUDA(iterate_init());
  if (dist && dist->cuda_stream) {
    p->st = static_cast<cudaStream_t>(dist->cuda_stream);
    p->own_stream = false;
  } else {
    RS_CUDA(cudaStreamCreateWithFlags(&p->st, cudaStreamNonBlocking));
    p->own_stream = true;
  }
  p->rank = dist ? dist->rank : 0;
  p->world = dist ? dist->world : 1;
  p->coll = dist ? dist->collective : RS_COLL_NCCL;
  if (p->world > 1 && p->coll == RS_COLL_HOST) {
    char name[129];
    std::memcpy(name, dist->nccl_unique_id, 128);
    name[128] = 0;
    std::string err;
    p->hcoll = hostcoll_create(name, p->rank, p->world, &err);
    if (!p->hcoll) return fail(RS_ENCCL, "host collective: " + err);
  } else if (p->world > 1) {
    std::string err;
    const NcclApi* api = nccl_api(&err);
    if (!api) return fail(RS_ENCCL, err);
    ncclUniqueId id;
    std::memcpy(&id, dist->nccl_unique_id, sizeof(id));
    ncclResult_t ne = api->ncclCommInitRank(&p->comm, p->world, id, p->rank);
    if (ne != ncclSuccess) {
      p->comm = nullptr;
      return fail(RS_ENCCL, std::string("ncclCommInitRank: ") + api->ncclGetErrorString(ne));
    }
  }
  RS_CUDA(cudaMallocHost(&p->ctrl_host, sizeof(Ctrl)));
  RS_TRY(dalloc(&p->ctrl, 1));
  return RS_OK;
}

rs_status validate_dist(const rs_dist* dist, long long total) {
  if (!dist) return RS_OK;
  if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world)
    return fail(RS_EINVAL, "rs_dist: need 0 <= rank < world");
  if (dist->world > 1 && !dist->nccl_unique_id)
    return fail(RS_EINVAL, "rs_dist: world > 1 needs nccl_unique_id (the group id)");
  if (dist->collective != RS_COLL_NCCL && dist->collective != RS_COLL_HOST)
    return fail(RS_EINVAL, "rs_dist: bad collective");
  if (dist->shard_begin < 0 || dist->shard_len < 0 || dist->shard_begin + dist->shard_len > total)
    return fail(RS_EINVAL, "rs_dist: shard out of range");
  if (dist->world == 1 && (dist->shard_begin != 0 || dist->shard_len != total))
    return fail(RS_EINVAL, "rs_dist: world == 1 must hold the whole matrix");
  return RS_OK;
}


// m-vectors and b-norm (shared by dense and CSR creation)
rs_status finish_setup(Problem* p) {
  RS_TRY(dalloc(&p->w, p->m));
  RS_TRY(dalloc(&p->dw, p->m));
  RS_TRY(dalloc(&p->r, p->m));
  RS_TRY(dalloc(&p->dr, p->m));
  RS_TRY(dalloc(&p->sdelta, p->m));
  RS_CUDA(launch_fill(p->sdelta, p->m, 0.0, p->st));
  RS_TRY(dalloc(&p->scratch, 4));
  RS_CUDA(launch_dot_self(p->b, p->m, p->scratch, p->st));
  RS_CUDA(cudaMemcpyAsync(&p->bnorm2, p->scratch, sizeof(double), cudaMemcpyDeviceToHost, p->st));
  RS_CUDA(cudaStreamSynchronize(p->st));
  return RS_OK;
}

static rs_status create_dense(rs_problem* out, int64_t n, int64_t d, const double* X_local,
                              int64_t ldx, const double* y, double lambda, rs_route route,
                              rs_as_mode mode, rs_mem mem, const rs_dist* dist) {
  if (!out) return fail(RS_EINVAL, "out is NULL");
  *out = nullptr;
  if (n < 1 || d < 1) return fail(RS_EINVAL, "need n >= 1 and d >= 1");
  if (!(lambda > 0.0) || !std::isfinite(lambda)) return fail(RS_EINVAL, "need finite lambda > 0 (P:L36)");
  if (!X_local || !y) return fail(RS_EINVAL, "X and y must be non-NULL");
  if (mem != RS_MEM_HOST && mem != RS_MEM_DEVICE_COPY && mem != RS_MEM_DEVICE_BORROW)
    return fail(RS_EINVAL, "bad rs_mem");
  if (route != RS_ROUTE_AUTO && route != RS_ROUTE_PRIMAL && route != RS_ROUTE_DUAL)
    return fail(RS_EINVAL, "bad route");
  if (mode != RS_AS_IMPLICIT && mode != RS_AS_EXPLICIT && mode != RS_AS_GRAM)
    return fail(RS_EINVAL, "bad as_mode");
  const int rt = route == RS_ROUTE_AUTO ? (d <= n ? 1 : 2) : (route == RS_ROUTE_PRIMAL ? 1 : 2);
  // dense dual in IMPLICIT / GRAM mode: the primal machinery on R = X^T (d x n), whose A = R^T R +
  // lambda I = X X^T + lambda I; feature shards of X are row shards of R
  const bool dual_r = rt == 2 && mode != RS_AS_EXPLICIT;
  if (rt == 2 && mode == RS_AS_EXPLICIT && dist && dist->world > 1)
    return fail(RS_EUNSUPPORTED, "dense dual EXPLICIT route: one GPU in this version");
  if (mode == RS_AS_GRAM && (dual_r ? n : d) > 4096)
    return fail(RS_EUNSUPPORTED, "GRAM mode needs m <= 4096 (the X pass)");
  RS_TRY(validate_dist(dist, rt == 1 ? n : d));
  const long long rows = rt == 1 && dist ? dist->shard_len : n;
  const long long cols = rt == 2 && dist ? dist->shard_len : d;   // columns of the local X block
  if (ldx < cols) return fail(RS_EINVAL, "ldx < columns of the local X block");

  Problem* p = new Problem();
  auto guard = [&](rs_status s) {
    if (s != RS_OK) delete p;
    return s;
  };
  rs_status s = setup_common(p, dist);
  if (s != RS_OK) return guard(s);
  p->fmt = 0;
  p->route = rt;
  p->mode = mode;
  p->n = n;
  p->d = d;
  p->m = rt == 1 ? d : n;   // primal: w in R^d; dual: alpha in R^n
  p->rows_loc = rows;
  p->lambda = lambda;

  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // Host X for an EXPLICIT primal build of >= 2 GB: streamed in row chunks on a copy stream while
  // A = sum_c X_c^T X_c accumulates chunk by chunk on the solver stream (the H2D copy, not the
  // DMMA contraction, bounds rs_create then; c5: 65.5 GB).  setup_seconds covers both.
  const bool streamed = mem == RS_MEM_HOST && mode == RS_AS_EXPLICIT && rt == 1 && rows > 0 &&
                        (double)rows * (double)d * 8.0 >= 2e9;
  // X: library copy with ld a multiple of 4 doubles (16-byte cp.async rows), unless borrowable
  if (mem == RS_MEM_DEVICE_BORROW && ldx % 4 == 0) {
    p->X = const_cast<double*>(X_local);
    p->ldx = ldx;
    p->own_X = false;
  } else {
    p->ldx = round_up(cols, 4);
    s = dalloc(&p->X, (size_t)std::max<long long>(rows, 1) * p->ldx);
    if (s != RS_OK) return guard(s);
    p->own_X = true;
    if (rows > 0 && cols > 0 && !streamed) {
      cudaError_t ce = cudaMemcpy2DAsync(p->X, p->ldx * 8, X_local, ldx * 8, cols * 8, rows,
                                         kind_of(mem), p->st);
      if (ce != cudaSuccess) return guard(fail(RS_ECUDA, std::string("copy X: ") + cudaGetErrorString(ce)));
    }
  }
  s = dalloc(&p->y, std::max<long long>(rows, 1));
  if (s != RS_OK) return guard(s);
  if (rows > 0) {
    cudaError_t ce = cudaMemcpyAsync(p->y, y, rows * 8, kind_of(mem), p->st);
    if (ce != cudaSuccess) return guard(fail(RS_ECUDA, std::string("copy y: ") + cudaGetErrorString(ce)));
  }
  // streamed EXPLICIT build: chunk c's H2D (copy stream) overlaps chunk c-1's lower-tile DMMA
  // contraction (solver stream); the finiteness count runs on each chunk as it lands
  unsigned long long* cnt = nullptr;
  s = dalloc(&cnt, 1);
  if (s != RS_OK) return guard(s);
  cudaMemsetAsync(cnt, 0, 8, p->st);
  if (streamed) {
    p->lda = round_up(d, 4);
    s = dalloc(&p->A, (size_t)d * p->lda);
    double* tacc = nullptr;
    if (s == RS_OK) s = dalloc(&tacc, (size_t)d * p->lda);
    if (s != RS_OK) return guard(s);
    const int nch = (int)std::max<double>(2.0, std::ceil((double)rows * d * 8.0 / 4e9));
    const long long rc = (rows + nch - 1) / nch;
    std::vector<TmaGemm> plans;
    size_t wmax = 0;
    for (long long r0 = 0; r0 < rows; r0 += rc) {
      TmaGemm tgc{};
      const double* Xc = p->X + r0 * p->ldx;
      cudaError_t ce = tma_gemm_plan(&tgc, Xc, p->ldx, Xc, p->ldx, d, d, std::min(rc, rows - r0), p->num_sms, 1);
      if (ce != cudaSuccess) return guard(fail(RS_ECUDA, std::string("A build plan: ") + cudaGetErrorString(ce)));
      tgc.lower = 1;
      wmax = std::max(wmax, tgc.work_elems);
      plans.push_back(tgc);
    }
    double* swork = nullptr;
    if (wmax) s = dalloc(&swork, wmax);
    if (s != RS_OK) return guard(s);
    cudaStream_t cs = nullptr;
    RS_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    std::vector<cudaEvent_t> landed(plans.size());
    for (auto& ev : landed) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(e0, p->st);
    RS_CUDA(cudaStreamWaitEvent(cs, e0, 0));   // y copied, counters cleared
    cudaError_t ce = cudaSuccess;
    for (size_t c = 0; c < plans.size() && ce == cudaSuccess; ++c) {
      const long long r0 = (long long)c * rc, nr = std::min(rc, rows - r0);
      ce = cudaMemcpy2DAsync(p->X + r0 * p->ldx, p->ldx * 8, X_local + r0 * ldx, ldx * 8, d * 8, nr,
                             cudaMemcpyHostToDevice, cs);
      if (ce == cudaSuccess) ce = cudaEventRecord(landed[c], cs);
      if (ce == cudaSuccess) ce = cudaStreamWaitEvent(p->st, landed[c], 0);
      if (ce == cudaSuccess) ce = launch_count_nonfinite(p->X + r0 * p->ldx, p->ldx, nr, d, cnt, p->st);
      if (ce == cudaSuccess) ce = tma_gemm_launch(plans[c], c == 0 ? p->A : tacc, p->lda, swork, nullptr, p->st);
      if (ce == cudaSuccess && c > 0) ce = launch_add_lower(p->A, tacc, p->lda, d, p->st);
    }
    cudaError_t ce2 = cudaStreamSynchronize(p->st);
    for (auto& ev : landed) cudaEventDestroy(ev);
    cudaStreamDestroy(cs);
    dfree(swork);
    dfree(tacc);
    if (ce == cudaSuccess) ce = ce2;
    if (ce != cudaSuccess) return guard(fail(RS_ECUDA, std::string("streamed A build: ") + cudaGetErrorString(ce)));
  }
  // finiteness check of the local data
  {
    if (!streamed) launch_count_nonfinite(p->X, p->ldx, rows, cols, cnt, p->st);
    launch_count_nonfinite(p->y, 1, rows, 1, cnt, p->st);
    unsigned long long h = 0;
    cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, p->st);
    cudaError_t ce = cudaStreamSynchronize(p->st);
    dfree(cnt);
    if (ce != cudaSuccess) return guard(fail(RS_ECUDA, cudaGetErrorString(ce)));
    if (h) return guard(fail(RS_EINVAL, "X or y has non-finite entries"));
  }
  if (dual_r) {   // R = X_local^T (cols x n, ld a multiple of 4), b = y; X kept for w = X^T alpha
    const long long ldr = round_up(n, 4);
    double* R = nullptr;
    s = dalloc(&R, (size_t)std::max<long long>(cols, 1) * ldr);
    if (s == RS_OK) s = dalloc(&p->b, n);
    if (s != RS_OK) {
      dfree(R);
      return guard(s);
    }
    cudaEventRecord(e0, p->st);
    cudaError_t ce = cols > 0 ? launch_transpose(p->X, p->ldx, n, cols, R, ldr, p->st) : cudaSuccess;
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(p->b, p->y, n * 8, cudaMemcpyDeviceToDevice, p->st);
    cudaEventRecord(e1, p->st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(p->st);
    if (ce != cudaSuccess) {
      dfree(R);
      return guard(fail(RS_ECUDA, std::string("dual R = X^T: ") + cudaGetErrorString(ce)));
    }
    p->Xo = p->X;
    p->ldxo = p->ldx;
    p->own_Xo = p->own_X;
    p->X = R;
    p->ldx = ldr;
    p->own_X = true;
    p->rows_loc = cols;
    p->dual_r = true;
    p->col0 = dist ? dist->shard_begin : 0;
    p->cols_loc = cols;
    s = finish_setup(p);
    if (s != RS_OK) return guard(s);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    p->setup_seconds = ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *out = reinterpret_cast<rs_problem>(p);
    return RS_OK;
  }
  // every buffer of the setup is allocated before e0 (and freed after e1), so setup_seconds is the
  // device work of b = X^T y and the explicit A build, not host allocator time
  const long long m = p->m;
  s = dalloc(&p->b, m);
  if (s != RS_OK) return guard(s);
  double* xty_work = nullptr;
  s = dalloc(&xty_work, dense_xty_work(rows, d));
  if (s != RS_OK) return guard(s);
  double* xt = nullptr;   // dual: X^T (d x ldt), the operand of A = X X^T = (X^T)^T X^T
  long long ldt = 0;
  double* a_work = nullptr;
  TmaGemm tg{};
  GemmPlan gp{};
  cudaError_t ce = cudaSuccess;
  if (mode == RS_AS_EXPLICIT && rt == 2) {
    p->lda = round_up(n, 4);
    s = dalloc(&p->A, (size_t)n * p->lda);
    if (s != RS_OK) return guard(s);
    ldt = round_up(n, 4);
    s = dalloc(&xt, (size_t)d * ldt);
    if (s != RS_OK) return guard(s);
    ce = tma_gemm_plan(&tg, xt, ldt, xt, ldt, n, n, d, p->num_sms, 1);
    tg.lower = 1;
    if (ce == cudaSuccess && tg.work_elems) s = dalloc(&a_work, tg.work_elems);
    if (s != RS_OK) return guard(s);
    if (ce != cudaSuccess) return guard(fail(RS_ECUDA, std::string("A build: ") + cudaGetErrorString(ce)));
  } else if (mode == RS_AS_EXPLICIT && !streamed) {
    p->lda = round_up(d, 4);
    s = dalloc(&p->A, (size_t)d * p->lda);
    if (s != RS_OK) return guard(s);
    if (rows > 0) {
      ce = tma_gemm_plan(&tg, p->X, p->ldx, p->X, p->ldx, d, d, rows, p->num_sms, 1);
      if (std::getenv("RS_VERBOSE"))
        fprintf(stderr, "[rs] A build: TMA variant %d (%dx%d), splits %d\n", tg.variant, tg.bm, tg.bn, tg.splits);
      tg.lower = 1;
      if (ce == cudaSuccess && tg.work_elems) s = dalloc(&a_work, tg.work_elems);
    }
    if (s != RS_OK) return guard(s);
    if (ce != cudaSuccess) return guard(fail(RS_ECUDA, std::string("A build: ") + cudaGetErrorString(ce)));
  }
  if (!streamed) cudaEventRecord(e0, p->st);   // (streamed: recorded before the first chunk)
  if (rt == 2) {   // dual: b = y, A = X X^T + lambda I on the lower DMMA tiles of X^T
    ce = cudaMemcpyAsync(p->b, p->y, n * 8, cudaMemcpyDeviceToDevice, p->st);
    if (ce == cudaSuccess) ce = launch_transpose(p->X, p->ldx, n, d, xt, ldt, p->st);
    if (ce == cudaSuccess) ce = tma_gemm_launch(tg, p->A, p->lda, a_work, nullptr, p->st);
    if (ce == cudaSuccess) ce = launch_mirror_lower(p->A, p->lda, n, p->st);
    if (ce != cudaSuccess) return guard(fail(RS_ECUDA, std::string("dual A build: ") + cudaGetErrorString(ce)));
    launch_add_diag(p->A, p->lda, n, lambda, p->st);
  } else {
  // b = X^T y  (primal), summed over ranks
  ce = launch_dense_xty(p->X, p->ldx, rows, d, p->y, p->b, xty_work, p->st);
  if (ce != cudaSuccess) return guard(fail(RS_ECUDA, cudaGetErrorString(ce)));
  s = p->allreduce(p->b, d);
  if (s != RS_OK) return guard(s);
  }
  if (mode == RS_AS_EXPLICIT && rt == 1) {  // A = X^T X + lambda I, built once (DSYRK-shaped DMMA contraction)
    // lower-triangle tiles only on the TMA/DMMA contraction (d^2 n flop instead of 2 d^2 n), then
    // the upper triangle mirrored: A is symmetric
    if (streamed) {   // the chunks' lower tiles are summed already
      ce = launch_mirror_lower(p->A, p->lda, d, p->st);
    } else if (rows > 0) {
      ce = tma_gemm_launch(tg, p->A, p->lda, a_work, nullptr, p->st);
      if (ce == cudaSuccess) ce = launch_mirror_lower(p->A, p->lda, d, p->st);
    } else {
      ce = launch_fill(p->A, (long long)d * p->lda, 0.0, p->st);
    }
    if (ce != cudaSuccess) return guard(fail(RS_ECUDA, std::string("A build: ") + cudaGetErrorString(ce)));
    s = p->allreduce(p->A, (size_t)d * p->lda);
    if (s != RS_OK) return guard(s);
    launch_add_diag(p->A, p->lda, d, lambda, p->st);
  }
  cudaEventRecord(e1, p->st);
  ce = cudaStreamSynchronize(p->st);
  dfree(xty_work);
  dfree(a_work);
  dfree(xt);
  if (ce != cudaSuccess) return guard(fail(RS_ECUDA, cudaGetErrorString(ce)));
  s = finish_setup(p);
  if (s != RS_OK) return guard(s);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  p->setup_seconds = ms * 1e-3;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ce = cudaGetLastError();
  if (ce != cudaSuccess) return guard(fail(RS_ECUDA, cudaGetErrorString(ce)));
  *out = reinterpret_cast<rs_problem>(p);
  return RS_OK;
}

// ------------------------------------------------------------------------------------------------
static rs_status validate_opts(const Problem* p, const rs_solve_opts* o, int* ksum) {
  if (!o) return fail(RS_EINVAL, "opts is NULL");
  if (o->kind != RS_SKETCH_SUBSAMPLE && o->kind != RS_SKETCH_COUNT && o->kind != RS_SKETCH_SUBCOUNT)
    return fail(RS_EINVAL, "bad sketch kind");
  if (o->tau < 1 || o->tau > p->m) return fail(RS_EINVAL, "need 1 <= tau <= m");
  if (!(o->gamma > 0.0 && o->gamma <= 1.0)) return fail(RS_EINVAL, "need gamma in (0, 1] (P:L566)");
  if (!(o->beta >= 0.0 && o->beta <= 1.0)) return fail(RS_EINVAL, "need beta in [0, 1] (P:L566)");
  if (!(o->tol >= 0.0) || !std::isfinite(o->tol)) return fail(RS_EINVAL, "need finite tol >= 0");
  if (o->max_iter < 0) return fail(RS_EINVAL, "need max_iter >= 0");
  if (o->trace_cap < 0 || (o->trace_cap > 0 && !o->trace)) return fail(RS_EINVAL, "bad trace buffer");
  if (o->momentum < RS_MOM_CONSTANT || o->momentum > RS_MOM_COR1)
    return fail(RS_EINVAL, "bad momentum schedule");
  if (o->momentum != RS_MOM_CONSTANT && !(o->eta > 0.0 && o->eta < 1.0))
    return fail(RS_EINVAL, "need eta in (0, 1) for a momentum schedule (P:L620)");
  *ksum = 1;
  if (o->kind == RS_SKETCH_SUBCOUNT) {
    long long k = o->subcount_k;
    if (k < 0) return fail(RS_EINVAL, "subcount_k < 0");
    if (k == 0) k = (10 * o->tau <= p->m) ? 10 : p->m / o->tau;
    if (k * o->tau > p->m) return fail(RS_EINVAL, "subcount: k * tau > m");
    *ksum = (int)k;
  }
  if (o->kind == RS_SKETCH_COUNT && o->tau > 1536)
    return fail(RS_EUNSUPPORTED, "count sketch with tau > 1536 not implemented");
  if (o->kind != RS_SKETCH_COUNT && (long long)o->tau * *ksum > 8192)
    return fail(RS_EUNSUPPORTED, "selection of more than 8192 coordinates not implemented");
  if (p->m > 0x7fffffffLL) return fail(RS_EUNSUPPORTED, "m >= 2^31");
  return RS_OK;
}

// Sketch-ahead pipeline (bfactor.cu) applies to dense primal EXPLICIT and GRAM modes with
// tau <= bfactor_max_tau(): there G_k needs no per-iteration contraction of the iterate's data.
static bool pipeline_applies(const Problem* p, int tau) {
  const bool dense = (p->fmt == 0 && (p->route == 1 || p->dual_r) &&
                      (p->mode == RS_AS_EXPLICIT || p->mode == RS_AS_GRAM)) ||
                     p->mode == RS_AS_EXPLICIT;   // CSR explicit: dense A built in rs_create_csr
  const bool csr = p->fmt == 1 && p->mode == RS_AS_GRAM;
  return (dense || csr) && tau <= bfactor_max_tau();
}

// Diagonal super-blocks of the group kernel's blocked inverse (tau > 224; RS_SB_NB=n forces n)
static int sb_blocks(int tau) {
  static const int nb_env = [] {
    const char* e = std::getenv("RS_SB_NB");
    return e ? std::atoi(e) : -1;
  }();
  if (tau <= 224) return 1;
  return nb_env >= 1 ? nb_env : (tau >= 512 ? 2 : 1);
}

rs_status Problem::ensure_workspace(int kind, int tau, int ksum, int depth, bool xg) {
  if (ws_kind == kind && ws_tau == tau && ws_ksum == ksum && ws_depth == depth && ws_xg == (int)xg)
    return RS_OK;
  cudaStreamSynchronize(st);
  free_workspace();
  const size_t L = sketch_max_len(kind, (int)m, tau, ksum);
  sk.kind = kind;
  sk.m = (int)m;
  sk.tau = tau;
  sk.len = (int)L;
  sk.ksum = ksum;
  RS_TRY(dalloc(&sk.coord, L));
  RS_TRY(dalloc(&sk.sign, L));
  RS_TRY(dalloc(&sk.bucket, L));
  RS_TRY(dalloc(&sk.bptr, tau + 1));
  if (kind == SK_COUNT) RS_TRY(dalloc(&sk.cmap, m));
  if (fmt == 1 && mode == RS_AS_GRAM) {   // CSR GRAM: buffers in csr_gram_workspace
  } else if (fmt == 1 && mode != RS_AS_EXPLICIT) {   // CSR IMPLICIT: AS row-major m x tau
    ld_as = round_up(tau, 4);
    RS_TRY(dalloc(&ASt, (size_t)m * ld_as));
  } else if (depth > 0 && mode == RS_AS_EXPLICIT) {   // pipelined explicit: A S^T per slot
    ld_as = round_up(m, 4);
    as_stride = (long long)tau * ld_as;
  } else if (mode == RS_AS_GRAM) {   // no A S at all: XS, G, u
    ld_as = round_up(m, 4);
    ld_xs = round_up(tau, 4);
    RS_TRY(dalloc(&XS, (size_t)std::max<long long>(rows_loc, 1) * ld_xs));
    ld_gram = round_up(tau, 4);
    RS_TRY(dalloc(&Gram, (size_t)tau * ld_gram));
    RS_TRY(dalloc(&xp_part, std::max(xpass_partials(m, num_sms), gram_fused_partials(num_sms))));
    RS_TRY(dalloc(&uvec, m));
    gram_fused = gram_fused_ok(kind, tau);
    if (gram_fused && rows_loc > 0 && !XT) {
      // the Gram reads the tau sketched columns as contiguous rows of X^T: built once per
      // problem when it fits next to X (2 GiB margin)
      const long long ldt = round_up(rows_loc, 64);   // zero padding >= one 32-row K chunk
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      if ((double)m * ldt * 8.0 + 2.0 * (1 << 30) < (double)fr) {
        RS_TRY(dalloc(&XT, (size_t)m * ldt));
        ldxt = ldt;
        RS_CUDA(cudaMemsetAsync(XT, 0, (size_t)m * ldt * sizeof(double), st));
        RS_CUDA(launch_transpose(X, ldx, rows_loc, m, XT, ldxt, st));
      }
    }
    if (rows_loc > 0 && !gram_fused) {
      RS_CUDA(tma_gemm_plan(&tg_gram, XS, ld_xs, XS, ld_xs, tau, tau, rows_loc, num_sms, 1));
      tg_gram.lower = 1;   // G is symmetric and only its lower triangle is read (R12)
      if (tg_gram.work_elems) RS_TRY(dalloc(&gemm_work, tg_gram.work_elems));
      if (std::getenv("RS_VERBOSE"))
        fprintf(stderr, "[rs] gram gemm M=N=%d K=%lld: variant %d (%dx%d), splits %d\n", tau,
                rows_loc, tg_gram.variant, tg_gram.bm, tg_gram.bn, tg_gram.splits);
    }
  } else {          // dense: AS^T row-major tau x m
    ld_as = round_up(m, 4);
    RS_TRY(dalloc(&ASt, (size_t)tau * ld_as));
  }
  if (fmt == 0 && mode == RS_AS_IMPLICIT) {
    ld_xs = round_up(tau, 4);
    RS_TRY(dalloc(&XS, (size_t)std::max<long long>(rows_loc, 1) * ld_xs));
    use_tma = rows_loc > 0;   // an empty shard contributes zeros through the cp.async GEMM
    if (use_tma) {
      RS_CUDA(tma_gemm_plan(&tg, XS, ld_xs, X, ldx, tau, m, rows_loc, num_sms));
      if (tg.work_elems) RS_TRY(dalloc(&gemm_work, tg.work_elems));
    } else {
      gp = plan_tn_gemm(tau, m, rows_loc, num_sms);
      if (gp.work_elems) RS_TRY(dalloc(&gemm_work, gp.work_elems));
    }
    if (std::getenv("RS_VERBOSE"))
      fprintf(stderr, "[rs] gemm M=%d N=%lld K=%lld: %s variant %d (%dx%d), splits %d\n", tau, m,
              rows_loc, use_tma ? "TMA" : "cp.async", use_tma ? tg.variant : gp.variant,
              use_tma ? tg.bm : gp.bm, use_tma ? tg.bn : gp.bn, use_tma ? tg.splits : gp.splits);
  }
  if (fmt == 1 && mode != RS_AS_EXPLICIT) RS_TRY(csr_ensure_workspace(kind, tau, ksum));
  if (depth > 0) {   // sketch-ahead slots (two sets of `depth` for the fused pipeline)
    pipe = true;
    pipe_xg = xg;
    P = depth;
    if (xg) depth *= 2;
    skb = sk;   // same geometry, `depth` slots
    skb.coord = nullptr; skb.sign = nullptr; skb.bucket = nullptr; skb.bptr = nullptr; skb.cmap = nullptr;
    RS_TRY(dalloc(&skb.coord, L * depth));
    RS_TRY(dalloc(&skb.sign, L * depth));
    RS_TRY(dalloc(&skb.bucket, L * depth));
    RS_TRY(dalloc(&skb.bptr, (size_t)(tau + 1) * depth));
    if (kind == SK_COUNT) RS_TRY(dalloc(&skb.cmap, (size_t)m * depth));
    // slots the device skips (beyond max_iter) are never written, but the PDL-chained kernels read
    // a slot's sketch before they learn that the solve has stopped: keep every slot well-formed
    RS_CUDA(cudaMemsetAsync(skb.coord, 0, L * depth * sizeof(int), st));
    RS_CUDA(cudaMemsetAsync(skb.sign, 0, L * depth, st));
    RS_CUDA(cudaMemsetAsync(skb.bucket, 0, L * depth * sizeof(int), st));
    RS_CUDA(cudaMemsetAsync(skb.bptr, 0, (size_t)(tau + 1) * depth * sizeof(int), st));
    if (mode == RS_AS_EXPLICIT) {   // count: A S^T rows per slot; subsample / SubCount read A directly
      if (kind == SK_COUNT) RS_TRY(dalloc(&ASt_slots, (size_t)as_stride * depth));
    } else {
      gram_stride = (long long)tau * ld_gram;
      RS_TRY(dalloc(&Gram_slots, (size_t)gram_stride * depth));
    }
    ld_gi = round_up(tau, 4);
    gi_stride = (long long)tau * ld_gi;
    RS_TRY(dalloc(&Ginv_slots, (size_t)gi_stride * depth));
    RS_TRY(dalloc(&slot_flags, depth));
    // (two slot sets: the second region also serves the first set's tail, factored beside the
    // first group)
    if (bfactor_work_elems(tau)) RS_TRY(dalloc(&bf_work, bfactor_work_elems(tau) * depth));
    if (xg) RS_TRY(dalloc(&bf_claim, 2 * BF_CLAIM_WORDS));   // two concurrent launches' claims
    // EXPLICIT: the group's iterations as one persistent kernel (iterate.cu)
    use_iterate = mode == RS_AS_EXPLICIT && iterate_ok(sk, m, xg ? ov_sms : num_sms);
    if (use_iterate) RS_TRY(dalloc(&it_scratch, 2 * (size_t)tau + num_sms));
    // the group kernel solves with a blocked inverse: the factorisation inverts only the nb
    // diagonal super-blocks of L (2 tau^3 / 3 -> (1 + 1/nb^2) tau^3 / 3 flop) and the iteration
    // substitutes block by block (2 (nb - 1) more grid barriers per iteration); DESIGN §1
    bf_sb = 0;
    if (use_iterate && tau > 224) {
      const int nb = sb_blocks(tau), pairs = (tau + 63) / 64;
      if (nb > 1) bf_sb = (pairs + nb - 1) / nb * 64;
    }
  }
  sw = plan_solve(tau, num_sms);
  RS_TRY(dalloc(&sw.Gx, solve_gx_elems(tau)));
  RS_TRY(dalloc(&sw.delta, tau));
  RS_TRY(dalloc(&partials, update_partials(m)));
  ws_kind = kind;
  ws_tau = tau;
  ws_ksum = ksum;
  ws_depth = xg ? depth / 2 : depth;
  ws_xg = (int)xg;
  return RS_OK;
}

// One iteration of Alg. 2 as a launch sequence; `ev` (optional) = 2*RS_K_NCLASSES
// events bracketing each kernel class.
rs_status Problem::enqueue_iteration(const rs_solve_opts* o, cudaEvent_t* ev) {
  auto mark = [&](int cls, int edge) {
    if (ev) cudaEventRecordWithFlags(ev[2 * cls + edge], st, cudaEventRecordExternal);
  };
  mark(RS_K_SKETCH, 0);
  RS_CUDA(launch_sketch(sk, o->seed, ctrl, -1, st));                       // a1
  mark(RS_K_SKETCH, 1);
  if (fmt == 1 && mode == RS_AS_GRAM) return csr_enqueue_gram(o, ev);
  if (fmt == 0 && mode == RS_AS_GRAM) {
    if (!gram_fused) {
      mark(RS_K_XS, 0);
      RS_CUDA(launch_dense_xs(X, ldx, rows_loc, sk, XS, ld_xs, ctrl, st));  // a2  XS
      mark(RS_K_XS, 1);
    }
    mark(RS_K_GRAM, 0);
    if (rows_loc > 0 && XT)                                                  // (XS)^T XS from X^T
      RS_CUDA(launch_gram_xt(XT, ldxt, rows_loc, sk, xp_part, Gram, ld_gram, num_sms, ctrl, st));
    else if (rows_loc > 0 && gram_fused)                                     // gather + (XS)^T XS
      RS_CUDA(launch_gram_fused(X, ldx, rows_loc, sk, xp_part, Gram, ld_gram, num_sms, ctrl, st));
    else if (rows_loc > 0)
      RS_CUDA(tma_gemm_launch(tg_gram, Gram, ld_gram, gemm_work, ctrl, st));   // (XS)^T XS
    else
      RS_CUDA(launch_fill(Gram, (long long)sk.tau * ld_gram, 0.0, st));
    RS_TRY(allreduce(Gram, (size_t)sk.tau * ld_gram));
    mark(RS_K_GRAM, 1);
    mark(RS_K_SOLVE, 0);
    RS_CUDA(launch_sketched_solve(nullptr, 0, false, Gram, ld_gram, lambda, r, sk, sw, sdelta,
                                  ctrl, st));                                // a4 + a5
    mark(RS_K_SOLVE, 1);
    mark(RS_K_AS, 0);
    if (rows_loc > 0)
      RS_CUDA(launch_xpass(X, ldx, rows_loc, m, sdelta, xp_part, uvec, num_sms, ctrl, st, &sk,
                           sw.delta));
    else
      RS_CUDA(launch_fill(uvec, m, 0.0, st));
    RS_TRY(allreduce(uvec, (size_t)m));                                     // X^T X S delta
    mark(RS_K_AS, 1);
    mark(RS_K_UPDATE, 0);
    RS_CUDA(launch_update_vec(uvec, lambda, sdelta, w, dw, r, dr, m, o->gamma, o->beta, partials,
                              ctrl, st));                                    // a6 + a7
    mark(RS_K_UPDATE, 1);
    return RS_OK;
  }
  if (fmt == 0 && mode == RS_AS_IMPLICIT) {
    mark(RS_K_XS, 0);
    RS_CUDA(launch_dense_xs(X, ldx, rows_loc, sk, XS, ld_xs, ctrl, st));    // a2  XS
    mark(RS_K_XS, 1);
    mark(RS_K_AS, 0);
    if (use_tma)                                                             // a3  (X^T XS)^T
      RS_CUDA(tma_gemm_launch(tg, ASt, ld_as, gemm_work, ctrl, st));
    else
      RS_CUDA(launch_tn_gemm(XS, ld_xs, X, ldx, sk.tau, m, rows_loc, ASt, ld_as, gp, gemm_work,
                             ctrl, st));
    RS_TRY(allreduce(ASt, (size_t)sk.tau * ld_as));                         // sum over row shards
    RS_CUDA(launch_add_lambda_s(lambda, sk, ASt, ld_as, false, ctrl, st));         // + lambda S
    mark(RS_K_AS, 1);
  } else if (mode == RS_AS_EXPLICIT) {
    mark(RS_K_XS, 0);
    RS_CUDA(launch_explicit_rows(A, lda, m, sk, ASt, ld_as, ctrl, st));      // a2  rows of A
    mark(RS_K_XS, 1);
  } else {
    RS_TRY(csr_enqueue_as(o, ev));
  }
  mark(RS_K_SOLVE, 0);
  const bool as_rm = fmt == 1 && mode != RS_AS_EXPLICIT;   // CSR IMPLICIT stores AS row-major
  RS_CUDA(launch_sketched_solve(ASt, ld_as, as_rm, nullptr, 0, 0.0, r, sk, sw, sdelta, ctrl, st));
  mark(RS_K_SOLVE, 1);
  mark(RS_K_UPDATE, 0);
  RS_CUDA(launch_update(ASt, ld_as, as_rm, sk.tau, sw.delta, sdelta, w, dw, r, dr, m, o->gamma, o->beta,
                        partials, ctrl, st));                                // a6 + a7
  mark(RS_K_UPDATE, 1);
  return RS_OK;
}

// Group precompute of the sketch-ahead pipeline: sketches S_{k0..k0+ns-1} (k0 = ctrl->k), their
// A S^T rows (explicit) or Grams (XS)^T XS (gram), and the batched factorisation Ginv = G^{-1}.
rs_status Problem::enqueue_precompute(const rs_solve_opts* o, int ns, cudaEvent_t* ev, int split) {
  // ev (optional): the event sets of iterations k0 .. k0+ns-1, 2 * RS_K_NCLASSES each; the group's
  // sketches and factorisation are recorded on iteration k0's, slot q's Gram on iteration k0+q's
  auto mark = [&](int q, int cls, int edge) {
    if (ev) cudaEventRecordWithFlags(ev[(size_t)q * 2 * RS_K_NCLASSES + 2 * cls + edge], st,
                                     cudaEventRecordExternal);
  };
  mark(0, RS_K_PRE, 0);
  RS_CUDA(launch_sketch_batch(skb, ns, o->seed, ctrl, -1, st));                 // a1 x ns
  FactorSrc src{};
  if (mode == RS_AS_EXPLICIT && ASt_slots) {                                     // a2 x ns
    RS_CUDA(launch_explicit_rows_batch(A, lda, m, skb, ns, ASt_slots, ld_as, as_stride, ctrl, st));
    src.ASt = ASt_slots;
    src.ld_as = ld_as;
    src.as_stride = as_stride;
  } else if (mode == RS_AS_EXPLICIT) {   // G = S^T A S gathered from A inside the factor kernel
    src.A = A;
    src.lda = lda;
  }
  mark(0, RS_K_PRE, 1);
  if (mode != RS_AS_EXPLICIT) {                                                  // Gram x ns
    for (int q = 0; q < ns; ++q) {
      const DevSketch sq = skb.at(q);
      double* Gq = Gram_slots + (long long)q * gram_stride;
      if (fmt == 1) {
        RS_TRY(csr_gram_into(sq, Gq, ev ? ev + (size_t)q * 2 * RS_K_NCLASSES : nullptr, q, false));
        continue;
      }
      mark(q, RS_K_GRAM, 0);
      if (rows_loc > 0 && XT) {
        RS_CUDA(launch_gram_xt(XT, ldxt, rows_loc, sq, xp_part, Gq, ld_gram, num_sms, ctrl, st, q));
      } else if (rows_loc > 0 && gram_fused) {
        RS_CUDA(launch_gram_fused(X, ldx, rows_loc, sq, xp_part, Gq, ld_gram, num_sms, ctrl, st, q));
      } else if (rows_loc > 0) {
        RS_CUDA(launch_dense_xs(X, ldx, rows_loc, sq, XS, ld_xs, ctrl, st, q));
        RS_CUDA(tma_gemm_launch(tg_gram, Gq, ld_gram, gemm_work, ctrl, st));
      } else {
        RS_CUDA(launch_fill(Gq, gram_stride, 0.0, st));
      }
      mark(q, RS_K_GRAM, 1);
    }
    // the ns partial Grams of the rank's rows, summed over ranks in ONE collective per group
    RS_TRY(allreduce(Gram_slots, (size_t)ns * gram_stride));
    src.Gram = Gram_slots;
    src.ld_gram = ld_gram;
    src.gram_stride = gram_stride;
    src.lambda = lambda;
  }
  mark(0, RS_K_FACTOR, 0);
  if (split > 0 && split < ns) {   // the overlapped pipeline's first set (see solve): slots [0, split)
    // here, one per SM; slots [split, ns) on st2 with their own scratch, flagged -1 until factored
    RS_CUDA(launch_bfactor(src, skb, split, Ginv_slots, ld_gi, gi_stride, slot_flags, bf_work, ctrl,
                           st, false, nullptr, bf_sb));                                     // a4+a5
    RS_CUDA(cudaMemsetAsync(slot_flags + split, 0xff, sizeof(int) * (size_t)(ns - split), st));
    RS_CUDA(cudaEventRecord(ev_pro, st));
    RS_CUDA(cudaStreamWaitEvent(st2, ev_pro, 0));
    FactorSrc s2 = src;
    if (s2.ASt) s2.ASt += (long long)split * as_stride;
    const BfClaim cl{bf_claim + BF_CLAIM_WORDS, num_sms - ov_sms, num_sms};
    RS_CUDA(launch_bfactor(s2, skb.at(split), ns - split, Ginv_slots + (long long)split * gi_stride,
                           ld_gi, gi_stride, slot_flags + split,
                           bf_work + (long long)bfactor_work_elems((int)o->tau) * P, ctrl, st2, false,
                           &cl, bf_sb));
    RS_CUDA(cudaEventRecord(ev_pro_tail, st2));
  } else {
    RS_CUDA(launch_bfactor(src, skb, ns, Ginv_slots, ld_gi, gi_stride, slot_flags, bf_work, ctrl,
                           st, bf_dual, nullptr, bf_sb));                                   // a4+a5
  }
  mark(0, RS_K_FACTOR, 1);
  return RS_OK;
}

// One iteration of Alg. 2 on precomputed slot `slot`: delta = Ginv S^T r, A S delta, update.
rs_status Problem::enqueue_pipelined_iteration(const rs_solve_opts* o, int slot, cudaEvent_t* ev) {
  auto mark = [&](int cls, int edge) {
    if (ev) cudaEventRecordWithFlags(ev[2 * cls + edge], st, cudaEventRecordExternal);
  };
  const DevSketch sq = skb.at(slot);
  mark(RS_K_SOLVE, 0);
  // slot 0 follows the group's factorisation (ordinary launch); later slots chain by PDL
  const bool rows_of_A = mode == RS_AS_EXPLICIT && !ASt_slots;   // k_update_rows reads A rows
  RS_CUDA(launch_apply_ginv(Ginv_slots + (long long)slot * gi_stride, ld_gi, sq, slot_flags + slot,
                            r, sw.Gx, sw.delta, sdelta, ctrl, st, slot == 0,
                            rows_of_A ? A : nullptr, lda, m));                     // a4 + a5
  mark(RS_K_SOLVE, 1);
  if (mode == RS_AS_EXPLICIT) {
    mark(RS_K_UPDATE, 0);
    if (ASt_slots)
      RS_CUDA(launch_update(ASt_slots + (long long)slot * as_stride, ld_as, false, sq.tau, sw.delta,
                            sdelta, w, dw, r, dr, m, o->gamma, o->beta, partials, ctrl, st));  // a6+a7
    else   // A S delta from the sketched rows of A
      RS_CUDA(launch_update_rows(A, lda, sq, sw.delta, sdelta, w, dw, r, dr, m, o->gamma, o->beta,
                                 partials, num_sms, ctrl, st));          // a6+a7
    mark(RS_K_UPDATE, 1);
    return RS_OK;
  }
  mark(RS_K_AS, 0);
  if (fmt == 1)
    RS_TRY(csr_gram_apply(sdelta, uvec, &sq));                                   // R^T R S delta
  else if (rows_loc > 0)
    RS_CUDA(launch_xpass(X, ldx, rows_loc, m, sdelta, xp_part, uvec, num_sms, ctrl, st, &sq,
                         sw.delta));
  else
    RS_CUDA(launch_fill(uvec, m, 0.0, st));
  RS_TRY(allreduce(uvec, (size_t)m));                                            // X^T X S delta
  mark(RS_K_AS, 1);
  mark(RS_K_UPDATE, 0);
  RS_CUDA(launch_update_vec(uvec, lambda, sdelta, w, dw, r, dr, m, o->gamma, o->beta, partials,
                            ctrl, st));                                          // a6 + a7
  mark(RS_K_UPDATE, 1);
  return RS_OK;
}

// The ns iterations of a precomputed EXPLICIT group as one persistent cooperative kernel.
rs_status Problem::enqueue_iterate_group(const rs_solve_opts* o, int ns, cudaEvent_t* ev, int slot0,
                                         int grid) {
  if (ev) cudaEventRecordWithFlags(ev[2 * RS_K_UPDATE], st, cudaEventRecordExternal);
  IterArgs ia{};
  ia.Ginv = Ginv_slots + (long long)slot0 * gi_stride;
  ia.ld_gi = ld_gi;
  ia.gi_stride = gi_stride;
  ia.skb = skb.at(slot0);
  ia.flags = slot_flags + slot0;
  ia.A = A;
  ia.lda = lda;
  ia.ASt = ASt_slots ? ASt_slots + (long long)slot0 * as_stride : nullptr;
  ia.ld_as = ld_as;
  ia.as_stride = as_stride;
  ia.m = m;
  ia.w = w;
  ia.dw = dw;
  ia.r = r;
  ia.dr = dr;
  ia.sdelta = sdelta;
  ia.tvec = it_scratch;
  ia.dvec = it_scratch + skb.tau;
  ia.partials = it_scratch + 2 * (long long)skb.tau;
  ia.gamma = o->gamma;
  ia.beta = o->beta;
  ia.nslots = ns;
  ia.big = skb.tau > 224;
  ia.sb = bf_sb;
  ia.wait = pipe_ov ? 1 : 0;   // the first set's tail may still be factored on st2 (solve)
  if (grid <= 0) {   // all SMs, but no fewer than 64 columns per CTA (small m: cheaper grid syncs)
    static const int g_env = [] {
      const char* e = std::getenv("RS_IT_GRID");
      return e ? std::atoi(e) : 0;
    }();
    grid = g_env > 0 ? g_env : (int)std::min<long long>(num_sms, std::max<long long>(16, (m + 63) / 64));
  }
  RS_CUDA(launch_iterate(ia, grid, ctrl, st));
  if (ev) cudaEventRecordWithFlags(ev[2 * RS_K_UPDATE + 1], st, cudaEventRecordExternal);
  return RS_OK;
}

// One group of an overlapped EXPLICIT pipeline (tau > 224) on slot set g: the sketches of the next
// group (set 1 - g, iterations k0 + P ..) are drawn first; then, concurrently, st2 gathers and
// factors them (k_bf_gather + k_bfactor_lp on the num_sms - ov_sms SMs) while st runs this group's
// P iterations (k_iterate on the ov_sms SMs left free).  The factorisation kernels read ctrl->k only
// to skip slots beyond max_iter; the concurrent iterations can only make that test skip fewer slots.
rs_status Problem::enqueue_group_ov(const rs_solve_opts* o, int g, cudaEvent_t* ev) {
  auto mark = [&](cudaStream_t s, int q, int cls, int edge) {
    if (ev) cudaEventRecordWithFlags(ev[(size_t)q * 2 * RS_K_NCLASSES + 2 * cls + edge], s,
                                     cudaEventRecordExternal);
  };
  const int cur = g, nxt = 1 - g;
  const DevSketch sn = skb.at(nxt * P);
  mark(st, 0, RS_K_PRE, 0);
  RS_CUDA(launch_sketch_batch(sn, P, o->seed, ctrl, -1, st, P));   // a1 x P (next group)
  mark(st, 0, RS_K_PRE, 1);
  RS_CUDA(cudaEventRecord(ev_fork, st));
  RS_CUDA(cudaStreamWaitEvent(st2, ev_fork, 0));
  FactorSrc src{};
  mark(st2, 0, RS_K_FACTOR, 0);
  if (ASt_slots) {   // count: the slots' rows of A S^T
    double* as_n = ASt_slots + (long long)nxt * P * as_stride;
    RS_CUDA(launch_explicit_rows_batch(A, lda, m, sn, P, as_n, ld_as, as_stride, ctrl, st2));
    src.ASt = as_n;
    src.ld_as = ld_as;
    src.as_stride = as_stride;
  } else {
    src.A = A;
    src.lda = lda;
  }
  // at most num_sms - ov_sms SMs (BfClaim)
  const BfClaim cl{bf_claim, num_sms - ov_sms, num_sms};
  RS_CUDA(launch_bfactor(src, sn, P, Ginv_slots + (long long)nxt * P * gi_stride, ld_gi, gi_stride,
                         slot_flags + (long long)nxt * P, bf_work, ctrl, st2, bf_dual, &cl, bf_sb));   // a4 + a5 ahead
  mark(st2, 0, RS_K_FACTOR, 1);
  RS_CUDA(cudaEventRecord(ev_join, st2));
  RS_TRY(enqueue_iterate_group(o, P, ev, cur * P, ov_sms));                       // a4-a7 x P
  RS_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
  return RS_OK;
}

static int status_of(int st) {
  switch (st) {
    case ST_DIVERGED: return RS_EDIVERGED;
    case ST_NOTSPD: return RS_ENOTSPD;
    case ST_OVERFLOW: return RS_EUNSUPPORTED;
    case ST_SKETCHFAIL: return RS_EUNSUPPORTED;
    default: return RS_OK;
  }
}

// THEORY schedule (Eq. parameterswitchtheory through Thm. 1, R24): (gamma_k, beta_k)
// until eta has switched to 1, after which zeta is frozen and the last pair repeats.
static std::vector<double> theory_table(double eta) {
  std::vector<double> t;
  double S = 0.0, e = eta, zeta = 0.0;   // sum_{t<k} eta_t (1 - eta_t), eta_k, zeta_k
  bool switched = false;
  for (int k = 0; k < 10000000; ++k) {
    const double S1 = S + e * (1.0 - e);
    double e1 = switched ? 1.0 : eta;
    double z1 = S1 / e1;
    double g = e / (z1 + 1.0), b = zeta / (z1 + 1.0);
    if (!switched && b >= 0.5) {
      switched = true;
      e1 = 1.0;
      z1 = S1 / e1;
      g = e / (z1 + 1.0);
      b = zeta / (z1 + 1.0);
    }
    t.push_back(g);
    t.push_back(b);
    if (e == 1.0) break;
    S = S1;
    e = e1;
    zeta = z1;
  }
  return t;
}

rs_status Problem::solve(const rs_solve_opts* o, double* w_out, rs_mem w_mem, double* alpha_out,
                         rs_report* rep) {
  int ksum = 1;
  RS_TRY(validate_opts(this, o, &ksum));
  if (!w_out) return fail(RS_EINVAL, "w_out is NULL");
  // RS_TIMING: host time of the solve's phases on stderr (diagnostics of the timed regions)
  static const bool timing = std::getenv("RS_TIMING") != nullptr;
  const auto h0 = std::chrono::steady_clock::now();
  auto hms = [&](std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
  };
  RS_CUDA(cudaSetDevice(device));
  const bool want_pipe = pipeline_applies(this, (int)o->tau);
  // iterations per CUDA-graph launch (between host reads of the stop flag)
  int chunk = (int)(o->check_every > 0 ? std::min<long long>(o->check_every, 1024)
                                       : (want_pipe ? (o->tau > 224 ? num_sms : 64) : 16));
  // overlapped pipeline: the batched factorisation runs two slots per SM (k_bfactor_lp<4>), so a
  // wave holds 2 x (free SMs) slots (RS_BF_DUAL=0: the 8-warp shape, one per SM)
  static const bool dual_env = [] {
    const char* e = std::getenv("RS_BF_DUAL");
    return !(e && e[0] == '0');
  }();
  // EXPLICIT with tau > 224: overlap the next group's factorisation with the current group's
  // iterations on a split of the SMs when that shortens an iteration, the split chosen by a model
  // of both (measured on this B200): the group kernel's phase C reads len rows (count:
  // tau rows of A S^T) x 64-column chunks per CTA at ~45 GB/s per SM, ~4.5 TB/s in all, plus ~12 us
  // of phases A/B and barriers; one G_k costs ~1924 (tau / 256)^0.70 SM-us of factorisation
  // (k_bfactor_lp: tau 256 and 1024 measured; the small-tau end is latency-bound).  RS_OV_SMS=n
  // forces the group kernel's SM count.
  const double tau_d = (double)o->tau;
  const double len_d = (double)sketch_max_len((int)o->kind, (int)m, (int)o->tau, ksum);
  const double rows_it = o->kind == RS_SKETCH_COUNT ? tau_d : len_d;
  auto it_us = [&](int sms) {
    const long long cw = (m + sms - 1) / sms;
    const double cols = 64.0 * (double)((cw + 63) / 64);
    return std::max(rows_it * 8.0 * cols / 45e3, rows_it * (double)m * 8.0 / 4.5e6) + 12.0;
  };
  // (blocked inverse, nb super-blocks: the inverse step -- ~0.32 of the full-inverse slot time on
  // c5 -- shrinks to 1/nb^2 of its flop; measured c5 factor per slot 53 -> 40.5 us at nb = 2)
  const int nb_sb = len_d <= 8192 ? sb_blocks((int)o->tau) : 1;
  const double fslot = 1924.0 * std::pow(tau_d / 256.0, 0.702) * (0.68 + 0.32 / (nb_sb * nb_sb));
  const int it_grid = (int)std::min<long long>(num_sms, std::max<long long>(16, (m + 63) / 64));
  const double seq_us = fslot / num_sms + it_us(it_grid);
  static const int ov_env = [] {
    const char* e = std::getenv("RS_OV_SMS");
    return e ? std::atoi(e) : 0;
  }();
  int ov_best = 0;
  double ov_us = 1e30;
  for (int sms = 16; sms <= num_sms - 16; sms += 2) {
    const double v = std::max(fslot / (num_sms - sms), it_us(sms));
    if (v < ov_us) {
      ov_us = v;
      ov_best = sms;
    }
  }
  if (ov_env > 0 && ov_env < num_sms) {
    ov_best = ov_env;
    ov_us = 0.0;
  }
  const bool want_ov = want_pipe && mode == RS_AS_EXPLICIT && o->tau > 224 && ov_best > 0 &&
                       len_d <= 8192 && ov_us < seq_us;
  if (want_ov) ov_sms = ov_best;
  bf_dual = want_ov && dual_env;
  const int cps = bf_dual ? 2 : 1;
  if (want_ov) chunk = 2 * cps * (num_sms - ov_sms);
  const bool want_xg = want_ov;   // two slot sets
  if (want_xg) chunk = std::max(2, chunk & ~1);   // two groups of P = chunk / 2
  int depth = 0;
  if (want_pipe) {   // one batched factorisation wave: <= num_sms slots, <= ~6 GB of slots
    const long long slot_bytes =
        8LL * o->tau * (mode == RS_AS_EXPLICIT ? (o->kind == RS_SKETCH_COUNT ? round_up(m, 4) : 0)
                                               : round_up(o->tau, 4)) +
        8LL * o->tau * round_up(o->tau, 4) + 16LL * m + 8LL * (long long)bfactor_work_elems((int)o->tau);
    depth = (int)std::max<long long>(1, std::min<long long>({(long long)chunk, (long long)cps * num_sms,
                                                             6000000000LL / slot_bytes}));
    if (want_xg) {
      depth = std::min<long long>({(long long)depth, (long long)chunk / 2, 5000000000LL / slot_bytes});
      chunk = 2 * depth;
    }
  }
  RS_TRY(ensure_workspace((int)o->kind, (int)o->tau, ksum, depth, want_xg));
  pipe_ov = want_ov && pipe_xg;
  if (pipe_ov && !st2) {
    RS_CUDA(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
    RS_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    RS_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    RS_CUDA(cudaEventCreateWithFlags(&ev_pro, cudaEventDisableTiming));
    RS_CUDA(cudaEventCreateWithFlags(&ev_pro_tail, cudaEventDisableTiming));
  }
  // state: w^{-1} = w^0 = 0, r^{-1} = r^0 = -b
  RS_CUDA(launch_fill(w, m, 0.0, st));
  RS_CUDA(launch_fill(dw, m, 0.0, st));
  RS_CUDA(launch_fill(dr, m, 0.0, st));
  RS_CUDA(launch_fill(sdelta, m, 0.0, st));
  RS_CUDA(launch_axpby_neg(b, r, m, st));
  dfree(trace_dev);
  trace_dev = nullptr;
  if (o->trace_cap > 0) RS_TRY(dalloc(&trace_dev, o->trace_cap));
  Ctrl c{};
  c.k = 0;
  c.bnorm2 = bnorm2;
  c.rnorm2 = bnorm2;
  c.tol = o->tol;
  c.max_iter = o->max_iter;
  c.trace = trace_dev;
  c.trace_cap = o->trace_cap;
  c.mom_kind = o->momentum == RS_MOM_HEURISTIC ? 1 : o->momentum == RS_MOM_THEORY ? 2
             : o->momentum == RS_MOM_COR1 ? 3 : 0;
  c.mom_eta = o->eta;
  dfree(mom_tab_dev);
  mom_tab_dev = nullptr;
  if (o->momentum == RS_MOM_THEORY) {
    const std::vector<double> tab = theory_table(o->eta);
    RS_TRY(dalloc(&mom_tab_dev, tab.size()));
    RS_CUDA(cudaMemcpyAsync(mom_tab_dev, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, st));
    c.mom_tab = mom_tab_dev;
    c.mom_ntab = (long long)tab.size() / 2;
  }
  c.status = ST_RUNNING;
  if (bnorm2 == 0.0 || o->tol >= 1.0) {   // ||r^0|| <= tol ||r^0||: w = 0 is returned
    c.done = 1;
    c.status = ST_CONVERGED;
  } else if (o->max_iter == 0) {
    c.done = 1;
    c.status = ST_MAXITER;
  }
  *ctrl_host = c;
  RS_CUDA(cudaMemcpyAsync(ctrl, ctrl_host, sizeof(Ctrl), cudaMemcpyHostToDevice, st));

  // CUDA graph of `chunk` iterations, reused by later solves with the same launch parameters
  const GraphKey key{(int)o->kind, (int)o->tau, ksum, chunk, o->profile ? 1 : 0, o->seed, o->gamma,
                     o->beta};
  const bool rebuild = !graph_exec || !(key == graph_key);
  if (rebuild) {
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    graph_exec = nullptr;
    for (auto ev : prof_events) cudaEventDestroy(ev);
    prof_events.clear();
    if (o->profile) {
      prof_events.resize((size_t)chunk * 2 * RS_K_NCLASSES);
      for (auto& ev : prof_events) RS_CUDA(cudaEventCreate(&ev));
    }
  }
  RS_CUDA(cudaStreamSynchronize(st));
  if (rebuild) {
    cudaGraph_t g = nullptr;
    RS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    rs_status s = RS_OK;
    auto evs = [&](int i) { return o->profile ? &prof_events[(size_t)i * 2 * RS_K_NCLASSES] : nullptr; };
    for (int i = 0; i < chunk && s == RS_OK;) {
      if (pipe_xg) {   // two groups, alternating slot sets
        s = enqueue_group_ov(o, (i / P) & 1, evs(i));
        i += P;
      } else if (pipe) {   // group: precompute ns slots, then ns iterations on them
        const int ns = std::min(P, chunk - i);
        s = enqueue_precompute(o, ns, evs(i));
        if (use_iterate && s == RS_OK)
          s = enqueue_iterate_group(o, ns, evs(i));
        else
          for (int q = 0; q < ns && s == RS_OK; ++q) s = enqueue_pipelined_iteration(o, q, evs(i + q));
        i += ns;
      } else {
        s = enqueue_iteration(o, evs(i));
        ++i;
      }
    }
    cudaError_t ce = cudaStreamEndCapture(st, &g);
    if (s != RS_OK) {
      if (g) cudaGraphDestroy(g);
      return s;
    }
    if (ce != cudaSuccess) return fail(RS_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    {   // kernel nodes per graph launch (rs_report.gpu_launches)
      size_t nn = 0;
      cudaGraphGetNodes(g, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      cudaGraphGetNodes(g, nodes.data(), &nn);
      kernels_per_iter = 0;
      for (auto nd : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nd, &t);
        if (t == cudaGraphNodeTypeKernel) ++kernels_per_iter;
      }
    }
    ce = cudaGraphInstantiate(&graph_exec, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return fail(RS_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
    graph_key = key;
  }
  double kms[RS_K_NCLASSES] = {0};
  long long klaunch[RS_K_NCLASSES] = {0};
  cudaEvent_t t0, t1;
  RS_CUDA(cudaEventCreate(&t0));
  RS_CUDA(cudaEventCreate(&t1));
  if (timing) fprintf(stderr, "[rs] solve preamble %.3f ms (graph %s)\n", hms(h0), rebuild ? "built" : "reused");
  const auto h1 = std::chrono::steady_clock::now();
  RS_CUDA(cudaEventRecord(t0, st));
  // overlapped pipeline: slot set 0 (iterations 0 .. P-1) is formed and factored up front -- with two
  // slots per SM in the steady state (P > num_sms), its first num_sms slots as one wave of the 8-warp
  // shape on every SM, the rest on st2 beside the first group, whose iterations wait per slot
  bool pro_tail = false;
  if (pipe_xg && !ctrl_host->done) {
    static const bool split_env = [] {   // RS_OV_SPLIT=0: the whole first set up front
      const char* e = std::getenv("RS_OV_SPLIT");
      return !(e && e[0] == '0');
    }();
    const int split = pipe_ov && split_env && P > num_sms ? num_sms : P;
    RS_TRY(enqueue_precompute(o, P, nullptr, split));
    pro_tail = split < P;
  }
  long long k_prev = 0, graph_launches = 0;
  while (!ctrl_host->done) {
    RS_CUDA(cudaGraphLaunch(graph_exec, st));
    ++graph_launches;
    RS_CUDA(cudaMemcpyAsync(ctrl_host, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaStreamSynchronize(st));
    if (o->profile) {
      const long long ran = std::min<long long>(ctrl_host->k - k_prev, chunk);
      for (long long i = 0; i < ran; ++i)
        for (int cls = 0; cls < RS_K_NCLASSES; ++cls) {
          float ms = 0;
          cudaEvent_t* ev = &prof_events[(size_t)i * 2 * RS_K_NCLASSES];
          if (cudaEventElapsedTime(&ms, ev[2 * cls], ev[2 * cls + 1]) == cudaSuccess && ms > 0) {
            kms[cls] += ms;
            klaunch[cls] += 1;
          }
        }
      cudaGetLastError();
    }
    if (world > 1 && hostcoll_failed(hcoll))
      return fail(RS_ENCCL, "host collective: a rank timed out in an allreduce");
    if (world > 1 && comm) {
      std::string err;
      const NcclApi* api = nccl_api(&err);
      ncclResult_t ae = ncclSuccess;
      if (api && api->ncclCommGetAsyncError(comm, &ae) == ncclSuccess && ae != ncclSuccess) {
        api->ncclCommAbort(comm);
        comm = nullptr;
        return fail(RS_ENCCL, std::string("NCCL async error: ") + api->ncclGetErrorString(ae));
      }
    }
    k_prev = ctrl_host->k;
  }
  if (pro_tail) RS_CUDA(cudaStreamWaitEvent(st, ev_pro_tail, 0));   // (stops early once done)
  RS_CUDA(cudaEventRecord(t1, st));
  RS_CUDA(cudaEventSynchronize(t1));
  const auto h2 = std::chrono::steady_clock::now();
  float solve_ms = 0;
  cudaEventElapsedTime(&solve_ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  last_status = ctrl_host->status;

  const Ctrl& h = *ctrl_host;
  rs_report R{};
  R.iterations = h.k;
  R.converged = h.status == ST_CONVERGED;
  R.rel_residual = bnorm2 > 0 ? std::sqrt(h.rnorm2) / std::sqrt(bnorm2) : 0.0;
  R.setup_seconds = setup_seconds;
  R.solve_seconds = solve_ms * 1e-3;
  R.trace_len = std::min<long long>(h.k, o->trace_cap);
  for (int cls = 0; cls < RS_K_NCLASSES; ++cls) {
    R.kernel_ms[cls] = kms[cls];
    R.kernel_launches[cls] = klaunch[cls];
  }
  R.gpu_launches = graph_launches * kernels_per_iter;   // kernel nodes per graph launch
  R.overlap_sms = pipe_ov ? ov_sms : 0;
  R.inverse_blocks = 0;
  if (pipe && o->tau > 224) {
    const long long sbw = bf_sb > 0 ? bf_sb : o->tau;
    R.inverse_blocks = use_iterate ? (int)((o->tau + sbw - 1) / sbw) : 1;
  }
  if (rep) *rep = R;
  if (o->trace && R.trace_len > 0)
    RS_CUDA(cudaMemcpy(o->trace, trace_dev, R.trace_len * 8, cudaMemcpyDeviceToHost));
  const int rc = status_of(h.status);
  if (h.status == ST_SKETCHFAIL)
    return fail(RS_EUNSUPPORTED, "sketch selection: more than 1024 coordinates share one 64-bit key");
  if (rc == RS_EUNSUPPORTED)
    return fail(RS_EUNSUPPORTED, "CSR dual: sketched-row hash table overflow (bucket too dense)");
  if (rc == RS_ENOTSPD)
    return fail(RS_ENOTSPD, "Cholesky pivot <= 0 in S^T A S at iteration " + std::to_string(h.k));
  // outputs (also on divergence: the last iterate)
  RS_TRY(write_weights(w_out, w_mem, alpha_out));
  if (timing)
    fprintf(stderr, "[rs] solve loop %.3f ms host (%.3f device), %lld graph launches; outputs %.3f ms\n",
            std::chrono::duration<double, std::milli>(h2 - h1).count(), solve_ms, graph_launches, hms(h2));
  if (rc == RS_EDIVERGED)
    return fail(RS_EDIVERGED, "residual diverged (non-finite or > 1e8 relative) at iteration " +
                                  std::to_string(h.k));
  return RS_OK;
}

rs_status Problem::write_weights(double* w_out, rs_mem w_mem, double* alpha_out) {
  const cudaMemcpyKind kd = w_mem == RS_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (route == 1) {
    RS_CUDA(cudaMemcpyAsync(w_out, w, m * 8, kd, st));
  } else if (fmt == 0) {   // dense dual: w = X^T alpha; feature shards assembled
    const double* Xd = dual_r ? Xo : X;
    const long long ldd = dual_r ? ldxo : ldx, dl = dual_r ? cols_loc : d;
    double *wd = nullptr, *work = nullptr;
    RS_TRY(dalloc(&wd, d));
    rs_status s = dalloc(&work, dense_xty_work(n, std::max<long long>(dl, 1)));
    if (s == RS_OK && world > 1 && launch_fill(wd, d, 0.0, st) != cudaSuccess) s = fail(RS_ECUDA, "dual weights");
    if (s == RS_OK && dl > 0 && launch_dense_xty(Xd, ldd, n, dl, w, wd + (world > 1 ? col0 : 0), work, st) != cudaSuccess)
      s = fail(RS_ECUDA, "dual weights");
    if (s == RS_OK && world > 1) s = allreduce(wd, (size_t)d);   // zero-padded feature blocks
    if (s == RS_OK && cudaMemcpyAsync(w_out, wd, d * 8, kd, st) != cudaSuccess) s = fail(RS_ECUDA, "copy w");
    cudaStreamSynchronize(st);
    dfree(wd);
    dfree(work);
    RS_TRY(s);
    if (alpha_out) RS_CUDA(cudaMemcpyAsync(alpha_out, w, m * 8, cudaMemcpyDeviceToHost, st));
  } else {
    RS_TRY(csr_dual_weights(w_out, kd));
    if (alpha_out) RS_CUDA(cudaMemcpyAsync(alpha_out, w, m * 8, cudaMemcpyDeviceToHost, st));
  }
  RS_CUDA(cudaStreamSynchronize(st));
  return RS_OK;
}

}  // namespace rs

// ================================================================================================
// C ABI
using rs::Problem;
using rs::fail;

extern "C" {

rs_status rs_create_dense(rs_problem* out, int64_t n, int64_t d, const double* X_local, int64_t ldx,
                          const double* y, double lambda, rs_route route, rs_as_mode mode,
                          rs_mem mem, const rs_dist* dist) {
  return rs::create_dense(out, n, d, X_local, ldx, y, lambda, route, mode, mem, dist);
}

rs_status rs_create_csr(rs_problem* out, int64_t n, int64_t d, int64_t nnz_local,
                        const int64_t* rowptr, const int32_t* colidx, const double* vals,
                        const double* y, double lambda, rs_route route, rs_as_mode mode, rs_mem mem,
                        const rs_dist* dist) {
  return rs::create_csr(out, n, d, nnz_local, rowptr, colidx, vals, y, lambda, route, mode, mem,
                        dist);
}

rs_status rs_solve(rs_problem p, const rs_solve_opts* opts, double* w_out, rs_mem w_mem,
                   double* alpha_out, rs_report* report) {
  if (!p) return fail(RS_EINVAL, "problem is NULL");
  return reinterpret_cast<Problem*>(p)->solve(opts, w_out, w_mem, alpha_out, report);
}

rs_status rs_get_state(rs_problem p, double* w_sys, double* r, rs_mem mem) {
  if (!p) return fail(RS_EINVAL, "problem is NULL");
  Problem* q = reinterpret_cast<Problem*>(p);
  if (!q->w) return fail(RS_EINVAL, "no state");
  const cudaMemcpyKind kd = mem == RS_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  cudaSetDevice(q->device);
  if (w_sys) RS_CUDA(cudaMemcpyAsync(w_sys, q->w, q->m * 8, kd, q->st));
  if (r) RS_CUDA(cudaMemcpyAsync(r, q->r, q->m * 8, kd, q->st));
  RS_CUDA(cudaStreamSynchronize(q->st));
  return RS_OK;
}

rs_status rs_get_info(rs_problem p, int64_t* m, int* route) {
  if (!p) return fail(RS_EINVAL, "problem is NULL");
  Problem* q = reinterpret_cast<Problem*>(p);
  if (m) *m = q->m;
  if (route) *route = q->route;
  return RS_OK;
}

rs_status rs_sketch_draw(rs_sketch_kind kind, int64_t m, int64_t tau, int64_t subcount_k,
                         uint64_t seed, int64_t iter, int device, int32_t* coord, int32_t* bucket,
                         int8_t* sign, int64_t* len_out) {
  if (m < 1 || m > 0x7fffffffLL || tau < 1 || tau > m || iter < 0 || iter > 0xffffffffLL)
    return fail(RS_EINVAL, "need 1 <= tau <= m < 2^31 and 0 <= iter < 2^32");
  if (!coord || !bucket || !sign || !len_out) return fail(RS_EINVAL, "NULL output");
  long long k = 1;
  if (kind == RS_SKETCH_SUBCOUNT) {
    k = subcount_k > 0 ? subcount_k : ((10 * tau <= m) ? 10 : m / tau);
    if (k * tau > m) return fail(RS_EINVAL, "subcount: k * tau > m");
  } else if (kind != RS_SKETCH_SUBSAMPLE && kind != RS_SKETCH_COUNT) {
    return fail(RS_EINVAL, "bad sketch kind");
  }
  if (kind == RS_SKETCH_COUNT && tau > 1536) return fail(RS_EUNSUPPORTED, "count tau > 1536");
  if (kind != RS_SKETCH_COUNT && tau * k > 8192) return fail(RS_EUNSUPPORTED, "selection > 8192");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(RS_ECUDA, "no CUDA device");
  RS_CUDA(cudaSetDevice(device));
  RS_CUDA(rs::sketch_init());
  rs::DevSketch sk{};
  sk.kind = (int)kind;
  sk.m = (int)m;
  sk.tau = (int)tau;
  sk.ksum = (int)k;
  sk.len = (int)rs::sketch_max_len(sk.kind, sk.m, sk.tau, sk.ksum);
  const size_t L = sk.len;
  RS_CUDA(cudaMalloc(&sk.coord, L * 4));
  RS_CUDA(cudaMalloc(&sk.bucket, L * 4));
  RS_CUDA(cudaMalloc(&sk.sign, L));
  RS_CUDA(cudaMalloc(&sk.bptr, (tau + 1) * 4));
  if (kind == RS_SKETCH_COUNT) RS_CUDA(cudaMalloc(&sk.cmap, m * 4));
  cudaError_t e = rs::launch_sketch(sk, seed, nullptr, iter, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(coord, sk.coord, L * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(bucket, sk.bucket, L * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(sign, sk.sign, L, cudaMemcpyDeviceToHost);
  int serr = 0;
  if (e == cudaSuccess) e = rs::sketch_err_take(&serr);
  cudaFree(sk.coord);
  cudaFree(sk.bucket);
  cudaFree(sk.sign);
  cudaFree(sk.bptr);
  if (sk.cmap) cudaFree(sk.cmap);
  if (e != cudaSuccess) return fail(RS_ECUDA, std::string("sketch draw: ") + cudaGetErrorString(e));
  if (serr) return fail(RS_EUNSUPPORTED, "sketch selection: more than 1024 coordinates share one 64-bit key");
  *len_out = (int64_t)L;
  return RS_OK;
}

rs_status rs_shard_range(int64_t total, int rank, int world, int64_t* begin, int64_t* len) {
  if (total < 0 || world < 1 || rank < 0 || rank >= world || !begin || !len)
    return fail(RS_EINVAL, "bad shard arguments");
  const int64_t q = total / world, rem = total % world;
  *begin = rank * q + std::min<int64_t>(rank, rem);
  *len = q + (rank < rem ? 1 : 0);
  return RS_OK;
}

rs_status rs_shard_rows_nnz(int64_t n_rows, const int64_t* rowptr, int rank, int world,
                            int64_t* begin, int64_t* len) {
  if (n_rows < 0 || !rowptr || world < 1 || rank < 0 || rank >= world || !begin || !len)
    return fail(RS_EINVAL, "bad shard arguments");
  // boundary t (t = 1..world-1) = first row whose prefix nnz reaches t * nnz / world
  const int64_t nnz = rowptr[n_rows];
  auto boundary = [&](int t) -> int64_t {
    if (t <= 0) return 0;
    if (t >= world) return n_rows;
    const long double target = (long double)nnz * t / world;
    int64_t lo = 0, hi = n_rows;   // smallest row index i with rowptr[i] >= target
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if ((long double)rowptr[mid] >= target) hi = mid;
      else lo = mid + 1;
    }
    return lo;
  };
  const int64_t b0 = boundary(rank), b1 = boundary(rank + 1);
  *begin = b0;
  *len = std::max<int64_t>(0, b1 - b0);
  return RS_OK;
}

rs_status rs_nccl_unique_id(void* out128) {
  if (!out128) return fail(RS_EINVAL, "NULL output");
  std::string err;
  const rs::NcclApi* api = rs::nccl_api(&err);
  if (!api) return fail(RS_ENCCL, err);
  ncclUniqueId id;
  ncclResult_t e = api->ncclGetUniqueId(&id);
  if (e != ncclSuccess) return fail(RS_ENCCL, api->ncclGetErrorString(e));
  std::memcpy(out128, &id, sizeof(id));
  return RS_OK;
}

rs_status rs_host_coll_id(void* out128) {
  if (!out128) return fail(RS_EINVAL, "NULL output");
  rs::hostcoll_new_name(static_cast<char*>(out128));
  return RS_OK;
}

void rs_destroy(rs_problem p) { delete reinterpret_cast<Problem*>(p); }

const char* rs_status_string(rs_status s) {
  switch (s) {
    case RS_OK: return "RS_OK";
    case RS_EINVAL: return "RS_EINVAL: invalid argument";
    case RS_EUNSUPPORTED: return "RS_EUNSUPPORTED: not implemented";
    case RS_ENOMEM: return "RS_ENOMEM: device allocation failed";
    case RS_ECUDA: return "RS_ECUDA: CUDA failure";
    case RS_ENCCL: return "RS_ENCCL: NCCL failure";
    case RS_ENOTSPD: return "RS_ENOTSPD: sketched system not positive definite";
    case RS_EDIVERGED: return "RS_EDIVERGED: residual diverged";
  }
  return "unknown rs_status";
}

const char* rs_last_error(void) { return rs::g_last_error.c_str(); }

int rs_abi_version(void) { return RS_ABI_VERSION; }

}  // extern "C"
