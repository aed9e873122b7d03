// Problem object of the host engine (internal).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <string>
#include <vector>

#include "../../include/ridgesketch.h"
#include "rs_internal.cuh"
#include "hostcoll.h"

namespace rs {

rs_status fail(rs_status s, const std::string& msg);
rs_status validate_dist(const rs_dist* dist, long long total);
rs_status create_csr(rs_problem* out, int64_t n, int64_t d, int64_t nnz_local, const int64_t* rowptr,
                     const int32_t* colidx, const double* vals, const double* y, double lambda,
                     rs_route route, rs_as_mode mode, rs_mem mem, const rs_dist* dist);

struct CsrData;   // csr.cu

// Launch parameters baked into the captured iteration graph (tol / max_iter live in Ctrl).
struct GraphKey {
  int kind = -1, tau = 0, ksum = 0, chunk = 0, profile = 0;
  uint64_t seed = 0;
  double gamma = 0.0, beta = 0.0;
  bool operator==(const GraphKey& o) const {
    return kind == o.kind && tau == o.tau && ksum == o.ksum && chunk == o.chunk &&
           profile == o.profile && seed == o.seed && gamma == o.gamma && beta == o.beta;
  }
};

struct Problem {
  // placement
  int device = -1, num_sms = 148;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  int coll = 0;                    // rs_collective
  struct HostColl* hcoll = nullptr;   // RS_COLL_HOST
  // problem
  int fmt = 0;      // 0 dense, 1 CSR
  int route = 1;    // 1 primal (m = d), 2 dual (m = n)
  int mode = 0;     // rs_as_mode
  long long n = 0, d = 0, m = 0;
  long long rows_loc = 0;   // dense primal: local rows of X
  double lambda = 0.0;
  double* X = nullptr;
  long long ldx = 0;
  bool own_X = false;
  // dense dual in IMPLICIT / GRAM mode: X above is R = X_local^T (cols_loc x n); Xo is X_local
  // (n x cols_loc) for w = X^T alpha; col0 = the rank's first feature
  bool dual_r = false;
  double* Xo = nullptr;
  long long ldxo = 0, col0 = 0, cols_loc = 0;
  bool own_Xo = false;
  double* y = nullptr;
  double* b = nullptr;
  double bnorm2 = 0.0;
  double* A = nullptr;
  long long lda = 0;
  CsrData* csr = nullptr;
  double setup_seconds = 0.0;
  // iteration state (x, dx = x^k - x^{k-1}), R13
  double *w = nullptr, *dw = nullptr, *r = nullptr, *dr = nullptr, *sdelta = nullptr;
  Ctrl* ctrl = nullptr;
  Ctrl* ctrl_host = nullptr;
  double* trace_dev = nullptr;
  double* mom_tab_dev = nullptr;   // THEORY momentum schedule table
  double* scratch = nullptr;
  int last_status = 0;
  // per-(kind, tau) workspace
  int ws_kind = -1, ws_tau = -1, ws_ksum = -1, ws_depth = -1;
  DevSketch sk{};
  double* XS = nullptr;
  long long ld_xs = 0;
  double* ASt = nullptr;
  long long ld_as = 0;
  double* gemm_work = nullptr;
  GemmPlan gp{};
  TmaGemm tg{};
  // GRAM mode (NEXT-2)
  TmaGemm tg_gram{};
  double* Gram = nullptr;
  long long ld_gram = 0;
  double* xp_part = nullptr;
  double* uvec = nullptr;
  bool gram_fused = false;
  double* XT = nullptr;          // dense GRAM, subsample tau <= 200: transposed local rows (d x ldxt)
  long long ldxt = 0;
  bool use_tma = true;
  // sketch-ahead pipeline (bfactor.cu): P slots of (sketch, A S^T or Gram, Ginv, flag)
  bool pipe = false;
  int P = 0;
  DevSketch skb{};
  double* ASt_slots = nullptr;
  long long as_stride = 0;
  double* Gram_slots = nullptr;
  long long gram_stride = 0;
  double* Ginv_slots = nullptr;
  long long ld_gi = 0, gi_stride = 0;
  int* slot_flags = nullptr;
  int* bf_claim = nullptr;   // overlapped pipeline: factor SM registry + tickets (BfClaim)
  double* bf_work = nullptr;     // tau > 224: per-slot work matrices of the batched factorisation
  double* it_scratch = nullptr;  // EXPLICIT group kernel (iterate.cu): t, delta (tau each), partials
  bool use_iterate = false;
  int bf_sb = 0;               // super-block width of the blocked slot inverse (0: W = L^{-1} in full)
  // EXPLICIT, tau > 224: two slot sets of P; the next group's factorisation (st2) overlaps the
  // current group's iterations (st, k_iterate on the SMs the factor grid leaves free)
  bool pipe_xg = false;   // two slot sets
  bool pipe_ov = false;
  bool bf_dual = false;   // tau > 224: the 4-warp factorisation, two slots per SM
  int ov_sms = 32;        // overlapped pipeline: SMs of the group kernel (solve's model)
  int ws_xg = -1;
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_pro = nullptr, ev_pro_tail = nullptr;   // first set's tail on st2 (solve)
  SolveWork sw{};
  double* partials = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  GraphKey graph_key{};
  std::vector<cudaEvent_t> prof_events;
  long long kernels_per_iter = 0;   // kernel nodes of one graph launch (chunk iterations)

  ~Problem();
  void free_workspace();
  rs_status allreduce(double* buf, size_t count);
  rs_status ensure_workspace(int kind, int tau, int ksum, int depth, bool xg = false);
  rs_status enqueue_iteration(const rs_solve_opts* o, cudaEvent_t* ev);
  // split < nslots: the overlapped pipeline's first set, slots [split, nslots) factored on st2
  rs_status enqueue_precompute(const rs_solve_opts* o, int nslots, cudaEvent_t* ev, int split = 0);
  rs_status enqueue_pipelined_iteration(const rs_solve_opts* o, int slot, cudaEvent_t* ev);
  rs_status enqueue_iterate_group(const rs_solve_opts* o, int ns, cudaEvent_t* ev, int slot0 = 0,
                                  int grid = 0);
  rs_status enqueue_group_ov(const rs_solve_opts* o, int g, cudaEvent_t* ev);
  rs_status solve(const rs_solve_opts* o, double* w_out, rs_mem w_mem, double* alpha_out,
                  rs_report* rep);
  rs_status write_weights(double* w_out, rs_mem w_mem, double* alpha_out);
  // CSR parts (csr.cu)
  void csr_free();
  void csr_free_workspace();
  rs_status csr_ensure_workspace(int kind, int tau, int ksum);
  rs_status csr_enqueue_as(const rs_solve_opts* o, cudaEvent_t* ev);
  rs_status csr_dual_weights(double* w_out, cudaMemcpyKind kd);
  // CSR GRAM mode (csr_gram.cu)
  void csr_gram_free();
  rs_status csr_build_explicit();                              // csr_explicit.cu
  rs_status csr_gram_workspace(int kind, int tau);
  rs_status csr_enqueue_gram(const rs_solve_opts* o, cudaEvent_t* ev);
  rs_status csr_gram_into(const DevSketch& s, double* G, cudaEvent_t* ev, int slot = 0,
                          bool reduce = true);   // (R S)^T (R S)
  rs_status csr_gram_apply(const double* v, double* u,          // u = R^T (R v), local part
                           const DevSketch* s = nullptr);
};

rs_status finish_setup(Problem* p);
rs_status setup_common(Problem* p, const rs_dist* dist);

#define RS_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      return ::rs::fail(_e == cudaErrorMemoryAllocation ? RS_ENOMEM : RS_ECUDA,        \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));           \
  } while (0)

#define RS_TRY(expr)                  \
  do {                                \
    rs_status _s = (expr);            \
    if (_s != RS_OK) return _s;       \
  } while (0)

template <class T>
inline rs_status dalloc(T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
  if (e != cudaSuccess)
    return fail(RS_ENOMEM, std::string("cudaMalloc(") + std::to_string(n * sizeof(T)) +
                               " bytes): " + cudaGetErrorString(e));
  return RS_OK;
}

inline void dfree(void* p) {
  if (p) cudaFree(p);
}

inline long long round_up(long long x, long long q) { return (x + q - 1) / q * q; }

inline cudaMemcpyKind kind_of(rs_mem mem) {
  return mem == RS_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
}

}  // namespace rs
