// Internal declarations shared by the CUDA translation units of libridgesketch.so.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rs {

// ---------------------------------------------------------------------------------------------
// Device-resident control block: iteration counter, stop flag, residual norms.  Every per-iteration
// kernel reads `done` first and returns immediately when it is set, so a CUDA graph of K captured
// iterations stops exactly at the iteration where the stop rule fired (P:L729 while-condition).
enum : int {
  ST_RUNNING = 0, ST_CONVERGED = 1, ST_MAXITER = 2,
  // errors (>= ST_DIVERGED): set by the kernel that detects them; the update kernel turns them
  // into `done` (a cooperative kernel must never set `done` itself, see chol.cu)
  ST_DIVERGED = 3, ST_NOTSPD = 4, ST_OVERFLOW = 5,
  ST_SKETCHFAIL = 6   // sketch selection met > 1024 equal 64-bit keys (never seen; fails loudly)
};

struct Ctrl {
  long long k;          // iterations performed so far (the sketch of the next step is S_k)
  int done;             // 1: stop
  int status;           // ST_*
  double rnorm2;        // ||r^k||^2 of the maintained residual
  double bnorm2;        // ||r^0||^2 = ||b||^2
  double tol;
  long long max_iter;
  unsigned int arrive;  // last-block-done counter of the update kernel
  int pad;
  double* trace;        // device, may be null
  long long trace_cap;
  // momentum schedule (rs_momentum): 0 constant (kernel arguments), 1 heuristic, 2 table, 3 Cor. 1
  int mom_kind;
  int mom_pad;
  double mom_eta;
  const double* mom_tab;   // kind 2: (gamma_k, beta_k) pairs, k < mom_ntab; the last pair repeats
  long long mom_ntab;
};

// Programmatic dependent launch (PDL).  A kernel launched by launch_pdl may start while its
// predecessor in the stream is still running.  Everything it reads before pdl_wait() must have been
// written before the last ordinarily launched kernel of the chain (static data: A, the sketches, the
// factor slots, and ctrl->done of the previous iteration); pdl_wait() blocks until the predecessor
// grid has completed and its writes are visible (a no-op without the launch attribute);
// pdl_trigger() lets the successor launch.  RS_PDL=0 in the environment turns PDL off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}

// (gamma_k, beta_k) of iteration k = ctrl->k (read by the update kernels before ctrl->k moves on)
__device__ __forceinline__ void mom_at(const Ctrl* c, double& gamma, double& beta) {
  const int kind = c->mom_kind;
  if (kind == 0) return;
  const long long k = c->k;
  if (kind == 2) {
    const long long i = k < c->mom_ntab ? k : c->mom_ntab - 1;
    gamma = c->mom_tab[2 * i];
    beta = c->mom_tab[2 * i + 1];
    return;
  }
  const double eta = c->mom_eta;
  const double den = (double)(k + 1) * (1.0 - eta) + 1.0;
  beta = 1.0 - (2.0 - eta) / den;
  gamma = kind == 3 ? eta / den : 1.0;
}

// Sketch-ahead slot q of the group that starts at iteration ctrl->k is needed only if
// k + q < max_iter (and the solve is still running).
__device__ __forceinline__ bool slot_unused(const Ctrl* c, long long q) {
  return c && (c->done || c->k + q >= c->max_iter);
}

// ---------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11) -- the sketch-stream generator, DESIGN.md Section 3.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const unsigned lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    if (r < 9) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
  }
  return c;
}

// Sketch stream ids.
enum : unsigned { STREAM_SELECT = 0, STREAM_COUNT = 1, STREAM_SUBCOUNT_SIGN = 2 };
enum : int { SK_SUBSAMPLE = 0, SK_COUNT = 1, SK_SUBCOUNT = 2 };

// Device sketch in bucket order: entries e in [bptr[b], bptr[b+1]) belong to bucket b;
// S[coord[e], b] = sign[e].  For the count sketch cmap[i] = (bucket << 1) | (sign < 0) for every
// coordinate i (the per-coordinate table used by the CSR primal kernel).
struct DevSketch {
  int kind;
  int m, tau, len, ksum;  // len = number of entries; ksum = SubCount k
  int* coord;             // [len_cap]
  signed char* sign;      // [len_cap]
  int* bucket;            // [len_cap]
  int* bptr;              // [tau + 1]
  int* cmap;              // [m] (count only)
  // Batched sketches (pipelined modes): slot s of an array of sketches laid out with strides
  // len (coord/sign/bucket), tau + 1 (bptr) and m (cmap).
  __host__ __device__ DevSketch at(int s) const {
    DevSketch o = *this;
    o.coord += (long long)s * len;
    o.sign += (long long)s * len;
    o.bucket += (long long)s * len;
    o.bptr += (long long)s * (tau + 1);
    if (cmap) o.cmap += (long long)s * m;
    return o;
  }
};

// ---------------------------------------------------------------------------------------------
// Kernel launchers (each returns cudaGetLastError()).  All take the control block so that they can
// no-op once the solve has stopped.

// One-time per-process kernel setup (attributes, flags); must run outside any stream capture.
cudaError_t sketch_init();
cudaError_t gemm_init();
cudaError_t chol_init();
cudaError_t update_init();

// a1 sketch draw.  uses seed key and iteration k read from ctrl (or `fixed_k` >= 0 if given).
cudaError_t launch_sketch(const DevSketch& sk, uint64_t seed, const Ctrl* ctrl, long long fixed_k,
                          cudaStream_t st);
// Batched: slot s of `skb` (DevSketch::at) receives S_{k0 + s}, s < nslots, k0 = ctrl->k at launch
// (or fixed_k >= 0).  One CTA per slot.
// kofs: slot s receives S_{ctrl->k + kofs + s} (fixed_k < 0).
cudaError_t launch_sketch_batch(const DevSketch& skb, int nslots, uint64_t seed, const Ctrl* ctrl,
                                long long fixed_k, cudaStream_t st, long long kofs = 0);
size_t sketch_max_len(int kind, int m, int tau, int ksum);
// rs_sketch_draw (no control block): the select's failure flag, read and cleared
cudaError_t sketch_err_take(int* out);

// a2 dense: XS[i, b] = sum_{e in b} sign_e X[i, coord_e],  i < rows, row-major ld_xs (>= tau, pad
// columns zeroed).
cudaError_t launch_dense_xs(const double* X, long long ldx, long long rows, const DevSketch& sk,
                            double* XS, long long ld_xs, const Ctrl* ctrl, cudaStream_t st,
                            int slot = 0);
// a2 explicit: AS^T[b, :] = sum_{e in b} sign_e A[coord_e, :]  (A symmetric, m x m, ld lda).
cudaError_t launch_explicit_rows(const double* A, long long lda, long long m, const DevSketch& sk,
                                 double* ASt, long long ld_as, const Ctrl* ctrl, cudaStream_t st);
// Batched over `nslots` sketch slots: AS^T of slot s at ASt + s * as_stride.
cudaError_t launch_explicit_rows_batch(const double* A, long long lda, long long m,
                                       const DevSketch& skb, int nslots, double* ASt,
                                       long long ld_as, long long as_stride, const Ctrl* ctrl,
                                       cudaStream_t st);

// a3 dense TN contraction on FP64 tensor cores (DMMA):  C[M' x N'] (row-major, ldc) =
//   sum_{k < K} Aop[k, 0:M'] (x) Bop[k, 0:N']  with Aop row-major (lda), Bop row-major (ldb),
// split over `splits` K-ranges into `work` and reduced deterministically.  If work == nullptr,
// splits must be 1.
struct GemmPlan {
  int variant, bm, bn, splits;
  long long k_per_split;
  size_t work_elems;
};
GemmPlan plan_tn_gemm(long long M, long long N, long long K, int num_sms);
cudaError_t launch_tn_gemm(const double* Aop, long long lda, const double* Bop, long long ldb,
                           long long M, long long N, long long K, double* C, long long ldc,
                           const GemmPlan& plan, double* work, const Ctrl* ctrl, cudaStream_t st);

// Same contraction, TMA + mbarrier warp-specialised pipeline (gemm_tma.cu).  tmA / tmB hold two
// CUtensorMap descriptors (64-byte aligned opaque blobs) encoded by tma_gemm_plan.
struct TmaGemm {
  alignas(64) unsigned char tmA[128];
  alignas(64) unsigned char tmB[128];
  int variant = 0, splits = 1, bm = 0, bn = 0;
  int lower = 0;   // 1: only tiles touching the lower triangle (C symmetric, e.g. A = X^T X)
  long long M = 0, N = 0, K = 0, k_per_split = 0, ldw = 0;
  size_t work_elems = 0;
};
// A[j][i] = A[i][j] for i > j (upper triangle from the lower one), m x m, ld lda.
cudaError_t launch_mirror_lower(double* A, long long lda, long long m, cudaStream_t st);
cudaError_t tma_gemm_init();
cudaError_t tma_gemm_plan(TmaGemm* g, const double* Aop, long long lda, const double* Bop,
                          long long ldb, long long M, long long N, long long K, int num_sms, int lower = 0);
cudaError_t tma_gemm_launch(const TmaGemm& g, double* C, long long ldc, double* work,
                            const Ctrl* ctrl, cudaStream_t st);

// The EXPLICIT iterations of a sketch-ahead group as one persistent cooperative kernel (iterate.cu).
struct IterArgs {
  const double* Ginv;            // factor slots: G^{-1} (tau <= 224) or W lower / W^T upper
  long long ld_gi, gi_stride;
  DevSketch skb;                 // slot q's sketch: skb.at(q)
  const int* flags;              // slot not SPD
  const double* A;               // explicit A (rows of A S for subsample / SubCount), or
  long long lda;
  const double* ASt;             // the slots' A S^T rows (count sketch), null otherwise
  long long ld_as, as_stride;
  long long m;
  double *w, *dw, *r, *dr, *sdelta;
  double *tvec, *dvec;           // tau each
  double* partials;              // one per CTA (grid = num_sms)
  double gamma, beta;
  int nslots;                    // iterations of the group
  int big;                       // tau > 224
  int sb;                        // tau > 224: super-block width of the slot's blocked inverse
                                 // (bfactor.cu; 0 or >= tau: W = L^{-1} in full)
  int wait;                      // flags[q] < 0: slot q is still being factored (by a concurrent
                                 // kernel), spin until it is 0 or 1
};
size_t iterate_smem();
bool iterate_ok(const DevSketch& sk, long long m, int grid);   // the group kernel applies
cudaError_t iterate_init();
cudaError_t launch_iterate(const IterArgs& args, int grid, Ctrl* ctrl, cudaStream_t st);

// lambda S:  AS^T[b_e, coord_e] += lambda * sign_e  (as_rowmajor: AS[coord_e, b_e]).
cudaError_t launch_add_lambda_s(double lambda, const DevSketch& sk, double* ASt, long long ld_as,
                                bool as_rowmajor, const Ctrl* ctrl, cudaStream_t st);
// A += lambda I on a dense m x m.
cudaError_t launch_add_diag(double* A, long long lda, long long m, double lambda, cudaStream_t st);
// A[r][c] += T[r][c] for c <= r < m (lower triangles, ld lda)
cudaError_t launch_add_lower(double* A, const double* T, long long lda, long long m, cudaStream_t st);

// a4 + a5: G = S^T (A S) (lower), g = S^T r, empty-bucket rule, Cholesky, solves; writes
// sdelta[coord_e] = sign_e * delta[b_e].  Gx / delta are workspace.
struct SolveWork {
  double* Gx;        // (tau + 1) x ldg, row-major, lower triangle + border row tau = g
  long long ldg;
  double* delta;     // tau
  int grid;          // cooperative grid size for the Cholesky
};
SolveWork plan_solve(int tau, int num_sms);
size_t solve_gx_elems(int tau);
// AS layout: as_rowmajor = false -> AS^T stored tau x m (ld_as); true -> AS stored m x tau (ld_as).
// Gram mode (Gram != nullptr): G = Gram (tau x tau, ld_gram, lower read) + lambda diag(|bucket|).
cudaError_t launch_sketched_solve(const double* ASt, long long ld_as, bool as_rowmajor,
                                  const double* Gram, long long ld_gram, double lambda,
                                  const double* r, const DevSketch& sk, SolveWork& sw,
                                  double* sdelta, Ctrl* ctrl, cudaStream_t st);

// a6 fused update: u = AS delta (from AS^T rows), r/dr and w/dw heavy-ball, sdelta cleared,
// ||r||^2, stop flag and iteration counter.
size_t update_partials(long long m);
cudaError_t launch_update(const double* ASt, long long ld_as, bool as_rowmajor, int tau,
                          const double* delta, double* sdelta, double* w, double* dw, double* r,
                          double* dr, long long m, double gamma, double beta, double* partials,
                          Ctrl* ctrl, cudaStream_t st);

// Gram mode (gram.cu): u = X^T (X v) in one pass over X (d <= 4096), partials reduced in order.
size_t xpass_partials(long long d, int num_sms);
// Transposed copy XT (d x ldxt) of the local rows of X, and the Gram (XS)^T XS of a subsample
// sketch (tau <= 200) read from it as tau contiguous rows (partials: gram_fused_partials).
cudaError_t launch_transpose(const double* X, long long ldx, long long rows, long long d, double* XT,
                             long long ldxt, cudaStream_t st);
cudaError_t launch_gram_xt(const double* XT, long long ldxt, long long rows, const DevSketch& sk,
                           double* partials, double* G, long long ldg, int num_sms,
                           const Ctrl* ctrl, cudaStream_t st, int slot = 0);
// v = S delta (dense, m); when the sketch and delta are given and d <= 2048, the row-owner kernel
// forms <X_i, v> from the sketch entries only.
cudaError_t launch_xpass(const double* X, long long ldx, long long rows, long long d,
                         const double* v, double* partials, double* u, int num_sms,
                         const Ctrl* ctrl, cudaStream_t st, const DevSketch* sk = nullptr,
                         const double* delta = nullptr);
// Fused gather + Gram (subsample, tau <= 200): G lower = sum_i X[i,C]^T X[i,C], no XS written.
bool gram_fused_ok(int kind, int tau);
size_t gram_fused_partials(int num_sms);
cudaError_t gram_init();
cudaError_t launch_gram_fused(const double* X, long long ldx, long long rows, const DevSketch& sk,
                              double* partials, double* G, long long ldg, int num_sms,
                              const Ctrl* ctrl, cudaStream_t st,
                              int slot = 0);
// explicit A, sketch with few entries (subsample / SubCount):
//   u_j = sum_e sign_e delta[bucket_e] A[coord_e][j]  (= (A S delta)_j, A symmetric), then the update
cudaError_t launch_update_rows(const double* A, long long lda, const DevSketch& sk,
                               const double* delta, double* sdelta, double* w, double* dw,
                               double* r, double* dr, long long m, double gamma, double beta,
                               double* partials, int num_sms, Ctrl* ctrl, cudaStream_t st);
// update with a dense u = X^T X S delta:  u_j + lambda sdelta_j  is A S delta
cudaError_t launch_update_vec(const double* u, double lambda, double* sdelta, double* w, double* dw,
                              double* r, double* dr, long long m, double gamma, double beta,
                              double* partials, Ctrl* ctrl, cudaStream_t st);

// ---------------------------------------------------------------------------------------------
// Sketch-ahead pipeline (bfactor.cu).  G_k = S_k^T A S_k depends only on S_k (drawn from (seed, k),
// P:L214) and on the data, never on the iterate, so for a group of P future iterations the
// sketches, G_k and its factorisation are computed ahead in one batched pass (one CTA per G_k):
//   G = L L^T (Cholesky, lower triangle read, R12), W = L^{-1}, Ginv = W^T W  (full tau x tau).
// The iteration itself then needs only  delta = Ginv (S^T r).
struct FactorSrc {
  const double* ASt;      // AS^T slots (tau x ld_as each, slot stride as_stride), or null
  long long ld_as, as_stride;
  const double* Gram;     // Gram slots (XS)^T XS (tau x ld_gram, stride gram_stride), or null
  long long ld_gram, gram_stride;
  double lambda;          // Gram source: G = Gram + lambda S^T S
  const double* A;        // explicit A (m x m, lda): G[a][c] = sum_{e in a, f in c} s_e s_f A[e][f]
  long long lda;
};
int bfactor_max_tau();
cudaError_t bfactor_init();
// flags[s] = 1 if G of slot s was not SPD (a pivot <= 0 or non-finite after the empty-bucket rule)
// tau > 224: `work` = nslots x bfactor_work_elems(tau) doubles of scratch (null otherwise).
size_t bfactor_work_elems(int tau);
// tau > 224: `dual` selects the 4-warp k_bfactor_lp, two CTAs (slots) per SM -- for a wave of about
// 2 x (free SMs) slots; else the 8-warp shape, one CTA per SM.  claim (optional): slots are claimed
// dynamically by CTAs on every SM, of which those beyond max_sms distinct SMs step aside, leaving
// num_sms - max_sms SMs to a concurrent kernel; `words` (BF_CLAIM_WORDS ints, reset by the launch)
// is the launch's ticket and SM registry -- one per concurrently running launch.
constexpr int BF_CLAIM_WORDS = 4 + 256;
struct BfClaim {
  int* words;
  int max_sms, num_sms;
};
cudaError_t launch_bfactor(const FactorSrc& src, const DevSketch& skb, int nslots, double* Ginv,
                           long long ldgi, long long gi_stride, int* flags, double* work,
                           const Ctrl* ctrl, cudaStream_t st, bool dual = false,
                           const BfClaim* claim = nullptr, int sb = 0);
// delta = Ginv (S^T r), sdelta[coord_e] = sign_e delta[bucket_e]; flag != 0 -> status NOTSPD.
// tau <= 224: the slot holds G^{-1} (full); tau > 224: it holds W = L^{-1} (lower) and
// delta = W^T (W g).  gbuf: 2 tau doubles of scratch (g, W g).
cudaError_t launch_apply_ginv(const double* Ginv, long long ldgi, const DevSketch& sk,
                              const int* flag, const double* r, double* gbuf, double* delta,
                              double* sdelta, Ctrl* ctrl, cudaStream_t st, bool first = true,
                              const double* pfA = nullptr, long long pf_lda = 0, long long pf_m = 0);

// misc
// *out += number of non-finite entries of the rows x cols block.
cudaError_t launch_count_nonfinite(const double* X, long long ldx, long long rows, long long cols,
                                   unsigned long long* out, cudaStream_t st);
cudaError_t launch_fill(double* p, long long n, double v, cudaStream_t st);
cudaError_t launch_axpby_neg(const double* b, double* r, long long m, cudaStream_t st);  // r = -b
cudaError_t launch_dot_self(const double* x, long long n, double* out, cudaStream_t st);  // out = ||x||^2
// y_out[j] = sum_i X[i, j] y[i]  (dense X^T y, rows x cols, deterministic two-pass).
cudaError_t launch_dense_xty(const double* X, long long ldx, long long rows, long long cols,
                             const double* y, double* out, double* work, cudaStream_t st);
size_t dense_xty_work(long long rows, long long cols);

}  // namespace rs
