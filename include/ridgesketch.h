/* ridgesketch.h -- C ABI of the B200-native momentum sketch-and-project ridge solver.
 *
 * Method: RidgeSketch (Gazagnadou, Ibrahim, Gower, arXiv 2105.05565).  Citations "P:Lnnn" are
 * lines of the paper text (/root/reference/PAPER.md, not needed at run time).
 *
 *   Ridge regression  min_w 1/2||X w - y||^2 + lambda/2 ||w||^2, lambda > 0     (Eq. ridge)
 *   is solved as the SPD system  A w = b                                          (Eq. Axb)
 *     primal (d <= n):  A = X^T X + lambda I (m = d),  b = X^T y
 *     dual   (n <  d):  A = X X^T + lambda I (m = n),  b = y,  w = X^T alpha
 *   by Alg. 2, sketch-and-project with heavy-ball momentum:
 *     delta_k = (S_k^T A S_k)^{-1} S_k^T r^k
 *     w^{k+1} = w^k - gamma S_k delta_k + beta (w^k - w^{k-1})
 *     r^{k+1} = r^k - gamma A S_k delta_k + beta (r^k - r^{k-1})                  (Eq. res_update_mom)
 *   stopping when ||r^k|| <= tol ||r^0|| or k = max_iter
 *   with S_k a subsample, count or SubCount sketch drawn
 *   from the seeded counter-based sketch stream of DESIGN.md Section 3.
 *
 * All floating point is IEEE binary64.  Every computational step of an iteration runs in this
 * library's CUDA kernels (sm_100a); the host only launches them.  There is no CPU fallback: a
 * missing or unusable GPU is reported as RS_ECUDA.
 *
 * Conventions.
 *   - Every function returns rs_status; on failure nothing is written to outputs and a
 *     human-readable detail is available from rs_last_error() (thread-local).
 *   - "device" pointers are CUDA device (or managed) pointers of the current process; "host"
 *     pointers are ordinary (optionally pinned) host memory.
 *   - Dense matrices are row-major with a leading dimension (elements between rows).
 *   - CSR: rowptr int64[n_rows+1] (monotone, rowptr[0] = 0, rowptr[n_rows] = nnz), colidx
 *     int32[nnz] (strictly increasing within each row, in range), vals double[nnz].
 *   - When world > 1 every call taking an rs_problem is collective over the ranks.
 *   - Handles are not thread-safe; distinct handles may be used from distinct threads.
 */
#ifndef RIDGESKETCH_H
#define RIDGESKETCH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 5

typedef struct rs_problem_t* rs_problem;

typedef enum {
  RS_OK = 0,
  RS_EINVAL = 1,        /* invalid argument: dimensions, lambda <= 0, non-finite data, CSR
                           invariants, tau not in [1, m], subcount k*tau > m, gamma not in (0,1],
                           beta not in [0,1], tol < 0, max_iter < 0, NULL pointers            */
  RS_EUNSUPPORTED = 2,  /* valid but not implemented (e.g. CSR GRAM with tau > 1536, kernel
                           ridge with world > 1)                                              */
  RS_ENOMEM = 3,        /* device allocation failed                                           */
  RS_ECUDA = 4,         /* CUDA runtime / launch failure, or no usable device                 */
  RS_ENCCL = 5,         /* NCCL failure; the communicator is aborted, only rs_destroy is legal */
  RS_ENOTSPD = 6,       /* a Cholesky pivot of S^T A S was <= 0 or not finite                 */
  RS_EDIVERGED = 7      /* maintained residual non-finite or ||r||/||b|| > 1e8; the
                           norms are fp64 sums of squares, so this is also the outcome when
                           ||b||^2 leaves the fp64 range (||b|| > ~1e154)                      */
} rs_status;

typedef enum { RS_ROUTE_AUTO = 0, RS_ROUTE_PRIMAL = 1, RS_ROUTE_DUAL = 2 } rs_route;

/* How A S is formed (R10).
 *   IMPLICIT: A S = X^T (X S) + lambda S (primal) or X (X^T S) + lambda S (dual); A never formed.
 *   EXPLICIT: A = B + lambda I is built once in rs_create (dense X: lower-tile DMMA product;
 *             CSR X: dense A from the sparse rows, RS_ENOMEM if m x m doubles do
 *             not fit), and every iteration gathers / sums the sketched rows of A (A symmetric,
 *             so rows = columns).
 *   GRAM    : (dense primal, CSR primal and dual) A S is never formed:
 *             G = (RS)^T(RS) + lambda S^T S with R = X (primal) or X^T (dual), and
 *             A S delta = R^T (R S delta) + lambda S delta (one streaming pass over X per iteration).
 *             Same iterates as IMPLICIT in exact arithmetic.                       */
typedef enum { RS_AS_IMPLICIT = 0, RS_AS_EXPLICIT = 1, RS_AS_GRAM = 2 } rs_as_mode;

typedef enum {
  RS_SKETCH_SUBSAMPLE = 0,   /* S = I_C, |C| = tau, uniform over tau-subsets (Eq. subsample)   */
  RS_SKETCH_COUNT = 1,       /* each coordinate -> one hashed bucket with a random sign         */
  RS_SKETCH_SUBCOUNT = 2     /* S^T = Sigma D I_C, |C| = s = k tau (Eq. Sigmacount)             */
} rs_sketch_kind;

/* Where caller buffers live and who owns them.
 *   HOST          : host memory; copied (H2D) into library-owned device memory.
 *   DEVICE_COPY   : device memory; copied (D2D) into library-owned device memory.
 *   DEVICE_BORROW : device memory used in place; the caller keeps it alive and unchanged until
 *                   rs_destroy.  (Dense X is copied anyway if ldx is not a multiple of 4.)
 * Device inputs must be complete when the call is made: the library works on its own stream
 * (or rs_dist.cuda_stream), which is not ordered with the producer's stream -- synchronise the
 * producer (or pass its stream in rs_dist) first. */
typedef enum { RS_MEM_HOST = 0, RS_MEM_DEVICE_COPY = 1, RS_MEM_DEVICE_BORROW = 2 } rs_mem;

/* Collective backend of a multi-rank problem (rs_dist.collective).
 *   NCCL : ncclAllReduce (sum, fp64) on the solver stream, one process per GPU -- production.
 *   HOST : host-staged sum over a POSIX shared-memory segment of the world's processes on one
 *          machine, the ranks' buffers summed in rank order (the same result on every rank); each
 *          allreduce is a D2H copy, a host function node and an H2D copy on the solver stream (so
 *          it is captured in the iteration graph like the NCCL call).  No kernel waits on another
 *          rank, so several ranks may share one GPU: this is how the multi-rank path is executed
 *          and tested on a single-GPU machine.  A rank waiting more than 300 s for the others
 *          fails the solve with RS_ENCCL. */
typedef enum { RS_COLL_NCCL = 0, RS_COLL_HOST = 1 } rs_collective;

/* Process layout (one process per GPU, or, with RS_COLL_HOST, any number of rank processes on one
 * machine).  NULL means world = 1 on the current device with the whole X.  Primal: X_local holds
 * rows [shard_begin, shard_begin + shard_len) of X.  Dual: X_local holds columns
 * [shard_begin, shard_begin + shard_len) (features).  Sketches are regenerated on every rank from
 * (seed, k); the per-iteration exchange is a sum-allreduce of the partial A S (IMPLICIT) or of
 * u = R^T R S delta (GRAM, plus one allreduce of a sketch-ahead group's Grams); EXPLICIT iterations
 * need none. */
typedef struct {
  int device;                  /* CUDA device ordinal used by this rank                         */
  int rank, world;
  const void* nccl_unique_id;  /* 128 bytes, the same on every rank, ignored when world == 1:
                                  NCCL: from rs_nccl_unique_id() on rank 0;
                                  HOST: from rs_host_coll_id() on rank 0 (a segment name)       */
  void* cuda_stream;           /* cudaStream_t to run on, or NULL for a library-owned stream     */
  int64_t shard_begin, shard_len;
  int collective;              /* rs_collective (0 = NCCL)                                      */
} rs_dist;

/* Create a problem from dense X (n x d, row-major, leading dimension ldx >= d) and y (n).
 * n, d are the GLOBAL dimensions.  Primal route: for world > 1, X_local / y are the rank's shard of
 * rows (y the matching rows).  Dual route (n < d): X_local is the rank's block of columns
 * [shard_begin, shard_begin + shard_len) (n x shard_len, ld ldx) and y is whole; EXPLICIT builds
 * A = X X^T + lambda I (one GPU), IMPLICIT / GRAM run the primal machinery on R = X^T (A = R^T R +
 * lambda I, feature shards = row shards of R); rs_solve returns w = X^T alpha.  GRAM needs
 * m <= 4096 (m = d primal, n dual). */
rs_status rs_create_dense(rs_problem* out, int64_t n, int64_t d, const double* X_local,
                          int64_t ldx, const double* y, double lambda, rs_route route,
                          rs_as_mode mode, rs_mem mem, const rs_dist* dist);

/* Create a problem from CSR X (local rows / local column block as in rs_create_dense; for a dual
 * column shard, colidx are LOCAL column indices in [0, shard_len)). */
rs_status rs_create_csr(rs_problem* out, int64_t n, int64_t d, int64_t nnz_local,
                        const int64_t* rowptr, const int32_t* colidx, const double* vals,
                        const double* y, double lambda, rs_route route, rs_as_mode mode,
                        rs_mem mem, const rs_dist* dist);

/* Kernel ridge regression (Section "Using a kernel"): the n x n system
 * K (K + lambda I) alpha = K y (Eq. kernelridge) with the Gaussian kernel
 * K_ij = exp(-||x_i - x_j||^2 / (2 sigma^2)) (Eq. Gausskernel), i.e. A = K^T (K + lambda I) and
 * b = K^T y, built on the device (K from X, A = K K + lambda K on FP64 tensor cores)
 * and solved by the EXPLICIT-mode path.  X: n x d row-major (ldx >= d), y: n; both copied (mem:
 * HOST or DEVICE_COPY/BORROW, read only during the call).  rs_solve returns alpha (n doubles) as
 * the weight vector; predictions on the inputs are K alpha.  Memory: 2 n^2 doubles
 * during setup, n^2 after.  Errors: RS_EINVAL (n, d < 1, lambda <= 0, sigma <= 0, ldx < d,
 * non-finite data), RS_EUNSUPPORTED (dist with world > 1: one GPU in this version). */
rs_status rs_create_kernel(rs_problem* out, int64_t n, int64_t d, const double* X, int64_t ldx,
                           const double* y, double lambda, double sigma, rs_mem mem,
                           const rs_dist* dist);

typedef struct {
  rs_sketch_kind kind;
  int64_t tau;          /* sketch size, 1 <= tau <= m                                         */
  int64_t subcount_k;   /* SubCount sum size k; 0 = the paper's rule                  */
  double gamma, beta;   /* constant step size in (0,1] and momentum in [0,1]  */
  double tol;           /* stop when ||r^k|| <= tol ||r^0|| (0: run exactly max_iter steps)    */
  int64_t max_iter;
  uint64_t seed;        /* sketch-stream seed                           */
  int64_t check_every;  /* iterations per CUDA-graph launch between host flag reads (0: 16)    */
  double* trace;        /* host, may be NULL: ||r^k||/||r^0|| for k = 1..trace_cap             */
  int64_t trace_cap;
  int profile;          /* 1: time every kernel class with CUDA events inside the graph       */
  int momentum;         /* rs_momentum: how (gamma_k, beta_k) evolve           */
  double eta;           /* schedule parameter eta in (0, 1) (HEURISTIC, THEORY, COR1)          */
} rs_solve_opts;

/* Momentum parameter schedules (Section "Momentum"):
 *   CONSTANT : gamma_k = gamma, beta_k = beta ("constant beta setting")
 *   HEURISTIC: gamma_k = 1, beta_k = 1 - (2 - eta) / ((k+1)(1-eta) + 1)  (Eq. parametersheurististic,
 *              P:L937-942); eta = 0.995 in the equations, 0.5 in the figure captions (DESIGN R17)
 *   THEORY   : eta_k = eta while beta < 0.5, then 1 (Eq. parameterswitchtheory; DESIGN
 *              R24), zeta_k from Thm. 1 (Eq. zeta_kaptheo), mapped to (gamma_k, beta_k) by
 *              Eq. etalambdatogammbetagen
 *   COR1     : constant eta < 1, gamma_k = eta / ((k+1)(1-eta) + 1), beta_k as HEURISTIC (Cor. 1,
 *              Eq. cst_eta_lambda_to_gamma_beta_formula)
 * gamma and beta of the options are ignored by the non-constant schedules.  Errors: RS_EINVAL for
 * an unknown schedule or eta outside (0, 1). */
typedef enum { RS_MOM_CONSTANT = 0, RS_MOM_HEURISTIC = 1, RS_MOM_THEORY = 2, RS_MOM_COR1 = 3 } rs_momentum;

/* Kernel classes reported in rs_report.kernel_ms (summed over the solve) when profile = 1. */
enum {
  RS_K_SKETCH = 0,   /* a1 sketch draw                                                  */
  RS_K_XS = 1,       /* a2 column gather / signed segmented sum (X S, X^T S, rows of A)  */
  RS_K_AS = 2,       /* a3 contraction A S (+ split-K reduce, allreduce, + lambda S);
                        GRAM mode: the X^T (X S delta) streaming pass                     */
  RS_K_SOLVE = 3,    /* a4 + a5 S^T A S, S^T r, Cholesky, triangular solves, S delta     */
  RS_K_UPDATE = 4,   /* a6 fused momentum update + ||r||^2 + stop flag                   */
  RS_K_GRAM = 5,     /* GRAM mode: G = (XS)^T XS contraction (+ allreduce)               */
  RS_K_PRE = 6,      /* sketch-ahead group precompute (EXPLICIT / GRAM modes): the P sketches
                        (and A S^T rows); the P Grams are counted under GRAM (and, CSR, the
                        hashed rows of R S under XS), per iteration they belong to            */
  RS_K_FACTOR = 7,   /* sketch-ahead: batched Cholesky + inverse of the P matrices G_k, counted
                        once per group of P iterations                                        */
  RS_K_NCLASSES = 8
};

typedef struct {
  int64_t iterations;        /* number of updates performed                                    */
  int converged;             /* 1 if ||r|| <= tol ||r^0||                                       */
  double rel_residual;       /* ||r^t|| / ||r^0|| of the maintained residual                    */
  double setup_seconds;      /* rs_create device work (b = X^T y, explicit A build)             */
  double solve_seconds;      /* CUDA-event time of the iteration loop on the solver stream      */
  int64_t trace_len;
  double kernel_ms[RS_K_NCLASSES];       /* profile = 1 only                                    */
  int64_t kernel_launches[RS_K_NCLASSES];
  int64_t gpu_launches;      /* CUDA kernels launched by the iteration loop (graph nodes run,
                                including no-op launches after the stop flag in the last chunk) */
  int32_t overlap_sms;       /* EXPLICIT, tau > 224, overlapped pipeline: SMs running the group
                                kernel while the next group's factorisation runs on the others;
                                0 when the solve did not overlap                                  */
  int32_t inverse_blocks;    /* tau > 224 on the group kernel: diagonal super-blocks nb of the
                                factor slots' blocked inverse (W_bb = L_bb^{-1} on the diagonal,
                                L below; per G_k tau^3/3 + tau^3/(3 nb^2) flop); 1 = W = L^{-1} in
                                full; 0 when no large-tau factor slots were used                    */
} rs_report;

/* Run Alg. 2 from w^0 = 0.  w_out: d doubles (the ridge weights; dual: X^T alpha), host memory
 * when w_mem == RS_MEM_HOST else device.  alpha_out: n doubles (dual only, host), may be NULL. */
rs_status rs_solve(rs_problem p, const rs_solve_opts* opts, double* w_out, rs_mem w_mem,
                   double* alpha_out, rs_report* report);

/* Copy the state after the last rs_solve: the system iterate (w if primal, alpha if dual; m
 * doubles) and the maintained residual r (m doubles).  Either pointer may be NULL.  mem: HOST or
 * DEVICE_COPY (device destination). */
rs_status rs_get_state(rs_problem p, double* w_sys, double* r, rs_mem mem);

/* System size m and route actually used (1 primal, 2 dual). */
rs_status rs_get_info(rs_problem p, int64_t* m, int* route);

/* Draw sketch S_it on the GPU with the same kernel the solver uses, and return its entries in
 * bucket order: coord[e], bucket[e] (int32) and sign[e] (+1/-1, int8), e < len, where len = tau
 * (subsample), m (count) or s = k tau (subcount).  Output arrays are host memory with room for
 * m entries.  device: CUDA ordinal. */
rs_status rs_sketch_draw(rs_sketch_kind kind, int64_t m, int64_t tau, int64_t subcount_k,
                         uint64_t seed, int64_t iter, int device, int32_t* coord,
                         int32_t* bucket, int8_t* sign, int64_t* len_out);

/* Host-only helpers (no GPU needed). */
/* Balanced shard of [0, total) for rank r of world (contiguous, sizes differ by at most 1). */
rs_status rs_shard_range(int64_t total, int rank, int world, int64_t* begin, int64_t* len);
/* nnz-balanced contiguous split of CSR rows: begin/len of rank's row block minimising the
 * maximum nnz per rank (greedy prefix split on rowptr). */
rs_status rs_shard_rows_nnz(int64_t n_rows, const int64_t* rowptr, int rank, int world,
                            int64_t* begin, int64_t* len);
/* Write 128 bytes of NCCL unique id (rank 0 only), loading NCCL on demand. */
rs_status rs_nccl_unique_id(void* out128);
/* Write 128 bytes naming a fresh RS_COLL_HOST group (rank 0 only; host only, no GPU needed). */
rs_status rs_host_coll_id(void* out128);

void rs_destroy(rs_problem p);
const char* rs_status_string(rs_status s);
const char* rs_last_error(void);
int rs_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RIDGESKETCH_H */
