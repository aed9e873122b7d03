// CSR-X data of a problem (internal; csr.cu, csr_gram.cu).
#pragma once
#include <cuda_runtime.h>

#include "rs_internal.cuh"

namespace rs {

struct CsrData {
  long long rows = 0, cols = 0, nnz = 0;   // local block: rows x cols
  long long* rowptr = nullptr;
  int* colidx = nullptr;
  double* vals = nullptr;
  long long* colptr = nullptr;   // CSC
  int* rowidx = nullptr;
  double* cvals = nullptr;
  long long max_row_nnz = 0;
  long long col_offset = 0;      // dual: first global feature of this rank's column block
  // workspace
  int* cmap_all = nullptr;       // coordinate -> (bucket << 1 | neg) or -1 (subsample / SubCount)
  int hash_slots = 0, hash_log2 = 0, group = 0, chunks = 0;
  size_t dual_smem = 0;
  // GRAM mode (csr_gram.cu): the hashed rows of R = X (primal) or X^T (dual), the band plan of
  // the lower triangle of (RS)^T (RS), and the two SpMV vectors
  int* hb = nullptr;             // [nnz] bucket of the k-th merged entry of a row (ascending)
  double* hv = nullptr;          // [nnz] its value sum_{j in row, h(j) = b} sign_j R_ij
  int* hcnt = nullptr;           // [R rows] merged entries per row
  int* band_a0 = nullptr;        // [nbands + 1] first G row of every band
  long long* chunk_r0 = nullptr; // [nchunks + 1] first R row of every chunk (nnz-balanced)
  int nbands = 0, nchunks = 0;
  double* gpart = nullptr;       // [nchunks][tau (tau + 1) / 2] packed lower-triangle partials
  long long gpart_stride = 0;
  double* fsc = nullptr;         // per-bucket fixed-point scales 2^e_b of the current slot's Gram
  double* cnorm = nullptr;       // column norms of R (static; bounds of the bucket columns of R S)
  double* tvec = nullptr;        // [R rows]  t = R (S delta)
  // rows longer than `heavy` are handled one CTA per row (Zipf-popular features of c4)
  long long heavyR = 0, heavyRt = 0;
  int* heavy_rowsR = nullptr;
  int* heavy_rowsRt = nullptr;
  int nheavyR = 0, nheavyRt = 0;
  int* chunk_h0 = nullptr;       // [nchunks + 1] first heavy row (sorted list) of every chunk
  // dual GRAM with a subsample / SubCount sketch: R = X^T rows are formed from the s selected
  // samples only.  cscpos[p] = R (CSC) position of X's CSR entry p; cmR[q] = (bucket << 1 | neg)
  // of R entry q for this sketch, else -1; tflag / tlist / tcount: the touched R rows
  int* cscpos = nullptr;
  int* cmR = nullptr;
  int* tflag = nullptr;
  int* tlist = nullptr;
  int* tcount = nullptr;
  // heavy R rows on the selected-row path: hidx[f] = position of feature f in heavy_rowsR or -1;
  // hacc: per heavy row its row of R S as a dense tau-vector (ld ldh); their Gram contribution
  // H^T H is one lower-tile DMMA GEMM (tg_heavy) into gh, added by the band reduction
  int* hidx = nullptr;
  double* hacc = nullptr;
  long long ldh = 0;
  TmaGemm tg_heavy{};
  double* gh = nullptr;
  double* gh_work = nullptr;
  int* chunk_h0_none = nullptr;   // [nchunks + 1] zeros: k_gram_bands without its heavy phase
  size_t hr_smem = 0, gb_smem = 0;
  int gb_cap = 0;          // band capacity (doubles) before the per-warp row staging
  bool gb_stage = false;   // k_gram_bands<true>: light rows staged in shared memory
};

// per-iteration map coordinate -> (bucket << 1 | neg), -1 outside the sketch (subsample / SubCount)
cudaError_t launch_cmap_build(const DevSketch& sk, int* cmap_all, long long m, const Ctrl* ctrl,
                              cudaStream_t st, int slot = 0);

}  // namespace rs
