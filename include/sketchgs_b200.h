/*
 * sketchgs_b200.h -- C ABI of the B200 (sm_100a) randomized Gram-Schmidt /
 * randomized-GMRES hot path.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * passed as `void*`; no torch or numpy types cross this boundary.  All calls
 * are asynchronous on the given stream and return 0 on success or a negative
 * SGS_E* code (details in sgs_last_error()).  Numerical outcomes that the
 * reference reports by raising (BreakdownError, LinAlgError) are recorded in
 * the device-resident `sgs_status` block and read back by the host at sync
 * points; once a status code is set every later kernel that is handed the
 * same block returns immediately, so a host may enqueue ahead.
 *
 * The reference (`sketchgs`, pure Python) has no native boundary; each entry
 * point below replaces the reference function cited next to it
 * (paths relative to the reference's pkg/src/sketchgs/).
 *
 * Layouts (all column-major, "ld" = elements between consecutive columns):
 *   X, W, Q        n x ncols, ld >= n (ld % 4 == 0 for the vectorised kernels)
 *   S, P           k x cap  (fine dtype)
 *   R              cap x cap fp64, upper triangular
 *   Theta^T        n x ldt fp64 row-major (= Theta column-major), dense kinds
 *   sign_bits      one bit per local row, bit set = +1 (LSB-first in uint32)
 *   samples        nblocks x k int32, sorted ascending within each block
 */
#ifndef SKETCHGS_B200_H
#define SKETCHGS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGS_ABI_VERSION 1

/* dtype codes */
#define SGS_F32 0
#define SGS_F64 1

/* return codes */
#define SGS_OK 0
#define SGS_EINVAL (-1)
#define SGS_ECUDA (-2)
#define SGS_ENOMEM (-3)

/* sgs_status.code values (device-side outcomes) */
#define SGS_ST_OK 0
#define SGS_ST_BREAKDOWN 1   /* reference: gram_schmidt.BreakdownError (gram_schmidt.py:323-326) */
#define SGS_ST_RANK 2        /* reference: np.linalg.LinAlgError (gram_schmidt.py:186-189) */
#define SGS_ST_CONVERGED 3   /* reference: gmres early exit est <= tol (krylov.py:300-301) */
#define SGS_ST_TIMEOUT 4     /* a wait on another rank's published data gave up */
/* (no code 4: a NaN r_ii flows through as in the reference, which has no
   non-finite guard - gram_schmidt.py:322-326 only compares r_ii <= tol) */

/* Device-resident status block (64 bytes, 8-byte aligned). */
typedef struct sgs_status {
  int64_t code;      /* SGS_ST_* */
  int64_t column;    /* 1-based column the code refers to */
  int64_t ncols;     /* columns committed to Q/R/S (RgsState.m) */
  int64_t iters;     /* GMRES iterations completed in this cycle */
  double r_ii;       /* last diagonal (or offending r_ii on breakdown) */
  double tol;        /* breakdown tolerance that was compared against */
  double diag_max;   /* running max |diag R_S| of the sketched-basis QR */
  double diag_min;   /* running min |diag R_S| */
} sgs_status;

/* ---- library ------------------------------------------------------------ */
int sgs_abi_version(void);
/* debug: %globaltimer stamps per column (8 x u64 each) into buf; NULL disables */
void sgs_debug_timeline(void* buf);
void sgs_debug_timeline_col(int64_t col);
const char* sgs_last_error(void);
/* number of kernels this library has launched (process-wide counter) */
uint64_t sgs_launch_count(void);
int sgs_device_sm_count(int device);
int sgs_status_init(sgs_status* st, void* stream);

/* ---- sketch operators ----------------------------------------------------
 * Replaces SketchOperator.apply / apply_block (sketch.py:168-198) and fwht
 * (sketch.py:90-109).  A P-SRHT of the reference is nblocks=1 with
 * log2_block = log2(next_pow2(n)); a block-SRHT is nblocks contiguous
 * 2^log2_block-row blocks each with its own signs/samples.  Partials are
 * per-CTA unscaled k-vectors: partials[(c*nparts + p)*k + j].  The number of
 * parts is a pure function of (n_local, log2_block) so every caller that
 * sketches the same vector gets bit-identical results. */
int sgs_srht_nparts(int64_t n_local, int log2_block);
int sgs_srht_partials(const void* X, int x_dtype, int64_t ldx, int ncols,
                      int64_t n_local, int64_t row0, int log2_block,
                      const uint32_t* sign_bits, const int32_t* samples, int k,
                      double* partials, const sgs_status* st, void* stream);
/* sgs_srht_partials with the CTA geometry of 4096-row tiles chosen: 0 as
 * sgs_srht_partials (by size), 1 one CTA per 4 consecutive tiles (a small
 * grid: a following cluster launch can be resident alongside), 2 one tile
 * per CTA with a 4-CTA cluster sum.  Bit-identical partials for all three. */
int sgs_srht_partials_geom(const void* X, int x_dtype, int64_t ldx, int ncols,
                           int64_t n_local, int64_t row0, int log2_block,
                           const uint32_t* sign_bits, const int32_t* samples, int k,
                           double* partials, int geom, const sgs_status* st, void* stream);
/* Two SRHT-kind sketches of the same columns in one pass (the P batch of
 * rgs_factorize with a certification sketch Phi: P = Theta W and
 * P_phi = Phi W, gram_schmidt.py:303-305 per column).  Both need 4096-row
 * tiles (log2 blocks >= 12); each partials array equals sgs_srht_partials'
 * of its sketch bit for bit.  W is read from HBM once; the second transform
 * re-reads each tile from L1/L2. */
int sgs_srht_partials_pair(const void* X, int x_dtype, int64_t ldx, int ncols,
                           int64_t n_local, int64_t row0, int log2_block,
                           const uint32_t* sign_bits, const int32_t* samples, int k,
                           double* partials, int log2_block2, const uint32_t* sign_bits2,
                           const int32_t* samples2, int k2, double* partials2,
                           const sgs_status* st, void* stream);

/* Dense sketch (Gaussian, absent from the reference's SketchKind; duck-typed
 * in through sketch.py:120-206; a column block sketched as the dense
 * contraction sketch.py:186-198 does column by column): partials of
 * Theta^T' X on the fp64 tensor cores (DMMA, mma.sync m8n8k4 f64).  The rows
 * are split into sub-chunks, each a chain of 4-row DMMA steps in ascending
 * order; 8 consecutive sub-chunks are summed in a thread-block cluster, so
 * sgs_gaussian_nparts(n) (<= 37) partials per column.  ncols == 1 runs the
 * same chains, so apply_block is bit-identical to apply.
 * SGS_DENSE_LEGACY=1 selects the DFMA GEMV / split-K GEMM with
 * sgs_dense_nparts(n) partials instead. */
int sgs_gaussian_nparts(int64_t n);
/* Row chunks of the packed-sign Rademacher partials (and of the legacy dense
 * kernels): min(296, ceil(n / 32)). */
int sgs_dense_nparts(int64_t n);
/* Partial k-vectors per column written by sgs_rgs_update_dense (its own
 * 16-row-aligned chunking, about two chunks per SM). */
int sgs_dense_column_nparts(int64_t n_local, int k);
int sgs_dense_partials(const double* thetaT, int64_t ldt, int k,
                       const void* X, int x_dtype, int64_t ldx, int ncols,
                       int64_t n, double* partials, const sgs_status* st,
                       void* stream);

/* Rademacher sketch generated on the device (SketchKind.RADEMACHER,
 * sketch.py:153-158): column j of the unscaled +-1 matrix is numpy
 * Philox(key = (seed << 64) | (col0 + j)).integers(0, 2, size=k), reproduced
 * bit for bit (Philox4x64-10, top bit of each 32-bit draw) into row j of an
 * n x ceil(k/32) uint32 array (bit r % 32 of word r / 32 set = +1). */
int sgs_rademacher_bits(uint64_t seed, int64_t col0, int64_t n, int k, uint32_t* bits,
                        void* stream);
/* Partials of Theta^T' X from the packed signs: the sgs_dense_partials
 * chunking (sgs_dense_nparts(n) parts) and per-output chains, so bit-identical
 * to it on the materialised matrix. */
int sgs_rademacher_partials(const uint32_t* bits, int k, const void* X, int x_dtype,
                            int64_t ldx, int ncols, int64_t n, double* partials,
                            const sgs_status* st, void* stream);

/* ---- Matrix Market ingest (io.read_matrix_market, io.py:24-70) -----------
 * Host-side, native: real/integer/double coordinate files, general or
 * symmetric storage, square; SGS_EINVAL with the reference's message in
 * sgs_last_error() otherwise (the Python layer raises MatrixMarketError).
 * Entries come back 0-based in file order (CSR assembly, duplicate summing and
 * the symmetric mirror are SparseMatrix.from_coo's). */
int sgs_mm_read_header(const char* path, int64_t* nrows, int64_t* ncols, int64_t* nnz,
                       int* symmetric);
int sgs_mm_read_entries(const char* path, int64_t nnz, int64_t* rows, int64_t* cols,
                        double* vals);

/* Y[:, c] = cast(scale * sum_p partials[c][p][:]) in fixed p order. */
int sgs_partials_reduce(const double* partials, int nparts, int k, int ncols,
                        double scale, void* Y, int y_dtype, int64_t ldy,
                        const sgs_status* st, void* stream);

/* as sgs_partials_reduce, then divided by den[0]: the certification sketch
 * S_phi[:, i] = (Phi q'_i) / r_ii of gram_schmidt.py:333-335 */
int sgs_partials_reduce_div(const double* partials, int nparts, int k, int ncols,
                            double scale, const double* den, void* Y, int y_dtype,
                            int64_t ldy, const sgs_status* st, void* stream);

/* Unnormalised Sylvester FWHT along axis 0 of a power-of-two length vector,
 * batched over columns (sketch.py:90-109). */
int sgs_fwht(double* X, int64_t s, int ncols, int64_t ldx, void* stream);

/* ---- RGS column step -----------------------------------------------------
 * Step 3 of RgsState.push (gram_schmidt.py:316-319):
 *   Q[:, i] = cast_crs(w) - Q[:, :i] @ r_crs        (coarse arithmetic)
 * When normalize_prev != 0 column i-1 holds the unnormalised q'_{i-1} and is
 * first normalised in place, Q[:, i-1] = cast_crs(q'_{i-1} / R[i-1, i-1])
 * (step 7, gram_schmidt.py:329), inside the same pass.  i == 0 stores
 * cast_crs(w) (gram_schmidt.py:307-310). */
int sgs_rgs_update(void* Q, int q_dtype, int64_t ldq, int64_t n, int i,
                   const void* w, int w_dtype, const void* r_crs,
                   int normalize_prev, const double* R, int64_t ldr,
                   const sgs_status* st, void* stream);

/* Fused column kernel: sgs_rgs_update plus, when do_sketch != 0, the P-SRHT /
 * block-SRHT sketch of the new column (step 4, gram_schmidt.py:320) in the
 * epilogue, without re-reading q'.  One CTA per 4096-row tile (requires
 * log2_block >= 12 and row0 % 4096 == 0), Q streamed through a TMA bulk-copy
 * ring; partials as sgs_srht_partials, one k-vector per 4-CTA cluster (4 tiles),
 * sgs_column_nparts(n_local) of them.  w_div != NULL (device scalar): the
 * column is cast(w / w_div[0]) - the lagged w_{i} = A q'_{i-1} / r_{i-1,i-1}
 * of the one-synchronisation Arnoldi. */
int sgs_column_nparts(int64_t n_local);
int sgs_rgs_update_srht(void* Q, int q_dtype, int64_t ldq, int64_t n, int i,
                        const void* w, int w_dtype, const double* w_div /* nullable */,
                        const void* r_crs, int normalize_prev, const double* R, int64_t ldr,
                        int do_sketch, int64_t row0, int log2_block,
                        const uint32_t* sign_bits, const int32_t* samples, int k,
                        double* partials, const sgs_status* st, void* stream);
/* sgs_rgs_update_srht with the certification sketch Phi of q' in the same
 * epilogue (reference RgsState.push, gram_schmidt.py:333-335: S_phi gets
 * Phi q'_i / r_ii).  Phi must be a P-SRHT / block-SRHT with log2 block >= 12
 * (4096-row tiles); phi_partials receives sgs_column_nparts(n) kphi-vectors,
 * bit-identical to sgs_srht_partials of Q[:, i] with Phi.  do_sketch must be
 * set.  phi_partials == NULL is sgs_rgs_update_srht. */
int sgs_rgs_update_srht_phi(void* Q, int q_dtype, int64_t ldq, int64_t n, int i,
                            const void* w, int w_dtype, const double* w_div /* nullable */,
                            const void* r_crs, int normalize_prev, const double* R, int64_t ldr,
                            int do_sketch, int64_t row0, int log2_block,
                            const uint32_t* sign_bits, const int32_t* samples, int k,
                            double* partials, const uint32_t* phi_sign_bits,
                            const int32_t* phi_samples, int kphi, int phi_log2_block,
                            double* phi_partials, const sgs_status* st, void* stream);

/* Fused column kernel for dense sketches: sgs_rgs_update over the row chunks
 * of sgs_dense_partials, q' kept in shared memory, then (do_sketch != 0) the
 * Theta^T GEMV of the chunk - bit-identical partials to sgs_dense_partials. */
int sgs_rgs_update_dense(void* Q, int q_dtype, int64_t ldq, int64_t n, int i,
                         const void* w, int w_dtype, const void* r_crs,
                         int normalize_prev, const double* R, int64_t ldr,
                         int do_sketch, const double* thetaT, int64_t ldt, int k,
                         double* partials, const sgs_status* st, void* stream);
/* The same fused column step for the device-generated Rademacher sketch
 * (SketchKind.RADEMACHER, sketch.py:153-166): q'_i = w - Q r streamed once,
 * then Theta q' from the packed signs of sgs_rademacher_bits (1 bit per entry,
 * n x ceil(k/32) words) - no second read of q', no fp64 Theta stream.  The
 * chunking and partial count are sgs_dense_column_nparts(n, k). */
int sgs_rgs_update_rademacher(void* Q, int q_dtype, int64_t ldq, int64_t n, int i,
                              const void* w, int w_dtype, const void* r_crs,
                              int normalize_prev, const double* R, int64_t ldr,
                              int do_sketch, const uint32_t* rbits, int k,
                              double* partials, const sgs_status* st, void* stream);

/* Q[:, col] = cast_crs(Q[:, col] / R[col, col])   (gram_schmidt.py:329) */
int sgs_normalize_column(void* Q, int q_dtype, int64_t ldq, int64_t n,
                         int col, const double* R, int64_t ldr,
                         const sgs_status* st, void* stream);

/* z = A_crs[:, :ncols] @ y in fp64 (A upcast), optionally z *= scale_num/scale_den[0]
 * (krylov.py:308-310: z = Q[:, :k].astype(f64) @ y; x = (b_norm/alpha) z). */
int sgs_gemv_f64(const void* A, int a_dtype, int64_t lda, int64_t n, int ncols,
                 const double* y, double* z, void* stream);

/* ---- sketched least squares (steps 2, 5, 6 and the LS append) ------------
 * One launch of a thread-block cluster that replicates the k-dimensional
 * work of RgsState.push (gram_schmidt.py:303-337) on device:
 *   finalize: s' = scale*sum(partials) (or P[:,0] for column 0), r_ii = ||s'||,
 *             breakdown guard, S[:, i] = s'/r_ii, R[i,i] = r_ii, and append
 *             s_i to an incrementally maintained QR of S (orthonormal factor
 *             Qs, explicit inverse Rinv of R_S), which replaces
 *             _IncrementalHouseholderQR.append (gram_schmidt.py:148-171).
 *   solve:    r = argmin ||S[:, :i] r - p|| = Rinv Qs^T p with the reference's
 *             rank check (gram_schmidt.py:180-190); writes R[:i, col] and the
 *             coarse copy r_crs used by sgs_rgs_update.
 * Fine dtype is fp64 (UNIFIED64, MIXED32_64) or fp32 (UNIFIED32). */
typedef struct sgs_ls_args {
  int k;                 /* sketch rows */
  int cap;               /* allocated columns of S/P/Qs/Rinv/R */
  int fine_dtype;        /* SGS_F32 / SGS_F64 */
  int coarse_dtype;      /* dtype of r_crs */
  int do_finalize;       /* finalize + append column `col_fin` */
  int col_fin;
  const double* s_partials; int s_nparts; double s_scale;
  int do_solve;          /* solve for column `col_sol` (uses col_sol columns) */
  int col_sol;
  const double* p_partials; int p_nparts; double p_scale; /* NULL: P[:,col_sol] is already stored */
  double bf_ucrs;        /* breakdown_factor * u_crs */
  void* S; void* P;      /* k x cap, fine, ld = k */
  double* R;             /* cap x cap, ld = cap */
  void* Qs; void* Rinv;  /* k x cap and cap x cap, fine: unnormalised orthogonal
                            factor T of S and R_S^{-1} */
  void* alpha;           /* cap, fine: column norms of T (Qs = T diag(1/alpha)) */
  double* scratch;       /* sgs_ls_scratch_elems(k, cap) doubles */
  void* r_crs;           /* cap, coarse */
  sgs_status* st;
  long long* trace;      /* optional (NULL): clock64() at phase boundaries, CTA 0 */
  int cache_cols;        /* set by the library: columns of T cached in shared memory */
  unsigned long long* timeline;  /* set by the library (debug timeline) */
  int* t_pend;           /* optional (NULL: off), 2 ints, -1 = none: [0] column of T whose formation
                            is deferred, [1] last column finalized without forming t */
  void* t_coef;          /* cap, fine: its projection coefficients (with t_pend).  A finalize
                            that sees no cancellation (||t||^2 >= ||s||^2/2 by Pythagoras)
                            publishes r without forming t = s - T c; the next launch forms
                            T[:, t_pend] before its dependency wait, overlapping the column
                            kernel.  Bit-identical T; alpha from the Pythagorean norm. */
  int p_lag;             /* finalize + solve with p_partials: they hold p' = Theta A q'_fin of the
                            one-synchronisation Arnoldi, p = p' / r_fin,fin
                            (stored to P[:, col_sol]); the solve runs after the one exchange */
  int giv_on;            /* with do_finalize, col_fin >= 1: also the progressive Givens update of
                            GMRES step col_fin - 1 (as sgs_givens_step, same arithmetic) */
  double* giv_cs; double* giv_sn; double* giv_g; double* giv_T; long long giv_ldt;
  double* giv_hist; double giv_tol;  /* giv_tol < 0: no stop test */
  const void* peer;      /* optional (NULL: off): device sgs_peer_desc (sgs_peer_desc_create) of a
                            row-sharded state.  The finalize then sums s' across the ranks itself:
                            each CTA reduces its rows of the local partials (s_partials), stores
                            them into every rank's receive slots over NVLink, flags them, waits
                            for every rank's flags and adds the ranks' rows in rank order - the
                            k-vector all-reduce of sgs_partials_reduce + NCCL done inside the LS
                            launch (fp64 fine dtype) */
} sgs_ls_args;

int64_t sgs_ls_scratch_elems(int k, int cap);

/* ---- peer memory of a row-sharded state (one node, NVLink / NVSwitch) --------
 * Replaces the per-column NCCL all-reduce of s' (the paper's distributed RGS,
 * PAPER.md:255-261, absent from the reference) by stores into the peers'
 * memory from the LS launch.  sgs_peer_alloc allocates this rank's exchange
 * area (receive slots + flags, zeroed; size sgs_peer_bytes), sgs_peer_export /
 * sgs_peer_import trade CUDA IPC handles (64 bytes) between the ranks (the
 * caller moves them, e.g. all_gather_object), sgs_peer_desc_create builds the
 * device descriptor the LS reads (area[q] = rank q's area as mapped here; the
 * own area for q == rank).  sgs_peer_begin(desc) opens a factorisation
 * (a new flag generation; enqueue it on every rank).  world <= 8. */
int64_t sgs_peer_bytes(int world, int k, int cl);
int sgs_peer_alloc(int64_t bytes, void** area);
int sgs_peer_free(void* area);
int sgs_peer_export(void* area, unsigned char* handle64);
int sgs_peer_import(const unsigned char* handle64, void** area);
int sgs_peer_unimport(void* area);
int sgs_peer_desc_create(int world, int rank, int k, void* const* areas, void** desc);
int sgs_peer_desc_free(void* desc);
int sgs_peer_begin(void* desc, void* stream);
int sgs_ls_cluster_size(int k);
int sgs_ls_step(const sgs_ls_args* a, void* stream);

/* ---- Krylov ---------------------------------------------------------------
 * SparseMatrix.matvec (krylov.py:81-83) fused with the 1/alpha scaling of
 * gmres (krylov.py:276): y = (A x) / alpha[0] (alpha == NULL: no scaling).
 * x is fp64 or a coarse column of Q; xdiv != NULL forms x = cast(q / xdiv[0])
 * on the fly (the basis column before its deferred normalisation).  CSR with
 * int32 indices, fp64 values. */
int sgs_csr_spmv(int64_t n, const int32_t* row_ptr, const int32_t* col_idx,
                 const double* vals, const void* x, int x_dtype, const double* xdiv,
                 const double* alpha, double* y, const sgs_status* st,
                 void* stream);

/* The Arnoldi step's w = A v (krylov.py:81-83, 276) and its sketch Theta w
 * (gram_schmidt.py:297, sketch.py:90-109) in one launch, for an SRHT on
 * 4096-row tiles (P-SRHT or block-SRHT, log2_block >= 12, k <= 2048): y as
 * sgs_csr_spmv, and the partials of Theta y exactly as sgs_srht_partials
 * writes them for one column of n rows (same bits; sgs_srht_nparts(n,
 * log2_block) partials of k).  row0: global row of local row 0 (tile
 * aligned); sign_bits: the sign words of the local rows.  Scratch: tilevec
 * (sgs_spmv_srht_tilevec_elems doubles) and counters
 * (sgs_spmv_srht_counter_elems u64, zero before the first call, never reset
 * after; one stream at a time). */
int sgs_csr_spmv_srht(int64_t n, const int32_t* row_ptr, const int32_t* col_idx,
                      const double* vals, const void* x, int x_dtype, const double* xdiv,
                      const double* alpha, double* y, int64_t row0, int log2_block,
                      const uint32_t* sign_bits, const int32_t* samples, int k,
                      double* tilevec, unsigned long long* counters, double* partials,
                      const sgs_status* st, void* stream);
int64_t sgs_spmv_srht_tilevec_elems(int64_t n, int k);
int64_t sgs_spmv_srht_counter_elems(int64_t n);

/* deterministic ||x||_2 (fp64 or fp32 input, fp64 result on device) */
int sgs_norm2(const void* x, int x_dtype, int64_t n, double* out, double* work,
              void* stream);
int64_t sgs_norm2_work_elems(int64_t n);
/* divide != 0: y = x / den[0];  else y = x * (num / den[0]) (den == NULL: x * num).
 * fp64; mirrors `v / nw` (krylov.py:224) and `(b_norm / alpha) * z` (krylov.py:309). */
int sgs_scale(const double* x, double num, const double* den, int divide, double* y,
              int64_t n, void* stream);
/* y = b - y (fp64), in place (residual r = b - A x of the restart wrapper) */
int sgs_rsub(const double* b, double* y, int64_t n, void* stream);
/* dst = cast(src / den[0]) (den == NULL: plain cast); e.g. push(b / b_norm) */
int sgs_cast_div(const void* src, int src_dtype, void* dst, int dst_dtype,
                 const double* den, int64_t n, void* stream);
/* v[r] = cos(r + 1): start vector of _operator_norm_estimate (krylov.py:218) */
int sgs_cos_init(double* v, int64_t n, void* stream);
/* The same start vector's entries [first, first + n) (a rank's row block). */
int sgs_cos_init_at(double* v, int64_t n, int64_t first, void* stream);

/* Power-iteration step of _operator_norm_estimate (krylov.py:213-226):
 * given w = A v and ||w|| in nrm[0], sets v = w / ||w|| and sigma[0] = ||w||;
 * a zero norm freezes sigma at -1 (the reference returns 0.0). */
int sgs_power_step(const double* w, const double* nrm, double* v,
                   double* sigma, int64_t n, void* stream);

/* Progressive Givens step of gmres (krylov.py:282-301) on device:
 * hcol = R[:i+2, i+1] rotated by the previous i rotations (cs/sn), new
 * rotation, T[:i+2, i] = hcol, g update, est = |g[i+1]|/beta appended to
 * hist[i]; sets st->code = SGS_ST_CONVERGED when tol > 0 and est <= tol and
 * advances st->iters. */
int sgs_givens_step(const double* R, int64_t ldr, int i, double* cs,
                    double* sn, double* g, double* T, int64_t ldt,
                    double* hist, double tol, sgs_status* st, void* stream);

/* Head of one RGMRES step (fused engine): normalise basis column `col` of Q
 * in place, q = cast(q' / R[col][col]) as RgsState.push step 7
 * (gram_schmidt.py:330-332), with all blocks but one, and - when gi >= 0 -
 * the progressive Givens update of step gi (as sgs_givens_step) with the
 * remaining block, concurrently.  The normalisation does not consult st (the
 * Givens update may set CONVERGED meanwhile); *norm_flag = col records it.
 * col < 0: Givens only. */
int sgs_arnoldi_head(void* Q, int q_dtype, int64_t ldq, int64_t n, int col, const double* R,
                     int64_t ldr, int* norm_flag, int gi, double* cs, double* sn, double* g,
                     double* T, int64_t ldt, double* hist, double tol, sgs_status* st,
                     void* stream);

/* Column-major transpose for staging host row-major inputs:
 * dst[c*ldd + r] = src[r*lds + c], r < rows, c < cols. */
int sgs_transpose(const void* src, int64_t lds, void* dst, int64_t ldd,
                  int64_t rows, int64_t cols, int dtype, void* stream);

/* ---- ILU(0) right preconditioning (krylov.py:86-151) ----------------------
 * Level-scheduled, sync-free row kernels: sgs_ilu0_analyse gives every row
 * its dependency level in the lower and the upper triangle and sorts the
 * rows by level; the factorization and the sweeps hand rows out in that
 * order through a ticket counter and wait on their dependencies row by row
 * (no per-level launches).  `ctl` (zeroed once by the caller) is owned by one
 * preconditioner and reused by its launches, which advance it themselves, so
 * they need no host bookkeeping and can be captured in a CUDA graph. */
typedef struct sgs_ilu_ctl {
  uint64_t ticket;   /* next row block to hand out */
  uint32_t done;     /* finished blocks of the running launch */
  uint32_t epoch;    /* launches completed (factor flags: row i ready when == epoch+1) */
} sgs_ilu_ctl;

/* int32 elements of the `work` buffer sgs_ilu0_analyse needs. */
int64_t sgs_ilu0_analysis_work_elems(int64_t n);

/* perm_lower / perm_upper (n int32 each) = rows ordered by level in the
 * lower (j < i) / upper (j > i) dependency graph of the pattern (rp, ci). */
int sgs_ilu0_analyse(int64_t n, const int32_t* rp, const int32_t* ci, int32_t* perm_lower,
                     int32_t* perm_upper, int32_t* work, sgs_ilu_ctl* ctl, void* stream);

/* ILU(0) of the CSR matrix (rp, ci, vals) into F (nnz doubles, same pattern):
 * row-oriented IKJ elimination (krylov.py:103-151), bit-identical to the
 * reference's sequential loop (no FMA contraction).  aux[0] = first row with a
 * structural zero diagonal (n if none; reference raises ValueError), aux[1] =
 * 2*i (+1) for the first row i at which the reference raises
 * ZeroDivisionError: +1 = row i's own pivot, +0 = row 0's pivot used by row i
 * (UINT64_MAX if none).  diag_pos: n int32 out; flags: n uint32, zeroed once. */
int sgs_ilu0_factor(int64_t n, const int32_t* rp, const int32_t* ci, const double* vals,
                    double* F, int32_t* diag_pos, const int32_t* perm_lower, uint32_t* flags,
                    sgs_ilu_ctl* ctl, uint64_t* aux, double pivot_tol, void* stream);

/* Arms a sweep buffer (fills it with the "not yet written" sentinel).  The
 * `tmp` of sgs_ilu0_solve must be armed once before its first solve; each
 * solve leaves it armed again. */
int sgs_ilu0_pending_fill(double* v, int64_t n, void* stream);

/* out = U^{-1} L^{-1} x (Ilu0Preconditioner.solve, krylov.py:95-99): forward
 * sweep with the unit lower part of F into tmp, then backward sweep with the
 * upper part into out.  x is binary32 or binary64; when xdiv is non-null the
 * input is cast(x / *xdiv) to x's dtype first (the normalised Arnoldi vector,
 * as sgs_csr_spmv).  x, tmp and out must be distinct.  Returns at once when
 * st->code is set. */
int sgs_ilu0_solve(int64_t n, const int32_t* rp, const int32_t* ci, const double* F,
                   const int32_t* perm_lower, const int32_t* perm_upper, const void* x,
                   int x_dtype, const double* xdiv, double* tmp, double* out, sgs_ilu_ctl* ctl,
                   const sgs_status* st, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SKETCHGS_B200_H */
