/*
 * bilu.h -- C-ABI of the B200-native numeric phase of the Crout-type block ILU
 * (BILU) of Bollhoefer, Schenk, Verbosio, "High Performance Block Incomplete LU
 * Factorization", arXiv:1908.10169.
 *
 * What the library computes:
 *   Given a sparse A, a symmetric permutation perm and a partition of the
 *   permuted matrix Ã = A(perm, perm) into contiguous diagonal blocks, compute
 *       Ã ≈ L · D^{-1} · U        ("Technically we compute A ≈ L D^{-1} U",
 *                                    PAPER.md:772-773)
 *   with L unit block-lower, U unit block-upper, D block diagonal holding the
 *   explicit inverses of the pivot blocks, by the Crout
 *   recurrence of Alg. 1 generalised to blocks: a row i of
 *   block column K of L is dropped iff max_t |(l_iK l_KK^{-1})_t| <= tau, a column
 *   j of block row K of U iff max_t |(u_KK^{-1} u_Kj)_t| <= tau (
 *   max-abs norm: DESIGN.md reading R1).  Consecutive blocks are merged
 *   ("progressive aggregation", Sec. 3.5) when
 *   nu <= 1.2 mu or nu <= mu + 2(p+q), and p+q <= max_block.
 *
 * Storage of the factors (hybrid layout of Fig. 1),
 * per final block K with rows/cols [s_K, e_K), b_K = e_K - s_K:
 *   L : sorted kept row indices i >= e_K and one dense m_K x b_K panel, row-major
 *   Ũ : sorted kept column indices j >= e_K and one dense b_K x c_K panel,
 *       column-major, holding the UNSCALED rows Ũ = D^{-1} U (so U = D_K Ũ)
 *   D : D_K = P_K^{-1}, b_K x b_K column-major (P_K = the pivot block)
 *
 * Ownership and errors:
 *   - Every input pointer is BORROWED for the duration of the call only.
 *   - The context owns all device memory (factors, arenas, workspaces).
 *   - No function aborts or throws across the ABI; each returns a status.  On
 *     failure bilu_last_error(ctx) (or bilu_last_error(NULL) for failures
 *     before a context exists) holds a one-line reason.
 *   - All entry points are synchronous with respect to the host unless noted.
 */
#ifndef BILU_H
#define BILU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BILU_OK = 0,
  BILU_ERR_ARG = 1,        /* NULL pointer, n < 1, unsorted/duplicate CSR,
                              perm not a bijection, sum(block_sizes) != n,
                              a block size < 1 or > max_block                   */
  BILU_ERR_BREAKDOWN = 2,  /* exactly singular pivot block P_K (stats->breakdown_block) */
  BILU_ERR_OOM = 3,        /* device allocation failed                          */
  BILU_ERR_CUDA = 4,       /* CUDA runtime error                                */
  BILU_ERR_NCCL = 5,       /* reserved for the multi-GPU path                   */
  BILU_ERR_STATE = 6,      /* e.g. bilu_apply / bilu_export before bilu_factor  */
  BILU_ERR_NOT_BUILT = 7   /* library compiled without a usable device          */
} bilu_status;

typedef struct bilu_ctx bilu_ctx;   /* opaque; owns all device state */

typedef struct {
  int32_t device;        /* CUDA device ordinal                                  */
  int32_t max_block;     /* cap on merged block size, and on initial blocks (<=128; R9) */
  int32_t aggregate;     /* 1 = progressive aggregation (Sec. 3.5), 0 = off      */
  int32_t n_ctas;        /* persistent CTAs of the factor kernel (0 = auto)      */
  double  near_rel;      /* decisions with |max/tau - 1| <= near_rel are logged  */
  int64_t arena_hint;    /* initial factor arena, doubles (0 = auto); grows on overflow */
  void   *stream;        /* cudaStream_t to run on (NULL = the legacy default stream) */
  int32_t rank, world;   /* reserved (multi-GPU runs through bilu_dist_setup; world = 1) */
  void   *nccl_comm;     /* reserved                                             */
  /* Sec. 3.6 perturbation of singular / ill-conditioned pivot blocks (PAPER.md:1505-1538,
   * DESIGN.md R19): off by default (an exactly singular pivot block is then a breakdown).
   * When on, a pivot block with a zero column / row, an exactly zero pivot or a 1-norm
   * condition number |P|_1 |P^{-1}|_1 > cond_max is perturbed with the absolute / relative
   * tolerances perturb_tau (x max|a_ij|) and perturb_rho. */
  int32_t perturb;       /* 0 = off (default), 1 = on                            */
  double  perturb_tau;   /* default 1e-2 (the paper's practice)                   */
  double  perturb_rho;   /* default 1e-1                                          */
  double  cond_max;      /* default 1e12                                          */
  /* Dense trailing zone: the longest suffix of blocks, all at most 8 wide,
   * whose dense panel buffers (2 x 64 B x blocks x unknowns of the suffix) fit this many
   * bytes keeps its block columns / rows in those buffers; its contributors push their
   * Schur updates there when they finish (same products, another summation order), so a
   * ready block of the suffix (the top separators of a nested dissection) reads only its
   * own panel.  0 = default budget (min(24 GiB, 1/4 of free memory)), < 0 = off.  Ignored
   * by the distributed factorization. */
  int64_t zone_bytes;
} bilu_options;

/* Fills *opt with the defaults (device 0, max_block 128, aggregate 1, near_rel
 * 1e-8, auto sizes, default stream, world 1, perturbation off with tau 1e-2, rho 1e-1,
 * cond_max 1e12). */
void bilu_options_default(bilu_options *opt);

typedef struct {
  double  flops;          /* algorithmic flops of the executed structure */
  double  bytes_min;      /* compulsory bytes: read Ã once, write L, Ũ, D + indices once */
  double  t_factor_ms;    /* device time of the numeric phase (CUDA events)      */
  double  t_merge_ms;     /* of which: progressive aggregation post-pass         */
  int64_t nnz_L, nnz_U, nnz_D;   /* stored doubles of the final factors          */
  int32_t n_blocks_init, n_blocks_final, n_merges;
  int32_t breakdown_block;       /* original block id of a singular pivot, or -1 */
  int32_t n_retries;             /* workspace regrow-and-retry rounds             */
  int32_t n_kernel_launches;     /* kernels launched by the last bilu_factor      */
  int64_t n_decisions;           /* drop/keep decisions taken                     */
  int64_t n_near;                /* of which |max/tau - 1| <= near_rel            */
  double  min_margin;            /* min |max/tau - 1| over all decisions (tau>0)  */
  int64_t n_perturbed;           /* pivot blocks modified by the Sec. 3.6 perturbation */
  int32_t zone_blocks;           /* blocks of the dense trailing zone */
  int32_t zone_unknowns;         /* ... and their unknowns                        */
} bilu_factor_stats;

/*
 * bilu_analyze -- symbolic phase (host preprocessing + device upload).
 *   n            order of A (>= 1)
 *   row_ptr      HOST, int64[n+1], CSR row offsets of A (0-based, row_ptr[0]=0)
 *   col_idx      HOST, int32[nnz], strictly increasing within each row
 *   val          HOST, double[nnz], values of A (may be NULL: set later with
 *                bilu_set_values before bilu_factor)
 *   perm         HOST, int32[n] or NULL (identity): Ã(i,j) = A(perm[i], perm[j])
 *                (the caller's fill-reducing ordering)
 *   block_sizes  HOST, int32[n_blocks], initial partition of Ã, sum = n,
 *                each in [1, max_block] (the caller's initial blocking,
 *                PAPER.md:923-965, 1171-1242)
 *   opt          options or NULL (defaults)
 *   out          receives the context (set to NULL on failure)
 * Builds Ã in CSR and CSC on the device, the block adjacency graph and the
 * initial dependency counts of the dataflow schedule.
 */
bilu_status bilu_analyze(int32_t n, const int64_t *row_ptr, const int32_t *col_idx,
                         const double *val, const int32_t *perm,
                         const int32_t *block_sizes, int32_t n_blocks,
                         const bilu_options *opt, bilu_ctx **out);

/*
 * bilu_set_values -- replace the values of A (same pattern as at analyze time).
 *   val          double[nnz] in A's original CSR order; HOST memory if
 *                on_device == 0, DEVICE memory (same device) if on_device != 0.
 *                Host memory should be pinned for an asynchronous copy.
 */
bilu_status bilu_set_values(bilu_ctx *h, const double *val, int32_t on_device);

/*
 * bilu_factor -- numeric phase: Crout block ILU with tau-dropping and, if
 * enabled, progressive aggregation (PAPER.md:158-175, 205-228, 767-799,
 * 1405-1453).  May be called again (new tau or new values); each call rebuilds
 * the factors from scratch.
 *   tau   drop tolerance >= 0 (0 keeps every row/column that is not exactly 0)
 *   st    optional statistics (may be NULL)
 * Returns BILU_ERR_BREAKDOWN (st->breakdown_block set) if a pivot block is
 * exactly singular (or, with opt.perturb, still singular / ill-conditioned after the
 * Sec. 3.6 perturbation).
 */
bilu_status bilu_factor(bilu_ctx *h, double tau, bilu_factor_stats *st);

/*
 * bilu_apply -- y = M^{-1} x with M = Pᵀ-permuted L D^{-1} U, i.e. solves
 * A y ≈ x through the factors of Ã (forward substitution with L, multiply by
 * the D blocks, backward substitution with U).
 *   x, y   DEVICE double[n] in A's ORIGINAL ordering; may not alias.
 *   stream cudaStream_t or NULL (context stream).  Asynchronous on that stream.
 */
bilu_status bilu_apply(bilu_ctx *h, const double *x, double *y, void *stream);

/*
 * bilu_export -- HOST copy of the final factors in the hybrid layout of Fig. 1
 * (PAPER.md:220-228): per final block the sorted kept L rows + dense panel, the
 * sorted kept U columns + dense panel of Ũ (U = D_K Ũ), and D_K; plus the log of
 * near-threshold drop decisions (|max/tau - 1| <= near_rel) for decision replay.
 * All arrays are malloc'd by the library and owned by the view; release them
 * with bilu_factor_view_free.  BILU_ERR_STATE before a successful bilu_factor.
 */
typedef struct {
  int32_t n, n_blocks;
  int32_t *bstart;          /* n_blocks+1 */
  int64_t *Lp;  int32_t *Li;  int64_t *Lvp; double *Lv;   /* rows, m x b row-major */
  int64_t *Up;  int32_t *Ui;  int64_t *Uvp; double *Uv;   /* cols, b x c col-major */
  int64_t *Dp;  double *Dv;                               /* b x b col-major */
  int64_t n_near;           /* near-threshold decisions logged (<= cap)      */
  int32_t *near_blk, *near_side, *near_idx, *near_keep;   /* original block id, 0=L row 1=U col */
  double *near_margin;
} bilu_factor_view;

bilu_status bilu_export(bilu_ctx *h, bilu_factor_view *v);
void bilu_factor_view_free(bilu_factor_view *v);

/* ---- preconditioned Krylov solve ----
 * bilu_gmres -- solves A x = b with restarted, right-preconditioned GMRES(m) on the device,
 * M = the factors of the last bilu_factor ("restarted GMRES ... restart length 30 ... b
 * with all ones"; R16: x0 = 0, modified Gram-Schmidt, Givens
 * rotations, inner steps counted, convergence on the true residual |b - A x| / |b| <= tol
 * checked at the end of every cycle).
 *   b, x   DEVICE double[n], A's ORIGINAL ordering; x is overwritten; may not alias.
 *   m      restart length (1..1000); tol > 0; max_restarts >= 1
 * The workspace ((2m+2) n doubles) is owned by the context.  Synchronous. */
typedef struct {
  int32_t iterations;        /* inner (Arnoldi) steps                                  */
  int32_t restarts;          /* cycles started                                         */
  int32_t converged;         /* 1 if |b - A x| / |b| <= tol                            */
  double  rel_residual;      /* final true relative residual                           */
  double  t_solve_ms;        /* device time (CUDA events on the context stream)        */
  int64_t n_kernel_launches;
} bilu_solve_stats;

bilu_status bilu_gmres(bilu_ctx *h, const double *b, double *x, int32_t m, double tol, int32_t max_restarts,
                       bilu_solve_stats *st);

/* ---- multi-GPU factorization over nested-dissection subtrees ----
 * One context per rank (one process per GPU), every rank with the same global matrix,
 * ordering and partition.  Sequence, on every rank:
 *   bilu_dist_setup(ctx, owner, rank)          once, before the first factorization
 *   bilu_factor_local(ctx, tau, &st)           phase A: this rank's subtree blocks
 *   bilu_interface_pack(ctx, NULL, 0, &bytes)  size of this rank's packed interface panels
 *   bilu_interface_pack(ctx, buf, bytes, &bytes)  ... packed into the caller's device buffer
 *   -- the caller exchanges the packed buffers (all-gather of variable-size device
 *      buffers, e.g. NCCL broadcasts from every rank) --
 *   bilu_interface_unpack(ctx, buf_r, bytes_r) for every other rank r
 *   bilu_factor_separators(ctx, &st)           phase B: the separator blocks (replicated)
 * Inside an ND subtree every contributor of a block is a block of the same subtree, so
 * phase A needs no communication; the separator blocks' Schur updates need the kept L rows
 * and Ũ columns of the subtree blocks that lie in separator rows / columns ("interface"
 * panels), which is what the ranks exchange.  Aggregation (Sec. 3.5)
 * does not cross the ownership boundaries (R18).  The final factors are
 * distributed: each rank holds its own subtree blocks and all separator blocks; bilu_export
 * reports the other ranks' blocks as empty (L, Ũ with no rows / columns) and bilu_apply
 * returns BILU_ERR_STATE.
 *
 * bilu_dist_setup -- owner: HOST int32[n_blocks]: rank owning each initial block (its ND
 *   subtree), or -1 for separator blocks (factored by every rank).  Returns BILU_ERR_ARG if
 *   blocks of different ranks are coupled in Ã or a subtree block follows a separator block
 *   it is coupled to (not a nested-dissection partition), BILU_ERR_STATE after a
 *   factorization.
 * bilu_factor_local -- phase A (same arithmetic as bilu_factor on this rank's blocks).
 * bilu_interface_pack -- dst: DEVICE buffer of `capacity` bytes owned by the caller (16-byte
 *   aligned); *bytes receives the packed size.  With dst == NULL or capacity < the size it
 *   only reports the size.  Format: int64 header {magic, count, bytes, rank}, `count` table
 *   entries {J, b, m, c, byte offsets of the row list, L panel, column list, Ũ panel}, then
 *   the payload.
 * bilu_interface_unpack -- buf: DEVICE pointer (same device) to another rank's packed
 *   buffer of `bytes` bytes, borrowed for the call.  BILU_ERR_ARG for a malformed buffer,
 *   one of this rank, or blocks that are not remote subtree blocks.
 * bilu_factor_separators -- phase B and the aggregation post-pass; st covers both phases
 *   (flops, device time; the caller times the exchange).
 */
bilu_status bilu_dist_setup(bilu_ctx *h, const int32_t *owner, int32_t rank);
bilu_status bilu_factor_local(bilu_ctx *h, double tau, bilu_factor_stats *st);
bilu_status bilu_interface_pack(bilu_ctx *h, void *dst, int64_t capacity, int64_t *bytes);
bilu_status bilu_interface_unpack(bilu_ctx *h, const void *buf, int64_t bytes);
bilu_status bilu_factor_separators(bilu_ctx *h, bilu_factor_stats *st);

/*
 * Distributed preconditioner application y = (L D^{-1} U)^{-1} x over the ranks' factors
 * (after bilu_factor_separators).  The forward sweep L w = x splits at
 * the ND separators: a subtree block's L rows lie in its own subtree and in separator rows,
 * a separator block's only in later separators (PAPER.md:164-171 dependency, ND order), so
 *   bilu_apply_dist_begin   forward sweep over this rank's subtree blocks; writes this rank's
 *                           contributions to the separator rows (contrib)
 *   (caller)                contrib_sum = sum of every rank's contrib (one all-reduce)
 *   bilu_apply_dist_end     forward sweep over the separator blocks (replicated), D multiply
 *                           and backward sweep over separator + own subtree blocks; y receives
 *                           this rank's subtree rows, the separator rows if write_separators,
 *                           and 0 elsewhere, so the ranks' y sum to the full result.
 *   x, y        DEVICE, double[n], A's original ordering; x the same on every rank
 *   contrib, contrib_sum   DEVICE, double[m], m from bilu_dist_separator_rows
 * Errors: BILU_ERR_STATE (not a distributed context, not factored, end before begin),
 * BILU_ERR_ARG, BILU_ERR_CUDA.  Asynchronous on stream (NULL = the context's stream).
 */
bilu_status bilu_dist_separator_rows(bilu_ctx *h, int64_t *m);
bilu_status bilu_apply_dist_begin(bilu_ctx *h, const double *x, double *contrib, void *stream);
bilu_status bilu_apply_dist_end(bilu_ctx *h, const double *contrib_sum, double *y, int32_t write_separators,
                                void *stream);

/* Destroys the context and frees all device memory.  NULL-safe. */
void bilu_destroy(bilu_ctx *h);

const char *bilu_status_string(bilu_status s);
/*
 * bilu_ilu1_blocks -- initial block partition by the ILU(1,tau) simulation of Sec. 3.4
 * (readings in DESIGN.md R20), computed on the device.
 *   n, row_ptr, col_idx, val, perm   HOST, as in bilu_analyze (val required); the estimate
 *                works on Ã = A(perm, perm)
 *   tau          drop tolerance of the simulation (>= 0)
 *   max_size     cap on a block (1..128; BASELINE: "initial block size up to 8")
 *   device, stream   CUDA device ordinal and cudaStream_t (NULL = legacy default stream)
 *   block_sizes  HOST, int32[n] (capacity n): receives the partition of Ã, sum = n
 *   n_blocks     receives the number of blocks
 *   n_kernel_launches   optional (may be NULL): kernels launched
 * Column k of L is estimated as I~_k = {i>k : |a_ik| >= tau|a_kk|} u {i>k : exists j<k,
 * |a_ij a_jk| >= tau|a_jj a_kk|} (and row k of U symmetrically); a block grows from k0 while
 * f_{l+1} <= 4/3 c' or f_{l+1} <= c' + 4(l+1).  Result identical to the oracle's.  Synchronous;
 * device memory is allocated and freed inside.  Errors: BILU_ERR_ARG (bad CSR / perm / tau /
 * max_size), BILU_ERR_OOM, BILU_ERR_CUDA, BILU_ERR_NOT_BUILT.
 */
bilu_status bilu_ilu1_blocks(int32_t n, const int64_t *row_ptr, const int32_t *col_idx, const double *val,
                             const int32_t *perm, double tau, int32_t max_size, int32_t device, void *stream,
                             int32_t *block_sizes, int32_t *n_blocks, int32_t *n_kernel_launches);

/*
 * bilu_cosine_blocks -- cosine-based initial blocking of Sec. 3.2 (readings
 * in DESIGN.md R21), computed on the device from the pattern of A.
 *   n, row_ptr, col_idx   HOST CSR of A as in bilu_analyze (values are not used)
 *   tau          similarity threshold in [0,1] (the paper's 0.8)
 *   max_size     cap on a group (1..128)
 *   device, stream   CUDA device ordinal and cudaStream_t (NULL = legacy default stream)
 *   q            HOST, int32[n]: the grouping permutation Q (new -> old), Ã = A(q, q)
 *   block_sizes  HOST, int32[n] (capacity n): group sizes in Q's order, sum = n
 *   n_blocks     receives the number of groups
 *   n_kernel_launches   optional (may be NULL)
 * Rows i, j join when nz(a_i n a_j)^2 >= tau nz(a_i) nz(a_j); rows / columns with more than
 * mu + 2 sigma nonzeros are ignored; groups follow Saad's greedy in row order.  Result identical
 * to the oracle's.  Synchronous; device memory allocated and freed inside.  Errors: BILU_ERR_ARG
 * (bad CSR / tau / max_size), BILU_ERR_OOM, BILU_ERR_CUDA, BILU_ERR_NOT_BUILT.
 */
bilu_status bilu_cosine_blocks(int32_t n, const int64_t *row_ptr, const int32_t *col_idx, double tau, int32_t max_size,
                               int32_t device, void *stream, int32_t *q, int32_t *block_sizes, int32_t *n_blocks,
                               int32_t *n_kernel_launches);

/*
 * bilu_mwm -- Sec. 3.1 preprocessing on the device (reading in DESIGN.md R22):
 * the maximum product transversal of A and its scalings, so that D_l A D_r Pi has unit
 * diagonal and off-diagonal entries of modulus at most 1 (the matching + scaling the paper
 * applies before the reordering; MC64's column-normalised costs
 * c_ij = log(max_k |a_kj|) - log|a_ij| on the stored nonzeros, explicit zeros excluded).
 *   n, row_ptr, col_idx, val   HOST CSR of A as in bilu_analyze (values required)
 *   device, stream   CUDA device ordinal and cudaStream_t (NULL = legacy default stream)
 *   sigma       HOST int32[n]: sigma[i] = column matched to row i (a permutation)
 *   dl, dr      HOST double[n]: row / column scalings, |dl_i a_ij dr_j| <= 1 (+ 1e-10 relative)
 *               and = 1 on the matching
 *   n_kernel_launches   optional (may be NULL)
 * Parallel forward auction with eps-scaling down to 1e-10 (relative cost range) / n: the
 * objective sum_i c_{i,sigma(i)} is optimal up to that margin (the oracle's Hungarian method
 * finds the same transversal when the optimum is unique).  Synchronous; device memory
 * allocated and freed inside.  Errors: BILU_ERR_ARG (bad CSR, or no perfect matching: an empty
 * row / column or a structurally singular pattern), BILU_ERR_OOM, BILU_ERR_CUDA,
 * BILU_ERR_NOT_BUILT.
 */
bilu_status bilu_mwm(int32_t n, const int64_t *row_ptr, const int32_t *col_idx, const double *val, int32_t device,
                     void *stream, int32_t *sigma, double *dl, double *dr, int32_t *n_kernel_launches);

const char *bilu_last_error(const bilu_ctx *h);

/* Number of kernels the library launched since the context was created
 * (evidence counter for benchmarks). */
int64_t bilu_kernel_launches(const bilu_ctx *h);

/* ---- diagnostics (tests and microbenchmarks; not needed by users) ----
 * bilu_diag_dgemm -- the library's CTA-level FP64 tensor-core GEMM (DMMA
 * m8n8k4, used for the Schur-update products PAPER.md:371-374 and the merged
 * panels PAPER.md:1348-1387) on its own: for b = 0..batch-1 (one CTA each)
 *     C_b = alpha * A_b * B_b + beta * C_b,   A_b = A + b*sa (M x K), B_b = B + b*sb
 *     (K x N), C_b = C + b*sc (M x N); element (i, j) of X at X[i*xrs + j*xcs].
 * All pointers DEVICE memory; asynchronous on `stream` (NULL = default stream).
 * Returns 0, 1 (bad argument) or 4 (launch error). */
int bilu_diag_dgemm(int M, int N, int K, double alpha, const double *A, int64_t ars, int64_t acs,
                    const double *B, int64_t brs, int64_t bcs, double beta, double *C, int64_t crs,
                    int64_t ccs, int batch, int64_t sa, int64_t sb, int64_t sc, void *stream);
/* bilu_diag_tsgemm -- the tall-skinny variant (B staged in shared memory, warps streaming
 * 8-row tiles of A; used for the per-contributor Schur updates and the panel scaling of
 * blocks wider than 16), same arguments; requires K <= 128 and N <= 128 (else 1). */
int bilu_diag_tsgemm(int M, int N, int K, double alpha, const double *A, int64_t ars, int64_t acs,
                     const double *B, int64_t brs, int64_t bcs, double beta, double *C, int64_t crs,
                     int64_t ccs, int batch, int64_t sa, int64_t sb, int64_t sc, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BILU_H */
