/*
 * bilu_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, scalar-loop CPU oracle of the paper's Crout-type block ILU
 * (Bollhoefer, Schenk, Verbosio, arXiv:1908.10169).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  It shares no code, header, helper or constant with the CUDA
 * product path (paper_1908_10169_b200/).
 *
 * Conventions:
 *   input  : Ã (already symmetrically permuted), CSR, 0-based, sorted, no dups.
 *   output : Ã ≈ L · P · U = L · D^{-1} · U   (Sec. 2.2)
 *            L unit block-lower, stored per final block K as the kept rows
 *              i >= e_K (sorted) and one dense m_K x b_K panel, row-major.
 *            Ũ = P·U (unscaled U rows), stored per block as the kept cols
 *              j >= e_K (sorted) and one dense b_K x c_K panel, column-major.
 *            D_K = P_K^{-1}, dense b_K x b_K, column-major.
 */
#ifndef BILU_ORACLE_H
#define BILU_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t n, nblk;      /* final partition (after progressive aggregation) */
  int32_t *bstart;      /* nblk+1 */
  int64_t *Lp;          /* nblk+1 offsets into Li (rows)                    */
  int32_t *Li;          /* kept L rows, global index                        */
  int64_t *Lvp;         /* nblk+1 offsets into Lv                           */
  double  *Lv;          /* m x b row-major panels                           */
  int64_t *Up;          /* nblk+1 offsets into Ui (cols)                    */
  int32_t *Ui;
  int64_t *Uvp;         /* nblk+1 offsets into Uv                           */
  double  *Uv;          /* b x c column-major panels (unscaled Ũ)          */
  int64_t *Dp;          /* nblk+1 offsets into Dv                           */
  double  *Dv;          /* b x b column-major, D_K = P_K^{-1}               */
  /* statistics */
  double  flops;            /* algorithmic flops of the executed structure  */
  double  t_factor_s;       /* steady-clock seconds of the numeric phase    */
  int32_t n_merges;
  int32_t breakdown_block;  /* -1 if none */
  int64_t n_decisions;      /* drop/keep decisions taken                    */
  int64_t n_near;           /* decisions with margin <= near_rel            */
  double  min_margin;       /* min |max/tau - 1| over all decisions         */
  int64_t n_perturbed;      /* pivot blocks modified by the Sec. 3.6 perturbation */
  int64_t n_override_applied; /* replayed decisions (each within OVR_GUARD of tau) */
} orc_factor;

/* Sec. 3.6 perturbation parameters (R19); perturb = 0 disables it. */
typedef struct { int32_t perturb; double tau, rho, cond_max; } orc_perturb;

/* One forced decision (decision replay, SURVEY.md 8(c) reading 15).
 * side 0 = L row `idx` of original block `blk`, side 1 = U col `idx`. */
typedef struct { int32_t blk, side, idx, keep; } orc_override;

/* Returns 0 on success, 1 bad argument, 2 breakdown (singular pivot block),
 * 3 out of memory, 5 an override names a decision whose margin |max/tau - 1| exceeds
 * OVR_GUARD = 1e-6 (refused: only near-threshold decisions may be replayed, R15).  On success *f owns malloc'd arrays (free with orc_free). */
int orc_bilu_factor(int32_t n, const int64_t *row_ptr, const int32_t *col_idx,
                    const double *val, int32_t nblk, const int32_t *bsizes,
                    double tau, int32_t aggregate, int32_t max_block,
                    const orc_override *ovr, int64_t n_ovr, double near_rel,
                    orc_factor *f);

/* As orc_bilu_factor, with aggregation segments: seg[K] (initial block K) -- block K is
 * merged into the aggregate ending at K-1 only if seg[K] == seg[K-1] (R18). */
int orc_bilu_factor_seg(int32_t n, const int64_t *row_ptr, const int32_t *col_idx,
                        const double *val, int32_t nblk, const int32_t *bsizes,
                        double tau, int32_t aggregate, int32_t max_block,
                        const orc_override *ovr, int64_t n_ovr, double near_rel,
                        const int32_t *seg, orc_factor *f);

/* As orc_bilu_factor_seg, with the diagonal-block perturbation of Sec. 3.6 (pt may be NULL). */
int orc_bilu_factor_pt(int32_t n, const int64_t *row_ptr, const int32_t *col_idx,
                       const double *val, int32_t nblk, const int32_t *bsizes,
                       double tau, int32_t aggregate, int32_t max_block,
                       const orc_override *ovr, int64_t n_ovr, double near_rel,
                       const int32_t *seg, const orc_perturb *pt, orc_factor *f);

/* y = (L P U)^{-1} x in the permuted ordering (forward/backward substitution
 * with D multiplies).  x, y host arrays of length n. */
int orc_bilu_apply(const orc_factor *f, const double *x, double *y);

/* The progressive-aggregation test of Sec. 3.5. */
int orc_aggregate_test(int64_t p, int64_t q, int64_t r, int64_t s, int64_t t,
                       int64_t r2, int64_t s2, int64_t t2, int64_t u, int64_t v,
                       int64_t max_block);

/* ILU(1,tau) initial block estimate of Sec. 3.4 (R20) on an
 * already-permuted CSR matrix; out receives the block sizes (capacity n).  Returns the number
 * of blocks, -1 on a bad argument. */
int32_t orc_ilu1_blocks(int32_t n, const int64_t *rp, const int32_t *ci, const double *val, double tau,
                        int32_t max_size, int32_t *out);

/* One estimated set of Sec. 3.4 (lower = 1: I~_k of column k of L, 0: J~_k of row k of U),
 * ascending in out (capacity n); returns its size, -1 on a bad argument. */
int32_t orc_ilu1_set(int32_t n, const int64_t *rp, const int32_t *ci, const double *val, double tau, int32_t k,
                     int32_t lower, int32_t *out);

/* Cosine-based blocking of Sec. 3.2 (R21) on the pattern of A:
 * q (capacity n) receives the grouping permutation (new -> old), sizes (capacity n) the group
 * sizes; returns the number of groups, -1 on a bad argument. */
int32_t orc_cosine_blocks(int32_t n, const int64_t *rp, const int32_t *ci, double tau, int32_t max_size,
                          int32_t *q, int32_t *sizes);

/* Maximum product transversal + MC64-style scalings of Sec. 3.1 (DESIGN.md
 * R22) by the dense O(n^3) Hungarian method (small n): sigma[i] = column matched to row i,
 * dl, dr the row / column scalings.  Returns 0, -1 bad argument, -2 structurally singular. */
int orc_mwm(int32_t n, const int64_t *rp, const int32_t *ci, const double *val, int32_t *sigma, double *dl,
            double *dr);

void orc_free(orc_factor *f);

#ifdef __cplusplus
}
#endif
#endif
