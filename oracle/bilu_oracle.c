/*
 * bilu_oracle.c -- TEST INFRASTRUCTURE ONLY (see bilu_oracle.h).
 *
 * A plain, slow, obviously-correct CPU implementation of the numeric phase of
 * the paper's Crout-type block ILU with tau-dropping and progressive
 * aggregation.  Scalar loops, fp64, no BLAS, no threads.  It follows the
 * paper's steps in the paper's order:
 *
 *   Alg. 1 "Crout ILU"                 PAPER.md:158-175  (Sec. 2.1)
 *   block generalisation, drop rule     PAPER.md:205-212  (Sec. 2.2)
 *   hybrid storage (Fig. 1)
 *   gather / GEMM / scatter update      PAPER.md:368-374  (Fig. 2)
 *   A ~ L D^{-1} U, inverted pivots
 *   no pivoting outside diagonal blocks PAPER.md:792-799
 *   L_head/L_list/L_first row access
 *   progressive aggregation (mu/nu)     PAPER.md:1405-1453 (Sec. 3.5)
 *
 * Readings where the paper is silent or garbled are listed in DESIGN.md
 * ("Readings of the paper"); the ones used here are cited inline as R<n>.
 */
#include "bilu_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef struct {
  int32_t s, b;       /* first row/col and size of the (possibly merged) block */
  int32_t is_void;    /* merged into its successor        */
  int32_t m;          /* kept L rows (all >= e)                                */
  int32_t *Li;
  double *Lv;         /* m x b, row-major                                      */
  int32_t c;          /* kept U cols (all >= e)                                */
  int32_t *Ui;
  double *Uv;         /* b x c, column-major: the unscaled rows Ũ = P U        */
  double *D;          /* b x b, column-major: D = P^{-1}                        */
  int32_t firstL, firstU; /* L_first / U_first              */
  int32_t nextL, nextU;   /* L_list / U_list                                   */
} oblk;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void *xmalloc(size_t bytes) { return malloc(bytes ? bytes : 1); }
static void *xcalloc(size_t cnt, size_t sz) { return calloc(cnt ? cnt : 1, sz ? sz : 1); }

/* ---------------- progressive aggregation test (Sec. 3.5) ---------------- */
/* mu = p(p+r+s+r'+s') + q(q+t+t')
 * nu = (p+q)(p+q+u+v)
 * merge iff nu <= 1.2 mu or nu <= mu + 2(p+q)
 * R10: 1.2 evaluated exactly as 5 nu <= 6 mu.   R9: p+q <= max_block
 * ("the maximum block size should be limited").          */
int orc_aggregate_test(int64_t p, int64_t q, int64_t r, int64_t s, int64_t t,
                       int64_t r2, int64_t s2, int64_t t2, int64_t u, int64_t v,
                       int64_t max_block) {
  int64_t mu = p * (p + r + s + r2 + s2) + q * (q + t + t2);
  int64_t nu = (p + q) * (p + q + u + v);
  if (p + q > max_block) return 0;
  return (5 * nu <= 6 * mu) || (nu <= mu + 2 * (p + q));
}

/* ---------------- dense inverse by Gauss-Jordan, partial pivoting -------- */
/* "factorizing and inverting the diagonal blocks using dense matrix kernels"
 * (PAPER.md:788-790), pivoting only inside the block.
 * a: b x b column-major (destroyed), inv: b x b column-major.
 * Pivot = first row of maximal |a_ik| (R6).  Returns 1 on an exact zero pivot. */
static int gauss_jordan_inverse(int b, double *a, double *inv) {
  int i, j, k;
  for (j = 0; j < b; ++j)
    for (i = 0; i < b; ++i) inv[i + (size_t)j * b] = (i == j) ? 1.0 : 0.0;
  for (k = 0; k < b; ++k) {
    int piv = k;
    double best = fabs(a[k + (size_t)k * b]);
    for (i = k + 1; i < b; ++i) {
      double v = fabs(a[i + (size_t)k * b]);
      if (v > best) { best = v; piv = i; }
    }
    if (best == 0.0) return 1;
    if (piv != k) {
      for (j = 0; j < b; ++j) {
        double t = a[k + (size_t)j * b]; a[k + (size_t)j * b] = a[piv + (size_t)j * b]; a[piv + (size_t)j * b] = t;
        t = inv[k + (size_t)j * b]; inv[k + (size_t)j * b] = inv[piv + (size_t)j * b]; inv[piv + (size_t)j * b] = t;
      }
    }
    double d = a[k + (size_t)k * b];
    for (j = 0; j < b; ++j) { a[k + (size_t)j * b] /= d; inv[k + (size_t)j * b] /= d; }
    for (i = 0; i < b; ++i) {
      if (i == k) continue;
      double f = a[i + (size_t)k * b];
      if (f == 0.0) continue;
      for (j = 0; j < b; ++j) {
        a[i + (size_t)j * b] -= f * a[k + (size_t)j * b];
        inv[i + (size_t)j * b] -= f * inv[k + (size_t)j * b];
      }
    }
  }
  return 0;
}

/* ---------------- diagonal-block perturbation (Sec. 3.6) ----------------
 * alpha = max |a_ij| of the matrix; tau_p, rho the absolute / relative tolerances (the paper
 * uses 1e-2 and 1e-1).  Column j of the pivot block with entries d and
 * delta_j = max|d|: the largest entry d_kj (the diagonal d_jj instead whenever
 * 2|d_jj| >= |d_kj|) becomes d_kj (1 + rho beta_j) + sign(d_kj) tau_p alpha
 * (PAPER.md:1524), beta_j := delta_j (beta_j is undefined in the paper, R19,
 * as in SPEC), sign(0) := +1; "after that we proceed analogously with respect to the rows"
 * (PAPER.md:1526-1527).  Trigger (R19): a zero column / row ("if d = 0") perturbs that
 * column / row; a singular block (zero pivot in the Gauss-Jordan elimination) or an
 * ill-conditioned one (kappa_1 = |P|_1 |P^{-1}|_1 > cond_max) perturbs every column, then
 * every row; if that is still singular / ill-conditioned, sign(p_ii) tau_p alpha is added to
 * every diagonal entry; if that fails too, the block is reported as a breakdown. */
static double sgn1(double x) { return x < 0.0 ? -1.0 : 1.0; }

static void perturb_col(int b, double *P, int j, double alpha, double tau_p, double rho) {
  int i, k = 0;
  double dmax = -1.0;
  for (i = 0; i < b; ++i) {
    double v = fabs(P[i + (size_t)j * b]);
    if (v > dmax) { dmax = v; k = i; }
  }
  if (2.0 * fabs(P[j + (size_t)j * b]) >= fabs(P[k + (size_t)j * b])) k = j;
  double *d = &P[k + (size_t)j * b];
  *d = *d * (1.0 + rho * dmax) + sgn1(*d) * tau_p * alpha;
}

static void perturb_row(int b, double *P, int i, double alpha, double tau_p, double rho) {
  int j, k = 0;
  double dmax = -1.0;
  for (j = 0; j < b; ++j) {
    double v = fabs(P[i + (size_t)j * b]);
    if (v > dmax) { dmax = v; k = j; }
  }
  if (2.0 * fabs(P[i + (size_t)i * b]) >= fabs(P[i + (size_t)k * b])) k = i;
  double *d = &P[i + (size_t)k * b];
  *d = *d * (1.0 + rho * dmax) + sgn1(*d) * tau_p * alpha;
}

static double norm1(int b, const double *M) {
  double best = 0.0;
  for (int j = 0; j < b; ++j) {
    double s = 0.0;
    for (int i = 0; i < b; ++i) s += fabs(M[i + (size_t)j * b]);
    if (s > best) best = s;
  }
  return best;
}

/* inverse of P (column-major, b x b; P is modified: it ends as the perturbed block), with the
 * perturbation of Sec. 3.6 when enabled.  Returns 0 (D = inverse), 1 (breakdown).
 * *perturbed is set to 1 if the block was modified. */
static int pivot_inverse(int b, double *P, double *D, double *A, int perturb, double alpha, double tau_p,
                         double rho, double cond_max, int *perturbed) {
  int i, j, zero_any = 0;
  *perturbed = 0;
  if (!perturb) {
    memcpy(A, P, sizeof(double) * (size_t)b * b);
    return gauss_jordan_inverse(b, A, D);
  }
  for (j = 0; j < b; ++j) {
    double m = 0.0;
    for (i = 0; i < b; ++i) m = fmax(m, fabs(P[i + (size_t)j * b]));
    if (m == 0.0) { perturb_col(b, P, j, alpha, tau_p, rho); zero_any = 1; }
  }
  for (i = 0; i < b; ++i) {
    double m = 0.0;
    for (j = 0; j < b; ++j) m = fmax(m, fabs(P[i + (size_t)j * b]));
    if (m == 0.0) { perturb_row(b, P, i, alpha, tau_p, rho); zero_any = 1; }
  }
  for (int stage = 0; stage < 3; ++stage) {
    if (stage == 1) {
      for (j = 0; j < b; ++j) perturb_col(b, P, j, alpha, tau_p, rho);
      for (i = 0; i < b; ++i) perturb_row(b, P, i, alpha, tau_p, rho);
    } else if (stage == 2) {
      for (i = 0; i < b; ++i) P[i + (size_t)i * b] += sgn1(P[i + (size_t)i * b]) * tau_p * alpha;
    }
    memcpy(A, P, sizeof(double) * (size_t)b * b);
    if (!gauss_jordan_inverse(b, A, D) && norm1(b, P) * norm1(b, D) <= cond_max) {
      *perturbed = zero_any || stage > 0;
      return 0;
    }
  }
  return 1;
}

/* ---------------- helpers ---------------- */
static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}
static int cmp_ovr(const void *a, const void *b) {
  const orc_override *x = (const orc_override *)a, *y = (const orc_override *)b;
  if (x->blk != y->blk) return (x->blk > y->blk) - (x->blk < y->blk);
  if (x->side != y->side) return (x->side > y->side) - (x->side < y->side);
  return (x->idx > y->idx) - (x->idx < y->idx);
}
/* first position p in sorted list[lo..hi) with list[p] >= key */
static int32_t lower_bound(const int32_t *list, int32_t lo, int32_t hi, int32_t key) {
  while (lo < hi) {
    int32_t mid = lo + (hi - lo) / 2;
    if (list[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}
/* size of the union of two sorted, duplicate-free lists */
static int64_t union_count(const int32_t *a, int32_t na, const int32_t *b, int32_t nb) {
  int32_t i = 0, j = 0; int64_t cnt = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i; else if (a[i] > b[j]) ++j; else { ++i; ++j; }
    ++cnt;
  }
  return cnt + (na - i) + (nb - j);
}
/* union of two sorted lists into out, returns its size */
static int32_t union_merge(const int32_t *a, int32_t na, const int32_t *b, int32_t nb, int32_t *out) {
  int32_t i = 0, j = 0, k = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) out[k++] = a[i++];
    else if (a[i] > b[j]) out[k++] = b[j++];
    else { out[k++] = a[i++]; ++j; }
  }
  while (i < na) out[k++] = a[i++];
  while (j < nb) out[k++] = b[j++];
  return k;
}

static const orc_override *find_override(const orc_override *ov, int64_t nov, int32_t blk,
                                         int32_t side, int32_t idx) {
  int64_t lo = 0, hi = nov;
  orc_override key; key.blk = blk; key.side = side; key.idx = idx; key.keep = 0;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    int c = cmp_ovr(&ov[mid], &key);
    if (c == 0) return &ov[mid];
    if (c < 0) lo = mid + 1; else hi = mid;
  }
  return NULL;
}

typedef struct {
  const orc_override *ov; int64_t nov;
  double tau, near_rel;
  int64_t n_decisions, n_near; double min_margin;
  int64_t n_applied;      /* overrides that matched a decision                        */
  int64_t n_refused;      /* overrides of decisions farther than OVR_GUARD from tau   */
} decider;

/* An override (decision replay, R15) may only flip a decision that is near tau in the
 * oracle's OWN arithmetic: north_star exempts only decisions within 1e-8 relative of the
 * threshold; OVR_GUARD leaves two decades for the rounding differences of the two sides.
 * A GPU-supplied override farther from tau than this is refused and the factorization
 * fails (status 5), so a margin bug on the GPU cannot make the oracle copy its decisions. */
#define OVR_GUARD 1e-6

/* Keep iff max_t |x_t| > tau (R1: max-abs norm; R2: ties drop, "<=" in
 * PAPER.md:167,173; R3: the *scaled* row l_ik l_kk^{-1}). */
static int decide(decider *d, int32_t blk, int32_t side, int32_t idx, double mx) {
  int keep = mx > d->tau;
  d->n_decisions++;
  if (d->tau > 0.0) {
    double margin = fabs(mx / d->tau - 1.0);
    if (margin < d->min_margin) d->min_margin = margin;
    if (margin <= d->near_rel) d->n_near++;
  }
  if (d->nov) {
    const orc_override *o = find_override(d->ov, d->nov, blk, side, idx);
    if (o) {
      if (!(d->tau > 0.0) || !(fabs(mx / d->tau - 1.0) <= OVR_GUARD)) { d->n_refused++; return keep; }
      keep = o->keep != 0;
      d->n_applied++;
    }
  }
  return keep;
}

/* ---------------- the factorization ---------------- */
/* seg (may be NULL): aggregation segment of every initial block; block K is merged into
 * the aggregate ending at K-1 only if seg[K] == seg[K-1] (the distributed factorization
 * keeps aggregation inside each rank's blocks, reading R18). */
static int factor_impl(int32_t n, const int64_t *row_ptr, const int32_t *col_idx,
                       const double *val, int32_t nblk, const int32_t *bsizes,
                       double tau, int32_t aggregate, int32_t max_block,
                       const orc_override *ovr, int64_t n_ovr, double near_rel,
                       const int32_t *seg, const orc_perturb *pt, orc_factor *f) {
  int32_t i, K;
  int64_t e64;
  memset(f, 0, sizeof(*f));
  f->breakdown_block = -1;
  if (n < 1 || nblk < 1 || !row_ptr || !col_idx || !val || !bsizes || !(tau >= 0.0) || max_block < 1)
    return 1;
  /* ---- validate the partition and the CSR ---- */
  int32_t *bs = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(nblk + 1));
  bs[0] = 0;
  for (K = 0; K < nblk; ++K) {
    if (bsizes[K] < 1 || bsizes[K] > max_block) { free(bs); return 1; }
    bs[K + 1] = bs[K] + bsizes[K];
  }
  if (bs[nblk] != n || row_ptr[0] != 0) { free(bs); return 1; }
  for (i = 0; i < n; ++i) {
    if (row_ptr[i + 1] < row_ptr[i]) { free(bs); return 1; }
    for (e64 = row_ptr[i]; e64 < row_ptr[i + 1]; ++e64) {
      if (col_idx[e64] < 0 || col_idx[e64] >= n) { free(bs); return 1; }
      if (e64 > row_ptr[i] && col_idx[e64] <= col_idx[e64 - 1]) { free(bs); return 1; }
    }
  }
  int64_t nnz = row_ptr[n];
  int32_t *block_of = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)n);
  for (K = 0; K < nblk; ++K) for (i = bs[K]; i < bs[K + 1]; ++i) block_of[i] = K;

  /* ---- column access to A (CSC by counting transpose) ---- */
  int64_t *cp = (int64_t *)xcalloc((size_t)n + 1, sizeof(int64_t));
  int32_t *cr = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)nnz);
  double *cv = (double *)xmalloc(sizeof(double) * (size_t)nnz);
  for (e64 = 0; e64 < nnz; ++e64) cp[col_idx[e64] + 1]++;
  for (i = 0; i < n; ++i) cp[i + 1] += cp[i];
  {
    int64_t *fill = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)n);
    memcpy(fill, cp, sizeof(int64_t) * (size_t)n);
    for (i = 0; i < n; ++i)
      for (e64 = row_ptr[i]; e64 < row_ptr[i + 1]; ++e64) {
        int64_t q = fill[col_idx[e64]]++;
        cr[q] = i; cv[q] = val[e64];
      }
    free(fill);
  }

  orc_override *ov = NULL;
  if (n_ovr > 0 && ovr) {
    ov = (orc_override *)xmalloc(sizeof(orc_override) * (size_t)n_ovr);
    memcpy(ov, ovr, sizeof(orc_override) * (size_t)n_ovr);
    qsort(ov, (size_t)n_ovr, sizeof(orc_override), cmp_ovr);
  }
  decider dec; dec.ov = ov; dec.nov = ov ? n_ovr : 0; dec.tau = tau; dec.near_rel = near_rel;
  dec.n_decisions = 0; dec.n_near = 0; dec.min_margin = INFINITY; dec.n_applied = 0; dec.n_refused = 0;

  /* ---- state ---- */
  oblk *B = (oblk *)xcalloc((size_t)nblk, sizeof(oblk));
  int32_t *Lhead = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)nblk);
  int32_t *Uhead = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)nblk);
  for (K = 0; K < nblk; ++K) { Lhead[K] = -1; Uhead[K] = -1; }
  int32_t *rslot = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)n);
  int32_t *cslot = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)n);
  for (i = 0; i < n; ++i) { rslot[i] = -1; cslot[i] = -1; }
  int32_t *rrows = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)n);  /* slot -> row */
  int32_t *ccols = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)n);  /* slot -> col */
  int32_t *Lc = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)nblk);
  int32_t *Uc = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)nblk);
  size_t wcap = 1024;
  double *wl = NULL, *wu = NULL;   /* (slots) x b each */
  size_t wl_cap = 0, wu_cap = 0;
  double *P = (double *)xmalloc(sizeof(double) * (size_t)max_block * max_block);
  double *Pw = (double *)xmalloc(sizeof(double) * (size_t)max_block * max_block);
  double alpha = 0.0;                      /* max |a_ij| (Sec. 3.6) */
  for (e64 = 0; e64 < row_ptr[n]; ++e64) alpha = fmax(alpha, fabs(val[e64]));
  double *tmp = (double *)xmalloc(sizeof(double) * (size_t)max_block * 2);
  int32_t *keep_idx = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)n);
  int status = 0;
  double flops = 0.0;
  int32_t n_merges = 0;
  (void)wcap;

  double t0 = now_s();
  for (K = 0; K < nblk && status == 0; ++K) {
    const int32_t s = bs[K], e = bs[K + 1], b = e - s;
    int32_t nLc = 0, nUc = 0, J, p, q, t, u;
    /* -- contributors via the linked lists: Uhead[K] holds
     *    blocks whose next Ũ column lies in K  -> feed the L side (Alg.1 l.3-4);
     *    Lhead[K] holds blocks whose next L row lies in K -> feed U (l.9-10).
     *    Void (merged-away) blocks drop out.          -- */
    for (J = Uhead[K]; J >= 0; J = B[J].nextU) if (!B[J].is_void) Lc[nLc++] = J;
    for (J = Lhead[K]; J >= 0; J = B[J].nextL) if (!B[J].is_void) Uc[nUc++] = J;
    /* R13: ascending order (any order is exact; this one is deterministic) */
    qsort(Lc, (size_t)nLc, sizeof(int32_t), cmp_i32);
    qsort(Uc, (size_t)nUc, sizeof(int32_t), cmp_i32);

    /* -- L side: block column buffer over rows >= s -- */
    int32_t nr = 0;
    for (i = s; i < e; ++i) { rslot[i] = nr; rrows[nr++] = i; }   /* diagonal block rows */
    /* count candidate rows first to size the buffer */
    for (int32_t c = s; c < e; ++c)
      for (e64 = cp[c]; e64 < cp[c + 1]; ++e64)
        if (cr[e64] >= e && rslot[cr[e64]] < 0) { rslot[cr[e64]] = nr; rrows[nr++] = cr[e64]; }
    for (int32_t a = 0; a < nLc; ++a) {
      oblk *Jb = &B[Lc[a]];
      for (p = Jb->firstL; p < Jb->m; ++p) {
        int32_t row = Jb->Li[p];
        if (row >= e && rslot[row] < 0) { rslot[row] = nr; rrows[nr++] = row; }
      }
    }
    if ((size_t)nr * b > wl_cap) { free(wl); wl_cap = (size_t)nr * b * 2; wl = (double *)xmalloc(sizeof(double) * wl_cap); }
    memset(wl, 0, sizeof(double) * (size_t)nr * b);
    /* Alg. 1 line 2: l_ik <- a_ik, i >= k */
    for (int32_t c = s; c < e; ++c)
      for (e64 = cp[c]; e64 < cp[c + 1]; ++e64)
        if (cr[e64] >= s) wl[(size_t)rslot[cr[e64]] * b + (c - s)] = cv[e64];
    /* Alg. 1 lines 3-4, blocked: W[i, K] -= L_J[i, :] * Ũ_J[:, K]   (Fig. 2) */
    for (int32_t a = 0; a < nLc; ++a) {
      oblk *Jb = &B[Lc[a]];
      const int32_t bJ = Jb->b;
      int32_t q0 = Jb->firstU, q1 = q0;
      while (q1 < Jb->c && Jb->Ui[q1] < e) ++q1;
      for (p = Jb->firstL; p < Jb->m; ++p) {
        double *wrow = wl + (size_t)rslot[Jb->Li[p]] * b;
        const double *lrow = Jb->Lv + (size_t)p * bJ;
        for (q = q0; q < q1; ++q) {
          const double *ucol = Jb->Uv + (size_t)q * bJ;
          double acc = 0.0;
          for (t = 0; t < bJ; ++t) acc += lrow[t] * ucol[t];
          wrow[Jb->Ui[q] - s] -= acc;
        }
      }
      flops += 2.0 * bJ * (double)(Jb->m - Jb->firstL) * (double)(q1 - q0);
    }

    /* -- U side: block row buffer over cols >= e -- */
    int32_t nc = 0;
    for (int32_t r = s; r < e; ++r)
      for (e64 = row_ptr[r]; e64 < row_ptr[r + 1]; ++e64)
        if (col_idx[e64] >= e && cslot[col_idx[e64]] < 0) { cslot[col_idx[e64]] = nc; ccols[nc++] = col_idx[e64]; }
    for (int32_t a = 0; a < nUc; ++a) {
      oblk *Jb = &B[Uc[a]];
      int32_t q0 = Jb->firstU;
      while (q0 < Jb->c && Jb->Ui[q0] < e) ++q0;
      for (q = q0; q < Jb->c; ++q)
        if (cslot[Jb->Ui[q]] < 0) { cslot[Jb->Ui[q]] = nc; ccols[nc++] = Jb->Ui[q]; }
    }
    if ((size_t)nc * b > wu_cap) { free(wu); wu_cap = (size_t)nc * b * 2 + 1; wu = (double *)xmalloc(sizeof(double) * wu_cap); }
    memset(wu, 0, sizeof(double) * (size_t)nc * b);
    /* Alg. 1 line 8: u_ki <- a_ki, i > k (the diagonal block lives in W_L) */
    for (int32_t r = s; r < e; ++r)
      for (e64 = row_ptr[r]; e64 < row_ptr[r + 1]; ++e64)
        if (col_idx[e64] >= e) wu[(size_t)cslot[col_idx[e64]] * b + (r - s)] = val[e64];
    /* Alg. 1 lines 9-10, blocked: W[K, j] -= L_J[K, :] * Ũ_J[:, j] */
    for (int32_t a = 0; a < nUc; ++a) {
      oblk *Jb = &B[Uc[a]];
      const int32_t bJ = Jb->b;
      int32_t p0 = Jb->firstL, p1 = p0;
      while (p1 < Jb->m && Jb->Li[p1] < e) ++p1;
      int32_t q0 = Jb->firstU;
      while (q0 < Jb->c && Jb->Ui[q0] < e) ++q0;
      for (q = q0; q < Jb->c; ++q) {
        double *wcol = wu + (size_t)cslot[Jb->Ui[q]] * b;
        const double *ucol = Jb->Uv + (size_t)q * bJ;
        for (p = p0; p < p1; ++p) {
          const double *lrow = Jb->Lv + (size_t)p * bJ;
          double acc = 0.0;
          for (t = 0; t < bJ; ++t) acc += lrow[t] * ucol[t];
          wcol[Jb->Li[p] - s] -= acc;
        }
      }
      flops += 2.0 * bJ * (double)(p1 - p0) * (double)(Jb->c - q0);
    }

    /* -- pivot block P_K and D_K = P_K^{-1} -- */
    oblk *Kb = &B[K];
    Kb->s = s; Kb->b = b; Kb->is_void = 0;
    Kb->D = (double *)xmalloc(sizeof(double) * (size_t)b * b);
    for (int32_t r = 0; r < b; ++r)
      for (int32_t c = 0; c < b; ++c) P[r + (size_t)c * b] = wl[(size_t)r * b + c];
    {
      int pert = 0;
      if (pivot_inverse(b, P, Kb->D, Pw, pt && pt->perturb, alpha, pt ? pt->tau : 0.0, pt ? pt->rho : 0.0,
                        pt ? pt->cond_max : 0.0, &pert)) {
        status = 2; f->breakdown_block = K; break;
      }
      f->n_perturbed += pert;
    }
    flops += 2.0 * b * b * (double)b + 2.0 * b * b * (double)((nr - b) + nc);

    /* -- L rows: l_i = w_i D_K, keep iff max|l_i| > tau -- */
    int32_t nk = 0;
    for (int32_t sl = b; sl < nr; ++sl) {
      const double *w = wl + (size_t)sl * b;
      double mx = 0.0;
      for (int32_t c = 0; c < b; ++c) {
        double acc = 0.0;
        for (t = 0; t < b; ++t) acc += w[t] * Kb->D[t + (size_t)c * b];
        if (fabs(acc) > mx) mx = fabs(acc);
      }
      if (decide(&dec, K, 0, rrows[sl], mx)) keep_idx[nk++] = rrows[sl];
    }
    qsort(keep_idx, (size_t)nk, sizeof(int32_t), cmp_i32);
    Kb->m = nk;
    Kb->Li = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)nk);
    Kb->Lv = (double *)xmalloc(sizeof(double) * (size_t)nk * b);
    for (p = 0; p < nk; ++p) {
      const double *w = wl + (size_t)rslot[keep_idx[p]] * b;
      Kb->Li[p] = keep_idx[p];
      for (int32_t c = 0; c < b; ++c) {
        double acc = 0.0;
        for (t = 0; t < b; ++t) acc += w[t] * Kb->D[t + (size_t)c * b];
        Kb->Lv[(size_t)p * b + c] = acc;
      }
    }
    /* -- U cols: u_j = D_K z_j, keep iff max|u_j| > tau; store Ũ_j = z_j -- */
    nk = 0;
    for (int32_t sl = 0; sl < nc; ++sl) {
      const double *z = wu + (size_t)sl * b;
      double mx = 0.0;
      for (int32_t r = 0; r < b; ++r) {
        double acc = 0.0;
        for (t = 0; t < b; ++t) acc += Kb->D[r + (size_t)t * b] * z[t];
        if (fabs(acc) > mx) mx = fabs(acc);
      }
      if (decide(&dec, K, 1, ccols[sl], mx)) keep_idx[nk++] = ccols[sl];
    }
    qsort(keep_idx, (size_t)nk, sizeof(int32_t), cmp_i32);
    Kb->c = nk;
    Kb->Ui = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)nk);
    Kb->Uv = (double *)xmalloc(sizeof(double) * (size_t)nk * b);
    for (q = 0; q < nk; ++q) {
      Kb->Ui[q] = keep_idx[q];
      memcpy(Kb->Uv + (size_t)q * b, wu + (size_t)cslot[keep_idx[q]] * b, sizeof(double) * (size_t)b);
    }
    /* reset the buffers' index maps */
    for (int32_t sl = 0; sl < nr; ++sl) rslot[rrows[sl]] = -1;
    for (int32_t sl = 0; sl < nc; ++sl) cslot[ccols[sl]] = -1;

    /* -- advance L_first/U_first of the blocks that fed K, relink -- */
    {
      int32_t cnt = 0;
      for (J = Lhead[K]; J >= 0; J = B[J].nextL) Uc[cnt++] = J;   /* reuse as scratch */
      for (int32_t a = 0; a < cnt; ++a) {
        oblk *Jb = &B[Uc[a]];
        if (Jb->is_void) continue;
        while (Jb->firstL < Jb->m && Jb->Li[Jb->firstL] < e) Jb->firstL++;
        if (Jb->firstL < Jb->m) {
          int32_t T = block_of[Jb->Li[Jb->firstL]];
          Jb->nextL = Lhead[T]; Lhead[T] = Uc[a];
        }
      }
      cnt = 0;
      for (J = Uhead[K]; J >= 0; J = B[J].nextU) Lc[cnt++] = J;
      for (int32_t a = 0; a < cnt; ++a) {
        oblk *Jb = &B[Lc[a]];
        if (Jb->is_void) continue;
        while (Jb->firstU < Jb->c && Jb->Ui[Jb->firstU] < e) Jb->firstU++;
        if (Jb->firstU < Jb->c) {
          int32_t T = block_of[Jb->Ui[Jb->firstU]];
          Jb->nextU = Uhead[T]; Uhead[T] = Lc[a];
        }
      }
      Lhead[K] = -1; Uhead[K] = -1;
    }

    /* -- progressive aggregation of the previous (aggregated) block and K (Sec. 3.5) -- */
    if (aggregate && K > 0 && !B[K - 1].is_void && (!seg || seg[K] == seg[K - 1])) {
      oblk *Pb = &B[K - 1];
      const int32_t pp = Pb->b, qq = b;
      /* rows of L_{k-1} inside block k (r) and below it (s); same for U */
      int32_t lr0 = lower_bound(Pb->Li, 0, Pb->m, s), lr1 = lower_bound(Pb->Li, 0, Pb->m, e);
      int32_t uc0 = lower_bound(Pb->Ui, 0, Pb->c, s), uc1 = lower_bound(Pb->Ui, 0, Pb->c, e);
      int64_t rr = lr1 - lr0, ss = Pb->m - lr1, tt = Kb->m;
      int64_t rr2 = uc1 - uc0, ss2 = Pb->c - uc1, tt2 = Kb->c;
      /* u, v: union of index sets ignoring cancellation */
      int64_t uu = union_count(Pb->Li + lr1, Pb->m - lr1, Kb->Li, Kb->m);
      int64_t vv = union_count(Pb->Ui + uc1, Pb->c - uc1, Kb->Ui, Kb->c);
      if (orc_aggregate_test(pp, qq, rr, ss, tt, rr2, ss2, tt2, uu, vv, max_block)) {
        const int32_t pq = pp + qq;
        /* L10 = L_{k,k-1} (q x p, dense, zero for dropped rows), row-major */
        double *L10 = (double *)xcalloc((size_t)qq * pp, sizeof(double));
        for (p = lr0; p < lr1; ++p)
          memcpy(L10 + (size_t)(Pb->Li[p] - s) * pp, Pb->Lv + (size_t)p * pp, sizeof(double) * (size_t)pp);
        /* U01 = U_{k-1,k} = D_{k-1} Ũ_{k-1,k} (p x q), column-major */
        double *U01 = (double *)xcalloc((size_t)pp * qq, sizeof(double));
        for (q = uc0; q < uc1; ++q) {
          int32_t c = Pb->Ui[q] - s;
          for (int32_t r = 0; r < pp; ++r) {
            double acc = 0.0;
            for (t = 0; t < pp; ++t) acc += Pb->D[r + (size_t)t * pp] * Pb->Uv[(size_t)q * pp + t];
            U01[r + (size_t)c * pp] = acc;
          }
        }
        /* merged rows: L^_{>,k-1} = L_{>,k-1} - L_{>,k} L_{k,k-1}; L_{>,k} unchanged
         * (\rdel PAPER.md:1399-1401; identity PAPER.md:1348-1387) */
        int32_t *Ru = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)uu);
        int32_t nu = union_merge(Pb->Li + lr1, Pb->m - lr1, Kb->Li, Kb->m, Ru);
        double *Lm = (double *)xcalloc((size_t)nu * pq, sizeof(double));
        {
          int32_t ia = lr1, ib = 0;
          for (p = 0; p < nu; ++p) {
            double *out = Lm + (size_t)p * pq;
            const double *la = NULL, *lb = NULL;
            if (ia < Pb->m && Pb->Li[ia] == Ru[p]) la = Pb->Lv + (size_t)(ia++) * pp;
            if (ib < Kb->m && Kb->Li[ib] == Ru[p]) lb = Kb->Lv + (size_t)(ib++) * qq;
            for (int32_t c = 0; c < pp; ++c) {
              double acc = la ? la[c] : 0.0;
              if (lb) for (t = 0; t < qq; ++t) acc -= lb[t] * L10[(size_t)t * pp + c];
              out[c] = acc;
            }
            for (int32_t c = 0; c < qq; ++c) out[pp + c] = lb ? lb[c] : 0.0;
          }
        }
        /* merged cols: Ũ^ = [Ũ_{k-1,>} ; Ũ_{k,>} + L_{k,k-1} Ũ_{k-1,>}] */
        int32_t *Cu = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)vv);
        int32_t nv = union_merge(Pb->Ui + uc1, Pb->c - uc1, Kb->Ui, Kb->c, Cu);
        double *Um = (double *)xcalloc((size_t)nv * pq, sizeof(double));
        {
          int32_t ia = uc1, ib = 0;
          for (q = 0; q < nv; ++q) {
            double *out = Um + (size_t)q * pq;
            const double *za = NULL, *zb = NULL;
            if (ia < Pb->c && Pb->Ui[ia] == Cu[q]) za = Pb->Uv + (size_t)(ia++) * pp;
            if (ib < Kb->c && Kb->Ui[ib] == Cu[q]) zb = Kb->Uv + (size_t)(ib++) * qq;
            for (int32_t r = 0; r < pp; ++r) out[r] = za ? za[r] : 0.0;
            for (int32_t r = 0; r < qq; ++r) {
              double acc = zb ? zb[r] : 0.0;
              if (za) for (t = 0; t < pp; ++t) acc += L10[(size_t)r * pp + t] * za[t];
              out[pp + r] = acc;
            }
          }
        }
        /* merged inverse: D^ = [[D1 + U01 D2 L10, -U01 D2], [-D2 L10, D2]]  (R7) */
        double *Dm = (double *)xcalloc((size_t)pq * pq, sizeof(double));
        {
          double *D2L10 = (double *)xcalloc((size_t)qq * pp, sizeof(double));  /* q x p col-major */
          double *U01D2 = (double *)xcalloc((size_t)pp * qq, sizeof(double));  /* p x q col-major */
          for (int32_t r = 0; r < qq; ++r)
            for (int32_t c = 0; c < pp; ++c) {
              double acc = 0.0;
              for (t = 0; t < qq; ++t) acc += Kb->D[r + (size_t)t * qq] * L10[(size_t)t * pp + c];
              D2L10[r + (size_t)c * qq] = acc;
            }
          for (int32_t r = 0; r < pp; ++r)
            for (int32_t c = 0; c < qq; ++c) {
              double acc = 0.0;
              for (t = 0; t < qq; ++t) acc += U01[r + (size_t)t * pp] * Kb->D[t + (size_t)c * qq];
              U01D2[r + (size_t)c * pp] = acc;
            }
          for (int32_t r = 0; r < pp; ++r)
            for (int32_t c = 0; c < pp; ++c) {
              double acc = Pb->D[r + (size_t)c * pp];
              for (t = 0; t < qq; ++t) acc += U01D2[r + (size_t)t * pp] * L10[(size_t)t * pp + c];
              Dm[r + (size_t)c * pq] = acc;
            }
          for (int32_t r = 0; r < pp; ++r)
            for (int32_t c = 0; c < qq; ++c) Dm[r + (size_t)(pp + c) * pq] = -U01D2[r + (size_t)c * pp];
          for (int32_t r = 0; r < qq; ++r)
            for (int32_t c = 0; c < pp; ++c) Dm[(pp + r) + (size_t)c * pq] = -D2L10[r + (size_t)c * qq];
          for (int32_t r = 0; r < qq; ++r)
            for (int32_t c = 0; c < qq; ++c) Dm[(pp + r) + (size_t)(pp + c) * pq] = Kb->D[r + (size_t)c * qq];
          free(D2L10); free(U01D2);
        }
        flops += 2.0 * uu * qq * pp + 2.0 * pp * qq * vv + 4.0 * pp * qq * (double)(pp + qq);
        /* block k-1 becomes void, the aggregate takes id k */
        int32_t s_new = Pb->s;
        free(Pb->Li); free(Pb->Lv); free(Pb->Ui); free(Pb->Uv); free(Pb->D);
        Pb->Li = NULL; Pb->Lv = NULL; Pb->Ui = NULL; Pb->Uv = NULL; Pb->D = NULL;
        Pb->m = 0; Pb->c = 0; Pb->b = 0; Pb->is_void = 1;
        free(Kb->Li); free(Kb->Lv); free(Kb->Ui); free(Kb->Uv); free(Kb->D);
        Kb->s = s_new; Kb->b = pq;
        Kb->m = nu; Kb->Li = Ru; Kb->Lv = Lm;
        Kb->c = nv; Kb->Ui = Cu; Kb->Uv = Um;
        Kb->D = Dm;
        free(L10); free(U01);
        n_merges++;
      }
    }
    /* -- link the finished block K into the lists by its first row / col -- */
    Kb->firstL = 0; Kb->firstU = 0; Kb->nextL = -1; Kb->nextU = -1;
    if (Kb->m > 0) { int32_t T = block_of[Kb->Li[0]]; Kb->nextL = Lhead[T]; Lhead[T] = K; }
    if (Kb->c > 0) { int32_t T = block_of[Kb->Ui[0]]; Kb->nextU = Uhead[T]; Uhead[T] = K; }
  }
  double t1 = now_s();

  if (status == 0) {
    /* ---- pack the final (non-void) blocks ---- */
    int32_t nf = 0; int64_t nL = 0, nLv = 0, nU = 0, nUv = 0, nD = 0;
    for (K = 0; K < nblk; ++K) if (!B[K].is_void) {
      nf++; nL += B[K].m; nLv += (int64_t)B[K].m * B[K].b;
      nU += B[K].c; nUv += (int64_t)B[K].c * B[K].b; nD += (int64_t)B[K].b * B[K].b;
    }
    f->n = n; f->nblk = nf;
    f->bstart = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(nf + 1));
    f->Lp = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(nf + 1));
    f->Lvp = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(nf + 1));
    f->Up = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(nf + 1));
    f->Uvp = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(nf + 1));
    f->Dp = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(nf + 1));
    f->Li = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)nL);
    f->Lv = (double *)xmalloc(sizeof(double) * (size_t)nLv);
    f->Ui = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)nU);
    f->Uv = (double *)xmalloc(sizeof(double) * (size_t)nUv);
    f->Dv = (double *)xmalloc(sizeof(double) * (size_t)nD);
    int32_t k2 = 0;
    f->Lp[0] = f->Lvp[0] = f->Up[0] = f->Uvp[0] = f->Dp[0] = 0;
    for (K = 0; K < nblk; ++K) if (!B[K].is_void) {
      oblk *Kb = &B[K];
      f->bstart[k2] = Kb->s;
      memcpy(f->Li + f->Lp[k2], Kb->Li, sizeof(int32_t) * (size_t)Kb->m);
      memcpy(f->Lv + f->Lvp[k2], Kb->Lv, sizeof(double) * (size_t)Kb->m * Kb->b);
      memcpy(f->Ui + f->Up[k2], Kb->Ui, sizeof(int32_t) * (size_t)Kb->c);
      memcpy(f->Uv + f->Uvp[k2], Kb->Uv, sizeof(double) * (size_t)Kb->c * Kb->b);
      memcpy(f->Dv + f->Dp[k2], Kb->D, sizeof(double) * (size_t)Kb->b * Kb->b);
      f->Lp[k2 + 1] = f->Lp[k2] + Kb->m;
      f->Lvp[k2 + 1] = f->Lvp[k2] + (int64_t)Kb->m * Kb->b;
      f->Up[k2 + 1] = f->Up[k2] + Kb->c;
      f->Uvp[k2 + 1] = f->Uvp[k2] + (int64_t)Kb->c * Kb->b;
      f->Dp[k2 + 1] = f->Dp[k2] + (int64_t)Kb->b * Kb->b;
      k2++;
    }
    f->bstart[nf] = n;
  }
  f->flops = flops;
  f->t_factor_s = t1 - t0;
  f->n_merges = n_merges;
  f->n_decisions = dec.n_decisions;
  f->n_near = dec.n_near;
  f->min_margin = dec.min_margin;
  f->n_override_applied = dec.n_applied;
  if (status == 0 && dec.n_refused > 0) status = 5;

  for (K = 0; K < nblk; ++K) {
    free(B[K].Li); free(B[K].Lv); free(B[K].Ui); free(B[K].Uv); free(B[K].D);
  }
  free(B); free(Lhead); free(Uhead); free(rslot); free(cslot); free(rrows); free(ccols);
  free(Lc); free(Uc); free(wl); free(wu); free(P); free(Pw); free(tmp); free(keep_idx);
  free(cp); free(cr); free(cv); free(block_of); free(bs); free(ov);
  return status;
}

/* ---------------- preconditioner application ---------------- */
/* Solve (L P U) y = x with P = D^{-1}:  forward  L w = x (unit block-lower,
 * column-oriented over the L panels), then backward y_K = D_K (w_K - Ũ_K y_C)
 * (U = D Ũ is unit block-upper).  PAPER.md:788-790 ("multiplying with D
 * instead of solving a sequence of dense linear systems"). */
int orc_bilu_apply(const orc_factor *f, const double *x, double *y) {
  int32_t K, n = f->n;
  if (!f || !f->bstart || !x || !y) return 1;
  double *w = (double *)xmalloc(sizeof(double) * (size_t)n);
  memcpy(w, x, sizeof(double) * (size_t)n);
  for (K = 0; K < f->nblk; ++K) {
    int32_t s = f->bstart[K], b = f->bstart[K + 1] - s;
    for (int64_t p = f->Lp[K]; p < f->Lp[K + 1]; ++p) {
      const double *l = f->Lv + f->Lvp[K] + (p - f->Lp[K]) * b;
      double acc = 0.0;
      for (int32_t t = 0; t < b; ++t) acc += l[t] * w[s + t];
      w[f->Li[p]] -= acc;
    }
  }
  double *z = (double *)xmalloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (K = f->nblk - 1; K >= 0; --K) {
    int32_t s = f->bstart[K], b = f->bstart[K + 1] - s;
    for (int32_t t = 0; t < b; ++t) z[t] = w[s + t];
    for (int64_t q = f->Up[K]; q < f->Up[K + 1]; ++q) {
      const double *u = f->Uv + f->Uvp[K] + (q - f->Up[K]) * b;
      double yj = y[f->Ui[q]];
      for (int32_t t = 0; t < b; ++t) z[t] -= u[t] * yj;
    }
    const double *D = f->Dv + f->Dp[K];
    for (int32_t r = 0; r < b; ++r) {
      double acc = 0.0;
      for (int32_t t = 0; t < b; ++t) acc += D[r + (size_t)t * b] * z[t];
      y[s + r] = acc;
    }
  }
  free(w); free(z);
  return 0;
}

void orc_free(orc_factor *f) {
  if (!f) return;
  free(f->bstart); free(f->Lp); free(f->Li); free(f->Lvp); free(f->Lv);
  free(f->Up); free(f->Ui); free(f->Uvp); free(f->Uv); free(f->Dp); free(f->Dv);
  memset(f, 0, sizeof(*f));
}

int orc_bilu_factor(int32_t n, const int64_t *row_ptr, const int32_t *col_idx,
                    const double *val, int32_t nblk, const int32_t *bsizes,
                    double tau, int32_t aggregate, int32_t max_block,
                    const orc_override *ovr, int64_t n_ovr, double near_rel,
                    orc_factor *f) {
  return factor_impl(n, row_ptr, col_idx, val, nblk, bsizes, tau, aggregate, max_block, ovr, n_ovr,
                     near_rel, NULL, NULL, f);
}

int orc_bilu_factor_pt(int32_t n, const int64_t *row_ptr, const int32_t *col_idx,
                       const double *val, int32_t nblk, const int32_t *bsizes,
                       double tau, int32_t aggregate, int32_t max_block,
                       const orc_override *ovr, int64_t n_ovr, double near_rel,
                       const int32_t *seg, const orc_perturb *pt, orc_factor *f) {
  return factor_impl(n, row_ptr, col_idx, val, nblk, bsizes, tau, aggregate, max_block, ovr, n_ovr,
                     near_rel, seg, pt, f);
}

int orc_bilu_factor_seg(int32_t n, const int64_t *row_ptr, const int32_t *col_idx,
                        const double *val, int32_t nblk, const int32_t *bsizes,
                        double tau, int32_t aggregate, int32_t max_block,
                        const orc_override *ovr, int64_t n_ovr, double near_rel,
                        const int32_t *seg, orc_factor *f) {
  return factor_impl(n, row_ptr, col_idx, val, nblk, bsizes, tau, aggregate, max_block, ovr, n_ovr,
                     near_rel, seg, NULL, f);
}

/* ---------------- ILU(1,tau) initial block estimate (Sec. 3.4) ----------------
 * For step k the estimated pattern of column k of L is
 *   I~_k = { i > k : a_ik != 0, |a_ik| >= tau |a_kk| }                                  (I^)
 *        u { i > k : exists j < k, a_jk != 0, a_ij != 0, |a_ij a_jk| >= tau |a_jj a_kk| }  (ILU(1) fill)
 * and of row k of U, symmetrically,
 *   J~_k = { j > k : a_kj != 0, |a_kj| >= tau |a_kk| }
 *        u { j > k : exists i < k, a_ki != 0, a_ij != 0, |a_ki a_ij| >= tau |a_ii a_kk| }.
 * Blocks grow greedily from k0: with l columns in the block, r / s the
 * sizes of the unions of I~_t / J~_t (t in the block) outside the block, f_l = (r + s + l) l;
 * the scalar count of the block is c' = sum_t (|I~_t| + |J~_t| + 1) (R20: "f_l - c"
 * is the scalar nnz, c the wasted zeros); column k0+l joins iff
 *   3 f_{l+1} <= 4 c'  or  f_{l+1} <= c' + 4 (l+1)   (exact integers for 4/3)
 * and l+1 <= max_size.  Returns the number of blocks, sizes in out (n entries capacity). */
static int cmp_int(const void *a, const void *b) { int x = *(const int *)a, y = *(const int *)b; return (x > y) - (x < y); }

static int32_t est_set(int32_t n, const int64_t *rp, const int32_t *ci, const double *val, const int64_t *cp,
                       const int32_t *cr, const int64_t *cmap, const double *diag, int32_t k, double tau, int lower,
                       int32_t *buf) {
  /* lower: column k of L via the CSC (rows i > k); else row k of U via the CSR (cols j > k) */
  int32_t m = 0;
  const double akk = diag[k];
  if (lower) {
    for (int64_t p = cp[k]; p < cp[k + 1]; ++p) {
      const int32_t i = cr[p];
      if (i > k && fabs(val[cmap[p]]) >= tau * fabs(akk)) buf[m++] = i;
    }
    for (int64_t p = cp[k]; p < cp[k + 1]; ++p) {          /* j < k with a_jk != 0 */
      const int32_t j = cr[p];
      if (j >= k) continue;
      const double ajk = val[cmap[p]];
      for (int64_t q = cp[j]; q < cp[j + 1]; ++q) {         /* i > k with a_ij != 0 */
        const int32_t i = cr[q];
        if (i > k && fabs(val[cmap[q]] * ajk) >= tau * fabs(diag[j] * akk)) buf[m++] = i;
      }
    }
  } else {
    for (int64_t p = rp[k]; p < rp[k + 1]; ++p) {
      const int32_t j = ci[p];
      if (j > k && fabs(val[p]) >= tau * fabs(akk)) buf[m++] = j;
    }
    for (int64_t p = rp[k]; p < rp[k + 1]; ++p) {          /* i < k with a_ki != 0 */
      const int32_t i = ci[p];
      if (i >= k) continue;
      const double aki = val[p];
      for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {         /* j > k with a_ij != 0 */
        const int32_t j = ci[q];
        if (j > k && fabs(aki * val[q]) >= tau * fabs(diag[i] * akk)) buf[m++] = j;
      }
    }
  }
  qsort(buf, (size_t)m, sizeof(int32_t), cmp_int);
  int32_t u = 0;
  for (int32_t x = 0; x < m; ++x) if (x == 0 || buf[x] != buf[x - 1]) buf[u++] = buf[x];
  return u;
}

/* CSC of the matrix (rows ascending within a column) with a map to the CSR entries, and the diagonal */
static void est_csc(int32_t n, const int64_t *rp, const int32_t *ci, const double *val, int64_t **cp_o,
                    int32_t **cr_o, int64_t **cmap_o, double **diag_o) {
  const int64_t nnz = rp[n];
  int64_t *cp = (int64_t *)xcalloc((size_t)n + 1, sizeof(int64_t));
  int32_t *cr = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
  int64_t *cmap = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
  double *diag = (double *)xcalloc((size_t)n, sizeof(double));
  for (int64_t p = 0; p < nnz; ++p) cp[ci[p] + 1]++;
  for (int32_t j = 0; j < n; ++j) cp[j + 1] += cp[j];
  int64_t *fill = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)n);
  for (int32_t j = 0; j < n; ++j) fill[j] = cp[j];
  for (int32_t i = 0; i < n; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t q = fill[ci[p]]++;
      cr[q] = i; cmap[q] = p;
      if (ci[p] == i) diag[i] = val[p];
    }
  free(fill);
  *cp_o = cp; *cr_o = cr; *cmap_o = cmap; *diag_o = diag;
}

static int64_t est_bound(const int64_t *rp, const int32_t *ci, const int64_t *cp, const int32_t *cr, int32_t k,
                         int lower) {
  int64_t bound = 0;
  if (lower) { bound = cp[k + 1] - cp[k]; for (int64_t p = cp[k]; p < cp[k + 1]; ++p) if (cr[p] < k) bound += cp[cr[p] + 1] - cp[cr[p]]; }
  else { bound = rp[k + 1] - rp[k]; for (int64_t p = rp[k]; p < rp[k + 1]; ++p) if (ci[p] < k) bound += rp[ci[p] + 1] - rp[ci[p]]; }
  return bound;
}

/* One estimated set (test/diagnostic export): lower = 1 -> I~_k, 0 -> J~_k, ascending in out
 * (capacity n).  Returns its size, -1 on a bad argument. */
int32_t orc_ilu1_set(int32_t n, const int64_t *rp, const int32_t *ci, const double *val, double tau, int32_t k,
                     int32_t lower, int32_t *out) {
  if (n < 1 || !rp || !ci || !val || !out || k < 0 || k >= n || !(tau >= 0.0)) return -1;
  int64_t *cp, *cmap; int32_t *cr; double *diag;
  est_csc(n, rp, ci, val, &cp, &cr, &cmap, &diag);
  const int64_t bound = est_bound(rp, ci, cp, cr, k, lower);
  int32_t *buf = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(bound > 0 ? bound : 1));
  const int32_t m = est_set(n, rp, ci, val, cp, cr, cmap, diag, k, tau, lower, buf);
  memcpy(out, buf, sizeof(int32_t) * (size_t)m);
  free(buf); free(cp); free(cr); free(cmap); free(diag);
  return m;
}

int32_t orc_ilu1_blocks(int32_t n, const int64_t *rp, const int32_t *ci, const double *val, double tau,
                        int32_t max_size, int32_t *out) {
  if (n < 1 || !rp || !ci || !val || !out || max_size < 1 || !(tau >= 0.0)) return -1;
  const int64_t nnz = rp[n];
  int64_t *cp, *cmap; int32_t *cr; double *diag;
  est_csc(n, rp, ci, val, &cp, &cr, &cmap, &diag);
  /* per step: sorted estimated sets */
  int64_t *Ip = (int64_t *)xcalloc((size_t)n + 1, sizeof(int64_t)), *Jp = (int64_t *)xcalloc((size_t)n + 1, sizeof(int64_t));
  int64_t capI = nnz + n, capJ = nnz + n, usedI = 0, usedJ = 0;
  int32_t *Is = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)capI), *Js = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)capJ);
  int64_t bufcap = 1024;
  int32_t *buf = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)bufcap);
  for (int32_t k = 0; k < n; ++k) {
    for (int side = 0; side < 2; ++side) {
      const int64_t bound = est_bound(rp, ci, cp, cr, k, side == 0);   /* candidate count */
      if (bound > bufcap) { free(buf); bufcap = 2 * bound; buf = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)bufcap); }
      const int32_t m = est_set(n, rp, ci, val, cp, cr, cmap, diag, k, tau, side == 0, buf);
      int64_t *used = side == 0 ? &usedI : &usedJ, *cap = side == 0 ? &capI : &capJ;
      int32_t **S = side == 0 ? &Is : &Js;
      if (*used + m > *cap) {
        *cap = 2 * (*used + m);
        *S = (int32_t *)realloc(*S, sizeof(int32_t) * (size_t)*cap);
      }
      memcpy(*S + *used, buf, sizeof(int32_t) * (size_t)m);
      *used += m;
      (side == 0 ? Ip : Jp)[k + 1] = *used;
    }
  }
  /* greedy block growing */
  char *inI = (char *)xcalloc((size_t)n, 1), *inJ = (char *)xcalloc((size_t)n, 1);
  int32_t *listI = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)n), *listJ = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)n);
  int32_t nb = 0, k0 = 0;
  while (k0 < n) {
    int32_t l = 1, nI = 0, nJ = 0;
    int64_t sc = (Ip[k0 + 1] - Ip[k0]) + (Jp[k0 + 1] - Jp[k0]) + 1;     /* scalar count c' */
    for (int64_t p = Ip[k0]; p < Ip[k0 + 1]; ++p) if (!inI[Is[p]]) { inI[Is[p]] = 1; listI[nI++] = Is[p]; }
    for (int64_t p = Jp[k0]; p < Jp[k0 + 1]; ++p) if (!inJ[Js[p]]) { inJ[Js[p]] = 1; listJ[nJ++] = Js[p]; }
    while (k0 + l < n && l + 1 <= max_size) {
      const int32_t t = k0 + l;
      /* unions with column t's sets, counted outside the grown block [k0, k0+l+1) */
      int64_t r = 0, s = 0;
      for (int32_t x = 0; x < nI; ++x) r += listI[x] > t;
      for (int32_t x = 0; x < nJ; ++x) s += listJ[x] > t;
      for (int64_t p = Ip[t]; p < Ip[t + 1]; ++p) if (!inI[Is[p]] && Is[p] > t) r++;
      for (int64_t p = Jp[t]; p < Jp[t + 1]; ++p) if (!inJ[Js[p]] && Js[p] > t) s++;
      const int64_t l1 = l + 1;
      const int64_t f = (r + s + l1) * l1;
      const int64_t c2 = sc + (Ip[t + 1] - Ip[t]) + (Jp[t + 1] - Jp[t]) + 1;
      if (!(3 * f <= 4 * c2 || f <= c2 + 4 * l1)) break;
      sc = c2;
      for (int64_t p = Ip[t]; p < Ip[t + 1]; ++p) if (!inI[Is[p]]) { inI[Is[p]] = 1; listI[nI++] = Is[p]; }
      for (int64_t p = Jp[t]; p < Jp[t + 1]; ++p) if (!inJ[Js[p]]) { inJ[Js[p]] = 1; listJ[nJ++] = Js[p]; }
      ++l;
    }
    for (int32_t x = 0; x < nI; ++x) inI[listI[x]] = 0;
    for (int32_t x = 0; x < nJ; ++x) inJ[listJ[x]] = 0;
    out[nb++] = l;
    k0 += l;
  }
  free(cp); free(cr); free(cmap); free(diag); free(Ip); free(Jp); free(Is); free(Js); free(buf);
  free(inI); free(inJ); free(listI); free(listJ);
  return nb;
}

/* ---------------- cosine-based blocking (Sec. 3.2; R21) ----------------
 * Pattern vectors c_i of the rows of A; rows i, j are grouped when
 *   nz(a_i n a_j)^2 >= tau nz(a_i) nz(a_j)
 * scanning i = 0, 1, ... : an unassigned row i opens a group and takes every unassigned j > i
 * with (A A^T)_ij != 0 that passes the test, in increasing j, until the group has max_size rows
 * (Saad's greedy over the upper triangle of A A^T).  Rows / columns with more
 * than mu + 2 sigma nonzeros (mu = nnz/n, sigma the population standard deviation of the row /
 * column counts) are ignored: an ignored column does not count in nz(.) or in
 * the intersections, an ignored row forms its own group.  The mu + 2 sigma test is evaluated in
 * exact integers: c > mu + 2 sigma  <=>  n c - S1 > 0 and (n c - S1)^2 > 4 (n S2 - S1^2).
 * Output: q (new -> old, groups in the order of their first row, rows ascending inside) and the
 * group sizes; returns the number of groups, -1 on a bad argument. */
static int cos_heavy(int64_t c, int64_t n, int64_t S1, int64_t S2) {
  const __int128 a = (__int128)n * c - S1;
  if (a <= 0) return 0;
  return a * a > (__int128)4 * ((__int128)n * S2 - (__int128)S1 * S1);
}

int32_t orc_cosine_blocks(int32_t n, const int64_t *rp, const int32_t *ci, double tau, int32_t max_size,
                          int32_t *q, int32_t *sizes) {
  if (n < 1 || !rp || !ci || !q || !sizes || max_size < 1 || !(tau >= 0.0)) return -1;
  const int64_t nnz = rp[n];
  int64_t *rc = (int64_t *)xcalloc((size_t)n, sizeof(int64_t)), *cc = (int64_t *)xcalloc((size_t)n, sizeof(int64_t));
  for (int32_t i = 0; i < n; ++i) rc[i] = rp[i + 1] - rp[i];
  for (int64_t p = 0; p < nnz; ++p) cc[ci[p]]++;
  int64_t S1r = 0, S2r = 0, S1c = 0, S2c = 0;
  for (int32_t i = 0; i < n; ++i) { S1r += rc[i]; S2r += rc[i] * rc[i]; S1c += cc[i]; S2c += cc[i] * cc[i]; }
  char *row_ign = (char *)xcalloc((size_t)n, 1), *col_ign = (char *)xcalloc((size_t)n, 1);
  for (int32_t i = 0; i < n; ++i) {
    row_ign[i] = (char)cos_heavy(rc[i], n, S1r, S2r);
    col_ign[i] = (char)cos_heavy(cc[i], n, S1c, S2c);
  }
  /* nz(a_i) over the columns kept; CSC of the kept columns */
  int64_t *nz = (int64_t *)xcalloc((size_t)n, sizeof(int64_t));
  int64_t *cp = (int64_t *)xcalloc((size_t)n + 1, sizeof(int64_t));
  for (int32_t i = 0; i < n; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (!col_ign[ci[p]]) { nz[i]++; cp[ci[p] + 1]++; }
  for (int32_t j = 0; j < n; ++j) cp[j + 1] += cp[j];
  int32_t *cr = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(cp[n] > 0 ? cp[n] : 1));
  int64_t *fill = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)n);
  for (int32_t j = 0; j < n; ++j) fill[j] = cp[j];
  for (int32_t i = 0; i < n; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (!col_ign[ci[p]]) cr[fill[ci[p]]++] = i;          /* rows ascending in each column */
  int32_t *group = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)n);
  for (int32_t i = 0; i < n; ++i) group[i] = -1;
  int64_t *cnt = (int64_t *)xcalloc((size_t)n, sizeof(int64_t));
  int32_t *touched = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)n);
  int32_t nb = 0, pos = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (group[i] >= 0) continue;
    group[i] = nb;
    q[pos++] = i;
    int32_t size = 1;
    if (!row_ign[i] && nz[i] > 0) {
      /* nz(a_i n a_j) for every j > i sharing a kept column: row i of A A^T */
      int32_t nt = 0;
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int32_t c = ci[p];
        if (col_ign[c]) continue;
        for (int64_t x = cp[c]; x < cp[c + 1]; ++x) {
          const int32_t j = cr[x];
          if (j <= i) continue;
          if (cnt[j] == 0) touched[nt++] = j;
          cnt[j]++;
        }
      }
      qsort(touched, (size_t)nt, sizeof(int32_t), cmp_int);
      for (int32_t t = 0; t < nt; ++t) {
        const int32_t j = touched[t];
        const int64_t c = cnt[j];
        cnt[j] = 0;
        if (size >= max_size || group[j] >= 0 || row_ign[j]) continue;
        if ((double)c * (double)c >= tau * ((double)nz[i] * (double)nz[j])) {
          group[j] = nb;
          q[pos++] = j;
          size++;
        }
      }
    }
    sizes[nb++] = size;
  }
  free(rc); free(cc); free(row_ign); free(col_ign); free(nz); free(cp); free(cr); free(fill); free(group);
  free(cnt); free(touched);
  return nb;
}

/* ---------------- maximum weight matching + scaling (Sec. 3.1; R22) ----------------
 * Maximum product transversal: a permutation sigma maximising prod_i |a_{i,sigma(i)}|, i.e.
 * minimising sum_i c_{i,sigma(i)} with c_ij = log(cmax_j) - log|a_ij| >= 0 (cmax_j the largest
 * |a_ij| of column j; MC64's normalisation), over the stored nonzeros only.
 * Solved by the textbook O(n^3) Hungarian method with potentials u (rows), v (columns) on the
 * dense cost matrix (missing entries excluded); at the optimum u_i + v_j <= c_ij with equality
 * on the matching, so with D_l = diag(exp(u_i)) and D_r = diag(exp(v_j) / cmax_j)
 *   |(D_l A D_r)_ij| <= 1 and |(D_l A D_r)_{i,sigma(i)}| = 1,
 * and A^ = D_l A D_r Pi has the matched entries on its diagonal (Pi maps column sigma(i) to i).
 * Test infrastructure for small n (dense O(n^2) memory).  sigma[i] = column matched to row i.
 * Returns 0, -1 on a bad argument, -2 if A is structurally singular (no perfect matching). */
int orc_mwm(int32_t n, const int64_t *rp, const int32_t *ci, const double *val, int32_t *sigma, double *dl,
            double *dr) {
  if (n < 1 || n > 8192 || !rp || !ci || !val || !sigma || !dl || !dr) return -1;
  const double INF = HUGE_VAL;
  double *cmax = (double *)xcalloc((size_t)n, sizeof(double));
  for (int32_t i = 0; i < n; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (fabs(val[p]) > cmax[ci[p]]) cmax[ci[p]] = fabs(val[p]);
  /* dense costs, 1-based as in the textbook statement: c[i][j], i, j = 1..n */
  double *c = (double *)xmalloc(sizeof(double) * (size_t)(n + 1) * (size_t)(n + 1));
  for (size_t x = 0; x < (size_t)(n + 1) * (size_t)(n + 1); ++x) c[x] = INF;
  for (int32_t i = 0; i < n; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (val[p] != 0.0) c[(size_t)(i + 1) * (n + 1) + ci[p] + 1] = log(cmax[ci[p]]) - log(fabs(val[p]));
  double *u = (double *)xcalloc((size_t)n + 1, sizeof(double)), *v = (double *)xcalloc((size_t)n + 1, sizeof(double));
  double *minv = (double *)xmalloc(sizeof(double) * (size_t)(n + 1));
  int32_t *p = (int32_t *)xcalloc((size_t)n + 1, sizeof(int32_t)), *way = (int32_t *)xcalloc((size_t)n + 1, sizeof(int32_t));
  char *used = (char *)xmalloc((size_t)n + 1);
  int rc = 0;
  for (int32_t i = 1; i <= n && rc == 0; ++i) {
    p[0] = i;
    int32_t j0 = 0;
    for (int32_t j = 0; j <= n; ++j) { minv[j] = INF; used[j] = 0; }
    do {
      used[j0] = 1;
      const int32_t i0 = p[j0];
      double delta = INF;
      int32_t j1 = -1;
      for (int32_t j = 1; j <= n; ++j) {
        if (used[j]) continue;
        const double cij = c[(size_t)i0 * (n + 1) + j];
        if (cij < INF) {
          const double cur = cij - u[i0] - v[j];
          if (cur < minv[j]) { minv[j] = cur; way[j] = j0; }
        }
        if (minv[j] < delta) { delta = minv[j]; j1 = j; }
      }
      if (j1 < 0) { rc = -2; break; }                       /* no augmenting path */
      for (int32_t j = 0; j <= n; ++j) {
        if (used[j]) { u[p[j]] += delta; v[j] -= delta; }
        else minv[j] -= delta;
      }
      j0 = j1;
    } while (p[j0] != 0);
    if (rc) break;
    do {
      const int32_t j1 = way[j0];
      p[j0] = p[j1];
      j0 = j1;
    } while (j0);
  }
  if (rc == 0) {
    for (int32_t j = 1; j <= n; ++j) sigma[p[j] - 1] = j - 1;
    for (int32_t i = 0; i < n; ++i) dl[i] = exp(u[i + 1]);
    for (int32_t j = 0; j < n; ++j) dr[j] = exp(v[j + 1]) / cmax[j];
  }
  free(cmax); free(c); free(u); free(v); free(minv); free(p); free(way); free(used);
  return rc;
}
