// bilu_factor.cu -- sm_100a numeric phase of the Crout-type block ILU.
//
// One persistent, dataflow-scheduled kernel (`factor_kernel`): every CTA pops a
// ready block K from a device queue and computes block column K of L, block
// row K of U and D_K = P_K^{-1} (Alg. 1 generalised to blocks,
// PAPER.md:205-228, 361-374, 767-799):
//   a-2  contributor lists      (replace L_head/L_list/L_first)
//   a-3  candidate row/col sets (sorted unions, CTA bitonic sort)
//   a-4  scatter of Ã's block column / block row into the dense buffers
//        ("load the associated scalar sparse columns of A into block column
//        buffer")
//   a-5  Schur updates W -= L_J Ũ_J: gather -> dense product -> scatter
//        (Fig. 2); operands are contiguous slices of the
//        hybrid panels, staged in shared memory
//   a-6  pivot block inverse, Gauss-Jordan with partial pivoting inside the block
//        (PAPER.md:788-794), warp argmax pivot search
//   a-7/8 scaling l_i = w_i D_K, u_j = D_K z_j, tau-dropping (PAPER.md:167, 173,
//        209-212) and compaction into the factor arenas
//   a-1  release of the blocks that depend on K (dataflow "chain" rule)
// Readiness rule: K may start once every block M < K
// that is adjacent to K in the block graph of Ã, or that precedes K in the
// sorted neighbour set N(J) of a finished block J, is finished.
#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>

#include "bilu_internal.h"

namespace bilu {

constexpr int NT = 256;
constexpr int NW = NT / 32;

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ int ld_vol(const int *p) { return *(const volatile int *)p; }
__device__ __forceinline__ unsigned long long ld_vol64(const unsigned long long *p) {
  return *(const volatile unsigned long long *)p;
}
__device__ __forceinline__ void st_vol(int *p, int v) { *(volatile int *)p = v; }

__device__ __forceinline__ void raise_abort(const DevFactor &F, int code, int blk) {
  if (atomicCAS(&F.ctrl[CTRL_ABORT], 0ull, (unsigned long long)code) == 0ull)
    atomicExch(&F.ctrl[CTRL_ERRBLK], (unsigned long long)blk);
}
__device__ __forceinline__ bool aborted(const DevFactor &F) { return ld_vol64(&F.ctrl[CTRL_ABORT]) != 0ull; }

// first position p in a[lo, hi) with a[p] >= key
__device__ __forceinline__ int lbound(const int *a, int lo, int hi, int key) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int lbound_cg(const int *a, int lo, int hi, int key) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__ldcg(a + mid) < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// exclusive scan of a[0..n) in place (any memory), returns the total. CTA-wide.
__device__ int cta_scan(int *a, int n, int *s_tmp /* >= NW+1 ints */) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (n + NT - 1) / NT;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int sum = 0;
  for (int i = lo; i < hi; ++i) sum += a[i];
  int x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_tmp[wid] = x;
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int w = 0; w < NW; ++w) { int t = s_tmp[w]; s_tmp[w] = acc; acc += t; }
    s_tmp[NW] = acc;
  }
  __syncthreads();
  int run = s_tmp[wid] + x - sum;
  for (int i = lo; i < hi; ++i) { int t = a[i]; a[i] = run; run += t; }
  int total = s_tmp[NW];
  __syncthreads();
  return total;
}

// CTA bitonic sort of a[0..m), m a power of two.
__device__ void cta_bitonic(int *a, int m) {
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < m; i += NT) {
        int ixj = i ^ j;
        if (ixj > i) {
          int x = a[i], y = a[ixj];
          bool up = (i & k) == 0;
          if ((x > y) == up) { a[i] = y; a[ixj] = x; }
        }
      }
      __syncthreads();
    }
  }
}

// sort a[0..n) (buffer capacity >= next pow2), drop duplicates and INT_MAX padding,
// compact in place; returns the number of distinct values.  CTA-wide.
__device__ int cta_sort_unique(int *a, int n, int *flags, int *s_tmp) {
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = n + threadIdx.x; i < m; i += NT) a[i] = INT_MAX;
  __syncthreads();
  if (m > 1) cta_bitonic(a, m);
  for (int i = threadIdx.x; i < n; i += NT) flags[i] = (i == 0 || a[i] != a[i - 1]) ? 1 : 0;
  __syncthreads();
  int total = cta_scan(flags, n, s_tmp);
  // in-place compaction, chunk by chunk (writes never pass unread elements);
  // "first of its run" is read off the scanned flags, not the (overwritten) values
  for (int base = 0; base < n; base += NT) {
    int i = base + threadIdx.x;
    int v = 0, pos = -1;
    if (i < n) {
      v = a[i];
      int nxt = (i + 1 < n) ? flags[i + 1] : total;
      if (nxt > flags[i]) pos = flags[i];
    }
    __syncthreads();
    if (pos >= 0) a[pos] = v;
    __syncthreads();
  }
  return total;
}

// ------------------------------------------------------------- chunked lists
__device__ __forceinline__ const int *list_rec(const ChunkList &L, int T, int idx) {
  int id = __ldcg(&L.dir[(size_t)T * DIR_SLOTS + idx / CHUNK]);
  return L.pool + ((size_t)id * CHUNK + (idx % CHUNK)) * L.rec_ints;
}

__device__ bool list_append(const DevFactor &F, const ChunkList &L, int T, const int *rec) {
  int idx = atomicAdd(&L.cnt[T], 1);
  int slot = idx / CHUNK;
  if (slot >= DIR_SLOTS) { raise_abort(F, DEV_OVF_LIST, T); return false; }
  int *dptr = &L.dir[(size_t)T * DIR_SLOTS + slot];
  int id;
  if (idx % CHUNK == 0) {
    unsigned long long c = atomicAdd(&F.ctrl[L.ctrl_cursor], 1ull);
    if (c >= (unsigned long long)L.pool_cap) {
      atomicExch(dptr, -2);
      raise_abort(F, DEV_OVF_POOL, T);
      return false;
    }
    id = (int)c;
    __threadfence();
    atomicExch(dptr, id);
  } else {
    while ((id = ld_vol(dptr)) == -1) {
      if (aborted(F)) return false;
      __nanosleep(20);
    }
    if (id < 0) return false;
  }
  int *dst = L.pool + ((size_t)id * CHUNK + (idx % CHUNK)) * L.rec_ints;
  for (int i = 0; i < L.rec_ints; ++i) dst[i] = rec[i];
  return true;
}

// ------------------------------------------------------ per-block allocator
struct Bump {
  unsigned char *sbase; int sused, scap;
  double *gbase; int64_t gused, gcap;
  bool ovf;
};
__device__ __forceinline__ void *balloc(Bump &A, int64_t bytes) {
  bytes = (bytes + 15) & ~int64_t(15);
  if (A.sused + bytes <= A.scap) {
    void *p = A.sbase + A.sused;
    A.sused += (int)bytes;
    return p;
  }
  int64_t d = bytes / 8;
  if (A.gused + d <= A.gcap) {
    void *p = A.gbase + A.gused;
    A.gused += d;
    return p;
  }
  A.ovf = true;
  return A.gbase;  // caller checks ovf
}

// --------------------------------------------------------------- the kernel
struct Shared {
  int K;
  int misc[8];
  int tmp[NW + 1];
  int piv;
  double pivd;
  unsigned long long off[4];
};

__device__ void process_block(const DevFactor &F, int K, Shared &S, unsigned char *smem) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int s = F.bstart[K], e = F.bstart[K + 1], b = e - s;
  Bump A;
  A.sbase = smem; A.sused = 0; A.scap = F.smem_bytes;
  A.gbase = F.work + (size_t)blockIdx.x * F.work_per_cta; A.gused = 0; A.gcap = F.work_per_cta;
  A.ovf = false;
  double flops = 0.0;

  // ---------------- a-2: contributor lists (Lc: J with Ũ cols in K; Uc: J with L rows in K)
  const int nLc = __ldcg(&F.lc.cnt[K]);
  const int nUc = __ldcg(&F.uc.cnt[K]);
  int *lrec = (int *)balloc(A, (int64_t)nLc * REC_INTS * 4);
  int *urec = (int *)balloc(A, (int64_t)nUc * REC_INTS * 4);
  int mL = 1; while (mL < nLc) mL <<= 1;
  int mU = 1; while (mU < nUc) mU <<= 1;
  int *lkey = (int *)balloc(A, (int64_t)mL * 4);
  int *ukey = (int *)balloc(A, (int64_t)mU * 4);
  if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; }
  for (int i = tid; i < nLc * REC_INTS; i += NT) {
    const int *r = list_rec(F.lc, K, i / REC_INTS);
    lrec[i] = __ldcg(r + (i % REC_INTS));
  }
  for (int i = tid; i < nUc * REC_INTS; i += NT) {
    const int *r = list_rec(F.uc, K, i / REC_INTS);
    urec[i] = __ldcg(r + (i % REC_INTS));
  }
  __syncthreads();
  // deterministic ascending-J order (R13): key = J << 10 | record index
  for (int i = tid; i < mL; i += NT) lkey[i] = i < nLc ? (lrec[i * REC_INTS] << 10) | i : INT_MAX;
  for (int i = tid; i < mU; i += NT) ukey[i] = i < nUc ? (urec[i * REC_INTS] << 10) | i : INT_MAX;
  __syncthreads();
  if (mL > 1) cta_bitonic(lkey, mL);
  if (mU > 1) cta_bitonic(ukey, mU);

  // ---------------- a-3: candidate rows R_K (>= e) and columns C_K (>= e)
  // item counts: b columns of Ã + nLc contributors (rows), b rows of Ã + nUc (cols)
  int *rcnt = (int *)balloc(A, (int64_t)(b + nLc + 1) * 4);
  int *ccnt = (int *)balloc(A, (int64_t)(b + nUc + 1) * 4);
  if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; }
  for (int i = tid; i < b + nLc; i += NT) {
    if (i < b) {
      int c = s + i;
      int64_t lo = F.cp[c], hi = F.cp[c + 1];
      int64_t p = lo, q = hi;  // first entry with row >= e
      while (p < q) { int64_t mid = (p + q) >> 1; if (F.cr[mid] < e) p = mid + 1; else q = mid; }
      rcnt[i] = (int)(hi - p);
    } else {
      const int *r = lrec + (i - b) * REC_INTS;
      int J = r[0];
      rcnt[i] = __ldcg(&F.Lm[J]) - r[4];
    }
  }
  for (int i = tid; i < b + nUc; i += NT) {
    if (i < b) {
      int rr = s + i;
      int64_t lo = F.rp[rr], hi = F.rp[rr + 1];
      int64_t p = lo, q = hi;
      while (p < q) { int64_t mid = (p + q) >> 1; if (F.ci[mid] < e) p = mid + 1; else q = mid; }
      ccnt[i] = (int)(hi - p);
    } else {
      const int *r = urec + (i - b) * REC_INTS;
      int J = r[0];
      ccnt[i] = __ldcg(&F.Uc[J]) - r[3];
    }
  }
  __syncthreads();
  const int totR = cta_scan(rcnt, b + nLc, S.tmp);
  const int totC = cta_scan(ccnt, b + nUc, S.tmp);
  // candidate buffers (+flags), power-of-two capacity
  int pR = 1; while (pR < totR) pR <<= 1;
  int pC = 1; while (pC < totC) pC <<= 1;
  const int saved = A.sused; const int64_t gsaved = A.gused;
  int *candR = (int *)balloc(A, (int64_t)pR * 4);
  int *flagR = (int *)balloc(A, (int64_t)pR * 4);
  if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; }
  // warp per item copy
  for (int it = wid; it < b + nLc; it += NW) {
    int off = rcnt[it];
    if (it < b) {
      int c = s + it;
      int64_t hi = F.cp[c + 1];
      int n_it = (it + 1 < b + nLc ? rcnt[it + 1] : totR) - off;
      int64_t lo = hi - n_it;
      for (int64_t p = lo + lane; p < hi; p += 32) candR[off + (p - lo)] = F.cr[p];
    } else {
      const int *r = lrec + (it - b) * REC_INTS;
      int J = r[0];
      int n_it = (it + 1 < b + nLc ? rcnt[it + 1] : totR) - off;
      const int *rows = F.Lidx + __ldcg(&F.Lrow_off[J]) + r[4];
      for (int p = lane; p < n_it; p += 32) candR[off + p] = __ldcg(rows + p);
    }
  }
  __syncthreads();
  const int nR = cta_sort_unique(candR, totR, flagR, S.tmp);
  // release the temporary part of the allocation, keep R (same address unless
  // the candidates spilled to global memory and R now fits in shared memory)
  A.sused = saved; A.gused = gsaved;
  int *R = (int *)balloc(A, (int64_t)nR * 4);
  if (R != candR) {
    for (int i = threadIdx.x; i < nR; i += NT) R[i] = candR[i];
    __syncthreads();
  }
  const int saved2 = A.sused; const int64_t gsaved2 = A.gused;
  int *candC = (int *)balloc(A, (int64_t)pC * 4);
  int *flagC = (int *)balloc(A, (int64_t)pC * 4);
  if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; }
  for (int it = wid; it < b + nUc; it += NW) {
    int off = ccnt[it];
    int n_it = (it + 1 < b + nUc ? ccnt[it + 1] : totC) - off;
    if (it < b) {
      int rr = s + it;
      int64_t hi = F.rp[rr + 1];
      int64_t lo = hi - n_it;
      for (int64_t p = lo + lane; p < hi; p += 32) candC[off + (p - lo)] = F.ci[p];
    } else {
      const int *r = urec + (it - b) * REC_INTS;
      int J = r[0];
      const int *cols = F.Uidx + __ldcg(&F.Ucol_off[J]) + r[3];
      for (int p = lane; p < n_it; p += 32) candC[off + p] = __ldcg(cols + p);
    }
  }
  __syncthreads();
  const int nC = cta_sort_unique(candC, totC, flagC, S.tmp);
  A.sused = saved2; A.gused = gsaved2;
  int *C = (int *)balloc(A, (int64_t)nC * 4);
  if (C != candC) {
    for (int i = threadIdx.x; i < nC; i += NT) C[i] = candC[i];
    __syncthreads();
  }

  // ---------------- a-4: dense buffers, scatter Ã
  // W_L: (b + nR) x b row-major (rows: the b diagonal rows, then R);  W_U: nC x b (column j contiguous)
  double *WL = (double *)balloc(A, (int64_t)(b + nR) * b * 8);
  double *WU = (double *)balloc(A, (int64_t)nC * b * 8);
  double *P = (double *)balloc(A, (int64_t)b * b * 8);
  int *keepR = (int *)balloc(A, (int64_t)(nR + 1) * 4);
  int *keepC = (int *)balloc(A, (int64_t)(nC + 1) * 4);
  if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; }
  for (int i = tid; i < (b + nR) * b; i += NT) WL[i] = 0.0;
  for (int i = tid; i < nC * b; i += NT) WU[i] = 0.0;
  __syncthreads();
  for (int it = wid; it < b; it += NW) {
    int c = s + it;
    int64_t lo = F.cp[c], hi = F.cp[c + 1];
    for (int64_t p = lo + lane; p < hi; p += 32) {
      int row = F.cr[p];
      if (row < s) continue;
      int w = row < e ? row - s : b + lbound(R, 0, nR, row);
      WL[(int64_t)w * b + it] = F.cval[p];
    }
    int rr = s + it;
    lo = F.rp[rr]; hi = F.rp[rr + 1];
    for (int64_t p = lo + lane; p < hi; p += 32) {
      int col = F.ci[p];
      if (col < e) continue;
      WU[(int64_t)lbound(C, 0, nC, col) * b + it] = F.val[p];
    }
  }
  __syncthreads();

  // ---------------- a-5: Schur updates, L side (and diagonal block)
  //   W_L[rows(L_J) >= s, cols(Ũ_J) in K] -= L_J[rows >= s, :] * Ũ_J[:, cols in K]
  const int mark = A.sused; const int64_t gmark = A.gused;
  for (int a = 0; a < nLc; ++a) {
    const int *r = lrec + (lkey[a] & 1023) * REC_INTS;
    const int J = r[0], c0 = r[1], c1 = r[2], lrs = r[3];
    const int bJ = F.bstart[J + 1] - F.bstart[J];
    const int mJ = __ldcg(&F.Lm[J]);
    const int nrow = mJ - lrs, ncol = c1 - c0;
    if (nrow <= 0 || ncol <= 0) continue;
    A.sused = mark; A.gused = gmark;
    double *sL = (double *)balloc(A, (int64_t)nrow * bJ * 8);
    double *sU = (double *)balloc(A, (int64_t)ncol * bJ * 8);
    int *wrow = (int *)balloc(A, (int64_t)nrow * 4);
    int *wcol = (int *)balloc(A, (int64_t)ncol * 4);
    if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; }
    const double *gL = F.Lval + __ldcg(&F.Lval_off[J]) + (int64_t)lrs * bJ;
    const double *gU = F.Uval + __ldcg(&F.Uval_off[J]) + (int64_t)c0 * bJ;
    const int *grow = F.Lidx + __ldcg(&F.Lrow_off[J]) + lrs;
    const int *gcol = F.Uidx + __ldcg(&F.Ucol_off[J]) + c0;
    for (int i = tid; i < nrow * bJ; i += NT) sL[i] = __ldcg(gL + i);
    for (int i = tid; i < ncol * bJ; i += NT) sU[i] = __ldcg(gU + i);
    for (int i = tid; i < nrow; i += NT) {
      int row = __ldcg(grow + i);
      wrow[i] = row < e ? row - s : b + lbound(R, 0, nR, row);
    }
    for (int i = tid; i < ncol; i += NT) wcol[i] = __ldcg(gcol + i) - s;
    __syncthreads();
    for (int it = tid; it < nrow * ncol; it += NT) {
      int p = it / ncol, q = it - p * ncol;
      const double *l = sL + (int64_t)p * bJ, *u = sU + (int64_t)q * bJ;
      double acc = 0.0;
      for (int t = 0; t < bJ; ++t) acc = fma(l[t], u[t], acc);
      WL[(int64_t)wrow[p] * b + wcol[q]] -= acc;
    }
    flops += 2.0 * bJ * (double)nrow * (double)ncol;
    __syncthreads();
  }
  // ---------------- a-5: Schur updates, U side
  //   W_U[rows(L_J) in K, cols(Ũ_J) >= e] -= L_J[rows in K, :] * Ũ_J[:, cols >= e]
  for (int a = 0; a < nUc; ++a) {
    const int *r = urec + (ukey[a] & 1023) * REC_INTS;
    const int J = r[0], r0 = r[1], r1 = r[2], cus = r[3];
    const int bJ = F.bstart[J + 1] - F.bstart[J];
    const int cJ = __ldcg(&F.Uc[J]);
    const int nrow = r1 - r0, ncol = cJ - cus;
    if (nrow <= 0 || ncol <= 0) continue;
    A.sused = mark; A.gused = gmark;
    double *sL = (double *)balloc(A, (int64_t)nrow * bJ * 8);
    double *sU = (double *)balloc(A, (int64_t)ncol * bJ * 8);
    int *wrow = (int *)balloc(A, (int64_t)nrow * 4);
    int *wcol = (int *)balloc(A, (int64_t)ncol * 4);
    if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; }
    const double *gL = F.Lval + __ldcg(&F.Lval_off[J]) + (int64_t)r0 * bJ;
    const double *gU = F.Uval + __ldcg(&F.Uval_off[J]) + (int64_t)cus * bJ;
    const int *grow = F.Lidx + __ldcg(&F.Lrow_off[J]) + r0;
    const int *gcol = F.Uidx + __ldcg(&F.Ucol_off[J]) + cus;
    for (int i = tid; i < nrow * bJ; i += NT) sL[i] = __ldcg(gL + i);
    for (int i = tid; i < ncol * bJ; i += NT) sU[i] = __ldcg(gU + i);
    for (int i = tid; i < nrow; i += NT) wrow[i] = __ldcg(grow + i) - s;
    for (int i = tid; i < ncol; i += NT) wcol[i] = lbound(C, 0, nC, __ldcg(gcol + i));
    __syncthreads();
    for (int it = tid; it < nrow * ncol; it += NT) {
      int q = it / nrow, p = it - q * nrow;
      const double *l = sL + (int64_t)p * bJ, *u = sU + (int64_t)q * bJ;
      double acc = 0.0;
      for (int t = 0; t < bJ; ++t) acc = fma(l[t], u[t], acc);
      WU[(int64_t)wcol[q] * b + wrow[p]] -= acc;
    }
    flops += 2.0 * bJ * (double)nrow * (double)ncol;
    __syncthreads();
  }
  A.sused = mark; A.gused = gmark;

  // ---------------- a-6: D_K = P_K^{-1}, Gauss-Jordan with partial pivoting (column-major P)
  for (int i = tid; i < b * b; i += NT) {
    int rr = i % b, cc = i / b;
    P[i] = WL[(int64_t)rr * b + cc];
  }
  int *ipiv = (int *)balloc(A, (int64_t)b * 4);
  double *fcol = (double *)balloc(A, (int64_t)b * 8);
  if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; }
  __syncthreads();
  bool singular = false;
  for (int k = 0; k < b; ++k) {
    if (wid == 0) {
      double best = -1.0; int bi = k;
      for (int i = k + lane; i < b; i += 32) {
        double v = fabs(P[i + (int64_t)k * b]);
        if (v > best) { best = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ob = __shfl_down_sync(0xffffffffu, best, o);
        int oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) { S.piv = bi; S.pivd = best; ipiv[k] = bi; }
    }
    __syncthreads();
    if (S.pivd == 0.0) { singular = true; break; }
    const int pv = S.piv;
    if (pv != k)
      for (int j = tid; j < b; j += NT) {
        double t = P[k + (int64_t)j * b]; P[k + (int64_t)j * b] = P[pv + (int64_t)j * b]; P[pv + (int64_t)j * b] = t;
      }
    __syncthreads();
    const double d = 1.0 / P[k + (int64_t)k * b];
    __syncthreads();
    if (tid == 0) P[k + (int64_t)k * b] = 1.0;
    __syncthreads();
    for (int j = tid; j < b; j += NT) P[k + (int64_t)j * b] *= d;
    for (int i = tid; i < b; i += NT) fcol[i] = (i == k) ? 0.0 : P[i + (int64_t)k * b];
    __syncthreads();
    for (int it = tid; it < b * b; it += NT) {
      int i = it % b, j = it / b;
      if (i == k) continue;
      double base = (j == k) ? 0.0 : P[i + (int64_t)j * b];
      P[i + (int64_t)j * b] = base - fcol[i] * P[k + (int64_t)j * b];
    }
    __syncthreads();
  }
  if (singular) {
    if (tid == 0) raise_abort(F, DEV_BREAKDOWN, K);
    return;
  }
  // undo the row interchanges as column interchanges, in reverse order
  for (int k = b - 1; k >= 0; --k) {
    int pv = ipiv[k];
    if (pv != k)
      for (int i = tid; i < b; i += NT) {
        double t = P[i + (int64_t)k * b]; P[i + (int64_t)k * b] = P[i + (int64_t)pv * b]; P[i + (int64_t)pv * b] = t;
      }
    __syncthreads();
  }
  {
    double *Dg = F.D + F.D_off[K];
    for (int i = tid; i < b * b; i += NT) Dg[i] = P[i];
  }
  flops += 2.0 * b * b * (double)b + 2.0 * b * b * (double)(nR + nC);

  // ---------------- a-7/a-8: scale, drop, compact -- L rows
  const double tau = F.tau;
  for (int i = tid; i < nR; i += NT) {
    const double *w = WL + (int64_t)(b + i) * b;
    double mx = 0.0;
    for (int c = 0; c < b; ++c) {
      double acc = 0.0;
      for (int t = 0; t < b; ++t) acc = fma(w[t], P[t + (int64_t)c * b], acc);
      mx = fmax(mx, fabs(acc));
    }
    int keep = mx > tau;
    keepR[i] = keep;
    if (tau > 0.0) {
      double margin = fabs(mx / tau - 1.0);
      if (margin <= F.near_rel) {
        unsigned long long slot = atomicAdd(&F.ctrl[CTRL_NEAR], 1ull);
        if (slot < (unsigned long long)F.near_cap) {
          F.near_i[4 * slot] = K; F.near_i[4 * slot + 1] = 0;
          F.near_i[4 * slot + 2] = R[i]; F.near_i[4 * slot + 3] = keep;
          F.near_m[slot] = margin;
        }
      }
    }
  }
  for (int j = tid; j < nC; j += NT) {
    const double *z = WU + (int64_t)j * b;
    double mx = 0.0;
    for (int rr = 0; rr < b; ++rr) {
      double acc = 0.0;
      for (int t = 0; t < b; ++t) acc = fma(P[rr + (int64_t)t * b], z[t], acc);
      mx = fmax(mx, fabs(acc));
    }
    int keep = mx > tau;
    keepC[j] = keep;
    if (tau > 0.0) {
      double margin = fabs(mx / tau - 1.0);
      if (margin <= F.near_rel) {
        unsigned long long slot = atomicAdd(&F.ctrl[CTRL_NEAR], 1ull);
        if (slot < (unsigned long long)F.near_cap) {
          F.near_i[4 * slot] = K; F.near_i[4 * slot + 1] = 1;
          F.near_i[4 * slot + 2] = C[j]; F.near_i[4 * slot + 3] = keep;
          F.near_m[slot] = margin;
        }
      }
    }
  }
  __syncthreads();
  const int mK = cta_scan(keepR, nR, S.tmp);   // keepR -> exclusive positions
  const int cK = cta_scan(keepC, nC, S.tmp);
  keepR[nR] = mK;   // sentinel so keep(i) = keepR[i+1] > keepR[i]
  keepC[nC] = cK;
  if (tid == 0) {
    unsigned long long oi = atomicAdd(&F.ctrl[CTRL_CUR_LIDX], (unsigned long long)mK);
    unsigned long long ov = atomicAdd(&F.ctrl[CTRL_CUR_LVAL], (unsigned long long)mK * b);
    unsigned long long ui = atomicAdd(&F.ctrl[CTRL_CUR_UIDX], (unsigned long long)cK);
    unsigned long long uv = atomicAdd(&F.ctrl[CTRL_CUR_UVAL], (unsigned long long)cK * b);
    S.off[0] = oi; S.off[1] = ov; S.off[2] = ui; S.off[3] = uv;
    atomicAdd(&F.ctrl[CTRL_NDEC], (unsigned long long)(nR + nC));
  }
  __syncthreads();
  if (S.off[0] + mK > (unsigned long long)F.cap_Lidx || S.off[1] + (unsigned long long)mK * b > (unsigned long long)F.cap_Lval ||
      S.off[2] + cK > (unsigned long long)F.cap_Uidx || S.off[3] + (unsigned long long)cK * b > (unsigned long long)F.cap_Uval) {
    if (tid == 0) raise_abort(F, DEV_OVF_ARENA, K);
    return;
  }
  const int64_t oLi = (int64_t)S.off[0], oLv = (int64_t)S.off[1], oUi = (int64_t)S.off[2], oUv = (int64_t)S.off[3];
  // kept row/col lists in shared memory for registration (R / C compacted in place)
  for (int i = tid; i < nR; i += NT)
    if (keepR[i + 1] > keepR[i]) F.Lidx[oLi + keepR[i]] = R[i];
  for (int it = tid; it < nR * b; it += NT) {
    int i = it / b, c = it - i * b;
    if (keepR[i + 1] > keepR[i]) {
      const double *w = WL + (int64_t)(b + i) * b;
      double acc = 0.0;
      for (int t = 0; t < b; ++t) acc = fma(w[t], P[t + (int64_t)c * b], acc);
      F.Lval[oLv + (int64_t)keepR[i] * b + c] = acc;
    }
  }
  for (int j = tid; j < nC; j += NT)
    if (keepC[j + 1] > keepC[j]) F.Uidx[oUi + keepC[j]] = C[j];
  for (int it = tid; it < nC * b; it += NT) {
    int j = it / b;
    if (keepC[j + 1] > keepC[j]) F.Uval[oUv + (int64_t)keepC[j] * b + (it - j * b)] = WU[it];
  }
  __syncthreads();
  // compact R -> kept rows, C -> kept cols (chunked in place)
  for (int base = 0; base < nR; base += NT) {
    int i = base + tid; int v = 0, pos = -1;
    if (i < nR && keepR[i + 1] > keepR[i]) { v = R[i]; pos = keepR[i]; }
    __syncthreads();
    if (pos >= 0) R[pos] = v;
    __syncthreads();
  }
  for (int base = 0; base < nC; base += NT) {
    int j = base + tid; int v = 0, pos = -1;
    if (j < nC && keepC[j + 1] > keepC[j]) { v = C[j]; pos = keepC[j]; }
    __syncthreads();
    if (pos >= 0) C[pos] = v;
    __syncthreads();
  }
  if (tid == 0) {
    F.Lrow_off[K] = oLi; F.Lm[K] = mK; F.Lval_off[K] = oLv;
    F.Ucol_off[K] = oUi; F.Uc[K] = cK; F.Uval_off[K] = oUv;
    F.blk_ncand[2 * K] = nR; F.blk_ncand[2 * K + 1] = nC;
  }

  // ---------------- a-2 (producer side): register K with the blocks it feeds,
  // and the chain edges of the readiness rule.
  // run starts of kept rows / cols by target block
  int *rrun = keepR;  // reuse: run flags -> positions
  int *crun = keepC;
  for (int i = tid; i < mK; i += NT) rrun[i] = (i == 0 || F.block_of[R[i]] != F.block_of[R[i - 1]]) ? 1 : 0;
  for (int j = tid; j < cK; j += NT) crun[j] = (j == 0 || F.block_of[C[j]] != F.block_of[C[j - 1]]) ? 1 : 0;
  __syncthreads();
  const int nRr = cta_scan(rrun, mK, S.tmp);
  const int nCr = cta_scan(crun, cK, S.tmp);
  int *rstart = (int *)balloc(A, (int64_t)(nRr + 1) * 4);
  int *cstart = (int *)balloc(A, (int64_t)(nCr + 1) * 4);
  int pN = 1; while (pN < nRr + nCr) pN <<= 1;
  int *nb = (int *)balloc(A, (int64_t)pN * 4);
  int *nbf = (int *)balloc(A, (int64_t)pN * 4);
  if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; }
  for (int i = tid; i < mK; i += NT) {
    bool st = (i == 0) || F.block_of[R[i]] != F.block_of[R[i - 1]];
    if (st) rstart[rrun[i]] = i;
  }
  for (int j = tid; j < cK; j += NT) {
    bool st = (j == 0) || F.block_of[C[j]] != F.block_of[C[j - 1]];
    if (st) cstart[crun[j]] = j;
  }
  if (tid == 0) { rstart[nRr] = mK; cstart[nCr] = cK; }
  __syncthreads();
  for (int x = tid; x < nRr; x += NT) {
    const int r0 = rstart[x], r1 = rstart[x + 1];
    const int T = F.block_of[R[r0]];
    int rec[REC_INTS] = {K, r0, r1, lbound(C, 0, cK, F.bstart[T + 1]), 0, 0, 0, 0};
    list_append(F, F.uc, T, rec);
    nb[x] = T;
  }
  for (int x = tid; x < nCr; x += NT) {
    const int c0 = cstart[x], c1 = cstart[x + 1];
    const int T = F.block_of[C[c0]];
    int rec[REC_INTS] = {K, c0, c1, lbound(R, 0, mK, F.bstart[T]), lbound(R, 0, mK, F.bstart[T + 1]), 0, 0, 0};
    list_append(F, F.lc, T, rec);
    nb[nRr + x] = T;
  }
  __syncthreads();
  const int nN = cta_sort_unique(nb, nRr + nCr, nbf, S.tmp);
  // chain edges n_i -> n_{i+1}: n_{i+1} additionally waits for n_i
  for (int x = tid; x + 1 < nN; x += NT) {
    atomicAdd(&F.pending[nb[x + 1]], 1);
    int rec1 = nb[x + 1];
    list_append(F, F.succ, nb[x], &rec1);
  }
  if (tid == 0) { F.blk_flops[K] = flops; atomicAdd((double *)&F.ctrl[CTRL_FLOPS], flops); }
  __threadfence();
  __syncthreads();

  // ---------------- a-1: release successors (static adjacency of Ã + chain edges)
  const int a0 = F.adj_ptr[K], a1 = F.adj_ptr[K + 1];
  const int nS = __ldcg(&F.succ.cnt[K]);
  for (int x = tid; x < (a1 - a0) + nS; x += NT) {
    int T = x < (a1 - a0) ? F.adj[a0 + x] : __ldcg(list_rec(F.succ, K, x - (a1 - a0)));
    if (atomicSub(&F.pending[T], 1) == 1) {
      unsigned long long slot = atomicAdd(&F.ctrl[CTRL_QHEAD], 1ull);
      __threadfence();
      st_vol(&F.queue[slot], T);
    }
  }
  if (tid == 0) atomicAdd(&F.ctrl[CTRL_DONE], 1ull);
}

__global__ void __launch_bounds__(NT) factor_kernel(DevFactor F) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Shared S;
  while (true) {
    if (threadIdx.x == 0) {
      int K = -1;
      unsigned long long idx = aborted(F) ? ~0ull : atomicAdd(&F.ctrl[CTRL_QTAIL], 1ull);
      if (idx < (unsigned long long)F.N) {
        while (true) {
          K = ld_vol(&F.queue[idx]);
          if (K >= 0) break;
          if (aborted(F)) { K = -1; break; }
          __nanosleep(32);
        }
      }
      S.K = K;
    }
    __syncthreads();
    const int K = S.K;
    if (K < 0) break;
    __threadfence();
    process_block(F, K, S, smem);
    __syncthreads();
  }
}

// ----------------------------------------------------------------- launchers
extern "C" cudaError_t bilu_launch_factor(const DevFactor &F, int grid, cudaStream_t st) {
  cudaError_t err = cudaFuncSetAttribute(factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, F.smem_bytes);
  if (err != cudaSuccess) return err;
  factor_kernel<<<grid, NT, F.smem_bytes, st>>>(F);
  return cudaGetLastError();
}

extern "C" cudaError_t bilu_factor_occupancy(int smem_bytes, int *blocks_per_sm) {
  cudaError_t err = cudaFuncSetAttribute(factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (err != cudaSuccess) return err;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, factor_kernel, NT, smem_bytes);
}

}  // namespace bilu
