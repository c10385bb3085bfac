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
#include "dgemm_cta.cuh"

namespace bilu {

#ifndef BILU_NT
#define BILU_NT 512
#endif
constexpr int NT = BILU_NT;
constexpr int NW = NT / 32;

// progress markers for the host-side deadlock watchdog (BILU_DEBUG_TIMEOUT)
#define DBGP(i) do { if (threadIdx.x == 0 && F.dbg) { F.dbg[4 * blockIdx.x + 1] = (i); } } while (0)
#define DBGK(k) do { if (threadIdx.x == 0 && F.dbg) { F.dbg[4 * blockIdx.x] = (k); F.dbg[4 * blockIdx.x + 1] = 0; \
  F.dbg[4 * blockIdx.x + 2]++; } } while (0)
#ifdef BILU_PROFILE
__device__ unsigned long long g_prof[32];
__device__ unsigned long long *g_blkprof;   // [N * 16]: t0, t1 (globaltimer ns), phase cycles, sizes
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}
#define PROF_T0 long long _pt = clock64(); if (threadIdx.x == 0 && g_blkprof) g_blkprof[32 * (size_t)K] = gtimer();
#define PROF_T0C long long _pt = clock64();
#define PROF(i) do { DBGP(i); if (threadIdx.x == 0) { long long _n = clock64(); atomicAdd(&g_prof[i], (unsigned long long)(_n - _pt)); \
  if (g_blkprof) g_blkprof[32 * (size_t)K + 1 + (i)] = (unsigned long long)(_n - _pt); _pt = _n; } } while (0)
#define SUBP(i) do { if (threadIdx.x == 0 && g_blkprof) { long long _n2 = clock64(); \
  g_blkprof[32 * (size_t)K + 16 + (i)] += (unsigned long long)(_n2 - _sp); _sp = _n2; } } while (0)
#define SUBP_T0 long long _sp = clock64();
#define PROF_END(a, b_, c, d) do { if (threadIdx.x == 0 && g_blkprof) { g_blkprof[32 * (size_t)K + 10] = gtimer(); \
  g_blkprof[32 * (size_t)K + 11] = (a); g_blkprof[32 * (size_t)K + 12] = (b_); g_blkprof[32 * (size_t)K + 13] = (c); \
  g_blkprof[32 * (size_t)K + 14] = (d); g_blkprof[32 * (size_t)K + 15] = blockIdx.x; } } while (0)
// the time block T became ready and the block whose release did it (profile slots 18, 26)
#define READY_MARK(T, K) do { if (g_blkprof) { g_blkprof[32 * (size_t)(T) + 18] = gtimer(); \
  g_blkprof[32 * (size_t)(T) + 26] = (unsigned long long)(K); } } while (0)
#else
#define READY_MARK(T, K) do {} while (0)
#define PROF_END(a, b_, c, d) do {} while (0)
#define SUBP(i) do {} while (0)
#define SUBP_T0
#define PROF_T0
#define PROF_T0C
#define PROF(i) DBGP(i)
#endif

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ int ld_vol(const int *p) { return *(const volatile int *)p; }
__device__ __forceinline__ unsigned long long ld_vol64(const unsigned long long *p) {
  return *(const volatile unsigned long long *)p;
}
__device__ __forceinline__ void st_vol(int *p, int v) { *(volatile int *)p = v; }

// high-priority queue: push tasks and the blocks they release (the dependency chains of the
// zone) are taken before the main queue's backlog
__device__ __forceinline__ void enqueue_hi(const DevFactor &F, int item) {
  const unsigned long long slot = atomicAdd(&F.ctrl[CS * CTRL_HQHEAD], 1ull);
  __threadfence();
  if (slot < (unsigned long long)F.hqcap) { st_vol(&F.hq[slot], item); return; }
  const unsigned long long s2 = atomicAdd(&F.ctrl[CS * CTRL_QHEAD], 1ull);   // full: main queue
  st_vol(&F.queue[s2], item);
}
__device__ __forceinline__ bool try_dequeue_hi(const DevFactor &F, int &item) {
  while (true) {
    const unsigned long long t = ld_vol64(&F.ctrl[CS * CTRL_HQTAIL]);
    const unsigned long long h = min(ld_vol64(&F.ctrl[CS * CTRL_HQHEAD]), (unsigned long long)F.hqcap);
    if (t >= h) return false;
    if (atomicCAS(&F.ctrl[CS * CTRL_HQTAIL], t, t + 1) == t) {
      int v;
      while ((v = ld_vol(&F.hq[t])) == -1) __nanosleep(32);   // producer between its ticket and its store
      item = v;
      return true;
    }
  }
}
__device__ __forceinline__ void raise_abort(const DevFactor &F, int code, int blk) {
  if (atomicCAS(&F.ctrl[CS * CTRL_ABORT], 0ull, (unsigned long long)code) == 0ull)
    atomicExch(&F.ctrl[CS * CTRL_ERRBLK], (unsigned long long)blk);
}
__device__ __forceinline__ bool aborted(const DevFactor &F) { return ld_vol64(&F.ctrl[CS * CTRL_ABORT]) != 0ull; }

// first position p in a[lo, hi) with a[p] >= key
__device__ __forceinline__ int lbound(const int *a, int lo, int hi, int key) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// exclusive scan of a[0..n) in place (any memory), returns the total. CTA-wide.
// Each warp owns a contiguous chunk and walks it in coalesced 32-element tiles
// (no shared-memory bank conflicts): pass 1 sums, pass 2 scans with the carry.
__device__ int cta_scan(int *a, int n, int *s_tmp /* >= NW+1 ints */) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int chunk = ((n + NW - 1) / NW + 31) & ~31;
  const int lo = min(n, wid * chunk), hi = min(n, lo + chunk);
  int sum = 0;
  for (int i = lo + lane; i < hi; i += 32) sum += a[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) s_tmp[wid] = sum;
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int w = 0; w < NW; ++w) { int t = s_tmp[w]; s_tmp[w] = acc; acc += t; }
    s_tmp[NW] = acc;
  }
  __syncthreads();
  int carry = s_tmp[wid];
  for (int base = lo; base < hi; base += 32) {
    const int i = base + lane;
    const int v = i < hi ? a[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (i < hi) a[i] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  const int total = s_tmp[NW];
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
    unsigned long long c = atomicAdd(&F.ctrl[CS * L.ctrl_cursor], 1ull);
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
  unsigned char *sbase; int sused, stop, scap;     // shared: bottom (persistent) / top (scratch)
  double *gbase; int64_t gused, gtop, gcap;        // global spill region, same scheme (doubles)
  bool ovf;
  bool bottom_global;                              // persistent allocations in global memory only
  bool pool;                                       // ... from the shared heavy-block pool (split blocks)
};
__device__ __forceinline__ void *balloc(Bump &A, int64_t bytes) {
  bytes = (bytes + 15) & ~int64_t(15);
  if (!A.bottom_global && A.sused + bytes <= A.stop) {
    void *p = A.sbase + A.sused;
    A.sused += (int)bytes;
    return p;
  }
  int64_t d = bytes / 8;
  if (A.gused + d <= A.gtop) {
    void *p = A.gbase + A.gused;
    A.gused += d;
    return p;
  }
  A.ovf = true;
  return A.gbase;  // caller checks ovf
}
__device__ __forceinline__ void *balloc_top(Bump &A, int64_t bytes) {
  bytes = (bytes + 15) & ~int64_t(15);
  if (A.stop - bytes >= A.sused) {
    A.stop -= (int)bytes;
    return A.sbase + A.stop;
  }
  int64_t d = bytes / 8;
  if (A.gtop - d >= A.gused) {
    A.gtop -= d;
    return A.gbase + A.gtop;
  }
  A.ovf = true;
  return A.gbase;
}

// --------------------------------------------------------------- the kernel
struct Shared {
  int K;
  int next;              // block made ready by this CTA, run next (release_block)
  unsigned long long ticket;   // main-queue slot this CTA holds (~0: none)
  int tmp[NW + 1];
  int piv;
  double pivd;
  int cnt[4];
  unsigned long long off[4];
  double sflops[2];      // Schur-update flops of each side
  int maxbJ[2];          // widest contributor of each side
  int maxkey[2];         // largest candidate key contributed to each side
};

// per-contributor descriptor kept in shared memory while block K is processed
struct Contrib {
  int J, bJ;
  int n_items;        // L side: rows >= s_K of L_J; U side: cols >= e_K of Ũ_J
  int n_cand_skip;    // L side: rows of the suffix that lie inside K (not candidates)
  int ncol;           // L side: Ũ_J columns inside K;  U side: L_J rows inside K
  int item_off;       // prefix over n_items
  int64_t rows;       // L side: Lidx offset of the first row >= s_K; U side: of row r0
  int64_t lval;       // matching Lval offset
  int64_t cols;       // L side: Uidx offset of column c0;  U side: of the first col >= e_K
  int64_t uval;       // matching Uval offset
  int last;           // largest candidate key of this contributor (-1: none)
};

// rank sort of distinct keys: out[rank(x)] = x (n small; thread per element)
__device__ void cta_rank_sort(const int *keys, int n, int *out) {
  for (int x = threadIdx.x; x < n; x += NT) {
    const int k = keys[x];
    int r = 0;
    for (int y = 0; y < n; ++y) r += keys[y] < k;
    out[r] = x;
  }
  __syncthreads();
}

// Both contributor lists of block K in one pass (records -> descriptors), each sorted
// by J (R13) and prefix-summed over its items (warp 0: Lc, warp 1: Uc).
// Lc(K): J has Ũ columns in K -> items = rows of L_J >= s_K
// Uc(K): J has L rows in K    -> items = cols of Ũ_J >= e_K
__device__ void load_contribs2(const DevFactor &F, int K, Contrib *CL, Contrib *CU, int nLc, int nUc, int *keys,
                               Shared &S) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nt = nLc + nUc;
  for (int x = tid; x < nt; x += NT) {
    const int side = x < nLc ? 0 : 1;
    const int xi = side ? x - nLc : x;
    const ChunkList &L = side ? F.uc : F.lc;
    const int *r = list_rec(L, K, xi);
    const int J = __ldcg(r);
    keys[x] = J;
    Contrib c;
    c.J = J;
    const int sJ = F.bstart[J];
    c.bJ = F.bstart[J + 1] - sJ;
    const int64_t lro = __ldcg(&F.Lrow_off[J]), lvo = __ldcg(&F.Lval_off[J]);
    const int64_t uco = __ldcg(&F.Ucol_off[J]), uvo = __ldcg(&F.Uval_off[J]);
    if (side == 0) {
      const int c0 = __ldcg(r + 1), c1 = __ldcg(r + 2), lrs = __ldcg(r + 3), lre = __ldcg(r + 4);
      const int mJ = __ldcg(&F.Lm[J]);
      c.n_items = mJ - lrs;
      c.n_cand_skip = lre - lrs;
      c.ncol = c1 - c0;
      c.rows = lro + lrs;
      c.lval = lvo + (int64_t)lrs * c.bJ;
      c.cols = uco + c0;
      c.uval = uvo + (int64_t)c0 * c.bJ;
      c.last = c.n_items > c.n_cand_skip ? __ldcg(&F.Lidx[c.rows + c.n_items - 1]) : -1;
      CL[nLc + xi] = c;
    } else {
      const int r0 = __ldcg(r + 1), r1 = __ldcg(r + 2), cus = __ldcg(r + 3);
      const int cJ = __ldcg(&F.Uc[J]);
      c.n_items = cJ - cus;
      c.n_cand_skip = 0;
      c.ncol = r1 - r0;
      c.rows = lro + r0;
      c.lval = lvo + (int64_t)r0 * c.bJ;
      c.cols = uco + cus;
      c.uval = uvo + (int64_t)cus * c.bJ;
      c.last = c.n_items > 0 ? __ldcg(&F.Uidx[c.cols + c.n_items - 1]) : -1;
      CU[nUc + xi] = c;
    }
  }
  __syncthreads();
  for (int x = tid; x < nt; x += NT) {       // ascending J within each list (J distinct)
    const int side = x < nLc ? 0 : 1;
    const int xi = side ? x - nLc : x, n = side ? nUc : nLc;
    const int *kk = keys + (side ? nLc : 0);
    const int k = kk[xi];
    int rk = 0;
    for (int y = 0; y < n; ++y) rk += kk[y] < k;
    Contrib *C = side ? CU : CL;
    C[rk] = C[n + xi];
  }
  __syncthreads();
  if (wid < 2) {
    Contrib *C = wid ? CU : CL;
    const int n = wid ? nUc : nLc;
    int carry = 0, mb = 0, mk = -1;
    double fl = 0.0;
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const int v = i < n ? C[i].n_items : 0;
      if (i < n) {
        fl += 2.0 * C[i].bJ * (double)C[i].n_items * (double)C[i].ncol;
        mb = max(mb, C[i].bJ);
        mk = max(mk, C[i].last);
      }
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (i < n) C[i].item_off = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      fl += __shfl_xor_sync(0xffffffffu, fl, o);
      mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
      mk = max(mk, __shfl_xor_sync(0xffffffffu, mk, o));
    }
    if (lane == 0) { S.cnt[wid] = carry; S.sflops[wid] = fl; S.maxbJ[wid] = mb; S.maxkey[wid] = mk; }
  }
  __syncthreads();
}

__device__ __forceinline__ int contrib_of(const Contrib *C, int nc, int t) {
  int lo = 0, hi = nc - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (C[mid].item_off <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}


// key -> buffer line of the candidate set of one side.  Two representations:
//  * bitmap (range of keys [e, e + 32*words) small enough for shared memory): bit per
//    key, per-word prefix counts; lines are in ascending key order
//  * pos map (fallback for wide ranges): per-CTA global array, last writer wins
struct LineMap {
  const unsigned *bm; const int *pre; int words;   // bitmap path
  const int *pos;                                   // pos-map path (bm == nullptr)
  const unsigned *l1; const int *pre1;              // two-level bitmap: pages of 1024 keys
  int e, base;
  __device__ __forceinline__ int operator()(int key) const {
    if (bm) {
      const int r = key - e;
      int w = r >> 5;
      if (l1) {                                     // page slot, then the word inside the page
        const int p = r >> 10, w1 = p >> 5;
        w = (pre1[w1] + __popc(l1[w1] & ((1u << (p & 31)) - 1u))) * 32 + (w & 31);
      }
      return base + pre[w] + __popc(bm[w] & ((1u << (r & 31)) - 1u));
    }
    return pos[key];
  }
};

// state of one side of block K after a-3/a-4
struct SideState {
  double *W;       // dense buffer, line-major (lines x b)
  int *lineOf;     // line -> matrix index
  int nU;          // candidate lines (excl. the pivot block)
  bool sorted;     // lines in ascending index order (bitmap path)
  LineMap M;
  const unsigned *gbm; const int *gpre;   // global copies of the bitmap map (split blocks)
  const unsigned *gl1; const int *gpre1;  // ... and of its page level (two-level maps)
};

constexpr int MAX_PARTS = 32;          // update parts per block (both sides)
constexpr int MAX_SPARTS = 32;         // scaling parts per block (wide split blocks)
constexpr int TASK_STRIDE = MAX_PARTS + MAX_SPARTS;   // task = N + ctx * TASK_STRIDE + part

// a split heavy block (see process_block)
struct HeavyCtx {
  int K, nc[2], T[2], np[2];
  int left;                 // parts not yet completed
  const Contrib *C[2];
  SideState R[2];
  double flops;
  int wide;                 // parts run per-contributor DMMA products over contributor ranges
  const int *iline[2];      // wide: destination line of every item of each side
  int cb[2][MAX_PARTS / 2 + 1];   // wide: contributor range of every part
  // wide: scaling split (finish_block mode 1 -> scale parts -> mode 2)
  double *Lsc, *Usc, *Lmx, *Umx;
  int ns, left2;
  int sortedR, sortedC;
};

// One side of block K (SIDE 0: block column of L incl. the pivot block; SIDE 1:
// block row of U):
//   a-3  candidate set: keys >= e_K of Ã's block column (resp. row) and of every
//        contributor's kept L rows (resp. Ũ columns)
//   a-4  dense buffer W (SIDE 0: (b + nR) x b row-major, rows 0..b-1 = the pivot
//        block; SIDE 1: nC columns of b), Ã's entries scattered in ("load the
//        associated scalar sparse columns of A into block column buffer")
//   a-5  W -= L_J Ũ_J for every contributor J in ascending J (R13) -- "gather ... GEMM
//        ... scatter": one thread per item (a row of L_J >= s_K,
//        resp. a column of Ũ_J >= e_K), the next contributor's operands prefetched
//        into registers while the current one is applied.
template <int SIDE>
__device__ bool side_prepare(const DevFactor &F, int K, int s, int e, int b, const Contrib *C, int nc, int T,
                             int64_t a0, int64_t ae, int64_t a1, Bump &A, Shared &S, SideState &R) {
  const int tid = threadIdx.x;
  const int32_t *arc = SIDE == 0 ? F.AL_rc : F.AU_rc;
  const double *aval = SIDE == 0 ? F.AL_val : F.AU_val;
  const int32_t *cidx = SIDE == 0 ? F.Lidx : F.Uidx;     // index list of the item side
  const int nA = (int)(a1 - ae);                           // Ã entries that are candidates
  SUBP_T0
  // -- range of candidate keys: Ã's block column / row is sorted by key, so its last entry
  //    is its largest key; the contributors' largest keys come from load_contribs2
  const int hi = max(max(e - 1, S.maxkey[SIDE]), a1 > ae ? (arc[a1 - 1] >> 7) : e - 1);
  const int words = (hi - e + 1 + 31) >> 5;
  const int base = SIDE == 0 ? b : 0;            // buffer line of the first candidate
  LineMap M;
  M.e = e; M.base = base; M.bm = nullptr; M.pre = nullptr; M.words = words; M.l1 = nullptr; M.pre1 = nullptr;
  M.pos = F.posmap + (size_t)blockIdx.x * F.n;
  int nU = 0;
  unsigned *bm = nullptr;
  int *pre = nullptr;
  if (words <= 8192) {
    // ---- bitmap path: dedup by atomicOr in shared memory, sorted for free
    bm = (unsigned *)balloc_top(A, (int64_t)(words + 1) * 4);
    pre = (int *)balloc_top(A, (int64_t)(words + 1) * 4);
    if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return false; }
    for (int w = tid; w < words; w += NT) bm[w] = 0u;
    __syncthreads();
    for (int64_t p = ae + tid; p < a1; p += NT) {
      const int r = (arc[p] >> 7) - e;
      atomicOr(&bm[r >> 5], 1u << (r & 31));
    }
    {
      int a = 0;
      for (int t0 = tid; t0 < T; t0 += 4 * NT) {
        int r4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = t0 + u * NT;
          r4[u] = -1;
          if (t < T) {
            while (a + 1 < nc && C[a + 1].item_off <= t) ++a;
            const int i = t - C[a].item_off;
            if (i >= C[a].n_cand_skip)                       // rows inside K are the pivot block
              r4[u] = cidx[(SIDE == 0 ? C[a].rows : C[a].cols) + i] - e;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (r4[u] >= 0) atomicOr(&bm[r4[u] >> 5], 1u << (r4[u] & 31));
      }
    }
    __syncthreads();
    for (int w = tid; w < words; w += NT) pre[w] = __popc(bm[w]);
    __syncthreads();
    nU = cta_scan(pre, words, S.tmp);
    M.bm = bm; M.pre = pre;

  } else {
    // ---- pos-map path: every occurrence writes its id, the surviving writer appends
    const int occ = nA + T;
    int *pos = F.posmap + (size_t)blockIdx.x * F.n;
    {
      int a = 0;
      for (int o = tid; o < occ; o += NT) {
        int key;
        if (o < nA) key = arc[ae + o] >> 7;
        else {
          const int t = o - nA;
          while (a + 1 < nc && C[a + 1].item_off <= t) ++a;
          const int i = t - C[a].item_off;
          if (i < C[a].n_cand_skip) continue;
          key = cidx[(SIDE == 0 ? C[a].rows : C[a].cols) + i];
        }
        pos[key] = o;
      }
    }
    if (tid == 0) S.cnt[2] = 0;
    __syncthreads();
    int *uniq = (int *)balloc_top(A, (int64_t)(occ + 1) * 4);
    if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return false; }
    {
      int a = 0;
      for (int o = tid; o < occ; o += NT) {
        int key;
        if (o < nA) key = arc[ae + o] >> 7;
        else {
          const int t = o - nA;
          while (a + 1 < nc && C[a + 1].item_off <= t) ++a;
          const int i = t - C[a].item_off;
          if (i < C[a].n_cand_skip) continue;
          key = cidx[(SIDE == 0 ? C[a].rows : C[a].cols) + i];
        }
        if (pos[key] == o) uniq[atomicAdd(&S.cnt[2], 1)] = key;
      }
    }
    __syncthreads();
    nU = S.cnt[2];
    for (int x = tid; x < nU; x += NT) pos[uniq[x]] = base + x;
    __syncthreads();
    // keep uniq (it becomes lineOf below)
    pre = uniq;
  }
  SUBP(8 * SIDE + 0);
  const int nW = base + nU;
  double *W;
  int *lineOf;
  if (A.pool) {
    // a split block: W, the line map and a copy of the bitmap map live in the global pool
    // (read by the helpers), allocated exactly now that the candidate count is known
    const int64_t wd = (int64_t)nW * b, ld = ((int64_t)nW + 2) / 2 + 1;
    const int64_t md = M.bm ? (int64_t)words + 2 : 0;     // bitmap + prefix (2 x words ints)
    if (tid == 0) S.off[3] = atomicAdd(&F.ctrl[CS * CTRL_HPOOL], (unsigned long long)(wd + ld + md));
    __syncthreads();
    const unsigned long long o = S.off[3];
    __syncthreads();
    if (o + wd + ld + md > (unsigned long long)F.hpool_cap) { if (tid == 0) raise_abort(F, DEV_OVF_HPOOL, K); return false; }
    W = F.hpool + o;
    lineOf = (int *)(W + wd);
    if (M.bm) {
      unsigned *gbm = (unsigned *)(W + wd + ld);
      int *gpre = (int *)(gbm + words + 1);
      for (int w = tid; w < words; w += NT) { gbm[w] = bm[w]; gpre[w] = pre[w]; }
      R.gbm = gbm; R.gpre = gpre; R.gl1 = nullptr; R.gpre1 = nullptr;
    }
  } else {
    W = (double *)balloc(A, (int64_t)nW * b * 8);
    lineOf = (int *)balloc(A, (int64_t)(nW + 1) * 4);
    if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return false; }
  }
  for (int x = tid; x < base; x += NT) lineOf[x] = s + x;
  if (M.bm) {
    for (int w = tid; w < words; w += NT) {
      unsigned m = bm[w];
      int at = base + pre[w];
      while (m) {
        const int bit = __ffs(m) - 1;
        lineOf[at++] = e + (w << 5) + bit;
        m &= m - 1;
      }
    }
  } else {
    for (int x = tid; x < nU; x += NT) lineOf[base + x] = pre[x];
  }
  if (!A.pool)                           // the global pool is zero at every launch
    for (int x = tid; x < nW * b; x += NT) W[x] = 0.0;
  __syncthreads();
  // -- a-4: scatter Ã
  for (int64_t p = a0 + tid; p < a1; p += NT) {
    const int rc = arc[p], key = rc >> 7;
    const int w = (SIDE == 0 && key < e) ? key - s : M(key);
    W[(int64_t)w * b + (rc & 127)] = aval[p];
  }
  __syncthreads();
  SUBP(8 * SIDE + 1);
  R.W = W; R.lineOf = lineOf; R.nU = nU; R.M = M;
  R.sorted = M.bm != nullptr;   // bitmap path: lines in ascending key order
  return true;
}

// a-3 / a-4 of both sides in lockstep (bitmap path on both sides): one pass per step over
// the two sides' Ã entries and items, one prefix scan over the two bitmaps, so the two
// sides' memory latencies overlap and the barriers are shared.  Same result as
// side_prepare<0> followed by side_prepare<1>.  Returns false (nothing done) when either
// side's key range needs the pos-map path.
__device__ int prep_words(const Shared &S, int side, int e, const int32_t *arc, int64_t ae, int64_t a1) {
  const int hi = max(max(e - 1, S.maxkey[side]), a1 > ae ? (arc[a1 - 1] >> 7) : e - 1);
  return (hi - e + 1 + 31) >> 5;
}

// a-4: scatter Ã's block column (incl. the pivot block) into W_L and its block row into W_U
// ("load the associated scalar sparse columns of A into block column buffer", PAPER.md:
// 370-371); four entries in flight per thread.  CTA-wide, ends with a barrier.
__device__ void scatter_A(const DevFactor &F, int s, int e, int b, int64_t aL0, int64_t aL1, int64_t aU0, int64_t aU1,
                          const LineMap &ML, const LineMap &MU, double *WL, double *WU) {
  const int nL0 = (int)(aL1 - aL0), nAU = (int)(aU1 - aU0);
  for (int x0 = threadIdx.x; x0 < nL0 + nAU; x0 += 4 * NT) {
    int rc4[4]; double v4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int x = x0 + u * NT;
      rc4[u] = -1; v4[u] = 0.0;
      if (x < nL0) { rc4[u] = F.AL_rc[aL0 + x]; v4[u] = F.AL_val[aL0 + x]; }
      else if (x < nL0 + nAU) { rc4[u] = F.AU_rc[aU0 + (x - nL0)]; v4[u] = F.AU_val[aU0 + (x - nL0)]; }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int x = x0 + u * NT;
      if (rc4[u] < 0) continue;
      const int key = rc4[u] >> 7;
      if (x < nL0) WL[(int64_t)(key < e ? key - s : ML(key)) * b + (rc4[u] & 127)] = v4[u];
      else WU[(int64_t)MU(key) * b + (rc4[u] & 127)] = v4[u];
    }
  }
  __syncthreads();
}

__device__ bool prepare_both(const DevFactor &F, int K, int s, int e, int b, const Contrib *CL, int nLc, int TL,
                             const Contrib *CU, int nUc, int TU, int64_t aL0, int64_t aLe, int64_t aL1, int64_t aU0,
                             int64_t aU1, Bump &A, Shared &S, SideState &RL, SideState &RU, bool &ok) {
  const int tid = threadIdx.x;
  ok = true;
  const int wL = prep_words(S, 0, e, F.AL_rc, aLe, aL1), wU = prep_words(S, 1, e, F.AU_rc, aU0, aU1);
  if (wL > 8192 || wU > 8192) return false;
  unsigned *bm = (unsigned *)balloc_top(A, (int64_t)(wL + wU + 2) * 4);
  int *pre = (int *)balloc_top(A, (int64_t)(wL + wU + 2) * 4);
  if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); ok = false; return true; }
  unsigned *bmL = bm, *bmU = bm + wL;
  for (int w = tid; w < wL + wU; w += NT) bm[w] = 0u;
  __syncthreads();
  // Ã's distinct candidate keys of both sides, then the items of both sides
  {
    const int64_t kL0 = F.AKL_ptr[K], kU0 = F.AKU_ptr[K];
    const int nKL = (int)(F.AKL_ptr[K + 1] - kL0), nKU = (int)(F.AKU_ptr[K + 1] - kU0);
    for (int x = tid; x < nKL + nKU; x += NT) {
      if (x < nKL) { const int r = F.AKL[kL0 + x] - e; atomicOr(&bmL[r >> 5], 1u << (r & 31)); }
      else { const int r = F.AKU[kU0 + (x - nKL)] - e; atomicOr(&bmU[r >> 5], 1u << (r & 31)); }
    }
  }
  {
    int aL = 0, aU = 0;
    for (int t0 = tid; t0 < TL + TU; t0 += 4 * NT) {
      int r4[4], sd[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = t0 + u * NT;
        r4[u] = -1; sd[u] = 0;
        if (t < TL) {
          while (aL + 1 < nLc && CL[aL + 1].item_off <= t) ++aL;
          const int i = t - CL[aL].item_off;
          if (i >= CL[aL].n_cand_skip) r4[u] = F.Lidx[CL[aL].rows + i] - e;   // pivot rows excluded
        } else if (t < TL + TU) {
          const int tu = t - TL;
          while (aU + 1 < nUc && CU[aU + 1].item_off <= tu) ++aU;
          r4[u] = F.Uidx[CU[aU].cols + (tu - CU[aU].item_off)] - e;
          sd[u] = 1;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (r4[u] >= 0) atomicOr(&(sd[u] ? bmU : bmL)[r4[u] >> 5], 1u << (r4[u] & 31));
    }
  }
  __syncthreads();
  for (int w = tid; w < wL + wU; w += NT) pre[w] = __popc(bm[w]);
  __syncthreads();
  const int tot = cta_scan(pre, wL + wU, S.tmp);
  const int nUL = wU > 0 ? pre[wL] : tot, nUU = tot - nUL;
  // line maps: L lines start at b (pivot rows first); U prefix sums are offset by nUL
  LineMap ML, MU;
  ML.e = e; ML.base = b; ML.bm = bmL; ML.pre = pre; ML.words = wL; ML.pos = nullptr; ML.l1 = nullptr; ML.pre1 = nullptr;
  MU.e = e; MU.base = -nUL; MU.bm = bmU; MU.pre = pre + wL; MU.words = wU; MU.pos = nullptr; MU.l1 = nullptr; MU.pre1 = nullptr;
  const int nWL = b + nUL, nWU = nUU;
  double *WL, *WU;
  int *lineL, *lineU;
  if (A.pool) {
    const int64_t wdL = (int64_t)nWL * b, ldL = ((int64_t)nWL + 2) / 2 + 1, mdL = (int64_t)wL + 2;
    const int64_t wdU = (int64_t)nWU * b, ldU = ((int64_t)nWU + 2) / 2 + 1, mdU = (int64_t)wU + 2;
    const int64_t d = wdL + ldL + mdL + wdU + ldU + mdU;
    if (tid == 0) S.off[3] = atomicAdd(&F.ctrl[CS * CTRL_HPOOL], (unsigned long long)d);
    __syncthreads();
    const unsigned long long o = S.off[3];
    __syncthreads();
    if (o + d > (unsigned long long)F.hpool_cap) { if (tid == 0) raise_abort(F, DEV_OVF_HPOOL, K); ok = false; return true; }
    WL = F.hpool + o;
    lineL = (int *)(WL + wdL);
    unsigned *gbmL = (unsigned *)(WL + wdL + ldL);
    WU = WL + wdL + ldL + mdL;
    lineU = (int *)(WU + wdU);
    unsigned *gbmU = (unsigned *)(WU + wdU + ldU);
    int *gpreL = (int *)(gbmL + wL + 1), *gpreU = (int *)(gbmU + wU + 1);
    for (int w = tid; w < wL; w += NT) { gbmL[w] = bmL[w]; gpreL[w] = pre[w]; }
    for (int w = tid; w < wU; w += NT) { gbmU[w] = bmU[w]; gpreU[w] = pre[wL + w]; }
    RL.gbm = gbmL; RL.gpre = gpreL; RU.gbm = gbmU; RU.gpre = gpreU;   // global copies (same bases)
    RL.gl1 = RU.gl1 = nullptr; RL.gpre1 = RU.gpre1 = nullptr;
  } else {
    WL = (double *)balloc(A, (int64_t)nWL * b * 8);
    lineL = (int *)balloc(A, (int64_t)(nWL + 1) * 4);
    WU = (double *)balloc(A, (int64_t)nWU * b * 8);
    lineU = (int *)balloc(A, (int64_t)(nWU + 1) * 4);
    if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); ok = false; return true; }
  }
  for (int x = tid; x < b; x += NT) lineL[x] = s + x;
  for (int w = tid; w < wL + wU; w += NT) {
    const bool u = w >= wL;
    unsigned m = bm[w];
    int at = u ? pre[w] - nUL : b + pre[w];
    int *lo = u ? lineU : lineL;
    const int wb = u ? w - wL : w;
    while (m) {
      const int bit = __ffs(m) - 1;
      lo[at++] = e + (wb << 5) + bit;
      m &= m - 1;
    }
  }
  if (!A.pool) {
    for (int x = tid; x < nWL * b; x += NT) WL[x] = 0.0;
    for (int x = tid; x < nWU * b; x += NT) WU[x] = 0.0;
  }
  __syncthreads();
  scatter_A(F, s, e, b, aL0, aL1, aU0, aU1, ML, MU, WL, WU);
  RL.W = WL; RL.lineOf = lineL; RL.nU = nUL; RL.M = ML; RL.sorted = true;
  RU.W = WU; RU.lineOf = lineU; RU.nU = nUU; RU.M = MU; RU.sorted = true;
  return true;
}

// a-3 / a-4 of both sides when a key range is too wide for the flat bitmap: a two-level
// bitmap in shared memory -- a page bit per 1024 keys, then one 32-word bitmap per occupied
// page -- so the candidate lines stay in ascending key order (sorted, no pos map) for any n.
// Two passes over the occurrences (Ã's distinct candidate keys and the contributors' items), four loads in flight per thread.  Same result as side_prepare<0>
// followed by side_prepare<1>.  Returns false (nothing done) if the occupied pages do not
// fit in the shared-memory budget.
__device__ bool prepare_both2(const DevFactor &F, int K, int s, int e, int b, const Contrib *CL, int nLc, int TL,
                              const Contrib *CU, int nUc, int TU, int64_t aL0, int64_t aLe, int64_t aL1, int64_t aU0,
                              int64_t aU1, Bump &A, Shared &S, SideState &RL, SideState &RU, bool &ok) {
  const int tid = threadIdx.x;
  ok = true;
  const int hiL = max(max(e - 1, S.maxkey[0]), aL1 > aLe ? (F.AL_rc[aL1 - 1] >> 7) : e - 1);
  const int hiU = max(max(e - 1, S.maxkey[1]), aU1 > aU0 ? (F.AU_rc[aU1 - 1] >> 7) : e - 1);
  const int w1L = ((hiL - e + 1 + 1023) >> 10) / 32 + 1, w1U = ((hiU - e + 1 + 1023) >> 10) / 32 + 1;
  const int64_t kL0 = F.AKL_ptr[K], kU0 = F.AKU_ptr[K];
  const int nKL = (int)(F.AKL_ptr[K + 1] - kL0), nKU = (int)(F.AKU_ptr[K + 1] - kU0);
  const int nocc = nKL + nKU + TL + TU;
  const int stop0 = A.stop;
  const int64_t gtop0 = A.gtop;
  // level 1 (+ its prefix) and the slot -> page table
  unsigned *l1 = (unsigned *)balloc_top(A, (int64_t)(w1L + w1U + 2) * 4);
  int *pre1 = (int *)balloc_top(A, (int64_t)(w1L + w1U + 2) * 4);
  if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); ok = false; return true; }
  for (int w = tid; w < w1L + w1U; w += NT) l1[w] = 0u;
  __syncthreads();
  // the key of occurrence x (-1: not a candidate) and its side
  auto occ = [&](int x, int &aL, int &aU, int &side) -> int {
    if (x < nKL) { side = 0; return F.AKL[kL0 + x]; }
    if (x < nKL + nKU) { side = 1; return F.AKU[kU0 + (x - nKL)]; }
    int t = x - nKL - nKU;
    if (t < TL) {
      while (aL + 1 < nLc && CL[aL + 1].item_off <= t) ++aL;
      const int i = t - CL[aL].item_off;
      side = 0;
      return i >= CL[aL].n_cand_skip ? F.Lidx[CL[aL].rows + i] : -1;   // pivot rows excluded
    }
    t -= TL;
    while (aU + 1 < nUc && CU[aU + 1].item_off <= t) ++aU;
    side = 1;
    return F.Uidx[CU[aU].cols + (t - CU[aU].item_off)];
  };
  {   // pass A: occupied pages
    int aL = 0, aU = 0;
    for (int x0 = tid; x0 < nocc; x0 += 4 * NT) {
      int k4[4], s4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { const int x = x0 + u * NT; k4[u] = x < nocc ? occ(x, aL, aU, s4[u]) : -1; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k4[u] >= 0) { const int pg = (k4[u] - e) >> 10; atomicOr(&l1[(s4[u] ? w1L : 0) + (pg >> 5)], 1u << (pg & 31)); }
    }
  }
  __syncthreads();
  for (int w = tid; w < w1L + w1U; w += NT) pre1[w] = __popc(l1[w]);
  __syncthreads();
  const int npu = cta_scan(pre1, w1L + w1U, S.tmp);
  const int npuL = pre1[w1L];
  // page bitmaps: budget -- fall back to the pos map beyond it
  const int64_t need = (int64_t)npu * 32 * 8 + (int64_t)npu * 4 + 64;
  if (need > (int64_t)(A.stop - A.sused) - 16 * 1024) {
    A.stop = stop0; A.gtop = gtop0;       // release l1 / pre1
    __syncthreads();
    return false;
  }
  unsigned *bm = (unsigned *)balloc_top(A, (int64_t)npu * 32 * 4 + 4);
  int *pre = (int *)balloc_top(A, (int64_t)npu * 32 * 4 + 4);
  int *pg = (int *)balloc_top(A, (int64_t)npu * 4 + 4);
  for (int w = tid; w < npu * 32; w += NT) bm[w] = 0u;
  for (int w = tid; w < w1L + w1U; w += NT) {
    unsigned m = l1[w];
    int at = pre1[w];
    const int pb = (w < w1L ? w : w - w1L) << 5;
    while (m) { const int bit = __ffs(m) - 1; pg[at++] = pb + bit; m &= m - 1; }
  }
  __syncthreads();
  {   // pass B: key bits inside the pages
    int aL = 0, aU = 0;
    for (int x0 = tid; x0 < nocc; x0 += 4 * NT) {
      int k4[4], s4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { const int x = x0 + u * NT; k4[u] = x < nocc ? occ(x, aL, aU, s4[u]) : -1; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k4[u] >= 0) {
          const int r = k4[u] - e, p = r >> 10, w1 = (s4[u] ? w1L : 0) + (p >> 5);
          const int slot = pre1[w1] + __popc(l1[w1] & ((1u << (p & 31)) - 1u));
          atomicOr(&bm[slot * 32 + ((r >> 5) & 31)], 1u << (r & 31));
        }
    }
  }
  __syncthreads();
  for (int w = tid; w < npu * 32; w += NT) pre[w] = __popc(bm[w]);
  __syncthreads();
  const int tot = cta_scan(pre, npu * 32, S.tmp);
  const int nUL = npuL < npu ? pre[npuL * 32] : tot, nUU = tot - nUL;
  LineMap ML, MU;
  ML.e = e; ML.base = b; ML.bm = bm; ML.pre = pre; ML.words = npu * 32; ML.pos = nullptr; ML.l1 = l1; ML.pre1 = pre1;
  MU.e = e; MU.base = -nUL; MU.bm = bm; MU.pre = pre; MU.words = npu * 32; MU.pos = nullptr; MU.l1 = l1 + w1L;
  MU.pre1 = pre1 + w1L;
  const int nWL = b + nUL, nWU = nUU;
  double *WL, *WU;
  int *lineL, *lineU;
  if (A.pool) {
    const int64_t wdL = (int64_t)nWL * b, ldL = ((int64_t)nWL + 2) / 2 + 1;
    const int64_t wdU = (int64_t)nWU * b, ldU = ((int64_t)nWU + 2) / 2 + 1;
    const int64_t md = ((int64_t)npu * 64 + 2 * (w1L + w1U) + 8) / 2 + 2;      // bm, pre, l1, pre1 (ints)
    const int64_t d = wdL + ldL + wdU + ldU + md;
    if (tid == 0) S.off[3] = atomicAdd(&F.ctrl[CS * CTRL_HPOOL], (unsigned long long)d);
    __syncthreads();
    const unsigned long long o = S.off[3];
    __syncthreads();
    if (o + d > (unsigned long long)F.hpool_cap) { if (tid == 0) raise_abort(F, DEV_OVF_HPOOL, K); ok = false; return true; }
    WL = F.hpool + o;
    lineL = (int *)(WL + wdL);
    WU = WL + wdL + ldL;
    lineU = (int *)(WU + wdU);
    unsigned *gbm = (unsigned *)(WU + wdU + ldU);
    int *gpre = (int *)(gbm + npu * 32);
    unsigned *gl1 = (unsigned *)(gpre + npu * 32);
    int *gpre1 = (int *)(gl1 + w1L + w1U);
    for (int w = tid; w < npu * 32; w += NT) { gbm[w] = bm[w]; gpre[w] = pre[w]; }
    for (int w = tid; w < w1L + w1U; w += NT) { gl1[w] = l1[w]; gpre1[w] = pre1[w]; }
    RL.gbm = gbm; RL.gpre = gpre; RU.gbm = gbm; RU.gpre = gpre;
    RL.gl1 = gl1; RL.gpre1 = gpre1; RU.gl1 = gl1 + w1L; RU.gpre1 = gpre1 + w1L;
  } else {
    WL = (double *)balloc(A, (int64_t)nWL * b * 8);
    lineL = (int *)balloc(A, (int64_t)(nWL + 1) * 4);
    WU = (double *)balloc(A, (int64_t)nWU * b * 8);
    lineU = (int *)balloc(A, (int64_t)(nWU + 1) * 4);
    if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); ok = false; return true; }
  }
  for (int x = tid; x < b; x += NT) lineL[x] = s + x;
  for (int w = tid; w < npu * 32; w += NT) {
    const int sl = w >> 5;
    const bool u = sl >= npuL;
    unsigned m = bm[w];
    int at = u ? pre[w] - nUL : b + pre[w];
    int *lo = u ? lineU : lineL;
    const int kb = e + (pg[sl] << 10) + ((w & 31) << 5);
    while (m) { const int bit = __ffs(m) - 1; lo[at++] = kb + bit; m &= m - 1; }
  }
  if (!A.pool) {
    for (int x = tid; x < nWL * b; x += NT) WL[x] = 0.0;
    for (int x = tid; x < nWU * b; x += NT) WU[x] = 0.0;
  }
  __syncthreads();
  scatter_A(F, s, e, b, aL0, aL1, aU0, aU1, ML, MU, WL, WU);
  RL.W = WL; RL.lineOf = lineL; RL.nU = nUL; RL.M = ML; RL.sorted = true;
  RU.W = WU; RU.lineOf = lineU; RU.nU = nUU; RU.M = MU; RU.sorted = true;
  return true;
}

// a-5 for the items [t0, t1) of one side: W -= L_J Ũ_J, "gather ... GEMM ... scatter"
// (Fig. 2): one thread per item (a row of L_J >= s_K, resp. a column of
// Ũ_J >= e_K); contributions are added atomically (shared-memory W) or with native
// global fp64 reductions (GLOBAL: W of a split heavy block), so the summation order is
// unspecified (exact in exact arithmetic, R13; differences are rounding only).
__device__ __forceinline__ void red_add_f64(double *p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
template <int SIDE, bool GLOBAL>
__device__ void side_items(const DevFactor &F, int s, int e, const Contrib *C, int nc, int t0, int t1, int b,
                           const LineMap &M, double *W) {
  const int32_t *cidx = SIDE == 0 ? F.Lidx : F.Uidx;
  int a = contrib_of(C, nc, min(t0 + (int)threadIdx.x, t1 - 1));
#pragma unroll 2
  for (int t = t0 + threadIdx.x; t < t1; t += NT) {
    while (a + 1 < nc && C[a + 1].item_off <= t) ++a;
    const Contrib &c = C[a];
    const int i = t - c.item_off, bJ = c.bJ, ncol = c.ncol;
    const int key = cidx[(SIDE == 0 ? c.rows : c.cols) + i];
    const int ln = (SIDE == 0 && key < e) ? key - s : M(key);
    const double *vi = (SIDE == 0 ? F.Lval + c.lval : F.Uval + c.uval) + (int64_t)i * bJ;
    const double *sm = SIDE == 0 ? F.Uval + c.uval : F.Lval + c.lval;
    const int32_t *sidx = SIDE == 0 ? F.Uidx + c.cols : F.Lidx + c.rows;
    double *wl = W + (int64_t)ln * b;
    if (bJ <= 16) {
      double v[16];
#pragma unroll
      for (int t2 = 0; t2 < 16; ++t2) v[t2] = t2 < bJ ? vi[t2] : 0.0;
      for (int q = 0; q < ncol; ++q) {
        const double *u = sm + (int64_t)q * bJ;
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
        for (int t2 = 0; t2 < 16; t2 += 2) {
          if (t2 < bJ) acc0 = fma(v[t2], u[t2], acc0);
          if (t2 + 1 < bJ) acc1 = fma(v[t2 + 1], u[t2 + 1], acc1);
        }
        if (GLOBAL) red_add_f64(&wl[sidx[q] - s], -(acc0 + acc1));
        else atomicAdd(&wl[sidx[q] - s], -(acc0 + acc1));
      }
    } else {
      for (int q = 0; q < ncol; ++q) {
        const double *u = sm + (int64_t)q * bJ;
        double acc = 0.0;
        for (int t2 = 0; t2 < bJ; ++t2) acc = fma(vi[t2], u[t2], acc);
        if (GLOBAL) red_add_f64(&wl[sidx[q] - s], -acc);
        else atomicAdd(&wl[sidx[q] - s], -acc);
      }
    }
  }
}

// a-5 for wide blocks: per contributor J (ascending, R13) one dense product on the FP64
// tensor pipe, "gather ... GEMM ... scatter" (Fig. 2):
//   SIDE 0: W_L[line(rows of L_J >= s_K), cols of Ũ_J in K] -= L_J(rows >= s_K, :) · Ũ_J(:, cols in K)
//   SIDE 1: W_U[line(cols of Ũ_J >= e_K), rows of L_J in K] -= Ũ_J(:, cols >= e_K)^T · L_J(rows in K, :)^T
// Both operands are contiguous slices of the hybrid panels; each output element is
// scattered once per product, so no atomics are needed.
template <int SIDE>
struct EpiScatter {
  const int32_t *ikey, *jkey;   // matrix index of output row i / column j
  int s, e, b;
  LineMap M;
  double *W;
  __device__ __forceinline__ void operator()(int i, int j, double v) const {
    const int key = ikey[i];
    const int ln = (SIDE == 0 && key < e) ? key - s : M(key);
    W[(int64_t)ln * b + (jkey[j] - s)] -= v;
  }
};

// B of one contributor's product (SIDE 0: Ũ_J(:, cols in K), b_J x ncol; SIDE 1:
// L_J(rows in K, :)^T, b_J x ncol) staged in shared memory, then the tall-skinny product
// over the contributor's items.  bs: scratch of >= 128 x TsB<128>::LDB doubles.
template <int SIDE, int NMAX>
__device__ void contrib_tsgemm(const DevFactor &F, int s, int e, int b, const Contrib &c, const LineMap &M, double *W,
                               double *bs) {
  if (SIDE == 0) {
    tsgemm_stage_b<NT, NMAX>(c.bJ, c.ncol, DMat{F.Uval + c.uval, 1, c.bJ}, bs);
    EpiScatter<0> ep{F.Lidx + c.rows, F.Uidx + c.cols, s, e, b, M, W};
    cta_tsgemm<NT, NMAX>(c.n_items, c.ncol, c.bJ, DMat{F.Lval + c.lval, c.bJ, 1}, bs, ep);
  } else {
    tsgemm_stage_b<NT, NMAX>(c.bJ, c.ncol, DMat{F.Lval + c.lval, 1, c.bJ}, bs);
    EpiScatter<1> ep{F.Uidx + c.cols, F.Lidx + c.rows, s, e, b, M, W};
    cta_tsgemm<NT, NMAX>(c.n_items, c.ncol, c.bJ, DMat{F.Uval + c.uval, c.bJ, 1}, bs, ep);
  }
  __syncthreads();   // bs is restaged by the next contributor
}

// split wide blocks: the item's line comes from the owner's per-item table; reductions
// into the global W of the block (several parts update it concurrently)
struct EpiScatterRed {
  const int *iline;        // line of output row i (this contributor's items)
  const int32_t *jkey;     // matrix index of output column j
  int s, b;
  double *W;
  __device__ __forceinline__ void operator()(int i, int j, double v) const {
    red_add_f64(&W[(int64_t)iline[i] * b + (jkey[j] - s)], -v);
  }
};

template <int SIDE, int NMAX>
__device__ void contrib_tsgemm_red(const DevFactor &F, int s, int b, const Contrib &c, const int *iline, double *W,
                                   double *bs) {
  if (SIDE == 0) {
    tsgemm_stage_b<NT, NMAX>(c.bJ, c.ncol, DMat{F.Uval + c.uval, 1, c.bJ}, bs);
    cta_tsgemm<NT, NMAX>(c.n_items, c.ncol, c.bJ, DMat{F.Lval + c.lval, c.bJ, 1}, bs,
                         EpiScatterRed{iline + c.item_off, F.Uidx + c.cols, s, b, W});
  } else {
    tsgemm_stage_b<NT, NMAX>(c.bJ, c.ncol, DMat{F.Lval + c.lval, 1, c.bJ}, bs);
    cta_tsgemm<NT, NMAX>(c.n_items, c.ncol, c.bJ, DMat{F.Uval + c.uval, c.bJ, 1}, bs,
                         EpiScatterRed{iline + c.item_off, F.Lidx + c.rows, s, b, W});
  }
  __syncthreads();
}

template <int SIDE>
__device__ void side_gemms(const DevFactor &F, int s, int e, int b, const Contrib *C, int nc, const LineMap &M,
                           double *W, double *gs) {
  for (int a = 0; a < nc; ++a) {
    const Contrib &c = C[a];
    if (c.n_items == 0 || c.ncol == 0) continue;
    if (c.ncol <= 64) contrib_tsgemm<SIDE, 64>(F, s, e, b, c, M, W, gs);
    else contrib_tsgemm<SIDE, 128>(F, s, e, b, c, M, W, gs);
  }
}


// ---------------------------------------------------------- split heavy blocks
// A block whose Schur-update item count is large is processed as several tasks of the
// dataflow queue: the owner CTA builds the candidate sets and a global-memory W
// (a-2..a-4) and publishes a HeavyCtx; "part" tasks apply disjoint item ranges with
// native global fp64 reductions (a-5) on any idle CTA; the CTA that completes the last
// part runs a-6..a-1 (finish_block).  Same values as the one-CTA path up to the
// summation order (R13).

// zone panels: unknown with path coordinate zdv in zone block T's panel
__device__ __forceinline__ int zone_loc(const DevFactor &F, int T, int zdv) { return F.zA[T] - zdv; }
__device__ __forceinline__ void zone_bit(unsigned *B, const DevFactor &F, int T, int zdv) {
  const int loc = zone_loc(F, T, zdv);
  atomicOr(&B[F.zwb[T] + (loc >> 5)], 1u << (loc & 31));
}
// local panel index -> unknown, from the run table of the block's path (shared memory)
__device__ __forceinline__ int zone_unknown(const int2 *runs, int nr, int z) {
  int r = nr - 1;
  while (r > 0 && runs[r].x > z) --r;
  return runs[r].y + (z - runs[r].x);
}

__device__ void finish_block(const DevFactor &F, int K, Shared &S, Bump &A, double *WL, double *WU, const int *rowOf,
                             const int *colOf, int nR, int nC, bool sortedR, bool sortedC, double flops,
                             HeavyCtx *X = nullptr, int mode = 0);

// a-1: release the blocks that wait for K (static adjacency of Ã + chain edges); K's writes
// are fenced by the caller
// The CTA keeps the first block it makes ready and runs it next (S.next), without a trip
// through the queue: a dependency chain advances on one SM as soon as its predecessor is
// done instead of waiting behind the blocks queued before it.
// Among the blocks K makes ready, the CTA keeps the one with the largest etree subtree (the
// one nearest the root: the long dependency chains run through the separators) and pushes
// the others.
// own: K's static adjacency and chain successors; extra[0 .. nex): further blocks whose
// pending count K holds (the early-release edges of process_zone_lean); last: K is done (the
// CTA keeps the best ready block as its continuation, K counts as finished), else every
// ready block goes to the queue (the CTA still has work for K)
__device__ void release_block(const DevFactor &F, int K, Shared &S, bool own = true, const int *extra = nullptr,
                              int nex = 0, bool last = true) {
  const int tid = threadIdx.x;
  const int a0 = F.adj_ptr[K], a1 = own ? F.adj_ptr[K + 1] : a0;
  const int nS = own ? __ldcg(&F.succ.cnt[K]) : 0;
  if (tid == 0) { S.cnt[0] = 0; S.off[0] = 0ull; }
  __syncthreads();
  int mine = -1;
  for (int x = tid; x < (a1 - a0) + nS + nex; x += NT) {
    int T = x < (a1 - a0) ? F.adj[a0 + x] : x < (a1 - a0) + nS ? __ldcg(list_rec(F.succ, K, x - (a1 - a0))) : extra[x - (a1 - a0) - nS];
    if (atomicSub(&F.pending[T], 1) == 1 && (F.owned == nullptr || F.owned[T])) {
      READY_MARK(T, K);
      if (!last) {
        unsigned long long slot = atomicAdd(&F.ctrl[CS * CTRL_QHEAD], 1ull);
        __threadfence();
        st_vol(&F.queue[slot], T);
      } else if (mine >= 0) {   // a thread that releases two keeps the better candidate, pushes the other
        const int worse = F.prio[mine] >= F.prio[T] ? T : mine;
        mine = worse == T ? mine : T;
        unsigned long long slot = atomicAdd(&F.ctrl[CS * CTRL_QHEAD], 1ull);
        __threadfence();
        st_vol(&F.queue[slot], worse);
      } else {
        mine = T;
      }
    }
  }
  if (mine >= 0) atomicMax(&S.off[0], ((unsigned long long)(unsigned)F.prio[mine] << 32) | (unsigned)mine);
  __syncthreads();
  const unsigned long long best = S.off[0];
  if (mine >= 0 && (best == 0ull || (int)(best & 0xffffffffu) != mine)) {
    unsigned long long slot = atomicAdd(&F.ctrl[CS * CTRL_QHEAD], 1ull);
    __threadfence();
    st_vol(&F.queue[slot], mine);
  }
  if (tid == 0 && last) {
    if (best != 0ull) S.next = (int)(best & 0xffffffffu);
    atomicAdd(&F.ctrl[CS * CTRL_DONE], 1ull);
  }
  __syncthreads();
}

// the destination line of every item of one side, into the global pool (split wide blocks)
template <int SIDE>
__device__ bool item_lines(const DevFactor &F, int K, int s, int e, const Contrib *C, int nc, int T, const LineMap &M,
                           Shared &S, int **out) {
  const int tid = threadIdx.x;
  const int32_t *cidx = SIDE == 0 ? F.Lidx : F.Uidx;
  const int64_t d = ((int64_t)T + 1) / 2 + 1;
  if (tid == 0) S.off[3] = atomicAdd(&F.ctrl[CS * CTRL_HPOOL], (unsigned long long)d);
  __syncthreads();
  const unsigned long long o = S.off[3];
  __syncthreads();
  if (o + d > (unsigned long long)F.hpool_cap) { if (tid == 0) raise_abort(F, DEV_OVF_HPOOL, K); return false; }
  int *il = (int *)(F.hpool + o);
  int a = contrib_of(C, nc, tid < T ? tid : 0);
  for (int t = tid; t < T; t += NT) {
    while (a + 1 < nc && C[a + 1].item_off <= t) ++a;
    const int i = t - C[a].item_off;
    const int key = cidx[(SIDE == 0 ? C[a].rows : C[a].cols) + i];
    il[t] = (SIDE == 0 && key < e) ? key - s : M(key);
  }
  __syncthreads();
  *out = il;
  return true;
}

__device__ void process_block(const DevFactor &F, int K, Shared &S, unsigned char *smem) {
  const int tid = threadIdx.x;
  const int s = F.bstart[K], e = F.bstart[K + 1], b = e - s;
  Bump A;
  A.sbase = smem; A.sused = 0; A.scap = F.smem_bytes; A.stop = F.smem_bytes;
  A.gbase = F.work + (size_t)blockIdx.x * F.work_per_cta; A.gused = 0; A.gcap = F.work_per_cta; A.gtop = F.work_per_cta;
  A.ovf = false; A.bottom_global = false; A.pool = false;
  PROF_T0
#define OVF_CHECK() do { if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; } } while (0)

  // ---------------- a-2: contributor lists (Lc: J with Ũ cols in K; Uc: J with L rows in K)
  const int nLc0 = __ldcg(&F.lc.cnt[K]), nUc0 = __ldcg(&F.uc.cnt[K]);
  Contrib *CL = (Contrib *)balloc(A, (int64_t)2 * nLc0 * sizeof(Contrib));
  Contrib *CU = (Contrib *)balloc(A, (int64_t)2 * nUc0 * sizeof(Contrib));
  int *tkeys = (int *)balloc(A, (int64_t)(nLc0 + nUc0 + 1) * 4);
  OVF_CHECK();
  load_contribs2(F, K, CL, CU, nLc0, nUc0, tkeys, S);
  const int nLc = nLc0, nUc = nUc0;
  const int TL = S.cnt[0], TU = S.cnt[1];
  const int64_t aL0 = F.AL_ptr[K], aLe = F.AL_ge[K], aL1 = F.AL_ptr[K + 1];
  const int64_t aU0 = F.AU_ptr[K], aU1 = F.AU_ptr[K + 1];
  const double flops = S.sflops[0] + S.sflops[1];
  const int maxbJ = max(S.maxbJ[0], S.maxbJ[1]);
  PROF(1);

  // ---------------- split decision: heavy blocks take their buffers from the global pool
  // split only when CTAs are idle (tickets taken but not yet filled)
  if (tid == 0) {
    const long long idle = (long long)ld_vol64(&F.ctrl[CS * CTRL_QTAIL]) - (long long)ld_vol64(&F.ctrl[CS * CTRL_QHEAD]);
    const int wide_ = b > 16 || maxbJ > 16;
    const bool big = F.heavy_T > 0 && (wide_ ? (S.sflops[0] + S.sflops[1] >= F.wide_flops) : (TL + TU >= F.heavy_T));
    // big blocks keep W in global memory (native fp64 reductions); they are split into
    // parts only when CTAs are idle, else this CTA applies every part itself
    S.cnt[3] = big ? ((idle >= F.heavy_idle ? 2 : 0) | 1) : 0;
  }
  __syncthreads();
  const bool heavy = (S.cnt[3] & 1) != 0;
  const bool publish = (S.cnt[3] & 2) != 0;
  // big blocks: W and the line maps in global memory -- the shared pool if the block is
  // split into parts (read by the helpers), else this CTA's reusable workspace
  if (heavy) { A.bottom_global = true; A.pool = publish; }

  // ---------------- a-3 / a-4 for both sides
  SideState RL, RU;
  RL.gbm = RU.gbm = nullptr; RL.gpre = RU.gpre = nullptr; RL.gl1 = RU.gl1 = nullptr; RL.gpre1 = RU.gpre1 = nullptr;
  const bool wide = b > 16 || maxbJ > 16;
  double *gs = nullptr;
  if (wide) {   // staging of the contributors' B operands (b_J <= 128 rows of TsB<128>::LDB)
    gs = (double *)balloc_top(A, (int64_t)max(maxbJ, 1) * TsB<128>::LDB * 8);
    OVF_CHECK();
  }
  bool both_ok = true;
  bool both = prepare_both(F, K, s, e, b, CL, nLc, TL, CU, nUc, TU, aL0, aLe, aL1, aU0, aU1, A, S, RL, RU, both_ok);
  if (!both_ok) return;
  if (!both) {
    both = prepare_both2(F, K, s, e, b, CL, nLc, TL, CU, nUc, TU, aL0, aLe, aL1, aU0, aU1, A, S, RL, RU, both_ok);
    if (!both_ok) return;
  }
  if (!both && !side_prepare<0>(F, K, s, e, b, CL, nLc, TL, aL0, aLe, aL1, A, S, RL)) return;
  PROF(2);
  int *ilineL = nullptr, *ilineU = nullptr;
  if (publish && wide) {   // the line of every item, so that the helpers need no line map
    if (!item_lines<0>(F, K, s, e, CL, nLc, TL, RL.M, S, &ilineL)) return;
  }
  // the pos-map candidate path (key ranges wider than the shared bitmap) keeps its line map
  // in a per-CTA global array that the other side's preparation reuses: apply this side's
  // updates first
  bool l_done = false;
  if (!both && !RL.sorted && !(publish && wide)) {
    if (wide) side_gemms<0>(F, s, e, b, CL, nLc, RL.M, RL.W, gs);
    else if (heavy) side_items<0, true>(F, s, e, CL, nLc, 0, TL, b, RL.M, RL.W);
    else side_items<0, false>(F, s, e, CL, nLc, 0, TL, b, RL.M, RL.W);
    __syncthreads();
    l_done = true;
  }
  if (!both && !side_prepare<1>(F, K, s, e, b, CU, nUc, TU, aU0, aU0, aU1, A, S, RU)) return;
  PROF(3);
  if (publish && wide) {
    if (!item_lines<1>(F, K, s, e, CU, nUc, TU, RU.M, S, &ilineU)) return;
  }

  if (publish && (wide || (RL.sorted && RU.sorted))) {
    // publish the context and the part tasks; this CTA is free afterwards
#ifdef BILU_PROFILE
    if (tid == 0 && g_blkprof) { g_blkprof[32 * (size_t)K + 19] = gtimer(); g_blkprof[32 * (size_t)K + 20] = ~0ull; }
#endif
    const int64_t cd = ((int64_t)(nLc + nUc) * (int64_t)sizeof(Contrib) + 7) / 8 + 2;
    if (tid == 0) S.off[3] = atomicAdd(&F.ctrl[CS * CTRL_HPOOL], (unsigned long long)cd);
    __syncthreads();
    if (S.off[3] + cd > (unsigned long long)F.hpool_cap) { if (tid == 0) raise_abort(F, DEV_OVF_HPOOL, K); return; }
    Contrib *gCL = (Contrib *)(F.hpool + S.off[3]);
    Contrib *gCU = gCL + nLc;
    for (int x = tid; x < nLc; x += NT) gCL[x] = CL[x];
    for (int x = tid; x < nUc; x += NT) gCU[x] = CU[x];
    int pL = min(MAX_PARTS / 2, (TL + F.part_items - 1) / F.part_items);
    int pU = min(MAX_PARTS / 2, (TU + F.part_items - 1) / F.part_items);
    if (wide) {   // parts = flop-balanced contributor ranges
      pL = (int)min((double)min(MAX_PARTS / 2, nLc), ceil(S.sflops[0] / F.wide_part_flops));
      pU = (int)min((double)min(MAX_PARTS / 2, nUc), ceil(S.sflops[1] / F.wide_part_flops));
      pL = max(pL, nLc > 0 ? 1 : 0); pU = max(pU, nUc > 0 ? 1 : 0);
    }
    __threadfence();   // W, the line maps and the contributor copies written by every thread
    __syncthreads();
    if (tid == 0) {
      const unsigned long long h = atomicAdd(&F.ctrl[CS * CTRL_HCTX], 1ull);
      if (h >= (unsigned long long)F.hctx_cap) { raise_abort(F, DEV_OVF_HCTX, K); S.off[1] = ~0ull; }
      else {
        HeavyCtx &X = F.hctx[h];
        X.K = K; X.nc[0] = nLc; X.nc[1] = nUc; X.T[0] = TL; X.T[1] = TU; X.np[0] = pL; X.np[1] = pU;
        X.C[0] = gCL; X.C[1] = gCU; X.R[0] = RL; X.R[1] = RU; X.flops = flops;
        X.R[0].M.bm = RL.gbm; X.R[0].M.pre = RL.gpre; X.R[1].M.bm = RU.gbm; X.R[1].M.pre = RU.gpre;
        X.R[0].M.l1 = RL.gl1; X.R[0].M.pre1 = RL.gpre1; X.R[1].M.l1 = RU.gl1; X.R[1].M.pre1 = RU.gpre1;
        X.wide = wide ? 1 : 0;
        X.iline[0] = ilineL; X.iline[1] = ilineU;
        if (wide) {
          for (int sd = 0; sd < 2; ++sd) {
            const Contrib *Cs = sd ? CU : CL;
            const int nc = sd ? nUc : nLc, np = sd ? pU : pL;
            const double tot = S.sflops[sd];
            int a = 0;
            double acc = 0.0;
            X.cb[sd][0] = 0;
            for (int p = 1; p < np; ++p) {
              const double goal = tot * p / np;
              while (a < nc && acc + 0.5 * 2.0 * Cs[a].bJ * (double)Cs[a].n_items * Cs[a].ncol < goal) {
                acc += 2.0 * Cs[a].bJ * (double)Cs[a].n_items * Cs[a].ncol;
                ++a;
              }
              X.cb[sd][p] = a;
            }
            X.cb[sd][np] = nc;
          }
        }
        X.left = pL + pU;
        __threadfence();
        const unsigned long long slot = atomicAdd(&F.ctrl[CS * CTRL_QHEAD], (unsigned long long)(pL + pU));
        if (slot + pL + pU > (unsigned long long)F.qcap) raise_abort(F, DEV_OVF_HCTX, K);
        else
          for (int p = 0; p < pL + pU; ++p) st_vol(&F.queue[slot + p], F.N + (int)h * TASK_STRIDE + p);
        S.off[1] = h;
      }
    }
    __syncthreads();
    return;
  }

  // ---------------- a-5, this CTA: every (contributor, item) pair
  if (wide) {
    if (!l_done) side_gemms<0>(F, s, e, b, CL, nLc, RL.M, RL.W, gs);
    side_gemms<1>(F, s, e, b, CU, nUc, RU.M, RU.W, gs);
  } else if (heavy) {
    if (!l_done) side_items<0, true>(F, s, e, CL, nLc, 0, TL, b, RL.M, RL.W);
    side_items<1, true>(F, s, e, CU, nUc, 0, TU, b, RU.M, RU.W);
  } else {
    if (!l_done) side_items<0, false>(F, s, e, CL, nLc, 0, TL, b, RL.M, RL.W);
    side_items<1, false>(F, s, e, CU, nUc, 0, TU, b, RU.M, RU.W);
  }
  __syncthreads();
  PROF(4);
  if (heavy) {   // finish scratch: shared memory from the start, the workspace after W (if W is there)
    A.sbase = smem; A.sused = 0; A.scap = F.smem_bytes; A.stop = F.smem_bytes; A.bottom_global = false;
    if (A.pool) {
      A.gbase = F.work + (size_t)blockIdx.x * F.work_per_cta; A.gused = 0; A.gcap = F.work_per_cta; A.gtop = F.work_per_cta;
    } else {
      A.gtop = A.gcap;
    }
    A.pool = false;
  } else {
    A.stop = A.scap; A.gtop = A.gcap;   // release the bitmaps / scratch
  }
  finish_block(F, K, S, A, RL.W, RU.W, RL.lineOf, RU.lineOf, RL.nU, RU.nU, RL.sorted, RU.sorted, flops);
#undef OVF_CHECK
}

// one scaling part of a wide split block: rows [r0, r1) of the candidates, L rows scaled by
// D_K from the right, U columns from the left (the trsm-equivalent of PAPER.md:210-212),
// with row maxima for the drop test; the CTA completing the last part finishes the block
__device__ void run_scale_part(const DevFactor &F, HeavyCtx &X, int p, Shared &S, unsigned char *smem) {
  const int tid = threadIdx.x;
  const int K = X.K;
  const int s = F.bstart[K], e = F.bstart[K + 1], b = e - s;
  const int nR = X.R[0].nU, nC = X.R[1].nU, tot = nR + nC;
  const int per = (tot + X.ns - 1) / X.ns;
  const int r0 = min(tot, p * per), r1 = min(tot, r0 + per);
  const double *D = F.D + F.D_off[K];
  double *bs = (double *)smem;
  const double *WL = X.R[0].W, *WU = X.R[1].W;
  // L rows [r0, min(r1, nR)): Lsc = W_L[b + i, :] D_K
  if (r0 < nR) {
    const int a = r0, z = min(r1, nR);
    if (b <= 64) {
      tsgemm_stage_b<NT, 64>(b, b, DMat{D, 1, b}, bs);
      cta_tsgemm<NT, 64>(z - a, b, b, DMat{WL + (int64_t)(b + a) * b, b, 1}, bs,
                         EpiAxpby{1.0, 0.0, X.Lsc + (int64_t)a * b, b, 1}, X.Lmx + a);
    } else {
      tsgemm_stage_b<NT, 128>(b, b, DMat{D, 1, b}, bs);
      cta_tsgemm<NT, 128>(z - a, b, b, DMat{WL + (int64_t)(b + a) * b, b, 1}, bs,
                          EpiAxpby{1.0, 0.0, X.Lsc + (int64_t)a * b, b, 1}, X.Lmx + a);
    }
    __syncthreads();
  }
  if (r1 > nR) {
    const int a = max(r0, nR) - nR, z = r1 - nR;
    if (b <= 64) {
      tsgemm_stage_b<NT, 64>(b, b, DMat{D, b, 1}, bs);
      cta_tsgemm<NT, 64>(z - a, b, b, DMat{WU + (int64_t)a * b, b, 1}, bs,
                         EpiAxpby{1.0, 0.0, X.Usc + (int64_t)a * b, b, 1}, X.Umx + a);
    } else {
      tsgemm_stage_b<NT, 128>(b, b, DMat{D, b, 1}, bs);
      cta_tsgemm<NT, 128>(z - a, b, b, DMat{WU + (int64_t)a * b, b, 1}, bs,
                          EpiAxpby{1.0, 0.0, X.Usc + (int64_t)a * b, b, 1}, X.Umx + a);
    }
    __syncthreads();
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) S.piv = atomicSub(&X.left2, 1);
  __syncthreads();
  if (S.piv != 1) return;
  __threadfence();
  Bump A;
  A.sbase = smem; A.sused = 0; A.scap = F.smem_bytes; A.stop = F.smem_bytes;
  A.gbase = F.work + (size_t)blockIdx.x * F.work_per_cta; A.gused = 0; A.gcap = F.work_per_cta; A.gtop = F.work_per_cta;
  A.ovf = false; A.bottom_global = false; A.pool = false;
  finish_block(F, K, S, A, X.R[0].W, X.R[1].W, X.R[0].lineOf, X.R[1].lineOf, nR, nC, X.sortedR != 0,
               X.sortedC != 0, X.flops, &X, 2);
}

// one part task: items of one side of a split heavy block; the CTA that completes the
// last part finishes the block
__device__ void run_part(const DevFactor &F, int task, Shared &S, unsigned char *smem) {
  const int tid = threadIdx.x;
  const int h = (task - F.N) / TASK_STRIDE, p = (task - F.N) % TASK_STRIDE;
  if (p >= MAX_PARTS) { run_scale_part(F, F.hctx[h], p - MAX_PARTS, S, smem); return; }
  HeavyCtx &X = F.hctx[h];
  const int K = X.K;
  const int s = F.bstart[K], e = F.bstart[K + 1], b = e - s;
  const int side = p < X.np[0] ? 0 : 1;
  const int pp = side == 0 ? p : p - X.np[0], np = X.np[side], T = X.T[side];
  const int per = (T + np - 1) / np;
  const int t0 = min(T, pp * per), t1 = min(T, t0 + per);
  const SideState &R = X.R[side];
  const int nc = X.nc[side];
  Contrib *C = (Contrib *)smem;
  bool cs = false;
  if (X.wide) {
    // contributors [cb[pp], cb[pp+1]) of this side: one DMMA product each, reductions into W
    const int a0 = X.cb[side][pp], a1 = X.cb[side][pp + 1];
    int mb = 0;
    for (int a = a0; a < a1; ++a) mb = max(mb, X.C[side][a].bJ);
    // B staging: shared memory when it fits, else this CTA's global workspace
    double *bs = (int64_t)mb * TsB<128>::LDB * 8 <= (int64_t)F.smem_bytes ? (double *)smem
                                                                          : F.work + (size_t)blockIdx.x * F.work_per_cta;
#ifdef BILU_PROFILE
    if (tid == 0 && g_blkprof) {
      atomicMin(&g_blkprof[32 * (size_t)K + 20], gtimer());
      atomicAdd(&g_blkprof[32 * (size_t)K + 22], 1ull);
    }
#endif
    for (int a = a0; a < a1; ++a) {
      const Contrib c = X.C[side][a];
      if (c.n_items == 0 || c.ncol == 0) continue;
      if (side == 0) {
        if (c.ncol <= 64) contrib_tsgemm_red<0, 64>(F, s, b, c, X.iline[0], R.W, bs);
        else contrib_tsgemm_red<0, 128>(F, s, b, c, X.iline[0], R.W, bs);
      } else {
        if (c.ncol <= 64) contrib_tsgemm_red<1, 64>(F, s, b, c, X.iline[1], R.W, bs);
        else contrib_tsgemm_red<1, 128>(F, s, b, c, X.iline[1], R.W, bs);
      }
    }
#ifdef BILU_PROFILE
    __syncthreads();
    if (tid == 0 && g_blkprof) atomicMax(&g_blkprof[32 * (size_t)K + 21], gtimer());
#endif
  } else {
  // the contributor descriptors of this side, staged in shared memory
  cs = (int64_t)nc * (int64_t)sizeof(Contrib) <= (int64_t)F.smem_bytes;
  if (cs) for (int x = tid; x < nc; x += NT) C[x] = X.C[side][x];
  __syncthreads();
#ifdef BILU_PROFILE
  if (tid == 0 && g_blkprof) {
    const unsigned long long t = gtimer();
    atomicMin(&g_blkprof[32 * (size_t)K + 20], t);            // first part start (buffer zeroed: use ~0 init)
    atomicAdd(&g_blkprof[32 * (size_t)K + 22], 1ull);
  }
  long long _pc0 = clock64();
#endif
  if (side == 0) side_items<0, true>(F, s, e, cs ? C : X.C[0], nc, t0, t1, b, R.M, R.W);
  else side_items<1, true>(F, s, e, cs ? C : X.C[1], nc, t0, t1, b, R.M, R.W);
#ifdef BILU_PROFILE
  __syncthreads();
  if (tid == 0 && g_blkprof) {
    atomicMax(&g_blkprof[32 * (size_t)K + 21], gtimer());     // last part end
    atomicAdd(&g_blkprof[32 * (size_t)K + 23], (unsigned long long)(clock64() - _pc0));   // part cycles
  }
#endif
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) S.piv = atomicSub(&X.left, 1);
  __syncthreads();
  if (S.piv != 1) return;
  __threadfence();
  Bump A;
  A.sbase = smem; A.sused = 0; A.scap = F.smem_bytes; A.stop = F.smem_bytes;
  A.gbase = F.work + (size_t)blockIdx.x * F.work_per_cta; A.gused = 0; A.gcap = F.work_per_cta; A.gtop = F.work_per_cta;
  A.ovf = false; A.bottom_global = false; A.pool = false;
  // stage the finished buffers in shared memory when they fit in half of it
  double *WL = X.R[0].W, *WU = X.R[1].W;
  const int *rowOf = X.R[0].lineOf, *colOf = X.R[1].lineOf;
  const int nR = X.R[0].nU, nC = X.R[1].nU;
  const int64_t nwl = (int64_t)(b + nR) * b, nwu = (int64_t)nC * b;
  if ((nwl + nwu) * 8 + (int64_t)(b + nR + nC + 2) * 4 + 64 <= F.smem_bytes - 24 * 1024) {
    double *sWL = (double *)balloc(A, nwl * 8), *sWU = (double *)balloc(A, nwu * 8);
    int *sR = (int *)balloc(A, (int64_t)(b + nR + 1) * 4), *sC = (int *)balloc(A, (int64_t)(nC + 1) * 4);
    for (int64_t x = tid; x < nwl; x += NT) sWL[x] = __ldcg(WL + x);
    for (int64_t x = tid; x < nwu; x += NT) sWU[x] = __ldcg(WU + x);
    for (int x = tid; x < b + nR; x += NT) sR[x] = __ldcg(rowOf + x);
    for (int x = tid; x < nC; x += NT) sC[x] = __ldcg(colOf + x);
    __syncthreads();
    WL = sWL; WU = sWU; rowOf = sR; colOf = sC;
  }
  const int fmode = (X.wide && b > 16 && nR + nC >= F.scale_split) ? 1 : 0;
  finish_block(F, K, S, A, WL, WU, rowOf, colOf, nR, nC, X.R[0].sorted, X.R[1].sorted, X.flops, &X, fmode);
}

// Gauss-Jordan inverse for 8 < b <= BR with P_K held in registers: the first BR * G threads
// take part (G = 4 column groups, named barrier 1); thread t owns row i = t % BR and the
// columns g*RP .. g*RP+RP-1 of it (g = t / BR), so lanes run over rows and every shared-memory
// access is conflict-free (column-major P) or a broadcast (a row).  Each step k reads the
// matrix of step k-1 from one of two shared copies (P and P + b^2, ping-pong) and writes its
// updated entries to the other, so one barrier per step suffices; the update is branch-free
// (rows k and bi, swapped, are patched afterwards).  The pivot of step k (argmax_{i>=k}
// |a_ik|, ties -> lowest row, R6) comes from the per-warp maxima (signed value, row) that the
// owners of column k reduced with shuffles at the end of step k-1.  Same arithmetic as the
// shared-memory version below.  P: 2 b^2 doubles; pv: >= 8 doubles.
template <int BR, int RP>
__device__ bool gj_invert_reg(double *P, int b, int *ipiv, double *fcol, double *pv, Shared &S) {
  // P and pv are in shared memory (checked by the caller), P with room for 2 BR^2 doubles: the
  // elimination runs on diag(P_K, I) padded to BR x BR (leading dimension BR), so every shared
  // access has a compile-time offset from one per-thread base and needs no bounds check (the
  // identity part never changes: its rows are 0 in the pivot columns and the pivot rows are 0
  // in its columns); 32-bit ld/st.shared instead of generic 64-bit pointer arithmetic
  constexpr int G = 4, NTH = BR * G, NWS = BR / 32;   // warps per column group
  constexpr unsigned CST = 8u * BR;                     // bytes between columns
  static_assert(G * RP == BR && NTH <= NT && BR % 32 == 0, "shape");
  const int tid = threadIdx.x, i = tid % BR, g = tid / BR, c0 = g * RP, lane = tid & 31;
  const unsigned sP = (unsigned)__cvta_generic_to_shared(P), sV = (unsigned)__cvta_generic_to_shared(pv);
  const unsigned buf1 = sP + 8u * BR * BR;
  auto lds = [](unsigned a) { double v; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory"); return v; };
  auto sts = [](unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory"); };
  auto ldsi = [](unsigned a) { int v; asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory"); return v; };
  auto stsi = [](unsigned a, int v) { asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); };
  if (tid < NTH) {
    const bool act = i < b;
    double x[RP];
#pragma unroll
    for (int u = 0; u < RP; ++u)
      x[u] = (act && c0 + u < b) ? lds(sP + 8u * (unsigned)(i + (c0 + u) * b)) : (i == c0 + u ? 1.0 : 0.0);
    // warp maxima of column col over rows >= from (owners of col only; whole warps): exact
    // argmax of |v|, lowest row on ties, by two integer max-reductions of the 64-bit key
    // bits(|v|) + 1 (0: not a candidate; the bits of a non-negative double order like its value)
    auto publish = [&](int col, int from) {
      double v = 0.0;
#pragma unroll
      for (int u = 0; u < RP; ++u) if (c0 + u == col) v = x[u];
      const unsigned long long key = (act && i >= from) ? (unsigned long long)__double_as_longlong(fabs(v)) + 1ull : 0ull;
      const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      const int w = __ffs(__ballot_sync(0xffffffffu, hi == mh && lo == ml)) - 1;
      const double vw = __shfl_sync(0xffffffffu, v, w);
      if (lane == 0) {
        const bool none = (mh | ml) == 0u;
        const unsigned slot = sV + 8u * (unsigned)((col & 1) * 2 * NWS);
        sts(slot + 8u * (i / 32), none ? 0.0 : vw);
        stsi(slot + 8u * NWS + 4u * (i / 32), none ? INT_MAX : i + w);
      }
    };
    asm volatile("bar.sync 1, %0;" ::"r"(NTH) : "memory");   // P read into registers before the padded copy
    {
      const unsigned my = sP + 8u * i + CST * c0;
#pragma unroll
      for (int u = 0; u < RP; ++u) sts(my + CST * u, x[u]);
    }
    if (g == 0) publish(0, 0);
    asm volatile("bar.sync 1, %0;" ::"r"(NTH) : "memory");
    bool sing = false;
    for (int k = 0; k < b; ++k) {
      const unsigned cur = (k & 1) ? buf1 : sP;
      const unsigned nxt = (k & 1) ? sP : buf1;
      const unsigned slot = sV + 8u * (unsigned)((k & 1) * 2 * NWS);
      double vb = lds(slot), best = fabs(vb);
      int bi = ldsi(slot + 8u * NWS);
#pragma unroll
      for (int q = 1; q < NWS; ++q) {           // warps in row order: the first maximum wins
        const double vq = lds(slot + 8u * q);
        if (fabs(vq) > best) { best = fabs(vq); vb = vq; bi = ldsi(slot + 8u * NWS + 4u * q); }
      }
      if (!(best > 0.0)) { sing = true; break; }   // identical decision in every thread
      // every shared-memory read of the step before any write
      double pr[RP];
      {
        const unsigned rowbi = cur + 8u * bi + CST * c0;
#pragma unroll
        for (int u = 0; u < RP; ++u) pr[u] = lds(rowbi + CST * u);   // old row bi
      }
      const double aik = lds(cur + 8u * i + CST * k);
      const double d = 1.0 / vb;
#pragma unroll
      for (int u = 0; u < RP; ++u) pr[u] *= d;  // the new pivot row, scaled
      const bool kin = k / RP == g;             // this column group owns column k (warp-uniform)
      if (i == bi && i != k) {                  // row bi takes old row k (one lane)
        const double ckk = lds(cur + 8u * k + CST * k);
        const unsigned rowk = cur + 8u * k + CST * c0;
#pragma unroll
        for (int u = 0; u < RP; ++u) x[u] = (c0 + u == k) ? -ckk * d : fma(-ckk, pr[u], lds(rowk + CST * u));
      } else if (i == k) {                      // the pivot row (one lane)
#pragma unroll
        for (int u = 0; u < RP; ++u) x[u] = (c0 + u == k) ? d : pr[u];
      } else {
#pragma unroll
        for (int u = 0; u < RP; ++u) x[u] = fma(-aik, pr[u], x[u]);
        if (kin) {
#pragma unroll
          for (int u = 0; u < RP; ++u) if (c0 + u == k) x[u] = -aik * d;
        }
      }
      {
        const unsigned my = nxt + 8u * i + CST * c0;
#pragma unroll
        for (int u = 0; u < RP; ++u) sts(my + CST * u, x[u]);
      }
      if (k + 1 < b && (k + 1) / RP == g) publish(k + 1, k + 1);
      if (tid == 0) ipiv[k] = bi;
      asm volatile("bar.sync 1, %0;" ::"r"(NTH) : "memory");
    }
    if (!sing) {
      // undo the row interchanges as column interchanges, in reverse order: composite map
      if (tid == 0) {
        for (int jj = 0; jj < b; ++jj) fcol[2 * b + jj] = jj;
        for (int k = b - 1; k >= 0; --k) {
          const int pvk = ipiv[k];
          if (pvk != k) { const double t = fcol[2 * b + k]; fcol[2 * b + k] = fcol[2 * b + pvk]; fcol[2 * b + pvk] = t; }
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(NTH) : "memory");
      // column jd of the result = column fcol[2b + jd] of the eliminated matrix (in the copy
      // written last), back to P with leading dimension b: read into registers, then write
      const unsigned fin = (b & 1) ? buf1 : sP;
      double o[RP];
#pragma unroll
      for (int u = 0; u < RP; ++u) {
        const int jd = g + G * u;
        o[u] = (act && jd < b) ? lds(fin + 8u * i + CST * (unsigned)(int)fcol[2 * b + jd]) : 0.0;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(NTH) : "memory");
#pragma unroll
      for (int u = 0; u < RP; ++u) {
        const int jd = g + G * u;
        if (act && jd < b) sts(sP + 8u * (unsigned)(i + jd * b), o[u]);
      }
    }
    if (tid == 0) S.piv = sing ? 1 : 0;
  }
  __syncthreads();
  return S.piv != 0;
}

// Blocked Gauss-Jordan inverse for 8 < b <= 64 (same pivot rule and the same elementary steps
// as the unblocked versions, R6).  The b steps run in panels of NB columns:
// warp 0 holds the panel (rows lane and lane + 32, NB columns in registers) and runs its NB
// steps with shuffles only -- pivot search, row interchange, the in-place elimination -- while
// tracking the composite row permutation src of the panel's interchanges.  Every other column j
// (earlier transform columns and later matrix columns) sees the panel's steps as one product
// T = (I + Q) Pi: column j becomes Pi a_j + Q (Pi a_j)[panel rows], where Q = (final panel
// columns) - (identity columns) -- the in-place stored panel column k equals (I + Q) e_k (the
// later interchanges of the panel do not move e_k).  All threads apply that rank-NB update,
// reading the matrix before the panel from one shared copy and writing the other (ping-pong,
// one barrier per panel instead of one per step).  P: 2 b^2 doubles; fcol: 3 b doubles.
// Measured (tools/micro/gj_standalone.cu, one CTA): b = 64 93K cycles (unblocked register
// version 110K), b = 33 46K (60K); a panel step costs ~1,000 cycles of one warp's dependent
// chain (pivot reductions, row shuffles, the division, the update).  A depth-1 lookahead
// (trailing update by the other warps during the next panel) was slower (b = 64 100K).
// Off by default: faster alone (above) but slower inside factor_kernel -- c4 136.5 -> 143.4 ms
// in an interleaved A/B (tools/ab_cfg.sh, profiles/r02_gj_blocked.md).  -DBILU_GJ_BLK_MIN=33
// switches it on for b >= 33.
#ifndef BILU_GJ_BLK_MIN
#define BILU_GJ_BLK_MIN 1000
#endif
template <int NB>
__device__ bool gj_invert_blk(double *P, int b, int *ipiv, double *fcol, Shared &S) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int *src = (int *)fcol;                       // b ints (fcol[0 .. b/2]); fcol[2b .. 3b) below
  const unsigned sP = (unsigned)__cvta_generic_to_shared(P);
  auto lds = [](unsigned a) { double v; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory"); return v; };
  auto sts = [](unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory"); };
  const unsigned CB = 8u * (unsigned)b;         // bytes between columns
  unsigned cur = sP, nxt = sP + 8u * (unsigned)(b * b);
  for (int p = 0; p < b; p += NB) {
    const int nbp = min(NB, b - p);
    if (wid == 0) {
      const int r0 = lane, r1 = lane + 32;
      const bool v0 = r0 < b, v1 = r1 < b;
      double x0[NB], x1[NB];
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        x0[u] = (v0 && u < nbp) ? lds(cur + 8u * r0 + CB * (unsigned)(p + u)) : 0.0;
        x1[u] = (v1 && u < nbp) ? lds(cur + 8u * r1 + CB * (unsigned)(p + u)) : 0.0;
      }
      int s0 = r0, s1 = r1;
      bool sing = false;
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        if (u < nbp && !sing) {
          const int k = p + u;
          // argmax_{i >= k} |a_ik|, lowest row on ties: exact max of the 64-bit key
          // bits(|v|) + 1 by two integer reductions, then the lowest row holding it
          const double a0 = fabs(x0[u]), a1 = fabs(x1[u]);
          const bool c0 = v0 && r0 >= k, c1 = v1 && r1 >= k;
          const unsigned long long k0 = c0 ? (unsigned long long)__double_as_longlong(a0) + 1ull : 0ull;
          const unsigned long long k1 = c1 ? (unsigned long long)__double_as_longlong(a1) + 1ull : 0ull;
          const unsigned long long kl = k1 > k0 ? k1 : k0;
          const int rl = k1 > k0 ? r1 : r0;
          const unsigned hi = (unsigned)(kl >> 32), lo = (unsigned)kl;
          const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
          const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
          const int bi = (int)__reduce_min_sync(0xffffffffu, (hi == mh && lo == ml && kl != 0ull) ? (unsigned)rl : 0x7fffffffu);
          const int lb = bi & 31, lk = k & 31;
          const bool sb = bi >= 32, sk = k >= 32;
          double pr[NB], rk[NB];
#pragma unroll
          for (int w = 0; w < NB; ++w) {
            pr[w] = __shfl_sync(0xffffffffu, sb ? x1[w] : x0[w], lb);
            rk[w] = __shfl_sync(0xffffffffu, sk ? x1[w] : x0[w], lk);
          }
          const int sbi = __shfl_sync(0xffffffffu, sb ? s1 : s0, lb);
          const int skk = __shfl_sync(0xffffffffu, sk ? s1 : s0, lk);
          const double vb = pr[u];
          if (!(fabs(vb) > 0.0)) { sing = true; continue; }   // warp-uniform
          const double d = 1.0 / vb, ckk = rk[u];
#pragma unroll
          for (int w = 0; w < NB; ++w) pr[w] *= d;
          auto step = [&](double (&x)[NB], int r, int &s) {
            if (r == k) {                         // the pivot row
#pragma unroll
              for (int w = 0; w < NB; ++w) x[w] = (w == u) ? d : pr[w];
              s = sbi;
            } else if (r == bi) {                 // takes old row k
#pragma unroll
              for (int w = 0; w < NB; ++w) x[w] = (w == u) ? -ckk * d : fma(-ckk, pr[w], rk[w]);
              s = skk;
            } else {
              const double aik = x[u];
#pragma unroll
              for (int w = 0; w < NB; ++w) x[w] = (w == u) ? -aik * d : fma(-aik, pr[w], x[w]);
            }
          };
          step(x0, r0, s0);
          step(x1, r1, s1);
          if (lane == 0) ipiv[k] = bi;
        }
      }
      if (!sing) {
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          if (u < nbp) {
            if (v0) sts(nxt + 8u * r0 + CB * (unsigned)(p + u), x0[u]);
            if (v1) sts(nxt + 8u * r1 + CB * (unsigned)(p + u), x1[u]);
          }
        }
        if (v0) src[r0] = s0;
        if (v1) src[r1] = s1;
      }
      if (lane == 0) S.piv = sing ? 1 : 0;
    }
    __syncthreads();
    if (S.piv) return true;
    // the other columns: new a_j = Pi a_j + Q (Pi a_j)[p .. p+nbp)
    {
      const int ng = NT / b, ncol = b - nbp;
      if (tid < ng * b) {
        const int i = tid % b, g = tid / b;
        const unsigned si = 8u * (unsigned)src[i];
        double q[NB];
        unsigned sp[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          q[u] = u < nbp ? lds(nxt + 8u * i + CB * (unsigned)(p + u)) - (i == p + u ? 1.0 : 0.0) : 0.0;
          sp[u] = u < nbp ? 8u * (unsigned)src[p + u] : 0u;
        }
        for (int jj = g; jj < ncol; jj += 2 * ng) {
          const bool two = jj + ng < ncol;
          const int j0 = jj < p ? jj : jj + nbp, j1t = jj + ng, j1 = j1t < p ? j1t : j1t + nbp;
          const unsigned c0 = cur + CB * (unsigned)j0, c1 = cur + CB * (unsigned)(two ? j1 : j0);
          double a0[NB], a1[NB];
          double acc0 = lds(c0 + si), acc1 = lds(c1 + si);
#pragma unroll
          for (int u = 0; u < NB; ++u) {
            a0[u] = u < nbp ? lds(c0 + sp[u]) : 0.0;
            a1[u] = u < nbp ? lds(c1 + sp[u]) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < NB; ++u) { acc0 = fma(q[u], a0[u], acc0); acc1 = fma(q[u], a1[u], acc1); }
          sts(nxt + 8u * (unsigned)i + CB * (unsigned)j0, acc0);
          if (two) sts(nxt + 8u * (unsigned)i + CB * (unsigned)j1, acc1);
        }
      }
    }
    __syncthreads();
    const unsigned t = cur; cur = nxt; nxt = t;
  }
  // undo the row interchanges as column interchanges, in reverse order: composite map
  if (tid == 0) {
    for (int jj = 0; jj < b; ++jj) fcol[2 * b + jj] = jj;
    for (int k = b - 1; k >= 0; --k) {
      const int pvk = ipiv[k];
      if (pvk != k) { const double t = fcol[2 * b + k]; fcol[2 * b + k] = fcol[2 * b + pvk]; fcol[2 * b + pvk] = t; }
    }
  }
  __syncthreads();
  // column jd of the result = column fcol[2b + jd] of the final copy, back to P (ld b)
  constexpr int MAXE = (64 * 64 + NT - 1) / NT;
  double o[MAXE];
#pragma unroll
  for (int e = 0; e < MAXE; ++e) {
    const int x = tid + e * NT;
    o[e] = x < b * b ? lds(cur + 8u * (unsigned)(x % b) + CB * (unsigned)(int)fcol[2 * b + x / b]) : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < MAXE; ++e) {
    const int x = tid + e * NT;
    if (x < b * b) sts(sP + 8u * (unsigned)x, o[e]);
  }
  __syncthreads();
  return false;
}

// D_K = P_K^{-1} in place (P column-major b x b in shared memory; b > 8 needs 2 b^2 doubles
// of P and 3 b of fcol), Gauss-Jordan with partial pivoting inside the block
// (ties -> lowest row, R6).  CTA-wide; returns true if a pivot is exactly 0.
__device__ __noinline__ bool gj_invert(double *P, int b, int *ipiv, double *fcol, Shared &S, bool reg = true) {
  if (reg && b >= BILU_GJ_BLK_MIN && b <= 64 && __isShared(P)) return gj_invert_blk<8>(P, b, ipiv, fcol, S);
  if (reg && b > 8 && b <= 64 && __isShared(P)) {
    __shared__ double pvbuf[8];
    if (b <= 32) return gj_invert_reg<32, 8>(P, b, ipiv, fcol, pvbuf, S);
    return gj_invert_reg<64, 16>(P, b, ipiv, fcol, pvbuf, S);
  }
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  bool singular = false;
  if (b <= 8) {
    // one warp, lane j holds column j of P_K in registers; pivot search by the lane
    // that owns column k, broadcasts by shuffles (pivoting inside
    // the block only; ties -> lowest row, R6)
    if (wid == 0) {
      double col[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) col[i] = (lane < b && i < b) ? P[i + lane * b] : 0.0;
      int piv_of[8];
      bool sing = false;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k < b && !sing) {
          // argmax_{i >= k} |a_ik| on lane k
          int bi = k; double best = -1.0;
#pragma unroll
          for (int i = 0; i < 8; ++i) if (i >= k && i < b) { const double v = fabs(col[i]); if (v > best) { best = v; bi = i; } }
          bi = __shfl_sync(0xffffffffu, bi, k);
          best = __shfl_sync(0xffffffffu, best, k);
          if (best == 0.0) { sing = true; }
          else {
            piv_of[k] = bi;
            // swap rows k and bi in every column
            double ck = 0.0, cb = 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i) { if (i == k) ck = col[i]; if (i == bi) cb = col[i]; }
#pragma unroll
            for (int i = 0; i < 8; ++i) { if (i == k) col[i] = cb; else if (i == bi) col[i] = ck; }
            // f_i = a_ik (column k, lane k), d = 1 / a_kk
            double f[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = __shfl_sync(0xffffffffu, col[i], k);
            const double d = 1.0 / f[k];
            const double pr = (lane == k) ? d : col[k] * d;
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (i != k) col[i] = ((lane == k) ? 0.0 : col[i]) - f[i] * pr;
            col[k] = pr;
          }
        }
      }
      if (!sing) {
        // undo the row interchanges as column interchanges, in reverse order
#pragma unroll
        for (int k = 7; k >= 0; --k) {
          if (k < b) {
            const int pv = piv_of[k];
            const int partner = (lane == k) ? pv : (lane == pv ? k : lane);
#pragma unroll
            for (int i = 0; i < 8; ++i) col[i] = __shfl_sync(0xffffffffu, col[i], partner);
          }
        }
        if (lane < b) {
#pragma unroll
          for (int i = 0; i < 8; ++i) if (i < b) P[i + lane * b] = col[i];
        }
      }
      if (lane == 0) S.piv = sing ? 1 : 0;
    }
    __syncthreads();
    singular = S.piv != 0;
  } else {
    // all warps; column j owned by warp j % NW (lanes over rows); the pivot column of step k
    // is read from a double buffer written by its owner at the end of step k-1, so one CTA
    // barrier per step suffices (P_K column-major in shared memory)
    double *cbuf = fcol;                         // 2 x b doubles
    if (wid == 0) for (int i = lane; i < b; i += 32) cbuf[i] = P[i];
    __syncthreads();
    bool sing = false;
    for (int k = 0; k < b; ++k) {
      const double *cb = cbuf + (k & 1) * b;
      double best = -1.0; int bi = k;
      for (int i = k + lane; i < b; i += 32) {
        const double v = fabs(cb[i]);
        if (v > best) { best = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, o);
        const int oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      best = __shfl_sync(0xffffffffu, best, 0);
      bi = __shfl_sync(0xffffffffu, bi, 0);
      if (best == 0.0) { sing = true; break; }     // identical decision in every warp
      if (tid == 0) ipiv[k] = bi;
      const double d = 1.0 / cb[bi];
      double *nb_ = cbuf + ((k + 1) & 1) * b;
      for (int j = wid; j < b; j += NW) {
        double *pc = P + (int64_t)j * b;
        if (bi != k && lane == 0) { const double t = pc[k]; pc[k] = pc[bi]; pc[bi] = t; }
        __syncwarp();
        const double pr = (j == k) ? d : pc[k] * d;
        for (int i = lane; i < b; i += 32) {
          if (i == k) continue;
          const double f = (i == bi) ? cb[k] : cb[i];          // column k after the row swap
          pc[i] = ((j == k) ? 0.0 : pc[i]) - f * pr;
        }
        __syncwarp();
        if (lane == 0) pc[k] = pr;
        __syncwarp();
        if (j == k + 1) for (int i = lane; i < b; i += 32) nb_[i] = pc[i];
      }
      __syncthreads();
    }
    if (!sing) {
      // undo the row interchanges as column interchanges, in reverse order: composite map
      if (tid == 0) {
        for (int j = 0; j < b; ++j) fcol[2 * b + j] = j;
        for (int k = b - 1; k >= 0; --k) {
          const int pv = ipiv[k];
          if (pv != k) { const double t = fcol[2 * b + k]; fcol[2 * b + k] = fcol[2 * b + pv]; fcol[2 * b + pv] = t; }
        }
      }
      __syncthreads();
      double *Q = P + (int64_t)b * b;              // permuted copy, then back
      for (int it = tid; it < b * b; it += NT) {
        const int i = it % b, j = it / b;
        Q[it] = P[i + (int64_t)(int)fcol[2 * b + j] * b];
      }
      __syncthreads();
      for (int it = tid; it < b * b; it += NT) P[it] = Q[it];
    }
    if (tid == 0) S.piv = sing ? 1 : 0;
    __syncthreads();
    singular = S.piv != 0;
  }
  return singular;
}

// Sec. 3.6 perturbation passes on the pivot block Pp (column-major, shared memory), lanes of
// warp 0 over columns / rows (R19): the largest entry of column j (the diagonal if
// 2|d_jj| >= |d_kj|) becomes d (1 + rho delta_j) + sign(d) tau_p alpha.  which: 0 = only zero
// columns then zero rows (returns whether any), 1 = every column then every row, 2 = sign-aware
// tau_p alpha on the diagonal.
__device__ bool perturb_pass(double *Pp, int b, int which, double alpha, double tp, double rho, Shared &S) {
  const int tid = threadIdx.x;
  if (tid == 0) S.cnt[3] = 0;
  __syncthreads();
  if (tid < 32) {
    if (which == 2) {
      for (int i = tid; i < b; i += 32) {
        double &d = Pp[i + (int64_t)i * b];
        d += (d < 0.0 ? -1.0 : 1.0) * tp * alpha;
      }
    } else {
      for (int j = tid; j < b; j += 32) {           // columns
        double dm = -1.0; int k = 0;
        for (int i = 0; i < b; ++i) { const double v = fabs(Pp[i + (int64_t)j * b]); if (v > dm) { dm = v; k = i; } }
        if (which == 0 && dm != 0.0) continue;
        if (2.0 * fabs(Pp[j + (int64_t)j * b]) >= fabs(Pp[k + (int64_t)j * b])) k = j;
        double &d = Pp[k + (int64_t)j * b];
        d = d * (1.0 + rho * dm) + (d < 0.0 ? -1.0 : 1.0) * tp * alpha;
        S.cnt[3] = 1;
      }
      __syncwarp();
      for (int i = tid; i < b; i += 32) {           // rows
        double dm = -1.0; int k = 0;
        for (int j = 0; j < b; ++j) { const double v = fabs(Pp[i + (int64_t)j * b]); if (v > dm) { dm = v; k = j; } }
        if (which == 0 && dm != 0.0) continue;
        if (2.0 * fabs(Pp[i + (int64_t)i * b]) >= fabs(Pp[i + (int64_t)k * b])) k = i;
        double &d = Pp[i + (int64_t)k * b];
        d = d * (1.0 + rho * dm) + (d < 0.0 ? -1.0 : 1.0) * tp * alpha;
        S.cnt[3] = 1;
      }
    }
  }
  __syncthreads();
  return S.cnt[3] != 0;
}

// |M|_1 (max column sum), warp 0, broadcast through shared memory
__device__ double norm1_cta(const double *M, int b, Shared &S) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    double best = 0.0;
    for (int j = tid; j < b; j += 32) {
      double sum = 0.0;
      for (int i = 0; i < b; ++i) sum += fabs(M[i + (int64_t)j * b]);
      best = fmax(best, sum);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (tid == 0) S.pivd = best;
  }
  __syncthreads();
  const double r = S.pivd;
  __syncthreads();
  return r;
}

// a-6 .. a-1 of block K once W_L (pivot block + candidate rows) and W_U are complete
__device__ void finish_block(const DevFactor &F, int K, Shared &S, Bump &A, double *WL, double *WU, const int *rowOf,
                             const int *colOf, int nR, int nC, bool sortedR, bool sortedC, double flops,
                             HeavyCtx *X, int mode) {
  const int tid = threadIdx.x;
  const int s = F.bstart[K], e = F.bstart[K + 1], b = e - s;
  PROF_T0C
#define OVF_CHECK() do { if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; } } while (0)
  // wide blocks: shared staging of D_K for the scaling products, reserved first so that it
  // stays in shared memory
  double *gsc = nullptr;
  if (b > 16) {
    gsc = (double *)balloc_top(A, (int64_t)b * (b <= 64 ? TsB<64>::LDB : TsB<128>::LDB) * 8);
    OVF_CHECK();
  }
  // mode 0: a-6 .. a-1 here.  mode 1 (wide split block): a-6, then the scaling of the
  // candidate rows / columns is published as parts.  mode 2: the parts are done, a-8 .. a-1.
  double *P = nullptr;
  if (mode == 2) goto scaled;
  {
  // ---------------- a-6: D_K = P_K^{-1}, Gauss-Jordan with partial pivoting (column-major P)
  // b in (8, 64]: room for the padded ping-pong copies of the register Gauss-Jordan
  P = (double *)balloc(A, (b <= 8 ? (int64_t)b * b : b <= 32 ? 2 * 32 * 32 : b <= 64 ? 2 * 64 * 64 : 2 * (int64_t)b * b) * 8);
  int *ipiv = (int *)balloc(A, (int64_t)b * 4);
  double *fcol = (double *)balloc(A, (int64_t)b * 8 * 3);
  OVF_CHECK();
  for (int i = tid; i < b * b; i += NT) {
    int rr = i % b, cc = i / b;
    P[i] = WL[(int64_t)rr * b + cc];
  }
  __syncthreads();
  bool singular;
  if (!F.perturb) {
    singular = gj_invert(P, b, ipiv, fcol, S);
  } else {
    // Sec. 3.6 (R19): zero columns / rows first; a singular or
    // ill-conditioned block (kappa_1 > cond_max) then gets every column and row perturbed,
    // then a diagonal shift; otherwise a breakdown
    double *Pp = (double *)balloc(A, (int64_t)b * b * 8);
    OVF_CHECK();
    for (int i = tid; i < b * b; i += NT) Pp[i] = P[i];
    __syncthreads();
    const double alpha = *F.alpha;
    bool changed = perturb_pass(Pp, b, 0, alpha, F.ptau, F.prho, S);
    singular = true;
    for (int stage = 0; stage < 3 && singular; ++stage) {
      if (stage > 0) { perturb_pass(Pp, b, stage, alpha, F.ptau, F.prho, S); changed = true; }
      for (int i = tid; i < b * b; i += NT) P[i] = Pp[i];
      __syncthreads();
      singular = gj_invert(P, b, ipiv, fcol, S);
      if (!singular) singular = norm1_cta(Pp, b, S) * norm1_cta(P, b, S) > F.cond_max;
    }
    if (!singular && changed && tid == 0) atomicAdd(&F.ctrl[CS * CTRL_NPERT], 1ull);
  }
  if (singular) {
    if (tid == 0) raise_abort(F, DEV_BREAKDOWN, K);
    return;
  }
  {
    double *Dg = F.D + F.D_off[K];
    for (int i = tid; i < b * b; i += NT) Dg[i] = P[i];
  }
  flops += 2.0 * b * b * (double)b + 2.0 * b * b * (double)(nR + nC);
  PROF(5);
  if (mode == 1) {
    // scale parts: rows [r0, r1) of the nR L candidates followed by the nC U candidates;
    // D_K is read back from F.D by every part (every thread's D writes fenced first)
    __threadfence();
    __syncthreads();
    const int64_t d = (int64_t)(nR + nC) * (b + 1) + 4;
    if (tid == 0) S.off[3] = atomicAdd(&F.ctrl[CS * CTRL_HPOOL], (unsigned long long)d);
    __syncthreads();
    if (S.off[3] + d > (unsigned long long)F.hpool_cap) { if (tid == 0) raise_abort(F, DEV_OVF_HPOOL, K); return; }
    if (tid == 0) {
      double *base = F.hpool + S.off[3];
      X->Lsc = base; X->Usc = base + (int64_t)nR * b;
      X->Lmx = base + (int64_t)(nR + nC) * b; X->Umx = X->Lmx + nR;
      X->ns = min(MAX_SPARTS, max(1, (nR + nC + F.scale_rows - 1) / F.scale_rows));
      X->left2 = X->ns;
      X->flops = flops;
      X->sortedR = sortedR; X->sortedC = sortedC;
      __threadfence();
      const unsigned long long slot = atomicAdd(&F.ctrl[CS * CTRL_QHEAD], (unsigned long long)X->ns);
      const int h = (int)(X - F.hctx);
      if (slot + X->ns > (unsigned long long)F.qcap) raise_abort(F, DEV_OVF_HCTX, K);
      else
        for (int p2 = 0; p2 < X->ns; ++p2) st_vol(&F.queue[slot + p2], F.N + h * TASK_STRIDE + MAX_PARTS + p2);
    }
    __syncthreads();
    return;
  }
  }
scaled:

  // ---------------- a-7/a-8: scale, drop (R1-R3), compact
  // L rows: l = w D_K, kept iff max|l| > tau; the scaled row overwrites W_L's row
  const double tau = F.tau;
  SUBP_T0
  int *keepR = (int *)balloc(A, (int64_t)(nR + 1) * 4);
  int *keepC = (int *)balloc(A, (int64_t)(nC + 1) * 4);
  OVF_CHECK();
  // wide blocks: the scaled candidates L_cand = W_L D_K and U_cand^T = Z^T D_K^T on the
  // FP64 tensor pipe (the trsm-equivalent of PAPER.md:788-790, 210-212)
  double *Lsc = nullptr, *Usc = nullptr, *Lmx = nullptr, *Umx = nullptr;
  if (mode == 2) {
    Lsc = X->Lsc; Usc = X->Usc; Lmx = X->Lmx; Umx = X->Umx;
  } else if (b > 16) {
    Lmx = (double *)balloc(A, (int64_t)nR * 8);
    Umx = (double *)balloc(A, (int64_t)nC * 8);
    Lsc = (double *)balloc(A, (int64_t)nR * b * 8);
    Usc = (double *)balloc(A, (int64_t)nC * b * 8);
    double *gs = gsc;
    if (b <= 64) {
      tsgemm_stage_b<NT, 64>(b, b, DMat{P, 1, b}, gs);
      cta_tsgemm<NT, 64>(nR, b, b, DMat{WL + (int64_t)b * b, b, 1}, gs, EpiAxpby{1.0, 0.0, Lsc, b, 1}, Lmx);
      __syncthreads();
      tsgemm_stage_b<NT, 64>(b, b, DMat{P, b, 1}, gs);
      cta_tsgemm<NT, 64>(nC, b, b, DMat{WU, b, 1}, gs, EpiAxpby{1.0, 0.0, Usc, b, 1}, Umx);
    } else {
      tsgemm_stage_b<NT, 128>(b, b, DMat{P, 1, b}, gs);
      cta_tsgemm<NT, 128>(nR, b, b, DMat{WL + (int64_t)b * b, b, 1}, gs, EpiAxpby{1.0, 0.0, Lsc, b, 1}, Lmx);
      __syncthreads();
      tsgemm_stage_b<NT, 128>(b, b, DMat{P, b, 1}, gs);
      cta_tsgemm<NT, 128>(nC, b, b, DMat{WU, b, 1}, gs, EpiAxpby{1.0, 0.0, Usc, b, 1}, Umx);
    }
    __syncthreads();
  }
  for (int i = tid; i < nR; i += NT) {
    double *w = WL + (int64_t)(b + i) * b;
    double mx = 0.0;
    if (b <= 8) {
      double wr[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) wr[t] = t < b ? w[t] : 0.0;     // the row once, into registers
      double l[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t) if (t < b && c < b) acc = fma(wr[t], P[t + c * b], acc);
        l[c] = acc;
        mx = fmax(mx, fabs(acc));
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) if (c < b) w[c] = l[c];
    } else if (b <= 16) {
      double wr[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) wr[t] = t < b ? w[t] : 0.0;
      double l[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < 16; ++t) if (t < b && c < b) acc = fma(wr[t], P[t + c * b], acc);
        l[c] = acc;
        mx = fmax(mx, fabs(acc));
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) if (c < b) w[c] = l[c];
    } else {
      mx = Lmx[i];
    }
    const int keep = mx > tau;
    keepR[i] = keep;
    if (tau > 0.0) {
      double margin = fabs(mx / tau - 1.0);
      if (margin <= F.near_rel) {
        unsigned long long slot = atomicAdd(&F.ctrl[CS * CTRL_NEAR], 1ull);
        if (slot < (unsigned long long)F.near_cap) {
          F.near_i[4 * slot] = K; F.near_i[4 * slot + 1] = 0;
          F.near_i[4 * slot + 2] = rowOf[b + i]; F.near_i[4 * slot + 3] = keep;
          F.near_m[slot] = margin;
        }
      }
    }
  }
  // U cols: u = D_K z, kept iff max|u| > tau; Ũ stores z (unscaled)
  for (int j = tid; j < nC; j += NT) {
    const double *z = WU + (int64_t)j * b;
    double mx = 0.0;
    if (b > 16) {
      mx = Umx[j];
    } else if (b <= 8) {
      double zr[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) zr[t] = t < b ? z[t] : 0.0;    // the column once, into registers
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t) if (t < b && rr < b) acc = fma(P[rr + t * b], zr[t], acc);
        mx = fmax(mx, fabs(acc));
      }
    } else {
      double zr[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) zr[t] = t < b ? z[t] : 0.0;
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < 16; ++t) if (t < b && rr < b) acc = fma(P[rr + t * b], zr[t], acc);
        mx = fmax(mx, fabs(acc));
      }
    }
    const int keep = mx > tau;
    keepC[j] = keep;
    if (tau > 0.0) {
      double margin = fabs(mx / tau - 1.0);
      if (margin <= F.near_rel) {
        unsigned long long slot = atomicAdd(&F.ctrl[CS * CTRL_NEAR], 1ull);
        if (slot < (unsigned long long)F.near_cap) {
          F.near_i[4 * slot] = K; F.near_i[4 * slot + 1] = 1;
          F.near_i[4 * slot + 2] = colOf[j]; F.near_i[4 * slot + 3] = keep;
          F.near_m[slot] = margin;
        }
      }
    }
  }
  __syncthreads();
  SUBP(11);
  const int mK = cta_scan(keepR, nR, S.tmp);
  const int cK = cta_scan(keepC, nC, S.tmp);
  SUBP(12);
  if (tid == 0) { keepR[nR] = mK; keepC[nC] = cK; }
  // kept rows / cols (buffer indices), then sorted by matrix index
  int *kr = (int *)balloc(A, (int64_t)(mK + 1) * 4);
  int *krow = (int *)balloc(A, (int64_t)(mK + 1) * 4);
  int *kc = (int *)balloc(A, (int64_t)(cK + 1) * 4);
  int *kcol = (int *)balloc(A, (int64_t)(cK + 1) * 4);
  int *R = (int *)balloc(A, (int64_t)(mK + 1) * 4);     // sorted kept rows
  int *Cs = (int *)balloc(A, (int64_t)(cK + 1) * 4);    // sorted kept cols
  int *ordR = (int *)balloc(A, (int64_t)(mK + 1) * 4);
  int *ordC = (int *)balloc(A, (int64_t)(cK + 1) * 4);
  OVF_CHECK();
  __syncthreads();
  for (int i = tid; i < nR; i += NT)
    if (keepR[i + 1] > keepR[i]) { kr[keepR[i]] = b + i; krow[keepR[i]] = rowOf[b + i]; }
  for (int j = tid; j < nC; j += NT)
    if (keepC[j + 1] > keepC[j]) { kc[keepC[j]] = j; kcol[keepC[j]] = colOf[j]; }
  __syncthreads();
  if (sortedR) {
    for (int x = tid; x < mK; x += NT) ordR[x] = x;
    __syncthreads();
  } else if (mK <= 1024) cta_rank_sort(krow, mK, ordR);
  else {
    // large: bitonic on (row << 0) keys carrying positions via a second pass
    for (int x = tid; x < mK; x += NT) R[x] = krow[x];
    __syncthreads();
    int m2 = 1; while (m2 < mK) m2 <<= 1;
    int *tmpk = (int *)balloc(A, (int64_t)m2 * 4);
    OVF_CHECK();
    for (int x = tid; x < m2; x += NT) tmpk[x] = x < mK ? R[x] : INT_MAX;
    __syncthreads();
    cta_bitonic(tmpk, m2);
    for (int x = tid; x < mK; x += NT) {
      const int r = lbound(tmpk, 0, mK, krow[x]);
      ordR[r] = x;
    }
    __syncthreads();
  }
  if (sortedC) {
    for (int x = tid; x < cK; x += NT) ordC[x] = x;
    __syncthreads();
  } else if (cK <= 1024) cta_rank_sort(kcol, cK, ordC);
  else {
    int m2 = 1; while (m2 < cK) m2 <<= 1;
    int *tmpk = (int *)balloc(A, (int64_t)m2 * 4);
    OVF_CHECK();
    for (int x = tid; x < m2; x += NT) tmpk[x] = x < cK ? kcol[x] : INT_MAX;
    __syncthreads();
    cta_bitonic(tmpk, m2);
    for (int x = tid; x < cK; x += NT) ordC[lbound(tmpk, 0, cK, kcol[x])] = x;
    __syncthreads();
  }
  SUBP(13);
  for (int x = tid; x < mK; x += NT) R[x] = krow[ordR[x]];
  for (int x = tid; x < cK; x += NT) Cs[x] = kcol[ordC[x]];
  if (tid < 5) {
    // 128-byte aligned slices: no L1 line is ever shared by two blocks' panels; the four
    // arena cursors are bumped by four threads at once (one round trip)
    const unsigned long long amt[5] = {((unsigned long long)mK + 31) & ~31ull,
                                       ((unsigned long long)mK * b + 15) & ~15ull,
                                       ((unsigned long long)cK + 31) & ~31ull,
                                       ((unsigned long long)cK * b + 15) & ~15ull,
                                       (unsigned long long)(nR + nC)};
    const int which[5] = {CTRL_CUR_LIDX, CTRL_CUR_LVAL, CTRL_CUR_UIDX, CTRL_CUR_UVAL, CTRL_NDEC};
    const unsigned long long o = atomicAdd(&F.ctrl[CS * which[tid]], amt[tid]);
    if (tid < 4) S.off[tid] = o;
  }
  __syncthreads();
  if (S.off[0] + mK > (unsigned long long)F.cap_Lidx || S.off[1] + (unsigned long long)mK * b > (unsigned long long)F.cap_Lval ||
      S.off[2] + cK > (unsigned long long)F.cap_Uidx || S.off[3] + (unsigned long long)cK * b > (unsigned long long)F.cap_Uval) {
    if (tid == 0) raise_abort(F, DEV_OVF_ARENA, K);
    return;
  }
  SUBP(14);
  const int64_t oLi = (int64_t)S.off[0], oLv = (int64_t)S.off[1], oUi = (int64_t)S.off[2], oUv = (int64_t)S.off[3];
  for (int x = tid; x < mK; x += NT) F.Lidx[oLi + x] = R[x];
  for (int it = tid; it < mK * b; it += NT) {
    const int x = it / b, c = it - x * b;
    if (b <= 16) F.Lval[oLv + it] = WL[(int64_t)kr[ordR[x]] * b + c];
    else F.Lval[oLv + it] = Lsc[(int64_t)(kr[ordR[x]] - b) * b + c];
  }
  for (int x = tid; x < cK; x += NT) F.Uidx[oUi + x] = Cs[x];
  for (int it = tid; it < cK * b; it += NT) {
    const int x = it / b;
    F.Uval[oUv + it] = WU[(int64_t)kc[ordC[x]] * b + (it - x * b)];
  }
  if (tid == 0) {
    F.Lrow_off[K] = oLi; F.Lm[K] = mK; F.Lval_off[K] = oLv;
    F.Ucol_off[K] = oUi; F.Uc[K] = cK; F.Uval_off[K] = oUv;
    F.blk_ncand[2 * K] = nR; F.blk_ncand[2 * K + 1] = nC;
  }
  __syncthreads();
  SUBP(15);
  PROF(6);

  // ---------------- a-2 (producer side): register K with the blocks it feeds,
  // and the chain edges of the readiness rule.
  // block of every kept row / column (sorted, so runs are contiguous)
  int *rb = (int *)balloc(A, (int64_t)(mK + cK + 1) * 4);
  int *cb = rb + mK;
  int *run = keepR;   // reuse: run-start flags of rows then columns, scanned together
  if (nR + 1 < mK + cK + 1) run = (int *)balloc(A, (int64_t)(mK + cK + 1) * 4);
  OVF_CHECK();
  for (int i = tid; i < mK; i += NT) rb[i] = F.block_of[R[i]];
  for (int j = tid; j < cK; j += NT) cb[j] = F.block_of[Cs[j]];
  __syncthreads();
  for (int i = tid; i < mK; i += NT) run[i] = (i == 0 || rb[i] != rb[i - 1]) ? 1 : 0;
  for (int j = tid; j < cK; j += NT) run[mK + j] = (j == 0 || cb[j] != cb[j - 1]) ? 1 : 0;
  __syncthreads();
  const int nRun = cta_scan(run, mK + cK, S.tmp);
  const int nRr = cK > 0 ? run[mK] : nRun, nCr = nRun - nRr;
  int *rstart = (int *)balloc(A, (int64_t)(nRr + 1) * 4);
  int *cstart = (int *)balloc(A, (int64_t)(nCr + 1) * 4);
  int *rblk = (int *)balloc(A, (int64_t)(nRr + 1) * 4);
  int *cblk = (int *)balloc(A, (int64_t)(nCr + 1) * 4);
  int *pdr = (int *)balloc(A, (int64_t)(nRr + 1) * 4);
  int *nb = (int *)balloc(A, (int64_t)(nRr + nCr + 1) * 4);
  OVF_CHECK();
  for (int i = tid; i < mK; i += NT)
    if (i == 0 || rb[i] != rb[i - 1]) { rstart[run[i]] = i; rblk[run[i]] = rb[i]; }
  for (int j = tid; j < cK; j += NT)
    if (j == 0 || cb[j] != cb[j - 1]) { cstart[run[mK + j] - nRr] = j; cblk[run[mK + j] - nRr] = cb[j]; }
  if (tid == 0) { rstart[nRr] = mK; cstart[nCr] = cK; }
  __syncthreads();
  // ---------------- dense trailing zone: push K's Schur update into the
  // panels of the zone blocks it feeds.  Every pair (i, j) of a kept row i and a kept column
  // j, both in the zone, receives -L_K[i, :] Ũ_K[:, j] ("gather ... GEMM ... scatter",
  // PAPER.md:371-374): in block column T = block(j) if T <= block(i), else in block row
  // block(i) -- the same products the Crout path applies when T is processed (each pair once,
  // at T = min(block(i), block(j))), in another summation order (R13).  Candidate bits: row
  // i of every zone column block T < block(i) of K's columns, column j of every zone row
  // block T < block(j) of K's rows (a-3: the union of the contributors' kept rows / columns).
  if (F.nzb > 0) {
    // K's kept rows / columns that are zone unknowns (with their path coordinates zd), and
    // its row / column runs that are zone blocks
    int *zx = (int *)balloc(A, (int64_t)(mK + cK + 2) * 4);
    int *zi = (int *)balloc(A, (int64_t)(mK + cK + 2) * 4);
    int *zrr = (int *)balloc(A, (int64_t)(nRr + nCr + 2) * 4);
    OVF_CHECK();
    if (tid == 0) { S.cnt[0] = 0; S.cnt[1] = 0; S.cnt[2] = 0; S.cnt[3] = 0; }
    __syncthreads();
    for (int x = tid; x < mK + cK; x += NT) {
      const int u = x < mK ? R[x] : Cs[x - mK];
      const int zl = F.zd[u];
      if (zl >= 0) {
        const int q = atomicAdd(&S.cnt[x < mK ? 0 : 1], 1);
        if (x < mK) { zx[q] = x; zi[q] = zl; }
        else { zx[mK + q] = x - mK; zi[mK + q] = zl; }
      }
    }
    for (int x = tid; x < nRr + nCr; x += NT) {
      const int T = x < nRr ? rblk[x] : cblk[x - nRr];
      if (F.zk[T] >= 0) {
        const int q = atomicAdd(&S.cnt[x < nRr ? 2 : 3], 1);
        if (x < nRr) zrr[q] = T; else zrr[nRr + q] = T;
      }
    }
    __syncthreads();
    const int nx = S.cnt[0], ny = S.cnt[1], nzr = S.cnt[2], nzc = S.cnt[3];
    __syncthreads();
    if (nx > 0 && ny > 0) {
      // products, one per (zone row, zone column) pair
      for (int p = tid; p < nx * ny; p += NT) {
        const int px = p / ny, py = p - px * ny;
        const int x = zx[px], y = zx[mK + py];
        const double *l = b <= 16 ? WL + (int64_t)kr[ordR[x]] * b : Lsc + (int64_t)(kr[ordR[x]] - b) * b;
        const double *u = WU + (int64_t)kc[ordC[y]] * b;
        double d0 = 0.0, d1 = 0.0;
        int t = 0;
        for (; t + 1 < b; t += 2) { d0 = fma(l[t], u[t], d0); d1 = fma(l[t + 1], u[t + 1], d1); }
        if (t < b) d0 = fma(l[t], u[t], d0);
        const int Ti = rb[x], Tj = cb[y];
        if (Tj <= Ti)
          red_add_f64(F.SL + (size_t)(F.zpb[Tj] + F.zA[Tj] - zi[px]) * 8 + (Cs[y] - F.bstart[Tj]), -(d0 + d1));
        else
          red_add_f64(F.SU + (size_t)(F.zpb[Ti] + F.zA[Ti] - zi[mK + py]) * 8 + (R[x] - F.bstart[Ti]), -(d0 + d1));
      }
      // candidate bits: zone row i in every zone column block T < block(i) of K's columns,
      // zone column j in every zone row block T < block(j) of K's rows (zone rows / columns
      // only meet zone blocks: the zone is closed under etree ancestors)
      for (int p = tid; p < nx * nzc; p += NT) {
        const int px = p / nzc, T = zrr[nRr + (p - px * nzc)];
        if (T < rb[zx[px]]) zone_bit(F.BL, F, T, zi[px]);
      }
      for (int p = tid; p < ny * nzr; p += NT) {
        const int py = p / nzr, T = zrr[p - py * nzr];
        if (T < cb[zx[mK + py]]) zone_bit(F.BU, F, T, zi[mK + py]);
      }
      if (tid == 0) atomicAdd((double *)&F.ctrl[CS * CTRL_FLOPS], 2.0 * b * (double)nx * (double)ny);
    }
  }
  for (int x = tid; x < nRr; x += NT) {
    const int T = rblk[x];
    const int p = lbound(cblk, 0, nCr, T);
    pdr[x] = (p < nCr && cblk[p] == T) ? 1 : 0;    // T is also a column block
  }
  __syncthreads();
  // N(K) = row blocks ∪ column blocks, both sorted: rank of v in the union =
  // #(rblk < v) + #(cblk < v) - #(common values < v)
  const int ndup = cta_scan(pdr, nRr, S.tmp);
  const int nN = nRr + nCr - ndup;
  for (int x = tid; x < nRr; x += NT) nb[x + lbound(cblk, 0, nCr, rblk[x]) - pdr[x]] = rblk[x];
  for (int y = tid; y < nCr; y += NT) {
    const int v = cblk[y], L = lbound(rblk, 0, nRr, v);
    if (L < nRr && rblk[L] == v) continue;
    nb[L + y - (L < nRr ? pdr[L] : ndup)] = v;
  }
  __syncthreads();
  // one parallel pass: register K in Uc(T) / Lc(T) of every run, and the readiness edges.
  // K's update can only create entries of a block T1 in a block T2 > T1 when one of them is
  // a row block and the other a column block of K (W_L[T2 rows, T1] -= L_K[T2 rows] Ũ_K[:, T1
  // cols], W_U[T1, T2 cols] -= L_K[T1 rows] Ũ_K[:, T2 cols]), so the exact
  // edges are the (row block, column block) pairs of N(K).  When there
  // are few of them they are added as such; otherwise the chain n_i -> n_{i+1} over N(K) --
  // whose transitive closure contains every pair -- keeps the edge count linear.
  const bool pairs = nRr * nCr <= F.pair_cap;
  const int nEdge = pairs ? nRr * nCr : max(nN - 1, 0);
  for (int x = tid; x < nRr + nCr + nEdge; x += NT) {
    if (x < nRr) {
      const int r0 = rstart[x], r1 = rstart[x + 1], T = rblk[x];
      if (F.nzb == 0 || F.zk[T] < 0) {   // zone targets read no contributor lists (their panels are pushed)
        int rec[REC_INTS] = {K, r0, r1, lbound(Cs, 0, cK, F.bstart[T + 1]), 0, 0, 0, 0};
        list_append(F, F.uc, T, rec);
      }
    } else if (x < nRr + nCr) {
      const int y = x - nRr;
      const int c0 = cstart[y], c1 = cstart[y + 1], T = cblk[y];
      if (F.nzb == 0 || F.zk[T] < 0) {
        int rec[REC_INTS] = {K, c0, c1, lbound(R, 0, mK, F.bstart[T]), lbound(R, 0, mK, F.bstart[T + 1]), 0, 0, 0};
        list_append(F, F.lc, T, rec);
      }
    } else if (pairs) {
      const int z = x - nRr - nCr, xr = z / nCr;
      const int r = rblk[xr], c = cblk[z - xr * nCr];
      if (r == c) continue;
      // a pair of two blocks that are both row and column blocks appears twice: keep r < c
      if (r > c) {
        const int pc = lbound(cblk, 0, nCr, r), pr = lbound(rblk, 0, nRr, c);
        if (pc < nCr && cblk[pc] == r && pr < nRr && rblk[pr] == c) continue;
      }
      const int lo = min(r, c), hi = max(r, c);
      atomicAdd(&F.pending[hi], 1);
      list_append(F, F.succ, lo, &hi);
    } else {
      const int z = x - nRr - nCr;
      atomicAdd(&F.pending[nb[z + 1]], 1);
      int rec1 = nb[z + 1];
      list_append(F, F.succ, nb[z], &rec1);
    }
  }
  if (tid == 0) { F.blk_flops[K] = flops; atomicAdd((double *)&F.ctrl[CS * CTRL_FLOPS], flops); }
  __threadfence();
  __syncthreads();
  PROF(7);

  // ---------------- a-1: release successors (static adjacency of Ã + chain edges)
  release_block(F, K, S);
  PROF(8);
  PROF_END(0, 0, nR, nC);
#undef OVF_CHECK
}

// The whole step of a narrow zone block (b <= 8, no perturbation, at most ZL_MAXLINES
// candidate lines) with few barriers and memory round trips: gather the panel (a-2..a-5,
// pushed by the contributors), a-6 pivot inverse, a-7/a-8 scaling, dropping and
// compaction, the push of K's own update into the zone, the chain edges of the readiness
// rule and a-1 the release.  Same arithmetic as process_zone_block + finish_block.
// Returns false (nothing consumed) if the block needs the general path.
constexpr int ZL_MAXLINES = 1024;
__device__ __forceinline__ int align16i(int x) { return (x + 15) & ~15; }

__device__ bool process_zone_lean(const DevFactor &F, int K, Shared &S, unsigned char *smem) {
  const int tid = threadIdx.x;
  const int s = F.bstart[K], e = F.bstart[K + 1], b = e - s;
  if (b > 8 || F.perturb) return false;
  const int k = F.zk[K];
  const int le = b;                                       // panel index of the first unknown >= e_K
  const int w0 = le >> 5, nw = ((F.zA[K] + 31) >> 5) - w0;
  const int rr0 = F.zrp[k], nrn = F.zrp[k + 1] - rr0;      // runs of K's etree path
  PROF_T0
  unsigned char *sp = smem;
  int2 *zr = (int2 *)sp; sp += align16i(nrn * 8);
  unsigned *bm = (unsigned *)sp; sp += align16i(2 * nw * 4);
  int *pre = (int *)sp; sp += align16i((2 * nw + 1) * 4);
  if ((int)(sp - smem) > F.smem_bytes) return false;
  unsigned *gL = F.BL + F.zwb[K] + w0, *gU = F.BU + F.zwb[K] + w0;
  for (int w = tid; w < 2 * nw; w += NT) {
    const unsigned m = __ldcg(w < nw ? gL + w : gU + (w - nw));
    bm[w] = m;
    pre[w] = __popc(m);
  }
  for (int x = tid; x < nrn; x += NT) zr[x] = F.zrun[rr0 + x];
  __syncthreads();
  const int tot = cta_scan(pre, 2 * nw, S.tmp);
  const int nR = nw > 0 ? pre[nw] : 0, nC = tot - nR;
  const int nL = b + nR, nl = nL + nC;
  // shared-memory plan: lines (panel indices, then unknowns), their path coordinates, W (8
  // doubles per line), flags / positions, D
  int *zl = (int *)sp; sp += align16i(nl * 4);
  int *zq = (int *)sp; sp += align16i(nl * 4);
  int *gb = (int *)sp; sp += align16i(nl * 4);                // block of every line
  int *fl = (int *)sp; sp += align16i((nR + nC + 1) * 4);      // keep flags -> kept positions
  int *kl = (int *)sp; sp += align16i((nR + nC + 1) * 4);      // kept lines (L then U)
  int *run = (int *)sp; sp += align16i((nR + nC + 2) * 4);     // row / column runs
  int *nb = (int *)sp; sp += align16i((nR + nC + 2) * 4);      // N(K)
  double *D = (double *)sp; sp += 64 * 8;
  int *ipiv = (int *)sp; sp += 64;
  double *fcol = (double *)sp; sp += 24 * 8;
  double *W = (double *)sp; sp += (size_t)nl * 64;
  if (nl > ZL_MAXLINES || (int)(sp - smem) > F.smem_bytes) return false;
  // committed: clear the bitmap words behind us
  for (int w = tid; w < 2 * nw; w += NT)
    if (bm[w]) *(w < nw ? gL + w : gU + (w - nw)) = 0u;
  for (int x = tid; x < b; x += NT) zl[x] = le - b + x;
  for (int w = tid; w < 2 * nw; w += NT) {
    unsigned m = bm[w];
    int at = w < nw ? b + pre[w] : nL + (pre[w] - nR);
    const int base = (w0 + (w < nw ? w : w - nw)) << 5;
    while (m) { const int bit = __ffs(m) - 1; zl[at++] = base + bit; m &= m - 1; }
  }
  __syncthreads();
  // gather the lines (64 B each, 16-byte loads, all in flight) and zero them behind
  for (int ln = tid; ln < nl; ln += NT) {
    double2 *src = (double2 *)((ln < nL ? F.SL : F.SU) + (size_t)(F.zpb[K] + zl[ln]) * 8);
    double2 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = __ldcg(src + q);
    const int u = zone_unknown(zr, nrn, zl[ln]);
    const int g = F.block_of[u];
    zl[ln] = u;
    zq[ln] = F.zd[u];
    double2 *dst = (double2 *)(W + (size_t)ln * 8);
#pragma unroll
    for (int q = 0; q < 4; ++q) { dst[q] = v[q]; src[q] = make_double2(0.0, 0.0); }
    gb[ln] = g;
  }
  __syncthreads();
  PROF(2);
  // a-6: D_K = P_K^{-1} (P column-major from the pivot lines; gj_invert: warp 0, R6)
  for (int x = tid; x < b * b; x += NT) D[x] = W[(x % b) * 8 + x / b];
  __syncthreads();
  if (gj_invert(D, b, ipiv, fcol, S)) { if (tid == 0) raise_abort(F, DEV_BREAKDOWN, K); return true; }
  {
    double *Dg = F.D + F.D_off[K];
    for (int x = tid; x < b * b; x += NT) Dg[x] = D[x];
  }
  PROF(5);
  // a-7/a-8: l = w D_K (kept iff max|l| > tau, stored scaled), u = D_K z (kept iff max|u| > tau,
  // Ũ stores z); near-threshold decisions logged (R1-R3, R15)
  const double tau = F.tau;
  for (int x = tid; x < nR + nC; x += NT) {
    const bool Lside = x < nR;
    double *w = W + (size_t)(Lside ? b + x : nL + (x - nR)) * 8;
    double wr[8], o[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) wr[t] = t < b ? w[t] : 0.0;
    double mx = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (t < b && c < b) acc = fma(wr[t], Lside ? D[t + c * b] : D[c + t * b], acc);
      o[c] = acc;
      mx = fmax(mx, fabs(acc));
    }
    if (Lside) {
#pragma unroll
      for (int c = 0; c < 8; ++c) if (c < b) w[c] = o[c];
    }
    const int keep = mx > tau;
    fl[x] = keep;
    if (tau > 0.0) {
      const double margin = fabs(mx / tau - 1.0);
      if (margin <= F.near_rel) {
        unsigned long long slot = atomicAdd(&F.ctrl[CS * CTRL_NEAR], 1ull);
        if (slot < (unsigned long long)F.near_cap) {
          F.near_i[4 * slot] = K; F.near_i[4 * slot + 1] = Lside ? 0 : 1;
          F.near_i[4 * slot + 2] = zl[Lside ? b + x : nL + (x - nR)]; F.near_i[4 * slot + 3] = keep;
          F.near_m[slot] = margin;
        }
      }
    }
  }
  __syncthreads();
  const int nk = cta_scan(fl, nR + nC, S.tmp);
  const int mK = nR > 0 ? (nC > 0 ? fl[nR] : nk) : 0, cK = nk - mK;
  for (int x = tid; x < nR + nC; x += NT) {
    const int nxt = x + 1 < nR + nC ? fl[x + 1] : nk;
    if (nxt > fl[x]) kl[fl[x]] = x < nR ? b + x : nL + (x - nR);
  }
  if (tid < 5) {
    const unsigned long long amt[5] = {((unsigned long long)mK + 31) & ~31ull, ((unsigned long long)mK * b + 15) & ~15ull,
                                       ((unsigned long long)cK + 31) & ~31ull, ((unsigned long long)cK * b + 15) & ~15ull,
                                       (unsigned long long)(nR + nC)};
    const int which[5] = {CTRL_CUR_LIDX, CTRL_CUR_LVAL, CTRL_CUR_UIDX, CTRL_CUR_UVAL, CTRL_NDEC};
    const unsigned long long o = atomicAdd(&F.ctrl[CS * which[tid]], amt[tid]);
    if (tid < 4) S.off[tid] = o;
  }
  __syncthreads();
  if (S.off[0] + mK > (unsigned long long)F.cap_Lidx || S.off[1] + (unsigned long long)mK * b > (unsigned long long)F.cap_Lval ||
      S.off[2] + cK > (unsigned long long)F.cap_Uidx || S.off[3] + (unsigned long long)cK * b > (unsigned long long)F.cap_Uval) {
    if (tid == 0) raise_abort(F, DEV_OVF_ARENA, K);
    return true;
  }
  const int64_t oLi = (int64_t)S.off[0], oLv = (int64_t)S.off[1], oUi = (int64_t)S.off[2], oUv = (int64_t)S.off[3];
  for (int x = tid; x < nk; x += NT) {
    const int ln = kl[x], g = zl[ln];
    if (x < mK) F.Lidx[oLi + x] = g; else F.Uidx[oUi + (x - mK)] = g;
  }
  for (int it = tid; it < nk * b; it += NT) {
    const int x = it / b, c = it - x * b;
    const double v = W[(size_t)kl[x] * 8 + c];
    if (x < mK) F.Lval[oLv + it] = v; else F.Uval[oUv + (it - mK * b)] = v;
  }
  if (tid == 0) {
    F.Lrow_off[K] = oLi; F.Lm[K] = mK; F.Lval_off[K] = oLv;
    F.Ucol_off[K] = oUi; F.Uc[K] = cK; F.Uval_off[K] = oUv;
    F.blk_ncand[2 * K] = nR; F.blk_ncand[2 * K + 1] = nC;
  }
  PROF(6);
  // runs of the kept rows / columns by block (sorted): run[r] = start of run r
  for (int x = tid; x < nk; x += NT) {
    const bool first = (x == 0 || x == mK) ? true : gb[kl[x]] != gb[kl[x - 1]];
    fl[x] = first ? 1 : 0;
  }
  __syncthreads();
  const int nrun = cta_scan(fl, nk, S.tmp);
  for (int x = tid; x < nk; x += NT) {
    const bool first = (x == 0 || x == mK) ? true : gb[kl[x]] != gb[kl[x - 1]];
    if (first) run[fl[x]] = x;
  }
  if (tid == 0) run[nrun] = nk;
  __syncthreads();
  const int nrr = mK > 0 ? (cK > 0 ? fl[mK] : nrun) : 0;     // row runs, then column runs
  // N(K): sorted union of the row-run and column-run blocks
  if (tid == 0) {
    int i = 0, j = nrr, q = 0;
    while (i < nrr || j < nrun) {
      const int vi = i < nrr ? gb[kl[run[i]]] : INT_MAX, vj = j < nrun ? gb[kl[run[j]]] : INT_MAX;
      const int v = min(vi, vj);
      nb[q++] = v;
      if (vi == v) ++i;
      if (vj == v) ++j;
    }
    S.cnt[0] = q;
    const double fl_ = 2.0 * b * b * (double)b + 2.0 * b * b * (double)(nR + nC) + 2.0 * b * (double)mK * (double)cK;
    F.blk_flops[K] = fl_;
    atomicAdd((double *)&F.ctrl[CS * CTRL_FLOPS], fl_);
  }
  __syncthreads();
  const int nN = S.cnt[0];
  // readiness: the chain edges n_z -> n_{z+1} of the readiness rule, and an edge K -> n_z for
  // every target, released below as soon as K's push into n_z is complete (every n_z waits
  // for K's release, so its pending count is > 0 here)
  for (int z = tid; z < nN; z += NT) {
    atomicAdd(&F.pending[nb[z]], 1);
    if (z + 1 < nN) {
      atomicAdd(&F.pending[nb[z + 1]], 1);
      int rec1 = nb[z + 1];
      list_append(F, F.succ, nb[z], &rec1);
    }
  }
  // push K's update into the zone (every kept row / column of a zone block is a zone unknown):
  // pair (x, y) goes to block column Tj if Tj <= Ti, else to block row Ti, i.e. to the target
  // min(Ti, Tj).  Every block K pushes into waits for its explicit edge K -> n_z.  The first
  // target n0 = min N(K) -- the next block of the dependency chain -- is pushed here by the
  // whole CTA (the rows in n0 times every column, every row times the columns in n0) and
  // released together with K's own edges (static adjacency, chain successors: they need
  // nothing more from K); the other targets go to a push task that any idle CTA runs from
  // K's stored factors (run_push_task), releasing each target when its pairs are complete.
  // This CTA continues with the next ready block ("early release").
  const int n0 = nN > 0 ? nb[0] : -1;
  const int r0 = (nrr > 0 && gb[kl[run[0]]] == n0) ? run[1] : 0;                // kept rows in n0
  const int c0 = (nrun > nrr && gb[kl[run[nrr]]] == n0) ? run[nrr + 1] - mK : 0;  // kept columns in n0
  {
    const int p1a = r0 * cK, p1 = p1a + (mK - r0) * c0;
    for (int p = tid; p < p1; p += NT) {
      int x, y;
      if (p < p1a) { x = p / cK; y = p - x * cK; }
      else { const int q = p - p1a; x = q / c0; y = q - x * c0; x += r0; }
      const int lx = kl[x], ly = kl[mK + y];
      const double *l = W + (size_t)lx * 8, *u = W + (size_t)ly * 8;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int t = 0; t < 8; t += 2) {
        if (t < b) d0 = fma(l[t], u[t], d0);
        if (t + 1 < b) d1 = fma(l[t + 1], u[t + 1], d1);
      }
      const int Ti = gb[lx], Tj = gb[ly];
      if (Tj <= Ti)
        red_add_f64(F.SL + (size_t)(F.zpb[Tj] + F.zA[Tj] - zq[lx]) * 8 + (zl[ly] - F.bstart[Tj]), -(d0 + d1));
      else
        red_add_f64(F.SU + (size_t)(F.zpb[Ti] + F.zA[Ti] - zq[ly]) * 8 + (zl[lx] - F.bstart[Ti]), -(d0 + d1));
    }
    // candidate bits of n0: the rows after n0 if n0 is a column block, the columns after n0
    // if n0 is a row block (a-3: the union of the contributors' kept rows / columns)
    if (c0 > 0) for (int x = r0 + tid; x < mK; x += NT) zone_bit(F.BL, F, n0, zq[kl[x]]);
    if (r0 > 0) for (int y = c0 + tid; y < cK; y += NT) zone_bit(F.BU, F, n0, zq[kl[mK + y]]);
  }
  __threadfence();
  __syncthreads();
  // the other targets: a push task (push_mode 1: high-priority queue, 2: main queue; 3: only if
  // CTAs are idle), else (push_mode 0) this CTA pushes them after releasing n0
  if (tid == 0) {
    bool task = nN > 1 && F.push_mode != 0;
    if (task && F.push_mode == 3)
      task = (long long)ld_vol64(&F.ctrl[CS * CTRL_QTAIL]) - (long long)ld_vol64(&F.ctrl[CS * CTRL_QHEAD]) >= 1;
    if (task) {   // published before any release
      if (F.push_mode == 1) enqueue_hi(F, -2 - K);
      else {
        const unsigned long long slot = atomicAdd(&F.ctrl[CS * CTRL_QHEAD], 1ull);
        __threadfence();
        st_vol(&F.queue[slot], -2 - K);
      }
    }
    S.cnt[2] = (nN > 1 && !task) ? 1 : 0;
  }
  __syncthreads();
  if (S.cnt[2]) {
    release_block(F, K, S, true, nb, 1, false);
    const int q1 = cK - c0;
    for (int p = tid; p < (mK - r0) * q1; p += NT) {
      const int x = r0 + p / q1, y = c0 + (p - (p / q1) * q1);
      const int lx = kl[x], ly = kl[mK + y];
      const double *l = W + (size_t)lx * 8, *u = W + (size_t)ly * 8;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int t = 0; t < 8; t += 2) {
        if (t < b) d0 = fma(l[t], u[t], d0);
        if (t + 1 < b) d1 = fma(l[t + 1], u[t + 1], d1);
      }
      const int Ti = gb[lx], Tj = gb[ly];
      if (Tj <= Ti)
        red_add_f64(F.SL + (size_t)(F.zpb[Tj] + F.zA[Tj] - zq[lx]) * 8 + (zl[ly] - F.bstart[Tj]), -(d0 + d1));
      else
        red_add_f64(F.SU + (size_t)(F.zpb[Ti] + F.zA[Ti] - zq[ly]) * 8 + (zl[lx] - F.bstart[Ti]), -(d0 + d1));
    }
    // candidate bits of the other targets: zone row i in every column-run block T (after n0)
    // with T < block(i); zone column j in every row-run block T (after n0) with T < block(j)
    {
      const int cr0 = nrr + (c0 > 0 ? 1 : 0), ncr = nrun - cr0, rb0 = r0 > 0 ? 1 : 0, nrb = nrr - rb0;
      for (int p = tid; p < mK * ncr; p += NT) {
        const int x = p / ncr, T = gb[kl[run[cr0 + (p - x * ncr)]]];
        if (T < gb[kl[x]]) zone_bit(F.BL, F, T, zq[kl[x]]);
      }
      for (int p = tid; p < cK * nrb; p += NT) {
        const int y = p / nrb, T = gb[kl[run[rb0 + (p - y * nrb)]]];
        if (T < gb[kl[mK + y]]) zone_bit(F.BU, F, T, zq[kl[mK + y]]);
      }
    }
    __threadfence();
    __syncthreads();
    PROF(7);
    release_block(F, K, S, false, nb + 1, nN - 1, true);
  } else {
    PROF(7);
    release_block(F, K, S, true, nb, nN > 0 ? 1 : 0, true);
  }
  PROF(8);
  PROF_END(0, 0, nR, nC);
  return true;
}

// The push of a finished zone block K into its targets n_1 .. n_{|N(K)|-1} (n_0 was pushed and
// released by K's own CTA, process_zone_lean): the same products, from K's stored factors --
// the kept rows of L_K (scaled, row-major) and the kept columns of Ũ_K -- each target pushed by
// one warp (n_z by warp z mod NW) and released by it when its pairs and candidate bits are
// complete (explicit edge K -> n_z).  No CTA barrier between targets.
__device__ void run_push_task(const DevFactor &F, int K, Shared &S, unsigned char *smem) {
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int s = F.bstart[K], b = F.bstart[K + 1] - s;
  const int mK = F.Lm[K], cK = F.Uc[K], nk = mK + cK;
  const int64_t oLi = F.Lrow_off[K], oLv = F.Lval_off[K], oUi = F.Ucol_off[K], oUv = F.Uval_off[K];
  int *gu = (int *)smem;            // unknown of kept row x / kept column mK + y
  int *gbk = gu + nk;               // ... its block
  int *gq = gbk + nk;               // ... its path coordinate
  int *fl = gq + nk;                // run-start flags -> run numbers
  int *run = fl + nk + 1;           // run starts (row runs, then column runs)
  int *nb = run + nk + 2;           // N(K)
  if ((int64_t)(6 * nk + 8) * 4 > F.smem_bytes) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; }
  for (int x = tid; x < nk; x += NT) {
    const int u = x < mK ? F.Lidx[oLi + x] : F.Uidx[oUi + (x - mK)];
    gu[x] = u; gbk[x] = F.block_of[u]; gq[x] = F.zd[u];
  }
  __syncthreads();
  for (int x = tid; x < nk; x += NT) fl[x] = (x == 0 || x == mK || gbk[x] != gbk[x - 1]) ? 1 : 0;
  __syncthreads();
  const int nrun = cta_scan(fl, nk, S.tmp);
  for (int x = tid; x < nk; x += NT)
    if (x == 0 || x == mK || gbk[x] != gbk[x - 1]) run[fl[x]] = x;
  if (tid == 0) run[nrun] = nk;
  __syncthreads();
  const int nrr = mK > 0 ? (cK > 0 ? fl[mK] : nrun) : 0;
  if (tid == 0) {
    int i = 0, j = nrr, q = 0;
    while (i < nrr || j < nrun) {
      const int vi = i < nrr ? gbk[run[i]] : INT_MAX, vj = j < nrun ? gbk[run[j]] : INT_MAX;
      const int v = min(vi, vj);
      nb[q++] = v;
      if (vi == v) ++i;
      if (vj == v) ++j;
    }
    S.cnt[0] = q;
  }
  __syncthreads();
  const int nN = S.cnt[0];
  const double *Lv = F.Lval + oLv, *Uv = F.Uval + oUv;
  auto rows_below = [&](int v) { int lo = 0, hi = mK; while (lo < hi) { const int m = (lo + hi) >> 1; if (gbk[m] < v) lo = m + 1; else hi = m; } return lo; };
  auto cols_below = [&](int v) { int lo = 0, hi = cK; while (lo < hi) { const int m = (lo + hi) >> 1; if (gbk[mK + m] < v) lo = m + 1; else hi = m; } return lo; };
  for (int z = 1 + wid; z < nN; z += NW) {
    const int T = nb[z];
    const int ra = rows_below(T), rb2 = rows_below(T + 1), ca = cols_below(T), cb2 = cols_below(T + 1);
    // pairs: rows in T x columns >= T, then rows after T x columns in T
    const int P1 = (rb2 - ra) * (cK - ca), P2 = (mK - rb2) * (cb2 - ca);
    for (int p = lane; p < P1 + P2; p += 32) {
      int x, y;
      if (p < P1) { const int w = cK - ca; x = p / w; y = ca + (p - x * w); x += ra; }
      else { const int q = p - P1, w = cb2 - ca; x = q / w; y = ca + (q - x * w); x += rb2; }
      const double *l = Lv + (int64_t)x * b, *u = Uv + (int64_t)y * b;
      double d0 = 0.0, d1 = 0.0;
      int t = 0;
      for (; t + 1 < b; t += 2) { d0 = fma(l[t], u[t], d0); d1 = fma(l[t + 1], u[t + 1], d1); }
      if (t < b) d0 = fma(l[t], u[t], d0);
      const int Ti = gbk[x], Tj = gbk[mK + y];
      if (Tj <= Ti)
        red_add_f64(F.SL + (size_t)(F.zpb[Tj] + F.zA[Tj] - gq[x]) * 8 + (gu[mK + y] - F.bstart[Tj]), -(d0 + d1));
      else
        red_add_f64(F.SU + (size_t)(F.zpb[Ti] + F.zA[Ti] - gq[mK + y]) * 8 + (gu[x] - F.bstart[Ti]), -(d0 + d1));
    }
    if (cb2 > ca) for (int x = rb2 + lane; x < mK; x += 32) zone_bit(F.BL, F, T, gq[x]);
    if (rb2 > ra) for (int y = cb2 + lane; y < cK; y += 32) zone_bit(F.BU, F, T, gq[mK + y]);
    __threadfence();
    __syncwarp();
    if (lane == 0 && atomicSub(&F.pending[T], 1) == 1) {
      READY_MARK(T, K);
      enqueue_hi(F, T);
    }
  }
  __syncthreads();
}

// a-2 .. a-5 of a block of the dense trailing zone: when the block is ready
// every contributor has pushed its update into the block's panel (finish_block), so the
// block gathers the candidate lines its bitmaps mark -- Ã's entries and the pushed
// products already summed -- zeroes them behind it (the zone buffers are all zero whenever
// no factorization runs), and continues with a-6 .. a-1.
__device__ void process_zone_block(const DevFactor &F, int K, Shared &S, unsigned char *smem) {
  const int tid = threadIdx.x;
  const int s = F.bstart[K], e = F.bstart[K + 1], b = e - s;
  const int k = F.zk[K];
  Bump A;
  A.sbase = smem; A.sused = 0; A.scap = F.smem_bytes; A.stop = F.smem_bytes;
  A.gbase = F.work + (size_t)blockIdx.x * F.work_per_cta; A.gused = 0; A.gcap = F.work_per_cta; A.gtop = F.work_per_cta;
  A.ovf = false; A.bottom_global = false; A.pool = false;
  PROF_T0
  const int le = b;                                      // panel index of the first unknown >= e_K
  const int w0 = le >> 5, nw = ((F.zA[K] + 31) >> 5) - w0; // bitmap words of the path unknowns >= e_K
  const int rr0 = F.zrp[k], nrn = F.zrp[k + 1] - rr0;      // runs of K's etree path
  unsigned *bm = (unsigned *)balloc_top(A, (int64_t)(2 * nw + 2) * 4);
  int *pre = (int *)balloc_top(A, (int64_t)(2 * nw + 2) * 4);
  int2 *zr = (int2 *)balloc_top(A, (int64_t)(nrn + 1) * 8);
  if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; }
  unsigned *gL = F.BL + F.zwb[K] + w0, *gU = F.BU + F.zwb[K] + w0;
  for (int x = tid; x < nrn; x += NT) zr[x] = F.zrun[rr0 + x];
  for (int w = tid; w < 2 * nw; w += NT) {
    unsigned *g = w < nw ? gL + w : gU + (w - nw);
    const unsigned m = __ldcg(g);
    bm[w] = m;
    pre[w] = __popc(m);
    if (m) *g = 0u;
  }
  __syncthreads();
  const int tot = cta_scan(pre, 2 * nw, S.tmp);
  const int nR = nw > 0 ? pre[nw] : 0, nC = tot - nR;
  double *WL = (double *)balloc(A, (int64_t)(b + nR) * b * 8);
  double *WU = (double *)balloc(A, (int64_t)nC * b * 8);
  int *zlL = (int *)balloc(A, (int64_t)(b + nR + 1) * 4);      // panel indices of the lines
  int *zlU = (int *)balloc(A, (int64_t)(nC + 1) * 4);
  int *lineL = (int *)balloc(A, (int64_t)(b + nR + 1) * 4);    // ... and the unknowns
  int *lineU = (int *)balloc(A, (int64_t)(nC + 1) * 4);
  if (A.ovf) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, K); return; }
  for (int x = tid; x < b; x += NT) zlL[x] = le - b + x;
  for (int w = tid; w < 2 * nw; w += NT) {
    unsigned m = bm[w];
    const bool u = w >= nw;
    int at = pre[w] - (u ? nR : 0);
    const int base = (w0 + (u ? w - nw : w)) << 5;
    while (m) {
      const int bit = __ffs(m) - 1;
      if (u) zlU[at++] = base + bit; else zlL[b + at++] = base + bit;
      m &= m - 1;
    }
  }
  __syncthreads();
  for (int x = tid; x < b + nR + nC; x += NT) {
    if (x < b + nR) lineL[x] = zone_unknown(zr, nrn, zlL[x]); else lineU[x - b - nR] = zone_unknown(zr, nrn, zlU[x - b - nR]);
  }
  // the lines (64 B each in the zone buffers), zeroed behind
  const int nl = (b + nR + nC) * b;
  for (int it = tid; it < nl; it += NT) {
    const int ln = it / b, c = it - ln * b;
    double *src;
    if (ln < b + nR) src = F.SL + (size_t)(F.zpb[K] + zlL[ln]) * 8 + c;
    else src = F.SU + (size_t)(F.zpb[K] + zlU[ln - b - nR]) * 8 + c;
    const double v = __ldcg(src);
    if (ln < b + nR) WL[it] = v; else WU[it - (b + nR) * b] = v;
    if (v != 0.0) *src = 0.0;
  }
  __syncthreads();
  PROF(2);
  A.stop = A.scap; A.gtop = A.gcap;   // release the bitmaps
  finish_block(F, K, S, A, WL, WU, lineL, lineU, nR, nC, true, true, 0.0);
}

__global__ void __launch_bounds__(NT, 1) factor_kernel(DevFactor F) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ Shared S;
  if (threadIdx.x == 0) { S.next = -1; S.ticket = ~0ull; }
  __syncthreads();
  while (true) {
    if (threadIdx.x == 0) {
#ifdef BILU_PROFILE
      long long _w0 = clock64();
#endif
      int K = -1;
      if (S.next >= 0) { K = S.next; S.next = -1; }                // continuation (release_block)
      else if (!try_dequeue_hi(F, K)) {
        // the main queue: hold a ticket (kept across high-priority items taken meanwhile)
        if (S.ticket == ~0ull && !aborted(F)) S.ticket = atomicAdd(&F.ctrl[CS * CTRL_QTAIL], 1ull);
        if (S.ticket < (unsigned long long)F.qcap) {
          unsigned ns = 32, polls = 0;
          while (true) {
            K = ld_vol(&F.queue[S.ticket]);
            if (K != -1) { S.ticket = ~0ull; break; }          // a block, a part task or a push task (<= -2)
            if (try_dequeue_hi(F, K)) break;
            if ((++polls & 15u) == 0 &&
                (aborted(F) || ld_vol64(&F.ctrl[CS * CTRL_DONE]) >= (unsigned long long)F.n_target)) { K = -1; break; }
            __nanosleep(ns);
            if (ns < 256) ns <<= 1;
          }
        } else {
          K = -1;
        }
      }
      S.K = K;
#ifdef BILU_PROFILE
      atomicAdd(&g_prof[0], (unsigned long long)(clock64() - _w0));
      if (K >= 0) atomicAdd(&g_prof[31], 1ull);
#endif
    }
    __syncthreads();
    const int K = S.K;
    if (K == -1) break;
    DBGK(K);
    __threadfence();
    if (K <= -2) {
      run_push_task(F, -2 - K, S, smem);
    } else if (K < F.N) {
      if (F.nzb > 0 && F.zk[K] >= 0) {
        if (!process_zone_lean(F, K, S, smem)) process_zone_block(F, K, S, smem);
      }
      else process_block(F, K, S, smem);
    } else {
      run_part(F, K, S, smem);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ distributed phases
// Multi-GPU factorization over the subtrees of a nested-dissection ordering (SURVEY.md
// 8(e)): phase A factors each rank's own subtree blocks (no communication: inside an ND
// subtree every contributor is a block of the same subtree); the ranks then exchange the
// panels of their "interface" blocks -- subtree blocks with kept L rows or Ũ columns in
// separator blocks, i.e. the operands of the separator Schur updates -- and phase B
// factors the separator blocks (replicated on every rank).  Before phase B the separator
// blocks' contributor lists, successor lists and pending counts are rebuilt from the
// interface blocks of all ranks (register_kernel) and the static separator adjacency.

// separator targets: empty contributor / successor lists, pending = static separator count
__global__ void sep_reset_kernel(DevFactor F, const int32_t *sep_list, int nsep, const int32_t *static_sep) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < nsep; x += gridDim.x * blockDim.x) {
    const int K = sep_list[x];
    F.lc.cnt[K] = 0; F.uc.cnt[K] = 0; F.succ.cnt[K] = 0;
    for (int d = 0; d < DIR_SLOTS; ++d) {
      F.lc.dir[(size_t)K * DIR_SLOTS + d] = -1;
      F.uc.dir[(size_t)K * DIR_SLOTS + d] = -1;
      F.succ.dir[(size_t)K * DIR_SLOTS + d] = -1;
    }
    F.pending[K] = static_sep[x];
  }
}

// register interface block J with the separator blocks it feeds (records of Lc/Uc, the
// same as finish_block's a-2) and the chain edges between consecutive separator blocks
// of N(J) (the readiness rule; the subtree blocks of N(J) are finished)
constexpr int REG_CAP = 4096;
__global__ void __launch_bounds__(NT) register_kernel(DevFactor F, const int32_t *blocks, int nb, const uint8_t *sep) {
  __shared__ int nbk[REG_CAP];
  __shared__ int flags[REG_CAP];
  __shared__ Shared S;
  const int tid = threadIdx.x;
  for (int x = blockIdx.x; x < nb; x += gridDim.x) {
    const int J = blocks[x];
    const int32_t *R = F.Lidx + F.Lrow_off[J];
    const int mK = F.Lm[J];
    const int32_t *Cs = F.Uidx + F.Ucol_off[J];
    const int cK = F.Uc[J];
    if (tid == 0) S.cnt[0] = 0;
    __syncthreads();
    for (int p = tid; p < mK; p += NT) {
      const int T = F.block_of[R[p]];
      if (!sep[T] || (p > 0 && F.block_of[R[p - 1]] == T)) continue;
      int r1 = p + 1;
      while (r1 < mK && F.block_of[R[r1]] == T) ++r1;
      int rec[REC_INTS] = {J, p, r1, lbound(Cs, 0, cK, F.bstart[T + 1]), 0, 0, 0, 0};
      list_append(F, F.uc, T, rec);
      const int slot = atomicAdd(&S.cnt[0], 1);
      if (slot < REG_CAP) nbk[slot] = T;
    }
    for (int p = tid; p < cK; p += NT) {
      const int T = F.block_of[Cs[p]];
      if (!sep[T] || (p > 0 && F.block_of[Cs[p - 1]] == T)) continue;
      int c1 = p + 1;
      while (c1 < cK && F.block_of[Cs[c1]] == T) ++c1;
      int rec[REC_INTS] = {J, p, c1, lbound(R, 0, mK, F.bstart[T]), lbound(R, 0, mK, F.bstart[T + 1]), 0, 0, 0};
      list_append(F, F.lc, T, rec);
      const int slot = atomicAdd(&S.cnt[0], 1);
      if (slot < REG_CAP) nbk[slot] = T;
    }
    __syncthreads();
    const int cnt = S.cnt[0];
    if (cnt > REG_CAP) { if (tid == 0) raise_abort(F, DEV_OVF_WORK, J); return; }
    const int nN = cta_sort_unique(nbk, cnt, flags, S.tmp);
    for (int z = tid; z + 1 < nN; z += NT) {
      atomicAdd(&F.pending[nbk[z + 1]], 1);
      int rec1 = nbk[z + 1];
      list_append(F, F.succ, nbk[z], &rec1);
    }
    __threadfence();
    __syncthreads();
  }
}

__global__ void sep_ready_kernel(DevFactor F, const int32_t *sep_list, int nsep) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < nsep; x += gridDim.x * blockDim.x) {
    const int K = sep_list[x];
    if (F.pending[K] == 0) {
      const unsigned long long slot = atomicAdd(&F.ctrl[CS * CTRL_QHEAD], 1ull);
      F.queue[slot] = K;
    }
  }
}

// own block J is an interface block iff its last kept row or column lies in a separator
// (rows / columns are sorted and the separators follow the subtree in the ND order)
__global__ void interface_flag_kernel(DevFactor F, const int32_t *own_list, int nown, const uint8_t *sep,
                                      uint8_t *flag) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < nown; x += gridDim.x * blockDim.x) {
    const int J = own_list[x];
    const int m = F.Lm[J], c = F.Uc[J];
    bool f = false;
    if (m > 0) f = f || sep[F.block_of[F.Lidx[F.Lrow_off[J] + m - 1]]];
    if (c > 0) f = f || sep[F.block_of[F.Uidx[F.Ucol_off[J] + c - 1]]];
    flag[x] = f ? 1 : 0;
  }
}

__global__ void pack_kernel(DevFactor F, const PackEntry *tab, int count, unsigned char *buf) {
  for (int x = blockIdx.x; x < count; x += gridDim.x) {
    const PackEntry e = tab[x];
    const int J = (int)e.J;
    int32_t *li = (int32_t *)(buf + e.offLi);
    int32_t *ui = (int32_t *)(buf + e.offUi);
    double *lv = (double *)(buf + e.offLv);
    double *uv = (double *)(buf + e.offUv);
    const int64_t lro = F.Lrow_off[J], lvo = F.Lval_off[J], uco = F.Ucol_off[J], uvo = F.Uval_off[J];
    for (int64_t i = threadIdx.x; i < e.Lm; i += blockDim.x) li[i] = F.Lidx[lro + i];
    for (int64_t i = threadIdx.x; i < e.Uc; i += blockDim.x) ui[i] = F.Uidx[uco + i];
    for (int64_t i = threadIdx.x; i < e.Lm * e.b; i += blockDim.x) lv[i] = F.Lval[lvo + i];
    for (int64_t i = threadIdx.x; i < e.Uc * e.b; i += blockDim.x) uv[i] = F.Uval[uvo + i];
  }
}

// remote interface blocks into this rank's arenas at base[4 x] = (Li, Lv, Ui, Uv) offsets
__global__ void unpack_kernel(DevFactor F, const unsigned char *buf, const PackEntry *tab, int count,
                              const int64_t *base) {
  for (int x = blockIdx.x; x < count; x += gridDim.x) {
    const PackEntry e = tab[x];
    const int J = (int)e.J;
    const int32_t *li = (const int32_t *)(buf + e.offLi);
    const int32_t *ui = (const int32_t *)(buf + e.offUi);
    const double *lv = (const double *)(buf + e.offLv);
    const double *uv = (const double *)(buf + e.offUv);
    const int64_t bLi = base[4 * x], bLv = base[4 * x + 1], bUi = base[4 * x + 2], bUv = base[4 * x + 3];
    for (int64_t i = threadIdx.x; i < e.Lm; i += blockDim.x) F.Lidx[bLi + i] = li[i];
    for (int64_t i = threadIdx.x; i < e.Uc; i += blockDim.x) F.Uidx[bUi + i] = ui[i];
    for (int64_t i = threadIdx.x; i < e.Lm * e.b; i += blockDim.x) F.Lval[bLv + i] = lv[i];
    for (int64_t i = threadIdx.x; i < e.Uc * e.b; i += blockDim.x) F.Uval[bUv + i] = uv[i];
    if (threadIdx.x == 0) {
      F.Lrow_off[J] = bLi; F.Lm[J] = (int32_t)e.Lm; F.Lval_off[J] = bLv;
      F.Ucol_off[J] = bUi; F.Uc[J] = (int32_t)e.Uc; F.Uval_off[J] = bUv;
    }
  }
}

extern "C" cudaError_t bilu_launch_sep_prepare(const DevFactor &F, const int32_t *sep_list, int nsep,
                                               const int32_t *static_sep, const int32_t *ifc, int nifc,
                                               const uint8_t *sep, cudaStream_t st) {
  if (nsep > 0) sep_reset_kernel<<<(nsep + 255) / 256, 256, 0, st>>>(F, sep_list, nsep, static_sep);
  if (nifc > 0) register_kernel<<<nifc < 1184 ? nifc : 1184, NT, 0, st>>>(F, ifc, nifc, sep);
  if (nsep > 0) sep_ready_kernel<<<(nsep + 255) / 256, 256, 0, st>>>(F, sep_list, nsep);
  return cudaGetLastError();
}

extern "C" cudaError_t bilu_launch_interface_flags(const DevFactor &F, const int32_t *own_list, int nown,
                                                   const uint8_t *sep, uint8_t *flag, cudaStream_t st) {
  if (nown > 0) interface_flag_kernel<<<(nown + 255) / 256, 256, 0, st>>>(F, own_list, nown, sep, flag);
  return cudaGetLastError();
}

extern "C" cudaError_t bilu_launch_pack(const DevFactor &F, const PackEntry *tab, int count, unsigned char *buf,
                                        cudaStream_t st) {
  if (count > 0) pack_kernel<<<count < 2048 ? count : 2048, 256, 0, st>>>(F, tab, count, buf);
  return cudaGetLastError();
}

extern "C" cudaError_t bilu_launch_unpack(const DevFactor &F, const unsigned char *buf, const PackEntry *tab,
                                          int count, const int64_t *base, cudaStream_t st) {
  if (count > 0) unpack_kernel<<<count < 2048 ? count : 2048, 256, 0, st>>>(F, buf, tab, count, base);
  return cudaGetLastError();
}

// Ã's entries inside the dense trailing zone into the zone panels, with their candidate
// bits ("load the associated scalar sparse columns of A into block column buffer",
// PAPER.md:370-371); the buffers are zero before (invariant kept by the zone blocks).
__global__ void zone_init_kernel(DevFactor F, const int32_t *zblocks) {
  for (int k = blockIdx.x; k < F.nzb; k += gridDim.x) {
    const int K = zblocks[k], e = F.bstart[K + 1];
    for (int64_t p = F.AL_ptr[K] + threadIdx.x; p < F.AL_ptr[K + 1]; p += blockDim.x) {
      const int rc = F.AL_rc[p], i = rc >> 7, zi = F.zd[i];
      F.SL[(size_t)(F.zpb[K] + zone_loc(F, K, zi)) * 8 + (rc & 127)] = F.AL_val[p];
      if (i >= e) zone_bit(F.BL, F, K, zi);
    }
    for (int64_t p = F.AU_ptr[K] + threadIdx.x; p < F.AU_ptr[K + 1]; p += blockDim.x) {
      const int rc = F.AU_rc[p], zj = F.zd[rc >> 7];
      F.SU[(size_t)(F.zpb[K] + zone_loc(F, K, zj)) * 8 + (rc & 127)] = F.AU_val[p];
      zone_bit(F.BU, F, K, zj);
    }
  }
}

extern "C" cudaError_t bilu_launch_zone_init(const DevFactor &F, const int32_t *zblocks, cudaStream_t st) {
  if (F.nzb > 0) zone_init_kernel<<<F.nzb < 4096 ? F.nzb : 4096, 128, 0, st>>>(F, zblocks);
  return cudaGetLastError();
}

// ----------------------------------------------------------------- launchers
extern "C" cudaError_t bilu_launch_factor(const DevFactor &F, int grid, cudaStream_t st) {
  cudaError_t err = cudaFuncSetAttribute(factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, F.smem_bytes);
  if (err != cudaSuccess) return err;
  // shared memory carve-out just large enough for the CTAs of one SM; the rest stays L1
  // (the Schur updates read contributor panels through L1)
  {
    int carve = 50;
    if (const char *cv = tune_env("BILU_CARVEOUT")) carve = atoi(cv);
    cudaFuncSetAttribute(factor_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  }
  factor_kernel<<<grid, NT, F.smem_bytes, st>>>(F);
  return cudaGetLastError();
}

extern "C" int bilu_heavyctx_size() { return (int)sizeof(HeavyCtx); }
extern "C" int bilu_max_parts() { return TASK_STRIDE; }

extern "C" cudaError_t bilu_factor_occupancy(int smem_bytes, int *blocks_per_sm) {
  cudaError_t err = cudaFuncSetAttribute(factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (err != cudaSuccess) return err;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, factor_kernel, NT, smem_bytes);
}

}  // namespace bilu

namespace bilu {
extern "C" int bilu_prof_set_blk(unsigned long long *dev_ptr) {
#ifdef BILU_PROFILE
  return cudaMemcpyToSymbol(g_blkprof, &dev_ptr, sizeof(dev_ptr)) == cudaSuccess;
#else
  (void)dev_ptr;
  return 0;
#endif
}
extern "C" int bilu_prof_read(unsigned long long *out, int reset) {
#ifdef BILU_PROFILE
  cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * 32);
  if (reset) { unsigned long long z[32] = {0}; cudaMemcpyToSymbol(g_prof, z, sizeof(z)); }
  return 1;
#else
  (void)out; (void)reset;
  return 0;
#endif
}
}
