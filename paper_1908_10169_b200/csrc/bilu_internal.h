// bilu_internal.h -- shared between the host orchestrator (bilu_host.cpp) and
// the sm_100a kernels (bilu_kernels.cu).  Not part of the public ABI.
#pragma once
#include <stdint.h>
#include <stdlib.h>
#include <vector_types.h>

// Tuning and diagnostic switches (BILU_HEAVY_T, BILU_SMEM_KB, BILU_DEBUG_TIMEOUT, ...) are
// read from the environment only in the builds of tools/ (-DBILU_TUNING, or the per-phase
// profiling build -DBILU_PROFILE).  The product library ignores the environment.
static inline const char *tune_env(const char *name) {
#if defined(BILU_TUNING) || defined(BILU_PROFILE)
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

namespace bilu {

// Records of the per-target contributor lists (replace the paper's
// L_head/L_list/L_first linked lists).  8 x int32.
//   Lc(T) entry: J has Ũ columns in T: {J, c0, c1, lrs, lre, 0, 0, 0}
//       c0..c1  = positions of J's kept columns inside T
//       lrs     = first position of J's kept rows >= s_T
//       lre     = first position of J's kept rows >= e_T
//   Uc(T) entry: J has L rows in T:    {J, r0, r1, cus, 0, 0, 0, 0}
//       r0..r1  = positions of J's kept rows inside T
//       cus     = first position of J's kept columns >= e_T
constexpr int REC_INTS = 8;
constexpr int CHUNK = 32;        // records per chunk of a chunked list
constexpr int DIR_SLOTS = 32;    // chunks per target -> 1024 records max

// error codes raised on the device (ctrl[CTRL_ABORT])
enum : int {
  DEV_OK = 0,
  DEV_BREAKDOWN = 1,
  DEV_OVF_ARENA = 2,
  DEV_OVF_LIST = 3,
  DEV_OVF_WORK = 4,
  DEV_OVF_POOL = 5,
  DEV_OVF_HPOOL = 6,     // heavy-block pool
  DEV_OVF_HCTX = 7,      // heavy-block context table or task queue
};

// control block indices (int64 each)
enum : int {
  CTRL_QHEAD = 0,
  CTRL_QTAIL,
  CTRL_ABORT,
  CTRL_ERRBLK,
  CTRL_CUR_LIDX,
  CTRL_CUR_LVAL,
  CTRL_CUR_UIDX,
  CTRL_CUR_UVAL,
  CTRL_POOL_LC,
  CTRL_POOL_UC,
  CTRL_POOL_SUCC,
  CTRL_NEAR,
  CTRL_DONE,
  CTRL_NDEC,
  CTRL_FLOPS,
  CTRL_HPOOL,      // doubles used in the heavy-block pool
  CTRL_HCTX,       // heavy contexts used
  CTRL_NPERT,      // pivot blocks perturbed (Sec. 3.6)
  CTRL_HQHEAD,     // high-priority queue (push tasks and the blocks they release)
  CTRL_HQTAIL,
  CTRL_COUNT = 24
};
constexpr int CS = 16;   // ctrl stride: every control word on its own 128-byte line

struct ChunkList {
  int *cnt;        // [N]   records appended per target
  int *dir;        // [N * DIR_SLOTS] chunk ids (-1 = none, -2 = overflow)
  int *pool;       // [pool_cap * CHUNK * rec_ints]
  int pool_cap;    // chunks
  int rec_ints;
  int ctrl_cursor; // index into ctrl of the pool cursor
};

struct HeavyCtx;   // bilu_factor.cu

struct DevFactor {
  // problem
  int32_t n, N;
  const int32_t *bstart;     // [N+1]
  const int32_t *block_of;   // [n]
  // Ã per block: AL = entries of block column K with row >= s_K (sorted by row),
  // packed rc = row << 7 | (col - s_K); AU = entries of block row K with col >= e_K,
  // rc = col << 7 | (row - s_K).  AL_ge[K] = first AL entry with row >= e_K.
  const int64_t *AL_ptr; const int64_t *AL_ge; const int32_t *AL_rc; const double *AL_val;
  const int64_t *AKL_ptr; const int32_t *AKL;   // distinct candidate keys of Ã per block (AL rows >= e_K)
  const int64_t *AKU_ptr; const int32_t *AKU;   // ... (AU columns)
  const int64_t *AU_ptr; const int32_t *AU_rc; const double *AU_val;
  // static schedule: block adjacency of sym(Ã), successors > J
  const int32_t *adj_ptr; const int32_t *adj;
  int32_t *pending;          // [N]
  int32_t *queue;            // [qcap]: block ids (< N) and part tasks (>= N) of split heavy blocks
  const int32_t *prio;       // [N] continuation priority: etree subtree size (unknowns), >= 1
  int64_t qcap;
  unsigned long long *ctrl;  // [CTRL_COUNT * CS]
  int32_t *hq; int64_t hqcap;  // high-priority queue (-1 = empty slot)
  int push_mode;               // zone push of the targets after n0
  // factors (per original block)
  int64_t *Lrow_off; int32_t *Lm; int64_t *Lval_off;
  int64_t *Ucol_off; int32_t *Uc; int64_t *Uval_off;
  const int64_t *D_off;      // static prefix of b^2
  int32_t *Lidx; double *Lval; int64_t cap_Lidx, cap_Lval;
  int32_t *Uidx; double *Uval; int64_t cap_Uidx, cap_Uval;
  double *D;
  double *blk_flops;         // [N]
  int32_t *blk_ncand;        // [2N] candidate rows / cols
  // lists
  ChunkList lc, uc, succ;
  // near-threshold log
  int32_t *near_i; double *near_m; int64_t near_cap;
  // per-CTA global workspace
  double *work; int64_t work_per_cta;   // doubles per CTA
  int *posmap;                          // [grid * n] index -> occurrence / buffer line
  volatile int *dbg;                    // mapped host memory for the deadlock watchdog (or NULL)
  // distributed factorization (bilu_dist_setup): blocks this launch may enqueue and the
  // finished-block count at which it stops
  const uint8_t *owned;                 // [N] or NULL (every block)
  int64_t n_target;
  // split heavy blocks
  HeavyCtx *hctx; int64_t hctx_cap;
  double *hpool; int64_t hpool_cap;     // doubles
  int heavy_T;                          // item count from which a block is split (0 = never)
  int pair_cap;                         // readiness edges: (row, column) block pairs up to this many, else the chain
  int heavy_idle;                       // ... if at least this many CTAs are idle
  int part_items;                       // items per update-part task
  double wide_flops;                    // blocks wider than 16 are split from this many update flops
  double wide_part_flops;               // ... into parts of about this many flops
  int scale_split;                      // wide split blocks: candidates from which the scaling is split
  int scale_rows;                       // ... into parts of this many rows
  int smem_bytes;
  double tau, near_rel;
  // Sec. 3.6 perturbation of singular / ill-conditioned pivot blocks (R19)
  int perturb; double ptau, prho, cond_max;
  const double *alpha;                  // device scalar: max |a_ij|
  // dense zone: the top blocks of the block elimination tree (a set closed
  // under ancestors, every block at most 8 wide) keep their panels in dense per-block
  // buffers that their contributors update when THEY finish (a right-looking push), so a
  // ready zone block only gathers its own panel.  Panel rows of block T are the unknowns on
  // T's etree path to the root (the only rows / columns T can have), in increasing order:
  // unknown i has the path coordinate zd[i] = A(B) - (i - s_B) (B = block of i, A(X) = the
  // unknowns from X up to the root), and sits at local index zA[T] - zd[i] in T's panel.
  //   SL[(zpb[T] + loc) * 8 + c]   entry (i, s_T + c) of block column T (i >= s_T)
  //   SU[(zpb[T] + loc) * 8 + r]   entry (s_T + r, j) of block row T    (j >= e_T)
  //   BL / BU[zwb[T] + (loc >> 5)]  candidate rows / columns (bit loc & 31)
  //   zrun[zrp[zk[T]] ..]          runs (first local index, first unknown) of T's path
  // nzb = 0: no zone.
  int nzb;
  const int32_t *zk;                    // [N] zone index of block K, or -1
  const int32_t *zA;                    // [N] unknowns on the etree path from K to the root
  const int64_t *zpb, *zwb;             // [N] first panel row / first bitmap word of zone block K
  const int32_t *zd;                    // [n] path coordinate of zone unknown i, -1 outside the zone
  const int32_t *zrp;                   // [nzb + 1] run table offsets (by zone index)
  const int2 *zrun;                     // runs of the paths
  double *SL, *SU;
  unsigned *BL, *BU;
};

struct MergeArgs {
  int n, N, max_block;
  const int32_t *bstart;
  const int64_t *Lrow_off; const int32_t *Lm; const int64_t *Lval_off;
  const int64_t *Ucol_off; const int32_t *Uc; const int64_t *Uval_off;
  const int32_t *Lidx; const int32_t *Uidx;
  const double *Lval; const double *Uval; const double *D; const int64_t *D_off;
  // outputs / workspace
  uint32_t *T;            // [4N] test bitmasks, bit d-1 <=> merge(a = k-d, k)
  const int64_t *wofs;    // [N+1] offsets of the per-block windows (W_k + 1 entries each)
  int32_t *UV;            // [2 * sum(W_k + 1)] union sizes u(d), v(d) of the test
  uint8_t *chunkmap;      // [nchunks * 128] scan state maps
  uint8_t *chunkstart;    // [nchunks]
  int32_t *flag;          // [N] run-start flags
  int32_t *first;         // [N+1] first original block of each final block
  int32_t *nF;            // [1]
  const int32_t *seg;     // [N] aggregation segments (merges only inside one segment) or NULL
  int32_t *fbstart;       // [N+1]
  int32_t *fLm, *fUc;     // [N]
  int64_t *fLrow_off, *fLval_off, *fUcol_off, *fUval_off, *fD_off;  // [N] / [N+1]
  unsigned long long *tot;  // [16] cursors and maxima
  int32_t *Lidx_out; double *Lval_out; int32_t *Uidx_out; double *Uval_out;
  double *fD;
  int *work; int64_t work_ints;  // per-CTA workspace (ints)
  double *flops;          // [1]
  int *ovf;               // [1]
  // test windows wider than the shared-memory hash table: per-CTA global tables of hbig_cap
  // slots (keys int32, dmin int32, flag uint8), bytes per CTA = 9 * hbig_cap
  unsigned char *hbig; int64_t hbig_cap;
  int *ticket;            // [1] merge_arith: next final block (dynamic, heaviest-first order)
};

// Apply (forward/backward block triangular solves) -- dataflow over final blocks.
struct ApplyArgs {
  int n, nF;
  const int32_t *fbstart;
  const int64_t *Lrow_off, *Lval_off, *Ucol_off, *Uval_off, *D_off;
  const int32_t *Lm, *Uc;
  const int32_t *Lidx, *Uidx;
  const double *Lval, *Uval, *D;
  // forward pull lists: for target T, records (J, r0, r1) at fl_ptr[T]..fl_ptr[T+1]
  const int32_t *fl_ptr, *fl_rec;
  const int32_t *fs_ptr, *fs;     // forward successors of J
  const int32_t *bs_ptr, *bs;     // backward successors of T (blocks with U cols in T)
  int32_t *cnt;                   // [nF] working counters
  int32_t *queue;                 // [nF]
  unsigned long long *ctrl;       // [4]: qhead, qtail
  double *w, *y;                  // permuted work vectors
  int ntarget;                    // blocks this sweep processes (nF; a rank's share when distributed)
  unsigned long long *prof;       // diagnostics (BILU_APPLY_PROF): per block popped/computed/released times, or NULL
};

// packed interface blocks exchanged between ranks (bilu_interface_pack/unpack)
struct PackEntry {
  int64_t J, b, Lm, Uc;
  int64_t offLi, offLv, offUi, offUv;   // byte offsets into the packed buffer
};
constexpr int64_t PACK_MAGIC = 0x42494c5550414b31LL;   // "BILUPAK1"
constexpr int64_t PACK_HEADER = 4;                     // int64 words: magic, count, bytes, rank

}  // namespace bilu
