// bilu_host.cpp -- host orchestrator behind the C-ABI of include/bilu.h.
//
// bilu_analyze: validation, symmetric permutation Ã = A(perm, perm) (CSR and
//   CSC), the block graph of sym(Ã) (static part of the dataflow schedule) and
//   device upload.  (Host preprocessing is allowed by the task; the caller's
//   ordering/blocking are inputs: PAPER.md:1541-1573.)
// bilu_factor:  resets the device schedule state, launches the persistent
//   factor kernel (bilu_factor.cu), regrows workspaces on overflow, runs the
//   progressive-aggregation post-pass (bilu_merge.cu) and collects statistics.
// bilu_apply:   level-free dataflow triangular solves (bilu_apply.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <chrono>
#include <ctime>
#include <unistd.h>

#include "../../include/bilu.h"
#include "bilu_internal.h"

using namespace bilu;

namespace bilu {
extern "C" cudaError_t bilu_launch_factor(const DevFactor &F, int grid, cudaStream_t st);
extern "C" cudaError_t bilu_launch_zone_init(const DevFactor &F, const int32_t *zblocks, cudaStream_t st);
extern "C" cudaError_t bilu_factor_occupancy(int smem_bytes, int *blocks_per_sm);
extern "C" cudaError_t bilu_launch_gather(double *dst, const double *src, const int64_t *map,
                                          int64_t n, cudaStream_t st);
extern "C" cudaError_t bilu_launch_permute(double *y, const double *x, const int32_t *perm,
                                           int32_t n, int inverse, cudaStream_t st);
extern "C" cudaError_t bilu_merge_plan(const MergeArgs &M, int grid, cudaStream_t st);
extern "C" int bilu_merge_plan_launches();
extern "C" int bilu_merge_test_grid(int grid);
extern "C" cudaError_t bilu_merge_bound(const MergeArgs &M, unsigned long long *out, int sms, cudaStream_t st);
extern "C" int bilu_heavyctx_size();
extern "C" cudaError_t bilu_launch_spmv(int n, const int64_t *rp, const int32_t *ci, const double *val, const double *x,
                                        double *y, int lpr, int sms, cudaStream_t st);
extern "C" cudaError_t bilu_launch_dot(int n, const double *x, const double *y, double *partials, double *out,
                                       int sqrt_out, int sms, cudaStream_t st);
extern "C" cudaError_t bilu_launch_axpy_dev(int n, const double *coef, double sign, const double *x, double *y, int sms,
                                            cudaStream_t st);
extern "C" cudaError_t bilu_launch_scale_dev(int n, const double *coef, const double *x, double *y, int sms,
                                             cudaStream_t st);
extern "C" cudaError_t bilu_launch_update(int n, int k, const double *Z, int64_t ld, const double *c, double *x, int sms,
                                          cudaStream_t st);
extern "C" cudaError_t bilu_launch_residual(int n, const double *b, double *r, int sms, cudaStream_t st);
extern "C" cudaError_t bilu_launch_maxabs(double *out, const double *x, int64_t n, cudaStream_t st);
extern "C" cudaError_t bilu_launch_sep_prepare(const DevFactor &F, const int32_t *sep_list, int nsep,
                                               const int32_t *static_sep, const int32_t *ifc, int nifc,
                                               const uint8_t *sep, cudaStream_t st);
extern "C" cudaError_t bilu_launch_interface_flags(const DevFactor &F, const int32_t *own_list, int nown,
                                                   const uint8_t *sep, uint8_t *flag, cudaStream_t st);
extern "C" cudaError_t bilu_launch_pack(const DevFactor &F, const PackEntry *tab, int count, unsigned char *buf,
                                        cudaStream_t st);
extern "C" cudaError_t bilu_launch_unpack(const DevFactor &F, const unsigned char *buf, const PackEntry *tab,
                                          int count, const int64_t *base, cudaStream_t st);
extern "C" int bilu_max_parts();
extern "C" int bilu_merge_nchunks(int N);
extern "C" cudaError_t bilu_merge_arith(const MergeArgs &M, double *dwork, int64_t dwork_per_cta, int grid,
                                        cudaStream_t st);
extern "C" cudaError_t bilu_launch_apply(const ApplyArgs &A, int grid, int backward, cudaStream_t st);
extern "C" cudaError_t bilu_launch_sep_gather(int m, const int32_t *idx, const double *src, double *out, cudaStream_t st);
extern "C" cudaError_t bilu_launch_sep_contrib(int m, const int32_t *idx, const double *w, const double *xsep,
                                               double *out, cudaStream_t st);
extern "C" cudaError_t bilu_launch_sep_set(int m, const int32_t *idx, const double *xsep, const double *sum, double *w,
                                           cudaStream_t st);
extern "C" cudaError_t bilu_launch_permute_out_masked(int n, const int32_t *perm, const uint8_t *mask, int write_sep,
                                                      const double *yp, double *y, cudaStream_t st);
extern "C" cudaError_t bilu_ilu1_run(int n, const int64_t *rp, const int32_t *ci, const double *val,
                                     const int32_t *pm, const int32_t *ipm, double tau, int max_size, int sms,
                                     cudaStream_t st, int32_t *h_sizes, int32_t *nblocks, int *launches);
extern "C" cudaError_t bilu_cosine_run(int n, const int64_t *rp, const int32_t *ci, double tau, int max_size, int sms,
                                       cudaStream_t st, int32_t *h_q, int32_t *h_sizes, int32_t *nblocks,
                                       int *launches, int *rounds);
}  // namespace bilu

// Final (post-aggregation) factor: per final block F, descriptors into the
// L/U arenas of DevFactor and a final D arena.
struct FinalFactor {
  int nF = 0;
  int32_t *bstart = nullptr;                      // [nF+1]
  int64_t *Lrow_off = nullptr, *Lval_off = nullptr, *Ucol_off = nullptr, *Uval_off = nullptr;
  int32_t *Lm = nullptr, *Uc = nullptr;
  int64_t *D_off = nullptr;                       // [nF+1]
  double *D = nullptr;
  int64_t nnzL = 0, nnzU = 0, nnzD = 0, nidxL = 0, nidxU = 0;   // final factor sizes
  int64_t usedLi = 0, usedLv = 0, usedUi = 0, usedUv = 0;       // arena prefixes in use
  bool owns = false;                              // arrays allocated for merges
};

static thread_local std::string g_last_error;

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
};

struct bilu_ctx {
  bilu_options opt;
  cudaStream_t stream = nullptr;
  int n = 0, N = 0;
  int64_t nnz = 0;
  std::string err;
  int sms = 0;
  int64_t launches = 0;
  bool factored = false;
  int max_b = 0;
  // host copies
  std::vector<int32_t> bstart, ready0;
  std::vector<int32_t> adj_ptr_h, adj_h, pending0_h;   // block graph (successors > K), static counts
  // distributed factorization (bilu_dist_setup)
  bool dist = false, dist_local_done = false;
  int32_t rank = 0;
  std::vector<int32_t> owner, seg, own_list, sep_list, static_sep, own_ifc, remote_ifc;
  int32_t *d_own_list = nullptr, *d_sep_list = nullptr, *d_static_sep = nullptr, *d_seg = nullptr;
  int32_t *d_ifc = nullptr; int64_t ifc_cap = 0;
  uint8_t *d_own_mask = nullptr, *d_sep_mask = nullptr, *d_flag = nullptr;
  std::vector<PackEntry> pack_tab; int64_t pack_bytes = 0; bool pack_valid = false;
  int64_t *d_base = nullptr; int64_t base_cap = 0;
  unsigned long long cur[4] = {0, 0, 0, 0};      // arena cursors after phase A + unpacks
  unsigned long long qhead0 = 0, ctrl_init[CTRL_COUNT * CS];
  int32_t *d_own_ready = nullptr; int32_t n_own_ready = 0;
  unsigned long long *d_mbound = nullptr;           // merge test: widest window
  int *d_mticket = nullptr;                          // merge arith: dynamic block ticket
  unsigned char *d_mhbig = nullptr; int64_t mhbig_cap = 0;   // merge test: per-CTA global tables
  double flops_local = 0.0, t_local_ms = 0.0;
  double *d_alpha = nullptr;
  // dense trailing zone
  bool zone_dirty = false;            // zone buffers may hold data (a launch did not complete)
  int32_t *d_zblocks = nullptr;       // zone index -> block
  size_t zone_val_bytes = 0, zone_bit_bytes = 0;
  int64_t zone_unknowns = 0;
  // GMRES: A's CSR structure (original ordering) and the Krylov workspace
  int64_t *d_rp = nullptr; int32_t *d_ci = nullptr;
  double *d_kry = nullptr; int64_t kry_cap = 0;
  int64_t npert_local = 0;
  int64_t ndec_local = 0, nnear_local = 0;
  std::vector<int64_t> D_off;
  std::vector<int64_t> map_csr;            // Ã entry -> original CSR entry
  std::vector<int32_t> perm;
  // device buffers (owned)
  std::vector<void *> owned;
  int32_t *d_bstart = nullptr, *d_block_of = nullptr;
  double *d_val_orig = nullptr;
  int64_t *d_AL_ptr = nullptr, *d_AL_ge = nullptr, *d_AU_ptr = nullptr;
  int32_t *d_AL_rc = nullptr, *d_AU_rc = nullptr;
  int64_t *d_AKL_ptr = nullptr, *d_AKU_ptr = nullptr;
  int32_t *d_AKL = nullptr, *d_AKU = nullptr;
  double *d_AL_val = nullptr, *d_AU_val = nullptr;
  int64_t *d_AL_map = nullptr, *d_AU_map = nullptr;
  int64_t nAL = 0, nAU = 0;
  int32_t *d_adj_ptr = nullptr, *d_adj = nullptr, *d_pending0 = nullptr, *d_ready0 = nullptr;
  int32_t *d_perm = nullptr;
  int32_t nready0 = 0;
  unsigned long long nready0_ull = 0;
  unsigned long long ctrl_full[CTRL_COUNT * CS];
  // dynamic
  DevFactor F{};
  int grid = 0;
  int64_t cap_val = 0, cap_idx = 0, work_per_cta = 0, hpool_cap = 0, hpool_dirty = 0;
  int pool_lc = 0, pool_uc = 0, pool_succ = 0;
  int64_t near_cap = 1 << 20;
  // results
  FinalFactor fin;
  bilu_factor_stats last{};
  // merge workspace
  MergeArgs M{};
  bool merge_alloc = false;
  int64_t merge_work_ints = 0, merge_dwork = 0, fD_cap = 0;
  double *d_mdwork = nullptr;
  volatile int *dbg_host = nullptr;
  // apply structure (built lazily after each factorization)
  bool apply_ready = false;
  ApplyArgs AA{};
  int32_t *d_fl_ptr = nullptr, *d_fl_rec = nullptr, *d_fs_ptr = nullptr, *d_fs = nullptr;
  int32_t *d_bs_ptr = nullptr, *d_bs = nullptr, *d_cnt_f0 = nullptr, *d_cnt_b0 = nullptr;
  int32_t *d_q_f0 = nullptr, *d_q_b0 = nullptr;
  int32_t nq_f0 = 0, nq_b0 = 0;
  unsigned long long nq_f0_ull = 0, nq_b0_ull = 0;
  int32_t nt_f0 = 0, nt_b0 = 0;                      // blocks per sweep (nF unless distributed)
  // distributed apply: forward over the separator blocks (phase 2), separator rows, row mask
  int32_t *d_cnt_f2 = nullptr, *d_q_f2 = nullptr; int32_t nq_f2 = 0, nt_f2 = 0;
  unsigned long long nq_f2_ull = 0;
  int32_t *d_seprows = nullptr; int32_t nsep_rows = 0;
  double *d_xsep = nullptr;
  uint8_t *d_rowmask = nullptr;
  bool dist_apply_begun = false;
  double *d_w = nullptr, *d_y = nullptr;
};

static void set_err(bilu_ctx *h, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  if (h) h->err = buf;
}

#define CUDA_TRY(h, x)                                                              \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      set_err(h, "CUDA error %s at %s:%d", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return e_ == cudaErrorMemoryAllocation ? BILU_ERR_OOM : BILU_ERR_CUDA;         \
    }                                                                               \
  } while (0)

template <typename T>
static cudaError_t dalloc(bilu_ctx *h, T **p, size_t count) {
  void *q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) return e;
  h->owned.push_back(q);
  *p = (T *)q;
  return cudaSuccess;
}
template <typename T>
static void dfree(bilu_ctx *h, T *&p) {
  if (!p) return;
  auto it = std::find(h->owned.begin(), h->owned.end(), (void *)p);
  if (it != h->owned.end()) h->owned.erase(it);
  cudaFree(p);
  p = nullptr;
}

extern "C" void bilu_options_default(bilu_options *opt) {
  if (!opt) return;
  memset(opt, 0, sizeof(*opt));
  opt->device = 0;
  opt->max_block = 128;
  opt->aggregate = 1;
  opt->n_ctas = 0;
  opt->near_rel = 1e-8;
  opt->arena_hint = 0;
  opt->stream = nullptr;
  opt->rank = 0;
  opt->world = 1;
  opt->nccl_comm = nullptr;
  opt->perturb = 0;
  opt->perturb_tau = 1e-2;
  opt->perturb_rho = 1e-1;
  opt->cond_max = 1e12;
}

extern "C" const char *bilu_status_string(bilu_status s) {
  switch (s) {
    case BILU_OK: return "ok";
    case BILU_ERR_ARG: return "invalid argument";
    case BILU_ERR_BREAKDOWN: return "breakdown: singular pivot block";
    case BILU_ERR_OOM: return "out of device memory";
    case BILU_ERR_CUDA: return "CUDA error";
    case BILU_ERR_NCCL: return "NCCL error";
    case BILU_ERR_STATE: return "invalid state";
    case BILU_ERR_NOT_BUILT: return "no usable CUDA device";
  }
  return "unknown status";
}

extern "C" const char *bilu_last_error(const bilu_ctx *h) {
  if (h) return h->err.c_str();
  return g_last_error.c_str();
}

extern "C" int64_t bilu_kernel_launches(const bilu_ctx *h) { return h ? h->launches : 0; }

// --------------------------------------------------------------- destroy
extern "C" void bilu_destroy(bilu_ctx *h) {
  if (!h) return;
  if (h->opt.device >= 0) cudaSetDevice(h->opt.device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void *p : h->owned) cudaFree(p);
  h->owned.clear();
  delete h;
}

// --------------------------------------------------------------- CSR / permutation input
// Validates a host CSR (sorted, duplicate-free rows) and a permutation (NULL = identity).
static bilu_status check_csr_perm(const char *fn, int32_t n, const int64_t *row_ptr, const int32_t *col_idx,
                                  const int32_t *perm, std::vector<int32_t> &pm, std::vector<int32_t> &ipm) {
  if (row_ptr[0] != 0) { set_err(nullptr, "%s: row_ptr[0] != 0", fn); return BILU_ERR_ARG; }
  for (int32_t i = 0; i < n; ++i) {
    if (row_ptr[i + 1] < row_ptr[i]) { set_err(nullptr, "%s: row_ptr decreases at row %d", fn, i); return BILU_ERR_ARG; }
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      if (col_idx[p] < 0 || col_idx[p] >= n) { set_err(nullptr, "%s: column index out of range in row %d", fn, i); return BILU_ERR_ARG; }
      if (p > row_ptr[i] && col_idx[p] <= col_idx[p - 1]) { set_err(nullptr, "%s: row %d not strictly increasing (unsorted or duplicate)", fn, i); return BILU_ERR_ARG; }
    }
  }
  pm.assign(n, 0);
  ipm.assign(n, -1);
  for (int32_t i = 0; i < n; ++i) {
    int32_t p = perm ? perm[i] : i;
    if (p < 0 || p >= n || ipm[p] != -1) { set_err(nullptr, "%s: perm is not a bijection (position %d)", fn, i); return BILU_ERR_ARG; }
    pm[i] = p; ipm[p] = i;
  }
  return BILU_OK;
}

// Ã = A(pm, pm) in CSR with sorted rows; map[q] = position of Ã's entry q in A's arrays.
static void permute_csr(int32_t n, const int64_t *row_ptr, const int32_t *col_idx, const std::vector<int32_t> &pm,
                        const std::vector<int32_t> &ipm, std::vector<int64_t> &rp, std::vector<int32_t> &ci,
                        std::vector<int64_t> &map) {
  const int64_t nnz = row_ptr[n];
  rp.assign(n + 1, 0);
  for (int32_t i = 0; i < n; ++i) rp[i + 1] = rp[i] + (row_ptr[pm[i] + 1] - row_ptr[pm[i]]);
  ci.resize(nnz);
  map.resize(nnz);
  std::vector<std::pair<int32_t, int64_t>> tmp;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t o = pm[i];
    tmp.clear();
    for (int64_t p = row_ptr[o]; p < row_ptr[o + 1]; ++p) tmp.emplace_back(ipm[col_idx[p]], p);
    std::sort(tmp.begin(), tmp.end());
    int64_t q = rp[i];
    for (auto &t : tmp) { ci[q] = t.first; map[q] = t.second; ++q; }
  }
}

// --------------------------------------------------------------- analyze
extern "C" bilu_status bilu_analyze(int32_t n, const int64_t *row_ptr, const int32_t *col_idx,
                                    const double *val, const int32_t *perm,
                                    const int32_t *block_sizes, int32_t n_blocks,
                                    const bilu_options *opt_in, bilu_ctx **out) {
  if (!out) { set_err(nullptr, "bilu_analyze: out is NULL"); return BILU_ERR_ARG; }
  *out = nullptr;
  bilu_options opt;
  if (opt_in) opt = *opt_in; else bilu_options_default(&opt);
  if (n < 1 || !row_ptr || !col_idx || !block_sizes || n_blocks < 1) {
    set_err(nullptr, "bilu_analyze: null pointer or empty problem (n=%d, n_blocks=%d)", n, n_blocks);
    return BILU_ERR_ARG;
  }
  if (opt.max_block < 1 || opt.max_block > 128) {
    set_err(nullptr, "bilu_analyze: max_block must be in [1,128] (got %d)", opt.max_block);
    return BILU_ERR_ARG;
  }
  if (n >= (1 << 24)) { set_err(nullptr, "bilu_analyze: n must be < 2^24 (got %d)", n); return BILU_ERR_ARG; }
  if (n_blocks >= (1 << 21)) {
    set_err(nullptr, "bilu_analyze: at most 2^21-1 blocks supported (got %d)", n_blocks);
    return BILU_ERR_ARG;
  }
  if (opt.world != 1) {
    set_err(nullptr, "bilu_analyze: world > 1 is not supported by this build");
    return BILU_ERR_ARG;
  }
  std::vector<int32_t> pm, ipm;
  {
    bilu_status st = check_csr_perm("bilu_analyze", n, row_ptr, col_idx, perm, pm, ipm);
    if (st != BILU_OK) return st;
  }
  const int64_t nnz = row_ptr[n];
  // ---- validate partition
  std::vector<int32_t> bstart(n_blocks + 1, 0);
  int max_b = 0;
  for (int32_t K = 0; K < n_blocks; ++K) {
    if (block_sizes[K] < 1 || block_sizes[K] > opt.max_block) {
      set_err(nullptr, "bilu_analyze: block %d has size %d outside [1, max_block=%d]", K, block_sizes[K], opt.max_block);
      return BILU_ERR_ARG;
    }
    bstart[K + 1] = bstart[K] + block_sizes[K];
    max_b = std::max(max_b, (int)block_sizes[K]);
    if (bstart[K + 1] > n) break;
  }
  if (bstart[n_blocks] != n) { set_err(nullptr, "bilu_analyze: sum(block_sizes) != n"); return BILU_ERR_ARG; }

  bilu_ctx *h = new bilu_ctx();
  h->opt = opt;
  h->n = n; h->N = n_blocks; h->nnz = nnz; h->max_b = max_b;
  h->bstart = bstart;
  h->perm = pm;
  if (cudaSetDevice(opt.device) != cudaSuccess) {
    set_err(h, "bilu_analyze: cannot use CUDA device %d", opt.device);
    g_last_error = h->err;
    delete h;
    return BILU_ERR_NOT_BUILT;
  }
  h->stream = (cudaStream_t)opt.stream;
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, opt.device);

  // ---- Ã = A(perm, perm), CSR (rows sorted)
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  permute_csr(n, row_ptr, col_idx, pm, ipm, rp, ci, h->map_csr);
  // ---- block graph of sym(Ã): successors > K and pending counts
  std::vector<int32_t> block_of(n);
  for (int32_t K = 0; K < n_blocks; ++K)
    for (int32_t i = bstart[K]; i < bstart[K + 1]; ++i) block_of[i] = K;
  std::vector<uint64_t> edges;
  {
    std::vector<int32_t> mark(n_blocks, -1);
    for (int32_t I = 0; I < n_blocks; ++I) {
      for (int32_t i = bstart[I]; i < bstart[I + 1]; ++i)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
          int32_t J = block_of[ci[p]];
          if (J == I || mark[J] == I) continue;
          mark[J] = I;
          int32_t a = std::min(I, J), b = std::max(I, J);
          edges.push_back(((uint64_t)a << 32) | (uint32_t)b);
        }
    }
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
  }
  // ---- per-block lists of Ã's entries: AL (block column K, rows >= s_K, sorted by
  // (row, col)) and AU (block row K, cols >= e_K, sorted by (col, row)); values are
  // gathered into this order by bilu_set_values.
  std::vector<int64_t> AL_ptr(n_blocks + 1, 0), AL_ge(n_blocks, 0), AU_ptr(n_blocks + 1, 0);
  std::vector<int32_t> AL_rc, AU_rc;
  std::vector<int64_t> AL_map, AU_map;
  AL_rc.reserve(nnz); AL_map.reserve(nnz); AU_rc.reserve(nnz); AU_map.reserve(nnz);
  {
    // bucket every entry (i, j) by its owning block: block(j) <= block(i) -> AL of block(j), else AU of block(i)
    std::vector<int64_t> cntL(n_blocks + 1, 0), cntU(n_blocks + 1, 0);
    for (int32_t i = 0; i < n; ++i)
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int32_t bi = block_of[i], bj = block_of[ci[p]];
        if (bj <= bi) cntL[bj + 1]++; else cntU[bi + 1]++;
      }
    for (int32_t K = 0; K < n_blocks; ++K) { cntL[K + 1] += cntL[K]; cntU[K + 1] += cntU[K]; }
    AL_ptr = cntL; AU_ptr = cntU;
    AL_rc.assign(cntL[n_blocks], 0); AL_map.assign(cntL[n_blocks], 0);
    AU_rc.assign(cntU[n_blocks], 0); AU_map.assign(cntU[n_blocks], 0);
    std::vector<int64_t> fl(cntL.begin(), cntL.end() - 1), fu(cntU.begin(), cntU.end() - 1);
    // rows ascending, and within a row columns ascending -> AL sorted by (row, col)
    for (int32_t i = 0; i < n; ++i)
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        const int32_t j = ci[p], bi = block_of[i], bj = block_of[j];
        if (bj <= bi) {
          const int64_t q = fl[bj]++;
          AL_rc[q] = (i << 7) | (j - bstart[bj]);
          AL_map[q] = h->map_csr[p];
        } else {
          const int64_t q = fu[bi]++;
          AU_rc[q] = (j << 7) | (i - bstart[bi]);
          AU_map[q] = h->map_csr[p];
        }
      }
    // AU: sort each block's list by (col, row)
    for (int32_t K = 0; K < n_blocks; ++K) {
      std::vector<std::pair<int32_t, int64_t>> tmp;
      for (int64_t q = AU_ptr[K]; q < AU_ptr[K + 1]; ++q) tmp.emplace_back(AU_rc[q], AU_map[q]);
      std::sort(tmp.begin(), tmp.end());
      for (size_t x = 0; x < tmp.size(); ++x) { AU_rc[AU_ptr[K] + x] = tmp[x].first; AU_map[AU_ptr[K] + x] = tmp[x].second; }
      int64_t q = AL_ptr[K];
      while (q < AL_ptr[K + 1] && (AL_rc[q] >> 7) < bstart[K + 1]) ++q;
      AL_ge[K] = q;
    }
  }
  h->nAL = AL_ptr[n_blocks]; h->nAU = AU_ptr[n_blocks];
  // distinct candidate keys of Ã per block (rows >= e_K of AL, columns of AU): the a-3 passes
  // read these instead of every entry
  std::vector<int64_t> AKL_ptr(n_blocks + 1, 0), AKU_ptr(n_blocks + 1, 0);
  std::vector<int32_t> AKL, AKU;
  for (int32_t K = 0; K < n_blocks; ++K) {
    for (int64_t q = AL_ge[K]; q < AL_ptr[K + 1]; ++q)
      if (q == AL_ge[K] || (AL_rc[q] >> 7) != (AL_rc[q - 1] >> 7)) AKL.push_back(AL_rc[q] >> 7);
    for (int64_t q = AU_ptr[K]; q < AU_ptr[K + 1]; ++q)
      if (q == AU_ptr[K] || (AU_rc[q] >> 7) != (AU_rc[q - 1] >> 7)) AKU.push_back(AU_rc[q] >> 7);
    AKL_ptr[K + 1] = (int64_t)AKL.size(); AKU_ptr[K + 1] = (int64_t)AKU.size();
  }
  std::vector<int32_t> adj_ptr(n_blocks + 1, 0), adj(edges.size()), pending0(n_blocks, 0);
  for (uint64_t eg : edges) { adj_ptr[(eg >> 32) + 1]++; pending0[(uint32_t)eg]++; }
  for (int32_t K = 0; K < n_blocks; ++K) adj_ptr[K + 1] += adj_ptr[K];
  for (size_t x = 0; x < edges.size(); ++x) adj[x] = (int32_t)(uint32_t)edges[x];  // sorted by (a, b)
  for (int32_t K = 0; K < n_blocks; ++K) if (pending0[K] == 0) h->ready0.push_back(K);
  h->adj_ptr_h = adj_ptr; h->adj_h = adj; h->pending0_h = pending0;
  h->nready0 = (int32_t)h->ready0.size();
  h->nready0_ull = (unsigned long long)h->nready0;
  h->D_off.assign(n_blocks + 1, 0);
  for (int32_t K = 0; K < n_blocks; ++K) {
    int64_t b = bstart[K + 1] - bstart[K];
    h->D_off[K + 1] = h->D_off[K] + b * b;
  }

  // ---- device upload
#define ALLOC(ptr, cnt) do { cudaError_t e_ = dalloc(h, &ptr, cnt); if (e_ != cudaSuccess) { set_err(h, "bilu_analyze: cudaMalloc failed (%s)", cudaGetErrorString(e_)); g_last_error = h->err; bilu_destroy(h); return BILU_ERR_OOM; } } while (0)
#define H2D(dst, src, cnt) do { cudaError_t e_ = cudaMemcpy(dst, src, (cnt) * sizeof(*(src)), cudaMemcpyHostToDevice); if (e_ != cudaSuccess) { set_err(h, "bilu_analyze: copy failed (%s)", cudaGetErrorString(e_)); g_last_error = h->err; bilu_destroy(h); return BILU_ERR_CUDA; } } while (0)
  ALLOC(h->d_bstart, n_blocks + 1); H2D(h->d_bstart, bstart.data(), n_blocks + 1);
  ALLOC(h->d_block_of, n); H2D(h->d_block_of, block_of.data(), n);
  ALLOC(h->d_AL_ptr, n_blocks + 1); H2D(h->d_AL_ptr, AL_ptr.data(), n_blocks + 1);
  ALLOC(h->d_AL_ge, n_blocks); H2D(h->d_AL_ge, AL_ge.data(), n_blocks);
  ALLOC(h->d_AU_ptr, n_blocks + 1); H2D(h->d_AU_ptr, AU_ptr.data(), n_blocks + 1);
  ALLOC(h->d_AL_rc, h->nAL); if (h->nAL) H2D(h->d_AL_rc, AL_rc.data(), h->nAL);
  ALLOC(h->d_AU_rc, h->nAU); if (h->nAU) H2D(h->d_AU_rc, AU_rc.data(), h->nAU);
  ALLOC(h->d_AL_map, h->nAL); if (h->nAL) H2D(h->d_AL_map, AL_map.data(), h->nAL);
  ALLOC(h->d_AKL_ptr, n_blocks + 1); H2D(h->d_AKL_ptr, AKL_ptr.data(), n_blocks + 1);
  ALLOC(h->d_AKU_ptr, n_blocks + 1); H2D(h->d_AKU_ptr, AKU_ptr.data(), n_blocks + 1);
  ALLOC(h->d_AKL, std::max<size_t>(AKL.size(), 1)); if (!AKL.empty()) H2D(h->d_AKL, AKL.data(), AKL.size());
  ALLOC(h->d_AKU, std::max<size_t>(AKU.size(), 1)); if (!AKU.empty()) H2D(h->d_AKU, AKU.data(), AKU.size());
  ALLOC(h->d_AU_map, h->nAU); if (h->nAU) H2D(h->d_AU_map, AU_map.data(), h->nAU);
  ALLOC(h->d_AL_val, h->nAL); ALLOC(h->d_AU_val, h->nAU); ALLOC(h->d_val_orig, nnz);
  ALLOC(h->d_adj_ptr, n_blocks + 1); H2D(h->d_adj_ptr, adj_ptr.data(), n_blocks + 1);
  ALLOC(h->d_adj, adj.size()); if (!adj.empty()) H2D(h->d_adj, adj.data(), adj.size());
  ALLOC(h->d_pending0, n_blocks); H2D(h->d_pending0, pending0.data(), n_blocks);
  ALLOC(h->d_ready0, std::max<int32_t>(h->nready0, 1));
  if (h->nready0) H2D(h->d_ready0, h->ready0.data(), h->nready0);
  ALLOC(h->d_perm, n); H2D(h->d_perm, pm.data(), n);
  ALLOC(h->d_rp, (size_t)n + 1); H2D(h->d_rp, row_ptr, (size_t)n + 1);      // A's CSR (bilu_gmres SpMV)
  ALLOC(h->d_ci, (size_t)std::max<int64_t>(nnz, 1)); if (nnz) H2D(h->d_ci, col_idx, nnz);
  {
    int64_t *d_Doff = nullptr;
    ALLOC(d_Doff, n_blocks + 1); H2D(d_Doff, h->D_off.data(), n_blocks + 1);
    h->F.D_off = d_Doff;
  }
#undef H2D

  // ---- schedule state and factor descriptors (sizes independent of values)
  DevFactor &F = h->F;
  F.n = n; F.N = n_blocks;
  F.bstart = h->d_bstart; F.block_of = h->d_block_of;
  F.AL_ptr = h->d_AL_ptr; F.AL_ge = h->d_AL_ge; F.AL_rc = h->d_AL_rc; F.AL_val = h->d_AL_val;
  F.AU_ptr = h->d_AU_ptr; F.AU_rc = h->d_AU_rc; F.AU_val = h->d_AU_val;
  F.AKL_ptr = h->d_AKL_ptr; F.AKL = h->d_AKL; F.AKU_ptr = h->d_AKU_ptr; F.AKU = h->d_AKU;
  F.adj_ptr = h->d_adj_ptr; F.adj = h->d_adj;
  ALLOC(F.pending, n_blocks);
  // heavy-block splitting: contexts, part tasks in the queue
  F.hctx_cap = std::max<int64_t>(256, n_blocks);          // a block is split at most once
  F.qcap = 2 * (int64_t)n_blocks + F.hctx_cap * bilu_max_parts();   // blocks, push tasks, part tasks
  ALLOC(F.queue, F.qcap);
  F.hqcap = 2 * (int64_t)n_blocks + 64;
  F.push_mode = 0;   // 0: the CTA pushes every target (n0 first, released early); 1-3: push tasks (tools/ builds)
  if (const char *pm = tune_env("BILU_PUSH_MODE")) F.push_mode = atoi(pm);
  ALLOC(F.hq, F.hqcap);
  {
    void *hc = nullptr;
    if (cudaMalloc(&hc, (size_t)F.hctx_cap * bilu_heavyctx_size()) != cudaSuccess) {
      set_err(nullptr, "bilu_analyze: out of device memory"); bilu_destroy(h); return BILU_ERR_OOM;
    }
    h->owned.push_back(hc);
    F.hctx = (HeavyCtx *)hc;
  }
  F.perturb = opt.perturb ? 1 : 0;
  F.ptau = opt.perturb_tau; F.prho = opt.perturb_rho; F.cond_max = opt.cond_max;
  {
    double *da = nullptr;
    if (cudaMalloc(&da, sizeof(double)) != cudaSuccess) {
      set_err(nullptr, "bilu_analyze: out of device memory"); bilu_destroy(h); return BILU_ERR_OOM;
    }
    h->owned.push_back(da);
    cudaMemset(da, 0, sizeof(double));
    F.alpha = da;
    h->d_alpha = da;
  }
  F.heavy_T = 1024;
  F.pair_cap = 128;
  if (const char *pc = tune_env("BILU_PAIR_CAP")) F.pair_cap = atoi(pc);
  if (const char *ht = tune_env("BILU_HEAVY_T")) F.heavy_T = atoi(ht);
  F.heavy_idle = 8;
  F.part_items = 512;
  F.wide_flops = 4e6;
  F.scale_split = 1024;
  F.scale_rows = 384;
  if (const char *ss = tune_env("BILU_SCALE_SPLIT")) F.scale_split = atoi(ss);
  if (const char *sr = tune_env("BILU_SCALE_ROWS")) F.scale_rows = std::max(32, atoi(sr));
  F.wide_part_flops = 2e6;
  if (const char *wf = tune_env("BILU_WIDE_FLOPS")) F.wide_flops = atof(wf);
  if (const char *wp = tune_env("BILU_WIDE_PART_FLOPS")) F.wide_part_flops = atof(wp);
  if (const char *pi = tune_env("BILU_PART_ITEMS")) F.part_items = std::max(64, atoi(pi));
  if (const char *hi = tune_env("BILU_HEAVY_IDLE")) F.heavy_idle = atoi(hi);
  ALLOC(F.ctrl, CTRL_COUNT * CS);
  ALLOC(F.Lrow_off, n_blocks); ALLOC(F.Lm, n_blocks); ALLOC(F.Lval_off, n_blocks);
  ALLOC(F.Ucol_off, n_blocks); ALLOC(F.Uc, n_blocks); ALLOC(F.Uval_off, n_blocks);
  ALLOC(F.D, h->D_off[n_blocks]);
  // ---- block elimination tree of sym(Ã) (Liu's algorithm over the lower neighbours of every
  // block; edges are sorted by (a, b)) and the subtree sizes in unknowns
  std::vector<int32_t> par(n_blocks, -1);
  {
    std::vector<int32_t> anc(n_blocks, -1), lp(n_blocks + 1, 0), lo(edges.size(), 0);
    for (uint64_t eg : edges) lp[(uint32_t)eg + 1]++;
    for (int32_t K = 0; K < n_blocks; ++K) lp[K + 1] += lp[K];
    std::vector<int32_t> fill(lp.begin(), lp.end() - 1);
    for (uint64_t eg : edges) lo[fill[(uint32_t)eg]++] = (int32_t)(eg >> 32);
    for (int32_t K = 0; K < n_blocks; ++K)
      for (int32_t q = lp[K]; q < lp[K + 1]; ++q) {
        int32_t r = lo[q];
        while (anc[r] != -1 && anc[r] != K) { const int32_t nx = anc[r]; anc[r] = K; r = nx; }
        if (anc[r] == -1) { anc[r] = K; par[r] = K; }
      }
  }
  std::vector<int64_t> sub(n_blocks, 0);
  for (int32_t K = 0; K < n_blocks; ++K) {
    sub[K] += bstart[K + 1] - bstart[K];
    if (par[K] >= 0) sub[par[K]] += sub[K];
  }
  {
    // continuation priority of release_block: the etree subtree size
    std::vector<int32_t> pr(n_blocks);
    for (int32_t K = 0; K < n_blocks; ++K) pr[K] = (int32_t)std::min<int64_t>(sub[K], INT32_MAX);
    int32_t *dpr = nullptr;
    ALLOC(dpr, n_blocks);
    cudaMemcpy(dpr, pr.data(), n_blocks * sizeof(int32_t), cudaMemcpyHostToDevice);
    F.prio = dpr;
  }
  // ---- dense zone: the top of the block elimination tree of sym(Ã).  The
  // exact-LU structure of a block column / row lies on its etree path to the root (and the
  // ILU structure inside it), so block T's panel has one row per unknown of that path.  A set
  // closed under etree ancestors is taken by decreasing etree-subtree size (a parent's is
  // larger than its child's, so every prefix is ancestor-closed) while the blocks are at most
  // 8 wide and the panels (2 x 64 B per path unknown) and bitmaps fit the budget.
  F.nzb = 0;
  F.zk = F.zA = F.zd = F.zrp = nullptr;
  F.zpb = F.zwb = nullptr;
  F.zrun = nullptr;
  F.SL = F.SU = nullptr; F.BL = F.BU = nullptr;
  h->zone_unknowns = 0;
  if (opt.zone_bytes >= 0 && n_blocks >= 2) {
    // path lengths A(K) = b_K + A(par K), parents first (par K > K)
    std::vector<int64_t> pathA(n_blocks, 0);
    for (int32_t K = n_blocks - 1; K >= 0; --K)
      pathA[K] = (bstart[K + 1] - bstart[K]) + (par[K] >= 0 ? pathA[par[K]] : 0);
    std::vector<int32_t> order(n_blocks);
    for (int32_t K = 0; K < n_blocks; ++K) order[K] = K;
    std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return sub[x] != sub[y] ? sub[x] > sub[y] : x > y; });
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const double budget = opt.zone_bytes > 0 ? (double)opt.zone_bytes : std::min(64.0 * (1ull << 30), 0.45 * (double)fr);
    int64_t nzb = 0, rows = 0, words = 0;
    double bytes = 0.0;
    for (int32_t x = 0; x < n_blocks; ++x) {
      const int32_t K = order[x], bK = bstart[K + 1] - bstart[K];
      if (bK > 8 || pathA[K] > INT32_MAX / 2) break;
      const int64_t wK = (pathA[K] + 31) / 32;
      const double add = 2.0 * (double)pathA[K] * 64.0 + 2.0 * (double)wK * 4.0;
      if (bytes + add > budget) break;
      bytes += add; nzb++; rows += pathA[K]; words += wK;
    }
    if (nzb >= 2) {
      std::vector<int32_t> zblocks(order.begin(), order.begin() + nzb);
      std::sort(zblocks.begin(), zblocks.end());
      std::vector<int32_t> zk(n_blocks, -1), zA(n_blocks, 0), zd(n, -1), zrp(nzb + 1, 0);
      std::vector<int64_t> zpb(n_blocks, -1), zwb(n_blocks, -1);
      int64_t pr = 0, pw = 0, nzu = 0;
      for (int64_t k = 0; k < nzb; ++k) {
        const int32_t K = zblocks[k];
        zk[K] = (int32_t)k; zA[K] = (int32_t)pathA[K];
        zpb[K] = pr; zwb[K] = pw;
        pr += pathA[K]; pw += (pathA[K] + 31) / 32;
        for (int32_t i = bstart[K]; i < bstart[K + 1]; ++i) zd[i] = (int32_t)(pathA[K] - (i - bstart[K]));
        nzu += bstart[K + 1] - bstart[K];
      }
      // run tables, parents first: runs(K) = [(0, s_K)] + runs(par K) shifted by b_K, the
      // parent's first run merged into K's when par K = K + 1 (consecutive unknowns)
      std::vector<std::vector<int2>> runs(nzb);
      for (int64_t k = nzb - 1; k >= 0; --k) {
        const int32_t K = zblocks[k], bK = bstart[K + 1] - bstart[K];
        std::vector<int2> &r = runs[k];
        r.push_back(make_int2(0, bstart[K]));
        if (par[K] >= 0) {
          const std::vector<int2> &rp = runs[zk[par[K]]];
          for (size_t q = (par[K] == K + 1 ? 1 : 0); q < rp.size(); ++q) r.push_back(make_int2(rp[q].x + bK, rp[q].y));
        }
      }
      std::vector<int2> zrun;
      for (int64_t k = 0; k < nzb; ++k) { zrp[k] = (int32_t)zrun.size(); zrun.insert(zrun.end(), runs[k].begin(), runs[k].end()); }
      zrp[nzb] = (int32_t)zrun.size();
      double *sl = nullptr, *su = nullptr;
      unsigned *bl = nullptr, *bu = nullptr;
      int32_t *dzk = nullptr, *dzA = nullptr, *dzd = nullptr, *dzrp = nullptr, *dzb = nullptr;
      int64_t *dpb = nullptr, *dwb = nullptr;
      int2 *drun = nullptr;
      if (dalloc(h, &sl, (size_t)(pr * 8)) == cudaSuccess && dalloc(h, &su, (size_t)(pr * 8)) == cudaSuccess &&
          dalloc(h, &bl, (size_t)pw) == cudaSuccess && dalloc(h, &bu, (size_t)pw) == cudaSuccess &&
          dalloc(h, &dzk, (size_t)n_blocks) == cudaSuccess && dalloc(h, &dzA, (size_t)n_blocks) == cudaSuccess &&
          dalloc(h, &dzd, (size_t)n) == cudaSuccess && dalloc(h, &dzrp, (size_t)(nzb + 1)) == cudaSuccess &&
          dalloc(h, &dzb, (size_t)nzb) == cudaSuccess && dalloc(h, &dpb, (size_t)n_blocks) == cudaSuccess &&
          dalloc(h, &dwb, (size_t)n_blocks) == cudaSuccess && dalloc(h, &drun, zrun.size()) == cudaSuccess) {
        h->zone_val_bytes = (size_t)pr * 8 * sizeof(double);
        h->zone_bit_bytes = (size_t)pw * sizeof(unsigned);
        cudaMemset(sl, 0, h->zone_val_bytes); cudaMemset(su, 0, h->zone_val_bytes);
        cudaMemset(bl, 0, h->zone_bit_bytes); cudaMemset(bu, 0, h->zone_bit_bytes);
        cudaMemcpy(dzk, zk.data(), n_blocks * sizeof(int32_t), cudaMemcpyHostToDevice);
        cudaMemcpy(dzA, zA.data(), n_blocks * sizeof(int32_t), cudaMemcpyHostToDevice);
        cudaMemcpy(dzd, zd.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice);
        cudaMemcpy(dzrp, zrp.data(), (nzb + 1) * sizeof(int32_t), cudaMemcpyHostToDevice);
        cudaMemcpy(dzb, zblocks.data(), nzb * sizeof(int32_t), cudaMemcpyHostToDevice);
        cudaMemcpy(dpb, zpb.data(), n_blocks * sizeof(int64_t), cudaMemcpyHostToDevice);
        cudaMemcpy(dwb, zwb.data(), n_blocks * sizeof(int64_t), cudaMemcpyHostToDevice);
        cudaMemcpy(drun, zrun.data(), zrun.size() * sizeof(int2), cudaMemcpyHostToDevice);
        F.nzb = (int)nzb;
        F.zk = dzk; F.zA = dzA; F.zd = dzd; F.zrp = dzrp; F.zpb = dpb; F.zwb = dwb; F.zrun = drun;
        h->d_zblocks = dzb;
        h->zone_unknowns = nzu;
        F.SL = sl; F.SU = su; F.BL = bl; F.BU = bu;
      } else {
        cudaGetLastError();   // no zone if it does not fit (the buffers allocated so far stay owned)
      }
    }
  }
  ALLOC(F.blk_flops, n_blocks);
  ALLOC(F.blk_ncand, 2 * (size_t)n_blocks);
  ALLOC(F.lc.cnt, n_blocks); ALLOC(F.uc.cnt, n_blocks); ALLOC(F.succ.cnt, n_blocks);
  ALLOC(F.lc.dir, (size_t)n_blocks * DIR_SLOTS);
  ALLOC(F.uc.dir, (size_t)n_blocks * DIR_SLOTS);
  ALLOC(F.succ.dir, (size_t)n_blocks * DIR_SLOTS);
  ALLOC(F.near_i, 4 * (size_t)h->near_cap); ALLOC(F.near_m, (size_t)h->near_cap);
  F.near_cap = h->near_cap;
  F.lc.rec_ints = REC_INTS; F.uc.rec_ints = REC_INTS; F.succ.rec_ints = 1;
  F.lc.ctrl_cursor = CTRL_POOL_LC; F.uc.ctrl_cursor = CTRL_POOL_UC; F.succ.ctrl_cursor = CTRL_POOL_SUCC;
#undef ALLOC

  // launch geometry: persistent CTAs, all co-resident
  F.smem_bytes = 110 * 1024;
  if (const char *sk = tune_env("BILU_SMEM_KB")) F.smem_bytes = std::max(16, std::min(220, atoi(sk))) * 1024;
  int per_sm = 0;
  if (bilu_factor_occupancy(F.smem_bytes, &per_sm) != cudaSuccess || per_sm < 1) per_sm = 1;
  const int occ = per_sm;
  per_sm = 1;   // one CTA per SM: the rest of the unified L1/shared array caches panels
  if (const char *cp = tune_env("BILU_CTAS_PER_SM")) per_sm = std::max(1, std::min(occ, atoi(cp)));
  h->grid = opt.n_ctas > 0 ? opt.n_ctas : h->sms * per_sm;

  // initial capacities (grown on overflow)
  {
    // factor arenas (grow on overflow): values ~ max(4 nnz, 400 n) doubles each for L and Ũ
    // (3D ND stencils keep ~300-400 values per row at tau = 1e-3, block-sparse inputs ~nnz/2),
    // indices one per kept row / column, capped at half of the free device memory
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const double avg_b = (double)n / std::max<int32_t>(n_blocks, 1);
    int64_t cv = opt.arena_hint > 0 ? opt.arena_hint : std::max<int64_t>(4 * nnz, 400 * (int64_t)n);
    const int64_t budget = (int64_t)(0.5 * (double)fr / (16.0 + 8.0 / avg_b));
    if (opt.arena_hint <= 0) cv = std::max<int64_t>(std::min(cv, budget), (int64_t)n * max_b);
    h->cap_val = cv;
    h->cap_idx = (int64_t)((double)cv / avg_b) + 2 * (int64_t)n + 1024;
  }
  h->work_per_cta = 256 * 1024;
  {
    // split-block pool: W buffers of the blocks processed as parallel tasks (grows on demand)
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    h->hpool_cap = std::min<int64_t>(std::max<int64_t>(1 << 22, 64 * nnz), (int64_t)(fr / 8 / 8));
  }
  h->pool_lc = h->pool_uc = std::max(2 * n_blocks, 1024);
  h->pool_succ = std::max(2 * n_blocks, 1024);

  if (val) {
    bilu_status st = bilu_set_values(h, val, 0);
    if (st != BILU_OK) { g_last_error = h->err; bilu_destroy(h); return st; }
  }
  *out = h;
  return BILU_OK;
}

// ------------------------------------------------------------ set values
extern "C" bilu_status bilu_set_values(bilu_ctx *h, const double *val, int32_t on_device) {
  if (!h || !val) { set_err(h, "bilu_set_values: null argument"); return BILU_ERR_ARG; }
  cudaSetDevice(h->opt.device);
  CUDA_TRY(h, cudaMemcpyAsync(h->d_val_orig, val, h->nnz * sizeof(double),
                              on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, bilu_launch_maxabs(h->d_alpha, h->d_val_orig, h->nnz, h->stream));   // alpha of Sec. 3.6
  h->launches += 1;
  if (h->nAL) CUDA_TRY(h, bilu_launch_gather(h->d_AL_val, h->d_val_orig, h->d_AL_map, h->nAL, h->stream));
  if (h->nAU) CUDA_TRY(h, bilu_launch_gather(h->d_AU_val, h->d_val_orig, h->d_AU_map, h->nAU, h->stream));
  h->launches += 2;
  h->factored = false;
  return BILU_OK;
}

// ------------------------------------------------------------ capacities
static bilu_status ensure_aux(bilu_ctx *h);
static bilu_status ensure_capacity(bilu_ctx *h) {
  DevFactor &F = h->F;
  if (F.cap_Lval != h->cap_val) {
    dfree(h, F.Lval); dfree(h, F.Uval);
    CUDA_TRY(h, dalloc(h, &F.Lval, h->cap_val));
    CUDA_TRY(h, dalloc(h, &F.Uval, h->cap_val));
    F.cap_Lval = F.cap_Uval = h->cap_val;
  }
  if (F.cap_Lidx != h->cap_idx) {
    dfree(h, F.Lidx); dfree(h, F.Uidx);
    CUDA_TRY(h, dalloc(h, &F.Lidx, h->cap_idx));
    CUDA_TRY(h, dalloc(h, &F.Uidx, h->cap_idx));
    F.cap_Lidx = F.cap_Uidx = h->cap_idx;
  }
  return ensure_aux(h);
}

// workspaces that hold no factor data (safe to reallocate between phases)
static bilu_status ensure_aux(bilu_ctx *h) {
  DevFactor &F = h->F;
  if (!F.posmap) CUDA_TRY(h, dalloc(h, &F.posmap, (size_t)h->grid * h->n));
  if (F.hpool_cap != h->hpool_cap) {
    dfree(h, F.hpool);
    CUDA_TRY(h, dalloc(h, &F.hpool, (size_t)h->hpool_cap));
    F.hpool_cap = h->hpool_cap;
    // invariant: the pool is zero when a launch starts (split blocks' W need no zero fill)
    CUDA_TRY(h, cudaMemsetAsync(F.hpool, 0, (size_t)h->hpool_cap * 8, h->stream));
    h->hpool_dirty = 0;
  }
  if (F.work_per_cta != h->work_per_cta) {
    dfree(h, F.work);
    CUDA_TRY(h, dalloc(h, &F.work, (size_t)h->work_per_cta * h->grid));
    F.work_per_cta = h->work_per_cta;
  }
  if (F.lc.pool_cap != h->pool_lc) {
    dfree(h, F.lc.pool);
    CUDA_TRY(h, dalloc(h, &F.lc.pool, (size_t)h->pool_lc * CHUNK * REC_INTS));
    F.lc.pool_cap = h->pool_lc;
  }
  if (F.uc.pool_cap != h->pool_uc) {
    dfree(h, F.uc.pool);
    CUDA_TRY(h, dalloc(h, &F.uc.pool, (size_t)h->pool_uc * CHUNK * REC_INTS));
    F.uc.pool_cap = h->pool_uc;
  }
  if (F.succ.pool_cap != h->pool_succ) {
    dfree(h, F.succ.pool);
    CUDA_TRY(h, dalloc(h, &F.succ.pool, (size_t)h->pool_succ * CHUNK));
    F.succ.pool_cap = h->pool_succ;
  }
  return BILU_OK;
}

static bilu_status reset_schedule(bilu_ctx *h, const int32_t *d_ready, int32_t nready) {
  DevFactor &F = h->F;
  cudaStream_t st = h->stream;
  const size_t N = h->N;
  h->qhead0 = (unsigned long long)nready;
  CUDA_TRY(h, cudaMemcpyAsync(F.pending, h->d_pending0, N * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(h, cudaMemsetAsync(F.queue, 0xFF, F.qcap * sizeof(int32_t), st));
  CUDA_TRY(h, cudaMemsetAsync(F.hq, 0xFF, F.hqcap * sizeof(int32_t), st));
  if (nready)
    CUDA_TRY(h, cudaMemcpyAsync(F.queue, d_ready, nready * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(h, cudaMemsetAsync(F.ctrl, 0, CTRL_COUNT * CS * sizeof(unsigned long long), st));
  CUDA_TRY(h, cudaMemcpyAsync(F.ctrl + CS * CTRL_QHEAD, &h->qhead0, sizeof(unsigned long long),
                              cudaMemcpyHostToDevice, st));
  CUDA_TRY(h, cudaMemsetAsync(F.lc.cnt, 0, N * sizeof(int), st));
  CUDA_TRY(h, cudaMemsetAsync(F.uc.cnt, 0, N * sizeof(int), st));
  CUDA_TRY(h, cudaMemsetAsync(F.succ.cnt, 0, N * sizeof(int), st));
  CUDA_TRY(h, cudaMemsetAsync(F.lc.dir, 0xFF, N * DIR_SLOTS * sizeof(int), st));
  CUDA_TRY(h, cudaMemsetAsync(F.uc.dir, 0xFF, N * DIR_SLOTS * sizeof(int), st));
  CUDA_TRY(h, cudaMemsetAsync(F.succ.dir, 0xFF, N * DIR_SLOTS * sizeof(int), st));
  return BILU_OK;
}

// ------------------------------------------------------------ finalize
// Grows one arena to hold `need` elements, keeping the first `used` ones.
template <typename T>
static bilu_status grow_keep(bilu_ctx *h, T *&p, int64_t &cap, int64_t need, int64_t used) {
  if (need <= cap) return BILU_OK;
  int64_t nc = std::max<int64_t>(need + need / 4, 2 * cap);
  T *q = nullptr;
  CUDA_TRY(h, dalloc(h, &q, nc));
  if (used > 0) CUDA_TRY(h, cudaMemcpyAsync(q, p, used * sizeof(T), cudaMemcpyDeviceToDevice, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  dfree(h, p);
  p = q;
  cap = nc;
  return BILU_OK;
}

static bilu_status finalize(bilu_ctx *h, const unsigned long long *ctrl, bilu_factor_stats &S, int &launches) {
  DevFactor &F = h->F;
  FinalFactor &fin = h->fin;
  const int N = h->N;
  double fl;
  memcpy(&fl, &ctrl[CTRL_FLOPS], sizeof(double));
  S.flops = fl;
  h->apply_ready = false;
  if (!h->opt.aggregate) {
    fin.nF = N;
    fin.bstart = h->d_bstart;
    fin.Lrow_off = F.Lrow_off; fin.Lval_off = F.Lval_off; fin.Lm = F.Lm;
    fin.Ucol_off = F.Ucol_off; fin.Uval_off = F.Uval_off; fin.Uc = F.Uc;
    fin.D_off = const_cast<int64_t *>(F.D_off); fin.D = F.D;
    fin.nidxL = fin.usedLi = (int64_t)ctrl[CTRL_CUR_LIDX]; fin.nnzL = fin.usedLv = (int64_t)ctrl[CTRL_CUR_LVAL];
    fin.nidxU = fin.usedUi = (int64_t)ctrl[CTRL_CUR_UIDX]; fin.nnzU = fin.usedUv = (int64_t)ctrl[CTRL_CUR_UVAL];
    fin.nnzD = h->D_off[N];
    S.n_blocks_final = N;
    S.n_merges = 0;
  } else {
    MergeArgs &M = h->M;
    if (!h->merge_alloc) {
      CUDA_TRY(h, dalloc(h, &M.T, 4 * (size_t)N));
      CUDA_TRY(h, dalloc(h, &M.first, (size_t)N + 1));
      CUDA_TRY(h, dalloc(h, &M.nF, 1));
      CUDA_TRY(h, dalloc(h, &M.fbstart, (size_t)N + 1));
      CUDA_TRY(h, dalloc(h, &M.fLm, (size_t)N)); CUDA_TRY(h, dalloc(h, &M.fUc, (size_t)N));
      CUDA_TRY(h, dalloc(h, &M.fLrow_off, (size_t)N)); CUDA_TRY(h, dalloc(h, &M.fLval_off, (size_t)N));
      CUDA_TRY(h, dalloc(h, &M.fUcol_off, (size_t)N)); CUDA_TRY(h, dalloc(h, &M.fUval_off, (size_t)N));
      CUDA_TRY(h, dalloc(h, &M.fD_off, (size_t)N + 1));
      CUDA_TRY(h, dalloc(h, &M.tot, 16)); CUDA_TRY(h, dalloc(h, &M.flops, 1)); CUDA_TRY(h, dalloc(h, &M.ovf, 1));
      // test windows: W_k = largest W <= 127 with s_k - s_{k-W} + q_k <= max_block
      {
        std::vector<int64_t> wofs(N + 1);
        int64_t acc = 0;
        const std::vector<int32_t> &bs = h->bstart;
        for (int k = 0; k < N; ++k) {
          int W = 0;
          if (k > 0) {
            const int sk = bs[k], q = bs[k + 1] - sk;
            while (k - 1 - W >= 0 && (sk - bs[k - 1 - W]) + q <= h->opt.max_block && W < 127 &&
                   (h->seg.empty() || h->seg[k - 1 - W] == h->seg[k]))
              ++W;
          }
          wofs[k] = acc;
          acc += W + 1;
        }
        wofs[N] = acc;     // W_k = wofs[k+1] - wofs[k] - 1
        int64_t *d_wofs = nullptr;
        CUDA_TRY(h, dalloc(h, &d_wofs, (size_t)N + 1));
        CUDA_TRY(h, cudaMemcpy(d_wofs, wofs.data(), (N + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
        M.wofs = d_wofs;
        CUDA_TRY(h, dalloc(h, &M.UV, 2 * (size_t)std::max<int64_t>(acc, 1)));
        const int nch = bilu_merge_nchunks(N);
        CUDA_TRY(h, dalloc(h, &M.chunkmap, (size_t)std::max(nch, 1) * 128));
        CUDA_TRY(h, dalloc(h, &M.chunkstart, (size_t)std::max(nch, 1)));
        CUDA_TRY(h, dalloc(h, &M.flag, (size_t)N));
      }
      h->merge_work_ints = 16384;
      CUDA_TRY(h, dalloc(h, &M.work, (size_t)h->merge_work_ints * 2 * h->sms));
      h->fD_cap = std::max<int64_t>(h->D_off[N], 1);
      CUDA_TRY(h, dalloc(h, &M.fD, h->fD_cap));
      h->merge_alloc = true;
    }
    M.n = h->n; M.N = N; M.max_block = h->opt.max_block;
    M.seg = h->dist ? h->d_seg : nullptr;
    M.bstart = h->d_bstart;
    M.Lrow_off = F.Lrow_off; M.Lm = F.Lm; M.Lval_off = F.Lval_off;
    M.Ucol_off = F.Ucol_off; M.Uc = F.Uc; M.Uval_off = F.Uval_off;
    M.D = F.D; M.D_off = F.D_off;
    M.work_ints = h->merge_work_ints;
    {   // windows too wide for the test's shared-memory table use per-CTA global tables
      M.Lidx = F.Lidx; M.Uidx = F.Uidx;
      if (!h->d_mbound) CUDA_TRY(h, dalloc(h, &h->d_mbound, 1));
      if (!h->d_mticket) CUDA_TRY(h, dalloc(h, &h->d_mticket, 1));
      M.ticket = h->d_mticket;
      CUDA_TRY(h, bilu_merge_bound(M, h->d_mbound, h->sms, h->stream));
      launches += 1;
      unsigned long long mx = 0;
      CUDA_TRY(h, cudaMemcpyAsync(&mx, h->d_mbound, sizeof(mx), cudaMemcpyDeviceToHost, h->stream));
      CUDA_TRY(h, cudaStreamSynchronize(h->stream));
      int64_t cap = 64;
      while (cap < 2 * (int64_t)mx) cap <<= 1;
      if (cap > 8192 && cap > h->mhbig_cap) {
        if (h->d_mhbig) dfree(h, h->d_mhbig);
        h->d_mhbig = nullptr;
        CUDA_TRY(h, dalloc(h, &h->d_mhbig, (size_t)bilu_merge_test_grid(h->grid) * 9 * (size_t)cap));
        h->mhbig_cap = cap;
      }
      M.hbig = h->d_mhbig;
      M.hbig_cap = h->mhbig_cap;
    }
    unsigned long long tot[16];
    for (int attempt = 0;; ++attempt) {
      M.Lidx = F.Lidx; M.Uidx = F.Uidx; M.Lval = F.Lval; M.Uval = F.Uval;
      unsigned long long cur[4] = {ctrl[CTRL_CUR_LIDX], ctrl[CTRL_CUR_LVAL], ctrl[CTRL_CUR_UIDX], ctrl[CTRL_CUR_UVAL]};
      CUDA_TRY(h, cudaMemcpyAsync(M.tot, cur, sizeof(cur), cudaMemcpyHostToDevice, h->stream));
      CUDA_TRY(h, cudaMemsetAsync(M.ovf, 0, sizeof(int), h->stream));
      CUDA_TRY(h, cudaMemsetAsync(M.flops, 0, sizeof(double), h->stream));
      CUDA_TRY(h, cudaMemsetAsync(h->d_mticket, 0, sizeof(int), h->stream));
      CUDA_TRY(h, bilu_merge_plan(M, h->grid, h->stream));
      launches += bilu_merge_plan_launches();
      int ovf = 0;
      CUDA_TRY(h, cudaMemcpyAsync(tot, M.tot, sizeof(tot), cudaMemcpyDeviceToHost, h->stream));
      CUDA_TRY(h, cudaMemcpyAsync(&ovf, M.ovf, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
      CUDA_TRY(h, cudaStreamSynchronize(h->stream));
      if (!ovf) break;
      if (attempt > 8) { set_err(h, "bilu_factor: merge workspace overflow"); return BILU_ERR_OOM; }
      dfree(h, M.work);
      h->merge_work_ints *= 4;
      CUDA_TRY(h, dalloc(h, &M.work, (size_t)h->merge_work_ints * 2 * h->sms));
      M.work_ints = h->merge_work_ints;
      S.n_retries++;
    }
    const int nF = (int)(N - (int64_t)tot[11]);
    // arenas: merged panels are appended after the factor kernel's cursors
    bilu_status bs;
    if ((bs = grow_keep(h, F.Lidx, F.cap_Lidx, (int64_t)tot[4], (int64_t)ctrl[CTRL_CUR_LIDX])) != BILU_OK) return bs;
    if ((bs = grow_keep(h, F.Lval, F.cap_Lval, (int64_t)tot[5], (int64_t)ctrl[CTRL_CUR_LVAL])) != BILU_OK) return bs;
    if ((bs = grow_keep(h, F.Uidx, F.cap_Uidx, (int64_t)tot[6], (int64_t)ctrl[CTRL_CUR_UIDX])) != BILU_OK) return bs;
    if ((bs = grow_keep(h, F.Uval, F.cap_Uval, (int64_t)tot[7], (int64_t)ctrl[CTRL_CUR_UVAL])) != BILU_OK) return bs;
    h->cap_val = std::max(F.cap_Lval, F.cap_Uval); h->cap_idx = std::max(F.cap_Lidx, F.cap_Uidx);
    F.cap_Lval = F.cap_Uval = h->cap_val; F.cap_Lidx = F.cap_Uidx = h->cap_idx;
    if ((int64_t)tot[8] > h->fD_cap) {
      dfree(h, M.fD);
      h->fD_cap = (int64_t)tot[8] + (int64_t)tot[8] / 4;
      CUDA_TRY(h, dalloc(h, &M.fD, h->fD_cap));
    }
    // per-CTA dense L_aa, U_aa of runs wider than the shared-memory tile
    const int64_t need_dw = 3 * (int64_t)h->opt.max_block * h->opt.max_block + (int64_t)tot[9];
    const int mgrid = 2 * h->sms;
    if (need_dw > h->merge_dwork) {
      dfree(h, h->d_mdwork);
      h->merge_dwork = need_dw;
      CUDA_TRY(h, dalloc(h, &h->d_mdwork, (size_t)need_dw * mgrid));
    }
    M.Lidx = F.Lidx; M.Uidx = F.Uidx; M.Lval = F.Lval; M.Uval = F.Uval;
    M.Lidx_out = F.Lidx; M.Uidx_out = F.Uidx; M.Lval_out = F.Lval; M.Uval_out = F.Uval;
    double mfl = 0.0;
    for (int attempt = 0;; ++attempt) {
      int ovf = 0;
      CUDA_TRY(h, cudaMemsetAsync(M.ovf, 0, sizeof(int), h->stream));
      CUDA_TRY(h, cudaMemsetAsync(M.flops, 0, sizeof(double), h->stream));
      if (!h->d_mticket) CUDA_TRY(h, dalloc(h, &h->d_mticket, 1));
      CUDA_TRY(h, cudaMemsetAsync(h->d_mticket, 0, sizeof(int), h->stream));
      M.ticket = h->d_mticket;
      CUDA_TRY(h, bilu_merge_arith(M, h->d_mdwork, h->merge_dwork, mgrid, h->stream));
      launches += 1;
      CUDA_TRY(h, cudaMemcpyAsync(&mfl, M.flops, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
      CUDA_TRY(h, cudaMemcpyAsync(&ovf, M.ovf, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
      CUDA_TRY(h, cudaStreamSynchronize(h->stream));
      if (!ovf) break;
      if (ovf == 2) { set_err(h, "bilu_factor: merged union size differs from the aggregation test"); return BILU_ERR_STATE; }
      if (attempt > 8) { set_err(h, "bilu_factor: merge workspace overflow in arithmetic"); return BILU_ERR_OOM; }
      dfree(h, M.work);
      h->merge_work_ints *= 4;
      CUDA_TRY(h, dalloc(h, &M.work, (size_t)h->merge_work_ints * 2 * h->sms));
      M.work_ints = h->merge_work_ints;
      S.n_retries++;
    }
    S.flops += mfl;
    fin.nF = nF;
    fin.bstart = M.fbstart;
    fin.Lrow_off = M.fLrow_off; fin.Lval_off = M.fLval_off; fin.Lm = M.fLm;
    fin.Ucol_off = M.fUcol_off; fin.Uval_off = M.fUval_off; fin.Uc = M.fUc;
    fin.D_off = M.fD_off; fin.D = M.fD;
    fin.usedLi = (int64_t)tot[4]; fin.usedLv = (int64_t)tot[5];
    fin.usedUi = (int64_t)tot[6]; fin.usedUv = (int64_t)tot[7];
    fin.nnzD = (int64_t)tot[8];
    fin.nnzL = (int64_t)tot[12]; fin.nnzU = (int64_t)tot[13];
    fin.nidxL = (int64_t)tot[14]; fin.nidxU = (int64_t)tot[15];
    S.n_blocks_final = nF;
    S.n_merges = (int32_t)tot[11];
  }
  S.nnz_D = fin.nnzD;
  S.nnz_L = fin.nnzL;
  S.nnz_U = fin.nnzU;
  S.bytes_min = 12.0 * (double)h->nnz + 4.0 * (h->n + 1) + 8.0 * (double)(fin.nnzL + fin.nnzU + fin.nnzD) +
                4.0 * (double)(fin.nidxL + fin.nidxU);
  return BILU_OK;
}

// ------------------------------------------------------------ factor
enum Phase { PH_ALL = 0, PH_LOCAL = 1, PH_SEP = 2 };

static bilu_status prepare_separators(bilu_ctx *h);

// One launch of the persistent factor kernel over the blocks of `ph` (all blocks, this
// rank's subtree blocks, or the separator blocks), with the regrow-and-retry loop for the
// device workspaces.  e0/e1 bracket the successful attempt.
static bilu_status run_phase(bilu_ctx *h, Phase ph, bilu_factor_stats &S, unsigned long long *ctrl, cudaEvent_t e0,
                             cudaEvent_t e1, int &launches) {
  DevFactor &F = h->F;
  for (int attempt = 0;; ++attempt) {
    bilu_status bs = ph == PH_SEP ? ensure_aux(h) : ensure_capacity(h);
    if (bs != BILU_OK) return bs;
    CUDA_TRY(h, cudaEventRecord(e0, h->stream));
    if (ph == PH_ALL) { F.owned = nullptr; F.n_target = h->N; bs = reset_schedule(h, h->d_ready0, h->nready0); }
    else if (ph == PH_LOCAL) {
      F.owned = h->d_own_mask; F.n_target = (int64_t)h->own_list.size();
      bs = reset_schedule(h, h->d_own_ready, h->n_own_ready);
    } else {
      F.owned = h->d_sep_mask; F.n_target = h->N;
      bs = prepare_separators(h);
    }
    if (bs != BILU_OK) return bs;
    const char *dbg_env = tune_env("BILU_DEBUG_TIMEOUT");
    if (dbg_env && !F.dbg) {
      void *hp = nullptr, *dp = nullptr;
      CUDA_TRY(h, cudaHostAlloc(&hp, 4 * sizeof(int) * h->grid, cudaHostAllocMapped));
      memset(hp, 0, 4 * sizeof(int) * h->grid);
      CUDA_TRY(h, cudaHostGetDevicePointer(&dp, hp, 0));
      F.dbg = (volatile int *)dp;
      h->dbg_host = (volatile int *)hp;
    }
    if (h->hpool_dirty > 0) {   // re-zero what the previous launch used
      CUDA_TRY(h, cudaMemsetAsync(F.hpool, 0, (size_t)std::min(h->hpool_dirty, F.hpool_cap) * 8, h->stream));
      h->hpool_dirty = 0;
    }
    if (F.nzb > 0) {            // dense zone: Ã's entries in (zero buffers)
      if (h->zone_dirty) {
        CUDA_TRY(h, cudaMemsetAsync(F.SL, 0, h->zone_val_bytes, h->stream));
        CUDA_TRY(h, cudaMemsetAsync(F.SU, 0, h->zone_val_bytes, h->stream));
        CUDA_TRY(h, cudaMemsetAsync(F.BL, 0, h->zone_bit_bytes, h->stream));
        CUDA_TRY(h, cudaMemsetAsync(F.BU, 0, h->zone_bit_bytes, h->stream));
      }
      CUDA_TRY(h, bilu_launch_zone_init(F, h->d_zblocks, h->stream));
      launches += 1;
      h->zone_dirty = true;
    }
    CUDA_TRY(h, bilu_launch_factor(F, h->grid, h->stream));
    launches += 1;
    if (dbg_env) {
      const double limit = atof(dbg_env);
      const double t_start = (double)clock() / CLOCKS_PER_SEC;
      while (cudaStreamQuery(h->stream) == cudaErrorNotReady) {
        if ((double)clock() / CLOCKS_PER_SEC - t_start > limit) {
          fprintf(stderr, "bilu watchdog: factor kernel still running after %.0f s; CTA progress (K, phase, blocks done):\n", limit);
          for (int c = 0; c < h->grid; ++c)
            if (h->dbg_host[4 * c + 2])
              fprintf(stderr, "  cta %3d: K=%d phase=%d done=%d\n", c, h->dbg_host[4 * c], h->dbg_host[4 * c + 1], h->dbg_host[4 * c + 2]);
          fflush(stderr);
          _exit(3);
        }
      }
    }
    CUDA_TRY(h, cudaEventRecord(e1, h->stream));
    CUDA_TRY(h, cudaMemcpyAsync(h->ctrl_full, F.ctrl, sizeof(h->ctrl_full), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    for (int i = 0; i < CTRL_COUNT; ++i) ctrl[i] = h->ctrl_full[CS * i];
    h->hpool_dirty = std::min<int64_t>((int64_t)ctrl[CTRL_HPOOL], F.hpool_cap);
    const int code = (int)ctrl[CTRL_ABORT];
    if (code == DEV_OK) {
      if (ctrl[CTRL_DONE] == (unsigned long long)F.n_target) h->zone_dirty = false;   // every zone block consumed its panel
      if (ctrl[CTRL_DONE] != (unsigned long long)F.n_target) {
        set_err(h, "bilu_factor: schedule finished %llu of %lld blocks", ctrl[CTRL_DONE], (long long)F.n_target);
        return BILU_ERR_STATE;
      }
      return BILU_OK;
    }
    if (code == DEV_BREAKDOWN) {
      S.breakdown_block = (int32_t)ctrl[CTRL_ERRBLK];
      set_err(h, "bilu_factor: pivot block %d is exactly singular", S.breakdown_block);
      return BILU_ERR_BREAKDOWN;
    }
    if (tune_env("BILU_VERBOSE"))
      fprintf(stderr, "bilu_factor retry %d (phase %d): code %d block %llu hpool %lld/%lld hctx %llu/%lld work %lld\n",
              attempt, (int)ph, code, ctrl[CTRL_ERRBLK], (long long)ctrl[CTRL_HPOOL], (long long)h->hpool_cap,
              ctrl[CTRL_HCTX], (long long)F.hctx_cap, (long long)h->work_per_cta);
    if (attempt >= 12) { set_err(h, "bilu_factor: workspace overflow persists (code %d)", code); return BILU_ERR_OOM; }
    S.n_retries++;
    switch (code) {
      case DEV_OVF_ARENA:
        if (ph == PH_SEP) {   // keep the factors of phase A and of the received interface blocks
          bilu_status gs;
          if ((gs = grow_keep(h, F.Lidx, F.cap_Lidx, 2 * F.cap_Lidx, (int64_t)h->cur[0])) != BILU_OK) return gs;
          if ((gs = grow_keep(h, F.Lval, F.cap_Lval, 2 * F.cap_Lval, (int64_t)h->cur[1])) != BILU_OK) return gs;
          if ((gs = grow_keep(h, F.Uidx, F.cap_Uidx, 2 * F.cap_Uidx, (int64_t)h->cur[2])) != BILU_OK) return gs;
          if ((gs = grow_keep(h, F.Uval, F.cap_Uval, 2 * F.cap_Uval, (int64_t)h->cur[3])) != BILU_OK) return gs;
          h->cap_val = std::max(F.cap_Lval, F.cap_Uval); h->cap_idx = std::max(F.cap_Lidx, F.cap_Uidx);
        } else {
          h->cap_val *= 2; h->cap_idx *= 2;
        }
        break;
      case DEV_OVF_WORK: h->work_per_cta *= 4; break;
      case DEV_OVF_POOL: h->pool_lc *= 2; h->pool_uc *= 2; h->pool_succ *= 2; break;
      case DEV_OVF_HPOOL:
        h->hpool_cap = std::max<int64_t>(2 * h->hpool_cap, (int64_t)ctrl[CTRL_HPOOL] + (int64_t)ctrl[CTRL_HPOOL] / 4);
        break;
      case DEV_OVF_HCTX: F.heavy_T *= 2; F.wide_flops *= 2; break;   // fewer split blocks
      default: set_err(h, "bilu_factor: device list overflow (code %d, block %llu)", code, ctrl[CTRL_ERRBLK]); return BILU_ERR_OOM;
    }
  }
}

static void factor_setup(bilu_ctx *h, double tau) {
  DevFactor &F = h->F;
  F.tau = tau;
  F.near_rel = h->opt.near_rel;
}

// finalize (aggregation post-pass) + statistics shared by bilu_factor and the separator phase
static bilu_status finish_factor(bilu_ctx *h, bilu_factor_stats &S, unsigned long long *ctrl, cudaEvent_t e0,
                                 cudaEvent_t e1, cudaEvent_t e2, int launches, bilu_factor_stats *st_out) {
  h->launches += launches;
  S.n_decisions += (int64_t)ctrl[CTRL_NDEC];
  S.n_near += (int64_t)ctrl[CTRL_NEAR];
  S.n_perturbed += (int64_t)ctrl[CTRL_NPERT];
  int mlaunch = 0;
  bilu_status ms = finalize(h, ctrl, S, mlaunch);
  if (ms != BILU_OK) return ms;
  launches += mlaunch;
  h->launches += mlaunch;
  CUDA_TRY(h, cudaEventRecord(e2, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  float ms1 = 0.f, ms2 = 0.f;
  cudaEventElapsedTime(&ms1, e0, e1);
  cudaEventElapsedTime(&ms2, e1, e2);
  S.t_factor_ms += ms1 + ms2;
  S.t_merge_ms = ms2;
  S.n_kernel_launches += launches;
  h->factored = true;
  h->last = S;
  if (st_out) *st_out = S;
  return BILU_OK;
}

struct Events {
  cudaEvent_t e[3] = {nullptr, nullptr, nullptr};
  ~Events() { for (auto x : e) if (x) cudaEventDestroy(x); }
};

extern "C" bilu_status bilu_factor(bilu_ctx *h, double tau, bilu_factor_stats *st_out) {
  if (!h) { set_err(nullptr, "bilu_factor: null context"); return BILU_ERR_ARG; }
  if (!(tau >= 0.0)) { set_err(h, "bilu_factor: tau must be >= 0"); return BILU_ERR_ARG; }
  if (h->dist) { set_err(h, "bilu_factor: distributed context; use bilu_factor_local / bilu_factor_separators"); return BILU_ERR_STATE; }
  cudaSetDevice(h->opt.device);
  factor_setup(h, tau);
  bilu_factor_stats S{};
  S.breakdown_block = -1;
  S.n_blocks_init = h->N;
  S.zone_blocks = h->F.nzb;
  S.zone_unknowns = h->F.nzb > 0 ? (int32_t)h->zone_unknowns : 0;
  Events ev;
  for (auto &x : ev.e) CUDA_TRY(h, cudaEventCreate(&x));
  h->factored = false;
  int launches = 0;
  unsigned long long ctrl[CTRL_COUNT];
  bilu_status bs = run_phase(h, PH_ALL, S, ctrl, ev.e[0], ev.e[1], launches);
  if (bs != BILU_OK) { if (st_out) *st_out = S; return bs; }
  return finish_factor(h, S, ctrl, ev.e[0], ev.e[1], ev.e[2], launches, st_out);
}

// ------------------------------------------------------------ distributed
extern "C" bilu_status bilu_dist_setup(bilu_ctx *h, const int32_t *owner, int32_t rank) {
  if (!h || !owner || rank < 0) { set_err(h, "bilu_dist_setup: null argument or negative rank"); return BILU_ERR_ARG; }
  if (h->merge_alloc || h->factored) {
    set_err(h, "bilu_dist_setup: must be called before the first factorization");
    return BILU_ERR_STATE;
  }
  const int N = h->N;
  h->owner.assign(owner, owner + N);
  h->rank = rank;
  h->F.nzb = 0;   // the distributed phases run the contributor-list path only
  h->own_list.clear(); h->sep_list.clear();
  for (int K = 0; K < N; ++K) {
    if (owner[K] < -1) { set_err(h, "bilu_dist_setup: owner[%d] = %d < -1", K, owner[K]); return BILU_ERR_ARG; }
    if (owner[K] == rank) h->own_list.push_back(K);
    else if (owner[K] == -1) h->sep_list.push_back(K);
  }
  // the partition must separate: no coupling between blocks of different ranks, and no
  // subtree block after a separator block it is coupled to (it could not finish in phase A)
  h->static_sep.assign(h->sep_list.size(), 0);
  std::vector<int32_t> sep_pos(N, -1);
  for (size_t x = 0; x < h->sep_list.size(); ++x) sep_pos[h->sep_list[x]] = (int32_t)x;
  for (int a = 0; a < N; ++a)
    for (int32_t q = h->adj_ptr_h[a]; q < h->adj_ptr_h[a + 1]; ++q) {
      const int b = h->adj_h[q];   // a < b, coupled
      if (owner[a] >= 0 && owner[b] >= 0 && owner[a] != owner[b]) {
        set_err(h, "bilu_dist_setup: blocks %d (rank %d) and %d (rank %d) are coupled", a, owner[a], b, owner[b]);
        return BILU_ERR_ARG;
      }
      if (owner[a] == -1 && owner[b] >= 0) {
        set_err(h, "bilu_dist_setup: subtree block %d follows separator block %d it is coupled to", b, a);
        return BILU_ERR_ARG;
      }
      if (owner[a] == -1 && owner[b] == -1) h->static_sep[sep_pos[b]]++;
    }
  std::vector<int32_t> ready, segv(N);
  std::vector<uint8_t> own_mask(N, 0), sep_mask(N, 0);
  for (int K : h->own_list) { own_mask[K] = 1; if (h->pending0_h[K] == 0) ready.push_back(K); }
  for (int K : h->sep_list) sep_mask[K] = 1;
  for (int K = 0; K < N; ++K) segv[K] = (owner[K] == rank || owner[K] == -1) ? owner[K] : -(K + 2);
  h->seg = segv;
  h->n_own_ready = (int32_t)ready.size();
  const size_t nown = h->own_list.size(), nsep = h->sep_list.size();
  CUDA_TRY(h, dalloc(h, &h->d_own_mask, (size_t)N)); CUDA_TRY(h, dalloc(h, &h->d_sep_mask, (size_t)N));
  CUDA_TRY(h, dalloc(h, &h->d_own_list, std::max<size_t>(nown, 1))); CUDA_TRY(h, dalloc(h, &h->d_sep_list, std::max<size_t>(nsep, 1)));
  CUDA_TRY(h, dalloc(h, &h->d_static_sep, std::max<size_t>(nsep, 1)));
  CUDA_TRY(h, dalloc(h, &h->d_seg, (size_t)N));
  CUDA_TRY(h, dalloc(h, &h->d_own_ready, std::max<size_t>(ready.size(), 1)));
  CUDA_TRY(h, dalloc(h, &h->d_flag, std::max<size_t>(nown, 1)));
  CUDA_TRY(h, cudaMemcpy(h->d_own_mask, own_mask.data(), N, cudaMemcpyHostToDevice));
  CUDA_TRY(h, cudaMemcpy(h->d_sep_mask, sep_mask.data(), N, cudaMemcpyHostToDevice));
  if (nown) CUDA_TRY(h, cudaMemcpy(h->d_own_list, h->own_list.data(), nown * 4, cudaMemcpyHostToDevice));
  if (nsep) CUDA_TRY(h, cudaMemcpy(h->d_sep_list, h->sep_list.data(), nsep * 4, cudaMemcpyHostToDevice));
  if (nsep) CUDA_TRY(h, cudaMemcpy(h->d_static_sep, h->static_sep.data(), nsep * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(h, cudaMemcpy(h->d_seg, segv.data(), (size_t)N * 4, cudaMemcpyHostToDevice));
  if (!ready.empty()) CUDA_TRY(h, cudaMemcpy(h->d_own_ready, ready.data(), ready.size() * 4, cudaMemcpyHostToDevice));
  h->dist = true;
  h->dist_local_done = false;
  return BILU_OK;
}

extern "C" bilu_status bilu_factor_local(bilu_ctx *h, double tau, bilu_factor_stats *st_out) {
  if (!h) { set_err(nullptr, "bilu_factor_local: null context"); return BILU_ERR_ARG; }
  if (!h->dist) { set_err(h, "bilu_factor_local: call bilu_dist_setup first"); return BILU_ERR_STATE; }
  if (!(tau >= 0.0)) { set_err(h, "bilu_factor_local: tau must be >= 0"); return BILU_ERR_ARG; }
  cudaSetDevice(h->opt.device);
  factor_setup(h, tau);
  DevFactor &F = h->F;
  bilu_factor_stats S{};
  S.breakdown_block = -1;
  S.n_blocks_init = h->N;
  S.zone_blocks = h->F.nzb;
  S.zone_unknowns = h->F.nzb > 0 ? (int32_t)h->zone_unknowns : 0;
  Events ev;
  for (auto &x : ev.e) CUDA_TRY(h, cudaEventCreate(&x));
  h->factored = false;
  h->dist_local_done = false;
  h->remote_ifc.clear();
  h->own_ifc.clear();
  // descriptors of every block empty: blocks of other ranks stay absent
  {
    bilu_status bs = ensure_capacity(h);
    if (bs != BILU_OK) return bs;
    const size_t N = h->N;
    CUDA_TRY(h, cudaMemsetAsync(F.Lm, 0, N * 4, h->stream)); CUDA_TRY(h, cudaMemsetAsync(F.Uc, 0, N * 4, h->stream));
    CUDA_TRY(h, cudaMemsetAsync(F.Lrow_off, 0, N * 8, h->stream)); CUDA_TRY(h, cudaMemsetAsync(F.Lval_off, 0, N * 8, h->stream));
    CUDA_TRY(h, cudaMemsetAsync(F.Ucol_off, 0, N * 8, h->stream)); CUDA_TRY(h, cudaMemsetAsync(F.Uval_off, 0, N * 8, h->stream));
  }
  int launches = 0;
  unsigned long long ctrl[CTRL_COUNT];
  bilu_status bs = run_phase(h, PH_LOCAL, S, ctrl, ev.e[0], ev.e[1], launches);
  if (bs != BILU_OK) { if (st_out) *st_out = S; return bs; }
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev.e[0], ev.e[1]);
  for (int i = 0; i < 4; ++i) h->cur[i] = ctrl[CTRL_CUR_LIDX + i];
  memcpy(&h->flops_local, &ctrl[CTRL_FLOPS], sizeof(double));
  h->t_local_ms = ms;
  h->ndec_local = (int64_t)ctrl[CTRL_NDEC];
  h->nnear_local = (int64_t)ctrl[CTRL_NEAR];
  h->npert_local = (int64_t)ctrl[CTRL_NPERT];
  h->launches += launches;
  h->dist_local_done = true;
  h->pack_valid = false;
  S.flops = h->flops_local;
  S.t_factor_ms = ms;
  S.n_decisions = h->ndec_local;
  S.n_near = h->nnear_local;
  S.n_kernel_launches = launches;
  if (st_out) *st_out = S;
  return BILU_OK;
}

static int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

extern "C" bilu_status bilu_interface_pack(bilu_ctx *h, void *dst, int64_t capacity, int64_t *nbytes) {
  if (!h || !nbytes) { set_err(h, "bilu_interface_pack: null argument"); return BILU_ERR_ARG; }
  if (!h->dist_local_done) { set_err(h, "bilu_interface_pack: bilu_factor_local has not run"); return BILU_ERR_STATE; }
  cudaSetDevice(h->opt.device);
  DevFactor &F = h->F;
  if (!h->pack_valid) {
    const int nown = (int)h->own_list.size();
    std::vector<uint8_t> flag(std::max(nown, 1));
    std::vector<int32_t> Lm(h->N), Uc(h->N);
    CUDA_TRY(h, bilu_launch_interface_flags(F, h->d_own_list, nown, h->d_sep_mask, h->d_flag, h->stream));
    if (nown) CUDA_TRY(h, cudaMemcpyAsync(flag.data(), h->d_flag, nown, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaMemcpyAsync(Lm.data(), F.Lm, h->N * 4, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaMemcpyAsync(Uc.data(), F.Uc, h->N * 4, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    h->launches += 1;
    h->own_ifc.clear();
    for (int x = 0; x < nown; ++x) if (flag[x]) h->own_ifc.push_back(h->own_list[x]);
    const int cnt = (int)h->own_ifc.size();
    h->pack_tab.assign(cnt, PackEntry{});
    int64_t off = align_up((PACK_HEADER * 8) + (int64_t)cnt * (int64_t)sizeof(PackEntry), 16);
    for (int x = 0; x < cnt; ++x) {
      const int J = h->own_ifc[x];
      PackEntry &e = h->pack_tab[x];
      e.J = J; e.b = h->bstart[J + 1] - h->bstart[J]; e.Lm = Lm[J]; e.Uc = Uc[J];
      e.offLi = off; off = align_up(off + e.Lm * 4, 16);
      e.offUi = off; off = align_up(off + e.Uc * 4, 16);
      e.offLv = off; off = align_up(off + e.Lm * e.b * 8, 16);
      e.offUv = off; off = align_up(off + e.Uc * e.b * 8, 16);
    }
    h->pack_bytes = off;
    h->pack_valid = true;
  }
  *nbytes = h->pack_bytes;
  if (!dst || capacity < h->pack_bytes) return BILU_OK;   // size query
  const int cnt = (int)h->pack_tab.size();
  unsigned char *buf = (unsigned char *)dst;
  const int64_t hdr[PACK_HEADER] = {PACK_MAGIC, cnt, h->pack_bytes, h->rank};
  CUDA_TRY(h, cudaMemcpyAsync(buf, hdr, sizeof(hdr), cudaMemcpyHostToDevice, h->stream));
  if (cnt) CUDA_TRY(h, cudaMemcpyAsync(buf + PACK_HEADER * 8, h->pack_tab.data(), cnt * sizeof(PackEntry), cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, bilu_launch_pack(F, (const PackEntry *)(buf + PACK_HEADER * 8), cnt, buf, h->stream));
  h->launches += cnt > 0;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return BILU_OK;
}

extern "C" bilu_status bilu_interface_unpack(bilu_ctx *h, const void *dbuf, int64_t nbytes) {
  if (!h || !dbuf || nbytes < PACK_HEADER * 8) { set_err(h, "bilu_interface_unpack: bad argument"); return BILU_ERR_ARG; }
  if (!h->dist_local_done) { set_err(h, "bilu_interface_unpack: bilu_factor_local has not run"); return BILU_ERR_STATE; }
  cudaSetDevice(h->opt.device);
  DevFactor &F = h->F;
  int64_t hdr[PACK_HEADER];
  CUDA_TRY(h, cudaMemcpy(hdr, dbuf, sizeof(hdr), cudaMemcpyDeviceToHost));
  if (hdr[0] != PACK_MAGIC || hdr[2] != nbytes || hdr[1] < 0) { set_err(h, "bilu_interface_unpack: not a packed interface buffer"); return BILU_ERR_ARG; }
  if (hdr[3] == h->rank) { set_err(h, "bilu_interface_unpack: buffer of this rank"); return BILU_ERR_ARG; }
  const int cnt = (int)hdr[1];
  std::vector<PackEntry> tab(cnt);
  if (cnt) CUDA_TRY(h, cudaMemcpy(tab.data(), (const unsigned char *)dbuf + PACK_HEADER * 8, cnt * sizeof(PackEntry), cudaMemcpyDeviceToHost));
  std::vector<int64_t> base(4 * (size_t)std::max(cnt, 1));
  unsigned long long c[4] = {h->cur[0], h->cur[1], h->cur[2], h->cur[3]};
  for (int x = 0; x < cnt; ++x) {
    const PackEntry &e = tab[x];
    if (e.J < 0 || e.J >= h->N || h->owner[e.J] == h->rank || h->owner[e.J] < 0) {
      set_err(h, "bilu_interface_unpack: block %lld is not a remote subtree block", (long long)e.J);
      return BILU_ERR_ARG;
    }
    base[4 * x] = (int64_t)c[0]; c[0] += ((unsigned long long)e.Lm + 31) & ~31ull;
    base[4 * x + 1] = (int64_t)c[1]; c[1] += ((unsigned long long)(e.Lm * e.b) + 15) & ~15ull;
    base[4 * x + 2] = (int64_t)c[2]; c[2] += ((unsigned long long)e.Uc + 31) & ~31ull;
    base[4 * x + 3] = (int64_t)c[3]; c[3] += ((unsigned long long)(e.Uc * e.b) + 15) & ~15ull;
  }
  bilu_status gs;
  if ((gs = grow_keep(h, F.Lidx, F.cap_Lidx, (int64_t)c[0], (int64_t)h->cur[0])) != BILU_OK) return gs;
  if ((gs = grow_keep(h, F.Lval, F.cap_Lval, (int64_t)c[1], (int64_t)h->cur[1])) != BILU_OK) return gs;
  if ((gs = grow_keep(h, F.Uidx, F.cap_Uidx, (int64_t)c[2], (int64_t)h->cur[2])) != BILU_OK) return gs;
  if ((gs = grow_keep(h, F.Uval, F.cap_Uval, (int64_t)c[3], (int64_t)h->cur[3])) != BILU_OK) return gs;
  h->cap_val = std::max(F.cap_Lval, F.cap_Uval); h->cap_idx = std::max(F.cap_Lidx, F.cap_Uidx);
  if ((int64_t)base.size() > h->base_cap) {
    dfree(h, h->d_base);
    CUDA_TRY(h, dalloc(h, &h->d_base, base.size()));
    h->base_cap = (int64_t)base.size();
  }
  CUDA_TRY(h, cudaMemcpyAsync(h->d_base, base.data(), base.size() * 8, cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, bilu_launch_unpack(F, (const unsigned char *)dbuf, (const PackEntry *)((const unsigned char *)dbuf + PACK_HEADER * 8),
                                 cnt, h->d_base, h->stream));
  h->launches += cnt > 0;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  for (int i = 0; i < 4; ++i) h->cur[i] = c[i];
  for (int x = 0; x < cnt; ++x) h->remote_ifc.push_back((int32_t)tab[x].J);
  return BILU_OK;
}

// phase-B schedule: control block with the arena cursors of phase A + unpacks, empty queue,
// separator lists / pending rebuilt from every interface block
static bilu_status prepare_separators(bilu_ctx *h) {
  DevFactor &F = h->F;
  cudaStream_t st = h->stream;
  const int nsep = (int)h->sep_list.size();
  memset(h->ctrl_init, 0, sizeof(h->ctrl_init));
  for (int i = 0; i < 4; ++i) h->ctrl_init[CS * (CTRL_CUR_LIDX + i)] = h->cur[i];
  h->ctrl_init[CS * CTRL_DONE] = (unsigned long long)(h->N - nsep);
  CUDA_TRY(h, cudaMemcpyAsync(F.ctrl, h->ctrl_init, sizeof(h->ctrl_init), cudaMemcpyHostToDevice, st));
  CUDA_TRY(h, cudaMemsetAsync(F.queue, 0xFF, F.qcap * sizeof(int32_t), st));
  CUDA_TRY(h, cudaMemsetAsync(F.hq, 0xFF, F.hqcap * sizeof(int32_t), st));
  std::vector<int32_t> ifc(h->own_ifc);
  ifc.insert(ifc.end(), h->remote_ifc.begin(), h->remote_ifc.end());
  if ((int64_t)ifc.size() > h->ifc_cap) {
    dfree(h, h->d_ifc);
    CUDA_TRY(h, dalloc(h, &h->d_ifc, std::max<size_t>(ifc.size(), 1)));
    h->ifc_cap = (int64_t)ifc.size();
  }
  if (!ifc.empty()) CUDA_TRY(h, cudaMemcpyAsync(h->d_ifc, ifc.data(), ifc.size() * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(h, bilu_launch_sep_prepare(F, h->d_sep_list, nsep, h->d_static_sep, h->d_ifc, (int)ifc.size(), h->d_sep_mask, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  h->launches += 3;
  return BILU_OK;
}

extern "C" bilu_status bilu_factor_separators(bilu_ctx *h, bilu_factor_stats *st_out) {
  if (!h) { set_err(nullptr, "bilu_factor_separators: null context"); return BILU_ERR_ARG; }
  if (!h->dist_local_done) { set_err(h, "bilu_factor_separators: bilu_factor_local has not run"); return BILU_ERR_STATE; }
  cudaSetDevice(h->opt.device);
  bilu_factor_stats S{};
  S.breakdown_block = -1;
  S.n_blocks_init = h->N;
  S.zone_blocks = h->F.nzb;
  S.zone_unknowns = h->F.nzb > 0 ? (int32_t)h->zone_unknowns : 0;
  Events ev;
  for (auto &x : ev.e) CUDA_TRY(h, cudaEventCreate(&x));
  int launches = 0;
  unsigned long long ctrl[CTRL_COUNT];
  bilu_status bs = run_phase(h, PH_SEP, S, ctrl, ev.e[0], ev.e[1], launches);
  if (bs != BILU_OK) { if (st_out) *st_out = S; return bs; }
  S.n_decisions = h->ndec_local;
  S.n_near = h->nnear_local;
  S.n_perturbed = h->npert_local;
  S.t_factor_ms = h->t_local_ms;
  bs = finish_factor(h, S, ctrl, ev.e[0], ev.e[1], ev.e[2], launches, nullptr);
  if (bs != BILU_OK) return bs;
  S = h->last;
  S.flops += h->flops_local;
  h->last = S;
  h->dist_local_done = false;
  if (st_out) *st_out = S;
  return BILU_OK;
}

// ------------------------------------------------------------ GMRES
// Restarted, right-preconditioned GMRES(m) on the device (readings
// R16: x0 = 0, modified Gram-Schmidt, Givens rotations, inner steps counted, the true
// residual checked at the end of every cycle).  Vectors live in device memory; the
// Hessenberg column of each step (m+2 doubles) is the only host round trip.
extern "C" bilu_status bilu_gmres(bilu_ctx *h, const double *b, double *x, int32_t m, double tol, int32_t max_restarts,
                                  bilu_solve_stats *st_out) {
  if (!h || !b || !x) { set_err(h, "bilu_gmres: null argument"); return BILU_ERR_ARG; }
  if (m < 1 || m > 1000 || !(tol > 0.0) || max_restarts < 1) { set_err(h, "bilu_gmres: bad restart / tol / max_restarts"); return BILU_ERR_ARG; }
  if (!h->factored) { set_err(h, "bilu_gmres: no factorization"); return BILU_ERR_STATE; }
  if (h->dist) { set_err(h, "bilu_gmres: distributed context"); return BILU_ERR_STATE; }
  cudaSetDevice(h->opt.device);
  cudaStream_t st = h->stream;
  const int n = h->n, sms = h->sms;
  const int64_t ld = n;
  const int64_t need = (int64_t)(2 * m + 2) * n + 8LL * sms + 4 * (int64_t)m + 16;
  if (need > h->kry_cap) {
    dfree(h, h->d_kry);
    CUDA_TRY(h, dalloc(h, &h->d_kry, (size_t)need));
    h->kry_cap = need;
  }
  double *V = h->d_kry, *Z = V + (int64_t)(m + 1) * n, *r = Z + (int64_t)m * n;
  double *part = r + n, *dH = part + 8 * sms, *dtmp = dH + (m + 2), *dY = dtmp + 4;
  int lpr = 1;
  {
    const double avg = (double)h->nnz / std::max(1, n);
    while (lpr < 32 && lpr < avg / 2) lpr <<= 1;
  }
  bilu_solve_stats S{};
  cudaEvent_t e0, e1;
  CUDA_TRY(h, cudaEventCreate(&e0)); CUDA_TRY(h, cudaEventCreate(&e1));
  CUDA_TRY(h, cudaEventRecord(e0, st));
  int64_t launches = 0;
  const int64_t l0 = h->launches;
  double hh[4];
  CUDA_TRY(h, cudaMemsetAsync(x, 0, (size_t)n * 8, st));
  CUDA_TRY(h, bilu_launch_dot(n, b, b, part, dtmp, 1, sms, st)); launches += 2;
  CUDA_TRY(h, cudaMemcpyAsync(hh, dtmp, 2 * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  const double bnorm = hh[1];
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m), col(m + 2);
  int its = 0;
  bool conv = bnorm == 0.0;
  double beta = bnorm;
  if (!conv) CUDA_TRY(h, cudaMemcpyAsync(r, b, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
  for (int cycle = 0; cycle < max_restarts && !conv; ++cycle) {
    if (beta / bnorm <= tol) { conv = true; break; }
    S.restarts = cycle + 1;
    // V0 = r / beta (beta on the device: dtmp[1])
    CUDA_TRY(h, bilu_launch_scale_dev(n, dtmp + 1, r, V, sms, st)); launches += 1;
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int k_used = 0;
    for (int k = 0; k < m; ++k) {
      double *vk = V + (int64_t)k * ld, *zk = Z + (int64_t)k * ld, *w = V + (int64_t)(k + 1) * ld;
      bilu_status as = bilu_apply(h, vk, zk, st);
      if (as != BILU_OK) return as;
      CUDA_TRY(h, bilu_launch_spmv(n, h->d_rp, h->d_ci, h->d_val_orig, zk, w, lpr, sms, st)); launches += 1;
      for (int i = 0; i <= k; ++i) {            // modified Gram-Schmidt, coefficients stay on the device
        CUDA_TRY(h, bilu_launch_dot(n, w, V + (int64_t)i * ld, part, dH + i, 0, sms, st));
        CUDA_TRY(h, bilu_launch_axpy_dev(n, dH + i, -1.0, V + (int64_t)i * ld, w, sms, st));
        launches += 3;
      }
      CUDA_TRY(h, bilu_launch_dot(n, w, w, part, dtmp, 1, sms, st)); launches += 2;
      CUDA_TRY(h, cudaMemcpyAsync(col.data(), dH, (size_t)(k + 1) * 8, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(h, cudaMemcpyAsync(hh, dtmp, 2 * 8, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(h, cudaStreamSynchronize(st));
      for (int i = 0; i <= k; ++i) H[(size_t)i * m + k] = col[i];
      const double hnext = hh[1];
      H[(size_t)(k + 1) * m + k] = hnext;
      for (int i = 0; i < k; ++i) {             // previous rotations
        const double t = cs[i] * H[(size_t)i * m + k] + sn[i] * H[(size_t)(i + 1) * m + k];
        H[(size_t)(i + 1) * m + k] = -sn[i] * H[(size_t)i * m + k] + cs[i] * H[(size_t)(i + 1) * m + k];
        H[(size_t)i * m + k] = t;
      }
      const double den = std::hypot(H[(size_t)k * m + k], H[(size_t)(k + 1) * m + k]);
      cs[k] = den != 0.0 ? H[(size_t)k * m + k] / den : 1.0;
      sn[k] = den != 0.0 ? H[(size_t)(k + 1) * m + k] / den : 0.0;
      H[(size_t)k * m + k] = den;
      H[(size_t)(k + 1) * m + k] = 0.0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      its += 1;
      k_used = k + 1;
      if (std::fabs(g[k + 1]) / bnorm <= tol || hnext == 0.0) break;
      CUDA_TRY(h, bilu_launch_scale_dev(n, dtmp + 1, w, w, sms, st)); launches += 1;   // V[k+1] = w / hnext
    }
    for (int i = k_used - 1; i >= 0; --i) {     // back substitution
      double acc = g[i];
      for (int j = i + 1; j < k_used; ++j) acc -= H[(size_t)i * m + j] * y[j];
      y[i] = acc / H[(size_t)i * m + i];
    }
    CUDA_TRY(h, cudaMemcpyAsync(dY, y.data(), (size_t)k_used * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(h, bilu_launch_update(n, k_used, Z, ld, dY, x, sms, st));
    CUDA_TRY(h, bilu_launch_spmv(n, h->d_rp, h->d_ci, h->d_val_orig, x, r, lpr, sms, st));
    CUDA_TRY(h, bilu_launch_residual(n, b, r, sms, st));
    CUDA_TRY(h, bilu_launch_dot(n, r, r, part, dtmp, 1, sms, st)); launches += 5;
    CUDA_TRY(h, cudaMemcpyAsync(hh, dtmp, 2 * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    beta = hh[1];
    if (beta / bnorm <= tol) conv = true;
  }
  CUDA_TRY(h, cudaEventRecord(e1, st));
  CUDA_TRY(h, cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  h->launches += launches;
  S.iterations = its;
  S.converged = conv ? 1 : 0;
  S.rel_residual = bnorm > 0.0 ? beta / bnorm : 0.0;
  S.t_solve_ms = ms;
  S.n_kernel_launches = launches + (h->launches - l0 - launches);
  if (st_out) *st_out = S;
  return BILU_OK;
}

// ------------------------------------------------------------ export
extern "C" bilu_status bilu_export(bilu_ctx *h, bilu_factor_view *v) {
  if (!h || !v) { set_err(h, "bilu_export: null argument"); return BILU_ERR_ARG; }
  memset(v, 0, sizeof(*v));
  if (!h->factored) { set_err(h, "bilu_export: no factorization"); return BILU_ERR_STATE; }
  cudaSetDevice(h->opt.device);
  const FinalFactor &fin = h->fin;
  const int nF = fin.nF;
  cudaStream_t st = h->stream;
  std::vector<int32_t> fb(nF + 1), Lm(nF), Uc(nF), Li(fin.usedLi), Ui(fin.usedUi);
  std::vector<int64_t> Lro(nF), Lvo(nF), Uco(nF), Uvo(nF), Doff(nF + 1);
  std::vector<double> Lv(fin.usedLv), Uv(fin.usedUv), Dv(fin.nnzD);
  CUDA_TRY(h, cudaMemcpyAsync(fb.data(), fin.bstart, (nF + 1) * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(Lm.data(), fin.Lm, nF * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(Uc.data(), fin.Uc, nF * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(Lro.data(), fin.Lrow_off, nF * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(Lvo.data(), fin.Lval_off, nF * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(Uco.data(), fin.Ucol_off, nF * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(Uvo.data(), fin.Uval_off, nF * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(Doff.data(), fin.D_off, (nF + 1) * 8, cudaMemcpyDeviceToHost, st));
  if (fin.usedLi) CUDA_TRY(h, cudaMemcpyAsync(Li.data(), h->F.Lidx, fin.usedLi * 4, cudaMemcpyDeviceToHost, st));
  if (fin.usedUi) CUDA_TRY(h, cudaMemcpyAsync(Ui.data(), h->F.Uidx, fin.usedUi * 4, cudaMemcpyDeviceToHost, st));
  if (fin.usedLv) CUDA_TRY(h, cudaMemcpyAsync(Lv.data(), h->F.Lval, fin.usedLv * 8, cudaMemcpyDeviceToHost, st));
  if (fin.usedUv) CUDA_TRY(h, cudaMemcpyAsync(Uv.data(), h->F.Uval, fin.usedUv * 8, cudaMemcpyDeviceToHost, st));
  if (fin.nnzD) CUDA_TRY(h, cudaMemcpyAsync(Dv.data(), fin.D, fin.nnzD * 8, cudaMemcpyDeviceToHost, st));
  int64_t nnear = std::min<int64_t>(h->last.n_near, h->near_cap);
  std::vector<int32_t> ni(4 * nnear);
  std::vector<double> nm(nnear);
  if (nnear) {
    CUDA_TRY(h, cudaMemcpyAsync(ni.data(), h->F.near_i, 4 * nnear * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaMemcpyAsync(nm.data(), h->F.near_m, nnear * 8, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(h, cudaStreamSynchronize(st));
  v->n = h->n; v->n_blocks = nF;
  v->bstart = (int32_t *)malloc(sizeof(int32_t) * (nF + 1));
  v->Lp = (int64_t *)malloc(sizeof(int64_t) * (nF + 1));
  v->Lvp = (int64_t *)malloc(sizeof(int64_t) * (nF + 1));
  v->Up = (int64_t *)malloc(sizeof(int64_t) * (nF + 1));
  v->Uvp = (int64_t *)malloc(sizeof(int64_t) * (nF + 1));
  v->Dp = (int64_t *)malloc(sizeof(int64_t) * (nF + 1));
  v->Lp[0] = v->Lvp[0] = v->Up[0] = v->Uvp[0] = v->Dp[0] = 0;
  for (int F = 0; F < nF; ++F) {
    int64_t b = fb[F + 1] - fb[F];
    v->bstart[F] = fb[F];
    v->Lp[F + 1] = v->Lp[F] + Lm[F];
    v->Lvp[F + 1] = v->Lvp[F] + Lm[F] * b;
    v->Up[F + 1] = v->Up[F] + Uc[F];
    v->Uvp[F + 1] = v->Uvp[F] + Uc[F] * b;
    v->Dp[F + 1] = v->Dp[F] + b * b;
  }
  v->bstart[nF] = fb[nF];
  v->Li = (int32_t *)malloc(sizeof(int32_t) * std::max<int64_t>(v->Lp[nF], 1));
  v->Lv = (double *)malloc(sizeof(double) * std::max<int64_t>(v->Lvp[nF], 1));
  v->Ui = (int32_t *)malloc(sizeof(int32_t) * std::max<int64_t>(v->Up[nF], 1));
  v->Uv = (double *)malloc(sizeof(double) * std::max<int64_t>(v->Uvp[nF], 1));
  v->Dv = (double *)malloc(sizeof(double) * std::max<int64_t>(v->Dp[nF], 1));
  for (int F = 0; F < nF; ++F) {
    int64_t b = fb[F + 1] - fb[F];
    if (Lm[F]) {
      memcpy(v->Li + v->Lp[F], Li.data() + Lro[F], sizeof(int32_t) * Lm[F]);
      memcpy(v->Lv + v->Lvp[F], Lv.data() + Lvo[F], sizeof(double) * Lm[F] * b);
    }
    if (Uc[F]) {
      memcpy(v->Ui + v->Up[F], Ui.data() + Uco[F], sizeof(int32_t) * Uc[F]);
      memcpy(v->Uv + v->Uvp[F], Uv.data() + Uvo[F], sizeof(double) * Uc[F] * b);
    }
    memcpy(v->Dv + v->Dp[F], Dv.data() + Doff[F], sizeof(double) * b * b);
  }
  v->n_near = nnear;
  v->near_blk = (int32_t *)malloc(sizeof(int32_t) * std::max<int64_t>(nnear, 1));
  v->near_side = (int32_t *)malloc(sizeof(int32_t) * std::max<int64_t>(nnear, 1));
  v->near_idx = (int32_t *)malloc(sizeof(int32_t) * std::max<int64_t>(nnear, 1));
  v->near_keep = (int32_t *)malloc(sizeof(int32_t) * std::max<int64_t>(nnear, 1));
  v->near_margin = (double *)malloc(sizeof(double) * std::max<int64_t>(nnear, 1));
  for (int64_t i = 0; i < nnear; ++i) {
    v->near_blk[i] = ni[4 * i]; v->near_side[i] = ni[4 * i + 1];
    v->near_idx[i] = ni[4 * i + 2]; v->near_keep[i] = ni[4 * i + 3];
    v->near_margin[i] = nm[i];
  }
  return BILU_OK;
}

extern "C" void bilu_factor_view_free(bilu_factor_view *v) {
  if (!v) return;
  free(v->bstart); free(v->Lp); free(v->Li); free(v->Lvp); free(v->Lv);
  free(v->Up); free(v->Ui); free(v->Uvp); free(v->Uv); free(v->Dp); free(v->Dv);
  free(v->near_blk); free(v->near_side); free(v->near_idx); free(v->near_keep); free(v->near_margin);
  memset(v, 0, sizeof(*v));
}

// ------------------------------------------------------------ apply
// Dependency lists of the two sweeps, built once per factorization from the
// final index lists (host side, like the schedule tables of bilu_analyze).
static bilu_status build_apply(bilu_ctx *h) {
  const FinalFactor &fin = h->fin;
  const int nF = fin.nF, n = h->n;
  cudaStream_t st = h->stream;
  std::vector<int32_t> fb(nF + 1), Lm(nF), Uc(nF), Li(fin.usedLi), Ui(fin.usedUi);
  std::vector<int64_t> Lro(nF), Uco(nF);
  CUDA_TRY(h, cudaMemcpyAsync(fb.data(), fin.bstart, (nF + 1) * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(Lm.data(), fin.Lm, nF * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(Uc.data(), fin.Uc, nF * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(Lro.data(), fin.Lrow_off, nF * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpyAsync(Uco.data(), fin.Ucol_off, nF * 8, cudaMemcpyDeviceToHost, st));
  if (fin.usedLi) CUDA_TRY(h, cudaMemcpyAsync(Li.data(), h->F.Lidx, fin.usedLi * 4, cudaMemcpyDeviceToHost, st));
  if (fin.usedUi) CUDA_TRY(h, cudaMemcpyAsync(Ui.data(), h->F.Uidx, fin.usedUi * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  std::vector<int32_t> fbo(n);
  for (int F = 0; F < nF; ++F) for (int i = fb[F]; i < fb[F + 1]; ++i) fbo[i] = F;
  // distributed: role of every final block (1 own subtree, 2 separator, 0 another rank's);
  // only own and separator blocks take part in this rank's sweeps
  std::vector<uint8_t> role(nF, 1);
  if (h->dist) {
    for (int F = 0; F < nF; ++F) {
      const int K = (int)(std::upper_bound(h->bstart.begin(), h->bstart.end(), fb[F]) - h->bstart.begin()) - 1;
      const int o = h->owner[K];
      role[F] = o == h->rank ? 1 : (o < 0 ? 2 : 0);
    }
  }
  // forward: target T pulls (J, r0, r1) for every J with L rows in T
  std::vector<int32_t> fl_cnt(nF + 1, 0), fs_ptr(nF + 1, 0), bs_cnt(nF + 1, 0), cnt_b(nF, 0);
  for (int J = 0; J < nF; ++J) {
    if (!role[J]) continue;
    const int32_t *r = Li.data() + Lro[J];
    for (int p = 0; p < Lm[J]; ++p) if (p == 0 || fbo[r[p]] != fbo[r[p - 1]]) { fl_cnt[fbo[r[p]] + 1]++; fs_ptr[J + 1]++; }
    const int32_t *c = Ui.data() + Uco[J];
    for (int q = 0; q < Uc[J]; ++q) if (q == 0 || fbo[c[q]] != fbo[c[q - 1]]) { bs_cnt[fbo[c[q]] + 1]++; cnt_b[J]++; }
  }
  std::vector<int32_t> fl_ptr(nF + 1, 0), bs_ptr(nF + 1, 0), cnt_f(nF, 0);
  for (int F = 0; F < nF; ++F) {
    fl_ptr[F + 1] = fl_ptr[F] + fl_cnt[F + 1];
    bs_ptr[F + 1] = bs_ptr[F] + bs_cnt[F + 1];
    fs_ptr[F + 1] += fs_ptr[F];
    cnt_f[F] = fl_cnt[F + 1];
  }
  std::vector<int32_t> fl_rec(3 * (size_t)fl_ptr[nF] + 3), fs(fs_ptr[nF] + 1), bs(bs_ptr[nF] + 1);
  std::vector<int32_t> flf(fl_ptr.begin(), fl_ptr.end() - 1), bsf(bs_ptr.begin(), bs_ptr.end() - 1);
  for (int J = 0; J < nF; ++J) {
    if (!role[J]) continue;
    const int32_t *r = Li.data() + Lro[J];
    int xs = fs_ptr[J];
    for (int p = 0; p < Lm[J];) {
      int T = fbo[r[p]], p1 = p;
      while (p1 < Lm[J] && fbo[r[p1]] == T) ++p1;
      int x = flf[T]++;
      fl_rec[3 * x] = J; fl_rec[3 * x + 1] = p; fl_rec[3 * x + 2] = p1;
      fs[xs++] = T;
      p = p1;
    }
    const int32_t *c = Ui.data() + Uco[J];
    for (int q = 0; q < Uc[J];) {
      int T = fbo[c[q]], q1 = q;
      while (q1 < Uc[J] && fbo[c[q1]] == T) ++q1;
      bs[bsf[T]++] = J;
      q = q1;
    }
  }
  std::vector<int32_t> qf, qb, qf2, cnt_f2;
  int nt_f = nF, nt_b = nF, nt_f2 = 0;
  if (h->dist) {
    // forward phase 1: own blocks (their contributors are own blocks); phase 2: separators,
    // counting separator contributors only; backward: own + separators.  Blocks outside a
    // phase never reach zero.
    const int32_t BIG = 1 << 30;
    cnt_f2.assign(nF, BIG);
    for (int F = 0; F < nF; ++F) {
      if (role[F] != 2) continue;
      int c = 0;
      for (int x = fl_ptr[F]; x < fl_ptr[F + 1]; ++x) c += role[fl_rec[3 * x]] == 2;
      cnt_f2[F] = c;
      if (c == 0) qf2.push_back(F);
    }
    nt_f = nt_f2 = nt_b = 0;
    for (int F = 0; F < nF; ++F) {
      nt_f += role[F] == 1; nt_f2 += role[F] == 2; nt_b += role[F] != 0;
      if (role[F] != 1) cnt_f[F] += BIG;
      if (role[F] == 0) cnt_b[F] += BIG;
    }
    std::vector<int32_t> seprows;
    std::vector<uint8_t> rmask(n, 0);
    for (int F = 0; F < nF; ++F)
      for (int i = fb[F]; i < fb[F + 1]; ++i) {
        rmask[i] = role[F];
        if (role[F] == 2) seprows.push_back(i);
      }
    dfree(h, h->d_seprows); dfree(h, h->d_xsep); dfree(h, h->d_rowmask);
    h->nsep_rows = (int32_t)seprows.size();
    CUDA_TRY(h, dalloc(h, &h->d_seprows, std::max<size_t>(seprows.size(), 1)));
    CUDA_TRY(h, dalloc(h, &h->d_xsep, std::max<size_t>(seprows.size(), 1)));
    CUDA_TRY(h, dalloc(h, &h->d_rowmask, (size_t)n));
    if (!seprows.empty()) CUDA_TRY(h, cudaMemcpy(h->d_seprows, seprows.data(), seprows.size() * 4, cudaMemcpyHostToDevice));
    CUDA_TRY(h, cudaMemcpy(h->d_rowmask, rmask.data(), (size_t)n, cudaMemcpyHostToDevice));
  }
  for (int F = 0; F < nF; ++F) if (cnt_f[F] == 0) qf.push_back(F);
  for (int F = nF - 1; F >= 0; --F) if (cnt_b[F] == 0) qb.push_back(F);
  h->nt_f0 = nt_f; h->nt_b0 = nt_b; h->nt_f2 = nt_f2;
  dfree(h, h->d_cnt_f2); dfree(h, h->d_q_f2);
  h->nq_f2 = (int32_t)qf2.size();
  h->nq_f2_ull = (unsigned long long)h->nq_f2;
  dfree(h, h->d_fl_ptr); dfree(h, h->d_fl_rec); dfree(h, h->d_fs_ptr); dfree(h, h->d_fs);
  dfree(h, h->d_bs_ptr); dfree(h, h->d_bs); dfree(h, h->d_cnt_f0); dfree(h, h->d_cnt_b0);
  dfree(h, h->d_q_f0); dfree(h, h->d_q_b0);
  auto up = [&](int32_t *&d, const std::vector<int32_t> &v) -> bilu_status {
    CUDA_TRY(h, dalloc(h, &d, std::max<size_t>(v.size(), 1)));
    if (!v.empty()) CUDA_TRY(h, cudaMemcpy(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
    return BILU_OK;
  };
  bilu_status bs_;
  if ((bs_ = up(h->d_fl_ptr, fl_ptr)) || (bs_ = up(h->d_fl_rec, fl_rec)) || (bs_ = up(h->d_fs_ptr, fs_ptr)) ||
      (bs_ = up(h->d_fs, fs)) || (bs_ = up(h->d_bs_ptr, bs_ptr)) || (bs_ = up(h->d_bs, bs)) ||
      (bs_ = up(h->d_cnt_f0, cnt_f)) || (bs_ = up(h->d_cnt_b0, cnt_b)) || (bs_ = up(h->d_q_f0, qf)) ||
      (bs_ = up(h->d_q_b0, qb)) || (bs_ = up(h->d_cnt_f2, cnt_f2)) || (bs_ = up(h->d_q_f2, qf2)))
    return bs_;
  h->nq_f0 = (int32_t)qf.size(); h->nq_b0 = (int32_t)qb.size();
  h->nq_f0_ull = (unsigned long long)h->nq_f0; h->nq_b0_ull = (unsigned long long)h->nq_b0;
  ApplyArgs &A = h->AA;
  if (!A.cnt) {
    CUDA_TRY(h, dalloc(h, &A.cnt, (size_t)h->N));
    CUDA_TRY(h, dalloc(h, &A.queue, (size_t)h->N));
    CUDA_TRY(h, dalloc(h, &A.ctrl, 4));
    CUDA_TRY(h, dalloc(h, &h->d_w, (size_t)n));
    CUDA_TRY(h, dalloc(h, &h->d_y, (size_t)n));
  }
  A.n = n; A.nF = nF;
  A.fbstart = fin.bstart;
  A.Lrow_off = fin.Lrow_off; A.Lval_off = fin.Lval_off; A.Ucol_off = fin.Ucol_off; A.Uval_off = fin.Uval_off;
  A.D_off = fin.D_off; A.Lm = fin.Lm; A.Uc = fin.Uc;
  A.Lidx = h->F.Lidx; A.Uidx = h->F.Uidx; A.Lval = h->F.Lval; A.Uval = h->F.Uval; A.D = fin.D;
  A.fl_ptr = h->d_fl_ptr; A.fl_rec = h->d_fl_rec; A.fs_ptr = h->d_fs_ptr; A.fs = h->d_fs;
  A.bs_ptr = h->d_bs_ptr; A.bs = h->d_bs;
  A.w = h->d_w; A.y = h->d_y;
  h->apply_ready = true;
  return BILU_OK;
}

// one dataflow sweep over ntarget blocks, starting from the counters cnt0 and ready queue q0
static bilu_status run_sweep(bilu_ctx *h, const int32_t *cnt0, const int32_t *q0, int nq,
                             const unsigned long long *nq_ull, int ntarget, int backward, cudaStream_t st) {
  ApplyArgs &A = h->AA;
  const int nF = h->fin.nF;
  if (ntarget <= 0) return BILU_OK;
  A.ntarget = ntarget;
  const int grid = std::max(1, std::min((ntarget + 15) / 16, h->sms * 2));   // 16 warp-workers per CTA
  CUDA_TRY(h, cudaMemcpyAsync(A.cnt, cnt0, nF * 4, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(h, cudaMemsetAsync(A.queue, 0xFF, nF * 4, st));
  if (nq) CUDA_TRY(h, cudaMemcpyAsync(A.queue, q0, nq * 4, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(h, cudaMemsetAsync(A.ctrl, 0, 4 * sizeof(unsigned long long), st));
  CUDA_TRY(h, cudaMemcpyAsync(A.ctrl, nq_ull, sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
  const char *prof_path = tune_env("BILU_APPLY_PROF");   // diagnostics: per-block times to <path>.<sweep>
  unsigned long long *d_prof = nullptr;
  if (prof_path) {
    CUDA_TRY(h, cudaMalloc(&d_prof, sizeof(unsigned long long) * 3 * nF));
    CUDA_TRY(h, cudaMemsetAsync(d_prof, 0, sizeof(unsigned long long) * 3 * nF, st));
  }
  A.prof = d_prof;
  CUDA_TRY(h, bilu_launch_apply(A, grid, backward, st));
  A.prof = nullptr;
  h->launches += 1;
  if (prof_path) {
    std::vector<unsigned long long> t(3 * (size_t)nF);
    CUDA_TRY(h, cudaMemcpyAsync(t.data(), d_prof, t.size() * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
    cudaFree(d_prof);
    std::string fn = std::string(prof_path) + (backward ? ".bwd" : ".fwd");
    if (FILE *fp = fopen(fn.c_str(), "wb")) { fwrite(t.data(), 8, t.size(), fp); fclose(fp); }
  }
  return BILU_OK;
}

extern "C" bilu_status bilu_apply(bilu_ctx *h, const double *x, double *y, void *stream) {
  if (h && h->dist) {
    set_err(h, "bilu_apply: distributed factors are spread over the ranks (use bilu_apply_dist_begin/_end)");
    return BILU_ERR_STATE;
  }
  if (!h || !x || !y) { set_err(h, "bilu_apply: null argument"); return BILU_ERR_ARG; }
  if (x == y) { set_err(h, "bilu_apply: x and y may not alias"); return BILU_ERR_ARG; }
  if (!h->factored) { set_err(h, "bilu_apply: no factorization"); return BILU_ERR_STATE; }
  cudaSetDevice(h->opt.device);
  if (!h->apply_ready) { bilu_status s = build_apply(h); if (s != BILU_OK) return s; }
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  CUDA_TRY(h, bilu_launch_permute(h->d_w, x, h->d_perm, h->n, 0, st));
  const int only = tune_env("BILU_APPLY_ONLY") ? atoi(tune_env("BILU_APPLY_ONLY")) : -1;   // diagnostics
  bilu_status s;
  if (only != 1 && (s = run_sweep(h, h->d_cnt_f0, h->d_q_f0, h->nq_f0, &h->nq_f0_ull, h->nt_f0, 0, st)) != BILU_OK)
    return s;
  if (only != 0 && (s = run_sweep(h, h->d_cnt_b0, h->d_q_b0, h->nq_b0, &h->nq_b0_ull, h->nt_b0, 1, st)) != BILU_OK)
    return s;
  CUDA_TRY(h, bilu_launch_permute(y, h->d_y, h->d_perm, h->n, 1, st));
  h->launches += 2;
  return BILU_OK;
}

// ---- distributed apply: phase 1 (own subtrees) / exchange by the caller / phases 2-3
static bilu_status dist_apply_check(bilu_ctx *h, const char *fn) {
  if (!h) { set_err(nullptr, "%s: null context", fn); return BILU_ERR_ARG; }
  if (!h->dist) { set_err(h, "%s: not a distributed context (use bilu_apply)", fn); return BILU_ERR_STATE; }
  if (!h->factored) { set_err(h, "%s: bilu_factor_separators has not run", fn); return BILU_ERR_STATE; }
  cudaSetDevice(h->opt.device);
  if (!h->apply_ready) { bilu_status s = build_apply(h); if (s != BILU_OK) return s; }
  return BILU_OK;
}

extern "C" bilu_status bilu_dist_separator_rows(bilu_ctx *h, int64_t *m) {
  bilu_status s = dist_apply_check(h, "bilu_dist_separator_rows");
  if (s != BILU_OK) return s;
  if (!m) { set_err(h, "bilu_dist_separator_rows: null argument"); return BILU_ERR_ARG; }
  *m = h->nsep_rows;
  return BILU_OK;
}

extern "C" bilu_status bilu_apply_dist_begin(bilu_ctx *h, const double *x, double *contrib, void *stream) {
  bilu_status s = dist_apply_check(h, "bilu_apply_dist_begin");
  if (s != BILU_OK) return s;
  if (!x || (!contrib && h->nsep_rows > 0)) { set_err(h, "bilu_apply_dist_begin: null argument"); return BILU_ERR_ARG; }
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  CUDA_TRY(h, bilu_launch_permute(h->d_w, x, h->d_perm, h->n, 0, st));
  CUDA_TRY(h, bilu_launch_sep_gather(h->nsep_rows, h->d_seprows, h->d_w, h->d_xsep, st));
  if ((s = run_sweep(h, h->d_cnt_f0, h->d_q_f0, h->nq_f0, &h->nq_f0_ull, h->nt_f0, 0, st)) != BILU_OK) return s;
  CUDA_TRY(h, bilu_launch_sep_contrib(h->nsep_rows, h->d_seprows, h->d_w, h->d_xsep, contrib, st));
  h->launches += 3;
  h->dist_apply_begun = true;
  return BILU_OK;
}

extern "C" bilu_status bilu_apply_dist_end(bilu_ctx *h, const double *contrib_sum, double *y, int32_t write_separators,
                                           void *stream) {
  bilu_status s = dist_apply_check(h, "bilu_apply_dist_end");
  if (s != BILU_OK) return s;
  if (!y || (!contrib_sum && h->nsep_rows > 0)) { set_err(h, "bilu_apply_dist_end: null argument"); return BILU_ERR_ARG; }
  if (!h->dist_apply_begun) { set_err(h, "bilu_apply_dist_end: bilu_apply_dist_begin has not run"); return BILU_ERR_STATE; }
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  CUDA_TRY(h, bilu_launch_sep_set(h->nsep_rows, h->d_seprows, h->d_xsep, contrib_sum, h->d_w, st));
  if ((s = run_sweep(h, h->d_cnt_f2, h->d_q_f2, h->nq_f2, &h->nq_f2_ull, h->nt_f2, 0, st)) != BILU_OK) return s;
  if ((s = run_sweep(h, h->d_cnt_b0, h->d_q_b0, h->nq_b0, &h->nq_b0_ull, h->nt_b0, 1, st)) != BILU_OK) return s;
  CUDA_TRY(h, bilu_launch_permute_out_masked(h->n, h->d_perm, h->d_rowmask, write_separators, h->d_y, y, st));
  h->launches += 2;
  h->dist_apply_begun = false;
  return BILU_OK;
}

// --------------------------------------------------------------- ILU(1,tau) initial blocking
extern "C" bilu_status bilu_ilu1_blocks(int32_t n, const int64_t *row_ptr, const int32_t *col_idx, const double *val,
                                        const int32_t *perm, double tau, int32_t max_size, int32_t device,
                                        void *stream, int32_t *block_sizes, int32_t *n_blocks,
                                        int32_t *n_kernel_launches) {
  if (n_blocks) *n_blocks = 0;
  if (n < 1 || !row_ptr || !col_idx || !val || !block_sizes || !n_blocks) {
    set_err(nullptr, "bilu_ilu1_blocks: null pointer or n < 1");
    return BILU_ERR_ARG;
  }
  if (!(tau >= 0.0) || max_size < 1 || max_size > 128) {
    set_err(nullptr, "bilu_ilu1_blocks: need tau >= 0 and max_size in [1,128] (got %g, %d)", tau, max_size);
    return BILU_ERR_ARG;
  }
  if (n >= (1 << 30)) { set_err(nullptr, "bilu_ilu1_blocks: n must be < 2^30"); return BILU_ERR_ARG; }
  const auto t_host0 = std::chrono::steady_clock::now();
  std::vector<int32_t> pm, ipm;
  bilu_status st = check_csr_perm("bilu_ilu1_blocks", n, row_ptr, col_idx, perm, pm, ipm);
  if (st != BILU_OK) return st;
  const int64_t nnz = row_ptr[n];
  if (cudaSetDevice(device) != cudaSuccess) {
    set_err(nullptr, "bilu_ilu1_blocks: cannot use CUDA device %d", device);
    return BILU_ERR_NOT_BUILT;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaStream_t s = (cudaStream_t)stream;
  int64_t *d_rp = nullptr;
  int32_t *d_ci = nullptr, *d_pm = nullptr, *d_ipm = nullptr;
  double *d_v = nullptr;
  cudaError_t e = cudaMalloc(&d_rp, sizeof(int64_t) * (n + 1));
  if (e == cudaSuccess) e = cudaMalloc(&d_ci, sizeof(int32_t) * (nnz > 0 ? nnz : 1));
  if (e == cudaSuccess) e = cudaMalloc(&d_v, sizeof(double) * (nnz > 0 ? nnz : 1));
  if (e == cudaSuccess && perm) e = cudaMalloc(&d_pm, sizeof(int32_t) * n);
  if (e == cudaSuccess && perm) e = cudaMalloc(&d_ipm, sizeof(int32_t) * n);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_rp, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && nnz > 0) e = cudaMemcpyAsync(d_ci, col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && nnz > 0) e = cudaMemcpyAsync(d_v, val, sizeof(double) * nnz, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && perm) e = cudaMemcpyAsync(d_pm, pm.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && perm) e = cudaMemcpyAsync(d_ipm, ipm.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s);
  int launches = 0;
  cudaStreamSynchronize(s);
  const auto t_dev0 = std::chrono::steady_clock::now();
  if (e == cudaSuccess)
    e = bilu_ilu1_run(n, d_rp, d_ci, d_v, d_pm, d_ipm, tau, max_size, sms, s, block_sizes, n_blocks, &launches);
  cudaStreamSynchronize(s);
  if (tune_env("BILU_VERBOSE")) {
    const auto t_dev1 = std::chrono::steady_clock::now();
    fprintf(stderr, "[bilu] ilu1_blocks: host validate+upload %.2f ms, device permute+estimate %.2f ms (%d launches)\n",
            std::chrono::duration<double, std::milli>(t_dev0 - t_host0).count(),
            std::chrono::duration<double, std::milli>(t_dev1 - t_dev0).count(), launches);
  }
  cudaFree(d_rp); cudaFree(d_ci); cudaFree(d_v); cudaFree(d_pm); cudaFree(d_ipm);
  if (n_kernel_launches) *n_kernel_launches = launches;
  if (e != cudaSuccess) {
    set_err(nullptr, "bilu_ilu1_blocks: %s", cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? BILU_ERR_OOM : BILU_ERR_CUDA;
  }
  return BILU_OK;
}

// --------------------------------------------------------------- cosine-based blocking
extern "C" bilu_status bilu_cosine_blocks(int32_t n, const int64_t *row_ptr, const int32_t *col_idx, double tau,
                                          int32_t max_size, int32_t device, void *stream, int32_t *q,
                                          int32_t *block_sizes, int32_t *n_blocks, int32_t *n_kernel_launches) {
  if (n_blocks) *n_blocks = 0;
  if (n < 1 || !row_ptr || !col_idx || !q || !block_sizes || !n_blocks) {
    set_err(nullptr, "bilu_cosine_blocks: null pointer or n < 1");
    return BILU_ERR_ARG;
  }
  if (!(tau >= 0.0 && tau <= 1.0) || max_size < 1 || max_size > 128) {
    set_err(nullptr, "bilu_cosine_blocks: need tau in [0,1] and max_size in [1,128] (got %g, %d)", tau, max_size);
    return BILU_ERR_ARG;
  }
  if (n >= (1 << 30)) { set_err(nullptr, "bilu_cosine_blocks: n must be < 2^30"); return BILU_ERR_ARG; }
  std::vector<int32_t> pm, ipm;
  bilu_status st = check_csr_perm("bilu_cosine_blocks", n, row_ptr, col_idx, nullptr, pm, ipm);
  if (st != BILU_OK) return st;
  const int64_t nnz = row_ptr[n];
  if (cudaSetDevice(device) != cudaSuccess) {
    set_err(nullptr, "bilu_cosine_blocks: cannot use CUDA device %d", device);
    return BILU_ERR_NOT_BUILT;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaStream_t s = (cudaStream_t)stream;
  int64_t *d_rp = nullptr;
  int32_t *d_ci = nullptr;
  cudaError_t e = cudaMalloc(&d_rp, sizeof(int64_t) * (n + 1));
  if (e == cudaSuccess) e = cudaMalloc(&d_ci, sizeof(int32_t) * (nnz > 0 ? nnz : 1));
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_rp, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && nnz > 0) e = cudaMemcpyAsync(d_ci, col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s);
  int launches = 0, rounds = 0;
  if (e == cudaSuccess) e = bilu_cosine_run(n, d_rp, d_ci, tau, max_size, sms, s, q, block_sizes, n_blocks, &launches, &rounds);
  cudaStreamSynchronize(s);
  cudaFree(d_rp); cudaFree(d_ci);
  if (tune_env("BILU_VERBOSE")) fprintf(stderr, "[bilu] cosine_blocks: %d launches, %d greedy rounds\n", launches, rounds);
  if (n_kernel_launches) *n_kernel_launches = launches;
  if (e != cudaSuccess) {
    set_err(nullptr, "bilu_cosine_blocks: %s", cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? BILU_ERR_OOM : BILU_ERR_CUDA;
  }
  return BILU_OK;
}

// ------------------------------------------------------------ Sec. 3.1 matching + scaling
extern "C" int bilu_mwm_device(int n, const int64_t *rp, const int32_t *ci, const double *val, int32_t *assign,
                               double *dl, double *dr, void *work, cudaStream_t st, int *launches, int *rounds);

extern "C" bilu_status bilu_mwm(int32_t n, const int64_t *row_ptr, const int32_t *col_idx, const double *val,
                                int32_t device, void *stream, int32_t *sigma, double *dl, double *dr,
                                int32_t *n_kernel_launches) {
  if (n < 1 || !row_ptr || !col_idx || !val || !sigma || !dl || !dr) {
    set_err(nullptr, "bilu_mwm: null pointer or n < 1");
    return BILU_ERR_ARG;
  }
  if (n >= (1 << 30)) { set_err(nullptr, "bilu_mwm: n must be < 2^30"); return BILU_ERR_ARG; }
  std::vector<int32_t> pm, ipm;
  bilu_status st = check_csr_perm("bilu_mwm", n, row_ptr, col_idx, nullptr, pm, ipm);
  if (st != BILU_OK) return st;
  const int64_t nnz = row_ptr[n];
  if (cudaSetDevice(device) != cudaSuccess) {
    set_err(nullptr, "bilu_mwm: cannot use CUDA device %d", device);
    return BILU_ERR_NOT_BUILT;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int64_t *d_rp = nullptr;
  int32_t *d_ci = nullptr, *d_as = nullptr;
  double *d_v = nullptr, *d_dl = nullptr, *d_dr = nullptr;
  void *d_work = nullptr;
  const size_t work_bytes = (size_t)n * (4 * 8 + 3 * 4) + 64 + 16 + (size_t)std::max<int64_t>(nnz, 1) * 8;
  cudaError_t e = cudaMalloc(&d_rp, sizeof(int64_t) * (n + 1));
  if (e == cudaSuccess) e = cudaMalloc(&d_ci, sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  if (e == cudaSuccess) e = cudaMalloc(&d_v, sizeof(double) * std::max<int64_t>(nnz, 1));
  if (e == cudaSuccess) e = cudaMalloc(&d_as, sizeof(int32_t) * n);
  if (e == cudaSuccess) e = cudaMalloc(&d_dl, sizeof(double) * n);
  if (e == cudaSuccess) e = cudaMalloc(&d_dr, sizeof(double) * n);
  if (e == cudaSuccess) e = cudaMalloc(&d_work, work_bytes);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_rp, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && nnz > 0) e = cudaMemcpyAsync(d_ci, col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && nnz > 0) e = cudaMemcpyAsync(d_v, val, sizeof(double) * nnz, cudaMemcpyHostToDevice, s);
  int launches = 0, rounds = 0, rc = 0;
  if (e == cudaSuccess) {
    rc = bilu_mwm_device(n, d_rp, d_ci, d_v, d_as, d_dl, d_dr, d_work, s, &launches, &rounds);
    if (rc > 0) e = (cudaError_t)rc;
  }
  if (e == cudaSuccess && rc == 0) {
    e = cudaMemcpyAsync(sigma, d_as, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dl, d_dl, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dr, d_dr, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  if (tune_env("BILU_VERBOSE")) fprintf(stderr, "[bilu] mwm: %d bidding rounds, %d launches\n", rounds, launches);
  cudaFree(d_rp); cudaFree(d_ci); cudaFree(d_v); cudaFree(d_as); cudaFree(d_dl); cudaFree(d_dr); cudaFree(d_work);
  if (n_kernel_launches) *n_kernel_launches = launches;
  if (e != cudaSuccess) {
    set_err(nullptr, "bilu_mwm: %s", cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? BILU_ERR_OOM : BILU_ERR_CUDA;
  }
  if (rc == -2) {
    set_err(nullptr, "bilu_mwm: the pattern has no perfect matching (structurally singular)");
    return BILU_ERR_ARG;
  }
  return BILU_OK;
}
