// bilu_merge.cu -- progressive aggregation (Sec. 3.5) as a
// post-pass over the finished (unmerged) factors.
//
// Merging k-1 into k leaves the operator L·P·U unchanged (identity displayed at
// PAPER.md:1348-1387), so the values of every later block are the same whether
// the merge happens during or after the factorization;
// the decisions only depend on index sets ("checking the union of nonzero index
// sets ignoring any cancellations").  The sequential scan of
// the paper is made parallel in three steps:
//   merge_test_kernel   the test of Sec. 3.5 for every (aggregate start a = k-d,
//                       block k) pair that max_block allows -> bitmask T[k] and
//                       the union sizes u(d), v(d)
//   merge_scan_kernel   the paper's left-to-right scan as a composition of
//                       per-chunk state maps (state = distance to the run start)
//   merge_offsets_kernel descriptors and arena offsets of the final blocks
//   merge_arith_kernel  the merged factors of each run a..k, formed with block
//                       triangular solves over the member blocks:
//     D^ = U_aa^{-1} D_agg L_aa^{-1},  L^ = L_{>,agg} L_aa^{-1},  Ũ^ = L_aa Ũ_{agg,>}
//   (the paper's pairwise update applied k-a times; DESIGN.md derives it).
#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>

#include "bilu_internal.h"
#include "dgemm_cta.cuh"

namespace bilu {

constexpr int MT = 256;
constexpr int MW = MT / 32;
constexpr int TEST_T = 256;            // threads of merge_test_kernel
constexpr int SCAN_CHUNK = 256;        // blocks per chunk of the parallel scan
constexpr int ARITH_KEYS = 4096;       // union keys sorted in shared memory
constexpr int ARITH_PSMEM = 64;        // runs with P <= this keep L_aa, U_aa in shared memory

// ----------------------------------------------------------- CTA helpers
template <int NTH>
__device__ int m_scan(int *a, int n, int *s_tmp) {
  constexpr int NWp = NTH / 32;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (n + NTH - 1) / NTH;
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
    for (int w = 0; w < NWp; ++w) { int t = s_tmp[w]; s_tmp[w] = acc; acc += t; }
    s_tmp[NWp] = acc;
  }
  __syncthreads();
  int run = s_tmp[wid] + x - sum;
  for (int i = lo; i < hi; ++i) { int t = a[i]; a[i] = run; run += t; }
  int total = s_tmp[NWp];
  __syncthreads();
  return total;
}

__device__ void m_bitonic(int *a, int m) {
  for (int k = 2; k <= m; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < m; i += MT) {
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

__device__ __forceinline__ int m_lbound(const int *a, int lo, int hi, int key) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ bool m_contains(const int *a, int n, int key) {
  int p = m_lbound(a, 0, n, key);
  return p < n && a[p] == key;
}

// the test of Sec. 3.5: mu = p(p+r+s+r'+s') + q(q+t+t'), nu = (p+q)(p+q+u+v);
// merge iff nu <= 1.2 mu (exactly: 5 nu <= 6 mu, R10) or nu <= mu + 2(p+q); p+q <= max_block
__device__ __forceinline__ bool agg_test(long long p, long long q, long long r, long long s, long long t,
                                         long long r2, long long s2, long long t2, long long u, long long v,
                                         long long max_block) {
  if (p + q > max_block) return false;
  long long mu = p * (p + r + s + r2 + s2) + q * (q + t + t2);
  long long nu = (p + q) * (p + q + u + v);
  return (5 * nu <= 6 * mu) || (nu <= mu + 2 * (p + q));
}


// ---------------------------------------------------------------- M1: test
// One side (rows of L or columns of Ũ) of block k: the lists l_d = kept indices
// >= s_k of member k-d (d = 0..W).  For the aggregate a..k-1 with a = k-d:
//   r(d) = |∪_{1..d} l_d' ∩ block k|, s(d) = |∪_{1..d} l_d' ∩ [e_k, n)|,
//   u(d) = |l_0 ∪ (∪_{1..d} l_d' ∩ [e_k, n))|, t = |l_0|.
// An element of l_d is counted at d iff it is in none of l_1..l_{d-1}.
struct TestSide {
  int t;
  int r[128], s[128], u[128];   // cumulative, index d (0 unused)
};

// Per distinct key x of the window's lists: dmin(x) = smallest d >= 1 with x in l_d and
// whether x is in l_0, from an open-addressing hash table (O(total list length) per block):
// in shared memory when 2 * total <= TEST_HT, else in the CTA's global-memory table
// (M.hbig, sized by merge_bound_kernel for the widest window).
constexpr int TEST_HT = 8192;      // shared hash slots (power of two)

__device__ __forceinline__ unsigned t_hash(int key, unsigned mask) { return ((unsigned)key * 0x9E3779B1u) >> 5 & mask; }

__device__ void test_side(const MergeArgs &M, int k, int W, bool rows, int *s_hkeys, int *s_hdmin, uint8_t *s_hflag,
                          int *s_len, int *s_off, const int **s_ptr, TestSide &R) {
  const int tid = threadIdx.x;
  const int s_k = M.bstart[k], e_k = M.bstart[k + 1];
  const int32_t *idx = rows ? M.Lidx : M.Uidx;
  const int64_t *off = rows ? M.Lrow_off : M.Ucol_off;
  const int32_t *len = rows ? M.Lm : M.Uc;
  for (int d = tid; d <= W; d += TEST_T) {
    const int j = k - d;
    const int32_t *L = idx + off[j];
    const int m = len[j];
    const int p0 = m_lbound(L, 0, m, s_k);
    s_len[d] = m - p0;
    s_ptr[d] = L + p0;
  }
  for (int d = tid; d < 128; d += TEST_T) { R.r[d] = 0; R.s[d] = 0; R.u[d] = 0; }
  __syncthreads();
  if (tid < 32) {   // exclusive prefix of the W+1 list lengths, one warp
    const int lane = tid;
    int carry = 0;
    for (int base = 0; base <= W; base += 32) {
      const int d = base + lane;
      const int v = d <= W ? s_len[d] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (d <= W) s_off[d] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) { s_off[W + 1] = carry; R.t = s_len[0]; }
  }
  __syncthreads();
  const int total = s_off[W + 1];
  unsigned hs = 64;
  while (hs < 2u * (unsigned)total) hs <<= 1;
  int *hkeys = s_hkeys, *hdmin = s_hdmin;
  uint8_t *hflag = s_hflag;
  if (hs > (unsigned)TEST_HT) {      // the CTA's global table (capacity checked by the host's bound)
    unsigned char *base = M.hbig + (size_t)blockIdx.x * 9 * (size_t)M.hbig_cap;
    hkeys = (int *)base;
    hdmin = hkeys + M.hbig_cap;
    hflag = (uint8_t *)(hdmin + M.hbig_cap);
  }
  const unsigned mask = hs - 1;
  for (unsigned h = tid; h < hs; h += TEST_T) { hkeys[h] = -1; hdmin[h] = 255; hflag[h] = 0; }
  __syncthreads();
  for (int x = tid; x < total; x += TEST_T) {
    int lo = 0, hi = W;
    while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (s_off[mid] <= x) lo = mid; else hi = mid - 1; }
    const int d = lo;
    const int key = s_ptr[d][x - s_off[d]];
    unsigned h = t_hash(key, mask);
    while (true) {
      const int old = atomicCAS(&hkeys[h], -1, key);
      if (old == -1 || old == key) break;
      h = (h + 1) & mask;
    }
    if (d == 0) hflag[h] = 1;
    else atomicMin(&hdmin[h], d);
  }
  __syncthreads();
  for (unsigned h = tid; h < hs; h += TEST_T) {
    const int key = hkeys[h], d = hdmin[h];
    if (key < 0 || d > W) continue;
    if (key < e_k) atomicAdd(&R.r[d], 1);
    else {
      atomicAdd(&R.s[d], 1);
      if (!hflag[h]) atomicAdd(&R.u[d], 1);
    }
  }
  __syncthreads();
  if (tid == 0) {
    int r = 0, s = 0, u = R.t;
    for (int d = 1; d <= W; ++d) { r += R.r[d]; s += R.s[d]; u += R.u[d]; R.r[d] = r; R.s[d] = s; R.u[d] = u; }
  }
  __syncthreads();
}

// widest test window: max over k and both sides of the window's total list length
__global__ void __launch_bounds__(256) merge_bound_kernel(MergeArgs M, unsigned long long *out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int k = gw; k < M.N; k += nw) {
    const int W = (int)(M.wofs[k + 1] - M.wofs[k]) - 1;
    if (W <= 0) continue;
    const int s_k = M.bstart[k];
    long long tl = 0, tu = 0;
    for (int d = lane; d <= W; d += 32) {
      const int j = k - d;
      const int ml = M.Lm[j], mu = M.Uc[j];
      tl += ml - m_lbound(M.Lidx + M.Lrow_off[j], 0, ml, s_k);
      tu += mu - m_lbound(M.Uidx + M.Ucol_off[j], 0, mu, s_k);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tl += __shfl_xor_sync(0xffffffffu, tl, o);
      tu += __shfl_xor_sync(0xffffffffu, tu, o);
    }
    if (lane == 0) atomicMax(out, (unsigned long long)(tl > tu ? tl : tu));
  }
}

__global__ void __launch_bounds__(TEST_T) merge_test_kernel(MergeArgs M) {
  extern __shared__ __align__(16) unsigned char tsm[];
  int *hkeys = (int *)tsm;
  int *hdmin = hkeys + TEST_HT;
  uint8_t *hflag = (uint8_t *)(hdmin + TEST_HT);
  __shared__ int s_len[129], s_off[130];
  __shared__ const int *s_ptr[129];
  __shared__ TestSide SR, SC;
  __shared__ uint32_t s_mask[4];
  const int tid = threadIdx.x;
  __shared__ int s_k;
  while (true) {
    // dynamic assignment, last block first (the separators' wide windows start early)
    __syncthreads();
    if (tid == 0) s_k = M.N - 1 - atomicAdd(M.ticket, 1);
    __syncthreads();
    const int k = s_k;
    if (k < 0) break;
    if (tid < 4) s_mask[tid] = 0u;
    const int W = (int)(M.wofs[k + 1] - M.wofs[k]) - 1;     // the host's window (same rule)
    __syncthreads();
    if (W > 0) {
      test_side(M, k, W, true, hkeys, hdmin, hflag, s_len, s_off, s_ptr, SR);
      test_side(M, k, W, false, hkeys, hdmin, hflag, s_len, s_off, s_ptr, SC);
      const int s_k = M.bstart[k], q = M.bstart[k + 1] - s_k;
      int32_t *uv = M.UV + 2 * M.wofs[k];
      for (int d = 1 + tid; d <= W; d += TEST_T) {
        const long long p = s_k - M.bstart[k - d];
        if (agg_test(p, q, SR.r[d], SR.s[d], SR.t, SC.r[d], SC.s[d], SC.t, SR.u[d], SC.u[d], M.max_block))
          atomicOr(&s_mask[(d - 1) >> 5], 1u << ((d - 1) & 31));
        uv[2 * d] = SR.u[d];
        uv[2 * d + 1] = SC.u[d];
      }
    }
    __syncthreads();
    if (tid < 4) M.T[4 * (size_t)k + tid] = s_mask[tid];
    __syncthreads();
  }
}

// ---------------------------------------------------------------- M2: scan
// The paper's order: after block k is finished, merge it into the aggregate
// that ends at k-1 iff the test passes.  State before block
// k: d = (k-1) - a, a = start of the current run; k merges iff bit d of T[k] is set
// (then d' = d+1, else d' = 0).  Chunks of SCAN_CHUNK blocks map every start state
// (0..127) to an end state in parallel; one thread composes the chunk maps; every
// chunk is then replayed from its true start state.
__global__ void __launch_bounds__(128) merge_chunkmap_kernel(MergeArgs M) {
  const int c = blockIdx.x, st0 = threadIdx.x;
  const int k0 = 1 + c * SCAN_CHUNK, k1 = min(M.N, k0 + SCAN_CHUNK);
  int d = st0;
  for (int k = k0; k < k1; ++k) {
    const uint32_t w = __ldg(&M.T[4 * (size_t)k + (d >> 5)]);
    d = (d < 127 && ((w >> (d & 31)) & 1u)) ? d + 1 : 0;
  }
  M.chunkmap[(size_t)c * 128 + st0] = (uint8_t)d;
}

__global__ void __launch_bounds__(1024) merge_scan_kernel(MergeArgs M, int nchunks) {
  __shared__ int s_tmp[33];
  const int tid = threadIdx.x;
  // compose the chunk maps (sequential over chunks, one thread)
  if (tid == 0) {
    int d = 0;
    for (int c = 0; c < nchunks; ++c) { M.chunkstart[c] = (uint8_t)d; d = M.chunkmap[(size_t)c * 128 + d]; }
  }
  __syncthreads();
  // replay: flag[k] = 1 iff a run starts at k
  int *flag = M.flag;
  if (tid == 0) flag[0] = 1;
  for (int c = tid; c < nchunks; c += blockDim.x) {
    const int k0 = 1 + c * SCAN_CHUNK, k1 = min(M.N, k0 + SCAN_CHUNK);
    int d = M.chunkstart[c];
    for (int k = k0; k < k1; ++k) {
      const uint32_t w = M.T[4 * (size_t)k + (d >> 5)];
      const bool merge = d < 127 && ((w >> (d & 31)) & 1u);
      flag[k] = merge ? 0 : 1;
      d = merge ? d + 1 : 0;
    }
  }
  __syncthreads();
  // exclusive scan of the flags -> run ids; first[run] = k
  const int N = M.N;
  const int per = (N + 1023) / 1024;
  const int lo = min(N, tid * per), hi = min(N, lo + per);
  int sum = 0;
  for (int i = lo; i < hi; ++i) sum += flag[i];
  const int lane = tid & 31, wid = tid >> 5;
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
    for (int w = 0; w < 32; ++w) { int t = s_tmp[w]; s_tmp[w] = acc; acc += t; }
    s_tmp[32] = acc;
  }
  __syncthreads();
  int run = s_tmp[wid] + x - sum;
  for (int i = lo; i < hi; ++i)
    if (flag[i]) M.first[run++] = i;
  if (tid == 0) { M.first[s_tmp[32]] = N; *M.nF = s_tmp[32]; }
}

// --------------------------------------------------- M3: descriptors, offsets
template <int NV>
__device__ void block_scan_ull(unsigned long long (&v)[NV], unsigned long long (&tot)[NV]) {
  __shared__ unsigned long long sw[NV][32];
  __shared__ unsigned long long st[NV];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    unsigned long long x = v[j];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sw[j][wid] = x;
    v[j] = x - v[j];   // exclusive within the warp
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      unsigned long long x = lane < nw ? sw[j][lane] : 0ull, x0 = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane < nw) sw[j][lane] = x - x0;
      if (lane == 31) st[j] = x;      // total (nw <= 32)
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; ++j) { v[j] += sw[j][wid]; tot[j] = st[j]; }
  __syncthreads();
}

// Singletons keep their arena slices; merged blocks are appended after the factor
// kernel's cursors (tot[0..3] on entry).  Union sizes of merged runs a..k come
// from the test: u(k-a), v(k-a) of block k.  One CTA of 1024 threads.
__global__ void __launch_bounds__(1024) merge_offsets_kernel(MergeArgs M) {
  const int nF = *M.nF;
  const int per = (nF + blockDim.x - 1) / blockDim.x;
  const int lo = min(nF, (int)threadIdx.x * per), hi = min(nF, lo + per);
  // per-thread sums: D, Li, Lv, Ui, Uv (merged only), nL, nU, iL, iU, nmerged
  unsigned long long v[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long maxws = 0;
  for (int F = lo; F < hi; ++F) {
    const int a = M.first[F], k = M.first[F + 1] - 1;
    const unsigned long long P = M.bstart[k + 1] - M.bstart[a];
    unsigned long long u, w;
    if (a == k) { u = M.Lm[k]; w = M.Uc[k]; }
    else {
      const int32_t *uv = M.UV + 2 * (M.wofs[k] + (k - a));
      u = uv[0]; w = uv[1];
    }
    M.fbstart[F] = M.bstart[a];
    M.fLm[F] = (int32_t)u; M.fUc[F] = (int32_t)w;
    v[0] += P * P;
    if (a != k) {
      v[1] += u; v[2] += u * P; v[3] += w; v[4] += w * P; v[9] += k - a;
      const unsigned long long ws = (u > w ? u : w) * P;
      if (ws > maxws) maxws = ws;
    }
    v[5] += u * P; v[6] += w * P; v[7] += u; v[8] += w;
  }
  unsigned long long tot[10];
  block_scan_ull<10>(v, tot);
  unsigned long long cD = v[0], cLi = M.tot[0] + v[1], cLv = M.tot[1] + v[2], cUi = M.tot[2] + v[3],
                     cUv = M.tot[3] + v[4];
  for (int F = lo; F < hi; ++F) {
    const int a = M.first[F], k = M.first[F + 1] - 1;
    const unsigned long long P = M.bstart[k + 1] - M.bstart[a];
    M.fD_off[F] = (int64_t)cD;
    cD += P * P;
    if (a == k) {
      M.fLrow_off[F] = M.Lrow_off[k]; M.fLval_off[F] = M.Lval_off[k];
      M.fUcol_off[F] = M.Ucol_off[k]; M.fUval_off[F] = M.Uval_off[k];
    } else {
      const unsigned long long u = M.fLm[F], w = M.fUc[F];
      M.fLrow_off[F] = (int64_t)cLi; cLi += u;
      M.fLval_off[F] = (int64_t)cLv; cLv += u * P;
      M.fUcol_off[F] = (int64_t)cUi; cUi += w;
      M.fUval_off[F] = (int64_t)cUv; cUv += w * P;
    }
  }
  __shared__ unsigned long long smax;
  if (threadIdx.x == 0) smax = 0;
  __syncthreads();
  atomicMax(&smax, maxws);
  __syncthreads();
  if (threadIdx.x == 0) {
    M.fbstart[nF] = M.n;
    M.fD_off[nF] = (int64_t)tot[0];
    M.tot[4] = M.tot[0] + tot[1]; M.tot[5] = M.tot[1] + tot[2];
    M.tot[6] = M.tot[2] + tot[3]; M.tot[7] = M.tot[3] + tot[4];
    M.tot[8] = tot[0]; M.tot[9] = smax; M.tot[10] = 0;
    M.tot[11] = tot[9];
    M.tot[12] = tot[5]; M.tot[13] = tot[6]; M.tot[14] = tot[7]; M.tot[15] = tot[8];
  }
}

// ---------------------------------------------------------------- M4: arithmetic
// Sorted union of the members' kept indices >= e_k, written to out[0..u): the members'
// suffixes are concatenated (each sorted); an element is "first" if no earlier member's
// suffix contains it; its rank in the union is the number of first elements smaller than it,
// summed over the suffixes via a prefix scan of the first-flags and binary searches.
// Returns the number of distinct keys (must equal the test's union size), -1 if the
// buffers are too small.
__device__ int build_union(const MergeArgs &M, int a, int k, bool rows, int *keys, int *flags, int cap,
                           int *s_cnt, int *s_tmp, int *out, int *sout) {
  const int tid = threadIdx.x;
  const int e_k = M.bstart[k + 1];
  const int32_t *idx = rows ? M.Lidx : M.Uidx;
  const int64_t *off = rows ? M.Lrow_off : M.Ucol_off;
  const int32_t *len = rows ? M.Lm : M.Uc;
  const int nm = k - a + 1;
  for (int x = tid; x < nm; x += MT) {
    const int j = a + x;
    const int32_t *L = idx + off[j];
    const int m = len[j];
    s_cnt[x] = m - m_lbound(L, 0, m, e_k);
  }
  __syncthreads();
  const int total = m_scan<MT>(s_cnt, nm, s_tmp);     // s_cnt[x] = start of member x's suffix
  if (total + 1 > cap) return -1;
  if (tid == 0) s_cnt[nm] = total;
  for (int x = 0; x < nm; ++x) {
    const int j = a + x;
    const int32_t *L = idx + off[j];
    const int m = len[j];
    const int c = (x + 1 < nm ? s_cnt[x + 1] : total) - s_cnt[x];
    for (int i = tid; i < c; i += MT) keys[s_cnt[x] + i] = L[m - c + i];
  }
  __syncthreads();
  // member of element t: the last x with s_cnt[x] <= t
  for (int t = tid; t < total; t += MT) {
    int lo = 0, hi = nm - 1;
    while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (s_cnt[mid] <= t) lo = mid; else hi = mid - 1; }
    const int key = keys[t];
    bool first = true;
    for (int x2 = 0; x2 < lo && first; ++x2) {
      const int b0 = s_cnt[x2], b1 = s_cnt[x2 + 1];
      const int p = m_lbound(keys, b0, b1, key);
      first = !(p < b1 && keys[p] == key);
    }
    flags[t] = first ? 1 : 0;
  }
  __syncthreads();
  const int u = m_scan<MT>(flags, total, s_tmp);      // exclusive prefix of the first-flags
  if (tid == 0) flags[total] = u;
  __syncthreads();
  for (int t = tid; t < total; t += MT) {
    const int f = (t + 1 <= total ? flags[t + 1] : u) - flags[t];
    if (!f) continue;
    const int key = keys[t];
    int rank = 0;
    for (int x2 = 0; x2 < nm; ++x2) {
      const int b0 = s_cnt[x2], b1 = s_cnt[x2 + 1];
      rank += flags[m_lbound(keys, b0, b1, key)] - flags[b0];
    }
    out[rank] = key;
  }
  __syncthreads();
  if (sout && u <= ARITH_KEYS) {   // shared copy for the lookups (the key buffer is dead now)
    for (int x = tid; x < u; x += MT) sout[x] = out[x];
    __syncthreads();
  }
  return u;
}

// per merged run a..k (P = e_k - s_a <= max_block), member blocks j with offsets
// o_j = s_j - s_a:
//   L_aa (unit lower, identity member diagonal blocks), U_aa = D_j Ũ_j inside the run
//   Linv:  X L_aa = I                 (member-block steps, last to first)
//   D^:    U_aa D^ = D_agg Linv        (member-block steps, last to first)
//   L^ =   L_{>,agg} · Linv            (DMMA GEMM, u x P x P)
//   Ũ^ =   L_aa · Ũ_{agg,>}            (DMMA GEMM, P x v x P)
// Global workspace per CTA: [L_aa, U_aa if P > ARITH_PSMEM] Linv (P^2), G (max(u,v) P).
__global__ void __launch_bounds__(MT) merge_arith_kernel(MergeArgs M, double *dwork, int64_t dwork_per_cta) {
  extern __shared__ __align__(16) unsigned char msm_raw[];
  double *sLU = (double *)msm_raw;                                            // 2 * 64^2 doubles
  unsigned char *scratch = msm_raw + 2 * ARITH_PSMEM * ARITH_PSMEM * 8;       // union keys | GEMM staging
  int *skeys = (int *)scratch;                                                // ARITH_KEYS
  int *sflags = skeys + ARITH_KEYS;                                           // ARITH_KEYS
  int *sunion = skeys;                                                        // the union, for lookups
  double *sgemm = (double *)scratch;
  __shared__ int s_tmp[MW + 1];
  __shared__ int s_cnt[130];
  __shared__ int s_mo[130];       // member offsets o_j, j = a..k+1
  __shared__ int s_mi[130], s_ci[130];   // per member: kept rows / cols inside the run (a prefix)
  const int tid = threadIdx.x;
  const int nF = *M.nF;
  double *gbase = dwork + (size_t)blockIdx.x * dwork_per_cta;
  int *gkeys = M.work + (size_t)blockIdx.x * M.work_ints;
  double flops = 0.0;
  __shared__ int s_F;
  while (true) {
    // dynamic assignment, last final block first: the separator runs (largest P, widest
    // unions) sit at the end of the ordering and start before the cheap copies
    __syncthreads();
    if (tid == 0) s_F = nF - 1 - atomicAdd(M.ticket, 1);
    __syncthreads();
    const int F = s_F;
    if (F < 0) break;
    const int a = M.first[F], k = M.first[F + 1] - 1;
    const int sa = M.bstart[a], ek = M.bstart[k + 1];
    const int P = ek - sa;
    double *Dout = M.fD + M.fD_off[F];
    if (a == k) {
      const double *Din = M.D + M.D_off[k];
      for (int i = tid; i < P * P; i += MT) Dout[i] = Din[i];
      continue;
    }
    const int nm = k - a + 1;
    for (int x = tid; x <= nm; x += MT) s_mo[x] = M.bstart[a + x] - sa;
    for (int x = tid; x < nm; x += MT) {   // one binary search per member list, shared by all threads
      const int j = a + x;
      s_mi[x] = m_lbound(M.Lidx + M.Lrow_off[j], 0, M.Lm[j], ek);
      s_ci[x] = m_lbound(M.Uidx + M.Ucol_off[j], 0, M.Uc[j], ek);
    }
    double *Laa, *Uaa, *Linv, *G;
    if (P <= ARITH_PSMEM) { Laa = sLU; Uaa = sLU + P * P; Linv = gbase; }
    else { Laa = gbase; Uaa = gbase + (size_t)P * P; Linv = Uaa + (size_t)P * P; }
    G = Linv + (size_t)P * P;
    for (int i = tid; i < P * P; i += MT) {
      const int r = i / P, c = i - r * P;
      Laa[i] = (r == c) ? 1.0 : 0.0;
      Uaa[i] = (r == c) ? 1.0 : 0.0;
      Linv[i] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    // L_aa, U_aa from the members
    for (int x = 0; x < nm; ++x) {
      const int j = a + x;
      const int oj = s_mo[x], bj = s_mo[x + 1] - oj;
      const int32_t *rows = M.Lidx + M.Lrow_off[j];
      const double *Lv = M.Lval + M.Lval_off[j];
      const int mi = s_mi[x];      // rows inside the run are a prefix
      for (int it = tid; it < mi * bj; it += MT) {
        const int p = it / bj, t = it - p * bj;
        Laa[(size_t)(rows[p] - sa) * P + oj + t] = Lv[it];
      }
      const int32_t *cols = M.Uidx + M.Ucol_off[j];
      const double *Uv = M.Uval + M.Uval_off[j];
      const double *Dj = M.D + M.D_off[j];
      const int ci = s_ci[x];
      for (int it = tid; it < ci * bj; it += MT) {
        const int q = it / bj, r = it - q * bj;
        double acc = 0.0;
        for (int t = 0; t < bj; ++t) acc = fma(Dj[r + (size_t)t * bj], Uv[(size_t)q * bj + t], acc);
        Uaa[(size_t)(oj + r) * P + (cols[q] - sa)] = acc;
      }
    }
    __syncthreads();
    // Linv (row-major): X L_aa = I, members last to first: X[:, c in m] -= X[:, later] L_aa[later, c]
    for (int x = nm - 2; x >= 0; --x) {
      const int om = s_mo[x], bm = s_mo[x + 1] - om, e = s_mo[x + 1];
      for (int it = tid; it < P * bm; it += MT) {
        const int i = it / bm, c = om + it % bm;
        if (i < e) continue;                 // rows above the later members stay e_i
        const double *xr = Linv + (size_t)i * P;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int t = e;
        for (; t + 3 <= i; t += 4) {
          a0 = fma(xr[t], Laa[(size_t)t * P + c], a0); a1 = fma(xr[t + 1], Laa[(size_t)(t + 1) * P + c], a1);
          a2 = fma(xr[t + 2], Laa[(size_t)(t + 2) * P + c], a2); a3 = fma(xr[t + 3], Laa[(size_t)(t + 3) * P + c], a3);
        }
        for (; t <= i; ++t) a0 = fma(xr[t], Laa[(size_t)t * P + c], a0);
        Linv[(size_t)i * P + c] = -((a0 + a1) + (a2 + a3));
      }
      __syncthreads();
    }
    // D^ (column-major): T = D_agg Linv, then U_aa D^ = T, members last to first; computed in
    // the shared scratch (idle in this phase) when it fits, then stored to Dout
    double *Dw = (P <= ARITH_PSMEM) ? (double *)scratch : Dout;
    for (int x = 0; x < nm; ++x) {
      const int om = s_mo[x], bm = s_mo[x + 1] - om;
      const double *Dj = M.D + M.D_off[a + x];
      for (int it = tid; it < P * bm; it += MT) {
        const int r = it % bm, c = it / bm;
        double acc = 0.0;
        for (int t = 0; t < bm; ++t) acc = fma(Dj[r + (size_t)t * bm], Linv[(size_t)(om + t) * P + c], acc);
        Dw[(size_t)c * P + om + r] = acc;
      }
    }
    __syncthreads();
    for (int x = nm - 2; x >= 0; --x) {
      const int om = s_mo[x], bm = s_mo[x + 1] - om, e = s_mo[x + 1];
      for (int it = tid; it < P * bm; it += MT) {
        const int r = om + it % bm, c = it / bm;
        const double *ur = Uaa + (size_t)r * P;
        const double *dc = Dw + (size_t)c * P;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int t = e;
        for (; t + 3 < P; t += 4) {
          a0 = fma(ur[t], dc[t], a0); a1 = fma(ur[t + 1], dc[t + 1], a1);
          a2 = fma(ur[t + 2], dc[t + 2], a2); a3 = fma(ur[t + 3], dc[t + 3], a3);
        }
        for (; t < P; ++t) a0 = fma(ur[t], dc[t], a0);
        Dw[(size_t)c * P + r] -= (a0 + a1) + (a2 + a3);
      }
      __syncthreads();
    }
    if (Dw != Dout) {
      for (int i = tid; i < P * P; i += MT) Dout[i] = Dw[i];
      __syncthreads();
    }
    // ---- L^ rows: union, gathered L_g (u x P row-major) in G, L^ = G Linv
    const int u = M.fLm[F], v = M.fUc[F];
    {
      int *R = M.Lidx_out + M.fLrow_off[F];
      int uu = build_union(M, a, k, true, skeys, sflags, ARITH_KEYS, s_cnt, s_tmp, R, sunion);
      if (uu < 0) uu = build_union(M, a, k, true, gkeys, gkeys + M.work_ints / 2, (int)(M.work_ints / 2), s_cnt, s_tmp, R, sunion);
      const int *Rl = uu <= ARITH_KEYS ? sunion : R;     // lookups in shared memory when it fits
      if (uu != u) { if (tid == 0) atomicExch(M.ovf, uu < 0 ? 1 : 2); return; }
      if (u > 0) {
        for (int i = tid; i < u * P; i += MT) G[i] = 0.0;
        __syncthreads();
        for (int x = 0; x < nm; ++x) {
          const int j = a + x;
          const int oj = s_mo[x], bj = s_mo[x + 1] - oj;
          const int32_t *rows = M.Lidx + M.Lrow_off[j];
          const double *Lv = M.Lval + M.Lval_off[j];
          const int mj = M.Lm[j];
          const int mi = s_mi[x];
          for (int p = mi + tid; p < mj; p += MT) {     // one search per row, then its b_j values
            double *g = G + (size_t)m_lbound(Rl, 0, u, rows[p]) * P + oj;
            const double *lv = Lv + (size_t)p * bj;
            for (int t = 0; t < bj; ++t) g[t] = lv[t];
          }
        }
        __syncthreads();
        cta_dgemm<MT>(u, P, P, 1.0, DMat{G, P, 1}, DMat{Linv, P, 1}, 0.0, M.Lval_out + M.fLval_off[F], P, 1,
                      sgemm);
      }
    }
    // ---- Ũ^ columns: union, gathered Ũ_g (P x v column-major) in G, Ũ^ = L_aa G
    {
      int *Cc = M.Uidx_out + M.fUcol_off[F];
      int vv = build_union(M, a, k, false, skeys, sflags, ARITH_KEYS, s_cnt, s_tmp, Cc, sunion);
      if (vv < 0) vv = build_union(M, a, k, false, gkeys, gkeys + M.work_ints / 2, (int)(M.work_ints / 2), s_cnt, s_tmp, Cc, sunion);
      const int *Cl = vv <= ARITH_KEYS ? sunion : Cc;
      if (vv != v) { if (tid == 0) atomicExch(M.ovf, vv < 0 ? 1 : 2); return; }
      if (v > 0) {
        for (int i = tid; i < v * P; i += MT) G[i] = 0.0;
        __syncthreads();
        for (int x = 0; x < nm; ++x) {
          const int j = a + x;
          const int oj = s_mo[x], bj = s_mo[x + 1] - oj;
          const int32_t *cols = M.Uidx + M.Ucol_off[j];
          const double *Uv = M.Uval + M.Uval_off[j];
          const int cj = M.Uc[j];
          const int ci = s_ci[x];
          for (int q = ci + tid; q < cj; q += MT) {     // one search per column, then its b_j values
            double *g = G + (size_t)m_lbound(Cl, 0, v, cols[q]) * P + oj;
            const double *uv = Uv + (size_t)q * bj;
            for (int t = 0; t < bj; ++t) g[t] = uv[t];
          }
        }
        __syncthreads();
        cta_dgemm<MT>(P, v, P, 1.0, DMat{Laa, P, 1}, DMat{G, 1, P}, 0.0, M.Uval_out + M.fUval_off[F], 1, P, sgemm);
      }
    }
    if (tid == 0) {
      const double Pd = P;
      flops += 2.0 * Pd * Pd * Pd / 3.0 + 2.0 * Pd * Pd * Pd / 2.0 + Pd * Pd * Pd + (double)(u + v) * Pd * Pd;
    }
    __syncthreads();
  }
  if (tid == 0 && flops > 0.0) atomicAdd(M.flops, flops);
}

// ----------------------------------------------------------------- launchers
extern "C" cudaError_t bilu_merge_plan(const MergeArgs &M, int grid, cudaStream_t st) {
  const int nchunks = M.N > 1 ? (M.N - 1 + SCAN_CHUNK - 1) / SCAN_CHUNK : 0;
  const int tsmem = TEST_HT * 9;
  cudaError_t e = cudaFuncSetAttribute(merge_test_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem);
  if (e != cudaSuccess) return e;
  merge_test_kernel<<<grid * 3, TEST_T, tsmem, st>>>(M);   // bilu_merge_test_grid
  if (nchunks > 0) merge_chunkmap_kernel<<<nchunks, 128, 0, st>>>(M);
  merge_scan_kernel<<<1, 1024, 0, st>>>(M, nchunks);
  merge_offsets_kernel<<<1, 1024, 0, st>>>(M);
  return cudaGetLastError();
}

extern "C" int bilu_merge_plan_launches() { return 4; }
extern "C" int bilu_merge_test_grid(int grid) { return grid * 3; }

extern "C" cudaError_t bilu_merge_bound(const MergeArgs &M, unsigned long long *out, int sms, cudaStream_t st) {
  cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
  merge_bound_kernel<<<sms * 8, 256, 0, st>>>(M, out);
  return cudaGetLastError();
}
extern "C" int bilu_merge_nchunks(int N) { return N > 1 ? (N - 1 + SCAN_CHUNK - 1) / SCAN_CHUNK : 0; }

extern "C" cudaError_t bilu_merge_arith(const MergeArgs &M, double *dwork, int64_t dwork_per_cta, int grid,
                                        cudaStream_t st) {
  const int smem = 2 * ARITH_PSMEM * ARITH_PSMEM * 8 + (2 * ARITH_KEYS * 4 > DGEMM_SMEM_DOUBLES * 8 ? 2 * ARITH_KEYS * 4 : DGEMM_SMEM_DOUBLES * 8);
  cudaError_t e = cudaFuncSetAttribute(merge_arith_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  merge_arith_kernel<<<grid, MT, smem, st>>>(M, dwork, dwork_per_cta);   // grid = 2 CTAs per SM
  return cudaGetLastError();
}

extern "C" int bilu_merge_args_size() { return (int)sizeof(MergeArgs); }

}  // namespace bilu
