// bilu_blocking.cu -- the ILU(1,tau) initial block estimate of Sec. 3.4 (PAPER.md:1171-1242,
// DESIGN.md R20) on the device: the input of bilu_analyze's block partition.
//
//  0. Ã = A(perm, perm) on the device (rows left unsorted).
//  1. CSC of Ã and its diagonal (count / scan / scatter; the order
//     inside a column is irrelevant: only sets are built from it).
//  2. Estimated patterns I~_k (column k of L) and J~_k (row k of U), one warp per step k:
//     the direct entries |a_ik| >= tau |a_kk| plus the ILU(1) fill |a_ij a_jk| >= tau |a_jj a_kk|
//     (j < k < i) collected in a warp-private shared-memory hash table.
//     Two passes (count, scan, write) give exact storage; a step whose candidate bound does
//     not fit the table is redone by the same code on a per-warp global-memory table.
//  3. Greedy growth is sequential in the block starts, so it runs
//     speculatively: one warp per possible start k0 computes L(k0), the block length the greedy
//     rule picks when a block starts at k0 (unions of the sets in hash tables, r and s counted
//     outside the grown block, 3 f <= 4 c' or f <= c' + 4(l+1), l <= max_size).
//  4. The partition is the chain 0 -> L(0) -> ...: per chunk of CH positions a table of
//     exit offsets for every entry offset in [0, max_size), a sequential composition over
//     chunks, and a parallel walk that emits the block sizes.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <vector>

namespace bilu {

constexpr int BT = 256;          // threads per CTA
constexpr int BW = BT / 32;      // warps per CTA
constexpr int SET_CAP = 2048;    // warp-private set table (ints)
constexpr int GROW_CAP = 1024;   // per union table (ints), two per warp
constexpr int CH = 256;          // chain chunk
constexpr int SCAN_TILE = 2048;  // 256 threads x 8

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// open addressing, linear probing, -1 = empty; keys are indices >= 0
struct Table {
  int32_t *t;
  uint32_t mask;
};
__device__ __forceinline__ uint32_t slot0(int32_t key, uint32_t mask) {
  uint32_t h = (uint32_t)key * 0x9E3779B1u;
  return (h ^ (h >> 15)) & mask;
}
__device__ __forceinline__ int t_insert(Table T, int32_t key) {
  uint32_t s = slot0(key, T.mask);
  while (true) {
    const int32_t old = atomicCAS(T.t + s, -1, key);
    if (old == -1) return 1;
    if (old == key) return 0;
    s = (s + 1) & T.mask;
  }
}
__device__ __forceinline__ int t_find(Table T, int32_t key) {
  uint32_t s = slot0(key, T.mask);
  while (true) {
    const int32_t v = ((volatile int32_t *)T.t)[s];
    if (v == key) return 1;
    if (v == -1) return 0;
    s = (s + 1) & T.mask;
  }
}
__device__ __forceinline__ void t_clear(Table T, int lane) {
  for (uint32_t i = lane; i <= T.mask; i += 32) T.t[i] = -1;
  __syncwarp();
}
// writes the table's keys to out (arbitrary order), returns the count (warp-uniform)
__device__ __forceinline__ int t_emit(Table T, int32_t *out, int lane) {
  int base = 0;
  for (uint32_t s0 = 0; s0 <= T.mask; s0 += 32) {
    const int32_t v = T.t[s0 + lane];
    const unsigned b = __ballot_sync(0xffffffffu, v >= 0);
    if (v >= 0) out[base + __popc(b & ((1u << lane) - 1u))] = v;
    base += __popc(b);
  }
  return base;
}

struct EstArgs {
  int n;
  const int64_t *rp;  const int32_t *ci;  const double *val;   // Ã, CSR
  const int64_t *cp;  const int32_t *cr;  const double *cv;    // Ã, CSC
  const double *diag;
  double tau;
};

// candidate count of step k (direct entries + the fill candidates): the table bound
template <bool LOWER>
__device__ int64_t set_bound(const EstArgs &E, int k, int lane) {
  const int64_t *P = LOWER ? E.cp : E.rp;
  const int32_t *X = LOWER ? E.cr : E.ci;
  int64_t b = 0;
  for (int64_t p = P[k] + lane; p < P[k + 1]; p += 32) {
    const int32_t j = X[p];
    if (j < k) b += P[j + 1] - P[j];
  }
  return warp_sum64(b) + (P[k + 1] - P[k]);
}

// I~_k (LOWER: column k, through the CSC) or J~_k (row k, through the CSR) into T (cleared);
// returns the set size.  PAPER.md:1183-1198; the products are the oracle's (R20).  With a
// limit (optimistic shared-memory attempt) the build stops once the distinct keys, counted in
// *nkeys, reach it (<= half the table, overshoot < 32): returns -1 then.
template <bool LOWER>
__device__ int build_set(const EstArgs &E, int k, Table T, int lane, int *nkeys = nullptr, int limit = 0) {
  const int64_t *P = LOWER ? E.cp : E.rp;
  const int32_t *X = LOWER ? E.cr : E.ci;
  const double *V = LOWER ? E.cv : E.val;
  volatile int *vk = nkeys;
  const double akk = E.diag[k];
  const double thr = E.tau * fabs(akk);
  int64_t cnt = 0;
  for (int64_t p = P[k] + lane; p < P[k + 1]; p += 32) {
    const int32_t x = X[p];
    if (x > k && fabs(V[p]) >= thr) {
      const int nw = t_insert(T, x);
      cnt += nw;
      if (limit && nw) atomicAdd(nkeys, 1);
    }
  }
  __syncwarp();
  for (int64_t p = P[k]; p < P[k + 1]; ++p) {          // j < k with a_jk != 0 (resp. i < k, a_ki != 0)
    const int32_t j = X[p];
    if (j >= k) continue;
    if (limit && *vk >= limit) return -1;
    const double ajk = V[p];
    const double thr2 = E.tau * fabs(E.diag[j] * akk);
    for (int64_t q = P[j] + lane; q < P[j + 1]; q += 32) {
      if (limit && *vk >= limit) break;
      const int32_t x = X[q];
      if (x > k && fabs(V[q] * ajk) >= thr2) {
        const int nw = t_insert(T, x);
        cnt += nw;
        if (limit && nw) atomicAdd(nkeys, 1);
      }
    }
    __syncwarp();
  }
  __syncwarp();
  if (limit && *vk >= limit) return -1;
  return (int)warp_sum64(cnt);
}

struct SetOut {
  int64_t *cnt;           // count pass: set sizes
  const int64_t *off;     // write pass: offsets
  int32_t *out;
  int32_t *ovf_list;
  int *ovf_n;
  unsigned long long *ovf_max;
};

// steps whose candidate bound exceeds half the table are tried optimistically (candidates
// repeat); a step whose distinct keys do not fit goes to the global tables
template <bool LOWER, bool WRITE>
__global__ void __launch_bounds__(BT) sets_kernel(EstArgs E, SetOut O) {
  extern __shared__ int32_t s_tab[];
  __shared__ int s_nkeys[BW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const Table T{s_tab + w * SET_CAP, SET_CAP - 1};
  for (int k = blockIdx.x * BW + w; k < E.n; k += gridDim.x * BW) {
    const int64_t b = set_bound<LOWER>(E, k, lane);
    const int limit = 2 * b > SET_CAP ? SET_CAP / 2 : 0;
    t_clear(T, lane);
    if (lane == 0) s_nkeys[w] = 0;
    __syncwarp();
    const int c = build_set<LOWER>(E, k, T, lane, s_nkeys + w, limit);
    if (c < 0) {
      if (!WRITE && lane == 0) {
        O.ovf_list[atomicAdd(O.ovf_n, 1)] = k;
        atomicMax(O.ovf_max, (unsigned long long)b);
      }
      __syncwarp();
      continue;
    }
    if (WRITE) t_emit(T, O.out + O.off[k], lane);
    else if (lane == 0) O.cnt[k] = c;
    __syncwarp();
  }
}

// overflowed steps: same code on per-warp global tables of cap entries
template <bool LOWER, bool WRITE>
__global__ void __launch_bounds__(BT) sets_big_kernel(EstArgs E, SetOut O, int nlist, int32_t *region, uint32_t cap) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * BT + threadIdx.x) >> 5, nw = gridDim.x * BW;
  const Table T{region + (int64_t)gw * cap, cap - 1};
  for (int x = gw; x < nlist; x += nw) {
    const int k = O.ovf_list[x];
    t_clear(T, lane);
    const int c = build_set<LOWER>(E, k, T, lane);
    if (WRITE) t_emit(T, O.out + O.off[k], lane);
    else if (lane == 0) O.cnt[k] = c;
    __syncwarp();
  }
}

struct GrowArgs {
  int n, max_size;
  const int64_t *Io; const int32_t *Is;
  const int64_t *Jo; const int32_t *Js;
  int32_t *L;
  int32_t *ovf_list;
  int *ovf_n;
  unsigned long long *ovf_max;
};

// L(k0): the greedy block length from start k0 (R20)
__device__ int grow_block(const GrowArgs &G, int k0, Table TI, Table TJ, int lane) {
  t_clear(TI, lane);
  t_clear(TJ, lane);
  for (int64_t p = G.Io[k0] + lane; p < G.Io[k0 + 1]; p += 32) t_insert(TI, G.Is[p]);
  for (int64_t p = G.Jo[k0] + lane; p < G.Jo[k0 + 1]; p += 32) t_insert(TJ, G.Js[p]);
  __syncwarp();
  int64_t nI = G.Io[k0 + 1] - G.Io[k0], nJ = G.Jo[k0 + 1] - G.Jo[k0];
  int64_t sc = nI + nJ + 1, inbI = 0, inbJ = 0;   // scalar count c', union entries inside the block
  int l = 1;
  while (k0 + l < G.n && l + 1 <= G.max_size) {
    const int t = k0 + l;
    int64_t aI = 0, aJ = 0;                        // entries of I~_t / J~_t new to the unions
    for (int64_t p = G.Io[t] + lane; p < G.Io[t + 1]; p += 32) aI += 1 - t_find(TI, G.Is[p]);
    for (int64_t p = G.Jo[t] + lane; p < G.Jo[t + 1]; p += 32) aJ += 1 - t_find(TJ, G.Js[p]);
    aI = warp_sum64(aI);
    aJ = warp_sum64(aJ);
    const int iI = t_find(TI, t), iJ = t_find(TJ, t);   // t moves inside the block
    const int64_t r = nI + aI - (inbI + iI), s = nJ + aJ - (inbJ + iJ);
    const int64_t l1 = l + 1, f = (r + s + l1) * l1;
    const int64_t c2 = sc + (G.Io[t + 1] - G.Io[t]) + (G.Jo[t + 1] - G.Jo[t]) + 1;
    if (!(3 * f <= 4 * c2 || f <= c2 + 4 * l1)) break;
    __syncwarp();
    for (int64_t p = G.Io[t] + lane; p < G.Io[t + 1]; p += 32) t_insert(TI, G.Is[p]);
    for (int64_t p = G.Jo[t] + lane; p < G.Jo[t + 1]; p += 32) t_insert(TJ, G.Js[p]);
    __syncwarp();
    nI += aI; nJ += aJ; inbI += iI; inbJ += iJ; sc = c2;
    ++l;
  }
  return l;
}

__device__ __forceinline__ int64_t grow_bound(const GrowArgs &G, int k0) {
  const int e = min(k0 + G.max_size, G.n);
  return max(G.Io[e] - G.Io[k0], G.Jo[e] - G.Jo[k0]);
}

__global__ void __launch_bounds__(BT) grow_kernel(GrowArgs G) {
  extern __shared__ int32_t s_tab[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const Table TI{s_tab + (2 * w) * GROW_CAP, GROW_CAP - 1}, TJ{s_tab + (2 * w + 1) * GROW_CAP, GROW_CAP - 1};
  for (int k0 = blockIdx.x * BW + w; k0 < G.n; k0 += gridDim.x * BW) {
    const int64_t b = grow_bound(G, k0);
    if (2 * b > GROW_CAP) {
      if (lane == 0) {
        G.ovf_list[atomicAdd(G.ovf_n, 1)] = k0;
        atomicMax(G.ovf_max, (unsigned long long)b);
      }
      continue;
    }
    const int l = grow_block(G, k0, TI, TJ, lane);
    if (lane == 0) G.L[k0] = l;
    __syncwarp();
  }
}

__global__ void __launch_bounds__(BT) grow_big_kernel(GrowArgs G, int nlist, int32_t *region, uint32_t cap) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * BT + threadIdx.x) >> 5, nw = gridDim.x * BW;
  const Table TI{region + (int64_t)(2 * gw) * cap, cap - 1}, TJ{region + (int64_t)(2 * gw + 1) * cap, cap - 1};
  for (int x = gw; x < nlist; x += nw) {
    const int k0 = G.ovf_list[x];
    const int l = grow_block(G, k0, TI, TJ, lane);
    if (lane == 0) G.L[k0] = l;
    __syncwarp();
  }
}

// ---- chain resolution
__global__ void chain_table_kernel(int n, int ms, int nch, const int32_t *__restrict__ L, int32_t *T) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)nch * ms) return;
  const int c = (int)(id / ms), e = (int)(id % ms);
  const int64_t end = min((int64_t)(c + 1) * CH, (int64_t)n);
  int64_t s = (int64_t)c * CH + e;
  while (s < end) s += L[s];
  T[id] = (int32_t)(s - (int64_t)(c + 1) * CH);
}

// one thread: entry offset of every chunk (chunk 0 entered at 0)
__global__ void chain_compose_kernel(int nch, int ms, const int32_t *T, int32_t *entry) {
  int e = 0;
  for (int c = 0; c < nch; ++c) {
    entry[c] = e;
    e = T[(int64_t)c * ms + e];
  }
}

// pass 0: blocks starting in each chunk; pass 1: write their sizes at base[c]
__global__ void chain_walk_kernel(int n, int nch, const int32_t *__restrict__ L, const int32_t *entry, int64_t *cnt,
                                  const int64_t *base, int32_t *sizes) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nch) return;
  const int64_t end = min((int64_t)(c + 1) * CH, (int64_t)n);
  int64_t s = (int64_t)c * CH + entry[c], m = 0;
  while (s < end) {
    const int l = L[s];
    if (sizes) sizes[base[c] + m] = l;
    ++m;
    s += l;
  }
  if (!sizes) cnt[c] = m;
}

// ---- CSC
__global__ void csc_count_kernel(int n, const int64_t *rp, const int32_t *ci, unsigned long long *colcnt) {
  const int64_t nnz = rp[n];
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(colcnt + ci[p], 1ull);
}
__global__ void csc_fill_kernel(int n, const int64_t *rp, const int32_t *ci, const double *val,
                                unsigned long long *cur, int32_t *cr, double *cv, double *diag) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int i = gw; i < n; i += (gridDim.x * blockDim.x) >> 5) {
    if (lane == 0) diag[i] = 0.0;
    __syncwarp();
    for (int64_t p = rp[i] + lane; p < rp[i + 1]; p += 32) {
      const int32_t j = ci[p];
      const int64_t q = (int64_t)atomicAdd(cur + j, 1ull);
      cr[q] = i;
      cv[q] = val[p];
      if (j == i) diag[i] = val[p];
    }
  }
}

// ---- Ã = A(pm, pm) without sorting the rows (only sets are built from them)
__global__ void perm_len_kernel(int n, const int64_t *rp, const int32_t *pm, int64_t *len) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    len[i] = rp[pm[i] + 1] - rp[pm[i]];
}
__global__ void perm_rows_kernel(int n, const int64_t *rp, const int32_t *ci, const double *val, const int32_t *pm,
                                 const int32_t *ipm, const int64_t *nrp, int32_t *nci, double *nval) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int i = gw; i < n; i += (gridDim.x * blockDim.x) >> 5) {
    const int o = pm[i];
    const int64_t src = rp[o], dst = nrp[i], m = rp[o + 1] - src;
    for (int64_t x = lane; x < m; x += 32) {
      nci[dst + x] = ipm[ci[src + x]];
      nval[dst + x] = val[src + x];
    }
  }
}

// ---- exclusive scan of int64 (out has n+1 entries; out[n] = total)
__global__ void __launch_bounds__(256) scan_tiles_kernel(const int64_t *in, int64_t n, int64_t *part) {
  __shared__ int64_t sw[8];
  const int64_t b0 = (int64_t)blockIdx.x * SCAN_TILE;
  int64_t acc = 0;
  for (int x = 0; x < 8; ++x) {
    const int64_t i = b0 + threadIdx.x * 8 + x;
    if (i < n) acc += in[i];
  }
  acc = warp_sum64(acc);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t s = 0;
    for (int w = 0; w < 8; ++w) s += sw[w];
    part[blockIdx.x] = s;
  }
}
__global__ void scan_top_kernel(int64_t *part, int nb, int64_t *total) {
  if (threadIdx.x != 0) return;
  int64_t s = 0;
  for (int b = 0; b < nb; ++b) {
    const int64_t v = part[b];
    part[b] = s;
    s += v;
  }
  *total = s;
}
__global__ void __launch_bounds__(256) scan_apply_kernel(const int64_t *in, int64_t n, const int64_t *part,
                                                         int64_t *out) {
  __shared__ int64_t sw[8];
  const int64_t b0 = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * 8;
  int64_t v[8], acc = 0;
  for (int x = 0; x < 8; ++x) {
    v[x] = (b0 + x < n) ? in[b0 + x] : 0;
    acc += v[x];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t incl = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sw[w] = incl;
  __syncthreads();
  int64_t wbase = 0;
  for (int u = 0; u < w; ++u) wbase += sw[u];
  int64_t s = part[blockIdx.x] + wbase + incl - acc;
  for (int x = 0; x < 8; ++x) {
    if (b0 + x < n) out[b0 + x] = s;
    s += v[x];
  }
}

// ================================================================ cosine-based blocking
// Sec. 3.2 (R21): rows i, j with nz(a_i n a_j)^2 >= tau nz(a_i) nz(a_j)
// are grouped by Saad's greedy (rows in increasing order, an unassigned row takes the unassigned
// j > i that pass, up to max_size).  On the device: the pairs that pass (one warp per row i, the
// row of A A^T in a count hash), then the greedy as a fixed point: j is decided once every
// smaller neighbour is: it joins the first leader i among them whose earlier joiners leave room
// (its slot = 1 + their number), else it leads.  Decisions only read decided states, so the
// in-place rounds are deterministic; a one-thread sweep in index order finishes long chains.

// exact "count > mu + 2 sigma" (population sigma): n c - S1 > 0 and (n c - S1)^2 > 4 (n S2 - S1^2)
__device__ __forceinline__ int cos_heavy_dev(long long c, long long n, long long S1, long long S2) {
  const __int128 a = (__int128)n * c - S1;
  if (a <= 0) return 0;
  return a * a > (__int128)4 * ((__int128)n * S2 - (__int128)S1 * S1);
}

// S[0..3] = sum rc, sum rc^2, sum cc, sum cc^2 (integers: exact in any order)
__global__ void cos_stats_kernel(int n, const int64_t *rp, const unsigned long long *cc, unsigned long long *S) {
  unsigned long long a = 0, b = 0, c = 0, d = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long r = (unsigned long long)(rp[i + 1] - rp[i]), k = cc[i];
    a += r; b += r * r; c += k; d += k * k;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o); b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o); d += __shfl_xor_sync(0xffffffffu, d, o);
  }
  if ((threadIdx.x & 31) == 0) { atomicAdd(S, a); atomicAdd(S + 1, b); atomicAdd(S + 2, c); atomicAdd(S + 3, d); }
}

// ignore flags; kept-column counts (for the kept CSC) and nz(a_i) over kept columns
__global__ void cos_flags_kernel(int n, const int64_t *rp, const int32_t *ci, const unsigned long long *cc,
                                 const unsigned long long *S, uint8_t *rign, uint8_t *cign, int64_t *kcnt,
                                 int64_t *nz) {
  const long long S1r = (long long)S[0], S2r = (long long)S[1], S1c = (long long)S[2], S2c = (long long)S[3];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    rign[i] = (uint8_t)cos_heavy_dev(rp[i + 1] - rp[i], n, S1r, S2r);
    const int ig = cos_heavy_dev((long long)cc[i], n, S1c, S2c);
    cign[i] = (uint8_t)ig;
    kcnt[i] = ig ? 0 : (int64_t)cc[i];
  }
}
__global__ void cos_nz_kernel(int n, const int64_t *rp, const int32_t *ci, const uint8_t *cign, int64_t *nz) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int i = gw; i < n; i += (gridDim.x * blockDim.x) >> 5) {
    int64_t c = 0;
    for (int64_t p = rp[i] + lane; p < rp[i + 1]; p += 32) c += !cign[ci[p]];
    c = warp_sum64(c);
    if (lane == 0) nz[i] = c;
  }
}
__global__ void cos_csc_kernel(int n, const int64_t *rp, const int32_t *ci, const uint8_t *cign,
                               unsigned long long *cur, int32_t *cr) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int i = gw; i < n; i += (gridDim.x * blockDim.x) >> 5)
    for (int64_t p = rp[i] + lane; p < rp[i + 1]; p += 32) {
      const int32_t c = ci[p];
      if (!cign[c]) cr[atomicAdd(cur + c, 1ull)] = i;
    }
}

struct CosArgs {
  int n;
  const int64_t *rp; const int32_t *ci;     // A
  const int64_t *cp; const int32_t *cr;     // kept columns
  const uint8_t *rign, *cign;
  const int64_t *nz;
  double tau;
};

__device__ __forceinline__ int64_t cos_bound(const CosArgs &C, int i, int lane) {
  int64_t b = 0;
  for (int64_t p = C.rp[i] + lane; p < C.rp[i + 1]; p += 32) {
    const int32_t c = C.ci[p];
    if (!C.cign[c]) b += C.cp[c + 1] - C.cp[c];
  }
  return warp_sum64(b);
}

// row i of A A^T (j > i, kept rows) in T (keys) / V (counts), both cleared.  With a limit
// (optimistic shared-memory attempt) the distinct keys are counted in *nkeys and the build
// stops once they reach the limit (<= half the table, overshoot < 32): returns 0 then.
__device__ int cos_row(const CosArgs &C, int i, Table T, int32_t *V, int lane, int *nkeys, int limit) {
  volatile int *vk = nkeys;
  for (int64_t p = C.rp[i]; p < C.rp[i + 1]; ++p) {
    const int32_t c = C.ci[p];
    if (C.cign[c]) continue;
    for (int64_t x = C.cp[c] + lane; x < C.cp[c + 1]; x += 32) {
      if (limit && *vk >= limit) break;
      const int32_t j = C.cr[x];
      if (j <= i || C.rign[j]) continue;
      uint32_t s = slot0(j, T.mask);
      while (true) {
        const int32_t old = atomicCAS(T.t + s, -1, j);
        if (old == -1) { if (limit) atomicAdd(nkeys, 1); break; }
        if (old == j) break;
        s = (s + 1) & T.mask;
      }
      atomicAdd(V + s, 1);
    }
    __syncwarp();
    if (limit && *vk >= limit) return 0;
  }
  __syncwarp();
  return 1;
}

// passing j of the table, written to out (arbitrary order); returns their number
__device__ int cos_emit(const CosArgs &C, int i, Table T, const int32_t *V, int32_t *out, int lane) {
  const double ni = (double)C.nz[i];
  int base = 0;
  for (uint32_t s0 = 0; s0 <= T.mask; s0 += 32) {
    const int32_t j = T.t[s0 + lane];
    bool ok = false;
    if (j >= 0) {
      const double c = (double)V[s0 + lane];
      ok = c * c >= C.tau * (ni * (double)C.nz[j]);
    }
    const unsigned b = __ballot_sync(0xffffffffu, ok);
    if (ok && out) out[base + __popc(b & ((1u << lane) - 1u))] = j;
    base += __popc(b);
  }
  return base;
}

// src[0..m) distinct -> dst ascending (rank sort, one warp)
__device__ void rank_sort_copy(const int32_t *src, int32_t *dst, int m, int lane) {
  for (int x = lane; x < m; x += 32) {
    const int32_t v = src[x];
    int r = 0;
    for (int y = 0; y < m; ++y) r += src[y] < v;
    dst[r] = v;
  }
}

struct CosOut {
  int64_t *cnt; const int64_t *off; int32_t *tmp; int32_t *up;
  int32_t *ovf_list; int *ovf_n; unsigned long long *ovf_max;
};

// returns 0 if the optimistic attempt (limit > 0) overflowed
template <bool WRITE>
__device__ int cos_one(const CosArgs &C, const CosOut &O, int i, Table T, int32_t *V, int lane, int *nkeys, int limit) {
  t_clear(T, lane);
  for (uint32_t x = lane; x <= T.mask; x += 32) V[x] = 0;
  if (lane == 0 && nkeys) *nkeys = 0;
  __syncwarp();
  if (!cos_row(C, i, T, V, lane, nkeys, limit)) return 0;
  if (!WRITE) {
    const int m = cos_emit(C, i, T, V, nullptr, lane);
    if (lane == 0) O.cnt[i] = m;
  } else {
    const int m = cos_emit(C, i, T, V, O.tmp + O.off[i], lane);
    __syncwarp();
    rank_sort_copy(O.tmp + O.off[i], O.up + O.off[i], m, lane);
  }
  __syncwarp();
  return 1;
}

// rows whose candidate bound exceeds half the shared table are tried optimistically (most of
// their candidates repeat); a row whose distinct keys do not fit goes to the global tables
template <bool WRITE>
__global__ void __launch_bounds__(BT) cos_pairs_kernel(CosArgs C, CosOut O) {
  extern __shared__ int32_t s_tab[];
  __shared__ int s_nkeys[BW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int CAP = SET_CAP / 2;
  const Table T{s_tab + w * 2 * CAP, CAP - 1};
  int32_t *V = s_tab + w * 2 * CAP + CAP;
  for (int i = blockIdx.x * BW + w; i < C.n; i += gridDim.x * BW) {
    if (C.rign[i] || C.nz[i] == 0) { if (!WRITE && lane == 0) O.cnt[i] = 0; continue; }
    const int64_t b = cos_bound(C, i, lane);
    const int limit = 2 * b > CAP ? CAP / 2 : 0;
    if (!cos_one<WRITE>(C, O, i, T, V, lane, s_nkeys + w, limit)) {
      if (!WRITE && lane == 0) { O.ovf_list[atomicAdd(O.ovf_n, 1)] = i; atomicMax(O.ovf_max, (unsigned long long)b); }
      __syncwarp();
    }
  }
}
template <bool WRITE>
__global__ void __launch_bounds__(BT) cos_pairs_big_kernel(CosArgs C, CosOut O, int nlist, int32_t *region, uint32_t cap) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * BT + threadIdx.x) >> 5, nw = gridDim.x * BW;
  const Table T{region + (int64_t)gw * 2 * cap, cap - 1};
  int32_t *V = region + (int64_t)gw * 2 * cap + cap;
  for (int x = gw; x < nlist; x += nw) cos_one<WRITE>(C, O, O.ovf_list[x], T, V, lane, nullptr, 0);
}

// lower lists: low(j) = { i < j : j in up(i) }
__global__ void cos_low_count_kernel(int n, const int64_t *uoff, const int32_t *up, unsigned long long *lcnt) {
  const int64_t tot = uoff[n];
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < tot; p += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(lcnt + up[p], 1ull);
}
__global__ void cos_low_fill_kernel(int n, const int64_t *uoff, const int32_t *up, unsigned long long *cur, int32_t *tmp) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int i = gw; i < n; i += (gridDim.x * blockDim.x) >> 5)
    for (int64_t p = uoff[i] + lane; p < uoff[i + 1]; p += 32) tmp[atomicAdd(cur + up[p], 1ull)] = i;
}
__global__ void cos_low_sort_kernel(int n, const int64_t *loff, const int32_t *tmp, int32_t *low) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int j = gw; j < n; j += (gridDim.x * blockDim.x) >> 5)
    rank_sort_copy(tmp + loff[j], low + loff[j], (int)(loff[j + 1] - loff[j]), lane);
}

struct CosGreedy {
  int n, max_size;
  const int64_t *uoff; const int32_t *up;    // up(i) ascending
  const int64_t *loff; const int32_t *low;   // low(j) ascending
  int32_t *state;                            // -2 undecided, -1 leader, >= 0 leader it joined
  int32_t *slot;                             // rank inside the group
  int *progress;
};

// one decision attempt for j (undecided); returns 1 if decided
__device__ int cos_decide(const CosGreedy &G, int j) {
  volatile int32_t *st = G.state;
  for (int64_t p = G.loff[j]; p < G.loff[j + 1]; ++p) {
    const int i = G.low[p];
    const int si = st[i];
    if (si == -2) return 0;
    if (si >= 0) continue;                   // i joined a group: it claims nobody
    int cnt = 0;                             // earlier joiners of i
    for (int64_t x = G.uoff[i]; x < G.uoff[i + 1]; ++x) {
      const int jj = G.up[x];
      if (jj >= j) break;
      const int sj = st[jj];
      if (sj == -2) return 0;
      cnt += (sj == i);
    }
    if (cnt < G.max_size - 1) {
      G.slot[j] = cnt + 1;
      __threadfence();
      st[j] = i;
      return 1;
    }
  }
  G.slot[j] = 0;
  __threadfence();
  st[j] = -1;
  return 1;
}

__global__ void cos_init_kernel(int n, int32_t *state) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) state[j] = -2;
}

__global__ void cos_round_kernel(CosGreedy G) {
  int done = 0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < G.n; j += gridDim.x * blockDim.x)
    if (((volatile int32_t *)G.state)[j] == -2) done += cos_decide(G, j);
  if (done) atomicAdd(G.progress, done);
}
__global__ void cos_undecided_kernel(int n, const int32_t *state, int64_t *flag) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) flag[j] = state[j] == -2;
}
__global__ void cos_list_kernel(int n, const int64_t *flag, const int64_t *pos, int32_t *list) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    if (flag[j]) list[pos[j]] = j;
}
// one thread over the undecided rows in index order: every dependency is decided first
__global__ void cos_sweep_kernel(CosGreedy G, const int32_t *list, const int64_t *m) {
  for (int64_t x = 0; x < *m; ++x) cos_decide(G, list[x]);
}

// groups: leaders numbered in index order; size = 1 + joiners; q[gstart[g] + slot[j]] = j
__global__ void cos_leader_kernel(int n, const int32_t *state, int64_t *lead) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) lead[j] = state[j] == -1;
}
__global__ void cos_size_kernel(int n, const int32_t *state, const int64_t *gid, unsigned long long *gsize) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    atomicAdd(gsize + gid[state[j] == -1 ? j : state[j]], 1ull);
}
__global__ void cos_place_kernel(int n, const int32_t *state, const int32_t *slot, const int64_t *gid,
                                 const int64_t *gstart, int32_t *q) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int L = state[j] == -1 ? j : state[j];
    q[gstart[gid[L]] + slot[j]] = j;
  }
}
__global__ void cos_sizes_kernel(int nb, const unsigned long long *gsize, int32_t *sizes) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < nb; g += gridDim.x * blockDim.x) sizes[g] = (int32_t)gsize[g];
}

// ---------------------------------------------------------------- host orchestration
namespace {
// scratch from the stream-ordered allocator: repeated calls reuse the device's pool instead of
// paying cudaMalloc / cudaFree (which synchronise) for GB-sized arrays
struct Pool {
  std::vector<void *> ptrs;
  cudaStream_t st;
  cudaError_t err = cudaSuccess;
  explicit Pool(cudaStream_t s) : st(s) {
    static bool once = false;
    if (!once) {
      int dev = 0;
      cudaMemPool_t mp;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess) {
        uint64_t keep = (uint64_t)8 << 30;          // retain up to 8 GiB between calls
        cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      once = true;
    }
  }
  template <class T>
  T *get(int64_t count) {
    void *p = nullptr;
    if (err != cudaSuccess) return nullptr;
    err = cudaMallocAsync(&p, (size_t)(count > 0 ? count : 1) * sizeof(T), st);
    if (err != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return (T *)p;
  }
  ~Pool() {
    for (void *p : ptrs) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
  }
};

cudaError_t scan_excl(const int64_t *in, int64_t n, int64_t *out, Pool &pool, cudaStream_t st) {
  const int nb = (int)((n + SCAN_TILE - 1) / SCAN_TILE);
  int64_t *part = pool.get<int64_t>(nb > 0 ? nb : 1);
  if (!part) return pool.err;
  if (nb > 0) scan_tiles_kernel<<<nb, 256, 0, st>>>(in, n, part);
  scan_top_kernel<<<1, 32, 0, st>>>(part, nb, out + n);
  if (nb > 0) scan_apply_kernel<<<nb, 256, 0, st>>>(in, n, part, out);
  return cudaGetLastError();
}

uint32_t pow2_at_least(int64_t x) {
  uint32_t c = 64;
  while ((int64_t)c < x && c < (1u << 30)) c <<= 1;
  return c;
}

// builds one side's sets: offsets off[n+1], entries *sets
template <bool LOWER>
cudaError_t build_sets(const EstArgs &E, int grid, int sms, int64_t **off_o, int32_t **sets_o, int *launches,
                       Pool &pool, cudaStream_t st) {
  const int n = E.n;
  int64_t *cnt = pool.get<int64_t>(n), *off = pool.get<int64_t>(n + 1);
  int32_t *list = pool.get<int32_t>(n);
  int *d_novf = pool.get<int>(1);
  unsigned long long *d_max = pool.get<unsigned long long>(1);
  if (pool.err != cudaSuccess) return pool.err;
  cudaMemsetAsync(d_novf, 0, sizeof(int), st);
  cudaMemsetAsync(d_max, 0, sizeof(unsigned long long), st);
  SetOut O{cnt, off, nullptr, list, d_novf, d_max};
  const size_t smem = (size_t)BW * SET_CAP * sizeof(int32_t);
  sets_kernel<LOWER, false><<<grid, BT, smem, st>>>(E, O);
  ++*launches;
  int novf = 0;
  unsigned long long mx = 0;
  cudaMemcpyAsync(&novf, d_novf, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&mx, d_max, sizeof(mx), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  int32_t *region = nullptr;
  uint32_t cap = 0;
  int bgrid = 0;
  if (novf > 0) {
    cap = pow2_at_least(2 * (int64_t)mx);
    int64_t warps = ((int64_t)1 << 28) / cap;            // <= 1 GiB of tables
    warps = warps < 1 ? 1 : warps;
    warps = warps > (int64_t)sms * BW * 4 ? (int64_t)sms * BW * 4 : warps;
    warps = warps > novf ? novf : warps;
    bgrid = (int)((warps + BW - 1) / BW);
    region = pool.get<int32_t>((int64_t)bgrid * BW * cap);
    if (!region) return pool.err;
    sets_big_kernel<LOWER, false><<<bgrid, BT, 0, st>>>(E, O, novf, region, cap);
    ++*launches;
  }
  if ((e = scan_excl(cnt, n, off, pool, st)) != cudaSuccess) return e;
  *launches += 3;
  int64_t total = 0;
  cudaMemcpyAsync(&total, off + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  int32_t *sets = pool.get<int32_t>(total);
  if (!sets) return pool.err;
  O.out = sets;
  sets_kernel<LOWER, true><<<grid, BT, smem, st>>>(E, O);
  ++*launches;
  if (novf > 0) {
    sets_big_kernel<LOWER, true><<<bgrid, BT, 0, st>>>(E, O, novf, region, cap);
    ++*launches;
  }
  *off_o = off;
  *sets_o = sets;
  return cudaGetLastError();
}
}  // namespace

// Runs the whole estimate on the permuted CSR already on the device.  h_sizes (HOST,
// capacity n) receives the block sizes, *nblocks their number; *launches the kernels run.
// pm / ipm (device, may be NULL = identity): the estimate runs on Ã = A(pm, pm).
extern "C" cudaError_t bilu_ilu1_run(int n, const int64_t *rp, const int32_t *ci, const double *val,
                                     const int32_t *pm, const int32_t *ipm, double tau, int max_size, int sms,
                                     cudaStream_t st, int32_t *h_sizes, int32_t *nblocks, int *launches) {
  Pool pool(st);
  *launches = 0;
  int64_t nnz = 0;
  cudaError_t e = cudaMemcpyAsync(&nnz, rp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess || (e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (pm) {
    int64_t *len = pool.get<int64_t>(n), *nrp = pool.get<int64_t>(n + 1);
    int32_t *nci = pool.get<int32_t>(nnz);
    double *nval = pool.get<double>(nnz);
    if (pool.err != cudaSuccess) return pool.err;
    perm_len_kernel<<<sms * 4, 256, 0, st>>>(n, rp, pm, len);
    if ((e = scan_excl(len, n, nrp, pool, st)) != cudaSuccess) return e;
    perm_rows_kernel<<<sms * 8, 256, 0, st>>>(n, rp, ci, val, pm, ipm, nrp, nci, nval);
    *launches += 5;
    rp = nrp; ci = nci; val = nval;
  }
  // 1. CSC
  unsigned long long *colcnt = pool.get<unsigned long long>(n);
  int64_t *cp = pool.get<int64_t>(n + 1);
  int32_t *cr = pool.get<int32_t>(nnz);
  double *cv = pool.get<double>(nnz), *diag = pool.get<double>(n);
  if (pool.err != cudaSuccess) return pool.err;
  cudaMemsetAsync(colcnt, 0, sizeof(unsigned long long) * n, st);
  const int egrid = sms * 8;
  csc_count_kernel<<<egrid, 256, 0, st>>>(n, rp, ci, colcnt);
  if ((e = scan_excl((const int64_t *)colcnt, n, cp, pool, st)) != cudaSuccess) return e;
  cudaMemcpyAsync(colcnt, cp, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st);
  csc_fill_kernel<<<egrid, 256, 0, st>>>(n, rp, ci, val, colcnt, cr, cv, diag);
  *launches += 5;
  const EstArgs E{n, rp, ci, val, cp, cr, cv, diag, tau};
  // 2. sets
  static bool attr = false;
  if (!attr) {
    const int s1 = BW * SET_CAP * (int)sizeof(int32_t), s2 = 2 * BW * GROW_CAP * (int)sizeof(int32_t);
    cudaFuncSetAttribute(sets_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1);
    cudaFuncSetAttribute(sets_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1);
    cudaFuncSetAttribute(sets_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1);
    cudaFuncSetAttribute(sets_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1);
    cudaFuncSetAttribute(grow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, s2);
    attr = true;
  }
  const int grid = sms * 3;
  int64_t *Io = nullptr, *Jo = nullptr;
  int32_t *Is = nullptr, *Js = nullptr;
  if ((e = build_sets<true>(E, grid, sms, &Io, &Is, launches, pool, st)) != cudaSuccess) return e;
  if ((e = build_sets<false>(E, grid, sms, &Jo, &Js, launches, pool, st)) != cudaSuccess) return e;
  // 3. speculative growth
  int32_t *L = pool.get<int32_t>(n), *list = pool.get<int32_t>(n);
  int *d_novf = pool.get<int>(1);
  unsigned long long *d_max = pool.get<unsigned long long>(1);
  if (pool.err != cudaSuccess) return pool.err;
  cudaMemsetAsync(d_novf, 0, sizeof(int), st);
  cudaMemsetAsync(d_max, 0, sizeof(unsigned long long), st);
  GrowArgs G{n, max_size, Io, Is, Jo, Js, L, list, d_novf, d_max};
  grow_kernel<<<grid, BT, (size_t)2 * BW * GROW_CAP * sizeof(int32_t), st>>>(G);
  ++*launches;
  int novf = 0;
  unsigned long long mx = 0;
  cudaMemcpyAsync(&novf, d_novf, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&mx, d_max, sizeof(mx), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (novf > 0) {
    const uint32_t cap = pow2_at_least(2 * (int64_t)mx);
    int64_t warps = ((int64_t)1 << 27) / cap;
    warps = warps < 1 ? 1 : warps;
    warps = warps > (int64_t)sms * BW * 4 ? (int64_t)sms * BW * 4 : warps;
    warps = warps > novf ? novf : warps;
    const int bgrid = (int)((warps + BW - 1) / BW);
    int32_t *region = pool.get<int32_t>((int64_t)bgrid * BW * 2 * cap);
    if (!region) return pool.err;
    grow_big_kernel<<<bgrid, BT, 0, st>>>(G, novf, region, cap);
    ++*launches;
  }
  // 4. chain
  const int nch = (n + CH - 1) / CH;
  int32_t *T = pool.get<int32_t>((int64_t)nch * max_size), *entry = pool.get<int32_t>(nch);
  int64_t *ccnt = pool.get<int64_t>(nch), *cbase = pool.get<int64_t>(nch + 1);
  int32_t *sizes = pool.get<int32_t>(n);
  if (pool.err != cudaSuccess) return pool.err;
  const int64_t nt = (int64_t)nch * max_size;
  chain_table_kernel<<<(int)((nt + 255) / 256), 256, 0, st>>>(n, max_size, nch, L, T);
  chain_compose_kernel<<<1, 1, 0, st>>>(nch, max_size, T, entry);
  chain_walk_kernel<<<(nch + 255) / 256, 256, 0, st>>>(n, nch, L, entry, ccnt, nullptr, nullptr);
  if ((e = scan_excl(ccnt, nch, cbase, pool, st)) != cudaSuccess) return e;
  chain_walk_kernel<<<(nch + 255) / 256, 256, 0, st>>>(n, nch, L, entry, nullptr, cbase, sizes);
  *launches += 7;
  int64_t nb = 0;
  cudaMemcpyAsync(&nb, cbase + nch, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (nb < 1 || nb > n) return cudaErrorUnknown;
  cudaMemcpyAsync(h_sizes, sizes, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  *nblocks = (int32_t)nb;
  return cudaGetLastError();
}

// Cosine-based blocking of the pattern of A (device CSR).  h_q (HOST, n): the grouping
// permutation (new -> old); h_sizes (HOST, capacity n): group sizes; *nblocks their number.
extern "C" cudaError_t bilu_cosine_run(int n, const int64_t *rp, const int32_t *ci, double tau, int max_size, int sms,
                                       cudaStream_t st, int32_t *h_q, int32_t *h_sizes, int32_t *nblocks,
                                       int *launches, int *rounds) {
  Pool pool(st);
  *launches = 0;
  *rounds = 0;
  int64_t nnz = 0;
  cudaError_t e = cudaMemcpyAsync(&nnz, rp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess || (e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  const int egrid = sms * 8;
  unsigned long long *cc = pool.get<unsigned long long>(n), *S = pool.get<unsigned long long>(4);
  uint8_t *rign = pool.get<uint8_t>(n), *cign = pool.get<uint8_t>(n);
  int64_t *kcnt = pool.get<int64_t>(n), *nz = pool.get<int64_t>(n), *cp = pool.get<int64_t>(n + 1);
  int32_t *cr = pool.get<int32_t>(nnz);
  if (pool.err != cudaSuccess) return pool.err;
  cudaMemsetAsync(cc, 0, sizeof(unsigned long long) * n, st);
  cudaMemsetAsync(S, 0, sizeof(unsigned long long) * 4, st);
  csc_count_kernel<<<egrid, 256, 0, st>>>(n, rp, ci, cc);
  cos_stats_kernel<<<egrid, 256, 0, st>>>(n, rp, cc, S);
  cos_flags_kernel<<<egrid, 256, 0, st>>>(n, rp, ci, cc, S, rign, cign, kcnt, nz);
  cos_nz_kernel<<<egrid, 256, 0, st>>>(n, rp, ci, cign, nz);
  if ((e = scan_excl(kcnt, n, cp, pool, st)) != cudaSuccess) return e;
  cudaMemcpyAsync(cc, cp, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st);
  cos_csc_kernel<<<egrid, 256, 0, st>>>(n, rp, ci, cign, cc, cr);
  *launches += 8;
  const CosArgs C{n, rp, ci, cp, cr, rign, cign, nz, tau};
  // similar pairs: count, scan, write (+ global-table fallback)
  int64_t *cnt = pool.get<int64_t>(n), *uoff = pool.get<int64_t>(n + 1);
  int32_t *list = pool.get<int32_t>(n);
  int *d_novf = pool.get<int>(1);
  unsigned long long *d_max = pool.get<unsigned long long>(1);
  if (pool.err != cudaSuccess) return pool.err;
  cudaMemsetAsync(d_novf, 0, sizeof(int), st);
  cudaMemsetAsync(d_max, 0, sizeof(unsigned long long), st);
  CosOut O{cnt, uoff, nullptr, nullptr, list, d_novf, d_max};
  static bool attr = false;
  const int smem = BW * SET_CAP * (int)sizeof(int32_t);
  if (!attr) {
    cudaFuncSetAttribute(cos_pairs_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(cos_pairs_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const int grid = sms * 3;
  cos_pairs_kernel<false><<<grid, BT, smem, st>>>(C, O);
  ++*launches;
  int novf = 0;
  unsigned long long mx = 0;
  cudaMemcpyAsync(&novf, d_novf, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&mx, d_max, sizeof(mx), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  int32_t *region = nullptr;
  uint32_t cap = 0;
  int bgrid = 0;
  if (novf > 0) {
    cap = pow2_at_least(2 * (int64_t)mx);
    int64_t warps = ((int64_t)1 << 27) / cap;
    warps = warps < 1 ? 1 : warps;
    warps = warps > (int64_t)sms * BW * 4 ? (int64_t)sms * BW * 4 : warps;
    warps = warps > novf ? novf : warps;
    bgrid = (int)((warps + BW - 1) / BW);
    region = pool.get<int32_t>((int64_t)bgrid * BW * 2 * cap);
    if (!region) return pool.err;
    cos_pairs_big_kernel<false><<<bgrid, BT, 0, st>>>(C, O, novf, region, cap);
    ++*launches;
  }
  if ((e = scan_excl(cnt, n, uoff, pool, st)) != cudaSuccess) return e;
  *launches += 3;
  int64_t npairs = 0;
  cudaMemcpyAsync(&npairs, uoff + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  int32_t *tmp = pool.get<int32_t>(npairs), *up = pool.get<int32_t>(npairs), *low = pool.get<int32_t>(npairs);
  int64_t *loff = pool.get<int64_t>(n + 1);
  unsigned long long *lcnt = pool.get<unsigned long long>(n);
  if (pool.err != cudaSuccess) return pool.err;
  O.tmp = tmp; O.up = up;
  cos_pairs_kernel<true><<<grid, BT, smem, st>>>(C, O);
  ++*launches;
  if (novf > 0) { cos_pairs_big_kernel<true><<<bgrid, BT, 0, st>>>(C, O, novf, region, cap); ++*launches; }
  cudaMemsetAsync(lcnt, 0, sizeof(unsigned long long) * n, st);
  cos_low_count_kernel<<<egrid, 256, 0, st>>>(n, uoff, up, lcnt);
  if ((e = scan_excl((const int64_t *)lcnt, n, loff, pool, st)) != cudaSuccess) return e;
  cudaMemcpyAsync(lcnt, loff, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st);
  cos_low_fill_kernel<<<egrid, 256, 0, st>>>(n, uoff, up, lcnt, tmp);
  cos_low_sort_kernel<<<egrid, 256, 0, st>>>(n, loff, tmp, low);
  *launches += 6;
  // greedy fixed point
  int32_t *state = pool.get<int32_t>(n), *slot = pool.get<int32_t>(n);
  int *progress = pool.get<int>(1);
  if (pool.err != cudaSuccess) return pool.err;
  cos_init_kernel<<<egrid, 256, 0, st>>>(n, state);
  ++*launches;
  const CosGreedy G{n, max_size, uoff, up, loff, low, state, slot, progress};
  int64_t decided = 0;
  const int rgrid = (int)(((int64_t)n + 255) / 256 < (int64_t)sms * 16 ? ((int64_t)n + 255) / 256 : (int64_t)sms * 16);
  while (decided < n) {
    cudaMemsetAsync(progress, 0, sizeof(int), st);
    cos_round_kernel<<<rgrid, 256, 0, st>>>(G);
    ++*launches;
    ++*rounds;
    int pr = 0;
    cudaMemcpyAsync(&pr, progress, sizeof(int), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    decided += pr;
    if (decided < n && (*rounds >= 64 || pr < (n - decided) / 64)) {   // long chains: finish in order
      int64_t *flag = pool.get<int64_t>(n), *pos = pool.get<int64_t>(n + 1);
      int32_t *ulist = pool.get<int32_t>(n);
      if (pool.err != cudaSuccess) return pool.err;
      cos_undecided_kernel<<<egrid, 256, 0, st>>>(n, state, flag);
      if ((e = scan_excl(flag, n, pos, pool, st)) != cudaSuccess) return e;
      cos_list_kernel<<<egrid, 256, 0, st>>>(n, flag, pos, ulist);
      cos_sweep_kernel<<<1, 1, 0, st>>>(G, ulist, pos + n);
      *launches += 6;
      break;
    }
  }
  // groups
  int64_t *lead = pool.get<int64_t>(n), *gid = pool.get<int64_t>(n + 1);
  if (pool.err != cudaSuccess) return pool.err;
  cos_leader_kernel<<<egrid, 256, 0, st>>>(n, state, lead);
  if ((e = scan_excl(lead, n, gid, pool, st)) != cudaSuccess) return e;
  int64_t nb = 0;
  cudaMemcpyAsync(&nb, gid + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (nb < 1 || nb > n) return cudaErrorUnknown;
  unsigned long long *gsize = pool.get<unsigned long long>(nb);
  int64_t *gstart = pool.get<int64_t>(nb + 1);
  int32_t *q = pool.get<int32_t>(n), *sizes = pool.get<int32_t>(nb);
  if (pool.err != cudaSuccess) return pool.err;
  cudaMemsetAsync(gsize, 0, sizeof(unsigned long long) * nb, st);
  cos_size_kernel<<<egrid, 256, 0, st>>>(n, state, gid, gsize);
  if ((e = scan_excl((const int64_t *)gsize, nb, gstart, pool, st)) != cudaSuccess) return e;
  cos_place_kernel<<<egrid, 256, 0, st>>>(n, state, slot, gid, gstart, q);
  cos_sizes_kernel<<<egrid, 256, 0, st>>>((int)nb, gsize, sizes);
  *launches += 8;
  cudaMemcpyAsync(h_q, q, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(h_sizes, sizes, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  *nblocks = (int32_t)nb;
  return cudaGetLastError();
}

}  // namespace bilu
