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
// returns the set size.  PAPER.md:1183-1198; the products are the oracle's (R20).
template <bool LOWER>
__device__ int build_set(const EstArgs &E, int k, Table T, int lane) {
  const int64_t *P = LOWER ? E.cp : E.rp;
  const int32_t *X = LOWER ? E.cr : E.ci;
  const double *V = LOWER ? E.cv : E.val;
  const double akk = E.diag[k];
  const double thr = E.tau * fabs(akk);
  int64_t cnt = 0;
  for (int64_t p = P[k] + lane; p < P[k + 1]; p += 32) {
    const int32_t x = X[p];
    if (x > k && fabs(V[p]) >= thr) cnt += t_insert(T, x);
  }
  for (int64_t p = P[k]; p < P[k + 1]; ++p) {          // j < k with a_jk != 0 (resp. i < k, a_ki != 0)
    const int32_t j = X[p];
    if (j >= k) continue;
    const double ajk = V[p];
    const double thr2 = E.tau * fabs(E.diag[j] * akk);
    for (int64_t q = P[j] + lane; q < P[j + 1]; q += 32) {
      const int32_t x = X[q];
      if (x > k && fabs(V[q] * ajk) >= thr2) cnt += t_insert(T, x);
    }
  }
  __syncwarp();
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

template <bool LOWER, bool WRITE>
__global__ void __launch_bounds__(BT) sets_kernel(EstArgs E, SetOut O) {
  extern __shared__ int32_t s_tab[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const Table T{s_tab + w * SET_CAP, SET_CAP - 1};
  for (int k = blockIdx.x * BW + w; k < E.n; k += gridDim.x * BW) {
    const int64_t b = set_bound<LOWER>(E, k, lane);
    if (2 * b > SET_CAP) {
      if (!WRITE && lane == 0) {
        O.ovf_list[atomicAdd(O.ovf_n, 1)] = k;
        atomicMax(O.ovf_max, (unsigned long long)b);
      }
      continue;
    }
    t_clear(T, lane);
    const int c = build_set<LOWER>(E, k, T, lane);
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

// ---------------------------------------------------------------- host orchestration
namespace {
struct Pool {
  std::vector<void *> ptrs;
  cudaError_t err = cudaSuccess;
  template <class T>
  T *get(int64_t count) {
    void *p = nullptr;
    if (err != cudaSuccess) return nullptr;
    err = cudaMalloc(&p, (size_t)(count > 0 ? count : 1) * sizeof(T));
    if (err != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return (T *)p;
  }
  ~Pool() {
    for (void *p : ptrs) cudaFree(p);
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
  Pool pool;
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

}  // namespace bilu
