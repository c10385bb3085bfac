// bilu_merge.cu -- progressive aggregation (Sec. 3.5) as a
// post-pass over the finished (unmerged) factors.
//
// Merging k-1 into k leaves the operator L·P·U unchanged (identity displayed at
// PAPER.md:1348-1387), so the values of every later block are the same whether
// the merge happens during or after the factorization;
// the decisions only depend on index sets ("checking the union of nonzero index
// sets ignoring any cancellations").  The sequential scan of
// the paper is made parallel by evaluating the test for every (aggregate start
// a, block k) pair that max_block allows (merge_test_kernel), after which the
// scan itself is a walk over bitmasks (merge_scan_kernel).  The merged factors
// of a whole run a..k are then formed in closed form (merge_arith_kernel):
//   L^ = L_{>,agg} L_aa^{-1},  Ũ^ = L_aa Ũ_{agg,>},  D^ = U_aa^{-1} D_agg L_aa^{-1}
// which is the paper's pairwise update applied k-a times (DESIGN.md derives it).
#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>

#include "bilu_internal.h"

namespace bilu {

constexpr int MT = 256;
constexpr int MW = MT / 32;

// MergeArgs: see bilu_internal.h

// ----------------------------------------------------------- CTA helpers
__device__ int m_scan(int *a, int n, int *s_tmp) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (n + MT - 1) / MT;
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
    for (int w = 0; w < MW; ++w) { int t = s_tmp[w]; s_tmp[w] = acc; acc += t; }
    s_tmp[MW] = acc;
  }
  __syncthreads();
  int run = s_tmp[wid] + x - sum;
  for (int i = lo; i < hi; ++i) { int t = a[i]; a[i] = run; run += t; }
  int total = s_tmp[MW];
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

// the test of Sec. 3.5: mu = p(p+r+s+r'+s') + q(q+t+t'), nu = (p+q)(p+q+u+v);
// merge iff nu <= 1.2 mu (exactly: 5 nu <= 6 mu) or nu <= mu + 2(p+q); p+q <= max_block
__device__ __forceinline__ bool agg_test(long long p, long long q, long long r, long long s, long long t,
                                         long long r2, long long s2, long long t2, long long u, long long v,
                                         long long max_block) {
  if (p + q > max_block) return false;
  long long mu = p * (p + r + s + r2 + s2) + q * (q + t + t2);
  long long nu = (p + q) * (p + q + u + v);
  return (5 * nu <= 6 * mu) || (nu <= mu + 2 * (p + q));
}

// ---------------------------------------------------------------- M1: test
// For block k and every candidate start a = k-d (d = 1..W), compute r,s,u (rows)
// and r',s',v (cols) of the aggregate (a..k-1) against k from the histogram of
// dmin(x) = distance k-j of the closest member j whose kept set contains x.
__device__ void count_side(const MergeArgs &M, int k, int W, bool rows, int *keys, int cap,
                           int *hist /* 3*(W+2) */, int *cnt /* W+2 */, int *s_tmp, int &t_out) {
  const int tid = threadIdx.x;
  const int s_k = M.bstart[k], e_k = M.bstart[k + 1];
  const int32_t *idx = rows ? M.Lidx : M.Uidx;
  const int64_t *off = rows ? M.Lrow_off : M.Ucol_off;
  const int32_t *len = rows ? M.Lm : M.Uc;
  // members j = k-W .. k (d = k - j); suffix >= s_k
  for (int d = tid; d <= W; d += MT) {
    int j = k - d;
    const int32_t *L = idx + off[j];
    int m = len[j];
    int p0 = 0, p1 = m;
    while (p0 < p1) { int mid = (p0 + p1) >> 1; if (L[mid] < s_k) p0 = mid + 1; else p1 = mid; }
    cnt[d] = m - p0;
  }
  for (int i = tid; i < 3 * (W + 2); i += MT) hist[i] = 0;
  __syncthreads();
  t_out = cnt[0];
  int total = m_scan(cnt, W + 1, s_tmp);
  { int pw0 = 1; while (pw0 < total) pw0 <<= 1;
    if (pw0 > cap) { if (tid == 0) atomicExch(M.ovf, 1); return; } }
  for (int d = 0; d <= W; ++d) {
    int j = k - d;
    const int32_t *L = idx + off[j];
    int m = len[j];
    int c = (d < W ? cnt[d + 1] : total) - cnt[d];
    for (int i = tid; i < c; i += MT) keys[cnt[d] + i] = (L[m - c + i] << 8) | d;
  }
  int pw = 1; while (pw < total) pw <<= 1;
  for (int i = total + tid; i < pw; i += MT) keys[i] = INT_MAX;
  __syncthreads();
  if (pw > 1) m_bitonic(keys, pw);
  for (int i = tid; i < total; i += MT) {
    int key = keys[i], x = key >> 8, d = key & 255;
    if (i > 0 && (keys[i - 1] >> 8) == x) continue;   // not the first of its value
    bool inK = (d == 0);
    int dmin = d;
    if (inK) dmin = (i + 1 < total && (keys[i + 1] >> 8) == x) ? (keys[i + 1] & 255) : -1;
    if (x < e_k) {                       // inside block k: r (d >= 1 always here)
      atomicAdd(&hist[dmin], 1);
    } else {
      if (dmin > 0) atomicAdd(&hist[(W + 2) + dmin], 1);           // s
      atomicAdd(&hist[2 * (W + 2) + (inK ? 1 : dmin)], 1);         // u
    }
  }
  __syncthreads();
  if (tid == 0) {
    for (int d = 1; d <= W; ++d) {
      hist[d] += hist[d - 1];
      hist[(W + 2) + d] += hist[(W + 2) + d - 1];
      hist[2 * (W + 2) + d] += hist[2 * (W + 2) + d - 1];
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(MT) merge_test_kernel(MergeArgs M) {
  extern __shared__ int msm[];
  __shared__ int s_tmp[MW + 1];
  const int tid = threadIdx.x;
  const int cap = (int)M.work_ints;
  int *keys = M.work + (size_t)blockIdx.x * M.work_ints;
  int *hr = msm;              // 3 * 130
  int *hc = msm + 3 * 130;    // 3 * 130
  int *cnt = msm + 6 * 130;   // 130
  for (int k = blockIdx.x; k < M.N; k += gridDim.x) {
    uint32_t mask[4] = {0, 0, 0, 0};
    if (k > 0) {
      const int s_k = M.bstart[k], q = M.bstart[k + 1] - s_k;
      int W = 0;
      while (k - 1 - W >= 0 && (s_k - M.bstart[k - 1 - W]) + q <= M.max_block && W < 127) ++W;
      if (W > 0) {
        int t = 0, t2 = 0;
        count_side(M, k, W, true, keys, cap, hr, cnt, s_tmp, t);
        __syncthreads();
        count_side(M, k, W, false, keys, cap, hc, cnt, s_tmp, t2);
        __syncthreads();
        if (tid == 0) {
          for (int d = 1; d <= W; ++d) {
            long long p = s_k - M.bstart[k - d];
            long long r = hr[d], s = hr[(W + 2) + d], u = hr[2 * (W + 2) + d];
            long long r2 = hc[d], s2 = hc[(W + 2) + d], v = hc[2 * (W + 2) + d];
            if (agg_test(p, q, r, s, t, r2, s2, t2, u, v, M.max_block)) mask[(d - 1) >> 5] |= 1u << ((d - 1) & 31);
          }
        }
      }
    }
    if (tid == 0) for (int w = 0; w < 4; ++w) M.T[4 * (size_t)k + w] = mask[w];
    __syncthreads();
  }
}

// ---------------------------------------------------------------- M2: scan
// The paper's order: after block k is finished, merge it into the aggregate
// that ends at k-1 iff the test passes.
__global__ void merge_scan_kernel(MergeArgs M) {
  __shared__ uint32_t sT[4 * 1024];
  int a = 0, nF = 0;
  if (threadIdx.x == 0) { M.first[0] = 0; nF = 1; }
  for (int base = 0; base < M.N; base += 1024) {
    int cnt = min(1024, M.N - base);
    for (int i = threadIdx.x; i < 4 * cnt; i += blockDim.x) sT[i] = M.T[4 * (size_t)base + i];
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = (base == 0 ? 1 : 0); i < cnt; ++i) {
        int k = base + i;
        int d = k - a;
        bool merge = d >= 1 && d <= 128 && ((sT[4 * i + ((d - 1) >> 5)] >> ((d - 1) & 31)) & 1u);
        if (!merge) { a = k; M.first[nF++] = k; }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { M.first[nF] = M.N; *M.nF = nF; }
}

// --------------------------------------------------- M3: union sizes, descriptors
// union of the members' kept indices >= e_k (rows of L^ / cols of Ũ^)
__device__ int gather_union(const MergeArgs &M, int a, int k, bool rows, int *keys, int cap, int *cnt, int *s_tmp,
                            int *flags) {
  const int tid = threadIdx.x;
  const int e_k = M.bstart[k + 1];
  const int32_t *idx = rows ? M.Lidx : M.Uidx;
  const int64_t *off = rows ? M.Lrow_off : M.Ucol_off;
  const int32_t *len = rows ? M.Lm : M.Uc;
  const int nm = k - a + 1;
  for (int x = tid; x < nm; x += MT) {
    int j = a + x;
    const int32_t *L = idx + off[j];
    int m = len[j];
    int p0 = 0, p1 = m;
    while (p0 < p1) { int mid = (p0 + p1) >> 1; if (L[mid] < e_k) p0 = mid + 1; else p1 = mid; }
    cnt[x] = m - p0;
  }
  __syncthreads();
  int total = m_scan(cnt, nm, s_tmp);
  int pw = 1; while (pw < total) pw <<= 1;
  if (2 * pw > cap) { if (tid == 0) atomicExch(M.ovf, 1); return -1; }
  for (int x = 0; x < nm; ++x) {
    int j = a + x;
    const int32_t *L = idx + off[j];
    int m = len[j];
    int c = (x + 1 < nm ? cnt[x + 1] : total) - cnt[x];
    for (int i = tid; i < c; i += MT) keys[cnt[x] + i] = L[m - c + i];
  }
  for (int i = total + tid; i < pw; i += MT) keys[i] = INT_MAX;
  __syncthreads();
  if (pw > 1) m_bitonic(keys, pw);
  for (int i = tid; i < total; i += MT) flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
  __syncthreads();
  int u = m_scan(flags, total, s_tmp);
  for (int base = 0; base < total; base += MT) {
    int i = base + tid; int v = 0, pos = -1;
    if (i < total) { v = keys[i]; int nxt = i + 1 < total ? flags[i + 1] : u; if (nxt > flags[i]) pos = flags[i]; }
    __syncthreads();
    if (pos >= 0) keys[pos] = v;
    __syncthreads();
  }
  return u;
}

__global__ void __launch_bounds__(MT) merge_count_kernel(MergeArgs M) {
  extern __shared__ int msm[];
  __shared__ int s_tmp[MW + 1];
  const int nF = *M.nF;
  int *keys = M.work + (size_t)blockIdx.x * M.work_ints;
  const int cap = (int)M.work_ints;
  int *cnt = msm;
  for (int F = blockIdx.x; F < nF; F += gridDim.x) {
    const int a = M.first[F], k = M.first[F + 1] - 1;
    if (threadIdx.x == 0) M.fbstart[F] = M.bstart[a];
    if (a == k) {
      if (threadIdx.x == 0) { M.fLm[F] = M.Lm[k]; M.fUc[F] = M.Uc[k]; }
      continue;
    }
    int u = gather_union(M, a, k, true, keys, cap, cnt, s_tmp, keys + cap / 2);
    __syncthreads();
    int v = gather_union(M, a, k, false, keys, cap, cnt, s_tmp, keys + cap / 2);
    if (threadIdx.x == 0) { M.fLm[F] = u; M.fUc[F] = v; }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) M.fbstart[nF] = M.n;
}

// descriptors: singletons keep their arena slices; merged blocks are appended
// after the factor kernel's cursors (tot[0..3] on entry).  One CTA.
// block-wide exclusive scan of NV 64-bit values per thread (1024 threads)
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

// descriptors: singletons keep their arena slices; merged blocks are appended after
// the factor kernel's cursors (tot[0..3] on entry).  One CTA of 1024 threads, each
// owning a contiguous range of final blocks.
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
    const unsigned long long u = M.fLm[F], w = M.fUc[F];
    v[0] += P * P;
    if (a != k) {
      v[1] += u; v[2] += u * P; v[3] += w; v[4] += w * P; v[9] += 1;
      const unsigned long long ws = 6ull * P * P + (u + w) * P + 64;
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
  // max workspace: reduce
  __shared__ unsigned long long smax;
  if (threadIdx.x == 0) smax = 0;
  __syncthreads();
  atomicMax(&smax, maxws);
  __syncthreads();
  if (threadIdx.x == 0) {
    M.fD_off[nF] = (int64_t)tot[0];
    M.tot[4] = M.tot[0] + tot[1]; M.tot[5] = M.tot[1] + tot[2];
    M.tot[6] = M.tot[2] + tot[3]; M.tot[7] = M.tot[3] + tot[4];
    M.tot[8] = tot[0]; M.tot[9] = smax; M.tot[10] = tot[9];
    M.tot[11] = (unsigned long long)(M.N - nF);
    M.tot[12] = tot[5]; M.tot[13] = tot[6]; M.tot[14] = tot[7]; M.tot[15] = tot[8];
  }
}

// ---------------------------------------------------------------- M4: arithmetic
// per merged run a..k (P = e_k - s_a <= max_block):
//   L_aa (unit lower), U_aa = D_j Ũ_j inside the run (unit upper), D_agg = diag(D_j)
//   D^ = U_aa^{-1} D_agg L_aa^{-1};  L^ = L_{>,agg} L_aa^{-1};  Ũ^ = L_aa Ũ_{agg,>}
// Work buffers in global memory (per CTA): Laa, Uaa, Linv, Uinv, T1 (P x P each,
// row-major), Lg (u x P), Ug (v x P).
__global__ void __launch_bounds__(MT) merge_arith_kernel(MergeArgs M, double *dwork, int64_t dwork_per_cta) {
  extern __shared__ int msm[];
  __shared__ int s_tmp[MW + 1];
  const int tid = threadIdx.x;
  const int nF = *M.nF;
  int *keys = M.work + (size_t)blockIdx.x * M.work_ints;
  const int cap = (int)M.work_ints;
  int *cnt = msm;
  double *base = dwork + (size_t)blockIdx.x * dwork_per_cta;
  double flops = 0.0;
  for (int F = blockIdx.x; F < nF; F += gridDim.x) {
    const int a = M.first[F], k = M.first[F + 1] - 1;
    const int sa = M.bstart[a], ek = M.bstart[k + 1];
    const int P = ek - sa;
    double *Dout = M.fD + M.fD_off[F];
    if (a == k) {
      const double *Din = M.D + M.D_off[k];
      for (int i = tid; i < P * P; i += MT) Dout[i] = Din[i];
      continue;
    }
    double *Laa = base, *Uaa = Laa + P * P, *Linv = Uaa + P * P, *Uinv = Linv + P * P, *T1 = Uinv + P * P;
    double *Lg = T1 + P * P;
    const int u = M.fLm[F], v = M.fUc[F];
    double *Ug = Lg + (size_t)u * P;
    for (int i = tid; i < P * P; i += MT) {
      int r = i / P, c = i % P;
      Laa[i] = (r == c) ? 1.0 : 0.0;
      Uaa[i] = (r == c) ? 1.0 : 0.0;
    }
    for (int i = tid; i < (u + v) * P; i += MT) Lg[i] = 0.0;
    __syncthreads();
    // L_aa and U_aa from the members' rows / cols inside the run
    for (int j = a; j <= k; ++j) {
      const int sj = M.bstart[j], ej = M.bstart[j + 1], bj = ej - sj;
      const int32_t *rows = M.Lidx + M.Lrow_off[j];
      const double *Lv = M.Lval + M.Lval_off[j];
      const int mj = M.Lm[j];
      for (int it = tid; it < mj * bj; it += MT) {
        int p = it / bj, t = it % bj;
        int x = rows[p];
        if (x < ek) Laa[(size_t)(x - sa) * P + (sj - sa) + t] = Lv[it];
      }
      const int32_t *cols = M.Uidx + M.Ucol_off[j];
      const double *Uv = M.Uval + M.Uval_off[j];
      const double *Dj = M.D + M.D_off[j];
      const int cj = M.Uc[j];
      for (int it = tid; it < cj * bj; it += MT) {
        int q = it / bj, r = it % bj;
        int y = cols[q];
        if (y < ek) {
          double acc = 0.0;
          for (int t = 0; t < bj; ++t) acc = fma(Dj[r + (size_t)t * bj], Uv[(size_t)q * bj + t], acc);
          Uaa[(size_t)(sj - sa + r) * P + (y - sa)] = acc;
        }
      }
    }
    __syncthreads();
    // unit triangular inverses, one column per thread
    for (int c = tid; c < P; c += MT) {
      for (int i = 0; i < P; ++i) {
        double x;
        if (i < c) x = 0.0;
        else if (i == c) x = 1.0;
        else {
          double acc = 0.0;
          for (int t = c; t < i; ++t) acc = fma(Laa[(size_t)i * P + t], Linv[(size_t)t * P + c], acc);
          x = -acc;
        }
        Linv[(size_t)i * P + c] = x;
      }
      for (int i = P - 1; i >= 0; --i) {
        double x;
        if (i > c) x = 0.0;
        else if (i == c) x = 1.0;
        else {
          double acc = 0.0;
          for (int t = i + 1; t <= c; ++t) acc = fma(Uaa[(size_t)i * P + t], Uinv[(size_t)t * P + c], acc);
          x = -acc;
        }
        Uinv[(size_t)i * P + c] = x;
      }
    }
    __syncthreads();
    // T1 = D_agg Linv
    for (int it = tid; it < P * P; it += MT) {
      int r = it / P, c = it % P;
      int j = a;
      while (M.bstart[j + 1] - sa <= r) ++j;
      const int sj = M.bstart[j] - sa, bj = M.bstart[j + 1] - M.bstart[j];
      const double *Dj = M.D + M.D_off[j];
      double acc = 0.0;
      for (int t = 0; t < bj; ++t) acc = fma(Dj[(r - sj) + (size_t)t * bj], Linv[(size_t)(sj + t) * P + c], acc);
      T1[it] = acc;
    }
    __syncthreads();
    // D^ = Uinv T1, stored column-major
    for (int it = tid; it < P * P; it += MT) {
      int c = it / P, r = it % P;
      double acc = 0.0;
      for (int t = r; t < P; ++t) acc = fma(Uinv[(size_t)r * P + t], T1[(size_t)t * P + c], acc);
      Dout[it] = acc;
    }
    // union rows / cols (recomputed; same as merge_count_kernel)
    int uu = gather_union(M, a, k, true, keys, cap, cnt, s_tmp, keys + cap / 2);
    if (uu < 0) return;
    for (int i = tid; i < uu; i += MT) M.Lidx_out[M.fLrow_off[F] + i] = keys[i];
    __syncthreads();
    for (int j = a; j <= k; ++j) {
      const int sj = M.bstart[j], bj = M.bstart[j + 1] - sj;
      const int32_t *rows = M.Lidx + M.Lrow_off[j];
      const double *Lv = M.Lval + M.Lval_off[j];
      const int mj = M.Lm[j];
      for (int it = tid; it < mj * bj; it += MT) {
        int p = it / bj, t = it % bj;
        int x = rows[p];
        if (x >= ek) Lg[(size_t)m_lbound(keys, 0, uu, x) * P + (sj - sa) + t] = Lv[it];
      }
    }
    __syncthreads();
    double *Lout = M.Lval_out + M.fLval_off[F];
    for (int it = tid; it < uu * P; it += MT) {
      int x = it / P, c = it % P;
      double acc = 0.0;
      for (int t = c; t < P; ++t) acc = fma(Lg[(size_t)x * P + t], Linv[(size_t)t * P + c], acc);
      Lout[it] = acc;
    }
    __syncthreads();
    int vv = gather_union(M, a, k, false, keys, cap, cnt, s_tmp, keys + cap / 2);
    if (vv < 0) return;
    for (int i = tid; i < vv; i += MT) M.Uidx_out[M.fUcol_off[F] + i] = keys[i];
    __syncthreads();
    for (int j = a; j <= k; ++j) {
      const int sj = M.bstart[j], bj = M.bstart[j + 1] - sj;
      const int32_t *cols = M.Uidx + M.Ucol_off[j];
      const double *Uv = M.Uval + M.Uval_off[j];
      const int cj = M.Uc[j];
      for (int it = tid; it < cj * bj; it += MT) {
        int q = it / bj, t = it % bj;
        int y = cols[q];
        if (y >= ek) Ug[(size_t)m_lbound(keys, 0, vv, y) * P + (sj - sa) + t] = Uv[it];
      }
    }
    __syncthreads();
    double *Uout = M.Uval_out + M.fUval_off[F];
    for (int it = tid; it < vv * P; it += MT) {
      int y = it / P, r = it % P;
      double acc = 0.0;
      for (int t = 0; t <= r; ++t) acc = fma(Laa[(size_t)r * P + t], Ug[(size_t)y * P + t], acc);
      Uout[it] = acc;
    }
    __syncthreads();
    if (tid == 0) {
      double Pd = P;
      flops += 2.0 * Pd * Pd * Pd / 3.0 + 2.0 * Pd * Pd * Pd / 2.0 + Pd * Pd * Pd + (double)(uu + vv) * Pd * Pd;
    }
  }
  if (tid == 0 && flops > 0.0) atomicAdd(M.flops, flops);
}

// ----------------------------------------------------------------- launchers
extern "C" cudaError_t bilu_merge_plan(const MergeArgs &M, int grid, cudaStream_t st) {
  const int smem = 7 * 130 * 4;
  merge_test_kernel<<<grid, MT, smem, st>>>(M);
  merge_scan_kernel<<<1, 256, 0, st>>>(M);
  merge_count_kernel<<<grid, MT, 1024 * 4, st>>>(M);
  merge_offsets_kernel<<<1, 1024, 0, st>>>(M);
  return cudaGetLastError();
}

extern "C" cudaError_t bilu_merge_arith(const MergeArgs &M, double *dwork, int64_t dwork_per_cta, int grid,
                                        cudaStream_t st) {
  merge_arith_kernel<<<grid, MT, 1024 * 4, st>>>(M, dwork, dwork_per_cta);
  return cudaGetLastError();
}

extern "C" int bilu_merge_args_size() { return (int)sizeof(MergeArgs); }

}  // namespace bilu
