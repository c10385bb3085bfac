// bilu_apply.cu -- y = (L D^{-1} U)^{-1} x with the final (merged) factors.
//
// "This requires factorizing and inverting the diagonal blocks ... but
// simplifies ... the forward/backward substitution inside a Krylov subspace
// method": with P_K = D_K^{-1} and U = D Ũ,
//   forward   w_F = x_F - sum_J L_J[rows in F, :] w_J          (unit block-lower L)
//   backward  y_F = D_F (w_F - Ũ_F y[cols(Ũ_F)])              (U = D Ũ unit upper)
// Both sweeps are persistent dataflow kernels over the final blocks, one warp per block
// (16 independent warps per CTA): the forward sweep pushes L_J w_J into its targets with
// native fp64 reductions (summation order unspecified: rounding only), the backward sweep
// pulls from the blocks in its Ũ columns.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bilu_internal.h"

namespace bilu {

constexpr int AT = 512;             // 16 warps per CTA, each an independent worker
constexpr int AW = AT / 32;

__device__ __forceinline__ int a_ld_vol(const int *p) { return *(const volatile int *)p; }
__device__ __forceinline__ unsigned long long a_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void a_prof(const ApplyArgs &A, int F, int k) {
  if (A.prof && (threadIdx.x & 31) == 0) A.prof[3 * (size_t)F + k] = a_clock();
}
__device__ __forceinline__ void a_red_add(double *p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// successor list of F loaded right after the pop (independent of F's arithmetic): lane x
// holds successor x for lists of <= 32 entries; longer lists are re-read at release
struct Succ {
  int32_t x0, n, T;
};
__device__ __forceinline__ Succ a_succ_prefetch(const int32_t *ptr, const int32_t *succ, int F) {
  Succ S;
  S.x0 = ptr[F];
  S.n = ptr[F + 1] - S.x0;
  const int lane = threadIdx.x & 31;
  S.T = lane < S.n ? succ[S.x0 + lane] : -1;
  return S;
}
__device__ __forceinline__ void a_release_pre(const ApplyArgs &A, const int32_t *succ, const Succ &S) {
  __threadfence();
  __syncwarp();
  const int lane = threadIdx.x & 31;
  for (int x = lane; x < S.n; x += 32) {
    const int T = x < 32 ? S.T : succ[S.x0 + x];
    if (atomicSub(&A.cnt[T], 1) == 1) {
      const unsigned long long slot = atomicAdd(&A.ctrl[0], 1ull);
      __threadfence();
      *(volatile int *)&A.queue[slot] = T;
    }
  }
}

// ---- heavy blocks shared by the CTA's warps.  A warp that pops a wide block with a large
// panel publishes it here (one at a time per CTA); warps waiting for their queue slot take
// parts of it.  A part is claimed by one atomic on `next` = (generation << 32) | part; the
// claim is valid iff the descriptor still carries that generation and part < n (a new
// generation is only published after every part of the previous one is done).
constexpr int HEAVY_ELEMS = 16384;     // panel entries from which a wide block is split
constexpr int FWD_PART_ROWS = 64;      // rows of L_J per forward part
constexpr int YCH = 128;               // columns of Ũ_F per backward part / gather chunk

struct Help {
  unsigned long long next;
  int F, n, done, lock, owner_w;
  unsigned gen;
};

__device__ __forceinline__ void help_init(Help &H) {
  if (threadIdx.x == 0) { H.next = 0ull; H.F = -1; H.n = 0; H.done = 0; H.lock = 0; H.owner_w = 0; H.gen = 0u; }
  __syncthreads();
}

// claim a part: returns its index (warp-uniform) or -1; F and owner_w of the block
__device__ __forceinline__ int help_claim(Help &H, int &F, int &ow) {
  int p = -1, f = -1, w = 0;
  if ((threadIdx.x & 31) == 0) {
    volatile Help &V = H;
    if ((int)(V.next & 0xffffffffull) < V.n) {
      const unsigned long long old = atomicAdd(&H.next, 1ull);
      const unsigned g = (unsigned)(old >> 32);
      const int pp = (int)(old & 0xffffffffull);
      __threadfence_block();
      if (V.gen == g && pp < V.n) { p = pp; f = V.F; w = V.owner_w; }
    }
  }
  p = __shfl_sync(0xffffffffu, p, 0);
  F = __shfl_sync(0xffffffffu, f, 0);
  ow = __shfl_sync(0xffffffffu, w, 0);
  return p;
}

__device__ __forceinline__ void help_part_done(Help &H) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) { __threadfence(); atomicAdd(&H.done, 1); }
  __syncwarp();
}

// try to publish block F with n parts (lane 0 takes the CTA lock); warp-uniform result
__device__ __forceinline__ bool help_publish(Help &H, int F, int n) {
  __threadfence_block();          // the owner's staged w_J / zeroed z before the descriptor
  __syncwarp();
  int ok = 0;
  if ((threadIdx.x & 31) == 0 && atomicCAS(&H.lock, 0, 1) == 0) {
    volatile Help &V = H;
    const unsigned g = V.gen + 1u;
    V.F = F; V.n = n; V.done = 0; V.owner_w = threadIdx.x >> 5; V.gen = g;
    __threadfence_block();
    atomicExch(&H.next, (unsigned long long)g << 32);
    ok = 1;
  }
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

__device__ __forceinline__ void help_wait_unlock(Help &H, int n) {
  if ((threadIdx.x & 31) == 0) {
    volatile Help &V = H;
    while (V.done < n) __nanosleep(32);
    __threadfence_block();
    V.n = 0;
    __threadfence_block();
    atomicExch(&H.lock, 0);
  }
  __syncwarp();
}

// forward part: rows [p0, p1) of a wide L_J (b_J >= 32): lanes across a row (coalesced),
// 8 rows per step; w[rows] -= L_J w_J by native fp64 reductions
__device__ void fwd_rows(const ApplyArgs &A, int J, const double *wj, int p0, int p1) {
  const int lane = threadIdx.x & 31;
  const int bJ = A.fbstart[J + 1] - A.fbstart[J];
  const int32_t *rows = A.Lidx + A.Lrow_off[J];
  const double *Lv = A.Lval + A.Lval_off[J];
  const int nt = (bJ - lane + 31) >> 5;
  double wl[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) wl[k] = k < nt ? wj[lane + 32 * k] : 0.0;
  constexpr int RG = 8;
  for (int q = p0; q < p1; q += RG) {
    double v[RG][4];
#pragma unroll
    for (int i = 0; i < RG; ++i) {
      const double *l = Lv + (int64_t)min(q + i, p1 - 1) * bJ + lane;
#pragma unroll
      for (int k = 0; k < 4; ++k) v[i][k] = k < nt ? l[32 * k] : 0.0;
    }
    double acc[RG];
#pragma unroll
    for (int i = 0; i < RG; ++i) {
      acc[i] = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[i] = fma(v[i][k], wl[k], acc[i]);
    }
#pragma unroll
    for (int i = 0; i < RG; ++i)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
    double mine = 0.0;
#pragma unroll
    for (int i = 0; i < RG; ++i) mine = lane == i ? acc[i] : mine;
    if (lane < RG && q + lane < p1) a_red_add(A.w + rows[q + lane], -mine);
  }
}

// backward part: columns [q0, q1) of a wide Ũ_F (b > 16): y gathered in chunks of YCH into
// yq, lane owns rows lane + 32k, 8 columns per step; z += Ũ_F[:, q0:q1] y (atomic if shared)
__device__ void bwd_cols(const ApplyArgs &A, int F, int q0, int q1, double *z, bool shared, double *yq) {
  const int lane = threadIdx.x & 31;
  const int b = A.fbstart[F + 1] - A.fbstart[F];
  const int32_t *cols = A.Uidx + A.Ucol_off[F];
  const double *Uv = A.Uval + A.Uval_off[F];
  const int nr = (b - lane + 31) >> 5;
  double a[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  for (int c0 = q0; c0 < q1; c0 += YCH) {
    const int qn = min(YCH, q1 - c0);
    __syncwarp();
    for (int j = lane; j < qn; j += 32) yq[j] = __ldcg(A.y + cols[c0 + j]);
    __syncwarp();
    const double *u = Uv + (int64_t)c0 * b + lane;
    int j = 0;
    for (; j + 7 < qn; j += 8) {
      const double *u0 = u + (int64_t)j * b;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < nr) {
          double v[8];
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) v[c8] = u0[(int64_t)c8 * b + 32 * k];
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) a[k][c8 & 1] = fma(v[c8], yq[j + c8], a[k][c8 & 1]);
        }
    }
    for (; j < qn; ++j) {
      const double yj = yq[j];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < nr) a[k][0] = fma(u[(int64_t)j * b + 32 * k], yj, a[k][0]);
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (k < nr) {
      const double v = a[k][0] + a[k][1];
      if (shared) atomicAdd(z + lane + 32 * k, v);
      else z[lane + 32 * k] += v;
    }
  __syncwarp();
}

// pop the next ready block (warp-uniform; -1 when this sweep's blocks are exhausted); while
// the ticket's slot is empty, take parts of the CTA's published heavy block
template <bool BWD>
__device__ int a_pop_help(const ApplyArgs &A, Help &H, double (*s_a)[128], double *yq_own) {
  unsigned long long idx = 0;
  if ((threadIdx.x & 31) == 0) idx = atomicAdd(&A.ctrl[1], 1ull);
  idx = __shfl_sync(0xffffffffu, idx, 0);
  if (idx >= (unsigned long long)A.ntarget) return -1;
  while (true) {
    int F = -1;
    if ((threadIdx.x & 31) == 0) F = a_ld_vol(&A.queue[idx]);
    F = __shfl_sync(0xffffffffu, F, 0);
    if (F >= 0) return F;
    int HF, ow;
    const int p = help_claim(H, HF, ow);
    if (p >= 0) {
      if (BWD) {
        const int c = A.Uc[HF];
        bwd_cols(A, HF, p * YCH, min(c, (p + 1) * YCH), s_a[ow], true, yq_own);
      } else {
        const int m = A.Lm[HF];
        fwd_rows(A, HF, s_a[ow], p * FWD_PART_ROWS, min(m, (p + 1) * FWD_PART_ROWS));
      }
      help_part_done(H);
      continue;
    }
    if ((threadIdx.x & 31) == 0) __nanosleep(20);
    __syncwarp();
  }
}

// forward sweep, push form: when block J is final (every block with L rows in J has pushed),
// w[rows of L_J] -= L_J w_J with native fp64 reductions, then J's targets are released
__global__ void __launch_bounds__(AT) apply_fwd_kernel(ApplyArgs A) {
  __shared__ double s_w[AW][128];
  __shared__ double s_y[AW][YCH];
  __shared__ Help H;
  help_init(H);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double *wj = s_w[wid];
  while (true) {
    const int J = a_pop_help<false>(A, H, s_w, s_y[wid]);
    if (J < 0) break;
    a_prof(A, J, 0);
    __threadfence();
    const Succ SJ = a_succ_prefetch(A.fs_ptr, A.fs, J);
    const int sJ = A.fbstart[J], bJ = A.fbstart[J + 1] - sJ;
    for (int t = lane; t < bJ; t += 32) wj[t] = __ldcg(A.w + sJ + t);
    __syncwarp();
    const int m = A.Lm[J];
    if (bJ >= 32) {
      const int np = (m + FWD_PART_ROWS - 1) / FWD_PART_ROWS;
      if (np > 1 && (int64_t)m * bJ >= HEAVY_ELEMS && help_publish(H, J, np)) {
        int HF, ow;
        for (int p; (p = help_claim(H, HF, ow)) >= 0;) {
          fwd_rows(A, HF, s_w[ow], p * FWD_PART_ROWS, min(A.Lm[HF], (p + 1) * FWD_PART_ROWS));
          help_part_done(H);
        }
        help_wait_unlock(H, np);
      } else {
        fwd_rows(A, J, wj, 0, m);
      }
    } else {
      const int32_t *rows = A.Lidx + A.Lrow_off[J];
      const double *Lv = A.Lval + A.Lval_off[J];
      for (int p = lane; p < m; p += 32) {
        const double *l = Lv + (int64_t)p * bJ;
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        int t = 0;
        for (; t + 3 < bJ; t += 4) {
          acc0 = fma(l[t], wj[t], acc0); acc1 = fma(l[t + 1], wj[t + 1], acc1);
          acc2 = fma(l[t + 2], wj[t + 2], acc2); acc3 = fma(l[t + 3], wj[t + 3], acc3);
        }
        for (; t < bJ; ++t) acc0 = fma(l[t], wj[t], acc0);
        a_red_add(A.w + rows[p], -((acc0 + acc1) + (acc2 + acc3)));
      }
    }
    a_prof(A, J, 1);
    a_release_pre(A, A.fs, SJ);
    a_prof(A, J, 2);
  }
}

// backward sweep, pull form: y_F = D_F (w_F - Ũ_F y[cols(Ũ_F)]) once every block in F's Ũ
// columns is final.  Wide blocks (b > 16): lanes over rows, shared by the CTA when heavy;
// narrow ones: groups of lanes split the columns
__global__ void __launch_bounds__(AT) apply_bwd_kernel(ApplyArgs A) {
  __shared__ double s_z[AW][128];
  __shared__ double s_y[AW][YCH];
  __shared__ Help H;
  help_init(H);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double *z = s_z[wid];
  double *yq = s_y[wid];
  while (true) {
    const int F = a_pop_help<true>(A, H, s_z, yq);
    if (F < 0) break;
    a_prof(A, F, 0);
    __threadfence();
    const Succ SF = a_succ_prefetch(A.bs_ptr, A.bs, F);
    const int s = A.fbstart[F], b = A.fbstart[F + 1] - s;
    // independent of the pull: w_F and (b <= 16) the lane's row of D_F
    const double wF = lane < b ? __ldcg(A.w + s + lane) : 0.0;
    double drow[16];
    if (b <= 16) {
      const double *D = A.D + A.D_off[F];
#pragma unroll
      for (int t = 0; t < 16; ++t) drow[t] = (t < b && lane < b) ? D[lane + (int64_t)t * b] : 0.0;
    }
    const int c = A.Uc[F];
    const int32_t *cols = A.Uidx + A.Ucol_off[F];
    const double *Uv = A.Uval + A.Uval_off[F];
    int R = 1;
    while (R < b && R < 32) R <<= 1;                 // lanes per row group
    const int G = 32 / R, gi = lane / R, rl = lane % R;
    for (int r = lane; r < b; r += 32) z[r] = 0.0;
    __syncwarp();
    if (R == 32) {
      const int np = (c + YCH - 1) / YCH;
      if (np > 1 && (int64_t)c * b >= HEAVY_ELEMS && help_publish(H, F, np)) {
        int HF, ow;
        for (int p; (p = help_claim(H, HF, ow)) >= 0;) {
          bwd_cols(A, HF, p * YCH, min(A.Uc[HF], (p + 1) * YCH), s_z[ow], true, yq);
          help_part_done(H);
        }
        help_wait_unlock(H, np);
        __threadfence_block();
      } else {
        bwd_cols(A, F, 0, c, z, false, yq);
      }
    } else {
      // the gathers of chunk q0 + YCH are issued before chunk q0's products (registers)
      for (int j = lane; j < min(YCH, c); j += 32) yq[j] = __ldcg(A.y + cols[j]);
      __syncwarp();
      for (int q0 = 0; q0 < c; q0 += YCH) {
        const int qn = min(YCH, c - q0);
        const int nq0 = q0 + YCH, nqn = min(YCH, c - nq0);
        double pre[YCH / 32];
#pragma unroll
        for (int k = 0; k < YCH / 32; ++k) {
          const int j = lane + 32 * k;
          pre[k] = j < nqn ? __ldcg(A.y + cols[nq0 + j]) : 0.0;
        }
        for (int r0 = 0; r0 < b; r0 += R) {
          const int r = r0 + rl;
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          if (r < b) {
            const double *ucol = Uv + (int64_t)q0 * b + r;
            int j = gi;
            for (; j + 3 * G < qn; j += 4 * G) {
              a0 = fma(ucol[(int64_t)j * b], yq[j], a0);
              a1 = fma(ucol[(int64_t)(j + G) * b], yq[j + G], a1);
              a2 = fma(ucol[(int64_t)(j + 2 * G) * b], yq[j + 2 * G], a2);
              a3 = fma(ucol[(int64_t)(j + 3 * G) * b], yq[j + 3 * G], a3);
            }
            for (; j < qn; j += G) a0 = fma(ucol[(int64_t)j * b], yq[j], a0);
          }
          double acc = (a0 + a1) + (a2 + a3);
          for (int o = R; o < 32; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (gi == 0 && r < b) z[r] += acc;
        }
        __syncwarp();
        if (nqn > 0) {
#pragma unroll
          for (int k = 0; k < YCH / 32; ++k) {
            const int j = lane + 32 * k;
            if (j < nqn) yq[j] = pre[k];
          }
          __syncwarp();
        }
      }
    }
    for (int r = lane; r < b; r += 32) z[r] = (r < 32 ? wF : __ldcg(A.w + s + r)) - z[r];
    __syncwarp();
    // y_F = D_F z: lane owns rows lane, lane+32, .. (up to 4 independent chains), one pass over
    // the columns of D_F (column-major: coalesced across lanes), 2-way unrolled
    const double *D = A.D + A.D_off[F];
    if (b <= 16) {
      double acc = 0.0, acc2 = 0.0;
#pragma unroll
      for (int t = 0; t < 16; t += 2) {
        if (t < b) acc = fma(drow[t], z[t], acc);
        if (t + 1 < b) acc2 = fma(drow[t + 1], z[t + 1], acc2);
      }
      if (lane < b) A.y[s + lane] = acc + acc2;
    } else {
      const int nr = (b - lane + 31) >> 5;
      double acc[4] = {0.0, 0.0, 0.0, 0.0}, acc2[4] = {0.0, 0.0, 0.0, 0.0};
      int t = 0;
      for (; t + 1 < b; t += 2) {
        const double z0 = z[t], z1 = z[t + 1];
        const double *d0 = D + (int64_t)t * b + lane, *d1 = d0 + b;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < nr) {
            acc[k] = fma(d0[32 * k], z0, acc[k]);
            acc2[k] = fma(d1[32 * k], z1, acc2[k]);
          }
      }
      if (t < b) {
        const double z0 = z[t];
        const double *d0 = D + (int64_t)t * b + lane;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < nr) acc[k] = fma(d0[32 * k], z0, acc[k]);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < nr) A.y[s + lane + 32 * k] = acc[k] + acc2[k];
    }
    __syncwarp();
    a_prof(A, F, 1);
    a_release_pre(A, A.bs, SF);
    a_prof(A, F, 2);
  }
}

// ---- distributed apply (bilu_apply_dist_begin / _end): separator rows of the permuted vectors
__global__ void sep_gather_kernel(int m, const int32_t *idx, const double *src, double *out) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < m; x += gridDim.x * blockDim.x) out[x] = src[idx[x]];
}
// out = w[sep] - x[sep]: this rank's (negated) contributions L_J w_J to the separator rows
__global__ void sep_contrib_kernel(int m, const int32_t *idx, const double *w, const double *xsep, double *out) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < m; x += gridDim.x * blockDim.x) out[x] = w[idx[x]] - xsep[x];
}
// w[sep] = x[sep] + (sum over ranks of the contributions)
__global__ void sep_set_kernel(int m, const int32_t *idx, const double *xsep, const double *sum, double *w) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < m; x += gridDim.x * blockDim.x) w[idx[x]] = xsep[x] + sum[x];
}
// y[perm[i]] = y_perm[i] on the rows this rank reports (mask 1: own subtree, 2: separator if
// write_sep), 0 elsewhere: the ranks' outputs sum to the full vector
__global__ void permute_out_masked_kernel(int n, const int32_t *perm, const uint8_t *mask, int write_sep,
                                          const double *yp, double *y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int m = mask[i];
    y[perm[i]] = (m == 1 || (m == 2 && write_sep)) ? yp[i] : 0.0;
  }
}

extern "C" cudaError_t bilu_launch_sep_gather(int m, const int32_t *idx, const double *src, double *out, cudaStream_t st) {
  if (m > 0) sep_gather_kernel<<<(m + 255) / 256, 256, 0, st>>>(m, idx, src, out);
  return cudaGetLastError();
}
extern "C" cudaError_t bilu_launch_sep_contrib(int m, const int32_t *idx, const double *w, const double *xsep,
                                               double *out, cudaStream_t st) {
  if (m > 0) sep_contrib_kernel<<<(m + 255) / 256, 256, 0, st>>>(m, idx, w, xsep, out);
  return cudaGetLastError();
}
extern "C" cudaError_t bilu_launch_sep_set(int m, const int32_t *idx, const double *xsep, const double *sum, double *w,
                                           cudaStream_t st) {
  if (m > 0) sep_set_kernel<<<(m + 255) / 256, 256, 0, st>>>(m, idx, xsep, sum, w);
  return cudaGetLastError();
}
extern "C" cudaError_t bilu_launch_permute_out_masked(int n, const int32_t *perm, const uint8_t *mask, int write_sep,
                                                      const double *yp, double *y, cudaStream_t st) {
  permute_out_masked_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, perm, mask, write_sep, yp, y);
  return cudaGetLastError();
}

extern "C" cudaError_t bilu_launch_apply(const ApplyArgs &A, int grid, int backward, cudaStream_t st) {
  if (backward) apply_bwd_kernel<<<grid, AT, 0, st>>>(A);
  else apply_fwd_kernel<<<grid, AT, 0, st>>>(A);
  return cudaGetLastError();
}

}  // namespace bilu
