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
__device__ __forceinline__ void a_red_add(double *p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// one warp pops the next ready block (lane 0), broadcast to the warp; -1 when all done
__device__ __forceinline__ int a_pop_warp(const ApplyArgs &A) {
  int F = -1;
  if ((threadIdx.x & 31) == 0) {
    const unsigned long long idx = atomicAdd(&A.ctrl[1], 1ull);
    if (idx < (unsigned long long)A.ntarget) {
      while ((F = a_ld_vol(&A.queue[idx])) < 0) __nanosleep(20);
    }
  }
  return __shfl_sync(0xffffffffu, F, 0);
}

__device__ __forceinline__ void a_release_warp(const ApplyArgs &A, const int32_t *ptr, const int32_t *succ, int F) {
  __threadfence();
  __syncwarp();
  for (int x = ptr[F] + (threadIdx.x & 31); x < ptr[F + 1]; x += 32) {
    const int T = succ[x];
    if (atomicSub(&A.cnt[T], 1) == 1) {
      const unsigned long long slot = atomicAdd(&A.ctrl[0], 1ull);
      __threadfence();
      *(volatile int *)&A.queue[slot] = T;
    }
  }
}

// forward sweep, push form: when block J is final (every block with L rows in J has pushed),
// w[rows of L_J] -= L_J w_J with native fp64 reductions, then J's targets are released
__global__ void __launch_bounds__(AT) apply_fwd_kernel(ApplyArgs A) {
  __shared__ double s_w[AW][128];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double *wj = s_w[wid];
  while (true) {
    const int J = a_pop_warp(A);
    if (J < 0) break;
    __threadfence();
    const int sJ = A.fbstart[J], bJ = A.fbstart[J + 1] - sJ;
    for (int t = lane; t < bJ; t += 32) wj[t] = __ldcg(A.w + sJ + t);
    __syncwarp();
    const int m = A.Lm[J];
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
    a_release_warp(A, A.fs_ptr, A.fs, J);
  }
}

// backward sweep, pull form: y_F = D_F (w_F - Ũ_F y[cols(Ũ_F)]) once every block in F's Ũ
// columns is final.  Lanes over the rows of F (groups of lanes split the columns when b < 32)
constexpr int YCH = 128;            // gathered y values staged per warp and chunk
__global__ void __launch_bounds__(AT) apply_bwd_kernel(ApplyArgs A) {
  __shared__ double s_z[AW][128];
  __shared__ double s_y[AW][YCH];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double *z = s_z[wid];
  double *yq = s_y[wid];
  while (true) {
    const int F = a_pop_warp(A);
    if (F < 0) break;
    __threadfence();
    const int s = A.fbstart[F], b = A.fbstart[F + 1] - s;
    const int c = A.Uc[F];
    const int32_t *cols = A.Uidx + A.Ucol_off[F];
    const double *Uv = A.Uval + A.Uval_off[F];
    int R = 1;
    while (R < b && R < 32) R <<= 1;                 // lanes per row group
    const int G = 32 / R, gi = lane / R, rl = lane % R;
    for (int r = lane; r < b; r += 32) z[r] = 0.0;
    __syncwarp();
    for (int q0 = 0; q0 < c; q0 += YCH) {
      const int qn = min(YCH, c - q0);
      for (int j = lane; j < qn; j += 32) yq[j] = __ldcg(A.y + cols[q0 + j]);   // independent gathers
      __syncwarp();
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
    }
    for (int r = lane; r < b; r += 32) z[r] = __ldcg(A.w + s + r) - z[r];
    __syncwarp();
    const double *D = A.D + A.D_off[F];
    for (int r = lane; r < b; r += 32) {
      double acc = 0.0;
      for (int t = 0; t < b; ++t) acc = fma(D[r + (int64_t)t * b], z[t], acc);
      A.y[s + r] = acc;
    }
    __syncwarp();
    a_release_warp(A, A.bs_ptr, A.bs, F);
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
