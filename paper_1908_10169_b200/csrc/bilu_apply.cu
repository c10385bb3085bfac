// bilu_apply.cu -- y = (L D^{-1} U)^{-1} x with the final (merged) factors.
//
// "This requires factorizing and inverting the diagonal blocks ... but
// simplifies ... the forward/backward substitution inside a Krylov subspace
// method": with P_K = D_K^{-1} and U = D Ũ,
//   forward   w_F = x_F - sum_J L_J[rows in F, :] w_J          (unit block-lower L)
//   backward  y_F = D_F (w_F - Ũ_F y[cols(Ũ_F)])              (U = D Ũ unit upper)
// Both sweeps are persistent dataflow kernels over the final blocks (a block
// starts when every block it reads is finished), pulling in a fixed order so
// that the result is deterministic.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bilu_internal.h"

namespace bilu {

constexpr int AT = 128;

__device__ __forceinline__ int a_ld_vol(const int *p) { return *(const volatile int *)p; }

__device__ __forceinline__ int a_pop(const ApplyArgs &A, int *s_blk) {
  if (threadIdx.x == 0) {
    int F = -1;
    unsigned long long idx = atomicAdd(&A.ctrl[1], 1ull);
    if (idx < (unsigned long long)A.nF) {
      while ((F = a_ld_vol(&A.queue[idx])) < 0) __nanosleep(32);
    }
    *s_blk = F;
  }
  __syncthreads();
  int F = *s_blk;
  __syncthreads();
  return F;
}

__device__ __forceinline__ void a_release(const ApplyArgs &A, const int32_t *ptr, const int32_t *succ, int F) {
  __threadfence();
  __syncthreads();
  for (int x = ptr[F] + threadIdx.x; x < ptr[F + 1]; x += AT) {
    int T = succ[x];
    if (atomicSub(&A.cnt[T], 1) == 1) {
      unsigned long long slot = atomicAdd(&A.ctrl[0], 1ull);
      __threadfence();
      *(volatile int *)&A.queue[slot] = T;
    }
  }
}

__global__ void __launch_bounds__(AT) apply_fwd_kernel(ApplyArgs A) {
  __shared__ int s_blk;
  __shared__ double s_w[128];
  while (true) {
    const int F = a_pop(A, &s_blk);
    if (F < 0) break;
    __threadfence();
    const int s = A.fbstart[F], b = A.fbstart[F + 1] - s;
    for (int i = threadIdx.x; i < b; i += AT) s_w[i] = __ldcg(A.w + s + i);
    __syncthreads();
    for (int x = A.fl_ptr[F]; x < A.fl_ptr[F + 1]; ++x) {
      const int J = A.fl_rec[3 * x], r0 = A.fl_rec[3 * x + 1], r1 = A.fl_rec[3 * x + 2];
      const int sJ = A.fbstart[J], bJ = A.fbstart[J + 1] - sJ;
      const int32_t *rows = A.Lidx + A.Lrow_off[J];
      const double *Lv = A.Lval + A.Lval_off[J];
      for (int p = r0 + threadIdx.x; p < r1; p += AT) {
        const double *l = Lv + (int64_t)p * bJ;
        double acc = 0.0;
        for (int t = 0; t < bJ; ++t) acc = fma(l[t], __ldcg(A.w + sJ + t), acc);
        s_w[rows[p] - s] -= acc;
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < b; i += AT) A.w[s + i] = s_w[i];
    a_release(A, A.fs_ptr, A.fs, F);
  }
}

__global__ void __launch_bounds__(AT) apply_bwd_kernel(ApplyArgs A) {
  __shared__ int s_blk;
  __shared__ double s_z[128];
  while (true) {
    const int F = a_pop(A, &s_blk);
    if (F < 0) break;
    __threadfence();
    const int s = A.fbstart[F], b = A.fbstart[F + 1] - s;
    const int c = A.Uc[F];
    const int32_t *cols = A.Uidx + A.Ucol_off[F];
    const double *Uv = A.Uval + A.Uval_off[F];
    for (int r = threadIdx.x; r < b; r += AT) {
      double acc = A.w[s + r];
      for (int q = 0; q < c; ++q) acc = fma(-Uv[(int64_t)q * b + r], __ldcg(A.y + cols[q]), acc);
      s_z[r] = acc;
    }
    __syncthreads();
    const double *D = A.D + A.D_off[F];
    for (int r = threadIdx.x; r < b; r += AT) {
      double acc = 0.0;
      for (int t = 0; t < b; ++t) acc = fma(D[r + (int64_t)t * b], s_z[t], acc);
      A.y[s + r] = acc;
    }
    a_release(A, A.bs_ptr, A.bs, F);
  }
}

extern "C" cudaError_t bilu_launch_apply(const ApplyArgs &A, int grid, int backward, cudaStream_t st) {
  if (backward) apply_bwd_kernel<<<grid, AT, 0, st>>>(A);
  else apply_fwd_kernel<<<grid, AT, 0, st>>>(A);
  return cudaGetLastError();
}

}  // namespace bilu
