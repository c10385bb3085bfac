// bilu_util.cu -- small HBM-bound kernels: value gather for bilu_set_values
// (a-4 prework: Ã's values in CSR and CSC order from A's original CSR order),
// permutation of vectors for bilu_apply, and final-D assembly.
#include <cuda_runtime.h>
#include <stdint.h>

namespace bilu {

__global__ void gather_kernel(double *__restrict__ dst, const double *__restrict__ src,
                              const int64_t *__restrict__ map, int64_t n) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = __ldg(src + __ldg(map + i));
}

// y[i] = x[perm[i]]  (to the permuted ordering)   or   y[perm[i]] = x[i]  (back)
__global__ void permute_kernel(double *__restrict__ y, const double *__restrict__ x,
                               const int32_t *__restrict__ perm, int32_t n, int inverse) {
  int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (inverse) y[perm[i]] = x[i]; else y[i] = x[perm[i]];
  }
}

// max |x_i| (non-negative doubles order like their bit patterns): alpha of Sec. 3.6
__global__ void maxabs_kernel(unsigned long long *out, const double *__restrict__ x, int64_t n) {
  double m = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) m = fmax(m, fabs(x[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

static int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

extern "C" cudaError_t bilu_launch_gather(double *dst, const double *src, const int64_t *map,
                                          int64_t n, cudaStream_t st) {
  gather_kernel<<<grid_for(n), 256, 0, st>>>(dst, src, map, n);
  return cudaGetLastError();
}

extern "C" cudaError_t bilu_launch_maxabs(double *out, const double *x, int64_t n, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  if (n > 0) maxabs_kernel<<<grid_for(n), 256, 0, st>>>((unsigned long long *)out, x, n);
  return cudaGetLastError();
}

extern "C" cudaError_t bilu_launch_permute(double *y, const double *x, const int32_t *perm,
                                           int32_t n, int inverse, cudaStream_t st) {
  permute_kernel<<<grid_for(n), 256, 0, st>>>(y, x, perm, n, inverse);
  return cudaGetLastError();
}

}  // namespace bilu

// ------------------------------------------------------------ diagnostics
// cta_dgemm (DMMA m8n8k4) exercised on its own: `batch` independent products,
// one CTA each, C_b = alpha A_b B_b + beta C_b (bilu.h: bilu_diag_dgemm).
#include "dgemm_cta.cuh"
namespace bilu {
__global__ void __launch_bounds__(256) diag_dgemm_kernel(int M, int N, int K, double alpha, const double *A,
                                                         int64_t ars, int64_t acs, const double *B, int64_t brs,
                                                         int64_t bcs, double beta, double *C, int64_t crs,
                                                         int64_t ccs, int64_t sa, int64_t sb, int64_t sc) {
  __shared__ double sm[DGEMM_SMEM_DOUBLES];
  const int b = blockIdx.x;
  cta_dgemm<256>(M, N, K, alpha, DMat{A + b * sa, ars, acs}, DMat{B + b * sb, brs, bcs}, beta, C + b * sc, crs,
                 ccs, sm);
}
template <int NMAX>
__global__ void __launch_bounds__(256) diag_tsgemm_kernel(int M, int N, int K, double alpha, const double *A,
                                                          int64_t ars, int64_t acs, const double *B, int64_t brs,
                                                          int64_t bcs, double beta, double *C, int64_t crs,
                                                          int64_t ccs, int64_t sa, int64_t sb, int64_t sc) {
  extern __shared__ double bsm[];
  const int b = blockIdx.x;
  tsgemm_stage_b<256, NMAX>(K, N, DMat{B + b * sb, brs, bcs}, bsm);
  cta_tsgemm<256, NMAX>(M, N, K, DMat{A + b * sa, ars, acs}, bsm, EpiAxpby{alpha, beta, C + b * sc, crs, ccs});
}
}  // namespace bilu

// tall-skinny variant (K, N <= 128): mode 1 of bilu_diag_dgemm
extern "C" int bilu_diag_tsgemm(int M, int N, int K, double alpha, const double *A, int64_t ars, int64_t acs,
                                const double *B, int64_t brs, int64_t bcs, double beta, double *C, int64_t crs,
                                int64_t ccs, int batch, int64_t sa, int64_t sb, int64_t sc, void *stream) {
  if (M < 0 || N < 0 || K < 0 || batch < 1 || N > 128 || K > 128) return 1;
  if (M == 0 || N == 0) return 0;
  if (!A || !B || !C) return 1;
  if (N <= 64) {
    const int smem = K * bilu::TsB<64>::LDB * 8;
    cudaFuncSetAttribute(bilu::diag_tsgemm_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bilu::diag_tsgemm_kernel<64><<<batch, 256, smem, (cudaStream_t)stream>>>(M, N, K, alpha, A, ars, acs, B, brs,
                                                                              bcs, beta, C, crs, ccs, sa, sb, sc);
  } else {
    const int smem = K * bilu::TsB<128>::LDB * 8;
    cudaFuncSetAttribute(bilu::diag_tsgemm_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bilu::diag_tsgemm_kernel<128><<<batch, 256, smem, (cudaStream_t)stream>>>(M, N, K, alpha, A, ars, acs, B, brs,
                                                                               bcs, beta, C, crs, ccs, sa, sb, sc);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

extern "C" int bilu_diag_dgemm(int M, int N, int K, double alpha, const double *A, int64_t ars, int64_t acs,
                               const double *B, int64_t brs, int64_t bcs, double beta, double *C, int64_t crs,
                               int64_t ccs, int batch, int64_t sa, int64_t sb, int64_t sc, void *stream) {
  if (M < 0 || N < 0 || K < 0 || batch < 1) return 1;
  if (M == 0 || N == 0) return 0;
  if (!A || !B || !C) return 1;
  bilu::diag_dgemm_kernel<<<batch, 256, 0, (cudaStream_t)stream>>>(M, N, K, alpha, A, ars, acs, B, brs, bcs, beta,
                                                                   C, crs, ccs, sa, sb, sc);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
