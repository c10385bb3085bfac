// bilu_krylov.cu -- device kernels of the preconditioned GMRES(m) solver (bilu_gmres):
// the Krylov method the paper drives BILU with ("restarted GMRES ... restart length 30
// ... the vector b with all ones").  HBM-bound vector kernels: CSR
// SpMV with A, two-pass deterministic dot products, AXPYs whose coefficient is read from
// device memory (no host round trip inside modified Gram-Schmidt), the solution update.
#include <cuda_runtime.h>
#include <stdint.h>

namespace bilu {

constexpr int KT = 256;

// y = A x, A in CSR (original ordering); LPR lanes per row (power of two <= 32)
template <int LPR>
__global__ void __launch_bounds__(KT) spmv_kernel(int n, const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                                  const double *__restrict__ val, const double *__restrict__ x,
                                                  double *__restrict__ y) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / LPR;
  const int sub = threadIdx.x % LPR;
  for (int64_t row = gt / LPR; row < n; row += stride) {
    double acc = 0.0;
    for (int64_t p = rp[row] + sub; p < rp[row + 1]; p += LPR) acc = fma(val[p], __ldg(x + ci[p]), acc);
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (sub == 0) y[row] = acc;
  }
}

// partials[block] = sum of x_i y_i over the block's grid-stride share (fixed order)
__global__ void __launch_bounds__(KT) dot_partial_kernel(int n, const double *__restrict__ x,
                                                         const double *__restrict__ y, double *partials) {
  __shared__ double sw[KT / 32];
  double acc = 0.0;
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) acc = fma(x[i], y[i], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < KT / 32; ++w) s += sw[w];
    partials[blockIdx.x] = s;
  }
}

// out = sum of partials[0..np) (one warp, fixed order); sqrt_out: also out[1] = sqrt(out[0])
__global__ void dot_final_kernel(const double *partials, int np, double *out, int sqrt_out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += 32) acc += partials[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (threadIdx.x == 0) {
    out[0] = acc;
    if (sqrt_out) out[1] = sqrt(acc);
  }
}

// y += sign * (*coef) * x
__global__ void __launch_bounds__(KT) axpy_dev_kernel(int n, const double *coef, double sign, const double *__restrict__ x,
                                                      double *__restrict__ y) {
  const double a = sign * *coef;
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) y[i] = fma(a, x[i], y[i]);
}

// y = x / (*coef)
__global__ void __launch_bounds__(KT) scale_dev_kernel(int n, const double *coef, const double *__restrict__ x,
                                                       double *__restrict__ y) {
  const double a = 1.0 / *coef;
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) y[i] = a * x[i];
}

// x += sum_j Z[j] c[j] (k vectors of length n, row stride ld)
__global__ void __launch_bounds__(KT) update_kernel(int n, int k, const double *__restrict__ Z, int64_t ld,
                                                    const double *__restrict__ c, double *__restrict__ x) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) {
    double acc = x[i];
    for (int j = 0; j < k; ++j) acc = fma(Z[(int64_t)j * ld + i], c[j], acc);
    x[i] = acc;
  }
}

// r = b - r  (r holds A x on entry)
__global__ void __launch_bounds__(KT) residual_kernel(int n, const double *__restrict__ b, double *__restrict__ r) {
  for (int i = blockIdx.x * KT + threadIdx.x; i < n; i += gridDim.x * KT) r[i] = b[i] - r[i];
}

static int kgrid(int64_t n, int sms) {
  int64_t g = (n + KT - 1) / KT;
  const int64_t cap = (int64_t)sms * 8;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

extern "C" cudaError_t bilu_launch_spmv(int n, const int64_t *rp, const int32_t *ci, const double *val, const double *x,
                                        double *y, int lpr, int sms, cudaStream_t st) {
  const int g = kgrid((int64_t)n * lpr, sms * 2);
  switch (lpr) {
    case 1: spmv_kernel<1><<<g, KT, 0, st>>>(n, rp, ci, val, x, y); break;
    case 2: spmv_kernel<2><<<g, KT, 0, st>>>(n, rp, ci, val, x, y); break;
    case 4: spmv_kernel<4><<<g, KT, 0, st>>>(n, rp, ci, val, x, y); break;
    case 8: spmv_kernel<8><<<g, KT, 0, st>>>(n, rp, ci, val, x, y); break;
    case 16: spmv_kernel<16><<<g, KT, 0, st>>>(n, rp, ci, val, x, y); break;
    default: spmv_kernel<32><<<g, KT, 0, st>>>(n, rp, ci, val, x, y); break;
  }
  return cudaGetLastError();
}

// out[0] = x . y (and out[1] = sqrt if sqrt_out); partials: >= kgrid doubles
extern "C" cudaError_t bilu_launch_dot(int n, const double *x, const double *y, double *partials, double *out,
                                       int sqrt_out, int sms, cudaStream_t st) {
  const int g = kgrid(n, sms);
  dot_partial_kernel<<<g, KT, 0, st>>>(n, x, y, partials);
  dot_final_kernel<<<1, 32, 0, st>>>(partials, g, out, sqrt_out);
  return cudaGetLastError();
}

extern "C" cudaError_t bilu_launch_axpy_dev(int n, const double *coef, double sign, const double *x, double *y, int sms,
                                            cudaStream_t st) {
  axpy_dev_kernel<<<kgrid(n, sms), KT, 0, st>>>(n, coef, sign, x, y);
  return cudaGetLastError();
}

extern "C" cudaError_t bilu_launch_scale_dev(int n, const double *coef, const double *x, double *y, int sms,
                                             cudaStream_t st) {
  scale_dev_kernel<<<kgrid(n, sms), KT, 0, st>>>(n, coef, x, y);
  return cudaGetLastError();
}

extern "C" cudaError_t bilu_launch_update(int n, int k, const double *Z, int64_t ld, const double *c, double *x, int sms,
                                          cudaStream_t st) {
  if (k > 0) update_kernel<<<kgrid(n, sms), KT, 0, st>>>(n, k, Z, ld, c, x);
  return cudaGetLastError();
}

extern "C" cudaError_t bilu_launch_residual(int n, const double *b, double *r, int sms, cudaStream_t st) {
  residual_kernel<<<kgrid(n, sms), KT, 0, st>>>(n, b, r);
  return cudaGetLastError();
}

}  // namespace bilu
