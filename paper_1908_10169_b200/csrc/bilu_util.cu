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

extern "C" cudaError_t bilu_launch_permute(double *y, const double *x, const int32_t *perm,
                                           int32_t n, int inverse, cudaStream_t st) {
  permute_kernel<<<grid_for(n), 256, 0, st>>>(y, x, perm, n, inverse);
  return cudaGetLastError();
}

}  // namespace bilu
