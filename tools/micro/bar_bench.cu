// cycles per __syncthreads for a 512-thread CTA, with and without a dependent double divide
#include <cstdio>
__global__ void __launch_bounds__(512, 1) k(int iters, int mode, long long *out, double *sink) {
  __shared__ double buf[2][64];
  const int tid = threadIdx.x;
  double x = tid;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode >= 1 && tid < 64) buf[i & 1][tid] = x;
    __syncthreads();
    if (mode >= 1) x += buf[i & 1][(tid + 1) & 63];
    if (mode >= 2) x = 1.0 / x;
    if (mode >= 3) { __syncthreads(); }
  }
  long long t1 = clock64();
  if (tid == 0) out[mode] = (t1 - t0) / iters;
  sink[tid] = x;
}
int main() {
  long long *o; double *s; cudaMalloc(&o, 64); cudaMalloc(&s, 4096 * 8);
  for (int m = 0; m < 4; ++m) { k<<<1, 512>>>(1000, m, o, s); k<<<1, 512>>>(1000, m, o, s); }
  long long h[4]; cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
  printf("cycles/iter: bar only %lld, +smem %lld, +div %lld, +2nd bar %lld\n", h[0], h[1], h[2], h[3]);
}
