// Micro-benchmarks of the per-block primitives the factor kernel is built from.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long out[64];
__global__ void k_sync(int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
__global__ void k_lds_chain(int iters, int *gsrc) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int *g = s;                     // generic pointer to smem
  int x = threadIdx.x & 1023;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = g[x];
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[1] = (t1 - t0) / iters; out[10] = x; }
}
__global__ void k_ddiv(int iters, double v) {
  double x = v;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / (x + 1.0);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[2] = (t1 - t0) / iters; out[11] = (unsigned long long)(x * 1e6); }
}
__global__ void k_atomic_ret(int iters, unsigned long long *ctr) {
  unsigned long long x = 0;
  long long t0 = clock64();
  if (threadIdx.x == 0) for (int i = 0; i < iters; ++i) x += atomicAdd(ctr, 1ull + (x & 1));
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[3] = (t1 - t0) / iters; out[12] = x; }
}
__global__ void k_gload_chain(int iters, const int *g) {
  int x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __ldcg(g + x);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[4] = (t1 - t0) / iters; out[13] = x; }
}
__global__ void k_sync_after_work(int iters) {
  // barrier when warp 0 does a little smem work each time
  __shared__ double s[256];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 32) s[threadIdx.x] = s[(threadIdx.x + 1) & 31] * 1.0000001;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0) / iters;
}
int main() {
  int *g; cudaMalloc(&g, 1 << 22);
  int h[1 << 20]; for (int i = 0; i < (1 << 20); ++i) h[i] = (i * 7919 + 13) & ((1 << 20) - 1);
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  unsigned long long *ctr; cudaMalloc(&ctr, 8); cudaMemset(ctr, 0, 8);
  unsigned long long r[64];
  for (int nt : {32, 256}) {
    k_sync<<<1, nt>>>(10000); k_lds_chain<<<1, nt>>>(10000, g); k_ddiv<<<1, nt>>>(1000, 0.5);
    k_atomic_ret<<<1, nt>>>(1000, ctr); k_gload_chain<<<1, nt>>>(1000, g); k_sync_after_work<<<1, nt>>>(10000);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(r, out, sizeof(r));
    printf("threads %d: syncthreads %llu cyc, generic-smem load chain %llu cyc, fp64 1/x chain %llu cyc, "
           "atomicAdd w/ return %llu cyc, L2 load chain %llu cyc, sync after warp-0 smem work %llu cyc\n",
           nt, r[0], r[1], r[2], r[3], r[4], r[5]);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock rate attr %d kHz\n", clk);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
