// dependent-chain latencies (cycles per op) of DFMA, DADD, DSETP+select, double divide, LDS.64
#include <cstdio>
__global__ void k(double a, double b, long long *o, double *sink, int n) {
  __shared__ double sh[64];
  sh[threadIdx.x & 63] = threadIdx.x;
  __syncthreads();
  double x = a; long long t0, t1;
  t0 = clock64(); for (int i = 0; i < n; ++i) x = fma(x, b, a); t1 = clock64(); o[0] = (t1 - t0) / n;
  t0 = clock64(); for (int i = 0; i < n; ++i) x = x + b; t1 = clock64(); o[1] = (t1 - t0) / n;
  t0 = clock64(); for (int i = 0; i < n; ++i) x = (x > b) ? x - b : x + a; t1 = clock64(); o[2] = (t1 - t0) / n;
  t0 = clock64(); for (int i = 0; i < n; ++i) x = a / x; t1 = clock64(); o[3] = (t1 - t0) / n;
  int idx = 0;
  t0 = clock64(); for (int i = 0; i < n; ++i) { x = sh[idx]; idx = ((int)x) & 63; } t1 = clock64(); o[4] = (t1 - t0) / n;
  float y = (float)a;
  t0 = clock64(); for (int i = 0; i < n; ++i) y = fmaf(y, (float)b, (float)a); t1 = clock64(); o[5] = (t1 - t0) / n;
  sink[threadIdx.x] = x + y;
}
int main() {
  long long *o; double *s; cudaMalloc(&o, 64); cudaMalloc(&s, 4096);
  k<<<1, 32>>>(1.0000001, 0.9999999, o, s, 1000); k<<<1, 32>>>(1.0000001, 0.9999999, o, s, 1000);
  long long h[6]; cudaMemcpy(h, o, 48, cudaMemcpyDeviceToHost);
  printf("latency cycles: dfma %lld dadd %lld dsetp+sel %lld ddiv %lld lds %lld ffma %lld\n", h[0], h[1], h[2], h[3], h[4], h[5]);
}
