// pointer-chase latency: buf[i] = next index (stride-permutation over a region), 1 thread
#include <cstdio>
#include <cuda_runtime.h>
__global__ void init(unsigned *buf, unsigned n, unsigned stride) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    buf[i] = (unsigned)(((unsigned long long)i + stride) % n);
}
__global__ void chase(const unsigned *buf, int steps, unsigned *out, long long *cyc) {
  unsigned x = 0;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) x = buf[x];
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}
__global__ void chase_cg(const unsigned *buf, int steps, unsigned *out, long long *cyc) {
  unsigned x = 0;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) x = __ldcg(buf + x);
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}
int main() {
  unsigned *buf, *out; long long *cyc; char *flush;
  const size_t N = 1ull << 28;   // 1 GB of uint32
  cudaMalloc(&buf, N * 4); cudaMalloc(&out, 64); cudaMalloc(&cyc, 8); cudaMalloc(&flush, 512 << 20);
  for (unsigned mb : {1u, 16u, 64u, 1024u}) {
    unsigned n = mb * (1u << 18);
    unsigned stride = 4096 * 16 + 33;     // > a page apart
    init<<<1024, 256>>>(buf, n, stride % n);
    cudaMemset(flush, 1, 512 << 20);
    for (int k = 0; k < 2; ++k) {
      long long c;
      chase<<<1, 1>>>(buf, 2000, out, cyc); cudaDeviceSynchronize(); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%5u MB chase %s: %.0f cycles/load\n", mb, k ? "warm" : "cold", c / 2000.0);
    }
    long long c;
    cudaMemset(flush, 2, 512 << 20);
    chase_cg<<<1, 1>>>(buf, 2000, out, cyc); cudaDeviceSynchronize(); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%5u MB chase ldcg cold: %.0f cycles/load\n", mb, c / 2000.0);
  }
  return 0;
}
