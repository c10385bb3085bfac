// Latency probe: one CTA of 512 threads, each thread chases `steps` dependent 64-byte reads at
// pseudo-random offsets inside a region of `mb` MB (inside a 6 GB allocation).  Compares the
// per-access latency for regions that fit L2, miss L2 but fit the TLB reach, and beyond.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void chase(const unsigned long long *buf, unsigned long long words, int steps, unsigned long long *out,
                      long long *cyc) {
  unsigned long long x = (threadIdx.x * 2654435761ull) % words;
  unsigned long long acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) {
    const unsigned long long v = buf[x];
    acc += v;
    x = (x * 6364136223846793005ull + 1442695040888963407ull + v) % words;
    x &= ~7ull;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  const size_t total = 6ull << 30;
  unsigned long long *buf, *out; long long *cyc;
  cudaMalloc(&buf, total); cudaMemset(buf, 0, total);
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
  int mbs[] = {16, 64, 256, 1024, 2048, 4096, 6000};
  for (int m : mbs) {
    unsigned long long words = (unsigned long long)m * (1ull << 20) / 8;
    for (int rep = 0; rep < 2; ++rep) {
      chase<<<1, 512>>>(buf, words, 64, out, cyc);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      if (rep) printf("region %5d MB: %.0f cycles per dependent access (512 threads in flight)\n", m, c / 64.0);
    }
  }
  // one thread only (pure latency)
  for (int m : mbs) {
    unsigned long long words = (unsigned long long)m * (1ull << 20) / 8;
    chase<<<1, 1>>>(buf, words, 256, out, cyc);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("region %5d MB: %.0f cycles per access (1 thread)\n", m, c / 256.0);
  }
  return 0;
}
