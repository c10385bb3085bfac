// calibration: one CTA of 512 threads, each loads K random 64-byte rows (4 x LDG.128) from a
// 1 GB arena (L2 flushed), all issued before use (K in flight) or one at a time (dependent use)
#include <cstdio>
#include <cuda_runtime.h>
template <int K, bool DEP>
__global__ void __launch_bounds__(512, 1) ld(const double *arena, long long n, double *out, long long *cyc) {
  const int tid = threadIdx.x;
  double s = 0.0;
  unsigned long long h = tid * 2654435761ull + 12345;
  long long t0 = clock64();
  if (!DEP) {
    double2 r[K][4];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      h = h * 6364136223846793005ull + 1442695040888963407ull;
      const double2 *p = (const double2 *)(arena + ((h >> 20) % (n / 8)) * 8);
#pragma unroll
      for (int i = 0; i < 4; ++i) r[k][i] = p[i];
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int i = 0; i < 4; ++i) s += r[k][i].x + r[k][i].y;
  } else {
    for (int k = 0; k < K; ++k) {
      h = h * 6364136223846793005ull + 1442695040888963407ull + (unsigned long long)(s != 0.0);
      const double2 *p = (const double2 *)(arena + ((h >> 20) % (n / 8)) * 8);
      double2 r[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) r[i] = p[i];
#pragma unroll
      for (int i = 0; i < 4; ++i) s += r[i].x + r[i].y;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[tid] = s;
  if (tid == 0) *cyc = t1 - t0;
}
int main() {
  const long long n = 128ll << 20;
  double *arena, *out; long long *cyc; char *fl;
  cudaMalloc(&arena, n * 8); cudaMemset(arena, 0, n * 8); cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 8);
  cudaMalloc(&fl, 512 << 20);
  auto run = [&](auto k, const char *nm) {
    for (int r = 0; r < 2; ++r) {
      cudaMemset(fl, r, 512 << 20);
      k<<<1, 512>>>(arena, n, out, cyc); cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      if (r) printf("%-30s %8.0f cycles = %6.2f us\n", nm, (double)c, c / 1965.0);
    }
  };
  run(ld<1, false>, "1 row/thread");
  run(ld<4, false>, "4 rows in flight");
  run(ld<8, false>, "8 rows in flight");
  run(ld<8, true>, "8 rows dependent");
  run(ld<16, true>, "16 rows dependent");
  return 0;
}
