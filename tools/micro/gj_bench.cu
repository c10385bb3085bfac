// Microbenchmark of the pivot-block inverse (a-6) inside one 512-thread CTA: cycles of
// gj_invert for b = 16..64 (register version) and the shared-memory version, plus the
// max |D P - I| check.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I include -I paper_1908_10169_b200/csrc tools/micro/gj_bench.cu -o /tmp/gj_bench
#include "../../paper_1908_10169_b200/csrc/bilu_factor.cu"
#include <cstdio>
#include <vector>
#include <cmath>
using namespace bilu;
__global__ void __launch_bounds__(NT, 1) gjk(const double *A, int b, int variant, double *out, long long *cyc) {
  extern __shared__ double sm[];
  __shared__ Shared S;
  double *P = sm, *fcol = sm + 2 * 64 * 64;   // room for the padded copies (b <= 64)
  int *ipiv = (int *)(fcol + 3 * b);
  for (int i = threadIdx.x; i < b * b; i += NT) P[i] = A[i];
  __syncthreads();
  long long t0 = clock64();
  bool s;
  s = gj_invert(P, b, ipiv, fcol, S, variant == 0);   // 0: registers, 1: shared-memory CTA version
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = s; }
  for (int i = threadIdx.x; i < b * b; i += NT) out[i] = P[i];
}
int main() {
  for (int b : {9, 16, 24, 32, 33, 40, 56, 64}) {
    std::vector<double> A(b * b);
    srand(b);
    for (int j = 0; j < b; ++j) for (int i = 0; i < b; ++i) A[i + j * b] = (rand() / (double)RAND_MAX - 0.5) + (i == j ? 0.0 : 0.0);
    double *dA, *dO; long long *dc;
    cudaMalloc(&dA, b * b * 8); cudaMalloc(&dO, b * b * 8); cudaMalloc(&dc, 16);
    cudaMemcpy(dA, A.data(), b * b * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(gjk, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    for (int v = 0; v < 2; ++v) {
      long long c[2];
      for (int rep = 0; rep < 3; ++rep) gjk<<<1, NT, 100000>>>(dA, b, v, dO, dc);
      cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
      std::vector<double> D(b * b);
      cudaMemcpy(D.data(), dO, b * b * 8, cudaMemcpyDeviceToHost);
      double err = 0;
      for (int i = 0; i < b; ++i) for (int j = 0; j < b; ++j) {
        double s = 0; for (int t = 0; t < b; ++t) s += D[i + t * b] * A[t + j * b];
        err = fmax(err, fabs(s - (i == j)));
      }
      printf("b=%d variant=%d cycles=%lld (%.1f us) sing=%lld err=%.2e %s\n", b, v, c[0], c[0] / 1965.0, c[1], err,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
}
