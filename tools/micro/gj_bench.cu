// Microbenchmark of the pivot-block inverse (a-6) inside one 512-thread CTA: cycles of
// gj_invert for b = 16..64 (register version) and the shared-memory version, plus the
// max |D P - I| check.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I include -I paper_1908_10169_b200/csrc tools/micro/gj_bench.cu -o /tmp/gj_bench
#define BILU_GJ_BLK_MIN 1000
#include "../../paper_1908_10169_b200/csrc/bilu_factor.cu"
__device__ bool gj_invert_reg_only(double *P, int b, int *ipiv, double *fcol, bilu::Shared &S, bool reg) { return bilu::gj_invert(P, b, ipiv, fcol, S, reg); }
#include <cstdio>
#include <vector>
#include <cmath>
using namespace bilu;
__global__ void __launch_bounds__(NT, 1) gjk(const double *A, int b, int variant, double *out, long long *cyc) {
  extern __shared__ double sm[];
  __shared__ Shared S;
  double *P = sm, *fcol = sm + 2 * 64 * 64;   // room for the padded copies (b <= 64)
  int *ipiv = (int *)(fcol + 3 * b);
  bool s = false;
  for (int rep = 0; rep < 2; ++rep) {       // rep 0: cold instruction cache, rep 1: warm
    for (int i = threadIdx.x; i < b * b; i += NT) P[i] = A[i];
    __syncthreads();
    long long t0 = clock64();
    if (variant == 2) s = gj_invert_blk<8>(P, b, ipiv, fcol, S);        // 2: blocked (panels of 8)
    else if (variant == 3) s = gj_invert_blk<16>(P, b, ipiv, fcol, S);  // 3: blocked (panels of 16)
    else s = gj_invert_reg_only(P, b, ipiv, fcol, S, variant == 0);   // 0: registers, 1: shared-memory CTA version
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[rep] = t1 - t0; cyc[2] = s; }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < b * b; i += NT) out[i] = P[i];
}
int main() {
  for (int b : {9, 16, 17, 24, 32, 33, 40, 48, 56, 63, 64}) {
    std::vector<double> A(b * b);
    srand(b);
    for (int j = 0; j < b; ++j) for (int i = 0; i < b; ++i) A[i + j * b] = (rand() / (double)RAND_MAX - 0.5) + (i == j ? 0.0 : 0.0);
    double *dA, *dO; long long *dc;
    cudaMalloc(&dA, b * b * 8); cudaMalloc(&dO, b * b * 8); cudaMalloc(&dc, 24);
    cudaMemcpy(dA, A.data(), b * b * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(gjk, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    for (int v = 0; v < 4; ++v) {
      long long c[3];
      for (int rep = 0; rep < 3; ++rep) gjk<<<1, NT, 100000>>>(dA, b, v, dO, dc);
      cudaMemcpy(c, dc, 24, cudaMemcpyDeviceToHost);
      std::vector<double> D(b * b);
      cudaMemcpy(D.data(), dO, b * b * 8, cudaMemcpyDeviceToHost);
      double err = 0;
      for (int i = 0; i < b; ++i) for (int j = 0; j < b; ++j) {
        double s = 0; for (int t = 0; t < b; ++t) s += D[i + t * b] * A[t + j * b];
        err = fmax(err, fabs(s - (i == j)));
      }
      printf("b=%d variant=%d cycles cold=%lld warm=%lld (%.1f us) sing=%lld err=%.2e %s\n", b, v, c[0], c[1], c[1] / 1965.0, c[2], err,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
}
