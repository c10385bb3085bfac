"""Extract gj_invert_blk from bilu_factor.cu into a small standalone microbenchmark
(seconds to compile instead of minutes): python tools/micro/mk_gj_standalone.py && nvcc ..."""
import os
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
s = open(os.path.join(R, 'paper_1908_10169_b200/csrc/bilu_factor.cu')).read()
a = s.index('#ifndef BILU_GJ_BLK_MIN')
b_ = s.index('// D_K = P_K^{-1} in place (P column-major b x b in shared memory; b > 8 needs 2 b^2 doubles')
fn = s[a:b_]
src = '''#include <cstdio>
#include <vector>
#include <cmath>
#include <climits>
namespace bilu {
constexpr int NT = 512;
struct Shared { int piv; };
''' + fn + '''
}
using namespace bilu;
__global__ void __launch_bounds__(NT, 1) gjk(const double *A, int b, double *out, long long *cyc) {
  extern __shared__ double sm[];
  __shared__ Shared S;
  double *P = sm, *fcol = sm + 2 * 64 * 64;
  int *ipiv = (int *)(fcol + 3 * 64);
  bool s = false;
  for (int rep = 0; rep < 2; ++rep) {
    for (int i = threadIdx.x; i < b * b; i += NT) P[i] = A[i];
    __syncthreads();
    long long t0 = clock64();
    s = gj_invert_blk<8>(P, b, ipiv, fcol, S);
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = s; }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < b * b; i += NT) out[i] = P[i];
}
int main() {
  for (int b : {9, 16, 17, 24, 32, 33, 40, 48, 56, 63, 64}) {
    for (int kind = 0; kind < 3; ++kind) {   // 0: random, 1: needs pivoting everywhere (tiny diagonal), 2: singular
      std::vector<double> A(b * b);
      srand(b * 7 + kind);
      for (int j = 0; j < b; ++j) for (int i = 0; i < b; ++i) A[i + j * b] = (rand() / (double)RAND_MAX - 0.5);
      if (kind == 1) for (int i = 0; i < b; ++i) A[i + i * b] = 1e-9;
      if (kind == 2) for (int i = 0; i < b; ++i) A[i + 3 * b] = 2.0 * A[i + 1 * b];
      double *dA, *dO; long long *dc;
      cudaMalloc(&dA, b * b * 8); cudaMalloc(&dO, b * b * 8); cudaMalloc(&dc, 16);
      cudaMemcpy(dA, A.data(), b * b * 8, cudaMemcpyHostToDevice);
      cudaFuncSetAttribute(gjk, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
      gjk<<<1, NT, 100000>>>(dA, b, dO, dc);
      long long c[2];
      cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
      std::vector<double> D(b * b);
      cudaMemcpy(D.data(), dO, b * b * 8, cudaMemcpyDeviceToHost);
      double err = 0;
      for (int i = 0; i < b; ++i) for (int j = 0; j < b; ++j) {
        double s = 0; for (int t = 0; t < b; ++t) s += D[i + t * b] * A[t + j * b];
        err = fmax(err, fabs(s - (i == j)));
      }
      printf("b=%d kind=%d cycles=%lld (%.1f us) sing=%lld err=%.2e %s\\n", b, kind, c[0], c[0] / 1965.0, c[1], err,
             cudaGetErrorString(cudaGetLastError()));
      cudaFree(dA); cudaFree(dO); cudaFree(dc);
    }
  }
}
'''
open(os.path.join(R, 'tools/micro/gj_standalone.cu'), 'w').write(src)
