// where do the cycles of one register Gauss-Jordan step go (thread 0's view)?
#include <cstdio>
#include <vector>
#include <cmath>
constexpr int NT = 512;
__global__ void __launch_bounds__(NT, 1) k(const double *A, int b, long long *cyc, double *out) {
  constexpr int BC = 64, RP = 8, G = NT / BC;
  __shared__ double pv[2 * (3 * BC + 2 * G)];
  const int tid = threadIdx.x, j = tid % BC, g = tid / BC, r0 = g * RP;
  const bool act = j < b;
  double x[RP];
#pragma unroll
  for (int u = 0; u < RP; ++u) x[u] = (act && r0 + u < b) ? A[r0 + u + j * b] : 0.0;
  auto buf = [&](int par) { return pv + par * (3 * BC + 2 * G); };
  if (j == 0) {
    double best = -1.0; int bi = 0;
#pragma unroll
    for (int u = 0; u < RP; ++u)
      if (r0 + u < b) { const double v = fabs(x[u]); if (v > best) { best = v; bi = r0 + u; } }
    double *B0 = buf(0);
    B0[3 * BC + g] = best; ((int *)(B0 + 3 * BC + G))[g] = bi;
  }
  __syncthreads();
  long long c[6] = {0, 0, 0, 0, 0, 0};
  for (int kk = 0; kk < b; ++kk) {
    long long t0 = clock64();
    double *B = buf(kk & 1);
    double best = -1.0; int bi = kk;
    for (int q = 0; q < G; ++q) {
      const double v = B[3 * BC + q];
      if (v > best) { best = v; bi = ((const int *)(B + 3 * BC + G))[q]; }
    }
    if (best == 0.0) break;
    double *rowK = B, *rowB = B + BC, *colK = B + 2 * BC;
    if (act) {
#pragma unroll
      for (int u = 0; u < RP; ++u) {
        const int i = r0 + u;
        if (i == bi) rowK[j] = x[u];
        if (i == kk) rowB[j] = x[u];
        if (j == kk && i < b) colK[i] = x[u];
      }
    }
    long long t1 = clock64();
    __syncthreads();
    long long t2 = clock64();
    if (act) {
      const double d = 1.0 / rowK[kk];
      const double pr = (j == kk) ? d : rowK[j] * d;
      const double ckk = colK[kk];
#pragma unroll
      for (int u = 0; u < RP; ++u) {
        const int i = r0 + u;
        if (i >= b) continue;
        if (i == kk) { x[u] = pr; continue; }
        const double xi = (i == bi) ? rowB[j] : x[u];
        const double f = (i == bi) ? ckk : colK[i];
        x[u] = ((j == kk) ? 0.0 : xi) - f * pr;
      }
      if (j == kk + 1) {
        double bst = -1.0; int bix = kk + 1;
#pragma unroll
        for (int u = 0; u < RP; ++u)
          if (r0 + u > kk && r0 + u < b) { const double v = fabs(x[u]); if (v > bst) { bst = v; bix = r0 + u; } }
        double *Bn = buf((kk + 1) & 1);
        Bn[3 * BC + g] = bst; ((int *)(Bn + 3 * BC + G))[g] = bix;
      }
    }
    long long t3 = clock64();
    __syncthreads();
    long long t4 = clock64();
    c[0] += t1 - t0; c[1] += t2 - t1; c[2] += t3 - t2; c[3] += t4 - t3;
  }
  if (tid == 0) for (int i = 0; i < 4; ++i) cyc[i] = c[i];
  if (tid == 64 * 7 + 3) for (int i = 0; i < 4; ++i) cyc[4 + i] = c[i];
#pragma unroll
  for (int u = 0; u < RP; ++u) out[tid * RP + u] = x[u];
}
int main() {
  int b = 40;
  std::vector<double> A(b * b);
  for (int i = 0; i < b * b; ++i) A[i] = rand() / (double)RAND_MAX - 0.5;
  double *dA, *dO; long long *dc;
  cudaMalloc(&dA, b * b * 8); cudaMalloc(&dO, NT * 8 * 8); cudaMalloc(&dc, 64);
  cudaMemcpy(dA, A.data(), b * b * 8, cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) k<<<1, NT>>>(dA, b, dc, dO);
  long long c[8]; cudaMemcpy(c, dc, 64, cudaMemcpyDeviceToHost);
  printf("b=%d per step: t0: pivot-read+publish %.0f bar1 %.0f update %.0f bar2 %.0f | t451: %.0f %.0f %.0f %.0f\n", b,
         c[0] / (double)b, c[1] / (double)b, c[2] / (double)b, c[3] / (double)b, c[4] / (double)b, c[5] / (double)b,
         c[6] / (double)b, c[7] / (double)b);
}
