// fine-grained cycle split of one register Gauss-Jordan step (thread 0 and a lane of warp 14)
#include <cstdio>
#include <vector>
#include <climits>
constexpr int NT = 512;
__global__ void __launch_bounds__(NT, 1) k(const double *A, int b, long long *cyc, double *out) {
  constexpr int BC = 64, RP = 8, G = NT / BC;
  extern __shared__ double P[];
  __shared__ double pv[4 * G];
  const int tid = threadIdx.x, j = tid % BC, g = tid / BC, r0 = g * RP;
  const bool act = j < b;
  const long long bb = (long long)b * b;
  for (int i = tid; i < b * b; i += NT) P[i] = A[i];
  __syncthreads();
  double x[RP];
#pragma unroll
  for (int u = 0; u < RP; ++u) x[u] = (act && r0 + u < b) ? P[r0 + u + j * b] : 0.0;
  auto slot_v = [&](int par) { return pv + par * 2 * G; };
  auto slot_i = [&](int par) { return (int *)(pv + par * 2 * G + G); };
  auto publish = [&](int col, int from) {
    double av[RP], sv[RP]; int iv[RP];
#pragma unroll
    for (int u = 0; u < RP; ++u) { const bool ok = r0 + u >= from && r0 + u < b; av[u] = ok ? fabs(x[u]) : -1.0; sv[u] = x[u]; iv[u] = r0 + u; }
#pragma unroll
    for (int w = 1; w < RP; w <<= 1)
#pragma unroll
      for (int u = 0; u + w < RP; u += 2 * w)
        if (av[u + w] > av[u]) { av[u] = av[u + w]; sv[u] = sv[u + w]; iv[u] = iv[u + w]; }
    slot_v(col & 1)[g] = av[0] < 0.0 ? 0.0 : sv[0];
    slot_i(col & 1)[g] = av[0] < 0.0 ? INT_MAX : iv[0];
  };
  if (j == 0) publish(0, 0);
  __syncthreads();
  long long c[8] = {0};
  for (int kk = 0; kk < b; ++kk) {
    long long t0 = clock64();
    const double *cur = (kk & 1) ? P + bb : P;
    double *nxt = (kk & 1) ? P : P + bb;
    double vv[G], av[G]; int ii[G];
#pragma unroll
    for (int q = 0; q < G; ++q) { vv[q] = slot_v(kk & 1)[q]; ii[q] = slot_i(kk & 1)[q]; }
#pragma unroll
    for (int q = 0; q < G; ++q) av[q] = fabs(vv[q]);
#pragma unroll
    for (int w = 1; w < G; w <<= 1)
#pragma unroll
      for (int q = 0; q + w < G; q += 2 * w)
        if (av[q + w] > av[q]) { av[q] = av[q + w]; vv[q] = vv[q + w]; ii[q] = ii[q + w]; }
    const double vb = vv[0]; const int bi = ii[0];
    if (!(av[0] > 0.0)) break;
    long long t1 = clock64();
    long long t2 = t1, t3 = t1, t4 = t1;
    if (act) {
      double cv[RP];
#pragma unroll
      for (int u = 0; u < RP; ++u) cv[u] = (r0 + u < b) ? cur[r0 + u + (long long)kk * b] : 0.0;
      const double rowbi = cur[bi + (long long)j * b], rb = cur[kk + (long long)j * b], ckk = cur[kk + (long long)kk * b];
      const double d = 1.0 / vb;
      const double pr = (j == kk) ? d : rowbi * d;
      t2 = clock64();
#pragma unroll
      for (int u = 0; u < RP; ++u) {
        const int i = r0 + u;
        if (i == kk) x[u] = pr;
        else { const double xi = (i == bi) ? rb : x[u]; const double f = (i == bi) ? ckk : cv[u]; x[u] = ((j == kk) ? 0.0 : xi) - f * pr; }
      }
#pragma unroll
      for (int u = 0; u < RP; ++u) if (r0 + u < b) nxt[r0 + u + (long long)j * b] = x[u];
      t3 = clock64();
      if (j == kk + 1) publish(kk + 1, kk + 1);
      t4 = clock64();
    }
    __syncthreads();
    long long t5 = clock64();
    c[0] += t1 - t0; c[1] += t2 - t1; c[2] += t3 - t2; c[3] += t4 - t3; c[4] += t5 - t4;
  }
  if (tid == 0) for (int i = 0; i < 5; ++i) cyc[i] = c[i];
  if (tid == 64 * 7 + 33) for (int i = 0; i < 5; ++i) cyc[8 + i] = c[i];
#pragma unroll
  for (int u = 0; u < RP; ++u) out[tid * RP + u] = x[u];
}
int main() {
  for (int b : {40, 64}) {
    std::vector<double> A(b * b);
    for (int i = 0; i < b * b; ++i) A[i] = rand() / (double)RAND_MAX - 0.5;
    double *dA, *dO; long long *dc;
    cudaMalloc(&dA, b * b * 8); cudaMalloc(&dO, NT * 8 * 8); cudaMalloc(&dc, 128);
    cudaMemcpy(dA, A.data(), b * b * 8, cudaMemcpyHostToDevice);
    for (int r = 0; r < 3; ++r) k<<<1, NT, 2 * b * b * 8>>>(dA, b, dc, dO);
    long long c[16]; cudaMemcpy(c, dc, 128, cudaMemcpyDeviceToHost);
    printf("b=%d per step t0: pivot %.0f loads+div %.0f update+store %.0f publish %.0f barrier %.0f | t481: %.0f %.0f %.0f %.0f %.0f\n", b,
           c[0] / (double)b, c[1] / (double)b, c[2] / (double)b, c[3] / (double)b, c[4] / (double)b, c[8] / (double)b,
           c[9] / (double)b, c[10] / (double)b, c[11] / (double)b, c[12] / (double)b);
  }
}
