// FP64 peak microbenchmark: DMMA (mma.sync m8n8k4 f64) vs DFMA, on the B200.
// Measures the roofline denominator for FP64 (not in MEASURED_PEAKS.json).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template<int NACC>
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

template<int NACC>
__global__ void dfma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(c[i]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 1234.5) out[0] = s;
}

template<typename F>
double timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  double* out; CK(cudaMalloc(&out, 8));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 20000;
  for (int tpb : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int grid = sms * bps;
      double ms = timeit([&] { dmma_kernel<8><<<grid, tpb>>>(out, iters); });
      double flops = (double)grid * (tpb / 32) * iters * 8 * 512.0;
      printf("DMMA m8n8k4 tpb=%d blocks/SM=%d : %.2f TFLOP/s\n", tpb, bps, flops / ms / 1e9);
      ms = timeit([&] { dfma_kernel<16><<<grid, tpb>>>(out, iters); });
      flops = (double)grid * tpb * iters * 16 * 2.0;
      printf("DFMA          tpb=%d blocks/SM=%d : %.2f TFLOP/s\n", tpb, bps, flops / ms / 1e9);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
