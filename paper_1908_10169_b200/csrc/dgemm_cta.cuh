// dgemm_cta.cuh -- CTA-cooperative FP64 GEMM on the tensor pipe (DMMA) for sm_100a.
//
// FP64 has no tcgen05 kind on Blackwell (ptxas rejects .kind::f64);
// the FP64 tensor path is the warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).
// This routine computes
//     C[M x N] = alpha * A[M x K] * B[K x N] + beta * C
// for operands with arbitrary (row, col) strides in global or shared memory, by
// 64 x 64 output tiles: the K dimension is staged through shared memory in slabs of
// 16 (A slab 64 x 16, B slab stored transposed 64 x 16, row stride 20 doubles so the
// fragment loads are two wavefronts per warp, the minimum for 64-bit lanes), the
// next slab is prefetched into registers while the current one is multiplied.
// Warps tile the 64 x 64 output as WM x WN; each warp owns (64/WM) x (64/WN)
// accumulators in registers (m8n8 fragments: lane holds C[lane/4][2*(lane%4)+{0,1}]).
// Used for the Schur-update products of the factor kernel (Fig. 2)
// and the merged panels of progressive aggregation.
#pragma once
#include <stdint.h>

namespace bilu {

// dynamic shared memory of the calling kernel: a generic pointer into it, re-derived from this
// array, lets the compiler emit 32-bit ld/st.shared instead of generic 64-bit accesses
extern __shared__ double dyn_sm[];
template <class T>
__device__ __forceinline__ T *as_shared(T *p) {
  const unsigned off = (unsigned)__cvta_generic_to_shared(p) - (unsigned)__cvta_generic_to_shared(dyn_sm);
  return (T *)((char *)dyn_sm + off);
}

struct DMat {
  const double *p;
  int64_t rs, cs;   // element (i, j) at p[i * rs + j * cs]
};

__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int GT = 64;        // output tile (GT x GT)
constexpr int GK = 16;        // K slab
constexpr int GS = GK + 4;    // shared row stride (doubles)
constexpr int DGEMM_SMEM_DOUBLES = 2 * GT * GS;

// smem: DGEMM_SMEM_DOUBLES doubles (20 KB).  All threads of the CTA must call it.
// Ends with __syncthreads().  C may alias neither A nor B.
// Epilogue functor: epi(i, j, acc) receives every output element (i < M, j < N) once.
template <int NTH, class Epi>
__device__ __forceinline__ void cta_dgemm_epi_impl(int M, int N, int K, DMat A, DMat B, Epi epi, double *smem) {
  constexpr int NWARP = NTH / 32;
  constexpr int WN = NWARP >= 4 ? 4 : NWARP;          // warps along n
  constexpr int WM = NWARP / WN;                       // warps along m
  constexpr int TM = GT / WM / 8, TN = GT / WN / 8;    // m8n8 fragments per warp
  constexpr int LD = GT * GK / NTH;                    // staged elements per thread per operand
  static_assert(NWARP % WN == 0 && TM >= 1 && TN >= 1 && LD >= 1, "tile shape");
  double *As = smem, *Bs = smem + GT * GS;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wm = wid / WN, wn = wid % WN;
  const int g = lane >> 2, q = lane & 3;
  // staging maps: along k if that stride is 1 (coalesced), else along m / n
  const bool a_k = A.cs == 1, b_k = B.rs == 1;
  for (int m0 = 0; m0 < M; m0 += GT) {
    for (int n0 = 0; n0 < N; n0 += GT) {
      double acc[TM][TN][2];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      double ra[LD], rb[LD];
      auto load = [&](int k0) {
#pragma unroll
        for (int l = 0; l < LD; ++l) {
          const int e = tid + l * NTH;
          int mi, ki;
          if (a_k) { mi = e / GK; ki = e % GK; } else { mi = e % GT; ki = e / GT; }
          const int gm = m0 + mi, gk = k0 + ki;
          ra[l] = (gm < M && gk < K) ? A.p[gm * A.rs + gk * A.cs] : 0.0;
          int ni, kj;
          if (b_k) { ni = e / GK; kj = e % GK; } else { ni = e % GT; kj = e / GT; }
          const int gn = n0 + ni, gk2 = k0 + kj;
          rb[l] = (gn < N && gk2 < K) ? B.p[gk2 * B.rs + gn * B.cs] : 0.0;
        }
      };
      auto store = [&]() {
#pragma unroll
        for (int l = 0; l < LD; ++l) {
          const int e = tid + l * NTH;
          if (a_k) As[(e / GK) * GS + e % GK] = ra[l]; else As[(e % GT) * GS + e / GT] = ra[l];
          if (b_k) Bs[(e / GK) * GS + e % GK] = rb[l]; else Bs[(e % GT) * GS + e / GT] = rb[l];
        }
      };
      load(0);
      for (int k0 = 0; k0 < K; k0 += GK) {
        __syncthreads();
        store();
        __syncthreads();
        if (k0 + GK < K) load(k0 + GK);
#pragma unroll
        for (int kk = 0; kk < GK; kk += 4) {
          double af[TM], bf[TN];
#pragma unroll
          for (int i = 0; i < TM; ++i) af[i] = As[(wm * TM * 8 + i * 8 + g) * GS + kk + q];
#pragma unroll
          for (int j = 0; j < TN; ++j) bf[j] = Bs[(wn * TN * 8 + j * 8 + g) * GS + kk + q];
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
      }
      // epilogue
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gm = m0 + wm * TM * 8 + i * 8 + g;
            const int gn = n0 + wn * TN * 8 + j * 8 + 2 * q + h;
            if (gm < M && gn < N) epi(gm, gn, acc[i][j][h]);
          }
    }
  }
  __syncthreads();
}

template <int NTH, class Epi>
__device__ void cta_dgemm_epi(int M, int N, int K, DMat A, DMat B, Epi epi, double *smem) {
  if (__isShared(smem)) cta_dgemm_epi_impl<NTH>(M, N, K, A, B, epi, as_shared(smem));
  else cta_dgemm_epi_impl<NTH>(M, N, K, A, B, epi, smem);
}

// Tall-skinny product C[M x N] = A[M x K] * B[K x N] with K, N <= NMAX: B is staged once
// in shared memory (Bs, K rows of ldb = NMAX + 4 doubles, zero-padded to NMAX columns) and
// every warp streams its own 8-row tiles of A from global memory (one m8n8k4 A fragment
// per k-step: lane (g, q) loads A[row g][k + q]), so many independent tiles are in flight
// -- the shape of the Schur-update products (m rows of L_J x b_J) and of the panel
// scaling W·D_K.  Callers stage B with tsgemm_stage_b; epi(i, j, acc) gets each element.
template <int NMAX>
struct TsB {
  static constexpr int LDB = NMAX + 4;
};

// Bs[k * LDB + n] = B(k, n) for k < K, n < N, 0 for N <= n < NMAX.  CTA-wide; ends with a barrier.
template <int NTH, int NMAX>
__device__ void tsgemm_stage_b(int K, int N, DMat B, double *Bs) {
  constexpr int LDB = TsB<NMAX>::LDB;
  for (int e = threadIdx.x; e < K * NMAX; e += NTH) {
    const int k = e / NMAX, n = e - k * NMAX;
    Bs[k * LDB + n] = n < N ? B.p[k * B.rs + n * B.cs] : 0.0;
  }
  __syncthreads();
}

// rmax (optional): rmax[i] = max_j |C(i, j)| (every tile spans all N columns, so a 4-lane
// shuffle reduction gives complete row maxima)
template <int NTH, int NMAX, class Epi>
__device__ __forceinline__ void cta_tsgemm_impl(int M, int N, int K, DMat A, const double *Bs, Epi epi, double *rmax) {
  constexpr int NWARP = NTH / 32, NF = NMAX / 8, LDB = TsB<NMAX>::LDB;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int nf = (N + 7) >> 3;
  for (int m0 = wid * 8; m0 < M; m0 += NWARP * 8) {
    const int row = m0 + g;
    const bool rv = row < M;
    const double *ar = A.p + (int64_t)(rv ? row : 0) * A.rs;
    double acc[NF][2];
#pragma unroll
    for (int f = 0; f < NF; ++f) acc[f][0] = acc[f][1] = 0.0;
    // A fragments of 8 k-steps loaded together (independent loads in flight), then used
    for (int kc = 0; kc < K; kc += 32) {
      double a8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int kk = kc + 4 * u + q;
        a8[u] = (rv && kk < K) ? ar[(int64_t)kk * A.cs] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int kk = kc + 4 * u + q;
        if (kc + 4 * u >= K) break;                 // warp-uniform
        const bool kv = kk < K;
        const double *br = Bs + (kv ? kk : 0) * LDB + g;
#pragma unroll
        for (int f = 0; f < NF; ++f)
          if (f < nf) dmma_8x8x4(acc[f][0], acc[f][1], a8[u], kv ? br[f * 8] : 0.0);
      }
    }
    double mx = 0.0;
#pragma unroll
    for (int f = 0; f < NF; ++f)
      if (f < nf)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = f * 8 + 2 * q + h;
          if (rv && col < N) {
            epi(row, col, acc[f][h]);
            mx = fmax(mx, fabs(acc[f][h]));
          }
        }
    if (rmax) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      if (rv && q == 0) rmax[row] = mx;
    }
  }
}

template <int NTH, int NMAX, class Epi>
__device__ void cta_tsgemm(int M, int N, int K, DMat A, const double *Bs, Epi epi, double *rmax = nullptr) {
  if (__isShared(Bs)) cta_tsgemm_impl<NTH, NMAX>(M, N, K, A, as_shared(Bs), epi, rmax);
  else cta_tsgemm_impl<NTH, NMAX>(M, N, K, A, Bs, epi, rmax);
}

struct EpiAxpby {
  double alpha, beta; double *C; int64_t crs, ccs;
  __device__ __forceinline__ void operator()(int i, int j, double v) const {
    double *c = C + i * crs + j * ccs;
    *c = beta == 0.0 ? alpha * v : fma(alpha, v, beta * *c);
  }
};

// C = alpha A B + beta C
template <int NTH>
__device__ void cta_dgemm(int M, int N, int K, double alpha, DMat A, DMat B, double beta, double *C, int64_t crs,
                          int64_t ccs, double *smem) {
  cta_dgemm_epi<NTH>(M, N, K, A, B, EpiAxpby{alpha, beta, C, crs, ccs}, smem);
}

}  // namespace bilu
