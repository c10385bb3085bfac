// Microbenchmark of the narrow-block Schur update (a-5) of one target block in one CTA of
// NT threads: items = rows of contributor panels (b_J = 8 doubles, contiguous per
// contributor), each multiplied by the contributor's B (ncol x 8, the columns inside K) and
// added into a line of W (lines x 8).  Panels are spread over a 1 GB arena (DRAM-resident
// after a 512 MB flush).  Variants:
//   0  thread per item, strided (consecutive threads -> consecutive items), B from global,
//      native fp64 reductions into a global W
//   1  same, B staged in shared memory, W in shared memory with atomicAdd (CAS loop)
//   2  same as 1 but W in global memory with red.global.add.f64
//   3  same as 2 with 2 items per thread in flight
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#ifndef NT
#define NT 512
#endif
struct Con { int item_off, n, ncol, pad; long long voff, boff; int qoff, bsm; };
__device__ __forceinline__ void cp16(void *sdst, const void *gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void red_add(double *p, double v) { asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory"); }

template <int VAR>
__global__ void __launch_bounds__(NT, 1) upd(const Con *gC, int nc, int T, const double *arena, const int *line_of_item,
                                             const int *qcol, double *gW, int nlines, long long *cyc, const int *ord) {
  extern __shared__ double sm[];
  __shared__ Con C[256];
  __shared__ int coff[257];
  const int tid = threadIdx.x;
  for (int x = tid; x < nc; x += NT) { C[x] = gC[x]; coff[x] = gC[x].item_off; }
  if (tid == 0) coff[nc] = T;
  double *W = (VAR == 1 || VAR == 5 || VAR == 7) ? sm : gW;
  double *Bs = sm + nlines * 8;
  for (int x = tid; x < nlines * 8; x += NT) W[x] = 0.0;
  __syncthreads();
  long long t0 = clock64();
  if (VAR >= 4) {   // stage B operands: 8 independent loads in flight per thread
    const int nB = C[nc - 1].bsm + C[nc - 1].ncol * 8;
    for (int x0 = tid; x0 < nB; x0 += 8 * NT) {
      double r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int x = x0 + u * NT;
        r[u] = 0.0;
        if (x < nB) {
          int lo = 0, hi = nc - 1;
          while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (C[mid].bsm <= x) lo = mid; else hi = mid - 1; }
          r[u] = arena[C[lo].boff + (x - C[lo].bsm)];
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) if (x0 + u * NT < nB) Bs[x0 + u * NT] = r[u];
    }
    __syncthreads();
  } else if (VAR >= 1) {   // stage B operands
    int a = 0;
    const int nB = C[nc - 1].bsm + C[nc - 1].ncol * 8;
    for (int x = tid; x < nB; x += NT) {
      while (a + 1 < nc && C[a + 1].bsm <= x) ++a;
      Bs[x] = arena[C[a].boff + (x - C[a].bsm)];
    }
    __syncthreads();
  }
  __shared__ int sbsm[257], sqoff[257], sncol[257];
  int *Qs = (int *)(Bs + 8192);
  if (VAR >= 6) {
    for (int x = tid; x < nc; x += NT) { sbsm[x] = C[x].bsm; sqoff[x] = C[x].qoff; sncol[x] = C[x].ncol; }
    __syncthreads();
    const int nQ = C[nc - 1].qoff + C[nc - 1].ncol;
    for (int x0 = tid; x0 < nQ; x0 += 8 * NT) {
      int r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) { const int x = x0 + u * NT; r[u] = x < nQ ? qcol[x] : 0; }
#pragma unroll
      for (int u = 0; u < 8; ++u) if (x0 + u * NT < nQ) Qs[x0 + u * NT] = r[u];
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (VAR == 8 || VAR == 9) {
    // pull: items sorted by line (ord = host-sorted item ids), contiguous chunk per thread,
    // one write per line run (VAR 9: no writes at all -> cost of the arithmetic + loads)
    const int ch = (T + NT - 1) / NT;
    const int p0 = min(T, tid * ch), p1 = min(T, p0 + ch);
    double acc[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) acc[x] = 0.0;
    int gl = p0 < p1 ? line_of_item[ord[p0]] : 0;
    for (int p = p0; p < p1; ++p) {
      const int t = ord[p];
      int lo = 0, hi = nc - 1;
      while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (coff[mid] <= t) lo = mid; else hi = mid - 1; }
      double v[8];
      const double2 *pp = (const double2 *)(arena + C[lo].voff + (long long)(t - coff[lo]) * 8);
#pragma unroll
      for (int i = 0; i < 4; ++i) { double2 x = pp[i]; v[2 * i] = x.x; v[2 * i + 1] = x.y; }
      const int g2 = line_of_item[t];
      if (g2 != gl) {
        if (VAR == 8) {
#pragma unroll
          for (int x = 0; x < 8; ++x) if (acc[x] != 0.0) red_add(&W[gl * 8 + x], -acc[x]);
        }
#pragma unroll
        for (int x = 0; x < 8; ++x) acc[x] = 0.0;
        gl = g2;
      }
      const double *B = Bs + sbsm[lo];
      const int *Q = Qs + sqoff[lo];
      const int nq = sncol[lo];
      for (int q = 0; q < nq; ++q) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int i = 0; i < 8; i += 2) { d0 = fma(v[i], B[q * 8 + i], d0); d1 = fma(v[i + 1], B[q * 8 + i + 1], d1); }
        const int col = Q[q];
#pragma unroll
        for (int x = 0; x < 8; ++x) acc[x] += (x == col) ? d0 + d1 : 0.0;
      }
    }
#pragma unroll
    for (int x = 0; x < 8; ++x) if (acc[x] != 0.0) red_add(&W[gl * 8 + x], -acc[x]);
    __syncthreads();
  } else if (VAR >= 6) {
    double dummy = 0.0;
    for (int t0 = tid; t0 < T; t0 += 2 * NT) {
      double v[2][8];
      int aa[2], ln[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int t = t0 + u * NT;
        aa[u] = -1;
        if (t < T) {
          int lo = 0, hi = nc - 1;
          while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (coff[mid] <= t) lo = mid; else hi = mid - 1; }
          aa[u] = lo;
          ln[u] = line_of_item[t];
          const double2 *p = (const double2 *)(arena + C[lo].voff + (long long)(t - coff[lo]) * 8);
#pragma unroll
          for (int i = 0; i < 4; ++i) { double2 x = p[i]; v[u][2 * i] = x.x; v[u][2 * i + 1] = x.y; }
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (aa[u] < 0) continue;
        const int a = aa[u];
        const double *B = Bs + sbsm[a];
        const int *Q = Qs + sqoff[a];
        double *wl = W + (long long)ln[u] * 8;
        const int nq = sncol[a];
        for (int q = 0; q < nq; ++q) {
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int i = 0; i < 8; i += 2) { d0 = fma(v[u][i], B[q * 8 + i], d0); d1 = fma(v[u][i + 1], B[q * 8 + i + 1], d1); }
          if (VAR == 7) atomicAdd(&wl[Q[q]], -(d0 + d1));
          else if (VAR == 10) dummy += d0 + d1 + Q[q];
          else if (VAR == 11) dummy += d0 + d1;
          else red_add(&wl[Q[q]], -(d0 + d1));
        }
      }
    }
    if (dummy == 12345.0) gW[0] = dummy;
    __syncthreads();
  } else if (VAR == 4 || VAR == 5) {
    // items staged by cp.async in batches of NBI rows (double buffered), then computed from smem
    constexpr int NBI = 512;
    double *V = Bs + 8192 + 2048;
    const int nbat = (T + NBI - 1) / NBI;
    auto issue = [&](int bt) {
      double *dst = V + (bt & 1) * NBI * 8;
      // 4 x 16 B per item; thread x copies chunk x of the batch's NBI*4 chunks
      for (int x = tid; x < NBI * 4; x += NT) {
        const int t = bt * NBI + (x >> 2);
        if (t < T) {
          int lo = 0, hi = nc - 1;
          while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (coff[mid] <= t) lo = mid; else hi = mid - 1; }
          cp16(dst + (x >> 2) * 8 + (x & 3) * 2, arena + C[lo].voff + (long long)(t - coff[lo]) * 8 + (x & 3) * 2);
        }
      }
      cp_commit();
    };
    issue(0);
    for (int bt = 0; bt < nbat; ++bt) {
      if (bt + 1 < nbat) { issue(bt + 1); cp_wait<1>(); } else cp_wait<0>();
      __syncthreads();
      const double *vb = V + (bt & 1) * NBI * 8;
      for (int x = tid; x < NBI; x += NT) {
        const int t = bt * NBI + x;
        if (t >= T) break;
        int lo = 0, hi = nc - 1;
        while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (coff[mid] <= t) lo = mid; else hi = mid - 1; }
        const double *v = vb + x * 8;
        const double *B = Bs + C[lo].bsm;
        double *wl = W + (long long)line_of_item[t] * 8;
        for (int q = 0; q < C[lo].ncol; ++q) {
          double d = 0.0;
#pragma unroll
          for (int i = 0; i < 8; ++i) d = fma(v[i], B[q * 8 + i], d);
          if (VAR == 5) atomicAdd(&wl[qcol[C[lo].qoff + q]], -d); else red_add(&wl[qcol[C[lo].qoff + q]], -d);
        }
      }
      __syncthreads();
    }
  } else if (VAR == 3) {
    int a = 0;
    for (int t = tid; t < T; t += 2 * NT) {
      const int t2 = t + NT;
      while (a + 1 < nc && coff[a + 1] <= t) ++a;
      int a2 = a;
      while (a2 + 1 < nc && coff[a2 + 1] <= t2) ++a2;
      double v[8], w[8];
      const double2 *p = (const double2 *)(arena + C[a].voff + (long long)(t - coff[a]) * 8);
#pragma unroll
      for (int i = 0; i < 4; ++i) { double2 x = p[i]; v[2 * i] = x.x; v[2 * i + 1] = x.y; }
      const bool has2 = t2 < T;
      if (has2) {
        const double2 *p2 = (const double2 *)(arena + C[a2].voff + (long long)(t2 - coff[a2]) * 8);
#pragma unroll
        for (int i = 0; i < 4; ++i) { double2 x = p2[i]; w[2 * i] = x.x; w[2 * i + 1] = x.y; }
      }
      for (int u = 0; u < 2; ++u) {
        if (u == 1 && !has2) break;
        const int aa = u ? a2 : a, tt = u ? t2 : t;
        const double *vv = u ? w : v;
        const double *B = Bs + C[aa].bsm;
        double *wl = W + (long long)line_of_item[tt] * 8;
        for (int q = 0; q < C[aa].ncol; ++q) {
          double d = 0.0;
#pragma unroll
          for (int i = 0; i < 8; ++i) d = fma(vv[i], B[q * 8 + i], d);
          red_add(&wl[qcol[C[aa].qoff + q]], -d);
        }
      }
    }
  } else {
    int a = 0;
    for (int t = tid; t < T; t += NT) {
      while (a + 1 < nc && coff[a + 1] <= t) ++a;
      double v[8];
      const double2 *p = (const double2 *)(arena + C[a].voff + (long long)(t - coff[a]) * 8);
#pragma unroll
      for (int i = 0; i < 4; ++i) { double2 x = p[i]; v[2 * i] = x.x; v[2 * i + 1] = x.y; }
      const double *B = VAR == 0 ? arena + C[a].boff : Bs + C[a].bsm;
      double *wl = W + (long long)line_of_item[t] * 8;
      for (int q = 0; q < C[a].ncol; ++q) {
        double d = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) d = fma(v[i], B[q * 8 + i], d);
        const int c = qcol[C[a].qoff + q];
        if (VAR == 1) atomicAdd(&wl[c], -d); else red_add(&wl[c], -d);
      }
    }
  }
  __syncthreads();
  long long t2 = clock64();
  if (tid == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  if (VAR == 1 || VAR == 5 || VAR == 7) for (int x = tid; x < nlines * 8; x += NT) gW[x] = W[x];
}

int main() {
  const int nc = 184, nlines = 256;
  srand(1);
  std::vector<Con> C(nc);
  int T = 0, nB = 0, nQ = 0;
  const long long arena_n = (getenv("ARENA_MB") ? atoll(getenv("ARENA_MB")) : 1024) * (1ll << 17);
  std::vector<int> qcol, lines;
  for (int a = 0; a < nc; ++a) {
    Con c; c.item_off = T; c.n = 8 + rand() % 22; c.ncol = 1 + rand() % 8;
    c.voff = ((long long)rand() * 4096 + rand()) % (arena_n - 4096); c.voff &= ~15ll;
    c.boff = ((long long)rand() * 4096 + rand()) % (arena_n - 4096); c.boff &= ~15ll;
    c.bsm = nB; c.qoff = nQ; c.pad = 0;
    for (int q = 0; q < c.ncol; ++q) qcol.push_back(q);
    for (int i = 0; i < c.n; ++i) lines.push_back(rand() % nlines);
    T += c.n; nB += c.ncol * 8; nQ += c.ncol;
    C[a] = c;
  }
  printf("T=%d items, nB=%d doubles, lines=%d\n", T, nB, nlines);
  double *arena, *W, *flush; Con *dC; int *dl, *dq; long long *cyc;
  cudaMalloc(&arena, arena_n * 8); cudaMemset(arena, 0, arena_n * 8);
  cudaMalloc(&flush, 512 << 20);
  cudaMalloc(&W, nlines * 8 * 8); cudaMalloc(&dC, nc * sizeof(Con)); cudaMalloc(&dl, T * 4); cudaMalloc(&dq, nQ * 4);
  cudaMalloc(&cyc, 16);
  cudaMemcpy(dC, C.data(), nc * sizeof(Con), cudaMemcpyHostToDevice);
  cudaMemcpy(dl, lines.data(), T * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dq, qcol.data(), nQ * 4, cudaMemcpyHostToDevice);
  std::vector<int> ordv(T);
  for (int i = 0; i < T; ++i) ordv[i] = i;
  std::stable_sort(ordv.begin(), ordv.end(), [&](int x, int y) { return lines[x] < lines[y]; });
  int *dord; cudaMalloc(&dord, T * 4); cudaMemcpy(dord, ordv.data(), T * 4, cudaMemcpyHostToDevice);
  const int smem = (nlines * 8 + 8192 + 2048 + 8192) * 8;
  auto run = [&](auto kern, const char *name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(flush, rep, 512 << 20);
      cudaMemset(W, 0, nlines * 64);
      kern<<<1, NT, smem>>>(dC, nc, T, arena, dl, dq, W, nlines, cyc, dord);
      cudaDeviceSynchronize();
      long long c[2]; cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
      if (rep) printf("%-40s stage %6.2f us  items %6.2f us %s\n", name, c[0] / 1965.0, c[1] / 1965.0, cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(upd<0>, "0: B global, RED global W");
  run(upd<1>, "1: B smem, smem W atomicAdd");
  run(upd<2>, "2: B smem, RED global W");
  run(upd<3>, "3: B smem, RED global W, 2 items");
  run(upd<4>, "4: cp.async items, RED global W");
  run(upd<5>, "5: cp.async items, smem W atomicAdd");
  run(upd<6>, "6: staged B+pos, 2 items, RED global W");
  run(upd<7>, "7: staged B+pos, 2 items, smem W atomic");
  run(upd<8>, "8: pull, line-sorted chunks, RED per run");
  run(upd<9>, "9: pull without writes");
  run(upd<10>, "10: as 6 without RED");
  run(upd<11>, "11: as 6 without RED and Q");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
