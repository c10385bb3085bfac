// bilu_matching.cu -- Sec. 3.1 maximum weight matching + scaling on the
// device: the maximum product transversal of A with MC64's column-normalised costs
//     c_ij = log(max_k |a_kj|) - log |a_ij|  >= 0     (stored nonzeros only; R22)
// solved as an assignment problem by a parallel (Jacobi) forward auction with eps-scaling
// (every unassigned row bids at once, one warp per row; the highest bid wins a column).
// With benefits b_ij = -c_ij and prices p_j the auction ends in eps-complementary slackness
//     b_{i,sigma(i)} - p_{sigma(i)} >= max_k (b_ik - p_k) - eps,
// so u_i = c_{i,sigma(i)} + p_{sigma(i)}, v_j = -p_j satisfy c_ij - u_i - v_j >= -eps with
// equality on the matching, and the scalings D_l = diag(e^{u_i}), D_r = diag(e^{v_j} / cmax_j)
// give |d_i a_ij d_j| <= e^eps and |d_i a_{i,sigma(i)} d_{sigma(i)}| = 1 ("the maximum weight
// matching ... two dual vectors from which one has to take the exponential", PAPER.md:836-848,
// 861-867).  The final eps is below 1e-10 (relative to the cost range) / n, so the transversal
// is an optimal one whenever the optimum is unique up to that margin.
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <climits>
#include <cstring>

namespace bilu {

__global__ void mwm_colmax_kernel(int n, const int64_t *rp, const int32_t *ci, const double *val,
                                  unsigned long long *cmax_bits) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      atomicMax(&cmax_bits[ci[p]], (unsigned long long)__double_as_longlong(fabs(val[p])));
}

// costs (HUGE_VAL for explicit zeros: not an edge of the bipartite graph); range of the finite ones
__global__ void mwm_cost_kernel(int n, const int64_t *rp, const int32_t *ci, const double *val,
                                const unsigned long long *cmax_bits, double *c, unsigned long long *cmaxcost_bits,
                                int *bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (rp[i] == rp[i + 1]) atomicExch(bad, 1);
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const double a = fabs(val[p]);
      if (a == 0.0) { c[p] = HUGE_VAL; continue; }
      const double cm = __longlong_as_double((long long)cmax_bits[ci[p]]);
      const double cost = log(cm) - log(a);
      c[p] = cost > 0.0 ? cost : 0.0;
      atomicMax(cmaxcost_bits, (unsigned long long)__double_as_longlong(c[p]));
    }
  }
}

// one warp per unassigned row: best and second-best value b_ij - p_j over the row's edges;
// the bid p_j1 + (v1 - v2) + eps goes to column j1 (prices are >= 0, so bids are positive
// doubles whose bit patterns order like the values)
__global__ void mwm_bid_kernel(int n, const int64_t *rp, const int32_t *ci, const double *c, const double *price,
                               const int32_t *assign, unsigned long long *colbid, double *rowbid, int32_t *rowcol,
                               double eps, double solo) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    if (assign[i] >= 0) { if (lane == 0) rowcol[i] = -1; continue; }
    double v1 = -HUGE_VAL, v2 = -HUGE_VAL;
    int j1 = INT_MAX;
    for (int64_t p = rp[i] + lane; p < rp[i + 1]; p += 32) {
      if (c[p] == HUGE_VAL) continue;
      const int j = ci[p];
      const double v = -c[p] - price[j];
      if (v > v1 || (v == v1 && j < j1)) { v2 = v1; v1 = v; j1 = j; }
      else if (v > v2) v2 = v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov1 = __shfl_xor_sync(0xffffffffu, v1, o), ov2 = __shfl_xor_sync(0xffffffffu, v2, o);
      const int oj1 = __shfl_xor_sync(0xffffffffu, j1, o);
      if (ov1 > v1 || (ov1 == v1 && oj1 < j1)) { v2 = fmax(v1, ov2); v1 = ov1; j1 = oj1; }
      else v2 = fmax(v2, ov1);
    }
    if (lane == 0) {
      if (j1 == INT_MAX) { rowcol[i] = -2; continue; }    // no edge: structurally singular
      const double inc = (v2 == -HUGE_VAL ? solo : v1 - v2) + eps;
      const double bid = price[j1] + inc;
      rowbid[i] = bid;
      rowcol[i] = j1;
      atomicMax(&colbid[j1], (unsigned long long)__double_as_longlong(bid));
    }
  }
}

// the highest bid wins (ties: lowest row); the previous owner is unassigned
__global__ void mwm_resolve_kernel(int n, const double *rowbid, const int32_t *rowcol, const unsigned long long *colbid,
                                   int *colwin, int *bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int j = rowcol[i];
    if (j == -2) atomicExch(bad, 1);
    if (j < 0) continue;
    if ((unsigned long long)__double_as_longlong(rowbid[i]) == colbid[j]) atomicMin(&colwin[j], i);
  }
}

__global__ void mwm_assign_kernel(int n, const double *rowbid, const int32_t *rowcol, unsigned long long *colbid,
                                  int *colwin, int32_t *owner, int32_t *assign, double *price, int *unassigned) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int j = rowcol[i];
    if (j < 0) continue;
    if (colwin[j] == i) {
      const int old = owner[j];
      if (old >= 0) { assign[old] = -1; atomicAdd(unassigned, 1); }
      owner[j] = i;
      assign[i] = j;
      price[j] = rowbid[i];
      colbid[j] = 0ull;
      colwin[j] = INT_MAX;
    } else {
      atomicAdd(unassigned, 1);
    }
  }
}

// duals and scalings from the final prices (header comment)
__global__ void mwm_scale_kernel(int n, const int64_t *rp, const int32_t *ci, const double *c, const int32_t *assign,
                                 const double *price, const unsigned long long *cmax_bits, double *dl, double *dr) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int j = assign[i];
    double cij = 0.0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] == j) { cij = c[p]; break; }
    dl[i] = exp(cij + price[j]);
    dr[i] = exp(-price[i]) / __longlong_as_double((long long)cmax_bits[i]);
  }
}

__global__ void mwm_reset_kernel(int n, int32_t *assign, int32_t *owner, unsigned long long *colbid, int *colwin) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    assign[i] = -1; owner[i] = -1; colbid[i] = 0ull; colwin[i] = INT_MAX;
  }
}

// Host driver (device buffers owned by the caller's bilu_mwm).  Returns 0, -2 (no perfect
// matching: an empty row / column, a row without a usable edge, or no progress within the
// round budget), or a CUDA error code (> 0).  *launches counts the kernels, *rounds the
// bidding rounds.
extern "C" int bilu_mwm_device(int n, const int64_t *rp, const int32_t *ci, const double *val, int32_t *assign,
                               double *dl, double *dr, void *work, cudaStream_t st, int *launches, int *rounds) {
  // work layout: cmax bits [n], price [n], colbid [n], rowbid [n], colwin [n], rowcol [n], owner [n],
  // scalars [4]; then costs [nnz] (passed separately through the work tail)
  char *w = (char *)work;
  unsigned long long *cmax_bits = (unsigned long long *)w; w += (size_t)n * 8;
  double *price = (double *)w; w += (size_t)n * 8;
  unsigned long long *colbid = (unsigned long long *)w; w += (size_t)n * 8;
  double *rowbid = (double *)w; w += (size_t)n * 8;
  int *colwin = (int *)w; w += (size_t)n * 4;
  int32_t *rowcol = (int32_t *)w; w += (size_t)n * 4;
  int32_t *owner = (int32_t *)w; w += (size_t)n * 4;
  w = (char *)(((uintptr_t)w + 15) & ~(uintptr_t)15);
  unsigned long long *scal = (unsigned long long *)w; w += 64;   // [0] max cost bits, [1] unassigned, [2] bad
  double *c = (double *)w;
  int *unassigned = (int *)&scal[1];
  int *bad = (int *)&scal[2];
  const int tb = 256, gb = (n + tb - 1) / tb < 2048 ? (n + tb - 1) / tb : 2048;
  const int gw = (n * 32 + tb - 1) / tb < 4096 ? (n * 32 + tb - 1) / tb : 4096;
  cudaError_t e;
#define MWM_TRY(x) do { if ((e = (x)) != cudaSuccess) return (int)e; } while (0)
  MWM_TRY(cudaMemsetAsync(cmax_bits, 0, (size_t)n * 8, st));
  MWM_TRY(cudaMemsetAsync(price, 0, (size_t)n * 8, st));
  MWM_TRY(cudaMemsetAsync(scal, 0, 64, st));
  mwm_colmax_kernel<<<gb, tb, 0, st>>>(n, rp, ci, val, cmax_bits);
  mwm_cost_kernel<<<gb, tb, 0, st>>>(n, rp, ci, val, cmax_bits, c, &scal[0], bad);
  *launches += 2;
  // an empty column (cmax 0) means no perfect matching
  unsigned long long h[3];
  MWM_TRY(cudaGetLastError());
  MWM_TRY(cudaMemcpyAsync(h, scal, sizeof(h), cudaMemcpyDeviceToHost, st));
  MWM_TRY(cudaStreamSynchronize(st));
  if ((int)(h[2] & 0xffffffffull)) return -2;          // an empty row
  {
    // empty columns: count columns with cmax == 0 on the host side of the same buffer
    unsigned long long *hc = new unsigned long long[n];
    cudaMemcpy(hc, cmax_bits, (size_t)n * 8, cudaMemcpyDeviceToHost);
    bool empty = false;
    for (int j = 0; j < n && !empty; ++j) empty = hc[j] == 0ull;
    delete[] hc;
    if (empty) return -2;
  }
  double R;                                                         // cost range (costs are >= 0)
  memcpy(&R, &h[0], sizeof(double));
  const double eps_min = 1e-10 * (R > 1.0 ? R : 1.0) / n;
  const double solo = R + 1.0;                                      // increment of a row with one edge
  double eps = (R > 0.0 ? R : 1.0) / 4.0;
  const long long budget = 200000 + 50ll * n;
  long long total = 0;
  while (true) {
    mwm_reset_kernel<<<gb, tb, 0, st>>>(n, assign, owner, colbid, colwin);
    *launches += 1;
    int left = n;
    while (left > 0) {
      if (++total > budget) return -2;
      MWM_TRY(cudaMemsetAsync(unassigned, 0, 4, st));
      mwm_bid_kernel<<<gw, tb, 0, st>>>(n, rp, ci, c, price, assign, colbid, rowbid, rowcol, eps, solo);
      mwm_resolve_kernel<<<gb, tb, 0, st>>>(n, rowbid, rowcol, colbid, colwin, bad);
      mwm_assign_kernel<<<gb, tb, 0, st>>>(n, rowbid, rowcol, colbid, colwin, owner, assign, price, unassigned);
      *launches += 3;
      MWM_TRY(cudaGetLastError());
      unsigned long long hs[3];
      MWM_TRY(cudaMemcpyAsync(hs, scal, sizeof(hs), cudaMemcpyDeviceToHost, st));
      MWM_TRY(cudaStreamSynchronize(st));
      if ((int)(hs[2] & 0xffffffffull)) return -2;       // a row without an edge
      left = (int)(hs[1] & 0xffffffffull);
    }
    if (eps <= eps_min) break;
    eps = eps / 8.0 > eps_min ? eps / 8.0 : eps_min;
  }
  *rounds = (int)total;
  mwm_scale_kernel<<<gb, tb, 0, st>>>(n, rp, ci, c, assign, price, cmax_bits, dl, dr);
  *launches += 1;
  MWM_TRY(cudaGetLastError());
  return 0;
#undef MWM_TRY
}

}  // namespace bilu
