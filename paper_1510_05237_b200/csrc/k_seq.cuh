// k_seq.cuh -- sequential ALS (Alg. 3).
//
// Block b of k2 topics occupies columns [b0, b0 + k2) of the k-column
// factors; the columns < b0 are the converged topics U_1, V_1.  The update of
// Eq. (7) / Eq. (8),
//     F_2 = (T H_2 - O_1 H_1^T H_2)(H_2^T H_2 + eps I)^{-1}
// (V side: T = A^T, H = U, O = V; U side: T = A, H = V, O = U), runs through
// the k-column pipeline unchanged with three additions:
//   * W is the block inverse: (G_22 + eps I)^{-1} in the block, 0 elsewhere
//     (k_seq_gblock + the sweep + k_seq_wmask), so the product T H W writes
//     T H_2 W_22 into the block columns and 0 into the others;
//   * k_seq_deflate subtracts O_1 (G_12 W_22), G_12 = H_1^T H_2, from the block
//     columns (M = G_12 W_22 from k_seq_m);
//   * the converged columns of O are written back into the LS buffer before
//     the selection (k_coo_to_colmajor), which keeps them (<= t entries each).
#pragma once
#include "common.cuh"

namespace esk {

// Gs = G on the block, (tr G_22 / k2) on the other diagonal entries, 0 elsewhere:
// the sweep's eps = rho (tr Gs / k + 1) is then rho (tr G_22 / k2 + 1), reading C6
// on the block Gram (reading C19), and its inverse is block-diagonal.
__global__ void k_seq_gblock(const double* __restrict__ G, int k, int b0, int k2, double* __restrict__ Gs) {
  double tr = 0;
  for (int d = 0; d < k2; ++d) tr += G[(int64_t)(b0 + d) * k + b0 + d];
  const double mean = tr / k2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)k * k; q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / k), j = (int)(q - (int64_t)i * k);
    const bool bi = i >= b0 && i < b0 + k2, bj = j >= b0 && j < b0 + k2;
    Gs[q] = (bi && bj) ? G[q] : (i == j ? mean : 0.0);
  }
}

// zero W outside block x block
__global__ void k_seq_wmask(double* __restrict__ W, int k, int b0, int k2) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)k * k; q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / k), j = (int)(q - (int64_t)i * k);
    if (!(i >= b0 && i < b0 + k2 && j >= b0 && j < b0 + k2)) W[q] = 0.0;
  }
}

// M[c][d] = sum_e G[c][b0+e] W[b0+e][b0+d] for c < b0, d < k2 (fp64)
__global__ void k_seq_m(const double* __restrict__ G, const double* __restrict__ W, int k, int b0, int k2,
                        double* __restrict__ M) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)b0 * k2; q += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(q / k2), d = (int)(q - (int64_t)c * k2);
    double s = 0;
    for (int e = 0; e < k2; ++e) s = fma(G[(int64_t)c * k + b0 + e], W[(int64_t)(b0 + e) * k + b0 + d], s);
    M[q] = s;
  }
}

// X[b0+d][i] -= sum_{c < b0} O[i][c] M[c][d] for every active row i of O (rows
// of O that are empty have nothing to subtract).  One thread per (row, d).
__global__ void k_seq_deflate(const int32_t* __restrict__ active, const int64_t* __restrict__ n_active,
                              const float* __restrict__ dense, int kpad, int b0, int k2,
                              const double* __restrict__ M, float* __restrict__ X, int64_t ldx, int64_t row0,
                              int64_t rows) {
  const int64_t total = *n_active * k2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q / k2;
    const int d = (int)(q - r * k2);
    const int64_t lr = (int64_t)active[r] - row0;
    if (lr < 0 || lr >= rows) continue;
    const float* o = dense + r * kpad;
    double s = 0;
    for (int c = 0; c < b0; ++c) {
      const float oc = o[c];
      if (oc != 0.f) s = fma((double)oc, M[(int64_t)c * k2 + d], s);
    }
    float* x = X + (int64_t)(b0 + d) * ldx + lr;
    *x = (float)((double)*x - s);
  }
}

// U_0 block ("Set U_2 = U_0", U_0 in R^{n x k2}): the reading C10 formula
// with k2 columns (index i*k2 + c), masked as reading C18 when thr != ~0,
// written into columns [b0, b0 + k2) of the column-major buffer X.
__global__ void k_seq_u0_block(int64_t n, int k2, uint64_t seed, uint64_t thr, int b0, float* __restrict__ X,
                               int64_t ldx) {
  const int64_t total = n * k2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / k2;
    const int c = (int)(q - i * k2);
    const uint64_t x = splitmix64(seed ^ kU0Stream ^ (uint64_t)q);
    float v = (float)(((double)(x >> 41) + 0.5) * 0x1p-23);
    if (thr != ~0ULL && (splitmix64(seed ^ kU0Mask ^ (uint64_t)q) >> 11) >= thr) v = 0.f;
    X[(int64_t)(b0 + c) * ldx + i] = v;
  }
}

// E's trace term without the LS recovery (the deflated, block-masked LS of
// Alg. 3 no longer gives A V): T = tr(U^T A V) = sum over the entries a_ij of
// the active term rows i of U of a_ij (U_i . V_j), V_j from V's row view.
// One warp per active U row, U_i staged in shared memory, lanes over entries;
// fixed-order per-block partials.
__global__ void __launch_bounds__(256) k_err_trace_direct(const int32_t* __restrict__ active,
                                                          const int64_t* __restrict__ n_active,
                                                          const float* __restrict__ udense,
                                                          const int64_t* __restrict__ aptr,
                                                          const int2* __restrict__ aent,
                                                          const int32_t* __restrict__ vrowmap,
                                                          const float* __restrict__ vdense, int kpad, int k,
                                                          double* __restrict__ part) {
  extern __shared__ float su[];  // [8 warps][kpad]
  __shared__ double sm[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* ur = su + w * kpad;
  const int64_t na = *n_active;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < na; r += nwarps) {
    for (int c = lane; c < kpad; c += 32) ur[c] = udense[r * kpad + c];
    __syncwarp();
    const int64_t i = active[r];
    for (int64_t e = aptr[i] + lane; e < aptr[i + 1]; e += 32) {
      const int2 en = aent[e];
      const int32_t vr = vrowmap[en.x];
      if (vr < 0) continue;
      const float* v = vdense + (int64_t)vr * kpad;
      double s = 0;
      for (int c = 0; c < k; ++c) s = fma((double)ur[c], (double)v[c], s);
      acc = fma((double)__int_as_float(en.y), s, acc);
    }
    __syncwarp();
  }
  acc = block_sum(acc, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

}  // namespace esk
