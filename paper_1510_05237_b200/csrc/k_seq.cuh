// k_seq.cuh -- sequential ALS (Alg. 3).
//
// The handle runs the k2-column pipeline on the current block (U_2, V_2); the
// converged topics U_1, V_1 (the first b0 = b k2 of the k columns) live in
// separate "frozen" factors FU, FV.  The update of Eq. (7) / Eq. (8)
// (P:322-326),
//     F_2 = (T H_2 - O_1 H_1^T H_2)(H_2^T H_2 + eps I)^{-1}
// (V side: T = A^T, H = U, O = V; U side: T = A, H = V, O = U), is the block's
// own product T H_2 W_22 minus O_1 M with M = (H_1^T H_2) W_22:
//   k_seq_cross   C = H_1^T H_2  (b0 x k2, fp64, one block per (c, d))
//   k_seq_m       M = C W_22
//   k_seq_deflate X[:, d] -= O_1 M[:, d] over O_1's active rows
// Appending a finished block to FU / FV and updating the constants of the
// whole-factor records (T_1 = tr(U_1^T A V_1), S_11 = tr(G_U1 G_V1), ||U_1||^2)
// are the other kernels here.
#pragma once
#include "common.cuh"

namespace esk {

// C[c][d] = sum over the entries (i, v) of column c of H_1 of v * H_2[i][d]
// (H_2 through its row view: rowmap + dense rows of stride kpad)
__global__ void __launch_bounds__(256) k_seq_cross(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                                                   const float* __restrict__ val, const int32_t* __restrict__ rowmap,
                                                   const float* __restrict__ dense, int kpad, int k2,
                                                   double* __restrict__ C) {
  __shared__ double sm[32];
  const int c = blockIdx.x, d = blockIdx.y;
  double s = 0;
  for (int64_t e = colptr[c] + threadIdx.x; e < colptr[c + 1]; e += blockDim.x) {
    const int32_t r = rowmap[row[e]];
    if (r >= 0) s = fma((double)val[e], (double)dense[(int64_t)r * kpad + d], s);
  }
  s = block_sum(s, sm);
  if (threadIdx.x == 0) C[(int64_t)c * k2 + d] = s;
}

// M[c][d] = sum_e C[c][e] W[e][d]  (c < b0, d < k2; W is the block's k2 x k2 inverse)
__global__ void k_seq_m(const double* __restrict__ C, const double* __restrict__ W, int b0, int k2,
                        double* __restrict__ M) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)b0 * k2; q += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(q / k2), d = (int)(q - (int64_t)c * k2);
    double s = 0;
    for (int e = 0; e < k2; ++e) s = fma(C[(int64_t)c * k2 + e], W[(int64_t)e * k2 + d], s);
    M[q] = s;
  }
}

// X[d][i] -= sum_{c < b0} O[i][c] M[c][d] for every active row i of O (rows of
// O that are empty have nothing to subtract).  One thread per (row, d); O's
// dense rows have stride kpf.
__global__ void k_seq_deflate(const int32_t* __restrict__ active, const int64_t* __restrict__ n_active,
                              const float* __restrict__ dense, int kpf, int b0, int k2,
                              const double* __restrict__ M, float* __restrict__ X, int64_t ldx, int64_t row0,
                              int64_t rows) {
  const int64_t total = *n_active * k2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q / k2;
    const int d = (int)(q - r * k2);
    const int64_t lr = (int64_t)active[r] - row0;
    if (lr < 0 || lr >= rows) continue;
    const float* o = dense + r * kpf;
    double s = 0;
    for (int c = 0; c < b0; ++c) {
      const float oc = o[c];
      if (oc != 0.f) s = fma((double)oc, M[(int64_t)c * k2 + d], s);
    }
    float* x = X + (int64_t)d * ldx + lr;
    *x = (float)((double)*x - s);
  }
}

// append the block's COO (k2 columns) as columns [b0, b0 + k2) of the frozen
// factor F (ktot columns, canonical column-major): entries first ...
__global__ void k_seq_append_entries(const int64_t* __restrict__ bcolptr, const int32_t* __restrict__ brow,
                                     const float* __restrict__ bval, int k2, int b0,
                                     const int64_t* __restrict__ fcolptr, int32_t* __restrict__ frow,
                                     float* __restrict__ fval) {
  const int64_t base = fcolptr[b0], nb = bcolptr[k2];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nb; e += (int64_t)gridDim.x * blockDim.x) {
    frow[base + e] = brow[e];
    fval[base + e] = bval[e];
  }
}

// ... then the column pointers (one block; colptr[c] for c > b0 + k2 = new total)
__global__ void k_seq_append_colptr(const int64_t* __restrict__ bcolptr, int k2, int b0, int ktot,
                                    int64_t* __restrict__ fcolptr) {
  const int64_t base = fcolptr[b0];
  __syncthreads();
  for (int c = b0 + 1 + threadIdx.x; c <= ktot; c += blockDim.x) fcolptr[c] = base + bcolptr[min(c - b0, k2)];
}

// record constants when block (U_2, V_2) joins U_1, V_1 (one block): with
// C_U = U_1^T U_2, C_V = V_1^T V_2 (old U_1, V_1) and X = sum C_U o C_V,
//   T_1   += tr(U_2^T A V_2) = T_2' + X    (T_2' = the last record's LS-recovered
//                                          trace, scal[2]; A V_2 = LS_2 (G + eps I) + U_1 C_V)
//   S_11  += 2 X + tr(G_U2 G_V2)          (the Gram of [U_1 U_2] is [[G_11, C_U], [C_U^T, G_22]])
//   |U_1|^2 += tr G_U2
__global__ void k_seq_consts(const double* __restrict__ CU, const double* __restrict__ CV, int ncross,
                             const double* __restrict__ T2, const double* __restrict__ GU2,
                             const double* __restrict__ GV2, int k2, double* __restrict__ c) {
  __shared__ double sm[32];
  double X = 0, S = 0, tr = 0;
  for (int q = threadIdx.x; q < ncross; q += blockDim.x) X += CU[q] * CV[q];
  for (int q = threadIdx.x; q < k2 * k2; q += blockDim.x) S += GU2[q] * GV2[q];
  for (int d = threadIdx.x; d < k2; d += blockDim.x) tr += GU2[(int64_t)d * k2 + d];
  X = block_sum(X, sm);
  S = block_sum(S, sm);
  tr = block_sum(tr, sm);
  if (threadIdx.x == 0) {
    c[0] += *T2 + X;
    c[1] += 2.0 * X + S;
    c[2] += tr;
  }
}

}  // namespace esk
