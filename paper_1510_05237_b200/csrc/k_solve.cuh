// k_solve.cuh -- the k x k solve of Alg. 2 ("(U^T U)^{-1}") and the
// reassociated right factor Z = F W.
#pragma once
#include "common.cuh"

namespace esk {

// ---- W = (G + eps I)^{-1}, eps = rho (tr G / k + 1) (reading C6) ------
// Gauss-Jordan "sweep" of a symmetric positive definite matrix on its packed
// upper triangle: sweeping every pivot p maps A to -A^{-1}:
//   d = a_pp;  a_pp <- -1/d;  a_pj <- a_pj / d;  a_ij <- a_ij - a_ip a_pj / d.
// Pivots of an SPD matrix stay positive; a non-positive or non-finite pivot
// raises *singular.  One CTA; storage P is shared memory (k <= 224) or a
// global scratch buffer.  fp64 throughout.
ESNMF_DEV int64_t pk_idx(int i, int j, int k) {  // i <= j, packed upper, row-major
  return (int64_t)i * k - ((int64_t)i * (i - 1)) / 2 + (j - i);
}

__global__ void __launch_bounds__(1024) k_sweep_inverse(const double* __restrict__ G, int k, double rho,
                                                        double* __restrict__ W, double* __restrict__ eps_out,
                                                        int* __restrict__ singular, double* gscratch) {
  extern __shared__ double dsm[];
  __shared__ double red[32];
  __shared__ double piv;
  const int64_t np = (int64_t)k * (k + 1) / 2;
  double* v = dsm;                              // old pivot row, k doubles
  double* P = gscratch ? gscratch : dsm + k;    // packed matrix
  double tr = 0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) tr += G[(int64_t)i * k + i];
  tr = block_sum(tr, red);
  const double eps = rho * (tr / k + 1.0);
  for (int64_t q = threadIdx.x; q < (int64_t)k * k; q += blockDim.x) {
    int i = (int)(q / k), j = (int)(q - (int64_t)i * k);
    if (j >= i) P[pk_idx(i, j, k)] = G[q] + (i == j ? eps : 0.0);
  }
  __syncthreads();
  for (int p = 0; p < k; ++p) {
    for (int j = threadIdx.x; j < k; j += blockDim.x) v[j] = P[j <= p ? pk_idx(j, p, k) : pk_idx(p, j, k)];
    __syncthreads();
    if (threadIdx.x == 0) {
      double d = v[p];
      if (!(d > 0.0) || !isfinite(d)) {
        atomicExch(singular, 1);
        d = 1.0;
      }
      piv = d;
    }
    __syncthreads();
    const double d = piv, inv = 1.0 / d;
    for (int64_t q = threadIdx.x; q < np; q += blockDim.x) {
      // recover (i, j) of packed index q (row i holds k - i entries)
      int i = (int)((2.0 * k + 1.0 - sqrt((2.0 * k + 1.0) * (2.0 * k + 1.0) - 8.0 * (double)q)) * 0.5);
      while (i > 0 && pk_idx(i, i, k) > q) --i;
      while (i + 1 < k && pk_idx(i + 1, i + 1, k) <= q) ++i;
      int j = i + (int)(q - pk_idx(i, i, k));
      double a = P[q];
      if (i == p && j == p) a = -inv;
      else if (i == p) a = v[j] * inv;
      else if (j == p) a = v[i] * inv;
      else a = a - v[i] * v[j] * inv;
      P[q] = a;
    }
    __syncthreads();
  }
  for (int64_t q = threadIdx.x; q < (int64_t)k * k; q += blockDim.x) {
    int i = (int)(q / k), j = (int)(q - (int64_t)i * k);
    W[q] = -P[i <= j ? pk_idx(i, j, k) : pk_idx(j, i, k)];
  }
  if (threadIdx.x == 0) *eps_out = eps;
}

inline size_t sweep_smem_bytes(int k, bool global_scratch) {
  size_t b = sizeof(double) * (size_t)k;
  if (!global_scratch) b += sizeof(double) * (size_t)k * (k + 1) / 2;
  return b;
}

// ---- Z = F W for the active rows of the factor (fp64 accumulate, fp32 out) ----
// The LS rows of a half-step are T (F W): the product with A^T (or A) is
// reassociated onto Z (identical to (T F) W up to rounding).
// One warp per active row; lanes own columns c = lane + 32 j.
template <int CJ>
__global__ void __launch_bounds__(256) k_form_z(const float* __restrict__ dense, int kpad, int k,
                                                const int64_t* __restrict__ n_active,
                                                const double* __restrict__ W, float* __restrict__ Z) {
  const int lane = threadIdx.x & 31;
  const int64_t na = *n_active;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp0; r < na; r += nwarps) {
    float f[CJ];
#pragma unroll
    for (int j = 0; j < CJ; ++j) {
      int c = lane + 32 * j;
      f[j] = c < kpad ? dense[r * kpad + c] : 0.f;
    }
    double acc[CJ];
#pragma unroll
    for (int j = 0; j < CJ; ++j) acc[j] = 0.0;
#pragma unroll
    for (int jl = 0; jl < CJ; ++jl) {
      const int lmax = min(32, k - 32 * jl);
      for (int ll = 0; ll < lmax; ++ll) {
        const float fl = __shfl_sync(kFull, f[jl], ll);
        if (fl != 0.f) {
          const int l = 32 * jl + ll;
#pragma unroll
          for (int j = 0; j < CJ; ++j) {
            int c = lane + 32 * j;
            if (c < k) acc[j] += (double)fl * W[(int64_t)l * k + c];
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < CJ; ++j) {
      int c = lane + 32 * j;
      if (c < kpad) Z[r * kpad + c] = c < k ? (float)acc[j] : 0.f;
    }
  }
}

}  // namespace esk
