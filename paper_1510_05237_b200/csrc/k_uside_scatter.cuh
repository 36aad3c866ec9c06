// k_uside_scatter.cuh -- U-side product on one GPU, driven by the ACTIVE
// documents ("U = A V (V^T V)^{-1}", paper's order).
//
// Y = A V only involves the documents j with a non-empty row of V (<= k t of
// them, ~9 % of the documents at Large), so instead of streaming all of A the
// kernel walks the rows of A^T of those documents and scatters each product
// a_ij v_jc into Y[i][c]:
//  * the sums are accumulated as 64-bit FIXED-POINT integers with one global
//    scale S = 2^62 / (max_i rowsum_i(A) * max(V)) -- every term is >= 0 and no
//    sum can exceed 2^62, integer atomic addition is exact and order-free, so Y
//    is deterministic; the quantum max_i rowsum_i max(V) 2^-62 is ~1e-19 of the
//    largest possible entry;
//  * a second pass converts each row of Y to fp64, multiplies it by
//    W = (V^T V + eps I)^{-1} (fp64, zero entries skipped), writes the LS row
//    and clears the accumulator row for the next half-step.
#pragma once
#include "common.cuh"

namespace esk {

// one warp per active document of V (vactive[0..n_active)): scatter a_ij v_jc
__global__ void __launch_bounds__(256) k_uside_scatter(const int32_t* __restrict__ vactive,
                                                       const int64_t* __restrict__ n_active,
                                                       const uint64_t* __restrict__ vmap,
                                                       const int2* __restrict__ vent,
                                                       const int64_t* __restrict__ atptr,
                                                       const int2* __restrict__ atent,
                                                       const double* __restrict__ bound,  // max_i rowsum_i
                                                       const uint32_t* __restrict__ vmax, int kpad,
                                                       unsigned long long* __restrict__ Yq) {
  const int lane = threadIdx.x & 31;
  const int64_t na = *n_active;
  const double B = *bound * (double)__uint_as_float(*vmax);
  const double S = B > 0 ? 0x1p62 / B : 0.0;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < na; r += nwarps) {
    const int32_t doc = vactive[r];
    const uint64_t code = vmap[doc];
    const uint32_t p0 = (uint32_t)(code >> 32), cnt = (uint32_t)code;
    const int64_t s = atptr[doc], e = atptr[doc + 1];
    for (uint32_t p = 0; p < cnt; ++p) {
      const int2 pr = vent[p0 + p];  // (topic c, value v_jc), same for all lanes
      const double vs = (double)__int_as_float(pr.y) * S;
      for (int64_t q = s + lane; q < e; q += 32) {
        const int2 en = atent[q];
        const unsigned long long add = __double2ull_rn((double)__int_as_float(en.y) * vs);
        if (add) atomicAdd(&Yq[(int64_t)en.x * kpad + pr.x], add);
      }
    }
  }
}

// one warp per term row: LS row = (Yq row * quantum) W, Yq row cleared
template <int CQ>
__global__ void __launch_bounds__(256) k_uside_finish(int64_t rows, const double* __restrict__ bound,
                                                      const uint32_t* __restrict__ vmax,
                                                      const double* __restrict__ W, int k, int kpad,
                                                      unsigned long long* __restrict__ Yq, float* __restrict__ X,
                                                      int64_t ldx) {
  const int lane = threadIdx.x & 31;
  const double unit = *bound * (double)__uint_as_float(*vmax) * 0x1p-62;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < rows; i += nwarps) {
    unsigned long long* yr = Yq + i * kpad;
    double y[CQ];
    bool any = false;
#pragma unroll
    for (int q = 0; q < CQ; ++q) {
      const int c = lane + 32 * q;
      unsigned long long v = 0;
      if (c < kpad) {
        v = yr[c];
        if (v) yr[c] = 0ull;
      }
      y[q] = (double)v * unit;
      any |= v != 0ull;
    }
    double o[CQ];
#pragma unroll
    for (int q = 0; q < CQ; ++q) o[q] = 0.0;
    if (__any_sync(kFull, any)) {
#pragma unroll
      for (int q = 0; q < CQ; ++q) {
        unsigned nz = __ballot_sync(kFull, y[q] != 0.0);
        while (nz) {  // two nonzero columns per step: independent loads in flight
          const int l0 = __ffs(nz) - 1;
          nz &= nz - 1;
          const int l1 = nz ? __ffs(nz) - 1 : l0;
          const bool two = nz != 0;
          if (two) nz &= nz - 1;
          const double y0 = __shfl_sync(kFull, y[q], l0);
          const double y1 = two ? __shfl_sync(kFull, y[q], l1) : 0.0;
          const double* W0 = W + (int64_t)(32 * q + l0) * k;
          const double* W1 = W + (int64_t)(32 * q + l1) * k;
#pragma unroll
          for (int qq = 0; qq < CQ; ++qq) {
            const int c = lane + 32 * qq;
            if (c < k) {
              const double w0 = __ldg(W0 + c), w1 = __ldg(W1 + c);
              o[qq] = fma(y0, w0, o[qq]);
              o[qq] = fma(y1, w1, o[qq]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < CQ; ++q) {
      const int c = lane + 32 * q;
      if (c < k) X[(int64_t)c * ldx + i] = (float)o[q];
    }
  }
}

// max_i rowsum_i(A) for the global fixed-point scale (one block)
__global__ void k_max_to(const double* __restrict__ a, int64_t n, double* __restrict__ out) {
  __shared__ double sm[32];
  double m = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, a[i]);
  m = fmax(m, __shfl_xor_sync(kFull, m, 16));
  m = fmax(m, __shfl_xor_sync(kFull, m, 8));
  m = fmax(m, __shfl_xor_sync(kFull, m, 4));
  m = fmax(m, __shfl_xor_sync(kFull, m, 2));
  m = fmax(m, __shfl_xor_sync(kFull, m, 1));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, sm[w]);
    *out = r;
  }
}

}  // namespace esk
