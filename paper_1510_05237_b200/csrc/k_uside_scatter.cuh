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
                                                      int64_t ldx, const int* __restrict__ use_fp64) {
  if (use_fp64 && !*use_fp64) return;  // the fp32 kernel handles this system
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
        v = yr[c];  // (Yq is cleared by the host's double buffering: k_polish_u reads it after the select)
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

// The same Y = A V driven by V's columns: block (c, chunk) takes ndocs
// entries (doc j, v) of topic column c.  Each document row of A^T stores its
// head-term entries first (k_reorder_head, nh[j] of them): those accumulate in
// a per-block shared fixed-point row acc[head slot] (topic c only), flushed
// once per block; the tail entries go straight to Yq.  Integer atomics in both
// places: the result is the same exact sum as k_uside_scatter's.
constexpr int kScatDocs = 32;  // documents per block (32 / 64 / 128 / 256 measured: 0.242 / 0.247 / 0.251 / 0.254 ms)

__global__ void __launch_bounds__(256) k_uside_scatter_cols(const int64_t* __restrict__ vcolptr,
                                                            const int32_t* __restrict__ vrow,
                                                            const float* __restrict__ vval,
                                                            const int64_t* __restrict__ atptr,
                                                            const int32_t* __restrict__ nh,
                                                            const int2* __restrict__ atent,
                                                            const int32_t* __restrict__ headslot,
                                                            const int32_t* __restrict__ headterm, int hh,
                                                            const double* __restrict__ bound,
                                                            const uint32_t* __restrict__ vmax, int kpad,
                                                            unsigned long long* __restrict__ Yq, int ndocs) {
  extern __shared__ unsigned long long acc[];  // [hh]
  const int c = blockIdx.y;
  const int64_t cb = vcolptr[c] + (int64_t)blockIdx.x * ndocs, ce = min(vcolptr[c + 1], cb + ndocs);
  if (cb >= ce) return;  // block-uniform
  ESNMF_CHECK(c < kpad && (uint32_t)hh * 8u <= dyn_smem_bytes());
  for (int q = threadIdx.x; q < hh; q += blockDim.x) acc[q] = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double B = *bound * (double)__uint_as_float(*vmax);
  const double S = B > 0 ? 0x1p62 / B : 0.0;
  // half a warp per entry of V (two documents per warp), 4 document entries per
  // lane in flight: the chain entry -> document row -> A^T entries -> head slot
  // is latency-bound, so more independent chains per warp
  const int hl = lane & 15, hw = lane >> 4;
  for (int64_t e0 = cb + 2 * warp; e0 < ce; e0 += 2 * (blockDim.x >> 5)) {  // warp-uniform
    const int64_t e = e0 + hw;
    int64_t s = 0, eh = 0, ee = 0;
    double vs = 0;
    if (e < ce) {
      const int32_t doc = vrow[e];
      vs = (double)vval[e] * S;
      s = atptr[doc];
      eh = s + nh[doc];
      ee = atptr[doc + 1];
    }
    for (int64_t q0 = s + hl; q0 < eh; q0 += 64) {  // head terms: shared accumulator
      int2 en[4];
      int sl[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) en[u] = q0 + 16 * u < eh ? atent[q0 + 16 * u] : make_int2(0, 0);
#pragma unroll
      for (int u = 0; u < 4; ++u) sl[u] = q0 + 16 * u < eh ? headslot[en[u].x] : -1;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (sl[u] < 0) continue;
        ESNMF_CHECK(sl[u] < hh);
        const unsigned long long add = __double2ull_rn((double)__int_as_float(en[u].y) * vs);
        if (add) atomicAdd(&acc[sl[u]], add);
      }
    }
    for (int64_t q0 = eh + hl; q0 < ee; q0 += 64) {  // tail terms: straight to Yq
      int2 en[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) en[u] = q0 + 16 * u < ee ? atent[q0 + 16 * u] : make_int2(-1, 0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (en[u].x < 0) continue;
        const unsigned long long add = __double2ull_rn((double)__int_as_float(en[u].y) * vs);
        if (add) atomicAdd(&Yq[(int64_t)en[u].x * kpad + c], add);
      }
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < hh; q += blockDim.x)
    if (acc[q]) atomicAdd(&Yq[(int64_t)headterm[q] * kpad + c], acc[q]);
}

// W (fp64, k x k) -> fp32 rows of stride kpad (zero padded) for k_uside_finish_rt
__global__ void k_w_to_f32(const double* __restrict__ W, int k, int kpad, float* __restrict__ W32) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < k * kpad; q += gridDim.x * blockDim.x) {
    const int l = q / kpad, c = q - l * kpad;
    W32[q] = c < k ? (float)W[(int64_t)l * k + c] : 0.f;
  }
}

// LS row block = (Y rows) W in fp32 (k <= 224, when the tensor-core finish is not
// used): a warp converts RT = 8 rows of the fixed-point Y at a time into shared
// memory (transposed, ys[l][r]), clears them, and computes the 8 x k block with
// every W row read once from shared memory per 8 rows.  Dense in l: Y's zeros
// are multiplied, not skipped (the same fixed summation order for every row;
// deterministic).  The fp32 product keeps the column-relative error ~1e-7
// (DESIGN.md section 4).
constexpr int kFinRT = 8;

template <int CW>
__global__ void __launch_bounds__(256) k_uside_finish_rt(int64_t rows, const double* __restrict__ bound,
                                                         const uint32_t* __restrict__ vmax,
                                                         const float* __restrict__ W32, int k, int kpad,
                                                         unsigned long long* __restrict__ Yq, float* __restrict__ X,
                                                         int64_t ldx, const int* __restrict__ use_fp64) {
  if (*use_fp64) return;  // ill-conditioned: the fp64 kernel handles it
  extern __shared__ float4 ws4[];  // [k][kpad/4] W, then per warp ys[kpad][kFinRT]
  const int kq = kpad / 4;
  for (int q = threadIdx.x; q < k * kq; q += blockDim.x) ws4[q] = reinterpret_cast<const float4*>(W32)[q];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* ys = reinterpret_cast<float*>(ws4 + k * kq) + warp * kpad * kFinRT;
  __syncthreads();
  const double unit = *bound * (double)__uint_as_float(*vmax) * 0x1p-62;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ngroups = (rows + kFinRT - 1) / kFinRT;
  for (int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; grp < ngroups; grp += nwarps) {
    const int64_t i0 = grp * kFinRT;
    // the RT rows are one contiguous block of Yq: every 16-byte load is issued
    // before any is used (PER in flight per lane), then converted and cleared
    constexpr int PER = CW * 16;  // >= kFinRT * kpad / 2 / 32 for kpad <= 128 CW
    const int nch = (int)(min((int64_t)kFinRT, rows - i0) * kpad / 2);
    const ulonglong2* yg = reinterpret_cast<const ulonglong2*>(Yq + i0 * kpad);
    ulonglong2 buf[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int q = lane + 32 * u;
      buf[u] = q < nch ? yg[q] : make_ulonglong2(0ull, 0ull);
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int q = lane + 32 * u;
      if (q < kFinRT * kpad / 2) {
        const unsigned long long pr[2] = {buf[u].x, buf[u].y};
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int e = 2 * q + h2, r = e / kpad, c = e - r * kpad;
          ys[c * kFinRT + r] = pr[h2] ? (float)((double)pr[h2] * unit) : 0.f;
        }
      }
    }
    __syncwarp();
    float4 acc[kFinRT][CW];
#pragma unroll
    for (int r = 0; r < kFinRT; ++r)
#pragma unroll
      for (int j = 0; j < CW; ++j) acc[r][j] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int l = 0; l < k; ++l) {
      const float4 y0 = *reinterpret_cast<const float4*>(ys + l * kFinRT);
      const float4 y1 = *reinterpret_cast<const float4*>(ys + l * kFinRT + 4);
      const float yv[kFinRT] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const int ch = lane + 32 * j;
        if (ch < kq) {
          const float4 w = ws4[l * kq + ch];
#pragma unroll
          for (int r = 0; r < kFinRT; ++r) {
            const float2 lo = __ffma2_rn(make_float2(yv[r], yv[r]), make_float2(w.x, w.y),
                                         make_float2(acc[r][j].x, acc[r][j].y));
            const float2 hi = __ffma2_rn(make_float2(yv[r], yv[r]), make_float2(w.z, w.w),
                                         make_float2(acc[r][j].z, acc[r][j].w));
            acc[r][j] = make_float4(lo.x, lo.y, hi.x, hi.y);
          }
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < CW; ++j) {
      const int c0 = 4 * (lane + 32 * j);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (c0 + e >= k) continue;
        float v[kFinRT];
#pragma unroll
        for (int r = 0; r < kFinRT; ++r)
          v[r] = e == 0 ? acc[r][j].x : e == 1 ? acc[r][j].y : e == 2 ? acc[r][j].z : acc[r][j].w;
        float* xo = X + (int64_t)(c0 + e) * ldx + i0;
        if (i0 + kFinRT <= rows) {  // ldx and i0 are multiples of 8
          reinterpret_cast<float4*>(xo)[0] = make_float4(v[0], v[1], v[2], v[3]);
          reinterpret_cast<float4*>(xo)[1] = make_float4(v[4], v[5], v[6], v[7]);
        } else {
#pragma unroll
          for (int r = 0; r < kFinRT; ++r)
            if (i0 + r < rows) xo[r] = v[r];
        }
      }
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
