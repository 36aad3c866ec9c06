// k_uside_tc.cuh -- U side, second half: LS_U = Y W on the tensor cores
// ("U = A V (V^T V)^{-1}"), Y = A V the exact fixed-point accumulators of
// k_uside_scatter, W = (V^T V + eps I)^{-1}.
//
// A dense (n x k) x (k x k) product: 200k x 100 x 100 at Large.  The SIMT
// register-tiled kernel (k_uside_finish_rt) was bound by instruction issue;
// here per 128-row tile:
//   * 8 producer warps (16 rows each; lane = 4 consecutive columns, 16-byte
//     loads, 8-byte shared-memory stores; 8 rows in flight)
//     convert the tile's fixed-point rows, find each row's maximum, scale the
//     row by an exact power of two into [2^14, 2^15), split it into fp16 hi/lo
//     (22 significant bits) in the K-major shared-memory layout, and clear the
//     accumulator rows for the next half-step;
//   * W is split the same way once per CTA (per-column power-of-two scales)
//     and stays resident in shared memory as the B operand;
//   * one thread issues kind::f16 MMAs (hi*hi + hi*lo + lo*hi) into TMEM;
//   * 4 epilogue warps (thread = row) undo the two scales (exact) and store
//     the LS rows column-major (coalesced).
// Used when kappa_inf(G_V + eps I) <= 100 (device flag), like the fp32 SIMT
// path it replaces; the fp64 kernel handles the rest.
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc.cuh"

namespace esk {

constexpr int kUtcM = 128;
constexpr int kUtcRows = 8;                          // rows of a producer warp in flight
constexpr int kUtcProdWarps = 8;                     // 16 rows of a tile each
constexpr int kUtcProd = 32 * kUtcProdWarps;
constexpr int kUtcThreads = kUtcProd + 32 + 128;     // producers, MMA, epilogue

ESNMF_DEV int utc_exp(double x) {  // e with x 2^e in [2^14, 2^15), 0 for x == 0
  if (!(x > 0.0)) return 0;
  int ex;
  frexp(x, &ex);
  return 15 - ex;
}

// W (fp64 k x k) -> B operand [n = output column c][K = l] = W[l][c], fp16
// hi/lo with per-column scales; wscale[c] = 2^-eW_c.  One block per column.
__global__ void k_utc_wprep(const double* __restrict__ W, int k, int kn, int kk, uint8_t* __restrict__ wb,
                            float* __restrict__ wscale) {
  __shared__ double red[32];
  const int c = blockIdx.x;
  double mx = 0;
  for (int l = threadIdx.x; l < k; l += blockDim.x) mx = fmax(mx, fabs(W[(int64_t)l * k + c]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    red[0] = m;
  }
  __syncthreads();
  const int e = utc_exp(red[0]);
  if (threadIdx.x == 0) wscale[c] = ldexpf(1.f, -e);
  const uint32_t half = (uint32_t)kn * kk * 2;
  for (int l = threadIdx.x; l < kk; l += blockDim.x) {
    const float w = l < k ? (float)ldexp(W[(int64_t)l * k + c], e) : 0.f;
    const __half hi = __float2half_rn(w);
    const __half lo = __float2half_rn(w - __half2float(hi));
    const uint32_t off = tc::kmajor_off16(c, l, kk);
    *reinterpret_cast<__half*>(wb + off) = hi;
    *reinterpret_cast<__half*>(wb + half + off) = lo;
  }
}

// LS rows of tiles of 128 term rows; 2 A stages, W resident
__global__ void __launch_bounds__(kUtcThreads, 1)
    k_uside_tc(int64_t rows, int64_t ntiles, const double* __restrict__ bound, const uint32_t* __restrict__ vmax,
               const uint8_t* __restrict__ wb, const float* __restrict__ wscale, int k, int kpad, int kn, int kk,
               int acc_cols, unsigned long long* __restrict__ Yq, float* __restrict__ X, int64_t ldx,
               const int* __restrict__ use_fp64) {
  if (*use_fp64) return;  // ill-conditioned: the fp64 kernel handles it
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t wbar, afull[2], aempty[2], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  __shared__ float rscale[2][kUtcM];
  __shared__ __align__(16) float s_ws[256];  // the epilogue's column scales (0: padding)
  for (int c = threadIdx.x; c < 256; c += blockDim.x) s_ws[c] = c < k ? wscale[c] : 0.f;
  uint8_t* base = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t wbytes = (uint32_t)kn * kk * 4;               // hi + lo
  const uint32_t abytes = (uint32_t)kUtcM * kk * 4;            // hi + lo
  uint8_t* ws = base;
  uint8_t* as0 = base + ((wbytes + 1023u) & ~1023u);
  const uint32_t astride = (abytes + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tc::mbar_init(&wbar, 1);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&afull[s], kUtcProd);
      tc::mbar_init(&aempty[s], 1);
      tc::mbar_init(&tfull[s], 1);
      tc::mbar_init(&tempty[s], 128);
    }
    tc::fence_mbar_init();
  }
  if (warp == kUtcProdWarps) tc::tmem_alloc(&tmem_base, 2 * acc_cols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const double unit = *bound * (double)__uint_as_float(*vmax) * 0x1p-62;  // fixed point -> value

  if (warp < kUtcProdWarps) {  // ---- producers: warp w converts rows 16w..16w+15 of a tile ----
    if (threadIdx.x == 0) {
      tc::mbar_arrive_expect_tx(&wbar, wbytes);
      tc::bulk_g2s(ws, wb, wbytes, &wbar);
    }
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t ahalf = (uint32_t)kUtcM * kk * 2;
    const int c4 = 4 * lane;  // this lane's 4 consecutive columns
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      tc::mbar_wait(&aempty[stage], phase ^ 1);   // the MMAs of this stage's last tile are done
      tc::mbar_wait(&tempty[stage], phase ^ 1);   // ... and its epilogue (rscale[stage] is free)
      uint8_t* sa = as0 + stage * astride;
      for (int rr = 0; rr < kUtcM / kUtcProdWarps; rr += kUtcRows) {
        // kUtcRows rows in flight: all loads issued before any use (the clearing
        // stores come after, so they cannot serialise the loads)
        ulonglong2 qv[kUtcRows][2];
#pragma unroll
        for (int q = 0; q < kUtcRows; ++q) {
          const int64_t row = tile * kUtcM + warp * (kUtcM / kUtcProdWarps) + rr + q;
          const bool live = row < rows && c4 < kpad;  // kpad is a multiple of 4
          const ulonglong2* src = reinterpret_cast<const ulonglong2*>(Yq + row * kpad + c4);
          qv[q][0] = live ? __ldcs(src) : make_ulonglong2(0ull, 0ull);
          qv[q][1] = live ? __ldcs(src + 1) : make_ulonglong2(0ull, 0ull);
        }
#pragma unroll
        for (int q = 0; q < kUtcRows; ++q) {
          const int r = warp * (kUtcM / kUtcProdWarps) + rr + q;
          float y[4];
          y[0] = (float)((double)qv[q][0].x * unit);
          y[1] = (float)((double)qv[q][0].y * unit);
          y[2] = (float)((double)qv[q][1].x * unit);
          y[3] = (float)((double)qv[q][1].y * unit);
          float mx = fmaxf(fmaxf(y[0], y[1]), fmaxf(y[2], y[3]));
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
          int e = 0;
          if (mx > 0.f) {
            frexpf(mx, &e);
            e = 15 - e;
          }
          const float sc = __int_as_float((127 + e) << 23);  // 2^e, exact
          if (lane == 0) rscale[stage][r] = __int_as_float((127 - e) << 23);
          if (c4 < kk) {  // 4 consecutive K elements of row r: 8 contiguous bytes in the core matrix
            __half hi[4], lo[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float v = y[j] * sc;
              hi[j] = __float2half_rn(v);
              lo[j] = __float2half_rn(v - __half2float(hi[j]));
            }
            const uint32_t off = tc::kmajor_off16(r, c4, kk);
            ESNMF_CHECK(r < kUtcM && off + 8 <= ahalf && (uint32_t)(sa - smem_raw) + 2 * ahalf <= dyn_smem_bytes());
            *reinterpret_cast<uint2*>(sa + off) = *reinterpret_cast<const uint2*>(hi);
            *reinterpret_cast<uint2*>(sa + ahalf + off) = *reinterpret_cast<const uint2*>(lo);
          }
        }
      }
      tc::fence_async_smem();
      tc::mbar_arrive(&afull[stage]);
      if (++stage == 2) { stage = 0; phase ^= 1; }
    }
  } else if (warp == kUtcProdWarps) {
    if (lane == 0) {  // ---- MMA issuer ----
      tc::mbar_wait(&wbar, 0);
      const uint32_t idesc = tc::make_idesc_f16(kUtcM, kn);
      const uint32_t wh = tc::smem_u32(ws), wl = wh + (uint32_t)kn * kk * 2;
      const uint32_t sbo = (uint32_t)(kk / 8) * 128;
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        tc::mbar_wait(&tempty[stage], phase ^ 1);
        tc::mbar_wait(&afull[stage], phase);
        tc::fence_after();
        const uint32_t ah = tc::smem_u32(as0 + stage * astride), al = ah + (uint32_t)kUtcM * kk * 2;
        const uint32_t d = tmem + (uint32_t)(stage * acc_cols);
        for (int s = 0; s < kk / 16; ++s) {
          const uint32_t o = s * 256;
          const uint64_t dah = tc::make_sdesc(ah + o, 128, sbo), dal = tc::make_sdesc(al + o, 128, sbo);
          const uint64_t dwh = tc::make_sdesc(wh + o, 128, sbo), dwl = tc::make_sdesc(wl + o, 128, sbo);
          tc::mma_f16(d, dah, dwh, idesc, s != 0);
          tc::mma_f16(d, dah, dwl, idesc, 1);
          tc::mma_f16(d, dal, dwh, idesc, 1);
        }
        tc::mma_commit(&aempty[stage]);  // A stage free
        tc::mma_commit(&tfull[stage]);   // accumulator ready
        if (++stage == 2) { stage = 0; phase ^= 1; }
      }
    }
  } else {  // ---- epilogue (4 warps, one per TMEM lane quadrant): thread = row ----
    const int lg = warp & 3;
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      tc::mbar_wait(&tfull[stage], phase);
      tc::mbar_wait(&afull[stage], phase);  // acquire the producers' rscale writes
      tc::fence_after();
      const int r = lg * 32 + lane;
      const int64_t row = tile * kUtcM + r;
      const float rs = rscale[stage][r];
      const uint32_t ta = tmem + (uint32_t)(stage * acc_cols) + ((uint32_t)(lg * 32) << 16);
      for (int c0 = 0; c0 < kn; c0 += 16) {
        uint32_t v[16];
        tc::tmem_ld16(ta + (uint32_t)c0, v);
        tc::tmem_wait_ld();
        if (row < rows) {  // exact powers of two: row scale, column scale (shared memory)
          float ws[16];
#pragma unroll
          for (int v4 = 0; v4 < 4; ++v4) {
            const float4 w4 = reinterpret_cast<const float4*>(s_ws + c0)[v4];
            ws[4 * v4] = w4.x; ws[4 * v4 + 1] = w4.y; ws[4 * v4 + 2] = w4.z; ws[4 * v4 + 3] = w4.w;
          }
          float* xr = X + (int64_t)c0 * ldx + row;
          if (c0 + 16 <= k) {
#pragma unroll
            for (int j = 0; j < 16; ++j) xr[(int64_t)j * ldx] = __uint_as_float(v[j]) * rs * ws[j];
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (c0 + j < k) xr[(int64_t)j * ldx] = __uint_as_float(v[j]) * rs * ws[j];
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&tempty[stage]);
      if (++stage == 2) { stage = 0; phase ^= 1; }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == kUtcProdWarps) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 2 * acc_cols);
  }
}

inline size_t uside_tc_smem(int kn, int kk) {
  return (((size_t)kn * kk * 4 + 1023) & ~(size_t)1023) + 2 * (((size_t)kUtcM * kk * 4 + 1023) & ~(size_t)1023) +
         1024;
}

}  // namespace esk
