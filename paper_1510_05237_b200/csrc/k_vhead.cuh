// k_vhead.cuh -- tensor-core "head" of the V-side product LS_V = A^T Z
// ("A^T U (U^T U)^{-1}", reassociated as A^T (U W), W = (U^T U + eps I)^{-1}).
//
// Split of the product by term.  The h most frequent terms ("head", chosen at
// create time from the document frequencies of A) hold a dense-ish block of
// A^T (Large: the 512 most frequent terms hold 44 % of the stored entries at
// 13 % density), so their part of the product is a dense GEMM
//     LS_head[docs, :] = A^T[docs, head] * Z[head, :]
// that runs on the 5th-generation tensor cores (tcgen05.mma, accumulator in
// TMEM).  The remaining "tail" terms keep the row-gather kernel
// (k_spmm_docs.cuh) with the head terms masked out of its active-term bitmap.
//
// Precision (fp32-level, BJ:5 "relative 1e-5"): every operand is split into
// two fp16 halves, x = x_hi + x_lo with x_hi = fp16(x), x_lo = fp16(x - x_hi)
// (22 significant bits), after an exact power-of-two scaling that puts the
// operand's maximum in [2^14, 2^15): A by one scale per shard, Z by one scale
// per topic column.  Three MMAs per K-step accumulate a_hi z_hi + a_hi z_lo +
// a_lo z_hi in fp32 (the dropped a_lo z_lo is < 2^-22 relative); the epilogue
// multiplies by the inverse power of two (exact).
//
// Layouts (K-major, no swizzle; core matrix = 8 rows x 16 bytes):
//   head tiles  [tile of 128 documents][chunk of 64 head terms] -> 32 KB =
//               hi block (128 x 64 fp16) then lo block, built once at create;
//   Z chunks    [chunk][hi block (kn x 64 fp16), lo block], rebuilt per half-step.
// Pipeline (one CTA per SM, persistent over document tiles): warp 0 issues
// 1-D bulk copies (TMA engine) of a tile chunk and the matching Z chunk into a
// STAGES-deep shared-memory ring; warp 1 (one thread) issues the MMAs into one
// of two TMEM accumulators; warps 2-5 drain the other accumulator into the LS
// buffer (column-major, coalesced stores); the gather kernel runs next and adds
// the tail part (its read of X is cheap next to its k-wide gathers).
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc.cuh"

namespace esk {

constexpr int kHeadK = 64;                                   // head terms per chunk
constexpr int kHeadM = 128;                                  // documents per tile (MMA M)
constexpr uint32_t kHeadABytes = kHeadM * kHeadK * 2 * 2;    // hi + lo fp16 = 32 KB
constexpr uint32_t kHeadAHalf = kHeadM * kHeadK * 2;         // 16 KB
constexpr int kHeadThreads = 192;                            // producer, MMA, 4 epilogue warps

// exponent e such that x * 2^e lies in [2^14, 2^15) (0 for x == 0)
ESNMF_DEV int head_exp(float x) {
  if (!(x > 0.f)) return 0;
  int ex;
  frexpf(x, &ex);  // x = f 2^ex, f in [0.5, 1)
  return 15 - ex;
}

// max of the (non-negative) values of a CSR shard, as float bits
__global__ void k_absmax_ent(const int2* __restrict__ ent, int64_t nnz, unsigned* __restrict__ out) {
  unsigned m = 0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned)ent[q].y & 0x7FFFFFFFu);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// dense head tiles from the head prefix of the document rows (warp per row);
// buffer zeroed first
__global__ void k_head_build(const int64_t* __restrict__ ptr, const int32_t* __restrict__ nh,
                             const int2* __restrict__ ent, int64_t rows,
                             const int32_t* __restrict__ headslot, const unsigned* __restrict__ amax_bits,
                             int nchunks, uint8_t* __restrict__ atile) {
  const int eA = head_exp(__uint_as_float(*amax_bits));
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < rows; row += nw) {
    const int64_t s = ptr[row], e = s + nh[row];  // head entries lead the row (k_reorder_head)
    const int64_t tile = row / kHeadM;
    const int r = (int)(row % kHeadM);
    for (int64_t q = s + lane; q < e; q += 32) {
      const int2 en = ent[q];
      const int slot = headslot[en.x];
      if (slot < 0) continue;
      const float a = ldexpf(__int_as_float(en.y), eA);
      const __half hi = __float2half_rn(a);
      const __half lo = __float2half_rn(a - __half2float(hi));
      uint8_t* b = atile + ((size_t)tile * nchunks + (slot / kHeadK)) * kHeadABytes;
      const uint32_t off = tc::kmajor_off16(r, slot % kHeadK, kHeadK);
      *reinterpret_cast<__half*>(b + off) = hi;
      *reinterpret_cast<__half*>(b + kHeadAHalf + off) = lo;
    }
  }
}

// clear the head terms' bits from the gather kernel's active-term bitmap
__global__ void k_head_bits_clear(const int32_t* __restrict__ headterm, int h, uint32_t* __restrict__ bits) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < h) {
    const int32_t t = headterm[s];
    atomicAnd(&bits[t >> 5], ~(1u << (t & 31)));
  }
}

// Z chunks of the head terms (one CTA per topic column c): per-column scale,
// fp16 hi/lo split, K-major layout; colscale[c] = 2^-(eA + eZ_c)
__global__ void k_zhead_prep(const float* __restrict__ Z, int zs, const int32_t* __restrict__ headterm, int h,
                             int kn, const unsigned* __restrict__ amax_bits, uint8_t* __restrict__ zbuf,
                             float* __restrict__ colscale) {
  __shared__ float red[32];
  const int c = blockIdx.x;
  float mx = 0.f;
  for (int s = threadIdx.x; s < h; s += blockDim.x) mx = fmaxf(mx, fabsf(Z[(int64_t)headterm[s] * zs + c]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const int eZ = head_exp(red[0]);
  const int eA = head_exp(__uint_as_float(*amax_bits));
  if (threadIdx.x == 0) colscale[c] = ldexpf(1.f, -(eA + eZ));
  const uint32_t zhalf = (uint32_t)kn * kHeadK * 2;
  for (int s = threadIdx.x; s < h; s += blockDim.x) {
    const float z = ldexpf(Z[(int64_t)headterm[s] * zs + c], eZ);
    const __half hi = __float2half_rn(z);
    const __half lo = __float2half_rn(z - __half2float(hi));
    uint8_t* b = zbuf + (size_t)(s / kHeadK) * 2 * zhalf;
    const uint32_t off = tc::kmajor_off16(c, s % kHeadK, kHeadK);
    *reinterpret_cast<__half*>(b + off) = hi;
    *reinterpret_cast<__half*>(b + zhalf + off) = lo;
  }
}

ESNMF_DEV uint32_t head_stage_bytes(int kn) { return (kHeadABytes + (uint32_t)kn * kHeadK * 4 + 1023u) & ~1023u; }

// X[c][row] = A^T[row, head] Z[head, c] for every document row of the shard (the
// gather kernel then adds the tail terms: k_spmm_docs<.., ACCUM = true>)
template <int STAGES>
__global__ void __launch_bounds__(kHeadThreads, 1)
    k_vhead_tc(const uint8_t* __restrict__ atile, const uint8_t* __restrict__ zbuf,
               const float* __restrict__ colscale, int64_t rows, int64_t ntiles, int nchunks, int k, int kn,
               int acc_cols, float* __restrict__ X, int64_t ldx) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  uint8_t* base = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t zhalf = (uint32_t)kn * kHeadK * 2;
  const uint32_t zbytes = 2 * zhalf;
  const uint32_t stage_bytes = head_stage_bytes(kn);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full_bar[s], 1);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 128);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(&tmem_base, 2 * acc_cols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---- producer: bulk copies into the smem ring ----
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int q = 0; q < nchunks; ++q) {
          tc::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = base + stage * stage_bytes;
          tc::mbar_arrive_expect_tx(&full_bar[stage], kHeadABytes + zbytes);
          tc::bulk_g2s(sa, atile + ((size_t)tile * nchunks + q) * kHeadABytes, kHeadABytes, &full_bar[stage]);
          tc::bulk_g2s(sa + kHeadABytes, zbuf + (size_t)q * zbytes, zbytes, &full_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      const uint32_t idesc = tc::make_idesc_f16(kHeadM, kn);
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        tc::mbar_wait(&tempty[acc], aphase ^ 1);
        tc::fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * acc_cols);
        for (int q = 0; q < nchunks; ++q) {
          tc::mbar_wait(&full_bar[stage], phase);
          tc::fence_after();
          const uint32_t ah = tc::smem_u32(base + stage * stage_bytes);
          const uint32_t al = ah + kHeadAHalf, zh = ah + kHeadABytes, zl = zh + zhalf;
#pragma unroll
          for (int s = 0; s < kHeadK / 16; ++s) {
            const uint32_t o = s * 256;
            const uint64_t dah = tc::make_sdesc(ah + o, 128, 1024), dal = tc::make_sdesc(al + o, 128, 1024);
            const uint64_t dzh = tc::make_sdesc(zh + o, 128, 1024), dzl = tc::make_sdesc(zl + o, 128, 1024);
            tc::mma_f16(d, dah, dzh, idesc, (q | s) != 0);
            tc::mma_f16(d, dah, dzl, idesc, 1);
            tc::mma_f16(d, dal, dzh, idesc, 1);
          }
          tc::mma_commit(&empty_bar[stage]);  // frees the smem slot when these MMAs finish
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc::mma_commit(&tfull[acc]);          // accumulator ready for the epilogue
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else {  // ---- epilogue: TMEM -> registers -> X += head part ----
    const int lg = warp & 3;  // TMEM lanes 32*lg .. 32*lg+31
    int acc = 0;
    uint32_t aphase = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      tc::mbar_wait(&tfull[acc], aphase);
      tc::fence_after();
      const int64_t row = tile * kHeadM + lg * 32 + lane;
      const uint32_t ta = tmem + (uint32_t)(acc * acc_cols) + ((uint32_t)(lg * 32) << 16);
      for (int c0 = 0; c0 < kn; c0 += 16) {
        uint32_t v[16];
        tc::tmem_ld16(ta + (uint32_t)c0, v);
        tc::tmem_wait_ld();
        if (row < rows) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int c = c0 + j;
            if (c < k) X[(int64_t)c * ldx + row] = __uint_as_float(v[j]) * colscale[c];  // exact 2^-e scale
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 2 * acc_cols);
  }
}

}  // namespace esk
