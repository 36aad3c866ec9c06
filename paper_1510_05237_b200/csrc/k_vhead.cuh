// k_vhead.cuh -- tensor-core "head" of the V-side product LS_V = A^T Z
// ("A^T U (U^T U)^{-1}", reassociated as A^T (U W), W = (U^T U + eps I)^{-1}).
//
// Split of the product by term.  The h most frequent terms ("head", chosen at
// create time from the document frequencies of A) hold a dense-ish block of
// A^T (Large: the 1024 most frequent terms hold 52 % of the stored entries at
// 7.6 % density), so their part of the product is a GEMM
//     LS_head[docs, :] = A^T[docs, head] * Z[head, :]
// on the 5th-generation tensor cores (tcgen05.mma, accumulator in TMEM).  The
// remaining "tail" terms keep the row-gather kernel (k_spmm_tail.cuh), which
// reads only the tail part of every row (head entries are stored first, sorted
// by head slot, with the slot in place of the term id: k_reorder_head).
//
// Precision (fp32-level, BJ:5 "relative 1e-5"): every operand is split into
// two fp16 halves, x = x_hi + x_lo with x_hi = fp16(x), x_lo = fp16(x - x_hi)
// (22 significant bits), after an exact power-of-two scaling that puts the
// operand's maximum in [2^14, 2^15): A by one scale per shard, Z by one scale
// per topic column.  Three MMAs per K-step accumulate a_hi z_hi + a_hi z_lo +
// a_lo z_hi in fp32 (the dropped a_lo z_lo is < 2^-22 relative); the epilogue
// multiplies by the inverse power of two (exact).
//
// The A^T tiles are built ON CHIP from the sparse head entries (a dense copy
// would cost 4 bytes per cell: 4 GB per pass at h = 1024 for 7.6 % density).
// At create time the head entries are copied into per-(tile, chunk) segments
// (k_head_count / k_head_fill): entry = (row in tile * 64 + slot in chunk,
// value), so one chunk of one tile is one contiguous run.  Per chunk, 128
// producer threads zero a shared-memory stage (one row each), read the run
// coalesced and scatter it as fp16 hi/lo in the K-major layout, while one of
// them bulk-copies (TMA engine) the matching Z chunk.
// Layouts (K-major, no swizzle; core matrix = 8 rows x 16 bytes):
//   A stage   hi block (128 x 64 fp16) then lo block      (32 KB)
//   Z chunks  [chunk][hi block (kn x 64 fp16), lo block], rebuilt per half-step.
// Roles (one CTA per SM, persistent over document tiles): a loader thread
// bulk-copies runs + Z chunks STAGES ahead, warps 0-3 build A stages, warp 4
// (one thread) issues the MMAs into one of two TMEM accumulators, warps 6-13
// drain the other accumulator, add the tail part the gather staged row-major,
// and store the LS buffer column-major (32 consecutive rows per warp, coalesced).
#pragma once
#include <cuda_fp16.h>

#include <climits>

#include "common.cuh"
#include "k_vtail.cuh"
#include "tc.cuh"

namespace esk {

#ifndef ESNMF_HEAD_K
#define ESNMF_HEAD_K 64
#endif
constexpr int kHeadK = ESNMF_HEAD_K;                         // head terms per chunk (MMA K per stage)
static_assert(kHeadK == 32 || kHeadK == 64, "chunk entries encode the slot in 6 bits");
constexpr int kHeadM = 128;                                  // documents per tile (MMA M)
constexpr uint32_t kHeadABytes = kHeadM * kHeadK * 2 * 2;    // hi + lo fp16 = 32 KB
constexpr uint32_t kHeadAHalf = kHeadM * kHeadK * 2;         // 16 KB
constexpr int kHeadMax = 31 * ESNMF_HEAD_K;                    // largest head (terms): <= 31 sparse chunks (one run offset per loader lane)

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

// clear the head terms' bits from the gather kernel's active-term bitmap
__global__ void k_head_bits_clear(const int32_t* __restrict__ headterm, int h, uint32_t* __restrict__ bits,
                                  const int* __restrict__ gate) {
  if (gate && !*gate) return;
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

// Paper-order tail mode (k_vtail.cuh): one CTA per topic column c.
//   Z_head[s][c] = (U W)[headterm[s]][c]   (fp64, k_form_z64)
//   one accumulator scale 2^sc_c for both parts of LS_V[:, c]:
//     head:  A' = A 2^eA,             Z'[s][c] = Z 2^(sc_c - eA)
//     tail:  Y' = Y 2^(s_j - 15),     W'[j][c] = W 2^(sc_c - s_j + 15)
//   sc_c the largest exponent keeping max |Z'[:, c]| and every |W'[j][c]| below
//   2^15 (fp16 hi/lo operands); colscale[c] = 2^-sc_c.
// zbuf: head chunks as before; wbuf chunk q: [hi | lo] of kn x w_q (K-major,
// w_q = min(64, kn - 64 q), chunk stride kn * kHeadK * 4 bytes).  Rows c >= k of
// both and K columns j >= k of W' stay zero (cleared at create).
__global__ void k_vside_prep(const double* __restrict__ Z64, const int32_t* __restrict__ rowmap,
                             const int32_t* __restrict__ headterm, int h, const double* __restrict__ W, int k, int kn,
                             const unsigned* __restrict__ amax_bits, const int* __restrict__ shift,
                             uint8_t* __restrict__ zbuf, uint8_t* __restrict__ wbuf, float* __restrict__ colscale,
                             const int* __restrict__ fallback) {
  __shared__ double wc[256];
  __shared__ float zs[kHeadMax];
  __shared__ float redf[32];
  __shared__ int redi[32];
  const int c = blockIdx.x;
  for (int j = threadIdx.x; j < k; j += blockDim.x) wc[j] = W[(int64_t)j * k + c];
  __syncthreads();
  float zmax = 0.f;
  for (int s = threadIdx.x; s < h; s += blockDim.x) {
    const int32_t term = headterm[s];
    const double z = rowmap[term] >= 0 ? Z64[(int64_t)term * k + c] : 0.0;  // Z = U W (fp64, k_form_z64)
    zs[s] = (float)z;
    zmax = fmaxf(zmax, fabsf((float)z));
  }
  const bool fb = *fallback != 0;  // Z-row gather this iteration: no (Y_tail W) chunks
  // the W' bound: min_j (e(|W_jc|) + s_j - 15) over the nonzero entries
  int wlim = INT_MAX;
  // (a row j whose column of U has no tail entry multiplies Y_tail[:, j] = 0: skipped, W' = 0)
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const float wf = fabsf((float)wc[j]);
    if (wf > 0.f && shift[j] != kNoTail && !fb) wlim = min(wlim, head_exp(wf) + shift[j] - 15);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    zmax = fmaxf(zmax, __shfl_xor_sync(kFull, zmax, o));
    wlim = min(wlim, __shfl_xor_sync(kFull, wlim, o));
  }
  if ((threadIdx.x & 31) == 0) {
    redf[threadIdx.x >> 5] = zmax;
    redi[threadIdx.x >> 5] = wlim;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float zm = 0.f;
    int wl = INT_MAX;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      zm = fmaxf(zm, redf[w]);
      wl = min(wl, redi[w]);
    }
    const int eA = head_exp(__uint_as_float(*amax_bits));
    int sc = zm > 0.f ? eA + head_exp(zm) : INT_MAX;
    sc = min(sc, wl);
    if (sc == INT_MAX) sc = 0;
    redi[0] = sc;
    colscale[c] = ldexpf(1.f, -sc);
  }
  __syncthreads();
  const int sc = redi[0];
  const int eA = head_exp(__uint_as_float(*amax_bits));
  const uint32_t zhalf = (uint32_t)kn * kHeadK * 2;
  for (int s = threadIdx.x; s < h; s += blockDim.x) {
    const float z = ldexpf(zs[s], sc - eA);
    const __half hi = __float2half_rn(z);
    const __half lo = __float2half_rn(z - __half2float(hi));
    uint8_t* b = zbuf + (size_t)(s / kHeadK) * 2 * zhalf;
    const uint32_t off = tc::kmajor_off16(c, s % kHeadK, kHeadK);
    *reinterpret_cast<__half*>(b + off) = hi;
    *reinterpret_cast<__half*>(b + zhalf + off) = lo;
  }
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const float w = (shift[j] == kNoTail || fb) ? 0.f : (float)ldexp(wc[j], sc - shift[j] + 15);
    const __half hi = __float2half_rn(w);
    const __half lo = __float2half_rn(w - __half2float(hi));
    const int q = j / kHeadK, wq = min(kHeadK, kn - kHeadK * q);
    uint8_t* b = wbuf + (size_t)q * 2 * zhalf;
    const uint32_t off = tc::kmajor_off16(c, j % kHeadK, wq);
    *reinterpret_cast<__half*>(b + off) = hi;
    *reinterpret_cast<__half*>(b + (size_t)kn * wq * 2 + off) = lo;
  }
}

// Dense A^T head tiles for the first nd chunks (the densest slots, where a run
// would hold more entries than a stage can stage), built per (tile, group of
// kHeadDenseG chunks) in shared memory and written out whole (coalesced, no memset
// of the tiles first): 16 warps, a warp per document row of the tile scatters the
// row's entries of the group's chunks (distinct terms: distinct cells), then the
// block copies the tiles out.
constexpr int kHeadDenseG = 4;
__global__ void __launch_bounds__(512) k_head_dense_tiles(const int64_t* __restrict__ ptr,
                                                          const int32_t* __restrict__ nh,
                                                          const int2* __restrict__ ent, int64_t rows,
                                                          const int32_t* __restrict__ headslot,
                                                          const unsigned* __restrict__ amax_bits, int nd,
                                                          uint8_t* __restrict__ atile) {
  extern __shared__ __align__(16) uint8_t dt[];  // [kHeadDenseG][kHeadABytes]
  const int64_t tile = blockIdx.x;
  const int g0 = blockIdx.y * kHeadDenseG, ng = min(kHeadDenseG, nd - g0);
  const int eA = head_exp(__uint_as_float(*amax_bits));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < ng * (int)(kHeadABytes / 16); i += blockDim.x)
    reinterpret_cast<uint4*>(dt)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  for (int r = warp; r < kHeadM; r += nw) {
    const int64_t row = tile * kHeadM + r;
    if (row >= rows) break;  // warp-uniform
    const int64_t s = ptr[row], e = s + nh[row];
    for (int64_t q = s + lane; q < e; q += 32) {
      const int2 en = ent[q];
      const int sl = headslot[en.x], ch = sl / kHeadK - g0;
      if (ch < 0 || ch >= ng) continue;
      const float a = ldexpf(__int_as_float(en.y), eA);
      const __half hi = __float2half_rn(a);
      const __half lo = __float2half_rn(a - __half2float(hi));
      uint8_t* b = dt + (size_t)ch * kHeadABytes;
      const uint32_t off = tc::kmajor_off16(r, sl % kHeadK, kHeadK);
      *reinterpret_cast<__half*>(b + off) = hi;
      *reinterpret_cast<__half*>(b + kHeadAHalf + off) = lo;
    }
  }
  __syncthreads();
  uint4* dst = reinterpret_cast<uint4*>(atile + ((size_t)tile * nd + g0) * kHeadABytes);
  for (int i = threadIdx.x; i < ng * (int)(kHeadABytes / 16); i += blockDim.x) dst[i] = reinterpret_cast<uint4*>(dt)[i];
}

// per (tile, chunk) counts of head entries (warp per document; head entries
// lead each row, k_reorder_head)
__global__ void k_head_count(const int64_t* __restrict__ ptr, const int32_t* __restrict__ nh,
                             const int2* __restrict__ ent, int64_t rows, const int32_t* __restrict__ headslot,
                             int nd, int nsp, unsigned long long* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < rows; row += nw) {
    const int64_t s = ptr[row], e = s + nh[row], tile = row / kHeadM;
    for (int64_t q = s + lane; q < e; q += 32) {
      const int ch = headslot[ent[q].x] / kHeadK - nd;  // sparse chunk index
      if (ch >= 0) atomicAdd(&cnt[tile * nsp + ch], 1ull);
    }
  }
}

// scatter into the segments: (row in tile << 6 | slot in chunk, value); the
// order inside a segment is irrelevant (each entry lands in its own cell)
__global__ void k_head_fill(const int64_t* __restrict__ ptr, const int32_t* __restrict__ nh,
                            const int2* __restrict__ ent, int64_t rows, const int32_t* __restrict__ headslot,
                            int nd, int nsp, unsigned long long* __restrict__ cursor, int2* __restrict__ hseg) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < rows; row += nw) {
    const int64_t s = ptr[row], e = s + nh[row], tile = row / kHeadM;
    const int r = (int)(row % kHeadM);
    for (int64_t q = s + lane; q < e; q += 32) {
      const int2 en = ent[q];
      const int sl = headslot[en.x];
      const int ch = sl / kHeadK - nd;
      if (ch < 0) continue;
      const unsigned long long pos = atomicAdd(&cursor[tile * nsp + ch], 1ull);
      hseg[pos] = make_int2((r << 6) | (sl % kHeadK), en.y);
    }
  }
}

// *need = some column's predicted selection failed (done[c] == 0): the deferred
// LS buffer must be written after all (the gated head re-run)
__global__ void k_any_undone(const int32_t* __restrict__ done, int k, int* __restrict__ need) {
  int any = 0;
  for (int c = threadIdx.x; c < k; c += blockDim.x) any |= done[c] == 0;
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) *need = any;
}

// fused V-side selection pass 1 (k_sel_pred_sort): pred == nullptr = off
struct SelFuse {
  const uint32_t* pred;  // [k] predicted threshold bits
  int32_t* npos;         // [k] positives per column (+=)
  uint64_t* pcand;       // [k][pcap] candidate keys
  int32_t* pfill;        // [k]
  int pcap;
  int64_t row0;
};

#ifndef ESNMF_HEAD_EXP
#define ESNMF_HEAD_EXP 0
#endif
// -DESNMF_HEAD_EXP=3 (development): per-role barrier-wait cycles of CTAs 0 and 77,
// printed at the end of k_vhead_otf (loader: empty, producers: raw_full, MMA:
// a_full + tempty, epilogue: tfull)
#if ESNMF_HEAD_EXP == 3
#define HT_WAIT(bar, ph)                  \
  {                                       \
    const long long t0_ = clock64();      \
    tc::mbar_wait(bar, ph);               \
    ht_wait += clock64() - t0_;           \
  }
#else
#define HT_WAIT(bar, ph) tc::mbar_wait(bar, ph)
#endif
// waits off the critical path (the epilogue has a whole tile of slack) suspend
// instead of polling; ESNMF_HEAD_SLEEP_ALL=1 makes every role's wait suspend
#ifndef ESNMF_HEAD_SLEEP_NS
#define ESNMF_HEAD_SLEEP_NS 20000
#endif
#ifndef ESNMF_HEAD_SLEEP_ALL
#define ESNMF_HEAD_SLEEP_ALL 0
#endif
#if ESNMF_HEAD_EXP == 3
#define HT_WAIT_SLOW(bar, ph) HT_WAIT(bar, ph)
#else
#define HT_WAIT_SLOW(bar, ph) tc::mbar_wait_sleep(bar, ph, ESNMF_HEAD_SLEEP_NS)
#if ESNMF_HEAD_SLEEP_ALL
#undef HT_WAIT
#define HT_WAIT(bar, ph) tc::mbar_wait_sleep(bar, ph, ESNMF_HEAD_SLEEP_NS)
#endif
#endif
#ifndef ESNMF_HEAD_PROD_WARPS
#define ESNMF_HEAD_PROD_WARPS 4
#endif
constexpr int kHeadProdWarps = ESNMF_HEAD_PROD_WARPS;   // producer warps
constexpr int kHeadProd = 32 * kHeadProdWarps;          // producer threads
constexpr int kHeadMmaWarp = kHeadProdWarps, kHeadLoadWarp = kHeadProdWarps + 1, kHeadEpiWarp = kHeadProdWarps + 2;
constexpr int kHeadRaw = 16 * kHeadK;                  // entries of a chunk's run staged in smem
constexpr uint32_t kHeadRawBytes = kHeadRaw * 8 + 16;  // (+1 entry of alignment skew, rounded)
constexpr int kHeadEpi = 256;                          // epilogue threads (2 warps per TMEM lane quadrant)
constexpr int kHeadOtfThreads = kHeadProd + 32 + 32 + kHeadEpi;  // producers, MMA, loader, epilogue
#ifndef ESNMF_HEAD_PF
#define ESNMF_HEAD_PF 6
#endif
constexpr int kHeadPf = ESNMF_HEAD_PF;                             // rounds of L2 prefetch ahead of the copies

// one arrival per warp (after __syncwarp: the lanes' shared-memory writes and
// fences are ordered before lane 0's arrive) instead of one per thread: 4 / 8
// arrivals on the producers' and the epilogue's barriers instead of 128 / 256
#ifndef ESNMF_HEAD_WARP_ARRIVE
#define ESNMF_HEAD_WARP_ARRIVE 1
#endif
constexpr bool kHeadWarpArrive = ESNMF_HEAD_WARP_ARRIVE != 0;
// -DESNMF_HEAD_SKIP=bits (timing experiments only, results wrong): 1 no sparse
// build, 2 no dense A copies, 4 no MMAs, 8 no epilogue work, 16 no run copies
#ifndef ESNMF_HEAD_SKIP
#define ESNMF_HEAD_SKIP 0
#endif
ESNMF_DEV void head_arrive(uint64_t* bar) {
  if (kHeadWarpArrive) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) tc::mbar_arrive(bar);
  } else {
    tc::mbar_arrive(bar);
  }
}

// wide accumulators (2 kn TMEM columns each, the a_hi z_lo part beside the rest):
// 2 MMAs per K-step (tensor-core operand reads from shared memory: A_hi once)
#ifndef ESNMF_HEAD_WIDE
#define ESNMF_HEAD_WIDE 1
#endif
__host__ __device__ __forceinline__ bool head_wide(int kn) { return ESNMF_HEAD_WIDE && 2 * kn <= 256; }

// stage = [A hi|lo 32 KB][Z chunk hi|lo][raw entries of the chunk's run]
ESNMF_DEV uint32_t head_stage_bytes(int kn) {
  return (kHeadABytes + (uint32_t)kn * kHeadK * 4 + kHeadRawBytes + 1023u) & ~1023u;
}

// X[c][row] = Xt[row][c] + A^T[row, head] Z[head, c] for every document row of
// the shard (the tail gather stored its part row-major in Xt: k_spmm_tail<.., TROW>).
// Roles: warp 5 (one thread) bulk-copies each (tile, chunk) run of head
// entries and the Z chunk into a stage (TMA engine, STAGES ahead); warps 0-3
// zero the stage's A block and scatter the run into it; warp 4 (one thread)
// issues the MMAs; warps 6-13 drain TMEM into X (two per lane quadrant).
// Paper-order tail (k_vtail.cuh; nyc > 0): after the nchunks head chunks of a
// tile come nyc chunks of (Y_tail W): A operand = the tile's Y_tail chunk
// (ytile, fp16 hi/lo, 128 x w_q), B operand = W chunk q (wbuf, kn x w_q),
// w_q = min(64, kn - 64 q) -- the same stage, copied like a dense tile, into the
// same accumulator (the scales of Z, W and Y_tail are chosen per column so both
// parts carry 2^sc_c: k_vside_prep).  Xt is then null.
// Epilogue of one 128-row tile (one thread per row: TMEM lane quadrant lg, columns
// [cbeg, cend) of its warp): X[c][row] = Xt[row][c] + colscale[c] * acc[row][c], and the
// fused selection pass 1 (positive counts in cnt2, candidate keys to fz.pcand).
template <bool FUSE>
__device__ __forceinline__ void head_epi_tile(int64_t row, uint32_t ta, uint32_t lo_off, int cbeg, int cend,
                                              bool no_mma, bool xstore, int k,
                                              const float* s_cs, int64_t rows, float* __restrict__ X,
                                              int64_t ldx, const float* __restrict__ Xt, int kpad, const SelFuse& fz,
                                              const uint32_t* s_pred, uint32_t (&cnt2)[4][8]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < (FUSE ? 4 : 1); ++q) {
    for (int c0 = cbeg + 16 * q; c0 < (FUSE ? min(cend, cbeg + 16 * q + 1) : cend); c0 += 16) {
      uint32_t v[16];
      if (ESNMF_HEAD_SKIP & 64) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __float_as_uint((float)(j + c0) * 1e-30f);
      } else {
      tc::tmem_ld16(ta + (uint32_t)c0, v);
      if (lo_off) {  // wide accumulator: columns [kn, 2 kn) hold the a_hi z_lo part
        uint32_t v2[16];
        tc::tmem_ld16(ta + lo_off + (uint32_t)c0, v2);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(v2[j]));
      }
      tc::tmem_wait_ld();
      }
      if (no_mma) {  // no MMA wrote the accumulator (no head, tail staged in Xt)
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0u;
      }
      float x[16];
      const bool live = row < rows;
      if (Xt && live) {  // X = tail part (row-major staging, k_spmm_tail<TROW>) + head part
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4) {
          const int c = c0 + 4 * v4;
          const float4 t4 = c < kpad ? *reinterpret_cast<const float4*>(Xt + row * kpad + c)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
          x[4 * v4] = t4.x; x[4 * v4 + 1] = t4.y; x[4 * v4 + 2] = t4.z; x[4 * v4 + 3] = t4.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = 0.f;
      }
      {  // column scales from shared memory (0 for padding columns c >= k): exact 2^-e
        const float4* cs4 = reinterpret_cast<const float4*>(s_cs + c0);
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4) {
          const float4 cs = cs4[v4];
          x[4 * v4] = fmaf(__uint_as_float(v[4 * v4]), cs.x, x[4 * v4]);
          x[4 * v4 + 1] = fmaf(__uint_as_float(v[4 * v4 + 1]), cs.y, x[4 * v4 + 1]);
          x[4 * v4 + 2] = fmaf(__uint_as_float(v[4 * v4 + 2]), cs.z, x[4 * v4 + 2]);
          x[4 * v4 + 3] = fmaf(__uint_as_float(v[4 * v4 + 3]), cs.w, x[4 * v4 + 3]);
        }
      }
      if (!live) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = 0.f;
      }
      if (xstore && live && !(ESNMF_HEAD_SKIP & 32)) {
        ESNMF_CHECK(row < ldx);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c0 + j < k) X[(int64_t)(c0 + j) * ldx + row] = x[j];
      }
      if (FUSE) {  // padding columns c >= k hold x = 0: never counted
        uint32_t cdm = 0;  // columns j with a candidate in this lane
        const uint4* p4 = reinterpret_cast<const uint4*>(s_pred + c0);
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4) {
          const uint4 pr = p4[v4];
          const uint32_t pj[4] = {pr.x, pr.y, pr.z, pr.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int j = 4 * v4 + i;
            if (!(ESNMF_HEAD_SKIP & 256)) cnt2[q][j >> 1] += (uint32_t)(x[j] > 0.f) << (16 * (j & 1));
            cdm |= (uint32_t)(__float_as_int(x[j]) >= (int)pj[i]) << j;
          }
        }
        uint32_t wm = (ESNMF_HEAD_SKIP & 128) ? 0u : __reduce_or_sync(kFull, cdm);
        while (wm) {  // usually one column, one lane
          const int j = __ffs(wm) - 1;
          wm &= wm - 1;
          const int c = c0 + j;
          const bool cd = (cdm >> j) & 1;
          const unsigned mc = __ballot_sync(kFull, cd);
          int b0 = 0;
          if (lane == 0) b0 = atomicAdd(&fz.pfill[c], __popc(mc));
          b0 = __shfl_sync(kFull, b0, 0);
          const int slot = b0 + __popc(mc & ((1u << lane) - 1u));
          if (cd && slot < fz.pcap) {
            float xv = 0.f;
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) xv = jj == j ? x[jj] : xv;
            fz.pcand[(int64_t)c * fz.pcap + slot] = sel_key(xv, (uint32_t)(fz.row0 + row));
          }
        }
      }
    }
  }
}

template <int STAGES, bool FUSE>
__global__ void __launch_bounds__(kHeadOtfThreads, 1)
    k_vhead_otf(const uint8_t* __restrict__ atile, int nd, const int64_t* __restrict__ hoff,
                const int2* __restrict__ hseg, const unsigned* __restrict__ amax_bits, const uint8_t* __restrict__ zbuf,
                const float* __restrict__ colscale, int64_t rows, int64_t ntiles, int nchunks, int k, int kn,
                int acc_cols, float* __restrict__ X, int64_t ldx, const float* __restrict__ Xt, int kpad,
                SelFuse fz, const uint8_t* __restrict__ ytile, const uint8_t* __restrict__ wbuf, int nyc_arg,
                const int* __restrict__ fallback, int xstore, const int* __restrict__ gate) {
  // gate (the re-run after a fused selection whose prediction failed for some
  // column: the LS buffer is needed after all): nothing to do when *gate == 0
  if (gate && *gate == 0) return;
  // paper-order tail mode, ill-conditioned W (fallback set): the Z-row gather
  // staged the tail rows in Xt this time -- no (Y_tail W) chunks
  const bool fb = fallback && *fallback;
  const int nyc = fb ? 0 : nyc_arg;
  if (!fb && nyc_arg > 0) Xt = nullptr;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t raw_full[STAGES], a_full[STAGES], empty_bar[STAGES], tfull[2], tempty[2];
  __shared__ int64_t s_run[STAGES][2];  // sparse round: [sb, se) of its run (loader -> producers)
  __shared__ uint32_t tmem_base;
  __shared__ int s_npos[256];       // fused selection: positives per column counted by this CTA
  __shared__ __align__(16) uint32_t s_pred[256];  // ... and the predicted thresholds (0xFFFFFFFF: none)
  __shared__ __align__(16) float s_cs[256];       // the epilogue's column scales (0: padding)
  for (int c = threadIdx.x; c < 256; c += blockDim.x) {
    s_npos[c] = 0;
    // thresholds as signed bit patterns: a candidate is (int)bits(x) >= s_pred, which
    // also excludes x <= 0 (threshold >= 1) and, with 0x7FFFFFFF, every finite x
    const uint32_t pu = (FUSE && c < k) ? fz.pred[c] : 0xFFFFFFFFu;
    s_pred[c] = pu == 0u ? 1u : (pu > 0x7F800000u ? 0x7FFFFFFFu : pu);
    s_cs[c] = c < k ? colscale[c] : 0.f;
  }
  uint8_t* base = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ESNMF_CHECK((uint32_t)(base - smem_raw) + STAGES * head_stage_bytes(kn) <= dyn_smem_bytes());
  const uint32_t zhalf = (uint32_t)kn * kHeadK * 2;
  const uint32_t zbytes = 2 * zhalf;
  const uint32_t stage_bytes = head_stage_bytes(kn);
  const uint32_t raw_off = kHeadABytes + zbytes;
  const bool wide = head_wide(kn);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&raw_full[s], 1);
      tc::mbar_init(&a_full[s], kHeadWarpArrive ? kHeadProdWarps : kHeadProd);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], kHeadWarpArrive ? kHeadEpi / 32 : kHeadEpi);
    }
    tc::fence_mbar_init();
  }
  if (warp == kHeadMmaWarp) tc::tmem_alloc(&tmem_base, 2 * acc_cols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  long long ht_wait = 0;
  const long long ht_t0 = clock64();

  if (warp == kHeadLoadWarp) {  // ---- loader: run + Z chunk of each round, STAGES ahead ----
    // One lane issues the copies.  The run offsets hoff[tile * nsp + j] (j <= nsp) of
    // a tile are loaded by the whole warp a tile ahead (one per lane) and taken by
    // shuffle: no dependent global load on the copy path (the producers get a
    // round's run bounds through s_run[stage]).
    const int nsp = nchunks - nd;  // sparse chunks per tile (<= 31)
    const int nall = nchunks + nyc;
    int stage = 0;
    uint32_t phase = 0;
    auto offs_of = [&](int64_t t) -> int64_t {
      return (t < ntiles && lane <= nsp && nsp > 0) ? hoff[t * nsp + lane] : 0;
    };
    int64_t off_cur = offs_of(blockIdx.x);
    int64_t off_nxt = offs_of(blockIdx.x + gridDim.x);
    // L2 prefetch kHeadPf rounds ahead of the copies (a stage's copy is issued only
    // when the MMAs of the round STAGES earlier finish, so its latency is on the
    // critical path; from L2 it is ~1/3 of the HBM latency).  Rounds ahead of the
    // current tile belong to the next one (kHeadPf < nchunks + nyc).
    auto prefetch = [&](int64_t pt, int pq, int64_t offv) {
      int64_t sb = 0, se = 0;
      if (pq >= nd && pq < nchunks) {
        sb = __shfl_sync(kFull, offv, pq - nd);
        se = __shfl_sync(kFull, offv, pq - nd + 1);
      }
      if (lane != 0 || pt >= ntiles) return;
      if (pq >= nchunks) {
        const int yq = pq - nchunks;
        tc::bulk_prefetch_l2(ytile + (size_t)pt * kHeadM * kn * 4 + (size_t)yq * kHeadABytes,
                             (uint32_t)kHeadM * min(kHeadK, kn - kHeadK * yq) * 4u);
      } else if (pq < nd) {
        tc::bulk_prefetch_l2(atile + ((size_t)pt * nd + pq) * kHeadABytes, kHeadABytes);
      } else {
        const int64_t a = sb & ~(int64_t)1;
        const int64_t b = min((int64_t)((se + 1) & ~(int64_t)1), a + (int64_t)kHeadRaw);
        if (b > a) tc::bulk_prefetch_l2(hseg + a, (uint32_t)(b - a) * 8u);
      }
    };
    for (int i = 0; i < min(kHeadPf, nall); ++i) prefetch(blockIdx.x, i, off_cur);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      for (int q = 0; q < nall; ++q) {
        if (kHeadPf > 0) {  // prefetch round (tile, q) + kHeadPf
          const int pq = q + kHeadPf;
          if (pq < nall) prefetch(tile, pq, off_cur);
          else prefetch(tile + gridDim.x, pq - nall, off_nxt);
        }
        int64_t sb = 0, se = 0;
        if (q >= nd && q < nchunks) {
          sb = __shfl_sync(kFull, off_cur, q - nd);
          se = __shfl_sync(kFull, off_cur, q - nd + 1);
        }
        if (lane == 0) {
          HT_WAIT(&empty_bar[stage], phase ^ 1);
          uint8_t* st = base + stage * stage_bytes;
          const int yq = q - nchunks;
          if (q >= nchunks) {  // (Y_tail W) chunk: Y_tail tile chunk + W chunk
            const uint32_t w = (uint32_t)min(kHeadK, kn - kHeadK * yq);
            const uint32_t ab = (uint32_t)kHeadM * w * 4u, bb = (uint32_t)kn * w * 4u;
            ESNMF_CHECK(ab <= kHeadABytes && bb <= zbytes);
            tc::mbar_arrive_expect_tx(&raw_full[stage], ab + bb);
            tc::bulk_g2s(st, ytile + (size_t)tile * kHeadM * kn * 4 + (size_t)yq * kHeadABytes, ab, &raw_full[stage]);
            tc::bulk_g2s(st + kHeadABytes, wbuf + (size_t)yq * zbytes, bb, &raw_full[stage]);
          } else {
            if (q < nd) {  // dense chunk: the A tile itself
              if (ESNMF_HEAD_SKIP & 2) {
                tc::mbar_arrive_expect_tx(&raw_full[stage], zbytes);
              } else {
              tc::mbar_arrive_expect_tx(&raw_full[stage], zbytes + kHeadABytes);
              tc::bulk_g2s(st, atile + ((size_t)tile * nd + q) * kHeadABytes, kHeadABytes, &raw_full[stage]);
              }
            } else {         // sparse chunk: its run of entries
              const int64_t a = sb & ~(int64_t)1;  // 16-byte aligned start
              const int64_t b = min((int64_t)((se + 1) & ~(int64_t)1), a + (int64_t)kHeadRaw);  // even, capped
              const uint32_t rb = (uint32_t)(b - a) * 8u;
              ESNMF_CHECK(rb <= kHeadRawBytes && raw_off + rb <= stage_bytes);
              s_run[stage][0] = sb;
              s_run[stage][1] = se;
              if (ESNMF_HEAD_SKIP & 16) {
                tc::mbar_arrive_expect_tx(&raw_full[stage], zbytes);
              } else {
              tc::mbar_arrive_expect_tx(&raw_full[stage], zbytes + rb);
              if (rb) tc::bulk_g2s(st + raw_off, hseg + a, rb, &raw_full[stage]);
              }
            }
            tc::bulk_g2s(st + kHeadABytes, zbuf + (size_t)q * zbytes, zbytes, &raw_full[stage]);
          }
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      off_cur = off_nxt;
      off_nxt = offs_of(tile + 2 * (int64_t)gridDim.x);
    }
  } else if (warp < kHeadProdWarps) {  // ---- producers: zero + scatter one tile chunk per stage ----
    const int p = threadIdx.x;
    const int eA = head_exp(__uint_as_float(*amax_bits));
    // 2^eA as a float (a product by it rounds like ldexpf: both are correctly rounded)
    const bool fastA = eA >= -126 && eA <= 127;
    const float sA = fastA ? __int_as_float((127 + eA) << 23) : 1.f;
    int stage = 0;
    uint32_t phase = 0;
    auto put = [&](uint8_t* sa, int2 en) {
      const float a = fastA ? __int_as_float(en.y) * sA : ldexpf(__int_as_float(en.y), eA);
      const __half hi = __float2half_rn(a);
      const __half lo = __float2half_rn(a - __half2float(hi));
      ESNMF_CHECK((en.x >> 6) < kHeadM && (en.x & 63) < kHeadK);
      const uint32_t off = tc::kmajor_off16(en.x >> 6, en.x & 63, kHeadK);
      *reinterpret_cast<__half*>(sa + off) = hi;
      *reinterpret_cast<__half*>(sa + kHeadAHalf + off) = lo;
    };
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      for (int q = 0; q < nchunks + nyc; ++q) {
        uint8_t* sa = base + stage * stage_bytes;
        HT_WAIT(&raw_full[stage], phase);  // also: the MMAs of this stage's last round are done
        if (q < nd || q >= nchunks || (ESNMF_HEAD_SKIP & 1)) {  // dense or (Y_tail W) chunk: bulk-copied, nothing to build
          head_arrive(&a_full[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          continue;
        }
        const int64_t sb = s_run[stage][0], se = s_run[stage][1];  // written by the loader before raw_full
        const int64_t a = sb & ~(int64_t)1;
        const int64_t cap = a + (int64_t)kHeadRaw;  // staged: [a, min(se, cap)); the rest from global
        const int2* raw = reinterpret_cast<const int2*>(sa + raw_off);
        // zero the A block: row rz, 16-byte chunks j of its 8 (hi and lo blocks)
        constexpr int kZ = kHeadProd / kHeadM;  // threads per row
#pragma unroll
        for (int jj = 0; jj < (kHeadK / 8) / kZ; ++jj) {
          const int rz = p / kZ, j = (p % kZ) * ((kHeadK / 8) / kZ) + jj;
          const uint32_t off = (uint32_t)((rz >> 3) * (kHeadK / 8) * 128 + j * 128 + (rz & 7) * 16);
          *reinterpret_cast<uint4*>(sa + off) = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(sa + kHeadAHalf + off) = make_uint4(0u, 0u, 0u, 0u);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kHeadProd) : "memory");
        const int64_t se_s = min(se, cap);
        ESNMF_CHECK(sb >= a && se_s - a <= kHeadRaw);
        for (int64_t i = sb + p; i < se_s; i += kHeadProd) put(sa, raw[i - a]);
        for (int64_t i = cap + p; i < se; i += kHeadProd) put(sa, __ldcs(hseg + i));  // long runs only
        tc::fence_async_smem();  // generic-proxy writes -> visible to the tensor core
        head_arrive(&a_full[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == kHeadMmaWarp) {
    if (lane == 0) {  // ---- MMA issuer ----
      const uint32_t idesc = tc::make_idesc_f16(kHeadM, kn);
      // wide (2 kn <= 256): one MMA of A_hi against [Z_hi; Z_lo] (the lo block follows
      // the hi block as row groups kn/8.. of one K-major operand) into columns
      // [0, 2 kn), then A_lo Z_hi into [0, kn): 2 MMAs per K-step instead of 3, and
      // A_hi is read from shared memory once
      const uint32_t idesc_w = tc::make_idesc_f16(kHeadM, wide ? 2 * kn : kn);
      // head-chunk descriptors: everything but the 14-bit start address is fixed
      // (LBO = 128, SBO = (kHeadK / 8) * 128); the stage's addresses are added per round
      const uint64_t hdesc = tc::make_sdesc(0, 128, (kHeadK / 8) * 128);
      const uint32_t sbase = tc::smem_u32(base);
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        HT_WAIT(&tempty[acc], aphase ^ 1);
        tc::fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * acc_cols);
        for (int q = 0; q < nchunks + nyc; ++q) {
          HT_WAIT(&a_full[stage], phase);
          tc::fence_after();
          const uint32_t ah = sbase + (uint32_t)stage * stage_bytes;
          if (q < nchunks) {  // head chunk: K = kHeadK, descriptors advance 256 B (16 units) per K-step
            const uint64_t dah = hdesc | ((ah >> 4) & 0x3FFF), dal = dah + ((kHeadM * kHeadK * 2) >> 4);
            const uint64_t dzh = dah + (kHeadABytes >> 4), dzl = dzh + (((uint32_t)kn * kHeadK * 2) >> 4);
#pragma unroll
            for (uint32_t s = 0; s < kHeadK / 16; ++s) {
              if (ESNMF_HEAD_SKIP & 4) break;
              if (wide) {
                tc::mma_f16(d, dah + 16 * s, dzh + 16 * s, idesc_w, (q | s) != 0);
              } else {
                tc::mma_f16(d, dah + 16 * s, dzh + 16 * s, idesc, (q | s) != 0);
                tc::mma_f16(d, dah + 16 * s, dzl + 16 * s, idesc, 1);
              }
              tc::mma_f16(d, dal + 16 * s, dzh + 16 * s, idesc, 1);
            }
          } else {  // (Y_tail W) chunk: K = w (its tiles are w wide)
            const uint32_t w = (uint32_t)min(kHeadK, kn - kHeadK * (q - nchunks));
            const uint32_t al = ah + (uint32_t)kHeadM * w * 2u, zh = ah + kHeadABytes, zl = zh + (uint32_t)kn * w * 2u;
            const uint32_t sbo = (w / 8) * 128;  // K-major, no swizzle: 8-row core-matrix groups
            for (uint32_t s = 0; s < w / 16; ++s) {
              if (ESNMF_HEAD_SKIP & 4) break;
              const uint32_t o = s * 256;
              const uint64_t dah = tc::make_sdesc(ah + o, 128, sbo), dal = tc::make_sdesc(al + o, 128, sbo);
              const uint64_t dzh = tc::make_sdesc(zh + o, 128, sbo), dzl = tc::make_sdesc(zl + o, 128, sbo);
              if (wide) {
                tc::mma_f16(d, dah, dzh, idesc_w, (q | s) != 0);
              } else {
                tc::mma_f16(d, dah, dzh, idesc, (q | s) != 0);
                tc::mma_f16(d, dah, dzl, idesc, 1);
              }
              tc::mma_f16(d, dal, dzh, idesc, 1);
            }
          }
          tc::mma_commit(&empty_bar[stage]);  // frees the stage when these MMAs finish
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc::mma_commit(&tfull[acc]);          // accumulator ready for the epilogue
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else {  // ---- epilogue (warps 6-13): TMEM -> registers -> X += ----
    const int lg = warp & 3;  // TMEM lanes 32*lg .. 32*lg+31
    const int half = (warp - kHeadEpiWarp) >> 2;  // the two warps of a quadrant split the columns
    const int cmid = ((kn / 16 + 1) / 2) * 16;
    const int cbeg = half ? cmid : 0, cend = half ? kn : cmid;
    // fused selection pass 1 (kn <= 128: at most 4 chunks of 16 columns per warp):
    // per-thread positive counts, two 16-bit counters per register, reduced once
    // at the end; candidates (value bits >= the predicted threshold) are rare and
    // take a warp-aggregated slow path
    uint32_t cnt2[4][8];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int j = 0; j < 8; ++j) cnt2[q][j] = 0;
    int acc = 0;
    uint32_t aphase = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      HT_WAIT_SLOW(&tfull[acc], aphase);
      tc::fence_after();
      if (!(ESNMF_HEAD_SKIP & 8))
      head_epi_tile<FUSE>(tile * kHeadM + lg * 32 + lane, tmem + (uint32_t)(acc * acc_cols) + ((uint32_t)(lg * 32) << 16),
                          wide ? (uint32_t)kn : 0u, cbeg, cend, nchunks + nyc == 0, xstore != 0, k, s_cs, rows, X, ldx, Xt, kpad, fz, s_pred, cnt2);
      tc::fence_before();
      head_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
    if (FUSE) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c0 = cbeg + 16 * q;
        if (c0 >= cend) break;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int n = warp_sum((int)((cnt2[q][j >> 1] >> (16 * (j & 1))) & 0xFFFFu));
          if (lane == 0 && n) atomicAdd(&s_npos[c0 + j], n);
        }
      }
    }
  }
#if ESNMF_HEAD_EXP == 3
  if ((blockIdx.x == 0 || blockIdx.x == 77) && lane == 0 && (warp == 0 || warp == kHeadMmaWarp || warp == kHeadLoadWarp || warp == kHeadEpiWarp))
    printf("HT cta %d warp %d wait %lld total %lld\n", blockIdx.x, warp, ht_wait, clock64() - ht_t0);
#endif
  (void)ht_wait;
  (void)ht_t0;
  tc::fence_before();
  __syncthreads();
  if (warp == kHeadMmaWarp) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, 2 * acc_cols);
  }
  if (FUSE)
    for (int c = threadIdx.x; c < k; c += blockDim.x)
      if (s_npos[c]) atomicAdd(&fz.npos[c], s_npos[c]);
}

}  // namespace esk
