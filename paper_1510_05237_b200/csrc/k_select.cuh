// k_select.cuh -- projection + per-column enforced sparsity.
//
// For every column c of the LS buffer X (column-major, rows of this shard):
//   keep {j : X[c][j] > 0}                         ("negative entries to zero")
//   if more than t: keep the t largest             (per column P:304)
//   ties at the t-th value -> lower row first, so exactly min(t, #positive) survive (C4).
// Equivalently: keep the positives whose 64-bit key (value desc, row asc) is <=
// the t-th smallest key K*_c.  K*_c is found by a radix select:
//   1. k_sel_hist      histogram of the top 12 value bits (bits 30..19) per column;
//   2. k_sel_threshold bucket D holding the t-th largest, r = t - #(buckets > D);
//   3. k_sel_collect   count entries above D per chunk, gather bucket-D keys;
//   4. k_sel_refine    K*_c = r-th smallest bucket-D key (bitonic sort in shared
//                      memory; exact multi-pass radix fallback if the bucket is large);
//   5. k_sel_scan_cols / k_sel_colptr: per-chunk output offsets;
//   6. k_sel_write     ordered (row-ascending) compaction into column-major COO.
// Integer counts only; no float atomics; output independent of scheduling.
#pragma once
#include "common.cuh"

namespace esk {

// (pred != nullptr) also appends every positive with value bits >= pred[c] to a
// per-column candidate list (row-keyed, capacity cap): pred[c] is the previous
// select's t-th value lowered by ~10 %, so in steady state the list holds the
// column's top t and the second pass over X is skipped (k_sel_pred_final).
__global__ void __launch_bounds__(256) k_sel_hist(const float* __restrict__ X, int64_t ldx, int64_t rows,
                                                  uint32_t* __restrict__ hist, const uint32_t* __restrict__ pred = nullptr,
                                                  int64_t row0 = 0, uint64_t* __restrict__ pcand = nullptr,
                                                  int32_t* __restrict__ pfill = nullptr, int pcap = 0,
                                                  const int32_t* __restrict__ skip = nullptr) {
  __shared__ uint32_t h[kNumBins];
  const int c = blockIdx.y;
  if (skip && skip[c]) return;  // column already selected (fused path)
  const uint32_t pb = pred ? pred[c] : 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int b = threadIdx.x; b < kNumBins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const float* col = X + (int64_t)c * ldx;
  // chunks blockIdx.x, + gridDim.x, ... (a full grid takes one chunk per block)
  for (int64_t r0 = (int64_t)blockIdx.x * kSelChunk; r0 < rows; r0 += (int64_t)gridDim.x * kSelChunk) {
  const int64_t r1 = min(rows, r0 + kSelChunk);
  for (int64_t base = r0; base < r1; base += 4 * blockDim.x) {  // uniform trip count (ballots below)
    const int64_t j = base + 4 * threadIdx.x;
    float x[4];
    if (j + 3 < r1) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(col + j));
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = j + u < r1 ? col[j + u] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (x[u] > 0.f) atomicAdd(&h[sel_digit(x[u])], 1u);
    // predicted candidates (value bits >= pb: a few per column in a million) --
    // one vote per four entries, the per-entry votes only when one lane has a hit
    // (positive floats order like their bit patterns; pb = 0xFFFFFFFF: no prediction)
    const float xm = fmaxf(fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3])), 0.f);
    if (pred && __any_sync(kFull, xm > 0.f && f2u(xm) >= pb)) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool cd = x[u] > 0.f && f2u(x[u]) >= pb;
        const unsigned m = __ballot_sync(kFull, cd);
        if (m) {
          int b0 = 0;
          if (lane == 0) b0 = atomicAdd(&pfill[c], __popc(m));
          b0 = __shfl_sync(kFull, b0, 0);
          const int slot = b0 + __popc(m & lt);
          if (cd && slot < pcap) pcand[(int64_t)c * pcap + slot] = sel_key(x[u], (uint32_t)(row0 + j + u));
        }
      }
    }
  }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kNumBins; b += blockDim.x)
    if (h[b]) atomicAdd(&hist[(int64_t)c * kNumBins + b], h[b]);
}

// one block (1024 threads) per column; thread q owns bins [4095-4q-3, 4095-4q]
__global__ void __launch_bounds__(1024) k_sel_threshold(const uint32_t* __restrict__ hist, int64_t t,
                                                        ColSel* __restrict__ sel) {
  __shared__ int64_t sm[33];
  const int c = blockIdx.x;
  const uint32_t* hc = hist + (int64_t)c * kNumBins;
  int64_t cnt[4];
  int64_t mine = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    cnt[u] = hc[kNumBins - 1 - (4 * threadIdx.x + u)];
    mine += cnt[u];
  }
  int64_t total;
  const int64_t before = block_exscan(mine, sm, &total);  // # in higher bins
  if (threadIdx.x == 0) {
    ColSel s;
    s.pad_ = 0;
    s.npos = total;
    s.ncand = 0;
    s.r = 0;
    if (t < 0 || total <= t) { s.digit = -1; s.above = total; }
    else if (t == 0) { s.digit = kNumBins; s.above = 0; }
    else { s.digit = -2; s.above = 0; }   // filled by the owning thread below
    sel[c] = s;
  }
  __syncthreads();
  if (t > 0 && total > t) {
    int64_t acc = before;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (acc < t && acc + cnt[u] >= t) {
        ColSel s = sel[c];
        s.digit = kNumBins - 1 - (4 * threadIdx.x + u);
        s.above = acc;
        s.r = t - acc;
        s.ncand = cnt[u];
        sel[c] = s;
      }
      acc += cnt[u];
    }
  }
}

__global__ void __launch_bounds__(256) k_sel_collect(const float* __restrict__ X, int64_t ldx, int64_t rows,
                                                     int64_t row0, const ColSel* __restrict__ sel,
                                                     uint64_t* __restrict__ cand, int32_t* __restrict__ cand_fill,
                                                     int64_t* __restrict__ chunk_cnt, int64_t nseg, int ccap) {
  // counts of strictly-above entries per kSelSeg-row segment: with 256 threads x
  // float4 one loop iteration covers exactly one segment (1024 rows)
  __shared__ int32_t sm[8][kSelSegs];
  const int c = blockIdx.y;
  const ColSel s = sel[c];
  const int64_t r0 = (int64_t)blockIdx.x * kSelChunk;
  const int64_t r1 = min(rows, r0 + kSelChunk);
  const float* col = X + (int64_t)c * ldx;
  int32_t cnt[kSelSegs];
#pragma unroll
  for (int q = 0; q < kSelSegs; ++q) cnt[q] = 0;
#pragma unroll
  for (int q = 0; q < kSelSegs; ++q) {
    const int64_t j = r0 + (int64_t)q * kSelSeg + 4 * threadIdx.x;
    if (j >= r1) continue;
    int32_t above = 0;
    float x[4];
    if (j + 3 < r1) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(col + j));
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = j + u < r1 ? col[j + u] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int dg = x[u] > 0.f ? sel_digit(x[u]) : -1;
      above += dg > s.digit;
      // bucket-D candidates: one atomic per warp (a flat whole-factor column can
      // put millions of entries into the bucket)
      const bool cd = x[u] > 0.f && dg == s.digit;
      const unsigned m = __ballot_sync(__activemask(), cd);
      if (cd) {
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(m) - 1;
        int b0 = 0;
        if (lane == leader) b0 = atomicAdd(&cand_fill[c], __popc(m));
        b0 = __shfl_sync(m, b0, leader);
        const int slot = b0 + __popc(m & ((1u << lane) - 1u));
        if (slot < ccap) cand[(int64_t)c * ccap + slot] = sel_key(x[u], (uint32_t)(row0 + j + u));
      }
    }
    cnt[q] = above;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < kSelSegs; ++q) {
    const int32_t w = warp_sum(cnt[q]);
    if (lane == 0) sm[warp][q] = w;
  }
  __syncthreads();
  if (threadIdx.x < kSelSegs) {
    int64_t tot = 0;
    for (int w = 0; w < 8; ++w) tot += sm[w][threadIdx.x];
    const int64_t seg = (int64_t)blockIdx.x * kSelSegs + threadIdx.x;
    if (seg < nseg) chunk_cnt[(int64_t)c * nseg + seg] = tot;
  }
}

// bitonic sort of n (power of two) keys in shared memory, ascending
// one block-wide compare-exchange stage of the bitonic network (stride >= 128)
__device__ __forceinline__ void bitonic_stage_smem(uint64_t* a, int n, int size, int stride) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int jx = i ^ stride;
    if (jx > i) {
      bool up = (i & size) == 0;
      uint64_t x = a[i], y = a[jx];
      if ((x > y) == up) { a[i] = y; a[jx] = x; }
    }
  }
}

// the stages of strides < 128 on a 128-element chunk held 4 per lane (lane l:
// elements 4l .. 4l+3 of the chunk at global offset b), warp-synchronous
__device__ __forceinline__ void bitonic_warp_stages(uint64_t (&v)[4], int b, int size, int stride_hi) {
  const int lane = threadIdx.x & 31;
  for (int stride = stride_hi; stride > 0; stride >>= 1) {
    if (stride >= 4) {
      const int ld = stride >> 2;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t pv = __shfl_xor_sync(kFull, v[j], ld);
        const int i = b + 4 * lane + j;
        const bool up = (i & size) == 0, lower = (i & stride) == 0;
        const uint64_t mn = v[j] < pv ? v[j] : pv, mx = v[j] < pv ? pv : v[j];
        v[j] = (up == lower) ? mn : mx;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j & stride) continue;
        const int jp = j | stride;
        const int i = b + 4 * lane + j;
        const bool up = (i & size) == 0;
        if ((v[j] > v[jp]) == up) { const uint64_t t = v[j]; v[j] = v[jp]; v[jp] = t; }
      }
    }
  }
}

// Ascending bitonic sort of n (a power of two) keys in shared memory by the whole
// block (blockDim a multiple of 32).  From n = 128 on, every run of stages with
// strides < 128 is done warp-synchronously on 128-element chunks in registers
// (shuffles), so only the strides >= 128 cost a block barrier: 15 of the 78 stages
// at n = 4,096.
__device__ void bitonic_sort_smem(uint64_t* a, int n) {
  if (n < 128) {
    for (int size = 2; size <= n; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        bitonic_stage_smem(a, n, size, stride);
        __syncthreads();
      }
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int b = warp * 128; b < n; b += nw * 128) {  // sizes 2 .. 128 inside each chunk
    uint64_t v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = a[b + 4 * lane + j];
    for (int size = 2; size <= 128; size <<= 1) bitonic_warp_stages(v, b, size, size >> 1);
#pragma unroll
    for (int j = 0; j < 4; ++j) a[b + 4 * lane + j] = v[j];
  }
  __syncthreads();
  for (int size = 256; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride >= 128; stride >>= 1) {
      bitonic_stage_smem(a, n, size, stride);
      __syncthreads();
    }
    for (int b = warp * 128; b < n; b += nw * 128) {
      uint64_t v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = a[b + 4 * lane + j];
      bitonic_warp_stages(v, b, size, 64);
#pragma unroll
      for (int j = 0; j < 4; ++j) a[b + 4 * lane + j] = v[j];
    }
    __syncthreads();
  }
}

// K*_c and the per-chunk counts of the selected bucket-D entries.
__global__ void __launch_bounds__(1024) k_sel_refine(const float* __restrict__ X, int64_t ldx, int64_t rows,
                                                     int64_t row0, const ColSel* __restrict__ sel,
                                                     const uint64_t* __restrict__ cand,
                                                     const int32_t* __restrict__ cand_fill,
                                                     int64_t* __restrict__ chunk_cnt, int64_t nchunks,
                                                     uint64_t* __restrict__ kthr, int ccap) {
  __shared__ uint64_t keys[kSelCap];           // sort buffer
  const int c = blockIdx.x;
  const ColSel s = sel[c];
  // kthr[c] = (tb << 32) | tr: keep x > 0 iff bits(x) > tb or (bits(x) == tb and row <= tr)
  if (s.r == 0) {
    if (threadIdx.x == 0) kthr[c] = s.digit < 0 ? 0x00000000FFFFFFFFULL : 0xFFFFFFFF00000000ULL;
    return;
  }
  const int nc = cand_fill[c];
  uint64_t kstar;
  if (nc <= kSelCap) {
    int np = 1;
    while (np < nc) np <<= 1;
    for (int i = threadIdx.x; i < np; i += blockDim.x) keys[i] = i < nc ? cand[(int64_t)c * ccap + i] : ~0ULL;
    __syncthreads();
    bitonic_sort_smem(keys, np);
    kstar = keys[s.r - 1];
    for (int i = threadIdx.x; i < s.r; i += blockDim.x) {
      const int64_t lr = (int64_t)(uint32_t)(keys[i] & 0xFFFFFFFFu) - row0;
      atomicAdd((unsigned long long*)&chunk_cnt[(int64_t)c * nchunks + lr / kSelSeg], 1ULL);
    }
  } else {
    return;  // bucket larger than kSelCap: exact multi-block radix select (k_sel_lvl_*)
  }
  if (threadIdx.x == 0)
    kthr[c] = ((uint64_t)(0x7FFFFFFFu - (uint32_t)(kstar >> 32)) << 32) | (kstar & 0xFFFFFFFFULL);
}

// ---- exact fallback for a threshold bucket larger than kSelCap ----------------
// Radix select over the column restricted to bucket D, every level a grid-wide
// pass (a whole-factor selection is one column of k x rows entries: one block
// would take ~100 ms).  Key bits below the bucket: value bits 18..0 (stored
// inverted), then the row; levels (shift, width) = (39,12) (32,7) (20,12) (8,12)
// (0,8).  A level whose chosen bin is taken whole ends the search (lower bits
// set to ones), so without exact value ties two levels suffice.
struct SelLvl {
  uint64_t prefix, mask;
  int64_t r;
  int32_t active, done;
  int32_t incand, pad_;  // 1: the whole bucket is in the candidate list (levels over it, not over X)
};

__global__ void k_sel_lvl_init(const ColSel* __restrict__ sel, const int32_t* __restrict__ cand_fill, int k,
                               SelLvl* __restrict__ lvl, int ccap) {
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    const ColSel s = sel[c];
    SelLvl L;
    L.active = s.r > 0 && cand_fill[c] > kSelCap;
    L.incand = L.active && cand_fill[c] <= ccap;  // (ccap > kSelCap: the list holds the whole bucket)
    L.pad_ = 0;
    L.done = !L.active;
    L.prefix = L.active ? ((uint64_t)(0x7FFFFFFFu - ((uint32_t)s.digit << kSelShift)) >> kSelShift) << 51 : 0;
    L.mask = 0xFFFULL << 51;
    L.r = s.r;
    lvl[c] = L;
  }
}

__global__ void __launch_bounds__(256) k_sel_lvl_hist(const float* __restrict__ X, int64_t ldx, int64_t rows,
                                                      int64_t row0, const ColSel* __restrict__ sel,
                                                      const SelLvl* __restrict__ lvl, int sh, int wd,
                                                      uint32_t* __restrict__ ghist) {
  __shared__ uint32_t h[kNumBins];
  const int c = blockIdx.y;
  const SelLvl L = lvl[c];
  if (L.done || L.incand) return;
  const int digit = sel[c].digit;
  const int nb = 1 << wd;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * kSelChunk;
  const int64_t r1 = min(rows, r0 + kSelChunk);
  const float* col = X + (int64_t)c * ldx;
  for (int64_t j = r0 + threadIdx.x; j < r1; j += blockDim.x) {
    const float x = col[j];
    if (x > 0.f && sel_digit(x) == digit) {
      const uint64_t key = sel_key(x, (uint32_t)(row0 + j));
      if ((key & L.mask) == L.prefix) atomicAdd(&h[(key >> sh) & (nb - 1)], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (h[b]) atomicAdd(&ghist[(int64_t)c * kNumBins + b], h[b]);
}

// one block of 256 per column: bin of the r-th key, narrow the prefix; clears the histogram
__global__ void __launch_bounds__(256) k_sel_lvl_pick(uint32_t* __restrict__ ghist, int sh, int wd, bool last,
                                                      SelLvl* __restrict__ lvl) {
  __shared__ int64_t sm[33];
  __shared__ int64_t res[2];
  const int c = blockIdx.x;
  SelLvl L = lvl[c];
  if (L.done) return;
  uint32_t* hc = ghist + (int64_t)c * kNumBins;
  const int nb = 1 << wd, per = (nb + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  int64_t mine = 0;
  for (int b = b0; b < min(nb, b0 + per); ++b) mine += hc[b];
  int64_t tot;
  const int64_t before = block_exscan(mine, sm, &tot);
  if (before < L.r && before + mine >= L.r) {  // exactly one thread
    int64_t acc = before;
    int b = b0;
    for (; b < b0 + per - 1; ++b) {
      if (acc + hc[b] >= L.r) break;
      acc += hc[b];
    }
    res[0] = b;
    res[1] = L.r - acc;
    res[1] |= (int64_t)(res[1] == (int64_t)hc[b]) << 62;  // the whole bin is taken
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x) hc[b] = 0;
  if (threadIdx.x == 0) {
    const bool whole = (res[1] >> 62) & 1;
    L.r = res[1] & ((1LL << 62) - 1);
    L.prefix |= (uint64_t)res[0] << sh;
    L.mask |= (uint64_t)(nb - 1) << sh;
    if (whole || last) {
      if (whole) L.prefix |= (1ULL << sh) - 1;  // every key of the bin is <= K*
      L.done = 1;
    }
    lvl[c] = L;
  }
}

// per-segment counts of the kept bucket-D keys (key <= K*), and kthr of the column
__global__ void __launch_bounds__(256) k_sel_lvl_count(const float* __restrict__ X, int64_t ldx, int64_t rows,
                                                       int64_t row0, const ColSel* __restrict__ sel,
                                                       const SelLvl* __restrict__ lvl,
                                                       int64_t* __restrict__ chunk_cnt, int64_t nseg,
                                                       uint64_t* __restrict__ kthr) {
  __shared__ int32_t sm[8][kSelSegs];
  const int c = blockIdx.y;
  const SelLvl L = lvl[c];
  if (!L.active || L.incand) return;
  const uint64_t kstar = L.prefix;
  if (blockIdx.x == 0 && threadIdx.x == 0)
    kthr[c] = ((uint64_t)(0x7FFFFFFFu - (uint32_t)(kstar >> 32)) << 32) | (kstar & 0xFFFFFFFFULL);
  const int digit = sel[c].digit;
  const int64_t r0 = (int64_t)blockIdx.x * kSelChunk;
  const int64_t r1 = min(rows, r0 + kSelChunk);
  const float* col = X + (int64_t)c * ldx;
  int32_t cnt[kSelSegs];
#pragma unroll
  for (int q = 0; q < kSelSegs; ++q) {  // rows r0 + 1024 q + 4 t .. + 3: segment q
    const int64_t j = r0 + (int64_t)q * kSelSeg + 4 * threadIdx.x;
    float x[4];
    if (j + 3 < r1) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(col + j));
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = j + u < r1 ? col[j + u] : 0.f;
    }
    cnt[q] = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      cnt[q] += x[u] > 0.f && sel_digit(x[u]) == digit && sel_key(x[u], (uint32_t)(row0 + j + u)) <= kstar;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < kSelSegs; ++q) {
    const int32_t w = warp_sum(cnt[q]);
    if (lane == 0) sm[warp][q] = w;
  }
  __syncthreads();
  if (threadIdx.x < kSelSegs) {
    int64_t tot = 0;
    for (int w = 0; w < 8; ++w) tot += sm[w][threadIdx.x];
    const int64_t seg = (int64_t)blockIdx.x * kSelSegs + threadIdx.x;
    if (tot && seg < nseg) atomicAdd((unsigned long long*)&chunk_cnt[(int64_t)c * nseg + seg], (unsigned long long)tot);
  }
}

// the same levels over a column's candidate list (every bucket-D key of the
// column, when it fit the list: incand), 8 keys per thread
__global__ void __launch_bounds__(256) k_sel_lvl_hist_cand(const uint64_t* __restrict__ cand,
                                                           const int32_t* __restrict__ cand_fill, int ccap,
                                                           const SelLvl* __restrict__ lvl, int sh, int wd,
                                                           uint32_t* __restrict__ ghist) {
  __shared__ uint32_t h[kNumBins];
  const int c = blockIdx.y;
  const SelLvl L = lvl[c];
  if (L.done || !L.incand) return;
  const int nc = cand_fill[c];
  const int64_t b0 = (int64_t)blockIdx.x * 2048;
  if (b0 >= nc) return;
  const int nb = 1 << wd;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const uint64_t* cc = cand + (int64_t)c * ccap;
  for (int64_t i = b0 + threadIdx.x; i < min((int64_t)nc, b0 + 2048); i += blockDim.x) {
    const uint64_t key = cc[i];
    if ((key & L.mask) == L.prefix) atomicAdd(&h[(key >> sh) & (nb - 1)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (h[b]) atomicAdd(&ghist[(int64_t)c * kNumBins + b], h[b]);
}

// per-segment counts of the kept candidates (key <= K*) and kthr, incand columns
__global__ void __launch_bounds__(256) k_sel_cand_count(const uint64_t* __restrict__ cand,
                                                        const int32_t* __restrict__ cand_fill, int ccap,
                                                        const SelLvl* __restrict__ lvl, int64_t row0,
                                                        int64_t* __restrict__ chunk_cnt, int64_t nseg,
                                                        uint64_t* __restrict__ kthr) {
  const int c = blockIdx.y;
  const SelLvl L = lvl[c];
  if (!L.incand) return;
  const uint64_t kstar = L.prefix;
  if (blockIdx.x == 0 && threadIdx.x == 0)
    kthr[c] = ((uint64_t)(0x7FFFFFFFu - (uint32_t)(kstar >> 32)) << 32) | (kstar & 0xFFFFFFFFULL);
  const int nc = cand_fill[c];
  const uint64_t* cc = cand + (int64_t)c * ccap;
  const int64_t b0 = (int64_t)blockIdx.x * 2048;
  for (int64_t i = b0 + threadIdx.x; i < min((int64_t)nc, b0 + 2048); i += blockDim.x) {
    const uint64_t key = cc[i];
    if (key <= kstar) {
      const int64_t lr = (int64_t)(uint32_t)(key & 0xFFFFFFFFu) - row0;
      atomicAdd((unsigned long long*)&chunk_cnt[(int64_t)c * nseg + lr / kSelSeg], 1ULL);
    }
  }
}

// per column: exclusive scan of the chunk counts (in place), column total -> coltot[c]
__global__ void __launch_bounds__(1024) k_sel_scan_cols(int64_t* __restrict__ chunk_cnt, int64_t nchunks,
                                                        int64_t* __restrict__ coltot) {
  __shared__ int64_t sm[33];
  const int c = blockIdx.x;
  int64_t* a = chunk_cnt + (int64_t)c * nchunks;
  int64_t carry = 0;
  for (int64_t base = 0; base < nchunks; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < nchunks ? a[i] : 0;
    int64_t tot;
    const int64_t ex = block_exscan(v, sm, &tot);
    if (i < nchunks) a[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) coltot[c] = carry;
}

// colptr[0..k] = exclusive scan of coltot (k <= 256: one block of 256)
__global__ void k_sel_colptr(const int64_t* __restrict__ coltot, int k, int64_t* __restrict__ colptr) {
  __shared__ int64_t sm[33];
  const int64_t v = threadIdx.x < k ? coltot[threadIdx.x] : 0;
  int64_t tot;
  const int64_t ex = block_exscan(v, sm, &tot);
  if (threadIdx.x < k) colptr[threadIdx.x] = ex;
  if (threadIdx.x == 0) colptr[k] = tot;
}

__global__ void __launch_bounds__(256) k_sel_write(const float* __restrict__ X, int64_t ldx, int64_t rows,
                                                   int64_t row0, const ColSel* __restrict__ sel,
                                                   const uint64_t* __restrict__ kthr,
                                                   const int64_t* __restrict__ colptr,
                                                   const int64_t* __restrict__ chunk_off, int64_t nchunks,
                                                   int32_t* __restrict__ out_row, float* __restrict__ out_val) {
  // each warp owns one kSelSeg-row segment whose output offset is known from
  // the per-segment counts (k_sel_collect + k_sel_refine, scanned by
  // k_sel_scan_cols): one read of the segment as float4 (lane l holds rows
  // 4l..4l+3 of a 128-row step) and an in-order compaction with a warp scan
  (void)sel;
  const int c = blockIdx.y;
  const uint64_t ks = kthr[c];
  const uint32_t tb = (uint32_t)(ks >> 32), tr = (uint32_t)ks;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t seg = (int64_t)blockIdx.x * kSelSegs + warp;
  const int64_t r0 = seg * kSelSeg;
  const int64_t r1 = min(rows, r0 + kSelSeg);
  if (r0 >= rows) return;
  const float* col = X + (int64_t)c * ldx;
  auto load4 = [&](int64_t j, float (&x)[4], unsigned& mask) {
    mask = 0;
    if (j + 3 < r1) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(col + j));
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = j + u < r1 ? col[j + u] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t b = __float_as_uint(x[u]);
      const uint32_t gr = (uint32_t)(row0 + j + u);
      const bool kp = x[u] > 0.f && (b > tb || (b == tb && gr <= tr));
      mask |= (unsigned)kp << u;
    }
  };
  int64_t off = colptr[c] + chunk_off[(int64_t)c * nchunks + seg];
  // all eight 128-row steps of the segment loaded before any use
  float xs[kSelSeg / 128][4];
  unsigned mks[kSelSeg / 128];
#pragma unroll
  for (int i = 0; i < kSelSeg / 128; ++i) load4(r0 + 128 * i + 4 * lane, xs[i], mks[i]);
#pragma unroll
  for (int i = 0; i < kSelSeg / 128; ++i) {
    const int64_t base = r0 + 128 * i;
    const float* x = xs[i];
    const unsigned mk = mks[i];
    const int mine = __popc(mk);
    int inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    int64_t o = off + inc - mine;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if ((mk >> u) & 1u) {
        out_row[o] = (int32_t)(row0 + base + 4 * lane + u);
        out_val[o] = x[u];
        ++o;
      }
    off += __shfl_sync(kFull, inc, 31);
  }
}


// ---------------------------------------------------------------------------
// Two-pass variant for t <= kSelFastT (every BASELINE config but Box and the
// t = 10^4 / unlimited sweep points): after k_sel_hist + k_sel_threshold,
//   k_sel_collect2  one pass over X appends every positive of bucket > D to a
//                   per-column "above" list (row-keyed, < t of them) and every
//                   positive of bucket D to a "bucket" list (value-keyed), with
//                   warp-aggregated slot reservations;
//   k_sel_final     one block per column: sort the bucket keys, keep the r
//                   smallest (value desc, row asc), merge with the above list,
//                   sort the kept entries by row and write the column.
// The lists are filled in scheduling order but everything kept is sorted by a
// total order, so the output is deterministic.  A bucket larger than
// kSelCap falls back to an exact radix select over the column.
constexpr int64_t kSelFastT = 8192;

ESNMF_DEV uint64_t row_key(uint32_t row, float x) { return ((uint64_t)row << 32) | (uint64_t)f2u(x); }

// prediction for the next select: value bits 10 % below the kept minimum
// (0 = every positive is a candidate)
ESNMF_DEV uint32_t pred_of(uint32_t minbits) {
  if (minbits == 0xFFFFFFFFu || minbits == 0u) return 0u;
  return f2u(__uint_as_float(minbits) * 0.9f);
}

__global__ void __launch_bounds__(256) k_sel_collect2(const float* __restrict__ X, int64_t ldx, int64_t rows,
                                                      int64_t row0, const ColSel* __restrict__ sel, int64_t t,
                                                      uint64_t* __restrict__ above, int32_t* __restrict__ above_fill,
                                                      uint64_t* __restrict__ bucket,
                                                      int32_t* __restrict__ bucket_fill,
                                                      const int32_t* __restrict__ done = nullptr) {
  const int c = blockIdx.y;
  const ColSel s = sel[c];
  if (s.digit >= kNumBins) return;  // t == 0: nothing kept
  if (done && done[c]) return;      // selected from the predicted candidates
  const float* col = X + (int64_t)c * ldx;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  uint64_t* ab = above + (int64_t)c * t;
  uint64_t* bk = bucket + (int64_t)c * kSelCap;
  // chunks blockIdx.x, + gridDim.x, ...; every thread runs the same trip count (the
  // ballots need the full warp)
  for (int64_t r0 = (int64_t)blockIdx.x * kSelChunk; r0 < rows; r0 += (int64_t)gridDim.x * kSelChunk) {
  const int64_t r1 = min(rows, r0 + kSelChunk);
  for (int64_t base = r0; base < r1; base += 4 * blockDim.x) {
    const int64_t j = base + 4 * threadIdx.x;
    float x[4];
    if (j + 3 < r1) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(col + j));
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = j + u < r1 ? col[j + u] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool pos = x[u] > 0.f;
      const int dg = pos ? sel_digit(x[u]) : -1;
      const bool up = pos && dg > s.digit;
      const bool eq = pos && dg == s.digit;
      if (!__any_sync(kFull, up || eq)) continue;  // most entries sit below the threshold bucket
      const unsigned mu = __ballot_sync(kFull, up), me = __ballot_sync(kFull, eq);
      int bu = 0, be = 0;
      if (lane == 0) {
        if (mu) bu = atomicAdd(&above_fill[c], __popc(mu));
        if (me) be = atomicAdd(&bucket_fill[c], __popc(me));
      }
      bu = __shfl_sync(kFull, bu, 0);
      be = __shfl_sync(kFull, be, 0);
      const uint32_t gr = (uint32_t)(row0 + j + u);
      if (up) ab[bu + __popc(mu & lt)] = row_key(gr, x[u]);
      if (eq) {
        const int slot = be + __popc(me & lt);
        if (slot < kSelCap) bk[slot] = sel_key(x[u], gr);
      }
    }
  }
  }
}

// positives of the clamped LS over all columns (the record's peak nnz)
__global__ void k_sel_npos_sum(const ColSel* __restrict__ sel, int kc, int64_t* __restrict__ out) {
  __shared__ int64_t sm[32];
  int64_t v = 0;
  for (int c = threadIdx.x; c < kc; c += blockDim.x) v += sel[c].npos;
  v = block_sum(v, sm);
  if (threadIdx.x == 0) *out = v;
}

// colptr of the kept entries: min(t, #positive) per column (reading C4/C5)
// (and, when peak != nullptr, the positives of all columns: the record's peak nnz)
__global__ void k_sel_colptr_kept(const ColSel* __restrict__ sel, int k, int64_t t, int64_t* __restrict__ colptr,
                                  int64_t* __restrict__ peak = nullptr) {
  __shared__ int64_t sm[33];
  int64_t v = 0, np = 0;
  if (threadIdx.x < k) {
    np = sel[threadIdx.x].npos;
    v = t < 0 ? np : min(np, t);
  }
  int64_t tot, ptot;
  const int64_t ex = block_exscan(v, sm, &tot);
  if (threadIdx.x < k) colptr[threadIdx.x] = ex;
  if (threadIdx.x == 0) colptr[k] = tot;
  if (peak) {
    __syncthreads();
    block_exscan(np, sm, &ptot);
    if (threadIdx.x == 0) *peak = ptot;
  }
}

constexpr size_t kSelFinalSmem = sizeof(uint64_t) * (kSelCap + kSelFastT);

__global__ void __launch_bounds__(1024) k_sel_final(const float* __restrict__ X, int64_t ldx, int64_t rows,
                                                    int64_t row0, const ColSel* __restrict__ sel, int64_t t,
                                                    const uint64_t* __restrict__ above,
                                                    const int32_t* __restrict__ above_fill,
                                                    const uint64_t* __restrict__ bucket,
                                                    const int32_t* __restrict__ bucket_fill,
                                                    const int64_t* __restrict__ colptr, int32_t* __restrict__ out_row,
                                                    float* __restrict__ out_val,
                                                    const int32_t* __restrict__ done = nullptr,
                                                    uint32_t* __restrict__ pred_next = nullptr) {
  extern __shared__ uint64_t fin_smem[];
  uint64_t* kb = fin_smem;                                // [kSelCap] bucket keys
  uint64_t* kept = fin_smem + kSelCap;                    // [kSelFastT] kept row keys
  uint32_t* h = reinterpret_cast<uint32_t*>(kb);          // fallback histogram (aliases kb)
  __shared__ int64_t sm[4];
  __shared__ int nk_s;
  const int c = blockIdx.x;
  const ColSel s = sel[c];
  if (s.digit >= kNumBins) {
    if (pred_next && threadIdx.x == 0) pred_next[c] = 0xFFFFFFFFu;  // t == 0: no candidates
    return;
  }
  if (done && done[c]) return;  // selected from the predicted candidates
  const int na = above_fill[c];  // == s.above (all positives when s.digit < 0)
  const int nb = bucket_fill[c];
  const int r = (int)s.r;
  for (int i = threadIdx.x; i < na; i += blockDim.x) kept[i] = above[(int64_t)c * t + i];
  if (threadIdx.x == 0) nk_s = na;
  __syncthreads();
  if (r > 0) {
    if (nb <= kSelCap) {
      int np = 1;
      while (np < nb) np <<= 1;
      for (int i = threadIdx.x; i < np; i += blockDim.x) kb[i] = i < nb ? bucket[(int64_t)c * kSelCap + i] : ~0ULL;
      __syncthreads();
      bitonic_sort_smem(kb, np);
      for (int i = threadIdx.x; i < r; i += blockDim.x) {
        const uint64_t key = kb[i];
        const uint32_t row = (uint32_t)key;
        const float x = __uint_as_float(0x7FFFFFFFu - (uint32_t)(key >> 32));
        kept[na + i] = row_key(row, x);
      }
    } else {
      // exact fallback: radix select of the r-th smallest key of bucket D over the column
      const float* col = X + (int64_t)c * ldx;
      const int shifts[5] = {39, 32, 20, 8, 0};
      const int widths[5] = {12, 7, 12, 12, 8};
      uint64_t prefix = ((uint64_t)(0x7FFFFFFFu - ((uint32_t)s.digit << kSelShift)) >> kSelShift) << 51;
      uint64_t fixed_mask = 0xFFFULL << 51;
      int64_t rr = r;
      for (int lv = 0; lv < 5; ++lv) {
        const int sh = shifts[lv], wd = widths[lv];
        for (int b = threadIdx.x; b < kNumBins; b += blockDim.x) h[b] = 0;
        __syncthreads();
        for (int64_t j = threadIdx.x; j < rows; j += blockDim.x) {
          const float x = col[j];
          if (x > 0.f && sel_digit(x) == s.digit) {
            const uint64_t key = sel_key(x, (uint32_t)(row0 + j));
            if ((key & fixed_mask) == prefix) atomicAdd(&h[(key >> sh) & ((1u << wd) - 1)], 1u);
          }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          int64_t acc = 0;
          int b = 0;
          for (; b < (1 << wd); ++b) {
            if (acc + h[b] >= rr) break;
            acc += h[b];
          }
          sm[0] = b;
          sm[1] = rr - acc;
        }
        __syncthreads();
        prefix |= (uint64_t)sm[0] << sh;
        rr = sm[1];
        fixed_mask |= (uint64_t)((1u << wd) - 1) << sh;
        __syncthreads();
      }
      const uint64_t kstar = prefix;
      for (int64_t j = threadIdx.x; j < rows; j += blockDim.x) {
        const float x = col[j];
        if (x > 0.f && sel_digit(x) == s.digit && sel_key(x, (uint32_t)(row0 + j)) <= kstar) {
          const int slot = atomicAdd(&nk_s, 1);
          kept[slot] = row_key((uint32_t)(row0 + j), x);
        }
      }
    }
  }
  __syncthreads();
  const int nk = na + r;
  int np = 1;
  while (np < nk) np <<= 1;
  for (int i = nk + threadIdx.x; i < np; i += blockDim.x) kept[i] = ~0ULL;
  __syncthreads();
  bitonic_sort_smem(kept, np);
  const int64_t o = colptr[c];
  uint32_t mn = 0xFFFFFFFFu;
  for (int i = threadIdx.x; i < nk; i += blockDim.x) {
    const uint64_t key = kept[i];
    out_row[o + i] = (int32_t)(key >> 32);
    out_val[o + i] = __uint_as_float((uint32_t)key);
    mn = min(mn, (uint32_t)key);
  }
  if (pred_next) {
    mn = __reduce_min_sync(kFull, mn);
    __shared__ uint32_t wmin[32];
    if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = mn;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t m = 0xFFFFFFFFu;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = min(m, wmin[w]);
      // keep-all columns (s.digit < 0): predict 0 (every positive is a candidate)
      pred_next[c] = s.digit < 0 ? 0u : pred_of(m);
    }
  }
}

// ---- predicted-threshold fast path ----------------------------------------

// one block per column: if the candidates of the histogram pass contain the
// column's top min(t, #pos) (#candidates >= that, no overflow), select from
// them and mark the column done; else leave it to k_sel_collect2/k_sel_final.
// Like k_sel_final: candidates above the threshold bucket D (from the full
// histogram) are all kept, only bucket D's candidates are sorted by key, and
// the kept entries are sorted by row for the canonical order.
constexpr int kPredSort = 8192;  // candidate capacity (keys staged in shared memory)

__global__ void __launch_bounds__(1024) k_sel_pred_final(const ColSel* __restrict__ sel, int64_t t,
                                                         const uint64_t* __restrict__ pcand,
                                                         const int32_t* __restrict__ pfill, int pcap,
                                                         const int64_t* __restrict__ colptr,
                                                         int32_t* __restrict__ out_row, float* __restrict__ out_val,
                                                         int32_t* __restrict__ done, uint32_t* __restrict__ pred_next) {
  extern __shared__ uint64_t ps[];  // [kSelFastT] kept row keys, then [kSelCap] bucket keys
  uint64_t* kept = ps;
  uint64_t* bk = ps + kSelFastT;
  __shared__ int nkept, nbk;
  __shared__ uint32_t wmin[32];
  const int c = blockIdx.x;
  const ColSel s = sel[c];
  const int64_t need = min(t, s.npos);
  const int nc = pfill[c];
  bool ok = s.digit < kNumBins && nc <= pcap && (int64_t)nc >= need && need > 0 && need <= kSelFastT;
  if (!ok) {
    if (threadIdx.x == 0) {
      done[c] = s.digit >= kNumBins || need == 0 ? 1 : 0;
      if (need == 0) pred_next[c] = s.digit >= kNumBins ? 0xFFFFFFFFu : 0u;
    }
    return;
  }
  if (threadIdx.x == 0) {
    nkept = 0;
    nbk = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    const uint64_t key = pcand[(int64_t)c * pcap + i];  // sel_key: (value desc, row asc)
    const uint32_t bits = 0x7FFFFFFFu - (uint32_t)(key >> 32);
    const int dg = (int)(bits >> kSelShift);
    if (dg > s.digit) {
      const int slot = atomicAdd(&nkept, 1);
      if (slot < kSelFastT) kept[slot] = row_key((uint32_t)key, __uint_as_float(bits));
    } else if (dg == s.digit) {
      const int slot = atomicAdd(&nbk, 1);
      if (slot < kSelCap) bk[slot] = key;
    }
  }
  __syncthreads();
  const int na = nkept, nb = nbk;
  const int r = (int)(need - na);  // from bucket D (s.digit < 0: every positive is "above")
  if (na > kSelFastT || nb > kSelCap || r < 0 || r > nb) {  // cannot happen when the candidates are complete
    if (threadIdx.x == 0) done[c] = 0;
    return;
  }
  if (r > 0) {
    int np = 1;
    while (np < nb) np <<= 1;
    for (int i = nb + threadIdx.x; i < np; i += blockDim.x) bk[i] = ~0ULL;
    __syncthreads();
    bitonic_sort_smem(bk, np);
    for (int i = threadIdx.x; i < r; i += blockDim.x) {
      const uint64_t key = bk[i];
      kept[na + i] = row_key((uint32_t)key, __uint_as_float(0x7FFFFFFFu - (uint32_t)(key >> 32)));
    }
  }
  __syncthreads();
  const int nk = (int)need;
  int np = 1;
  while (np < nk) np <<= 1;
  for (int i = nk + threadIdx.x; i < np; i += blockDim.x) kept[i] = ~0ULL;
  __syncthreads();
  bitonic_sort_smem(kept, np);
  const int64_t o = colptr[c];
  uint32_t mn = 0xFFFFFFFFu;
  for (int i = threadIdx.x; i < nk; i += blockDim.x) {
    const uint64_t key = kept[i];
    out_row[o + i] = (int32_t)(key >> 32);
    out_val[o + i] = __uint_as_float((uint32_t)key);
    mn = min(mn, (uint32_t)key);
  }
  mn = __reduce_min_sync(kFull, mn);
  if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t m = 0xFFFFFFFFu;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = min(m, wmin[w]);
    done[c] = 1;
    pred_next[c] = s.npos <= t ? 0u : pred_of(m);
  }
}

// ---- V side fused with the head kernel's epilogue (k_vhead_otf) -------------
// The epilogue counted the positives of every column (npos) and appended every
// positive with value bits >= pred[c] as a candidate, so the LS buffer is not
// read again in steady state.  colptr (min(t, npos)) and the peak count first:
__global__ void k_sel_npos_colptr(const int32_t* __restrict__ npos, int k, int64_t t, int64_t* __restrict__ colptr,
                                  int64_t* __restrict__ peak) {
  __shared__ int64_t sm[33];
  int64_t v = 0, np = 0;
  if (threadIdx.x < k) {
    np = npos[threadIdx.x];
    v = t < 0 ? np : min(np, t);
  }
  int64_t tot, ptot;
  const int64_t ex = block_exscan(v, sm, &tot);
  __syncthreads();
  block_exscan(np, sm, &ptot);
  if (threadIdx.x < k) colptr[threadIdx.x] = ex;
  if (threadIdx.x == 0) {
    colptr[k] = tot;
    if (peak) *peak = ptot;
  }
}

// ... then per column: if the candidates hold at least min(t, npos) entries (so
// they contain the column's top min(t, npos): every entry >= the predicted
// threshold is a candidate), sort them by (value desc, row asc), keep the first
// min(t, npos), write them in row order and mark the column done; else leave it
// to the histogram path (k_sel_hist/threshold/collect2/final with `done`).
constexpr size_t kPredSortSmem = sizeof(uint64_t) * (kPredSort + kSelFastT);

__global__ void __launch_bounds__(1024) k_sel_pred_sort(const int32_t* __restrict__ npos, int64_t t,
                                                        const uint64_t* __restrict__ pcand,
                                                        const int32_t* __restrict__ pfill, int pcap,
                                                        const int64_t* __restrict__ colptr,
                                                        int32_t* __restrict__ out_row, float* __restrict__ out_val,
                                                        int32_t* __restrict__ done, uint32_t* __restrict__ pred) {
  extern __shared__ uint64_t ps[];
  uint64_t* keys = ps;                // [kPredSort] candidate keys
  uint64_t* kept = ps + kPredSort;    // [kSelFastT] kept row keys
  __shared__ uint32_t wmin[32];
  const int c = blockIdx.x;
  const int64_t np_c = npos[c];
  const int64_t need = min(t, np_c);
  const int nc = pfill[c];
  if (need == 0) {
    if (threadIdx.x == 0) {
      done[c] = 1;
      pred[c] = t == 0 ? 0xFFFFFFFFu : 0u;
    }
    return;
  }
  const bool ok = nc <= pcap && nc <= kPredSort && (int64_t)nc >= need && need <= kSelFastT;
  if (!ok) {
    if (threadIdx.x == 0) done[c] = 0;
    return;
  }
  int np = 1;
  while (np < nc) np <<= 1;
  for (int i = threadIdx.x; i < np; i += blockDim.x) keys[i] = i < nc ? pcand[(int64_t)c * pcap + i] : ~0ULL;
  __syncthreads();
  bitonic_sort_smem(keys, np);
  const int nk = (int)need;
  for (int i = threadIdx.x; i < nk; i += blockDim.x) {
    const uint64_t key = keys[i];
    kept[i] = row_key((uint32_t)key, __uint_as_float(0x7FFFFFFFu - (uint32_t)(key >> 32)));
  }
  int nq = 1;
  while (nq < nk) nq <<= 1;
  for (int i = nk + threadIdx.x; i < nq; i += blockDim.x) kept[i] = ~0ULL;
  __syncthreads();
  bitonic_sort_smem(kept, nq);
  const int64_t o = colptr[c];
  uint32_t mn = 0xFFFFFFFFu;
  for (int i = threadIdx.x; i < nk; i += blockDim.x) {
    const uint64_t key = kept[i];
    out_row[o + i] = (int32_t)(key >> 32);
    out_val[o + i] = __uint_as_float((uint32_t)key);
    mn = min(mn, (uint32_t)key);
  }
  mn = __reduce_min_sync(kFull, mn);
  if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t m = 0xFFFFFFFFu;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = min(m, wmin[w]);
    done[c] = 1;
    pred[c] = np_c <= t ? 0u : pred_of(m);
  }
}

}  // namespace esk
