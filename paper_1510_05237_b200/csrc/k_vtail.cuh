// k_vtail.cuh -- V-side "tail" in the paper's order ("V = A^T U (U^T U)^{-1}";
// P:133): Y_tail = A^T[:, tail] U, then LS_tail = Y_tail W on the tensor cores
// inside the head kernel (k_vhead.cuh: two or four extra K-chunks per tile whose
// A operand is Y_tail and whose B operand is W).
//
// Why this order for the tail.  Past the most frequent terms, the rows of U are
// short (Large steady state: ~4-20 nonzeros per row for term ranks 1k-2k, ~1.5
// per active row beyond): the paper's order costs r_i = nnz(U row i) products
// per stored entry (i, j) of A^T -- 0.15 G products at Large -- where the
// reassociated A^T (U W) order gathers a k-wide Z row per active entry (28 M x
// 400 B = 11-14 GB of L2 traffic per launch, round 1's k_spmm_tail).
//
// Data (built at create time, k_vt_count / k_vt_fill): per 128-document tile,
// the tile's tail entries in JAGGED-DIAGONAL order -- documents ranked by tail
// length (descending), then layer q holds the q-th tail entry of every document
// with more than q -- each entry (row in tile << 24 | term, value).  Consecutive
// entries therefore belong to different documents, so the lanes of a warp add
// into different shared-memory rows.
//
// Accumulation is FIXED POINT (unsigned 32-bit; every product a_ij u_ic >= 0):
// U's values are stored pre-scaled by 2^s_c (k_ut_scale) with s_c chosen so that
// max_j rowsum_j(A) * max_i U_ic * 2^s_c <= 2^30 (a bound on every Y entry);
// each product is rounded once to an integer and integer addition is exact and
// order-free, so the result does not depend on the atomic order (bitwise
// deterministic) and the quantisation error is <= 2^-31 of the bound per product.
// The finished tile is written as Y' = Y_fix 2^-15 (<= 2^15) split into fp16
// hi + lo halves in the UMMA K-major layout (tc.cuh) -- the head kernel copies
// it into a stage like a dense A tile.
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc.cuh"

namespace esk {

constexpr int kVtM = 128;           // documents per tile (= the head kernel's MMA M)
constexpr int kVtThreads = 512;     // k_ytail block
constexpr int kVtTermBits = 24;     // term id bits of a packed tail entry (n < 2^24)
constexpr uint32_t kVtTermMask = (1u << kVtTermBits) - 1u;

// tail entries of each tile: sum over its documents of (row length - head entries)
__global__ void k_vt_count(const int64_t* __restrict__ ptr, const int32_t* __restrict__ nh, int64_t rows,
                           int64_t* __restrict__ tcnt) {
  __shared__ int64_t sm[33];
  const int64_t tile = blockIdx.x;
  const int64_t row = tile * kVtM + threadIdx.x;
  int64_t c = 0;
  if (threadIdx.x < kVtM && row < rows) c = ptr[row + 1] - ptr[row] - (nh ? nh[row] : 0);
  int64_t tot;
  block_exscan(c, sm, &tot);
  if (threadIdx.x == 0) tcnt[tile] = tot;
}

// the tile's tail entries in jagged-diagonal order (one block of kVtM threads per tile)
__global__ void __launch_bounds__(kVtM) k_vt_fill(const int64_t* __restrict__ ptr, const int32_t* __restrict__ nh,
                                                  const int2* __restrict__ ent, int64_t rows,
                                                  const int64_t* __restrict__ toff, int2* __restrict__ tent) {
  __shared__ int cnt[kVtM];
  const int64_t tile = blockIdx.x;
  const int r = threadIdx.x;
  const int64_t row = tile * kVtM + r;
  int64_t s = 0;
  int c = 0;
  if (row < rows) {
    s = ptr[row] + (nh ? nh[row] : 0);
    c = (int)(ptr[row + 1] - s);
  }
  cnt[r] = c;
  __syncthreads();
  int rank = 0;  // position among the tile's documents by (tail length desc, row asc)
  for (int q = 0; q < kVtM; ++q) rank += (cnt[q] > c) || (cnt[q] == c && q < r);
  int64_t layer = toff[tile];
  for (int q = 0;; ++q) {
    const int nq = __syncthreads_count(c > q);  // documents with more than q tail entries
    if (nq == 0) break;
    if (c > q) {
      const int2 en = ent[s + q];
      tent[layer + rank] = make_int2((int)(((uint32_t)r << kVtTermBits) | (uint32_t)en.x), en.y);
    }
    layer += nq;
  }
}

// row sums of A^T (one warp per document; fixed order) -> max over the shard, as
// the bits of a float rounded UP (a valid bound for the fixed-point scale)
__global__ void k_doc_rowsum_max(const int64_t* __restrict__ ptr, const int2* __restrict__ ent, int64_t rows,
                                 unsigned* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned mx = 0;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows; r += nw) {
    double s = 0;
    for (int64_t q = ptr[r] + lane; q < ptr[r + 1]; q += 32) s += (double)__int_as_float(ent[q].y);
    s = warp_sum(s);
    mx = max(mx, __float_as_uint(__double2float_ru(s)));
  }
  if (lane == 0 && mx) atomicMax(out, mx);
}

// ---- U row view for the paper-order tail (k_vrows_count / scan / here / k_vrows_finish) ----
// scatter U's (column, value) pairs into rows; per-column max over the TAIL rows
// (headslot < 0) as float bits: the bound of the fixed-point scale
__global__ void k_urows_scatter(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                                const float* __restrict__ val, const int32_t* __restrict__ rowmap,
                                const int32_t* __restrict__ headslot, int64_t* __restrict__ cursor,
                                int2* __restrict__ uent, uint32_t* __restrict__ umax) {
  const int c_ = blockIdx.y;
  const int64_t cb = colptr[c_], ce = colptr[c_ + 1];
  uint32_t mx = 0;
  for (int64_t e = cb + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ce; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = row[e];
    const int64_t p = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(&cursor[rowmap[i]]), 1ull);
    uent[p] = make_int2(c_, __float_as_int(val[e]));
    if (!headslot || headslot[i] < 0) mx = max(mx, __float_as_uint(val[e]));  // values > 0
  }
  mx = __reduce_max_sync(kFull, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(&umax[c_], mx);
}

// publish umap[row] = (first << 32) | count for every active row of U; the rows
// published are listed in ulist (for the next clear), their number in *ulist_n
__global__ void k_urows_finish(const int32_t* __restrict__ active, const int64_t* __restrict__ n_active,
                               const int64_t* __restrict__ rptr, uint64_t* __restrict__ umap,
                               int32_t* __restrict__ ulist, int64_t* __restrict__ ulist_n) {
  const int64_t na = *n_active;
  if (blockIdx.x == 0 && threadIdx.x == 0) *ulist_n = na;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < na; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = active[r];
    umap[i] = ((uint64_t)rptr[r] << 32) | (uint64_t)(rptr[r + 1] - rptr[r]);
    ulist[r] = i;
  }
}

__global__ void k_urows_clear(const int32_t* __restrict__ ulist, const int64_t* __restrict__ ulist_n,
                              uint64_t* __restrict__ umap) {
  const int64_t na = *ulist_n;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < na; r += (int64_t)gridDim.x * blockDim.x)
    umap[ulist[r]] = 0ull;
}

// max over ranks of the per-rank {amax bits, rowsum bits} (allgathered, 16 bytes per rank)
__global__ void k_rank_max2(const unsigned* __restrict__ gathered, int world, unsigned* __restrict__ amax,
                            unsigned* __restrict__ rowsum) {
  unsigned a = 0, b = 0;
  for (int p = 0; p < world; ++p) {
    a = max(a, gathered[4 * p]);
    b = max(b, gathered[4 * p + 1]);
  }
  *amax = a;
  *rowsum = b;
}

// fixed-point exponent of column c: 2^s_c * rowsum_max * umax_c <= 2^30
ESNMF_DEV int vt_shift(uint32_t umax_bits, uint32_t rowsum_bits) {
  const float b = __uint_as_float(umax_bits) * __uint_as_float(rowsum_bits);  // rounded: slack below
  if (!(b > 0.f)) return 0;
  int e;
  frexpf(b, &e);           // b = f 2^e, f in [0.5, 1): b < 2^e
  return 29 - e;           // b 2^s < 2^29 (a factor 2 of slack for the float product's rounding)
}

// scale every pair's value by 2^s_c (exact) and publish s_c
__global__ void k_ut_scale(const int64_t* __restrict__ n_ent, int2* __restrict__ uent, int k,
                           const uint32_t* __restrict__ umax, const unsigned* __restrict__ rowsum_bits,
                           int* __restrict__ shift) {
  const uint32_t rb = *rowsum_bits;
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < k; c += blockDim.x) shift[c] = vt_shift(umax[c], rb);
  const int64_t n = *n_ent;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int2 p = uent[e];
    p.y = __float_as_int(ldexpf(__int_as_float(p.y), vt_shift(umax[p.x], rb)));
    uent[e] = p;
  }
}

// ---- Y_tail per tile, written as fp16 hi/lo K-major chunks ----
// Chunk q of a tile covers Y columns [64 q, 64 q + w_q), w_q = min(64, kn - 64 q);
// it is stored as [hi: 128 x w_q fp16][lo: 128 x w_q fp16], K-major (tc.cuh),
// at ytile + tile * 128 * kn * 4 + 64 q * 128 * 4.
// ys: shared row stride in words (odd: lanes on different rows, same column,
// fall in different banks).
__global__ void __launch_bounds__(kVtThreads) k_ytail(const int64_t* __restrict__ toff, const int2* __restrict__ tent,
                                                      int64_t ntiles, const uint64_t* __restrict__ umap,
                                                      const int2* __restrict__ uent, int kn, int ys,
                                                      uint8_t* __restrict__ ytile) {
  extern __shared__ uint32_t Ysm[];
  const int T = blockDim.x;
  const int ng = kn / 8;  // 8-column groups per row
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int i = threadIdx.x; i < kVtM * ys; i += T) Ysm[i] = 0u;
    __syncthreads();
    const int64_t e0 = toff[tile], e1 = toff[tile + 1];
    // two entries per thread per round: their map lookups are in flight together
    for (int64_t e = e0 + threadIdx.x; e < e1; e += 2 * (int64_t)T) {
      const int64_t f = e + T;
      const int2 a0 = __ldcs(tent + e);
      const int2 a1 = f < e1 ? __ldcs(tent + f) : make_int2(0, 0);
      const uint64_t m0 = umap[(uint32_t)a0.x & kVtTermMask];
      const uint64_t m1 = f < e1 ? umap[(uint32_t)a1.x & kVtTermMask] : 0ull;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int2 a = u ? a1 : a0;
        const uint64_t mp = u ? m1 : m0;
        const int cnt = (int)(mp & 0xFFFFFFFFull);
        if (cnt == 0) continue;
        const int2* up = uent + (mp >> 32);
        uint32_t* yrow = Ysm + ((uint32_t)a.x >> kVtTermBits) * ys;
        const float av = __int_as_float(a.y);
        int j = 0;
        for (; j + 2 <= cnt; j += 2) {
          const int2 p0 = up[j], p1 = up[j + 1];
          atomicAdd(yrow + p0.x, __float2uint_rn(av * __int_as_float(p0.y)));
          atomicAdd(yrow + p1.x, __float2uint_rn(av * __int_as_float(p1.y)));
        }
        if (j < cnt) {
          const int2 p0 = up[j];
          atomicAdd(yrow + p0.x, __float2uint_rn(av * __int_as_float(p0.y)));
        }
      }
    }
    __syncthreads();
    uint8_t* tbase = ytile + (size_t)tile * kVtM * kn * 4;
    for (int i = threadIdx.x; i < kVtM * ng; i += T) {
      const int r = i / ng, g = i - r * ng;
      const int c0 = 8 * g, q = c0 >> 6, w = min(64, kn - 64 * q);
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const float y0 = (float)Ysm[r * ys + c0 + 2 * v] * 0x1p-15f;
        const float y1 = (float)Ysm[r * ys + c0 + 2 * v + 1] * 0x1p-15f;
        const __half h0 = __float2half_rn(y0), h1 = __float2half_rn(y1);
        const __half l0 = __float2half_rn(y0 - __half2float(h0)), l1 = __float2half_rn(y1 - __half2float(h1));
        hw[v] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
        lw[v] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
      }
      uint8_t* cb = tbase + (size_t)64 * q * kVtM * 4;
      const uint32_t off = tc::kmajor_off16(r, c0 - 64 * q, w);
      *reinterpret_cast<uint4*>(cb + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4*>(cb + (size_t)kVtM * w * 2 + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
    __syncthreads();
  }
}

}  // namespace esk
