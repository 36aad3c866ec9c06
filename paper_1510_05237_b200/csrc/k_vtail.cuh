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
// Data (built at create time, k_vt_count / k_vt_fill / sort): per 128-document
// tile, the tile's tail entries sorted by (term, row), each (row in tile << 24 |
// term, value).  The lanes of a warp then read neighbouring activity-bitmap words
// and map words and, for a frequent term, the same U row; entries of one term
// belong to different documents (different shared-memory rows).
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
#ifndef ESNMF_VT_THREADS
#define ESNMF_VT_THREADS 512
#endif
constexpr int kVtThreads = ESNMF_VT_THREADS;  // k_ytail block
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

// (row << 24 | term, value) <-> (term << 7 | row, value): the keys of the per-tile
// sort by term (create time, cub segmented radix sort): consecutive entries of a
// tile then share bitmap words, U-row map words and U rows
__global__ void k_vt_to_keys(const int2* __restrict__ tent, int64_t n, uint32_t* __restrict__ key,
                             int32_t* __restrict__ val) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = (uint32_t)tent[e].x;
    key[e] = ((x & kVtTermMask) << 7) | (x >> kVtTermBits);
    val[e] = tent[e].y;
  }
}
__global__ void k_vt_from_keys(const uint32_t* __restrict__ key, const int32_t* __restrict__ val, int64_t n,
                               int2* __restrict__ tent) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = key[e];
    tent[e] = make_int2((int)(((k & 127u) << kVtTermBits) | (k >> 7)), val[e]);
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

// publish umap[row] = (first << 32) | count for every active row of U -- or, for a
// row with one pair (most rows past rank ~2k), the pair itself (bit 63 set), which
// spares k_ytail a dependent load per entry; runs after k_ut_scale.  The rows
// published are listed in ulist (for the next clear), their number in *ulist_n.
// The same pass sums the per-half-step cost model of the V-side tail
// from the document frequencies of A (termlen[i] = stored entries of term i):
//   cost[0] = sum over active tail rows i of termlen_i * r_i   (paper order: products, k_ytail)
//   cost[1] = sum over active tail rows i of termlen_i * k     (reassociated: FMAs of the Z-row gather)
//   cost[2] = sum over active tail rows i of termlen_i         (active tail entries of A^T)
//   cost[3] = sum over active head rows of termlen_i * r_i     (head products, for the report)
// (integer-valued fp64 sums: exact in any order; cost[] zeroed by k_urows_clear), and
// its last block (a ticket, reset by that block) takes the product order of the
// tail: Z-row gather (*zpath = 1) when the paper order's products outweigh the
// gather's FMAs at the measured relative cost of one shared-memory fixed-point
// product vs one gathered FMA (ratio).
__global__ void k_urows_finish(const int32_t* __restrict__ active, const int64_t* __restrict__ n_active,
                               const int64_t* __restrict__ rptr, const int64_t* __restrict__ cursor,
                               int2* __restrict__ uent, uint64_t* __restrict__ umap,
                               uint32_t* __restrict__ ubits, int32_t* __restrict__ ulist,
                               int64_t* __restrict__ ulist_n, const int32_t* __restrict__ termlen,
                               const int32_t* __restrict__ headslot, int k, double* __restrict__ cost,
                               unsigned* __restrict__ ticket, double ratio, int* __restrict__ zpath) {
  __shared__ double sm[32];
  __shared__ bool last;
  const int64_t na = *n_active;
  if (blockIdx.x == 0 && threadIdx.x == 0) *ulist_n = na;
  double p = 0, z = 0, a = 0, hp = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < na; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = active[r];
    const int64_t cnt = cursor[r] - rptr[r];
    if (cnt == 1) {  // the (scaled) pair itself: bit 63, column in bits 32-39, value bits below
      const int2 p = uent[rptr[r]];
      umap[i] = (1ull << 63) | ((uint64_t)(uint32_t)p.x << 32) | (uint64_t)(uint32_t)p.y;
    } else {  // (rows start at even offsets: an odd row ends in a (0, 0) pad)
      if (cnt & 1) uent[rptr[r] + cnt] = make_int2(0, 0);
      umap[i] = ((uint64_t)rptr[r] << 32) | (uint64_t)cnt;
    }
    atomicOr(&ubits[i >> 5], 1u << (i & 31));
    ulist[r] = i;
    const double len = (double)termlen[i];
    if (headslot && headslot[i] >= 0) {
      hp += len * (double)cnt;
    } else {
      p += len * (double)cnt;
      z += len * k;
      a += len;
    }
  }
  p = block_sum(p, sm);
  z = block_sum(z, sm);
  a = block_sum(a, sm);
  hp = block_sum(hp, sm);
  if (threadIdx.x == 0) {
    atomicAdd(&cost[0], p);
    atomicAdd(&cost[1], z);
    atomicAdd(&cost[2], a);
    atomicAdd(&cost[3], hp);
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    if (last) {
      __threadfence();
      *zpath = __ldcg(cost) * ratio > __ldcg(cost + 1);
      *ticket = 0u;
    }
  }
}

__global__ void k_urows_clear(const int32_t* __restrict__ ulist, const int64_t* __restrict__ ulist_n,
                              uint64_t* __restrict__ umap, uint32_t* __restrict__ ubits, double* __restrict__ cost) {
  if (blockIdx.x == 0 && threadIdx.x < 8) cost[threadIdx.x] = 0.0;
  const int64_t na = *ulist_n;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < na; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = ulist[r];
    umap[i] = 0ull;
    ubits[i >> 5] = 0u;  // every listed row is cleared: whole words may go
  }
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

// fixed-point exponent of column c: 2^s_c * rowsum_max * umax_c <= 2^30;
// kNoTail: column c of U has no entry in a tail row (Y_tail[:, c] = 0)
constexpr int kNoTail = -100000;
ESNMF_DEV int vt_shift(uint32_t umax_bits, uint32_t rowsum_bits) {
  const float b = __uint_as_float(umax_bits) * __uint_as_float(rowsum_bits);  // rounded: slack below
  if (!(b > 0.f)) return kNoTail;
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
    if ((unsigned)p.x >= (unsigned)k) continue;  // a pad slot not yet written (k_urows_finish writes it)
    const int sh = vt_shift(umax[p.x], rb);
    if (sh != kNoTail) p.y = __float_as_int(ldexpf(__int_as_float(p.y), sh));  // (else: a head row, never read)
    uent[e] = p;
  }
}

// ---- Y_tail per tile, written as fp16 hi/lo K-major chunks ----
// Chunk q of a tile covers Y columns [K q, K q + w_q), w_q = min(K, kn - K q), K = kHeadK;
// it is stored as [hi: 128 x w_q fp16][lo: 128 x w_q fp16], K-major (tc.cuh),
// at ytile + tile * 128 * kn * 4 + K q * 128 * 4.
#ifndef ESNMF_HEAD_K
#define ESNMF_HEAD_K 64
#endif
constexpr int kVtYChunk = ESNMF_HEAD_K;  // Y chunk width K: the head kernel's K per stage
// ys: shared row stride in words (odd).  Tiles are taken from a global counter
// (*next, zeroed before the launch): a CTA that starts late (an SM busy with the
// solve on the other stream) simply takes fewer tiles.
// Entries are sorted by term inside a tile, so the lanes of a warp hold the same
// or neighbouring terms: their rows of U are of similar length (the per-lane
// product loops stay nearly convergent), lanes of one term load the same pairs
// (broadcast) and add into different document rows (different banks: ys odd).
#ifndef ESNMF_VT_SUB
#define ESNMF_VT_SUB 4
#endif
#ifndef ESNMF_VT_MINB
#define ESNMF_VT_MINB 3
#endif
constexpr int kVtSub = ESNMF_VT_SUB;  // entries per thread per round (their loads in flight together)
constexpr int kVtMinB = ESNMF_VT_MINB;                      // resident CTAs per SM the launch asks for
#ifndef ESNMF_VT_NOBITS
#define ESNMF_VT_NOBITS 0
#endif
#ifndef ESNMF_VT_PF
#define ESNMF_VT_PF 1
#endif
constexpr bool kVtPf = ESNMF_VT_PF != 0;                     // L2 prefetch of the next tile's entries

ESNMF_DEV void vt_add(uint32_t* yrow, float av, int2 p) {
  ESNMF_CHECK(p.x >= 0 && p.x < 256);
  atomicAdd(yrow + p.x, __float2uint_rn(av * __int_as_float(p.y)));
}

__global__ void __launch_bounds__(kVtThreads, ESNMF_VT_MINB) k_ytail(const int64_t* __restrict__ toff,
                                                         const int2* __restrict__ tent, int64_t ntiles,
                                                         const uint32_t* __restrict__ ubits,
                                                         const uint64_t* __restrict__ umap,
                                                         const int2* __restrict__ uent, int kn, int ys,
                                                         uint8_t* __restrict__ ytile,
                                                         unsigned long long* __restrict__ next,
                                                         const int* __restrict__ zpath) {
  if (zpath && *zpath) return;  // the cost model chose the Z-row gather this half-step
  extern __shared__ __align__(16) uint32_t Ysm[];
  __shared__ int64_t s_tile, s_next;
  const int T = blockDim.x;
  // tiles are claimed one ahead: the next tile's entries are prefetched into L2
  // (one bulk prefetch) while this one is processed, so the first link of the
  // entry -> bitmap -> map -> pairs chain is an L2 hit instead of an HBM read
  auto claim = [&]() -> int64_t {
    const int64_t t = (int64_t)atomicAdd(next, 1ull);
    if (kVtPf && t < ntiles) {
      const int64_t a = toff[t] & ~(int64_t)1;  // 16-byte aligned, inside the array
      const int64_t b = min((toff[t + 1] + 1) & ~(int64_t)1, toff[ntiles] & ~(int64_t)1);
      if (b > a) tc::bulk_prefetch_l2(tent + a, (uint32_t)((b - a) * 8));
    }
    return t;
  };
  if (threadIdx.x == 0) s_next = claim();
  for (;;) {
    if (threadIdx.x == 0) {
      s_tile = s_next;
      s_next = s_tile < ntiles ? claim() : ntiles;
    }
    {  // zero the Y tile, 16 bytes per store (the tile is 16-byte aligned, ys odd: its rows are not)
      const int nz = kVtM * ys;
      uint4* z4 = reinterpret_cast<uint4*>(Ysm);
      for (int i = threadIdx.x; i < nz / 4; i += T) z4[i] = make_uint4(0u, 0u, 0u, 0u);
      for (int i = (nz & ~3) + threadIdx.x; i < nz; i += T) Ysm[i] = 0u;
    }
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) break;
    const int64_t e1 = toff[tile + 1];
    for (int64_t base = toff[tile] + threadIdx.x; base < e1; base += (int64_t)kVtSub * T) {
      int2 en[kVtSub];
      uint64_t mp[kVtSub];
#pragma unroll
      for (int u = 0; u < kVtSub; ++u) {
        const int64_t e = base + (int64_t)u * T;
        en[u] = e < e1 ? __ldcs(tent + e) : make_int2(0, 0);
      }
#pragma unroll
      for (int u = 0; u < kVtSub; ++u) {
        const uint32_t term = (uint32_t)en[u].x & kVtTermMask;
#if ESNMF_VT_NOBITS
        mp[u] = base + (int64_t)u * T < e1 ? umap[term] : 0ull;  // 0 for an inactive term
#else
        const bool act = base + (int64_t)u * T < e1 && ((__ldg(ubits + (term >> 5)) >> (term & 31)) & 1u);
        mp[u] = act ? umap[term] : 0ull;
#endif
      }
#pragma unroll
      for (int u = 0; u < kVtSub; ++u) {
        const uint64_t m = mp[u];
        uint32_t* yrow = Ysm + ((uint32_t)en[u].x >> kVtTermBits) * ys;
        const float av = __int_as_float(en[u].y);
        if (m >> 63) {  // a one-pair row, inline in its map word (k_urows_finish): no pair load
          vt_add(yrow, av, make_int2((int)((m >> 32) & 0xFFu), (int)(uint32_t)m));
          continue;
        }
        const int cnt = (int)(m & 0xFFFFFFFFull);
        const int2* up = uent + (m >> 32);
        ESNMF_CHECK(((uint32_t)en[u].x >> kVtTermBits) < (uint32_t)kVtM && cnt <= kn);
        // a row starts at an even pair offset (16-byte aligned; k_urows_*): two pairs per load
        for (int j = 0; j < cnt; j += 2) {
          const int4 q = __ldg(reinterpret_cast<const int4*>(up + j));
          vt_add(yrow, av, make_int2(q.x, q.y));
          if (j + 1 < cnt) vt_add(yrow, av, make_int2(q.z, q.w));
        }
      }
    }
    __syncthreads();
    // convert: a thread takes two adjacent columns of one row (lanes on adjacent
    // pairs of a row: 2-way bank conflicts on the reads), writes 4 + 4 bytes
    uint8_t* tbase = ytile + (size_t)tile * kVtM * kn * 4;
    const int np = kn / 2;
    // pair i = (row r, columns c, c + 1), i = r np + c / 2, stepped by T without a division per step
    const int dr = T / np, dc = T - dr * np;
    int r = threadIdx.x / np, cp = threadIdx.x - r * np;
    for (; r < kVtM; r += dr, cp += dc) {
      if (cp >= np) { cp -= np; ++r; if (r >= kVtM) break; }
      const int c = 2 * cp;
      const int q = c / kVtYChunk, w = min(kVtYChunk, kn - kVtYChunk * q);
      const float y0 = (float)Ysm[r * ys + c] * 0x1p-15f;
      const float y1 = (float)Ysm[r * ys + c + 1] * 0x1p-15f;
      const __half h0 = __float2half_rn(y0), h1 = __float2half_rn(y1);
      const __half l0 = __float2half_rn(y0 - __half2float(h0)), l1 = __float2half_rn(y1 - __half2float(h1));
      uint8_t* cb = tbase + (size_t)kVtYChunk * q * kVtM * 4;
      const uint32_t off = tc::kmajor_off16(r, c - kVtYChunk * q, w);
      *reinterpret_cast<uint32_t*>(cb + off) = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
      *reinterpret_cast<uint32_t*>(cb + (size_t)kVtM * w * 2 + off) =
          (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
    }
    __syncthreads();
  }
}

// Z64 = U W in fp64 for the active rows of U (row r of the dense active view,
// written at its term: Z64[active[r]][c]; rows of inactive terms are stale and
// never read): the exact Z rows behind k_vside_prep's head chunks and k_polish_v
// (term-indexed, so the polish needs no rowmap lookup).  One warp per active row,
// lanes over columns (CJ = ceil(k / 32)).
template <int CJ>
__global__ void __launch_bounds__(256) k_form_z64(const float* __restrict__ dense, int kpad, int k,
                                                  const int64_t* __restrict__ n_active,
                                                  const int32_t* __restrict__ active, const double* __restrict__ W,
                                                  double* __restrict__ Z64) {
  const int lane = threadIdx.x & 31;
  const int64_t na = *n_active;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < na; r += nwarps) {
    float f[CJ];
    double acc[CJ];
#pragma unroll
    for (int j = 0; j < CJ; ++j) {
      const int c = lane + 32 * j;
      f[j] = c < kpad ? dense[r * kpad + c] : 0.f;
      acc[j] = 0.0;
    }
#pragma unroll
    for (int jl = 0; jl < CJ; ++jl) {
      const int lmax = min(32, k - 32 * jl);
      // the row's nonzeros only, in ascending l (the same sum as a loop over every l
      // that skips zeros): most active rows of U hold a few entries
      unsigned m = __ballot_sync(kFull, f[jl] != 0.f) & (lmax >= 32 ? ~0u : lmax <= 0 ? 0u : (1u << lmax) - 1u);
      while (m) {
        const int ll = __ffs(m) - 1;
        m &= m - 1u;
        const float fl = __shfl_sync(kFull, f[jl], ll);
        const double* Wl = W + (int64_t)(32 * jl + ll) * k;
#pragma unroll
        for (int j = 0; j < CJ; ++j) {
          const int c = lane + 32 * j;
          if (c < k) acc[j] = fma((double)fl, Wl[c], acc[j]);
        }
      }
    }
    double* zr = Z64 + (int64_t)active[r] * k;  // term-indexed: the readers skip inactive terms
#pragma unroll
    for (int j = 0; j < CJ; ++j) {
      const int c = lane + 32 * j;
      if (c < k) zr[c] = acc[j];
    }
  }
}

// The kept entries of V (after the selection) recomputed exactly: for kept
// (document j, topic c) LS_jc = sum over the document's stored entries a_ji Z_ic
// with Z = U W in fp64 (Z64, k_form_z64, term-indexed; a term whose row of U
// is empty -- its bit in ubits clear -- contributes zero).  The selection chose the entries from the tensor-core values; this
// pass makes the VALUES exact to fp32 rounding (BJ:5 "relative 1e-5 on factor
// entries").  Grid (x, k): half a warp per kept entry of column blockIdx.y,
// lanes over the document's entries.
constexpr int kPolHalf = 16;  // lanes per kept entry (two entries per warp)
constexpr int kPolIn = 10;    // document entries per lane in flight (16 x 10 >= a typical row)
__global__ void k_polish_v(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                           float* __restrict__ val, int k, int64_t row0, const int64_t* __restrict__ ptr,
                           const int2* __restrict__ ent, const uint32_t* __restrict__ ubits,
                           const double* __restrict__ Z64) {
  const int lane = threadIdx.x & 31, hl = lane & (kPolHalf - 1), hw = lane / kPolHalf;
  const int c = blockIdx.y;  // grid (x, k): the entries of column c, two per warp
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t cend = colptr[c + 1];
  for (int64_t e0 = colptr[c] + 2 * ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); e0 < cend;
       e0 += 2 * nw) {  // warp-uniform
    const int64_t e = e0 + hw;
    const bool valid = e < cend;
    int64_t s0 = 0, s1 = 0;
    if (valid) {
      const int64_t r = (int64_t)row[e] - row0;
      s0 = ptr[r];
      s1 = ptr[r + 1];
    }
    double acc = 0;
    for (int64_t q0 = s0 + hl; q0 < s1; q0 += kPolHalf * kPolIn) {
      int2 en[kPolIn];
      bool act[kPolIn];
      double z[kPolIn];
#pragma unroll
      for (int u = 0; u < kPolIn; ++u)
        en[u] = q0 + kPolHalf * u < s1 ? __ldg(ent + q0 + kPolHalf * u) : make_int2(0, 0);
#pragma unroll
      for (int u = 0; u < kPolIn; ++u)  // the term's row of U is non-empty (U's bitmap, L1-resident)
        act[u] = q0 + kPolHalf * u < s1 && ((__ldg(ubits + ((uint32_t)en[u].x >> 5)) >> (en[u].x & 31)) & 1u);
#pragma unroll
      for (int u = 0; u < kPolIn; ++u) z[u] = act[u] ? __ldg(Z64 + (int64_t)en[u].x * k + c) : 0.0;
#pragma unroll
      for (int u = 0; u < kPolIn; ++u) acc = fma((double)__int_as_float(en[u].y), z[u], acc);
    }
#pragma unroll
    for (int o = kPolHalf / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);  // within the half
    // an entry kept for a tensor-core LS value within rounding of zero keeps that
    // (positive) value: a factor holds no zeros or negatives (P:63 clamp)
    if (valid && hl == 0 && (float)acc > 0.f) val[e] = (float)acc;
  }
}

// The kept entries of U recomputed exactly (one GPU): LS_ic = sum_j Y_ij W_jc
// with Y = A V from the U side's exact fixed-point accumulator (Yq, k_uside_*:
// Y_ij = Yq[i][j] * unit, unit = rowsum_max * max(V) * 2^-62) and W in fp64.
// Grid (x, k): half a warp per kept entry of column blockIdx.y, lanes over j
// (4 loads per lane in flight).
__global__ void k_polish_u(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                           float* __restrict__ val, int k, int kpad, const unsigned long long* __restrict__ Yq,
                           const double* __restrict__ bound, const uint32_t* __restrict__ vmax,
                           const double* __restrict__ W) {
  const int lane = threadIdx.x & 31, hl = lane & (kPolHalf - 1), hw = lane / kPolHalf;
  const int c = blockIdx.y;  // grid (x, k): the entries of column c, two per warp
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t cend = colptr[c + 1];
  const double unit = *bound * (double)__uint_as_float(*vmax) * 0x1p-62;
  const double* wr = W + (int64_t)c * k;  // W symmetric: column c = row c (coalesced)
  for (int64_t e0 = colptr[c] + 2 * ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); e0 < cend;
       e0 += 2 * nw) {  // warp-uniform
    const int64_t e = e0 + hw;
    const bool valid = e < cend;
    const unsigned long long* yr = Yq + (int64_t)(valid ? row[e] : 0) * kpad;
    double acc = 0;
    for (int j0 = valid ? hl : k; j0 < k; j0 += 4 * kPolHalf) {
      unsigned long long y[4];
      double w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + kPolHalf * u;
        y[u] = j < k ? __ldg(yr + j) : 0ull;
        w[u] = j < k ? __ldg(wr + j) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = fma((double)y[u] * unit, w[u], acc);
    }
#pragma unroll
    for (int o = kPolHalf / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);  // within the half
    if (valid && hl == 0 && (float)acc > 0.f) val[e] = (float)acc;
  }
}

// U side's paper-order products for the current V: sum over V's entries (d, c) of
// the stored entries of document d (this rank's documents; out zeroed by the caller)
__global__ void k_u_cost(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row, int k, int64_t row0,
                         int64_t rows, const int64_t* __restrict__ ptr, double* __restrict__ out) {
  __shared__ double sm[32];
  const int64_t total = colptr[k];
  double p = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = (int64_t)row[e] - row0;
    if (d >= 0 && d < rows) p += (double)(ptr[d + 1] - ptr[d]);
  }
  p = block_sum(p, sm);
  if (threadIdx.x == 0) atomicAdd(out, p);
}

// dynamic shared memory of k_ytail: the Y tile and the long-row list
inline size_t ytail_smem(int ys) { return sizeof(uint32_t) * (size_t)kVtM * ys; }

}  // namespace esk
