// k_spmm_terms.cuh -- U-side product LS_U = (A V)(V^T V + eps I)^{-1}
// ("U = A V (V^T V)^{-1}"), in the paper's order.
//
// V is very sparse (<= k t entries over m documents: ~9 % of the documents are
// active at Large, ~1.1 entries per active document), so instead of gathering a
// dense k-wide row per stored entry of A, every lane handles its own entry:
//  * activity test: one bit of `vbits` (m bits, L1-resident);
//  * vmap[doc] = (first << 32) | count of the doc's (column, value) pairs in
//    `vent` (row-CSR of V), looked up only for active entries;
//  * each product a_ij * v_jc is added, lane-parallel, into a per-warp
//    shared-memory accumulator of k 64-bit FIXED-POINT integers with the row
//    scale S_i = 2^62 / (rowsum_i(A) * max(V)).  Every term is >= 0 and the row
//    sum is <= 2^62, integer addition is exact and order-free, so the result
//    is deterministic whatever the atomic order; the quantisation error is
//    <= 2^-63 rowsum_i max(V) per product (~1e-16 relative);
//  * the finished row Y_i is converted to fp64 and multiplied by W = (V^T V +
//    eps I)^{-1} in fp64 (zero entries of Y_i skipped), rounded once to fp32.
// Rows longer than the split length arrive as several work items; their
// integer partial rows are summed exactly by k_terms_combine.
#pragma once
#include "common.cuh"

namespace esk {

// ---- V row view for the U side: vbits (m bits), vmap[m] (0 = inactive),
// vent (pairs of each active row, column ascending), vmax (max value bits) ----
__global__ void k_vrows_count(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                              const int32_t* __restrict__ rowmap, int64_t* __restrict__ rcnt) {
  const int c_ = blockIdx.y;
  const int64_t cb = colptr[c_], ce = colptr[c_ + 1];
  for (int64_t e = cb + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ce; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(&rcnt[rowmap[row[e]]]), 1ull);
}

// rptr = exclusive scan of rcnt (done by the caller); scatter pairs with a cursor
__global__ void k_vrows_scatter(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                                const float* __restrict__ val, const int32_t* __restrict__ rowmap,
                                int64_t* __restrict__ cursor, int2* __restrict__ vent, uint32_t* __restrict__ vmax) {
  const int c_ = blockIdx.y;
  const int64_t cb = colptr[c_], ce = colptr[c_ + 1];
  uint32_t mx = 0;
  for (int64_t e = cb + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ce; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(&cursor[rowmap[row[e]]]), 1ull);
    vent[p] = make_int2(c_, __float_as_int(val[e]));
    mx = max(mx, __float_as_uint(val[e]));  // values are > 0: bits order like values
  }
  mx = __reduce_max_sync(kFull, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(vmax, mx);
}

// one thread per active row: sort its pairs by column (<= k, usually 1-2),
// publish vmap / vbits for the row's document
__global__ void k_vrows_finish(const int32_t* __restrict__ active, const int64_t* __restrict__ n_active,
                               const int64_t* __restrict__ rptr, int2* __restrict__ vent, uint64_t* __restrict__ vmap,
                               uint32_t* __restrict__ vbits) {
  const int64_t na = *n_active;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < na; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = rptr[r], e = rptr[r + 1];
    for (int64_t a = s + 1; a < e; ++a) {
      const int2 key = vent[a];
      int64_t b = a - 1;
      while (b >= s && vent[b].x > key.x) {
        vent[b + 1] = vent[b];
        --b;
      }
      vent[b + 1] = key;
    }
    const int32_t doc = active[r];
    vmap[doc] = ((uint64_t)s << 32) | (uint64_t)(e - s);
    atomicOr(&vbits[doc >> 5], 1u << (doc & 31));
  }
}

// max(V) bits only (the U side's fixed-point scale) when the row-CSR is not needed
__global__ void k_vmax_only(const int64_t* __restrict__ colptr, const float* __restrict__ val, int k,
                            uint32_t* __restrict__ vmax) {
  const int64_t n = colptr[k];
  uint32_t mx = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, __float_as_uint(val[e]));  // values > 0: bits order like values
  mx = __reduce_max_sync(kFull, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(vmax, mx);
}

// clear the previous V's vmap / vbits entries (by its active list)
__global__ void k_vrows_clear(const int32_t* __restrict__ active, const int64_t* __restrict__ n_active,
                              uint64_t* __restrict__ vmap, uint32_t* __restrict__ vbits) {
  const int64_t na = *n_active;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < na; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t doc = active[r];
    vmap[doc] = 0;
    vbits[doc >> 5] = 0;
  }
}

// row sums of A (fp64) for the fixed-point scales, one block per row (grid-stride):
// A's term rows are Zipf-long (the top ones hold most documents), which left a
// warp per row running one long row alone; the block sum is a fixed tree
__global__ void __launch_bounds__(256) k_rowsum(const int64_t* __restrict__ ptr, const int2* __restrict__ ent,
                                                int64_t rows, double* __restrict__ rsum) {
  __shared__ double sm[32];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    double s = 0;
    for (int64_t q = ptr[r] + threadIdx.x; q < ptr[r + 1]; q += blockDim.x) s += (double)__int_as_float(ent[q].y);
    s = block_sum(s, sm);
    if (threadIdx.x == 0) rsum[r] = s;
  }
}

// Y_i (fixed point, lane-owned columns c = lane + 32 q) -> LS row = Y_i W (fp64)
template <int CQ>
ESNMF_DEV void terms_epilogue(const unsigned long long (&yq)[CQ], double unit, const double* __restrict__ W, int k,
                              int lane, double (&o)[CQ]) {
#pragma unroll
  for (int q = 0; q < CQ; ++q) o[q] = 0.0;
#pragma unroll
  for (int q = 0; q < CQ; ++q) {
    const double yv = (double)yq[q] * unit;
    unsigned nz = __ballot_sync(kFull, yq[q] != 0ull);
    while (nz) {
      const int ll = __ffs(nz) - 1;
      nz &= nz - 1;
      const double yl = __shfl_sync(kFull, yv, ll);
      const double* Wl = W + (int64_t)(32 * q + ll) * k;
#pragma unroll
      for (int qq = 0; qq < CQ; ++qq) {
        const int c = lane + 32 * qq;
        if (c < k) o[qq] = fma(yl, __ldg(Wl + c), o[qq]);
      }
    }
  }
}

template <int CQ>
__global__ void __launch_bounds__(256) k_spmm_terms(const WorkItem* __restrict__ items, int64_t nitems,
                                                    const int32_t* __restrict__ item_slot,
                                                    const int2* __restrict__ ent, const double* __restrict__ rsum,
                                                    const uint32_t* __restrict__ vbits,
                                                    const uint64_t* __restrict__ vmap,
                                                    const int2* __restrict__ vent, const uint32_t* __restrict__ vmax,
                                                    const double* __restrict__ W, int k, int kpad,
                                                    float* __restrict__ X, int64_t ldx,
                                                    unsigned long long* __restrict__ partial) {
  constexpr int NB = 4;  // batches of 32 entries in flight per warp
  __shared__ unsigned long long ysm[8][CQ * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long* ys = ysm[warp];
  const double maxv = (double)__uint_as_float(*vmax);
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; it < nitems; it += nwarps) {
    const WorkItem w = items[it];
    const double D = rsum[w.row] * maxv;             // bound of every entry of Y_i
    const double S = D > 0 ? 0x1p62 / D : 0.0;       // fixed-point scale
#pragma unroll
    for (int q = 0; q < CQ; ++q) ys[lane + 32 * q] = 0ull;
    __syncwarp();
    const int64_t e = w.start + w.len;
    if (S > 0) {
      for (int64_t base = w.start; base < e; base += 32 * NB) {
        int2 en[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const int64_t idx = base + b * 32 + lane;
          en[b] = idx < e ? __ldcs(ent + idx) : make_int2(-1, 0);
        }
        uint32_t word[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) word[b] = en[b].x >= 0 ? __ldg(vbits + (en[b].x >> 5)) : 0u;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          if ((word[b] >> (en[b].x & 31)) & 1u) {
            const unsigned long long code = __ldg(reinterpret_cast<const unsigned long long*>(vmap) + en[b].x);
            const uint32_t p0 = (uint32_t)(code >> 32), cnt = (uint32_t)code;
            const double as = (double)__int_as_float(en[b].y) * S;
            for (uint32_t p = 0; p < cnt; ++p) {
              const int2 pr = __ldg(vent + p0 + p);
              atomicAdd(&ys[pr.x], __double2ull_rn(as * (double)__int_as_float(pr.y)));
            }
          }
        }
      }
    }
    __syncwarp();
    unsigned long long yq[CQ];
#pragma unroll
    for (int q = 0; q < CQ; ++q) yq[q] = ys[lane + 32 * q];
    __syncwarp();
    const int32_t slot = item_slot[it];
    if (slot >= 0) {  // part of a split row: exact integer partial
#pragma unroll
      for (int q = 0; q < CQ; ++q)
        if (lane + 32 * q < kpad) partial[(int64_t)slot * kpad + lane + 32 * q] = yq[q];
      continue;
    }
    double o[CQ];
    terms_epilogue<CQ>(yq, D * 0x1p-62, W, k, lane, o);
#pragma unroll
    for (int q = 0; q < CQ; ++q) {
      const int c = lane + 32 * q;
      if (c < k) X[(int64_t)c * ldx + w.row] = (float)o[q];
    }
  }
}

// split rows: exact integer sum of the item partials, then Y_i W
template <int CQ>
__global__ void __launch_bounds__(256) k_terms_combine(const SplitRow* __restrict__ splits, int64_t nsplit,
                                                       const unsigned long long* __restrict__ partial,
                                                       const double* __restrict__ rsum,
                                                       const uint32_t* __restrict__ vmax,
                                                       const double* __restrict__ W, int k, int kpad,
                                                       float* __restrict__ X, int64_t ldx) {
  const int lane = threadIdx.x & 31;
  const double maxv = (double)__uint_as_float(*vmax);
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q0 < nsplit; q0 += nwarps) {
    const SplitRow sr = splits[q0];
    unsigned long long yq[CQ];
#pragma unroll
    for (int q = 0; q < CQ; ++q) {
      unsigned long long s = 0;
      const int c = lane + 32 * q;
      if (c < kpad)
        for (int p = 0; p < sr.count; ++p) s += partial[(int64_t)(sr.first + p) * kpad + c];
      yq[q] = s;
    }
    double o[CQ];
    terms_epilogue<CQ>(yq, rsum[sr.row] * maxv * 0x1p-62, W, k, lane, o);
#pragma unroll
    for (int q = 0; q < CQ; ++q) {
      const int c = lane + 32 * q;
      if (c < k) X[(int64_t)c * ldx + sr.row] = (float)o[q];
    }
  }
}

}  // namespace esk
