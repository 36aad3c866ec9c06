// k_csr.cuh -- input CSR handling at create time: packing, validation, A^T.
#pragma once
#include "common.cuh"

namespace esk {

// (int32 column, fp32 value) pairs -> one 8-byte entry per stored element
__global__ void k_pack(const int32_t* __restrict__ col, const float* __restrict__ val, int64_t nnz,
                       int2* __restrict__ ent) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    ent[e] = make_int2(col[e], __float_as_int(val[e]));
}


// ---- A^T from A on the device (used when the caller gives only CSR(A)) ----
__global__ void k_col_count(const int2* __restrict__ ent, int64_t nnz, int64_t* __restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd((unsigned long long*)&cnt[ent[e].x], 1ULL);
}

constexpr int kScanBlock = 2048;

// (rmask = 1: every count rounded up to even first -- 16-byte aligned pair rows)
__global__ void k_blocksum_i64(const int64_t* __restrict__ a, int64_t n, int64_t* __restrict__ bsum,
                               int64_t rmask = 0) {
  __shared__ int64_t sm[32];
  int64_t s = 0;
  const int64_t base = blockIdx.x * (int64_t)kScanBlock;
  for (int q = threadIdx.x; q < kScanBlock; q += blockDim.x) {
    const int64_t i = base + q;
    if (i < n) s += (a[i] + rmask) & ~rmask;
  }
  s = block_sum(s, sm);
  if (threadIdx.x == 0) bsum[blockIdx.x] = s;
}

// in place exclusive scan of a[0..n) given exclusive block offsets; 256 threads x 8
__global__ void k_scan_apply_i64(int64_t* __restrict__ a, int64_t n, const int64_t* __restrict__ boff,
                                 int64_t rmask = 0) {
  __shared__ int64_t sm[33];
  constexpr int per = kScanBlock / 256;
  const int64_t base = blockIdx.x * (int64_t)kScanBlock + threadIdx.x * per;
  int64_t v[per];
  int64_t s = 0;
#pragma unroll
  for (int q = 0; q < per; ++q) {
    v[q] = base + q < n ? (a[base + q] + rmask) & ~rmask : 0;
    s += v[q];
  }
  int64_t tot;
  int64_t off = boff[blockIdx.x] + block_exscan(s, sm, &tot);
#pragma unroll
  for (int q = 0; q < per; ++q) {
    if (base + q < n) a[base + q] = off;
    off += v[q];
  }
}


// sort every row of A^T by column (terms are distinct within a document):
// bitonic sort of 64-bit (col << 32 | value bits) keys.  Rows up to
// kRowSortCap entries sort in shared memory; longer rows in `scratch`.
constexpr int kRowSortCap = 4096;

__global__ void __launch_bounds__(256) k_sort_rows(const int64_t* __restrict__ ptr, int64_t rows,
                                                   int2* __restrict__ ent, uint64_t* __restrict__ scratch,
                                                   int long_rows_only) {
  __shared__ uint64_t keys[kRowSortCap];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t s = ptr[r], e = ptr[r + 1];
    const int64_t len = e - s;
    if (len <= 1 || len <= 512) continue;  // rows <= kRankRow: k_sort_rows_rank
    const bool fits = len <= kRowSortCap;
    if (fits == (bool)long_rows_only) continue;
    int64_t np = 1;
    while (np < len) np <<= 1;
    uint64_t* a = fits ? keys : scratch;
    for (int64_t i = threadIdx.x; i < np; i += blockDim.x)
      a[i] = i < len ? (((uint64_t)(uint32_t)ent[s + i].x << 32) | (uint32_t)ent[s + i].y) : ~0ULL;
    __syncthreads();
    for (int64_t size = 2; size <= np; size <<= 1) {
      for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (int64_t i = threadIdx.x; i < np; i += blockDim.x) {
          const int64_t j = i ^ stride;
          if (j > i) {
            const bool up = (i & size) == 0;
            const uint64_t x = a[i], y = a[j];
            if ((x > y) == up) { a[i] = y; a[j] = x; }
          }
        }
        __syncthreads();
      }
    }
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x)
      ent[s + i] = make_int2((int32_t)(a[i] >> 32), (int32_t)(uint32_t)(a[i] & 0xFFFFFFFFu));
    __syncthreads();
  }
}

}  // namespace esk

namespace esk {

// ---- row normalisation (NEXT-4): a_ij / nnz(row i of A), fp32 correctly rounded ----
// A's term rows (local rows r = global row0 + r)
__global__ void k_norm_rows(const int64_t* __restrict__ ptr, int2* __restrict__ ent, int64_t rows, int64_t row0,
                            const float* __restrict__ rowlen) {
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
       r += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const float len = rowlen[row0 + r];
    for (int64_t e = ptr[r] + (threadIdx.x & 31); e < ptr[r + 1]; e += 32) {
      int2 en = ent[e];
      en.y = __float_as_int(__fdiv_rn(__int_as_float(en.y), len));
      ent[e] = en;
    }
  }
}

// A^T's entries: the column index is the term
__global__ void k_norm_cols(int2* __restrict__ ent, int64_t nnz, const float* __restrict__ rowlen) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    int2 en = ent[e];
    en.y = __float_as_int(__fdiv_rn(__int_as_float(en.y), rowlen[en.x]));
    ent[e] = en;
  }
}

}  // namespace esk

namespace esk {

// ---- create-time CSR work in balanced units -----------------------------------
// A term row of A can hold half a million entries (Zipf head); one warp per row
// left the create-time passes waiting on the longest rows.  A RowChunk is <=
// kChunkLen consecutive entries of one row; one warp per chunk.
constexpr int64_t kChunkLen = 1024;
struct RowChunk {
  int64_t begin, end;
  int32_t row, pad_;
};

// CSR checks (row_ptr is checked on the host): column in range and strictly
// increasing within the row, value finite and >= 0
__global__ void k_validate_chunks(const RowChunk* __restrict__ ch, int64_t nch, const int64_t* __restrict__ ptr,
                                  const int2* __restrict__ ent, int64_t ncols, int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < nch; u += nwarps) {
    const RowChunk c = ch[u];
    const int64_t rs = ptr[c.row];
    int flags = 0;
    for (int64_t q = c.begin + lane; q < c.end; q += 32) {
      const int2 en = ent[q];
      if (en.x < 0 || en.x >= ncols) flags |= 2;
      if (q > rs && ent[q - 1].x >= en.x) flags |= 4;
      const float v = __int_as_float(en.y);
      if (!(v >= 0.f) || !isfinite(v)) flags |= 8;
    }
    flags = __reduce_or_sync(kFull, flags);
    if (lane == 0 && flags) atomicOr(bad, flags);
  }
}

// transpose scatter: entry (row r, col j, v) -> (r, v) at an atomic slot of row j
__global__ void k_transpose_chunks(const RowChunk* __restrict__ ch, int64_t nch, const int2* __restrict__ ent,
                                   unsigned long long* __restrict__ cursor, int2* __restrict__ tent) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < nch; u += nwarps) {
    const RowChunk c = ch[u];
    for (int64_t q = c.begin + lane; q < c.end; q += 32) {
      const int2 en = ent[q];
      const int64_t p = (int64_t)atomicAdd(&cursor[en.x], 1ULL);
      tent[p] = make_int2(c.row, en.y);
    }
  }
}

// order every row of <= kRankRow entries by column: one warp per row, the row
// staged in shared memory, each entry's slot = the number of smaller columns
// (columns are distinct within a row); longer rows: k_sort_rows(long_rows_only)
constexpr int kRankRow = 512;
// the rank sort of one row held in shared memory (b[0..len), len <= 32 * PER):
// entry i goes to position #{j : b[j].x < b[i].x} (the columns are distinct)
template <int PER>
__device__ __forceinline__ void rank_row(const int2* __restrict__ b, int len, int2* __restrict__ out, int lane) {
  int mine[PER], rank[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int i = lane + 32 * q;
    mine[q] = i < len ? b[i].x : 0x7FFFFFFF;
    rank[q] = 0;
  }
  for (int j = 0; j < len; ++j) {
    const int cj = b[j].x;  // broadcast
#pragma unroll
    for (int q = 0; q < PER; ++q) rank[q] += cj < mine[q];
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int i = lane + 32 * q;
    if (i < len) out[rank[q]] = b[i];
  }
}

__global__ void __launch_bounds__(256) k_sort_rows_rank(const int64_t* __restrict__ ptr, int64_t rows,
                                                        int2* __restrict__ ent) {
  __shared__ int2 buf[8][kRankRow];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int2* b = buf[w];
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows; r += nwarps) {
    const int64_t s = ptr[r];
    const int len = (int)(ptr[r + 1] - s);
    if (len <= 1 || len > kRankRow) continue;  // warp-uniform
    for (int i = lane; i < len; i += 32) b[i] = ent[s + i];
    __syncwarp();
    // as many entries per lane as the row needs (the compare loop is len x PER)
    if (len <= 64) rank_row<2>(b, len, ent + s, lane);
    else if (len <= 96) rank_row<3>(b, len, ent + s, lane);
    else if (len <= 128) rank_row<4>(b, len, ent + s, lane);
    else if (len <= 160) rank_row<5>(b, len, ent + s, lane);
    else if (len <= 192) rank_row<6>(b, len, ent + s, lane);
    else if (len <= 256) rank_row<8>(b, len, ent + s, lane);
    else rank_row<kRankRow / 32>(b, len, ent + s, lane);
    __syncwarp();
  }
}

}  // namespace esk
