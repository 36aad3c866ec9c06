// k_merge.cuh -- multi-GPU shard merge of the per-column top-t.
//
// Every rank selects, among its own rows, the top-t of each column (same key:
// value descending, GLOBAL row ascending).  The global top-t of a column is the
// top-t of the union of the local top-t sets (any entry of the global top-t is
// in the top-t of its own shard), so after an allgather of the local
// candidates every rank runs the same deterministic merge and obtains the
// factor a single GPU would produce, bit for bit.
//
// Exchange buffer of one rank (fixed size, so it can be allgathered as is):
//   int64 cnt[k]; int32 row[k * cap]; float val[k * cap]   (column c at c*cap)
// Rows are ascending within a column; ranks own increasing row ranges, so the
// concatenation over ranks of a column's candidates is ascending in row.
#pragma once
#include "common.cuh"

namespace esk {

struct ShardBuf {
  int64_t* cnt;
  int32_t* row;
  float* val;
};

ESNMF_DEV ShardBuf shard_view(void* base, int k, int64_t cap) {
  ShardBuf b;
  b.cnt = reinterpret_cast<int64_t*>(base);
  b.row = reinterpret_cast<int32_t*>(b.cnt + k);
  b.val = reinterpret_cast<float*>(b.row + (int64_t)k * cap);
  return b;
}

inline size_t shard_bytes(int k, int64_t cap) { return sizeof(int64_t) * k + (sizeof(int32_t) + sizeof(float)) * k * cap; }

// local COO (colptr, row, val) -> this rank's exchange buffer
__global__ void k_pack_shard(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                             const float* __restrict__ val, int k, int64_t cap, void* __restrict__ buf) {
  const ShardBuf b = shard_view(buf, k, cap);
  const int c = blockIdx.y;
  const int64_t s = colptr[c], n = colptr[c + 1] - s;
  if (blockIdx.x == 0 && threadIdx.x == 0) b.cnt[c] = n;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    b.row[(int64_t)c * cap + q] = row[s + q];
    b.val[(int64_t)c * cap + q] = val[s + q];
  }
}

// kept count per column = min(t, total candidates); colptr by exclusive scan
__global__ void k_merge_counts(const void* __restrict__ gathered, size_t rank_bytes, int world, int k, int64_t cap,
                               int64_t t, int64_t* __restrict__ colptr) {
  __shared__ int64_t sm[33];
  int64_t v = 0;
  if ((int)threadIdx.x < k) {
    for (int p = 0; p < world; ++p) {
      const ShardBuf b = shard_view((char*)gathered + p * rank_bytes, k, cap);
      v += b.cnt[threadIdx.x];
    }
    if (t >= 0 && v > t) v = t;
  }
  int64_t tot;
  const int64_t ex = block_exscan(v, sm, &tot);
  if ((int)threadIdx.x < k) colptr[threadIdx.x] = ex;
  if (threadIdx.x == 0) colptr[k] = tot;
}

// one block per column: threshold key of the t-th candidate, then an ordered
// (row-ascending) filter of the concatenated candidate lists
constexpr int kMergeCap = 4096;  // candidates sorted in shared memory (32 KB)

__global__ void __launch_bounds__(1024) k_merge_topt(const void* __restrict__ gathered, size_t rank_bytes, int world,
                                                     int k, int64_t cap, int64_t t,
                                                     const int64_t* __restrict__ colptr, int32_t* __restrict__ out_row,
                                                     float* __restrict__ out_val, uint64_t* __restrict__ scratch) {
  __shared__ uint64_t keys[kMergeCap];
  __shared__ int64_t base[65];
  __shared__ int64_t sm[33];
  const int c = blockIdx.x;
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int p = 0; p < world; ++p) {
      base[p] = acc;
      acc += shard_view((char*)gathered + p * rank_bytes, k, cap).cnt[c];
    }
    base[world] = acc;
  }
  __syncthreads();
  const int64_t n = base[world];
  auto entry = [&](int64_t q, int32_t& r, float& v) {
    int p = 0;
    while (q >= base[p + 1]) ++p;
    const ShardBuf b = shard_view((char*)gathered + p * rank_bytes, k, cap);
    const int64_t o = (int64_t)c * cap + (q - base[p]);
    r = b.row[o];
    v = b.val[o];
  };
  uint64_t kstar = ~0ULL;  // keep everything when n <= t
  if (t >= 0 && n > t) {
    // the t-th smallest key (value desc, row asc) among the n candidates
    uint64_t* ks = n <= kMergeCap ? keys : scratch + (int64_t)c * 2 * cap * world;
    int64_t np = 1;
    while (np < n) np <<= 1;
    for (int64_t q = threadIdx.x; q < np; q += blockDim.x) {
      uint64_t key = ~0ULL;
      if (q < n) {
        int32_t r;
        float v;
        entry(q, r, v);
        key = sel_key(v, (uint32_t)r);
      }
      ks[q] = key;
    }
    __syncthreads();
    for (int64_t size = 2; size <= np; size <<= 1) {
      for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (int64_t i = threadIdx.x; i < np; i += blockDim.x) {
          const int64_t j = i ^ stride;
          if (j > i) {
            const bool up = (i & size) == 0;
            const uint64_t x = ks[i], y = ks[j];
            if ((x > y) == up) { ks[i] = y; ks[j] = x; }
          }
        }
        __syncthreads();
      }
    }
    kstar = ks[t - 1];
    __syncthreads();
  }
  // ordered filter: candidates are row-ascending in concatenation order
  int64_t off = colptr[c];
  for (int64_t q0 = 0; q0 < n; q0 += blockDim.x) {
    const int64_t q = q0 + threadIdx.x;
    int32_t r = 0;
    float v = 0.f;
    bool keep = false;
    if (q < n) {
      entry(q, r, v);
      keep = sel_key(v, (uint32_t)r) <= kstar;
    }
    int64_t tot;
    const int64_t ex = block_exscan((int64_t)keep, sm, &tot);
    if (keep) {
      out_row[off + ex] = r;
      out_val[off + ex] = v;
    }
    off += tot;
  }
}

}  // namespace esk
