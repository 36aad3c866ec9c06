// common.cuh -- shared device helpers for libesnmf (sm_100a).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define ESNMF_DEV __device__ __forceinline__

// Device bounds checks (compute-sanitizer is not available on the GPU pool):
// built with -DESNMF_DEBUG_CHECKS=1 (tools/debug_checks.sh) every ESNMF_CHECK
// prints the failing condition with its block / thread and traps, so the test
// suite run on the debug library stops at the first out-of-range index; in the
// product build it compiles to nothing.
#ifndef ESNMF_DEBUG_CHECKS
#define ESNMF_DEBUG_CHECKS 0
#endif
#if ESNMF_DEBUG_CHECKS
#define ESNMF_CHECK(cond)                                                                                 \
  do {                                                                                                  \
    if (!(cond)) {                                                                                      \
      printf("ESNMF_CHECK failed: %s at %s:%d block %d thread %d\n", #cond, __FILE__, __LINE__,         \
             (int)blockIdx.x, (int)threadIdx.x);                                                        \
      __trap();                                                                                         \
    }                                                                                                   \
  } while (0)
#else
#define ESNMF_CHECK(cond) \
  do {                    \
  } while (0)
#endif

namespace esk {

// dynamic shared memory of the running launch, bytes (bounds checks)
ESNMF_DEV uint32_t dyn_smem_bytes() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// One unit of SpMM work: `len` stored entries of output row `row` starting at
// `start` of the operator CSR.  Rows longer than the split length are cut into
// several items whose partial rows are summed afterwards in a fixed order.
struct WorkItem {
  int64_t start;
  int32_t row;   // local output row
  int32_t len;
};

// A row split over several items: partial slots [first, first+count).
struct SplitRow {
  int32_t row;
  int32_t first;
  int32_t count;
  int32_t pad_;
};

// Per-column state of the top-t selection.
struct ColSel {
  int32_t digit;     // threshold bucket D: -1 keep all positives, kNumBins keep none
  int32_t pad_;
  int64_t r;         // entries still to take from bucket D
  int64_t above;     // positives in buckets > D
  int64_t ncand;     // positives in bucket D
  int64_t npos;      // positives in the column
};

constexpr int kSelBits = 12;             // first-level bucket: float bits 30..19
constexpr int kNumBins = 1 << kSelBits;  // 4096
constexpr int kSelShift = 31 - kSelBits; // 19
constexpr int kSelChunk = 8192;          // rows per selection block
constexpr int kSelSeg = 1024;            // rows per output segment (one warp in k_sel_write)
constexpr int kSelSegs = kSelChunk / kSelSeg;
constexpr int kSelCap = 4096;            // candidates sorted in shared memory

ESNMF_DEV uint32_t f2u(float x) { return __float_as_uint(x); }

// Ascending 64-bit key = (value descending, row ascending) for x > 0.
ESNMF_DEV uint64_t sel_key(float x, uint32_t row) {
  return ((uint64_t)(0x7FFFFFFFu - f2u(x)) << 32) | (uint64_t)row;
}

ESNMF_DEV int sel_digit(float x) { return (int)(f2u(x) >> kSelShift); }

template <typename T>
ESNMF_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Deterministic block sum (fixed shuffle tree, fixed warp order).  All
// threads must call; result valid in every thread.  smem: >= 32 doubles.
template <typename T>
__device__ T block_sum(T v, T* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  T s = 0;
  if (wid == 0) {
    s = lane < nw ? smem[lane] : T(0);
    s = warp_sum(s);
    if (lane == 0) smem[0] = s;
  }
  __syncthreads();
  s = smem[0];
  __syncthreads();
  return s;
}

// Exclusive block scan of int64 values (one per thread); returns the exclusive
// prefix, writes the block total to *total.  smem: >= 33 int64.
__device__ inline int64_t block_exscan(int64_t v, int64_t* smem, int64_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int64_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  __syncthreads();
  if (lane == 31) smem[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int64_t w = lane < nw ? smem[lane] : 0;
    int64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(kFull, wi, o);
      if (lane >= o) wi += y;
    }
    smem[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) smem[32] = wi;
  }
  __syncthreads();
  int64_t ex = smem[wid] + inc - v;
  *total = smem[32];
  __syncthreads();
  return ex;
}

inline unsigned grid_for(int64_t work, int per_block, int64_t max_blocks = 1 << 20) {
  int64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (unsigned)b;
}

}  // namespace esk
