// k_spmm.cuh -- the half-step product ("A^T U (U^T U)^{-1}", "A V (V^T V)^{-1}").
//
// LS[row, :] = sum over the stored (col, a) of operator row `row` of a * Z[rowmap[col], :]
// where Z = F (F^T F + eps I)^{-1} holds the active rows of the factor F (k_solve.cuh)
// and rowmap[col] < 0 marks an all-zero factor row (skipped: it contributes 0).
//
// Operator entries are packed (int32 col, fp32 value) pairs: one 8-byte,
// coalesced load per stored entry of A / A^T.  One warp per work item; the
// warp is split into NG = 32/G lane groups, each group gathers one factor row
// (KQ = kpad/4 float4 chunks, CPL chunks per lane) so NG entries are in flight
// per step.  Per-row accumulation order is fixed (deterministic), fp32.
#pragma once
#include "common.cuh"

namespace esk {

template <int G, int CPL>
struct SpmmAcc {
  float4 a[CPL];
};

template <int G, int CPL>
ESNMF_DEV void spmm_row(const int2* __restrict__ ent, int64_t s, int64_t e, const int32_t* __restrict__ rowmap,
                        const float4* __restrict__ Z, int KQ, SpmmAcc<G, CPL>& acc) {
  constexpr int NG = 32 / G;
  const int lane = threadIdx.x & 31;
  const int g = lane / G, lg = lane % G;
#pragma unroll
  for (int j = 0; j < CPL; ++j) acc.a[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t base = s; base < e; base += 32) {
    const int64_t idx = base + lane;
    int2 en = make_int2(0, 0);
    int32_t r = -1;
    if (idx < e) {
      en = __ldcs(ent + idx);  // streamed once per half-step: evict-first
      r = __ldg(rowmap + en.x);
    }
    const unsigned act = __ballot_sync(kFull, r >= 0);
    const int cnt = __popc(act);
    const float aval = __int_as_float(en.y);
    // NG entries per step, two steps unrolled: 2*NG factor-row gathers in flight
    for (int q0 = 0; q0 < cnt; q0 += 2 * NG) {
      const int qa = q0 + g, qb = q0 + NG + g;
      const int sa = qa < cnt ? (int)__fns(act, 0, qa + 1) : 0;
      const int sb = qb < cnt ? (int)__fns(act, 0, qb + 1) : 0;
      const float xa = __shfl_sync(kFull, aval, sa);
      const int32_t ra = __shfl_sync(kFull, r, sa);
      const float xb = __shfl_sync(kFull, aval, sb);
      const int32_t rb = __shfl_sync(kFull, r, sb);
      float4 za[CPL], zb[CPL];
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const int ch = lg + j * G;
        za[j] = (qa < cnt && ch < KQ) ? __ldg(Z + (int64_t)ra * KQ + ch) : make_float4(0.f, 0.f, 0.f, 0.f);
        zb[j] = (qb < cnt && ch < KQ) ? __ldg(Z + (int64_t)rb * KQ + ch) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        acc.a[j].x = fmaf(xa, za[j].x, acc.a[j].x);
        acc.a[j].y = fmaf(xa, za[j].y, acc.a[j].y);
        acc.a[j].z = fmaf(xa, za[j].z, acc.a[j].z);
        acc.a[j].w = fmaf(xa, za[j].w, acc.a[j].w);
      }
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        acc.a[j].x = fmaf(xb, zb[j].x, acc.a[j].x);
        acc.a[j].y = fmaf(xb, zb[j].y, acc.a[j].y);
        acc.a[j].z = fmaf(xb, zb[j].z, acc.a[j].z);
        acc.a[j].w = fmaf(xb, zb[j].w, acc.a[j].w);
      }
    }
  }
  // combine the lane groups (fixed xor tree -> deterministic)
#pragma unroll
  for (int o = G; o < 32; o <<= 1) {
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      acc.a[j].x += __shfl_xor_sync(kFull, acc.a[j].x, o);
      acc.a[j].y += __shfl_xor_sync(kFull, acc.a[j].y, o);
      acc.a[j].z += __shfl_xor_sync(kFull, acc.a[j].z, o);
      acc.a[j].w += __shfl_xor_sync(kFull, acc.a[j].w, o);
    }
  }
}

// Tiled variant for operators whose rows are never split (A^T: d entries per
// document).  A block owns 32 consecutive output rows at a time, stages them in
// shared memory and writes each LS column as a coalesced 128-byte run of the
// column-major LS buffer X[c * ldx + row].
template <int G, int CPL>
__global__ void __launch_bounds__(256) k_spmm_tiled(const int64_t* __restrict__ ptr, const int2* __restrict__ ent,
                                                    int64_t rows, const int32_t* __restrict__ rowmap,
                                                    const float4* __restrict__ Z, int KQ, int k,
                                                    float* __restrict__ X, int64_t ldx) {
  extern __shared__ float tile[];  // [kpad][33]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lg = lane % G;
  const int64_t ntiles = (rows + 31) / 32;
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int64_t r0 = tl * 32;
#pragma unroll 1
    for (int rr = warp; rr < 32; rr += 8) {
      const int64_t row = r0 + rr;
      SpmmAcc<G, CPL> acc;
      int64_t s = 0, e = 0;
      if (row < rows) { s = ptr[row]; e = ptr[row + 1]; }
      spmm_row<G, CPL>(ent, s, e, rowmap, Z, KQ, acc);
      if (lane < G) {
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          const int ch = lg + j * G;
          if (ch < KQ) {
            tile[(4 * ch + 0) * 33 + rr] = acc.a[j].x;
            tile[(4 * ch + 1) * 33 + rr] = acc.a[j].y;
            tile[(4 * ch + 2) * 33 + rr] = acc.a[j].z;
            tile[(4 * ch + 3) * 33 + rr] = acc.a[j].w;
          }
        }
      }
    }
    __syncthreads();
    const int nr = (int)(rows - r0 < 32 ? rows - r0 : 32);
    for (int q = threadIdx.x; q < k * 32; q += blockDim.x) {
      const int c = q >> 5, rr = q & 31;
      if (rr < nr) X[(int64_t)c * ldx + r0 + rr] = tile[c * 33 + rr];
    }
    __syncthreads();
  }
}

// Item variant for operators with long (Zipf) rows (A: term rows up to ~m
// entries).  Items covering a whole row write X directly; items of split rows
// write a partial row to `partial[slot]`, summed by k_spmm_combine.
template <int G, int CPL>
__global__ void __launch_bounds__(256) k_spmm_items(const WorkItem* __restrict__ items, int64_t nitems,
                                                    const int32_t* __restrict__ item_slot,
                                                    const int2* __restrict__ ent,
                                                    const int32_t* __restrict__ rowmap,
                                                    const float4* __restrict__ Z, int KQ, int k, int kpad,
                                                    float* __restrict__ X, int64_t ldx,
                                                    float* __restrict__ partial) {
  const int lane = threadIdx.x & 31;
  const int lg = lane % G;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = warp0; it < nitems; it += nwarps) {
    const WorkItem w = items[it];
    SpmmAcc<G, CPL> acc;
    spmm_row<G, CPL>(ent, w.start, w.start + w.len, rowmap, Z, KQ, acc);
    const int32_t slot = item_slot[it];
    if (lane < G) {
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const int ch = lg + j * G;
        if (ch < KQ) {
          const float v[4] = {acc.a[j].x, acc.a[j].y, acc.a[j].z, acc.a[j].w};
          if (slot < 0) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (4 * ch + u < k) X[(int64_t)(4 * ch + u) * ldx + w.row] = v[u];
          } else {
            reinterpret_cast<float4*>(partial + (int64_t)slot * kpad)[ch] = acc.a[j];
          }
        }
      }
    }
  }
}

// Sum the partial rows of split rows in slot order (fp64), one warp per row.
__global__ void k_spmm_combine(const SplitRow* __restrict__ splits, int64_t nsplit, const float* __restrict__ partial,
                               int k, int kpad, float* __restrict__ X, int64_t ldx) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = warp0; q < nsplit; q += nwarps) {
    const SplitRow sr = splits[q];
    for (int c = lane; c < k; c += 32) {
      double s = 0;
      for (int p = 0; p < sr.count; ++p) s += (double)partial[(int64_t)(sr.first + p) * kpad + c];
      X[(int64_t)c * ldx + sr.row] = (float)s;
    }
  }
}

}  // namespace esk
