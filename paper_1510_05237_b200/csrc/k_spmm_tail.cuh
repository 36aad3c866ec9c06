// k_spmm_tail.cuh -- V-side product over the "tail" terms, LS_V += A^T[:, tail] Z[tail, :]
// ("A^T U (U^T U)^{-1}", reassociated as A^T (U W)); the head terms run on
// the tensor cores first (k_vhead.cuh), so every document row of A^T is stored
// head entries first (k_reorder_head) and this kernel reads only
// [ptr[j] + nh[j], ptr[j+1]).
//
// What bounds it: after the head split each document keeps ~45 active tail
// entries (Large, h = 512), each a gather of a k-wide fp32 Z row (400 B, 13
// 32-byte sectors) that hits in L2 (~90 %) but rarely in L1 (~17 %): 45 M x
// 416 B = 19 GB of L2 -> SM traffic per launch, against an L2 ceiling of
// ~6300 B/clk (~12 TB/s; B300_MICROARCH.md "LTS throughput cap").  The kernel
// is therefore built to keep L2 requests in flight and to add no sectors:
//   * a warp owns RG = 4 documents; their tail segments are flattened and
//     loaded SUB = 4 entries per lane at a time, the next round (or the next
//     group's first round, bounds loaded one group ahead) prefetched while the
//     current one is gathered;
//   * active entries (bitmap test) are compacted, in row order, into a per-warp
//     shared list of (Z-row byte offset, value), each row's segment zero-padded
//     to a multiple of the gather step, so the gather loop has no predicates;
//   * U list slots per lane group in flight, packed FFMA2 accumulation; every
//     lane loads unconditionally (Z rows are zero-padded to G*CPL float4):
//     predicating the padding lanes' loads saves L2 sectors but measured
//     slower (1.90 vs 1.75 ms, Large, h = 512).
// Accumulation order per row is the row's entry order: deterministic.
#pragma once
#include "common.cuh"

namespace esk {

constexpr int kTailThreads = 256;
#ifndef ESNMF_TAIL_MINB
#define ESNMF_TAIL_MINB 3
#endif
constexpr int kTailMinBlocks = ESNMF_TAIL_MINB;
constexpr int kTailSub = 4;              // entries per lane per load round
constexpr int kTailRound = 32 * kTailSub;

// zero the Z rows of the terms listed (the previous V side's active terms)
// gate (all of this file's per-iteration kernels): null = run; else run only if *gate
// (the paper-order V side falls back to the Z-row gather for an ill-conditioned W)
__global__ void k_zrows_clear(const int32_t* __restrict__ terms, const int64_t* __restrict__ count,
                              float4* __restrict__ Z, int zq, const int* __restrict__ gate) {
  if (gate && !*gate) return;
  const int64_t cnt = *count;
  const int64_t total = cnt * zq;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q / zq;
    Z[(int64_t)terms[r] * zq + (q - r * zq)] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Z rows for the gather from the fp64 Z64 = U W already formed (paper-order mode,
// k_form_z64, term-indexed): Z[term][c] = fp32(Z64[term][c]) -- the rounding
// k_form_z applies to the same fp64 sums -- instead of a second k x k product per
// row.  One warp per active row; the rows' terms go to zlist for the next clear.
__global__ void k_form_z_from64(const int64_t* __restrict__ n_active, const int32_t* __restrict__ active, int k,
                                int zs, const double* __restrict__ Z64, float* __restrict__ Z,
                                int32_t* __restrict__ zlist, int64_t* __restrict__ zcount,
                                const int* __restrict__ gate) {
  if (gate && !*gate) return;
  const int lane = threadIdx.x & 31;
  const int64_t na = *n_active;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < na; r += nwarps) {
    const int32_t term = active[r];
    const double* zr64 = Z64 + (int64_t)term * k;
    float* zr = Z + (int64_t)term * zs;
    for (int c = lane; c < zs; c += 32) zr[c] = c < k ? (float)zr64[c] : 0.f;
    if (lane == 0) zlist[r] = term;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *zcount = na;
}

// term bitmap of the active rows of U (all bits cleared by the caller first)
__global__ void k_term_bits(const int32_t* __restrict__ active, const int64_t* __restrict__ n_active,
                            uint32_t* __restrict__ bits, const int* __restrict__ gate) {
  if (gate && !*gate) return;
  const int64_t na = *n_active;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < na; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = active[r];
    atomicOr(&bits[t >> 5], 1u << (t & 31));
  }
}

// Head entries (headslot >= 0) first, then the rest; both in their original
// order (stable).  Out-of-place; nh[row] = number of head entries.  The tensor
// core kernel reads its own copy of the head entries (k_head_fill); the tail
// gather reads [ptr + nh, ptr+1) and the U side reads whole rows.
__global__ void k_reorder_head(const int64_t* __restrict__ ptr, const int2* __restrict__ ent, int64_t rows,
                               const int32_t* __restrict__ headslot, int2* __restrict__ out,
                               int32_t* __restrict__ nh) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < rows; row += nw) {
    const int64_t s = ptr[row], e = ptr[row + 1];
    int64_t nhead = 0;
    for (int64_t b = s; b < e; b += 32) {  // pass 1: head entries
      const int64_t q = b + lane;
      int2 en = make_int2(0, 0);
      bool hd = false;
      if (q < e) {
        en = ent[q];
        hd = headslot[en.x] >= 0;
      }
      const unsigned m = __ballot_sync(kFull, hd);
      if (hd) out[s + nhead + __popc(m & lt)] = en;
      nhead += __popc(m);
    }
    int64_t ntail = 0;
    for (int64_t b = s; b < e; b += 32) {  // pass 2: the others
      const int64_t q = b + lane;
      int2 en = make_int2(0, 0);
      bool tl = false;
      if (q < e) {
        en = ent[q];
        tl = headslot[en.x] < 0;
      }
      const unsigned m = __ballot_sync(kFull, tl);
      if (tl) out[s + nhead + ntail + __popc(m & lt)] = en;
      ntail += __popc(m);
    }
    if (lane == 0) nh[row] = (int32_t)nhead;
  }
}

// packed fp32 FMA (FFMA2 on sm_100a): acc += x * z for two lanes of a float4
ESNMF_DEV void ffma4(float4& acc, float x, const float4& z) {
  const float2 lo = __ffma2_rn(make_float2(x, x), make_float2(z.x, z.y), make_float2(acc.x, acc.y));
  const float2 hi = __ffma2_rn(make_float2(x, x), make_float2(z.z, z.w), make_float2(acc.z, acc.w));
  acc = make_float4(lo.x, lo.y, hi.x, hi.y);
}

// G lanes per gathered Z row, CPL float4 per lane (Z rows are zs = G*CPL*4
// floats, zero-padded, so every lane loads unconditionally), U entries per lane
// group in flight, RG document rows per warp.
// TROW: store the rows ROW-MAJOR (stride ldx = kpad floats) into a staging
// buffer that the tensor-core head kernel reads and adds to the column-major LS
// buffer (400 contiguous bytes per row instead of 16-byte pieces of k columns);
// otherwise store column-major into the LS buffer directly (no head).
template <int G, int CPL, int U, int RG, bool TROW>
__global__ void __launch_bounds__(kTailThreads, kTailMinBlocks)
    k_spmm_tail(const int64_t* __restrict__ ptr, const int32_t* __restrict__ nh, const int2* __restrict__ ent,
                int64_t rows, const uint32_t* __restrict__ tbits, int nwords, const float4* __restrict__ Z, int zq,
                int kq, int k, float* __restrict__ X, int64_t ldx, const int* __restrict__ gate) {
  if (gate && !*gate) return;
  constexpr int NG = 32 / G;
  constexpr int STEP = U * NG;                         // list slots per gather step
  constexpr int LCAP = kTailRound + RG * (STEP - 1);   // compacted entries + per-row padding
  extern __shared__ uint32_t sbits_dyn[];
  __shared__ int2 stage[kTailThreads / 32][LCAP];
  __shared__ int64_t segb[kTailThreads / 32][RG];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / G, lg = lane % G;
  const uint32_t* sbits = nwords > 0 ? sbits_dyn : tbits;
  for (int q = threadIdx.x; q < nwords; q += blockDim.x) sbits_dyn[q] = tbits[q];
  __syncthreads();
  int2* st = stage[warp];
  int64_t* sb = segb[warp];
  const unsigned lt_mask = (1u << lane) - 1u;
  const char* zl = reinterpret_cast<const char*>(Z) + lg * 16;  // this lane's column chunk
  const uint32_t zrow = (uint32_t)zq * 16u;                      // bytes per Z row

  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ngroups = (rows + RG - 1) / RG;
  // Software pipeline across groups: the next group's row bounds are loaded at
  // the start of a group, and its first round of entries is fetched before the
  // current group's last gather loop, so no group starts on an HBM round trip.
  auto bounds = [&](int64_t gi, int64_t& ms, int& ml) {
    ms = 0;
    ml = 0;
    const int64_t r = gi * RG + lane;
    if (gi < ngroups && lane < RG && r < rows) {
      const int64_t a = ptr[r], b = ptr[r + 1];
      ms = a + (nh ? nh[r] : 0);
      ml = (int)(b - ms);
    }
  };
  int off[RG + 1];
  int L = 0;
  // flattened layout of a group: row q owns [off[q], off[q+1]); entry = sb[q] + index
  auto setup = [&](int64_t ms, int ml) {
    off[0] = 0;
#pragma unroll
    for (int q = 0; q < RG; ++q) off[q + 1] = off[q] + __shfl_sync(kFull, ml, q);
    int pre = 0;
#pragma unroll
    for (int q = 0; q < RG; ++q)
      if (lane == q) pre = off[q];
    __syncwarp();
    if (lane < RG) sb[lane] = ms - pre;
    __syncwarp();
    L = off[RG];
  };
  auto tag_of = [&](int idx) {
    int t = 0;
#pragma unroll
    for (int q = 1; q < RG; ++q) t += idx >= off[q];
    return t;
  };
  int2 en[kTailSub];
  auto fetch = [&](int rb) {
#pragma unroll
    for (int j = 0; j < kTailSub; ++j) {
      const int idx = rb + j * 32 + lane;
      en[j] = idx < L ? __ldcs(ent + sb[tag_of(idx)] + idx) : make_int2(0, 0);  // streamed once
    }
  };
  int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  {
    int64_t ms;
    int ml;
    bounds(grp, ms, ml);
    setup(ms, ml);
    fetch(0);
  }
  for (; grp < ngroups; grp += nwarps) {
    const int64_t r0 = grp * RG;
    int64_t nms;
    int nml;
    bounds(grp + nwarps, nms, nml);  // next group's bounds, consumed at this group's last round
    const int cL = L;
    float4 res[RG][CPL];
#pragma unroll
    for (int q = 0; q < RG; ++q)
#pragma unroll
      for (int j = 0; j < CPL; ++j) res[q][j] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int rb = 0; rb < cL; rb += kTailRound) {
      // pass 1: activity, per-row counts
      unsigned act[kTailSub];
      int tg[kTailSub];
      int cnt = 0;
      int rc[RG];
#pragma unroll
      for (int q = 0; q < RG; ++q) rc[q] = 0;
#pragma unroll
      for (int j = 0; j < kTailSub; ++j) {
        const int idx = rb + j * 32 + lane;
        tg[j] = tag_of(idx);
        const bool on = idx < cL && ((sbits[en[j].x >> 5] >> (en[j].x & 31)) & 1u);
        act[j] = __ballot_sync(kFull, on);
#pragma unroll
        for (int q = 0; q < RG - 1; ++q) rc[q] += __popc(__ballot_sync(kFull, on && tg[j] == q));
        cnt += __popc(act[j]);
      }
      {
        int sum = 0;
#pragma unroll
        for (int q = 0; q < RG - 1; ++q) sum += rc[q];
        rc[RG - 1] = cnt - sum;
      }
      // padded layout: row q's entries at [pb[q], pb[q] + rc[q]), zero slots up to a multiple of STEP
      // row q's slot shift (padding before it, < 256) packed into byte q of one
      // register: an indexed array here was placed in local memory
      static_assert(RG <= 4 && (RG - 1) * (STEP - 1) < 256, "packed row shifts");
      int pb[RG + 1];
      uint32_t shp = 0;
      pb[0] = 0;
      {
        int plain = 0;
#pragma unroll
        for (int q = 0; q < RG; ++q) {
          shp |= (uint32_t)(pb[q] - plain) << (8 * q);
          plain += rc[q];
          pb[q + 1] = pb[q] + (rc[q] + STEP - 1) / STEP * STEP;
        }
      }
      // pass 2: write (Z-row byte offset, value) in row order
      int run = 0;
#pragma unroll
      for (int j = 0; j < kTailSub; ++j) {
        if ((act[j] >> lane) & 1u) {
          const int sh = (int)((shp >> (8 * tg[j])) & 0xFFu);
          st[run + __popc(act[j] & lt_mask) + sh] = make_int2((int)((uint32_t)en[j].x * zrow), en[j].y);
        }
        run += __popc(act[j]);
      }
#pragma unroll
      for (int q = 0; q < RG; ++q)
        if (lane < pb[q + 1] - pb[q] - rc[q]) st[pb[q] + rc[q] + lane] = make_int2(0, 0);
      __syncwarp();
      // prefetch while this round is gathered: the group's next round, or the
      // next group's first round
      if (rb + kTailRound < cL) {
        fetch(rb + kTailRound);
      } else {
        setup(nms, nml);
        fetch(0);
      }
      // gather: U list slots per lane group in flight, no predication (zero padding)
#pragma unroll
      for (int q = 0; q < RG; ++q) {
        for (int p = pb[q]; p < pb[q + 1]; p += STEP) {
          float xv[U];
          float4 z[U][CPL];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int2 ev = st[p + u * NG + g];
            xv[u] = __int_as_float(ev.y);
            const float4* zp = reinterpret_cast<const float4*>(zl + (uint32_t)ev.x);
#pragma unroll
            for (int j = 0; j < CPL; ++j) z[u][j] = __ldg(zp + j * G);
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < CPL; ++j) ffma4(res[q][j], xv[u], z[u][j]);
        }
      }
      __syncwarp();
    }
    if (cL == 0) {  // empty group: the next group's first round was not fetched yet
      setup(nms, nml);
      fetch(0);
    }
    // lane groups hold partial sums of interleaved entries: reduce across groups
#pragma unroll
    for (int o = G; o < 32; o <<= 1)
#pragma unroll
      for (int q = 0; q < RG; ++q)
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          res[q][j].x += __shfl_xor_sync(kFull, res[q][j].x, o);
          res[q][j].y += __shfl_xor_sync(kFull, res[q][j].y, o);
          res[q][j].z += __shfl_xor_sync(kFull, res[q][j].z, o);
          res[q][j].w += __shfl_xor_sync(kFull, res[q][j].w, o);
        }
    if (TROW && lane < G) {
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const int c4 = lg + j * G;
        if (c4 < kq)
#pragma unroll
          for (int q = 0; q < RG; ++q)
            if (r0 + q < rows) *reinterpret_cast<float4*>(X + (r0 + q) * ldx + 4 * c4) = res[q][j];
      }
    } else if (lane < G) {
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const int c0 = 4 * (lg + j * G);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (c0 + u >= k) continue;
          float v[RG];
#pragma unroll
          for (int q = 0; q < RG; ++q)
            v[q] = u == 0 ? res[q][j].x : u == 1 ? res[q][j].y : u == 2 ? res[q][j].z : res[q][j].w;
          float* xo = X + (int64_t)(c0 + u) * ldx + r0;
          if (r0 + RG <= rows) {  // ldx and r0 are multiples of RG: aligned vector accesses
            if constexpr (RG % 4 == 0) {
#pragma unroll
              for (int q4 = 0; q4 < RG; q4 += 4)
                *reinterpret_cast<float4*>(xo + q4) = make_float4(v[q4], v[q4 + 1], v[q4 + 2], v[q4 + 3]);
            } else {
              *reinterpret_cast<float2*>(xo) = make_float2(v[0], v[1]);
            }
          } else {
#pragma unroll
            for (int q = 0; q < RG; ++q)
              if (r0 + q < rows) xo[q] = v[q];
          }
        }
      }
    }
    __syncwarp();
  }
}

}  // namespace esk

namespace esk {

// ---- narrow k (kpad <= 8: small blocks of sequential ALS, or small ranks) ----
// The V side is an SpMM with a skinny right factor: LS_V[j, :] = sum over the
// entries (i, a) of document j of a z_i with z = U W held compactly (KP floats
// per term, zc), instead of 64-byte-padded Z rows and a tensor-core head.  One
// warp per document, lanes over its entries, fixed-order warp reduction; z is
// small (4 KP n bytes, its Zipf head L1-resident), so the pass streams A^T.
template <int KP>
__global__ void __launch_bounds__(256) k_spmm_narrow(const int64_t* __restrict__ ptr, const int2* __restrict__ ent,
                                                     int64_t rows, const float* __restrict__ zc, int k,
                                                     float* __restrict__ X, int64_t ldx) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows; r += nwarps) {
    float acc[KP];
#pragma unroll
    for (int c = 0; c < KP; ++c) acc[c] = 0.f;
    for (int64_t q = ptr[r] + lane; q < ptr[r + 1]; q += 32) {
      const int2 en = __ldcs(ent + q);
      const float a = __int_as_float(en.y);
      if constexpr (KP == 1) {
        acc[0] = fmaf(a, __ldg(zc + en.x), acc[0]);
      } else {
#pragma unroll
        for (int c4 = 0; c4 < KP; c4 += 4) {
          const float4 z = __ldg(reinterpret_cast<const float4*>(zc + (int64_t)en.x * KP + c4));
          acc[c4] = fmaf(a, z.x, acc[c4]);
          acc[c4 + 1] = fmaf(a, z.y, acc[c4 + 1]);
          acc[c4 + 2] = fmaf(a, z.z, acc[c4 + 2]);
          acc[c4 + 3] = fmaf(a, z.w, acc[c4 + 3]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < KP; ++c) acc[c] = warp_sum(acc[c]);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < KP; ++c)
        if (c < k) X[(int64_t)c * ldx + r] = acc[c];
  }
}

// zc[t, :] = 0 for the terms of the previous call (before the list is rewritten) ...
__global__ void k_zc_clear(const int32_t* __restrict__ terms, const int64_t* __restrict__ count, int kp,
                           float* __restrict__ zc) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < *count * kp; q += (int64_t)gridDim.x * blockDim.x)
    zc[(int64_t)terms[q / kp] * kp + q % kp] = 0.f;
}
// ... and zc[t, :] = Z[t, 0:kp] for this call's terms
__global__ void k_zc_fill(const int32_t* __restrict__ terms, const int64_t* __restrict__ count,
                          const float* __restrict__ Z, int zs, int kp, float* __restrict__ zc) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < *count * kp; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = terms[q / kp];
    zc[t * kp + q % kp] = Z[t * zs + q % kp];
  }
}

}  // namespace esk
