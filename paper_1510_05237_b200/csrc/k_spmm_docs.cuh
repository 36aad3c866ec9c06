// k_spmm_docs.cuh -- V-side product LS_V = A^T Z ("A^T U (U^T U)^{-1}"),
// Z = U (U^T U + eps I)^{-1}, one document row of A^T per warp.
//
// The kernel is bound by the L1/TEX data path (every stored entry of A^T whose
// term is active gathers a k-wide fp32 row of Z), so the layout minimises L1
// wavefronts per entry:
//  * Z is indexed by TERM (n rows, zero rows for inactive terms) with a row
//    stride of zs = 32*CPL*4 floats: a row is a whole number of 128-byte lines
//    and every lane of a group issues an unconditional, aligned 16-byte load
//    (k = 100: 4 lines per gathered row, no per-entry index lookup);
//  * activity is one bit per term in a shared-memory bitmap (n/8 bytes), so the
//    only per-entry global traffic is the packed (term, value) entry itself
//    (8 bytes, coalesced, evict-first);
//  * each warp compacts the active entries of a 32-entry batch into a per-warp
//    shared list (ballot + popc) padded with references to term 0 with value 0,
//    then walks it U entries per lane group at a time: U independent loads in
//    flight, then 4U FMAs -- branch-free.
// Results go from registers straight to the column-major LS buffer (ACCUM:
// added to the head part the tensor-core kernel stored there, k_vhead.cuh).
// Accumulation order per row is fixed by the row's entry order (deterministic).
#pragma once
#include "common.cuh"

namespace esk {

constexpr int kDocStage = 64;  // per-warp entry list: 32 entries + zero padding

// zero the Z rows of the terms listed (the previous V side's active terms)
__global__ void k_zrows_clear(const int32_t* __restrict__ terms, const int64_t* __restrict__ count,
                              float4* __restrict__ Z, int zq) {
  const int64_t cnt = *count;
  const int64_t total = cnt * zq;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q / zq;
    Z[(int64_t)terms[r] * zq + (q - r * zq)] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// term bitmap of the active rows of U (all bits cleared by the caller first)
__global__ void k_term_bits(const int32_t* __restrict__ active, const int64_t* __restrict__ n_active,
                            uint32_t* __restrict__ bits) {
  const int64_t na = *n_active;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < na; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = active[r];
    atomicOr(&bits[t >> 5], 1u << (t & 31));
  }
}

constexpr int kDocThreads = 512;  // two CTAs per SM (128 registers per thread for the 8-row results)

template <int G, int CPL, bool ACCUM>
__global__ void __launch_bounds__(kDocThreads, 2)
    k_spmm_docs(const int64_t* __restrict__ ptr, const int2* __restrict__ ent, int64_t rows,
                const uint32_t* __restrict__ tbits, int nwords, const float4* __restrict__ Z, int zq, int kq,
                int k, float* __restrict__ X, int64_t ldx) {
  // zq: Z row stride in float4; kq: float4 chunks holding the k values
  constexpr int NG = 32 / G;
  constexpr int U = 4;         // entries per lane group per step
  extern __shared__ uint32_t sbits_dyn[];              // [nwords] active-term bitmap
  __shared__ int2 stage[kDocThreads / 32][kDocStage];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / G, lg = lane % G;
  // small n: bitmap staged in shared memory; large n (nwords == 0): read via L1
  const uint32_t* sbits = nwords > 0 ? sbits_dyn : tbits;
  for (int q = threadIdx.x; q < nwords; q += blockDim.x) sbits_dyn[q] = tbits[q];
  __syncthreads();
  int2* st = stage[warp];
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // each warp produces RG consecutive rows, kept in registers, then writes
  // every LS column as one 32-byte segment (RG = 8 rows)
  constexpr int RG = CPL == 1 ? 4 : 2;
  const int64_t ngroups = (rows + RG - 1) / RG;
  for (int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; grp < ngroups; grp += nwarps) {
  float4 res[RG][CPL];
#pragma unroll 1
  for (int rr = 0; rr < RG; ++rr) {
    const int64_t row = grp * RG + rr;
    float4 acc[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t s = row < rows ? ptr[row] : 0, e = row < rows ? ptr[row + 1] : 0;
    for (int64_t base = s; base < e; base += 32) {
      const int64_t idx = base + lane;
      int2 en = make_int2(0, 0);
      bool on = false;
      if (idx < e) {
        en = __ldcs(ent + idx);  // streamed once per half-step
        on = (sbits[en.x >> 5] >> (en.x & 31)) & 1u;
      }
      const unsigned act = __ballot_sync(kFull, on);
      const int cnt = __popc(act);
      if (on) st[__popc(act & lt_mask)] = en;
      st[cnt + lane] = make_int2(0, 0);  // padding: term 0, value 0
      __syncwarp();
      for (int q0 = 0; q0 < cnt; q0 += U * NG) {
        float xv[U];
        const float4* zr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int2 ev = st[q0 + u * NG + g];
          zr[u] = Z + (size_t)(uint32_t)ev.x * (uint32_t)zq + lg;
          xv[u] = __int_as_float(ev.y);
        }
        float4 z[U][CPL];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int j = 0; j < CPL; ++j)
            z[u][j] = (lg + j * G < kq) ? __ldg(zr[u] + j * G) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int j = 0; j < CPL; ++j) {
            acc[j].x = fmaf(xv[u], z[u][j].x, acc[j].x);
            acc[j].y = fmaf(xv[u], z[u][j].y, acc[j].y);
            acc[j].z = fmaf(xv[u], z[u][j].z, acc[j].z);
            acc[j].w = fmaf(xv[u], z[u][j].w, acc[j].w);
          }
      }
      __syncwarp();
    }
#pragma unroll
    for (int o = G; o < 32; o <<= 1) {
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        acc[j].x += __shfl_xor_sync(kFull, acc[j].x, o);
        acc[j].y += __shfl_xor_sync(kFull, acc[j].y, o);
        acc[j].z += __shfl_xor_sync(kFull, acc[j].z, o);
        acc[j].w += __shfl_xor_sync(kFull, acc[j].w, o);
      }
    }
    // keep the row's result (dynamic index rr -> unrolled select keeps it in registers)
#pragma unroll
    for (int q = 0; q < RG; ++q)
      if (q == rr)
#pragma unroll
        for (int j = 0; j < CPL; ++j) res[q][j] = acc[j];
  }
  if (lane < G) {
    const int64_t r0 = grp * RG;
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int c0 = 4 * (lg + j * G);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (c0 + u >= k) continue;
        float v[RG];
#pragma unroll
        for (int q = 0; q < RG; ++q) v[q] = u == 0 ? res[q][j].x : u == 1 ? res[q][j].y : u == 2 ? res[q][j].z : res[q][j].w;
        float* xo = X + (int64_t)(c0 + u) * ldx + r0;
        if (r0 + RG <= rows) {  // ldx and r0 are multiples of RG: one aligned vector store
          if constexpr (RG == 4) {
            float4 o = make_float4(v[0], v[1], v[2], v[3]);
            if constexpr (ACCUM) {
              const float4 p = *reinterpret_cast<const float4*>(xo);
              o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
            }
            *reinterpret_cast<float4*>(xo) = o;
          } else {
            float2 o = make_float2(v[0], v[1]);
            if constexpr (ACCUM) {
              const float2 p = *reinterpret_cast<const float2*>(xo);
              o.x += p.x; o.y += p.y;
            }
            *reinterpret_cast<float2*>(xo) = o;
          }
        } else {
#pragma unroll
          for (int q = 0; q < RG; ++q)
            if (r0 + q < rows) xo[q] = ACCUM ? xo[q] + v[q] : v[q];
        }
      }
    }
  }
  }
}

}  // namespace esk
