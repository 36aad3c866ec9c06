// k_metrics.cuh -- relative error E and the per-iteration record.
#pragma once
#include "common.cuh"
#include "../../include/esnmf.h"

namespace esk {

// T = tr(U^T (A V)) restricted to this shard's term rows.  (A V) is recovered
// from the pre-clamp LS rows of the U side: A V = U_ls (V^T V + eps I), using
// the regularised Gram the solve used (reading C9).  part[blk] = block partial.
__global__ void __launch_bounds__(256) k_err_trace(const int64_t* __restrict__ colptr,
                                                   const int32_t* __restrict__ row, const float* __restrict__ val,
                                                   int64_t row0, int64_t rows, const float* __restrict__ XU,
                                                   int64_t ldx, const double* __restrict__ GV, const double* eps_v,
                                                   int k, double* __restrict__ part) {
  __shared__ double sm[32];
  const int c_ = blockIdx.y;
  const int64_t cb = colptr[c_], ce = colptr[c_ + 1];
  const double eps = *eps_v;
  double acc = 0;
  for (int64_t e = cb + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ce; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lr = (int64_t)row[e] - row0;
    if (lr < 0 || lr >= rows) continue;
    double s = 0;
    for (int l = 0; l < k; ++l) s += (double)XU[(int64_t)l * ldx + lr] * GV[(int64_t)l * k + c_];
    s += (double)XU[(int64_t)c_ * ldx + lr] * eps;
    acc += (double)val[e] * s;
  }
  acc = block_sum(acc, sm);
  if (threadIdx.x == 0) part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = acc;
}

// Same T, one warp per active row i of U (row view: active list + dense rows):
// lanes load the k LS values X_U[l][i] at once, then every lane forms
// s_c = sum_l X_U[l][i] (G_V + eps I)[l][c] for its columns c = lane + 32 q and
// adds U_ic s_c.  part[blk] = block partial (fixed-order reduction).
template <int CQ>
__global__ void __launch_bounds__(256) k_err_trace_rows(const int32_t* __restrict__ active,
                                                        const int64_t* __restrict__ n_active,
                                                        const float* __restrict__ dense, int kpad, int64_t row0,
                                                        int64_t rows, const float* __restrict__ XU, int64_t ldx,
                                                        const double* __restrict__ GV, const double* eps_v, int k,
                                                        double* __restrict__ part) {
  __shared__ double sm[32];
  const int lane = threadIdx.x & 31;
  const double eps = *eps_v;
  const int64_t na = *n_active;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < na; r += nwarps) {
    const int64_t lr = (int64_t)active[r] - row0;
    if (lr < 0 || lr >= rows) continue;  // warp-uniform
    double x[CQ], u[CQ];
#pragma unroll
    for (int q = 0; q < CQ; ++q) {
      const int l = lane + 32 * q;
      x[q] = l < k ? (double)XU[(int64_t)l * ldx + lr] : 0.0;
      u[q] = l < k ? (double)dense[r * kpad + l] : 0.0;
    }
    // only the columns c with U_ic != 0 contribute: s_c = sum_l x_l (G_V + eps I)[c][l]
    // (G_V symmetric: row c is contiguous), reduced over the warp in a fixed tree
#pragma unroll
    for (int qc = 0; qc < CQ; ++qc) {
      unsigned nz = __ballot_sync(kFull, u[qc] != 0.0);
      while (nz) {
        const int cl = __ffs(nz) - 1;
        nz &= nz - 1;
        const int c = 32 * qc + cl;
        const double uc = __shfl_sync(kFull, u[qc], cl);
        double p = 0;
#pragma unroll
        for (int q = 0; q < CQ; ++q) {
          const int l = lane + 32 * q;
          if (l < k) p = fma(x[q], __ldg(GV + (int64_t)c * k + l) + (l == c ? eps : 0.0), p);
        }
        p = warp_sum(p);
        acc += lane == 0 ? uc * p : 0.0;
      }
    }
  }
  acc = block_sum(acc, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// Sum of a partial array in a fixed order by one block.
__device__ double reduce_fixed(const double* p, int64_t n, int64_t stride, double* sm) {
  double s = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += p[i * stride];
  return block_sum(s, sm);
}

struct RecordInputs {
  const double* rnew;   // 2 per block: (sum (v-old)^2, sum v^2)
  int64_t nrnew;
  const double* rold;   // 1 per block
  int64_t nrold;
  const double* tpart;  // error trace partials
  int64_t ntpart;
  const double* GU;
  const double* GV;
  const int64_t* colptr_u;
  const int64_t* colptr_v;
  const int64_t* nact_u;
  const int64_t* nact_v;
  const int64_t* peak_u;  // positives of the clamped LS before truncation (per side)
  const int64_t* peak_v;
  double normA2;
  int k;
  const double* t_reduced;  // if non-null: {T, peak_u, peak_v} already summed over ranks
  // sequential ALS (Alg. 3): the record covers U = [U_1 U_2 0], V = [V_1 V_2 0]; the
  // pipeline's factors are the block (k columns), U_1 / V_1 the frozen columns
  // [0, b0) of ktot.  seqc = {T_1, S_11, ||U_1||^2}; null otherwise.
  const double* seqc = nullptr;
  const int64_t* fcolptr_u = nullptr;
  const int64_t* fcolptr_v = nullptr;
  int ktot = 0, b0 = 0;
};

// One block: R, E, counts -> rec.  Also stores (Rnum, Rden, T) into scal[0..2].
// the record goes to rec[*nrec] (then ++*nrec): the slot is found on the device,
// so a captured iteration (CUDA graph) writes the next record on every replay
__global__ void k_finalize_record(RecordInputs in, esnmf_record* __restrict__ recs, int64_t* __restrict__ nrec,
                                  double* __restrict__ scal) {
  const int64_t slot = *nrec;
  esnmf_record* rec = recs + slot;
  __shared__ double sm[32];
  const double num = reduce_fixed(in.rnew, in.nrnew, 2, sm) + reduce_fixed(in.rold, in.nrold, 1, sm);
  const double den = reduce_fixed(in.rnew + 1, in.nrnew, 2, sm);
  const double T = in.t_reduced ? *in.t_reduced : reduce_fixed(in.tpart, in.ntpart, 1, sm);
  double S = 0;
  for (int q = threadIdx.x; q < in.k * in.k; q += blockDim.x) S += in.GU[q] * in.GV[q];
  S = block_sum(S, sm);
  int dead_u = 0, dead_v = 0;
  for (int c = threadIdx.x; c < in.k; c += blockDim.x) {
    dead_u += in.colptr_u[c + 1] == in.colptr_u[c];
    dead_v += in.colptr_v[c + 1] == in.colptr_v[c];
  }
  int64_t fnnz_u = 0, fnnz_v = 0;
  double seq_T = 0, seq_S = 0, seq_N = 0;
  if (in.seqc) {
    // E^2 ||A||^2 = ||A||^2 - 2 T_1 - 2 T_2' + S_11 + S_22: the cross terms
    // 2 tr(U_1^T U_2 V_2^T V_1) of ||U V^T||^2 and of T_2 = T_2' + that (A V_2
    // recovered from the deflated LS, reading C9) cancel
    for (int c = threadIdx.x; c < in.b0; c += blockDim.x) {
      dead_u += in.fcolptr_u[c + 1] == in.fcolptr_u[c];
      dead_v += in.fcolptr_v[c + 1] == in.fcolptr_v[c];
    }
    const int future = in.ktot - in.b0 - in.k;  // blocks not started: zero columns
    if (threadIdx.x == 0) dead_u += future, dead_v += future;
    fnnz_u = in.fcolptr_u[in.ktot];
    fnnz_v = in.fcolptr_v[in.ktot];
    seq_T = in.seqc[0];
    seq_S = in.seqc[1];
    seq_N = in.seqc[2];
  }
  dead_u = (int)block_sum((double)dead_u, sm);
  dead_v = (int)block_sum((double)dead_v, sm);
  if (threadIdx.x == 0) {
    esnmf_record r;
    r.it = (int)(slot + 1);
    r.R = den + seq_N > 0 ? sqrt(num) / sqrt(den + seq_N) : -1.0;
    double e2 = in.normA2 - 2.0 * (T + seq_T) + S + seq_S;
    if (e2 < 0) e2 = 0;
    r.E = sqrt(e2) / sqrt(in.normA2);
    r.nnz_u = in.colptr_u[in.k] + fnnz_u;
    r.nnz_v = in.colptr_v[in.k] + fnnz_v;
    r.dead_u = dead_u;
    r.dead_v = dead_v;
    r.active_u = *in.nact_u;
    r.active_v = *in.nact_v;
    // multi-rank: each rank counted the positives of its own rows; the sums
    // (integers < 2^53, exact in fp64) came back with T
    const int64_t pu = in.t_reduced ? (int64_t)in.t_reduced[1] : (in.peak_u ? *in.peak_u : -1);
    const int64_t pv = in.t_reduced ? (int64_t)in.t_reduced[2] : (in.peak_v ? *in.peak_v : -1);
    r.peak_u = pu >= 0 ? pu + fnnz_u : -1;
    r.peak_v = pv >= 0 ? pv + fnnz_v : -1;
    *rec = r;
    *nrec = slot + 1;
    scal[0] = num;
    scal[1] = den;
    scal[2] = T;
  }
}

// ||A||_F^2 partials over the packed entries
__global__ void k_frob2(const int2* __restrict__ ent, int64_t nnz, double* __restrict__ part) {
  __shared__ double sm[32];
  double s = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const double v = __int_as_float(ent[e].y);
    s += v * v;
  }
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_reduce_to(const double* __restrict__ part, int64_t n, double* __restrict__ out) {
  __shared__ double sm[32];
  const double s = reduce_fixed(part, n, 1, sm);
  if (threadIdx.x == 0) *out = s;
}

// multi-rank record scalars before their allreduce: out = {T partial of this
// rank, this rank's peak_u, peak_v} (the peaks as exact fp64 integers)
__global__ void k_rank_scalars(const double* __restrict__ part, int64_t n, const int64_t* __restrict__ peak_u,
                               const int64_t* __restrict__ peak_v, double* __restrict__ out) {
  __shared__ double sm[32];
  const double s = reduce_fixed(part, n, 1, sm);
  if (threadIdx.x == 0) {
    out[0] = s;
    out[1] = peak_u ? (double)*peak_u : -1.0;
    out[2] = peak_v ? (double)*peak_v : -1.0;
  }
}

}  // namespace esk

namespace esk {

// ---- clustering accuracy, Eq. (3)-(4) (NEXT-4) ----
// cnt[(coff + c) * nJ + label[row]] += 1 for every stored entry of column c
__global__ void k_acc_count(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                            const int32_t* __restrict__ label, int nJ, int coff, double* __restrict__ cnt) {
  const int c = blockIdx.y;
  for (int64_t e = colptr[c] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < colptr[c + 1];
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[(int64_t)(coff + c) * nJ + label[row[e]]], 1.0);  // integers < 2^53: exact
}

// Acc_c = (same - alpha) / (beta - alpha); same = sum_j C(n_j, 2), alpha = q (nJ (q-1) + 2 (nD mod nJ)) / 2
// with q = floor(nD / nJ), beta = nD (nD - 1) / 2; 1 for nD <= 1 or beta == alpha
__global__ void k_acc_final(const double* __restrict__ cnt, int k, int nJ, double* __restrict__ acc) {
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    long long nD = 0, same = 0;
    for (int j = 0; j < nJ; ++j) {
      const long long x = (long long)cnt[(int64_t)c * nJ + j];
      nD += x;
      same += x * (x - 1) / 2;
    }
    const long long q = nD / nJ;
    const long long alpha = q * ((long long)nJ * (q - 1) + 2 * (nD % nJ)) / 2;
    const long long beta = nD * (nD - 1) / 2;
    acc[c] = (nD <= 1 || beta == alpha) ? 1.0 : (double)(same - alpha) / (double)(beta - alpha);
  }
}

}  // namespace esk
