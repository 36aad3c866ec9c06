// k_solve.cuh -- the k x k solve of Alg. 2 ("(U^T U)^{-1}") and the
// reassociated right factor Z = F W.
#pragma once
#include "common.cuh"

namespace esk {

// ---- W = (G + eps I)^{-1}, eps = rho (tr G / k + 1) (reading C6) ------
// Gauss-Jordan "sweep" of a symmetric positive definite matrix on its packed
// upper triangle: sweeping every pivot p maps A to -A^{-1}:
//   d = a_pp;  a_pp <- -1/d;  a_pj <- a_pj / d;  a_ij <- a_ij - a_ip a_pj / d.
// Pivots of an SPD matrix stay positive; a non-positive or non-finite pivot
// raises *singular.  One CTA; storage P is shared memory (k <= 224) or a
// global scratch buffer.  fp64 throughout.
ESNMF_DEV int64_t pk_idx(int i, int j, int k) {  // i <= j, packed upper, row-major
  return (int64_t)i * k - ((int64_t)i * (i - 1)) / 2 + (j - i);
}

inline bool sweep_packed(int k) { return (int64_t)k * k * 8 + k * 8 > 200 * 1024; }

// Conditioning of the solve, computed by the sweep kernel itself after W is
// written (no extra launch): kappa_inf(G + eps I) = ||G + eps I||_inf ||W||_inf and
// the column amplification max_c sum_j |W_jc| / |W_cc| (W symmetric: row sums).
// *flag = kappa > kmax || (amax > 0 && amplification > amax) || (orflag && *orflag).
// Consumers: the U side's fp32 / tensor-core (Y W) (k_uside_*; flag = use fp64) and
// the V side's paper-order tail (k_vtail.cuh; flag = Z-row gather).
struct SweepCond {
  int* flag = nullptr;          // null: not computed
  double kmax = 0, amax = 0;
  const int* orflag = nullptr;
};

__device__ void sweep_cond(const double* __restrict__ G, const double* __restrict__ W, double eps, int k,
                           const SweepCond& sc) {
  __shared__ double sg[32], sw[32], sa[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double g = 0, w = 0, amp = 0;
  for (int i = warp; i < k; i += nw) {
    double rg = 0, rw = 0;
    for (int j = lane; j < k; j += 32) {
      rg += fabs(G[(int64_t)i * k + j] + (i == j ? eps : 0.0));
      rw += fabs(W[(int64_t)i * k + j]);
    }
    rg = warp_sum(rg);
    rw = warp_sum(rw);
    g = fmax(g, rg);
    w = fmax(w, rw);
    amp = fmax(amp, rw / fabs(W[(int64_t)i * k + i]));
  }
  if (lane == 0) sg[warp] = g, sw[warp] = w, sa[warp] = amp;
  __syncthreads();
  if (threadIdx.x == 0) {
    double gm = 0, wm = 0, am = 0;
    for (int q = 0; q < nw; ++q) gm = fmax(gm, sg[q]), wm = fmax(wm, sw[q]), am = fmax(am, sa[q]);
    *sc.flag = !(gm * wm <= sc.kmax) || (sc.amax > 0 && !(am <= sc.amax)) || (sc.orflag && *sc.orflag);
  }
}

// k <= 128: the whole matrix lives in registers.  Thread (ty = warp, tx = lane)
// owns elements (i, j) = (ty + 32a, tx + 32b), a, b < JB.  Per pivot the owner
// warp of row p publishes it to shared memory (double-buffered, so one barrier
// per pivot suffices); every thread applies the rank-1 update
//   a_ij <- a_ij - (a_ip / d) a_pj
// to its whole block (which turns row p and column p into zeros) and then the
// owners of row p / column p overwrite them with a_pj / d, a_ip / d, -1 / d.
// Row blocks a with ty + 32a >= k hold only padding and are skipped (warp-
// uniform).  ~1 DFMA per element and pivot instead of a select chain.
// 1/d to full fp64 precision: hardware approximation + two Newton steps (the
// IEEE division's slow path is on the sweep's serial critical path, once per pivot)
__device__ __forceinline__ double fast_rcp(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}

template <int JB>
__global__ void __launch_bounds__(1024) k_sweep_regs(const double* __restrict__ G, int k, double rho,
                                                     double* __restrict__ W, double* __restrict__ eps_out,
                                                     int* __restrict__ singular, SweepCond sc) {
  __shared__ double vbuf[2][32 * JB];
  __shared__ double red[32];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double tr = 0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) tr += G[(int64_t)i * k + i];
  tr = block_sum(tr, red);
  const double eps = rho * (tr / k + 1.0);
  double r[JB][JB];
#pragma unroll
  for (int a = 0; a < JB; ++a)
#pragma unroll
    for (int b = 0; b < JB; ++b) {
      const int i = ty + 32 * a, j = tx + 32 * b;
      r[a][b] = (i < k && j < k) ? G[(int64_t)i * k + j] + (i == j ? eps : 0.0) : 0.0;
    }
  int na = 0;  // live row blocks of this warp
#pragma unroll
  for (int a = 0; a < JB; ++a) na += (ty + 32 * a < k);
  bool bad = false;
  for (int p = 0; p < k; ++p) {
    double* v = vbuf[p & 1];
    const int pa = p >> 5, pl = p & 31;
    if (ty == pl) {  // owner warp publishes the old row p
#pragma unroll
      for (int a = 0; a < JB; ++a)
        if (a == pa)
#pragma unroll
          for (int b = 0; b < JB; ++b) v[tx + 32 * b] = r[a][b];
    }
    __syncthreads();
    double d = v[p];
    if (!(d > 0.0) || !isfinite(d)) {
      bad = true;
      d = 1.0;
    }
    const double inv = fast_rcp(d);
    double vj[JB], vi[JB];
#pragma unroll
    for (int b = 0; b < JB; ++b) vj[b] = v[tx + 32 * b];
#pragma unroll
    for (int a = 0; a < JB; ++a) vi[a] = v[min(ty + 32 * a, 32 * JB - 1)] * inv;  // a_ip / d (symmetric)
#pragma unroll
    for (int a = 0; a < JB; ++a)
      if (a < na)
#pragma unroll
        for (int b = 0; b < JB; ++b) r[a][b] = fma(-vi[a], vj[b], r[a][b]);
    // row p: a_pj / d (and -1/d on the diagonal); column p: a_ip / d
    if (ty == pl) {
#pragma unroll
      for (int a = 0; a < JB; ++a)
        if (a == pa)
#pragma unroll
          for (int b = 0; b < JB; ++b) r[a][b] = vj[b] * inv;
    }
    if (tx == pl) {
#pragma unroll
      for (int a = 0; a < JB; ++a)
#pragma unroll
        for (int b = 0; b < JB; ++b)
          if (b == pa) r[a][b] = (ty + 32 * a == p) ? -inv : vi[a];
    }
  }
  if (bad && threadIdx.x == 0) atomicExch(singular, 1);
#pragma unroll
  for (int a = 0; a < JB; ++a)
#pragma unroll
    for (int b = 0; b < JB; ++b) {
      const int i = ty + 32 * a, j = tx + 32 * b;
      if (i < k && j < k) W[(int64_t)i * k + j] = -r[a][b];
    }
  if (threadIdx.x == 0) *eps_out = eps;
  if (sc.flag) {
    __syncthreads();  // W (global) written by the whole block
    sweep_cond(G, W, eps, k, sc);
  }
}

// 2-D thread layout (32 x 32 warps): warp ty updates rows i = ty + 32 a (so the
// row-p test is warp-uniform), lane tx columns j = tx + 32 b, b < JB, with the
// old pivot row held in registers -- ~5 instructions per element and pivot.
template <int JB, bool PACKED>
__global__ void __launch_bounds__(1024) k_sweep_inverse(const double* __restrict__ G, int k, double rho,
                                                        double* __restrict__ W, double* __restrict__ eps_out,
                                                        int* __restrict__ singular, double* gscratch, SweepCond sc) {
  extern __shared__ double dsm[];
  __shared__ double red[32];
  double* v = dsm;                              // old pivot row
  double* P = gscratch ? gscratch : dsm + k;    // full k x k, or packed upper triangle
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, nty = blockDim.x >> 5;
  auto idx = [&](int i, int j) -> int64_t {
    if (!PACKED) return (int64_t)i * k + j;
    return i <= j ? pk_idx(i, j, k) : pk_idx(j, i, k);
  };
  double tr = 0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) tr += G[(int64_t)i * k + i];
  tr = block_sum(tr, red);
  const double eps = rho * (tr / k + 1.0);
  for (int i = ty; i < k; i += nty)
    for (int j = tx; j < k; j += 32)
      if (!PACKED || j >= i) P[idx(i, j)] = G[(int64_t)i * k + j] + (i == j ? eps : 0.0);
  __syncthreads();
  for (int p = 0; p < k; ++p) {
    for (int j = threadIdx.x; j < k; j += blockDim.x) v[j] = P[idx(p, j)];
    __syncthreads();
    double d = v[p];
    if (!(d > 0.0) || !isfinite(d)) {
      if (threadIdx.x == 0) atomicExch(singular, 1);
      d = 1.0;
    }
    const double inv = fast_rcp(d);
    double vj[JB];
#pragma unroll
    for (int b = 0; b < JB; ++b) {
      const int j = tx + 32 * b;
      vj[b] = j < k ? v[j] : 0.0;
    }
    for (int i = ty; i < k; i += nty) {
      if (i == p) {  // the pivot row: a_pj <- a_pj / d, a_pp <- -1/d
#pragma unroll
        for (int b = 0; b < JB; ++b) {
          const int j = tx + 32 * b;
          if (j < k && (!PACKED || j >= i)) P[idx(i, j)] = j == p ? -inv : vj[b] * inv;
        }
      } else {
        const double vi = v[i] * inv;
#pragma unroll
        for (int b = 0; b < JB; ++b) {
          const int j = tx + 32 * b;
          if (j < k && (!PACKED || j >= i)) {
            const int64_t q = idx(i, j);
            P[q] = j == p ? vi : fma(-vi, vj[b], P[q]);
          }
        }
      }
    }
    __syncthreads();
  }
  for (int i = ty; i < k; i += nty)
    for (int j = tx; j < k; j += 32) W[(int64_t)i * k + j] = -P[idx(i, j)];
  if (threadIdx.x == 0) *eps_out = eps;
  if (sc.flag) {
    __syncthreads();
    sweep_cond(G, W, eps, k, sc);
  }
}

// ---- blocked sweep (k <= 256): the same map A -> -A^{-1}, 32 pivots at a time ----
// Sweeping the pivot set P of A = [[A_PP, A_PR], [A_RP, A_RR]] at once is the
// composition of its scalar sweeps:
//   A_PP <- -A_PP^{-1},  A_PR <- A_PP^{-1} A_PR,  A_RP <- A_PR^T A_PP^{-1},
//   A_RR <- A_RR - A_RP A_PP^{-1} A_PR.
// Per block of b <= 32 pivots: four warps sweep the b x b diagonal block D (the
// scalar sweep above, so its internal pivots are the scalar sweep's and an SPD
// matrix keeps them positive), giving D^{-1}; the CTA forms C = D^{-1} A_PR and the
// symmetric rank-b update A_RR -= A_PR^T C on its upper triangle, both as 4 x 4
// register tiles per thread (fp64 FMA).  ~k^3 / 2 FMAs behind ~4 k / 32 barriers,
// against k^3 FMAs behind k barriers.  A keeps only its upper triangle (the map
// preserves symmetry); it lives in shared memory when it fits, else in the global
// scratch (L2-resident).  fp64 throughout.
constexpr int kBsThreads = 512;

ESNMF_DEV int bs_ld(int k) { return ((k + 31) / 32) * 32; }  // panel row stride (padded R)

inline size_t bsweep_smem_bytes(int k, bool* a_in_smem) {
  const size_t ld = (size_t)((k + 31) / 32) * 32;
  size_t b = sizeof(double) * (32 * 32 + 2 * 32 * ld);
  const bool fit = b + sizeof(double) * (size_t)k * k <= 220 * 1024;
  if (a_in_smem) *a_in_smem = fit;
  return fit ? b + sizeof(double) * (size_t)k * k : b;
}

__global__ void __launch_bounds__(kBsThreads) k_sweep_blocked(const double* __restrict__ G, int k, double rho,
                                                              double* __restrict__ W, double* __restrict__ eps_out,
                                                              int* __restrict__ singular, double* gscratch,
                                                              SweepCond sc) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ double red[32];
  __shared__ double Drow[2 * 32];
  const int ld = bs_ld(k);
  double* Dinv = dsm;           // 32 x 32 (symmetric)
  double* AP = Dinv + 32 * 32;  // 32 x ld: rows P of A, columns R (compact index r)
  double* Cp = AP + 32 * ld;    // 32 x ld: D^{-1} A_PR
  double* A = gscratch ? gscratch : Cp + 32 * ld;
  ESNMF_CHECK(k <= 256 && (size_t)(32 * 32 + 2 * 32 * ld + (gscratch ? 0 : k * k)) * 8 <= dyn_smem_bytes());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  auto up = [k](int i, int j) -> int64_t { return i <= j ? (int64_t)i * k + j : (int64_t)j * k + i; };
  double tr = 0;
  for (int i = tid; i < k; i += blockDim.x) tr += G[(int64_t)i * k + i];
  tr = block_sum(tr, red);
  const double eps = rho * (tr / k + 1.0);
  for (int i = warp; i < k; i += nw)
    for (int j = lane; j < k; j += 32) A[(int64_t)i * k + j] = G[(int64_t)i * k + j] + (i == j ? eps : 0.0);
  __syncthreads();
  bool bad = false;
#pragma unroll 1
  for (int p0 = 0; p0 < k; p0 += 32) {
    const int b = min(32, k - p0), nr = k - b;
    auto ridx = [p0, b](int r) { return r < p0 ? r : r + b; };
    if (warp < 4) {  // D^{-1}: the scalar sweep of D (padded with the identity) by 4 warps
      // Thread (warp w, lane j) holds d_ij for rows i = 8w + u in registers.  Per
      // pivot the owner warp publishes row q (double-buffered, one 128-thread named
      // barrier per pivot); D stays symmetric, so column q (d_iq) is row q.
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = warp * 8 + u;
        x[u] = (i < b && lane < b) ? A[up(p0 + i, p0 + lane)] : (i == lane ? 1.0 : 0.0);
      }
#pragma unroll 1
      for (int qb = 0; qb < b; qb += 8) {
#pragma unroll
        for (int uq = 0; uq < 8; ++uq) {  // pivot q = qb + uq: its row is register uq of warp qb / 8
          const int q = qb + uq;
          if (q < b) {  // block-uniform
            double* row = Drow + (q & 1) * 32;
            if (warp == (qb >> 3)) row[lane] = x[uq];
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const double rq = row[lane];  // d_qj
            double d = row[q];
            if (!(d > 0.0) || !isfinite(d)) {
              bad = true;
              d = 1.0;
            }
            const double inv = fast_rcp(d);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int i = warp * 8 + u;
              const double ci = row[i] * inv;  // d_iq / d
              x[u] = i == q ? (lane == q ? -inv : rq * inv) : (lane == q ? ci : fma(-ci, rq, x[u]));
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) Dinv[(warp * 8 + u) * 32 + lane] = -x[u];
    }
    for (int q = warp; q < 32; q += nw)
      for (int r = lane; r < ld; r += 32) AP[q * ld + r] = (q < b && r < nr) ? A[up(p0 + q, ridx(r))] : 0.0;
    __syncthreads();
    // C = D^{-1} A_PR: thread tile rows q0..q0+3 x columns r0..r0+3 (D^{-1} symmetric:
    // its column s is row s, read as two 16-byte vectors)
    for (int t = tid; t < 8 * (ld / 4); t += blockDim.x) {
      const int q0 = (t & 7) * 4, r0 = (t >> 3) * 4;
      double acc[4][4] = {};
#pragma unroll 4
      for (int s2 = 0; s2 < b; ++s2) {
        const double2 d01 = *reinterpret_cast<const double2*>(Dinv + s2 * 32 + q0);
        const double2 d23 = *reinterpret_cast<const double2*>(Dinv + s2 * 32 + q0 + 2);
        const double2 a01 = *reinterpret_cast<const double2*>(AP + s2 * ld + r0);
        const double2 a23 = *reinterpret_cast<const double2*>(AP + s2 * ld + r0 + 2);
        const double dv[4] = {d01.x, d01.y, d23.x, d23.y}, av[4] = {a01.x, a01.y, a23.x, a23.y};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(dv[u], av[v], acc[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        *reinterpret_cast<double2*>(Cp + (q0 + u) * ld + r0) = make_double2(acc[u][0], acc[u][1]);
        *reinterpret_cast<double2*>(Cp + (q0 + u) * ld + r0 + 2) = make_double2(acc[u][2], acc[u][3]);
      }
    }
    __syncthreads();
    // A_RR -= A_PR^T C on the upper triangle: warp tiles of 16 rows x 32 columns
    const int ti_n = (nr + 15) / 16, tj_n = (nr + 31) / 32;
    const int ly = lane >> 3, lx = lane & 7;
    for (int t = warp; t < ti_n * tj_n; t += nw) {
      const int ti = t / tj_n, tj = t - ti * tj_n;
      if (ti * 16 > tj * 32 + 31) continue;  // strictly below the diagonal (warp-uniform)
      const int i0 = ti * 16 + ly * 4, j0 = tj * 32 + lx * 4;
      double acc[4][4] = {};
#pragma unroll 4
      for (int q = 0; q < b; ++q) {
        const double2 a01 = *reinterpret_cast<const double2*>(AP + q * ld + i0);
        const double2 a23 = *reinterpret_cast<const double2*>(AP + q * ld + i0 + 2);
        const double2 c01 = *reinterpret_cast<const double2*>(Cp + q * ld + j0);
        const double2 c23 = *reinterpret_cast<const double2*>(Cp + q * ld + j0 + 2);
        const double av[4] = {a01.x, a01.y, a23.x, a23.y}, cv[4] = {c01.x, c01.y, c23.x, c23.y};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], cv[v], acc[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u;
        if (i >= nr) continue;
        double* arow = A + (int64_t)ridx(i) * k;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int j = j0 + v;
          if (i <= j && j < nr) arow[ridx(j)] -= acc[u][v];
        }
      }
    }
    // rows / columns P: C (upper-triangle position) and -D^{-1}; disjoint from A_RR
    for (int q = warp; q < b; q += nw) {
      for (int r = lane; r < nr; r += 32) A[up(p0 + q, ridx(r))] = Cp[q * ld + r];
      if (lane >= q && lane < b) A[(int64_t)(p0 + q) * k + p0 + lane] = -Dinv[q * 32 + lane];
    }
    __syncthreads();
  }
  if (bad) atomicExch(singular, 1);
  for (int i = warp; i < k; i += nw)
    for (int j = lane; j < k; j += 32) W[(int64_t)i * k + j] = -A[up(i, j)];
  if (tid == 0) *eps_out = eps;
  if (sc.flag) {
    __syncthreads();
    sweep_cond(G, W, eps, k, sc);
  }
}

inline size_t sweep_smem_bytes(int k, bool global_scratch) {
  size_t b = sizeof(double) * (size_t)k;
  if (!global_scratch)
    b += sweep_packed(k) ? sizeof(double) * (size_t)k * (k + 1) / 2 : sizeof(double) * (size_t)k * k;
  return b;
}

// ---- Z = F W for the active rows of the factor (fp64 accumulate, fp32 out) ----
// The LS rows of a half-step are T (F W): the product with A^T (or A) is
// reassociated onto Z (identical to (T F) W up to rounding).
// One warp per active row; lanes own columns c = lane + 32 j.
// Z row of active row r is written at Z[active[r] * zs] (term-indexed, stride
// zs >= kpad floats, zero padded); zlist/zcount record the rows written so the
// next call can zero them first (k_zrows_clear).
template <int CJ>
__global__ void __launch_bounds__(256) k_form_z(const float* __restrict__ dense, int kpad, int k,
                                                const int64_t* __restrict__ n_active,
                                                const int32_t* __restrict__ active, int zs,
                                                const double* __restrict__ W, float* __restrict__ Z,
                                                int32_t* __restrict__ zlist, int64_t* __restrict__ zcount,
                                                const int* __restrict__ gate) {
  if (gate && !*gate) return;  // (k_spmm_tail.cuh: the Z-row gather runs only when gated on)
  const int lane = threadIdx.x & 31;
  const int64_t na = *n_active;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp0; r < na; r += nwarps) {
    float f[CJ];
#pragma unroll
    for (int j = 0; j < CJ; ++j) {
      int c = lane + 32 * j;
      f[j] = c < kpad ? dense[r * kpad + c] : 0.f;
    }
    double acc[CJ];
#pragma unroll
    for (int j = 0; j < CJ; ++j) acc[j] = 0.0;
#pragma unroll
    for (int jl = 0; jl < CJ; ++jl) {
      const int lmax = min(32, k - 32 * jl);
      for (int ll = 0; ll < lmax; ++ll) {
        const float fl = __shfl_sync(kFull, f[jl], ll);
        if (fl != 0.f) {
          const int l = 32 * jl + ll;
#pragma unroll
          for (int j = 0; j < CJ; ++j) {
            int c = lane + 32 * j;
            if (c < k) acc[j] += (double)fl * W[(int64_t)l * k + c];
          }
        }
      }
    }
    const int32_t term = active[r];
    float* zr = Z + (int64_t)term * zs;
#pragma unroll
    for (int j = 0; j < CJ; ++j) {
      int c = lane + 32 * j;
      if (c < zs) zr[c] = c < k ? (float)acc[j] : 0.f;
    }
    for (int c = lane + 32 * CJ; c < zs; c += 32) zr[c] = 0.f;
    if (lane == 0) zlist[r] = term;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *zcount = na;
}

}  // namespace esk
