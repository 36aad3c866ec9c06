// k_factor.cuh -- factor storage kernels: U_0, row view, Gram, residual.
//
// A factor (U: n x k, V: m x k) is held as
//   * canonical column-major COO (colptr[k+1], row[], val[]) -- the paper's
//     sparse factor, at most t entries per column;
//   * a row view: rowmap[rows] (active index or -1), active[] (ascending rows),
//     and dense[n_active][kpad] fp32 rows (zeros where absent), which the
//     SpMM gathers and the Gram reads.
#pragma once
#include "common.cuh"

namespace esk {

// ---- U_0 ("initial guess U_0"; reading C10) -------------------------
// U0[i,c] = ((splitmix64(seed ^ K_U0 ^ (i*k + c)) >> 41) + 0.5) * 2^-23: an
// odd multiple of 2^-24 in (0,1), exact in fp32.  splitmix64 = one step of the
// standard generator from state x.
constexpr uint64_t kU0Stream = 0x55305F494E495430ULL;  // "U0_INIT0"

ESNMF_DEV uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void k_u0_dense(int64_t n, int k, int kpad, uint64_t seed, const float* __restrict__ user,
                           float* __restrict__ dense, int* __restrict__ bad) {
  int64_t total = n * kpad;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = q / kpad;
    int c = (int)(q - i * kpad);
    float v = 0.f;
    if (c < k) {
      if (user) {
        v = user[i * k + c];
        if (!(v > 0.f) || !isfinite(v)) atomicExch(bad, 1);
      } else {
        uint64_t x = splitmix64(seed ^ kU0Stream ^ (uint64_t)(i * k + c));
        v = (float)(((double)(x >> 41) + 0.5) * 0x1p-23);
      }
    }
    dense[q] = v;
  }
}

// sparse initial guess (reading C18): zero U0[i,c] unless the mask hash draw
// (splitmix64(seed ^ K_MASK ^ (i*k + c)) >> 11) < thr = init_nnz 2^53 / n
constexpr uint64_t kU0Mask = 0x55305F4D41534B30ULL;  // "U0_MASK0"

__global__ void k_u0_mask(int64_t n, int k, int kpad, uint64_t seed, uint64_t thr, float* __restrict__ dense) {
  const int64_t total = n * k;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / k;
    const int c = (int)(q - i * k);
    if ((splitmix64(seed ^ kU0Mask ^ (uint64_t)q) >> 11) >= thr) dense[i * kpad + c] = 0.f;
  }
}

// compact the (masked) dense U_0 into canonical column-major COO: one block per
// column, rows in order (block scan over chunks of blockDim rows).  Pass 1
// (colptr == nullptr) counts into ccount[c]; pass 2 writes at colptr[c].
__global__ void k_u0_compact(int64_t n, int k, int kpad, const float* __restrict__ dense,
                             int64_t* __restrict__ ccount, const int64_t* __restrict__ colptr,
                             int32_t* __restrict__ row, float* __restrict__ val) {
  __shared__ int64_t sm[33];
  const int c = blockIdx.x;
  int64_t base = 0;
  for (int64_t i0 = 0; i0 < n; i0 += blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const float v = i < n ? dense[i * kpad + c] : 0.f;
    const int64_t on = v > 0.f;
    int64_t tot;
    const int64_t ex = block_exscan(on, sm, &tot);
    if (on && colptr) {
      row[colptr[c] + base + ex] = (int32_t)i;
      val[colptr[c] + base + ex] = v;
    }
    base += tot;
  }
  if (threadIdx.x == 0 && !colptr) ccount[c] = base;
}

// every entry of the dense U_0 is stored (all are > 0)
__global__ void k_u0_coo(int64_t n, int k, int kpad, const float* __restrict__ dense, int64_t* __restrict__ colptr,
                         int32_t* __restrict__ row, float* __restrict__ val, int32_t* __restrict__ rowmap,
                         int32_t* __restrict__ active, int64_t* __restrict__ n_active) {
  int64_t total = n * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = e / n, i = e - c * n;
    row[e] = (int32_t)i;
    val[e] = dense[i * kpad + c];
    if (c == 0) {
      rowmap[i] = (int32_t)i;
      active[i] = (int32_t)i;
    }
    if (e <= k) colptr[e] = e * n;
    if (e == 0) *n_active = n;
  }
}

// ---- row view maintenance ---------------------------------------------------
// Column-parallel launch: grid.y = column, grid.x strides over its entries.
#define ESNMF_FOR_COL_ENTRIES(colptr, e)                                                           \
  const int c_ = blockIdx.y;                                                                       \
  const int64_t cb_ = colptr[c_], ce_ = colptr[c_ + 1];                                            \
  for (int64_t e = cb_ + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ce_;                   \
       e += (int64_t)gridDim.x * blockDim.x)

// factor entries -> column-major dense buffer X[c * ldx + row] (zeroed by the caller)
__global__ void k_coo_to_colmajor(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                                  const float* __restrict__ val, float* __restrict__ X, int64_t ldx) {
  ESNMF_FOR_COL_ENTRIES(colptr, e) { X[(int64_t)c_ * ldx + row[e]] = val[e]; }
}

// zero the dense cells of the factor's current entries (before it is replaced)
__global__ void k_clear_dense(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                              const int32_t* __restrict__ rowmap, float* __restrict__ dense, int kpad) {
  ESNMF_FOR_COL_ENTRIES(colptr, e) {
    int32_t r = rowmap[row[e]];
    if (r >= 0) dense[(int64_t)r * kpad + c_] = 0.f;
  }
}

__global__ void k_reset_rowmap(const int32_t* __restrict__ active, const int64_t* __restrict__ n_active,
                               int32_t* __restrict__ rowmap) {
  int64_t na = *n_active;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < na; r += (int64_t)gridDim.x * blockDim.x)
    rowmap[active[r]] = -1;
}

__global__ void k_mark_rows(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                            int32_t* __restrict__ rowmap) {
  ESNMF_FOR_COL_ENTRIES(colptr, e) { rowmap[row[e]] = 0; }
}

constexpr int kRowBlock = 2048;  // rows per compaction block (256 threads x 8)

__global__ void k_rows_count(const int32_t* __restrict__ rowmap, int64_t rows, int64_t* __restrict__ bcount) {
  __shared__ int64_t sm[32];
  int64_t base = blockIdx.x * (int64_t)kRowBlock;
  int64_t cnt = 0;
  for (int q = threadIdx.x; q < kRowBlock; q += blockDim.x) {
    int64_t i = base + q;
    if (i < rows && rowmap[i] >= 0) cnt += 1;
  }
  cnt = block_sum(cnt, sm);
  if (threadIdx.x == 0) bcount[blockIdx.x] = cnt;
}

// in-place exclusive scan of nb int64 with one block; total -> *total
__global__ void k_scan_small(int64_t* __restrict__ a, int64_t nb, int64_t* __restrict__ total) {
  __shared__ int64_t sm[33];
  int64_t carry = 0;
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < nb ? a[i] : 0;
    int64_t tot;
    int64_t ex = block_exscan(v, sm, &tot);
    if (i < nb) a[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void k_rows_assign(int32_t* __restrict__ rowmap, int64_t rows, const int64_t* __restrict__ boff,
                              int32_t* __restrict__ active) {
  __shared__ int64_t sm[33];
  constexpr int per = kRowBlock / 256;
  int64_t base = blockIdx.x * (int64_t)kRowBlock + threadIdx.x * per;
  int64_t cnt = 0;
#pragma unroll
  for (int q = 0; q < per; ++q) {
    int64_t i = base + q;
    cnt += (i < rows && rowmap[i] >= 0);
  }
  int64_t tot;
  int64_t off = boff[blockIdx.x] + block_exscan(cnt, sm, &tot);
#pragma unroll
  for (int q = 0; q < per; ++q) {
    int64_t i = base + q;
    if (i < rows && rowmap[i] >= 0) {
      rowmap[i] = (int32_t)off;
      active[off] = (int32_t)i;
      ++off;
    }
  }
}

__global__ void k_scatter_dense(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                                const float* __restrict__ val, const int32_t* __restrict__ rowmap,
                                float* __restrict__ dense, int kpad) {
  ESNMF_FOR_COL_ENTRIES(colptr, e) { dense[(int64_t)rowmap[row[e]] * kpad + c_] = val[e]; }
}

// ---- Gram matrix G = F^T F in fp64 ("U^T U", "V^T V") -----------
// G[a][b] = sum over the entries (i, u) of column a of u * F[i][b], with F[i]
// read from the dense row view.  grid = (k columns a, S segments); a block is
// ng groups of gb >= k threads (thread b of a group owns G[a][b]), the groups
// splitting the segment's entries (long columns -- whole-factor enforcement
// can put 10^5 entries in one -- are otherwise one long dependent loop);
// group sums and segment partials are added in a fixed order (k_gram_reduce):
// deterministic.
__global__ void __launch_bounds__(512) k_gram_partial_groups(const int64_t* __restrict__ colptr,
                                                      const int32_t* __restrict__ row,
                                                      const float* __restrict__ val,
                                                      const int32_t* __restrict__ rowmap,
                                                      const float* __restrict__ dense, int kpad, int k,
                                                      int64_t seglen, double* __restrict__ partial, int gb) {
  __shared__ double red[512];
  const int a = blockIdx.x, s = blockIdx.y;
  const int ng = blockDim.x / gb, g = threadIdx.x / gb, b = threadIdx.x - g * gb;
  const int64_t cb = colptr[a], ce = colptr[a + 1];
  const int64_t s0 = cb + (int64_t)s * seglen;
  const int64_t s1 = min(ce, s0 + seglen);
  const int64_t sub = (max(s1 - s0, (int64_t)0) + ng - 1) / ng;
  const int64_t b0 = s0 + g * sub, b1 = min(s1, b0 + sub);
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  if (b < k) {
    int64_t e = b0;
    for (; e + 4 <= b1; e += 4) {
      float u0 = val[e], u1 = val[e + 1], u2 = val[e + 2], u3 = val[e + 3];
      int32_t r0 = rowmap[row[e]], r1 = rowmap[row[e + 1]], r2 = rowmap[row[e + 2]], r3 = rowmap[row[e + 3]];
      acc0 += (double)u0 * (double)dense[(int64_t)r0 * kpad + b];
      acc1 += (double)u1 * (double)dense[(int64_t)r1 * kpad + b];
      acc2 += (double)u2 * (double)dense[(int64_t)r2 * kpad + b];
      acc3 += (double)u3 * (double)dense[(int64_t)r3 * kpad + b];
    }
    for (; e < b1; ++e) acc0 += (double)val[e] * (double)dense[(int64_t)rowmap[row[e]] * kpad + b];
  }
  red[threadIdx.x] = (acc0 + acc1) + (acc2 + acc3);
  __syncthreads();
  if (g == 0 && b < k) {
    double t = red[b];
    for (int q = 1; q < ng; ++q) t += red[q * gb + b];
    partial[((int64_t)s * k + a) * k + b] = t;
  }
}

// short segments (every column of a per-column factor): thread b owns G[a][b]
__global__ void __launch_bounds__(256) k_gram_partial(const int64_t* __restrict__ colptr,
                                                      const int32_t* __restrict__ row,
                                                      const float* __restrict__ val,
                                                      const int32_t* __restrict__ rowmap,
                                                      const float* __restrict__ dense, int kpad, int k,
                                                      int64_t seglen, double* __restrict__ partial) {
  const int a = blockIdx.x, s = blockIdx.y;
  const int64_t cb = colptr[a], ce = colptr[a + 1];
  const int64_t b0 = cb + (int64_t)s * seglen;
  const int64_t b1 = min(ce, b0 + seglen);
  for (int b = threadIdx.x; b < k; b += blockDim.x) {
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    int64_t e = b0;
    for (; e + 4 <= b1; e += 4) {
      float u0 = val[e], u1 = val[e + 1], u2 = val[e + 2], u3 = val[e + 3];
      int32_t r0 = rowmap[row[e]], r1 = rowmap[row[e + 1]], r2 = rowmap[row[e + 2]], r3 = rowmap[row[e + 3]];
      acc0 += (double)u0 * (double)dense[(int64_t)r0 * kpad + b];
      acc1 += (double)u1 * (double)dense[(int64_t)r1 * kpad + b];
      acc2 += (double)u2 * (double)dense[(int64_t)r2 * kpad + b];
      acc3 += (double)u3 * (double)dense[(int64_t)r3 * kpad + b];
    }
    for (; e < b1; ++e) acc0 += (double)val[e] * (double)dense[(int64_t)rowmap[row[e]] * kpad + b];
    partial[((int64_t)s * k + a) * k + b] = (acc0 + acc1) + (acc2 + acc3);
  }
}

// Dense variant (a factor whose columns are long, e.g. the dense U_0 of
// iteration 1): the same upper-triangle partials straight from the dense active
// rows, G_ab = sum_r D_ra D_rb (zeros of D contribute nothing; fp32 products are
// exact in fp64).  Grid (S, nb, nb): slab s of the active rows, output block
// (bi, bj) of 128 x 128 (bi <= bj); 256 threads, an 8 x 8 fp64 register tile each,
// rows staged 32 at a time in shared memory.
constexpr int kGdRows = 32;
__global__ void __launch_bounds__(256) k_gram_dense(const float* __restrict__ dense, int kpad, int k,
                                                    const int64_t* __restrict__ n_active, double* __restrict__ partial) {
  const int bi = blockIdx.y, bj = blockIdx.z;
  if (bi > bj) return;
  __shared__ __align__(16) float sa[kGdRows][128], sb[kGdRows][128];
  const int S = gridDim.x, s = blockIdx.x;
  const int64_t na = *n_active;
  const int64_t len = (na + S - 1) / S;
  const int64_t r0 = (int64_t)s * len, r1 = min(na, r0 + len);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i0 = bi * 128 + ty * 8, j0 = bj * 128 + tx * 8;
  const bool live = i0 <= j0 + 7 && i0 < k && j0 < k;  // tile touches the upper triangle
  double acc[8][8];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[u][v] = 0.0;
  for (int64_t rb = r0; rb < r1; rb += kGdRows) {
    __syncthreads();
    for (int e = threadIdx.x; e < kGdRows * 128; e += blockDim.x) {
      const int rr = e >> 7, c = e & 127;
      const int64_t r = rb + rr;
      const int ca = bi * 128 + c, cb = bj * 128 + c;
      sa[rr][c] = (r < r1 && ca < kpad) ? dense[r * kpad + ca] : 0.f;
      sb[rr][c] = (r < r1 && cb < kpad) ? dense[r * kpad + cb] : 0.f;
    }
    __syncthreads();
    if (live) {
      const int nr = (int)min((int64_t)kGdRows, r1 - rb);
      for (int rr = 0; rr < nr; ++rr) {
        const float4 a0 = *reinterpret_cast<const float4*>(&sa[rr][ty * 8]);
        const float4 a1 = *reinterpret_cast<const float4*>(&sa[rr][ty * 8 + 4]);
        const float4 b0 = *reinterpret_cast<const float4*>(&sb[rr][tx * 8]);
        const float4 b1 = *reinterpret_cast<const float4*>(&sb[rr][tx * 8 + 4]);
        const double a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const double b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int v = 0; v < 8; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int i = i0 + u, j = j0 + v;
      if (i <= j && j < k) partial[((int64_t)s * k + i) * k + j] = acc[u][v];
    }
}

// G[i][j] = G[j][i] = the segment sum of the upper-triangle partial (i <= j):
// both halves are the same sum, so G is exactly symmetric
__global__ void k_gram_reduce(const double* __restrict__ partial, int S, int k, double* __restrict__ G) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= k * k) return;
  const int i = q / k, j = q - i * k;
  const int64_t u = (int64_t)min(i, j) * k + max(i, j);
  double s = 0;
  for (int t = 0; t < S; ++t) s += partial[(int64_t)t * k * k + u];
  G[q] = s;
}


// ---- residual R = ||U_i - U_{i-1}||_F / ||U_i||_F, direct difference ----
// part[2*blk] += sum over new entries (v - old)^2, part[2*blk+1] += v^2
__global__ void k_resid_new(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                            const float* __restrict__ val, const int32_t* __restrict__ rowmap_old,
                            const float* __restrict__ dense_old, int kpad, double* __restrict__ part) {
  __shared__ double sm[32];
  double num = 0, den = 0;
  ESNMF_FOR_COL_ENTRIES(colptr, e) {
    double v = val[e];
    int32_t r = rowmap_old[row[e]];
    double o = r >= 0 ? (double)dense_old[(int64_t)r * kpad + c_] : 0.0;
    num += (v - o) * (v - o);
    den += v * v;
  }
  num = block_sum(num, sm);
  den = block_sum(den, sm);
  if (threadIdx.x == 0) {
    int64_t b = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
    part[2 * b] = num;
    part[2 * b + 1] = den;
  }
}

// part[blk] = sum over old entries that are absent from the new factor of v_old^2
__global__ void k_resid_old(const int64_t* __restrict__ colptr, const int32_t* __restrict__ row,
                            const float* __restrict__ val, const int32_t* __restrict__ rowmap_new,
                            const float* __restrict__ dense_new, int kpad, double* __restrict__ part) {
  __shared__ double sm[32];
  double s = 0;
  ESNMF_FOR_COL_ENTRIES(colptr, e) {
    int32_t r = rowmap_new[row[e]];
    bool present = r >= 0 && dense_new[(int64_t)r * kpad + c_] != 0.f;  // kept entries are > 0
    if (!present) s += (double)val[e] * (double)val[e];
  }
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
}

}  // namespace esk
