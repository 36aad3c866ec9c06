/*
 * oracle/esnmf_oracle.c -- plain, slow, fp64 CPU oracle of enforced-sparse ALS.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Paper: Gavin, Gadepally, Kepner, "Enforced Sparse Non-Negative Matrix
 * Factorization" (arXiv 1510.05237), PAPER.md line numbers cited as P:n.
 *   Alg. 2: V = A^T U (U^T U)^{-1}, clamp, keep t largest;
 *                       U = A V (V^T V)^{-1},   clamp, keep t largest.
 *   Per-column enforcement: keep the t largest of EACH column.
 *   Threshold rule: t-th largest, everything below dropped.
 *   R = ||U_i - U_{i-1}|| / ||U_i||;  E = ||A - U V^T|| / ||A||.
 * Readings of silent / ambiguous points:
 *   ties at the t-th value -> exactly min(t, #positive) kept, lower row first (C4);
 *   only strictly positive entries are ever kept (C5);
 *   (G + eps I)^{-1} with eps = rho (tr G / k + 1), rho = 1e-10 (C6);
 *   Frobenius norms (C7); U_0 dense, C10 formula (C10, C11).
 *
 * Everything is fp64 (the paper's MATLAB sparse is double); the input
 * values are fp32 and are read exactly.  Factors are held DENSE (rows x k,
 * zeros where absent) because that is the most obviously correct layout.
 * Build: gcc -O2 -fopenmp -shared -fPIC
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- C10: initial guess U_0 ("initial guess U_0", undefined there) ----
 * U0[i,c] = ((splitmix64(seed ^ K_U0 ^ (i*k + c)) >> 41) + 0.5) * 2^-23
 * splitmix64 here is the standard one-step generator: z = x + golden;
 * z = (z ^ z>>30) * C1; z = (z ^ z>>27) * C2; z ^= z>>31.                   */
#define OR_K_U0 0x55305F494E495430ULL /* "U0_INIT0" */

static uint64_t or_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t or_splitmix64_pub(uint64_t x) { return or_splitmix64(x); }

void or_u0(int64_t n, int32_t k, uint64_t seed, float* out) {
  for (int64_t i = 0; i < n; ++i)
    for (int32_t c = 0; c < k; ++c) {
      uint64_t x = or_splitmix64(seed ^ OR_K_U0 ^ (uint64_t)(i * (int64_t)k + c));
      double v = ((double)(x >> 41) + 0.5) * 0x1p-23;
      out[i * (int64_t)k + c] = (float)v; /* exact: (2j+1) 2^-24 */
    }
}

/* ---- sparse initial guess (P:289-298 vary the nnz of U_0; reading C18):
 * U0[i,c] kept iff (splitmix64(seed ^ K_MASK ^ (i*k + c)) >> 11) < init_nnz 2^53 / n,
 * i.e. an independent Bernoulli(init_nnz / n) draw per entry; others 0. ---- */
#define OR_K_U0_MASK 0x55305F4D41534B30ULL /* "U0_MASK0" */
void or_u0_sparsify(int64_t n, int32_t k, uint64_t seed, int64_t init_nnz, float* U) {
  if (init_nnz <= 0) return;
  const double p = (double)init_nnz / (double)n;
  const uint64_t thr = p >= 1.0 ? UINT64_MAX : (uint64_t)(p * 0x1p53);
  for (int64_t i = 0; i < n; ++i)
    for (int32_t c = 0; c < k; ++c) {
      uint64_t x = or_splitmix64(seed ^ OR_K_U0_MASK ^ (uint64_t)(i * (int64_t)k + c));
      if ((x >> 11) >= thr) U[i * (int64_t)k + c] = 0.0f;
    }
}

/* ---- Gram matrix F^T F ("U^T U", "V^T V") ---- */
void or_gram(int64_t rows, int32_t k, const double* F, double* G) {
  for (int32_t a = 0; a < k; ++a)
    for (int32_t b = 0; b < k; ++b) G[a * k + b] = 0.0;
#pragma omp parallel
  {
    double* Gl = (double*)calloc((size_t)k * k, sizeof(double));
#pragma omp for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
      const double* f = F + i * (int64_t)k;
      for (int32_t a = 0; a < k; ++a) {
        if (f[a] == 0.0) continue;
        for (int32_t b = 0; b < k; ++b) Gl[a * k + b] += f[a] * f[b];
      }
    }
#pragma omp critical
    for (int64_t q = 0; q < (int64_t)k * k; ++q) G[q] += Gl[q];
    free(Gl);
  }
}

/* ---- ridge + Cholesky of G + eps I ("(U^T U)^{-1}"; ridge reading C6) ----
 * L lower-triangular, row-major k x k.  Returns 0, or -1 if not positive definite. */
int or_cholesky(int32_t k, const double* G, double rho, double* L, double* eps_out) {
  double tr = 0.0;
  for (int32_t a = 0; a < k; ++a) tr += G[a * k + a];
  double eps = rho * (tr / k + 1.0);
  if (eps_out) *eps_out = eps;
  memset(L, 0, sizeof(double) * (size_t)k * k);
  for (int32_t j = 0; j < k; ++j) {
    double s = G[j * k + j] + eps;
    for (int32_t p = 0; p < j; ++p) s -= L[j * k + p] * L[j * k + p];
    if (!(s > 0.0) || !isfinite(s)) return -1;
    double ljj = sqrt(s);
    L[j * k + j] = ljj;
    for (int32_t i = j + 1; i < k; ++i) {
      double v = G[i * k + j];
      for (int32_t p = 0; p < j; ++p) v -= L[i * k + p] * L[j * k + p];
      L[i * k + j] = v / ljj;
    }
  }
  return 0;
}

/* x = y (L L^T)^{-1} for a row vector y (symmetric system, two triangular solves) */
static void or_solve_row(int32_t k, const double* L, const double* y, double* x) {
  /* forward: L z = y */
  for (int32_t i = 0; i < k; ++i) {
    double s = y[i];
    for (int32_t p = 0; p < i; ++p) s -= L[i * k + p] * x[p];
    x[i] = s / L[i * k + i];
  }
  /* backward: L^T x = z */
  for (int32_t i = k - 1; i >= 0; --i) {
    double s = x[i];
    for (int32_t p = i + 1; p < k; ++p) s -= L[p * k + i] * x[p];
    x[i] = s / L[i * k + i];
  }
}

void or_solve_rows(int64_t rows, int32_t k, const double* L, const double* Y, double* X) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < rows; ++j) or_solve_row(k, L, Y + j * (int64_t)k, X + j * (int64_t)k);
}

/* ---- product Y = T F ("A^T U", "A V"); T in CSR, F dense ----
 * Row j of Y = sum over the stored (i, a) of row j of T of a * F[i, :]. */
void or_spmm(int64_t rows_out, int32_t k, const int64_t* tp, const int32_t* ti, const float* tv,
             const double* F, double* Y) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t j = 0; j < rows_out; ++j) {
    double* y = Y + j * (int64_t)k;
    for (int32_t c = 0; c < k; ++c) y[c] = 0.0;
    for (int64_t e = tp[j]; e < tp[j + 1]; ++e) {
      const double a = (double)tv[e];
      const double* f = F + (int64_t)ti[e] * k;
      for (int32_t c = 0; c < k; ++c) y[c] += a * f[c];
    }
  }
}

/* same product for a list of output rows only (sampled parity at full size) */
void or_spmm_rows(int64_t nsel, const int64_t* sel, int32_t k, const int64_t* tp, const int32_t* ti,
                  const float* tv, const double* F, double* Y) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t q = 0; q < nsel; ++q) {
    int64_t j = sel[q];
    double* y = Y + q * (int64_t)k;
    for (int32_t c = 0; c < k; ++c) y[c] = 0.0;
    for (int64_t e = tp[j]; e < tp[j + 1]; ++e) {
      const double a = (double)tv[e];
      const double* f = F + (int64_t)ti[e] * k;
      for (int32_t c = 0; c < k; ++c) y[c] += a * f[c];
    }
  }
}

/* ---- projection + per-column enforcement (P:63-64 clamp; P:134,136,146 keep
 * the t largest; P:304,387 per column).  X: rows x k dense, modified in place:
 * negatives and zeros -> 0; in every column with more than t positive entries
 * only the t largest stay, ties ordered by lower row first (C4).  t < 0 means
 * unlimited (Alg. 1).  kept[c] receives the surviving count of column c. ---- */
typedef struct { double v; int64_t row; } or_entry;

static int or_cmp_entry(const void* pa, const void* pb) {
  const or_entry* a = (const or_entry*)pa;
  const or_entry* b = (const or_entry*)pb;
  if (a->v > b->v) return -1; /* value descending */
  if (a->v < b->v) return 1;
  return (a->row < b->row) ? -1 : (a->row > b->row); /* row ascending */
}

void or_clamp_top_t(int64_t rows, int32_t k, int64_t t, double* X, int64_t* kept) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t c = 0; c < k; ++c) {
    int64_t npos = 0;
    for (int64_t j = 0; j < rows; ++j) {
      double* x = X + j * (int64_t)k + c;
      if (*x > 0.0) ++npos; else *x = 0.0; /* "set negative entries to zero" */
    }
    if (t < 0 || npos <= t) { kept[c] = npos; continue; }
    or_entry* e = (or_entry*)malloc(sizeof(or_entry) * (size_t)npos);
    int64_t q = 0;
    for (int64_t j = 0; j < rows; ++j) {
      double v = X[j * (int64_t)k + c];
      if (v > 0.0) { e[q].v = v; e[q].row = j; ++q; }
    }
    qsort(e, (size_t)npos, sizeof(or_entry), or_cmp_entry);
    for (int64_t p = t; p < npos; ++p) X[e[p].row * (int64_t)k + c] = 0.0;
    kept[c] = t;
    free(e);
  }
}

/* ---- projection + WHOLE-MATRIX enforcement: Alg. 2 as printed ("keep
 * the t_v largest values of V", P:136 for U; "find the t-th largest").
 * Negatives and zeros -> 0; if more than t entries are positive, only the t
 * largest of the whole matrix stay, ties ordered by lower column, then lower
 * row (reading C17, the column-major order of the factor).  *kept receives the
 * surviving count. ---- */
typedef struct { double v; int64_t idx; } or_entry_w;  /* idx = c * rows + j */

static int or_cmp_entry_w(const void* pa, const void* pb) {
  const or_entry_w* a = (const or_entry_w*)pa;
  const or_entry_w* b = (const or_entry_w*)pb;
  if (a->v > b->v) return -1; /* value descending */
  if (a->v < b->v) return 1;
  return (a->idx < b->idx) ? -1 : (a->idx > b->idx); /* (column, row) ascending */
}

void or_clamp_top_t_whole(int64_t rows, int32_t k, int64_t t, double* X, int64_t* kept) {
  int64_t npos = 0;
  for (int64_t q = 0; q < rows * (int64_t)k; ++q) {
    if (X[q] > 0.0) ++npos; else X[q] = 0.0;
  }
  if (t < 0 || npos <= t) { *kept = npos; return; }
  or_entry_w* e = (or_entry_w*)malloc(sizeof(or_entry_w) * (size_t)npos);
  int64_t p = 0;
  for (int32_t c = 0; c < k; ++c)
    for (int64_t j = 0; j < rows; ++j) {
      double v = X[j * (int64_t)k + c];
      if (v > 0.0) { e[p].v = v; e[p].idx = (int64_t)c * rows + j; ++p; }
    }
  qsort(e, (size_t)npos, sizeof(or_entry_w), or_cmp_entry_w);
  for (int64_t q = t; q < npos; ++q) {
    const int64_t c = e[q].idx / rows, j = e[q].idx % rows;
    X[j * (int64_t)k + c] = 0.0;
  }
  *kept = t;
  free(e);
}

/* ---- R = ||U_i - U_{i-1}||_F / ||U_i||_F by direct difference (C8) ----
 * returns -1 when ||U_i|| == 0 (degenerate). */
double or_residual(int64_t rows, int32_t k, const double* Unew, const double* Uold) {
  double num = 0.0, den = 0.0;
#pragma omp parallel for reduction(+ : num, den) schedule(static)
  for (int64_t q = 0; q < rows * (int64_t)k; ++q) {
    double d = Unew[q] - Uold[q];
    num += d * d;
    den += Unew[q] * Unew[q];
  }
  if (den == 0.0) return -1.0;
  return sqrt(num) / sqrt(den);
}

/* ---- E = ||A - U V^T||_F / ||A||_F via the trace identity (BJ:5)
 * ||A - UV^T||^2 = ||A||^2 - 2 sum(U o (A V)) + sum((U^T U) o (V^T V)).
 * AV is passed in (the U-side product), GU = U^T U, GV = V^T V. ---- */
double or_error(int64_t n, int32_t k, const double* U, const double* AV, const double* GU,
                const double* GV, double normA2) {
  double T = 0.0, S = 0.0;
#pragma omp parallel for reduction(+ : T) schedule(static)
  for (int64_t q = 0; q < n * (int64_t)k; ++q) T += U[q] * AV[q];
  for (int64_t q = 0; q < (int64_t)k * k; ++q) S += GU[q] * GV[q];
  double e2 = normA2 - 2.0 * T + S;
  if (e2 < 0.0) e2 = 0.0;
  return sqrt(e2) / sqrt(normA2);
}

double or_frob2_f32(int64_t nnz, const float* v) {
  double s = 0.0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int64_t e = 0; e < nnz; ++e) s += (double)v[e] * (double)v[e];
  return s;
}
