/*
 * synth/zipfgen.c -- seeded synthetic term/document matrices (CPU side).
 *
 * INPUT GENERATION ONLY.  This module holds none of the method's arithmetic;
 * it is shared, as data, by the fp64 oracle (oracle/) and by the CUDA path
 * (paper_1510_05237_b200/).  synth/zipfgen_cuda.cu implements the same
 * counter-based recipe on the GPU; tests check the two are bitwise equal.
 *
 * Recipe (BASELINE.json configs; stands in for the paper's
 * Reuters / Wikipedia / PubMed term-document matrices):
 *   for every document j (a column of A, a row of A^T):
 *     draw q = 0,1,2,...: u = top-53-bits(hash(seed, TERM, j, q)) * 2^-53,
 *       term = upper_bound(cdf, u)       (Zipf(s) rank, 0-based)
 *       rejected if already in the document, until d distinct terms;
 *     terms sorted ascending;
 *     value(j, i) = interp(vtab, hash(seed, VAL, j, i))  -- lognormal(0,sigma)
 *       quantile table, linear interpolation in fp64 with explicitly ordered
 *       IEEE operations (no FMA contraction), rounded once to fp32.
 *   cdf[] and vtab[] are built once on the host by synth/__init__.py and are
 *   passed to BOTH generators, so the two agree bit for bit.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ZG_STREAM_TERM 1ULL
#define ZG_STREAM_VAL 2ULL

static inline uint64_t zg_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t zg_hash(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
  uint64_t h = zg_mix64(seed + 0x9E3779B97F4A7C15ULL * (stream + 1ULL));
  h = zg_mix64(h ^ (a * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL));
  h = zg_mix64(h ^ (b * 0xABC98388FB8FAC03ULL + 0x8CB92BA72F3D8DD7ULL));
  return h;
}

/* first index r in [0,n) with cdf[r] > u; cdf[n-1] == 1.0 and u < 1 */
static inline int64_t zg_upper_bound(const double* cdf, int64_t n, double u) {
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    int64_t mid = lo + ((hi - lo) >> 1);
    if (cdf[mid] > u) hi = mid; else lo = mid + 1;
  }
  return lo;
}

float zg_value(uint64_t seed, int64_t doc, int64_t term, const double* vtab) {
  uint64_t x = zg_hash(seed, ZG_STREAM_VAL, (uint64_t)doc, (uint64_t)term);
  uint32_t idx = (uint32_t)(x >> 48);                       /* 0..65535 */
  double f = (double)(uint32_t)((x >> 16) & 0xFFFFFFFFULL) * 0x1p-32;
  double lo = vtab[idx];
  double dv = vtab[idx + 1] - lo;   /* separate IEEE ops, no contraction */
  double t2 = dv * f;
  double v = lo + t2;
  return (float)v;
}

/*
 * Generates CSR(A^T): m document rows, each with exactly d distinct term ids
 * (sorted ascending) in [0,n).  at_col, at_val: m*d entries (row j occupies
 * [j*d, (j+1)*d)).  Returns 0, or -1 on invalid arguments.
 */
int zg_generate_at(int64_t n, int64_t m, int32_t d, uint64_t seed,
                   const double* cdf, const double* vtab,
                   int32_t* at_col, float* at_val) {
  if (n <= 0 || m <= 0 || d <= 0 || (int64_t)d * 2 > n) return -1;
  int failed = 0;
#pragma omp parallel
  {
    unsigned char* mark = (unsigned char*)calloc((size_t)n, 1);
    if (!mark) {
#pragma omp atomic write
      failed = 1;
    }
#pragma omp for schedule(dynamic, 256)
    for (int64_t j = 0; j < m; ++j) {
      if (!mark) continue;
      int32_t* row = at_col + j * (int64_t)d;
      int32_t cnt = 0;
      uint64_t q = 0;
      while (cnt < d) {
        uint64_t x = zg_hash(seed, ZG_STREAM_TERM, (uint64_t)j, q++);
        double u = (double)(x >> 11) * 0x1p-53;
        int64_t r = zg_upper_bound(cdf, n, u);
        if (!mark[r]) { mark[r] = 1; row[cnt++] = (int32_t)r; }
      }
      /* insertion sort (d <= a few hundred) */
      for (int32_t a = 1; a < d; ++a) {
        int32_t key = row[a], b = a - 1;
        while (b >= 0 && row[b] > key) { row[b + 1] = row[b]; --b; }
        row[b + 1] = key;
      }
      for (int32_t a = 0; a < d; ++a) {
        mark[row[a]] = 0;
        at_val[j * (int64_t)d + a] = zg_value(seed, j, row[a], vtab);
      }
    }
    free(mark);
  }
  return failed ? -1 : 0;
}

/*
 * Stable counting-sort transpose: CSR(A^T) (m rows over n columns) ->
 * CSR(A) (n rows over m columns).  Rows of A list documents ascending.
 */
int zg_transpose(int64_t n, int64_t m, const int64_t* at_ptr,
                 const int32_t* at_col, const float* at_val,
                 int64_t* a_ptr, int32_t* a_col, float* a_val) {
  int64_t nnz = at_ptr[m];
  memset(a_ptr, 0, sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t e = 0; e < nnz; ++e) a_ptr[at_col[e] + 1]++;
  for (int64_t i = 0; i < n; ++i) a_ptr[i + 1] += a_ptr[i];
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  if (!cur) return -1;
  memcpy(cur, a_ptr, sizeof(int64_t) * (size_t)n);
  for (int64_t j = 0; j < m; ++j)
    for (int64_t e = at_ptr[j]; e < at_ptr[j + 1]; ++e) {
      int64_t p = cur[at_col[e]]++;
      a_col[p] = (int32_t)j;
      a_val[p] = at_val[e];
    }
  free(cur);
  return 0;
}
