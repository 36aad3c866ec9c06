// synth/zipfgen_cuda.cu -- GPU twin of synth/zipfgen.c (INPUT GENERATION ONLY).
//
// Same counter-based recipe, same host-built cdf[] / vtab[] tables, explicitly
// ordered IEEE fp64 operations (__dsub_rn/__dmul_rn/__dadd_rn, so nvcc cannot
// contract them into an FMA): the output is bitwise identical to the CPU
// generator (checked by tests/test_synth.py).  Used by bench.py to build the
// Large / Box matrices directly in HBM; holds none of the method's arithmetic.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t zg_hash(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
  uint64_t h = mix64(seed + 0x9E3779B97F4A7C15ULL * (stream + 1ULL));
  h = mix64(h ^ (a * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL));
  h = mix64(h ^ (b * 0xABC98388FB8FAC03ULL + 0x8CB92BA72F3D8DD7ULL));
  return h;
}

constexpr int kMaxD = 256;

__global__ void gen_at_kernel(int64_t n, int64_t m, int32_t d, uint64_t seed,
                              const double* __restrict__ cdf, const double* __restrict__ vtab,
                              int32_t* __restrict__ at_col, float* __restrict__ at_val) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  int32_t row[kMaxD];
  int32_t cnt = 0;
  uint64_t q = 0;
  while (cnt < d) {
    uint64_t x = zg_hash(seed, 1ULL, (uint64_t)j, q++);
    double u = (double)(x >> 11) * 0x1p-53;  // exact: 53-bit integer times a power of two
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
      int64_t mid = lo + ((hi - lo) >> 1);
      if (__ldg(cdf + mid) > u) hi = mid; else lo = mid + 1;
    }
    int32_t r = (int32_t)lo;
    bool dup = false;
    for (int32_t a = 0; a < cnt; ++a) dup |= (row[a] == r);
    if (!dup) row[cnt++] = r;
  }
  for (int32_t a = 1; a < d; ++a) {
    int32_t key = row[a], b = a - 1;
    while (b >= 0 && row[b] > key) { row[b + 1] = row[b]; --b; }
    row[b + 1] = key;
  }
  int32_t* oc = at_col + j * (int64_t)d;
  float* ov = at_val + j * (int64_t)d;
  for (int32_t a = 0; a < d; ++a) {
    uint64_t x = zg_hash(seed, 2ULL, (uint64_t)j, (uint64_t)row[a]);
    uint32_t idx = (uint32_t)(x >> 48);
    double f = (double)(uint32_t)((x >> 16) & 0xFFFFFFFFULL) * 0x1p-32;
    double lo = __ldg(vtab + idx);
    double dv = __dsub_rn(__ldg(vtab + idx + 1), lo);
    double t2 = __dmul_rn(dv, f);
    double v = __dadd_rn(lo, t2);
    oc[a] = row[a];
    ov[a] = __double2float_rn(v);
  }
}

}  // namespace

extern "C" int zg_generate_at_cuda(int64_t n, int64_t m, int32_t d, uint64_t seed,
                                   const double* cdf_dev, const double* vtab_dev,
                                   int32_t* at_col_dev, float* at_val_dev, void* stream) {
  if (n <= 0 || m <= 0 || d <= 0 || d > kMaxD || (int64_t)d * 2 > n) return -1;
  int threads = 128;
  int64_t blocks = (m + threads - 1) / threads;
  gen_at_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(n, m, d, seed, cdf_dev, vtab_dev,
                                                                         at_col_dev, at_val_dev);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
