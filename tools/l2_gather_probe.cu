// L2 -> SM gather bandwidth for the V-side tail's access pattern:
// warps gather rows of a small L2-resident table (R rows x 128 floats, 512 B per row)
// by a random index stream, one float4 per lane per row, D rows in flight per warp,
// FMA-accumulated so nothing is dead.  No arithmetic of the method; a ceiling for the
// tail gather (k_spmm_tail) measured on this B200.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_gather_probe tools/l2_gather_probe.cu
//   ./l2_gather_probe [rows=12068] [gathers=28105323] [zipf_s=0 [zipf_offset=1024]]
// zipf_s > 0 draws row r with probability ~ 1 / (offset + r)^s (the tail's active terms
// are Zipf ranks after the head), else uniformly.
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int D, int LANES>
__global__ void __launch_bounds__(256) gather(const float4* __restrict__ z, const int* __restrict__ idx,
                                               const float* __restrict__ w, long n, float4* out) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const long per = (n + nw - 1) / nw;
  const long b = warp * per, e = min(n, b + per);
  for (long i = b; i < e; i += D) {
    float4 v[D];
    float a[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const long j = min(i + d, e - 1);
      const int r = __ldg(idx + j);
      a[d] = (i + d < e) ? __ldg(w + j) : 0.f;
      v[d] = lane < LANES ? __ldg(z + (long)r * 32 + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      acc.x += a[d] * v[d].x; acc.y += a[d] * v[d].y; acc.z += a[d] * v[d].z; acc.w += a[d] * v[d].w;
    }
  }
  out[warp * 32 + lane] = acc;
}

template <int D, int LANES>
void run(const char* name, const float4* z, const int* idx, const float* w, long n, float4* out, int blocks) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int r = 0; r < 3; ++r) gather<D, LANES><<<blocks, 256>>>(z, idx, w, n, out);
  CK(cudaEventRecord(e0));
  const int reps = 10;
  for (int r = 0; r < reps; ++r) gather<D, LANES><<<blocks, 256>>>(z, idx, w, n, out);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  ms /= reps;
  const double bytes = (double)n * 16 * LANES;
  printf("%-28s blocks %5d  %.3f ms  %.2f TB/s of row bytes (%d B per row)\n", name, blocks, ms, bytes / ms / 1e9,
         16 * LANES);
}

int main(int argc, char** argv) {
  const long rows = argc > 1 ? atol(argv[1]) : 12068;
  const long n = argc > 2 ? atol(argv[2]) : 28105323;
  const double zs = argc > 3 ? atof(argv[3]) : 0.0;
  const double zo = argc > 4 ? atof(argv[4]) : 1024.0;
  std::vector<double> cdf(rows);
  for (long r = 0; r < rows; ++r) cdf[r] = (r ? cdf[r - 1] : 0.0) + (zs > 0 ? 1.0 / pow(zo + r, zs) : 1.0);
  std::vector<int> hi(n);
  std::vector<float> hw(n);
  unsigned long long s = 88172645463325252ull;
  for (long i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const double u = (double)(s >> 11) * (1.0 / 9007199254740992.0) * cdf[rows - 1];
    hi[i] = (int)std::min<long>(rows - 1, std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
    hw[i] = 1.0f + (float)(s >> 40) * 1e-7f;
  }
  float4 *z, *out;
  int* idx;
  float* w;
  CK(cudaMalloc(&z, rows * 512));
  CK(cudaMemset(z, 0, rows * 512));
  CK(cudaMalloc(&idx, n * 4));
  CK(cudaMalloc(&w, n * 4));
  CK(cudaMemcpy(idx, hi.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(w, hw.data(), n * 4, cudaMemcpyHostToDevice));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int maxb = sms * 8;
  CK(cudaMalloc(&out, (long)maxb * 256 * 16));
  printf("table %ld rows (%.1f MB), %ld gathers, %d SMs, rows %s (s = %.2f, offset %.0f)\n", rows, rows * 512 / 1e6, n, sms,
         zs > 0 ? "Zipf" : "uniform", zs, zo);
  for (int bps : {3, 4, 6, 8}) {
    run<4, 32>("D=4 512B", z, idx, w, n, out, sms * bps);
    run<4, 25>("D=4 400B (25 lanes)", z, idx, w, n, out, sms * bps);
    run<8, 32>("D=8 512B", z, idx, w, n, out, sms * bps);
    run<8, 25>("D=8 400B (25 lanes)", z, idx, w, n, out, sms * bps);
  }
  return 0;
}
