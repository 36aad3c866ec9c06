// l2_smem_probe.cu -- L2 -> shared-memory bulk-copy throughput (development tool):
// every CTA (one per SM) streams CHUNK-byte cp.async.bulk copies of an L2-resident
// buffer (or an HBM one larger than L2) into NBUF shared buffers, NBUF in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1510_05237_b200/csrc \
//        tools/l2_smem_probe.cu -o scratch/l2_smem_probe && scratch/l2_smem_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"
using namespace esk;

__global__ void __launch_bounds__(64, 1) copyk(const uint8_t* src, size_t span, int chunk, int nbuf, int iters,
                                               unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_[];
  __shared__ __align__(8) uint64_t bar_[2][8];
  const int issuer = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0 || issuer >= (int)(gridDim.y)) return;
  uint64_t* bar = bar_[issuer];
  uint8_t* sm = sm_ + (size_t)issuer * nbuf * chunk;
  for (int b = 0; b < nbuf; ++b) tc::mbar_init(&bar[b], 1);
  tc::fence_mbar_init();
  uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const size_t nchunks = span / chunk;
  size_t pos = ((size_t)blockIdx.x * 7919 + issuer * 131) % nchunks;
  long long t0 = clock64();
  for (int i = 0; i < iters + nbuf; ++i) {
    const int b = i % nbuf;
    if (i >= nbuf) {
      tc::mbar_wait(&bar[b], ph[b]);
      ph[b] ^= 1;
    }
    if (i < iters) {
      tc::mbar_arrive_expect_tx(&bar[b], chunk);
      tc::bulk_g2s(sm + (size_t)b * chunk, src + pos * chunk, chunk, &bar[b]);
      pos = (pos + 148) % nchunks;
    }
  }
  if (issuer == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  uint8_t* g;
  const size_t big = 4ull << 30;
  cudaMalloc(&g, big);
  cudaMemset(g, 1, big);
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(copyk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nis : {1, 2})
  for (size_t span : {(size_t)8 << 20}) {
    for (int chunk : {4096, 16384, 32768}) {
      for (int nbuf : {1, 2, 4}) {
        if ((size_t)chunk * nbuf * nis > 200 * 1024) continue;
        const int iters = (int)(4000ll * 32768 / chunk > 40000 ? 40000 : 4000ll * 32768 / chunk);
        copyk<<<dim3(148, nis), 64, chunk * nbuf * nis>>>(g, span, chunk, nbuf, 100, d);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        copyk<<<dim3(148, nis), 64, chunk * nbuf * nis>>>(g, span, chunk, nbuf, iters, d);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = 148.0 * iters * chunk * nis;
        printf("issuers %d span %6zu MB chunk %6d nbuf %d: %.2f TB/s (%.1f B/clk/SM at 1.92 GHz)  %s\n", nis, span >> 20, chunk, nbuf,
               bytes / ms / 1e9, bytes / 148 / (ms * 1.92e6), cudaGetErrorString(err));
      }
    }
  }
  return 0;
}
