// tests/tc_probe.cu -- standalone check of the tcgen05 building blocks in
// paper_1510_05237_b200/csrc/tc.cuh: D[128 x N] = A[128 x K] B[N x K]^T with
// kind::tf32 MMAs (plain, or 3xTF32 = hi*hi + hi*lo + lo*hi), A/B staged in
// shared memory in the K-major no-swizzle layout, D in TMEM read back with
// tcgen05.ld.  Built and run by tests/test_tc_probe.py.
#include <cuda_runtime.h>

#include "../paper_1510_05237_b200/csrc/tc.cuh"

using namespace esk;

__global__ void __launch_bounds__(128) tc_probe_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                       float* __restrict__ D, int K, int N, int split) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int M = 128;
  float* a_hi = reinterpret_cast<float*>(sm);
  float* a_lo = a_hi + M * K;
  float* b_hi = a_lo + M * K;
  float* b_lo = b_hi + N * K;
  for (int q = threadIdx.x; q < M * K; q += blockDim.x) {
    const int r = q / K, k = q % K;
    const float x = A[q];
    const float hi = split ? tc::to_tf32(x) : x;
    *reinterpret_cast<float*>(reinterpret_cast<char*>(a_hi) + tc::kmajor_off(r, k, K)) = hi;
    *reinterpret_cast<float*>(reinterpret_cast<char*>(a_lo) + tc::kmajor_off(r, k, K)) = x - hi;
  }
  for (int q = threadIdx.x; q < N * K; q += blockDim.x) {
    const int r = q / K, k = q % K;
    const float x = B[q];
    const float hi = split ? tc::to_tf32(x) : x;
    *reinterpret_cast<float*>(reinterpret_cast<char*>(b_hi) + tc::kmajor_off(r, k, K)) = hi;
    *reinterpret_cast<float*>(reinterpret_cast<char*>(b_lo) + tc::kmajor_off(r, k, K)) = x - hi;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tc::tmem_alloc(&tmem_base, 256);
  if (threadIdx.x == 0) tc::mbar_init(&mbar, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::make_idesc_tf32(M, N);
    const uint32_t sboA = (K / 4) * 128, sboB = (K / 4) * 128;
    for (int s = 0; s < K / 8; ++s) {
      const uint64_t ah = tc::make_sdesc(tc::smem_u32(a_hi) + s * 256, 128, sboA);
      const uint64_t bh = tc::make_sdesc(tc::smem_u32(b_hi) + s * 256, 128, sboB);
      tc::mma_tf32(tmem, ah, bh, idesc, s > 0);
      if (split) {
        const uint64_t al = tc::make_sdesc(tc::smem_u32(a_lo) + s * 256, 128, sboA);
        const uint64_t bl = tc::make_sdesc(tc::smem_u32(b_lo) + s * 256, 128, sboB);
        tc::mma_tf32(tmem, ah, bl, idesc, 1);
        tc::mma_tf32(tmem, al, bh, idesc, 1);
      }
    }
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  const int row = 32 * warp + lane;
  for (int c0 = 0; c0 < N; c0 += 8) {
    float v[8];
    tc::tmem_ld8(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
    for (int i = 0; i < 8; ++i) D[row * N + c0 + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

extern "C" int tc_probe(const float* A, const float* B, float* D, int K, int N, int split) {
  float *dA, *dB, *dD;
  const int M = 128;
  cudaMalloc(&dA, sizeof(float) * M * K);
  cudaMalloc(&dB, sizeof(float) * N * K);
  cudaMalloc(&dD, sizeof(float) * M * N);
  cudaMemcpy(dA, A, sizeof(float) * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B, sizeof(float) * N * K, cudaMemcpyHostToDevice);
  const size_t smem = sizeof(float) * 2 * (M * K + N * K);
  cudaFuncSetAttribute(tc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tc_probe_kernel<<<1, 128, smem>>>(dA, dB, dD, K, N, split);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D, dD, sizeof(float) * M * N, cudaMemcpyDeviceToHost);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return (int)e;
}
