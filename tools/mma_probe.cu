// mma_probe.cu -- tcgen05 kind::f16 issue-rate probe (development tool): one CTA per
// SM, one thread issues NITER rounds of the head kernel's MMA pattern (4 K-steps x
// 3 passes, M = 128, K = 16 per MMA, operands in shared memory, K-major no-swizzle)
// and reports cycles per MMA for several N, against the floor 128 N / 256 cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1510_05237_b200/csrc \
//        tools/mma_probe.cu -o scratch/mma_probe && scratch/mma_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"
using namespace esk;

template <int N, int SW>
__global__ void __launch_bounds__(128, 1) probe(int niter, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (tc::smem_u32(sm) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (32768 + N * 64 * 4) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&tbase, 512);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::make_idesc_f16(128, N);
    const uint32_t a0 = tc::smem_u32(base), b0 = a0 + 32768;
    const uint32_t ahalf = 16384, bhalf = N * 64 * 2;
    const uint32_t sboA = (64 / 8) * 128, sboB = (64 / 8) * 128;
    long long t0 = clock64();
    for (int it = 0; it < niter; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t ko = ks * 2 * 128;
        const uint64_t ah = tc::make_sdesc(a0 + ko, 128, sboA), al = tc::make_sdesc(a0 + ahalf + ko, 128, sboA);
        const uint64_t bh = tc::make_sdesc(b0 + ko, 128, sboB), bl = tc::make_sdesc(b0 + bhalf + ko, 128, sboB);
        const uint32_t acc = (it | ks) ? 1u : 0u;
        tc::mma_f16(tmem + (SW ? 0 : 0), ah, bh, idesc, acc);
        tc::mma_f16(tmem + (SW ? 256 : 0), ah, bl, idesc, acc);
        tc::mma_f16(tmem + (SW ? 0 : 0), al, bh, idesc, 1u);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

template <int N, int SW>
void run(int nsm) {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * nsm);
  const int smem = 32768 + N * 64 * 4 + 1024;
  cudaFuncSetAttribute(probe<N, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int niter = 2000;
  probe<N, SW><<<nsm, 128, smem>>>(50, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<N, SW><<<nsm, 128, smem>>>(niter, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148]; cudaMemcpy(h, d, sizeof(unsigned long long) * nsm, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < nsm; ++i) avg += h[i]; avg /= nsm;
  const double nmma = 12.0 * niter;
  const double flops = 2.0 * 128 * N * 16 * nmma * nsm;
  printf("N=%3d sep_acc=%d grid=%3d: %.1f cycles/MMA (floor %.1f), %.3f ms, %.0f TFLOP/s  %s\n", N, SW, nsm,
         avg / nmma, 128.0 * N / 256, ms, flops / ms / 1e9, cudaGetErrorString(err));
  cudaFree(d);
}


// interference: the MMA pattern above while other warps load the SM like the head
// kernel does.  mode bit 0: 4 warps st.shared 16 B (zeroing); bit 1: one thread
// bulk-copies 32 KB global -> shared continuously; bit 2: 8 warps tcgen05.ld TMEM
// columns 256.. (epilogue drain); bit 3: 8 warps ld.shared 16 B.
template <int N>
__global__ void __launch_bounds__(448, 1) probe_mix(int niter, int mode, const uint8_t* gsrc,
                                                    unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (tc::smem_u32(sm) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar, cbar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t opbytes = 32768 + N * 64 * 4;
  uint8_t* scratch = base + ((opbytes + 1023) & ~1023u);  // 64 KB for the interference traffic
  for (int i = threadIdx.x; i < (int)(opbytes / 16); i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::mbar_init(&cbar, 1); tc::fence_mbar_init(); done = 0; }
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::make_idesc_f16(128, N);
    const uint32_t a0 = tc::smem_u32(base), b0 = a0 + 32768;
    const uint32_t ahalf = 16384, bhalf = N * 64 * 2;
    const uint32_t sbo = (64 / 8) * 128;
    long long t0 = clock64();
    for (int it = 0; it < niter; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t ko = ks * 2 * 128;
        const uint64_t ah = tc::make_sdesc(a0 + ko, 128, sbo), al = tc::make_sdesc(a0 + ahalf + ko, 128, sbo);
        const uint64_t bh = tc::make_sdesc(b0 + ko, 128, sbo), bl = tc::make_sdesc(b0 + bhalf + ko, 128, sbo);
        const uint32_t acc = (it | ks) ? 1u : 0u;
        tc::mma_f16(tmem, ah, bh, idesc, acc);
        tc::mma_f16(tmem, ah, bl, idesc, 1u);
        tc::mma_f16(tmem, al, bh, idesc, 1u);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
    done = 1;
  } else if (warp >= 1 && warp <= 4 && (mode & 1)) {
    int i = 0;
    while (!done) {
      for (int r = 0; r < 16; ++r, ++i)
        reinterpret_cast<uint4*>(scratch)[((i * 128) + threadIdx.x - 32) & 2047] = make_uint4(i, 0, 0, 0);
    }
  } else if (warp == 5 && lane == 0 && (mode & 2)) {
    uint32_t ph = 0;
    int i = 0;
    while (!done) {
      tc::mbar_arrive_expect_tx(&cbar, 32768);
      tc::bulk_g2s(scratch + 32768, gsrc + (size_t)(i & 63) * 32768, 32768, &cbar);
      tc::mbar_wait(&cbar, ph);
      ph ^= 1;
      ++i;
    }
  } else if (warp >= 6 && (mode & 4)) {
    const int lg = warp & 3;
    uint32_t v[16];
    uint32_t accx = 0;
    while (!done) {
      for (int c = 0; c < 128; c += 16) {
        tc::tmem_ld16(tmem + 256 + c + ((uint32_t)(lg * 32) << 16), v);
        tc::tmem_wait_ld();
        accx += v[0];
      }
    }
    if (accx == 12345) out[0] = 0;
  } else if (warp >= 6 && (mode & 8)) {
    uint4 accx = make_uint4(0, 0, 0, 0);
    int i = 0;
    while (!done) {
      for (int r = 0; r < 16; ++r, ++i) {
        const uint4 v = reinterpret_cast<const uint4*>(scratch)[((i * 256) + threadIdx.x) & 4095];
        accx.x += v.x;
      }
    }
    if (accx.x == 12345) out[0] = 0;
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

template <int N>
void run_mix(int mode, const uint8_t* gsrc) {
  const int nsm = 148;
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * nsm);
  const int smem = ((32768 + N * 64 * 4 + 1023) & ~1023) + 65536 + 1024;
  cudaFuncSetAttribute(probe_mix<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int niter = 2000;
  probe_mix<N><<<nsm, 448, smem>>>(niter, mode, gsrc, d);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(unsigned long long) * nsm, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  printf("mix N=%3d mode=%2d: %.1f cycles/MMA (floor %.1f)  %s\n", N, mode, avg / (12.0 * niter), 128.0 * N / 256,
         cudaGetErrorString(err));
  cudaFree(d);
}

// rotating operands: round r reads stage r % NS (A 32 KB + B N x 64 x 4), like the
// head kernel's pipeline stages (no copies in flight)
template <int N, int NS, int CM>
__global__ void __launch_bounds__(128, 1) probe_rot(int niter, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (tc::smem_u32(sm) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar, ebar[4];
  __shared__ uint32_t tbase;
  const uint32_t sb = ((32768 + N * 64 * 4) + 1023) & ~1023u;
  for (int i = threadIdx.x; i < (int)(NS * sb / 16); i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) tc::mbar_init(&ebar[i], 1); tc::fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&tbase, 512);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::make_idesc_f16(128, N);
    const uint64_t hdesc = tc::make_sdesc(0, 128, (64 / 8) * 128);
    const uint32_t s0 = tc::smem_u32(base);
    long long t0 = clock64();
    int st = 0;
    for (int it = 0; it < niter; ++it) {
      const uint32_t a = s0 + st * sb;
      const uint64_t dah = hdesc | ((a >> 4) & 0x3FFF), dal = dah + (16384 >> 4);
      const uint64_t dzh = dah + (32768 >> 4), dzl = dzh + ((N * 64 * 2) >> 4);
#pragma unroll
      for (uint32_t s = 0; s < 4; ++s) {
        tc::mma_f16(tmem, dah + 16 * s, dzh + 16 * s, idesc, (it | s) != 0);
        tc::mma_f16(tmem, dah + 16 * s, dzl + 16 * s, idesc, 1u);
        tc::mma_f16(tmem, dal + 16 * s, dzh + 16 * s, idesc, 1u);
      }
      if (CM & 1) tc::mma_commit(&ebar[st]);
      if (CM & 2) tc::fence_after();
      if (++st == NS) st = 0;
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

template <int N, int NS, int CM>
void run_rot() {
  const int nsm = 148;
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * nsm);
  const int smem = NS * (((32768 + N * 64 * 4) + 1023) & ~1023) + 1024;
  cudaFuncSetAttribute(probe_rot<N, NS, CM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int niter = 2000;
  probe_rot<N, NS, CM><<<nsm, 128, smem>>>(niter, d);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(unsigned long long) * nsm, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  printf("rot CM=%d N=%3d stages=%d: %.1f cycles/MMA (floor %.1f)  %s\n", CM, N, NS, avg / (12.0 * niter), 128.0 * N / 256,
         cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  run<112, 0>(148); run<112, 1>(148); run<128, 0>(148); run<64, 0>(148); run<256, 0>(148); run<208, 0>(148);
  run<104, 0>(148); run<96, 0>(148); run<88, 0>(148); run<80, 0>(148); run<120, 0>(148);
  run<112, 0>(1);
  uint8_t* g;
  cudaMalloc(&g, 64 << 20);
  cudaMemset(g, 0, 64 << 20);
  for (int mode : {0, 1, 2, 4, 8, 3, 7, 15}) run_mix<112>(mode, g);
  run_rot<112, 3, 0>(); run_rot<112, 3, 1>(); run_rot<112, 3, 2>(); run_rot<112, 3, 3>();
  return 0;
}
