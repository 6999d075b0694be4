// tcgen05.mma kind::f16 issue-rate microbenchmark: A from shared memory (SS) vs A
// from TMEM (TS), M = 128, small N (the weight-only decode shapes), one CTA per SM,
// resident operands, P independent accumulators in rotation. Reports cycles per MMA.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/ts_rate.cu -o tools/ts_rate
#include <cstdio>

#include "../paper_2310_09259_b200/csrc/sm100.cuh"

using namespace quikb200;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc)
      : "memory");
}

// whole warp converged, elect.sync per MMA (operands warp-uniform). STORERS > 0: four
// more warps keep writing TMEM (tcgen05.st, other columns) meanwhile, as the
// weight-only kernel's widening warps do.
template <int N, int STORERS = 0>
__global__ void __launch_bounds__(256, 1) rate_warp(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<1>(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = __shfl_sync(0xffffffffu, slot, 0);
  if (warp == 0) {
    const uint32_t sb = smem_u32(smem) + 32768;
    const uint64_t bd = umma_desc_sw128(sb);
    constexpr uint32_t idesc = idesc_make(1u, 0u, 128, N);
    const uint32_t a_tm = t + 256;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) mma_ts_elect(t, a_tm + 8 * k, bd + 2 * (k & 3), idesc);
    }
    if (threadIdx.x == 0) {
      mma_commit<1>(&bar);
      mbar_wait(&bar, 0);
      const unsigned long long t1 = clock64();
      if (blockIdx.x == 0) *cycles = t1 - t0;
    }
    __syncwarp();
  } else if (STORERS && warp >= 4 && warp < 8) {
    uint32_t r[32];
    for (int j = 0; j < 32; ++j) r[j] = 0x3c003c00u;
    const uint32_t ta = t + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 384;
    for (int it = 0; it < iters / 2; ++it) {
#pragma unroll
      for (int h = 0; h < 4; ++h) tmem_st32(ta + 32 * h, r);
      tmem_st_wait();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<1>(t, 512);
  }
}

template <int N, int STORERS = 0>
void run_warp(int sms) {
  auto k = rate_warp<N, STORERS>;
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* dc;
  cudaMalloc(&dc, 8);
  const int iters = 2048;
  k<<<sms, STORERS ? 256 : 128, smem>>>(iters, dc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("kind::f16 M=128 N=%3d TS, converged warp + elect.sync%s: %s  %.1f cycles/MMA\n", N,
         STORERS ? ", 4 warps storing TMEM meanwhile" : "",
         e == cudaSuccess ? "ok" : cudaGetErrorString(e), double(cyc) / (iters * 16.0));
  cudaFree(dc);
}

template <int N, bool TS, int P, int ISSUERS = 1>
__global__ void __launch_bounds__(128, 1) rate(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, ISSUERS);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<1>(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot;
  if (threadIdx.x % 32 == 0 && warp < ISSUERS) {
    const uint32_t sa = smem_u32(smem), sb = sa + 32768;
    const uint64_t ad = umma_desc_sw128(sa), bd = umma_desc_sw128(sb);
    constexpr uint32_t idesc = idesc_make(1u, 0u, 128, N);
    const uint32_t a_tm = t + 256;  // A in TMEM columns 256.. (contents irrelevant for timing)
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t d = t + (k % P) * N + warp * 64;
        if constexpr (TS) mma_ts(d, a_tm + 8 * (k & 15), bd + 2 * (k & 3), idesc, 1u);
        else mma_f16<1>(d, ad + 2 * (k & 3), bd + 2 * (k & 3), idesc, 1u);
      }
    }
    mma_commit<1>(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && warp == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<1>(t, 512);
  }
}

template <int N, bool TS, int P, int ISSUERS = 1>
void run(int sms) {
  auto k = rate<N, TS, P, ISSUERS>;
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* dc;
  cudaMalloc(&dc, 8);
  const int iters = 2048;
  k<<<sms, 128, smem>>>(iters, dc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("kind::f16 M=128 N=%3d %s P=%d issuers=%d: %s  %.1f cycles/MMA (all issuers)\n", N,
         TS ? "TS (A in TMEM)" : "SS (A in smem)", P, ISSUERS, e == cudaSuccess ? "ok" : cudaGetErrorString(e),
         double(cyc) / (iters * 16.0 * ISSUERS));
  cudaFree(dc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<16, false, 1>(sms);
  run<16, false, 8>(sms);
  run<16, true, 1>(sms);
  run<16, true, 8>(sms);
  run<32, false, 1>(sms);
  run<32, true, 1>(sms);
  run<32, true, 4>(sms);
  run<64, false, 1>(sms);
  run<64, true, 1>(sms);
  run<128, false, 1>(sms);
  run<128, true, 1>(sms);
  run<16, true, 1, 2>(sms);
  run<16, true, 1, 4>(sms);
  run<16, false, 1, 2>(sms);
  run_warp<16>(sms);
  run_warp<32>(sms);
  run_warp<16, 1>(sms);
  return 0;
}
