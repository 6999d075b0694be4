// Raw tcgen05 MMA issue-rate microbenchmark (no global memory traffic): one CTA
// (or CTA pair) per SM repeatedly issues MMAs on resident shared-memory operands.
// Reports dense-equivalent int8 TOPS for kind::i8 dense vs 2:4 sparse (.sp), at
// cta_group::1 / ::2 and several N, to pin the tensor-core ceiling the GEMM
// kernels are measured against.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/mma_rate.cu -o tools/mma_rate
#include <cstdio>
#include <vector>

#include "../paper_2310_09259_b200/csrc/sm100.cuh"

using namespace quikb200;

template <int CG, int N, bool SP, int CP = 0, bool TS = false>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<CG>(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  if (warp == 0 && threadIdx.x == 0 && rank == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    const uint64_t ad = umma_desc_sw128(sa), bd = umma_desc_sw128(sb);
    constexpr uint32_t idesc = idesc_make(2u, 1u, 128 * CG, N) | (SP ? (1u << 2) : 0u);
    const uint32_t te = tbase + N;  // metadata after the accumulator (zeros: fine for timing)
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        // CP: metadata refresh every 4 MMAs (one 256-logical-K stage), like the GEMM:
        // 1 = two 128x128b copies into a 4-slot ring, 2 = same slot every time
        uint32_t tek = te;
        if constexpr (CP != 0) {
          const uint32_t slot_k = CP == 1 ? static_cast<uint32_t>(((it * 2 + (k >> 2)) & 3) * 8) : 0u;
          tek = te + slot_k;
          if ((k & 3) == 0) {
            tmem_cp_128x128b<CG>(tek, smem_desc_rows16(sa + 32768));
            tmem_cp_128x128b<CG>(tek + 4, smem_desc_rows16(sa + 32768 + 2048));
          }
        }
        if constexpr (SP) mma_sp_i8<CG>(tbase, ad + 2 * (k & 3), bd + 4 * (k & 1), idesc, tek + 2 * (k & 3), 1u);
        else if constexpr (TS) mma_i8_ts<CG>(tbase, tbase + 256 + 8 * (k & 3), bd + 2 * (k & 3), idesc, 1u);
        else mma_i8<CG>(tbase, ad + 2 * (k & 3), bd + 2 * (k & 3), idesc, 1u);
      }
    }
    mma_commit<CG>(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<CG>(tbase, 512);
  }
}

template <int CG, int N, bool SP, int CP = 0, bool TS = false>
void run(int sms) {
  auto k = rate_kernel<CG, N, SP, CP, TS>;
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* dc;
  cudaMalloc(&dc, 8);
  const int iters = 4096;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms / CG * CG);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, iters, dc);  // warm
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, k, iters, dc);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  const double kl = SP ? 64 : 32;  // logical K per instruction
  const double macs_per_sm = double(iters) * 8 * 128 * N * kl;  // per CTA: M rows = 128 per CTA
  const double tops = 2.0 * macs_per_sm * (sms / CG * CG) / (ms * 1e-3) / 1e12;
  printf("cta_group::%d N=%3d %-6s%s cp=%d : %s  %.3f ms  %.0f TOPS (dense-equivalent)  %.0f MAC/clk/SM\n", CG, N,
         SP ? "sparse" : "dense", TS ? " A=TMEM" : "", CP, e == cudaSuccess ? "ok " : cudaGetErrorString(e), ms, tops, macs_per_sm / cyc);
  cudaFree(dc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1, 128, false>(sms);
  run<1, 256, false>(sms);
  run<1, 128, true>(sms);
  run<1, 256, true>(sms);
  run<2, 128, false>(sms);
  run<2, 256, false>(sms);
  run<2, 128, true>(sms);
  run<2, 192, true>(sms);
  run<2, 256, true>(sms);
  run<2, 192, true, 1>(sms);
  run<2, 192, true, 2>(sms);
  run<1, 128, true, 1>(sms);
  // A operand from TMEM (the INT4-weight GEMM): kind::i8 .ts vs .ss
  run<1, 64, false, 0, true>(sms);
  run<1, 128, false, 0, true>(sms);
  run<1, 256, false, 0, true>(sms);
  run<2, 128, false, 0, true>(sms);
  run<2, 192, false, 0, true>(sms);
  run<2, 192, false>(sms);
  run<2, 256, false, 0, true>(sms);
  return 0;
}
