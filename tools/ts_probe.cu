// Probe: tcgen05.mma kind::f16 with the A operand in TMEM (".ts" form). Pins the TMEM
// layout of A the weight-only kernel writes with tcgen05.st: lane = A row m, 32-bit
// column j = f16x2 {k = 2j (low half), 2j + 1 (high half)}, K = 16 per MMA, the next
// K step at +8 columns. Two MMAs (K = 32) into D (M = 128, N = 16), compared with the
// host product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/ts_probe.cu -o tools/ts_probe
#include <cuda_fp16.h>

#include <cstdio>
#include <vector>

#include "../paper_2310_09259_b200/csrc/sm100.cuh"

using namespace quikb200;

constexpr int kN = 16, kK = 32;

__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void probe(const float* A, const float* B, float* D) {
  __shared__ __align__(1024) uint8_t sb[kN * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, m = threadIdx.x;
  // B [kN][kK] f16, K-major, 128-byte swizzle (chunk c of row n at 16 * (c ^ (n & 7)))
  for (int i = threadIdx.x; i < kN * kK; i += blockDim.x) {
    const int n = i / kK, k = i % kK, c = (k * 2) / 16, w = (k * 2) % 16;
    *reinterpret_cast<__half*>(sb + n * 128 + ((c ^ (n & 7)) * 16) + w) = __float2half(B[i]);
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<1>(&slot, 64);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot;
  // A -> TMEM columns 32.. (lane m, column j = {k = 2j, 2j + 1})
  uint32_t r[32];
  for (int j = 0; j < 32; ++j) {
    if (j < kK / 2) {
      const __half2 h = __floats2half2_rn(A[m * kK + 2 * j], A[m * kK + 2 * j + 1]);
      r[j] = *reinterpret_cast<const uint32_t*>(&h);
    } else {
      r[j] = 0;
    }
  }
  tmem_st32(t + (static_cast<uint32_t>(warp * 32) << 16) + 32, r);
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_make(1u, 0u, 128, kN);
    const uint64_t bd = umma_desc_sw128(smem_u32(sb));
    mma_f16_ts(t, t + 32, bd, idesc, 0u);
    mma_f16_ts(t, t + 32 + 8, bd + 2, idesc, 1u);
    mma_commit<1>(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  uint32_t v[32];
  tmem_ld32(t + (static_cast<uint32_t>(warp * 32) << 16), v);
  tmem_ld_wait();
  for (int n = 0; n < kN; ++n) D[m * kN + n] = __uint_as_float(v[n]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<1>(t, 64);
  }
}

// kind::i8 with A in TMEM: lane = row, 32-bit column j = 4 int8 {k = 4j .. 4j+3}
// (byte b = k 4j + b), K = 32 per MMA, next K step at +8 columns.
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
constexpr int kK8 = 64;
__global__ void probe_i8(const int* A, const int* B, int* D) {
  __shared__ __align__(1024) uint8_t sb[kN * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, m = threadIdx.x;
  for (int i = threadIdx.x; i < kN * kK8; i += blockDim.x) {
    const int n = i / kK8, k = i % kK8, c = k / 16, w = k % 16;
    sb[n * 128 + ((c ^ (n & 7)) * 16) + w] = static_cast<uint8_t>(static_cast<int8_t>(B[i]));
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<1>(&slot, 64);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot;
  uint32_t r[32];
  for (int j = 0; j < 32; ++j) {
    uint32_t v = 0;
    if (j < kK8 / 4)
      for (int b = 0; b < 4; ++b) v |= (static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(A[m * kK8 + 4 * j + b]))) << (8 * b));
    r[j] = v;
  }
  tmem_st32(t + (static_cast<uint32_t>(warp * 32) << 16) + 32, r);
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_make(2u, 1u, 128, kN);
    const uint64_t bd = umma_desc_sw128(smem_u32(sb));
    mma_i8_ts(t, t + 32, bd, idesc, 0u);
    mma_i8_ts(t, t + 32 + 8, bd + 2, idesc, 1u);
    mma_commit<1>(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  uint32_t v[32];
  tmem_ld32(t + (static_cast<uint32_t>(warp * 32) << 16), v);
  tmem_ld_wait();
  for (int n = 0; n < kN; ++n) D[m * kN + n] = static_cast<int>(v[n]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<1>(t, 64);
  }
}

int run_i8() {
  std::vector<int> A(128 * kK8), B(kN * kK8), D(128 * kN);
  for (int m = 0; m < 128; ++m)
    for (int k = 0; k < kK8; ++k) A[m * kK8 + k] = ((m * 5 + k * 3) % 15) - 7;
  for (int n = 0; n < kN; ++n)
    for (int k = 0; k < kK8; ++k) B[n * kK8 + k] = ((n * 7 + k * 11 + (k * k) % 13) % 31) - 15;
  int *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  probe_i8<<<1, 128>>>(dA, dB, dD);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < kN; ++n) {
      int want = 0;
      for (int k = 0; k < kK8; ++k) want += A[m * kK8 + k] * B[n * kK8 + k];
      if (want != D[m * kN + n] && bad++ < 8) printf("i8 m=%d n=%d got %d want %d\n", m, n, D[m * kN + n], want);
    }
  printf("ts_probe i8: %s, %d mismatches of %d (layout: lane = row, column j = 4 x int8 {k=4j..4j+3}, +8 cols per K=32)\n",
         cudaGetErrorString(e), bad, 128 * kN);
  return bad != 0;
}

int main() {
  const int bad_i8 = run_i8();
  std::vector<float> A(128 * kK), B(kN * kK), D(128 * kN);
  for (int m = 0; m < 128; ++m)
    for (int k = 0; k < kK; ++k) A[m * kK + k] = static_cast<float>(((m * 3 + k * 5) % 9) - 4);
  for (int n = 0; n < kN; ++n)
    for (int k = 0; k < kK; ++k) B[n * kK + k] = static_cast<float>(((n * 7 + k * 3 + (k * k) % 11) % 5) - 2);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dA, dB, dD);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < kN; ++n) {
      float want = 0;
      for (int k = 0; k < kK; ++k) want += A[m * kK + k] * B[n * kK + k];
      if (want != D[m * kN + n] && bad++ < 8) printf("m=%d n=%d got %g want %g\n", m, n, D[m * kN + n], want);
    }
  printf("ts_probe: %s, %d mismatches of %d (layout: lane = row, column j = f16x2 {k=2j, 2j+1}, +8 cols per K=16)\n",
         cudaGetErrorString(e), bad, 128 * kN);
  return bad != 0 || bad_i8;
}
