// Probe 2: the 2:4-sparse integer MMA with cta_group::2 (CTA pair, M = 256):
// each CTA holds its own 128 compressed A rows, half of B and its own metadata;
// the leader issues tcgen05.cp.cta_group::2 (smem -> TMEM metadata) and
// tcgen05.mma.sp.cta_group::2. Checks that every CTA's rows decode with that CTA's
// metadata (pins the pair semantics used by the sparse GEMM path).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/sp_probe2.cu -o tools/sp_probe2
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2310_09259_b200/csrc/sm100.cuh"

using namespace quikb200;

constexpr int MR = 128, N = 64, KL = 64, NH = N / 2;

__host__ __device__ inline int sw128(int row, int byte) {
  const int chunk = (byte >> 4) ^ (row & 7);
  return row * 128 + chunk * 16 + (byte & 15);
}

__device__ __forceinline__ void tmem_st2(uint32_t taddr, uint32_t a, uint32_t b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) probe2(const int8_t* acomp /*[2*MR][32]*/, const uint32_t* meta /*[2*MR][2]*/,
                                                 int32_t* out /*[2*MR][N]*/, int mode) {
  __shared__ __align__(1024) uint8_t sa[MR * 128];
  __shared__ __align__(1024) uint8_t sb[NH * 128];
  __shared__ __align__(16) uint32_t sm_meta[MR * 4];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const uint32_t rank = cluster_ctarank();
  for (int i = tid; i < MR * 128; i += blockDim.x) sa[i] = 0;
  for (int i = tid; i < NH * 128; i += blockDim.x) sb[i] = 0;
  __syncthreads();
  for (int i = tid; i < MR * 32; i += blockDim.x)
    sa[sw128(i / 32, i % 32)] = static_cast<uint8_t>(acomp[rank * MR * 32 + i]);
  for (int i = tid; i < NH; i += blockDim.x) sb[sw128(i, rank * NH + i)] = 1;  // B[n][k] = (k == n)
  for (int i = tid; i < MR * 4; i += blockDim.x)
    sm_meta[i] = (i % 4) < 2 ? meta[(rank * MR + i / 4) * 2 + (i % 4)] : 0u;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<2>(&slot, 128);
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = slot;
  const uint32_t tmeta = tbase + 64;
  if (mode == 1 && warp < 4) {  // metadata by tcgen05.st, each CTA into its own TMEM
    const uint32_t m = rank * MR + warp * 32 + lane;
    tmem_st2(tbase + (static_cast<uint32_t>(warp * 32) << 16) + 64, meta[m * 2], meta[m * 2 + 1]);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (rank == 0 && tid == 0) {
    if (mode == 0) {
      uint64_t d = 0;
      d |= static_cast<uint64_t>((smem_u32(sm_meta) >> 4) & 0x3FFFu);
      d |= static_cast<uint64_t>(1u) << 16;
      d |= static_cast<uint64_t>(128u >> 4) << 32;
      d |= static_cast<uint64_t>(1u) << 46;
      asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(tmeta), "l"(d) : "memory");
    }
    const uint32_t idesc = idesc_make(2u, 1u, 2 * MR, N) | (1u << 2);
    const uint64_t ad = umma_desc_sw128(smem_u32(sa)), bd = umma_desc_sw128(smem_u32(sb));
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.sp.cta_group::2.kind::i8 [%0], %1, %2, [%5], %3, p;\n\t}\n" ::"r"(tbase),
        "l"(ad), "l"(bd), "r"(idesc), "r"(0), "r"(tmeta)
        : "memory");
    mma_commit<2>(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp < 4) {
    uint32_t v[32];
    for (int c = 0; c < N; c += 32) {
      tmem_ld32(tbase + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) out[(rank * MR + warp * 32 + lane) * N + c + j] = static_cast<int32_t>(v[j]);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc<2>(tbase, 128);
}

static const int kPairs[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

int main() {
  const int R = 2 * MR;
  std::vector<int8_t> a(R * 32);
  for (int m = 0; m < R; ++m)
    for (int b = 0; b < 32; ++b) a[m * 32 + b] = static_cast<int8_t>(1 + (m * 7 + b * 3) % 100);
  std::vector<uint32_t> meta(R * 2, 0);
  for (int m = 0; m < R; ++m)
    for (int g = 0; g < 16; ++g) {
      const int p = (m * 5 + g + (m >= MR ? 3 : 0)) % 6;
      meta[m * 2 + g / 8] |= static_cast<uint32_t>(kPairs[p][0] | (kPairs[p][1] << 2)) << (4 * (g % 8));
    }
  int8_t* da;
  uint32_t* dm;
  int32_t* dout;
  cudaMalloc(&da, a.size());
  cudaMalloc(&dm, meta.size() * 4);
  cudaMalloc(&dout, R * N * 4);
  cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dm, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dout, 0x7f, R * N * 4);
    probe2<<<2, 128>>>(da, dm, dout, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: kernel error %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    std::vector<int32_t> out(R * N);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    int bad[2] = {0, 0};
    for (int m = 0; m < R; ++m) {
      int32_t want[KL] = {};
      for (int g = 0; g < 16; ++g) {
        const int p = (m * 5 + g + (m >= MR ? 3 : 0)) % 6;
        want[4 * g + kPairs[p][0]] = a[m * 32 + 2 * g];
        want[4 * g + kPairs[p][1]] = a[m * 32 + 2 * g + 1];
      }
      for (int n = 0; n < N; ++n) bad[m / MR] += out[m * N + n] != want[n];
    }
    printf("mode %d (%s): mismatches CTA0 %d, CTA1 %d of %d each\n", mode,
           mode == 0 ? "tcgen05.cp.cta_group::2 from each CTA's smem" : "tcgen05.st per CTA", bad[0], bad[1],
           MR * N);
    for (int m : {0, 130}) {
      printf("row %3d:", m);
      for (int n = 0; n < 16; ++n) printf(" %3d", out[m * N + n]);
      printf("\n");
    }
  }
  return 0;
}
