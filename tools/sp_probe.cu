// Probe of the sm_100a 2:4-sparse integer MMA (tcgen05.mma.sp ... kind::i8):
// decodes where the compressed A values land for given metadata words, to pin
// the metadata layout used by the sparse GEMM path. One CTA, M = 128, N = 64,
// K = 64 logical (32 compressed bytes per A row), B = identity so that
// D[m][n] = A_logical[m][n].
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../include tools/sp_probe.cu -o sp_probe -lcuda
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2310_09259_b200/csrc/sm100.cuh"

using namespace quikb200;

constexpr int M = 128, N = 64, KL = 64;

__device__ __forceinline__ void tmem_st2(uint32_t taddr, uint32_t a, uint32_t b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}

// swizzled (128B) byte offset of (row, byte) inside a K-major tile of 128-byte rows
__host__ __device__ inline int sw128(int row, int byte) {
  const int chunk = (byte >> 4) ^ (row & 7);
  return row * 128 + chunk * 16 + (byte & 15);
}

__global__ void probe(const int8_t* acomp /*[M][32]*/, const uint32_t* meta /*[M][2]*/, int32_t* out /*[M][N]*/,
                      int meta_col_off, int id2, int cp_meta) {
  __shared__ __align__(1024) uint8_t sa[M * 128];
  __shared__ __align__(1024) uint8_t sb[N * 128];
  __shared__ __align__(16) uint32_t sm_meta[M * 4];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < M * 128; i += blockDim.x) sa[i] = 0;
  for (int i = tid; i < N * 128; i += blockDim.x) sb[i] = 0;
  __syncthreads();
  for (int i = tid; i < M * 32; i += blockDim.x) sa[sw128(i / 32, i % 32)] = static_cast<uint8_t>(acomp[i]);
  for (int n = tid; n < N; n += blockDim.x) sb[sw128(n, n)] = 1;  // B[n][k] = (k == n)
  // metadata copy source for tcgen05.cp 128x128b: [128 rows][16 B] row-major
  for (int i = tid; i < M * 4; i += blockDim.x) sm_meta[i] = (i % 4) < 2 ? meta[(i / 4) * 2 + (i % 4)] : 0u;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<1>(&slot, 128);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  const uint32_t tmeta = tbase + 64 + meta_col_off;
  if (!cp_meta && warp < 4) {
    const uint32_t m = warp * 32 + lane;
    tmem_st2(tbase + (static_cast<uint32_t>(warp * 32) << 16) + 64 + meta_col_off, meta[m * 2], meta[m * 2 + 1]);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    if (cp_meta) {
      // smem descriptor, no swizzle: core matrices 8 rows x 16 B contiguous (128 B),
      // SBO = 128 B between 8-row groups, LBO unused
      uint64_t d = 0;
      d |= static_cast<uint64_t>((smem_u32(sm_meta) >> 4) & 0x3FFFu);
      d |= static_cast<uint64_t>(1u) << 16;
      d |= static_cast<uint64_t>(128u >> 4) << 32;
      d |= static_cast<uint64_t>(1u) << 46;
      asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tmeta), "l"(d) : "memory");
    }
    uint32_t idesc = idesc_make(2u, 1u, M, N) | (1u << 2) | static_cast<uint32_t>(id2 & 3);
    const uint64_t ad = umma_desc_sw128(smem_u32(sa)), bd = umma_desc_sw128(smem_u32(sb));
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%5], %3, p;\n\t}\n" ::"r"(tbase),
        "l"(ad), "l"(bd), "r"(idesc), "r"(0), "r"(tmeta)
        : "memory");
    mma_commit<1>(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp < 4) {
    uint32_t v[32];
    for (int c = 0; c < N; c += 32) {
      tmem_ld32(tbase + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * N + c + j] = static_cast<int32_t>(v[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<1>(tbase, 128);
}

static const int kPairs[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

int main(int argc, char** argv) {
  const int id2 = argc > 1 ? atoi(argv[1]) : 0;
  std::vector<int8_t> a(M * 32);
  for (int m = 0; m < M; ++m)
    for (int b = 0; b < 32; ++b) a[m * 32 + b] = static_cast<int8_t>(1 + (m * 7 + b * 3) % 100);
  // per row: group g uses pair p = (m + g) % 6; nibble hypothesis H1: lo 2 bits = idx of
  // the first stored value, hi 2 bits = idx of the second; group g at bits 4g.
  std::vector<uint32_t> meta(M * 2, 0);
  for (int m = 0; m < M; ++m)
    for (int g = 0; g < 16; ++g) {
      const int p = (m + g) % 6;
      const uint32_t nib = static_cast<uint32_t>(kPairs[p][0] | (kPairs[p][1] << 2));
      meta[m * 2 + g / 8] |= nib << (4 * (g % 8));
    }
  int8_t* da;
  uint32_t* dm;
  int32_t* dout;
  cudaMalloc(&da, a.size());
  cudaMalloc(&dm, meta.size() * 4);
  cudaMalloc(&dout, M * N * 4);
  cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dm, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice);
  for (int cp = 0; cp < 2; ++cp) {
    cudaMemset(dout, 0x7f, M * N * 4);
    probe<<<1, 128>>>(da, dm, dout, 0, id2, cp);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("kernel error (cp=%d): %s\n", cp, cudaGetErrorString(e));
      return 1;
    }
    std::vector<int32_t> out(M * N);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < M; ++m) {
      int32_t want[KL] = {};
      for (int g = 0; g < 16; ++g) {
        const int p = (m + g) % 6;
        want[4 * g + kPairs[p][0]] = a[m * 32 + 2 * g];
        want[4 * g + kPairs[p][1]] = a[m * 32 + 2 * g + 1];
      }
      for (int n = 0; n < N; ++n) bad += out[m * N + n] != want[n];
    }
    printf("id2=%d metadata via %s: H1 mismatches = %d of %d\n", id2, cp ? "tcgen05.cp" : "tcgen05.st", bad, M * N);
    for (int m : {0, 1, 37}) {
      printf("row %3d:", m);
      for (int n = 0; n < 24; ++n) printf(" %3d", out[m * N + n]);
      printf("\n   comp:");
      for (int b = 0; b < 12; ++b) printf(" %3d", a[m * 32 + b]);
      printf("\n");
    }
  }
  return 0;
}
