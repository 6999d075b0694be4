// Weight-streaming split-K integer GEMM on INT4 weights for small token counts
// (M <= 64, quik mode; HBM-bound for small M, cfg1 / cfg4 small M):
//
//   acc_ws[t][n] += sum_{k in split} q[n][k] * X8[t][k]      (red.global.add.s32)
//
// followed by the fused kernel's AccInit mode (dequant + f16 outlier MMAs + store,
// bit-identical to the one-kernel V3 forward: integer sums commute).
//
// Same architecture as the weight-only kernel (wo.cu): the 4-bit weights never exist
// as int8 in shared memory. A weight producer TMA-streams 16 KB INT4 tiles (128 rows x
// 256 K) into a deep ring; G widening groups (4 warps each, one weight row per thread)
// sign-extend the nibbles with two integer ops per four values and tcgen05.st them into
// a TMEM A buffer (lane = weight row, column j = 4 int8 {k = 4j .. 4j+3}, pinned by
// tools/ts_probe.cu) and release the weight slot at once; each group's converged
// issuing warp runs 8 tcgen05.mma.kind::i8 (A from TMEM, the int8 activation-code tile
// from shared memory) per stage into its own int32 accumulator; four epilogue warps sum
// the G accumulators and red.add them into the workspace. Each ring stage has exactly
// one consumer sequence (see wo.cu).
//
// Warps: 0 weight producer, 1 TMEM allocator, 2 .. 4G+1 widening, then 4 epilogue, G
// issuers, 1 activation-tile producer.
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"

namespace quikb200 {

namespace {

constexpr int kS4WBytes = kBlockM * kKBlockBytes;  // 16 KB: 128 rows x 128 B INT4 = 256 K
constexpr int kS4TmemA = 64;                        // columns per A buffer (256 K of int8)

template <int BN>
struct S4Cfg {
  static constexpr int G = BN == 64 ? 2 : 3;
  static constexpr int kTAtom = BN * kKBlockBytes;  // BN rows x 128 K int8
  static constexpr int kSlotT = 2 * kTAtom;         // 256 K per stage
  static constexpr int kStagesW = BN == 64 ? 8 : 9;
  static constexpr int kStagesT = BN == 64 ? 4 : 6;
  static_assert(kStagesW % G == 0 && kStagesT % G == 0, "one consumer group per stage");
  static constexpr int kOffT = kStagesW * kS4WBytes;
  static constexpr int kRingBytes = kOffT + kStagesT * kSlotT;
  static constexpr int kBarBytes = (2 * (kStagesW + kStagesT) + 2 * G + 4) * 8 + 16;
  static constexpr int kSmemBytes = 1024 + kRingBytes + kBarBytes;
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
  static constexpr int kAccCol = G * kS4TmemA;
  static constexpr int kAccBuf = G * BN;  // G int32 accumulators, double-buffered
  static_assert(kAccCol + 2 * kAccBuf <= 512, "TMEM budget");
  static constexpr int kWidenEnd = 2 + 4 * G, kEpiEnd = kWidenEnd + 4, kIssEnd = kEpiEnd + G;
  static constexpr int kThreads = (kIssEnd + 1) * 32;
};

struct S4Params {
  CUtensorMap tm_w;  // INT4 [N][kpad / 2] (device nibble layout), box {128 B, 128}, SW128
  CUtensorMap tm_x;  // int8 [M][kpad], box {128 B, BN}, SW128
  int M, N, nstage, splits;  // nstage: 256-K stages over kpad
  int32_t* acc;              // [M][N] workspace
};

template <int BN>
__global__ void __launch_bounds__(S4Cfg<BN>::kThreads, 1) stream4_gemm_kernel(const __grid_constant__ S4Params p) {
  using C = S4Cfg<BN>;
  constexpr int G = C::G;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring_w = smem;
  uint8_t* ring_t = smem + C::kOffT;
  uint64_t* full_w = reinterpret_cast<uint64_t*>(smem + C::kRingBytes);
  uint64_t* empty_w = full_w + C::kStagesW;
  uint64_t* full_t = empty_w + C::kStagesW;
  uint64_t* empty_t = full_t + C::kStagesT;
  uint64_t* a_full = empty_t + C::kStagesT;  // [G] widening group g -> issuer g
  uint64_t* a_empty = a_full + G;            // [G] issuer g -> widening group g
  uint64_t* acc_full = a_empty + G;          // [2] the G issuers -> epilogue
  uint64_t* acc_empty = acc_full + 2;        // [2] epilogue -> issuers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tm_w);
    tma_prefetch(&p.tm_x);
  }
  if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < C::kStagesW; ++i) { mbar_init(&full_w[i], 1); mbar_init(&empty_w[i], 4); }
      for (int i = 0; i < C::kStagesT; ++i) { mbar_init(&full_t[i], 1); mbar_init(&empty_t[i], 1); }
      for (int i = 0; i < G; ++i) { mbar_init(&a_full[i], 4); mbar_init(&a_empty[i], 1); }
      for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], G); mbar_init(&acc_empty[i], 4); }
      fence_mbar_init();
    }
    __syncwarp();
    tmem_alloc<1>(tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // K1's codes are complete

  const int tiles_n = (p.N + kBlockM - 1) / kBlockM;
  const int num_units = tiles_n * p.splits;
  // unit -> (weight block, K split); consecutive units walk the blocks of one split
  auto decode = [&](int u, int& nb, int& k0, int& k1) {
    nb = u % tiles_n;
    const int s = u / tiles_n;
    k0 = static_cast<int>((static_cast<long long>(p.nstage) * s) / p.splits);
    k1 = static_cast<int>((static_cast<long long>(p.nstage) * (s + 1)) / p.splits);
  };

  if (warp == 0 || warp == C::kIssEnd) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();  // weights stream once
      const uint64_t pol_x = policy_evict_last();   // the code tile is re-read by every block
      const bool wprod = warp == 0;
      int bc = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        int nb, k0, k1;
        decode(u, nb, k0, k1);
        for (int i = k0; i < k1; ++i, ++bc) {
          if (wprod) {
            const int st = bc % C::kStagesW;
            mbar_wait_sleep(&empty_w[st], ((bc / C::kStagesW) & 1) ^ 1);
            mbar_arrive_expect_tx(&full_w[st], kS4WBytes);
            tma_load_2d(ring_w + st * kS4WBytes, &p.tm_w, i * kKBlockBytes, nb * kBlockM, &full_w[st], pol_w);
          } else {
            const int st = bc % C::kStagesT;
            mbar_wait_sleep(&empty_t[st], ((bc / C::kStagesT) & 1) ^ 1);
            uint8_t* slot = ring_t + st * C::kSlotT;
            mbar_arrive_expect_tx(&full_t[st], C::kSlotT);
            tma_load_2d(slot, &p.tm_x, (2 * i) * kKBlockBytes, 0, &full_t[st], pol_x);
            tma_load_2d(slot + C::kTAtom, &p.tm_x, (2 * i + 1) * kKBlockBytes, 0, &full_t[st], pol_x);
          }
        }
      }
    }
  } else if (warp >= C::kEpiEnd) {
    // issuer of widening group g (whole warp converged, elected lane issues)
    const int g = warp - C::kEpiEnd;
    constexpr uint32_t idesc = idesc_make(2u, 1u, kBlockM, BN);
    int bc = 0, it = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++it) {
      int nb, k0, k1;
      decode(u, nb, k0, k1);
      const int b = it & 1;
      mbar_wait_sleep(&acc_empty[b], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + C::kAccCol + b * C::kAccBuf + g * BN;
      bool first = true;
      for (int i = k0; i < k1; ++i, ++bc) {
        if (bc % G != g) continue;
        const int st = bc % C::kStagesT;
        mbar_wait_spin(&a_full[g], (bc / G) & 1);          // A widened into TMEM
        mbar_wait(&full_t[st], (bc / C::kStagesT) & 1);    // code tile landed
        tc_fence_after();
        const uint32_t a_tm = tmem_base + g * kS4TmemA;
        const uint64_t bd0 = umma_desc_sw128(smem_u32(ring_t + st * C::kSlotT));
#pragma unroll
        for (int j = 0; j < 8; ++j)
          mma_i8_ts_e(d, a_tm + 8 * j, bd0 + (j >> 2) * (C::kTAtom >> 4) + 2 * (j & 3), idesc,
                      (first && j == 0) ? 0u : 1u);
        first = false;
        commit_e(&a_empty[g]);
        commit_e(&empty_t[st]);
      }
      commit_e(&acc_full[b]);
    }
  } else if (warp >= 2 && warp < C::kWidenEnd) {
    // widening: thread = weight row r (TMEM lane r); chunk c (16 B) holds k = 32c + i
    // (low nibble of byte i) and k = 32c + 16 + i (high nibble) -> columns 8c + q
    // (low nibbles of word q) and 8c + 4 + q (high nibbles)
    const int quad = warp & 3, g = (warp - 2) >> 2;
    const int r = quad * 32 + lane;
    const uint32_t a_tm = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + g * kS4TmemA;
    int bc = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      int nb, k0, k1;
      decode(u, nb, k0, k1);
      for (int i = k0; i < k1; ++i, ++bc) {
        if (bc % G != g) continue;
        const int st = bc % C::kStagesW;
        mbar_wait_sleep(&full_w[st], (bc / C::kStagesW) & 1);
        mbar_wait_spin(&a_empty[g], ((bc / G) & 1) ^ 1);
        tc_fence_after();
        const uint8_t* wrow = ring_w + st * kS4WBytes + r * kKBlockBytes;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          uint32_t o[32];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int c = 4 * h + cc;
            const uint4 v = *reinterpret_cast<const uint4*>(wrow + ((c ^ (r & 7)) << 4));
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t lo = w[q] & 0x0F0F0F0Fu, hi = (w[q] >> 4) & 0x0F0F0F0Fu;
              o[8 * cc + q] = lo + (lo & 0x08080808u) * 0x1Eu;  // sign-extend each nibble
              o[8 * cc + 4 + q] = hi + (hi & 0x08080808u) * 0x1Eu;
            }
          }
          tmem_st32(a_tm + 32 * h, o);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&empty_w[st]);  // weight tile consumed (the MMAs read TMEM)
          mbar_arrive(&a_full[g]);
        }
      }
    }
  } else if (warp >= C::kWidenEnd) {
    // epilogue: TMEM lane = weight row n, column = token t; sum the G accumulators
    const int quad = warp & 3;
    int it = 0, bc0 = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++it) {
      int nb, k0, k1;
      decode(u, nb, k0, k1);
      uint32_t used = 0;
      for (int k = 0; k < k1 - k0 && k < G; ++k) used |= 1u << ((bc0 + k) % G);
      bc0 += k1 - k0;
      const int b = it & 1;
      mbar_wait_sleep(&acc_full[b], (it >> 1) & 1);
      tc_fence_after();
      const int n = nb * kBlockM + quad * 32 + lane;
      const uint32_t tacc = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + C::kAccCol + b * C::kAccBuf;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        int sum[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) sum[j] = 0;
        if constexpr (BN == 16) {
          uint32_t x0[32], x1[32];  // accumulators 0/1 in columns 0-31, 2 in 32-47
          tmem_ld32(tacc, x0);
          tmem_ld32(tacc + 32, x1);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j)
            sum[j] = ((used & 1u) ? static_cast<int>(x0[j]) : 0) + ((used & 2u) ? static_cast<int>(x0[16 + j]) : 0) +
                     ((used & 4u) ? static_cast<int>(x1[j]) : 0);
        } else {
#pragma unroll 1
          for (int g = 0; g < G; ++g) {
            if (!(used & (1u << g))) continue;
            uint32_t x[32];
            tmem_ld32(tacc + g * BN + c, x);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) sum[j] += static_cast<int>(x[j]);
          }
        }
        if (n < p.N) {
#pragma unroll
          for (int j = 0; j < (BN < 32 ? BN : 32); ++j) {
            const int t = c + j;
            if (t < p.M) atomicAdd(&p.acc[static_cast<long long>(t) * p.N + n], sum[j]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, 512);
  }
}

template <int BN>
cudaError_t launch_s4(const S4Params& sp, int num_sms, cudaStream_t stream) {
  using C = S4Cfg<BN>;
  auto kern = stream4_gemm_kernel<BN>;
  cudaError_t e = ensure_smem_attr(kern, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  const int units = ((sp.N + kBlockM - 1) / kBlockM) * sp.splits;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(units < num_sms ? units : num_sms));
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, sp);
}

}  // namespace

// Measured at OPT-66B fc1 (9216 -> 36864, 256 outliers), K1 + stream + AccInit vs the
// fused kernel on INT8 tiles: M = 1 51 vs 65 us, M = 16 54 vs 65 us, M = 64 equal
// (profiles/r1_stream4.jsonl): on for 4-bit layers at M <= 32.
int gemm_stream4_auto = [] {
  const char* e = getenv("QUIK_STREAM4");
  return e ? atoi(e) : 1;
}();

cudaError_t launch_stream4_gemm(const StreamArgs& a, int num_sms, cudaStream_t stream, const char** err_msg) {
  *err_msg = nullptr;
  if (a.M == 0 || a.N == 0 || a.kpad == 0) return cudaSuccess;
  if (a.M > 64) { *err_msg = "INT4 stream GEMM: M > 64"; return cudaErrorInvalidValue; }
  if (!a.w4) { *err_msg = "INT4 stream GEMM: no INT4 weights"; return cudaErrorInvalidValue; }
  const int bn = a.M <= 16 ? 16 : (a.M <= 32 ? 32 : 64);
  S4Params sp{};
  sp.M = static_cast<int>(a.M);
  sp.N = static_cast<int>(a.N);
  sp.nstage = static_cast<int>((a.kpad + 255) / 256);
  // K splits: minimise the busiest CTA's stage count (see wo.cu)
  const long long tiles = (a.N + kBlockM - 1) / kBlockM;
  int splits = 1;
  long long best = -1;
  for (int s = 1; s <= 16 && s <= sp.nstage; ++s) {
    const long long waves = (tiles * s + num_sms - 1) / num_sms;
    const long long cost = waves * ((sp.nstage + s - 1) / s + 1);
    if (best < 0 || cost < best) { best = cost; splits = s; }
  }
  if (a.splits > 0) splits = a.splits;
  sp.splits = splits;
  sp.acc = a.acc;
  // the INT4 rows hold kpad / 2 bytes; a 256-K stage past kpad reads zeros (OOB fill)
  const CUresult r1 = encode_map_2d(&sp.tm_w, a.w4, a.kpad / 2, a.N, a.kpad / 2, kKBlockBytes, kBlockM, true);
  const CUresult r2 = encode_map_2d(&sp.tm_x, a.x, a.kpad, a.M, a.kpad, kKBlockBytes, static_cast<uint32_t>(bn), true);
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) { *err_msg = "INT4 stream GEMM: tensor map encode failed"; return cudaErrorInvalidValue; }
  switch (bn) {
    case 16: return launch_s4<16>(sp, num_sms, stream);
    case 32: return launch_s4<32>(sp, num_sms, stream);
    default: return launch_s4<64>(sp, num_sms, stream);
  }
}

}  // namespace quikb200
