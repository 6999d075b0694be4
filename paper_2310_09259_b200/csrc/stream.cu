// Weight-streaming integer GEMM for small token counts (M <= 64): the regime where
// the layer is bound by reading the weights from HBM, not by the tensor cores
// (HBM-bound for M <~ 160; cfg1, cfg4 small M).
//
//   acc_ws[t][n] += sum_{k in split} W[n][k] * X8[t][k]      (red.global.add.s32)
//
// Work units are (weight block of 128 rows, K split), so even a 4096-row layer
// (32 blocks) keeps all 148 SMs streaming. INT4 layers stream the packed 4-bit
// weights (half the bytes of the INT8 copy): the producer TMA-loads each 128 x 128-K
// tile (8 KB) into a deep ring, four transform warps widen it to the swizzled INT8
// operand tile in one of three small buffers, the MMA warp issues tcgen05.mma kind::i8
// (M = 128, N = BN tokens) into a double-buffered TMEM accumulator, and four epilogue
// warps add the partial accumulators into the int32 workspace (exact: integer adds
// commute). The dequantisation epilogue + f16 outlier MMAs then run as the fused
// kernel's AccInit mode reading the workspace (bit-identical to the V3 forward,
// same arithmetic), which also clears the workspace for the next call.
//
// Warp roles (320 threads, 1 CTA per SM, persistent over units):
//   warp 0 TMA producer, warp 1 MMA issuer + TMEM allocator, warps 2-5 INT4 widening,
//   warps 6-9 epilogue (TMEM lane quadrant = warp % 4).
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"

namespace quikb200 {

namespace {

constexpr int kSThreads = 320;
// One stage = kKAtoms 128-byte K atoms (128 logical K each). INT8 weights: 1 atom
// (128 rows x 128 B). INT4 weights: 2 atoms, so that every weight row contributes one
// 128-byte segment per TMA box (the stream is bound by TMA row segments per second
// as much as by bytes: 64-byte segments ran at the same stage rate as 128-byte ones).
// widened INT8 atoms (16 KB each): the transform -> MMA -> commit -> transform cycle of
// one buffer includes the commit-arrival latency, so several are kept in flight
constexpr int kSA8Bufs = 6;
constexpr int kAtomBytes = kBlockM * kKBlockBytes;    // 16 KB: 128 rows x 128 B

template <int BN, bool W4>
struct SCfg {
  static constexpr int kKAtoms = W4 ? 2 : 1;
  static constexpr int kBAtomBytes = BN * kKBlockBytes;
  static constexpr int kBBytes = kKAtoms * kBAtomBytes;             // token tiles of one stage
  static constexpr int kABytes = kAtomBytes;                        // INT4: 128 rows x 128 B = 256 K
  static constexpr int kSlotBytes = kABytes + kBBytes;
  static constexpr int kA8Total = W4 ? kSA8Bufs * kAtomBytes : 0;
  static constexpr int kBudget = 227 * 1024 - 2048 - kA8Total;
  static constexpr int kStages = (kBudget / kSlotBytes) > 12 ? 12 : (kBudget / kSlotBytes);
  static constexpr int kBarBytes = (2 * kStages + 2 * kSA8Bufs + 4) * 8 + 16;
  static constexpr int kSmemBytes = 1024 + kA8Total + kStages * kSlotBytes + kBarBytes;
  static constexpr int kTmemCols = 2 * BN < 64 ? 64 : 2 * BN;  // 32-column TMEM loads stay in range
};

struct SParams {
  CUtensorMap tm_w;  // W4: int4 [N][kpad / 2] box {64 B, 128}; else int8 [N][kpad] box {128 B, 128} SW128
  CUtensorMap tm_x;  // int8 [M][kpad], box {128 B, BN}, SW128
  int M, N, kb_total, splits;  // kb_total: stages (K / (128 * kKAtoms))
  int32_t* acc;      // [M][N] workspace
  long long* trace;  // diagnostics (QUIK_STREAM_TRACE): CTA 0, per stage g < 256: [g][4]
};
__device__ __forceinline__ long long s_gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int BN, bool W4>
__global__ void __launch_bounds__(kSThreads, 1) stream_gemm_kernel(const __grid_constant__ SParams p) {
  using C = SCfg<BN, W4>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* a8 = smem;                         // [kSA8Bufs][16 KB] (W4)
  uint8_t* ring = smem + C::kA8Total;         // [kStages][slot]: (A4 | A8) then B
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + C::kStages * C::kSlotBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* a8_full = empty + C::kStages;     // transform -> MMA
  uint64_t* a8_empty = a8_full + kSA8Bufs;    // MMA -> transform
  uint64_t* acc_full = a8_empty + kSA8Bufs;   // [2] MMA -> epilogue
  uint64_t* acc_empty = acc_full + 2;         // [2] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tm_w);
    tma_prefetch(&p.tm_x);
  }
  if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < C::kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
      for (int i = 0; i < kSA8Bufs; ++i) { mbar_init(&a8_full[i], 1); mbar_init(&a8_empty[i], 1); }
      for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 4); }
      fence_mbar_init();
    }
    __syncwarp();
    tmem_alloc<1>(tmem_slot, C::kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: K1's codes are complete

  const int tiles_n = (p.N + kBlockM - 1) / kBlockM;
  const int num_units = tiles_n * p.splits;
  // unit u -> (weight block, split); consecutive units walk the blocks of one split
  auto krange = [&](int u, int& nb, int& k0, int& k1) {
    nb = u % tiles_n;
    const int s = u / tiles_n;
    k0 = static_cast<int>((static_cast<long long>(p.kb_total) * s) / p.splits);
    k1 = static_cast<int>((static_cast<long long>(p.kb_total) * (s + 1)) / p.splits);
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();  // weights are streamed once
      const uint64_t pol_x = policy_evict_last();   // the token tile is re-read by every unit
      int stage = 0;
      uint32_t phase = 0;
      int gcount = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        int nb, k0, k1;
        krange(u, nb, k0, k1);
        for (int kb = k0; kb < k1; ++kb, ++gcount) {
          mbar_wait_sleep(&empty[stage], phase ^ 1);
          if (p.trace && blockIdx.x == 0 && gcount < 256) p.trace[gcount * 4 + 0] = s_gtime();
          uint8_t* slot = ring + stage * C::kSlotBytes;
          mbar_arrive_expect_tx(&full[stage], C::kSlotBytes);
          tma_load_2d(slot, &p.tm_w, kb * kKBlockBytes, nb * kBlockM, &full[stage], pol_w);
#pragma unroll
          for (int a = 0; a < C::kKAtoms; ++a)
            tma_load_2d(slot + C::kABytes + a * C::kBAtomBytes, &p.tm_x, (kb * C::kKAtoms + a) * kKBlockBytes, 0,
                        &full[stage], pol_x);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_make(2u, 1u, kBlockM, BN);
      int stage = 0, ab = 0;
      uint32_t phase = 0, aphase = 0;
      int it = 0, gcount = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++it) {
        int nb, k0, k1;
        krange(u, nb, k0, k1);
        const int b = it & 1;
        mbar_wait_sleep(&acc_empty[b], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + b * BN;
        for (int kb = k0; kb < k1; ++kb, ++gcount) {
          uint8_t* slot = ring + stage * C::kSlotBytes;
          if constexpr (!W4) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
          }
#pragma unroll
          for (int a = 0; a < C::kKAtoms; ++a) {
            uint32_t a_addr = smem_u32(slot);
            if constexpr (W4) {
              mbar_wait_spin(&a8_full[ab], aphase);  // widened (implies the slot's B tiles landed)
              tc_fence_after();
              a_addr = smem_u32(a8 + ab * kAtomBytes);
            }
            const uint64_t ad = umma_desc_sw128(a_addr);
            const uint64_t bd = umma_desc_sw128(smem_u32(slot + C::kABytes + a * C::kBAtomBytes));
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_i8<1>(d, ad + 2 * k, bd + 2 * k, idesc, (kb != k0 || a || k) ? 1u : 0u);
            if constexpr (W4) {
              mma_commit<1>(&a8_empty[ab]);
              if (++ab == kSA8Bufs) { ab = 0; aphase ^= 1; }
            }
          }
          mma_commit<1>(&empty[stage]);
          if (p.trace && blockIdx.x == 0 && gcount < 256) p.trace[gcount * 4 + 3] = s_gtime();
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        mma_commit<1>(&acc_full[b]);
      }
    }
  } else if (warp >= 2 && warp <= 5) {
    if constexpr (W4) {
      // widening: ring slot's 4-bit tile -> INT8 buffer, SWIZZLE_128B layout (byte i of
      // input chunk c: k = 32c + i low nibble, k = 32c + 16 + i high nibble). Each warp
      // owns every 4th stage, so four stages are widened concurrently (one warp alone
      // is latency-bound: loads -> ALU -> stores -> proxy fence per stage).
      const int w = warp - 2;
      long long total = 0;  // K blocks this CTA streams
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        int nb, k0, k1;
        krange(u, nb, k0, k1);
        total += k1 - k0;
      }
      // atoms: g = 2 * stage_counter + half; warp w widens atoms g = w, w + 4, ...
      for (long long g = w; g < 2 * total; g += 4) {
        const long long sc = g >> 1;
        const int half = static_cast<int>(g & 1);
        const int stage = static_cast<int>(sc % C::kStages);
        const uint32_t phase = static_cast<uint32_t>((sc / C::kStages) & 1);
        const int ab = static_cast<int>(g % kSA8Bufs);
        const uint32_t aphase = static_cast<uint32_t>((g / kSA8Bufs) & 1);
        mbar_wait_sleep(&full[stage], phase);
        mbar_wait_spin(&a8_empty[ab], aphase ^ 1);
        if (p.trace && blockIdx.x == 0 && sc < 256 && lane == 0 && half == 1) p.trace[sc * 4 + 1] = s_gtime();
        // input: 128 rows x 64 B (chunks 4*half .. 4*half+3 of the 128-byte row)
        const uint8_t* s4 = ring + stage * C::kSlotBytes + half * 64;
        uint8_t* dst = a8 + ab * kAtomBytes;
#pragma unroll 1
        for (int part = 0; part < 2; ++part) {
          uint4 win[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int item = lane + (part * 8 + i) * 32;  // 512 = 128 rows x 4 chunks
            win[i] = *reinterpret_cast<const uint4*>(s4 + (item >> 2) * kKBlockBytes + (item & 3) * 16);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int item = lane + (part * 8 + i) * 32;
            const int r = item >> 2, c = item & 3;
            uint32_t lo[4], hi[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t v = (&win[i].x)[q];
              const uint32_t l = v & 0x0F0F0F0Fu, h = (v >> 4) & 0x0F0F0F0Fu;
              lo[q] = l + (l & 0x08080808u) * 0x1Eu;  // sign-extend each 4-bit value to 8 bits
              hi[q] = h + (h & 0x08080808u) * 0x1Eu;
            }
            uint8_t* row = dst + r * kKBlockBytes;
            *reinterpret_cast<uint4*>(row + (((2 * c) ^ (r & 7)) << 4)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            *reinterpret_cast<uint4*>(row + (((2 * c + 1) ^ (r & 7)) << 4)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a8_full[ab]);
        if (p.trace && blockIdx.x == 0 && sc < 256 && lane == 0 && half == 1) p.trace[sc * 4 + 2] = s_gtime();
      }
    }
  } else {
    // epilogue: TMEM lane = weight row n, column = token t -> red.add into acc[t][n]
    const int q = warp & 3;
    int it = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++it) {
      int nb, k0, k1;
      krange(u, nb, k0, k1);
      const int b = it & 1;
      mbar_wait_sleep(&acc_full[b], (it >> 1) & 1);
      tc_fence_after();
      const int n = nb * kBlockM + q * 32 + lane;
      const uint32_t tacc = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + b * BN;
#pragma unroll
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        tmem_ld32(tacc + c, v);
        tmem_ld_wait();
        if (n < p.N) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int t = c + j;
            if (t < p.M && (BN >= 32 || j < BN)) atomicAdd(&p.acc[static_cast<long long>(t) * p.N + n], static_cast<int>(v[j]));
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
    tmem_dealloc<1>(tmem_base, C::kTmemCols);
  }
}

template <int BN, bool W4>
cudaError_t launch_stream_t(const SParams& sp, int num_sms, cudaStream_t stream) {
  using C = SCfg<BN, W4>;
  auto kern = stream_gemm_kernel<BN, W4>;
  cudaError_t e = ensure_smem_attr(kern, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  const int units = ((sp.N + kBlockM - 1) / kBlockM) * sp.splits;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(units < num_sms ? units : num_sms));
  cfg.blockDim = dim3(kSThreads);
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

// Off by default: correct (bit-identical to the fused path, tested) but not yet faster.
// Measured at OPT-66B fc1, M = 16: INT8 stream 58 us (5.8 TB/s, HBM-bound), INT4 stream
// 52-54 us (widening-bound: 0.64 us per 16 KB atom per warp, 4 warps, and a ~1.5 us
// transform -> MMA -> commit hand-off lag), + 16 us AccInit epilogue, vs 60 us for the
// fused 1-CTA kernel reading INT8 weights. Next: more widening warps, B tiles copied out
// of the ring so slots free after widening, the f16 outlier MMAs inside this kernel.
int gemm_stream = 0;
int gemm_w4_stream = 1;

cudaError_t launch_stream_gemm(const StreamArgs& a, int num_sms, cudaStream_t stream, const char** err_msg) {
  *err_msg = nullptr;
  if (a.M == 0 || a.N == 0 || a.kpad == 0) return cudaSuccess;
  if (a.M > 64) { *err_msg = "stream GEMM: M > 64"; return cudaErrorInvalidValue; }
  const bool w4 = a.w4 != nullptr && a.kpad % (2 * kKBlockBytes) == 0;  // INT4 stages span 256 K
  const int bn = a.M <= 16 ? 16 : (a.M <= 32 ? 32 : 64);
  SParams sp{};
  sp.M = static_cast<int>(a.M);
  sp.N = static_cast<int>(a.N);
  sp.kb_total = static_cast<int>(a.kpad / (kKBlockBytes * (w4 ? 2 : 1)));
  // K splits: enough units to keep every SM streaming (>= 2 per SM), each >= 4 K blocks
  const int tiles_n = static_cast<int>((a.N + kBlockM - 1) / kBlockM);
  int splits = 1;
  while (tiles_n * splits < 2 * num_sms && sp.kb_total / (splits * 2) >= 4) splits *= 2;
  if (a.splits > 0) splits = a.splits;
  sp.splits = splits;
  sp.acc = a.acc;
  static const char* trace_path = getenv("QUIK_STREAM_TRACE");
  static long long* trace_buf = nullptr;
  if (trace_path) {
    if (!trace_buf) cudaMalloc(&trace_buf, 256 * 4 * 8);
    cudaMemsetAsync(trace_buf, 0, 256 * 4 * 8, stream);
    sp.trace = trace_buf;
  }
  const CUresult r1 =
      w4 ? encode_map_2d(&sp.tm_w, a.w4, a.kpad / 2, a.N, a.kpad / 2, kKBlockBytes, kBlockM, false)
         : encode_map_2d(&sp.tm_w, a.w8, a.kpad, a.N, a.kpad, kKBlockBytes, kBlockM, true);
  const CUresult r2 = encode_map_2d(&sp.tm_x, a.x, a.kpad, a.M, a.kpad, kKBlockBytes, static_cast<uint32_t>(bn), true);
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) { *err_msg = "stream GEMM: tensor map encode failed"; return cudaErrorInvalidValue; }
  if (trace_path) {
    cudaError_t e = cudaSuccess;
    switch (bn * 2 + (w4 ? 1 : 0)) {
      case 32: e = launch_stream_t<16, false>(sp, num_sms, stream); break;
      case 33: e = launch_stream_t<16, true>(sp, num_sms, stream); break;
      case 64: e = launch_stream_t<32, false>(sp, num_sms, stream); break;
      case 65: e = launch_stream_t<32, true>(sp, num_sms, stream); break;
      case 128: e = launch_stream_t<64, false>(sp, num_sms, stream); break;
      default: e = launch_stream_t<64, true>(sp, num_sms, stream); break;
    }
    long long h[1024];
    cudaStreamSynchronize(stream);
    cudaMemcpy(h, trace_buf, sizeof(h), cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(trace_path, "wb")) {
      fwrite(h, 8, 1024, f);
      fclose(f);
    }
    return e;
  }
  switch (bn * 2 + (w4 ? 1 : 0)) {
    case 32: return launch_stream_t<16, false>(sp, num_sms, stream);
    case 33: return launch_stream_t<16, true>(sp, num_sms, stream);
    case 64: return launch_stream_t<32, false>(sp, num_sms, stream);
    case 65: return launch_stream_t<32, true>(sp, num_sms, stream);
    case 128: return launch_stream_t<64, false>(sp, num_sms, stream);
    default: return launch_stream_t<64, true>(sp, num_sms, stream);
  }
}

}  // namespace quikb200
