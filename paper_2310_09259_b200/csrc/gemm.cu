// K2+K3+K4: the fused QUIK linear kernel for sm_100a.
//
// Computes, for one layer call (runtime.cpp:246-318, V3 path :279-303):
//   acc[n][t] = sum_k W8[n][k] * X8[t][k]                  (tcgen05 kind::i8, exact int32 in TMEM)
//   f[n][t]   = sum_o Wo[n][o] * Xo[t][o]                  (tcgen05 kind::f16, f32 in TMEM)
//   y[t][n]   = (bias[n] + f) + dequant_element(acc, ...)  (epilogue, runtime.cpp:70-77)
// "Swap-AB" orientation: weight rows are the UMMA M dimension (128 per tile),
// tokens are the UMMA N dimension (BN per tile), so small token counts use
// narrow N tiles instead of padding 128-row MMAs.
//
// Warp roles (256 threads, 1 CTA per SM, persistent over tiles):
//   warp 0      TMA producer (one elected lane)
//   warp 1      MMA issuer  (one elected lane)
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: TMEM -> registers -> dequant -> global
// Pipelines: smem ring (full/empty mbarriers, TMA <-> MMA) and a double-buffered
// TMEM accumulator (tmem_full/tmem_empty, MMA <-> epilogue).
#include <cudaTypedefs.h>

#include <mutex>

#include "kernels.h"
#include "sm100.cuh"

namespace quikb200 {

namespace {

constexpr int kThreads = 256;
constexpr int kEpiWarp0 = 4;

template <int BN>
struct Cfg {
  static constexpr int kABytes = kBlockM * kKBlockBytes;  // 16 KB
  static constexpr int kBBytes = BN * kKBlockBytes;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (200 * 1024 / kStageBytes) > 8 ? 8 : (200 * 1024 / kStageBytes);
  // Per accumulator buffer: BN int32 columns + BN f32 columns.
  static constexpr int kAccCols = 2 * BN;
  static constexpr int kAccBufs = (2 * kAccCols <= 512) ? 2 : 1;
  static constexpr int kTmemColsRaw = kAccBufs * kAccCols;
  static constexpr int kTmemCols =
      kTmemColsRaw <= 32 ? 32 : kTmemColsRaw <= 64 ? 64 : kTmemColsRaw <= 128 ? 128 : kTmemColsRaw <= 256 ? 256 : 512;
  static constexpr int kBarBytes = (2 * kStages + 2 * kAccBufs) * 8 + 16;
  static constexpr int kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes + kBarBytes;
};

struct KParams {
  CUtensorMap tm_w;   // int8 [N][kpad], box {128 B, 128 rows}
  CUtensorMap tm_x;   // int8 [M][kpad], box {128 B, BN rows}
  CUtensorMap tm_wo;  // f16 [N][opad], box {64, 128}
  CUtensorMap tm_xo;  // f16 [M][opad], box {64, BN}
  int M, N;
  int kb_int, kb_out;
  const float* w_scale;
  const float* wreduced;
  const float* bias;
  const float* a_scale;
  const float* a_zero;
  float half_range;
  void* out;
  long long ldo;
};

template <int BN, int MODE>
__global__ void __launch_bounds__(kThreads, 1) quik_gemm_kernel(const __grid_constant__ KParams p) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kAccBufs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + C::kAccBufs);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    if (p.kb_int) { tma_prefetch(&p.tm_w); tma_prefetch(&p.tm_x); }
    if (p.kb_out) { tma_prefetch(&p.tm_wo); tma_prefetch(&p.tm_xo); }
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < C::kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < C::kAccBufs; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int tiles_m = (p.M + BN - 1) / BN;
  const int tiles_n = (p.N + kBlockM - 1) / kBlockM;
  const int num_tiles = tiles_m * tiles_n;
  // Tile order: consecutive tile ids share the weight block (n) so the CTAs that
  // run concurrently read the same 128 weight rows through L2.
  const int kb_total = p.kb_int + p.kb_out;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int nb = tile / tiles_m, mb = tile % tiles_m;
        for (int kb = 0; kb < kb_total; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::kStageBytes;
          uint8_t* sb = sa + C::kABytes;
          mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
          if (kb < p.kb_int) {
            tma_load_2d(sa, &p.tm_w, kb * kKBlockBytes, nb * kBlockM, &full[stage], pol_w);
            tma_load_2d(sb, &p.tm_x, kb * kKBlockBytes, mb * BN, &full[stage], pol_x);
          } else {
            const int ko = (kb - p.kb_int) * 64;
            tma_load_2d(sa, &p.tm_wo, ko, nb * kBlockM, &full[stage], pol_w);
            tma_load_2d(sb, &p.tm_xo, ko, mb * BN, &full[stage], pol_x);
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_i8 = idesc_make(2u, 1u, kBlockM, BN);
      constexpr uint32_t id_f16 = idesc_make(1u, 0u, kBlockM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int abuf = 0;
      uint32_t aphase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[abuf], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_int = tmem_base + abuf * C::kAccCols;
        const uint32_t d_f32 = d_int + BN;
        for (int kb = 0; kb < kb_total; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t sb = sa + C::kABytes;
          const uint64_t adesc = umma_desc_sw128(sa);
          const uint64_t bdesc = umma_desc_sw128(sb);
          if (kb < p.kb_int) {
#pragma unroll
            for (int k = 0; k < 4; ++k)  // 4 x K=32 int8 = 128 bytes
              mma_i8(d_int, adesc + 2 * k, bdesc + 2 * k, id_i8, (kb | k) != 0);
          } else {
            const int ko = kb - p.kb_int;
#pragma unroll
            for (int k = 0; k < 4; ++k)  // 4 x K=16 f16 = 128 bytes
              mma_f16(d_f32, adesc + 2 * k, bdesc + 2 * k, id_f16, (ko | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[abuf]);
        if (C::kAccBufs == 2) { abuf ^= 1; if (abuf == 0) aphase ^= 1; } else { aphase ^= 1; }
      }
    }
  } else if (warp >= kEpiWarp0) {
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = q * 32 + lane;
    int abuf = 0;
    uint32_t aphase = 0;
    const bool has_int = p.kb_int > 0;
    const bool has_out = p.kb_out > 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int nb = tile / tiles_m, mb = tile % tiles_m;
      const int n = nb * kBlockM + row;
      const bool n_ok = n < p.N;
      float sw = 0.f, wr = 0.f, bs = 0.f;
      if (n_ok) {
        if (MODE == kModeF32 || MODE == kModeF16) { sw = __ldg(&p.w_scale[n]); wr = __ldg(&p.wreduced[n]); }
        if (MODE != kModeInt32 && p.bias) bs = __ldg(&p.bias[n]);
      }
      mbar_wait(&tfull[abuf], aphase);
      tc_fence_after();
      const uint32_t t_int = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + abuf * C::kAccCols;
      const uint32_t t_f32 = t_int + BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t vi[32], vf[32];
        if (MODE != kModeOutlierF32) {
          if (has_int) tmem_ld32(t_int + c, vi);
          else {
#pragma unroll
            for (int j = 0; j < 32; ++j) vi[j] = 0u;
          }
        }
        if (MODE != kModeInt32) {
          if (has_out) tmem_ld32(t_f32 + c, vf);
          else {
#pragma unroll
            for (int j = 0; j < 32; ++j) vf[j] = 0u;
          }
        }
        tmem_ld_wait();
        const int t0 = mb * BN + c;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int t = t0 + j;
          if (t >= p.M) continue;
          const long long off = static_cast<long long>(t) * p.ldo + n;
          if (MODE == kModeInt32) {
            if (n_ok) reinterpret_cast<int32_t*>(p.out)[off] = static_cast<int32_t>(vi[j]);
          } else {
            // orow = fp_linear(...) = bias + sum_o x_o w_o   (runtime.cpp:96-113)
            float o = bs;
            if (has_out) o = __fadd_rn(o, __uint_as_float(vf[j]));
            if (MODE != kModeOutlierF32) {
              const float sa = __ldg(&p.a_scale[t]);
              const float za = __ldg(&p.a_zero[t]);
              // dequant_element, runtime.cpp:70-77, op by op (no contraction)
              float v = __fmul_rn(__int2float_rn(static_cast<int32_t>(vi[j])), sa);
              v = __fmul_rn(v, sw);
              float sh = __fadd_rn(za, __fmul_rn(p.half_range, sa));
              sh = __fmul_rn(sh, wr);
              o = __fadd_rn(o, __fadd_rn(v, sh));  // runtime.cpp:298-299
            }
            if (n_ok) {
              if (MODE == kModeF16) reinterpret_cast<__half*>(p.out)[off] = __float2half_rn(o);
              else reinterpret_cast<float*>(p.out)[off] = o;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[abuf]);
      if (C::kAccBufs == 2) { abuf ^= 1; if (abuf == 0) aphase ^= 1; } else { aphase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// --------------------------------------------------------------------- host side

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

bool get_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

// 2D K-major tile map with 128-byte swizzle. inner = elements per row (logical
// extent), pitch in bytes, box = {box_inner elements (128 B), box_rows}.
bool make_map(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, uint64_t inner,
              uint64_t rows, uint64_t pitch_bytes, uint32_t box_rows) {
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kKBlockBytes / elem_bytes), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int MODE>
cudaError_t launch_bn_mode(const KParams& kp, int num_sms, cudaStream_t stream) {
  using C = Cfg<BN>;
  auto kern = quik_gemm_kernel<BN, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  const int tiles = static_cast<int>(((kp.M + BN - 1) / BN) * ((kp.N + kBlockM - 1) / kBlockM));
  const int grid = tiles < num_sms ? tiles : num_sms;
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, kThreads, C::kSmemBytes, stream>>>(kp);
  return cudaGetLastError();
}

template <int BN>
cudaError_t launch_bn(const KParams& kp, int mode, int num_sms, cudaStream_t stream) {
  switch (mode) {
    case kModeInt32: return launch_bn_mode<BN, kModeInt32>(kp, num_sms, stream);
    case kModeOutlierF32: return launch_bn_mode<BN, kModeOutlierF32>(kp, num_sms, stream);
    case kModeF32: return launch_bn_mode<BN, kModeF32>(kp, num_sms, stream);
    default: return launch_bn_mode<BN, kModeF16>(kp, num_sms, stream);
  }
}

}  // namespace

cudaError_t launch_quik_gemm(const GemmArgs& a, int num_sms, cudaStream_t stream, const char** err_msg) {
  *err_msg = nullptr;
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  if (!get_encoder()) { *err_msg = "cuTensorMapEncodeTiled unavailable"; return cudaErrorNotSupported; }
  // Token tile: the narrowest legal UMMA N that covers M (<=128), else 128.
  int bn = 128;
  if (a.M <= 32) bn = 32;
  else if (a.M <= 64) bn = 64;

  KParams kp{};
  kp.M = static_cast<int>(a.M);
  kp.N = static_cast<int>(a.N);
  kp.kb_int = static_cast<int>(a.kpad / kKBlockBytes);
  kp.kb_out = static_cast<int>(a.opad / 64);
  if (a.mode == kModeInt32) kp.kb_out = 0;
  if (a.mode == kModeOutlierF32) kp.kb_int = 0;
  if (kp.kb_int) {
    if (!make_map(&kp.tm_w, a.w, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.kpad, a.N, a.kpad, kBlockM) ||
        !make_map(&kp.tm_x, a.x, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.kpad, a.M, a.kpad, bn)) {
      *err_msg = "tensor map encode failed (int8 operands)";
      return cudaErrorInvalidValue;
    }
  }
  if (kp.kb_out) {
    if (!make_map(&kp.tm_wo, a.wo, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.opad, a.N, a.opad * 2, kBlockM) ||
        !make_map(&kp.tm_xo, a.xo, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.opad, a.M, a.opad * 2, bn)) {
      *err_msg = "tensor map encode failed (outlier operands)";
      return cudaErrorInvalidValue;
    }
  }
  kp.w_scale = a.w_scale;
  kp.wreduced = a.wreduced;
  kp.bias = a.bias;
  kp.a_scale = a.a_scale;
  kp.a_zero = a.a_zero;
  kp.half_range = a.half_range;
  kp.out = a.out;
  kp.ldo = a.ldo;
  switch (bn) {
    case 32: return launch_bn<32>(kp, a.mode, num_sms, stream);
    case 64: return launch_bn<64>(kp, a.mode, num_sms, stream);
    default: return launch_bn<128>(kp, a.mode, num_sms, stream);
  }
}

}  // namespace quikb200
