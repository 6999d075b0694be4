// K1: fused activation split + per-token asymmetric quantisation, plus the small
// layout kernels (ABI unpack, f32->f16, stand-alone dequantisation epilogue).
//
// Numerics contract (reference runtime.cpp:36-66, SPEC.md runtime module):
//   vmin/vmax over the base columns in permutation order, first element seeds,
//   strict < / > (the first of several equal extrema wins; matters only for the
//   sign of a zero minimum); non-finite base value -> NumericalError (device flag);
//   range = vmax - vmin; scale = range == 0 ? 1 : range / (2^b - 1) (IEEE div);
//   q = lround((v - vmin) / scale) (ties away from zero); stored = clamp(q - hr,
//   -hr, hr - 1). Every FP op is an explicit _rn intrinsic, so the result is
//   bit-identical to the reference compiled with -ffp-contract=off.
#include <cfloat>

#include "kernels.h"
#include "sm100.cuh"

namespace quikb200 {

namespace {

constexpr int kQThreads = 256;
constexpr int kGroup = 16;  // base positions per thread per step (one 16-byte int8 store)

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }

struct MinMax {
  float vmin, vmax;
  int imin, imax;  // column index of the extremum (first-seen tie-break)
  int nonfinite;
};

// Combines two partial reductions; on equal values the lower column index wins,
// which reproduces the sequential "first element seeds, strict < / >" scan.
__device__ __forceinline__ void mm_combine(MinMax& a, float vmin, int imin, float vmax, int imax, int nf) {
  if (vmin < a.vmin || (vmin == a.vmin && imin < a.imin)) { a.vmin = vmin; a.imin = imin; }
  if (vmax > a.vmax || (vmax == a.vmax && imax < a.imax)) { a.vmax = vmax; a.imax = imax; }
  a.nonfinite |= nf;
}

// One CTA per token row. The row is staged in shared memory with 16-byte loads;
// base positions are processed 16 at a time per thread (perm gather from smem).
template <typename T, int BITS>
__global__ void __launch_bounds__(kQThreads) quantize_rows_kernel(const QuantArgs a) {
  extern __shared__ __align__(16) uint8_t smem_q[];
  T* row = reinterpret_cast<T*>(smem_q);
  __shared__ MinMax red[kQThreads / 32];
  __shared__ float s_scale, s_zero;

  const int64_t t = blockIdx.x;
  const T* src = reinterpret_cast<const T*>(a.x) + t * a.ldx;
  const int tid = threadIdx.x;

  // ---- stage the row (vectorised when 16-byte aligned)
  constexpr int kVec = 16 / sizeof(T);
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && (a.K % kVec == 0);
  if (vec_ok) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(row);
    for (int64_t i = tid; i < a.K / kVec; i += kQThreads) d4[i] = __ldg(&s4[i]);
  } else {
    for (int64_t i = tid; i < a.K; i += kQThreads) row[i] = src[i];
  }
  __syncthreads();

  // ---- pass 1: min / max over base columns (+ finiteness)
  MinMax mm{FLT_MAX, -FLT_MAX, INT_MAX, INT_MAX, 0};
  bool any = false;
  for (int64_t j0 = static_cast<int64_t>(tid) * kGroup; j0 < a.kb; j0 += kQThreads * kGroup) {
    const int jn = static_cast<int>(a.kb - j0 < kGroup ? a.kb - j0 : kGroup);
    for (int u = 0; u < jn; ++u) {
      const int c = __ldg(&a.base_src[j0 + u]);
      const float v = to_f32<T>(row[c]);
      if (!isfinite(v)) mm.nonfinite = 1;
      if (!any) { mm.vmin = mm.vmax = v; mm.imin = mm.imax = c; any = true; }
      else {
        if (v < mm.vmin) { mm.vmin = v; mm.imin = c; }
        if (v > mm.vmax) { mm.vmax = v; mm.imax = c; }
      }
    }
  }
  // warp reduce
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float vmin = __shfl_xor_sync(0xffffffffu, mm.vmin, off);
    const float vmax = __shfl_xor_sync(0xffffffffu, mm.vmax, off);
    const int imin = __shfl_xor_sync(0xffffffffu, mm.imin, off);
    const int imax = __shfl_xor_sync(0xffffffffu, mm.imax, off);
    const int nf = __shfl_xor_sync(0xffffffffu, mm.nonfinite, off);
    mm_combine(mm, vmin, imin, vmax, imax, nf);
  }
  if ((tid & 31) == 0) red[tid >> 5] = mm;
  __syncthreads();
  if (tid == 0) {
    MinMax r = red[0];
    for (int w = 1; w < kQThreads / 32; ++w) mm_combine(r, red[w].vmin, red[w].imin, red[w].vmax, red[w].imax, red[w].nonfinite);
    if (r.nonfinite && a.err) atomicExch(a.err, 1);
    // The seeded min/max hold the actual values of the winning columns
    // (re-read so the sign of a zero extremum is the first-seen one).
    float vmin = 0.f, vmax = 0.f;
    if (a.kb > 0) { vmin = to_f32<T>(row[r.imin]); vmax = to_f32<T>(row[r.imax]); }
    const float range = __fsub_rn(vmax, vmin);
    constexpr float kLevels = static_cast<float>((1 << BITS) - 1);
    const float scale = range == 0.0f ? 1.0f : __fdiv_rn(range, kLevels);
    s_scale = scale;
    s_zero = vmin;
    a.scale[t] = scale;
    a.zero[t] = vmin;
  }
  __syncthreads();
  const float vmin = s_zero, scale = s_scale;
  constexpr int kHr = 1 << (BITS - 1);

  // ---- pass 2: quantise + pack
  const int64_t kend = a.q8 ? a.kpad : a.kb;
  uint8_t* prow = a.packed ? a.packed + t * (BITS == 4 ? (a.kb + 1) / 2 : a.kb) : nullptr;
  for (int64_t j0 = static_cast<int64_t>(tid) * kGroup; j0 < kend; j0 += kQThreads * kGroup) {
    int8_t code[kGroup];
#pragma unroll
    for (int u = 0; u < kGroup; ++u) {
      const int64_t j = j0 + u;
      int s = 0;
      if (j < a.kb) {
        const float v = to_f32<T>(row[__ldg(&a.base_src[j])]);
        const float qf = round_half_away(__fdiv_rn(__fsub_rn(v, vmin), scale));
        int q = static_cast<int>(fminf(fmaxf(qf, -1.0e6f), 1.0e6f));  // NaN-safe bound; NaN rows are flagged
        s = q - kHr;
        s = s < -kHr ? -kHr : (s > kHr - 1 ? kHr - 1 : s);
      }
      code[u] = static_cast<int8_t>(s);
    }
    if (a.q8) {
      uint4 v;
      memcpy(&v, code, 16);
      *reinterpret_cast<uint4*>(a.q8 + t * a.kpad + j0) = v;
    }
    if (prow) {
      const int jn = static_cast<int>(a.kb - j0 < kGroup ? a.kb - j0 : kGroup);
      if (BITS == 8) {
        for (int u = 0; u < jn; ++u) prow[j0 + u] = static_cast<uint8_t>(code[u]);
      } else {
        // i4p: low nibble = even base index, stored + 8; pad nibble of odd rows = 0
        for (int u = 0; u < jn; u += 2) {
          const uint8_t lo = static_cast<uint8_t>(code[u] + 8) & 0xF;
          const uint8_t hi = (u + 1 < jn) ? (static_cast<uint8_t>(code[u + 1] + 8) & 0xF) : 0;
          prow[(j0 + u) / 2] = static_cast<uint8_t>(lo | (hi << 4));
        }
      }
    }
  }

  // ---- outlier gather (ascending index order, runtime.cpp:217)
  if (a.xo16) {
    for (int64_t i = tid; i < a.opad; i += kQThreads) {
      const float v = i < a.n_out ? to_f32<T>(row[__ldg(&a.out_src[i])]) : 0.0f;
      a.xo16[t * a.opad + i] = __float2half_rn(v);
    }
  }
  if (a.xo32) {
    for (int64_t i = tid; i < a.n_out; i += kQThreads) a.xo32[t * a.n_out + i] = to_f32<T>(row[__ldg(&a.out_src[i])]);
  }
}

__global__ void split_kernel(const SplitArgs a) {
  const int64_t t = blockIdx.y;
  for (int64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < a.kb + a.opad; j += gridDim.x * blockDim.x) {
    if (j < a.kb) {
      const int64_t c = a.base_src[j];
      a.xbase[t * a.kb + j] = a.x_is_f32 ? reinterpret_cast<const float*>(a.x)[t * a.ldx + c]
                                         : __half2float(reinterpret_cast<const __half*>(a.x)[t * a.ldx + c]);
    } else if (a.xo16) {
      const int64_t i = j - a.kb;
      float v = 0.0f;
      if (i < a.n_out) {
        const int64_t c = a.out_src[i];
        v = a.x_is_f32 ? reinterpret_cast<const float*>(a.x)[t * a.ldx + c]
                       : __half2float(reinterpret_cast<const __half*>(a.x)[t * a.ldx + c]);
      }
      a.xo16[t * a.opad + i] = __float2half_rn(v);
    }
  }
}

__global__ void unpack_kernel(const uint8_t* __restrict__ packed, int64_t rows, int64_t cols, int bits,
                              int8_t* __restrict__ dst, int64_t kpad) {
  const int64_t r = blockIdx.y;
  const int64_t rb = bits == 4 ? (cols + 1) / 2 : cols;
  const uint8_t* src = packed + r * rb;
  for (int64_t c = blockIdx.x * blockDim.x + threadIdx.x; c < kpad; c += gridDim.x * blockDim.x) {
    int8_t v = 0;
    if (c < cols) {
      if (bits == 8) v = static_cast<int8_t>(src[c]);
      else {
        const uint8_t b = src[c / 2];
        v = static_cast<int8_t>(static_cast<int>((c & 1) ? (b >> 4) : (b & 0xF)) - 8);
      }
    }
    dst[r * kpad + c] = v;
  }
}

__global__ void f32_to_f16_kernel(const float* __restrict__ src, int64_t rows, int64_t cols,
                                  __half* __restrict__ dst, int64_t pitch) {
  const int64_t r = blockIdx.y;
  for (int64_t c = blockIdx.x * blockDim.x + threadIdx.x; c < pitch; c += gridDim.x * blockDim.x)
    dst[r * pitch + c] = __float2half_rn(c < cols ? src[r * cols + c] : 0.0f);
}

__device__ __forceinline__ float dequant_element(int32_t acc, float sa, float sw, float za, float hr, float wr) {
  float v = __fmul_rn(__int2float_rn(acc), sa);
  v = __fmul_rn(v, sw);
  float shift = __fadd_rn(za, __fmul_rn(hr, sa));
  shift = __fmul_rn(shift, wr);
  return __fadd_rn(v, shift);
}

__global__ void dequant_kernel(const int32_t* __restrict__ acc, int64_t M, int64_t N, const float* __restrict__ sa,
                               const float* __restrict__ za, float hr, const float* __restrict__ sw,
                               const float* __restrict__ wr, const float* __restrict__ fp_part, void* out,
                               int out_kind /*0 f32 deq only, 1 f32 add, 2 f16 add*/) {
  const int64_t t = blockIdx.y;
  for (int64_t r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    const int64_t i = t * N + r;
    const float d = dequant_element(acc[i], sa[t], sw[r], za[t], hr, wr[r]);
    if (out_kind == 0) reinterpret_cast<float*>(out)[i] = d;
    else {
      const float o = __fadd_rn(fp_part[i], d);  // runtime.cpp:314
      if (out_kind == 1) reinterpret_cast<float*>(out)[i] = o;
      else reinterpret_cast<__half*>(out)[i] = __float2half_rn(o);
    }
  }
}

dim3 grid2(int64_t cols, int64_t rows) {
  int64_t gx = (cols + 255) / 256;
  if (gx > 64) gx = 64;
  if (gx < 1) gx = 1;
  return dim3(static_cast<unsigned>(gx), static_cast<unsigned>(rows));
}

}  // namespace

cudaError_t launch_quantize(const QuantArgs& a, cudaStream_t stream) {
  if (a.M == 0) return cudaSuccess;
  const size_t smem = static_cast<size_t>(a.K) * (a.x_is_f32 ? 4 : 2) + 16;
  cudaError_t e;
#define QUIK_Q_LAUNCH(T, B)                                                                           \
  do {                                                                                                \
    e = cudaFuncSetAttribute(quantize_rows_kernel<T, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             static_cast<int>(smem));                                                 \
    if (e != cudaSuccess) return e;                                                                   \
    quantize_rows_kernel<T, B><<<static_cast<unsigned>(a.M), kQThreads, smem, stream>>>(a);          \
  } while (0)
  if (a.x_is_f32) {
    if (a.bits == 4) QUIK_Q_LAUNCH(float, 4); else QUIK_Q_LAUNCH(float, 8);
  } else {
    if (a.bits == 4) QUIK_Q_LAUNCH(__half, 4); else QUIK_Q_LAUNCH(__half, 8);
  }
#undef QUIK_Q_LAUNCH
  return cudaGetLastError();
}

cudaError_t launch_split(const SplitArgs& a, cudaStream_t stream) {
  if (a.M == 0 || a.kb + a.opad == 0) return cudaSuccess;
  split_kernel<<<grid2(a.kb + a.opad, a.M), 256, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_unpack_to_gemm(const uint8_t* packed, int64_t rows, int64_t cols, int bits, int8_t* dst,
                                  int64_t kpad, cudaStream_t stream) {
  if (rows == 0 || kpad == 0) return cudaSuccess;
  unpack_kernel<<<grid2(kpad, rows), 256, 0, stream>>>(packed, rows, cols, bits, dst, kpad);
  return cudaGetLastError();
}

cudaError_t launch_f32_to_f16_padded(const float* src, int64_t rows, int64_t cols, __half* dst, int64_t pitch,
                                     cudaStream_t stream) {
  if (rows == 0 || pitch == 0) return cudaSuccess;
  f32_to_f16_kernel<<<grid2(pitch, rows), 256, 0, stream>>>(src, rows, cols, dst, pitch);
  return cudaGetLastError();
}

cudaError_t launch_dequant(const int32_t* acc, int64_t M, int64_t N, const float* a_scale, const float* a_zero,
                           float half_range, const float* w_scale, const float* wreduced, float* out,
                           cudaStream_t stream) {
  if (M == 0 || N == 0) return cudaSuccess;
  dequant_kernel<<<grid2(N, M), 256, 0, stream>>>(acc, M, N, a_scale, a_zero, half_range, w_scale, wreduced,
                                                  nullptr, out, 0);
  return cudaGetLastError();
}

cudaError_t launch_dequant_add(const int32_t* acc, int64_t M, int64_t N, const float* a_scale,
                               const float* a_zero, float half_range, const float* w_scale,
                               const float* wreduced, const float* fp_part, void* out, int out_is_f16,
                               cudaStream_t stream) {
  if (M == 0 || N == 0) return cudaSuccess;
  dequant_kernel<<<grid2(N, M), 256, 0, stream>>>(acc, M, N, a_scale, a_zero, half_range, w_scale, wreduced,
                                                  fp_part, out, out_is_f16 ? 2 : 1);
  return cudaGetLastError();
}

}  // namespace quikb200
