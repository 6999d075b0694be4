// Weight-side helpers and the elementwise ops of the reference's small block graphs,
// on the device:
//   clip_search_kernel      clip_search (quantizer.cpp:266-290) for rtn_quantize_weights
//                           with use_clipping (quantizer.cpp:339-371)
//   wreduced_kernel         compute_wreduced (quantizer.cpp:373-382)
//   dequant_weights_kernel  dequantize_weights (quantizer.cpp:384-403)
//   elementwise_kernel      forward_model's Silu / Multiply / Add (runtime.cpp:339-360)
// Every floating-point operation is the reference's, as an explicit _rn intrinsic.
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.h"

namespace quikb200 {
namespace {

// quantize_to_grid (quantizer.cpp:17-22): nearest, ties away from zero, clamped.
__device__ __forceinline__ int grid_code(float v, double inv_scale, int maxq) {
  const double t = __dmul_rn(static_cast<double>(v), inv_scale);
  double q = floor(__dadd_rn(fabs(t), 0.5));
  if (q > maxq) q = maxq;
  return static_cast<int>(t < 0.0 ? -q : q);
}

// static_cast<float>(0.50 + 0.01 * step) without FMA contraction (the reference is
// built -ffp-contract=off)
__device__ __forceinline__ float clip_factor(int step) {
  return static_cast<float>(__dadd_rn(0.50, __dmul_rn(0.01, static_cast<double>(step))));
}

// One warp per weight row. The reference walks the 51 clip factors in ascending order
// and, for each, sums the squared round-trip error over the row sequentially; lane l
// owns factors l and l + 32 and keeps exactly that sequential order for them (the row
// is broadcast element by element), so every err is the reference's bit for bit.
// "err <= best" in ascending c = the largest c among the minimal errors.
__global__ void __launch_bounds__(256) clip_search_kernel(const float* __restrict__ w, int64_t N, int64_t K,
                                                          const int32_t* __restrict__ base_src, int64_t kb, int bits,
                                                          float* __restrict__ clip) {
  const int64_t r = blockIdx.x * 8LL + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= N) return;
  const float* row = w + r * K;
  const int maxq = (1 << (bits - 1)) - 1;
  double amax = 0.0;
  for (int64_t j = lane; j < kb; j += 32) amax = fmax(amax, static_cast<double>(fabsf(row[base_src[j]])));
  for (int off = 16; off; off >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  if (amax == 0.0 || kb == 0) {
    if (lane == 0) clip[r] = 1.0f;
    return;
  }
  double sc[2], inv[2], err[2] = {0.0, 0.0};
  float c[2];
  for (int u = 0; u < 2; ++u) {
    const int step = lane + 32 * u;
    c[u] = clip_factor(step <= 50 ? step : 50);
    sc[u] = __ddiv_rn(__dmul_rn(static_cast<double>(c[u]), amax), static_cast<double>(maxq));
    inv[u] = __ddiv_rn(1.0, sc[u]);
  }
  for (int64_t j0 = 0; j0 < kb; j0 += 32) {
    const int64_t jj = j0 + lane;
    const float mine = jj < kb ? row[base_src[jj]] : 0.0f;
    const int n = static_cast<int>(kb - j0 < 32 ? kb - j0 : 32);
    for (int i = 0; i < n; ++i) {
      const float v = __shfl_sync(0xffffffffu, mine, i);
      for (int u = 0; u < 2; ++u) {
        const double dq = __dmul_rn(static_cast<double>(grid_code(v, inv[u], maxq)), sc[u]);
        const double d = __dsub_rn(static_cast<double>(v), dq);
        err[u] = __dadd_rn(err[u], __dmul_rn(d, d));
      }
    }
  }
  // lanes 0..31 hold steps 0..31, lanes 0..18 also steps 32..50
  double best = err[0];
  int best_step = lane;
  if (lane + 32 <= 50 && err[1] <= best) {
    best = err[1];
    best_step = lane + 32;
  }
  for (int off = 16; off; off >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int os = __shfl_xor_sync(0xffffffffu, best_step, off);
    if (ob < best || (ob == best && os > best_step)) {
      best = ob;
      best_step = os;
    }
  }
  if (lane == 0) clip[r] = clip_factor(best_step);
}

// compute_wreduced: wreduced[r] = float(double(scale[r]) * double(sum_j q[r][j])).
__global__ void wreduced_kernel(const uint8_t* __restrict__ base, int64_t N, int64_t kb, int bits,
                                const float* __restrict__ scales, float* __restrict__ out) {
  const int64_t r = blockIdx.x * 8LL + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= N) return;
  const int64_t rb = bits == 4 ? (kb + 1) / 2 : kb;
  const uint8_t* row = base + r * rb;
  long long s = 0;
  for (int64_t p = lane; p < rb; p += 32) {
    const uint8_t b = row[p];
    if (bits == 8) s += static_cast<int8_t>(b);
    else {
      s += static_cast<int>(b & 0xF) - 8;
      if (2 * p + 1 < kb) s += static_cast<int>(b >> 4) - 8;
    }
  }
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) out[r] = __double2float_rn(__dmul_rn(static_cast<double>(scales[r]), static_cast<double>(s)));
}

// dequantize_weights: out[r][perm[j]] = float(q[r][j]) * scale[r] for base columns,
// out[r][idx[i]] = outlier_weights[r][i].
__global__ void dequant_weights_kernel(const uint8_t* __restrict__ base, int64_t N, int64_t K, int64_t kb, int bits,
                                       const float* __restrict__ scales, const int32_t* __restrict__ perm,
                                       const float* __restrict__ ow, float* __restrict__ out) {
  const int64_t rb = bits == 4 ? (kb + 1) / 2 : kb;
  const int64_t no = K - kb;
  for (int64_t r = blockIdx.y; r < N; r += gridDim.y)
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < K;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float v;
    if (j < kb) {
      int q;
      if (bits == 8) q = static_cast<int8_t>(base[r * rb + j]);
      else {
        const uint8_t b = base[r * rb + j / 2];
        q = static_cast<int>((j & 1) ? (b >> 4) : (b & 0xF)) - 8;
      }
      v = __fmul_rn(static_cast<float>(q), scales[r]);
    } else {
      v = ow[r * no + (j - kb)];
    }
    out[r * K + perm[j]] = v;
  }
}

// forward_model elementwise ops (runtime.cpp:339-360): 0 silu e / (1 + exp(-e)),
// 1 multiply, 2 add; f32.
__global__ void elementwise_kernel(int op, const float* __restrict__ a, const float* __restrict__ b,
                                   float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float e = a[i];
    float v;
    if (op == 0) v = __fdiv_rn(e, __fadd_rn(1.0f, expf(-e)));
    else if (op == 1) v = __fmul_rn(e, b[i]);
    else v = __fadd_rn(e, b[i]);
    out[i] = v;
  }
}

unsigned blocks_for(int64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }

}  // namespace

cudaError_t launch_clip_search(const float* w, int64_t N, int64_t K, const int32_t* base_src, int64_t kb, int bits,
                               float* clip, cudaStream_t stream) {
  if (N == 0) return cudaSuccess;
  clip_search_kernel<<<blocks_for(N, 8), 256, 0, stream>>>(w, N, K, base_src, kb, bits, clip);
  return cudaGetLastError();
}

cudaError_t launch_compute_wreduced(const uint8_t* base, int64_t N, int64_t kb, int bits, const float* scales,
                                    float* out, cudaStream_t stream) {
  if (N == 0) return cudaSuccess;
  wreduced_kernel<<<blocks_for(N, 8), 256, 0, stream>>>(base, N, kb, bits, scales, out);
  return cudaGetLastError();
}

cudaError_t launch_dequantize_weights(const uint8_t* base, int64_t N, int64_t K, int64_t kb, int bits,
                                      const float* scales, const int32_t* perm, const float* ow, float* out,
                                      cudaStream_t stream) {
  if (N == 0 || K == 0) return cudaSuccess;
  const unsigned gx = blocks_for(K, 256) > 64 ? 64 : blocks_for(K, 256);
  dequant_weights_kernel<<<dim3(gx, static_cast<unsigned>(std::min<int64_t>(N, 65535))), 256, 0, stream>>>(base, N, K, kb, bits, scales, perm,
                                                                                 ow, out);
  return cudaGetLastError();
}

cudaError_t launch_elementwise(int op, const float* a, const float* b, float* out, int64_t n, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const unsigned g = blocks_for(n, 256) > 148 * 16 ? 148 * 16 : blocks_for(n, 256);
  elementwise_kernel<<<g, 256, 0, stream>>>(op, a, b, out, n);
  return cudaGetLastError();
}

}  // namespace quikb200
