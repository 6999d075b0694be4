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
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include <cstdio>

#include "kernels.h"
#include "sm100.cuh"

namespace quikb200 {

namespace {

__device__ __forceinline__ float to_float(__half v) { return __half2float(v); }
__device__ __forceinline__ float to_float(float v) { return v; }

template <typename T>
__device__ __forceinline__ float elem(const uint4& v, int e) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t w = (&v.x)[e >> 1];
    const uint16_t h = (e & 1) ? static_cast<uint16_t>(w >> 16) : static_cast<uint16_t>(w & 0xFFFF);
    return __half2float(__ushort_as_half(h));
  } else {
    return __uint_as_float((&v.x)[e]);
  }
}

// Exact lround((x - vmin) / scale) for the quantizer (runtime.cpp:58) without an
// IEEE division per element. With d = fl(x - vmin) >= 0, r = fl(1/scale),
// qa = fl(d * r) and u = fl(qa + 0.5):
//   |qa - fl(d / scale)| <= (d/scale) * 3.0001 * 2^-24 <= 4.6e-5 (d/scale <= 256),
//   |u - (fl(d/scale) + 0.5)| <= 6.1e-5.
// lround(q) = floor(q + 0.5) for q >= 0 changes value only at integers of u, so
// whenever frac(u) is farther than 2^-12 from 0 and 1, floor(u) is exact; the
// other elements (about 5e-4 of them; exact .5 ties among them) take the IEEE
// quotient, rounded half away from zero. Bit-identical to the reference.
__device__ __forceinline__ float quant_slow(float d, float scale) { return round_half_away(__fdiv_rn(d, scale)); }
// |qa - round(qa)| >= kNearTie  <=>  qa within 2^-12 of a half-integer (a rounding
// boundary of lround); such elements take the exact IEEE quotient.
constexpr float kNearTie = 0.5f - 2.44140625e-4f;

__device__ __forceinline__ unsigned long long f32x2_pack(float lo, float hi) {
  return (static_cast<unsigned long long>(__float_as_uint(hi)) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ void f32x2_unpack(unsigned long long v, float& lo, float& hi) {
  lo = __uint_as_float(static_cast<uint32_t>(v));
  hi = __uint_as_float(static_cast<uint32_t>(v >> 32));
}
// (x - vmin) * rcp for two lanes at once (FADD2 / FMUL2, IEEE round-to-nearest).
__device__ __forceinline__ void sub_mul_x2(float x0, float x1, unsigned long long vmin2, unsigned long long rcp2,
                                           float& d0, float& d1, float& q0, float& q1) {
  unsigned long long d, qa;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f32x2_pack(x0, x1)), "l"(vmin2));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(qa) : "l"(d), "l"(rcp2));
  f32x2_unpack(d, d0, d1);
  f32x2_unpack(qa, q0, q1);
}

__device__ __forceinline__ __half2 u2h2(uint32_t u) {
  __half2 h;
  memcpy(&h, &u, 4);
  return h;
}
__device__ __forceinline__ uint32_t h22u(__half2 h) {
  uint32_t u;
  memcpy(&u, &h, 4);
  return u;
}

// One CTA per token row (the row held in registers, VPT 16-byte vectors per
// thread, read once from HBM with coalesced 128-bit loads):
//   pass 1  min / max over the base columns: packed half2 (or f32) min/max with
//           outlier lanes neutralised by the per-layer byte lane mask; NaN
//           propagates (flagged as NumericalError);
//   pass 2  codes for every column in registers (exact reciprocal fast path),
//           written UNCOMPACTED to shared memory with one 8-byte store per vector;
//   copy    base position j <- column gather[j] (per-layer u16 table): 16 codes per
//           thread gathered from shared memory, one 16-byte store to HBM;
//   outliers gathered from the shared-memory row copy into their f16 slots.
//
// min/max tie semantics (runtime.cpp:40-51: first element seeds, strict < / >):
// the extrema VALUES are order independent except for the sign of a zero
// minimum, which is resolved exactly: when the row minimum compares equal to 0
// the sign of the lowest-index zero wins (only the sign of vmin reaches an
// output; vmax's sign cannot change range = vmax - vmin).
// FULL: nvec == blockDim * VPT, K % E == 0 and the row is 16-byte aligned (host
// checked): no bounds checks or tails in the unrolled register code.
template <typename T, int BITS, int VPT, bool FULL>
__global__ void __launch_bounds__(512) quantize_rows_kernel(const QuantArgs a) {
  extern __shared__ __align__(16) uint8_t s_dyn[];
  __shared__ float s_min[16], s_max[16];
  __shared__ int s_nf[16];
  __shared__ unsigned s_key[16];
  constexpr int E = 16 / sizeof(T);  // elements per 16-byte vector (8 f16 / 4 f32)
  constexpr int kHr = 1 << (BITS - 1);
  constexpr float kLevels = static_cast<float>((1 << BITS) - 1);

  // let the dependent GEMM launch and run its prologue while this grid finishes
  // (it waits for this grid's completion with griddepcontrol.wait)
  asm volatile("griddepcontrol.launch_dependents;");
  const int t = blockIdx.x;
  const int tid = threadIdx.x;
  const int nt = blockDim.x;
  const int K = static_cast<int>(a.K);
  const int nvec = (K + E - 1) / E;
  const int kb = static_cast<int>(a.kb);
  // shared: codes [round_up(K,16) + 16] (uncompacted, zero tail) | row copy [nvec * 16] (outlier gather)
  const int code_bytes = ((K + 15) & ~15) + 16;
  uint8_t* s_codes = s_dyn;
  uint4* s_row = reinterpret_cast<uint4*>(s_dyn + code_bytes);
  const T* src = reinterpret_cast<const T*>(a.x) + static_cast<int64_t>(t) * a.ldx;
  const bool vec_ok = FULL || (((reinterpret_cast<uintptr_t>(src) & 15) == 0) && (K % E == 0));
  const bool has_out = a.lane_mask != nullptr;

  uint4 raw[VPT];
  uint32_t lm[VPT];  // lane-mask bytes of the vector's E columns (tail / beyond-row columns = 0xFF)
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int v = tid + i * nt;
    raw[i] = make_uint4(0, 0, 0, 0);
    lm[i] = 0xFFFFFFFFu;
    if (E == 8) lm[i] = 0xFFFFFFFFu;  // E == 8: two words, see lm_hi
    if (FULL || v < nvec) {
      if (vec_ok) {
        raw[i] = __ldg(reinterpret_cast<const uint4*>(src) + v);
      } else {
        T tmp[E];
#pragma unroll
        for (int e = 0; e < E; ++e) tmp[e] = (v * E + e < K) ? src[v * E + e] : T(0);
        memcpy(&raw[i], tmp, 16);
      }
      s_row[v] = raw[i];
    }
  }
  uint32_t lm_hi[VPT];  // bytes 4..7 of the lane mask (E == 8 only)
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int v = tid + i * nt;
    lm_hi[i] = 0xFFFFFFFFu;
    if (FULL || v < nvec) {
      const int c0 = v * E;
      if (has_out) {
        if (E == 8) {
          const uint2 m = __ldg(reinterpret_cast<const uint2*>(a.lane_mask + c0));
          lm[i] = m.x;
          lm_hi[i] = m.y;
        } else {
          lm[i] = __ldg(reinterpret_cast<const uint32_t*>(a.lane_mask + c0));
        }
      } else {
        lm[i] = 0u;
        lm_hi[i] = 0u;
      }
      if (!FULL && c0 + E > K) {  // row tail: columns >= K excluded
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (c0 + e >= K) {
            if (e < 4) lm[i] |= 0xFFu << (8 * e);
            else lm_hi[i] |= 0xFFu << (8 * (e - 4));
          }
      }
    }
  }

  // prefetch the gather-table entries of this thread's first two output chunks
  const int nchunk = a.q8 ? static_cast<int>(a.kpad / 16) : 0;
  uint4 gpre[4] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
  if (has_out) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int cidx = tid + k * nt;
      if (cidx < nchunk) {
        gpre[2 * k] = __ldg(reinterpret_cast<const uint4*>(a.gather + cidx * 16));
        gpre[2 * k + 1] = __ldg(reinterpret_cast<const uint4*>(a.gather + cidx * 16 + 8));
      }
    }
  }

  // ---- pass 1: min / max over base columns (NaN-propagating; +-inf caught by the
  // final finiteness test)
  float vmin, vmax;
  int nonfinite;
  if constexpr (sizeof(T) == 2) {
    __half2 hmin = u2h2(0x7C007C00u), hmax = u2h2(0xFC00FC00u);
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t x2 = (&raw[i].x)[w];
        // widen mask bytes (2w, 2w+1) to 16-bit lanes
        const uint32_t mword = w < 2 ? lm[i] : lm_hi[i];
        const uint32_t m = __byte_perm(mword, 0u, (w & 1) ? 0x3322u : 0x1100u);
        hmin = __hmin2_nan(hmin, u2h2((x2 & ~m) | (0x7C007C00u & m)));
        hmax = __hmax2_nan(hmax, u2h2((x2 & ~m) | (0xFC00FC00u & m)));
      }
    }
    const float2 fmn = __half22float2(hmin);
    const float2 fmx = __half22float2(hmax);
    // NaN propagates through the _nan min/max; +inf can only reach hmax and -inf
    // only hmin (the lane sentinels are the opposite infinities)
    nonfinite = isnan(fmn.x) || isnan(fmn.y) || isnan(fmx.x) || isnan(fmx.y) || fmx.x == INFINITY ||
                fmx.y == INFINITY || fmn.x == -INFINITY || fmn.y == -INFINITY;
    vmin = fminf(fmn.x, fmn.y);
    vmax = fmaxf(fmx.x, fmx.y);
  } else {
    vmin = __int_as_float(0x7f800000);
    vmax = -vmin;
    nonfinite = 0;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float x = __uint_as_float((&raw[i].x)[e]);
        const bool base = ((lm[i] >> (8 * e)) & 0xFFu) == 0;
        nonfinite |= base && !isfinite(x);
        vmin = fminf(vmin, base ? x : vmin);
        vmax = fmaxf(vmax, base ? x : vmax);
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, off));
    vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, off));
    nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, off);
  }
  if ((tid & 31) == 0) { s_min[tid >> 5] = vmin; s_max[tid >> 5] = vmax; s_nf[tid >> 5] = nonfinite; }
  for (int j = ((K + 15) & ~15) + tid; j < code_bytes; j += nt) s_codes[j] = 0;  // zero pad (gather target)
  __syncthreads();
  vmin = s_min[0];
  vmax = s_max[0];
  nonfinite = s_nf[0];
  for (int w = 1; w < nt / 32; ++w) {
    vmin = fminf(vmin, s_min[w]);
    vmax = fmaxf(vmax, s_max[w]);
    nonfinite |= s_nf[w];
  }
  if (kb == 0) { vmin = 0.f; vmax = 0.f; }
  if (vmin == 0.0f && kb > 0) {
    // rare: the sign of a zero minimum is the first-seen zero's (block-uniform branch)
    unsigned key = 0xFFFFFFFFu;
#pragma unroll 1
    for (int i = 0; i < VPT; ++i) {
      const int v = tid + i * nt;
      if (!FULL && v >= nvec) break;
      uint4 rv = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < VPT; ++j)
        if (j == i) rv = raw[j];
      uint32_t m0 = 0, m1 = 0;
#pragma unroll
      for (int j = 0; j < VPT; ++j)
        if (j == i) { m0 = lm[j]; m1 = lm_hi[j]; }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float x = elem<T>(rv, e);
        const uint32_t mbyte = ((e < 4 ? m0 : m1) >> (8 * (e & 3))) & 0xFFu;
        if (mbyte == 0 && x == 0.0f) {
          const unsigned k = (static_cast<unsigned>(v * E + e) << 1) | (__float_as_uint(x) >> 31);
          key = k < key ? k : key;
        }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned o = __shfl_xor_sync(0xffffffffu, key, off);
      key = o < key ? o : key;
    }
    __syncthreads();
    if ((tid & 31) == 0) s_key[tid >> 5] = key;
    __syncthreads();
    key = s_key[0];
    for (int w = 1; w < nt / 32; ++w) key = s_key[w] < key ? s_key[w] : key;
    vmin = (key & 1u) ? -0.0f : 0.0f;
  }
  const float range = __fsub_rn(vmax, vmin);
  const float scale = range == 0.0f ? 1.0f : __fdiv_rn(range, kLevels);
  const float rcp = __frcp_rn(scale);
  if (tid == 0) {
    if (nonfinite && a.err) atomicExch(a.err, 1);
    a.scale[t] = scale;
    a.zero[t] = vmin;
  }
  const unsigned long long vmin2 = f32x2_pack(vmin, vmin);
  const unsigned long long rcp2 = f32x2_pack(rcp, rcp);
  constexpr float kMagic = 12582912.0f - static_cast<float>(kHr);  // 1.5 * 2^23 - half_range
  const unsigned long long magic2 = f32x2_pack(kMagic, kMagic);

  // ---- pass 2: codes for every column (outlier lanes produce ignored codes)
  uint32_t near_vec = 0;  // bit i: vector i has an element near a rounding boundary
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int v = tid + i * nt;
    if (!FULL && v >= nvec) continue;
    // qa = (x - vmin) * fl(1/scale) (FADD2/FMUL2); t = qa + (1.5*2^23 - hr) rounds qa
    // to the nearest integer inside the mantissa, whose low byte is then the signed
    // code (q - hr) directly; r = qa - round(qa) tells how close qa is to a
    // rounding boundary (see quant_q / kNearTie). No float->int conversions.
    // ptxas may contract the packed mul+add into FFMA2 (t = rn(d*rcp + magic)); the
    // exactness argument holds either way: the unrounded product is even closer to
    // d/scale (<= 3.1e-5 at the top of the range) than fl(d*rcp), and the margin to
    // kNearTie is 2^-12, so an element is either flagged or its rounding is exact.
    float x[E];
    uint32_t tb[E];
    float rmax = 0.0f;
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = elem<T>(raw[i], e);
#pragma unroll
    for (int e = 0; e < E; e += 2) {
      unsigned long long d2, qa2, t2, rq2, r2;
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d2) : "l"(f32x2_pack(x[e], x[e + 1])), "l"(vmin2));
      asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(qa2) : "l"(d2), "l"(rcp2));
      asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t2) : "l"(qa2), "l"(magic2));
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(rq2) : "l"(t2), "l"(magic2));
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r2) : "l"(qa2), "l"(rq2));
      float r0, r1;
      f32x2_unpack(r2, r0, r1);
      rmax = fmaxf(rmax, fmaxf(fabsf(r0), fabsf(r1)));
      tb[e] = static_cast<uint32_t>(t2);
      tb[e + 1] = static_cast<uint32_t>(t2 >> 32);
    }
    const bool near_any = !(rmax < kNearTie);  // also catches NaN (flagged rows)
    // codes are in [0, levels] for finite rows (d >= 0, qa <= levels * (1 + 2^-22))
    const uint32_t w0 = __byte_perm(__byte_perm(tb[0], tb[1], 0x0040), __byte_perm(tb[2], tb[3], 0x0040), 0x5410);
    if (E == 8) {
      const uint32_t w1 =
          __byte_perm(__byte_perm(tb[4 % E], tb[5 % E], 0x0040), __byte_perm(tb[6 % E], tb[7 % E], 0x0040), 0x5410);
      *reinterpret_cast<uint2*>(s_codes + v * E) = make_uint2(w0, w1);
    } else {
      *reinterpret_cast<uint32_t*>(s_codes + v * E) = w0;
    }
    near_vec |= (near_any ? 1u : 0u) << i;
  }
  if (near_vec) {
    // rare: elements within 2^-12 of a rounding boundary take the exact IEEE
    // quotient (same d and u as above; this thread owns these code bytes)
    const T* row = reinterpret_cast<const T*>(s_row);
#pragma unroll 1
    for (uint32_t nv = near_vec; nv; nv &= nv - 1) {
      const int v = tid + (__ffs(nv) - 1) * nt;
#pragma unroll 1
      for (int e = 0; e < E; ++e) {
        const int c = v * E + e;
        if (c >= K) break;
        const float d = __fsub_rn(to_float(row[c]), vmin);
        const float qa = __fmul_rn(d, rcp);
        const float r = __fsub_rn(qa, __fsub_rn(__fadd_rn(qa, kMagic), kMagic));
        if (!(fabsf(r) < kNearTie))
          s_codes[c] = static_cast<uint8_t>(static_cast<int>(quant_slow(d, scale)) - kHr);
      }
    }
  }
  __syncthreads();

  // ---- outliers (ascending index order, runtime.cpp:217) from the row copy
  if (has_out) {
    const T* row = reinterpret_cast<const T*>(s_row);
    __half* xo16 = a.xo16 ? a.xo16 + static_cast<int64_t>(t) * a.opad : nullptr;
    float* xo32 = a.xo32 ? a.xo32 + static_cast<int64_t>(t) * a.n_out : nullptr;
    for (int i = tid; i < a.n_out; i += nt) {
      const float x = to_float(row[__ldg(&a.out_src[i])]);
      if (xo16) xo16[i] = __float2half_rn(x);
      if (xo32) xo32[i] = x;
    }
    if (xo16)
      for (int i = static_cast<int>(a.n_out) + tid; i < a.opad; i += nt) xo16[i] = __float2half_rn(0.0f);
  } else if (a.xo16) {
    for (int i = tid; i < a.opad; i += nt) a.xo16[static_cast<int64_t>(t) * a.opad + i] = __float2half_rn(0.0f);
  }

  // ---- compacted code row: base position j <- column gather[j] (16 per thread;
  // the first two chunks' gather entries were prefetched at kernel start)
  if (a.q8) {
    uint4* dst = reinterpret_cast<uint4*>(a.q8 + static_cast<int64_t>(t) * a.kpad);
#pragma unroll 1
    for (int k = 0, cidx = tid; cidx < nchunk; ++k, cidx += nt) {
      const int j0 = cidx * 16;
      uint32_t w[4];
      if (has_out) {
        uint4 g0, g1;
        if (k == 0) { g0 = gpre[0]; g1 = gpre[1]; }
        else if (k == 1) { g0 = gpre[2]; g1 = gpre[3]; }
        else {
          g0 = __ldg(reinterpret_cast<const uint4*>(a.gather + j0));
          g1 = __ldg(reinterpret_cast<const uint4*>(a.gather + j0 + 8));
        }
        const uint32_t gi[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t b0 = s_codes[gi[2 * kk] & 0xFFFFu], b1 = s_codes[gi[2 * kk] >> 16];
          const uint32_t b2 = s_codes[gi[2 * kk + 1] & 0xFFFFu], b3 = s_codes[gi[2 * kk + 1] >> 16];
          w[kk] = __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
        }
      } else {
        const uint4 c = *reinterpret_cast<const uint4*>(s_codes + j0);
        w[0] = c.x; w[1] = c.y; w[2] = c.z; w[3] = c.w;
        if (j0 + 16 > kb) {  // zero the pad positions j >= kb
#pragma unroll
          for (int kk = 0; kk < 16; ++kk)
            if (j0 + kk >= kb) w[kk >> 2] &= ~(0xFFu << (8 * (kk & 3)));
        }
      }
      dst[cidx] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  // ---- ABI packed codes (debug / parity entry points)
  if (a.packed) {
    uint8_t* prow = a.packed + static_cast<int64_t>(t) * (BITS == 4 ? (kb + 1) / 2 : kb);
    auto code_at = [&](int j) -> int {
      const int c = has_out ? static_cast<int>(__ldg(&a.gather[j])) : j;
      return static_cast<int8_t>(s_codes[c]);
    };
    if (BITS == 8) {
      for (int j = tid; j < kb; j += nt) prow[j] = static_cast<uint8_t>(code_at(j));
    } else {
      // i4p: low nibble = even base index, stored + 8; pad nibble of odd rows = 0
      for (int b = tid; b < (kb + 1) / 2; b += nt) {
        const uint8_t lo = static_cast<uint8_t>(code_at(2 * b) + 8) & 0xF;
        const uint8_t hi = (2 * b + 1 < kb) ? (static_cast<uint8_t>(code_at(2 * b + 1) + 8) & 0xF) : 0;
        prow[b] = static_cast<uint8_t>(lo | (hi << 4));
      }
    }
  }
}

// Hot-path K1 (f16 x, 16-byte aligned rows, K % 8 == 0, GEMM-layout outputs only).
// Same numerics as quantize_rows_kernel, organised for HBM throughput and a short
// instruction stream (the one-CTA-per-row kernel issues ~27 instructions per
// element and is issue-bound at ~2 TB/s):
//   * persistent CTAs walk rows blockIdx.x, +gridDim.x, ...; each row is fetched
//     into a shared-memory ring by one TMA bulk copy issued `stages` rows ahead
//     (a slot is refilled at barrier A of its own row, once the row is in registers);
//   * everything row-independent is hoisted out of the row loop: the per-vector
//     outlier lane masks live in registers; the compaction descriptors are
//     L1-resident per-layer tables;
//   * min/max: packed HMNMX2; outlier lanes are replaced (one LOP3 per word) by the
//     row's first base value, which cannot move the base min/max;
//   * codes are written uncompacted to shared memory (one 8-byte store per vector);
//   * compaction by 16-byte output chunk with a uniform two-window rule: byte p of
//     the chunk is window A[p] (p < len1) or window B[p]; each window is 5 aligned
//     32-bit shared loads + 4 byte permutes, the merge is 4 byte permutes. The few
//     chunks with more than one outlier gap ("general") are gathered per byte by
//     the first warps in a separate, warp-uniform loop.
// Thread tid owns vectors v = tid + i * nt (i < VPT) and chunk slots tid + k * nt.
__device__ __forceinline__ float redux_min(float v) {
  float r;
  asm volatile("redux.sync.min.NaN.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float redux_max(float v) {
  float r;
  asm volatile("redux.sync.max.NaN.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
// f32 = f16 - f32 in one instruction (FHADD), exact conversion then IEEE rn subtraction
__device__ __forceinline__ float sub_f16_f32(uint32_t h, float c) {
  float d;
  asm("sub.rn.f32.f16 %0, %1, %2;" : "=f"(d) : "h"(static_cast<unsigned short>(h)), "f"(c));
  return d;
}

// hstat / pre_stat key (kernels.h) -> the f16 value it encodes
__device__ __forceinline__ float hkey_to_float(uint32_t k) {
  const uint32_t u = k >= 0x8000u ? k - 0x8000u : (0x8000u | (0x7FFFu - k));
  return __half2float(__ushort_as_half(static_cast<unsigned short>(u)));
}

// FILL: no per-thread lane masks (48 registers at VPT 8): each row's outlier columns are
// overwritten in the ring slot by the row's first base value (a value of the base set,
// so it cannot move the base min / max, and a zero there carries the first base zero's
// sign) behind one more block barrier, so the kernel fits two CTAs per SM.
template <int BITS, int VPT, bool FULL, bool FILL>
__device__ __forceinline__ void quantize_hot_body(const QuantArgs& a, int stages, int row_stride) {
  extern __shared__ __align__(128) uint8_t s_dyn[];
  __shared__ float s_min[16], s_max[16];
  __shared__ int s_nf[16];
  __shared__ unsigned s_key[16];
  __shared__ __align__(8) uint64_t s_full[8];
  constexpr int kHr = 1 << (BITS - 1);
  constexpr float kLevels = static_cast<float>((1 << BITS) - 1);
  asm volatile("griddepcontrol.launch_dependents;");
  const int tid = threadIdx.x;
  const int nt = blockDim.x;
  const int nwarps = (nt + 31) >> 5;
  const int K = static_cast<int>(a.K);
  const int M = static_cast<int>(a.M);
  const int nvec = K >> 3;
  // FULL: nvec == blockDim * VPT (host checked), every vector slot is in the row
  auto in_row = [&](int v) { return FULL || v < nvec; };
  const int kb = static_cast<int>(a.kb);
  const int kr16 = (K + 15) & ~15;
  const uint32_t row_bytes = static_cast<uint32_t>(K) * 2u;
  // one code row (written after barrier A of row t+1, read before it for row t), then
  // the ring
  const int code_stride = (kr16 + 32 + 127) & ~127;
  // prescaled rows (a.pre_stat: min / max from the producing GEMM's epilogue): no
  // reduction pass; barrier A stays (it orders row t's compaction reads before row
  // t+1's code writes and frees the ring slot)
  uint4* const pre = a.pre_stat;
  uint8_t* s_codes = s_dyn;                          // [code_stride]: codes by column, zero tail
  uint8_t* s_ring = s_dyn + code_stride;             // [stages][row_stride]
  const bool has_out = a.lane_mask != nullptr;
  const int nchunk = static_cast<int>(a.kpad >> 4);
  const __half* xg = reinterpret_cast<const __half*>(a.x);
  const uint4* cdesc = reinterpret_cast<const uint4*>(a.chunk_desc);
  const int first_base = has_out ? static_cast<int>(a.gather[0]) : 0;  // column of base position 0

  // row-independent: outlier lane masks of this thread's vectors, the byte mask (lm, the
  // rare exact paths) and its expansion to one 16-bit lane mask per f16 (lmw, pass 1:
  // one LOP3 per word instead of a PRMT + LOP3)
  constexpr int kLm = FILL ? 1 : VPT;
  uint2 lm[kLm];
  uint4 lmw[kLm];
#pragma unroll
  for (int i = 0; i < kLm; ++i) {
    const int v = tid + i * nt;
    lm[i] = (!FILL && has_out && in_row(v)) ? __ldg(reinterpret_cast<const uint2*>(a.lane_mask) + v) : make_uint2(0u, 0u);
    lmw[i] = make_uint4(__byte_perm(lm[i].x, 0u, 0x1100u), __byte_perm(lm[i].x, 0u, 0x3322u),
                        __byte_perm(lm[i].y, 0u, 0x1100u), __byte_perm(lm[i].y, 0u, 0x3322u));
  }

  // row-independent: this thread's outlier slots (i = tid, tid + nt) -> source column, -1 = zero pad
  int osrc[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int i = tid + j * nt;
    osrc[j] = (has_out && i < a.n_out) ? __ldg(&a.out_src[i]) : -1;
  }
  const int opad = static_cast<int>(a.opad);
  const bool xo_hoisted = opad <= 2 * nt;

  if (tid == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&s_full[s], 1);
    fence_mbar_init();
  }
  if (tid < 8) reinterpret_cast<uint32_t*>(s_codes + kr16)[tid] = 0u;  // zero tail
  __syncthreads();
  if (tid == 0) {
    // PDL: everything above (tables, barriers) overlapped the previous kernel; its
    // outputs may be this layer's input and it may still read this kernel's output
    // buffers, so the first row loads (and hence every write) come after the wait
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int s = 0; s < stages; ++s) {
      const int r = blockIdx.x + s * gridDim.x;
      if (r >= M) break;
      mbar_arrive_expect_tx(&s_full[s], row_bytes);
      bulk_load_1d(s_ring + s * row_stride, xg + static_cast<int64_t>(r) * a.ldx, row_bytes, &s_full[s]);
    }
  }

  // prescaled: every thread that reads the keys (written by the previous kernel) waits on
  // the programmatic dependency itself (the others only consume TMA data issued after it)
  if (pre) asm volatile("griddepcontrol.wait;" ::: "memory");
  int s = 0;
  uint32_t ph = 0;
  // FILL: the next row's outlier overwrite is done before barrier B of the current row
  // (once its load has landed), so B doubles as its barrier F; `prepared` marks a row
  // whose slot is already overwritten, xov_next holds its outlier values
  bool prepared = false;
  uint16_t xov_next[2] = {0, 0};
#pragma unroll 1
  for (int t = blockIdx.x; t < M; t += gridDim.x) {
    const uint4* srow = reinterpret_cast<const uint4*>(s_ring + s * row_stride);
    if (a.hot_flags & 1) mbar_wait_sleep(&s_full[s], ph);  // waiting threads give up their issue slots
    else mbar_wait(&s_full[s], ph);
    uint4 pst = make_uint4(0u, 0u, 0u, 0u);
    if (pre) pst = __ldcg(pre + t);  // issued early: its latency overlaps the row loads

    uint4 raw[VPT];
    if constexpr (!FILL) {
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        const int v = tid + i * nt;
        raw[i] = in_row(v) ? srow[v] : make_uint4(0, 0, 0, 0);
      }
    }
    // this row's outlier values (the ring slot is refilled at barrier A)
    uint16_t xov[2] = {0, 0};
    if (prepared) {
      xov[0] = xov_next[0];
      xov[1] = xov_next[1];
    } else if (a.xo16 && xo_hoisted) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (osrc[j] >= 0) xov[j] = reinterpret_cast<const uint16_t*>(srow)[osrc[j]];
    }
    if constexpr (FILL) {
      // outlier columns := the first base value (each thread its own slots, after reading
      // them above; the non-hoisted outlier copy reads x from global memory)
      if (has_out && !pre && !prepared) {
        uint16_t* hrow = reinterpret_cast<uint16_t*>(s_ring + s * row_stride);
        const uint16_t h0 = hrow[first_base];  // a base column: never overwritten
        for (int i = tid; i < a.n_out; i += nt) hrow[__ldg(&a.out_src[i])] = h0;
        __syncthreads();  // (F)
      }
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        const int v = tid + i * nt;
        raw[i] = in_row(v) ? srow[v] : make_uint4(0, 0, 0, 0);
      }
    }
    float vmin = 0.f, vmax = 0.f;
    int nonfinite = 0;
    if (!pre) {
    // ---- pass 1: packed min / max over the base columns
    __half2 hmin = u2h2(0x7C007C00u), hmax = u2h2(0xFC00FC00u);
    if (has_out && !FILL) {
      const uint32_t h0 = reinterpret_cast<const uint16_t*>(srow)[first_base];
      const uint32_t fill = h0 | (h0 << 16);  // a base value of this row, in both halves
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        if (!in_row(tid + i * nt)) continue;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const uint32_t mk = (&lmw[FILL ? 0 : i].x)[w];
          const __half2 x2 = u2h2(((&raw[i].x)[w] & ~mk) | (fill & mk));
          hmin = __hmin2_nan(hmin, x2);
          hmax = __hmax2_nan(hmax, x2);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        if (!in_row(tid + i * nt)) continue;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const __half2 x2 = u2h2((&raw[i].x)[w]);
          hmin = __hmin2_nan(hmin, x2);
          hmax = __hmax2_nan(hmax, x2);
        }
      }
    }
    {
      const float2 fmn = __half22float2(hmin);
      const float2 fmx = __half22float2(hmax);
      nonfinite = isnan(fmn.x) || isnan(fmn.y) || isnan(fmx.x) || isnan(fmx.y) || fmx.x == INFINITY ||
                  fmx.y == INFINITY || fmn.x == -INFINITY || fmn.y == -INFINITY;
      vmin = fminf(fmn.x, fmn.y);
      vmax = fmaxf(fmx.x, fmx.y);
    }
    vmin = redux_min(vmin);
    vmax = redux_max(vmax);
    nonfinite = __reduce_or_sync(0xffffffffu, nonfinite);
    if ((tid & 31) == 0) { s_min[tid >> 5] = vmin; s_max[tid >> 5] = vmax; s_nf[tid >> 5] = nonfinite; }
    }
    __syncthreads();  // (A): every thread is done with the previous row and holds this one in registers
    if (tid == 0) {
      // refill this row's ring slot: after A nothing reads it (row in registers,
      // outlier values read above, the rare exact-division path selects from registers)
      const int rn = t + stages * gridDim.x;
      if (rn < M) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&s_full[s], row_bytes);
        bulk_load_1d(s_ring + s * row_stride, xg + static_cast<int64_t>(rn) * a.ldx, row_bytes, &s_full[s]);
      }
    }
    if (pre) {
      // the epilogue's keys (kernels.h): exact f16 values; a zero minimum takes the sign
      // of the first zero (its column in the key's upper bits); non-finite values were
      // flagged by the epilogue
      vmin = hkey_to_float(pst.x);
      vmax = hkey_to_float(pst.y);
      if (kb == 0) { vmin = 0.f; vmax = 0.f; }
      if (vmin == 0.0f && kb > 0 && pst.z != 0xFFFFFFFFu) vmin = (pst.z & 1u) ? -0.0f : 0.0f;
    } else {
    {
      const int l = tid & 31;
      vmin = redux_min(l < nwarps ? s_min[l] : INFINITY);
      vmax = redux_max(l < nwarps ? s_max[l] : -INFINITY);
      nonfinite = __reduce_or_sync(0xffffffffu, l < nwarps ? s_nf[l] : 0);
    }
    if (kb == 0) { vmin = 0.f; vmax = 0.f; }
    if (vmin == 0.0f && kb > 0) {
      // rare: the sign of a zero minimum is the first-seen zero's (block-uniform branch)
      unsigned key = 0xFFFFFFFFu;
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        const int v = tid + i * nt;
        if (!in_row(v)) continue;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float x = elem<__half>(raw[i], e);
          uint32_t mbyte = 0u;
          if constexpr (!FILL) mbyte = ((e < 4 ? lm[i].x : lm[i].y) >> (8 * (e & 3))) & 0xFFu;
          if (mbyte == 0 && x == 0.0f) {
            const unsigned k = (static_cast<unsigned>(v * 8 + e) << 1) | (__float_as_uint(x) >> 31);
            key = k < key ? k : key;
          }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const unsigned o = __shfl_xor_sync(0xffffffffu, key, off);
        key = o < key ? o : key;
      }
      if ((tid & 31) == 0) s_key[tid >> 5] = key;
      __syncthreads();
      key = s_key[0];
      for (int w = 1; w < nwarps; ++w) key = s_key[w] < key ? s_key[w] : key;
      vmin = (key & 1u) ? -0.0f : 0.0f;
    }
    }  // !pre
    const float range = __fsub_rn(vmax, vmin);
    const float scale = range == 0.0f ? 1.0f : __fdiv_rn(range, kLevels);
    const float rcp = __frcp_rn(scale);
    if (tid == 0) {
      if (nonfinite && a.err) atomicExch(a.err, 1);
      a.scale[t] = scale;
      a.zero[t] = vmin;
    }
    // Bracketed rounding (exact): with rcp = fl(1/scale), the reference quotient
    // fl(d / scale) lies strictly inside (d * rcp_lo, d * rcp_hi) for d > 0, since
    // |fl(d/scale) - d*rcp| <= 2 * 2^-24 * d*rcp < 2^-20 * d*rcp. One FMA each
    // rounds d*rcp_x + (1.5 * 2^23 - hr) to an integer (ties-to-even); if both land on
    // the same integer R, no half-integer lies strictly between the brackets, so
    // lround(fl(d/scale)) - hr = R - 1.5 * 2^23 exactly and the low byte of the FMA
    // result is the stored code. Otherwise (within ~2^-20 * q of a tie, incl. exact
    // ties) the element takes the IEEE quotient. 2 FFMA2 + 1 LOP3 per pair.
    const float rcp_lo = __fmul_rd(rcp, 1.0f - 0x1p-20f), rcp_hi = __fmul_ru(rcp, 1.0f + 0x1p-20f);
    const unsigned long long rlo2 = f32x2_pack(rcp_lo, rcp_lo), rhi2 = f32x2_pack(rcp_hi, rcp_hi);
    constexpr float kMagic = 12582912.0f - static_cast<float>(kHr);  // 1.5 * 2^23 - half_range
    const unsigned long long magic2 = f32x2_pack(kMagic, kMagic);

    // ---- pass 2: codes for every column
    uint32_t near_vec = 0;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int v = tid + i * nt;
      if (!in_row(v)) continue;
      uint32_t tb[8];
      uint32_t diff = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t xw = (&raw[i].x)[w];
        const unsigned long long d2 = f32x2_pack(sub_f16_f32(xw & 0xFFFFu, vmin), sub_f16_f32(xw >> 16, vmin));
        unsigned long long tl2, th2;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(tl2) : "l"(d2), "l"(rlo2), "l"(magic2));
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(th2) : "l"(d2), "l"(rhi2), "l"(magic2));
        const uint32_t l0 = static_cast<uint32_t>(tl2), l1 = static_cast<uint32_t>(tl2 >> 32);
        diff |= (l0 ^ static_cast<uint32_t>(th2)) | (l1 ^ static_cast<uint32_t>(th2 >> 32));
        tb[2 * w] = l0;
        tb[2 * w + 1] = l1;
      }
      near_vec |= (diff != 0u ? 1u : 0u) << i;
      const uint32_t w0 = __byte_perm(__byte_perm(tb[0], tb[1], 0x0040), __byte_perm(tb[2], tb[3], 0x0040), 0x5410);
      const uint32_t w1 = __byte_perm(__byte_perm(tb[4], tb[5], 0x0040), __byte_perm(tb[6], tb[7], 0x0040), 0x5410);
      *reinterpret_cast<uint2*>(s_codes + v * 8) = make_uint2(w0, w1);
    }
    if (near_vec) {
      // rare: elements whose brackets straddle a rounding boundary take the exact
      // IEEE quotient, rounded half away from zero (runtime.cpp:58)
#pragma unroll 1
      for (uint32_t nv = near_vec; nv; nv &= nv - 1) {
        const int iv = __ffs(nv) - 1;
        const int v = tid + iv * nt;
        uint4 rv = raw[0];
#pragma unroll
        for (int i = 1; i < VPT; ++i)
          if (i == iv) rv = raw[i];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int c = v * 8 + e;
          const uint32_t hw = (&rv.x)[e >> 1];
          const float d = __fsub_rn(__half2float(__ushort_as_half(static_cast<unsigned short>((e & 1) ? hw >> 16 : hw & 0xFFFFu))), vmin);
          if (__float_as_uint(__fmaf_rn(d, rcp_lo, kMagic)) != __float_as_uint(__fmaf_rn(d, rcp_hi, kMagic)))
            s_codes[c] = static_cast<uint8_t>(static_cast<int>(quant_slow(d, scale)) - kHr);
        }
      }
    }
    if constexpr (FILL) {
      // the next row of this CTA: wait for its slot, take its outlier values, overwrite
      // its outlier columns; barrier B below then orders these stores before its raw loads
      const int tn = t + static_cast<int>(gridDim.x);
      prepared = false;
      if (has_out && !pre && tn < M) {
        const int sn = s + 1 == stages ? 0 : s + 1;
        const uint32_t phn = s + 1 == stages ? ph ^ 1u : ph;
        if (a.hot_flags & 1) mbar_wait_sleep(&s_full[sn], phn);
        else mbar_wait(&s_full[sn], phn);
        uint16_t* hn = reinterpret_cast<uint16_t*>(s_ring + sn * row_stride);
        if (a.xo16 && xo_hoisted) {
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (osrc[j] >= 0) xov_next[j] = hn[osrc[j]];
        }
        const uint16_t h0n = hn[first_base];
        for (int i = tid; i < a.n_out; i += nt) hn[__ldg(&a.out_src[i])] = h0n;
        prepared = true;
      }
    }
    __syncthreads();  // (B) codes complete (FILL: and the next row's outlier columns overwritten)
    if (pre && tid == 0) pre[t] = make_uint4(0xFFFFFFFFu, 0u, 0xFFFFFFFFu, 0u);  // initial keys, next forward
    // this row's compaction descriptors (row-independent, L1-resident): all loads in
    // flight before the outlier gather instead of one at a time in the copy-out loop
    constexpr int kCk = VPT > 1 ? VPT / 2 : 1;
    uint4 dpre[kCk];
#pragma unroll
    for (int k = 0; k < kCk; ++k) {
      const int cidx = tid + k * nt;
      dpre[k] = cidx < nchunk ? __ldg(cdesc + cidx) : make_uint4(0xFFFFFFFFu, 0u, 0u, 0u);
    }

    // ---- outliers (ascending index order, runtime.cpp:217) from the row in the ring
    if (a.xo16) {
      uint16_t* xo = reinterpret_cast<uint16_t*>(a.xo16) + static_cast<int64_t>(t) * opad;
      if (xo_hoisted) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = tid + j * nt;
          if (i < opad) xo[i] = xov[j];
        }
      } else {  // more outliers than 2 per thread: from global memory (L2: the row was just read)
        const uint16_t* xrow = reinterpret_cast<const uint16_t*>(xg + static_cast<int64_t>(t) * a.ldx);
        for (int i = tid; i < opad; i += nt) xo[i] = (has_out && i < a.n_out) ? xrow[__ldg(&a.out_src[i])] : 0;
      }
    }
    // ---- compacted code row: two-window chunks, then the general chunks
    uint4* dst = reinterpret_cast<uint4*>(a.q8 + static_cast<int64_t>(t) * a.kpad);
#pragma unroll
    for (int k = 0; k < kCk; ++k) {
      const int cidx = tid + k * nt;
      const uint4 d = dpre[k];
      if (d.x == 0xFFFFFFFFu) continue;  // general chunk (second loop) or past the row
      const uint32_t* wa = reinterpret_cast<const uint32_t*>(s_codes + (d.x & 0xFFFFu));
      const uint32_t* wb = reinterpret_cast<const uint32_t*>(s_codes + (d.y & 0xFFFFu));
      const uint32_t sa = d.x >> 16, sb = d.y >> 16;
      const uint32_t a0 = wa[0], a1 = wa[1], a2 = wa[2], a3 = wa[3], a4 = wa[4];
      const uint32_t b0 = wb[0], b1 = wb[1], b2 = wb[2], b3 = wb[3], b4 = wb[4];
      const uint32_t o0 = __byte_perm(__byte_perm(a0, a1, sa), __byte_perm(b0, b1, sb), d.z & 0xFFFFu);
      const uint32_t o1 = __byte_perm(__byte_perm(a1, a2, sa), __byte_perm(b1, b2, sb), d.z >> 16);
      const uint32_t o2 = __byte_perm(__byte_perm(a2, a3, sa), __byte_perm(b2, b3, sb), d.w & 0xFFFFu);
      const uint32_t o3 = __byte_perm(__byte_perm(a3, a4, sa), __byte_perm(b3, b4, sb), d.w >> 16);
      dst[cidx] = make_uint4(o0, o1, o2, o3);
    }
    for (int gi = tid; gi < a.n_gen; gi += nt) {
      const int cidx = a.gen_chunk[gi];
      const uint4 g0 = __ldg(reinterpret_cast<const uint4*>(a.gather + cidx * 16));
      const uint4 g1 = __ldg(reinterpret_cast<const uint4*>(a.gather + cidx * 16 + 8));
      const uint32_t gw[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      uint32_t w[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t c0 = s_codes[gw[2 * kk] & 0xFFFFu], c1 = s_codes[gw[2 * kk] >> 16];
        const uint32_t c2 = s_codes[gw[2 * kk + 1] & 0xFFFFu], c3 = s_codes[gw[2 * kk + 1] >> 16];
        w[kk] = __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410);
      }
      dst[cidx] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (++s == stages) { s = 0; ph ^= 1u; }
  }
}

template <int BITS, int VPT, bool FULL>
__global__ void __launch_bounds__(VPT >= 4 ? 512 : 256) quantize_hot_kernel(const QuantArgs a, int stages, int row_stride) {
  quantize_hot_body<BITS, VPT, FULL, false>(a, stages, row_stride);
}
template <int BITS, int VPT, bool FULL>
__global__ void __launch_bounds__(VPT >= 4 ? 512 : 256, 2) quantize_hot_fill_kernel(const QuantArgs a, int stages,
                                                                                      int row_stride) {
  quantize_hot_body<BITS, VPT, FULL, true>(a, stages, row_stride);
}

// Wide rows (K beyond one CTA's ring: OPT-66B fc2 36864, Falcon-180B fc2 59392, the
// 28672-wide down projections): the hot kernel's algorithm with each row split over a
// thread-block cluster, one CTA per slice (quik_layer_create builds the slices: a
// contiguous column range covering a contiguous range of output chunks and outlier
// slots, neighbouring slices overlapping by < 8 columns). Each CTA streams its slice of
// every row through its own TMA ring, reduces min / max over its base columns, and the
// cluster exchanges the partials through distributed shared memory (every CTA stores
// its partial into every peer's slot [row parity][rank] with st.async, which completes
// transaction bytes on the peer's mbarrier; min / max are order independent, so all CTAs reach the same row
// scale). Codes, compaction (window offsets rebased to the slice) and the outlier copy
// then stay inside the CTA. The rare exact paths (near-tie quotients; the sign of a zero
// minimum, which takes a second cluster exchange of the first zero's key) match the hot
// kernel's, so the codes are bit-identical to it and to the reference.
// FILL (as the hot kernel's): no lane-mask registers; the slice's outlier columns (its
// own slots and the < 8 overlap columns past them) are overwritten in the ring slot by
// the slice's first base value, and the rare first-zero scan skips the columns before
// it (outliers or the previous slice's base columns, which that slice scans).
template <int BITS, int VPT, bool FILL>
__global__ void __launch_bounds__(VPT >= 8 ? 512 : 256) quantize_wide_kernel(const QuantArgs a, int stages, int row_stride) {
  extern __shared__ __align__(128) uint8_t s_dyn[];
  __shared__ float s_min[16], s_max[16];
  __shared__ int s_nf[16];
  __shared__ unsigned s_key[16];
  __shared__ __align__(8) uint64_t s_full[8];
  __shared__ __align__(16) uint4 s_x[2][8];  // [row parity][rank]: min, max, non-finite (bits)
  __shared__ __align__(16) uint4 s_k[2][8];  // zero-minimum key exchange
  __shared__ __align__(8) uint64_t s_xbar[2], s_kbar[2];
  constexpr int kHr = 1 << (BITS - 1);
  constexpr float kLevels = static_cast<float>((1 << BITS) - 1);
  asm volatile("griddepcontrol.launch_dependents;");
  const int tid = threadIdx.x;
  const int nt = blockDim.x;
  const int nwarps = (nt + 31) >> 5;
  const uint32_t rank = cluster_ctarank();
  const int C = a.n_slice;
  const int4 sd0 = __ldg(reinterpret_cast<const int4*>(a.slice_desc) + 2 * rank);
  const int4 sd1 = __ldg(reinterpret_cast<const int4*>(a.slice_desc) + 2 * rank + 1);
  const int in_lo = sd0.x, in_n = sd0.y, ch_lo = sd0.z, ch_hi = sd0.w;
  const int o_lo = sd1.x, o_hi = sd1.y, g_lo = sd1.z, g_hi = sd1.w;
  const int K = static_cast<int>(a.K);
  const int M = static_cast<int>(a.M);
  const int nvec = in_n >> 3;
  auto in_row = [&](int v) { return v < nvec; };
  const int kr16 = (K + 15) & ~15;
  const uint32_t row_bytes = static_cast<uint32_t>(in_n) * 2u;
  const int code_stride = a.slice_code_bytes;
  uint8_t* s_codes = s_dyn;                // [code_stride]: codes by local column, zero tail
  uint8_t* s_ring = s_dyn + code_stride;   // [stages][row_stride]
  const bool has_out = a.lane_mask != nullptr;
  const __half* xg = reinterpret_cast<const __half*>(a.x) + in_lo;
  const uint4* cdesc = reinterpret_cast<const uint4*>(a.chunk_desc);
  const int first_base = static_cast<int>(a.gather[16 * ch_lo]) - in_lo;  // a base column of the slice
  const int cl = blockIdx.x / C, ncl = gridDim.x / C;

  constexpr int kLm = FILL ? 1 : VPT;
  uint2 lm[kLm];
  uint4 lmw[kLm];
#pragma unroll
  for (int i = 0; i < kLm; ++i) {
    const int v = tid + i * nt;
    lm[i] = (!FILL && has_out && in_row(v)) ? __ldg(reinterpret_cast<const uint2*>(a.lane_mask + in_lo) + v)
                                             : make_uint2(0u, 0u);
    lmw[i] = make_uint4(__byte_perm(lm[i].x, 0u, 0x1100u), __byte_perm(lm[i].x, 0u, 0x3322u),
                        __byte_perm(lm[i].y, 0u, 0x1100u), __byte_perm(lm[i].y, 0u, 0x3322u));
  }
  // this CTA's outlier slots i = o_lo + tid (+ nt): source column in the slice, -1 = zero pad
  int osrc[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int i = o_lo + tid + j * nt;
    osrc[j] = (has_out && i < o_hi && i < a.n_out) ? __ldg(&a.out_src[i]) - in_lo : -1;
  }
  const int opad = static_cast<int>(a.opad);
  const bool xo_hoisted = o_hi - o_lo <= 2 * nt;

  if (tid == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&s_full[s], 1);
    // exchange barriers: this CTA's arrive (with C x 16 bytes expected) + the C peers'
    // st.async completions
    for (int s = 0; s < 2; ++s) { mbar_init(&s_xbar[s], 1); mbar_init(&s_kbar[s], 1); }
    fence_mbar_init();
  }
  if (rank == static_cast<uint32_t>(C - 1) && tid < 8)  // zero codes of the pad positions (kr16 + q)
    reinterpret_cast<uint32_t*>(s_codes + (kr16 - in_lo))[tid] = 0u;
  __syncthreads();
  cluster_sync();  // every peer's exchange barriers are initialised before the first remote arrive
  if (tid == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int s = 0; s < stages; ++s) {
      const int r = cl + s * ncl;
      if (r >= M) break;
      mbar_arrive_expect_tx(&s_full[s], row_bytes);
      bulk_load_1d(s_ring + s * row_stride, xg + static_cast<int64_t>(r) * a.ldx, row_bytes, &s_full[s]);
    }
  }

  int s = 0, it = 0, kround = 0;
  uint32_t ph = 0;
#pragma unroll 1
  for (int t = cl; t < M; t += ncl, ++it) {
    const uint4* srow = reinterpret_cast<const uint4*>(s_ring + s * row_stride);
    mbar_wait(&s_full[s], ph);
    uint4 raw[VPT];
    if constexpr (!FILL) {
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        const int v = tid + i * nt;
        raw[i] = in_row(v) ? srow[v] : make_uint4(0, 0, 0, 0);
      }
    }
    uint16_t xov[2] = {0, 0};
    if (a.xo16 && xo_hoisted) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (osrc[j] >= 0) xov[j] = reinterpret_cast<const uint16_t*>(srow)[osrc[j]];
    }
    if constexpr (FILL) {
      if (has_out) {
        uint16_t* hrow = reinterpret_cast<uint16_t*>(s_ring + s * row_stride);
        const uint16_t h0 = hrow[first_base];  // a base column: never overwritten
        const int i_end = o_hi + 8 < static_cast<int>(a.n_out) ? o_hi + 8 : static_cast<int>(a.n_out);
        for (int i = o_lo + tid; i < i_end; i += nt) {
          const int col = __ldg(&a.out_src[i]) - in_lo;
          if (col >= 0 && col < in_n) hrow[col] = h0;
        }
        __syncthreads();  // (F)
      }
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        const int v = tid + i * nt;
        raw[i] = in_row(v) ? srow[v] : make_uint4(0, 0, 0, 0);
      }
    }
    // ---- pass 1: packed min / max over the slice's base columns
    __half2 hmin = u2h2(0x7C007C00u), hmax = u2h2(0xFC00FC00u);
    {
      const uint32_t h0 = reinterpret_cast<const uint16_t*>(srow)[first_base];
      const uint32_t fill = h0 | (h0 << 16);
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        if (!in_row(tid + i * nt)) continue;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const uint32_t mk = FILL ? 0u : (&lmw[FILL ? 0 : i].x)[w];
          const __half2 x2 = u2h2(((&raw[i].x)[w] & ~mk) | (fill & mk));
          hmin = __hmin2_nan(hmin, x2);
          hmax = __hmax2_nan(hmax, x2);
        }
      }
    }
    float vmin, vmax;
    int nonfinite;
    {
      const float2 fmn = __half22float2(hmin);
      const float2 fmx = __half22float2(hmax);
      nonfinite = isnan(fmn.x) || isnan(fmn.y) || isnan(fmx.x) || isnan(fmx.y) || fmx.x == INFINITY ||
                  fmx.y == INFINITY || fmn.x == -INFINITY || fmn.y == -INFINITY;
      vmin = fminf(fmn.x, fmn.y);
      vmax = fmaxf(fmx.x, fmx.y);
    }
    vmin = redux_min(vmin);
    vmax = redux_max(vmax);
    nonfinite = __reduce_or_sync(0xffffffffu, nonfinite);
    if ((tid & 31) == 0) { s_min[tid >> 5] = vmin; s_max[tid >> 5] = vmax; s_nf[tid >> 5] = nonfinite; }
    __syncthreads();  // (A)
    const int xp = it & 1;
    if (tid == 0) {
      const int rn = t + stages * ncl;
      if (rn < M) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&s_full[s], row_bytes);
        bulk_load_1d(s_ring + s * row_stride, xg + static_cast<int64_t>(rn) * a.ldx, row_bytes, &s_full[s]);
      }
    }
    if (tid < 32) {
      // the CTA's partial -> every CTA of the cluster
      const int l = tid;
      float m0 = redux_min(l < nwarps ? s_min[l] : INFINITY);
      float m1 = redux_max(l < nwarps ? s_max[l] : -INFINITY);
      const int nf = __reduce_or_sync(0xffffffffu, l < nwarps ? s_nf[l] : 0);
      if (l == 0) mbar_arrive_expect_tx(&s_xbar[xp], 16u * C);
      if (l < C)
        st_async_cluster_v4(&s_x[xp][rank], static_cast<uint32_t>(l),
                            make_uint4(__float_as_uint(m0), __float_as_uint(m1), static_cast<uint32_t>(nf), 0u),
                            &s_xbar[xp]);
    }
    mbar_wait(&s_xbar[xp], (it >> 1) & 1);
    {
      const int l = tid & 31;
      const uint4 px = l < C ? s_x[xp][l] : make_uint4(__float_as_uint(INFINITY), __float_as_uint(-INFINITY), 0u, 0u);
      vmin = redux_min(__uint_as_float(px.x));
      vmax = redux_max(__uint_as_float(px.y));
      nonfinite = __reduce_or_sync(0xffffffffu, static_cast<int>(px.z));
    }
    if (vmin == 0.0f) {
      // rare: the sign of a zero minimum is the first-seen zero's (cluster-uniform branch)
      unsigned key = 0xFFFFFFFFu;
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        const int v = tid + i * nt;
        if (!in_row(v)) continue;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float x = elem<__half>(raw[i], e);
          uint32_t mbyte = 0u;
          if constexpr (!FILL) mbyte = ((e < 4 ? lm[i].x : lm[i].y) >> (8 * (e & 3))) & 0xFFu;
          else mbyte = (v * 8 + e < first_base) ? 1u : 0u;
          if (mbyte == 0 && x == 0.0f) {
            const unsigned k = (static_cast<unsigned>(in_lo + v * 8 + e) << 1) | (__float_as_uint(x) >> 31);
            key = k < key ? k : key;
          }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const unsigned o = __shfl_xor_sync(0xffffffffu, key, off);
        key = o < key ? o : key;
      }
      if ((tid & 31) == 0) s_key[tid >> 5] = key;
      __syncthreads();
      const int kp = kround & 1;
      if (tid < 32) {
        unsigned k = 0xFFFFFFFFu;
        for (int w = 0; w < nwarps; ++w) k = s_key[w] < k ? s_key[w] : k;
        if (tid == 0) mbar_arrive_expect_tx(&s_kbar[kp], 16u * C);
        if (tid < C)
          st_async_cluster_v4(&s_k[kp][rank], static_cast<uint32_t>(tid), make_uint4(k, 0u, 0u, 0u), &s_kbar[kp]);
      }
      mbar_wait(&s_kbar[kp], (kround >> 1) & 1);
      ++kround;
      key = 0xFFFFFFFFu;
      for (int r = 0; r < C; ++r) key = s_k[kp][r].x < key ? s_k[kp][r].x : key;
      vmin = (key & 1u) ? -0.0f : 0.0f;
    }
    const float range = __fsub_rn(vmax, vmin);
    const float scale = range == 0.0f ? 1.0f : __fdiv_rn(range, kLevels);
    const float rcp = __frcp_rn(scale);
    if (tid == 0 && rank == 0) {
      if (nonfinite && a.err) atomicExch(a.err, 1);
      a.scale[t] = scale;
      a.zero[t] = vmin;
    }
    const float rcp_lo = __fmul_rd(rcp, 1.0f - 0x1p-20f), rcp_hi = __fmul_ru(rcp, 1.0f + 0x1p-20f);
    const unsigned long long rlo2 = f32x2_pack(rcp_lo, rcp_lo), rhi2 = f32x2_pack(rcp_hi, rcp_hi);
    constexpr float kMagic = 12582912.0f - static_cast<float>(kHr);
    const unsigned long long magic2 = f32x2_pack(kMagic, kMagic);

    // ---- pass 2: codes for every column of the slice
    uint32_t near_vec = 0;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int v = tid + i * nt;
      if (!in_row(v)) continue;
      uint32_t tb[8];
      uint32_t diff = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t xw = (&raw[i].x)[w];
        const unsigned long long d2 = f32x2_pack(sub_f16_f32(xw & 0xFFFFu, vmin), sub_f16_f32(xw >> 16, vmin));
        unsigned long long tl2, th2;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(tl2) : "l"(d2), "l"(rlo2), "l"(magic2));
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(th2) : "l"(d2), "l"(rhi2), "l"(magic2));
        const uint32_t l0 = static_cast<uint32_t>(tl2), l1 = static_cast<uint32_t>(tl2 >> 32);
        diff |= (l0 ^ static_cast<uint32_t>(th2)) | (l1 ^ static_cast<uint32_t>(th2 >> 32));
        tb[2 * w] = l0;
        tb[2 * w + 1] = l1;
      }
      near_vec |= (diff != 0u ? 1u : 0u) << i;
      const uint32_t w0 = __byte_perm(__byte_perm(tb[0], tb[1], 0x0040), __byte_perm(tb[2], tb[3], 0x0040), 0x5410);
      const uint32_t w1 = __byte_perm(__byte_perm(tb[4], tb[5], 0x0040), __byte_perm(tb[6], tb[7], 0x0040), 0x5410);
      *reinterpret_cast<uint2*>(s_codes + v * 8) = make_uint2(w0, w1);
    }
    if (near_vec) {
#pragma unroll 1
      for (uint32_t nv = near_vec; nv; nv &= nv - 1) {
        const int iv = __ffs(nv) - 1;
        const int v = tid + iv * nt;
        uint4 rv = raw[0];
#pragma unroll
        for (int i = 1; i < VPT; ++i)
          if (i == iv) rv = raw[i];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int c = v * 8 + e;
          const uint32_t hw = (&rv.x)[e >> 1];
          const float d = __fsub_rn(__half2float(__ushort_as_half(static_cast<unsigned short>((e & 1) ? hw >> 16 : hw & 0xFFFFu))), vmin);
          if (__float_as_uint(__fmaf_rn(d, rcp_lo, kMagic)) != __float_as_uint(__fmaf_rn(d, rcp_hi, kMagic)))
            s_codes[c] = static_cast<uint8_t>(static_cast<int>(quant_slow(d, scale)) - kHr);
        }
      }
    }
    __syncthreads();  // (B) codes complete
    // ---- outliers of this slice (ascending index order, runtime.cpp:217)
    if (a.xo16) {
      uint16_t* xo = reinterpret_cast<uint16_t*>(a.xo16) + static_cast<int64_t>(t) * opad;
      if (xo_hoisted) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = o_lo + tid + j * nt;
          if (i < o_hi) xo[i] = xov[j];
        }
      } else {
        const uint16_t* xrow = reinterpret_cast<const uint16_t*>(xg + static_cast<int64_t>(t) * a.ldx);
        for (int i = o_lo + tid; i < o_hi; i += nt)
          xo[i] = (has_out && i < a.n_out) ? xrow[__ldg(&a.out_src[i]) - in_lo] : 0;
      }
    }
    // ---- compacted code chunks of this slice (window offsets rebased to the slice)
    uint4* dst = reinterpret_cast<uint4*>(a.q8 + static_cast<int64_t>(t) * a.kpad);
    for (int cidx = ch_lo + tid; cidx < ch_hi; cidx += nt) {
      const uint4 d = __ldg(cdesc + cidx);
      if (d.x == 0xFFFFFFFFu) continue;  // general chunk (below)
      const uint32_t* wa = reinterpret_cast<const uint32_t*>(s_codes + (d.x & 0xFFFFu) - in_lo);
      const uint32_t* wb = reinterpret_cast<const uint32_t*>(s_codes + (d.y & 0xFFFFu) - in_lo);
      const uint32_t sa = d.x >> 16, sb = d.y >> 16;
      const uint32_t a0 = wa[0], a1 = wa[1], a2 = wa[2], a3 = wa[3], a4 = wa[4];
      const uint32_t b0 = wb[0], b1 = wb[1], b2 = wb[2], b3 = wb[3], b4 = wb[4];
      const uint32_t o0 = __byte_perm(__byte_perm(a0, a1, sa), __byte_perm(b0, b1, sb), d.z & 0xFFFFu);
      const uint32_t o1 = __byte_perm(__byte_perm(a1, a2, sa), __byte_perm(b1, b2, sb), d.z >> 16);
      const uint32_t o2 = __byte_perm(__byte_perm(a2, a3, sa), __byte_perm(b2, b3, sb), d.w & 0xFFFFu);
      const uint32_t o3 = __byte_perm(__byte_perm(a3, a4, sa), __byte_perm(b3, b4, sb), d.w >> 16);
      dst[cidx] = make_uint4(o0, o1, o2, o3);
    }
    for (int gi = g_lo + tid; gi < g_hi; gi += nt) {
      const int cidx = a.gen_chunk[gi];
      const uint4 g0 = __ldg(reinterpret_cast<const uint4*>(a.gather + cidx * 16));
      const uint4 g1 = __ldg(reinterpret_cast<const uint4*>(a.gather + cidx * 16 + 8));
      const uint32_t gw[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      uint32_t w[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t c0 = s_codes[(gw[2 * kk] & 0xFFFFu) - in_lo], c1 = s_codes[(gw[2 * kk] >> 16) - in_lo];
        const uint32_t c2 = s_codes[(gw[2 * kk + 1] & 0xFFFFu) - in_lo], c3 = s_codes[(gw[2 * kk + 1] >> 16) - in_lo];
        w[kk] = __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410);
      }
      dst[cidx] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (++s == stages) { s = 0; ph ^= 1u; }
  }
  cluster_sync();  // no CTA leaves while a peer may still address its shared memory
}

__global__ void split_kernel(const SplitArgs a) {
  for (int64_t t = blockIdx.y; t < a.M; t += gridDim.y)  // rows beyond grid.y's 65535 limit
  for (int64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < a.kb + a.opad; j += gridDim.x * blockDim.x) {
    if (j < a.kb) {
      const int64_t c = a.base_src[j];
      a.xbase[t * a.kb + j] = a.x_is_f32 ? reinterpret_cast<const float*>(a.x)[t * a.ldx + c]
                                         : __half2float(reinterpret_cast<const __half*>(a.x)[t * a.ldx + c]);
    } else if (a.xo32) {
      const int64_t i = j - a.kb;
      if (i < a.n_out) {
        const int64_t c = a.out_src[i];
        a.xo32[t * a.n_out + i] = a.x_is_f32 ? reinterpret_cast<const float*>(a.x)[t * a.ldx + c]
                                             : __half2float(reinterpret_cast<const __half*>(a.x)[t * a.ldx + c]);
      }
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
  const int64_t rb = bits == 4 ? (cols + 1) / 2 : cols;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
  for (int64_t c = blockIdx.x * blockDim.x + threadIdx.x; c < kpad; c += gridDim.x * blockDim.x) {
    int8_t v = 0;
    if (c < cols) {
      if (bits == 8) v = static_cast<int8_t>(packed[r * rb + c]);
      else {
        const uint8_t b = packed[r * rb + c / 2];
        v = static_cast<int8_t>(static_cast<int>((c & 1) ? (b >> 4) : (b & 0xF)) - 8);
      }
    }
    dst[r * kpad + c] = v;
  }
}

__global__ void f32_to_f16_kernel(const float* __restrict__ src, int64_t rows, int64_t cols,
                                  __half* __restrict__ dst, int64_t pitch) {
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
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
  for (int64_t t = blockIdx.y; t < M; t += gridDim.y)
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

// rtn_quantize_weights (quantizer.cpp:339-371 with rtn_quantize_row :251-264 and
// quantize_to_grid :17-22): per output row, FP64 scale = amax / maxq, q =
// clamp(round-half-away(w / scale)), packed ABI codes, wreduced = scale_f32 * sum q.
// One CTA per row; every FP64 op is an explicit _rn intrinsic (bit-exact).
__global__ void __launch_bounds__(256) rtn_rows_kernel(const float* __restrict__ w, int64_t K,
                                                       const int32_t* __restrict__ base_src, int64_t kb,
                                                       const int32_t* __restrict__ out_src, int64_t n_out, int bits,
                                                       uint8_t* __restrict__ base, float* __restrict__ scales,
                                                       float* __restrict__ wreduced, float* __restrict__ outlier_w,
                                                       const float* __restrict__ clip) {
  __shared__ float s_amax[8];
  __shared__ long long s_sum[8];
  const int64_t r = blockIdx.x;
  const float* row = w + r * K;
  const int tid = threadIdx.x;
  float amax = 0.0f;
  for (int64_t j = tid; j < kb; j += blockDim.x) amax = fmaxf(amax, fabsf(row[base_src[j]]));
  for (int off = 16; off; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  if ((tid & 31) == 0) s_amax[tid >> 5] = amax;
  __syncthreads();
  amax = s_amax[0];
  for (int i = 1; i < 8; ++i) amax = fmaxf(amax, s_amax[i]);
  const int maxq = (1 << (bits - 1)) - 1;
  const bool zero_row = amax == 0.0f;
  // rtn_quantize_row: scale = double(clip_factor) * amax / maxq (clip_factor 1 without clipping)
  const double camax = clip ? __dmul_rn(static_cast<double>(clip[r]), static_cast<double>(amax))
                            : static_cast<double>(amax);
  const double scale = zero_row ? 1.0 : __ddiv_rn(camax, static_cast<double>(maxq));
  const double inv_scale = __ddiv_rn(1.0, scale);
  const int64_t rb = bits == 4 ? (kb + 1) / 2 : kb;
  long long qsum = 0;
  for (int64_t p = tid; p < rb; p += blockDim.x) {
    const int per = bits == 4 ? 2 : 1;
    uint8_t byte = 0;
    for (int u = 0; u < per; ++u) {
      const int64_t j = p * per + u;
      if (j >= kb) break;
      int qi = 0;
      if (!zero_row) {
        const double t = __dmul_rn(static_cast<double>(row[base_src[j]]), inv_scale);
        double qd = floor(__dadd_rn(fabs(t), 0.5));
        if (qd > maxq) qd = maxq;
        qi = static_cast<int>(t < 0.0 ? -qd : qd);
      }
      qsum += qi;
      if (bits == 8) byte = static_cast<uint8_t>(static_cast<int8_t>(qi));
      else byte |= static_cast<uint8_t>((qi + 8) & 0xF) << (4 * u);
    }
    base[r * rb + p] = byte;
  }
  for (int off = 16; off; off >>= 1) qsum += __shfl_xor_sync(0xffffffffu, qsum, off);
  if ((tid & 31) == 0) s_sum[tid >> 5] = qsum;
  __syncthreads();
  if (tid == 0) {
    long long total = 0;
    for (int i = 0; i < 8; ++i) total += s_sum[i];
    const float sf = __double2float_rn(scale);
    scales[r] = sf;
    wreduced[r] = __double2float_rn(__dmul_rn(static_cast<double>(sf), static_cast<double>(total)));
  }
  for (int64_t i = tid; i < n_out; i += blockDim.x) outlier_w[r * n_out + i] = row[out_src[i]];
}

// 2:4 compression of the GEMM-layout weights (layer create). Thread = one row x
// 32 logical K (8 groups of 4): two kept codes per group (the non-zero ones, padded
// with the lowest remaining positions), ascending, and the group's metadata nibble
// (index of the first kept value in bits [1:0], second in [3:2]).
__global__ void compress24_kernel(const int8_t* __restrict__ w8, int64_t N, int64_t kpad, int8_t* __restrict__ w_sp,
                                  uint8_t* __restrict__ meta, int64_t npad, int* bad) {
  const int64_t per_row = kpad / 32;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= N * per_row) return;
  const int64_t n = idx / per_row, o = idx % per_row;
  const uint4* src = reinterpret_cast<const uint4*>(w8 + n * kpad + 32 * o);
  const uint4 lo = src[0], hi = src[1];
  const uint32_t words[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
  uint32_t vals[4] = {0, 0, 0, 0};
  uint32_t nib = 0;
  bool over = false;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const uint32_t w = words[g];
    int i0 = -1, i1 = -1, cnt = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if ((w >> (8 * e)) & 0xFFu) {
        ++cnt;
        if (i0 < 0) i0 = e;
        else if (i1 < 0) i1 = e;
      }
    over |= cnt > 2;
    if (i0 < 0) {
      i0 = 0;
      i1 = 1;
    } else if (i1 < 0) {
      if (i0 == 3) i0 = 2, i1 = 3;
      else i1 = i0 + 1;
    }
    const uint32_t v0 = (w >> (8 * i0)) & 0xFFu, v1 = (w >> (8 * i1)) & 0xFFu;
    vals[g >> 1] |= (v0 | (v1 << 8)) << (16 * (g & 1));
    nib |= static_cast<uint32_t>(i0 | (i1 << 2)) << (4 * g);
  }
  if (over) atomicExch(bad, 1);
  *reinterpret_cast<uint4*>(w_sp + n * (kpad / 2) + 16 * o) = make_uint4(vals[0], vals[1], vals[2], vals[3]);
  const int64_t g0 = 8 * o, kb = g0 / 64, gl = g0 % 64, h = gl / 32;
  *reinterpret_cast<uint32_t*>(meta + ((2 * kb + h) * npad + n) * 16 + (gl % 32) / 2) = nib;
}

// INT4 weight repack for the W4 GEMM tiles: thread = one 16-byte output chunk.
__global__ void pack_w4_kernel(const int8_t* __restrict__ w8, int64_t N, int64_t kpad, uint8_t* __restrict__ w4) {
  const int64_t per_row = kpad / 32;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= N * per_row) return;
  const int64_t n = idx / per_row, c = idx % per_row;
  const uint4* src = reinterpret_cast<const uint4*>(w8 + n * kpad + 32 * c);
  const uint4 lo = src[0], hi = src[1];
  uint32_t out[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t a = (&lo.x)[k] & 0x0F0F0F0Fu, b = (&hi.x)[k] & 0x0F0F0F0Fu;
    out[k] = a | (b << 4);
  }
  *reinterpret_cast<uint4*>(w4 + n * (kpad / 2) + 16 * c) = make_uint4(out[0], out[1], out[2], out[3]);
}

// ABI i4p (stored = v + 8, low nibble = even column) -> device INT4 chunk layout:
// byte i of 16-byte chunk c = nibble(k = 32c + i) | nibble(k = 32c + 16 + i) << 4, with
// nibble = two's complement 4-bit v = stored ^ 8, zero past kb.
__global__ void pack_w4_abi_kernel(const uint8_t* __restrict__ src, int64_t N, int64_t kb, uint8_t* __restrict__ w4,
                                   int64_t kpad) {
  const int64_t per_row = kpad / 32;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= N * per_row) return;
  const int64_t n = idx / per_row, c = idx % per_row;
  const uint8_t* row = src + n * ((kb + 1) / 2);
  auto nib = [&](int64_t k) -> uint32_t {
    if (k >= kb) return 0u;
    const uint32_t b = row[k >> 1];
    return (((k & 1) ? (b >> 4) : b) & 0xFu) ^ 8u;
  };
  uint32_t out[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = 4 * w + b;
      v |= (nib(32 * c + i) | (nib(32 * c + 16 + i) << 4)) << (8 * b);
    }
    out[w] = v;
  }
  *reinterpret_cast<uint4*>(w4 + n * (kpad / 2) + 16 * c) = make_uint4(out[0], out[1], out[2], out[3]);
}

dim3 grid2(int64_t cols, int64_t rows) {
  int64_t gx = (cols + 255) / 256;
  if (gx > 64) gx = 64;
  if (gx < 1) gx = 1;
  // rows past grid.y's limit are walked by the kernels' row loops
  return dim3(static_cast<unsigned>(gx), static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(rows, 65535))));
}

}  // namespace

template <typename T, int B>
cudaError_t launch_quantize_t(const QuantArgs& a, cudaStream_t stream) {
  constexpr int E = 16 / sizeof(T);
  const int64_t nvec = (a.K + E - 1) / E;
  int threads = nvec > 256 * 4 ? 512 : 256;
  int64_t vpt = (nvec + threads - 1) / threads;
  if (vpt > 16) return cudaErrorInvalidValue;  // row wider than 512 x 16 vectors
  // exact fit (no bounds checks): threads * vpt == nvec with 16-byte aligned rows
  bool full = false;
  const bool aligned = (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && (a.ldx * static_cast<int64_t>(sizeof(T))) % 16 == 0 &&
                       a.K % E == 0;
  if (aligned) {
    for (int v : {4, 8, 2, 1}) {
      if (nvec % v == 0 && (nvec / v) % 32 == 0 && nvec / v >= 64 && nvec / v <= 512) {
        threads = static_cast<int>(nvec / v);
        vpt = v;
        full = true;
        break;
      }
    }
  }
  const size_t smem = static_cast<size_t>(round_up(a.K, 16) + 16) + static_cast<size_t>(nvec) * 16;
  const dim3 grid(static_cast<unsigned>(a.M));
#define QUIK_Q_LAUNCH(V)                                                                                   \
  do {                                                                                                     \
    if (full && V <= 8) {                                                                                  \
      cudaError_t e = ensure_smem_attr(quantize_rows_kernel<T, B, V, true>, static_cast<int>(smem));       \
      if (e != cudaSuccess) return e;                                                                      \
      quantize_rows_kernel<T, B, V, true><<<grid, threads, smem, stream>>>(a);                            \
    } else {                                                                                               \
      cudaError_t e = ensure_smem_attr(quantize_rows_kernel<T, B, V, false>, static_cast<int>(smem));      \
      if (e != cudaSuccess) return e;                                                                      \
      quantize_rows_kernel<T, B, V, false><<<grid, threads, smem, stream>>>(a);                           \
    }                                                                                                      \
  } while (0)
  if (vpt <= 1) QUIK_Q_LAUNCH(1);
  else if (vpt <= 2) QUIK_Q_LAUNCH(2);
  else if (vpt <= 4) QUIK_Q_LAUNCH(4);
  else if (vpt <= 8) QUIK_Q_LAUNCH(8);
  else QUIK_Q_LAUNCH(16);
#undef QUIK_Q_LAUNCH
  return cudaGetLastError();
}

template <int B>
cudaError_t launch_quantize_hot(const QuantArgs& a, cudaStream_t stream) {
  const int64_t nvec = a.K / 8;
  // about 4 warps per row (measured: 128-thread rows beat 256-thread ones at cfg2 q/k/v/o
  // 12.1 -> 10.7 us and cfg3 28.8 -> 28.2 us; fewer threads per block barrier)
  int vpt = 1;
  while (vpt < 8 && (nvec + vpt - 1) / vpt > 128) vpt *= 2;
  // an exact fit (FULL: no bounds checks, fewer registers) wins over the 4-warp target:
  // the exact fit with the fewest threads >= 128, else the one with the most threads
  // (4-vector rows up to 512 threads: K = 9216 fits exactly at 288 threads, OPT-66B fc1
  // K1 20.7 -> 19.8 us)
  int best = 0;
  int64_t best_thr = 0;
  for (int v = 1; v <= 8; v *= 2) {
    const int64_t thr = nvec / v;
    if (thr * v != nvec || thr % 32 || thr > (v >= 4 ? 512 : 256)) continue;
    const bool wide = thr >= 128, best_wide = best_thr >= 128;
    if (!best || (wide && (!best_wide || thr < best_thr)) || (!wide && !best_wide && thr > best_thr)) {
      best = v;
      best_thr = thr;
    }
  }
  if (best) vpt = best;
  static const int vpt_env = [] {  // tuning knob: QUIK_K1_VPT forces 16-byte vectors per thread
    const char* e = getenv("QUIK_K1_VPT");
    return e ? atoi(e) : 0;
  }();
  if ((vpt_env == 1 || vpt_env == 2 || vpt_env == 4 || vpt_env == 8) &&
      (nvec + vpt_env - 1) / vpt_env <= (vpt_env >= 4 ? 512 : 256))  // the kernel's launch bounds
    vpt = vpt_env;
  const int threads = static_cast<int>(round_up((nvec + vpt - 1) / vpt, 32));
  if (a.kpad / 16 > static_cast<int64_t>(vpt > 1 ? vpt / 2 : 1) * threads) return cudaErrorNotSupported;
  const int row_stride = static_cast<int>(round_up(a.K * 2, 128));
  const int codes = static_cast<int>(round_up(round_up(a.K, 16) + 32, 128));
  // ring depth: about 32 KB of rows per CTA (a slot is refilled as soon as its row is in
  // registers, so one stage still overlaps the next row's load), <= 8 stages
  static const int ring_kb = [] {  // tuning knob: QUIK_K1_RING_KB (ring bytes per CTA)
    const char* e = getenv("QUIK_K1_RING_KB");
    return e ? atoi(e) : 32;
  }();
  // One ring stage by default: a slot is refilled at barrier A of its own row, so one
  // stage still overlaps the next row's load with this row's codes, and the smaller CTA
  // fits more CTAs per SM (measured, k1_bench: 70B down 110.7 -> 96.6 us with FILL below,
  // 7B down 33.9 -> 27.6, cfg3 28.0 -> 27.4, 7B q/k/v/o 10.9 -> 10.4). QUIK_K1_STAGES=n
  // forces n stages, QUIK_K1_STAGES=0 the ring_kb rule above.
  int stages = static_cast<int>(std::max<int64_t>(2, std::min<int64_t>(8, (ring_kb * 1024) / row_stride)));
  static const int stages_env = [] {
    const char* e = getenv("QUIK_K1_STAGES");
    return e ? atoi(e) : 1;
  }();
  if (stages_env >= 1 && stages_env <= 8) stages = stages_env;
  // VPT 8 rows run the FILL kernel (no lane-mask registers: 64 instead of 106-121, two
  // CTAs per SM); QUIK_K1_FILL=0 keeps the masks in registers, =2 uses FILL from VPT 2
  // (measured mixed: OPT-66B fc1 19.9 -> 19.3 us, 7B q/k/v/o 10.4 -> 11.1)
  static const int fill_env = [] {
    const char* e = getenv("QUIK_K1_FILL");
    return e ? atoi(e) : 1;
  }();
  const bool fill = (fill_env == 1 && vpt == 8) || (fill_env == 2 && vpt >= 2);
  while (stages > 1 && codes + stages * row_stride > 200 * 1024) --stages;
  const int smem = codes + stages * row_stride;
  const bool full = static_cast<int64_t>(threads) * vpt == nvec;
  static const int wait_env = [] {  // tuning knob: QUIK_K1_WAIT=1 sleep-waits on the row ring
    const char* e = getenv("QUIK_K1_WAIT");
    return e ? atoi(e) : 0;
  }();
  static const int hot_pdl = [] {  // tuning: QUIK_K1_PDL=0 launches without programmatic serialization
    const char* e = getenv("QUIK_K1_PDL");
    return e ? atoi(e) : 1;
  }();
  QuantArgs ah = a;
  ah.hot_flags = wait_env ? 1 : 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#define QUIK_QH_LAUNCH(V)                                                                                  \
  do {                                                                                                     \
    auto kern = fill ? (full ? quantize_hot_fill_kernel<B, V, true> : quantize_hot_fill_kernel<B, V, false>)      \
                     : (full ? quantize_hot_kernel<B, V, true> : quantize_hot_kernel<B, V, false>);             \
    cudaError_t e = ensure_smem_attr(kern, smem);                                                          \
    if (e != cudaSuccess) return e;                                                                        \
    int per_sm = 0;                                                                                        \
    e = occupancy_cached(kern, threads, smem, &per_sm);                                                    \
    if (e != cudaSuccess) return e;                                                                        \
    const int64_t grid = std::min<int64_t>(a.M, static_cast<int64_t>(std::max(per_sm, 1)) * sms);          \
    cudaLaunchConfig_t cfg{};                                                                              \
    cfg.gridDim = dim3(static_cast<unsigned>(grid));                                                       \
    cfg.blockDim = dim3(threads);                                                                          \
    cfg.dynamicSmemBytes = smem;                                                                           \
    cfg.stream = stream;                                                                                   \
    cudaLaunchAttribute attr[1];                                                                           \
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                       \
    attr[0].val.programmaticStreamSerializationAllowed = 1;                                                \
    cfg.attrs = attr;                                                                                      \
    cfg.numAttrs = hot_pdl ? 1 : 0;                                                                        \
    e = cudaLaunchKernelEx(&cfg, kern, ah, stages, row_stride);                                            \
    if (e != cudaSuccess) return e;                                                                        \
  } while (0)
  if (vpt == 1) QUIK_QH_LAUNCH(1);
  else if (vpt == 2) QUIK_QH_LAUNCH(2);
  else if (vpt == 4) QUIK_QH_LAUNCH(4);
  else QUIK_QH_LAUNCH(8);
#undef QUIK_QH_LAUNCH
  return cudaGetLastError();
}

template <int B>
cudaError_t launch_quantize_wide(const QuantArgs& a, cudaStream_t stream) {
  // launched WITHOUT programmatic serialization by default: under PDL its clusters start
  // while the previous layer's GEMM still holds SMs and the persistent row ranges of the
  // late clusters stretch the launch (OPT-66B fc2 M = 2048 step 587 -> 540 us without;
  // QUIK_K1_WIDE_PDL=1 restores it)
  static const int wide_pdl = [] {
    const char* e = getenv("QUIK_K1_WIDE_PDL");
    return e ? atoi(e) : 0;
  }();
  const int C = a.n_slice;
  const int64_t nvec = a.slice_cols_max / 8;
  int vpt = 1;
  while (vpt < 8 && (nvec + vpt - 1) / vpt > 128) vpt *= 2;
  const int threads = static_cast<int>(round_up((nvec + vpt - 1) / vpt, 32));
  if (threads > (vpt >= 8 ? 512 : 256)) return cudaErrorNotSupported;
  const int row_stride = static_cast<int>(round_up(static_cast<int64_t>(a.slice_cols_max) * 2, 128));
  int stages = static_cast<int>(std::max<int64_t>(2, std::min<int64_t>(8, (32 * 1024) / row_stride)));
  // one ring stage by default (as the hot kernel; with the FILL kernel below: OPT-66B
  // fc2 82.4 -> 70.0 us, Falcon-180B fc2 139.0 -> 117.4); QUIK_K1_WIDE_STAGES=n forces n,
  // =0 the 32 KB rule above
  static const int wstages_env = [] {
    const char* e = getenv("QUIK_K1_WIDE_STAGES");
    return e ? atoi(e) : 1;
  }();
  if (wstages_env >= 1 && wstages_env <= 8) stages = wstages_env;
  while (stages > 1 && a.slice_code_bytes + stages * row_stride > 200 * 1024) --stages;
  const int smem = a.slice_code_bytes + stages * row_stride;
  // FILL kernel for eight-vector slices (no lane-mask registers; QUIK_K1_WIDE_FILL=0 off)
  static const int wfill_env = [] {
    const char* e = getenv("QUIK_K1_WIDE_FILL");
    return e ? atoi(e) : 1;
  }();
  const bool wfill = wfill_env != 0 && vpt == 8;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#define QUIK_QW_LAUNCH(V)                                                                                   \
  do {                                                                                                      \
    auto kern = wfill ? quantize_wide_kernel<B, V, true> : quantize_wide_kernel<B, V, false>;               \
    cudaError_t e = ensure_smem_attr(kern, smem);                                                           \
    if (e != cudaSuccess) return e;                                                                         \
    cudaLaunchConfig_t cfg{};                                                                               \
    cfg.blockDim = dim3(threads);                                                                           \
    cfg.dynamicSmemBytes = smem;                                                                            \
    cfg.stream = stream;                                                                                    \
    cudaLaunchAttribute attr[2];                                                                            \
    attr[0].id = cudaLaunchAttributeClusterDimension;                                                       \
    attr[0].val.clusterDim.x = C;                                                                           \
    attr[0].val.clusterDim.y = 1;                                                                           \
    attr[0].val.clusterDim.z = 1;                                                                           \
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                        \
    attr[1].val.programmaticStreamSerializationAllowed = 1;                                                 \
    cfg.attrs = attr;                                                                                       \
    cfg.numAttrs = wide_pdl ? 2 : 1;                                                                        \
    /* as many clusters as are co-resident (the row loop is persistent) */                                  \
    static int cached_key = -1, cached_clusters = 0;                                                        \
    const int key = (C << 24) ^ (threads << 12) ^ smem;                                                     \
    int clusters = 0;                                                                                       \
    if (key == cached_key) {                                                                                \
      clusters = cached_clusters;                                                                           \
    } else {                                                                                                \
      cfg.gridDim = dim3(static_cast<unsigned>(C * sms));                                                   \
      e = cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg);                                            \
      if (e != cudaSuccess) return e;                                                                       \
      cached_key = key;                                                                                     \
      cached_clusters = clusters;                                                                           \
    }                                                                                                       \
    if (clusters < 1) return cudaErrorNotSupported;                                                         \
    const int64_t ncl = std::min<int64_t>(a.M, clusters);                                                   \
    cfg.gridDim = dim3(static_cast<unsigned>(ncl * C));                                                     \
    e = cudaLaunchKernelEx(&cfg, kern, a, stages, row_stride);                                              \
    if (e != cudaSuccess) return e;                                                                         \
  } while (0)
  if (vpt == 1) QUIK_QW_LAUNCH(1);
  else if (vpt == 2) QUIK_QW_LAUNCH(2);
  else if (vpt == 4) QUIK_QW_LAUNCH(4);
  else QUIK_QW_LAUNCH(8);
#undef QUIK_QW_LAUNCH
  return cudaGetLastError();
}

cudaError_t launch_quantize(const QuantArgs& a, cudaStream_t stream) {
  if (a.M == 0) return cudaSuccess;
  // hot path: f16 rows, 16-byte aligned, GEMM-layout outputs only
  const bool hot = !a.x_is_f32 && a.q8 && !a.packed && !a.xo32 && a.chunk_desc && a.gather && a.K % 8 == 0 &&
                   a.K / 8 <= 512 * 8 && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && (a.ldx * 2) % 16 == 0;
  static const int variant = [] {  // tuning: QUIK_K1_VARIANT=0 forces the general kernel, 2 the one-CTA-per-row hot kernel
    const char* e = getenv("QUIK_K1_VARIANT");
    return e ? atoi(e) : 1;
  }();
  // wide rows: K1 over a cluster of CTAs per row (the layer's slices)
  const bool wide = !a.x_is_f32 && a.q8 && !a.packed && !a.xo32 && a.chunk_desc && a.gather && a.n_slice >= 2 &&
                    a.slice_desc && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && (a.ldx * 2) % 16 == 0;
  if (a.pre_stat) {
    // prescaled rows: the hot kernel consumes and resets the keys; any other kernel
    // reduces the rows itself, then the keys are reset for the next forward
    if (hot && variant != 0) {
      const cudaError_t e = a.bits == 4 ? launch_quantize_hot<4>(a, stream) : launch_quantize_hot<8>(a, stream);
      if (e != cudaErrorNotSupported) return e;
    }
    QuantArgs b = a;
    b.pre_stat = nullptr;
    const cudaError_t e = launch_quantize(b, stream);
    if (e != cudaSuccess) return e;
    return launch_hstat_init(a.pre_stat, a.M, stream);
  }
  if (wide && variant != 0 && variant != 2) {
    const cudaError_t e = a.bits == 4 ? launch_quantize_wide<4>(a, stream) : launch_quantize_wide<8>(a, stream);
    if (e != cudaErrorNotSupported) return e;
  }
  if (hot && variant != 0) {
    const cudaError_t e = a.bits == 4 ? launch_quantize_hot<4>(a, stream) : launch_quantize_hot<8>(a, stream);
    if (e != cudaErrorNotSupported) return e;  // else: shape outside the hot kernel's range
  }
  if (a.x_is_f32) return a.bits == 4 ? launch_quantize_t<float, 4>(a, stream) : launch_quantize_t<float, 8>(a, stream);
  return a.bits == 4 ? launch_quantize_t<__half, 4>(a, stream) : launch_quantize_t<__half, 8>(a, stream);
}

__global__ void hstat_init_kernel(uint4* stat, int64_t M) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < M) stat[i] = make_uint4(0xFFFFFFFFu, 0u, 0xFFFFFFFFu, 0u);
}

cudaError_t launch_hstat_init(uint4* stat, int64_t M, cudaStream_t stream) {
  if (M == 0) return cudaSuccess;
  hstat_init_kernel<<<static_cast<unsigned>((M + 255) / 256), 256, 0, stream>>>(stat, M);
  return cudaGetLastError();
}

cudaError_t launch_split(const SplitArgs& a, cudaStream_t stream) {
  if (a.M == 0 || a.kb + a.opad == 0) return cudaSuccess;
  split_kernel<<<grid2(a.kb + a.opad, a.M), 256, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_compress_24(const int8_t* w8, int64_t N, int64_t kpad, int8_t* w_sp, uint8_t* meta, int* bad,
                               cudaStream_t stream) {
  if (N == 0 || kpad == 0) return cudaSuccess;
  if (kpad % 256) return cudaErrorInvalidValue;
  const int64_t npad = round_up(N, kBlockM);
  cudaError_t e = cudaMemsetAsync(meta, 0, static_cast<size_t>(2 * (kpad / 256) * npad * 16), stream);
  if (e != cudaSuccess) return e;
  const int64_t work = N * (kpad / 32);
  compress24_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(w8, N, kpad, w_sp, meta, npad, bad);
  return cudaGetLastError();
}

cudaError_t launch_pack_w4(const int8_t* w8, int64_t N, int64_t kpad, uint8_t* w4, cudaStream_t stream) {
  if (N == 0 || kpad == 0) return cudaSuccess;
  const int64_t work = N * (kpad / 32);
  pack_w4_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(w8, N, kpad, w4);
  return cudaGetLastError();
}

cudaError_t launch_pack_w4_abi(const uint8_t* i4p, int64_t N, int64_t kb, uint8_t* w4, int64_t kpad,
                               cudaStream_t stream) {
  if (N == 0 || kpad == 0) return cudaSuccess;
  const int64_t work = N * (kpad / 32);
  pack_w4_abi_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, stream>>>(i4p, N, kb, w4, kpad);
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

cudaError_t launch_rtn_weights(const float* w, int64_t N, int64_t K, const int32_t* base_src, int64_t kb,
                               const int32_t* out_src, int64_t n_out, int bits, uint8_t* base, float* scales,
                               float* wreduced, float* outlier_w, const float* clip, cudaStream_t stream) {
  if (N == 0) return cudaSuccess;
  rtn_rows_kernel<<<static_cast<unsigned>(N), 256, 0, stream>>>(w, K, base_src, kb, out_src, n_out, bits, base,
                                                                scales, wreduced, outlier_w, clip);
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
