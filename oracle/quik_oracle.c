/*
 * quik_oracle.c — TEST INFRASTRUCTURE ONLY (see quik_oracle.h).
 *
 * C restatement of the reference's algorithm for the QUIK hot path. Every
 * function cites the reference file:line it follows (paths relative to
 * /root/reference/proj). Float arithmetic is written op by op and compiled with
 * -ffp-contract=off, like the reference.
 */
#include "quik_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

int64_t qo_row_bytes(int64_t cols, int bits) { return bits == 4 ? (cols + 1) / 2 : cols; }

/* packed.cpp:30-49 (int4: low nibble = even column, stored = v + 8, zero pad
 * nibble) and packed.cpp:51-60 (int8: two's complement bytes). */
int qo_pack(const int8_t* vals, int64_t rows, int64_t cols, int bits, uint8_t* out, int64_t* bad_row,
            int64_t* bad_col) {
  if (bits != 4 && bits != 8) return QO_INVALID_ARGUMENT;
  const int64_t rb = qo_row_bytes(cols, bits);
  memset(out, 0, (size_t)(rows * rb));
  const int lo = bits == 4 ? -8 : -128, hi = bits == 4 ? 7 : 127;
  for (int64_t r = 0; r < rows; ++r) {
    for (int64_t c = 0; c < cols; ++c) {
      const int v = vals[r * cols + c];
      if (v < lo || v > hi) {
        if (bad_row) *bad_row = r;
        if (bad_col) *bad_col = c;
        return QO_OUT_OF_RANGE;
      }
      if (bits == 8) {
        out[r * rb + c] = (uint8_t)(int8_t)v;
      } else {
        const uint8_t biased = (uint8_t)(v + 8);
        uint8_t* b = &out[r * rb + c / 2];
        *b = (c % 2 == 0) ? (uint8_t)((*b & 0xF0) | biased) : (uint8_t)((*b & 0x0F) | (biased << 4));
      }
    }
  }
  return QO_OK;
}

/* packed.cpp:68-91 */
void qo_unpack(const uint8_t* packed, int64_t rows, int64_t cols, int bits, int8_t* out) {
  const int64_t rb = qo_row_bytes(cols, bits);
  for (int64_t r = 0; r < rows; ++r) {
    for (int64_t c = 0; c < cols; ++c) {
      if (bits == 8) {
        out[r * cols + c] = (int8_t)packed[r * rb + c];
      } else {
        const uint8_t byte = packed[r * rb + c / 2];
        const uint8_t nib = (c % 2 == 0) ? (byte & 0x0F) : (byte >> 4);
        out[r * cols + c] = (int8_t)((int)nib - 8);
      }
    }
  }
}

/* packed.cpp:93-132: checks bits equal (:94-97), inner dims (:98-101), the
 * accumulator guard k <= 2^31 / (2^(b-1))^2 (:102-106); exact int32 sum. */
int qo_int_matmul(const uint8_t* x, int64_t t, int64_t xk, int xbits, const uint8_t* w, int64_t n, int64_t wk,
                  int wbits, int32_t* out) {
  if (xbits != wbits) return QO_INVALID_ARGUMENT;
  if (xk != wk) return QO_INVALID_ARGUMENT;
  if (xbits != 4 && xbits != 8) return QO_INVALID_ARGUMENT;
  const int64_t half = (int64_t)1 << (xbits - 1);
  if (xk > ((int64_t)1 << 31) / (half * half)) return QO_INVALID_ARGUMENT;
  const int64_t k = xk;
  int8_t* xv = (int8_t*)malloc((size_t)(t * k + 1));
  int8_t* wv = (int8_t*)malloc((size_t)(n * k + 1));
  qo_unpack(x, t, k, xbits, xv);
  qo_unpack(w, n, k, wbits, wv);
#pragma omp parallel for collapse(2) schedule(static) if (t * n * k > (1 << 16))
  for (int64_t i = 0; i < t; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      const int8_t* xr = xv + i * k;
      const int8_t* wr = wv + j * k;
      int32_t acc = 0;
      for (int64_t kk = 0; kk < k; ++kk) acc += (int32_t)xr[kk] * (int32_t)wr[kk];
      out[i * n + j] = acc;
    }
  }
  free(xv);
  free(wv);
  return QO_OK;
}

/* calibration.cpp:69-91 */
int qo_outlier_permutation(int64_t features, const int64_t* idx, int64_t n_idx, int64_t* perm) {
  char* is_out = (char*)calloc((size_t)features + 1, 1);
  for (int64_t i = 0; i < n_idx; ++i) {
    if (idx[i] < 0 || idx[i] >= features || (i > 0 && idx[i] <= idx[i - 1])) {
      free(is_out);
      return QO_INVALID_ARGUMENT;
    }
    is_out[idx[i]] = 1;
  }
  int64_t p = 0;
  for (int64_t f = 0; f < features; ++f)
    if (!is_out[f]) perm[p++] = f;
  for (int64_t i = 0; i < n_idx; ++i) perm[p++] = idx[i];
  free(is_out);
  return QO_OK;
}

static const float* g_sort_key;
static int cmp_desc_stable(const void* a, const void* b) {
  const int64_t ia = *(const int64_t*)a, ib = *(const int64_t*)b;
  const float ka = g_sort_key[ia], kb = g_sort_key[ib];
  if (ka > kb) return -1;
  if (ka < kb) return 1;
  return ia < ib ? -1 : (ia > ib ? 1 : 0); /* stable: lower index first */
}
static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* calibration.cpp:10-33 (max_abs, strict >) and :101-114 (stable_sort by
 * descending max-abs, first k, then OutlierSet::from_indices sorts ascending). */
int qo_select_outliers(const float* x, int64_t rows, int64_t features, int64_t k, int64_t* idx_out) {
  if (k < 0 || k > features) return QO_INVALID_ARGUMENT;
  float* max_abs = (float*)calloc((size_t)features + 1, sizeof(float));
  for (int64_t t = 0; t < rows; ++t)
    for (int64_t f = 0; f < features; ++f) {
      const float a = fabsf(x[t * features + f]);
      if (a > max_abs[f]) max_abs[f] = a;
    }
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * ((size_t)features + 1));
  for (int64_t f = 0; f < features; ++f) order[f] = f;
  g_sort_key = max_abs;
  qsort(order, (size_t)features, sizeof(int64_t), cmp_desc_stable);
  memcpy(idx_out, order, sizeof(int64_t) * (size_t)k);
  qsort(idx_out, (size_t)k, sizeof(int64_t), cmp_i64);
  free(order);
  free(max_abs);
  return QO_OK;
}

/* runtime.cpp:169-186 */
void qo_split_activations(const float* x, int64_t M, int64_t K, const int64_t* perm, int64_t kb,
                          const int64_t* idx, int64_t n_out, float* x_base, float* x_out) {
  for (int64_t t = 0; t < M; ++t) {
    const float* src = x + t * K;
    for (int64_t j = 0; j < kb; ++j) x_base[t * kb + j] = src[perm[j]];
    for (int64_t j = 0; j < n_out; ++j) x_out[t * n_out + j] = src[idx[j]];
  }
}

/* runtime.cpp:21-30 */
static void packed_store(uint8_t* row, int64_t c, int bits, int stored) {
  if (bits == 8) {
    row[c] = (uint8_t)(int8_t)stored;
    return;
  }
  const uint8_t biased = (uint8_t)(stored + 8);
  uint8_t* b = &row[c / 2];
  *b = (c % 2 == 0) ? (uint8_t)((*b & 0xF0) | biased) : (uint8_t)((*b & 0x0F) | (biased << 4));
}

/* runtime.cpp:36-66: min/max seeded by the first element, strict < / >, any
 * non-finite -> NumericalError; scale = range == 0 ? 1 : range / levels; codes
 * lround((v - vmin) / scale) - half_range clamped; idx == NULL means the row is
 * already base-only. */
static int quantize_token_row(const float* vals, const int64_t* idx, int64_t n, int bits, uint8_t* packed_row,
                              float* scale_out, float* zero_out) {
  const int levels = (1 << bits) - 1;
  const int half_range = 1 << (bits - 1);
  float vmin = 0.0f, vmax = 0.0f;
  int finite = 1;
  for (int64_t i = 0; i < n; ++i) {
    const float v = idx ? vals[idx[i]] : vals[i];
    finite = finite && isfinite(v);
    if (i == 0) {
      vmin = vmax = v;
    } else {
      if (v < vmin) vmin = v;
      if (v > vmax) vmax = v;
    }
  }
  if (!finite) return QO_NUMERICAL;
  const float range = vmax - vmin;
  const float scale = range == 0.0f ? 1.0f : range / (float)levels;
  for (int64_t i = 0; i < n; ++i) {
    const float v = idx ? vals[idx[i]] : vals[i];
    const long q = lroundf((v - vmin) / scale); /* ties away from zero */
    int stored = (int)q - half_range;
    if (stored < -half_range) stored = -half_range;
    if (stored > half_range - 1) stored = half_range - 1;
    packed_store(packed_row, i, bits, stored);
  }
  *scale_out = scale;
  *zero_out = vmin;
  return QO_OK;
}

/* runtime.cpp:188-197 */
int qo_quantize_activations(const float* x_base, int64_t M, int64_t K, int bits, uint8_t* packed, float* scale,
                            float* zero) {
  if (bits != 4 && bits != 8) return QO_INVALID_ARGUMENT;
  const int64_t rb = qo_row_bytes(K, bits);
  memset(packed, 0, (size_t)(M * rb));
  for (int64_t t = 0; t < M; ++t) {
    const int s = quantize_token_row(x_base + t * K, NULL, K, bits, packed + t * rb, &scale[t], &zero[t]);
    if (s) return s;
  }
  return QO_OK;
}

/* runtime.cpp:199-220 */
int qo_quantize_activations_fused(const float* x, int64_t M, int64_t K, const int64_t* perm, int64_t kb,
                                  const int64_t* idx, int64_t n_out, int bits, uint8_t* packed, float* scale,
                                  float* zero, float* x_out) {
  if (bits != 4 && bits != 8) return QO_INVALID_ARGUMENT;
  if (kb + n_out != K) return QO_INVALID_ARGUMENT;
  const int64_t rb = qo_row_bytes(kb, bits);
  memset(packed, 0, (size_t)(M * rb));
  for (int64_t t = 0; t < M; ++t) {
    const float* src = x + t * K;
    const int s = quantize_token_row(src, perm, kb, bits, packed + t * rb, &scale[t], &zero[t]);
    if (s) return s;
    if (x_out)
      for (int64_t j = 0; j < n_out; ++j) x_out[t * n_out + j] = src[idx[j]];
  }
  return QO_OK;
}

/* runtime.cpp:70-77 */
float qo_dequant_element(int32_t acc, float scale_act, float scale_w, float zero_act, float half_range,
                         float wreduced) {
  float v = (float)acc * scale_act;
  v *= scale_w;
  float shift = zero_act + half_range * scale_act;
  shift *= wreduced;
  return v + shift;
}

/* runtime.cpp:222-244 */
void qo_dequantize_epilogue(const int32_t* acc, int64_t M, int64_t N, const float* sa, const float* za,
                            int half_range, const float* sw, const float* wr, float* out) {
  const float hr = (float)half_range;
  for (int64_t t = 0; t < M; ++t)
    for (int64_t r = 0; r < N; ++r)
      out[t * N + r] = qo_dequant_element(acc[t * N + r], sa[t], sw[r], za[t], hr, wr[r]);
}

/* runtime.cpp:96-113 */
void qo_fp_linear(const float* x_out, int64_t M, int64_t O, const float* w_out, const float* bias, int64_t N,
                  float* out) {
#pragma omp parallel for schedule(static) if (M * N > 4096)
  for (int64_t t = 0; t < M; ++t) {
    const float* xr = x_out + t * O;
    for (int64_t r = 0; r < N; ++r) {
      float acc = bias ? bias[r] : 0.0f;
      const float* wrow = w_out + r * O;
      for (int64_t i = 0; i < O; ++i) acc += xr[i] * wrow[i];
      out[t * N + r] = acc;
    }
  }
}

/* runtime.cpp:246-318 (Quik mode). validate() runtime.cpp:150-167. */
int qo_quik_matmul(const qo_layer* L, const float* x, int64_t M, int variant, float* out) {
  if (L->bits != 4 && L->bits != 8) return QO_INVALID_ARGUMENT;
  if (L->act_bits != L->bits) return QO_INVALID_ARGUMENT;
  const int64_t K = L->in_features, N = L->out_features, O = L->n_outlier, kb = K - O;
  if (kb < 0) return QO_INVALID_ARGUMENT;
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * ((size_t)K + 1));
  if (qo_outlier_permutation(K, L->outlier_idx, O, perm)) {
    free(perm);
    return QO_INVALID_ARGUMENT;
  }
  const int64_t rb = qo_row_bytes(kb, L->bits);
  uint8_t* packed = (uint8_t*)malloc((size_t)(M * rb + 1));
  float* scale = (float*)malloc(sizeof(float) * ((size_t)M + 1));
  float* zero = (float*)malloc(sizeof(float) * ((size_t)M + 1));
  float* xo = (float*)malloc(sizeof(float) * ((size_t)(M * O) + 1));
  int st;
  if (variant == 0) {
    float* xb = (float*)malloc(sizeof(float) * ((size_t)(M * kb) + 1));
    qo_split_activations(x, M, K, perm, kb, L->outlier_idx, O, xb, xo);
    st = qo_quantize_activations(xb, M, kb, L->act_bits, packed, scale, zero);
    free(xb);
  } else {
    st = qo_quantize_activations_fused(x, M, K, perm, kb, L->outlier_idx, O, L->act_bits, packed, scale, zero, xo);
  }
  if (st == QO_OK) {
    int32_t* acc = (int32_t*)malloc(sizeof(int32_t) * ((size_t)(M * N) + 1));
    qo_int_matmul(packed, M, kb, L->act_bits, L->base, N, kb, L->bits, acc);
    qo_fp_linear(xo, M, O, L->outlier_weights, L->bias, N, out);
    const float hr = (float)(1 << (L->act_bits - 1));
    if (variant == 2) { /* runtime.cpp:288-303 */
      for (int64_t t = 0; t < M; ++t)
        for (int64_t r = 0; r < N; ++r)
          out[t * N + r] = out[t * N + r] +
                           qo_dequant_element(acc[t * N + r], scale[t], L->scales[r], zero[t], hr, L->wreduced[r]);
    } else { /* runtime.cpp:304-316 */
      float* deq = (float*)malloc(sizeof(float) * ((size_t)(M * N) + 1));
      qo_dequantize_epilogue(acc, M, N, scale, zero, 1 << (L->act_bits - 1), L->scales, L->wreduced, deq);
      for (int64_t i = 0; i < M * N; ++i) out[i] = out[i] + deq[i];
      free(deq);
    }
    free(acc);
  }
  free(perm);
  free(packed);
  free(scale);
  free(zero);
  free(xo);
  return st;
}

/* quantizer.cpp:17-22 */
static int8_t quantize_to_grid(double value, double inv_scale, int maxq) {
  const double t = value * inv_scale;
  double q = floor(fabs(t) + 0.5);
  if (q > maxq) q = maxq;
  return (int8_t)(t < 0.0 ? -q : q);
}

/* quantizer.cpp:339-371 with rtn_quantize_row (:251-264), clip factor 1. */
/* clip_search (quantizer.cpp:266-290): c in {0.50, 0.51, ..., 1.00} minimising the
 * sequential FP64 sum of squared round-trip errors; ties toward the larger c. */
static float clip_search(const float* w, const int64_t* perm, int64_t kb, int bits) {
  const int maxq = (1 << (bits - 1)) - 1;
  double amax = 0.0;
  for (int64_t j = 0; j < kb; ++j) {
    const double a = (double)fabsf(w[perm[j]]);
    if (a > amax) amax = a;
  }
  if (amax == 0.0) return 1.0f;
  double best_err = INFINITY;
  float best_c = 1.0f;
  for (int step = 0; step <= 50; ++step) {
    const float c = (float)(0.50 + 0.01 * step);
    const double scale = (double)c * amax / maxq;
    const double inv_scale = 1.0 / scale;
    double err = 0.0;
    for (int64_t j = 0; j < kb; ++j) {
      const float v = w[perm[j]];
      const double dq = (double)quantize_to_grid(v, inv_scale, maxq) * scale;
      const double d = (double)v - dq;
      err += d * d;
    }
    if (err <= best_err) {
      best_err = err;
      best_c = c;
    }
  }
  return best_c;
}

int qo_rtn_quantize_weights_clip(const float* w, int64_t N, int64_t K, const int64_t* idx, int64_t n_out, int bits,
                                 int use_clipping, uint8_t* base, float* scales, float* wreduced, float* outlier_w) {
  if (bits != 4 && bits != 8) return QO_INVALID_ARGUMENT;
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * ((size_t)K + 1));
  if (qo_outlier_permutation(K, idx, n_out, perm)) {
    free(perm);
    return QO_INVALID_ARGUMENT;
  }
  const int64_t kb = K - n_out;
  const int maxq = (1 << (bits - 1)) - 1;
  int8_t* q = (int8_t*)malloc((size_t)(N * kb) + 1);
  for (int64_t r = 0; r < N; ++r) {
    double amax = 0.0; /* row_amax, quantizer.cpp:24-28 */
    for (int64_t j = 0; j < kb; ++j) {
      const double a = (double)fabsf(w[r * K + perm[j]]);
      if (a > amax) amax = a;
    }
    /* rtn_quantize_weights :355: clip = use_clipping && n_base > 0 ? clip_search : 1 */
    const float clip = use_clipping && kb > 0 ? clip_search(w + r * K, perm, kb, bits) : 1.0f;
    float scale_f;
    int64_t qsum = 0;
    if (amax == 0.0) {
      for (int64_t j = 0; j < kb; ++j) q[r * kb + j] = 0;
      scale_f = 1.0f;
    } else {
      const double scale = (double)clip * amax / maxq; /* rtn_quantize_row, quantizer.cpp:258 */
      const double inv_scale = 1.0 / scale;
      for (int64_t j = 0; j < kb; ++j) {
        q[r * kb + j] = quantize_to_grid(w[r * K + perm[j]], inv_scale, maxq);
      }
      scale_f = (float)scale;
    }
    for (int64_t j = 0; j < kb; ++j) qsum += q[r * kb + j];
    scales[r] = scale_f;
    wreduced[r] = (float)((double)scale_f * (double)qsum);
    for (int64_t j = 0; j < n_out; ++j) outlier_w[r * n_out + j] = w[r * K + perm[kb + j]];
  }
  int st = qo_pack(q, N, kb, bits, base, NULL, NULL);
  free(q);
  free(perm);
  return st;
}

int qo_rtn_quantize_weights(const float* w, int64_t N, int64_t K, const int64_t* idx, int64_t n_out, int bits,
                            uint8_t* base, float* scales, float* wreduced, float* outlier_w) {
  return qo_rtn_quantize_weights_clip(w, N, K, idx, n_out, bits, 0, base, scales, wreduced, outlier_w);
}

/* dequantize_weights (quantizer.cpp:384-403): out[r][perm[j]] = (float)q * scale[r]
 * for base columns, the outlier weights in theirs. */
int qo_dequantize_weights(const uint8_t* base, int64_t N, int64_t K, const int64_t* idx, int64_t n_out, int bits,
                          const float* scales, const float* outlier_w, float* out) {
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * ((size_t)K + 1));
  if (qo_outlier_permutation(K, idx, n_out, perm)) {
    free(perm);
    return QO_INVALID_ARGUMENT;
  }
  const int64_t kb = K - n_out;
  int8_t* q = (int8_t*)malloc((size_t)(N * kb) + 1);
  qo_unpack(base, N, kb, bits, q);
  for (int64_t r = 0; r < N; ++r) {
    for (int64_t j = 0; j < kb; ++j) out[r * K + perm[j]] = (float)q[r * kb + j] * scales[r];
    for (int64_t j = 0; j < n_out; ++j) out[r * K + perm[kb + j]] = outlier_w[r * n_out + j];
  }
  free(q);
  free(perm);
  return 0;
}

/* quantizer.cpp:373-382 */
void qo_compute_wreduced(const uint8_t* base, int64_t N, int64_t kb, int bits, const float* scales, float* out) {
  int8_t* v = (int8_t*)malloc((size_t)(N * kb) + 1);
  qo_unpack(base, N, kb, bits, v);
  for (int64_t r = 0; r < N; ++r) {
    int64_t s = 0;
    for (int64_t j = 0; j < kb; ++j) s += v[r * kb + j];
    out[r] = (float)((double)scales[r] * (double)s);
  }
  free(v);
}

/* runtime.cpp:115-136 (LayerMode::WeightOnly). quik_matmul validates the layer first
 * (runtime.cpp:247, :150-167; act_bits need not match in this mode) and dispatches
 * here at :255: split_activations (:169-186), unpack_values of the base codes,
 * fp_linear (:96-113) for bias + outliers, then per output the sequential FP32 sum
 * acc += x_b[j] * (float(q[j]) * scale) added onto it. */
int qo_weight_only_forward(const qo_layer* L, const float* x, int64_t M, float* out) {
  if (L->bits != 4 && L->bits != 8) return QO_INVALID_ARGUMENT;
  const int64_t K = L->in_features, N = L->out_features, O = L->n_outlier, kb = K - O;
  if (kb < 0) return QO_INVALID_ARGUMENT;
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * ((size_t)K + 1));
  if (qo_outlier_permutation(K, L->outlier_idx, O, perm)) {
    free(perm);
    return QO_INVALID_ARGUMENT;
  }
  float* xb = (float*)malloc(sizeof(float) * ((size_t)(M * kb) + 1));
  float* xo = (float*)malloc(sizeof(float) * ((size_t)(M * O) + 1));
  int8_t* q = (int8_t*)malloc((size_t)(N * kb) + 1);
  qo_split_activations(x, M, K, perm, kb, L->outlier_idx, O, xb, xo);
  qo_unpack(L->base, N, kb, L->bits, q);
  qo_fp_linear(xo, M, O, L->outlier_weights, L->bias, N, out);
  for (int64_t t = 0; t < M; ++t) {
    const float* xr = xb + t * kb;
    for (int64_t r = 0; r < N; ++r) {
      const int8_t* qr = q + r * kb;
      const float scale = L->scales[r];
      float acc = 0.0f;
      for (int64_t j = 0; j < kb; ++j) acc += xr[j] * ((float)qr[j] * scale);
      out[t * N + r] += acc;
    }
  }
  free(q);
  free(xo);
  free(xb);
  free(perm);
  return QO_OK;
}
