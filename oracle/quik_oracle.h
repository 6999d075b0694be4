/*
 * quik_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's CPU algorithm for the QUIK linear-layer
 * hot path (/root/reference/proj, C++20). Used exclusively as the checker by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg; the product
 * (paper_2310_09259_b200/) never links, imports or calls it.
 *
 * Parity is pinned two ways (see tests/test_oracle.py):
 *   1. against every known-answer test of the reference's own unit tests for this
 *      path (proj/tests/test_packed.cpp, test_runtime.cpp, test_quantizer.cpp);
 *   2. bit-for-bit against the reference sources themselves, compiled unchanged
 *      into oracle/_ref/libquik_ref.so (golden fixtures in tests/golden/).
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off (the reference's FP-contraction rule,
 * proj/CMakeLists.txt:11-13), no -ffast-math.
 */
#ifndef QUIK_ORACLE_H_
#define QUIK_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the reference's exception types */
enum { QO_OK = 0, QO_INVALID_ARGUMENT = 1, QO_OUT_OF_RANGE = 2, QO_NUMERICAL = 3 };

int64_t qo_row_bytes(int64_t cols, int bits);

/* packed.cpp:30-66. On a range error returns QO_OUT_OF_RANGE and the offending row/col. */
int qo_pack(const int8_t* vals, int64_t rows, int64_t cols, int bits, uint8_t* out, int64_t* bad_row,
            int64_t* bad_col);
/* packed.cpp:68-91 */
void qo_unpack(const uint8_t* packed, int64_t rows, int64_t cols, int bits, int8_t* out);
/* packed.cpp:93-132 — same argument checks, exact int32 accumulation. */
int qo_int_matmul(const uint8_t* x, int64_t t, int64_t xk, int xbits, const uint8_t* w, int64_t n, int64_t wk,
                  int wbits, int32_t* out);

/* calibration.cpp:69-91: permutation = non-outliers ascending then outliers. */
int qo_outlier_permutation(int64_t features, const int64_t* idx, int64_t n_idx, int64_t* perm);
/* calibration.cpp:10-33 (max-abs only) + :101-114 (stable descending sort, ties by index). */
int qo_select_outliers(const float* x, int64_t rows, int64_t features, int64_t k, int64_t* idx_out);

/* runtime.cpp:169-186 */
void qo_split_activations(const float* x, int64_t M, int64_t K, const int64_t* perm, int64_t kb,
                          const int64_t* idx, int64_t n_out, float* x_base, float* x_out);
/* runtime.cpp:188-197 (unfused, on a pre-split base matrix) */
int qo_quantize_activations(const float* x_base, int64_t M, int64_t K, int bits, uint8_t* packed, float* scale,
                            float* zero);
/* runtime.cpp:199-220 (fused split + quantize + outlier gather) */
int qo_quantize_activations_fused(const float* x, int64_t M, int64_t K, const int64_t* perm, int64_t kb,
                                  const int64_t* idx, int64_t n_out, int bits, uint8_t* packed, float* scale,
                                  float* zero, float* x_out);
/* runtime.cpp:70-77 */
float qo_dequant_element(int32_t acc, float scale_act, float scale_w, float zero_act, float half_range,
                         float wreduced);
/* runtime.cpp:222-244 */
void qo_dequantize_epilogue(const int32_t* acc, int64_t M, int64_t N, const float* sa, const float* za,
                            int half_range, const float* sw, const float* wr, float* out);
/* runtime.cpp:96-113: out[t][r] = bias[r] + sum_i x_o[t][i] * w_o[r][i], sequential FP32 */
void qo_fp_linear(const float* x_out, int64_t M, int64_t O, const float* w_out, const float* bias, int64_t N,
                  float* out);

/* The layer as the reference holds it (QuikLinearLayer, runtime.hpp:33-44). */
typedef struct qo_layer {
  int64_t in_features, out_features, n_outlier;
  int bits, act_bits;
  const uint8_t* base;          /* packed [out][row_bytes(K_b)] */
  const float* scales;          /* [out] */
  const float* wreduced;        /* [out] */
  const float* outlier_weights; /* [out][n_outlier] */
  const int64_t* outlier_idx;   /* [n_outlier] sorted */
  const float* bias;            /* [out] or NULL */
} qo_layer;

/* runtime.cpp:246-318, LayerMode::Quik; variant 0=V1, 1=V2, 2=V3. */
int qo_quik_matmul(const qo_layer* layer, const float* x, int64_t M, int variant, float* out);
/* runtime.cpp:115-136, LayerMode::WeightOnly: fp_linear(x_o, W_o, bias) then
 * out[t][r] += sum_j x_b[t][j] * ((float)q[r][j] * scale[r]), sequential FP32. */
int qo_weight_only_forward(const qo_layer* layer, const float* x, int64_t M, float* out);

/* quantizer.cpp:339-371 (+ :251-264, :17-22): RTN symmetric per-row, FP64 internals. */
int qo_rtn_quantize_weights(const float* w, int64_t N, int64_t K, const int64_t* idx, int64_t n_out, int bits,
                            uint8_t* base, float* scales, float* wreduced, float* outlier_w);
/* the same with use_clipping (clip_search, quantizer.cpp:266-290, :355) */
int qo_rtn_quantize_weights_clip(const float* w, int64_t N, int64_t K, const int64_t* idx, int64_t n_out, int bits,
                                 int use_clipping, uint8_t* base, float* scales, float* wreduced, float* outlier_w);
/* quantizer.cpp:384-403 */
int qo_dequantize_weights(const uint8_t* base, int64_t N, int64_t K, const int64_t* idx, int64_t n_out, int bits,
                          const float* scales, const float* outlier_w, float* out);
/* quantizer.cpp:373-382 */
void qo_compute_wreduced(const uint8_t* base, int64_t N, int64_t kb, int bits, const float* scales, float* out);

#ifdef __cplusplus
}
#endif
#endif
