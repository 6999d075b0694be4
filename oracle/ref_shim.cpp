// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper around the reference's own C++ implementation so the test
// suite (and bench.py's reference / cpu_baseline leg) can call it from Python.
// Compiled together with the UNMODIFIED reference sources
//   /root/reference/proj/src/{packed,calibration,quantizer,runtime}.cpp
// into oracle/_ref/libquik_ref.so by paper_2310_09259_b200/build.py
// (flags: the reference's Release flags, proj/CMakeLists.txt:11-13).
// Nothing here re-implements the algorithm; it only marshals plain arrays.
#include <chrono>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#include "quik/calibration.hpp"
#include "quik/packed.hpp"
#include "quik/quantizer.hpp"
#include "quik/runtime.hpp"
#include "quik/layer_io.hpp"

namespace {

int status_of(const std::exception_ptr& e) {
  try {
    std::rethrow_exception(e);
  } catch (const quik::NumericalError&) {
    return 3;
  } catch (const quik::FormatError&) {
    return 7;
  } catch (const std::out_of_range&) {
    return 2;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (...) {
    return 9;
  }
}

quik::FpMatrix to_fp(const float* p, int64_t r, int64_t c) {
  quik::FpMatrix m(r, c);
  if (r * c) std::memcpy(m.data.data(), p, sizeof(float) * r * c);
  return m;
}

quik::PackedIntMatrix to_packed(const uint8_t* p, int64_t r, int64_t c, int bits) {
  quik::PackedIntMatrix m;
  m.rows = r;
  m.cols = c;
  m.bits = bits;
  m.data.assign(p, p + r * m.row_bytes());
  return m;
}

struct Layer {
  quik::QuikLinearLayer layer;
};

quik::QuikLinearLayer make_layer(int64_t in, int64_t out, int bits, int act_bits, const uint8_t* base,
                                 const float* scales, const float* wreduced, const float* ow, const int64_t* idx,
                                 int64_t n_out, const float* bias) {
  quik::QuikLinearLayer L;
  L.outliers = quik::OutlierSet::from_indices(in, std::vector<int64_t>(idx, idx + n_out));
  L.weights.base = to_packed(base, out, in - n_out, bits);
  L.weights.scales.assign(scales, scales + out);
  L.weights.wreduced.assign(wreduced, wreduced + out);
  L.weights.outlier_weights = to_fp(ow, out, n_out);
  if (bias) L.bias.assign(bias, bias + out);
  L.act_bits = act_bits;
  return L;
}

}  // namespace

extern "C" {

int qr_pack(const int8_t* vals, int64_t rows, int64_t cols, int bits, uint8_t* out) {
  try {
    auto m = quik::pack_values(std::span<const int8_t>(vals, rows * cols), rows, cols, bits);
    std::memcpy(out, m.data.data(), m.data.size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int qr_unpack(const uint8_t* packed, int64_t rows, int64_t cols, int bits, int8_t* out) {
  try {
    auto v = quik::unpack_values(to_packed(packed, rows, cols, bits));
    std::memcpy(out, v.data(), v.size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int qr_int_matmul(const uint8_t* x, int64_t t, int64_t xk, int xbits, const uint8_t* w, int64_t n, int64_t wk,
                  int wbits, int32_t* out) {
  try {
    auto r = quik::int_matmul(to_packed(x, t, xk, xbits), to_packed(w, n, wk, wbits));
    std::memcpy(out, r.data.data(), r.data.size() * 4);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int qr_select_outliers(const float* x, int64_t rows, int64_t features, int64_t k, int64_t* idx_out) {
  try {
    quik::CalibStats s;
    s.accumulate(to_fp(x, rows, features));
    auto o = quik::select_outliers(s, k);
    std::memcpy(idx_out, o.indices.data(), o.indices.size() * 8);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int qr_outlier_permutation(int64_t features, const int64_t* idx, int64_t n_idx, int64_t* perm) {
  try {
    auto o = quik::OutlierSet::from_indices(features, std::vector<int64_t>(idx, idx + n_idx));
    std::memcpy(perm, o.permutation.data(), o.permutation.size() * 8);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int qr_quantize_activations(const float* xb, int64_t M, int64_t K, int bits, uint8_t* packed, float* scale,
                            float* zero) {
  try {
    auto r = quik::quantize_activations(to_fp(xb, M, K), bits);
    std::memcpy(packed, r.packed.data.data(), r.packed.data.size());
    std::memcpy(scale, r.scale.data(), M * 4);
    std::memcpy(zero, r.zero.data(), M * 4);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int qr_quantize_activations_fused(const float* x, int64_t M, int64_t K, const int64_t* idx, int64_t n_out,
                                  int bits, uint8_t* packed, float* scale, float* zero, float* x_out) {
  try {
    auto o = quik::OutlierSet::from_indices(K, std::vector<int64_t>(idx, idx + n_out));
    auto [r, xo] = quik::quantize_activations_fused(to_fp(x, M, K), o, bits);
    std::memcpy(packed, r.packed.data.data(), r.packed.data.size());
    std::memcpy(scale, r.scale.data(), M * 4);
    std::memcpy(zero, r.zero.data(), M * 4);
    if (x_out && !xo.data.empty()) std::memcpy(x_out, xo.data.data(), xo.data.size() * 4);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int qr_dequantize_epilogue(const int32_t* acc, int64_t M, int64_t N, const float* sa, const float* za,
                           int half_range, const float* sw, const float* wr, float* out) {
  try {
    quik::Int32Matrix a(M, N);
    std::memcpy(a.data.data(), acc, M * N * 4);
    quik::ActQuantResult q;
    q.scale.assign(sa, sa + M);
    q.zero.assign(za, za + M);
    q.half_range = half_range;
    auto r = quik::dequantize_epilogue(a, q, std::span<const float>(sw, N), std::span<const float>(wr, N));
    std::memcpy(out, r.data.data(), M * N * 4);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// quik_matmul with per-stage timings (StageTimes, runtime.hpp:72-80) in ms:
// times[0..5] = split, quantize, int_matmul, fp_matmul, dequantize, add.
int qr_quik_matmul(int64_t in, int64_t out_f, int bits, int act_bits, const uint8_t* base, const float* scales,
                   const float* wreduced, const float* ow, const int64_t* idx, int64_t n_out, const float* bias,
                   const float* x, int64_t M, int variant, float* out, double* times) {
  try {
    auto L = make_layer(in, out_f, bits, act_bits, base, scales, wreduced, ow, idx, n_out, bias);
    quik::StageTimes st;
    auto r = quik::quik_matmul(L, to_fp(x, M, in), static_cast<quik::PipelineVariant>(variant), &st);
    std::memcpy(out, r.data.data(), r.data.size() * 4);
    if (times) {
      times[0] = st.split_ms;
      times[1] = st.quantize_ms;
      times[2] = st.int_matmul_ms;
      times[3] = st.fp_matmul_ms;
      times[4] = st.dequantize_ms;
      times[5] = st.add_ms;
    }
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// LayerMode::WeightOnly through the reference's own quik_matmul (runtime.cpp:255).
int qr_weight_only(int64_t in, int64_t out_f, int bits, int act_bits, const uint8_t* base, const float* scales,
                   const float* wreduced, const float* ow, const int64_t* idx, int64_t n_out, const float* bias,
                   const float* x, int64_t M, float* out) {
  try {
    auto L = make_layer(in, out_f, bits, act_bits, base, scales, wreduced, ow, idx, n_out, bias);
    L.mode = quik::LayerMode::WeightOnly;
    auto r = quik::quik_matmul(L, to_fp(x, M, in));
    std::memcpy(out, r.data.data(), r.data.size() * 4);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// Persistent layer handle so timing loops exclude layer assembly.
void* qr_layer_create(int64_t in, int64_t out_f, int bits, int act_bits, const uint8_t* base, const float* scales,
                      const float* wreduced, const float* ow, const int64_t* idx, int64_t n_out, const float* bias) {
  try {
    auto* h = new Layer{make_layer(in, out_f, bits, act_bits, base, scales, wreduced, ow, idx, n_out, bias)};
    return h;
  } catch (...) {
    return nullptr;
  }
}
void qr_layer_destroy(void* h) { delete static_cast<Layer*>(h); }

int qr_layer_forward(void* h, const float* x, int64_t M, int variant, float* out, double* times) {
  try {
    auto& L = static_cast<Layer*>(h)->layer;
    quik::StageTimes st;
    auto r = quik::quik_matmul(L, to_fp(x, M, L.in_features()), static_cast<quik::PipelineVariant>(variant), &st);
    std::memcpy(out, r.data.data(), r.data.size() * 4);
    if (times) {
      times[0] = st.split_ms;
      times[1] = st.quantize_ms;
      times[2] = st.int_matmul_ms;
      times[3] = st.fp_matmul_ms;
      times[4] = st.dequantize_ms;
      times[5] = st.add_ms;
    }
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// forward_model_trace over gated_mlp_ops (runtime.cpp:325-388) with layer handles
// {up, gate, down}: out = down(silu(gate(x)) * up(x)) [M][down out]; h (optional) =
// the Hadamard product value v4 [M][up out].
int qr_gated_mlp(void* up, void* gate, void* down, const float* x, int64_t M, float* out, float* h) {
  try {
    std::vector<quik::QuikLinearLayer> layers = {static_cast<Layer*>(up)->layer, static_cast<Layer*>(gate)->layer,
                                                 static_cast<Layer*>(down)->layer};
    const auto ops = quik::gated_mlp_ops();
    auto vals = quik::forward_model_trace(layers, ops, to_fp(x, M, layers[0].in_features()));
    std::memcpy(out, vals.back().data.data(), vals.back().data.size() * 4);
    if (h) std::memcpy(h, vals[4].data.data(), vals[4].data.size() * 4);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int qr_rtn_quantize_weights(const float* w, int64_t N, int64_t K, const int64_t* idx, int64_t n_out, int bits,
                            uint8_t* base, float* scales, float* wreduced, float* outlier_w) {
  try {
    auto o = quik::OutlierSet::from_indices(K, std::vector<int64_t>(idx, idx + n_out));
    auto q = quik::rtn_quantize_weights(to_fp(w, N, K), o, bits);
    std::memcpy(base, q.base.data.data(), q.base.data.size());
    std::memcpy(scales, q.scales.data(), N * 4);
    std::memcpy(wreduced, q.wreduced.data(), N * 4);
    if (n_out) std::memcpy(outlier_w, q.outlier_weights.data.data(), N * n_out * 4);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int qr_rtn_quantize_weights_clip(const float* w, int64_t N, int64_t K, const int64_t* idx, int64_t n_out, int bits,
                                 int use_clipping, uint8_t* base, float* scales, float* wreduced, float* outlier_w) {
  try {
    auto o = quik::OutlierSet::from_indices(K, std::vector<int64_t>(idx, idx + n_out));
    auto q = quik::rtn_quantize_weights(to_fp(w, N, K), o, bits, use_clipping != 0);
    std::memcpy(base, q.base.data.data(), q.base.data.size());
    std::memcpy(scales, q.scales.data(), N * 4);
    std::memcpy(wreduced, q.wreduced.data(), N * 4);
    if (n_out) std::memcpy(outlier_w, q.outlier_weights.data.data(), N * n_out * 4);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// compute_wreduced / dequantize_weights of a layer in the reference's formats
int qr_compute_wreduced(const uint8_t* base, int64_t N, int64_t kb, int bits, const float* scales, float* out) {
  try {
    quik::QuantizedWeights q;
    q.base.rows = N;
    q.base.cols = kb;
    q.base.bits = bits;
    q.base.data.assign(base, base + N * q.base.row_bytes());
    q.scales.assign(scales, scales + N);
    const auto r = quik::compute_wreduced(q);
    std::memcpy(out, r.data(), N * 4);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int qr_dequantize_weights(const uint8_t* base, int64_t N, int64_t K, const int64_t* idx, int64_t n_out, int bits,
                          const float* scales, const float* outlier_w, float* out) {
  try {
    auto o = quik::OutlierSet::from_indices(K, std::vector<int64_t>(idx, idx + n_out));
    quik::QuantizedWeights q;
    q.base.rows = N;
    q.base.cols = K - n_out;
    q.base.bits = bits;
    q.base.data.assign(base, base + N * q.base.row_bytes());
    q.scales.assign(scales, scales + N);
    q.outlier_weights = to_fp(outlier_w, N, n_out);
    const auto r = quik::dequantize_weights(q, o);
    std::memcpy(out, r.data.data(), r.data.size() * 4);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// The reference tests' layer fixture, exactly (tests/test_runtime.cpp:27-45
// make_layer): W ~ N(0, .5), x ~ N(0, 1) from mt19937(seed), `heavy` random
// columns x100, outliers = select_outliers(x), RTN weights, bias ~ N(0, .1).
// Sizes are fixed by the arguments; outputs are caller-allocated.
int qr_make_test_layer(uint32_t seed, int64_t tokens, int64_t in, int64_t out, int bits, int64_t outliers,
                       int64_t heavy_cols, int with_bias, float* x, float* w, int64_t* idx, uint8_t* base,
                       float* scales, float* wreduced, float* outlier_w, float* bias) {
  try {
    std::mt19937 rng(seed);
    auto randm = [&](int64_t r, int64_t c, float sd) {
      std::normal_distribution<float> dist(0.0f, sd);
      quik::FpMatrix m(r, c);
      for (float& v : m.data) v = dist(rng);
      return m;
    };
    quik::FpMatrix W = randm(out, in, 0.5f);
    quik::FpMatrix X = randm(tokens, in, 1.0f);
    if (heavy_cols > 0) {
      std::uniform_int_distribution<int64_t> pick(0, in - 1);
      for (int64_t i = 0; i < heavy_cols; ++i) {
        const int64_t c = pick(rng);
        for (int64_t r = 0; r < tokens; ++r) X.at(r, c) *= 100.0f;
      }
    }
    quik::CalibStats stats;
    stats.accumulate(X);
    auto o = quik::select_outliers(stats, outliers);
    auto q = quik::rtn_quantize_weights(W, o, bits);
    std::memcpy(x, X.data.data(), X.data.size() * 4);
    std::memcpy(w, W.data.data(), W.data.size() * 4);
    if (outliers) std::memcpy(idx, o.indices.data(), o.indices.size() * 8);
    std::memcpy(base, q.base.data.data(), q.base.data.size());
    std::memcpy(scales, q.scales.data(), out * 4);
    std::memcpy(wreduced, q.wreduced.data(), out * 4);
    if (outliers) std::memcpy(outlier_w, q.outlier_weights.data.data(), out * outliers * 4);
    if (with_bias) {
      std::normal_distribution<float> dist(0.0f, 0.1f);
      for (int64_t r = 0; r < out; ++r) bias[r] = dist(rng);
    }
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// sparsegpt_joint (quantizer.cpp:299-337): joint 2:4 pruning + quantization, the
// producer of the sparse layers (cfg5). hsum: row-major K x K Hessian sum (FP64)
// over `tokens` calibration rows, or NULL for Hessian::identity(K). Outputs as
// qr_rtn_quantize_weights plus the mask [N][K - n_out] (1 = kept).
int qr_sparsegpt_joint(const float* w, int64_t N, int64_t K, const int64_t* idx, int64_t n_out, int bits,
                       const double* hsum, int64_t tokens, uint8_t* base, float* scales, float* wreduced,
                       float* outlier_w, uint8_t* mask) {
  try {
    auto o = quik::OutlierSet::from_indices(K, std::vector<int64_t>(idx, idx + n_out));
    quik::Hessian h = quik::Hessian::identity(K);
    if (hsum) {
      h.dim = K;
      h.token_count = tokens;
      h.sum.assign(hsum, hsum + K * K);
    }
    auto q = quik::sparsegpt_joint(to_fp(w, N, K), h, o, bits);
    std::memcpy(base, q.base.data.data(), q.base.data.size());
    std::memcpy(scales, q.scales.data(), N * 4);
    std::memcpy(wreduced, q.wreduced.data(), N * 4);
    if (n_out) std::memcpy(outlier_w, q.outlier_weights.data.data(), N * n_out * 4);
    std::memcpy(mask, q.mask.kept.data(), q.mask.kept.size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// gptq_quantize (quantizer.cpp:292-297) / sparsegpt_joint (:299-337) with an explicit
// Hessian sum (identity when hsum is NULL), damping fraction and clipping flag.
int qr_gptq(const float* w, int64_t N, int64_t K, const int64_t* idx, int64_t n_out, int bits, const double* hsum,
            int64_t tokens, double damping, int use_clipping, int sparse, uint8_t* base, float* scales,
            float* wreduced, float* outlier_w, uint8_t* mask) {
  try {
    auto o = quik::OutlierSet::from_indices(K, std::vector<int64_t>(idx, idx + n_out));
    quik::Hessian h = quik::Hessian::identity(K, damping);
    if (hsum) {
      h.token_count = tokens;
      h.sum.assign(hsum, hsum + K * K);
    }
    auto q = sparse ? quik::sparsegpt_joint(to_fp(w, N, K), h, o, bits, use_clipping != 0)
                    : quik::gptq_quantize(to_fp(w, N, K), h, o, bits, use_clipping != 0);
    std::memcpy(base, q.base.data.data(), q.base.data.size());
    std::memcpy(scales, q.scales.data(), N * 4);
    std::memcpy(wreduced, q.wreduced.data(), N * 4);
    if (n_out) std::memcpy(outlier_w, q.outlier_weights.data.data(), N * n_out * 4);
    if (sparse && mask) std::memcpy(mask, q.mask.kept.data(), q.mask.kept.size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// build_hessian (quantizer.cpp:225-240) over one batch x [T][K]: the FP64 sum.
int qr_build_hessian(const float* x, int64_t T, int64_t K, double* hsum) {
  try {
    std::vector<quik::FpMatrix> b{to_fp(x, T, K)};
    quik::Hessian h = quik::build_hessian(b);
    std::memcpy(hsum, h.sum.data(), K * K * 8);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// save_layer (layer_io.cpp:7-30): writes a layer bundle exactly as the reference does
// (the fixtures of the bundle-loader tests). mask: [N][K - n_out] or NULL; wfp32:
// reference weights [N][K] or NULL.
int qr_save_layer(const char* dir, int64_t in, int64_t out_f, int bits, int act_bits, const uint8_t* base,
                  const float* scales, const float* wreduced, const float* outlier_w, const int64_t* idx,
                  int64_t n_out, const float* bias, const uint8_t* mask, const float* wfp32) {
  try {
    quik::QuikLinearLayer L;
    L.outliers = quik::OutlierSet::from_indices(in, std::vector<int64_t>(idx, idx + n_out));
    const int64_t kb = in - n_out;
    L.weights.base.rows = out_f;
    L.weights.base.cols = kb;
    L.weights.base.bits = bits;
    L.weights.base.data.assign(base, base + out_f * (bits == 4 ? (kb + 1) / 2 : kb));
    L.weights.scales.assign(scales, scales + out_f);
    L.weights.wreduced.assign(wreduced, wreduced + out_f);
    L.weights.outlier_weights = quik::FpMatrix(out_f, n_out);
    if (n_out) std::memcpy(L.weights.outlier_weights.data.data(), outlier_w, out_f * n_out * 4);
    if (bias) L.bias.assign(bias, bias + out_f);
    if (mask) {
      L.weights.mask.rows = out_f;
      L.weights.mask.cols = kb;
      L.weights.mask.kept.assign(mask, mask + out_f * kb);
    }
    if (wfp32) {
      L.reference_weights = quik::FpMatrix(out_f, in);
      std::memcpy(L.reference_weights.data.data(), wfp32, out_f * in * 4);
    }
    L.act_bits = act_bits;
    quik::save_layer(L, dir);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// The reference tests' seeded Gaussian generator (tests/test_helpers.hpp:128-134):
// std::mt19937(seed) + std::normal_distribution<float>(0, stddev), row-major.
void qr_random_matrix(uint32_t seed, int64_t rows, int64_t cols, float stddev, float* out) {
  std::mt19937 rng(seed);
  std::normal_distribution<float> dist(0.0f, stddev);
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = dist(rng);
}

}  // extern "C"
