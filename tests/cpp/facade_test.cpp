// C++ parity driver for the drop-in facade (include/quik_b200.hpp): the same
// calls as the reference's own tests (proj/tests/test_packed.cpp,
// test_runtime.cpp), against the plain-C oracle (oracle/quik_oracle.c) as the
// checker. Exit code = number of failed checks. Needs a B200.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include <cuda_fp16.h>

#include "quik_b200.hpp"

extern "C" {
#include "../../oracle/quik_oracle.h"
}

namespace Q = quik::b200;

static int g_fail = 0;
#define CHECK(cond)                                                       \
  do {                                                                    \
    if (!(cond)) {                                                        \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);         \
      ++g_fail;                                                           \
    }                                                                     \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static Q::FpMatrix rows(std::initializer_list<std::initializer_list<float>> init) {
  Q::FpMatrix m(static_cast<int64_t>(init.size()), static_cast<int64_t>(init.begin()->size()));
  size_t i = 0;
  for (auto& r : init)
    for (float v : r) m.data[i++] = v;
  return m;
}

int main(int argc, char** argv) {
  // test_packed.cpp:78-92 — int_matmul hand-computed 2x2, INT8 and INT4
  {
    const std::vector<int8_t> xv = {1, -2, 3, 4}, wv = {5, 6, -7, 8}, w4 = {5, 6, -7, 7};
    const auto out = Q::int_matmul(Q::pack_int8(xv, 2, 2), Q::pack_int8(wv, 2, 2));
    CHECK(out.at(0, 0) == -7 && out.at(0, 1) == -23 && out.at(1, 0) == 39 && out.at(1, 1) == 11);
    const auto out4 = Q::int_matmul(Q::pack_int4(xv, 2, 2), Q::pack_int4(w4, 2, 2));
    CHECK(out4.at(0, 0) == 1 * 5 + -2 * 6 && out4.at(1, 1) == 3 * -7 + 4 * 7);
    CHECK(throws<std::invalid_argument>([&] { Q::int_matmul(Q::pack_int4(xv, 2, 2), Q::pack_int8(wv, 2, 2)); }));
    CHECK(throws<std::out_of_range>([&] { Q::pack_int4(std::vector<int8_t>{0, 0, 8, 0}, 2, 2); }));
  }
  // test_packed.cpp:104-120 — int_matmul == naive on random shapes
  {
    std::mt19937 rng(7);
    std::uniform_int_distribution<int64_t> dim(1, 40);
    for (int trial = 0; trial < 50; ++trial) {
      const int bits = trial % 2 == 0 ? 4 : 8;
      const int lim = bits == 4 ? 7 : 127;
      std::uniform_int_distribution<int> val(-lim - 1, lim);
      const int64_t t = dim(rng), k = dim(rng), n = dim(rng);
      std::vector<int8_t> xv(t * k), wv(n * k);
      for (auto& v : xv) v = static_cast<int8_t>(val(rng));
      for (auto& v : wv) v = static_cast<int8_t>(val(rng));
      const auto x = Q::pack_values(xv, t, k, bits), w = Q::pack_values(wv, n, k, bits);
      const auto got = Q::int_matmul(x, w);
      std::vector<int32_t> want(t * n);
      qo_int_matmul(x.data.data(), t, k, bits, w.data.data(), n, k, bits, want.data());
      CHECK(got.data == want);
    }
  }
  // test_runtime.cpp:80-116 — quantizer known answers and errors
  {
    const auto r = Q::quantize_activations(rows({{0.0f, 0.5f, 1.0f, 1.5f}}), 4);
    CHECK(std::fabs(r.scale[0] - 0.1f) < 1e-7f && r.zero[0] == 0.0f && r.half_range == 8);
    CHECK((Q::unpack_values(r.packed) == std::vector<int8_t>{-8, -3, 2, 7}));
    const auto c = Q::quantize_activations(rows({{5.0f, 5.0f, 5.0f}}), 4);
    CHECK(c.scale[0] == 1.0f && c.zero[0] == 5.0f);
    auto bad = rows({{1.0f, 2.0f}});
    bad.at(0, 1) = NAN;
    CHECK(throws<Q::NumericalError>([&] { Q::quantize_activations(bad, 4); }));
  }
  // test_runtime.cpp:134-156 — fused quantizer == reference (oracle), bit-exact
  {
    for (uint32_t seed = 0; seed < 40; ++seed) {
      std::mt19937 local(seed);
      const int bits = seed % 2 == 0 ? 4 : 8;
      const int64_t in = 8 + static_cast<int64_t>(local() % 120);
      const int64_t tokens = 1 + static_cast<int64_t>(local() % 16);
      std::normal_distribution<float> dist(0.0f, 1.5f);
      Q::FpMatrix x(tokens, in);
      for (float& v : x.data) v = dist(local);
      const int64_t k = static_cast<int64_t>(local() % static_cast<uint64_t>(in));
      std::vector<int64_t> idx(k);
      qo_select_outliers(x.data.data(), tokens, in, k, idx.data());
      const auto o = Q::OutlierSet::from_indices(in, idx);
      const auto [fused, xo] = Q::quantize_activations_fused(x, o, bits);
      std::vector<uint8_t> pk(tokens * qo_row_bytes(in - k, bits) + 1);
      std::vector<float> sc(tokens), ze(tokens), xo_ref(tokens * k + 1);
      qo_quantize_activations_fused(x.data.data(), tokens, in, o.permutation.data(), in - k, o.indices.data(), k,
                                    bits, pk.data(), sc.data(), ze.data(), xo_ref.data());
      CHECK(std::memcmp(fused.packed.data.data(), pk.data(), fused.packed.data.size()) == 0);
      CHECK(std::memcmp(fused.scale.data(), sc.data(), tokens * 4) == 0);
      CHECK(std::memcmp(fused.zero.data(), ze.data(), tokens * 4) == 0);
      CHECK(std::memcmp(xo.data.data(), xo_ref.data(), xo.data.size() * 4) == 0);
    }
  }
  // test_runtime.cpp:172-186 — epilogue hand example
  {
    const auto aq = Q::quantize_activations(rows({{1.0f, 3.0f}}), 4);
    const auto acc = Q::int_matmul(aq.packed, Q::pack_int4(std::vector<int8_t>{2, -1}, 1, 2));
    CHECK(acc.at(0, 0) == -23);
    const std::vector<float> s = {0.5f}, wr = {0.5f};
    const auto out = Q::dequantize_epilogue(acc, aq, s, wr);
    CHECK(std::fabs(out.at(0, 0) + 0.5f) < 1e-6f);
  }
  // quik_matmul through the facade vs the reference algorithm (oracle):
  // bit-exact without outliers, and V1 == V2 == V3
  {
    std::mt19937 rng(131);
    std::normal_distribution<float> nd(0.0f, 1.0f);
    for (int trial = 0; trial < 6; ++trial) {
      const int bits = trial % 2 == 0 ? 4 : 8;
      const int64_t M = 5 + 11 * trial, K = 64 + 40 * trial, N = 24 + 30 * trial;
      const int64_t O = (trial % 3) * 8;
      Q::FpMatrix x(M, K), w(N, K);
      for (float& v : x.data) v = nd(rng);
      for (float& v : w.data) v = 0.5f * nd(rng);
      std::vector<int64_t> idx(O);
      qo_select_outliers(x.data.data(), M, K, O, idx.data());
      Q::QuikLinearLayer L;
      L.outliers = Q::OutlierSet::from_indices(K, idx);
      L.weights = Q::rtn_quantize_weights(w, L.outliers, bits);
      L.act_bits = bits;
      L.bias.assign(N, 0.25f);
      // weight-side parity: device RTN == reference RTN
      std::vector<uint8_t> base(N * qo_row_bytes(K - O, bits));
      std::vector<float> sc(N), wr(N), ow(N * O + 1);
      qo_rtn_quantize_weights(w.data.data(), N, K, idx.data(), O, bits, base.data(), sc.data(), wr.data(), ow.data());
      CHECK(L.weights.base.data == base);
      CHECK(std::memcmp(L.weights.scales.data(), sc.data(), N * 4) == 0);
      CHECK(std::memcmp(L.weights.wreduced.data(), wr.data(), N * 4) == 0);
      // x and outlier weights rounded to f16 so the device f16 outlier operands are exact
      for (float& v : x.data) v = __half2float(__float2half(v));
      for (float& v : L.weights.outlier_weights.data) v = __half2float(__float2half(v));
      const auto y1 = Q::quik_matmul(L, x, Q::PipelineVariant::V1Unfused);
      const auto y2 = Q::quik_matmul(L, x, Q::PipelineVariant::V2FusedQuant);
      const auto y3 = Q::quik_matmul(L, x);
      CHECK(y1.data == y2.data && y1.data == y3.data);
      qo_layer ql{K, N, O, bits, bits, L.weights.base.data.data(), L.weights.scales.data(), L.weights.wreduced.data(),
                  L.weights.outlier_weights.data.data(), L.outliers.indices.data(), L.bias.data()};
      std::vector<float> want(M * N);
      CHECK(qo_quik_matmul(&ql, x.data.data(), M, 2, want.data()) == QO_OK);
      if (O == 0) {
        CHECK(std::memcmp(y3.data.data(), want.data(), want.size() * 4) == 0);
      } else {
        double d2 = 0, r2 = 0;
        for (size_t i = 0; i < want.size(); ++i) {
          d2 += (double(y3.data[i]) - want[i]) * (double(y3.data[i]) - want[i]);
          r2 += double(want[i]) * want[i];
        }
        CHECK(std::sqrt(d2 / r2) < 1e-5);
      }
    }
  }
  // LayerMode::WeightOnly (test_runtime.cpp:284-300): FP32 activations, device result
  // vs the C restatement of weight_only_forward (itself pinned to the reference)
  {
    std::mt19937 rng(137);
    std::normal_distribution<float> nd(0.f, 1.f);
    for (int trial = 0; trial < 4; ++trial) {
      const int bits = trial % 2 == 0 ? 4 : 8;
      const int64_t M = 7 + 9 * trial, K = 64 + 96 * trial, N = 24 + 40 * trial, O = (trial % 2) * 8;
      Q::FpMatrix x(M, K), w(N, K);
      for (float& v : x.data) v = nd(rng);
      for (float& v : w.data) v = 0.5f * nd(rng);
      std::vector<int64_t> idx(O);
      qo_select_outliers(x.data.data(), M, K, O, idx.data());
      Q::QuikLinearLayer L;
      L.outliers = Q::OutlierSet::from_indices(K, idx);
      L.weights = Q::rtn_quantize_weights(w, L.outliers, bits);
      L.act_bits = bits == 4 ? 8 : 4;  // need not match the weights in this mode (runtime.cpp:163)
      L.bias.assign(N, -0.5f);
      L.mode = Q::LayerMode::WeightOnly;
      const auto y = Q::quik_matmul(L, x);
      qo_layer ql{K, N, O, bits, bits, L.weights.base.data.data(), L.weights.scales.data(), L.weights.wreduced.data(),
                  L.weights.outlier_weights.data.data(), L.outliers.indices.data(), L.bias.data()};
      std::vector<float> want(M * N);
      CHECK(qo_weight_only_forward(&ql, x.data.data(), M, want.data()) == QO_OK);
      double d2 = 0, r2 = 0;
      for (size_t i = 0; i < want.size(); ++i) {
        d2 += (double(y.data[i]) - want[i]) * (double(y.data[i]) - want[i]);
        r2 += double(want[i]) * want[i];
      }
      CHECK(std::sqrt(d2 / r2) < 1e-6);
    }
    Q::QuikLinearLayer R;
    R.outliers = Q::OutlierSet::from_indices(8, {});
    R.weights.base = Q::pack_int4(std::vector<int8_t>(16, 0), 2, 8);
    R.weights.scales = {1.f, 1.f};
    R.weights.wreduced = {0.f, 0.f};
    R.weights.outlier_weights = Q::FpMatrix(2, 0);
    R.mode = Q::LayerMode::FpReference;
    CHECK(throws<std::invalid_argument>([&] { Q::quik_matmul(R, Q::FpMatrix(1, 8)); }));
  }
  // GPTQ / SparseGPT on the device through the reference signatures (quantizer.hpp:18-90):
  // H = I means no compensation, so gptq_quantize equals RTN bit for bit; a calibrated
  // Hessian from build_hessian matches the host FP64 sum; sparsegpt_joint's mask keeps
  // exactly two of every full group of four (quantizer.cpp:299-337)
  {
    std::mt19937 rng(211);
    std::normal_distribution<float> nd(0.f, 1.f);
    const int64_t N = 24, K = 136, O = 8;
    Q::FpMatrix w(N, K), x(64, K);
    for (float& v : w.data) v = 0.5f * nd(rng);
    for (float& v : x.data) v = nd(rng);
    std::vector<int64_t> idx(O);
    qo_select_outliers(x.data.data(), 64, K, O, idx.data());
    const auto o = Q::OutlierSet::from_indices(K, idx);
    const auto g = Q::gptq_quantize(w, Q::Hessian::identity(K), o, 4);
    const auto rt = Q::rtn_quantize_weights(w, o, 4);
    CHECK(g.base.data == rt.base.data);
    CHECK(std::memcmp(g.scales.data(), rt.scales.data(), N * 4) == 0);
    const std::vector<Q::FpMatrix> batches = {x};
    const Q::Hessian h = Q::build_hessian(batches);
    double maxrel = 0;
    for (int64_t i = 0; i < K; ++i)
      for (int64_t j = 0; j < K; ++j) {
        double ref = 0;
        for (int64_t t = 0; t < 64; ++t) ref += double(x.data[t * K + i]) * double(x.data[t * K + j]);
        maxrel = std::max(maxrel, std::fabs(h.at(i, j) - ref) / (std::fabs(ref) + 1e-9));
      }
    CHECK(h.token_count == 64 && maxrel < 1e-12);
    double tr = 0;  // Hessian::lambda (quantizer.cpp:225-229)
    for (int64_t i = 0; i < K; ++i) tr += h.at(i, i);
    CHECK(h.lambda() == 0.01 * tr / static_cast<double>(K));
    const auto sp = Q::sparsegpt_joint(w, h, o, 4);
    bool groups_ok = sp.mask.rows == N && sp.mask.cols == K - O;
    for (int64_t r = 0; r < N && groups_ok; ++r)
      for (int64_t gi = 0; gi < (K - O) / 4; ++gi) {
        int kept = 0;
        for (int e = 0; e < 4; ++e) kept += sp.mask.kept_at(r, 4 * gi + e);
        groups_ok = groups_ok && kept == 2;
      }
    CHECK(groups_ok);
    CHECK(throws<std::invalid_argument>([&] { Q::gptq_quantize(w, Q::Hessian::identity(K + 1), o, 4); }));
  }
  // The rest of the reference surface on the device, against the oracle (quantizer.cpp /
  // runtime.cpp / packed.cpp): rtn_quantize_weights with use_clipping (clip_search),
  // compute_wreduced, dequantize_weights, split_activations, unpack_int4 / unpack_values,
  // per-stage StageTimes, forward_model(gated_mlp_ops)
  {
    std::mt19937 rng(99);
    std::normal_distribution<float> nd(0.f, 1.f);
    const int64_t N = 40, K = 300, O = 12, M = 7;
    Q::FpMatrix w(N, K), x(M, K);
    for (float& v : w.data) v = 0.5f * nd(rng);
    for (float& v : x.data) v = nd(rng);
    std::vector<int64_t> idx(O);
    qo_select_outliers(x.data.data(), M, K, O, idx.data());
    const auto o = Q::OutlierSet::from_indices(K, idx);
    for (int bits : {4, 8}) {
      const auto q = Q::rtn_quantize_weights(w, o, bits, true);
      std::vector<uint8_t> base(N * q.base.row_bytes());
      std::vector<float> sc(N), wr(N), ow(N * O);
      qo_rtn_quantize_weights_clip(w.data.data(), N, K, idx.data(), O, bits, 1, base.data(), sc.data(), wr.data(),
                                   ow.data());
      CHECK(q.base.data == base);
      CHECK(std::memcmp(q.scales.data(), sc.data(), N * 4) == 0 && std::memcmp(q.wreduced.data(), wr.data(), N * 4) == 0);
      const auto q0 = Q::rtn_quantize_weights(w, o, bits);
      CHECK(q0.scales != q.scales);  // clipping changes the scales
      const auto wred = Q::compute_wreduced(q);
      CHECK(std::memcmp(wred.data(), q.wreduced.data(), N * 4) == 0);
      const auto dq = Q::dequantize_weights(q, o);
      std::vector<float> want(N * K);
      qo_dequantize_weights(q.base.data.data(), N, K, idx.data(), O, bits, q.scales.data(),
                            q.outlier_weights.data.data(), want.data());
      CHECK(std::memcmp(dq.data.data(), want.data(), want.size() * 4) == 0);
      const auto vals = Q::unpack_values(q.base);
      std::vector<int8_t> wv(N * (K - O));
      qo_unpack(q.base.data.data(), N, K - O, bits, wv.data());
      CHECK(vals == wv);
      if (bits == 4) CHECK(Q::unpack_int4(q.base) == wv);
      else CHECK(throws<std::invalid_argument>([&] { Q::unpack_int4(q.base); }));
    }
    {
      const auto [xb, xo] = Q::split_activations(x, o);
      std::vector<float> wb(M * (K - O)), wo(M * O);
      qo_split_activations(x.data.data(), M, K, o.permutation.data(), K - O, idx.data(), O, wb.data(), wo.data());
      CHECK(xb.rows == M && xb.cols == K - O && xo.cols == O);
      CHECK(std::memcmp(xb.data.data(), wb.data(), wb.size() * 4) == 0 && std::memcmp(xo.data.data(), wo.data(), wo.size() * 4) == 0);
      CHECK(throws<std::invalid_argument>([&] { Q::split_activations(Q::FpMatrix(1, K + 1), o); }));
    }
    // StageTimes per stage: V3 reports K1 under quantize_ms and the fused GEMM under
    // int_matmul_ms; V1 fills split / quantize / int_matmul / fp_matmul
    {
      Q::QuikLinearLayer L;
      L.outliers = o;
      L.weights = Q::rtn_quantize_weights(w, o, 4);
      L.act_bits = 4;
      Q::StageTimes t3, t1;
      const auto y3 = Q::quik_matmul(L, x, Q::PipelineVariant::V3FusedEpilogue, &t3);
      const auto y1 = Q::quik_matmul(L, x, Q::PipelineVariant::V1Unfused, &t1);
      CHECK(t3.quantize_fused && t3.dequantize_fused && t3.quantize_ms > 0 && t3.int_matmul_ms > 0 &&
            t3.split_ms == 0 && t3.fp_matmul_ms == 0);
      CHECK(!t1.quantize_fused && t1.split_ms > 0 && t1.quantize_ms > 0 && t1.int_matmul_ms > 0 && t1.fp_matmul_ms > 0);
      CHECK(std::memcmp(y3.data.data(), y1.data.data(), y3.data.size() * 4) == 0);  // V1 == V3 bit for bit
    }
    // forward_model(gated_mlp_ops) on the device vs the oracle's layers + the
    // reference's elementwise ops (runtime.cpp:325-382)
    {
      const int64_t F = 64;
      Q::FpMatrix wu(F, K), wg(F, K), wd(K, F);
      for (float& v : wu.data) v = 0.05f * nd(rng);
      for (float& v : wg.data) v = 0.05f * nd(rng);
      for (float& v : wd.data) v = 0.5f * nd(rng);
      std::vector<Q::QuikLinearLayer> layers(3);
      layers[0].outliers = o;
      layers[0].weights = Q::rtn_quantize_weights(wu, o, 4);
      layers[1].outliers = o;
      layers[1].weights = Q::rtn_quantize_weights(wg, o, 4);
      const auto od = Q::OutlierSet::from_indices(F, {3, 17});
      layers[2].outliers = od;
      layers[2].weights = Q::rtn_quantize_weights(wd, od, 8);
      layers[2].act_bits = 8;
      const auto ops = Q::gated_mlp_ops();
      const auto tr = Q::forward_model_trace(layers, ops, x);
      CHECK(tr.size() == 6 && tr[5].rows == M && tr[5].cols == K);
      // values 1 / 2 exactly the single-layer forwards; 3 / 4 the reference's silu / multiply
      const auto u = Q::quik_matmul(layers[0], x), g = Q::quik_matmul(layers[1], x);
      CHECK(std::memcmp(tr[1].data.data(), u.data.data(), u.data.size() * 4) == 0);
      CHECK(std::memcmp(tr[2].data.data(), g.data.data(), g.data.size() * 4) == 0);
      double e3 = 0, e4 = 0;
      for (size_t i = 0; i < g.data.size(); ++i) {
        const float e = g.data[i];
        const float sil = e / (1.0f + std::exp(-e));
        e3 = std::max(e3, std::fabs(double(tr[3].data[i]) - sil) / (std::fabs(sil) + 1e-30));
        e4 = std::max(e4, std::fabs(double(tr[4].data[i]) - double(tr[3].data[i] * u.data[i])));
      }
      CHECK(e3 < 1e-6 && e4 == 0.0);
      const auto y = Q::forward_model(layers, ops, x);
      CHECK(std::memcmp(y.data.data(), tr[5].data.data(), y.data.size() * 4) == 0);
      const std::vector<Q::BlockOp> bad = {{Q::BlockOp::Kind::Silu, 7, -1, -1}};
      CHECK(throws<std::invalid_argument>([&] { Q::forward_model(layers, bad, x); }));
    }
  }
  // validation (runtime.cpp:150-167)
  {
    Q::QuikLinearLayer L;
    L.outliers = Q::OutlierSet::from_indices(8, {1, 2});
    L.weights.base = Q::pack_int4(std::vector<int8_t>(12, 0), 2, 6);
    L.weights.scales = {1.f, 1.f};
    L.weights.wreduced = {0.f, 0.f};
    L.weights.outlier_weights = Q::FpMatrix(2, 2);
    L.act_bits = 8;
    CHECK(throws<std::invalid_argument>([&] { Q::quik_matmul(L, Q::FpMatrix(1, 8)); }));
    L.act_bits = 4;
    CHECK(throws<std::invalid_argument>([&] { Q::quik_matmul(L, Q::FpMatrix(1, 9)); }));
  }
  // layer_io.cpp:32-74 through the bundle reader: reference bundles load with the same
  // fields, the sparse one keeps its mask; a missing bundle is a FormatError
  // (test_runtime.cpp:452-482). Bundles: tests/golden/bundle_* (reference save_layer).
  if (argc > 1) {
    const std::string root = argv[1];
    const Q::QuikLinearLayer d = Q::load_layer(root + "/bundle_f16_w4_o64");
    CHECK(d.in_features() == 512 && d.out_features() == 256 && d.outliers.outlier_count() == 64);
    CHECK(d.weights.bits() == 4 && d.act_bits == 4 && d.bias.size() == 256 && d.weights.mask.empty());
    const Q::QuikLinearLayer s = Q::load_layer(root + "/bundle_sp24_w4_o16");
    CHECK(!s.weights.mask.empty() && s.weights.mask.rows == 160 && s.weights.mask.cols == 240);
    Q::FpMatrix x(3, 256);
    for (int64_t i = 0; i < x.size(); ++i) x.data[static_cast<size_t>(i)] = static_cast<float>((i * 37) % 11) - 5.0f;
    const Q::FpMatrix y = Q::quik_matmul(s, x);  // sparse layer -> 2:4 GEMM
    CHECK(y.rows == 3 && y.cols == 160);
    CHECK(throws<Q::FormatError>([&] { Q::load_layer(root + "/missing"); }));
  }
  std::printf("facade_test: %d failure(s)\n", g_fail);
  return g_fail;
}
