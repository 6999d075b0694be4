// quik_b200.hpp — C++ facade with the reference's layer API, running on B200.
//
// Drop-in for the reference's namespace quik (proj/include/quik/{matrix,packed,
// calibration,quantizer,runtime}.hpp): the same type names, fields, function
// names, argument meaning and exception types, in namespace quik::b200. A caller
// switches with `namespace Q = quik::b200;` (or a using-declaration). Host data in,
// host data out, exactly like the reference; every number is computed by the
// sm_100a kernels behind the C ABI (quik_b200.h). For repeated forwards keep a
// DeviceLayer (weights uploaded and repacked once) instead of quik_matmul(layer, x).
//
// Header-only; link with -lquik_b200 -lcudart.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "quik_b200.h"

namespace quik::b200 {

// ---------------------------------------------------------------- errors (matrix.hpp:12-21)
class FormatError : public std::runtime_error {
 public:
  explicit FormatError(const std::string& m) : std::runtime_error(m) {}
};
class NumericalError : public std::runtime_error {
 public:
  explicit NumericalError(const std::string& m) : std::runtime_error(m) {}
};
class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

namespace detail {
inline void check(quik_status s) {
  if (s == QUIK_OK) return;
  const std::string m = quik_last_error();
  switch (s) {
    case QUIK_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case QUIK_ERR_OUT_OF_RANGE: throw std::out_of_range(m);
    case QUIK_ERR_NUMERICAL: throw NumericalError(m);
    case QUIK_ERR_FORMAT: throw FormatError(m);
    default: throw CudaError(m);
  }
}
inline void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
// Device buffer (RAII).
struct Buf {
  void* p = nullptr;
  explicit Buf(size_t n) { cuda(cudaMalloc(&p, n ? n : 1), "cudaMalloc"); }
  Buf(const void* host, size_t n) : Buf(n) {
    if (n) cuda(cudaMemcpy(p, host, n, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  }
  ~Buf() { cudaFree(p); }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  void get(void* host, size_t n) const {
    if (n) cuda(cudaMemcpy(host, p, n, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  }
};
// One context per host thread (scratch + error flag), on the current device.
inline quik_ctx_t ctx() {
  struct Holder {
    quik_ctx_t c = nullptr;
    ~Holder() { quik_ctx_destroy(c); }
  };
  thread_local Holder h;
  if (!h.c) {
    int dev = 0;
    cudaGetDevice(&dev);
    check(quik_ctx_create(dev, &h.c));
  }
  return h.c;
}
}  // namespace detail

// ---------------------------------------------------------------- value types (matrix.hpp:24-65)
struct FpMatrix {
  int64_t rows = 0, cols = 0;
  std::vector<float> data;
  FpMatrix() = default;
  FpMatrix(int64_t r, int64_t c) : rows(r), cols(c), data(static_cast<size_t>(r * c), 0.0f) {}
  float& at(int64_t r, int64_t c) { return data[static_cast<size_t>(r * cols + c)]; }
  float at(int64_t r, int64_t c) const { return data[static_cast<size_t>(r * cols + c)]; }
  const float* row(int64_t r) const { return data.data() + r * cols; }
  bool empty() const { return rows == 0 || cols == 0; }
  int64_t size() const { return rows * cols; }
};

struct Int32Matrix {
  int64_t rows = 0, cols = 0;
  std::vector<int32_t> data;
  Int32Matrix() = default;
  Int32Matrix(int64_t r, int64_t c) : rows(r), cols(c), data(static_cast<size_t>(r * c), 0) {}
  int32_t at(int64_t r, int64_t c) const { return data[static_cast<size_t>(r * cols + c)]; }
};

// packed.hpp:17-36 (i4p: low nibble = even column, stored = v + 8; bits 8 = two's complement)
struct PackedIntMatrix {
  int64_t rows = 0, cols = 0;
  int bits = 4;
  std::vector<uint8_t> data;
  int64_t row_bytes() const { return bits == 4 ? (cols + 1) / 2 : cols; }
  int get(int64_t r, int64_t c) const {
    if (bits == 8) return static_cast<int8_t>(data[static_cast<size_t>(r * cols + c)]);
    const uint8_t b = data[static_cast<size_t>(r * row_bytes() + c / 2)];
    return static_cast<int>((c % 2 == 0) ? (b & 0x0F) : (b >> 4)) - 8;
  }
  bool empty() const { return rows == 0 || cols == 0; }
};

// packed.cpp:30-66 (host-side format conversion; same range errors)
inline PackedIntMatrix pack_values(std::span<const int8_t> v, int64_t rows, int64_t cols, int bits) {
  if (bits != 4 && bits != 8) throw std::invalid_argument("pack_values: bits must be 4 or 8");
  if (static_cast<int64_t>(v.size()) != rows * cols)
    throw std::invalid_argument("pack: expected " + std::to_string(rows * cols) + " values, got " +
                                std::to_string(v.size()));
  PackedIntMatrix m;
  m.rows = rows;
  m.cols = cols;
  m.bits = bits;
  m.data.assign(static_cast<size_t>(rows * m.row_bytes()), 0);
  const int lo = bits == 4 ? -8 : -128, hi = bits == 4 ? 7 : 127;
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) {
      const int x = v[static_cast<size_t>(r * cols + c)];
      if (x < lo || x > hi)
        throw std::out_of_range("pack: value " + std::to_string(x) + " at row " + std::to_string(r) + ", col " +
                                std::to_string(c) + " outside [" + std::to_string(lo) + ", " + std::to_string(hi) +
                                "]");
      if (bits == 8) {
        m.data[static_cast<size_t>(r * cols + c)] = static_cast<uint8_t>(static_cast<int8_t>(x));
      } else {
        uint8_t& b = m.data[static_cast<size_t>(r * m.row_bytes() + c / 2)];
        const uint8_t s = static_cast<uint8_t>(x + 8);
        b = (c % 2 == 0) ? static_cast<uint8_t>((b & 0xF0) | s) : static_cast<uint8_t>((b & 0x0F) | (s << 4));
      }
    }
  return m;
}
inline PackedIntMatrix pack_int4(std::span<const int8_t> v, int64_t r, int64_t c) { return pack_values(v, r, c, 4); }
inline PackedIntMatrix pack_int8(std::span<const int8_t> v, int64_t r, int64_t c) { return pack_values(v, r, c, 8); }

// packed.cpp:86-91 (unpack_values) / :68-84 (unpack_int4), on the device
inline std::vector<int8_t> unpack_values(const PackedIntMatrix& m) {
  std::vector<int8_t> out(static_cast<size_t>(m.rows * m.cols));
  if (out.empty()) return out;
  detail::Buf dp(m.data.data(), m.data.size()), dout(out.size());
  detail::check(quik_unpack_values(detail::ctx(), static_cast<const uint8_t*>(dp.p), m.rows, m.cols, m.bits,
                                   static_cast<int8_t*>(dout.p), nullptr));
  detail::check(quik_ctx_sync(detail::ctx(), nullptr));
  dout.get(out.data(), out.size());
  return out;
}
inline std::vector<int8_t> unpack_int4(const PackedIntMatrix& m) {
  if (m.bits != 4) throw std::invalid_argument("unpack_int4: matrix is not 4-bit");
  return unpack_values(m);
}

// matrix.hpp:67-73
inline void check_same_shape(const FpMatrix& a, const FpMatrix& b, const char* what) {
  if (a.rows != b.rows || a.cols != b.cols)
    throw std::invalid_argument(std::string(what) + ": shape mismatch (" + std::to_string(a.rows) + "x" +
                                std::to_string(a.cols) + " vs " + std::to_string(b.rows) + "x" +
                                std::to_string(b.cols) + ")");
}

// calibration.hpp:37-48; from_indices calibration.cpp:69-91
struct OutlierSet {
  int64_t feature_count = 0;
  std::vector<int64_t> indices;
  std::vector<int64_t> permutation;
  static OutlierSet from_indices(int64_t feature_count, std::vector<int64_t> idx) {
    std::sort(idx.begin(), idx.end());
    for (size_t i = 0; i < idx.size(); ++i) {
      if (idx[i] < 0 || idx[i] >= feature_count)
        throw std::invalid_argument("OutlierSet: index " + std::to_string(idx[i]) + " outside feature range");
      if (i > 0 && idx[i] == idx[i - 1])
        throw std::invalid_argument("OutlierSet: duplicate index " + std::to_string(idx[i]));
    }
    OutlierSet o;
    o.feature_count = feature_count;
    o.indices = std::move(idx);
    std::vector<bool> is_out(static_cast<size_t>(feature_count), false);
    for (int64_t i : o.indices) is_out[static_cast<size_t>(i)] = true;
    for (int64_t f = 0; f < feature_count; ++f)
      if (!is_out[static_cast<size_t>(f)]) o.permutation.push_back(f);
    o.permutation.insert(o.permutation.end(), o.indices.begin(), o.indices.end());
    return o;
  }
  static OutlierSet none(int64_t feature_count) { return from_indices(feature_count, {}); }
  int64_t outlier_count() const { return static_cast<int64_t>(indices.size()); }
  int64_t base_count() const { return feature_count - outlier_count(); }
};

// quantizer.hpp:48-58
// quantizer.hpp:32-43: 2:4 structured mask over base weight positions
struct SparsityMask {
  int64_t rows = 0;
  int64_t cols = 0;
  std::vector<uint8_t> kept;
  bool empty() const { return kept.empty(); }
  bool kept_at(int64_t r, int64_t c) const { return kept[static_cast<size_t>(r * cols + c)] != 0; }
};

struct QuantizedWeights {
  PackedIntMatrix base;
  std::vector<float> scales;
  FpMatrix outlier_weights;
  std::vector<float> wreduced;
  SparsityMask mask;  // empty unless produced by sparsegpt_joint (-> 2:4 sparse GEMM)
  int bits() const { return base.bits; }
  int64_t out_features() const { return base.rows; }
  int64_t base_features() const { return base.cols; }
};

enum class PipelineVariant { V1Unfused, V2FusedQuant, V3FusedEpilogue };  // runtime.hpp:31

// runtime.hpp:25. Quik: the W4A4/W8A8 hot path; WeightOnly: activations stay FP
// (quik_linear_forward_weight_only); FpReference needs the original FP weights, which
// the device layer does not hold (std::invalid_argument, as the reference without them).
enum class LayerMode { Quik, WeightOnly, FpReference };

// runtime.hpp:33-44
struct QuikLinearLayer {
  QuantizedWeights weights;
  OutlierSet outliers;
  std::vector<float> bias;
  int act_bits = 4;
  LayerMode mode = LayerMode::Quik;
  int64_t in_features() const { return outliers.feature_count; }
  int64_t out_features() const { return weights.out_features(); }
  void validate() const {  // runtime.cpp:150-167
    if (outliers.outlier_count() != weights.outlier_weights.cols)
      throw std::invalid_argument("layer: outlier index count " + std::to_string(outliers.outlier_count()) +
                                  " != outlier weight columns " + std::to_string(weights.outlier_weights.cols));
    if (outliers.base_count() != weights.base_features())
      throw std::invalid_argument("layer: base column count mismatch");
    if (!bias.empty() && static_cast<int64_t>(bias.size()) != out_features())
      throw std::invalid_argument("layer: bias length != out_features");
    if (mode == LayerMode::Quik && act_bits != weights.bits())
      throw std::invalid_argument("layer: activation bits must match weight bits in quik mode");
    if (act_bits != 4 && act_bits != 8) throw std::invalid_argument("activation bits must be 4 or 8");
  }
};

// runtime.hpp:18-23
struct ActQuantResult {
  PackedIntMatrix packed;
  std::vector<float> scale;
  std::vector<float> zero;
  int half_range = 8;
};

inline float dequantize_activation(int q, float scale, float zero, int half_range) {  // runtime.hpp:60-62
  return (static_cast<float>(q) + static_cast<float>(half_range)) * scale + zero;
}

// runtime.hpp:72-80; filled from CUDA events around the device call
struct StageTimes {
  double split_ms = 0, quantize_ms = 0, int_matmul_ms = 0, fp_matmul_ms = 0, dequantize_ms = 0, add_ms = 0;
  bool quantize_fused = false, dequantize_fused = false;
  double total_ms() const { return split_ms + quantize_ms + int_matmul_ms + fp_matmul_ms + dequantize_ms + add_ms; }
};

// ---------------------------------------------------------------- device layer handle
class DeviceLayer {
 public:
  explicit DeviceLayer(const QuikLinearLayer& L, int64_t row_begin = 0, int64_t row_end = 0) {
    L.validate();
    if (L.mode == LayerMode::FpReference)
      throw std::invalid_argument("FpReference mode requires the original FP weights");
    mode_ = L.mode;
    quik_weights_desc d{};
    d.in_features = L.in_features();
    d.out_features = L.out_features();
    d.bits = L.weights.bits();
    d.act_bits = L.mode == LayerMode::WeightOnly ? L.weights.bits() : L.act_bits;  // unused in weight-only mode
    d.base = L.weights.base.data.data();
    d.scales = L.weights.scales.data();
    d.wreduced = L.weights.wreduced.data();
    d.outlier_weights = L.weights.outlier_weights.data.data();
    d.outlier_indices = L.outliers.indices.data();
    d.n_outlier = L.outliers.outlier_count();
    d.bias = L.bias.empty() ? nullptr : L.bias.data();
    d.row_begin = row_begin;
    d.row_end = row_end;
    d.sparsity = L.weights.mask.empty() ? 0 : 1;
    detail::check(quik_layer_create(detail::ctx(), &d, &h_));
    int64_t in = 0, out = 0;
    quik_layer_info(h_, &in, &out, nullptr, nullptr);
    in_ = in;
    out_ = out;
  }
  ~DeviceLayer() { quik_layer_destroy(h_); }
  DeviceLayer(const DeviceLayer&) = delete;
  DeviceLayer& operator=(const DeviceLayer&) = delete;
  quik_layer_t handle() const { return h_; }
  int64_t in_features() const { return in_; }
  int64_t out_features() const { return out_; }

  // Host FP32 in, host FP32 out (reference semantics), copies included.
  FpMatrix forward(const FpMatrix& x, PipelineVariant v = PipelineVariant::V3FusedEpilogue,
                   StageTimes* times = nullptr) const {
    if (x.cols != in_)
      throw std::invalid_argument("quik_matmul: input has " + std::to_string(x.cols) + " features, layer expects " +
                                  std::to_string(in_));
    FpMatrix y(x.rows, out_);
    if (x.rows == 0 || out_ == 0) return y;
    if (mode_ == LayerMode::WeightOnly) {  // runtime.cpp:255 -> weight_only_forward
      detail::Buf dx(x.data.data(), x.data.size() * 4), dy(y.data.size() * 4);
      detail::check(quik_linear_forward_weight_only(detail::ctx(), h_, dx.p, QUIK_F32, x.rows, dy.p, QUIK_F32, out_,
                                                    nullptr));
      detail::check(quik_ctx_sync(detail::ctx(), nullptr));
      dy.get(y.data.data(), y.data.size() * 4);
      return y;
    }
    if (v == PipelineVariant::V3FusedEpilogue && !times) {
      // host buffers straight through the chunked copy/compute pipeline
      detail::check(quik_linear_forward_host(detail::ctx(), h_, x.data.data(), QUIK_F32, x.rows, y.data.data(),
                                             QUIK_F32, 0, nullptr));
      detail::check(quik_ctx_sync(detail::ctx(), nullptr));
      return y;
    }
    detail::Buf dx(x.data.data(), x.data.size() * 4), dy(y.data.size() * 4);
    if (times) {
      // per-stage CUDA-event times (runtime.cpp:265-315 convention; see quik_linear_forward_timed)
      double ms[6] = {0, 0, 0, 0, 0, 0};
      int fused[2] = {0, 0};
      detail::check(quik_linear_forward_timed(detail::ctx(), h_, dx.p, QUIK_F32, x.rows, dy.p, QUIK_F32, out_,
                                              static_cast<quik_variant>(v), nullptr, ms, fused));
      times->split_ms = ms[0];
      times->quantize_ms = ms[1];
      times->int_matmul_ms = ms[2];
      times->fp_matmul_ms = ms[3];
      times->dequantize_ms = ms[4];
      times->add_ms = ms[5];
      times->quantize_fused = fused[0] != 0;
      times->dequantize_fused = fused[1] != 0;
    } else {
      detail::check(quik_linear_forward(detail::ctx(), h_, dx.p, QUIK_F32, x.rows, dy.p, QUIK_F32,
                                        static_cast<quik_variant>(v), nullptr));
    }
    detail::check(quik_ctx_sync(detail::ctx(), nullptr));
    dy.get(y.data.data(), y.data.size() * 4);
    return y;
  }

  // Device-resident forward: x / y device pointers, asynchronous on `stream`.
  void forward_device(const void* x, quik_dtype xdt, int64_t M, void* y, quik_dtype ydt, void* stream = nullptr,
                      PipelineVariant v = PipelineVariant::V3FusedEpilogue) const {
    detail::check(quik_linear_forward(detail::ctx(), h_, x, xdt, M, y, ydt, static_cast<quik_variant>(v), stream));
  }

  // Output-feature shard: this layer's f16 output columns go to column `col_offset` of
  // every destination (own y first, then peers' mapped outputs), the all-gather fused
  // into the GEMM epilogue (quik_linear_forward_sharded).
  void forward_sharded(const void* x, quik_dtype xdt, int64_t M, void* const* dsts, int n_dst, int64_t ldy,
                       int64_t col_offset, void* stream = nullptr) const {
    detail::check(quik_linear_forward_sharded(detail::ctx(), h_, x, xdt, M, dsts, n_dst, ldy, col_offset, stream));
  }

 private:
  quik_layer_t h_ = nullptr;
  int64_t in_ = 0, out_ = 0;
  LayerMode mode_ = LayerMode::Quik;
};

// ---------------------------------------------------------------- multi-GPU

// Contiguous, balanced output-row range of `rank` (the first n % world ranks get one more).
inline std::pair<int64_t, int64_t> shard_bounds(int64_t n, int world, int rank) {
  if (world <= 0 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank / world size");
  const int64_t base = n / world, extra = n % world;
  const int64_t b = rank * base + std::min<int64_t>(rank, extra);
  return {b, b + base + (rank < extra ? 1 : 0)};
}

// One process per GPU: this rank's output-feature shard of a QUIK layer with the
// all-gather fused into the GEMM epilogue. The [M][N] f16 outputs of every rank are
// mapped into every process through CUDA IPC (quik_ipc_handle_*); `exchange` is the
// caller's all-gather of byte blobs (MPI_Allgather, sockets, ...), used once at
// construction. Two output buffers alternate; after forward() the caller fences the
// ranks on `stream` (e.g. a one-element ncclAllReduce) before reading the result, which
// also orders readers of the buffer two steps back before its next writes.
class FusedShardedLayer {
 public:
  using Exchange = std::function<std::vector<std::vector<uint8_t>>(const std::vector<uint8_t>&)>;

  FusedShardedLayer(const QuikLinearLayer& full, int rank, int world, int64_t max_tokens, const Exchange& exchange)
      : rank_(rank), world_(world), n_(full.out_features()), max_tokens_(max_tokens) {
    const auto [b, e] = shard_bounds(n_, world, rank);
    begin_ = b;
    local_ = std::make_unique<DeviceLayer>(full, b, e);
    std::vector<uint8_t> mine;
    for (int i = 0; i < 2; ++i) {
      detail::cuda(cudaMalloc(&bufs_[i], static_cast<size_t>(max_tokens * n_ * 2)), "cudaMalloc");
      quik_ipc_handle h{};
      detail::check(quik_ipc_handle_get(detail::ctx(), bufs_[i], &h));
      const auto* p = reinterpret_cast<const uint8_t*>(&h);
      mine.insert(mine.end(), p, p + sizeof(h));
    }
    const std::vector<std::vector<uint8_t>> all = exchange(mine);
    if (static_cast<int>(all.size()) != world) throw std::invalid_argument("fused all-gather: exchange size != world");
    for (int i = 0; i < 2; ++i) {
      dst_[i].push_back(bufs_[i]);
      for (int r = 0; r < world; ++r) {
        if (r == rank) continue;
        if (all[r].size() != 2 * sizeof(quik_ipc_handle)) throw std::invalid_argument("fused all-gather: bad handle");
        quik_ipc_handle h{};
        std::memcpy(&h, all[r].data() + i * sizeof(h), sizeof(h));
        void* p = nullptr;
        detail::check(quik_ipc_handle_open(detail::ctx(), &h, &p));
        dst_[i].push_back(p);
        opened_.push_back({p, h});
      }
    }
  }
  ~FusedShardedLayer() {
    for (auto& [p, h] : opened_) quik_ipc_handle_close(detail::ctx(), p, &h);
    for (void* b : bufs_) cudaFree(b);
  }
  FusedShardedLayer(const FusedShardedLayer&) = delete;
  FusedShardedLayer& operator=(const FusedShardedLayer&) = delete;

  // x: device [M][in] (f16 or f32); returns this rank's copy of the full [M][N] f16 output.
  const void* forward(const void* x, quik_dtype xdt, int64_t M, void* stream = nullptr) {
    if (M > max_tokens_) throw std::invalid_argument("fused all-gather: more tokens than max_tokens");
    const int i = step_++ & 1;
    local_->forward_sharded(x, xdt, M, dst_[i].data(), world_, n_, begin_, stream);
    return bufs_[i];
  }
  int64_t out_features() const { return n_; }

 private:
  int rank_, world_;
  int64_t n_, max_tokens_, begin_ = 0;
  int step_ = 0;
  std::unique_ptr<DeviceLayer> local_;
  void* bufs_[2] = {nullptr, nullptr};
  std::vector<void*> dst_[2];
  std::vector<std::pair<void*, quik_ipc_handle>> opened_;
};

// ---------------------------------------------------------------- reference functions

// layer_io.hpp / layer_io.cpp:32-74: reference layer bundle -> host layer (FormatError
// on every reference failure mode; parsed by the C ABI bundle reader)
inline QuikLinearLayer load_layer(const std::string& dir) {
  quik_bundle_t b = nullptr;
  detail::check(quik_bundle_open(dir.c_str(), &b));
  struct Close {
    quik_bundle_t b;
    ~Close() { quik_bundle_close(b); }
  } close{b};
  quik_weights_desc d{};
  detail::check(quik_bundle_weights(b, &d));
  QuikLinearLayer L;
  L.act_bits = d.act_bits;
  L.outliers = OutlierSet::from_indices(d.in_features,
                                        std::vector<int64_t>(d.outlier_indices, d.outlier_indices + d.n_outlier));
  const int64_t kb = d.in_features - d.n_outlier;
  L.weights.base.rows = d.out_features;
  L.weights.base.cols = kb;
  L.weights.base.bits = d.bits;
  L.weights.base.data.assign(d.base, d.base + d.out_features * L.weights.base.row_bytes());
  L.weights.scales.assign(d.scales, d.scales + d.out_features);
  L.weights.wreduced.assign(d.wreduced, d.wreduced + d.out_features);
  L.weights.outlier_weights = FpMatrix(d.out_features, d.n_outlier);
  if (d.n_outlier)
    std::memcpy(L.weights.outlier_weights.data.data(), d.outlier_weights, d.out_features * d.n_outlier * 4);
  if (d.bias) L.bias.assign(d.bias, d.bias + d.out_features);
  if (d.sparsity) {
    const void* m = nullptr;
    int dt = 0, nd = 0;
    int64_t shape[4] = {0, 0, 0, 0};
    detail::check(quik_bundle_tensor(b, "sparsity_mask", &m, &dt, shape, &nd));
    L.weights.mask.rows = shape[0];
    L.weights.mask.cols = shape[1];
    L.weights.mask.kept.assign(static_cast<const uint8_t*>(m),
                               static_cast<const uint8_t*>(m) + shape[0] * shape[1]);
  }
  return L;
}

// runtime.hpp:85-87 (uploads the layer per call, like the reference re-reads its weights)
inline FpMatrix quik_matmul(const QuikLinearLayer& layer, const FpMatrix& x,
                            PipelineVariant v = PipelineVariant::V3FusedEpilogue, StageTimes* times = nullptr) {
  layer.validate();
  if (x.cols != layer.in_features())
    throw std::invalid_argument("quik_matmul: input has " + std::to_string(x.cols) + " features, layer expects " +
                                std::to_string(layer.in_features()));
  return DeviceLayer(layer).forward(x, v, times);
}

// runtime.hpp:55-56
inline std::pair<ActQuantResult, FpMatrix> quantize_activations_fused(const FpMatrix& x, const OutlierSet& o,
                                                                      int bits) {
  if (bits != 4 && bits != 8) throw std::invalid_argument("activation bits must be 4 or 8");
  if (x.cols != o.feature_count)
    throw std::invalid_argument("fused quantization: input features do not match outlier set");
  QuikLinearLayer carrier;  // permutation tables only (no weight rows)
  carrier.outliers = o;
  carrier.act_bits = bits;
  carrier.weights.base.rows = 0;
  carrier.weights.base.cols = o.base_count();
  carrier.weights.base.bits = bits;
  carrier.weights.outlier_weights = FpMatrix(0, o.outlier_count());
  DeviceLayer L(carrier);
  ActQuantResult r;
  r.packed.rows = x.rows;
  r.packed.cols = o.base_count();
  r.packed.bits = bits;
  r.packed.data.resize(static_cast<size_t>(x.rows * r.packed.row_bytes()));
  r.scale.resize(static_cast<size_t>(x.rows));
  r.zero.resize(static_cast<size_t>(x.rows));
  r.half_range = 1 << (bits - 1);
  FpMatrix xo(x.rows, o.outlier_count());
  if (x.rows == 0) return {std::move(r), std::move(xo)};
  detail::Buf dx(x.data.data(), x.data.size() * 4), dp(r.packed.data.size()), ds(x.rows * 4), dz(x.rows * 4),
      dxo(xo.data.size() * 4);
  detail::check(quik_quantize_activations_fused(detail::ctx(), L.handle(), dx.p, QUIK_F32, x.rows,
                                                static_cast<uint8_t*>(dp.p), static_cast<float*>(ds.p),
                                                static_cast<float*>(dz.p), static_cast<float*>(dxo.p), nullptr));
  detail::check(quik_ctx_sync(detail::ctx(), nullptr));
  dp.get(r.packed.data.data(), r.packed.data.size());
  ds.get(r.scale.data(), x.rows * 4);
  dz.get(r.zero.data(), x.rows * 4);
  dxo.get(xo.data.data(), xo.data.size() * 4);
  return {std::move(r), std::move(xo)};
}

// runtime.hpp:51
inline ActQuantResult quantize_activations(const FpMatrix& x_base, int bits) {
  if (bits != 4 && bits != 8) throw std::invalid_argument("activation bits must be 4 or 8");
  ActQuantResult r;
  r.packed.rows = x_base.rows;
  r.packed.cols = x_base.cols;
  r.packed.bits = bits;
  r.packed.data.resize(static_cast<size_t>(x_base.rows * r.packed.row_bytes()));
  r.scale.resize(static_cast<size_t>(x_base.rows));
  r.zero.resize(static_cast<size_t>(x_base.rows));
  r.half_range = 1 << (bits - 1);
  if (x_base.rows == 0) return r;
  detail::Buf dx(x_base.data.data(), x_base.data.size() * 4), dp(r.packed.data.size()), ds(x_base.rows * 4),
      dz(x_base.rows * 4);
  detail::check(quik_quantize_activations(detail::ctx(), dx.p, QUIK_F32, x_base.rows, x_base.cols, bits,
                                          static_cast<uint8_t*>(dp.p), static_cast<float*>(ds.p),
                                          static_cast<float*>(dz.p), nullptr));
  detail::check(quik_ctx_sync(detail::ctx(), nullptr));
  dp.get(r.packed.data.data(), r.packed.data.size());
  ds.get(r.scale.data(), x_base.rows * 4);
  dz.get(r.zero.data(), x_base.rows * 4);
  return r;
}

// packed.hpp:58
inline Int32Matrix int_matmul(const PackedIntMatrix& x, const PackedIntMatrix& w) {
  Int32Matrix out(x.rows, w.rows);
  detail::Buf dx(x.data.data(), x.data.size()), dw(w.data.data(), w.data.size()), dout(out.data.size() * 4);
  detail::check(quik_int_matmul(detail::ctx(), static_cast<const uint8_t*>(dx.p), x.rows, x.cols, x.bits,
                                static_cast<const uint8_t*>(dw.p), w.rows, w.cols, w.bits,
                                static_cast<int32_t*>(dout.p), nullptr));
  detail::check(quik_ctx_sync(detail::ctx(), nullptr));
  dout.get(out.data.data(), out.data.size() * 4);
  return out;
}

// runtime.hpp:66-68
inline FpMatrix dequantize_epilogue(const Int32Matrix& acc, const ActQuantResult& a,
                                   std::span<const float> weight_scales, std::span<const float> wreduced) {
  if (acc.rows != static_cast<int64_t>(a.scale.size()))
    throw std::invalid_argument("dequantize_epilogue: token count mismatch");
  if (static_cast<int64_t>(weight_scales.size()) != acc.cols || static_cast<int64_t>(wreduced.size()) != acc.cols)
    throw std::invalid_argument("dequantize_epilogue: per-row vector length mismatch");
  FpMatrix out(acc.rows, acc.cols);
  if (acc.rows == 0 || acc.cols == 0) return out;
  detail::Buf da(acc.data.data(), acc.data.size() * 4), ds(a.scale.data(), a.scale.size() * 4),
      dz(a.zero.data(), a.zero.size() * 4), dsw(weight_scales.data(), weight_scales.size() * 4),
      dwr(wreduced.data(), wreduced.size() * 4), dout(out.data.size() * 4);
  detail::check(quik_dequantize_epilogue(detail::ctx(), static_cast<const int32_t*>(da.p), acc.rows, acc.cols,
                                         static_cast<const float*>(ds.p), static_cast<const float*>(dz.p),
                                         a.half_range, static_cast<const float*>(dsw.p),
                                         static_cast<const float*>(dwr.p), static_cast<float*>(dout.p), nullptr));
  detail::check(quik_ctx_sync(detail::ctx(), nullptr));
  dout.get(out.data.data(), out.data.size() * 4);
  return out;
}

// quantizer.hpp:89-90, on the device, bit-exact (incl. clip_search with use_clipping)
inline QuantizedWeights rtn_quantize_weights(const FpMatrix& w, const OutlierSet& o, int bits,
                                             bool use_clipping = false) {
  if (o.feature_count != w.cols)
    throw std::invalid_argument("outlier set covers " + std::to_string(o.feature_count) + " features, weights have " +
                                std::to_string(w.cols));
  QuantizedWeights q;
  q.base.rows = w.rows;
  q.base.cols = o.base_count();
  q.base.bits = bits;
  q.base.data.resize(static_cast<size_t>(w.rows * q.base.row_bytes()));
  q.scales.resize(static_cast<size_t>(w.rows));
  q.wreduced.resize(static_cast<size_t>(w.rows));
  q.outlier_weights = FpMatrix(w.rows, o.outlier_count());
  if (w.rows == 0) return q;
  detail::Buf dw(w.data.data(), w.data.size() * 4), db(q.base.data.size()), ds(w.rows * 4), dr(w.rows * 4),
      dow(q.outlier_weights.data.size() * 4);
  detail::check(quik_rtn_quantize_weights(detail::ctx(), static_cast<const float*>(dw.p), w.rows, w.cols,
                                          o.indices.data(), o.outlier_count(), bits, use_clipping ? 1 : 0,
                                          static_cast<uint8_t*>(db.p),
                                          static_cast<float*>(ds.p), static_cast<float*>(dr.p),
                                          static_cast<float*>(dow.p), nullptr));
  detail::check(quik_ctx_sync(detail::ctx(), nullptr));
  db.get(q.base.data.data(), q.base.data.size());
  ds.get(q.scales.data(), w.rows * 4);
  dr.get(q.wreduced.data(), w.rows * 4);
  dow.get(q.outlier_weights.data.data(), q.outlier_weights.data.size() * 4);
  return q;
}

// quantizer.hpp:18-31: the calibration statistic H = sum x x^T (FP64), accumulated on
// the device (quik_hessian_accumulate), kept on the host like the reference's.
struct Hessian {
  int64_t dim = 0;
  int64_t token_count = 0;
  std::vector<double> sum;  // row-major dim x dim, before damping
  double damping_frac = 0.01;

  void accumulate(const FpMatrix& batch) {
    if (dim == 0 && token_count == 0) {
      dim = batch.cols;
      sum.assign(static_cast<size_t>(dim * dim), 0.0);
    }
    if (batch.cols != dim)
      throw std::invalid_argument("Hessian: batch has " + std::to_string(batch.cols) + " features, expected " +
                                  std::to_string(dim));
    if (batch.rows > 0) {
      detail::Buf dh(sum.data(), sum.size() * 8);
      detail::check(quik_hessian_accumulate(detail::ctx(), batch.data.data(), batch.rows, batch.cols,
                                            static_cast<double*>(dh.p)));
      dh.get(sum.data(), sum.size() * 8);
    }
    token_count += batch.rows;
  }
  double at(int64_t i, int64_t j) const { return sum[static_cast<size_t>(i * dim + j)]; }
  // quantizer.cpp:225-229: damping_frac * mean diagonal (trace summed in index order)
  double lambda() const {
    double trace = 0.0;
    for (int64_t i = 0; i < dim; ++i) trace += at(i, i);
    return damping_frac * trace / static_cast<double>(dim);
  }
  static Hessian identity(int64_t dim, double damping_frac = 0.01) {
    Hessian h;
    h.dim = dim;
    h.token_count = 1;
    h.damping_frac = damping_frac;
    h.sum.assign(static_cast<size_t>(dim * dim), 0.0);
    for (int64_t i = 0; i < dim; ++i) h.sum[static_cast<size_t>(i * dim + i)] = 1.0;
    return h;
  }
};

// quantizer.cpp:225-240
inline Hessian build_hessian(std::span<const FpMatrix> batches, double damping_frac = 0.01) {
  Hessian h;
  h.damping_frac = damping_frac;
  for (const FpMatrix& b : batches) h.accumulate(b);
  if (h.token_count == 0) throw std::invalid_argument("build_hessian: no calibration tokens");
  return h;
}

namespace detail {
inline QuantizedWeights gptq_device(const FpMatrix& w, const Hessian& h, const OutlierSet& o, int bits,
                                    bool use_clipping, bool sparse) {
  if (h.dim != w.cols)
    throw std::invalid_argument("Hessian dim " + std::to_string(h.dim) + " does not match weight columns " +
                                std::to_string(w.cols));
  if (o.feature_count != w.cols)
    throw std::invalid_argument("outlier set covers " + std::to_string(o.feature_count) + " features, weights have " +
                                std::to_string(w.cols));
  QuantizedWeights q;
  q.base.rows = w.rows;
  q.base.cols = o.base_count();
  q.base.bits = bits;
  q.base.data.resize(static_cast<size_t>(w.rows * q.base.row_bytes()));
  q.scales.resize(static_cast<size_t>(w.rows));
  q.wreduced.resize(static_cast<size_t>(w.rows));
  q.outlier_weights = FpMatrix(w.rows, o.outlier_count());
  if (sparse) {
    q.mask.rows = w.rows;
    q.mask.cols = o.base_count();
    q.mask.kept.resize(static_cast<size_t>(w.rows * o.base_count()));
  }
  if (w.rows == 0) return q;
  check(quik_gptq_quantize(ctx(), w.data.data(), w.rows, w.cols, h.sum.data(), h.damping_frac, o.indices.data(),
                           o.outlier_count(), bits, use_clipping ? 1 : 0, sparse ? 1 : 0, q.base.data.data(),
                           q.scales.data(), q.wreduced.data(), q.outlier_weights.data.data(),
                           sparse ? q.mask.kept.data() : nullptr));
  return q;
}
}  // namespace detail

// quantizer.cpp:292-297 / :299-337 on the device (FP64; quik_gptq_quantize)
inline QuantizedWeights gptq_quantize(const FpMatrix& w, const Hessian& h, const OutlierSet& o, int bits,
                                      bool use_clipping = false) {
  return detail::gptq_device(w, h, o, bits, use_clipping, false);
}
inline QuantizedWeights sparsegpt_joint(const FpMatrix& w, const Hessian& h, const OutlierSet& o, int bits,
                                        bool use_clipping = false) {
  return detail::gptq_device(w, h, o, bits, use_clipping, true);
}

// quantizer.hpp:94 / quantizer.cpp:373-382, on the device (bit-exact)
inline std::vector<float> compute_wreduced(const QuantizedWeights& q) {
  std::vector<float> out(static_cast<size_t>(q.base.rows));
  if (out.empty()) return out;
  detail::Buf db(q.base.data.data(), q.base.data.size()), ds(q.scales.data(), q.scales.size() * 4),
      dout(out.size() * 4);
  detail::check(quik_compute_wreduced(detail::ctx(), static_cast<const uint8_t*>(db.p), q.base.rows, q.base.cols,
                                      q.base.bits, static_cast<const float*>(ds.p), static_cast<float*>(dout.p),
                                      nullptr));
  detail::check(quik_ctx_sync(detail::ctx(), nullptr));
  dout.get(out.data(), out.size() * 4);
  return out;
}

// quantizer.hpp:98 / quantizer.cpp:384-403, on the device
inline FpMatrix dequantize_weights(const QuantizedWeights& q, const OutlierSet& o) {
  if (o.base_count() != q.base_features() || o.outlier_count() != q.outlier_weights.cols)
    throw std::invalid_argument("dequantize_weights: outlier set does not match weights");
  FpMatrix out(q.out_features(), o.feature_count);
  if (out.data.empty()) return out;
  detail::Buf db(q.base.data.data(), q.base.data.size()), ds(q.scales.data(), q.scales.size() * 4),
      dow(q.outlier_weights.data.data(), q.outlier_weights.data.size() * 4), dout(out.data.size() * 4);
  for (int64_t r0 = 0; r0 < out.rows; r0 += 65535) {
    const int64_t nr = std::min<int64_t>(65535, out.rows - r0);
    detail::check(quik_dequantize_weights(
        detail::ctx(), static_cast<const uint8_t*>(db.p) + r0 * q.base.row_bytes(), nr, o.feature_count, q.bits(),
        static_cast<const float*>(ds.p) + r0, static_cast<const float*>(dow.p) + r0 * o.outlier_count(),
        o.indices.data(), o.outlier_count(), static_cast<float*>(dout.p) + r0 * o.feature_count, nullptr));
  }
  detail::check(quik_ctx_sync(detail::ctx(), nullptr));
  dout.get(out.data.data(), out.data.size() * 4);
  return out;
}

// runtime.hpp:48 / runtime.cpp:169-186, on the device
inline std::pair<FpMatrix, FpMatrix> split_activations(const FpMatrix& x, const OutlierSet& o) {
  if (x.cols != o.feature_count)
    throw std::invalid_argument("split_activations: input has " + std::to_string(x.cols) +
                                " features, outlier set covers " + std::to_string(o.feature_count));
  FpMatrix base(x.rows, o.base_count()), outl(x.rows, o.outlier_count());
  if (x.rows == 0) return {std::move(base), std::move(outl)};
  QuikLinearLayer carrier;  // permutation tables only (no weight rows)
  carrier.outliers = o;
  carrier.weights.base.cols = o.base_count();
  carrier.weights.outlier_weights = FpMatrix(0, o.outlier_count());
  DeviceLayer L(carrier);
  detail::Buf dx(x.data.data(), x.data.size() * 4), db(base.data.size() * 4), dout(outl.data.size() * 4);
  detail::check(quik_split_activations(detail::ctx(), L.handle(), dx.p, QUIK_F32, x.rows, static_cast<float*>(db.p),
                                       static_cast<float*>(dout.p), nullptr));
  detail::check(quik_ctx_sync(detail::ctx(), nullptr));
  db.get(base.data.data(), base.data.size() * 4);
  dout.get(outl.data.data(), outl.data.size() * 4);
  return {std::move(base), std::move(outl)};
}

// ---------------------------------------------------------------- model graphs (runtime.hpp:91-111)
struct BlockOp {
  enum class Kind { Linear, Silu, Multiply, Add };
  Kind kind = Kind::Linear;
  int a = 0;
  int b = -1;
  int layer = -1;
};

// runtime.cpp:373-382: up/gate/SiLU/Hadamard/down over layers {0: up, 1: gate, 2: down}
inline std::vector<BlockOp> gated_mlp_ops() {
  using K = BlockOp::Kind;
  return {
      {K::Linear, 0, -1, 0},
      {K::Linear, 0, -1, 1},
      {K::Silu, 2, -1, -1},
      {K::Multiply, 3, 1, -1},
      {K::Linear, 4, -1, 2},
  };
}

// runtime.cpp:325-371 on the device: every value stays in device memory (f32); Linear ops
// run the QUIK forward of a DeviceLayer (uploaded once per call), Silu / Multiply / Add
// run quik_elementwise. Same op semantics and errors as the reference.
inline std::vector<FpMatrix> forward_model_trace(std::span<const QuikLinearLayer> layers,
                                                 std::span<const BlockOp> ops, const FpMatrix& x) {
  std::vector<std::unique_ptr<DeviceLayer>> dev(layers.size());
  std::vector<FpMatrix> values;
  std::vector<std::unique_ptr<detail::Buf>> dvals;
  values.reserve(ops.size() + 1);
  values.push_back(x);
  dvals.push_back(std::make_unique<detail::Buf>(x.data.data(), x.data.size() * 4));
  auto check_value = [&](int i) {
    if (i < 0 || i >= static_cast<int>(values.size()))
      throw std::invalid_argument("forward_model: op references undefined value " + std::to_string(i));
  };
  for (const BlockOp& op : ops) {
    switch (op.kind) {
      case BlockOp::Kind::Linear: {
        if (op.layer < 0 || op.layer >= static_cast<int>(layers.size()))
          throw std::invalid_argument("forward_model: op references undefined layer " + std::to_string(op.layer));
        check_value(op.a);
        const FpMatrix& in = values[static_cast<size_t>(op.a)];
        const QuikLinearLayer& L = layers[static_cast<size_t>(op.layer)];
        L.validate();
        if (in.cols != L.in_features())
          throw std::invalid_argument("quik_matmul: input has " + std::to_string(in.cols) +
                                      " features, layer expects " + std::to_string(L.in_features()));
        if (!dev[static_cast<size_t>(op.layer)]) dev[static_cast<size_t>(op.layer)] = std::make_unique<DeviceLayer>(L);
        FpMatrix v(in.rows, L.out_features());
        auto dv = std::make_unique<detail::Buf>(v.data.size() * 4);
        if (in.rows && v.cols) {
          const DeviceLayer& D = *dev[static_cast<size_t>(op.layer)];
          if (L.mode == LayerMode::WeightOnly)
            detail::check(quik_linear_forward_weight_only(detail::ctx(), D.handle(), dvals[op.a]->p, QUIK_F32, in.rows,
                                                          dv->p, QUIK_F32, v.cols, nullptr));
          else
            D.forward_device(dvals[op.a]->p, QUIK_F32, in.rows, dv->p, QUIK_F32);
        }
        values.push_back(std::move(v));
        dvals.push_back(std::move(dv));
        break;
      }
      case BlockOp::Kind::Silu: {
        check_value(op.a);
        FpMatrix v(values[op.a].rows, values[op.a].cols);
        auto dv = std::make_unique<detail::Buf>(v.data.size() * 4);
        detail::check(quik_elementwise(detail::ctx(), 0, static_cast<const float*>(dvals[op.a]->p), nullptr,
                                       static_cast<float*>(dv->p), v.size(), nullptr));
        values.push_back(std::move(v));
        dvals.push_back(std::move(dv));
        break;
      }
      case BlockOp::Kind::Multiply:
      case BlockOp::Kind::Add: {
        check_value(op.a);
        check_value(op.b);
        check_same_shape(values[op.a], values[op.b], "forward_model elementwise op");
        FpMatrix v(values[op.a].rows, values[op.a].cols);
        auto dv = std::make_unique<detail::Buf>(v.data.size() * 4);
        detail::check(quik_elementwise(detail::ctx(), op.kind == BlockOp::Kind::Multiply ? 1 : 2,
                                       static_cast<const float*>(dvals[op.a]->p),
                                       static_cast<const float*>(dvals[op.b]->p), static_cast<float*>(dv->p),
                                       v.size(), nullptr));
        values.push_back(std::move(v));
        dvals.push_back(std::move(dv));
        break;
      }
    }
  }
  if (values.size() == 1) throw std::invalid_argument("forward_model: empty op list");
  detail::check(quik_ctx_sync(detail::ctx(), nullptr));
  for (size_t i = 1; i < values.size(); ++i) dvals[i]->get(values[i].data.data(), values[i].data.size() * 4);
  return values;
}

inline FpMatrix forward_model(std::span<const QuikLinearLayer> layers, std::span<const BlockOp> ops,
                              const FpMatrix& x) {
  return std::move(forward_model_trace(layers, ops, x).back());
}

}  // namespace quik::b200
