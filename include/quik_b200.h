/*
 * quik_b200.h — C ABI of the B200-native QUIK hybrid W4A4 / W8A8 linear layer.
 *
 * Drop-in boundary for the reference's C++ layer API (namespace quik, in
 * /root/reference/proj). Each entry point names the reference interface it
 * replaces. Plain pointers and sizes only; no exceptions cross this boundary:
 * every call returns a quik_status and quik_last_error() holds the message
 * (thread-local). The C++ facade in quik_b200.hpp rethrows them as the
 * reference's exception types (std::invalid_argument, std::out_of_range,
 * quik::NumericalError).
 *
 * Memory: unless stated otherwise pointers are DEVICE pointers owned by the
 * caller, and calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy
 * default stream). Non-finite activations raise a device flag which the next
 * quik_ctx_sync() reports as QUIK_ERR_NUMERICAL (reference runtime.cpp:52).
 *
 * Threading: a layer handle is immutable after creation; forwards on the same
 * layer may run concurrently from different contexts (SPEC.md "forward passes
 * are pure and may run concurrently"). A context owns scratch memory and must
 * not be used from two host threads at once. Calls through one context on
 * different streams are ordered: each call waits (cudaStreamWaitEvent) for the
 * previous call's work when the stream changes, so they cannot race on the
 * scratch; a CUDA graph captured through a context must be replayed on one stream.
 *
 * Numerical errors: a non-finite activation sets the context's device flag; the
 * next quik_ctx_sync() reports QUIK_ERR_NUMERICAL and clears it. Asynchronous
 * forwards do not check it themselves; quik_ctx_clear_error() resets it before a
 * call whose errors should be reported on their own.
 */
#ifndef QUIK_B200_H_
#define QUIK_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QUIK_B200_ABI_VERSION 3

typedef enum quik_status {
  QUIK_OK = 0,
  QUIK_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  QUIK_ERR_OUT_OF_RANGE = 2,     /* reference: std::out_of_range (pack range errors) */
  QUIK_ERR_NUMERICAL = 3,        /* reference: quik::NumericalError (non-finite activations) */
  QUIK_ERR_CUDA = 4,             /* CUDA runtime / driver failure, or no sm_100 device */
  QUIK_ERR_NCCL = 5,             /* reserved: collective failure */
  QUIK_ERR_UNSUPPORTED = 6,
  QUIK_ERR_FORMAT = 7            /* reference: quik::FormatError (layer bundle I/O) */
} quik_status;

/* Element types of activation / output buffers. */
typedef enum quik_dtype { QUIK_F16 = 0, QUIK_F32 = 1 } quik_dtype;

/* reference: quik::PipelineVariant (runtime.hpp:31). All three are bit-identical. */
typedef enum quik_variant { QUIK_V1_UNFUSED = 0, QUIK_V2_FUSED_QUANT = 1, QUIK_V3_FUSED_EPILOGUE = 2 } quik_variant;

typedef struct quik_ctx_s* quik_ctx_t;
typedef struct quik_layer_s* quik_layer_t;

const char* quik_last_error(void);
const char* quik_status_string(quik_status s);
int quik_abi_version(void);

/* Context: device binding, scratch memory, device error flag. */
quik_status quik_ctx_create(int device, quik_ctx_t* out);
quik_status quik_ctx_destroy(quik_ctx_t ctx);
/* Synchronises `stream`, then reports (and clears) the non-finite-input flag. */
quik_status quik_ctx_sync(quik_ctx_t ctx, void* stream);
/* Clears the non-finite-input flag (asynchronously, on `stream`). */
quik_status quik_ctx_clear_error(quik_ctx_t ctx, void* stream);
/* Sizes the context's scratch for forwards of `layer` with up to M tokens (codes,
 * scales, outlier operands, the decode workspace and the INT4 weight copy at M <= 32;
 * for a gated layer also the quik_gated_mlp_forward statistics — reserve the block's
 * gated layer and its down projection),
 * so that later forwards can be captured into a CUDA graph: scratch cannot grow during
 * capture (those calls return QUIK_ERR_INVALID_ARGUMENT). Synchronous. */
quik_status quik_ctx_reserve(quik_ctx_t ctx, quik_layer_t layer, int64_t M);

/*
 * Layer weights, HOST memory, in the reference's formats.
 * reference: quik::QuantizedWeights (quantizer.hpp:48-58), quik::OutlierSet
 * (calibration.hpp:37-48), quik::QuikLinearLayer (runtime.hpp:33-44).
 *   base            packed [out_features][row_bytes]: bits 4 -> i4p (low nibble = even
 *                   column, stored = v + 8, packed.hpp:11-16), bits 8 -> two's complement
 *   scales          [out_features] per-row symmetric weight scales
 *   wreduced        [out_features] scale[r] * sum_j q[r][j] (quantizer.cpp:159-165)
 *   outlier_weights [out_features][n_outlier] f32 (rounded to f16 on the device)
 *   outlier_indices [n_outlier] sorted, unique, in [0, in_features)
 *   bias            [out_features] or NULL
 *   All arrays except outlier_indices may be host or device memory (UVA copy).
 *   row_begin/row_end: optional output-row shard [row_begin, row_end) of the layer
 *                   (multi-GPU column sharding); 0/0 = all rows.
 */
typedef struct quik_weights_desc {
  int64_t in_features;
  int64_t out_features;
  int bits;     /* base weight bits: 4 or 8 */
  int act_bits; /* activation bits; must equal bits (runtime.cpp:162-164) */
  const uint8_t* base;
  const float* scales;
  const float* wreduced;
  const float* outlier_weights;
  const int64_t* outlier_indices;
  int64_t n_outlier;
  const float* bias;
  int64_t row_begin;
  int64_t row_end;
  /* 1: the base weights are 2:4 structured sparse (reference: sparsegpt_joint,
   * quantizer.cpp:299-337 -- at most two non-zero codes per aligned group of 4
   * permuted base columns). The layer is compressed to half the codes + 4-bit
   * metadata and runs on tcgen05.mma.sp (exactly equal to the dense sum). If some
   * group has more than two non-zero codes the layer stays dense; see
   * quik_layer_is_sparse. 0: dense. (ABI version 2; absent in version 1.) */
  int sparsity;
  /* Device copy of 4-bit dense base weights (ABI version 3):
   *   QUIK_WEIGHTS_SPEED (0, default): INT8 GEMM-layout weights for the prefill GEMM
   *     (the tensor-bound regime runs at the full kind::i8 rate) and, made on the first
   *     decode-regime forward (or quik_ctx_reserve), an INT4 copy for M <= 32;
   *   QUIK_WEIGHTS_INT4 (1): ONLY the INT4 copy (half the weight bytes of INT8; QUIK's
   *     memory footprint): every GEMM streams INT4 tiles and widens them into TMEM.
   * 8-bit and 2:4-compressed layers have one device copy either way. */
  int weight_mode;
} quik_weights_desc;

#define QUIK_WEIGHTS_SPEED 0
#define QUIK_WEIGHTS_INT4 1

/* Uploads and repacks the weights into the device GEMM layout.
 * Replaces QuikLinearLayer::validate (runtime.cpp:150-167) + per-call unpack_int4
 * of the weights (packed.cpp:110-111), which the device path does once here. */
quik_status quik_layer_create(quik_ctx_t ctx, const quik_weights_desc* desc, quik_layer_t* out);
quik_status quik_layer_destroy(quik_layer_t layer);

/* Gated MLP projection (reference forward_model with gated_mlp_ops,
 * runtime.cpp:320-392): one layer computing h = silu(gate(x)) * up(x) [M][F] in a
 * single K1 + GEMM launch pair -- the up and gate rows are interleaved in blocks of 32
 * so every GEMM tile holds both projections of the same 32-feature blocks, and the
 * epilogue forms silu(gate) * up in f32 (silu(e) = e / (1 + exp(-e))) before the
 * f16/f32 store. up / gate: same shapes, bits and outlier set (the shared input x is
 * quantized once); F (and a row shard) a multiple of 32. The down projection is a
 * plain layer applied to h. quik_layer_info reports out_features = F. */
quik_status quik_layer_create_gated(quik_ctx_t ctx, const quik_weights_desc* up, const quik_weights_desc* gate,
                                   quik_layer_t* out);
/* Gated MLP block (reference forward_model with gated_mlp_ops,
 * runtime.cpp:373-388): y = down(silu(gate(x)) * up(x)). gated: a
 * quik_layer_create_gated layer, down: a plain layer with in_features = F.
 * h: device f16 [M][ldh] hidden state (written; ldh >= F, any pitch); y: [M][ldy] of ydt.
 * Above the decode regime the gated GEMM's epilogue also reduces the down projection's
 * per-token min / max over the base (non-outlier) columns of the f16 h it stores, and
 * the down projection's quantizer consumes them instead of its own reduction pass
 * (runtime.cpp:36-50 split across the two kernels). h, the down codes / scales and y
 * are bit-identical to quik_linear_forward(gated) followed by quik_linear_forward(down)
 * on h. Non-finite base values of h raise the context's numerical flag
 * (quik_ctx_sync -> QUIK_ERR_NUMERICAL), as the down quantizer would. Asynchronous. */
quik_status quik_gated_mlp_forward(quik_ctx_t ctx, quik_layer_t gated, quik_layer_t down, const void* x,
                                   quik_dtype xdt, int64_t M, void* h, int64_t ldh, void* y, quik_dtype ydt,
                                   int64_t ldy, void* stream);
quik_status quik_layer_info(quik_layer_t layer, int64_t* in_features, int64_t* out_features,
                            int64_t* n_outlier, int* bits);
/* 1 if the layer runs the 2:4 sparse GEMM (sparsity requested and compressible). */
int quik_layer_is_sparse(quik_layer_t layer);
/* Device GEMM layout of the layer's activation operands (what quik_quantize_activations_gemm
 * writes): codes int8 [M][kpad], x_outlier16 f16 [M][opad]. */
quik_status quik_layer_layout(quik_layer_t layer, int64_t* kpad, int64_t* opad);
/* Device memory the layer holds (weights in every copy it keeps, per-row vectors,
 * outlier tables), bytes; -1 for a null layer. */
int64_t quik_layer_device_bytes(quik_layer_t layer);

/*
 * Layer bundles: the reference's on-disk layer format
 * (<dir>/manifest.json + blob files; container.cpp, layer_io.cpp), read on the host
 * with every check of TensorContainer::read (container.cpp:167-226) and load_layer
 * (layer_io.cpp:32-74); failures return QUIK_ERR_FORMAT (quik::FormatError).
 * quik_bundle_weights fills a descriptor with host pointers into the bundle
 * (valid until quik_bundle_close; sparsity = 1 when a sparsity_mask is present),
 * ready for quik_layer_create (set row_begin / row_end for a shard).
 * quik_bundle_tensor exposes any tensor: dtype 0 = f32, 1 = i8, 2 = i4p; shape[<= 4].
 */
typedef struct quik_bundle_s* quik_bundle_t;
quik_status quik_bundle_open(const char* dir, quik_bundle_t* out);
quik_status quik_bundle_weights(quik_bundle_t bundle, quik_weights_desc* desc);
quik_status quik_bundle_tensor(quik_bundle_t bundle, const char* name, const void** data, int* dtype,
                               int64_t* shape, int* ndim);
quik_status quik_bundle_close(quik_bundle_t bundle);
/* open + quik_layer_create (shard [row_begin, row_end), 0/0 = all rows) + close:
 * bundle -> device GEMM layout in one call. */
quik_status quik_layer_load_bundle(quik_ctx_t ctx, const char* dir, int64_t row_begin, int64_t row_end,
                                   quik_layer_t* out);

/*
 * K1 fused quantizer. reference: quantize_activations_fused (runtime.hpp:55-56,
 * runtime.cpp:199-220). x: [M][in_features] (x_dtype). Outputs in the reference
 * formats: packed [M][row_bytes(K_b)] (i4p or i8), scale[M], zero[M] (row min),
 * x_outlier [M][n_outlier] f32. Any output pointer may be NULL.
 */
quik_status quik_quantize_activations_fused(quik_ctx_t ctx, quik_layer_t layer, const void* x, quik_dtype x_dtype,
                                            int64_t M, uint8_t* packed, float* scale, float* zero,
                                            float* x_outlier, void* stream);

/* K1 exactly as the hot path runs it, into caller buffers in the device GEMM
 * layout (diagnostics / parity): codes int8 [M][kpad] (kpad = round_up(K_b, 128),
 * signed stored codes in permuted base order, zero padded), scale[M], zero[M],
 * x_outlier16 f16 [M][opad] (opad = round_up(n_outlier, 64), zero padded). */
quik_status quik_quantize_activations_gemm(quik_ctx_t ctx, quik_layer_t layer, const void* x, quik_dtype x_dtype,
                                           int64_t M, int8_t* codes, float* scale, float* zero, void* x_outlier16,
                                           void* stream);

/* Unfused quantizer of an already-split base matrix [M][K].
 * reference: quantize_activations (runtime.hpp:51, runtime.cpp:188-197). */
quik_status quik_quantize_activations(quik_ctx_t ctx, const void* x_base, quik_dtype x_dtype, int64_t M, int64_t K,
                                      int bits, uint8_t* packed, float* scale, float* zero, void* stream);

/* Exact INT32 GEMM of two packed operands, out[i][j] = sum_k x[i][k] * w[j][k].
 * reference: int_matmul (packed.hpp:58, packed.cpp:93-132), same argument checks. */
quik_status quik_int_matmul(quik_ctx_t ctx, const uint8_t* x_packed, int64_t x_rows, int64_t x_cols, int x_bits,
                            const uint8_t* w_packed, int64_t w_rows, int64_t w_cols, int w_bits, int32_t* out,
                            void* stream);

/* out[t][r] = acc[t][r]*sa[t]*sw[r] + (za[t] + half_range*sa[t]) * wreduced[r], f32.
 * reference: dequantize_epilogue (runtime.hpp:66-68, runtime.cpp:222-244), bit-exact. */
quik_status quik_dequantize_epilogue(quik_ctx_t ctx, const int32_t* acc, int64_t M, int64_t N,
                                     const float* scale_act, const float* zero_act, int half_range,
                                     const float* weight_scales, const float* wreduced, float* out, void* stream);

/* The hot path: y[M][out_features] = quik_matmul(layer, x).
 * reference: quik_matmul (runtime.hpp:85-87, runtime.cpp:246-318), LayerMode::Quik.
 * x_dtype/y_dtype: QUIK_F16 (hot) or QUIK_F32. V3 runs two kernels: K1 and the
 * fused tcgen05 GEMM + epilogue. V1/V2 run the unfused stages for debugging. */
quik_status quik_linear_forward(quik_ctx_t ctx, quik_layer_t layer, const void* x, quik_dtype x_dtype, int64_t M,
                                void* y, quik_dtype y_dtype, quik_variant variant, void* stream);

/* Same, writing into a column slice of a wider output: y + col_offset with row
 * pitch ldy elements (used by sharded layers to place their shard in place). */
quik_status quik_linear_forward_strided(quik_ctx_t ctx, quik_layer_t layer, const void* x, quik_dtype x_dtype,
                                        int64_t M, void* y, quik_dtype y_dtype, int64_t ldy, quik_variant variant,
                                        void* stream);

/* Same as _strided; additionally records `mid_event` (a cudaEvent_t, may be NULL)
 * on `stream` between the quantizer and the GEMM launch (V3) for per-kernel timing. */
quik_status quik_linear_forward_ex(quik_ctx_t ctx, quik_layer_t layer, const void* x, quik_dtype x_dtype, int64_t M,
                                   void* y, quik_dtype y_dtype, int64_t ldy, quik_variant variant, void* stream,
                                   void* mid_event);

/* GPTQ / SparseGPT weight quantisation on the device: the reference's
 * gptq_quantize (quantizer.cpp:292-297, sparse = 0) or sparsegpt_joint (:299-337,
 * sparse = 1) with Hessian hessian_sum [K][K] f64 (sum x x^T before damping, host or
 * device) and damping_frac; FP64 throughout (cuSOLVER Cholesky, blocked column
 * recursion with DGEMM trailing updates). w [N][K] f32 and the outputs may be host or
 * device memory (UVA); outputs in the reference's layout: base i4p/i8 [N][row bytes of
 * K - n_outlier], scales/wreduced [N], outlier_weights [N][n_outlier], mask [N][K - n]
 * (sparse). Synchronous. QUIK_ERR_NUMERICAL when the damped Hessian is not positive
 * definite (the reference's NumericalError). */
quik_status quik_gptq_quantize(quik_ctx_t ctx, const float* w, int64_t N, int64_t K, const double* hessian_sum,
                               double damping_frac, const int64_t* outlier_indices, int64_t n_outlier, int bits,
                               int use_clipping, int sparse, uint8_t* base, float* scales, float* wreduced,
                               float* outlier_weights, uint8_t* mask);

/* Hessian::accumulate (quantizer.cpp:193-213): h_sum [K][K] f64 (DEVICE memory) += x^T x
 * for the calibration batch x [T][K] f32 (host or device). Synchronous. */
quik_status quik_hessian_accumulate(quik_ctx_t ctx, const float* x, int64_t T, int64_t K, double* h_sum);

/* Output-feature shard forward with the all-gather fused into the epilogue (SURVEY.md
 * §8e; replaces quik_matmul + ncclAllGather for one shard): the shard layer's f16
 * output tiles [M][shard columns] are TMA-stored at column `col_offset` of EVERY
 * destination y_dst[0..n_dst) (row pitch ldy elements): y_dst[0] is this GPU's output,
 * the others peer GPUs' outputs mapped into this process (cudaDeviceEnablePeerAccess
 * or cudaIpcOpenMemHandle), so the exchange rides NVLink tile by tile while the GEMM
 * runs. n_dst <= 8; col_offset and ldy multiples of 8. The caller orders readers
 * after every rank's call (stream events / a barrier), as after an all-gather. */
quik_status quik_linear_forward_sharded(quik_ctx_t ctx, quik_layer_t shard, const void* x, quik_dtype x_dtype,
                                        int64_t M, void* const* y_dst, int n_dst, int64_t ldy, int64_t col_offset,
                                        void* stream);

/* CUDA IPC plumbing for the fused all-gather across processes (one process per GPU):
 * quik_ipc_handle_get returns the IPC handle of the allocation holding `dev_ptr` and
 * the byte offset of dev_ptr inside it (works for pointers from caching allocators);
 * another process opens it with quik_ipc_handle_open (peer access enabled lazily) and
 * gets the same buffer mapped at *dev_ptr (offset applied), suitable as a y_dst of
 * quik_linear_forward_sharded; quik_ipc_handle_close unmaps it. */
typedef struct quik_ipc_handle {
  unsigned char bytes[64]; /* cudaIpcMemHandle_t */
  int64_t offset;          /* byte offset of the pointer inside the allocation */
} quik_ipc_handle;
quik_status quik_ipc_handle_get(quik_ctx_t ctx, const void* dev_ptr, quik_ipc_handle* out);
quik_status quik_ipc_handle_open(quik_ctx_t ctx, const quik_ipc_handle* handle, void** dev_ptr);
quik_status quik_ipc_handle_close(quik_ctx_t ctx, void* dev_ptr, const quik_ipc_handle* handle);

/* WeightOnly mode (reference LayerMode::WeightOnly, weight_only_forward,
 * runtime.cpp:115-136): activations stay floating point,
 *   y = (bias + x_o W_o^T) + x_b (q * scale)^T
 * on device buffers, asynchronous on `stream`. 4-bit layers stream INT4 weights (an
 * INT4 copy is made on the first call). Every product is exact; f32 accumulation in
 * a different order than the reference. f32 inputs are carried as two f16 planes
 * (hi + lo), f16 inputs exactly; inputs must be inside the f16 range. Not for gated
 * or 2:4-compressed layers (QUIK_ERR_UNSUPPORTED). */
quik_status quik_linear_forward_weight_only(quik_ctx_t ctx, quik_layer_t layer, const void* x, quik_dtype x_dtype,
                                            int64_t M, void* y, quik_dtype y_dtype, int64_t ldy, void* stream);

/* The hot path with HOST activations and outputs: what the reference's
 * quik_matmul(layer, FpMatrix) call (runtime.hpp:85-87) does with host data.
 * x_host [M][in_features] and y_host [M][out_features] are host memory (page-locked
 * for full overlap). The token rows are processed in chunks of `chunk_tokens`
 * (0 = automatic, about 16 chunks of multiples of 256): the host->device copy of
 * chunk c+1, the V3 kernels of chunk c and the device->host copy of chunk c-1 run
 * concurrently on context-owned copy streams. Asynchronous on `stream`: y_host is
 * complete once `stream` reaches this point (synchronise or use quik_ctx_sync). */
quik_status quik_linear_forward_host(quik_ctx_t ctx, quik_layer_t layer, const void* x_host, quik_dtype x_dtype,
                                     int64_t M, void* y_host, quik_dtype y_dtype, int64_t chunk_tokens, void* stream);

/* Round-to-nearest weight quantization on the device.
 * reference: rtn_quantize_weights (quantizer.hpp:89-90, quantizer.cpp:339-371); with
 * use_clipping the per-row clip factor of clip_search (quantizer.cpp:266-290: 51
 * factors 0.50..1.00, sequential FP64 error sums, ties to the larger factor); bit-exact
 * (FP64 scale, ties away from zero, wreduced in FP64).
 * w: DEVICE f32 [N][K]. outlier_indices: HOST, sorted unique. Outputs (DEVICE):
 * base packed [N][row_bytes(K - n_outlier)] (i4p / i8), scales [N], wreduced [N],
 * outlier_weights [N][n_outlier] f32 (original values, permuted-tail order). */
quik_status quik_rtn_quantize_weights(quik_ctx_t ctx, const float* w, int64_t N, int64_t K,
                                      const int64_t* outlier_indices, int64_t n_outlier, int bits, int use_clipping,
                                      uint8_t* base, float* scales, float* wreduced, float* outlier_weights,
                                      void* stream);

/* quik_matmul with StageTimes (runtime.hpp:72-80, runtime.cpp:265-315): the forward of
 * quik_linear_forward_strided timed with CUDA events at the kernel boundaries; waits for
 * completion. stage_ms[6] = {split, quantize, int_matmul, fp_matmul, dequantize, add}
 * (ms), fused_flags[2] = {quantize_fused, dequantize_fused}. A fused stage reports under
 * the first field it covers, as in the reference: V3 -> quantize_ms (K1: split +
 * quantize) and int_matmul_ms (the fused GEMM: int + outlier matmul + dequantize + add);
 * V1 -> split_ms, quantize_ms, int_matmul_ms (int32 GEMM) and fp_matmul_ms (one kernel:
 * outlier matmul + dequantize + add); V2 as V1 with split folded into quantize_ms. */
quik_status quik_linear_forward_timed(quik_ctx_t ctx, quik_layer_t layer, const void* x, quik_dtype x_dtype,
                                      int64_t M, void* y, quik_dtype y_dtype, int64_t ldy, quik_variant variant,
                                      void* stream, double* stage_ms, int* fused_flags);

/* split_activations (runtime.hpp:48, runtime.cpp:169-186): x [M][in_features] ->
 * x_base f32 [M][K_b] (permuted base columns) and x_outlier f32 [M][n_outlier]. */
quik_status quik_split_activations(quik_ctx_t ctx, quik_layer_t layer, const void* x, quik_dtype x_dtype, int64_t M,
                                   float* x_base, float* x_outlier, void* stream);

/* unpack_values / unpack_int4 (packed.hpp:48-51, packed.cpp:68-91): packed
 * [rows][row_bytes] -> int8 [rows][cols]. */
quik_status quik_unpack_values(quik_ctx_t ctx, const uint8_t* packed, int64_t rows, int64_t cols, int bits,
                               int8_t* out, void* stream);

/* compute_wreduced (quantizer.hpp:94, quantizer.cpp:373-382): wreduced[r] =
 * float(double(scales[r]) * sum_j q[r][j]), bit-exact. base packed [rows][row_bytes(cols)]. */
quik_status quik_compute_wreduced(quik_ctx_t ctx, const uint8_t* base, int64_t rows, int64_t cols, int bits,
                                  const float* scales, float* wreduced, void* stream);

/* dequantize_weights (quantizer.hpp:98, quantizer.cpp:384-403): the de-permuted f32
 * reconstruction out [rows][in_features]: q * scale in the base columns, the outlier
 * weights in theirs. base / scales / outlier_weights / out DEVICE; outlier_indices HOST
 * (sorted, unique); rows <= 65535 per call. Synchronous. */
quik_status quik_dequantize_weights(quik_ctx_t ctx, const uint8_t* base, int64_t rows, int64_t in_features, int bits,
                                    const float* scales, const float* outlier_weights, const int64_t* outlier_indices,
                                    int64_t n_outlier, float* out, void* stream);

/* forward_model's elementwise block ops (runtime.cpp:339-360) on f32 device buffers:
 * op 0 = Silu out = a / (1 + exp(-a)), 1 = Multiply out = a * b, 2 = Add out = a + b. */
quik_status quik_elementwise(quik_ctx_t ctx, int op, const float* a, const float* b, float* out, int64_t n,
                             void* stream);

/* Tuning/debug knob (process-wide): force the GEMM tile, cta_group in {1, 2} and
 * token block_n in {32, 64, 128} (1-CTA) or {128, 192, 256} (CTA pair; 2:4 sparse and
 * 4-bit (INT4-weight) layers use 192 where 256 is asked, 8-bit dense ones 256 for 192);
 * (0, 0) restores the heuristic. */
quik_status quik_set_gemm_tile(int cta_group, int block_n);

/* Tuning knob (process-wide): 1 runs the CTA-pair GEMM tiles of 8-bit dense layers in
 * 4-CTA clusters whose two pairs share (TMA-multicast) the activation tiles; 0 (default)
 * plain CTA pairs. */
quik_status quik_set_gemm_multicast(int on);

/* Tuning: dense layers at M <= 32 run the decode kernel (stream4.cu: split-K over all
 * SMs on INT4 weights widened into TMEM (4-bit) or INT8 tiles (8-bit), the fused
 * epilogue in the same kernel; bit-identical to the fused path). Default on; 0 = the
 * fused kernel. */
quik_status quik_set_int4_decode(int on);

/* Diagnostics (process-wide): when on, the V3 forward runs the fused GEMM
 * without writing the output (mainloop + TMEM drain only). Never for results. */
quik_status quik_set_probe_mode(int on);

/* Number of device kernels quik_linear_forward launches for (variant) — the
 * bench reports it as gpu_launches. */
int quik_linear_forward_launches(quik_variant variant);

#ifdef __cplusplus
}
#endif
#endif /* QUIK_B200_H_ */
