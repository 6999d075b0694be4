// Internal kernel launch interface shared by the C-ABI layer (capi.cu) and the
// kernel translation units. Not part of the public ABI.
#pragma once

#include <string>

#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace quikb200 {

// Device-private GEMM operand layout ("GEMM layout"): row-major, one signed
// int8 per element, row pitch kpad = round_up(cols, 128) bytes, padding = 0.
constexpr int kKBlockBytes = 128;  // one K-block = one 128-byte swizzle atom per row
constexpr int kBlockM = 128;       // UMMA M (weight rows / output features per tile)

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and device
// (it is a host-side call per launch otherwise, visible at small M).
cudaError_t ensure_smem_attr_impl(const void* kernel, int bytes);  // capi.cu
template <typename K>
cudaError_t ensure_smem_attr(K kernel, int bytes) {
  return ensure_smem_attr_impl(reinterpret_cast<const void*>(kernel), bytes);
}
cudaError_t occupancy_cached_impl(const void* kernel, int threads, int smem, int* per_sm);  // capi.cu
template <typename K>
cudaError_t occupancy_cached(K kernel, int threads, int smem, int* per_sm) {
  return occupancy_cached_impl(reinterpret_cast<const void*>(kernel), threads, smem, per_sm);
}

// Output of the fused layer: y = f16/f32( (bias + dequant(acc)) + x_out . W_out^T ),
// where the outlier product is accumulated by the tensor cores onto the f32
// value bias + dequant(acc) held in TMEM (SURVEY.md A.3 tolerance; bit-exact
// when the layer has no outliers).
enum GemmMode : int {
  kModeInt32 = 0,       // out int32 [M][ldo]: raw base accumulator (int_matmul, V1/V2 stage)
  kModeAccInitF32 = 1,  // acc read from global int32 (V1/V2 tail), out f32
  kModeF32 = 2,         // fused int GEMM + epilogue + outliers, out f32
  kModeF16 = 3,         // same, out f16 (hot path)
  kModeProbe = 4,       // diagnostics: mainloop + TMEM traffic, no global stores
  kModeAccInitF16 = 5,  // acc read from global int32 (V1/V2 tail), out f16
  kModeF16Stats = 6,    // kModeF16 + the gated epilogue's down-projection statistics
                        // (GemmArgs::hstat; set by the launcher, dense / W4 tiles)
};

struct GemmArgs {
  // Operand A (weights, "N" side of the layer) and B (tokens), GEMM layout.
  const int8_t* w;       // [n_rows][kpad]
  const int8_t* x;       // [m_rows][kpad]
  int64_t kpad;          // bytes per row (multiple of 128); 0 => no integer part
  // Outlier operands, fp16, row pitch opad elements (multiple of 64), 0 => none.
  const __half* wo;      // [n_rows][opad]
  const __half* xo;      // [m_rows][opad]
  int64_t opad;
  int64_t M;             // tokens
  int64_t N;             // output features
  const float* w_scale;  // [N]
  const float* wreduced; // [N]
  const float* bias;     // [N] or nullptr
  const float* a_scale;  // [M]
  const float* a_zero;   // [M]
  float half_range;
  void* out;             // [M][ldo]
  int64_t ldo;           // elements
  int mode;
  const int32_t* acc_in; // kModeAccInit*: int32 accumulators [M][ld_acc]
  int64_t ld_acc;
  int32_t* acc_clear;    // kModeAccInit*: if non-null (== acc_in), zeroed after reading
  // 2:4 sparse base weights (sparse != 0; kpad multiple of 256): compressed values
  // [N][kpad / 2] (two kept codes per group of 4, ascending position) and metadata
  // planes [(2 * kb + h) * round_up(N, 128) + n][16 B] for stage kb (256 logical K),
  // half h (128 logical K = 32 groups, nibble per group, low nibble first).
  int sparse;
  const int8_t* w_sp;
  const uint8_t* meta;
  // INT4 weights in the device nibble layout [N][kpad / 2] (or null): per 16-byte chunk
  // c of a row, byte i = (k = 32c + i) | (k = 32c + 16 + i) << 4, signed 4-bit values.
  const uint8_t* w4;
  // gated MLP layer (rows interleave up / gate in blocks of 32): out is [M][N / 2],
  // h = silu(gate) * up (modes kModeF16 / kModeF32, no tile splitting of the pairs)
  int gated;
  // fused all-gather: every output tile is also TMA-stored to these
  // destinations (same [M][ldo] layout, typically peer GPUs' outputs mapped into this
  // process), f16 TMA-store outputs only
  void* const* peer_out;
  int n_peer;
  // gated MLP block (second half): the epilogue also reduces the next
  // (down) projection's per-token base min / max over the f16 h it stores, so the down
  // layer's K1 skips its reduction pass (QuantArgs::pre_stat). hstat [M] x uint4 =
  // {min key, max key, first-zero key, 0} (order-preserving u32 keys of the f16 values,
  // atomics; quik_gated_mlp_forward); hmask [ceil(N / 2 / 32)] words, bit f set =
  // feature f is a down-projection outlier column (or past the row); herr: non-finite
  // base h flag. hstat == nullptr: no statistics.
  uint4* hstat;
  const uint32_t* hmask;
  int* herr;
};
constexpr int kMaxPeerOut = 7;

// Decode-regime quik forward on INT4 weights after K1 (stream4.cu): split-K integer
// GEMM (TMEM-widened A, kind::i8), outlier MMAs and the dequant epilogue in one kernel.
struct Stream4Args {
  const uint8_t* w4;   // [N][kpad / 2] device INT4 layout (4-bit layers)
  const int8_t* w8;    // [N][kpad] (8-bit layers, when w4 is null)
  const int8_t* x;     // [M][kpad] activation codes (K1)
  int64_t kpad, M, N;
  const __half* wo;    // [N][opad]
  const __half* xo;    // [M][opad]
  int64_t opad;
  const float *a_scale, *a_zero, *w_scale, *wreduced, *bias;
  float half_range;
  int32_t* acc;        // [M][N] int32 workspace, zero on entry and exit
  int* counters;       // [stream4_counter_count(N)], zero on entry and exit
  void* out;
  int64_t ldo;
  int out_f16;
  int gated;           // gated MLP layer (rows interleave up / gate): out is [M][N / 2]
  void* const* peer_out;
  int n_peer;
};
size_t stream4_counter_count(int64_t N);
cudaError_t launch_stream4(const Stream4Args& a, int num_sms, cudaStream_t stream, const char** err_msg);

// WeightOnly forward (wo.cu, reference weight_only_forward runtime.cpp:115-136).
struct WoArgs {
  const void* x;        // [M][ldx] f16 or f32
  int x_is_f32;
  int64_t M, ldx;
  const int32_t* base_src;  // [kb] permuted base column -> source column
  int64_t kb, kpad;
  const int32_t* out_src;   // [n_out]
  int64_t n_out, opad;
  const uint8_t* w4;        // INT4 device layout [N][kpad / 2] (4-bit layers) or null
  const int8_t* w8;         // [N][kpad] (used when w4 is null)
  const __half* wo;         // [N][opad] f16(w_o)
  const __half* wo_lo;      // [N][opad] f16(w_o - f16(w_o))
  const float* scale;       // [N]
  const float* bias;        // [N] or null
  int64_t N;
  __half* xb;               // workspace [P*M][kpad] (P = 2 for f32 input)
  __half* xo;               // workspace [P*M][opad]
  float* ws;                // workspace (wo_workspace_bytes)
  void* y;
  int y_is_f16;
  int64_t ldy;
};
// Workspace bytes for ws (0 when the GEMM writes y directly) and the token planes.
size_t wo_workspace_bytes(const WoArgs& a, int num_sms, size_t* plane_bytes_b, size_t* plane_bytes_o);
cudaError_t launch_weight_only(const WoArgs& a, int num_sms, cudaStream_t stream, const char** err_msg);
// dst[r][c] = f16(src[r][c] - f16(src[r][c])) (zero padded to pitch)
cudaError_t launch_f16_lo_padded(const float* src, int64_t rows, int64_t cols, __half* dst, int64_t pitch,
                                 cudaStream_t stream);

// GPTQ / SparseGPT on the device (gptq.cu); returns 0 ok, 1 invalid argument,
// 3 numerical (Hessian not positive definite), 4 CUDA / library failure.
struct GptqArgs {
  const float* w;            // [N][K] (host or device)
  int64_t N, K;
  const double* hessian_sum; // [K][K] sum x x^T before damping (host or device)
  double damping;
  const int64_t* outlier_idx;  // host, sorted
  int64_t n_out;
  int bits, use_clipping, sparse;
  uint8_t* base;             // [N][row_bytes(K - n_out)] i4p / i8
  float* scales;             // [N]
  float* wreduced;           // [N]
  float* outlier_weights;    // [N][n_out]
  uint8_t* mask;             // [N][K - n_out] when sparse (else unused)
};
int gptq_quantize_device(const GptqArgs& a, std::string* msg);
int hessian_accumulate_device(const float* x, int64_t T, int64_t K, double* h_dev, std::string* msg);

// 2D K-major tensor map (uint8), box {box_inner bytes, box_rows}, 128-byte swizzle or none.
CUresult encode_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t pitch,
                       uint32_t box_inner, uint32_t box_rows, bool swizzle128);

// GEMM-layout int8 weights [N][kpad] (values in [-8, 7]) -> device INT4 layout above.
cudaError_t launch_pack_w4(const int8_t* w8, int64_t N, int64_t kpad, uint8_t* w4, cudaStream_t stream);
// ABI i4p rows [N][ceil(kb/2)] (packed.hpp:11-16: low nibble = even column, stored = v + 8)
// -> the device INT4 layout [N][kpad / 2] (zero beyond kb)
cudaError_t launch_pack_w4_abi(const uint8_t* i4p, int64_t N, int64_t kb, uint8_t* w4, int64_t kpad,
                               cudaStream_t stream);

// Compresses dense int8 GEMM-layout weights [N][kpad] (kpad % 256 == 0) into the
// 2:4 sparse operands above. *bad is set to 1 if a group of 4 has more than two
// non-zero codes (the layer then stays dense).
cudaError_t launch_compress_24(const int8_t* w8, int64_t N, int64_t kpad, int8_t* w_sp, uint8_t* meta, int* bad,
                               cudaStream_t stream);

// Launches the fused persistent tcgen05 kernel (int8 GEMM + f16 outlier GEMM +
// dequantisation epilogue). Returns a cudaError_t / CUresult-derived status in
// *err_msg on failure.
extern int gemm_tile_override;  // (cta_group << 16) | block_n, 0 = heuristic
extern int gemm_multicast;      // 1: 4-CTA TMA-multicast clusters for CTA-pair tiles
extern int gemm_stream4_auto;   // 1: 4-bit layers at M <= 32 use the INT4 stream kernel (default)
cudaError_t launch_quik_gemm(const GemmArgs& a, int num_sms, cudaStream_t stream, const char** err_msg);

// K1: fused split + per-token asymmetric quantisation (runtime.cpp:36-66,
// :199-220). x is [M][K] (f16 when x_is_f32 == 0, else f32), row pitch ldx.
struct QuantArgs {
  const void* x;
  int x_is_f32;
  int64_t M, K, ldx;
  // Outlier map (calibration.cpp:69-91, permutation = non-outliers ascending then
  // outliers), as per-layer tables (K <= 65520):
  //   lane_mask [round_up(K, 16)] bytes: 0xFF = outlier column, 0 = base
  //   gather    [kpad] u16: source column of base position j; j >= kb -> round_up(K, 16)
  //             (a zero code slot)
  //   out_src   [n_out] i32: outlier columns ascending
  // lane_mask == nullptr: no outliers (identity permutation, gather unused).
  const uint8_t* lane_mask;
  const uint16_t* gather;
  const int32_t* out_src;
  //   chunk_desc [kpad / 16] x uint4, the hot kernel's compaction rule per 16-byte
  //             output chunk (row independent): byte p = p < len1 ? A[p] : B[p] where
  //             A / B are 16-byte windows of the uncompacted code row.
  //               .x = A word offset (bytes, 4-aligned) | A funnel selector << 16
  //               .y = B word offset | B funnel selector << 16
  //               .z / .w = merge selectors of output words 0,1 / 2,3 (16 bits each)
  //             .x == 0xFFFFFFFF: "general" chunk (more than one gap), listed in
  //   gen_chunk [n_gen] u16 and gathered per byte through `gather`.
  const uint32_t* chunk_desc;
  const uint16_t* gen_chunk;
  int n_gen;
  int64_t kb;               // base column count K_b
  int64_t n_out;
  int bits;                 // 4 or 8
  int hot_flags;            // hot K1 tuning (set by the launcher): bit 0 = sleep-wait on the row ring
  int8_t* q8;               // GEMM layout [M][kpad] or nullptr
  int64_t kpad;
  uint8_t* packed;          // ABI layout [M][row_bytes] (i4p / i8) or nullptr
  float* scale;             // [M]
  float* zero;              // [M]
  __half* xo16;             // [M][opad] fp16 outliers (GEMM layout) or nullptr
  int64_t opad;
  float* xo32;              // [M][n_out] fp32 outliers (ABI) or nullptr
  int* err;                 // device flag, set to 1 on non-finite base input
  // Row slices of the wide hot quantizer (K1 over a thread-block cluster, one CTA per
  // slice; n_slice >= 2): slice_desc [n_slice] x int32[8] = {first column (multiple of
  // 8), columns, first / end output chunk, first / end outlier slot, first / end index
  // into gen_chunk}; the sizes below are maxima over the slices.
  const int32_t* slice_desc;
  int n_slice;
  int slice_cols_max;       // columns of the widest slice
  int slice_chunks_max;     // output chunks of the busiest slice
  int slice_code_bytes;     // shared code-row bytes (window reads and the zero tail included)
  // Prescaled rows (hot kernel only): the per-token base min / max were reduced by the
  // producing GEMM's epilogue (GemmArgs::hstat); the kernel reads them instead of its own
  // reduction pass and restores the keys to their initial values for the next forward.
  uint4* pre_stat;
};
// hstat / pre_stat keys: f16 bits u (signed zeros canonicalised to +0) ->
// u >= 0 ? u | 0x8000 : 0x7FFF - (u & 0x7FFF); initial {0xFFFFFFFF, 0, 0xFFFFFFFF, 0}
cudaError_t launch_hstat_init(uint4* stat, int64_t M, cudaStream_t stream);
cudaError_t launch_quantize(const QuantArgs& a, cudaStream_t stream);

// V1 split (runtime.cpp:169-186): base columns in permutation order as f32
// [M][kb] and outlier columns as f16 GEMM operands [M][opad].
struct SplitArgs {
  const void* x;
  int x_is_f32;
  int64_t M, K, ldx;
  const int32_t* base_src;
  int64_t kb;
  const int32_t* out_src;
  int64_t n_out;
  float* xbase;
  __half* xo16;
  int64_t opad;
  float* xo32;  // split_activations: f32 outlier columns [M][n_out] (instead of xo16)
};
cudaError_t launch_split(const SplitArgs& a, cudaStream_t stream);

// Unpacks ABI packed rows (i4p or i8, packed.hpp:11-16) into the GEMM layout.
cudaError_t launch_unpack_to_gemm(const uint8_t* packed, int64_t rows, int64_t cols, int bits, int8_t* dst,
                                  int64_t kpad, cudaStream_t stream);

// f32 [rows][cols] -> f16 [rows][pitch], zero padded.
cudaError_t launch_f32_to_f16_padded(const float* src, int64_t rows, int64_t cols, __half* dst,
                                     int64_t pitch, cudaStream_t stream);

// rtn_quantize_weights (quantizer.cpp:339-371): f32 W [N][K] (device) -> ABI
// packed base [N][row_bytes(kb)], scales, wreduced, outlier weights [N][n_out].
cudaError_t launch_rtn_weights(const float* w, int64_t N, int64_t K, const int32_t* base_src, int64_t kb,
                               const int32_t* out_src, int64_t n_out, int bits, uint8_t* base, float* scales,
                               float* wreduced, float* outlier_w, const float* clip, cudaStream_t stream);

// weights.cu: clip_search per row (clip may then feed launch_rtn_weights), compute_wreduced,
// dequantize_weights, forward_model's elementwise ops (0 silu, 1 multiply, 2 add).
cudaError_t launch_clip_search(const float* w, int64_t N, int64_t K, const int32_t* base_src, int64_t kb, int bits,
                               float* clip, cudaStream_t stream);
cudaError_t launch_compute_wreduced(const uint8_t* base, int64_t N, int64_t kb, int bits, const float* scales,
                                    float* out, cudaStream_t stream);
cudaError_t launch_dequantize_weights(const uint8_t* base, int64_t N, int64_t K, int64_t kb, int bits,
                                      const float* scales, const int32_t* perm, const float* ow, float* out,
                                      cudaStream_t stream);
cudaError_t launch_elementwise(int op, const float* a, const float* b, float* out, int64_t n, cudaStream_t stream);

// dequantize_epilogue (runtime.cpp:222-244): out[t][r] = dequant_element(...).
cudaError_t launch_dequant(const int32_t* acc, int64_t M, int64_t N, const float* a_scale,
                           const float* a_zero, float half_range, const float* w_scale,
                           const float* wreduced, float* out, cudaStream_t stream);

// V1/V2 tail: out[t][r] = out[t][r] + dequant_element(acc[t][r], ...), f32 or f16 result.
cudaError_t launch_dequant_add(const int32_t* acc, int64_t M, int64_t N, const float* a_scale,
                               const float* a_zero, float half_range, const float* w_scale,
                               const float* wreduced, const float* fp_part, void* out, int out_is_f16,
                               cudaStream_t stream);

}  // namespace quikb200
