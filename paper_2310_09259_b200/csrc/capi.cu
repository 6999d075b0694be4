// C-ABI implementation (include/quik_b200.h). Argument checking mirrors the
// reference's exceptions (runtime.cpp / packed.cpp); device work is delegated
// to the kernels in gemm.cu and quantize.cu. No CPU compute fallback exists:
// every numerical result comes from a CUDA kernel.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <tuple>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/quik_b200.h"
#include "kernels.h"

using namespace quikb200;

namespace quikb200 {
// cudaFuncSetAttribute once per (kernel, device, size): a host call per launch
// otherwise, which shows up as GPU idle time at small token counts.
cudaError_t ensure_smem_attr_impl(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find({kernel, dev});
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[{kernel, dev}] = bytes;
  return e;
}
// Resident CTAs per SM, queried once per (kernel, device, block size, smem bytes).
cudaError_t occupancy_cached_impl(const void* kernel, int threads, int smem, int* per_sm) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int>, int> seen;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = seen.find({kernel, dev, threads, smem});
  if (it != seen.end()) { *per_sm = it->second; return cudaSuccess; }
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kernel, threads, smem);
  if (e == cudaSuccess) seen[{kernel, dev, threads, smem}] = *per_sm;
  return e;
}
}  // namespace quikb200

namespace {
thread_local std::string g_err;
}  // namespace

namespace quikb200 {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace quikb200

namespace {

int g_probe_mode = 0;  // diagnostics: V3 GEMM without output stores (quik_set_probe_mode)

quik_status fail(quik_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

struct CudaFail {
  cudaError_t e;
  const char* what;
};

#define QK_CUDA(expr)                                                \
  do {                                                               \
    cudaError_t _e = (expr);                                         \
    if (_e != cudaSuccess) throw CudaFail{_e, #expr};               \
  } while (0)

// The stream of the API call in progress on this thread: scratch growth (cudaFree /
// cudaMalloc) is not allowed while it is being captured into a CUDA graph.
thread_local cudaStream_t t_call_stream = nullptr;

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* ensure(size_t bytes) {
    if (bytes <= cap) return p;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(t_call_stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
      throw std::invalid_argument(
          "scratch memory would grow during CUDA graph capture: run one forward (or quik_ctx_reserve) at the "
          "largest token count before capturing");
    if (p) { QK_CUDA(cudaDeviceSynchronize()); QK_CUDA(cudaFree(p)); p = nullptr; cap = 0; }
    const size_t want = std::max<size_t>(bytes, 1 << 16);
    QK_CUDA(cudaMalloc(&p, want));
    cap = want;
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev_);
    if (prev_ != dev) cudaSetDevice(dev);
    dev_ = dev;
  }
  ~DeviceGuard() {
    if (prev_ != dev_) cudaSetDevice(prev_);
  }

 private:
  int prev_ = 0, dev_ = 0;
};

}  // namespace

constexpr int kMaxHostChunks = 32;

struct quik_ctx_s {
  int device = 0;
  int num_sms = 148;
  int* d_err = nullptr;
  DevBuf q8, scale, zero, xo16, acc, fp, xbase, xo32, wtmp, wo_ws, s4_out, s4_cnt, aux;
  // gated MLP block: the down projection's per-token min / max keys (kernels.h), kept at
  // their initial values between calls (the down K1 restores what it reads)
  DevBuf hstat;
  uint4* ensure_hstat(int64_t M, cudaStream_t st) {
    const size_t before = hstat.cap;
    void* p = hstat.ensure(static_cast<size_t>(M) * 16);
    if (hstat.cap != before) check_hstat(launch_hstat_init(static_cast<uint4*>(p), hstat.cap / 16, st));
    return static_cast<uint4*>(p);
  }
  static void check_hstat(cudaError_t e) {
    if (e != cudaSuccess) throw CudaFail{e, "hstat init"};
  }
  // per-weight-block arrival counters of the INT4 decode kernel (zero between calls)
  int* ensure_s4_counters(size_t n, cudaStream_t st) {
    const size_t before = s4_cnt.cap;
    void* p = s4_cnt.ensure(n * 4);
    if (s4_cnt.cap != before) QK_CUDA(cudaMemsetAsync(p, 0, s4_cnt.cap, st));
    return static_cast<int*>(p);
  }
  // host-buffer forward (quik_linear_forward_host): copy-in / copy-out streams and
  // per-chunk events, created on first use; device staging for x and y.
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_start = nullptr, ev_done = nullptr;
  cudaEvent_t ev_in[kMaxHostChunks] = {}, ev_out[kMaxHostChunks] = {};
  DevBuf xdev, ydev;
  // split-K workspace of the weight-streaming path: int32 [M][N], kept all-zero
  // between calls (the AccInit epilogue clears what it reads)
  DevBuf ws;
  int32_t* ensure_ws(size_t bytes, cudaStream_t st) {
    const size_t before = ws.cap;
    void* p = ws.ensure(bytes);
    if (ws.cap != before) QK_CUDA(cudaMemsetAsync(p, 0, ws.cap, st));
    return static_cast<int32_t*>(p);
  }
  // Scratch is shared by every call on this context: a call on a different stream than
  // the previous one waits for the previous call's last kernel (event), so forwards
  // issued on several streams through one context serialise instead of racing on the
  // codes / scales / decode workspace. Skipped while the stream is being captured
  // (a captured graph must be replayed on one stream per context).
  cudaEvent_t ev_last = nullptr;
  cudaStream_t last_stream = nullptr;
  bool have_last = false;
  bool begin_call(cudaStream_t st) {
    t_call_stream = st;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    QK_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone) return false;
    if (!ev_last) QK_CUDA(cudaEventCreateWithFlags(&ev_last, cudaEventDisableTiming));
    if (have_last && last_stream != st) QK_CUDA(cudaStreamWaitEvent(st, ev_last, 0));
    return true;
  }
  void end_call(cudaStream_t st, bool ordered) {
    if (!ordered) return;
    QK_CUDA(cudaEventRecord(ev_last, st));
    last_stream = st;
    have_last = true;
  }
  void ensure_pipeline() {
    if (s_in) return;
    QK_CUDA(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
    QK_CUDA(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    QK_CUDA(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
    QK_CUDA(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
    for (int i = 0; i < kMaxHostChunks; ++i) {
      QK_CUDA(cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming));
      QK_CUDA(cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming));
    }
  }
};

struct quik_layer_s {
  int device = 0;
  int64_t in_features = 0, out_features = 0, n_outlier = 0, kb = 0, kpad = 0, opad = 0;
  int bits = 4;
  int8_t* w8 = nullptr;      // [out][kpad] INT8 weights (8-bit dense layers; 4-bit dense in speed mode)
  int sparse = 0;            // 2:4 sparse GEMM operands below are in use
  int gated = 0;             // gated MLP layer: rows interleave up / gate (32-row blocks), output width N / 2
  int8_t* w_sp = nullptr;    // [out][kpad / 2]
  uint8_t* w4 = nullptr;     // [out][kpad / 2] INT4 weights of 4-bit dense layers, device nibble layout
                             // (INT4 mode: from create; speed mode: made for the decode regime)
  int int4_only = 0;         // QUIK_WEIGHTS_INT4: w4 is the only base-weight copy
  uint8_t* meta = nullptr;   // metadata planes (kernels.h GemmArgs)
  __half* wo16 = nullptr;    // [out][opad]
  __half* wo16_lo = nullptr; // [out][opad] f16(w_o - f16(w_o)): weight-only forward only, uploaded on its first call
  std::vector<__half> wo16_lo_host;  // host copy of wo16_lo until then (keeps it out of HBM for quik-mode layers)
  float* w_scale = nullptr;  // [out]
  float* wreduced = nullptr; // [out]
  float* bias = nullptr;     // [out] or null
  int32_t* base_src = nullptr;  // [kb]
  int32_t* out_src = nullptr;   // [n_outlier]
  uint8_t* lane_mask = nullptr;  // [round_up(in,16)] 0xFF = outlier column (null when n_outlier == 0)
  uint16_t* gather = nullptr;    // [kpad] base position -> source column; >= kb -> zero slot
  uint32_t* chunk_desc = nullptr;  // [kpad / 16] x uint4 hot-quantizer compaction descriptors
  uint16_t* gen_chunk = nullptr;   // [n_gen] chunks gathered per byte
  int n_gen = 0;
  // wide-row K1 slices (kernels.h QuantArgs::slice_desc), n_slice == 0: one CTA per row
  int32_t* slice_desc = nullptr;
  int n_slice = 0, slice_cols_max = 0, slice_chunks_max = 0, slice_code_bytes = 0;
  // [ceil(in / 32) + 1] words, bit f = input feature f is an outlier column (bits past
  // in_features set): the base-column mask a gated projection's epilogue reduces this
  // layer's K1 min / max over (quik_gated_mlp_forward)
  uint32_t* fmask = nullptr;
};

namespace {

template <typename F>
quik_status guarded(F&& f) {
  try {
    return f();
  } catch (const CudaFail& c) {
    return fail(QUIK_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(c.e) + " (" + c.what + ")");
  } catch (const std::bad_alloc&) {
    return fail(QUIK_ERR_CUDA, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(QUIK_ERR_INVALID_ARGUMENT, e.what());
  }
}

void check_launch(cudaError_t e, const char* what, const char* extra = nullptr) {
  if (e != cudaSuccess) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e) + (extra ? std::string(" (") + extra + ")" : "");
    throw CudaFail{e, what};
  }
}

int64_t packed_row_bytes(int64_t cols, int bits) { return bits == 4 ? (cols + 1) / 2 : cols; }

// Runs one API call's device work on `st` ordered after the context's previous call
// (quik_ctx_s::begin_call / end_call).
template <typename F>
quik_status on_stream(quik_ctx_t ctx, cudaStream_t st, F&& f) {
  const bool ordered = ctx->begin_call(st);
  const quik_status r = f();
  if (r == QUIK_OK) ctx->end_call(st, ordered);
  return r;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Wide rows: split each row of K1 over a cluster of CTAs (quantize.cu
// quantize_wide_kernel). Slice boundaries sit at output-chunk boundaries near c * K / C;
// a slice loads the columns from its first base column (rounded down to a 16-byte
// vector) to the next slice's start or its last base column (rounded up), whichever is
// later, so every column is loaded by some slice and neighbours overlap by < 8 columns.
// Outlier slots go to the slice whose [start, next start) holds their column.
// Used where one CTA per row cannot hold a row (K > 32768: OPT-66B fc2, Falcon-180B fc2);
// the per-row cluster exchange makes it slower than the one-CTA kernel below that
// (70B down 28672: 128 us in 2 slices vs 110 us). QUIK_K1_WIDE_MIN_K (default 32769) /
// QUIK_K1_SLICE_COLS (8192) tune it.
void build_k1_slices(quik_layer_s* L, const std::vector<int32_t>& base_src, const std::vector<int32_t>& out_src,
                     const std::vector<uint16_t>& gen, int64_t kr16) {
  static const int64_t min_k = [] {
    const char* e = getenv("QUIK_K1_WIDE_MIN_K");
    return e ? atoll(e) : 32769LL;
  }();
  static const int64_t slice_cols = [] {
    const char* e = getenv("QUIK_K1_SLICE_COLS");
    return e ? std::max(1024LL, atoll(e)) : 8192LL;
  }();
  const int64_t K = L->in_features, kb = L->kb, nch = L->kpad / 16;
  if (K < min_k || kb < 64 || K % 8) return;
  const int64_t nch_base = (kb + 15) / 16;  // chunks holding base positions
  int C = static_cast<int>(std::min<int64_t>(8, (K + slice_cols - 1) / slice_cols));
  if (C < 2) return;
  std::vector<int64_t> ch_lo;
  for (;; --C) {
    ch_lo.assign(1, 0);
    bool ok = true;
    for (int c = 1; c < C && ok; ++c) {
      const int64_t T = c * K / C;
      const int64_t pos = std::lower_bound(base_src.begin(), base_src.end(), static_cast<int32_t>(T)) - base_src.begin();
      const int64_t ch = pos / 16;
      ok = ch > ch_lo.back() && ch < nch_base;
      ch_lo.push_back(ch);
    }
    if (ok) break;
    if (C == 2) return;
  }
  ch_lo.push_back(nch);
  std::vector<int64_t> in_lo(C + 1);
  for (int c = 0; c < C; ++c) in_lo[c] = c == 0 ? 0 : (base_src[16 * ch_lo[c]] & ~int64_t{7});
  in_lo[C] = K;
  std::vector<int32_t> desc(static_cast<size_t>(8 * C));
  int64_t cols_max = 0, chunks_max = 0, code_bytes = 0;
  for (int c = 0; c < C; ++c) {
    const int64_t last_pos = std::min<int64_t>(16 * ch_lo[c + 1], kb) - 1;
    int64_t hi = c == C - 1 ? K : std::max(in_lo[c + 1], (static_cast<int64_t>(base_src[last_pos]) + 8) & ~int64_t{7});
    hi = std::min(hi, K);
    const int64_t n = hi - in_lo[c];
    auto first_out = [&](int64_t col) {
      return static_cast<int64_t>(std::lower_bound(out_src.begin(), out_src.end(), static_cast<int32_t>(col)) - out_src.begin());
    };
    const int64_t o_lo = c == 0 ? 0 : first_out(in_lo[c]);
    const int64_t o_hi = c == C - 1 ? L->opad : first_out(in_lo[c + 1]);
    auto first_gen = [&](int64_t ch) {
      return static_cast<int64_t>(std::lower_bound(gen.begin(), gen.end(), static_cast<uint16_t>(ch)) - gen.begin());
    };
    const int64_t g_lo = first_gen(ch_lo[c]), g_hi = c == C - 1 ? static_cast<int64_t>(gen.size()) : first_gen(ch_lo[c + 1]);
    int32_t* d = &desc[static_cast<size_t>(8 * c)];
    d[0] = static_cast<int32_t>(in_lo[c]);
    d[1] = static_cast<int32_t>(n);
    d[2] = static_cast<int32_t>(ch_lo[c]);
    d[3] = static_cast<int32_t>(ch_lo[c + 1]);
    d[4] = static_cast<int32_t>(o_lo);
    d[5] = static_cast<int32_t>(o_hi);
    d[6] = static_cast<int32_t>(g_lo);
    d[7] = static_cast<int32_t>(g_hi);
    cols_max = std::max(cols_max, n);
    chunks_max = std::max(chunks_max, ch_lo[c + 1] - ch_lo[c]);
    // window reads run up to 20 bytes past a chunk's source; the last slice also holds
    // the pad positions' zero codes at kr16
    code_bytes = std::max(code_bytes, std::max(n, c == C - 1 ? kr16 - in_lo[c] : 0) + 32);
  }
  QK_CUDA(cudaMalloc(&L->slice_desc, desc.size() * 4));
  QK_CUDA(cudaMemcpy(L->slice_desc, desc.data(), desc.size() * 4, cudaMemcpyHostToDevice));
  L->n_slice = C;
  L->slice_cols_max = static_cast<int>(cols_max);
  L->slice_chunks_max = static_cast<int>(chunks_max);
  L->slice_code_bytes = static_cast<int>(round_up(code_bytes, 128));
}

void set_slices(QuantArgs& q, const quik_layer_s* L) {
  q.slice_desc = L->slice_desc;
  q.n_slice = L->n_slice;
  q.slice_cols_max = L->slice_cols_max;
  q.slice_chunks_max = L->slice_chunks_max;
  q.slice_code_bytes = L->slice_code_bytes;
}

// Runs K1 into the context scratch (GEMM layout) for the hot path.
void run_k1(quik_ctx_t ctx, const quik_layer_s* L, const void* x, quik_dtype xdt, int64_t M, cudaStream_t st,
            uint4* pre_stat = nullptr, int64_t ldx = 0) {
  QuantArgs q{};
  q.x = x;
  q.x_is_f32 = xdt == QUIK_F32;
  q.M = M;
  q.K = L->in_features;
  q.ldx = ldx ? ldx : L->in_features;  // x row pitch (elements)
  q.lane_mask = L->lane_mask;
  q.gather = L->gather;
  q.chunk_desc = L->chunk_desc;
  q.gen_chunk = L->gen_chunk;
  q.n_gen = L->n_gen;
  set_slices(q, L);
  q.out_src = L->out_src;
  q.kb = L->kb;
  q.n_out = L->n_outlier;
  q.bits = L->bits;
  q.q8 = L->kpad ? static_cast<int8_t*>(ctx->q8.ensure(static_cast<size_t>(M * L->kpad))) : nullptr;
  q.kpad = L->kpad;
  q.scale = static_cast<float*>(ctx->scale.ensure(M * 4));
  q.zero = static_cast<float*>(ctx->zero.ensure(M * 4));
  q.xo16 = L->opad ? static_cast<__half*>(ctx->xo16.ensure(static_cast<size_t>(M * L->opad * 2))) : nullptr;
  q.opad = L->opad;
  q.err = ctx->d_err;
  q.pre_stat = pre_stat;
  check_launch(launch_quantize(q, st), "quantize kernel");
}

GemmArgs gemm_args(quik_ctx_t ctx, const quik_layer_s* L, int64_t M) {
  GemmArgs g{};
  g.w = L->w8;
  g.x = static_cast<const int8_t*>(ctx->q8.p);
  g.kpad = L->kpad;
  g.wo = L->wo16;
  g.xo = static_cast<const __half*>(ctx->xo16.p);
  g.opad = L->opad;
  g.M = M;
  g.N = L->out_features;
  g.gated = L->gated;
  g.w_scale = L->w_scale;
  g.wreduced = L->wreduced;
  g.bias = L->bias;
  g.a_scale = static_cast<const float*>(ctx->scale.p);
  g.a_zero = static_cast<const float*>(ctx->zero.p);
  g.half_range = static_cast<float>(1 << (L->bits - 1));
  g.sparse = L->sparse;
  g.w4 = L->int4_only ? L->w4 : nullptr;  // speed mode: the prefill GEMM reads the INT8 copy
  g.w_sp = L->w_sp;
  g.meta = L->meta;
  return g;
}

void run_gemm(quik_ctx_t ctx, const GemmArgs& g, cudaStream_t st) {
  const char* msg = nullptr;
  cudaError_t e = launch_quik_gemm(g, ctx->num_sms, st, &msg);
  check_launch(e, "quik gemm kernel", msg);
}

}  // namespace

extern "C" {

const char* quik_last_error(void) { return g_err.c_str(); }

const char* quik_status_string(quik_status s) {
  switch (s) {
    case QUIK_OK: return "ok";
    case QUIK_ERR_INVALID_ARGUMENT: return "invalid argument";
    case QUIK_ERR_OUT_OF_RANGE: return "out of range";
    case QUIK_ERR_NUMERICAL: return "numerical error";
    case QUIK_ERR_CUDA: return "cuda error";
    case QUIK_ERR_NCCL: return "nccl error";
    case QUIK_ERR_UNSUPPORTED: return "unsupported";
    case QUIK_ERR_FORMAT: return "format error";
  }
  return "unknown";
}

int quik_abi_version(void) { return QUIK_B200_ABI_VERSION; }

quik_status quik_set_probe_mode(int on) {
  g_probe_mode = on;
  return QUIK_OK;
}

quik_status quik_set_gemm_tile(int cta_group, int block_n) {
  if (cta_group == 0 && block_n == 0) {
    quikb200::gemm_tile_override = 0;
    return QUIK_OK;
  }
  const bool ok = (cta_group == 1 && (block_n == 32 || block_n == 64 || block_n == 128)) ||
                  (cta_group == 2 && (block_n == 128 || block_n == 192 || block_n == 256));
  if (!ok) return fail(QUIK_ERR_INVALID_ARGUMENT, "unsupported GEMM tile configuration");
  quikb200::gemm_tile_override = (cta_group << 16) | block_n;
  return QUIK_OK;
}

quik_status quik_set_int4_decode(int on) {
  quikb200::gemm_stream4_auto = on ? 1 : 0;
  return QUIK_OK;
}

quik_status quik_set_gemm_multicast(int on) {
  quikb200::gemm_multicast = on ? 1 : 0;
  return QUIK_OK;
}

int quik_linear_forward_launches(quik_variant v) {
  switch (v) {
    case QUIK_V1_UNFUSED: return 4;      // split, quantize, int gemm, epilogue + outlier gemm
    case QUIK_V2_FUSED_QUANT: return 3;  // fused quantize, int gemm, epilogue + outlier gemm
    default: return 2;                   // fused quantize, fused gemm+epilogue
  }
}

quik_status quik_ctx_create(int device, quik_ctx_t* out) {
  if (!out) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_ctx_create: null output");
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      return fail(QUIK_ERR_CUDA, "quik_ctx_create: no CUDA device visible (the B200 path has no CPU fallback)");
    if (device < 0 || device >= n) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_ctx_create: bad device index");
    cudaDeviceProp prop;
    QK_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      return fail(QUIK_ERR_CUDA, std::string("quik_ctx_create: device ") + prop.name +
                                     " is not sm_100 (kernels are built for sm_100a only)");
    DeviceGuard g(device);
    auto* c = new quik_ctx_s();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    QK_CUDA(cudaMalloc(&c->d_err, sizeof(int)));
    QK_CUDA(cudaMemset(c->d_err, 0, sizeof(int)));
    *out = c;
    return QUIK_OK;
  });
}

quik_status quik_ctx_destroy(quik_ctx_t ctx) {
  if (!ctx) return QUIK_OK;
  DeviceGuard g(ctx->device);
  cudaDeviceSynchronize();
  for (DevBuf* b : {&ctx->q8, &ctx->scale, &ctx->zero, &ctx->xo16, &ctx->acc, &ctx->fp, &ctx->xbase, &ctx->xo32,
                    &ctx->wtmp, &ctx->xdev, &ctx->ydev, &ctx->ws, &ctx->wo_ws, &ctx->s4_out, &ctx->s4_cnt, &ctx->aux,
                    &ctx->hstat})
    b->release();
  if (ctx->s_in) {
    cudaStreamDestroy(ctx->s_in);
    cudaStreamDestroy(ctx->s_out);
    cudaEventDestroy(ctx->ev_start);
    cudaEventDestroy(ctx->ev_done);
    for (int i = 0; i < kMaxHostChunks; ++i) {
      cudaEventDestroy(ctx->ev_in[i]);
      cudaEventDestroy(ctx->ev_out[i]);
    }
  }
  if (ctx->ev_last) cudaEventDestroy(ctx->ev_last);
  cudaFree(ctx->d_err);
  delete ctx;
  return QUIK_OK;
}

quik_status quik_ctx_sync(quik_ctx_t ctx, void* stream) {
  if (!ctx) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    QK_CUDA(cudaStreamSynchronize(as_stream(stream)));
    int flag = 0;
    QK_CUDA(cudaMemcpy(&flag, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) {
      QK_CUDA(cudaMemset(ctx->d_err, 0, sizeof(int)));
      return fail(QUIK_ERR_NUMERICAL, "activation quantization: non-finite input value");
    }
    return QUIK_OK;
  });
}

quik_status quik_layer_create(quik_ctx_t ctx, const quik_weights_desc* d, quik_layer_t* out) {
  if (!ctx || !d || !out) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_layer_create: null argument");
  if (d->bits != 4 && d->bits != 8) return fail(QUIK_ERR_INVALID_ARGUMENT, "weight bits must be 4 or 8");
  if (d->act_bits != 4 && d->act_bits != 8) return fail(QUIK_ERR_INVALID_ARGUMENT, "activation bits must be 4 or 8");
  if (d->act_bits != d->bits)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "layer: activation bits must match weight bits in quik mode");
  if (d->in_features < 0 || d->out_features < 0 || d->n_outlier < 0 || d->n_outlier > d->in_features)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "layer: bad feature counts");
  if (d->n_outlier > 0 && !d->outlier_indices)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "layer: outlier indices missing");
  for (int64_t i = 0; i < d->n_outlier; ++i) {
    const int64_t v = d->outlier_indices[i];
    if (v < 0 || v >= d->in_features)
      return fail(QUIK_ERR_INVALID_ARGUMENT, "OutlierSet: index " + std::to_string(v) + " outside feature range");
    if (i > 0 && v <= d->outlier_indices[i - 1])
      return fail(QUIK_ERR_INVALID_ARGUMENT, "OutlierSet: indices must be sorted and unique");
  }
  const int64_t rb = d->row_begin, re = (d->row_begin == 0 && d->row_end == 0) ? d->out_features : d->row_end;
  if (rb < 0 || re < rb || re > d->out_features) return fail(QUIK_ERR_INVALID_ARGUMENT, "layer: bad row shard");
  const int64_t kb = d->in_features - d->n_outlier;
  const int64_t rows = re - rb;
  if (rows > 0 && ((kb > 0 && !d->base) || !d->scales || !d->wreduced || (d->n_outlier > 0 && !d->outlier_weights)))
    return fail(QUIK_ERR_INVALID_ARGUMENT, "layer: missing weight arrays");
  if (rows > 0x7fffffffLL || kb > 0x7fffffffLL)
    return fail(QUIK_ERR_UNSUPPORTED, "layer: dimensions exceed 2^31");
  if (d->in_features > 65520) return fail(QUIK_ERR_UNSUPPORTED, "layer: in_features > 65520");
  if (d->weight_mode != QUIK_WEIGHTS_SPEED && d->weight_mode != QUIK_WEIGHTS_INT4)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "layer: unknown weight_mode");

  return guarded([&] {
    DeviceGuard g(ctx->device);
    auto* L = new quik_layer_s();
    std::unique_ptr<quik_layer_s> hold(L);
    L->device = ctx->device;
    L->in_features = d->in_features;
    L->out_features = rows;
    L->n_outlier = d->n_outlier;
    L->bits = d->bits;
    L->kb = kb;
    L->kpad = round_up(kb, d->sparsity ? 2 * kKBlockBytes : kKBlockBytes);
    L->opad = round_up(d->n_outlier, 64);

    // permutation tables (calibration.cpp:69-91): non-outliers ascending, outliers ascending
    std::vector<int32_t> base_src;
    base_src.reserve(kb);
    std::vector<char> is_out(static_cast<size_t>(d->in_features), 0);
    for (int64_t i = 0; i < d->n_outlier; ++i) is_out[d->outlier_indices[i]] = 1;
    for (int64_t f = 0; f < d->in_features; ++f)
      if (!is_out[f]) base_src.push_back(static_cast<int32_t>(f));
    std::vector<int32_t> out_src(d->outlier_indices, d->outlier_indices + d->n_outlier);
    const int64_t kr16 = round_up(d->in_features, 16);
    std::vector<uint8_t> lane_mask(static_cast<size_t>(kr16), 0);
    for (int64_t i = 0; i < d->n_outlier; ++i) lane_mask[d->outlier_indices[i]] = 0xFF;
    std::vector<uint16_t> gather(static_cast<size_t>(L->kpad), static_cast<uint16_t>(kr16));
    for (int64_t j = 0; j < kb; ++j) gather[j] = static_cast<uint16_t>(base_src[j]);
    {
      const int64_t nw = d->in_features / 32 + 1;
      std::vector<uint32_t> fm(static_cast<size_t>(nw), 0u);
      for (int64_t f = 0; f < nw * 32; ++f)
        if (f >= d->in_features || is_out[f]) fm[f >> 5] |= 1u << (f & 31);
      QK_CUDA(cudaMalloc(&L->fmask, nw * 4));
      QK_CUDA(cudaMemcpy(L->fmask, fm.data(), nw * 4, cudaMemcpyHostToDevice));
    }

    cudaStream_t st = nullptr;
    if (kb) {
      QK_CUDA(cudaMalloc(&L->base_src, kb * 4));
      QK_CUDA(cudaMemcpy(L->base_src, base_src.data(), kb * 4, cudaMemcpyHostToDevice));
    }
    if (d->n_outlier) {
      QK_CUDA(cudaMalloc(&L->out_src, d->n_outlier * 4));
      QK_CUDA(cudaMemcpy(L->out_src, out_src.data(), d->n_outlier * 4, cudaMemcpyHostToDevice));
      QK_CUDA(cudaMalloc(&L->lane_mask, kr16));
      QK_CUDA(cudaMemcpy(L->lane_mask, lane_mask.data(), kr16, cudaMemcpyHostToDevice));
    }
    if (L->kpad) {
      // compaction tables of the hot quantizer (also for outlier-free layers: identity).
      // Chunk c covers base positions 16c .. 16c+15; src[p] = code-row byte of position
      // p (pads past kb read the zero bytes at kr16 + q).
      const int64_t nch = L->kpad / 16;
      std::vector<uint32_t> desc(static_cast<size_t>(nch * 4), 0u);
      std::vector<uint16_t> gen;
      for (int64_t c = 0; c < nch; ++c) {
        int64_t src[16];
        for (int p = 0; p < 16; ++p) {
          const int64_t j = 16 * c + p;
          src[p] = j < kb ? gather[j] : kr16 + (j - std::max<int64_t>(kb, 16 * c));
        }
        int len1 = 1;
        while (len1 < 16 && src[len1] == src[0] + len1) ++len1;
        bool ok = true;
        for (int p = len1 + 1; p < 16; ++p) ok = ok && src[p] == src[len1] + (p - len1);
        uint32_t* dd = &desc[static_cast<size_t>(4 * c)];
        if (!ok) {
          dd[0] = 0xFFFFFFFFu;
          gen.push_back(static_cast<uint16_t>(c));
          continue;
        }
        const int64_t sa = src[0], sb = len1 < 16 ? src[len1] - len1 : src[0];
        dd[0] = static_cast<uint32_t>(sa & ~int64_t{3}) | ((0x3210u + 0x1111u * static_cast<uint32_t>(sa & 3)) << 16);
        dd[1] = static_cast<uint32_t>(sb & ~int64_t{3}) | ((0x3210u + 0x1111u * static_cast<uint32_t>(sb & 3)) << 16);
        uint32_t sel[4];
        for (int k = 0; k < 4; ++k) {
          sel[k] = 0;
          for (int b = 0; b < 4; ++b) sel[k] |= static_cast<uint32_t>(4 * k + b < len1 ? b : 4 + b) << (4 * b);
        }
        dd[2] = sel[0] | (sel[1] << 16);
        dd[3] = sel[2] | (sel[3] << 16);
      }
      L->n_gen = static_cast<int>(gen.size());
      QK_CUDA(cudaMalloc(&L->gather, L->kpad * 2));
      QK_CUDA(cudaMemcpy(L->gather, gather.data(), L->kpad * 2, cudaMemcpyHostToDevice));
      QK_CUDA(cudaMalloc(&L->chunk_desc, nch * 16));
      QK_CUDA(cudaMemcpy(L->chunk_desc, desc.data(), nch * 16, cudaMemcpyHostToDevice));
      QK_CUDA(cudaMalloc(&L->gen_chunk, std::max<size_t>(gen.size(), 1) * 2));
      if (!gen.empty()) QK_CUDA(cudaMemcpy(L->gen_chunk, gen.data(), gen.size() * 2, cudaMemcpyHostToDevice));
      build_k1_slices(L, base_src, out_src, gen, kr16);
    }
    if (rows > 0) {
      QK_CUDA(cudaMalloc(&L->w_scale, rows * 4));
      QK_CUDA(cudaMalloc(&L->wreduced, rows * 4));
      QK_CUDA(cudaMemcpy(L->w_scale, d->scales + rb, rows * 4, cudaMemcpyDefault));
      QK_CUDA(cudaMemcpy(L->wreduced, d->wreduced + rb, rows * 4, cudaMemcpyDefault));
      if (d->bias) {
        QK_CUDA(cudaMalloc(&L->bias, rows * 4));
        QK_CUDA(cudaMemcpy(L->bias, d->bias + rb, rows * 4, cudaMemcpyDefault));
      }
      if (kb) {
        // One device copy of the base weights: INT4 (device nibble layout, half the bytes
        // of INT8) for 4-bit layers, INT8 for 8-bit layers, the 2:4-compressed codes for
        // sparse layers. Staging buffers are released at the end of the call.
        const int64_t rbytes = packed_row_bytes(kb, d->bits);
        void* tmp = ctx->wtmp.ensure(static_cast<size_t>(rows * rbytes));
        QK_CUDA(cudaMemcpy(tmp, d->base + rb * rbytes, static_cast<size_t>(rows * rbytes), cudaMemcpyDefault));
        if (d->bits == 4 && !d->sparsity && d->weight_mode == QUIK_WEIGHTS_INT4) {
          QK_CUDA(cudaMalloc(&L->w4, static_cast<size_t>(rows * L->kpad / 2)));
          check_launch(launch_pack_w4_abi(static_cast<const uint8_t*>(tmp), rows, kb, L->w4, L->kpad, st),
                       "int4 weight pack");
          L->int4_only = 1;
        } else {
          QK_CUDA(cudaMalloc(&L->w8, static_cast<size_t>(rows * L->kpad)));
          check_launch(launch_unpack_to_gemm(static_cast<const uint8_t*>(tmp), rows, kb, d->bits, L->w8, L->kpad, st),
                       "weight unpack");
        }
        if (d->sparsity) {
          // 2:4 compression (tcgen05.mma.sp operands); stays dense if not compressible
          const int64_t npad = round_up(rows, kBlockM);
          QK_CUDA(cudaMalloc(&L->w_sp, static_cast<size_t>(rows * L->kpad / 2)));
          QK_CUDA(cudaMalloc(&L->meta, static_cast<size_t>(2 * (L->kpad / 256) * npad * 16)));
          int* d_bad = nullptr;
          QK_CUDA(cudaMalloc(&d_bad, sizeof(int)));
          QK_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
          check_launch(launch_compress_24(L->w8, rows, L->kpad, L->w_sp, L->meta, d_bad, st), "2:4 compression");
          int bad = 0;
          QK_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
          QK_CUDA(cudaStreamSynchronize(st));
          cudaFree(d_bad);
          if (bad) {
            cudaFree(L->w_sp);
            cudaFree(L->meta);
            L->w_sp = nullptr;
            L->meta = nullptr;
            if (d->bits == 4 && d->weight_mode == QUIK_WEIGHTS_INT4) {  // not 2:4: dense INT4 after all
              QK_CUDA(cudaMalloc(&L->w4, static_cast<size_t>(rows * L->kpad / 2)));
              check_launch(launch_pack_w4(L->w8, rows, L->kpad, L->w4, st), "int4 weight pack");
              QK_CUDA(cudaStreamSynchronize(st));
              QK_CUDA(cudaFree(L->w8));
              L->w8 = nullptr;
              L->int4_only = 1;
            }
          } else {
            L->sparse = 1;
            QK_CUDA(cudaFree(L->w8));
            L->w8 = nullptr;
          }
        }
      }
      if (d->n_outlier) {
        QK_CUDA(cudaMalloc(&L->wo16, static_cast<size_t>(rows * L->opad * 2)));
        void* tmp = ctx->fp.ensure(static_cast<size_t>(rows * d->n_outlier * 4));
        QK_CUDA(cudaMemcpy(tmp, d->outlier_weights + rb * d->n_outlier, static_cast<size_t>(rows * d->n_outlier * 4),
                           cudaMemcpyDefault));
        check_launch(launch_f32_to_f16_padded(static_cast<const float*>(tmp), rows, d->n_outlier, L->wo16, L->opad, st),
                     "outlier weight convert");
        // the weight-only forward's low f16 plane, computed here from the f32 weights and
        // parked in host memory (the quik-mode hot path never reads it)
        __half* lo = static_cast<__half*>(ctx->aux.ensure(static_cast<size_t>(rows * L->opad * 2)));
        check_launch(launch_f16_lo_padded(static_cast<const float*>(tmp), rows, d->n_outlier, lo, L->opad, st),
                     "outlier weight convert (lo)");
        L->wo16_lo_host.resize(static_cast<size_t>(rows * L->opad));
        QK_CUDA(cudaMemcpyAsync(L->wo16_lo_host.data(), lo, static_cast<size_t>(rows * L->opad * 2),
                                cudaMemcpyDeviceToHost, st));
      }
    }
    QK_CUDA(cudaStreamSynchronize(st));
    // the layer's device copy is complete: give the staging memory back (a cfg3 layer
    // would otherwise keep its 114 MB ABI copy + 29 MB f32 outliers in the context)
    ctx->wtmp.release();
    ctx->fp.release();
    ctx->aux.release();
    *out = hold.release();
    return QUIK_OK;
  });
}

quik_status quik_layer_create_gated(quik_ctx_t ctx, const quik_weights_desc* up, const quik_weights_desc* gate,
                                   quik_layer_t* out) {
  if (!ctx || !up || !gate || !out) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_layer_create_gated: null argument");
  if (up->in_features != gate->in_features || up->out_features != gate->out_features || up->bits != gate->bits ||
      up->act_bits != gate->act_bits || up->n_outlier != gate->n_outlier)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "gated MLP: up and gate layers differ in shape, bits or outlier count");
  for (int64_t i = 0; i < up->n_outlier; ++i)
    if (!up->outlier_indices || !gate->outlier_indices || up->outlier_indices[i] != gate->outlier_indices[i])
      return fail(QUIK_ERR_INVALID_ARGUMENT, "gated MLP: up and gate layers need the same outlier set (shared quantizer)");
  if ((up->bias == nullptr) != (gate->bias == nullptr))
    return fail(QUIK_ERR_INVALID_ARGUMENT, "gated MLP: bias on one projection only");
  const int64_t F = up->out_features;
  const int64_t rb = up->row_begin, re = (up->row_begin == 0 && up->row_end == 0) ? F : up->row_end;
  if (rb < 0 || re < rb || re > F || rb % 32 || (re - rb) % 32)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "gated MLP: feature count / shard must be a multiple of 32");
  if (up->sparsity != gate->sparsity) return fail(QUIK_ERR_INVALID_ARGUMENT, "gated MLP: mixed 2:4 sparsity");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    // interleave the two row sets in blocks of 32 (host copies; arrays may live on the device)
    const int64_t rows = re - rb, kb = up->in_features - up->n_outlier, O = up->n_outlier;
    const int64_t rbytes = packed_row_bytes(kb, up->bits);
    std::vector<uint8_t> base(static_cast<size_t>(2 * rows * rbytes));
    std::vector<float> sc(static_cast<size_t>(2 * rows)), wr(static_cast<size_t>(2 * rows)),
        ow(static_cast<size_t>(2 * rows * O)), bias(up->bias ? static_cast<size_t>(2 * rows) : 0);
    auto fetch = [&](void* dst, const void* src, size_t bytes) {
      if (bytes) QK_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault));
    };
    for (int64_t blk = 0; blk < rows / 32; ++blk)
      for (int which = 0; which < 2; ++which) {
        const quik_weights_desc* d = which ? gate : up;
        const int64_t src_row = rb + 32 * blk, dst_row = 64 * blk + 32 * which;
        fetch(base.data() + dst_row * rbytes, d->base + src_row * rbytes, static_cast<size_t>(32 * rbytes));
        fetch(sc.data() + dst_row, d->scales + src_row, 32 * 4);
        fetch(wr.data() + dst_row, d->wreduced + src_row, 32 * 4);
        if (O) fetch(ow.data() + dst_row * O, d->outlier_weights + src_row * O, static_cast<size_t>(32 * O * 4));
        if (d->bias) fetch(bias.data() + dst_row, d->bias + src_row, 32 * 4);
      }
    quik_weights_desc c = *up;
    c.out_features = 2 * rows;
    c.base = base.data();
    c.scales = sc.data();
    c.wreduced = wr.data();
    c.outlier_weights = O ? ow.data() : nullptr;
    c.bias = up->bias ? bias.data() : nullptr;
    c.row_begin = 0;
    c.row_end = 0;
    const quik_status st = quik_layer_create(ctx, &c, out);
    if (st == QUIK_OK) (*out)->gated = 1;
    return st;
  });
}

quik_status quik_layer_destroy(quik_layer_t L) {
  if (!L) return QUIK_OK;
  DeviceGuard g(L->device);
  cudaDeviceSynchronize();
  cudaFree(L->w8);
  cudaFree(L->w_sp);
  cudaFree(L->meta);
  cudaFree(L->w4);
  cudaFree(L->wo16);
  cudaFree(L->wo16_lo);
  cudaFree(L->w_scale);
  cudaFree(L->wreduced);
  cudaFree(L->bias);
  cudaFree(L->base_src);
  cudaFree(L->out_src);
  cudaFree(L->lane_mask);
  cudaFree(L->gather);
  cudaFree(L->chunk_desc);
  cudaFree(L->gen_chunk);
  cudaFree(L->slice_desc);
  cudaFree(L->fmask);
  delete L;
  return QUIK_OK;
}

int quik_layer_is_sparse(quik_layer_t L) { return L ? L->sparse : 0; }

quik_status quik_layer_info(quik_layer_t L, int64_t* in_f, int64_t* out_f, int64_t* n_out, int* bits) {
  if (!L) return fail(QUIK_ERR_INVALID_ARGUMENT, "null layer");
  if (in_f) *in_f = L->in_features;
  if (out_f) *out_f = L->gated ? L->out_features / 2 : L->out_features;
  if (n_out) *n_out = L->n_outlier;
  if (bits) *bits = L->bits;
  return QUIK_OK;
}

quik_status quik_quantize_activations_fused(quik_ctx_t ctx, quik_layer_t L, const void* x, quik_dtype xdt, int64_t M,
                                            uint8_t* packed, float* scale, float* zero, float* x_outlier,
                                            void* stream) {
  if (!ctx || !L) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context or layer");
  if (M < 0 || (M > 0 && !x)) return fail(QUIK_ERR_INVALID_ARGUMENT, "fused quantization: bad input");
  if (L->in_features * (xdt == QUIK_F32 ? 4 : 2) > 128 * 1024)
    return fail(QUIK_ERR_UNSUPPORTED, "fused quantization: row wider than 128 KiB (register-resident quantizer limit)");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    return on_stream(ctx, as_stream(stream), [&]() -> quik_status {
      QuantArgs q{};
      q.x = x;
      q.x_is_f32 = xdt == QUIK_F32;
      q.M = M;
      q.K = L->in_features;
      q.ldx = L->in_features;
      q.lane_mask = L->lane_mask;
      q.gather = L->gather;
      q.out_src = L->out_src;
      q.kb = L->kb;
      q.n_out = L->n_outlier;
      q.bits = L->bits;
      q.packed = packed;
      q.scale = scale ? scale : static_cast<float*>(ctx->scale.ensure(M * 4));
      q.zero = zero ? zero : static_cast<float*>(ctx->zero.ensure(M * 4));
      q.xo32 = x_outlier;
      q.err = ctx->d_err;
      check_launch(launch_quantize(q, as_stream(stream)), "quantize kernel");
      return QUIK_OK;
    });
  });
}

quik_status quik_quantize_activations_gemm(quik_ctx_t ctx, quik_layer_t L, const void* x, quik_dtype xdt, int64_t M,
                                           int8_t* codes, float* scale, float* zero, void* x_outlier16, void* stream) {
  if (!ctx || !L) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context or layer");
  if (M < 0 || (M > 0 && (!x || !scale || !zero || (L->kpad && !codes) || (L->opad && !x_outlier16))))
    return fail(QUIK_ERR_INVALID_ARGUMENT, "quantize (GEMM layout): bad arguments");
  if (L->in_features * (xdt == QUIK_F32 ? 4 : 2) > 128 * 1024)
    return fail(QUIK_ERR_UNSUPPORTED, "quantize: row wider than 128 KiB (register-resident quantizer limit)");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    return on_stream(ctx, as_stream(stream), [&]() -> quik_status {
      QuantArgs q{};
      q.x = x;
      q.x_is_f32 = xdt == QUIK_F32;
      q.M = M;
      q.K = L->in_features;
      q.ldx = L->in_features;
      q.lane_mask = L->lane_mask;
      q.gather = L->gather;
      q.chunk_desc = L->chunk_desc;
      q.gen_chunk = L->gen_chunk;
      q.n_gen = L->n_gen;
      set_slices(q, L);
      q.out_src = L->out_src;
      q.kb = L->kb;
      q.n_out = L->n_outlier;
      q.bits = L->bits;
      q.q8 = L->kpad ? codes : nullptr;
      q.kpad = L->kpad;
      q.scale = scale;
      q.zero = zero;
      q.xo16 = L->opad ? static_cast<__half*>(x_outlier16) : nullptr;
      q.opad = L->opad;
      q.err = ctx->d_err;
      check_launch(launch_quantize(q, as_stream(stream)), "quantize kernel");
      return QUIK_OK;
    });
  });
}

quik_status quik_quantize_activations(quik_ctx_t ctx, const void* x, quik_dtype xdt, int64_t M, int64_t K, int bits,
                                      uint8_t* packed, float* scale, float* zero, void* stream) {
  if (!ctx) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context");
  if (bits != 4 && bits != 8) return fail(QUIK_ERR_INVALID_ARGUMENT, "activation bits must be 4 or 8");
  if (M < 0 || K < 0 || (M > 0 && K > 0 && !x)) return fail(QUIK_ERR_INVALID_ARGUMENT, "quantize: bad input");
  if (K * (xdt == QUIK_F32 ? 4 : 2) > 128 * 1024)
    return fail(QUIK_ERR_UNSUPPORTED, "quantize: row wider than 128 KiB (register-resident quantizer limit)");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    return on_stream(ctx, as_stream(stream), [&]() -> quik_status {
      QuantArgs q{};
      q.x = x;
      q.x_is_f32 = xdt == QUIK_F32;
      q.M = M;
      q.K = K;
      q.ldx = K;
      q.kb = K;
      q.bits = bits;
      q.packed = packed;
      q.scale = scale ? scale : static_cast<float*>(ctx->scale.ensure(M * 4));
      q.zero = zero ? zero : static_cast<float*>(ctx->zero.ensure(M * 4));
      q.err = ctx->d_err;
      check_launch(launch_quantize(q, as_stream(stream)), "quantize kernel");
      return QUIK_OK;
    });
  });
}

quik_status quik_int_matmul(quik_ctx_t ctx, const uint8_t* xp, int64_t xr, int64_t xc, int xb, const uint8_t* wp,
                            int64_t wr, int64_t wc, int wb, int32_t* out, void* stream) {
  if (!ctx) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context");
  if (xb != wb)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "int_matmul: operand bit widths differ (" + std::to_string(xb) + " vs " +
                                               std::to_string(wb) + ")");
  if (xb != 4 && xb != 8) return fail(QUIK_ERR_INVALID_ARGUMENT, "int_matmul: bits must be 4 or 8");
  if (xc != wc)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "int_matmul: inner dimensions differ (" + std::to_string(xc) + " vs " +
                                               std::to_string(wc) + ")");
  const int64_t half = int64_t{1} << (xb - 1);
  if (xc > (int64_t{1} << 31) / (half * half))
    return fail(QUIK_ERR_INVALID_ARGUMENT, "int_matmul: inner dimension risks INT32 accumulator overflow");
  if (xr < 0 || wr < 0 || xc < 0) return fail(QUIK_ERR_INVALID_ARGUMENT, "int_matmul: negative dimension");
  if (xr > 0x7fffffffLL || wr > 0x7fffffffLL) return fail(QUIK_ERR_UNSUPPORTED, "int_matmul: dimension exceeds 2^31");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    return on_stream(ctx, as_stream(stream), [&]() -> quik_status {
      cudaStream_t st = as_stream(stream);
      if (xr == 0 || wr == 0) return QUIK_OK;
      if (xc == 0) {
        QK_CUDA(cudaMemsetAsync(out, 0, static_cast<size_t>(xr * wr * 4), st));
        return QUIK_OK;
      }
      const int64_t kpad = round_up(xc, kKBlockBytes);
      int8_t* x8 = static_cast<int8_t*>(ctx->q8.ensure(static_cast<size_t>(xr * kpad)));
      int8_t* w8 = static_cast<int8_t*>(ctx->wtmp.ensure(static_cast<size_t>(wr * kpad)));
      check_launch(launch_unpack_to_gemm(xp, xr, xc, xb, x8, kpad, st), "unpack x");
      check_launch(launch_unpack_to_gemm(wp, wr, wc, wb, w8, kpad, st), "unpack w");
      GemmArgs gm{};
      gm.w = w8;
      gm.x = x8;
      gm.kpad = kpad;
      gm.M = xr;
      gm.N = wr;
      gm.out = out;
      gm.ldo = wr;
      gm.mode = kModeInt32;
      run_gemm(ctx, gm, st);
      return QUIK_OK;
    });
  });
}

quik_status quik_dequantize_epilogue(quik_ctx_t ctx, const int32_t* acc, int64_t M, int64_t N, const float* sa,
                                     const float* za, int half_range, const float* sw, const float* wr, float* out,
                                     void* stream) {
  if (!ctx) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context");
  if (M < 0 || N < 0) return fail(QUIK_ERR_INVALID_ARGUMENT, "dequantize_epilogue: negative dimension");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    check_launch(launch_dequant(acc, M, N, sa, za, static_cast<float>(half_range), sw, wr, out, as_stream(stream)),
                 "dequant kernel");
    return QUIK_OK;
  });
}

}  // extern "C"

namespace {
// Speed mode: the INT4 copy of a 4-bit dense layer for the decode kernel, made on the
// first M <= 32 forward (not under stream capture: quik_ctx_reserve makes it ahead).
bool ensure_w4(quik_layer_s* L, cudaStream_t st) {
  if (L->w4) return true;
  if (L->bits != 4 || !L->w8 || L->sparse) return false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  QK_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone) return false;
  const int64_t rows = L->out_features;  // all rows (gated: up + gate)
  QK_CUDA(cudaMalloc(&L->w4, static_cast<size_t>(rows * L->kpad / 2)));
  check_launch(launch_pack_w4(L->w8, rows, L->kpad, L->w4, st), "int4 weight pack");
  return true;
}

// Events recorded at the stage boundaries of one forward (StageTimes, runtime.hpp:72-80);
// any may be null.
struct StageMarks {
  cudaEvent_t after_split = nullptr, after_quant = nullptr, after_int = nullptr;
};
void mark(cudaEvent_t e, cudaStream_t st) {
  if (e) QK_CUDA(cudaEventRecord(e, st));
}

// Gated MLP block link (quik_gated_mlp_forward): the gated projection's GEMM epilogue
// emits the down projection's per-token min / max keys (emit: hmask = the down layer's
// outlier mask; *emitted = whether the fused GEMM ran, i.e. the keys are complete), the
// down projection's K1 consumes them (consume).
struct MlpLink {
  uint4* hstat = nullptr;
  const uint32_t* hmask = nullptr;
  bool* emitted = nullptr;
  bool consume = false;
  int64_t ldx = 0;  // input row pitch (0: in_features), V3 / decode paths
};

quik_status forward_impl(quik_ctx_t ctx, quik_layer_t L, const void* x, quik_dtype xdt, int64_t M, void* y,
                         quik_dtype ydt, int64_t ldy, quik_variant variant, cudaStream_t st, const StageMarks& sm,
                         void* const* peers = nullptr, int n_peer = 0, const MlpLink& link = MlpLink{}) {
  uint4* const pre = link.consume ? link.hstat : nullptr;
  if (M == 0 || L->out_features == 0) return QUIK_OK;
  const int64_t N = L->out_features;
  // Decode regime (M <= 16, or M <= 32 for layers of >= 128 M weights, dense layers):
  // the weight-streaming kernel (stream4.cu) spreads small layers over every SM (4-bit:
  // INT4 weights widened into TMEM; 8-bit: INT8 tiles); default on (QUIK_STREAM4=0
  // disables). At 17-32 tokens the fused kernel (on the INT4 copy, QUIK_W4_MID_M) is as
  // fast or faster except for the largest layers (M = 32: cfg1 4096^2 12.7 us fused vs
  // 13.1 decode, 7B up 13.5 vs 15.9, 70B up 38.6 vs 38.7, OPT-66B fc1 44.2 vs 37.2).
  const bool decode_m = M <= 16 || (M <= 32 && N * L->kpad >= (int64_t{128} << 20));
  bool decode = variant == QUIK_V3_FUSED_EPILOGUE && decode_m && L->kpad && !L->sparse && !g_probe_mode &&
                quikb200::gemm_stream4_auto;
  if (decode && L->bits == 4) decode = ensure_w4(L, st);
  if (decode) {
    // under stream capture no workspace may be (re)allocated: use the fused path when
    // the decode workspace / counters are not sized yet (a warm-up call sizes them)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    QK_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone &&
        (ctx->ws.cap < static_cast<size_t>(M * N * 4) || ctx->s4_cnt.cap < quikb200::stream4_counter_count(N) * 4))
      decode = false;
  }
  if (decode) {
    // decode regime: K1 -> one kernel for the INT4 split-K GEMM and the fused epilogue
    // (dequant + outlier MMAs, stream4.cu); workspace / counters stay zeroed between calls
    run_k1(ctx, L, x, xdt, M, st, pre, link.ldx);
    mark(sm.after_quant, st);
    Stream4Args a{};
    a.w4 = L->bits == 4 ? L->w4 : nullptr;
    a.w8 = L->w8;
    a.x = static_cast<const int8_t*>(ctx->q8.p);
    a.kpad = L->kpad;
    a.M = M;
    a.N = N;
    a.wo = L->wo16;
    a.xo = static_cast<const __half*>(ctx->xo16.p);
    a.opad = L->opad;
    a.a_scale = static_cast<const float*>(ctx->scale.p);
    a.a_zero = static_cast<const float*>(ctx->zero.p);
    a.w_scale = L->w_scale;
    a.wreduced = L->wreduced;
    a.bias = L->bias;
    a.half_range = static_cast<float>(1 << (L->bits - 1));
    a.acc = ctx->ensure_ws(static_cast<size_t>(M * N * 4), st);
    a.counters = ctx->ensure_s4_counters(quikb200::stream4_counter_count(N), st);
    a.out = y;
    a.ldo = ldy;
    a.out_f16 = ydt == QUIK_F16;
    a.gated = L->gated;
    a.peer_out = peers;
    a.n_peer = n_peer;
    const char* msg = nullptr;
    check_launch(launch_stream4(a, ctx->num_sms, st, &msg), "int4 stream kernel", msg);
    return QUIK_OK;
  }
  if (variant == QUIK_V3_FUSED_EPILOGUE) {
    // speed mode, mid token counts: the GEMM streams the weights more than it computes,
    // so it reads the INT4 copy (half the bytes; the decode regime makes it anyway):
    // OPT-66B fc1 M = 64 61.9 -> 46.2 us, M = 128 66.5 -> 54.8 us; from M = 256 the
    // INT8 copy is faster again (84 vs 127 us). QUIK_W4_MID_M sets the bound (0: off).
    static const int64_t w4_mid_m = [] {
      const char* e = getenv("QUIK_W4_MID_M");
      return e ? atoll(e) : 128LL;
    }();
    const bool mid_w4 = !L->int4_only && L->bits == 4 && !L->sparse && !g_probe_mode && M <= w4_mid_m &&
                        ensure_w4(L, st);
    run_k1(ctx, L, x, xdt, M, st, pre, link.ldx);
    mark(sm.after_quant, st);
    GemmArgs gm = gemm_args(ctx, L, M);
    if (mid_w4) gm.w4 = L->w4;
    if (link.hmask && L->gated && !L->sparse && ydt == QUIK_F16 && !g_probe_mode &&
        (reinterpret_cast<uintptr_t>(y) & 15) == 0 && (ldy * 2) % 16 == 0) {  // TMA-store tiles
      gm.hstat = link.hstat;
      gm.hmask = link.hmask;
      gm.herr = ctx->d_err;
      if (link.emitted) *link.emitted = true;
    }
    gm.out = y;
    gm.ldo = ldy;
    gm.mode = ydt == QUIK_F16 ? kModeF16 : kModeF32;
    if (g_probe_mode) gm.mode = kModeProbe;
    gm.peer_out = peers;
    gm.n_peer = n_peer;
    run_gemm(ctx, gm, st);
    return QUIK_OK;
  }
  if (variant == QUIK_V1_UNFUSED) {
    // split (runtime.cpp:169-186) then unfused quantisation of the base matrix (:188-197):
    // the split is K1 in "copy" form writing f32 base/outlier columns, then K1 again
    // over the base matrix with the identity permutation.
    float* xb32 = static_cast<float*>(ctx->xbase.ensure(static_cast<size_t>(M * std::max<int64_t>(L->kb, 1) * 4)));
    // split pass: gather base columns in permutation order as f32 (exact) and the
    // outliers as f16 GEMM operands.
    SplitArgs s{};
    s.x = x;
    s.x_is_f32 = xdt == QUIK_F32;
    s.M = M;
    s.K = L->in_features;
    s.ldx = L->in_features;
    s.base_src = L->base_src;
    s.kb = L->kb;
    s.out_src = L->out_src;
    s.n_out = L->n_outlier;
    s.xbase = xb32;
    s.xo16 = L->opad ? static_cast<__half*>(ctx->xo16.ensure(static_cast<size_t>(M * L->opad * 2))) : nullptr;
    s.opad = L->opad;
    check_launch(launch_split(s, st), "split kernel");
    mark(sm.after_split, st);
    QuantArgs q{};
    q.x = xb32;
    q.x_is_f32 = 1;
    q.M = M;
    q.K = L->kb;
    q.ldx = L->kb;
    q.kb = L->kb;
    q.bits = L->bits;
    q.q8 = L->kpad ? static_cast<int8_t*>(ctx->q8.ensure(static_cast<size_t>(M * L->kpad))) : nullptr;
    q.kpad = L->kpad;
    q.scale = static_cast<float*>(ctx->scale.ensure(M * 4));
    q.zero = static_cast<float*>(ctx->zero.ensure(M * 4));
    q.err = ctx->d_err;
    check_launch(launch_quantize(q, st), "quantize kernel");
  } else {
    run_k1(ctx, L, x, xdt, M, st, pre, link.ldx);
  }
  mark(sm.after_quant, st);
  // V1/V2 tail: the int32 accumulator through global memory, then the same
  // epilogue + outlier MMAs as V3 reading it back (bit-identical to V3).
  int32_t* acc = static_cast<int32_t*>(ctx->acc.ensure(static_cast<size_t>(M * N * 4)));
  GemmArgs gi = gemm_args(ctx, L, M);
  gi.out = acc;
  gi.ldo = N;
  gi.mode = kModeInt32;
  if (L->kpad) run_gemm(ctx, gi, st);
  else QK_CUDA(cudaMemsetAsync(acc, 0, static_cast<size_t>(M * N * 4), st));
  mark(sm.after_int, st);
  GemmArgs go = gemm_args(ctx, L, M);
  go.acc_in = acc;
  go.ld_acc = N;
  go.out = y;
  go.ldo = ldy;
  go.mode = ydt == QUIK_F16 ? kModeAccInitF16 : kModeAccInitF32;
  run_gemm(ctx, go, st);
  return QUIK_OK;
}
}  // namespace

extern "C" {

quik_status quik_linear_forward_ex(quik_ctx_t ctx, quik_layer_t L, const void* x, quik_dtype xdt, int64_t M,
                                   void* y, quik_dtype ydt, int64_t ldy, quik_variant variant, void* stream,
                                   void* mid_event) {
  if (!ctx || !L) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context or layer");
  if (M < 0) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: negative token count");
  if (M > 0 && (!x || !y)) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: null input or output");
  if (M > 0x7fffffffLL) return fail(QUIK_ERR_UNSUPPORTED, "quik_matmul: token count exceeds 2^31");
  if (ldy < (L->gated ? L->out_features / 2 : L->out_features))
    return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: output pitch < out_features");
  if (L->in_features * (xdt == QUIK_F32 ? 4 : 2) > 128 * 1024)
    return fail(QUIK_ERR_UNSUPPORTED, "quik_matmul: row wider than 128 KiB (register-resident quantizer limit)");
  if (ctx->device != L->device) return fail(QUIK_ERR_INVALID_ARGUMENT, "context and layer live on different devices");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    StageMarks sm;
    sm.after_quant = reinterpret_cast<cudaEvent_t>(mid_event);
    return on_stream(ctx, as_stream(stream),
                     [&] { return forward_impl(ctx, L, x, xdt, M, y, ydt, ldy, variant, as_stream(stream), sm); });
  });
}

quik_status quik_gated_mlp_forward(quik_ctx_t ctx, quik_layer_t gated, quik_layer_t down, const void* x,
                                   quik_dtype xdt, int64_t M, void* h, int64_t ldh, void* y, quik_dtype ydt,
                                   int64_t ldy, void* stream) {
  if (!ctx || !gated || !down) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context or layer");
  if (!gated->gated) return fail(QUIK_ERR_INVALID_ARGUMENT, "gated MLP: first layer is not a gated projection");
  const int64_t F = gated->out_features / 2;
  if (down->in_features != F)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "gated MLP: down projection input != up/gate output features");
  if (down->gated) return fail(QUIK_ERR_INVALID_ARGUMENT, "gated MLP: down projection is gated");
  if (M < 0) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: negative token count");
  if (M > 0 && (!x || !h || !y)) return fail(QUIK_ERR_INVALID_ARGUMENT, "gated MLP: null input, hidden or output");
  if (M > 0x7fffffffLL) return fail(QUIK_ERR_UNSUPPORTED, "quik_matmul: token count exceeds 2^31");
  if (ldh < F) return fail(QUIK_ERR_INVALID_ARGUMENT, "gated MLP: hidden pitch < hidden features");
  if (ldy < down->out_features) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: output pitch < out_features");
  if (gated->in_features * (xdt == QUIK_F32 ? 4 : 2) > 128 * 1024 || F * 2 > 128 * 1024)
    return fail(QUIK_ERR_UNSUPPORTED, "quik_matmul: row wider than 128 KiB (register-resident quantizer limit)");
  if (ctx->device != gated->device || ctx->device != down->device)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "context and layers live on different devices");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    cudaStream_t st = as_stream(stream);
    return on_stream(ctx, st, [&] {
      if (M == 0) return QUIK_OK;
      static const int fuse_env = [] {  // QUIK_MLP_FUSE=0: no statistics link (two plain forwards)
        const char* e = getenv("QUIK_MLP_FUSE");
        return e ? atoi(e) : 1;
      }();
      MlpLink up_link, down_link;
      bool emitted = false;
      if (fuse_env && down->kpad) {
        up_link.hstat = ctx->ensure_hstat(M, st);
        up_link.hmask = down->fmask;
        up_link.emitted = &emitted;
      }
      StageMarks none;
      quik_status s1 = forward_impl(ctx, gated, x, xdt, M, h, QUIK_F16, ldh, QUIK_V3_FUSED_EPILOGUE, st, none, nullptr,
                                    0, up_link);
      if (s1 != QUIK_OK) return s1;
      if (emitted) {
        down_link.hstat = up_link.hstat;
        down_link.consume = true;
      }
      down_link.ldx = ldh;
      try {
        return forward_impl(ctx, down, h, QUIK_F16, M, y, ydt, ldy, QUIK_V3_FUSED_EPILOGUE, st, none, nullptr, 0,
                            down_link);
      } catch (...) {
        // the keys the gated epilogue posted were not consumed: restore them
        if (emitted) launch_hstat_init(up_link.hstat, M, st);
        throw;
      }
    });
  });
}

quik_status quik_linear_forward_strided(quik_ctx_t ctx, quik_layer_t L, const void* x, quik_dtype xdt, int64_t M,
                                        void* y, quik_dtype ydt, int64_t ldy, quik_variant variant, void* stream) {
  return quik_linear_forward_ex(ctx, L, x, xdt, M, y, ydt, ldy, variant, stream, nullptr);
}

quik_status quik_gptq_quantize(quik_ctx_t ctx, const float* w, int64_t N, int64_t K, const double* hessian_sum,
                               double damping_frac, const int64_t* outlier_indices, int64_t n_outlier, int bits,
                               int use_clipping, int sparse, uint8_t* base, float* scales, float* wreduced,
                               float* outlier_weights, uint8_t* mask) {
  if (!ctx) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context");
  if (N > 0 && (!w || !hessian_sum || !base || !scales || !wreduced || (n_outlier && !outlier_weights) ||
                (n_outlier && !outlier_indices) || (sparse && !mask)))
    return fail(QUIK_ERR_INVALID_ARGUMENT, "gptq: null argument");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    GptqArgs a{};
    a.w = w;
    a.N = N;
    a.K = K;
    a.hessian_sum = hessian_sum;
    a.damping = damping_frac;
    a.outlier_idx = outlier_indices;
    a.n_out = n_outlier;
    a.bits = bits;
    a.use_clipping = use_clipping;
    a.sparse = sparse;
    a.base = base;
    a.scales = scales;
    a.wreduced = wreduced;
    a.outlier_weights = outlier_weights;
    a.mask = mask;
    std::string msg;
    const int st = quikb200::gptq_quantize_device(a, &msg);
    if (st == 1) return fail(QUIK_ERR_INVALID_ARGUMENT, msg);
    if (st == 3) return fail(QUIK_ERR_NUMERICAL, msg);
    if (st != 0) return fail(QUIK_ERR_CUDA, msg);
    return QUIK_OK;
  });
}

quik_status quik_hessian_accumulate(quik_ctx_t ctx, const float* x, int64_t T, int64_t K, double* h_sum) {
  if (!ctx) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context");
  if (T < 0 || K < 0 || (T > 0 && K > 0 && (!x || !h_sum))) return fail(QUIK_ERR_INVALID_ARGUMENT, "hessian: bad argument");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    std::string msg;
    if (quikb200::hessian_accumulate_device(x, T, K, h_sum, &msg) != 0) return fail(QUIK_ERR_CUDA, msg);
    return QUIK_OK;
  });
}

quik_status quik_linear_forward_sharded(quik_ctx_t ctx, quik_layer_t L, const void* x, quik_dtype xdt, int64_t M,
                                        void* const* y_dst, int n_dst, int64_t ldy, int64_t col_offset, void* stream) {
  if (!ctx || !L) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context or layer");
  if (M < 0) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: negative token count");
  if (n_dst < 1 || n_dst > 1 + kMaxPeerOut) return fail(QUIK_ERR_INVALID_ARGUMENT, "sharded forward: 1..8 destinations");
  if (M > 0 && !x) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: null input");
  for (int i = 0; i < n_dst; ++i)
    if (M > 0 && !y_dst[i]) return fail(QUIK_ERR_INVALID_ARGUMENT, "sharded forward: null destination");
  const int64_t w = L->gated ? L->out_features / 2 : L->out_features;
  if (col_offset < 0 || col_offset + w > ldy)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "sharded forward: shard columns exceed the output pitch");
  if (((col_offset * 2) % 16) != 0 || ((ldy * 2) % 16) != 0)
    return fail(QUIK_ERR_UNSUPPORTED, "sharded forward: column offset and pitch must be multiples of 8 (f16 TMA store)");
  if (M > 0x7fffffffLL) return fail(QUIK_ERR_UNSUPPORTED, "quik_matmul: token count exceeds 2^31");
  if (L->in_features * (xdt == QUIK_F32 ? 4 : 2) > 128 * 1024)
    return fail(QUIK_ERR_UNSUPPORTED, "quik_matmul: row wider than 128 KiB (register-resident quantizer limit)");
  if (ctx->device != L->device) return fail(QUIK_ERR_INVALID_ARGUMENT, "context and layer live on different devices");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    void* peers[kMaxPeerOut] = {};
    for (int i = 1; i < n_dst; ++i) peers[i - 1] = static_cast<__half*>(y_dst[i]) + col_offset;
    return on_stream(ctx, as_stream(stream), [&] {
      return forward_impl(ctx, L, x, xdt, M, static_cast<__half*>(y_dst[0]) + col_offset, QUIK_F16, ldy,
                          QUIK_V3_FUSED_EPILOGUE, as_stream(stream), StageMarks{}, peers, n_dst - 1);
    });
  });
}

quik_status quik_linear_forward_weight_only(quik_ctx_t ctx, quik_layer_t L, const void* x, quik_dtype xdt,
                                            int64_t M, void* y, quik_dtype ydt, int64_t ldy, void* stream) {
  if (!ctx || !L) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context or layer");
  if (M < 0) return fail(QUIK_ERR_INVALID_ARGUMENT, "weight_only_forward: negative token count");
  if (M > 0 && (!x || !y)) return fail(QUIK_ERR_INVALID_ARGUMENT, "weight_only_forward: null input or output");
  if (M > 0x7fffffffLL) return fail(QUIK_ERR_UNSUPPORTED, "weight_only_forward: token count exceeds 2^31");
  if (L->gated) return fail(QUIK_ERR_UNSUPPORTED, "weight_only_forward: gated MLP layers run in quik mode only");
  if (ldy < L->out_features) return fail(QUIK_ERR_INVALID_ARGUMENT, "weight_only_forward: output pitch < out_features");
  if (L->sparse) return fail(QUIK_ERR_UNSUPPORTED, "weight_only_forward: 2:4-compressed layers run in quik mode only");
  if (ctx->device != L->device) return fail(QUIK_ERR_INVALID_ARGUMENT, "context and layer live on different devices");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    return on_stream(ctx, as_stream(stream), [&]() -> quik_status {
      cudaStream_t st = as_stream(stream);
      if (M == 0 || L->out_features == 0) return QUIK_OK;
      if (L->n_outlier && !L->wo16_lo) {  // first weight-only call: upload the low outlier plane
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        QK_CUDA(cudaStreamIsCapturing(st, &cs));
        if (cs != cudaStreamCaptureStatusNone)
          return fail(QUIK_ERR_INVALID_ARGUMENT, "weight_only_forward: run one call before capturing it in a graph");
        QK_CUDA(cudaMalloc(&L->wo16_lo, L->wo16_lo_host.size() * 2));
        QK_CUDA(cudaMemcpy(L->wo16_lo, L->wo16_lo_host.data(), L->wo16_lo_host.size() * 2, cudaMemcpyHostToDevice));
      }
      WoArgs a{};
      a.x = x;
      a.x_is_f32 = xdt == QUIK_F32;
      a.M = M;
      a.ldx = L->in_features;
      a.base_src = L->base_src;
      a.kb = L->kb;
      a.kpad = L->kpad;
      a.out_src = L->out_src;
      a.n_out = L->n_outlier;
      a.opad = L->opad;
      if (L->bits == 4 && !ensure_w4(L, st))
        return fail(QUIK_ERR_INVALID_ARGUMENT, "weight_only_forward: run one call before capturing it in a graph");
      a.w4 = L->bits == 4 ? L->w4 : nullptr;
      a.w8 = L->w8;
      a.wo = L->wo16;
      a.wo_lo = L->wo16_lo;
      a.scale = L->w_scale;
      a.bias = L->bias;
      a.N = L->out_features;
      a.y = y;
      a.y_is_f16 = ydt == QUIK_F16;
      a.ldy = ldy;
      size_t pb = 0, po = 0;
      const size_t wsb = wo_workspace_bytes(a, ctx->num_sms, &pb, &po);
      a.xb = static_cast<__half*>(ctx->xbase.ensure(std::max<size_t>(pb, 16)));
      a.xo = static_cast<__half*>(ctx->xo16.ensure(std::max<size_t>(po, 16)));
      a.ws = wsb ? static_cast<float*>(ctx->wo_ws.ensure(wsb)) : nullptr;
      const char* msg = nullptr;
      check_launch(launch_weight_only(a, ctx->num_sms, st, &msg), "weight-only kernel", msg);
      return QUIK_OK;
    });
  });
}

quik_status quik_linear_forward_host(quik_ctx_t ctx, quik_layer_t L, const void* x_host, quik_dtype xdt, int64_t M,
                                     void* y_host, quik_dtype ydt, int64_t chunk_tokens, void* stream) {
  if (!ctx || !L) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context or layer");
  if (M < 0) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: negative token count");
  if (M > 0 && (!x_host || !y_host)) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: null input or output");
  if (M > 0x7fffffffLL) return fail(QUIK_ERR_UNSUPPORTED, "quik_matmul: token count exceeds 2^31");
  if (chunk_tokens < 0) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: negative chunk size");
  if (L->in_features * (xdt == QUIK_F32 ? 4 : 2) > 128 * 1024)
    return fail(QUIK_ERR_UNSUPPORTED, "quik_matmul: row wider than 128 KiB (register-resident quantizer limit)");
  if (ctx->device != L->device) return fail(QUIK_ERR_INVALID_ARGUMENT, "context and layer live on different devices");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    return on_stream(ctx, as_stream(stream), [&]() -> quik_status {
      cudaStream_t st = as_stream(stream);
      const int64_t K = L->in_features, N = L->gated ? L->out_features / 2 : L->out_features;  // output width
      if (M == 0 || N == 0) return QUIK_OK;
      ctx->ensure_pipeline();
      const size_t xe = xdt == QUIK_F32 ? 4 : 2, ye = ydt == QUIK_F32 ? 4 : 2;
      // Chunking: copy-in of chunk c+1, the two kernels of chunk c and copy-out of
      // chunk c-1 run concurrently (PCIe is full duplex; the copies dominate). About
      // 16 chunks (pipeline fill / drain ~1/16 of the copies), each a multiple of 256 tokens.
      int64_t chunk = chunk_tokens;
      if (chunk == 0) chunk = std::max<int64_t>(256, round_up((M + 15) / 16, 256));
      if ((M + chunk - 1) / chunk > kMaxHostChunks) chunk = (M + kMaxHostChunks - 1) / kMaxHostChunks;
      const int64_t nchunks = (M + chunk - 1) / chunk;
      char* xd = static_cast<char*>(ctx->xdev.ensure(static_cast<size_t>(M * K) * xe));
      char* yd = static_cast<char*>(ctx->ydev.ensure(static_cast<size_t>(M * N) * ye));
      const char* xh = static_cast<const char*>(x_host);
      char* yh = static_cast<char*>(y_host);
      // everything already queued on `stream` (including an earlier call's use of the
      // staging buffers) happens before this call's copies
      QK_CUDA(cudaEventRecord(ctx->ev_start, st));
      QK_CUDA(cudaStreamWaitEvent(ctx->s_in, ctx->ev_start, 0));
      QK_CUDA(cudaStreamWaitEvent(ctx->s_out, ctx->ev_start, 0));
      for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t m0 = c * chunk, mc = std::min(chunk, M - m0);
        QK_CUDA(cudaMemcpyAsync(xd + m0 * K * xe, xh + m0 * K * xe, static_cast<size_t>(mc * K) * xe,
                                cudaMemcpyHostToDevice, ctx->s_in));
        QK_CUDA(cudaEventRecord(ctx->ev_in[c], ctx->s_in));
        QK_CUDA(cudaStreamWaitEvent(st, ctx->ev_in[c], 0));
        const quik_status s =
            forward_impl(ctx, L, xd + m0 * K * xe, xdt, mc, yd + m0 * N * ye, ydt, N, QUIK_V3_FUSED_EPILOGUE, st,
                         StageMarks{});
        if (s != QUIK_OK) return s;
        QK_CUDA(cudaEventRecord(ctx->ev_out[c], st));
        QK_CUDA(cudaStreamWaitEvent(ctx->s_out, ctx->ev_out[c], 0));
        QK_CUDA(cudaMemcpyAsync(yh + m0 * N * ye, yd + m0 * N * ye, static_cast<size_t>(mc * N) * ye,
                                cudaMemcpyDeviceToHost, ctx->s_out));
      }
      QK_CUDA(cudaEventRecord(ctx->ev_done, ctx->s_out));
      QK_CUDA(cudaStreamWaitEvent(st, ctx->ev_done, 0));
      return QUIK_OK;
    });
  });
}

quik_status quik_rtn_quantize_weights(quik_ctx_t ctx, const float* w, int64_t N, int64_t K,
                                      const int64_t* outlier_indices, int64_t n_outlier, int bits, int use_clipping,
                                      uint8_t* base, float* scales, float* wreduced, float* outlier_weights,
                                      void* stream) {
  if (!ctx) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context");
  if (bits != 4 && bits != 8) return fail(QUIK_ERR_INVALID_ARGUMENT, "weight bits must be 4 or 8");
  if (N < 0 || K < 0 || n_outlier < 0 || n_outlier > K)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "rtn_quantize_weights: bad dimensions");
  if (n_outlier > 0 && !outlier_indices) return fail(QUIK_ERR_INVALID_ARGUMENT, "outlier indices missing");
  for (int64_t i = 0; i < n_outlier; ++i) {
    const int64_t v = outlier_indices[i];
    if (v < 0 || v >= K)
      return fail(QUIK_ERR_INVALID_ARGUMENT, "OutlierSet: index " + std::to_string(v) + " outside feature range");
    if (i > 0 && v <= outlier_indices[i - 1])
      return fail(QUIK_ERR_INVALID_ARGUMENT, "OutlierSet: indices must be sorted and unique");
  }
  return guarded([&] {
    DeviceGuard g(ctx->device);
    return on_stream(ctx, as_stream(stream), [&]() -> quik_status {
      cudaStream_t st = as_stream(stream);
      const int64_t kb = K - n_outlier;
      std::vector<int32_t> tab(static_cast<size_t>(K));
      std::vector<char> is_out(static_cast<size_t>(K), 0);
      for (int64_t i = 0; i < n_outlier; ++i) is_out[outlier_indices[i]] = 1;
      int64_t p = 0;
      for (int64_t f = 0; f < K; ++f)
        if (!is_out[f]) tab[p++] = static_cast<int32_t>(f);
      for (int64_t i = 0; i < n_outlier; ++i) tab[p++] = static_cast<int32_t>(outlier_indices[i]);
      int32_t* dtab = static_cast<int32_t*>(ctx->xbase.ensure(static_cast<size_t>(std::max<int64_t>(K, 1) * 4)));
      if (K) QK_CUDA(cudaMemcpyAsync(dtab, tab.data(), K * 4, cudaMemcpyHostToDevice, st));
      float* clip = nullptr;
      if (use_clipping && kb > 0) {  // clip_search per row (quantizer.cpp:266-290, :355)
        clip = static_cast<float*>(ctx->aux.ensure(static_cast<size_t>(std::max<int64_t>(N, 1) * 4)));
        check_launch(launch_clip_search(w, N, K, dtab, kb, bits, clip, st), "clip search kernel");
      }
      check_launch(launch_rtn_weights(w, N, K, dtab, kb, dtab + kb, n_outlier, bits, base, scales, wreduced,
                                      outlier_weights, clip, st),
                   "rtn weight kernel");
      QK_CUDA(cudaStreamSynchronize(st));  // tab must outlive the copy
      return QUIK_OK;
    });
  });
}

namespace {
// cuMemGetAddressRange through the runtime's driver entry point (no -lcuda link)
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range_fn() {
  static AddrRangeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<AddrRangeFn>(f);
  }();
  return fn;
}
}  // namespace

quik_status quik_ipc_handle_get(quik_ctx_t ctx, const void* dev_ptr, quik_ipc_handle* out) {
  if (!ctx || !dev_ptr || !out) return fail(QUIK_ERR_INVALID_ARGUMENT, "ipc: null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    AddrRangeFn range = addr_range_fn();
    if (!range) return fail(QUIK_ERR_CUDA, "ipc: cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
      return fail(QUIK_ERR_INVALID_ARGUMENT, "ipc: pointer is not device memory");
    cudaIpcMemHandle_t h;
    QK_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    std::memcpy(out->bytes, &h, 64);
    out->offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
    return QUIK_OK;
  });
}

quik_status quik_ipc_handle_open(quik_ctx_t ctx, const quik_ipc_handle* handle, void** dev_ptr) {
  if (!ctx || !handle || !dev_ptr) return fail(QUIK_ERR_INVALID_ARGUMENT, "ipc: null argument");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle->bytes, 64);
    void* base = nullptr;
    QK_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr = static_cast<char*>(base) + handle->offset;
    return QUIK_OK;
  });
}

quik_status quik_ipc_handle_close(quik_ctx_t ctx, void* dev_ptr, const quik_ipc_handle* handle) {
  if (!ctx || !dev_ptr || !handle) return fail(QUIK_ERR_INVALID_ARGUMENT, "ipc: null argument");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    QK_CUDA(cudaIpcCloseMemHandle(static_cast<char*>(dev_ptr) - handle->offset));
    return QUIK_OK;
  });
}

int64_t quik_layer_device_bytes(quik_layer_t L) {
  if (!L) return -1;
  const int64_t rows = L->out_features, nch = L->kpad / 16;
  int64_t b = 0;
  if (L->w8) b += rows * L->kpad;
  if (L->w4) b += rows * L->kpad / 2;
  if (L->w_sp) b += rows * L->kpad / 2 + 2 * (L->kpad / 256) * round_up(rows, kBlockM) * 16;
  if (L->wo16) b += rows * L->opad * 2;
  if (L->wo16_lo) b += rows * L->opad * 2;
  b += rows * 4 * (2 + (L->bias ? 1 : 0));
  b += L->kb * 4 + L->n_outlier * 4 + (L->lane_mask ? round_up(L->in_features, 16) : 0);
  if (L->kpad) b += L->kpad * 2 + nch * 16 + std::max(L->n_gen, 1) * 2;
  return b;
}

quik_status quik_layer_layout(quik_layer_t L, int64_t* kpad, int64_t* opad) {
  if (!L) return fail(QUIK_ERR_INVALID_ARGUMENT, "null layer");
  if (kpad) *kpad = L->kpad;
  if (opad) *opad = L->opad;
  return QUIK_OK;
}

quik_status quik_ctx_clear_error(quik_ctx_t ctx, void* stream) {
  if (!ctx) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    QK_CUDA(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), as_stream(stream)));
    return QUIK_OK;
  });
}

quik_status quik_ctx_reserve(quik_ctx_t ctx, quik_layer_t L, int64_t M) {
  if (!ctx || !L) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context or layer");
  if (M < 0 || M > 0x7fffffffLL) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_ctx_reserve: bad token count");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    t_call_stream = nullptr;
    if (M == 0) return QUIK_OK;
    const int64_t N = L->out_features;
    if (L->kpad) ctx->q8.ensure(static_cast<size_t>(M * L->kpad));
    ctx->scale.ensure(M * 4);
    ctx->zero.ensure(M * 4);
    if (L->opad) ctx->xo16.ensure(static_cast<size_t>(M * L->opad * 2));
    if (L->gated) ctx->ensure_hstat(M, nullptr);  // quik_gated_mlp_forward statistics
    if (M <= 32 && L->kpad && !L->sparse) {  // decode kernel workspace + counters (zeroed)
      ctx->ensure_ws(static_cast<size_t>(M * N * 4), nullptr);
      ctx->ensure_s4_counters(quikb200::stream4_counter_count(N), nullptr);
      if (L->bits == 4) ensure_w4(L, nullptr);
    }
    QK_CUDA(cudaDeviceSynchronize());
    return QUIK_OK;
  });
}

quik_status quik_linear_forward_timed(quik_ctx_t ctx, quik_layer_t L, const void* x, quik_dtype xdt, int64_t M,
                                      void* y, quik_dtype ydt, int64_t ldy, quik_variant variant, void* stream,
                                      double* stage_ms, int* fused_flags) {
  if (!ctx || !L) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context or layer");
  if (M < 0) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: negative token count");
  if (M > 0 && (!x || !y)) return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: null input or output");
  if (M > 0x7fffffffLL) return fail(QUIK_ERR_UNSUPPORTED, "quik_matmul: token count exceeds 2^31");
  if (ldy < (L->gated ? L->out_features / 2 : L->out_features))
    return fail(QUIK_ERR_INVALID_ARGUMENT, "quik_matmul: output pitch < out_features");
  if (L->in_features * (xdt == QUIK_F32 ? 4 : 2) > 128 * 1024)
    return fail(QUIK_ERR_UNSUPPORTED, "quik_matmul: row wider than 128 KiB (register-resident quantizer limit)");
  if (ctx->device != L->device) return fail(QUIK_ERR_INVALID_ARGUMENT, "context and layer live on different devices");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    cudaStream_t st = as_stream(stream);
    cudaEvent_t ev[5] = {};
    for (auto& e : ev) QK_CUDA(cudaEventCreate(&e));
    struct Free {
      cudaEvent_t* e;
      ~Free() {
        for (int i = 0; i < 5; ++i) cudaEventDestroy(e[i]);
      }
    } free_ev{ev};
    StageMarks sm;
    const bool v1 = variant == QUIK_V1_UNFUSED, v3 = variant == QUIK_V3_FUSED_EPILOGUE;
    sm.after_split = v1 ? ev[1] : nullptr;
    sm.after_quant = ev[2];
    sm.after_int = v3 ? nullptr : ev[3];
    QK_CUDA(cudaEventRecord(ev[0], st));
    const quik_status r = on_stream(ctx, st, [&] { return forward_impl(ctx, L, x, xdt, M, y, ydt, ldy, variant, st, sm); });
    if (r != QUIK_OK) return r;
    QK_CUDA(cudaEventRecord(ev[4], st));
    QK_CUDA(cudaEventSynchronize(ev[4]));
    // StageTimes (runtime.hpp:72-80): a fused stage reports under the first field it covers
    // and flags itself fused. V3: K1 = split + quantize (quantize_ms, quantize_fused); the
    // fused GEMM = int matmul + outlier matmul + dequantize + add (int_matmul_ms,
    // dequantize_fused). V1 / V2: the int32 GEMM alone (int_matmul_ms), then one epilogue
    // kernel = outlier matmul + dequantize + add (fp_matmul_ms, dequantize_fused).
    double t[6] = {0, 0, 0, 0, 0, 0};
    float ms = 0.0f;
    if (M > 0 && L->out_features > 0) {
      cudaEvent_t prev = ev[0];
      if (v1) {
        QK_CUDA(cudaEventElapsedTime(&ms, prev, ev[1]));
        t[0] = ms;
        prev = ev[1];
      }
      QK_CUDA(cudaEventElapsedTime(&ms, prev, ev[2]));
      t[1] = ms;
      if (v3) {
        QK_CUDA(cudaEventElapsedTime(&ms, ev[2], ev[4]));
        t[2] = ms;
      } else {
        QK_CUDA(cudaEventElapsedTime(&ms, ev[2], ev[3]));
        t[2] = ms;
        QK_CUDA(cudaEventElapsedTime(&ms, ev[3], ev[4]));
        t[3] = ms;
      }
    }
    if (stage_ms)
      for (int i = 0; i < 6; ++i) stage_ms[i] = t[i];
    if (fused_flags) {
      fused_flags[0] = v1 ? 0 : 1;  // quantize_fused
      fused_flags[1] = 1;           // dequantize_fused
    }
    return QUIK_OK;
  });
}

quik_status quik_split_activations(quik_ctx_t ctx, quik_layer_t L, const void* x, quik_dtype xdt, int64_t M,
                                   float* x_base, float* x_outlier, void* stream) {
  if (!ctx || !L) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context or layer");
  if (M < 0 || (M > 0 && (!x || (L->kb && !x_base) || (L->n_outlier && !x_outlier))))
    return fail(QUIK_ERR_INVALID_ARGUMENT, "split_activations: bad arguments");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    return on_stream(ctx, as_stream(stream), [&]() -> quik_status {
      SplitArgs s{};
      s.x = x;
      s.x_is_f32 = xdt == QUIK_F32;
      s.M = M;
      s.K = L->in_features;
      s.ldx = L->in_features;
      s.base_src = L->base_src;
      s.kb = L->kb;
      s.out_src = L->out_src;
      s.n_out = L->n_outlier;
      s.xbase = x_base;
      s.xo32 = x_outlier;
      s.opad = L->n_outlier;
      check_launch(launch_split(s, as_stream(stream)), "split kernel");
      return QUIK_OK;
    });
  });
}

quik_status quik_unpack_values(quik_ctx_t ctx, const uint8_t* packed, int64_t rows, int64_t cols, int bits,
                               int8_t* out, void* stream) {
  if (!ctx) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context");
  if (bits != 4 && bits != 8) return fail(QUIK_ERR_INVALID_ARGUMENT, "unpack: bits must be 4 or 8");
  if (rows < 0 || cols < 0 || (rows > 0 && cols > 0 && (!packed || !out)))
    return fail(QUIK_ERR_INVALID_ARGUMENT, "unpack: bad arguments");
  if (rows > 0xffffLL * 0xffffLL) return fail(QUIK_ERR_UNSUPPORTED, "unpack: too many rows");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    check_launch(launch_unpack_to_gemm(packed, rows, cols, bits, out, cols, as_stream(stream)), "unpack kernel");
    return QUIK_OK;
  });
}

quik_status quik_compute_wreduced(quik_ctx_t ctx, const uint8_t* base, int64_t rows, int64_t cols, int bits,
                                  const float* scales, float* wreduced, void* stream) {
  if (!ctx) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context");
  if (bits != 4 && bits != 8) return fail(QUIK_ERR_INVALID_ARGUMENT, "weight bits must be 4 or 8");
  if (rows < 0 || cols < 0 || (rows > 0 && (!scales || !wreduced || (cols > 0 && !base))))
    return fail(QUIK_ERR_INVALID_ARGUMENT, "compute_wreduced: bad arguments");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    check_launch(launch_compute_wreduced(base, rows, cols, bits, scales, wreduced, as_stream(stream)),
                 "wreduced kernel");
    return QUIK_OK;
  });
}

quik_status quik_dequantize_weights(quik_ctx_t ctx, const uint8_t* base, int64_t rows, int64_t in_features, int bits,
                                    const float* scales, const float* outlier_weights, const int64_t* outlier_indices,
                                    int64_t n_outlier, float* out, void* stream) {
  if (!ctx) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context");
  if (bits != 4 && bits != 8) return fail(QUIK_ERR_INVALID_ARGUMENT, "weight bits must be 4 or 8");
  if (rows < 0 || in_features < 0 || n_outlier < 0 || n_outlier > in_features)
    return fail(QUIK_ERR_INVALID_ARGUMENT, "dequantize_weights: outlier set does not match weights");
  if (n_outlier > 0 && !outlier_indices) return fail(QUIK_ERR_INVALID_ARGUMENT, "outlier indices missing");
  for (int64_t i = 0; i < n_outlier; ++i) {
    const int64_t v = outlier_indices[i];
    if (v < 0 || v >= in_features || (i > 0 && v <= outlier_indices[i - 1]))
      return fail(QUIK_ERR_INVALID_ARGUMENT, "OutlierSet: indices must be sorted, unique and inside the feature range");
  }
  if (rows > 0xffffLL) return fail(QUIK_ERR_UNSUPPORTED, "dequantize_weights: more than 65535 rows per call");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    return on_stream(ctx, as_stream(stream), [&]() -> quik_status {
      cudaStream_t st = as_stream(stream);
      std::vector<int32_t> perm(static_cast<size_t>(in_features));
      std::vector<char> is_out(static_cast<size_t>(in_features), 0);
      for (int64_t i = 0; i < n_outlier; ++i) is_out[outlier_indices[i]] = 1;
      int64_t p = 0;
      for (int64_t f = 0; f < in_features; ++f)
        if (!is_out[f]) perm[p++] = static_cast<int32_t>(f);
      for (int64_t i = 0; i < n_outlier; ++i) perm[p++] = static_cast<int32_t>(outlier_indices[i]);
      int32_t* dperm = static_cast<int32_t*>(ctx->aux.ensure(static_cast<size_t>(std::max<int64_t>(in_features, 1) * 4)));
      if (in_features) QK_CUDA(cudaMemcpyAsync(dperm, perm.data(), in_features * 4, cudaMemcpyHostToDevice, st));
      check_launch(launch_dequantize_weights(base, rows, in_features, in_features - n_outlier, bits, scales, dperm,
                                             outlier_weights, out, st),
                   "dequantize weights kernel");
      QK_CUDA(cudaStreamSynchronize(st));  // perm must outlive the copy
      return QUIK_OK;
    });
  });
}

quik_status quik_elementwise(quik_ctx_t ctx, int op, const float* a, const float* b, float* out, int64_t n,
                             void* stream) {
  if (!ctx) return fail(QUIK_ERR_INVALID_ARGUMENT, "null context");
  if (op < 0 || op > 2) return fail(QUIK_ERR_INVALID_ARGUMENT, "elementwise: op must be silu (0), multiply (1), add (2)");
  if (n < 0 || (n > 0 && (!a || !out || (op > 0 && !b)))) return fail(QUIK_ERR_INVALID_ARGUMENT, "elementwise: bad arguments");
  return guarded([&] {
    DeviceGuard g(ctx->device);
    check_launch(launch_elementwise(op, a, b, out, n, as_stream(stream)), "elementwise kernel");
    return QUIK_OK;
  });
}

quik_status quik_linear_forward(quik_ctx_t ctx, quik_layer_t L, const void* x, quik_dtype xdt, int64_t M, void* y,
                                quik_dtype ydt, quik_variant variant, void* stream) {
  if (!L) return fail(QUIK_ERR_INVALID_ARGUMENT, "null layer");
  return quik_linear_forward_strided(ctx, L, x, xdt, M, y, ydt, L->gated ? L->out_features / 2 : L->out_features,
                                     variant, stream);
}

}  // extern "C"
