// WeightOnly forward (reference LayerMode::WeightOnly, weight_only_forward,
// runtime.cpp:115-136): activations stay floating point, the base
// weights stay INT4 / INT8 codes with a per-row scale:
//
//   y[t][n] = (bias[n] + sum_o x_o[t][o] w_o[n][o]) + sum_j x_b[t][j] (q[n][j] scale[n])
//
// the memory-bound decode regime. Every product is exact on the tensor
// cores: q (<= 8 bits) x f16 activation fits f32's mantissa; only the f32 summation
// order differs from the reference. f32 activations are split into two f16 "token
// planes" hi = f16(x), lo = f16(x - hi) (rows [0, M) and [M, 2M) of the B operand) and
// the outlier weights into hi/lo f16 planes, so f32 inputs keep ~2^-22 relative
// accuracy (the reference's own test bar is 1e-6 relative Frobenius vs f64).
//
// B200 design: the widened f16 weight tile never touches shared memory. The producer
// TMA-streams the packed INT4 (or INT8) weight tile into a shared-memory ring; eight
// widening warps (two per TMEM lane quadrant, alternating stages) read one weight row
// per thread, widen the codes to f16 with two integer ops + PRMT + one HSUB2 per pair
// (f16 bits 0x6400 | u == 1024 + u, u = q + 8), and write them with tcgen05.st into a
// TMEM A buffer; the MMA warp issues tcgen05.mma kind::f16 with A from TMEM (".ts":
// lane = weight row, column j = f16x2 {k = 2j, 2j+1}, pinned by tools/ts_probe.cu) and
// B (the f16 token tile) from shared memory. Shared-memory traffic per weight is the
// 0.5 B TMA write + 0.5 B read instead of 2 B write + 2 B MMA read for a widened
// shared-memory tile. The outlier columns are plain SS f16 MMAs (weights TMA-loaded as
// f16) into a second accumulator, so the epilogue can apply the per-row scale to the
// base sum only.
//
// Work units: (128-row weight block, token tile of BN plane rows, K split). With one
// split and f16 input the epilogue writes y directly; otherwise each unit writes its
// f32 partial to a workspace and a finalize kernel sums splits (and the hi/lo planes)
// in a fixed order (deterministic).
//
// Warp roles (512 threads, 1 CTA per SM, persistent): warp 0 TMA producer, warp 1
// outlier-MMA issuer + TMEM allocator, warps 2-9 widening (quadrant = warp % 4, group =
// (warp - 2) / 4 owns TMEM A buffer `group`), warps 10-13 epilogue, warps 14-15 base-MMA
// issuers (one per widening group).
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"

namespace quikb200 {

namespace {

constexpr int kWABytes = kBlockM * kKBlockBytes;  // 16 KB: packed weight tile or one f16 outlier tile
constexpr int kWTmemA = 128;                        // columns per TMEM A buffer (256 K as f16x2)

template <int BN>
struct WCfg {
  static constexpr int kBAtom = BN * kKBlockBytes;  // BN plane rows x 64 f16
  // G widening groups (each 4 warps, one TMEM A buffer of 128 columns, one issuing warp
  // and one base accumulator): 3 when the TMEM budget allows it (BN = 16)
  static constexpr int G = BN == 16 ? 3 : 2;
  // Three rings, each stage with exactly one consumer sequence (a consumer that skips
  // other consumers' items could otherwise run a whole ring cycle ahead and alias an
  // mbarrier phase):
  //  * weight tiles (16 KB, consumed by widening group bc % G, released as soon as the
  //    group has widened them: the MMAs read A from TMEM) - deep, it covers HBM latency;
  //  * token tiles of the base stages (L2-resident, consumed by base issuer bc % G);
  //  * outlier stages (f16 weight tile + token tile, consumed by warp 1).
  static constexpr int kSlotW = kWABytes;
  static constexpr int kSlotT = 4 * kBAtom;
  static constexpr int kSlotO = kWABytes + kBAtom;
  static constexpr int kStagesW = BN == 16 ? 9 : 6;
  static constexpr int kStagesT = BN == 16 ? 3 : 4;
  static constexpr int kStagesO = BN == 16 ? 3 : 2;
  static_assert(kStagesW % G == 0 && kStagesT % G == 0, "every base stage belongs to one group / issuer");
  static constexpr int kOffT = kStagesW * kSlotW, kOffO = kOffT + kStagesT * kSlotT;
  static constexpr int kRingBytes = kOffO + kStagesO * kSlotO;
  static constexpr int kBarBytes = (2 * (kStagesW + kStagesT + kStagesO) + 2 * G + 4) * 8 + 16;
  static constexpr int kSmemBytes = 1024 + kRingBytes + kBarBytes;
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
  static constexpr int kAccColG = G * kWTmemA;
  static constexpr int kAccBufG = (G + 1) * BN;  // G base accumulators + outliers, double-buffered
  static_assert(kAccColG + 2 * kAccBufG <= 512, "TMEM budget");
  // warps: 0 weight producer, 1 outlier issuer + TMEM allocator, 2 .. 4G+1 widening, 4
  // epilogue warps, G base issuers, 1 token / outlier producer
  static constexpr int kWidenEnd = 2 + 4 * G, kEpiEnd = kWidenEnd + 4, kIssEnd = kEpiEnd + G;
  static constexpr int kThreads = (kIssEnd + 1) * 32;
};

struct WParams {
  CUtensorMap tm_w;     // INT4 [N][kpad/2] or INT8 [N][kpad] bytes, box {128 B, 128}, SW128
  CUtensorMap tm_xb;    // f16 [R][kpad] as bytes, box {128 B, BN}, SW128
  CUtensorMap tm_wo;    // f16 [N][opad] as bytes, box {128 B, 128}, SW128
  CUtensorMap tm_wolo;  // f16 [N][opad] (lo plane)
  CUtensorMap tm_xo;    // f16 [R][opad] as bytes, box {128 B, BN}, SW128
  const float* scale;
  const float* bias;  // [N] or null
  void* out;          // mode 0: ws f32 [splits][R][N]; 1: y f32 [M][ldo]; 2: y f16 [M][ldo]
  int R, M, N, ldo;
  int nbase, nout;    // base stages (256 K INT4 / 128 K INT8) and outlier items (2 per 64 columns)
  int splits, tiles_t, w4, mode;
  long long* trace;  // diagnostics (QUIK_WO_TRACE): CTA 0, per item g < 256: [g][8] globaltimer
};
__device__ __forceinline__ long long wo_gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ uint32_t hsub2_u32(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
template <int BN>
__global__ void __launch_bounds__(WCfg<BN>::kThreads, 1) wo_gemm_kernel(const __grid_constant__ WParams p) {
  using C = WCfg<BN>;
  constexpr int G = C::G;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring_w = smem;
  uint8_t* ring_t = smem + C::kOffT;
  uint8_t* ring_o = smem + C::kOffO;
  uint64_t* full_w = reinterpret_cast<uint64_t*>(smem + C::kRingBytes);
  uint64_t* empty_w = full_w + C::kStagesW;
  uint64_t* full_t = empty_w + C::kStagesW;
  uint64_t* empty_t = full_t + C::kStagesT;
  uint64_t* full_o = empty_t + C::kStagesT;
  uint64_t* empty_o = full_o + C::kStagesO;
  uint64_t* a_full = empty_o + C::kStagesO;  // [G] widening group g -> base issuer g
  uint64_t* a_empty = a_full + 3;         // [G] base issuer g -> widening group g
  uint64_t* acc_full = a_empty + 3;       // [2] the G + 1 issuers -> epilogue
  uint64_t* acc_empty = acc_full + 2;     // [2] epilogue -> issuers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    if (p.nbase) {
      tma_prefetch(&p.tm_w);
      tma_prefetch(&p.tm_xb);
    }
    if (p.nout) {
      tma_prefetch(&p.tm_wo);
      tma_prefetch(&p.tm_wolo);
      tma_prefetch(&p.tm_xo);
    }
  }
  if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < C::kStagesW; ++i) { mbar_init(&full_w[i], 1); mbar_init(&empty_w[i], 4); }
      for (int i = 0; i < C::kStagesT; ++i) { mbar_init(&full_t[i], 1); mbar_init(&empty_t[i], 1); }
      for (int i = 0; i < C::kStagesO; ++i) { mbar_init(&full_o[i], 1); mbar_init(&empty_o[i], 1); }
      for (int i = 0; i < G; ++i) {
        mbar_init(&a_full[i], 4);
        mbar_init(&a_empty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&acc_full[i], G + 1);
        mbar_init(&acc_empty[i], 4);
      }
      fence_mbar_init();
    }
    __syncwarp();
    tmem_alloc<1>(tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: only the token / outlier-tile producer reads the planes kernel's output and
  // waits for it; the weight stream and its widening start right away
  asm volatile("griddepcontrol.launch_dependents;");   // let the finalize kernel launch early

  const int tiles_n = (p.N + kBlockM - 1) / kBlockM;
  const int num_units = tiles_n * p.tiles_t * p.splits;
  const int items = p.nbase + p.nout;
  const int natoms = p.w4 ? 4 : 2;  // 64-K token atoms per base stage
  // unit -> (weight block, token tile, split, item range); consecutive units walk the
  // weight blocks of one (token tile, split)
  auto decode = [&](int u, int& nb, int& tb, int& s, int& i0, int& i1) {
    nb = u % tiles_n;
    const int r = u / tiles_n;
    tb = r % p.tiles_t;
    s = r / p.tiles_t;
    i0 = static_cast<int>((static_cast<long long>(items) * s) / p.splits);
    i1 = static_cast<int>((static_cast<long long>(items) * (s + 1)) / p.splits);
  };
  auto nbase_in = [&](int i0, int i1) { return max(0, min(i1, p.nbase) - i0); };

  if (warp == 0 || warp == C::kIssEnd) {
    if (lane == 0) {
      // weights stream once per token tile (decode: once); token planes are re-read by
      // every weight block
      const uint64_t pol_w = p.tiles_t == 1 ? policy_evict_first() : policy_evict_normal();
      const uint64_t pol_x = policy_evict_last();
      const bool wprod = warp == 0;  // warp 0: weight ring; last warp: token + outlier rings
      if (!wprod) asm volatile("griddepcontrol.wait;" ::: "memory");  // the token planes are complete
      int bc = 0, oc = 0, gi = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        int nb, tb, s, i0, i1;
        decode(u, nb, tb, s, i0, i1);
        for (int i = i0; i < i1; ++i, ++gi) {
          if (i < p.nbase) {
            if (wprod) {
              const int st = bc % C::kStagesW;
              mbar_wait_sleep(&empty_w[st], ((bc / C::kStagesW) & 1) ^ 1);
              if (p.trace && blockIdx.x == 0 && gi < 256) p.trace[gi * 8 + 0] = wo_gtime();
              mbar_arrive_expect_tx(&full_w[st], kWABytes);
              tma_load_2d(ring_w + st * C::kSlotW, &p.tm_w, i * kKBlockBytes, nb * kBlockM, &full_w[st], pol_w);
            } else {
              const int st = bc % C::kStagesT;
              mbar_wait_sleep(&empty_t[st], ((bc / C::kStagesT) & 1) ^ 1);
              uint8_t* slot = ring_t + st * C::kSlotT;
              mbar_arrive_expect_tx(&full_t[st], natoms * C::kBAtom);
              for (int a = 0; a < natoms; ++a)
                tma_load_2d(slot + a * C::kBAtom, &p.tm_xb, (i * natoms + a) * kKBlockBytes, tb * BN, &full_t[st],
                            pol_x);
            }
            ++bc;
          } else {
            if (!wprod) {
              const int j = i - p.nbase, st = oc % C::kStagesO;
              mbar_wait_sleep(&empty_o[st], ((oc / C::kStagesO) & 1) ^ 1);
              uint8_t* slot = ring_o + st * C::kSlotO;
              mbar_arrive_expect_tx(&full_o[st], kWABytes + C::kBAtom);
              tma_load_2d(slot, (j & 1) ? &p.tm_wolo : &p.tm_wo, (j >> 1) * kKBlockBytes, nb * kBlockM, &full_o[st],
                          pol_w);
              tma_load_2d(slot + kWABytes, &p.tm_xo, (j >> 1) * kKBlockBytes, tb * BN, &full_o[st], pol_x);
            }
            ++oc;
          }
        }
      }
    }
  } else if (warp == 1 || warp >= C::kEpiEnd) {  // (warp C::kIssEnd is handled above)
    // MMA issuers. A single thread issues at most one small-N tcgen05.mma per ~45
    // cycles (tools/ts_rate.cu: 44.5 cycles at N = 16, 13.4 with four issuing warps),
    // and a 256-K INT4 stage is 16 K = 16 steps, so the base stages are issued by two
    // threads (warp 14: stages of widening group 0, warp 15: group 1), each into its own
    // accumulator; warp 1 issues the outlier stages into a third. Every issuer commits
    // acc_full once per unit (count 3).
    {  // the whole warp runs the loop (converged); elected lanes issue
      constexpr uint32_t idesc = idesc_make(1u, 0u, kBlockM, BN);
      const int role = warp == 1 ? G : warp - C::kEpiEnd;  // < G: base group, G: outliers
      int bc = 0, oc = 0, it = 0, gi = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++it) {
        int nb, tb, s, i0, i1;
        decode(u, nb, tb, s, i0, i1);
        const int b = it & 1;
        mbar_wait_sleep(&acc_empty[b], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + C::kAccColG + b * C::kAccBufG + role * BN;
        bool first = true;
        for (int i = i0; i < i1; ++i, ++gi) {
          if (i < p.nbase) {
            const int st = bc % C::kStagesT;
            uint8_t* slot = ring_t + st * C::kSlotT;
            const int g = bc % G, use = bc / G;
            if (role == g) {
              mbar_wait_spin(&a_full[g], use & 1);                     // A widened into TMEM
              mbar_wait(&full_t[st], (bc / C::kStagesT) & 1);          // token tile landed
              tc_fence_after();
              if (p.trace && lane == 0 && blockIdx.x == 0 && gi < 256) p.trace[gi * 8 + 6] = wo_gtime();
              const uint32_t a_tm = tmem_base + g * kWTmemA;
              const int ksteps = natoms * 4;
              const uint64_t bd0 = umma_desc_sw128(smem_u32(slot));
              for (int j = 0; j < ksteps; ++j)
                mma_f16_ts_e(d, a_tm + 8 * j, bd0 + (j >> 2) * (C::kBAtom >> 4) + 2 * (j & 3), idesc,
                             (first && j == 0) ? 0u : 1u);
              first = false;
              commit_e(&a_empty[g]);
              commit_e(&empty_t[st]);
              if (p.trace && lane == 0 && blockIdx.x == 0 && gi < 256) p.trace[gi * 8 + 7] = wo_gtime();
            }
            ++bc;
          } else {
            if (role == G) {
              const int st = oc % C::kStagesO;
              uint8_t* slot = ring_o + st * C::kSlotO;
              mbar_wait(&full_o[st], (oc / C::kStagesO) & 1);
              tc_fence_after();
              const uint64_t ad = umma_desc_sw128(smem_u32(slot));
              const uint64_t bd = umma_desc_sw128(smem_u32(slot + kWABytes));
#pragma unroll
              for (int k = 0; k < 4; ++k) mma_f16_ss_e(d, ad + 2 * k, bd + 2 * k, idesc, (first && k == 0) ? 0u : 1u);
              first = false;
              commit_e(&empty_o[st]);
            }
            ++oc;
          }
        }
        commit_e(&acc_full[b]);
      }
    }
  } else if (warp < C::kWidenEnd) {
    // widening: thread = weight row r of the 128-row tile (TMEM lane r)
    const int quad = warp & 3, g = (warp - 2) >> 2;  // TMEM lane quadrant = warp % 4
    const int r = quad * 32 + lane;
    const uint32_t a_tm = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + g * kWTmemA;
    int bc = 0, gi = 0;
    const bool tr = p.trace && blockIdx.x == 0 && lane == 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      int nb, tb, s, i0, i1;
      decode(u, nb, tb, s, i0, i1);
      for (int i = i0; i < i1; ++i, ++gi) {
        if (i < p.nbase) {
          if (bc % G == g) {
            const int st = bc % C::kStagesW;
            mbar_wait_sleep(&full_w[st], (bc / C::kStagesW) & 1);
            mbar_wait_spin(&a_empty[g], ((bc / G) & 1) ^ 1);
            tc_fence_after();
            if (tr && quad == 0 && gi < 256) p.trace[gi * 8 + 1] = wo_gtime();
            const uint8_t* wrow = ring_w + st * C::kSlotW + r * kKBlockBytes;
            if (p.w4) {
              // chunk c (16 B) holds k = 32c + i (low nibble of byte i) and 32c + 16 + i
              // (high nibble); column = k / 2
#pragma unroll 1
              for (int h = 0; h < 4; ++h) {
                uint32_t o[32];
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                  const int c = 2 * h + cc;
                  const uint4 v = *reinterpret_cast<const uint4*>(wrow + ((c ^ (r & 7)) << 4));
                  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                  for (int q = 0; q < 4; ++q) {
                    const uint32_t lo = (w[q] & 0x0F0F0F0Fu) ^ 0x08080808u;  // q + 8
                    const uint32_t hi = ((w[q] >> 4) & 0x0F0F0F0Fu) ^ 0x08080808u;
                    o[16 * cc + 2 * q] = hsub2_u32(prmt(lo, 0x64646464u, 0x4140u), 0x64086408u);
                    o[16 * cc + 2 * q + 1] = hsub2_u32(prmt(lo, 0x64646464u, 0x4342u), 0x64086408u);
                    o[16 * cc + 8 + 2 * q] = hsub2_u32(prmt(hi, 0x64646464u, 0x4140u), 0x64086408u);
                    o[16 * cc + 8 + 2 * q + 1] = hsub2_u32(prmt(hi, 0x64646464u, 0x4342u), 0x64086408u);
                  }
                }
                tmem_st32(a_tm + 32 * h, o);
              }
            } else {
              // INT8: chunk c holds k = 16c .. 16c + 15 in order; u = q + 128
#pragma unroll 1
              for (int h = 0; h < 2; ++h) {
                uint32_t o[32];
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                  const int c = 4 * h + cc;
                  const uint4 v = *reinterpret_cast<const uint4*>(wrow + ((c ^ (r & 7)) << 4));
                  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                  for (int q = 0; q < 4; ++q) {
                    const uint32_t uu = w[q] ^ 0x80808080u;
                    o[8 * cc + 2 * q] = hsub2_u32(prmt(uu, 0x64646464u, 0x4140u), 0x64806480u);
                    o[8 * cc + 2 * q + 1] = hsub2_u32(prmt(uu, 0x64646464u, 0x4342u), 0x64806480u);
                  }
                }
                tmem_st32(a_tm + 32 * h, o);
              }
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              mbar_arrive(&empty_w[st]);  // weight tile consumed (the MMAs read TMEM)
              mbar_arrive(&a_full[g]);
            }
            if (tr && gi < 256) p.trace[gi * 8 + 2 + quad] = wo_gtime();
          }
          ++bc;
        }
      }
    }
  } else {
    // epilogue (warps 10-13): TMEM lane = weight row n, column = plane row t
    const int quad = warp & 3;
    int it = 0, bc0 = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++it) {
      int nb, tb, s, i0, i1;
      decode(u, nb, tb, s, i0, i1);
      // accumulators written in this unit: base issuer g iff one of its stages is here
      const int nbi = nbase_in(i0, i1);
      uint32_t used = 0;  // bit g: base issuer g has a stage in this unit
      for (int k = 0; k < nbi && k < G; ++k) used |= 1u << ((bc0 + k) % G);
      const bool has_out = i1 > p.nbase;
      bc0 += nbi;
      const int b = it & 1;
      const int n = nb * kBlockM + quad * 32 + lane;
      const bool nok = n < p.N;
      const float sc = nok ? __ldg(p.scale + n) : 0.0f;
      const float bi = (nok && s == 0 && p.bias) ? __ldg(p.bias + n) : 0.0f;
      mbar_wait_sleep(&acc_full[b], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tacc = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + C::kAccColG + b * C::kAccBufG;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float vb[32];
        uint32_t vo[32];  // outlier accumulator columns (raw f32 bits)
        if constexpr (BN == 16) {
          // G = 3: base 0-2 in columns 0-47, outliers in 48-63
          uint32_t x0[32];
          tmem_ld32(tacc, x0);
          tmem_ld32(tacc + 32, vo);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float a = 0.0f;
            if (used & 1u) a = __uint_as_float(x0[j]);
            if (used & 2u) a = __fadd_rn(a, __uint_as_float(x0[16 + j]));
            if (used & 4u) a = __fadd_rn(a, __uint_as_float(vo[j]));
            vb[j] = a;
            vo[j] = vo[16 + j];
          }
        } else {
          // G = 2: one 32-column load per accumulator, summed in place
          tmem_ld32(tacc + c, vo);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) vb[j] = (used & 1u) ? __uint_as_float(vo[j]) : 0.0f;
          tmem_ld32(tacc + BN + c, vo);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (used & 2u) vb[j] = __fadd_rn(vb[j], __uint_as_float(vo[j]));
          tmem_ld32(tacc + 2 * BN + c, vo);
          tmem_ld_wait();
        }
        if (nok) {
#pragma unroll
          for (int j = 0; j < (BN < 32 ? BN : 32); ++j) {
            const int t = tb * BN + c + j;
            if (t < p.R) {
              float v = t < p.M ? bi : 0.0f;  // bias once: hi plane, first split
              if (has_out) v = __fadd_rn(v, __uint_as_float(vo[j]));
              if (used) v = __fmaf_rn(sc, vb[j], v);
              if (p.mode == 0)
                static_cast<float*>(p.out)[(static_cast<long long>(s) * p.R + t) * p.N + n] = v;
              else if (p.mode == 1)
                static_cast<float*>(p.out)[static_cast<long long>(t) * p.ldo + n] = v;
              else
                static_cast<__half*>(p.out)[static_cast<long long>(t) * p.ldo + n] = __float2half_rn(v);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, 512);
  }
}

// token planes: x -> xb f16 [P*M][kpad] (base columns in permutation order, zero
// padded) and xo f16 [P*M][opad]; P = 2 for f32 input (hi, lo planes)
__global__ void wo_planes_kernel(const WoArgs a, __half* __restrict__ xb, __half* __restrict__ xo, int planes) {
  // the GEMM (launched with programmatic serialisation) may start its prologue now; it
  // waits for this grid's completion before reading the planes
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t width = a.kpad + a.opad;
  for (int64_t t = blockIdx.y; t < a.M; t += gridDim.y)
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < width;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t src = -1;
    if (j < a.kpad) {
      if (j < a.kb) src = a.base_src[j];
    } else if (j - a.kpad < a.n_out) {
      src = a.out_src[j - a.kpad];
    }
    float v = 0.0f;
    if (src >= 0)
      v = a.x_is_f32 ? reinterpret_cast<const float*>(a.x)[t * a.ldx + src]
                     : __half2float(reinterpret_cast<const __half*>(a.x)[t * a.ldx + src]);
    const __half hi = __float2half_rn(v);
    __half* dst = j < a.kpad ? xb + t * a.kpad + j : xo + t * a.opad + (j - a.kpad);
    const int64_t plane_stride = j < a.kpad ? a.M * a.kpad : a.M * a.opad;
    *dst = hi;
    if (planes == 2) dst[plane_stride] = __float2half_rn(__fsub_rn(v, __half2float(hi)));
  }
}

__global__ void wo_finalize_kernel(const float* __restrict__ ws, int64_t M, int64_t N, int splits, int planes,
                                   void* y, int y_f16, int64_t ldy) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the GEMM's partials are complete
  const int64_t total = M * N;
  const int64_t R = M * planes;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = e / N, n = e % N;
    float v = 0.0f;
    for (int s = 0; s < splits; ++s) {
      v = __fadd_rn(v, ws[(s * R + t) * N + n]);
      if (planes == 2) v = __fadd_rn(v, ws[(s * R + M + t) * N + n]);
    }
    if (y_f16)
      static_cast<__half*>(y)[t * ldy + n] = __float2half_rn(v);
    else
      static_cast<float*>(y)[t * ldy + n] = v;
  }
}

__global__ void f16_lo_kernel(const float* __restrict__ src, int64_t rows, int64_t cols, __half* __restrict__ dst,
                              int64_t pitch) {
  const int64_t r = blockIdx.y;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < pitch;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float v = 0.0f;
    if (c < cols) {
      const float x = src[r * cols + c];
      v = __fsub_rn(x, __half2float(__float2half_rn(x)));
    }
    dst[r * pitch + c] = __float2half_rn(v);
  }
}

struct WoPlan {
  int bn, splits, tiles_t, nbase, nout, planes;
};

WoPlan plan(const WoArgs& a, int num_sms) {
  WoPlan pl{};
  pl.planes = a.x_is_f32 ? 2 : 1;
  const int64_t R = a.M * pl.planes;
  pl.bn = R <= 16 ? 16 : 32;  // 3 accumulators x 2 buffers x BN + 2 A buffers <= 512 TMEM columns
  pl.tiles_t = static_cast<int>((R + pl.bn - 1) / pl.bn);
  const int64_t kstage = a.w4 ? 256 : 128;
  pl.nbase = static_cast<int>((a.kpad + kstage - 1) / kstage);
  pl.nout = static_cast<int>(2 * (a.opad / 64));
  const int items = pl.nbase + pl.nout;
  const long long tiles = ((a.N + kBlockM - 1) / kBlockM) * static_cast<long long>(pl.tiles_t);
  // K splits: minimise the busiest CTA's stage count, ceil(units / SMs) x (stages per
  // unit + 1 for the unit's pipeline fill / epilogue); e.g. LLaMA-2-70B up (224 tiles x
  // 39 stages): 3 splits -> 5 x 14 instead of 2 splits -> 4 x 21
  int splits = 1;
  long long best = -1;
  for (int sp = 1; sp <= 16 && sp <= items; ++sp) {
    const long long waves = (tiles * sp + num_sms - 1) / num_sms;
    const long long cost = waves * ((items + sp - 1) / sp + 1);
    if (best < 0 || cost < best) { best = cost; splits = sp; }
  }
  pl.splits = splits;
  return pl;
}

template <int BN>
cudaError_t launch_wo_t(const WParams& wp, int units, int num_sms, cudaStream_t stream) {
  using C = WCfg<BN>;
  auto kern = wo_gemm_kernel<BN>;
  cudaError_t e = ensure_smem_attr(kern, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(units < num_sms ? units : num_sms));
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, wp);
}

}  // namespace

size_t wo_workspace_bytes(const WoArgs& a, int num_sms, size_t* plane_bytes_b, size_t* plane_bytes_o) {
  const WoPlan pl = plan(a, num_sms);
  const int64_t R = a.M * pl.planes;
  *plane_bytes_b = static_cast<size_t>(R * a.kpad * 2);
  *plane_bytes_o = static_cast<size_t>(R * a.opad * 2);
  const bool direct = pl.splits == 1 && pl.planes == 1;
  return direct ? 0 : static_cast<size_t>(pl.splits) * R * a.N * 4;
}

cudaError_t launch_weight_only(const WoArgs& a, int num_sms, cudaStream_t stream, const char** err_msg) {
  *err_msg = nullptr;
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  if (a.kpad % 128 || a.opad % 64) { *err_msg = "weight-only: bad padding"; return cudaErrorInvalidValue; }
  if (a.n_out > 0 && (!a.wo || !a.wo_lo)) { *err_msg = "weight-only: outlier weights missing"; return cudaErrorInvalidValue; }
  const WoPlan pl = plan(a, num_sms);
  const int64_t R = a.M * pl.planes;
  if (a.kpad + a.opad > 0) {
    dim3 grid(static_cast<unsigned>(std::min<int64_t>((a.kpad + a.opad + 255) / 256, 64)),
              static_cast<unsigned>(std::min<int64_t>(a.M, 65535)));
    wo_planes_kernel<<<grid, 256, 0, stream>>>(a, a.xb, a.xo, pl.planes);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const bool direct = pl.splits == 1 && pl.planes == 1;
  WParams wp{};
  CUresult r1 = CUDA_SUCCESS, r2 = CUDA_SUCCESS;
  if (pl.nbase) {
    r1 = a.w4 ? encode_map_2d(&wp.tm_w, a.w4, a.kpad / 2, a.N, a.kpad / 2, kKBlockBytes, kBlockM, true)
              : encode_map_2d(&wp.tm_w, a.w8, a.kpad, a.N, a.kpad, kKBlockBytes, kBlockM, true);
    r2 = encode_map_2d(&wp.tm_xb, a.xb, a.kpad * 2, R, a.kpad * 2, kKBlockBytes, pl.bn, true);
  }
  CUresult r3 = CUDA_SUCCESS, r4 = CUDA_SUCCESS, r5 = CUDA_SUCCESS;
  if (pl.nout) {
    r3 = encode_map_2d(&wp.tm_wo, a.wo, a.opad * 2, a.N, a.opad * 2, kKBlockBytes, kBlockM, true);
    r4 = encode_map_2d(&wp.tm_wolo, a.wo_lo, a.opad * 2, a.N, a.opad * 2, kKBlockBytes, kBlockM, true);
    r5 = encode_map_2d(&wp.tm_xo, a.xo, a.opad * 2, R, a.opad * 2, kKBlockBytes, pl.bn, true);
  }
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS || r3 != CUDA_SUCCESS || r4 != CUDA_SUCCESS || r5 != CUDA_SUCCESS) {
    *err_msg = "weight-only: tensor map encode failed";
    return cudaErrorInvalidValue;
  }
  wp.scale = a.scale;
  wp.bias = a.bias;
  wp.out = direct ? a.y : a.ws;
  wp.R = static_cast<int>(R);
  wp.M = static_cast<int>(a.M);
  wp.N = static_cast<int>(a.N);
  wp.ldo = static_cast<int>(a.ldy);
  wp.nbase = pl.nbase;
  wp.nout = pl.nout;
  wp.splits = pl.splits;
  wp.tiles_t = pl.tiles_t;
  wp.w4 = a.w4 ? 1 : 0;
  wp.mode = direct ? (a.y_is_f16 ? 2 : 1) : 0;
  const int units = static_cast<int>(((a.N + kBlockM - 1) / kBlockM) * pl.tiles_t * pl.splits);
  static const char* trace_path = getenv("QUIK_WO_TRACE");
  static long long* trace_buf = nullptr;
  if (trace_path) {
    if (!trace_buf) cudaMalloc(&trace_buf, 256 * 8 * 8);
    cudaMemsetAsync(trace_buf, 0, 256 * 8 * 8, stream);
    wp.trace = trace_buf;
  }
  cudaError_t e;
  switch (pl.bn) {
    case 16: e = launch_wo_t<16>(wp, units, num_sms, stream); break;
    default: e = launch_wo_t<32>(wp, units, num_sms, stream); break;
  }
  if (trace_path && e == cudaSuccess) {
    long long h[2048];
    cudaStreamSynchronize(stream);
    cudaMemcpy(h, trace_buf, sizeof(h), cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(trace_path, "wb")) {
      fwrite(h, 8, 2048, f);
      fclose(f);
    }
  }
  if (e != cudaSuccess || direct) return e;
  const int64_t total = a.M * a.N;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 4 * num_sms));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, wo_finalize_kernel, static_cast<const float*>(a.ws), a.M, a.N, pl.splits,
                            pl.planes, a.y, a.y_is_f16, a.ldy);
}

cudaError_t launch_f16_lo_padded(const float* src, int64_t rows, int64_t cols, __half* dst, int64_t pitch,
                                 cudaStream_t stream) {
  if (rows == 0 || pitch == 0) return cudaSuccess;
  dim3 grid(static_cast<unsigned>(std::min<int64_t>((pitch + 255) / 256, 64)), static_cast<unsigned>(rows));
  f16_lo_kernel<<<grid, 256, 0, stream>>>(src, rows, cols, dst, pitch);
  return cudaGetLastError();
}

}  // namespace quikb200
