// Weight-streaming integer GEMM on INT4 weights for small token counts (M <= 64, quik
// mode; HBM-bound for small M, cfg1 / cfg4 small M). Each CTA walks a
// sequence of segments (a 128-row weight block's K interval: round-robin units of whole
// blocks or K splits, or a stream-K range, host-chosen); a whole block finalises from
// registers, a cut one accumulates
//
//   acc_ws[t][n] += sum_{k in segment} q[n][k] * X8[t][k]      (red.global.add.s32)
//
// and, in the same kernel, the rest of the layer: the CTA that completes a weight block
// last (per-block arrival counter) finalises it exactly as the fused kernel's epilogue
// does: init = bias + dequant_element(acc) (op by op, runtime.cpp:70-77) written into a
// TMEM accumulator, the f16 outlier MMAs (x_o W_o^T) accumulated onto it, f16/f32 out.
// Same instructions in the same order, so the output is bit-identical to the fused V3
// forward (and to V1/V2). The workspace and counters are left zeroed for the next call.
//
// Same architecture as the weight-only kernel (wo.cu): the 4-bit weights never exist
// as int8 in shared memory. A weight producer TMA-streams 16 KB INT4 tiles (128 rows x
// 256 K) into a deep ring; G widening groups (4 warps each, one weight row per thread)
// move each nibble into the high half of its byte (16 x the value, 1-2 integer ops per
// four values; the epilogue shifts the exact sums right by 4, like the prefill GEMM),
// tcgen05.st them into a TMEM A buffer (lane = weight row, column j = 4 int8
// {k = 4j .. 4j+3}, pinned by tools/ts_probe.cu) and release the weight slot at once;
// each group's converged
// issuing warp runs 8 tcgen05.mma.kind::i8 (A from TMEM, the int8 activation-code tile
// from shared memory) per stage into its own int32 accumulator; four epilogue warps sum
// the G accumulators and red.add them into the workspace. Each ring stage has exactly
// one consumer sequence (see wo.cu).
//
// Warps: 0 weight producer, 1 TMEM allocator, 2 .. 4G+1 widening, then 4 epilogue, G
// issuers, 1 activation-tile producer.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"

namespace quikb200 {

namespace {

constexpr int kS4WBytes = kBlockM * kKBlockBytes;  // 16 KB: 128 rows x 128 B INT4 = 256 K
constexpr int kS4TmemA = 64;                        // columns per A buffer (256 K of int8)

template <int BN>
struct S4Cfg {
  static constexpr int G = BN == 64 ? 2 : 3;
  static constexpr int kTAtom = BN * kKBlockBytes;  // BN rows x 128 K int8 (or 64 f16)
  static constexpr int kSlotT = 2 * kTAtom;         // 256 K of codes per stage
  static constexpr int kStagesW = BN == 16 ? 9 : 6;
  static constexpr int kStagesT = BN == 64 ? 4 : 6;
  static_assert(kStagesW % G == 0 && kStagesT % G == 0, "one consumer group per stage");
  // finalisation buffer: two 64-column outlier blocks (f16 weight tile + x_o tile)
  static constexpr int kFinBlk = kS4WBytes + kTAtom;
  static constexpr int kOffT = kStagesW * kS4WBytes;
  static constexpr int kOffF = kOffT + kStagesT * kSlotT;
  static constexpr int kRingBytes = kOffF + 2 * kFinBlk;
  // TMEM A buffers per widening group: two at BN = 16 (the group widens its next stage
  // while its MMAs still read the previous one), one where TMEM is short
  static constexpr int NB = BN == 16 ? 2 : 1;
  static constexpr int kBarBytes = (2 * (kStagesW + kStagesT) + 2 * G * NB + 6) * 8 + 32;
  static constexpr int kSmemBytes = 1024 + kRingBytes + kBarBytes;
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
  static constexpr int kAccCol = NB * G * kS4TmemA;
  static constexpr int kAccBuf = G * BN;             // G int32 accumulators, double-buffered
  static constexpr int kFinCol = kAccCol + 2 * kAccBuf;  // f32 finalisation accumulator (BN)
  static_assert(kFinCol + BN <= 512, "TMEM budget");
  // warps: 0 weight producer, 1 TMEM allocator, 2 .. 4G+1 widening, 4 epilogue, G base
  // issuers, 1 code-tile producer
  static constexpr int kWidenEnd = 2 + 4 * G, kEpiEnd = kWidenEnd + 4, kIssEnd = kEpiEnd + G;
  static constexpr int kThreads = (kIssEnd + 1) * 32;
};

struct S4Params {
  CUtensorMap tm_w;   // INT4 [N][kpad / 2] (device nibble layout), box {128 B, 128}, SW128
  CUtensorMap tm_x;   // int8 [M][kpad], box {128 B, BN}, SW128
  CUtensorMap tm_wo;  // f16 [N][opad] as bytes, box {128 B, 128}, SW128
  CUtensorMap tm_xo;  // f16 [M][opad] as bytes, box {128 B, BN}, SW128
  int M, N, nstage, nout;  // nstage: K stages (INT4 256 K, INT8 128 K); nout: 64-column outlier blocks
  int splits;              // round-robin schedule: K splits per block (0: stream-K schedule)
  int w8;                          // INT8 weights (A from the weight ring, no widening)
  int32_t* acc;                    // [M][N] int32 workspace (zero on entry and exit)
  int* counters;                   // [tiles] arrivals per weight block (zero on entry and exit)
  const float* a_scale;
  const float* a_zero;
  const float* w_scale;
  const float* wreduced;
  const float* bias;
  float half_range;
  void* out;
  long long ldo;
  int out_f16;
  int gated;              // rows interleave up / gate (32-row blocks): out is [M][N / 2]
  int prefetch;           // outlier tiles load while the unit streams (QUIK_S4_PREFETCH=0: at finalisation)
  int n_dst;              // 1 + peers
  void* dst[8];           // output base pointers (dst[0] == out)
};

template <int BN>
__global__ void __launch_bounds__(S4Cfg<BN>::kThreads, 1) stream4_gemm_kernel(const __grid_constant__ S4Params p) {
  using C = S4Cfg<BN>;
  constexpr int G = C::G;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring_w = smem;
  uint8_t* ring_t = smem + C::kOffT;
  uint8_t* fin = smem + C::kOffF;
  uint64_t* full_w = reinterpret_cast<uint64_t*>(smem + C::kRingBytes);
  uint64_t* empty_w = full_w + C::kStagesW;
  uint64_t* full_t = empty_w + C::kStagesW;
  uint64_t* empty_t = full_t + C::kStagesT;
  uint64_t* fin_full = empty_t + C::kStagesT;  // finalisation: outlier tiles landed
  uint64_t* fin_mma = fin_full + 1;            // finalisation: outlier MMAs done
  constexpr int NB = C::NB;
  uint64_t* a_full = fin_mma + 1;              // [G][NB] widening group g, A buffer b -> issuer g
  uint64_t* a_empty = a_full + G * NB;       // [G][NB] issuer g -> widening group g
  uint64_t* acc_full = a_empty + G * NB;     // [2] the G issuers -> epilogue
  uint64_t* acc_empty = acc_full + 2;        // [2] epilogue -> issuers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tm_w);
    tma_prefetch(&p.tm_x);
    if (p.nout) {
      tma_prefetch(&p.tm_wo);
      tma_prefetch(&p.tm_xo);
    }
  }
  if (warp == 1) {
    if (lane == 0) {
      // INT4: a weight slot is released by its 4 widening warps; INT8: by its issuer's commit
      for (int i = 0; i < C::kStagesW; ++i) { mbar_init(&full_w[i], 1); mbar_init(&empty_w[i], p.w8 ? 1 : 4); }
      for (int i = 0; i < C::kStagesT; ++i) { mbar_init(&full_t[i], 1); mbar_init(&empty_t[i], 1); }
      mbar_init(fin_full, 1);
      mbar_init(fin_mma, 1);
      for (int i = 0; i < G * NB; ++i) { mbar_init(&a_full[i], 4); mbar_init(&a_empty[i], 1); }
      for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], G); mbar_init(&acc_empty[i], 4); }
      fence_mbar_init();
    }
    __syncwarp();
    tmem_alloc<1>(tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: only the roles that read K1's outputs (the code-tile producer; the epilogue,
  // which finalises with the per-token scales and outlier columns) wait for K1; the
  // weight stream and its widening start while K1 is still running.

  const int tiles_n = (p.N + kBlockM - 1) / kBlockM;
  // Two schedules, walked identically by every role as a sequence of segments (one
  // weight block's K interval each):
  //  * round robin (p.splits > 0): unit u = blockIdx.x + j * gridDim.x is block
  //    u % tiles_n, K split u / tiles_n of p.splits (whole blocks when p.splits == 1);
  //  * stream-K (p.splits == 0): the (block, K stage) pairs, block-major, are cut into
  //    gridDim.x contiguous equal ranges, one per CTA (no idle tail wave when the block
  //    count is a poor multiple of the grid).
  // A block cut into several segments is reduced through the workspace and finalised by
  // the last of its contributors; a whole block finalises from registers.
  // (32-bit state: two registers per role; the rest is re-read from the parameter space)
  const int work = tiles_n * p.nstage;
  struct Segs {
    int pos, end;  // stream-K: the CTA's work range; round robin: unit index and unit count
  };
  auto segs = [&]() {
    if (p.splits) return Segs{static_cast<int>(blockIdx.x), tiles_n * p.splits};
    return Segs{static_cast<int>(static_cast<long long>(work) * blockIdx.x / gridDim.x),
                static_cast<int>(static_cast<long long>(work) * (blockIdx.x + 1) / gridDim.x)};
  };
  auto next = [&](Segs& sg, int& nb, int& k0, int& k1) {
    if (sg.pos >= sg.end) return false;
    if (p.splits) {
      nb = sg.pos % tiles_n;
      const int sp = sg.pos / tiles_n;
      k0 = (p.nstage * sp) / p.splits;
      k1 = (p.nstage * (sp + 1)) / p.splits;
      sg.pos += gridDim.x;
      return true;
    }
    nb = sg.pos / p.nstage;
    k0 = sg.pos - nb * p.nstage;
    k1 = k0 + (sg.end - sg.pos) < p.nstage ? k0 + (sg.end - sg.pos) : p.nstage;
    sg.pos += k1 - k0;
    return true;
  };
  // after next(): that was the CTA's last segment
  auto done = [](const Segs& sg) { return sg.pos >= sg.end; };
  // stream-K: CTA whose range holds work item x (the largest c with floor(c * work / grid) <= x)
  auto owner = [&](int x) { return static_cast<int>(((x + 1LL) * gridDim.x - 1) / work); };
  auto contributors = [&](int nb) {
    if (p.splits) return p.splits;
    return owner((nb + 1) * p.nstage - 1) - owner(nb * p.nstage) + 1;
  };

  if (warp == 0 || warp == C::kIssEnd) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();  // weights stream once
      const uint64_t pol_x = policy_evict_last();   // code / x_o tiles are re-read by every block
      const bool wprod = warp == 0;
      if (!wprod) asm volatile("griddepcontrol.wait;" ::: "memory");  // K1's codes are complete
      int bc = 0, nb, k0, k1;
      for (Segs sg = segs(); next(sg, nb, k0, k1);) {
        if (wprod && done(sg))
          asm volatile("griddepcontrol.launch_dependents;");  // last segment: the next kernel may start its prologue
        {
          for (int i = k0; i < k1; ++i, ++bc) {
            if (wprod) {
              const int st = bc % C::kStagesW;
              mbar_wait_sleep(&empty_w[st], ((bc / C::kStagesW) & 1) ^ 1);
              mbar_arrive_expect_tx(&full_w[st], kS4WBytes);
              tma_load_2d(ring_w + st * kS4WBytes, &p.tm_w, i * kKBlockBytes, nb * kBlockM, &full_w[st], pol_w);
            } else {
              const int st = bc % C::kStagesT;
              mbar_wait_sleep(&empty_t[st], ((bc / C::kStagesT) & 1) ^ 1);
              uint8_t* slot = ring_t + st * C::kSlotT;
              if (p.w8) {  // 128-K stages: one code atom
                mbar_arrive_expect_tx(&full_t[st], C::kTAtom);
                tma_load_2d(slot, &p.tm_x, i * kKBlockBytes, 0, &full_t[st], pol_x);
              } else {
                mbar_arrive_expect_tx(&full_t[st], C::kSlotT);
                tma_load_2d(slot, &p.tm_x, (2 * i) * kKBlockBytes, 0, &full_t[st], pol_x);
                tma_load_2d(slot + C::kTAtom, &p.tm_x, (2 * i + 1) * kKBlockBytes, 0, &full_t[st], pol_x);
              }
            }
          }
        }
      }
    }
  } else if (warp >= C::kEpiEnd) {
    // issuer of widening group g (whole warp converged, elected lane issues); commits
    // acc_full once per unit
    const int g = warp - C::kEpiEnd;
    constexpr uint32_t idesc_i8 = idesc_make(2u, 1u, kBlockM, BN);
    int bc = 0, it = 0, nb, k0, k1;
    for (Segs sg = segs(); next(sg, nb, k0, k1); ++it) {
      const int b = it & 1;
      mbar_wait_sleep(&acc_empty[b], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + C::kAccCol + b * C::kAccBuf + g * BN;
      bool first = true;
      for (int i = k0; i < k1; ++i, ++bc) {
        if (bc % G != g) continue;
        const int st = bc % C::kStagesT;
        const uint64_t bd0 = umma_desc_sw128(smem_u32(ring_t + st * C::kSlotT));
        if (p.w8) {
          // INT8 weights: A straight from the weight ring (SS MMAs), 128 K per stage
          const int sw = bc % C::kStagesW;
          mbar_wait(&full_w[sw], (bc / C::kStagesW) & 1);
          mbar_wait(&full_t[st], (bc / C::kStagesT) & 1);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(smem_u32(ring_w + sw * kS4WBytes));
#pragma unroll
          for (int j = 0; j < 4; ++j)
            mma_i8_ss_e(d, ad + 2 * j, bd0 + 2 * j, idesc_i8, (first && j == 0) ? 0u : 1u);
          first = false;
          commit_e(&empty_w[sw]);
          commit_e(&empty_t[st]);
          continue;
        }
        // the group's n-th stage uses A buffer n % NB
        const int n = bc / G, ab = n % NB;
        mbar_wait_spin(&a_full[g * NB + ab], (n / NB) & 1);  // A widened into TMEM
        mbar_wait(&full_t[st], (bc / C::kStagesT) & 1);    // code tile landed
        tc_fence_after();
        const uint32_t a_tm = tmem_base + (ab * G + g) * kS4TmemA;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          mma_i8_ts_e(d, a_tm + 8 * j, bd0 + (j >> 2) * (C::kTAtom >> 4) + 2 * (j & 3), idesc_i8,
                      (first && j == 0) ? 0u : 1u);
        first = false;
        commit_e(&a_empty[g * NB + ab]);
        commit_e(&empty_t[st]);
      }
      commit_e(&acc_full[b]);
    }
  } else if (warp >= 2 && warp < C::kWidenEnd) {
    // widening: thread = weight row r (TMEM lane r); chunk c (16 B) holds k = 32c + i
    // (low nibble of byte i) and k = 32c + 16 + i (high nibble) -> columns 8c + q
    // (low nibbles of word q) and 8c + 4 + q (high nibbles)
    const int quad = warp & 3, g = (warp - 2) >> 2;
    const int r = quad * 32 + lane;
    const uint32_t a_lane = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
    int bc = 0, nb, k0, k1;
    for (Segs sg = segs(); !p.w8 && next(sg, nb, k0, k1);) {  // (INT8: nothing to widen)
      for (int i = k0; i < k1; ++i, ++bc) {
        if (bc % G != g) continue;
        const int st = bc % C::kStagesW;
        const int n = bc / G, ab = n % NB;
        const uint32_t a_tm = a_lane + (ab * G + g) * kS4TmemA;
        mbar_wait_sleep(&full_w[st], (bc / C::kStagesW) & 1);
        mbar_wait_spin(&a_empty[g * NB + ab], ((n / NB) & 1) ^ 1);
        tc_fence_after();
        const uint8_t* wrow = ring_w + st * kS4WBytes + r * kKBlockBytes;
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
              // 16 x the value: each nibble moved to the high half of its byte (3 ops per
              // word instead of a sign extension); the epilogue shifts the exact sums back
              o[8 * cc + q] = (w[q] << 4) & 0xF0F0F0F0u;
              o[8 * cc + 4 + q] = w[q] & 0xF0F0F0F0u;
            }
          }
          tmem_st32(a_tm + 32 * h, o);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&empty_w[st]);  // weight tile consumed (the MMAs read TMEM)
          mbar_arrive(&a_full[g * NB + ab]);
        }
      }
    }
  } else if (warp >= C::kWidenEnd) {
    // epilogue (4 warps): TMEM lane = weight row n, column = token t
    const int quad = warp & 3;
    const bool lead = warp == C::kWidenEnd;  // issues the finalisation TMA loads / MMAs
    asm volatile("griddepcontrol.wait;" ::: "memory");  // K1's scales / outlier columns
    int it = 0, bc0 = 0, fin_ld = 0, fin_mm = 0, nb, k0, k1;
    constexpr uint32_t idesc_f16 = idesc_make(1u, 0u, kBlockM, BN);
    for (Segs sg = segs(); next(sg, nb, k0, k1); ++it) {
      const int ncontrib = contributors(nb);
      // a block inside this CTA's range (BN <= 32): the sums stay in registers and
      // finalise at once (no workspace round trip, no arrival counter)
      const bool direct = ncontrib == 1 && BN <= 32;
      uint32_t used = 0;
      for (int k = 0; k < k1 - k0 && k < G; ++k) used |= 1u << ((bc0 + k) % G);
      bc0 += k1 - k0;
      auto load_blocks = [&](int j0) {
        const int nblk = p.nout - j0 < 2 ? p.nout - j0 : 2;
        if (lane == 0) {
          mbar_arrive_expect_tx(fin_full, nblk * C::kFinBlk);
          for (int q = 0; q < nblk; ++q) {
            tma_load_2d(fin + q * C::kFinBlk, &p.tm_wo, (j0 + q) * kKBlockBytes, nb * kBlockM, fin_full,
                        policy_evict_first());
            tma_load_2d(fin + q * C::kFinBlk + kS4WBytes, &p.tm_xo, (j0 + q) * kKBlockBytes, 0, fin_full,
                        policy_evict_last());
          }
        }
        return nblk;
      };
      // (0) the segment's first outlier tiles load while its K range streams (the buffer is
      // free: the previous segment's finalisation completed before this loop iteration)
      // when this CTA will (a whole block) or most likely will finalise the block: round
      // robin, the block's last split (the CTAs reach it last); stream-K, a cut block's
      // head segment, the last one its CTA reaches (the other contributors streamed their
      // parts at the start of their ranges)
      const bool prefetched =
          p.nout && p.prefetch && (direct || (p.splits ? k1 == p.nstage : (k0 == 0 && done(sg))));
      if (lead && prefetched) load_blocks(0);
      const int b = it & 1;
      mbar_wait_sleep(&acc_full[b], (it >> 1) & 1);
      tc_fence_after();
      const int n = nb * kBlockM + quad * 32 + lane;
      const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
      const uint32_t tacc = tmem_base + lane_off + C::kAccCol + b * C::kAccBuf;
      int sum[32];
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
#pragma unroll
        for (int j = 0; j < 32; ++j) sum[j] = 0;
#pragma unroll 1
        for (int g = 0; g < G; ++g) {
          if (!(used & (1u << g))) continue;
          uint32_t x[32];
          tmem_ld32(tacc + g * BN + c, x);  // (BN = 16: the next accumulator's columns are ignored)
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) sum[j] += static_cast<int>(x[j]);
        }
        if (direct) {
          const int sh = p.w8 ? 0 : 4;
#pragma unroll
          for (int j = 0; j < 32; ++j) sum[j] >>= sh;
        } else if (n < p.N && used) {
          const int sh = p.w8 ? 0 : 4;  // INT4: the MMAs summed 16 x the weight (exact shift)
#pragma unroll
          for (int j = 0; j < (BN < 32 ? BN : 32); ++j) {
            const int t = c + j;
            if (t < p.M) atomicAdd(&p.acc[static_cast<long long>(t) * p.N + n], sum[j] >> sh);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
      // completion: the last of this block's contributors finalises it (writes -> fence ->
      // counter; last arriver: fence -> reads)
      if (!direct) {
        __threadfence();
        named_barrier_sync(1, 128);
        if (lead && lane == 0) *last_flag = atomicAdd(&p.counters[nb], 1) == ncontrib - 1;
        named_barrier_sync(1, 128);
        if (!*last_flag) {
          if (lead && prefetched) {  // the prefetched outlier tiles are not needed: retire the phase
            mbar_wait(fin_full, fin_ld & 1);
            ++fin_ld;
          }
          continue;
        }
        __threadfence();
      }
      // (1) init = bias + dequant_element(acc) -> TMEM finalisation accumulator
      const uint32_t tfin = tmem_base + lane_off + C::kFinCol;
      {
        const bool nok = n < p.N;
        const float sw = nok ? __ldg(&p.w_scale[n]) : 0.f, wr = nok ? __ldg(&p.wreduced[n]) : 0.f;
        const float bs = (nok && p.bias) ? __ldg(&p.bias[n]) : 0.f;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          // per-token scale / zero: lane j holds token c + j (shuffled below); all
          // accumulator loads in flight before the workspace is cleared
          const int tl = c + lane;
          const float sa_l = tl < p.M ? __ldg(&p.a_scale[tl]) : 0.f;
          const float zs_l = tl < p.M ? __fadd_rn(__ldg(&p.a_zero[tl]), __fmul_rn(p.half_range, sa_l)) : 0.f;  // runtime.cpp:74
          int32_t accv[BN < 32 ? BN : 32];
          if (direct) {
#pragma unroll
            for (int j = 0; j < (BN < 32 ? BN : 32); ++j) accv[j] = sum[j];
          } else {
#pragma unroll
            for (int j = 0; j < (BN < 32 ? BN : 32); ++j)
              accv[j] = (c + j < p.M && nok) ? __ldcg(&p.acc[static_cast<long long>(c + j) * p.N + n]) : 0;
#pragma unroll
            for (int j = 0; j < (BN < 32 ? BN : 32); ++j)
              if (c + j < p.M && nok) p.acc[static_cast<long long>(c + j) * p.N + n] = 0;  // zeros for the next call
          }
          uint32_t v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float sa = __shfl_sync(0xffffffffu, sa_l, j);
            const float zs = __shfl_sync(0xffffffffu, zs_l, j);
            float init = 0.f;
            if (j < BN && c + j < p.M) {
              float x = __fmul_rn(__int2float_rn(accv[j < BN ? j : 0]), sa);
              x = __fmul_rn(x, sw);
              x = __fadd_rn(x, __fmul_rn(zs, wr));  // dequant_element, runtime.cpp:70-77
              init = __fadd_rn(bs, x);
            }
            v[j] = __float_as_uint(init);
          }
          tmem_st32(tfin + c, v);  // (BN = 16: columns 16-31 land in unused TMEM)
        }
        tmem_st_wait();
      }
      tc_fence_before();
      named_barrier_sync(1, 128);
      // (2) outlier MMAs onto init, two 64-column blocks per round trip
      if (lead && p.nout) {
        tc_fence_after();
        for (int j0 = 0; j0 < p.nout; j0 += 2) {
          const int nblk = (j0 == 0 && prefetched) ? (p.nout < 2 ? p.nout : 2) : load_blocks(j0);
          mbar_wait(fin_full, fin_ld & 1);
          ++fin_ld;
          tc_fence_after();
          for (int q = 0; q < nblk; ++q) {
            const uint64_t ad = umma_desc_sw128(smem_u32(fin + q * C::kFinBlk));
            const uint64_t bd = umma_desc_sw128(smem_u32(fin + q * C::kFinBlk + kS4WBytes));
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_f16_ss_e(tmem_base + C::kFinCol, ad + 2 * k, bd + 2 * k, idesc_f16, 1u);
          }
          commit_e(fin_mma);
          mbar_wait(fin_mma, fin_mm & 1);  // MMAs done: buffer reusable, accumulator final
          ++fin_mm;
        }
        tc_fence_before();
      }
      named_barrier_sync(1, 128);
      tc_fence_after();
      // (3) drain: f16 / f32 to every destination. Gated MLP layers (rows interleave up /
      // gate in blocks of 32: quadrants 0, 2 up, 1, 3 gate) emit h = silu(gate) * up at
      // output feature nb * 64 + (quad / 2) * 32 + lane, like the fused epilogue: the gate
      // warp hands silu(g) to its up warp through shared memory (the free finalisation
      // buffer) between two 64-thread named barriers.
      float* xch = reinterpret_cast<float*>(fin) + (quad >> 1) * 1024;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        tmem_ld32(tfin + c, v);
        tmem_ld_wait();
        if (p.gated) {
          const int pair_bar = 2 + (quad >> 1);
          if (quad & 1) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float g = __uint_as_float(v[j]);
              xch[j * 32 + lane] = __fdividef(g, 1.0f + __expf(-g));
            }
            named_barrier_sync(pair_bar, 64);
            named_barrier_sync(pair_bar, 64);  // the up warp has read the exchange buffer
            continue;
          }
          named_barrier_sync(pair_bar, 64);
          const int f = nb * (kBlockM / 2) + (quad >> 1) * 32 + lane;
          if (n < p.N) {
#pragma unroll
            for (int j = 0; j < (BN < 32 ? BN : 32); ++j) {
              const int t = c + j;
              if (t >= p.M) continue;
              const float h = __fmul_rn(xch[j * 32 + lane], __uint_as_float(v[j]));
              for (int di = 0; di < p.n_dst; ++di) {
                if (p.out_f16)
                  static_cast<__half*>(p.dst[di])[static_cast<long long>(t) * p.ldo + f] = __float2half_rn(h);
                else
                  static_cast<float*>(p.dst[di])[static_cast<long long>(t) * p.ldo + f] = h;
              }
            }
          }
          named_barrier_sync(pair_bar, 64);
          continue;
        }
        if (n < p.N) {
#pragma unroll
          for (int j = 0; j < (BN < 32 ? BN : 32); ++j) {
            const int t = c + j;
            if (t >= p.M) continue;
            const float y = __uint_as_float(v[j]);
            for (int di = 0; di < p.n_dst; ++di) {
              if (p.out_f16)
                static_cast<__half*>(p.dst[di])[static_cast<long long>(t) * p.ldo + n] = __float2half_rn(y);
              else
                static_cast<float*>(p.dst[di])[static_cast<long long>(t) * p.ldo + n] = y;
            }
          }
        }
      }
      tc_fence_before();
      if (lead && lane == 0 && !direct) p.counters[nb] = 0;
      named_barrier_sync(1, 128);  // the finalisation accumulator is free again
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, 512);
  }
}

template <int BN>
cudaError_t launch_s4(const S4Params& sp, int num_sms, cudaStream_t stream) {
  using C = S4Cfg<BN>;
  auto kern = stream4_gemm_kernel<BN>;
  cudaError_t e = ensure_smem_attr(kern, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  const long long tiles = (sp.N + kBlockM - 1) / kBlockM;
  const long long units = sp.splits ? tiles * sp.splits : tiles * sp.nstage;
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
  return cudaLaunchKernelEx(&cfg, kern, sp);
}

}  // namespace

// Measured (profiles/r2_decode_sweep.jsonl, K1 + this kernel, 10 forwards per CUDA
// graph): OPT-66B fc1 (9216 -> 36864, 256 outliers) M = 1: 33 us, M = 16: 37 us (cuBLAS
// f16: 108 us); LLaMA-2-70B up (8192 -> 28672) M = 1: 31 us; Falcon-180B fc1 M = 1: 79 us
// (cuBLAS 267 us). On for 4-bit layers at M <= 32 (QUIK_STREAM4=0 /
// quik_set_int4_decode(0) disables).
int gemm_stream4_auto = [] {
  const char* e = getenv("QUIK_STREAM4");
  return e ? atoi(e) : 1;
}();

size_t stream4_counter_count(int64_t N) { return static_cast<size_t>((N + kBlockM - 1) / kBlockM); }

cudaError_t launch_stream4(const Stream4Args& a, int num_sms, cudaStream_t stream, const char** err_msg) {
  *err_msg = nullptr;
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  if (a.M > 64) { *err_msg = "INT4 stream GEMM: M > 64"; return cudaErrorInvalidValue; }
  if ((!a.w4 && !a.w8) || a.kpad == 0) { *err_msg = "decode GEMM: no weights"; return cudaErrorInvalidValue; }
  if (a.n_peer < 0 || a.n_peer > 7) { *err_msg = "INT4 stream GEMM: at most 7 peer outputs"; return cudaErrorInvalidValue; }
  const int bn = a.M <= 16 ? 16 : (a.M <= 32 ? 32 : 64);
  S4Params sp{};
  sp.M = static_cast<int>(a.M);
  sp.N = static_cast<int>(a.N);
  sp.w8 = a.w4 ? 0 : 1;
  sp.nstage = static_cast<int>(sp.w8 ? a.kpad / 128 : (a.kpad + 255) / 256);
  sp.nout = static_cast<int>(a.opad / 64);
  // Schedule from a cost model in weight stages per CTA. Round robin with s K splits:
  // (full waves + the last wave's fill, counted as at least 0.75 of a wave: a partly
  // filled wave streams faster per CTA, the kernel being HBM-bound) x (stages per unit
  // + 1, + 4 per split unit for its workspace reduction). Stream-K: the CTA's range + 8
  // (its cut blocks finalise through the workspace at the end of the ranges), only for
  // ranges of >= 24 stages and when 15 % cheaper. Measured, M = 1: 70B up / gate
  // (224 blocks) whole blocks 27.1 us vs stream-K 30.1; Falcon-180B fc1 (464 blocks,
  // a 20-CTA last wave) stream-K 76.8 vs whole blocks 82.8 vs 3 splits 90; 7B up / gate
  // M = 16 13.8 us whole blocks vs 18.7 in 3 splits.
  const long long tiles = (a.N + kBlockM - 1) / kBlockM;
  int splits = 1;
  double best = -1.0;
  for (int s = 1; s <= 16 && s <= sp.nstage; ++s) {
    const long long units = tiles * s, full = units / num_sms, rest = units - full * num_sms;
    const double waves = static_cast<double>(full) + (rest ? std::max(0.75, static_cast<double>(rest) / num_sms) : 0.0);
    const double cost = waves * ((sp.nstage + s - 1) / s + 1 + (s > 1 ? 4 : 0));
    if (best < 0 || cost < best) { best = cost; splits = s; }
  }
  {
    const double range = std::ceil(static_cast<double>(tiles * sp.nstage) / num_sms);
    if (range >= 24 && best > 1.15 * (range + 8)) splits = 0;
  }
  static const int sched_env = [] {  // tuning: QUIK_S4_SPLITS=n forces n round-robin K splits, -1 stream-K
    const char* e = getenv("QUIK_S4_SPLITS");
    return e ? atoi(e) : 0;
  }();
  if (sched_env > 0) splits = std::min(sched_env, sp.nstage);
  if (sched_env < 0) splits = 0;
  sp.splits = splits;
  static const int prefetch_env = [] {  // tuning: QUIK_S4_PREFETCH=0 loads the outlier tiles at finalisation
    const char* e = getenv("QUIK_S4_PREFETCH");
    return e ? atoi(e) : 1;
  }();
  sp.prefetch = prefetch_env;
  sp.acc = a.acc;
  sp.counters = a.counters;
  sp.a_scale = a.a_scale;
  sp.a_zero = a.a_zero;
  sp.w_scale = a.w_scale;
  sp.wreduced = a.wreduced;
  sp.bias = a.bias;
  sp.half_range = a.half_range;
  sp.out = a.out;
  sp.ldo = a.ldo;
  sp.out_f16 = a.out_f16;
  sp.gated = a.gated;
  sp.n_dst = 1 + a.n_peer;
  sp.dst[0] = a.out;
  for (int i = 0; i < a.n_peer; ++i) sp.dst[1 + i] = a.peer_out[i];
  // the INT4 rows hold kpad / 2 bytes; a 256-K stage past kpad reads zeros (OOB fill)
  CUresult r = sp.w8 ? encode_map_2d(&sp.tm_w, a.w8, a.kpad, a.N, a.kpad, kKBlockBytes, kBlockM, true)
                     : encode_map_2d(&sp.tm_w, a.w4, a.kpad / 2, a.N, a.kpad / 2, kKBlockBytes, kBlockM, true);
  if (r == CUDA_SUCCESS) r = encode_map_2d(&sp.tm_x, a.x, a.kpad, a.M, a.kpad, kKBlockBytes, static_cast<uint32_t>(bn), true);
  if (r == CUDA_SUCCESS && sp.nout) {
    r = encode_map_2d(&sp.tm_wo, a.wo, a.opad * 2, a.N, a.opad * 2, kKBlockBytes, kBlockM, true);
    if (r == CUDA_SUCCESS)
      r = encode_map_2d(&sp.tm_xo, a.xo, a.opad * 2, a.M, a.opad * 2, kKBlockBytes, static_cast<uint32_t>(bn), true);
  }
  if (r != CUDA_SUCCESS) { *err_msg = "INT4 stream GEMM: tensor map encode failed"; return cudaErrorInvalidValue; }
  switch (bn) {
    case 16: return launch_s4<16>(sp, num_sms, stream);
    case 32: return launch_s4<32>(sp, num_sms, stream);
    default: return launch_s4<64>(sp, num_sms, stream);
  }
}

}  // namespace quikb200
