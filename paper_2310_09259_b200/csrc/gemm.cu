// K2+K3+K4: the fused QUIK linear kernel for sm_100a.
//
// For one layer call (reference runtime.cpp:246-318, V3 path :279-303):
//   acc[n][t] = sum_k W8[n][k] * X8[t][k]                   tcgen05 kind::i8, exact int32 in TMEM
//   init      = bias[n] + dequant_element(acc, ...)         epilogue, in place in TMEM (f32)
//   D         = init + sum_o Wo[n][o] * Xo[t][o]            tcgen05 kind::f16 accumulating onto init
//   y[t][n]   = f16(D)                                      epilogue -> smem -> TMA store
// dequant_element is evaluated op by op (runtime.cpp:70-77) so the whole layer is
// bit-identical to the reference when it has no outliers; with outliers the only
// difference is the summation order of the f16 products (SURVEY.md A.3 tolerance).
//
// "Swap-AB" orientation: weight rows are the UMMA M dimension, tokens are the
// UMMA N dimension (BN per tile), so small token counts use narrow N tiles.
// CG = 2 (large M): a CTA pair runs tcgen05.mma.cta_group::2 with M = 256; each
// CTA stages its own 128 weight rows and half of the BN token rows; the leader
// issues the MMAs, both CTAs' TMA loads complete on the leader's barrier, MMA
// commits are multicast to both CTAs.
//
// TMEM: two accumulator buffers of BN columns. Per tile the MMA warp issues
//   int k-blocks [0, kb/2) of tile i | outlier k-blocks of tile i-1 | int k-blocks [kb/2, kb) of tile i
// so that the epilogue's two passes over tile i-1 (convert int32 -> f32 init in
// place, then drain the finished f32 tile) overlap the integer MMAs of tile i.
//
// Warp roles (384 threads, 1 CTA per SM, persistent over tiles; 512 with W4):
//   warp 0      TMA producer (one lane)
//   warp 1      MMA issuer  (one lane, leader CTA only)
//   warp 2      TMEM allocator
//   warps 4..11 epilogue (TMEM lane quadrant = warp % 4, column half = (warp - 4) / 4)
//   warps 12..15 W4 only: INT4 -> INT8 widening of the weight tiles into TMEM
//
// W4 (4-bit layers; the default for them): the weights stay INT4 in HBM (half the
// bytes of an INT8 copy; packed.hpp:11-16 widened once per use instead of once per
// call, packed.cpp:110-111). Each CTA TMA-loads its 128 x 64-byte INT4 tile (64-byte
// swizzle) into the stage with its own barrier; four widening warps (one per TMEM lane
// quadrant, thread = weight row) sign-extend the nibbles and tcgen05.st the int8 row
// into a TMEM A-operand ring (lane = row, column j = k 4j..4j+3) as 16 x the value (the
// nibble in the high half of the byte: one or two logic ops per word; the epilogue
// shifts the exact int32 sums right by 4); the MMA warp issues tcgen05.mma kind::i8
// with A from TMEM and the activation codes from shared memory.
// The widened operand never touches shared memory, so per stage the SM's shared
// memory moves 8 KB of INT4 weights (TMA in + one read) instead of 16 KB twice.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>
#include <cstdio>

#include "kernels.h"
#include "sm100.cuh"

namespace quikb200 {

namespace {

constexpr int kEpiWarp0 = 4;
constexpr int kEpiWarps = 8;
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
constexpr int kWidenWarp0 = kEpiWarp0 + kEpiWarps;  // W4: warps 12..19 widen INT4 -> TMEM
constexpr int kWidenGroups = 2;                     // W4: widening warp groups (4 warps = 4 lane quadrants each)
constexpr int kThreadsW4 = kThreads + kWidenGroups * 4 * 32;
constexpr int kAStagesMax = 8;                      // W4: TMEM A-operand ring (32 columns each)
constexpr int kChunk = 32;                                     // tokens per epilogue step
constexpr int kStoreBufBytes = kChunk * 32 * 2;                // [32 tokens][32 features] f16
constexpr int kStagingBytes = kEpiWarps * 2 * kStoreBufBytes;  // double-buffered per warp

// SP (2:4 sparse base weights): one integer stage covers 256 logical K: the
// compressed weight tile (128 rows x 128 B = 256 logical K), two 128-byte swizzle
// atoms of activations and the 4 KB metadata tile [2 halves][128 rows][16 B],
// which the MMA warp copies into a TMEM ring (tcgen05.cp) ahead of the 4
// tcgen05.mma.sp (K = 64 each) that read it.
constexpr int kMetaSlots = 4;     // TMEM metadata ring (8 columns per stage)
constexpr int kMetaTileBytes = 4096;

// W4: the packed 4-bit weight tile of one k-block (128 rows x 64 B = 128 K, device
// nibble layout: byte i of 16-byte chunk c holds k = 32c + i (low nibble) and
// k = 32c + 16 + i (high nibble), two's complement), in the A region of the stage.
constexpr int kA4Bytes = kBlockM * kKBlockBytes / 2;  // 8 KB

template <int CG, int BN, bool SP = false, bool W4 = false>
struct Cfg {
  static constexpr int kBRows = BN / CG;                  // token rows staged per CTA
  static constexpr int kABytes = kBlockM * kKBlockBytes;  // 16 KB: 128 weight rows per CTA
  static constexpr int kBAtomBytes = kBRows * kKBlockBytes;
  static constexpr int kBBytes = kBAtomBytes * (SP ? 2 : 1);
  static constexpr int kMetaBytes = SP ? kMetaTileBytes : 0;
  // W4: the main ring carries only activation tiles; the INT4 weight tiles have their own
  // ring (released by the widening warps as soon as they have read a tile, so the HBM
  // weight stream is not held up by the MMAs) and the f16 outlier-weight tiles a two-slot
  // ring of their own.
  static constexpr int kStageBytes = W4 ? 2 * kBBytes : kABytes + kBBytes + kMetaBytes;  // W4: a k-block pair
  static constexpr int kA4Slots = 4;  // W4: INT4 ring slots of one k-block PAIR (2 x 8 KB) each
  static constexpr int kOASlots = 2;
  static constexpr int kRingFixed = W4 ? kOASlots * kABytes + kA4Slots * 2 * kA4Bytes : 0;
  static constexpr int kBudget = 227 * 1024 - 1024 - kStagingBytes - 1024 - kRingFixed;
  static constexpr int kStages = (kBudget / kStageBytes) > 8 ? 8 : (kBudget / kStageBytes);
  static constexpr int kOAOff = kStages * kStageBytes;             // W4: outlier-weight ring
  static constexpr int kA4Off = kOAOff + kOASlots * kABytes;       // W4: INT4 weight ring
  static constexpr int kAccCols = 2 * BN;                 // two accumulator buffers
  static constexpr int kMetaCol = kAccCols;               // SP: metadata ring after the accumulators
  static constexpr int kACol = kAccCols;                  // W4: A-operand ring after the accumulators
  // W4: as many 32-column A slots as fit next to the accumulators (up to 8): a slot is
  // reused only after the MMAs that read it completed, so the ring depth has to cover the
  // widen -> MMA -> commit round trip
  static constexpr int kAStages = (512 - kAccCols) / 32 > kAStagesMax ? kAStagesMax : (512 - kAccCols) / 32;
  static constexpr int kAPairs = kAStages / 2;  // W4: the ring is used in 64-column k-block pairs
  static constexpr int kTmemNeed = kAccCols + (SP ? 8 * kMetaSlots : 0) + (W4 ? 32 * kAStages : 0);
  static constexpr int kTmemCols = kTmemNeed <= 32 ? 32 : kTmemNeed <= 64 ? 64 : kTmemNeed <= 128 ? 128
                                 : kTmemNeed <= 256 ? 256 : 512;
  static_assert(kTmemNeed <= 512, "TMEM: accumulators + metadata / A-operand ring");
  static constexpr int kBarBytes = 1024;  // mbarriers + TMEM slot
  static constexpr int kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes + kRingFixed + kStagingBytes +
                                    kBarBytes;
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
  static constexpr int kTileRows = kBlockM * CG;          // weight rows per (cluster) tile
  static constexpr int kIntStageBytes = kABytes + kBBytes + kMetaBytes;  // expect-tx per CTA (not W4)
  static constexpr int kOutStageBytes = kABytes + kBAtomBytes;
};

struct KParams {
  CUtensorMap tm_w;   // int8 [N][kpad] (SP: compressed [N][kpad / 2]), box {128 B, 128 rows}
  CUtensorMap tm_e;   // SP: metadata [2 * n_kb * n_pad rows][16 B], box {16 B, 128 rows}
  CUtensorMap tm_w4;  // W4: packed int4 weights [N][kpad / 2], box {64 B, 128 rows}, 64-byte swizzle
  CUtensorMap tm_x;   // int8 [M][kpad], box {128 B, BN/CG rows}
  CUtensorMap tm_wo;  // f16 [N][opad], box {64, 128}
  CUtensorMap tm_xo;  // f16 [M][opad], box {64, BN/CG}
  CUtensorMap tm_y;   // f16 [M][ldo] output, box {32 features, 32 tokens} (valid when tma_store)
  int tma_store;
  int w_policy;  // L2 policy of the weight tiles: 0 normal, 1 evict_first, 2 evict_last
  int M, N;
  int kb_int, kb_out;
  const float* w_scale;
  const float* wreduced;
  const float* bias;
  const float* a_scale;
  const float* a_zero;
  float half_range;
  void* out;
  long long ldo;
  const int32_t* acc_in;
  long long ld_acc;
  int32_t* acc_clear;
  int meta_rows;  // SP: n_pad = round_up(N, 128) rows per metadata (stage, half) plane
  int split_num;  // h_a = kb_int * split_num / 8
  int dbg;        // diagnostics (QUIK_W4_DBG): skip W4 synchronisation steps to locate the
                  // bottleneck; results are garbage when non-zero. Never for results.
  // gated MLP: weight rows interleave up / gate in blocks of 32
  // (combined row 64b + w: w < 32 -> up feature 32b + w, else gate feature 32b + w - 32);
  // the epilogue emits h[t][f] = silu(gate) * up into an [M][N / 2] output
  int gated;
  // diagnostics (QUIK_GEMM_TRACE): per leader CTA and tile iteration (< kTraceTiles),
  // kTraceSlots globaltimer stamps; null in normal runs
  long long* trace;
  // fused all-gather: each output tile is also stored through these maps (peer outputs)
  int n_peer;
  CUtensorMap tm_peer[kMaxPeerOut];
  // gated MLP block: the down projection's per-token base min / max keys (GemmArgs::hstat)
  uint4* hstat;
  const uint32_t* hmask;
  int* herr;
};
__device__ __forceinline__ __half2 u2h2(uint32_t u) {
  __half2 h;
  memcpy(&h, &u, 4);
  return h;
}
constexpr int kTraceTiles = 64;
__device__ long long g_wstamps[2 * 128 * 8];  // W4 MMA / widening clock64 stamps (QUIK_GEMM_TRACE)
constexpr int kTraceSlots = 16;
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// slots: 0 MMA before tempty wait, 1 after it, 2 first-half int issued, 3 after tconv
// wait, 4 all issued, 5 summed full-barrier wait (ns); 6 epi before tint wait, 7 after,
// 8 pass 1 done, 9 after tfin wait, 10 pass 2 done; 11 MMA summed W4 ready wait (ns);
// W4 widening warp 12 of the leader: 12 summed full4 wait, 13 summed aempty wait,
// 14 tile start, 15 tile end

// Arrive on the barrier of this CTA pair's leader (cluster rank `leader_rank`).
template <int CG>
__device__ __forceinline__ void arrive_leader(uint64_t* bar, uint32_t leader_rank) {
  if constexpr (CG == 2) mbar_arrive_cluster(bar, leader_rank);
  else mbar_arrive(bar);
}

// MC (CG == 2 only): clusters of 4 CTAs = 2 CTA pairs that compute the tiles of two
// adjacent weight blocks on the same token block. The activation (B) tiles are
// identical for both pairs, so each is fetched once: CTA (pair p, rank r) loads
// half p of its B rows and TMA-multicasts it to (0, r) and (1, r). A stage is
// refilled only after both pairs' MMAs released it (empty barriers count 2, the
// MMA commits multicast to all 4 CTAs). Halves the L2->SM traffic of B.
template <int CG, int BN, int MODE, bool SP, bool MC, bool W4>
__global__ void __launch_bounds__(W4 ? kThreadsW4 : kThreads, 1) quik_gemm_kernel(const __grid_constant__ KParams p) {
  using C = Cfg<CG, BN, SP, W4>;
  static_assert(!MC || CG == 2, "multicast clusters pair CTA pairs");
  static_assert(!(W4 && (SP || MC)), "W4 is a dense-weight variant");
  constexpr int CL = MC ? 4 : CG;  // CTAs per cluster
  constexpr bool kAccGlobal = MODE == kModeAccInitF32 || MODE == kModeAccInitF16;
  constexpr bool kF16Out = MODE == kModeF16 || MODE == kModeAccInitF16 || MODE == kModeF16Stats;
  constexpr bool kStats = MODE == kModeF16Stats;  // gated MLP block: down K1 statistics
  constexpr bool kInt32Out = MODE == kModeInt32;
  constexpr bool kProbe = MODE == kModeProbe;

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned, derived by pointer arithmetic so the compiler keeps the shared
  // address space (STS / LDS instead of generic stores in the epilogue staging)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* staging = smem + C::kStages * C::kStageBytes + C::kRingFixed;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + kStagingBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tint = empty + C::kStages;  // [2] int MMAs of the tile done        (MMA -> epilogue)
  uint64_t* tconv = tint + 2;           // [2] init written into TMEM          (epilogue -> MMA)
  uint64_t* tfin = tconv + 2;           // [2] outlier MMAs done, tile final   (MMA -> epilogue)
  uint64_t* tempty = tfin + 2;          // [2] accumulator buffer drained      (epilogue -> MMA)
  uint64_t* full4 = tempty + 2;          // [kA4Slots] W4: this CTA's INT4 pair landed (TMA -> widen)
  uint64_t* empty4 = full4 + C::kA4Slots; // [kA4Slots] W4: INT4 pair read (widen -> producer)
  uint64_t* emptyo = empty4 + C::kA4Slots; // [kOASlots] W4: outlier-weight tile consumed (MMA -> producer)
  uint64_t* ready = emptyo + C::kOASlots; // [kAStages] W4: TMEM A slot widened, both CTAs (widen -> MMA)
  uint64_t* aempty = ready + kAStagesMax; // [kAStages] W4: TMEM A slot consumed (MMA -> widen)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + kAStagesMax);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t crank = CG == 2 ? cluster_ctarank() : 0u;
  const uint32_t rank = crank & 1u;   // rank inside the CTA pair
  const uint32_t pair = crank >> 1;   // pair inside the cluster (MC)
  const uint32_t leader_rank = crank & ~1u;
  const bool leader = rank == 0;
  const uint16_t pair_mask = static_cast<uint16_t>(3u << (2 * pair));

  const int kb_int = kAccGlobal ? 0 : p.kb_int;
  const int kb_out = kInt32Out ? 0 : p.kb_out;
  const bool two_phase = kb_out > 0;
  // int k-blocks of tile i issued before the outlier MMAs of tile i-1: the epilogue's
  // in-place dequantisation of tile i-1 must finish within them (p.split_num / 8)
  // (W4: even, the integer k-blocks go in pairs)
  const int h_a = W4 ? (((kb_int * p.split_num) >> 3) & ~1) : ((kb_int * p.split_num) >> 3);

  if (warp == 0 && lane == 0) {
    if (kb_int) { tma_prefetch(&p.tm_w); tma_prefetch(&p.tm_x); }
    if (SP && kb_int) tma_prefetch(&p.tm_e);
    if (W4 && kb_int) tma_prefetch(&p.tm_w4);
    if (kb_out) { tma_prefetch(&p.tm_wo); tma_prefetch(&p.tm_xo); }
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < C::kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], MC ? 2 : 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tint[i], 1);
      mbar_init(&tconv[i], kEpiWarps * CG);
      mbar_init(&tfin[i], 1);
      mbar_init(&tempty[i], kEpiWarps * CG);
    }
    if (W4) {
      for (int i = 0; i < C::kA4Slots; ++i) { mbar_init(&full4[i], 1); mbar_init(&empty4[i], 4); }
      for (int i = 0; i < C::kOASlots; ++i) mbar_init(&emptyo[i], 1);
      for (int i = 0; i < C::kAPairs; ++i) { mbar_init(&ready[i], 4 * CG); mbar_init(&aempty[i], 1); }
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<CG>(tmem_slot, C::kTmemCols);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: everything above overlapped the previous kernel
  // (the quantizer); wait for its results before touching them. Dense tiles: the
  // producer first issues the weight loads of its first ring stages (weights do not
  // depend on K1) and waits before the token tiles; the epilogue waits before reading
  // the per-token scales; the MMA warp only reads what the producer staged.
  constexpr bool kEarlyW = !MC && !W4;  // (W4: its own early-weight path in the producer)
  if constexpr (!kEarlyW && !W4) asm volatile("griddepcontrol.wait;" ::: "memory");

  const int tiles_m = (p.M + BN - 1) / BN;
  const int tiles_n = (p.N + C::kTileRows - 1) / C::kTileRows;
  // work units: tiles, or (MC) pairs of weight blocks on one token block
  const int num_tiles = tiles_m * (MC ? (tiles_n + 1) / 2 : tiles_n);
  const int cluster_id = blockIdx.x / CL;
  const int num_clusters = gridDim.x / CL;
  auto decode = [&](int tile, int& nb, int& mb) {
    nb = MC ? 2 * (tile / tiles_m) + static_cast<int>(pair) : tile / tiles_m;
    mb = tile % tiles_m;
  };
  // Tile order: consecutive tile ids share the weight block (n) so the clusters
  // that run concurrently read the same weight rows through L2.

  if (W4 && warp == 3) {
    // ---------------------------------------------------------------- W4 weight producer
    // INT4 weight tiles stream on their own thread, paced only by the widening warps
    // (empty4), so the HBM weight stream runs a full weight ring ahead of the widening
    // instead of being held to the activation ring's pace by one thread's program order.
    if (lane == 0) {
      const uint64_t pol_w =
          p.w_policy == 1 ? policy_evict_first() : (p.w_policy == 2 ? policy_evict_last() : policy_evict_normal());
      int a4 = 0;
      uint32_t aph = 0;
      // (weights only: no griddepcontrol.wait, the loads overlap K1 under PDL)
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        int nb, mb;
        decode(tile, nb, mb);
        const int wr = nb * C::kTileRows + static_cast<int>(rank) * kBlockM;
        for (int run = 0; run < 2; ++run) {  // the k-block pairs in the MMA warp's order
          const int k0 = run ? h_a : 0, k1 = run ? kb_int : h_a;
          for (int kb = k0; kb < k1; kb += 2) {
            const int n = kb + 1 < k1 ? 2 : 1;
            mbar_wait(&empty4[a4], aph ^ 1);
            mbar_arrive_expect_tx(&full4[a4], n * kA4Bytes);
            for (int i = 0; i < n; ++i)
              tma_load_2d(smem + C::kA4Off + (2 * a4 + i) * kA4Bytes, &p.tm_w4, (kb + i) * (kKBlockBytes / 2), wr,
                          &full4[a4], pol_w);
            if (++a4 == C::kA4Slots) { a4 = 0; aph ^= 1; }
          }
        }
      }
    }
  } else if (W4 && warp == 0) {
    // ---------------------------------------------------------------- W4 activation producer
    if (lane == 0) {
      const uint64_t pol_w =
          p.w_policy == 1 ? policy_evict_first() : (p.w_policy == 2 ? policy_evict_last() : policy_evict_normal());
      const uint64_t pol_x = policy_evict_last();
      int b = 0, o = 0;
      uint32_t bph = 0, oph = 0;
      // pair form for CG == 2: both CTAs' tiles complete on the leader's barrier
      auto tma_pair = [&](void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar, uint64_t pol) {
        if constexpr (CG == 1) tma_load_2d(dst, m, c0, c1, bar, pol);
        else tma_load_2d_pair(dst, m, c0, c1, bar, pol);
      };
      // activation codes of the k-block pair (kb, kb + 1 < k_end) -> one main-ring stage
      auto load_b = [&](int kb, int k_end, int trow) {
        const int n = kb + 1 < k_end ? 2 : 1;
        mbar_wait(&empty[b], bph ^ 1);
        if (leader) mbar_arrive_expect_tx(&full[b], CG * n * C::kBBytes);
        for (int i = 0; i < n; ++i)
          tma_pair(smem + b * C::kStageBytes + i * C::kBBytes, &p.tm_x, (kb + i) * kKBlockBytes, trow, &full[b],
                   pol_x);
        if (++b == C::kStages) { b = 0; bph ^= 1; }
      };
      // outlier block ko: f16 weight tile -> outlier ring, f16 activations -> main ring,
      // both on the main ring's full barrier
      auto load_out = [&](int ko, int wrow, int trow) {
        mbar_wait(&emptyo[o], oph ^ 1);
        mbar_wait(&empty[b], bph ^ 1);
        if (leader) mbar_arrive_expect_tx(&full[b], CG * (C::kABytes + C::kBBytes));
        tma_pair(smem + C::kOAOff + o * C::kABytes, &p.tm_wo, ko * 64, wrow, &full[b], pol_w);
        tma_pair(smem + b * C::kStageBytes, &p.tm_xo, ko * 64, trow, &full[b], pol_x);
        if (++o == C::kOASlots) { o = 0; oph ^= 1; }
        if (++b == C::kStages) { b = 0; bph ^= 1; }
      };
      auto rows_of = [&](int tile, int& wrow, int& trow) {
        int nb, mb;
        decode(tile, nb, mb);
        wrow = nb * C::kTileRows + static_cast<int>(rank) * kBlockM;
        trow = mb * BN + static_cast<int>(rank) * C::kBRows;
      };
      asm volatile("griddepcontrol.wait;" ::: "memory");  // K1's codes are complete
      int prev = -1;
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        int wr, tr;
        rows_of(tile, wr, tr);
        if (tile + num_clusters >= num_tiles) asm volatile("griddepcontrol.launch_dependents;");
        for (int kb = 0; kb < h_a; kb += 2) load_b(kb, h_a, tr);
        if (two_phase && prev >= 0) {
          int pw, pt;
          rows_of(prev, pw, pt);
          for (int ko = 0; ko < kb_out; ++ko) load_out(ko, pw, pt);
        }
        for (int kb = h_a; kb < kb_int; kb += 2) load_b(kb, kb_int, tr);
        prev = tile;
      }
      if (two_phase && prev >= 0) {
        int pw, pt;
        rows_of(prev, pw, pt);
        for (int ko = 0; ko < kb_out; ++ko) load_out(ko, pw, pt);
      }
    }
  } else if (W4 && warp == 1) {
    // ---------------------------------------------------------------- W4 MMA issuer
    // the whole (converged) warp runs the loop and one elected lane issues each MMA /
    // commit: back-to-back UTC*MMA instead of a per-instruction ELECT / branch loop
    // (~13 vs ~45-70 cycles per MMA, tools/ts_rate.cu), which at BN = 192 (96 cycles
    // of tensor work per K = 32 step) decides whether the tensor pipe stays busy
    if (leader) {
      constexpr uint32_t id_i8 = idesc_make(2u, 1u, kBlockM * CG, BN);
      constexpr uint32_t id_f16 = idesc_make(1u, 0u, kBlockM * CG, BN);
      int b = 0, o = 0, aslot = 0;
      uint32_t bph = 0, aph = 0;
      long long full_wait = 0, ready_wait = 0;
      int mit = 0;
      // k-block pairs: one activation-stage check, one widened-slot check, 8 MMAs and two
      // commits per pair (the per-k-block synchronisation is what bounds the MMA warp)
      auto int_blocks = [&](uint32_t d, int k0, int k1) {
        for (int kb = k0; kb < k1; kb += 2) {
          const int n = kb + 1 < k1 ? 2 : 1;
          long long* ms = (p.trace && cluster_id == 0 && mit < 128 && lane == 0) ? g_wstamps + mit * 8 : nullptr;
          ++mit;
          if (ms) ms[0] = clock64();
          mbar_wait(&full[b], bph);
          if (ms) ms[1] = clock64();
          mbar_wait(&ready[aslot], aph);
          if (ms) ms[2] = clock64();
          tc_fence_after();
          const uint64_t bd = umma_desc_sw128(smem_u32(smem + b * C::kStageBytes));
          const uint32_t a_tm = tmem_base + C::kACol + aslot * 64;  // both CTAs widened their rows here
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            if (i < n) {
#pragma unroll
              for (int k = 0; k < 4; ++k)  // 4 x K=32 int8 = 32 TMEM columns of A, 128 bytes of B
                mma_i8_ts_w<CG>(d, a_tm + 32 * i + 8 * k, bd + ((i * C::kBBytes) >> 4) + 2 * k, id_i8,
                                ((kb + i) | k) != 0);
            }
          }
          if (ms) ms[3] = clock64();
          mma_commit_w<CG>(&empty[b], static_cast<uint16_t>(3));
          mma_commit_w<CG>(&aempty[aslot], static_cast<uint16_t>(3));
          if (ms) ms[4] = clock64();
          if (++b == C::kStages) { b = 0; bph ^= 1; }
          if (++aslot == C::kAPairs) { aslot = 0; aph ^= 1; }
        }
      };
      auto out_blocks = [&](int it_prev) {
        const int bp = it_prev & 1;
        mbar_wait(&tconv[bp], (it_prev >> 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem_base + bp * BN;
        for (int ko = 0; ko < kb_out; ++ko) {
          mbar_wait(&full[b], bph);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(smem_u32(smem + C::kOAOff + o * C::kABytes));
          const uint64_t bd = umma_desc_sw128(smem_u32(smem + b * C::kStageBytes));
#pragma unroll
          for (int k = 0; k < 4; ++k)  // 4 x K=16 f16 = 128 bytes, accumulating onto init
            mma_f16_w<CG>(d, ad + 2 * k, bd + 2 * k, id_f16, 1u);
          mma_commit_w<CG>(&empty[b], static_cast<uint16_t>(3));
          mma_commit_w<CG>(&emptyo[o], static_cast<uint16_t>(3));
          if (++b == C::kStages) { b = 0; bph ^= 1; }
          if (++o == C::kOASlots) o = 0;
        }
        mma_commit_w<CG>(&tfin[bp], pair_mask);
      };
      int it = 0;
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters, ++it) {
        const int bb = it & 1;
        long long* tr =
            (p.trace && it < kTraceTiles && lane == 0) ? p.trace + (cluster_id * kTraceTiles + it) * kTraceSlots : nullptr;
        if (tr) { tr[0] = gtime(); full_wait = 0; ready_wait = 0; }
        mbar_wait(&tempty[bb], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        if (tr) tr[1] = gtime();
        const uint32_t d = tmem_base + bb * BN;
        int_blocks(d, 0, h_a);
        if (tr) tr[2] = gtime();
        if (two_phase && it > 0) out_blocks(it - 1);
        if (tr) tr[3] = gtime();
        int_blocks(d, h_a, kb_int);
        mma_commit_w<CG>(&tint[bb], pair_mask);
        if (tr) { tr[4] = gtime(); tr[5] = full_wait; tr[11] = ready_wait; }
      }
      if (two_phase && it > 0) out_blocks(it - 1);
    }
  } else if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w =
          p.w_policy == 1 ? policy_evict_first() : (p.w_policy == 2 ? policy_evict_last() : policy_evict_normal());
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      auto tma = [&](void* dst, const CUtensorMap* m, int c0, int c1, uint64_t pol) {
        if constexpr (CG == 1) tma_load_2d(dst, m, c0, c1, &full[stage], pol);
        else tma_load_2d_pair(dst, m, c0, c1, &full[stage], pol);
      };
      // B (token) tile of this CTA: MC -> half `pair`, multicast to both pairs
      const uint16_t mc_mask = static_cast<uint16_t>((1u << rank) | (1u << (2 + rank)));
      auto tma_b = [&](uint8_t* dst, const CUtensorMap* m, int c0, int trow, uint64_t pol) {
        if constexpr (MC) {
          constexpr int kHalfRows = C::kBRows / 2;
          tma_load_2d_pair_mc(dst + pair * kHalfRows * kKBlockBytes, m, c0, trow + static_cast<int>(pair) * kHalfRows,
                              &full[stage], mc_mask, pol);
        } else {
          tma(dst, m, c0, trow, pol);
        }
      };
      // outlier block (or dense integer block): A + one B atom at column kc
      auto load = [&](const CUtensorMap* ma, const CUtensorMap* mx, int kc, int wrow, int trow) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * C::kStageBytes;
        if (leader) mbar_arrive_expect_tx(&full[stage], CG * C::kOutStageBytes);
        tma(sa, ma, kc, wrow, pol_w);
        tma_b(sa + C::kABytes, mx, kc, trow, pol_x);
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      };
      // integer block kb: dense = load(); SP = compressed A + two B atoms + metadata tile
      auto load_int = [&](int kb, int wrow, int trow) {
        if constexpr (!SP) {
          load(&p.tm_w, &p.tm_x, kb * kKBlockBytes, wrow, trow);
        } else {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::kStageBytes;
          uint8_t* sb = sa + C::kABytes;
          uint8_t* se = sb + C::kBBytes;
          if (leader) mbar_arrive_expect_tx(&full[stage], CG * C::kIntStageBytes);
          tma(sa, &p.tm_w, kb * kKBlockBytes, wrow, pol_w);
          tma_b(sb, &p.tm_x, kb * 2 * kKBlockBytes, trow, pol_x);
          tma_b(sb + C::kBAtomBytes, &p.tm_x, kb * 2 * kKBlockBytes + kKBlockBytes, trow, pol_x);
          tma(se, &p.tm_e, 0, (2 * kb) * p.meta_rows + wrow, pol_w);
          tma(se + kMetaTileBytes / 2, &p.tm_e, 0, (2 * kb + 1) * p.meta_rows + wrow, pol_w);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      };
      auto rows_of = [&](int tile, int& wrow, int& trow) {
        int nb, mb;
        decode(tile, nb, mb);
        wrow = nb * C::kTileRows + static_cast<int>(rank) * kBlockM;
        trow = mb * BN + static_cast<int>(rank) * C::kBRows;
      };
      int pre = 0;  // integer blocks of the first tile whose weight tiles went out early
      if constexpr (kEarlyW) {
        int wr0 = 0, tr0 = 0;
        if (cluster_id < num_tiles) {
          rows_of(cluster_id, wr0, tr0);
          pre = h_a < C::kStages ? h_a : C::kStages;
          for (int kb = 0; kb < pre; ++kb) {  // fresh ring stages 0 .. pre-1
            stage = kb;
            uint8_t* sa = smem + kb * C::kStageBytes;
            if (leader) mbar_arrive_expect_tx(&full[kb], CG * (SP ? C::kIntStageBytes : C::kOutStageBytes));
            tma(sa, &p.tm_w, kb * kKBlockBytes, wr0, pol_w);
            if constexpr (SP) {  // 2:4 metadata of the stage (a weight-side tensor too)
              uint8_t* se = sa + C::kABytes + C::kBBytes;
              tma(se, &p.tm_e, 0, (2 * kb) * p.meta_rows + wr0, pol_w);
              tma(se + kMetaTileBytes / 2, &p.tm_e, 0, (2 * kb + 1) * p.meta_rows + wr0, pol_w);
            }
          }
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");  // K1's codes are complete
        for (int kb = 0; kb < pre; ++kb) {
          stage = kb;
          uint8_t* sb = smem + kb * C::kStageBytes + C::kABytes;
          if constexpr (SP) {
            tma_b(sb, &p.tm_x, kb * 2 * kKBlockBytes, tr0, pol_x);
            tma_b(sb + C::kBAtomBytes, &p.tm_x, kb * 2 * kKBlockBytes + kKBlockBytes, tr0, pol_x);
          } else {
            tma_b(sb, &p.tm_x, kb * kKBlockBytes, tr0, pol_x);
          }
        }
        stage = pre == C::kStages ? 0 : pre;
        phase = pre == C::kStages ? 1u : 0u;
      }
      int prev = -1;
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        int wr, tr;
        rows_of(tile, wr, tr);
        // last tile of this CTA: the next kernel (the next layer's quantizer) may start
        // its prologue on SMs this grid has left
        if (tile + num_clusters >= num_tiles) asm volatile("griddepcontrol.launch_dependents;");
        for (int kb = (tile == cluster_id ? pre : 0); kb < h_a; ++kb) load_int(kb, wr, tr);
        if (two_phase && prev >= 0) {
          int pw, pt;
          rows_of(prev, pw, pt);
          for (int ko = 0; ko < kb_out; ++ko) load(&p.tm_wo, &p.tm_xo, ko * 64, pw, pt);
        }
        for (int kb = h_a; kb < kb_int; ++kb) load_int(kb, wr, tr);
        prev = tile;
      }
      if (two_phase && prev >= 0) {
        int pw, pt;
        rows_of(prev, pw, pt);
        for (int ko = 0; ko < kb_out; ++ko) load(&p.tm_wo, &p.tm_xo, ko * 64, pw, pt);
      }
    }
  } else if (warp == 1) {
    // converged warp, one elected lane issues (see the W4 MMA issuer)
    if (leader) {
      constexpr uint32_t id_i8 = idesc_make(2u, 1u, kBlockM * CG, BN);
      constexpr uint32_t id_f16 = idesc_make(1u, 0u, kBlockM * CG, BN);
      constexpr uint32_t id_sp = idesc_make(2u, 1u, kBlockM * CG, BN) | (1u << 2);  // sparse flag
      (void)id_sp;
      int stage = 0;
      uint32_t phase = 0;
      long long full_wait = 0;
      auto next_stage = [&](uint64_t& adesc, uint64_t& bdesc) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * C::kStageBytes);
        adesc = umma_desc_sw128(sa);
        bdesc = umma_desc_sw128(sa + C::kABytes);
      };
      auto release_stage = [&]() {
        mma_commit_w<CG>(&empty[stage], MC ? static_cast<uint16_t>(0xF) : static_cast<uint16_t>(3));
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      };
      uint32_t meta_slot = 0;
      int mit = 0;
      auto int_blocks = [&](uint32_t d, int k0, int k1) {
        for (int kb = k0; kb < k1; ++kb) {
          long long* ms = (p.trace && cluster_id == 0 && mit < 128 && lane == 0) ? g_wstamps + mit * 8 : nullptr;
          ++mit;
          if (ms) ms[0] = clock64();
          uint64_t ad, bd;
          next_stage(ad, bd);
          if (ms) { ms[1] = clock64(); ms[2] = ms[1]; }
          if constexpr (!SP) {
#pragma unroll
            for (int k = 0; k < 4; ++k)  // 4 x K=32 int8 = 128 bytes
              mma_i8_w<CG>(d, ad + 2 * k, bd + 2 * k, id_i8, (kb | k) != 0);
          } else {
            // metadata tile -> TMEM ring slot (two 128 x 128-bit copies), then 4 sparse
            // MMAs of 64 logical K: A advances 32 compressed bytes, B 64 bytes (two atoms)
            const uint32_t te = tmem_base + C::kMetaCol + meta_slot * 8;
            const uint32_t se = smem_u32(smem + stage * C::kStageBytes + C::kABytes + C::kBBytes);
            tmem_cp_128x128b_w<CG>(te, smem_desc_rows16(se));
            tmem_cp_128x128b_w<CG>(te + 4, smem_desc_rows16(se + kMetaTileBytes / 2));
            const uint64_t bd1 = bd + ((C::kBAtomBytes >> 4) & 0x3FFF);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_sp_i8_w<CG>(d, ad + 2 * k, (k < 2 ? bd : bd1) + 4 * (k & 1), id_sp, te + 2 * k, (kb | k) != 0);
            if (++meta_slot == kMetaSlots) meta_slot = 0;
          }
          if (ms) ms[3] = clock64();
          release_stage();
          if (ms) ms[4] = clock64();
        }
      };
      auto out_blocks = [&](int it_prev) {
        const int bp = it_prev & 1;
        mbar_wait(&tconv[bp], (it_prev >> 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem_base + bp * BN;
        for (int ko = 0; ko < kb_out; ++ko) {
          uint64_t ad, bd;
          next_stage(ad, bd);
#pragma unroll
          for (int k = 0; k < 4; ++k)  // 4 x K=16 f16 = 128 bytes, accumulating onto init
            mma_f16_w<CG>(d, ad + 2 * k, bd + 2 * k, id_f16, 1u);
          release_stage();
        }
        mma_commit_w<CG>(&tfin[bp], pair_mask);
      };
      int it = 0;
      for (int tile = cluster_id; tile < num_tiles; tile += num_clusters, ++it) {
        const int b = it & 1;
        long long* tr =
            (p.trace && it < kTraceTiles && lane == 0) ? p.trace + (cluster_id * kTraceTiles + it) * kTraceSlots : nullptr;
        if (tr) { tr[0] = gtime(); full_wait = 0; }
        mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        if (tr) tr[1] = gtime();
        const uint32_t d = tmem_base + b * BN;
        int_blocks(d, 0, h_a);
        if (tr) tr[2] = gtime();
        if (two_phase && it > 0) out_blocks(it - 1);
        if (tr) tr[3] = gtime();
        int_blocks(d, h_a, kb_int);
        mma_commit_w<CG>(&tint[b], pair_mask);
        if (tr) { tr[4] = gtime(); tr[5] = full_wait; }
      }
      if (two_phase && it > 0) out_blocks(it - 1);
    }
  } else if (W4 && warp >= kWidenWarp0) {
    // INT4 -> INT8 widening into the TMEM A ring, k-block by k-block in the producer's
    // order (int blocks [0, h_a) | outlier blocks of the previous tile | [h_a, kb_int)).
    // Thread = weight row r of this CTA (TMEM lane quadrant q = warp % 4). The INT4 tile
    // lands 64-byte swizzled: 16-byte chunk c of row r sits at chunk c ^ ((r >> 1) & 3),
    // so the 8 rows of a quarter warp read 8 distinct bank groups. Byte i of chunk c
    // holds k = 32c + i (low nibble) and 32c + 16 + i (high nibble): word w of the chunk
    // widens to TMEM columns 8c + w (low) and 8c + 4 + w (high).
    // Two groups of four warps (one per TMEM lane quadrant each) take alternate k-block
    // PAIRS; ring positions follow from the pair index p (INT4 pair slot p % kA4Slots,
    // TMEM pair slot p % kAPairs, parities from the wrap counts), so the groups share no
    // state; each pair is one aempty check, two widened stores, one store wait / fence
    // and one ready arrival.
    const int q = warp & 3;
    const int g = (warp - kWidenWarp0) >> 2;
    const int r = q * 32 + lane;
    const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + C::kACol;
    const int swz = (r >> 1) & 3;
    const bool tw = p.trace && leader && warp == kWidenWarp0 && lane == 0;
    // Widening as 16 x the value: the nibble moved to the HIGH half of its byte is the
    // int8 16 * v (two's complement), one or two logic ops per word instead of a
    // sign extension; the MMA sums 16 * (w * a) exactly (|acc| <= 16 * 64 * K_b < 2^31)
    // and the epilogue shifts the accumulator right by 4 (exact).
    // k-block i (0 / 1) of the pair in INT4 pair slot `sl` (its full4 already waited for)
    auto load_tile = [&](int sl, int i, uint4 (&win)[4]) {
      const uint8_t* row = smem + C::kA4Off + (2 * sl + i) * kA4Bytes + r * (kKBlockBytes / 2);
      if (p.dbg & 16) {  // diagnostics: no shared-memory reads
#pragma unroll
        for (int c = 0; c < 4; ++c) win[c] = make_uint4(r, c, 3, 4);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) win[c] = *reinterpret_cast<const uint4*>(row + ((c ^ swz) << 4));
      }
    };
    // the INT4 pair is in registers (its values consumed): hand the slot back to the producer
    auto release_tile = [&](int sl) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty4[sl]);
    };
    // one k-block: 16 INT4 words -> 32 TMEM columns (slot j) of 16 x the int8 codes
    auto widen_store = [&](const uint4 (&win)[4], long long j) {
      uint32_t v[32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const uint32_t x = (&win[c].x)[w];
          v[8 * c + w] = (x << 4) & 0xF0F0F0F0u;  // k = 32c + 4w .. +3   (low nibbles) x 16
          v[8 * c + 4 + w] = x & 0xF0F0F0F0u;     // k = 32c + 16 + 4w .. (high nibbles) x 16
        }
      }
      if (!(p.dbg & 8)) tmem_st32(trow + static_cast<uint32_t>(j) * 32, v);  // j: TMEM 32-column slot
    };
    // the k-block pairs of each tile, in the MMA warp's order: [0, h_a) then [h_a, kb_int)
    // (h_a even); pair p goes to group p % 2 and TMEM pair slot p % kAPairs; k-block j of
    // the CTA's sequence sits in INT4 slot j % kA4Slots
    long long p_idx = 0;
    int wit = 0;
    auto do_pair = [&](int n, long long pp) {
      long long* ws = (tw && cluster_id == 0 && wit < 128) ? g_wstamps + 128 * 8 + wit * 8 : nullptr;
      ++wit;
      if (ws) ws[0] = clock64();
      const int sl = static_cast<int>(pp % C::kA4Slots);
      mbar_wait(&full4[sl], static_cast<uint32_t>((pp / C::kA4Slots) & 1));
      uint4 wa[4], wb[4];
      load_tile(sl, 0, wa);
      if (n > 1) load_tile(sl, 1, wb);
      if (ws) ws[1] = clock64();
      const int ps = static_cast<int>(pp % C::kAPairs);
      mbar_wait(&aempty[ps], static_cast<uint32_t>(((pp / C::kAPairs) & 1) ^ 1));  // MMAs of its last use done
      if (ws) ws[2] = clock64();
      tc_fence_after();
      widen_store(wa, 2LL * ps);
      if (n > 1) widen_store(wb, 2LL * ps + 1);
      release_tile(sl);
      if (ws) ws[3] = clock64();
      if (!(p.dbg & 2)) tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (ws) ws[4] = clock64();
      if (lane == 0) arrive_leader<CG>(&ready[ps], leader_rank);
      if (ws) ws[5] = clock64();
    };
    for (int tile = cluster_id; tile < num_tiles; tile += num_clusters) {
      for (int run = 0; run < 2; ++run) {
        const int k0 = run ? h_a : 0, k1 = run ? kb_int : h_a;
        for (int kb = k0; kb < k1; kb += 2, ++p_idx)
          if ((p_idx & 1) == g) do_pair(kb + 1 < k1 ? 2 : 1, p_idx);
      }
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps) {
    if constexpr (kEarlyW || W4) asm volatile("griddepcontrol.wait;" ::: "memory");  // per-token scales, acc_in
    const int e = warp - kEpiWarp0;
    const int q = warp & 3;  // TMEM lane quadrant (hardware: lanes 32*(warp%4) .. +31)
    const int h = e >> 2;
    constexpr int kHalf = BN / 2 < kChunk ? kChunk : BN / 2;
    const int c_begin = h * kHalf;
    const int c_end = (c_begin + kHalf) < BN ? (c_begin + kHalf) : BN;
    uint8_t* my_stage = staging + e * 2 * kStoreBufBytes;
    int sbuf = 0;
    // kStats gate warps: the previous chunk's staged h tile, reduced while the up warp
    // works on the current one (pend_t0 < 0: none)
    const __half* pend_hb = nullptr;
    int pend_n0s = 0, pend_t0 = -1;
    // gated MLP block (kStats): the down projection's K1 reduction (runtime.cpp:36-50
    // over the base columns of h), run by the gate warp on the up warp's staged f16 tile
    // hb (features n0s .. n0s + 31, tokens t0 ..) while the up warp goes on with its
    // next chunk
    auto down_stats = [&](const __half* hb, int n0s, int t0) {
      // Transposed: lane j reads token j's 32 features (16-byte pieces rotated by lane
      // pair: conflict-free), outlier features of the down layer (fm) replaced by a
      // base value of the same token,
      // packed f16 min / max (K1's pass 1), one atomic pair per token and chunk on
      // order-preserving keys (kernels.h). Signed zeros: a chunk whose minimum is a
      // zero reports its first base zero's column and sign (the row minimum is zero
      // only if every zero-holding chunk's minimum is). Non-finite: error flag.
      const uint32_t fm = __ldg(&p.hmask[n0s >> 5]);
      const int t = t0 + lane;
      if (fm != 0xFFFFFFFFu && t < p.M) {
        const uint16_t* rowh = reinterpret_cast<const uint16_t*>(hb) + lane * 32;
        const uint4* row4 = reinterpret_cast<const uint4*>(rowh);
        const uint32_t f0 = rowh[__ffs(~fm) - 1];
        const uint32_t fill = f0 | (f0 << 16);
        __half2 mn = u2h2(0x7C007C00u), mx = u2h2(0xFC00FC00u);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int kk = (k + (lane >> 1)) & 3;
          const uint4 q4 = row4[kk];
          const uint32_t byte = (fm >> (8 * kk)) & 0xFFu;
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const uint32_t i2 = (byte >> (2 * w)) & 3u;
            const uint32_t mk = (i2 & 1u ? 0x0000FFFFu : 0u) | (i2 & 2u ? 0xFFFF0000u : 0u);
            const __half2 x2 = u2h2(((&q4.x)[w] & ~mk) | (fill & mk));
            mn = __hmin2_nan(mn, x2);
            mx = __hmax2_nan(mx, x2);
          }
        }
        const float2 fmn = __half22float2(mn), fmx = __half22float2(mx);
        const bool bad = isnan(fmn.x) || isnan(fmn.y) || isnan(fmx.x) || isnan(fmx.y) || fmx.x == INFINITY ||
                         fmx.y == INFINITY || fmn.x == -INFINITY || fmn.y == -INFINITY;
        if (bad) atomicExch(p.herr, 1);
        const float vmn = fminf(fmn.x, fmn.y), vmx = fmaxf(fmx.x, fmx.y);
        auto key = [](float v) {  // f16-exact value -> order-preserving key (+-0 -> +0)
          const uint32_t u = __half_as_ushort(__float2half_rn(v));
          const uint32_t mag = u & 0x7FFFu;
          return ((u & 0x8000u) && mag) ? 0x7FFFu - mag : (mag | 0x8000u);
        };
        atomicMin(&p.hstat[t].x, key(vmn));
        atomicMax(&p.hstat[t].y, key(vmx));
        if (vmn == 0.0f) {  // rare: this chunk's first base zero (column, sign)
#pragma unroll 1
          for (int f = 0; f < 32; ++f) {
            const uint32_t u = rowh[f];
            if (!((fm >> f) & 1u) && (u & 0x7FFFu) == 0u) {
              atomicMin(&p.hstat[t].z, (static_cast<uint32_t>(n0s + f) << 1) | (u >> 15));
              break;
            }
          }
        }
      }
    };
    const bool tma_out = kF16Out && p.tma_store;
    const uint64_t pol_y = policy_evict_first();  // the output is not re-read by this kernel
    int it = 0;
    for (int tile = cluster_id; tile < num_tiles; tile += num_clusters, ++it) {
      const int b = it & 1;
      const uint32_t par = (it >> 1) & 1;
      int nb, mb;
      decode(tile, nb, mb);
      const int n0 = nb * C::kTileRows + static_cast<int>(rank) * kBlockM + q * 32;  // warp's first feature
      const int n = n0 + lane;
      const bool n_ok = n < p.N;
      float sw = 0.f, wr = 0.f, bs = 0.f;
      if (n_ok && !kInt32Out) {
        sw = __ldg(&p.w_scale[n]);
        wr = __ldg(&p.wreduced[n]);
        if (p.bias) bs = __ldg(&p.bias[n]);
      }
      const uint32_t tacc = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + b * BN;
      // per-token activation scale / shifted zero of this warp's chunks, loaded before
      // waiting for the accumulators so their latency is off the critical path
      // (the outlier MMAs of this tile wait for the dequantisation below)
      constexpr int kMaxChunks = (kHalf + kChunk - 1) / kChunk;
      float sa_pre[kMaxChunks], zs_pre[kMaxChunks];
#pragma unroll
      for (int ci = 0; ci < kMaxChunks; ++ci) {
        const int t_l = mb * BN + c_begin + ci * kChunk + lane;
        const bool ok = !kInt32Out && t_l < p.M && c_begin + ci * kChunk < c_end;
        const float sa_l = ok ? __ldg(&p.a_scale[t_l]) : 0.f;
        const float za_l = ok ? __ldg(&p.a_zero[t_l]) : 0.f;
        sa_pre[ci] = sa_l;
        zs_pre[ci] = __fadd_rn(za_l, __fmul_rn(p.half_range, sa_l));  // runtime.cpp:74
      }
      auto pick = [&](const float (&a)[kMaxChunks], int ci) {
        float r = a[0];
#pragma unroll
        for (int k = 1; k < kMaxChunks; ++k) r = ci == k ? a[k] : r;
        return r;
      };
      long long* tr = (p.trace && leader && warp == kEpiWarp0 && lane == 0 && it < kTraceTiles)
                          ? p.trace + (cluster_id * kTraceTiles + it) * kTraceSlots
                          : nullptr;
      if (tr) tr[6] = gtime();
      if (!kAccGlobal) {
        if constexpr (W4) mbar_wait_sleep(&tint[b], par);  // idle epilogue warps yield their issue slots
        else mbar_wait(&tint[b], par);
        tc_fence_after();
      }
      if (tr) tr[7] = gtime();

      // init = bias + dequant_element(acc, ...) for 32 tokens of this warp's 32 rows
      auto dequant_chunk = [&](int c, uint32_t (&v)[32]) {
        if (kAccGlobal) {
          // all 32 loads in flight first, then the clears (acc_clear aliases acc_in)
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int t = mb * BN + c + j;
            v[j] = (t < p.M && n_ok) ? static_cast<uint32_t>(__ldcg(&p.acc_in[static_cast<long long>(t) * p.ld_acc + n]))
                                     : 0u;
          }
          if (p.acc_clear) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int t = mb * BN + c + j;
              if (t < p.M && n_ok) p.acc_clear[static_cast<long long>(t) * p.ld_acc + n] = 0;  // workspace -> zeros
            }
          }
        } else if (kb_int > 0) {
          tmem_ld32(tacc + c, v);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0u;
        }
        const int ci = (c - c_begin) / kChunk;
        const float sa_l = pick(sa_pre, ci);
        const float zs_l = pick(zs_pre, ci);
        if (!kAccGlobal && kb_int > 0) tmem_ld_wait();
        if constexpr (W4) {  // the MMAs summed 16 x the products (INT4 widening), exact
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = static_cast<uint32_t>(static_cast<int32_t>(v[j]) >> 4);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float sa = __shfl_sync(0xffffffffu, sa_l, j);
          const float zs = __shfl_sync(0xffffffffu, zs_l, j);
          float x = __fmul_rn(__int2float_rn(static_cast<int32_t>(v[j])), sa);
          x = __fmul_rn(x, sw);
          x = __fadd_rn(x, __fmul_rn(zs, wr));  // dequant_element, runtime.cpp:70-77
          v[j] = __float_as_uint(__fadd_rn(bs, x));
        }
      };
      // gated: the gate warp (odd quadrant) hands its 32 x 32 f32 values to the up warp
      // (even quadrant, same column half) through the gate warp's staging buffer; the up
      // warp forms silu(gate) * up (reference forward_model: e / (1 + exp(-e)), then the
      // Hadamard product, f32) and stores it at feature f = n / 2
      const bool gate_warp = p.gated && (q & 1);
      const int pair_bar = 1 + (e >> 1);  // named barriers 1..4, 64 threads each
      float* xch = reinterpret_cast<float*>(staging + (e | 1) * 2 * kStoreBufBytes);
      const int n0_out = p.gated ? n0 / 2 : n0;
      // writes 32 tokens x 32 features of final values
      auto emit_chunk = [&](int c, uint32_t (&v)[32]) {
        if constexpr (kProbe) return;
        if (p.gated) {
          if (gate_warp) {
            if constexpr (kStats) {
              // barrier pair_bar + 4 (up -> gate): the up warp has read the exchange
              // buffer and staged its h tile; pair_bar (gate -> up): exchange buffer full.
              // The gate warp reduces the previous chunk's h tile while the up warp forms
              // and stores the current one.
              if (pend_t0 >= 0) named_barrier_sync(pair_bar + 4, 64);
#pragma unroll
              for (int j = 0; j < 32; ++j) xch[j * 32 + lane] = __uint_as_float(v[j]);
              named_barrier_arrive(pair_bar, 64);
              if (pend_t0 >= 0 && tma_out) down_stats(pend_hb, pend_n0s, pend_t0);
              pend_hb = reinterpret_cast<const __half*>(staging + (e - 1) * 2 * kStoreBufBytes + sbuf * kStoreBufBytes);
              pend_n0s = (n0 - 32) / 2;
              pend_t0 = mb * BN + c;
              sbuf ^= 1;  // mirrors the up warp's staging buffer
              return;
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) xch[j * 32 + lane] = __uint_as_float(v[j]);
            named_barrier_sync(pair_bar, 64);
            named_barrier_sync(pair_bar, 64);  // the up warp has read the exchange buffer
            return;
          }
          named_barrier_sync(pair_bar, 64);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float g = xch[j * 32 + lane];
            // fast exp / divide (a few ulp; the reference's own std::exp differs from any
            // device exp by ulps, so the gated output is compared within tolerance)
            const float silu = __fdividef(g, 1.0f + __expf(-g));
            v[j] = __float_as_uint(__fmul_rn(silu, __uint_as_float(v[j])));
          }
          if constexpr (!kStats) named_barrier_sync(pair_bar, 64);
        }
        if (tma_out) {
          __half* buf = reinterpret_cast<__half*>(my_stage + sbuf * kStoreBufBytes);
          if (lane == 0) bulk_wait_read<1>();  // the store issued from this buffer 2 chunks ago has read it
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 32; ++j) buf[j * 32 + lane] = __float2half_rn(__uint_as_float(v[j]));
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&p.tm_y, buf, n0_out, mb * BN + c, pol_y);
            // fused all-gather: the same staged tile to every peer output (NVLink P2P
            // stores overlap the next tiles' MMAs); one bulk group covers them all
            for (int i = 0; i < p.n_peer; ++i) tma_store_2d(&p.tm_peer[i], buf, n0_out, mb * BN + c, pol_y);
            bulk_commit();
          }
          if constexpr (kStats) {
            if (p.gated) named_barrier_arrive(pair_bar + 4, 64);  // the gate warp reduces the staged tile
          }
          sbuf ^= 1;
          return;
        }
        if constexpr (kStats) {
          if (p.gated) named_barrier_arrive(pair_bar + 4, 64);  // (no statistics without TMA tiles: host-checked)
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int t = mb * BN + c + j;
          if (t >= p.M || !n_ok) continue;
          const long long off = static_cast<long long>(t) * p.ldo + (p.gated ? n0_out + lane : n);
          if (kInt32Out) reinterpret_cast<int32_t*>(p.out)[off] = static_cast<int32_t>(v[j]);
          else if (kF16Out) reinterpret_cast<__half*>(p.out)[off] = __float2half_rn(__uint_as_float(v[j]));
          else reinterpret_cast<float*>(p.out)[off] = __uint_as_float(v[j]);
        }
      };

      if (kInt32Out) {
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += kChunk) {
          uint32_t v[32];
          tmem_ld32(tacc + c, v);
          tmem_ld_wait();
          if constexpr (W4) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = static_cast<uint32_t>(static_cast<int32_t>(v[j]) >> 4);
          }
          emit_chunk(c, v);
        }
      } else if (!two_phase) {
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += kChunk) {
          uint32_t v[32];
          dequant_chunk(c, v);
          emit_chunk(c, v);
        }
      } else {
        // pass 1: init into TMEM (in place over the int32 accumulator)
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += kChunk) {
          uint32_t v[32];
          dequant_chunk(c, v);
          tmem_st32(tacc + c, v);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader<CG>(&tconv[b], leader_rank);
        if (tr) tr[8] = gtime();
        // pass 2: outlier MMAs have accumulated onto init
        if constexpr (W4) mbar_wait_sleep(&tfin[b], par);
        else mbar_wait(&tfin[b], par);
        tc_fence_after();
        if (tr) tr[9] = gtime();
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += kChunk) {
          uint32_t v[32];
          tmem_ld32(tacc + c, v);
          tmem_ld_wait();
          emit_chunk(c, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader<CG>(&tempty[b], leader_rank);
      if (tr) tr[10] = gtime();
    }
    if constexpr (kStats) {
      if (p.gated && (q & 1) && pend_t0 >= 0) {  // the last chunk's statistics
        named_barrier_sync(1 + (e >> 1) + 4, 64);
        if (tma_out) down_stats(pend_hb, pend_n0s, pend_t0);
      }
    }
    if (lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, C::kTmemCols);
  }
}

// --------------------------------------------------------------------- host side

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

bool get_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

}  // namespace

CUresult encode_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t pitch,
                       uint32_t box_inner, uint32_t box_rows, bool swizzle128) {
  if (!get_encoder()) return CUDA_ERROR_NOT_SUPPORTED;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {pitch};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

namespace {

// 2D K-major tile map with 128-byte swizzle. inner = elements per row (logical
// extent), pitch in bytes, box = {box_inner elements (128 B), box_rows}.
bool make_map(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, uint64_t inner,
              uint64_t rows, uint64_t pitch_bytes, uint32_t box_rows) {
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kKBlockBytes / elem_bytes), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int CG, int BN, int MODE, bool SP, bool MC, bool W4 = false>
cudaError_t launch_cfg(const KParams& kp, int num_sms, cudaStream_t stream) {
  using C = Cfg<CG, BN, SP, W4>;
  constexpr int CL = MC ? 4 : CG;
  auto kern = quik_gemm_kernel<CG, BN, MODE, SP, MC, W4>;
  cudaError_t e = ensure_smem_attr(kern, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  const long long tn = (kp.N + C::kTileRows - 1) / C::kTileRows;
  const long long tiles = static_cast<long long>((kp.M + BN - 1) / BN) * (MC ? (tn + 1) / 2 : tn);
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(W4 ? kThreadsW4 : kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (kernel waits via griddepcontrol)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  // persistent grid: as many clusters as can be co-resident (clusters must fit inside
  // a GPC, so num_sms / CL over-counts; a second partial wave would double the time)
  static int resident[2][2][2] = {};
  int& max_clusters = resident[CL == 4][CG == 2][W4];
  if (max_clusters == 0) {
    cfg.gridDim = dim3(static_cast<unsigned>(num_sms / CL * CL));
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
      (void)cudaGetLastError();
      n = num_sms / CL;
    }
    max_clusters = n;
  }
  const int clusters = static_cast<int>(tiles < max_clusters ? tiles : max_clusters);
  if (clusters <= 0) return cudaSuccess;
  cfg.gridDim = dim3(clusters * CL);
  return cudaLaunchKernelEx(&cfg, kern, kp);
}

template <int CG, int BN, bool MC = false>
cudaError_t launch_mode(const KParams& kp, int mode, int num_sms, cudaStream_t stream) {
  switch (mode) {
    case kModeInt32: return launch_cfg<CG, BN, kModeInt32, false, MC>(kp, num_sms, stream);
    case kModeAccInitF32: return launch_cfg<CG, BN, kModeAccInitF32, false, MC>(kp, num_sms, stream);
    case kModeAccInitF16: return launch_cfg<CG, BN, kModeAccInitF16, false, MC>(kp, num_sms, stream);
    case kModeF32: return launch_cfg<CG, BN, kModeF32, false, MC>(kp, num_sms, stream);
    case kModeProbe: return launch_cfg<CG, BN, kModeProbe, false, MC>(kp, num_sms, stream);
    case kModeF16Stats: return launch_cfg<CG, BN, kModeF16Stats, false, MC>(kp, num_sms, stream);
    default: return launch_cfg<CG, BN, kModeF16, false, MC>(kp, num_sms, stream);
  }
}

// INT4 weights from HBM widened into TMEM (4-bit dense layers, every tile)
template <int CG, int BN>
cudaError_t launch_mode_w4(const KParams& kp, int mode, int num_sms, cudaStream_t stream) {
  switch (mode) {
    case kModeInt32: return launch_cfg<CG, BN, kModeInt32, false, false, true>(kp, num_sms, stream);
    case kModeF32: return launch_cfg<CG, BN, kModeF32, false, false, true>(kp, num_sms, stream);
    case kModeProbe: return launch_cfg<CG, BN, kModeProbe, false, false, true>(kp, num_sms, stream);
    case kModeF16: return launch_cfg<CG, BN, kModeF16, false, false, true>(kp, num_sms, stream);
    case kModeF16Stats: return launch_cfg<CG, BN, kModeF16Stats, false, false, true>(kp, num_sms, stream);
    default: return cudaErrorInvalidValue;  // AccInit tails read int32 accumulators, no weights
  }
}

// 2:4 sparse base weights: the fused modes and the raw int32 accumulator (parity)
template <int CG, int BN, bool MC = false>
cudaError_t launch_mode_sp(const KParams& kp, int mode, int num_sms, cudaStream_t stream) {
  switch (mode) {
    case kModeInt32: return launch_cfg<CG, BN, kModeInt32, true, MC>(kp, num_sms, stream);
    case kModeF32: return launch_cfg<CG, BN, kModeF32, true, MC>(kp, num_sms, stream);
    case kModeProbe: return launch_cfg<CG, BN, kModeProbe, true, MC>(kp, num_sms, stream);
    case kModeF16: return launch_cfg<CG, BN, kModeF16, true, MC>(kp, num_sms, stream);
    default: return cudaErrorInvalidValue;  // V1/V2 tails read int32 accumulators: dense kernel
  }
}

constexpr int kKeyMC = 1 << 30;  // dispatch key flag: 4-CTA multicast clusters
constexpr int kKeyW4 = 1 << 29;  // dispatch key flag: INT4 weights widened into TMEM

cudaError_t launch_sp_key(int key, const KParams& kp, int mode, int num_sms, cudaStream_t stream) {
  if (key & kKeyMC) {
    switch (key & ~kKeyMC) {
      case (2 << 16) | 128: return launch_mode_sp<2, 128, true>(kp, mode, num_sms, stream);
      case (2 << 16) | 192: return launch_mode_sp<2, 192, true>(kp, mode, num_sms, stream);
      default: return cudaErrorInvalidConfiguration;
    }
  }
  switch (key) {
    case (1 << 16) | 32: return launch_mode_sp<1, 32>(kp, mode, num_sms, stream);
    case (1 << 16) | 64: return launch_mode_sp<1, 64>(kp, mode, num_sms, stream);
    case (1 << 16) | 128: return launch_mode_sp<1, 128>(kp, mode, num_sms, stream);
    case (2 << 16) | 128: return launch_mode_sp<2, 128>(kp, mode, num_sms, stream);
    case (2 << 16) | 192: return launch_mode_sp<2, 192>(kp, mode, num_sms, stream);
    default: return cudaErrorInvalidConfiguration;
  }
}

cudaError_t launch_dense_key(int key, const KParams& kp, int mode, int num_sms, cudaStream_t stream) {
  if (key & kKeyW4) {
    switch (key & ~kKeyW4) {
      case (1 << 16) | 32: return launch_mode_w4<1, 32>(kp, mode, num_sms, stream);
      case (1 << 16) | 64: return launch_mode_w4<1, 64>(kp, mode, num_sms, stream);
      case (1 << 16) | 128: return launch_mode_w4<1, 128>(kp, mode, num_sms, stream);
      case (2 << 16) | 128: return launch_mode_w4<2, 128>(kp, mode, num_sms, stream);
      case (2 << 16) | 192: return launch_mode_w4<2, 192>(kp, mode, num_sms, stream);
      default: return cudaErrorInvalidConfiguration;
    }
  }
  if (key & kKeyMC) {
    switch (key & ~kKeyMC) {
      case (2 << 16) | 128: return launch_mode<2, 128, true>(kp, mode, num_sms, stream);
      case (2 << 16) | 256: return launch_mode<2, 256, true>(kp, mode, num_sms, stream);
      default: return cudaErrorInvalidConfiguration;
    }
  }
  switch (key) {
    case (1 << 16) | 32: return launch_mode<1, 32>(kp, mode, num_sms, stream);
    case (1 << 16) | 64: return launch_mode<1, 64>(kp, mode, num_sms, stream);
    case (1 << 16) | 128: return launch_mode<1, 128>(kp, mode, num_sms, stream);
    case (2 << 16) | 128: return launch_mode<2, 128>(kp, mode, num_sms, stream);
    case (2 << 16) | 256: return launch_mode<2, 256>(kp, mode, num_sms, stream);
    default: return cudaErrorInvalidConfiguration;
  }
}

}  // namespace

int gemm_tile_override = 0;
int gemm_multicast = 0;  // 1: 4-CTA multicast clusters for CTA-pair tiles (quik_set_gemm_multicast)

cudaError_t launch_quik_gemm(const GemmArgs& a, int num_sms, cudaStream_t stream, const char** err_msg) {
  *err_msg = nullptr;
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  if (!get_encoder()) { *err_msg = "cuTensorMapEncodeTiled unavailable"; return cudaErrorNotSupported; }
  // Token tile: narrow UMMA N for small M (memory-bound weight streaming, 1-CTA);
  // CTA-pair M = 256 tiles once the token count makes the GEMM compute-bound.
  const bool sp = a.sparse && a.mode != kModeAccInitF32 && a.mode != kModeAccInitF16;
  int cg = 1, bn = 128;
  if (a.M <= 32) bn = 32;
  else if (a.M <= 64) bn = 64;
  else if (a.M <= 128) bn = 128;
  else { cg = 2; bn = sp ? 192 : 256; }  // SP: 2 x 192 accumulator columns + metadata ring in TMEM
  if (gemm_tile_override) { cg = gemm_tile_override >> 16; bn = gemm_tile_override & 0xFFFF; }
  // INT4 weights (4-bit dense layers): every tile streams them and widens into TMEM
  const bool acc_tail = a.mode == kModeAccInitF32 || a.mode == kModeAccInitF16;
  const bool w4 = a.w4 != nullptr && !sp && !acc_tail;
  // 192 is the sparse and INT4 CTA-pair tile (2 x 192 accumulator columns + the
  // metadata / A-operand ring in TMEM), 256 the INT8 one
  if ((sp || w4) && cg == 2 && bn == 256) bn = 192;
  if (!(sp || w4) && cg == 2 && bn == 192) bn = 256;

  KParams kp{};
  kp.M = static_cast<int>(a.M);
  kp.N = static_cast<int>(a.N);
  kp.kb_int = static_cast<int>(a.kpad / kKBlockBytes);
  kp.kb_out = static_cast<int>(a.opad / 64);
  const bool acc_global = a.mode == kModeAccInitF32 || a.mode == kModeAccInitF16;
  if (a.mode == kModeInt32) kp.kb_out = 0;
  if (acc_global) kp.kb_int = 0;
  kp.acc_in = a.acc_in;
  kp.ld_acc = a.ld_acc;
  kp.acc_clear = a.acc_clear;
  // QUIK_GEMM_MC=1 enables the 4-CTA multicast clusters. Off by default: measured on
  // B200 the k-loop is bound by TMA latency x shared-memory ring capacity, not by
  // L2->SM bandwidth, and fewer 4-CTA clusters fit per GPC (tools/trace_view.py).
  static const int mc_env = [] {
    const char* e = getenv("QUIK_GEMM_MC");
    return e ? atoi(e) : 0;
  }();
  const bool mc = cg == 2 && !w4 && (mc_env != 0 || gemm_multicast != 0) && !acc_tail;
  const uint32_t brows = static_cast<uint32_t>(bn / cg / (mc ? 2 : 1));
  if (kp.kb_int && sp) {
    // compressed weights [N][kpad / 2], activations [M][kpad] (two atoms per stage),
    // metadata planes [(2 * kb + h) * n_pad + row][16 B]
    if (a.kpad % (2 * kKBlockBytes) != 0) { *err_msg = "sparse layer: kpad must be a multiple of 256"; return cudaErrorInvalidValue; }
    kp.kb_int = static_cast<int>(a.kpad / (2 * kKBlockBytes));
    kp.meta_rows = static_cast<int>(round_up(a.N, kBlockM));
    cuuint64_t edims[2] = {16, static_cast<cuuint64_t>(2) * kp.kb_int * kp.meta_rows};
    cuuint64_t estr[1] = {16};
    cuuint32_t ebox[2] = {16, static_cast<cuuint32_t>(kBlockM)};
    cuuint32_t eel[2] = {1, 1};
    if (!make_map(&kp.tm_w, a.w_sp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.kpad / 2, a.N, a.kpad / 2, kBlockM) ||
        !make_map(&kp.tm_x, a.x, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.kpad, a.M, a.kpad, brows) ||
        g_encode(&kp.tm_e, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.meta), edims, estr, ebox, eel,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      *err_msg = "tensor map encode failed (sparse operands)";
      return cudaErrorInvalidValue;
    }
  } else if (kp.kb_int && w4) {
    cuuint64_t wdims[2] = {static_cast<cuuint64_t>(a.kpad / 2), static_cast<cuuint64_t>(a.N)};
    cuuint64_t wstr[1] = {static_cast<cuuint64_t>(a.kpad / 2)};
    cuuint32_t wbox[2] = {static_cast<cuuint32_t>(kKBlockBytes / 2), static_cast<cuuint32_t>(kBlockM)};
    cuuint32_t wel[2] = {1, 1};
    if (g_encode(&kp.tm_w4, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.w4), wdims, wstr, wbox, wel,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        !make_map(&kp.tm_x, a.x, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.kpad, a.M, a.kpad, brows)) {
      *err_msg = "tensor map encode failed (int4 operands)";
      return cudaErrorInvalidValue;
    }
  } else if (kp.kb_int) {
    if (!make_map(&kp.tm_w, a.w, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.kpad, a.N, a.kpad, kBlockM) ||
        !make_map(&kp.tm_x, a.x, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.kpad, a.M, a.kpad, brows)) {
      *err_msg = "tensor map encode failed (int8 operands)";
      return cudaErrorInvalidValue;
    }
  }
  if (kp.kb_out) {
    if (!make_map(&kp.tm_wo, a.wo, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.opad, a.N, a.opad * 2, kBlockM) ||
        !make_map(&kp.tm_xo, a.xo, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.opad, a.M, a.opad * 2, brows)) {
      *err_msg = "tensor map encode failed (outlier operands)";
      return cudaErrorInvalidValue;
    }
  }
  static const int w_policy = [] {
    const char* e = getenv("QUIK_W_L2_POLICY");
    return e ? atoi(e) : 0;
  }();
  kp.w_policy = w_policy;
  static const int w4_dbg = [] {
    const char* e = getenv("QUIK_W4_DBG");
    return e ? atoi(e) : 0;
  }();
  kp.dbg = w4_dbg;
  static const int split_env = [] {  // tuning: QUIK_SPLIT_NUM in 1..7 (eighths of the int k-blocks)
    const char* e = getenv("QUIK_SPLIT_NUM");
    return e ? atoi(e) : 0;
  }();
  kp.split_num = (split_env >= 1 && split_env <= 7) ? split_env : (sp ? 6 : 4);
  kp.gated = a.gated && a.mode != kModeInt32 && a.mode != kModeProbe;  // raw accumulators stay per row
  kp.hstat = (kp.gated && a.mode == kModeF16 && !sp) ? a.hstat : nullptr;  // 2:4 tiles: no statistics
  kp.hmask = a.hmask;
  kp.herr = a.herr;
  static const char* trace_path = getenv("QUIK_GEMM_TRACE");  // diagnostics: timeline dump
  static long long* trace_buf = nullptr;
  // per-cluster tile stamps, then (W4) per-iteration widening stamps of cluster 0
  const size_t trace_bytes = static_cast<size_t>(num_sms) * kTraceTiles * kTraceSlots * 8;
  if (trace_path && a.mode != kModeInt32 && a.mode != kModeProbe) {
    if (!trace_buf && cudaMalloc(&trace_buf, trace_bytes) != cudaSuccess) trace_buf = nullptr;
    if (trace_buf) cudaMemsetAsync(trace_buf, 0, trace_bytes, stream);
    kp.trace = trace_buf;
  }
  kp.tma_store = 0;
  if ((a.mode == kModeF16 || a.mode == kModeAccInitF16) && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0 &&
      (a.ldo * 2) % 16 == 0) {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.gated ? a.N / 2 : a.N), static_cast<cuuint64_t>(a.M)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ldo * 2)};
    cuuint32_t box[2] = {32, static_cast<cuuint32_t>(kChunk)};
    cuuint32_t estr[2] = {1, 1};
    kp.tma_store = g_encode(&kp.tm_y, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.out, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    for (int i = 0; kp.tma_store && i < a.n_peer; ++i) {
      if (!a.peer_out[i] || (reinterpret_cast<uintptr_t>(a.peer_out[i]) & 15) != 0 ||
          g_encode(&kp.tm_peer[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.peer_out[i], dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        *err_msg = "peer output: null, misaligned or not encodable";
        return cudaErrorInvalidValue;
      }
    }
  }
  kp.n_peer = a.n_peer;
  if (a.n_peer > kMaxPeerOut || (a.n_peer > 0 && !kp.tma_store)) {
    *err_msg = "peer outputs need an f16, 16-byte aligned output (TMA store) and at most 7 peers";
    return cudaErrorInvalidValue;
  }
  kp.w_scale = a.w_scale;
  kp.wreduced = a.wreduced;
  kp.bias = a.bias;
  kp.a_scale = a.a_scale;
  kp.a_zero = a.a_zero;
  kp.half_range = a.half_range;
  kp.out = a.out;
  kp.ldo = a.ldo;
  const int key = ((cg << 16) | bn) | (mc ? kKeyMC : 0) | (w4 ? kKeyW4 : 0);
  const int mode = kp.hstat ? kModeF16Stats : a.mode;
  if (kp.hstat && !kp.tma_store) {  // the statistics read the staged TMA-store tile
    *err_msg = "gated MLP statistics need a 16-byte aligned f16 hidden state";
    return cudaErrorInvalidValue;
  }
  if (kp.trace) {
    // launch, then dump the timeline of this call (overwrites the file each call)
    cudaError_t e = sp ? launch_sp_key(key, kp, mode, num_sms, stream) : launch_dense_key(key, kp, mode, num_sms, stream);
    if (e != cudaSuccess) return e;
    std::vector<long long> h(trace_bytes / 8);
    cudaStreamSynchronize(stream);
    cudaMemcpy(h.data(), kp.trace, trace_bytes, cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(trace_path, "wb")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
    std::vector<long long> w(2 * 128 * 8);
    cudaMemcpyFromSymbol(w.data(), g_wstamps, w.size() * 8);
    const std::string wp = std::string(trace_path) + ".w";
    if (FILE* f = fopen(wp.c_str(), "wb")) {
      fwrite(w.data(), 8, w.size(), f);
      fclose(f);
    }
    return cudaSuccess;
  }
  if (sp) {
    const cudaError_t e = launch_sp_key(key, kp, mode, num_sms, stream);
    if (e == cudaErrorInvalidConfiguration) *err_msg = "unsupported sparse tile configuration";
    return e;
  }
  const cudaError_t e = launch_dense_key(key, kp, mode, num_sms, stream);
  if (e == cudaErrorInvalidConfiguration) *err_msg = "unsupported tile configuration";
  return e;
}

}  // namespace quikb200
