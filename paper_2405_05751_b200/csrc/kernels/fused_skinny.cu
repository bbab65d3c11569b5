// B200 backend — fused skinny-GEMM µGraph kernels (sm_100a, tcgen05 + TMA).
//
// One kernel family executes the GraphDefs of three benchmark µGraphs
// (fixtures.py):
//   GATED : out = SiLU(X·W1) ⊙ (X·W3)                    (GatedMLP)
//   RMS   : out = (X·G)·W / sqrt(Σ_k X² · D)             (RMSNorm -> MatMul)
//   LORA  : out = X·W + (X·A)·B̄                          (single-kernel LoRA)
// Each µGraph block graph accumulates φ-Accums over its for-loop; all of them
// are linear, so a block-graph instance (a 128-column tile) maps onto a CTA
// *cluster* that splits the for-loop (the K range) S ways: every CTA
// accumulates its share of the loop in TMEM, then the partial accumulators
// are exchanged point-to-point over DSMEM (st.async + mbarrier transaction
// counts, no cluster-wide barrier) so that each CTA owns 128/S rows of the
// tile, sums the S partials and runs the post-loop ops (SiLU·, /sqrt, +XA·B̄)
// for them.
//
// Block matmuls run on the 5th-gen tensor cores with swap-AB (weights on
// UMMA M=128, the 8 or 16 tokens on N=16): D^T[n, t] = W^T[n, k] · X^T[k, t].
// W tiles are TMA-staged MN-major with 128-byte swizzle; X^T is K-major.
// RMS: the B operand is the exact fp32 product x·g split into bf16 hi + lo
// rows (tokens 0-7 hi, 8-15 lo) so no rounding of the elementwise product
// reaches the tensor cores; the halves are summed in the epilogue.
// LoRA: XA = X·A (16 x 16 per CTA K range) runs on the CUDA cores of the
// otherwise idle epilogue warps, reading the same staged X^T tile and a raw
// [64 k][16 r] A box, while the tensor cores run X·W.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer + TMEM
// owner, warps 2-5: per-stage RMS B-tile builders (+ Σx²) / LoRA XA, then
// the epilogue.
// Programmatic dependent launch: the prologue overlaps the previous kernel;
// global inputs are touched only after griddepcontrol.wait.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "fused.cuh"
#include "sm100.cuh"
#include "smem_limit.cuh"

namespace tpo_fused {

using namespace sm100;

constexpr int kBK = 64;                   // K per pipeline stage (one 128-B swizzle atom)
constexpr int kTileN = 128;               // UMMA M (weight columns per tile)
constexpr uint32_t kWBox = kBK * 128;     // bytes of one 64-col x kBK-row W box
constexpr int kThreads = 192;

// Pipeline stage layout (one k block of 64):
//   [W boxes: NP planes x 2 x 8 KB] [B operand tile] [RMS: raw X, G | LoRA: A box(es)]
// GATED / LoRA: the B operand tile (X^T, K-major, 128-B swizzle) is a TMA box.
// LoRA: the stage also carries the A box [64 k][16 r]; the epilogue warps
// fold it into this CTA's XA partial (warp MMA) and release the stage; after
// the last k block XA_s·B̄ joins the accumulator as two more UMMAs (kFold*).
// RMS: TMA brings raw X and G; the four epilogue warps build the B tile
// (x·g as bf16 hi + lo rows) in place while the stage's W boxes land, and
// release it to the MMA issuer per stage (b_full).
//
// SPLIT (fp32 / fp64 callers, tpo_gpu.h TPO_PREC_AUTO): every weight matrix
// arrives as two bf16 planes, hi = bf16(w) and lo = bf16(w - hi), and both
// planes accumulate into the same TMEM accumulator; the activations arrive
// as hi rows + lo rows of the B operand (GATED: tokens 0-7 hi, 8-15 lo;
// LoRA: N = 32, tokens 0-15 hi, 16-31 lo; RMS: raw fp32 X and G, split in
// the B-tile build).  The sum (w_hi + w_lo)·(x_hi + x_lo) carries ~16
// mantissa bits per operand, so the result meets the fp32-level tolerance
// against the double reference on arbitrary inputs.  It costs 2x the weight
// bytes of the bf16 kernel.
template <int MODE, bool SPLIT>
struct Cfg {
  static constexpr int NA = MODE == MODE_GATED ? 2 : 1;  // weight matrices
  static constexpr int NP = NA * (SPLIT ? 2 : 1);         // weight planes (TMA maps)
  static constexpr int kTokN = MODE == MODE_LORA && SPLIT ? 32 : 16;  // UMMA N
  static constexpr uint32_t kXTileB = kTokN * 128;        // B operand tile bytes
  static constexpr bool kTmaX = MODE != MODE_RMS;        // per-stage B tile via TMA
  // LoRA XA on the epilogue warps' mma.sync from the ring stage (measured
  // against XA as a second M = 128 UMMA per k step: 10.7 vs 8.35 us per
  // evaluation, profiles/r02/lora_xa.txt — it doubles the MMA time in every
  // stage's turnaround; removed)
  static constexpr bool kXaRing = MODE == MODE_LORA;
  static constexpr int kNABox = SPLIT ? 2 : 1;             // LoRA A planes
  static constexpr uint32_t kABox = 2048;                  // LoRA A per plane [64 k][16 r]
  static constexpr uint32_t kAOff = 0;                     // W boxes
  static constexpr uint32_t kBOff = kAOff + NP * 2 * kWBox;  // B operand (X^T) tile
  static constexpr uint32_t kXRawBytes = SPLIT ? 2048 : 1024;  // RMS X box [8][64] (fp32 | bf16)
  static constexpr uint32_t kGBytes = SPLIT ? 256 : 128;       // RMS G box [64]
  static constexpr uint32_t kXRawOff = kBOff + kXTileB;    // RMS raw X
  static constexpr uint32_t kGOff = kXRawOff + kXRawBytes; // RMS G
  static constexpr uint32_t kLAOff = kBOff + kXTileB;      // LoRA A box(es)
  static constexpr uint32_t kStage = MODE == MODE_RMS               ? kGOff + 1024
                                     : MODE == MODE_LORA              ? kLAOff + kNABox * kABox
                                                                      : kBOff + kXTileB;
  static constexpr uint32_t kFullBytes = MODE == MODE_RMS ? NP * 2 * kWBox : kStage;
  static constexpr uint32_t kXGBytes = kXRawBytes + kGBytes;  // RMS: X box [8][64] + G box [64]
  static constexpr int kSide = MODE == MODE_RMS ? 8 : 0;  // RMS: Σx² per token, exchanged
  // stage releases: the UMMA commit, plus (LoRA) the four epilogue warps
  static constexpr uint32_t kEmptyCount = kXaRing ? 5 : 1;
  // LoRA: XA_s·B̄ folded into the accumulator on the tensor cores — after
  // the last k block the MMA issuer adds B̄ (TMA, [16 r][128 n], MN-major
  // like W; SPLIT: hi and lo planes) times XA_s^T (written by the XA warps
  // as bf16 hi + lo, K-major) as 2 (SPLIT 4) more K = 16 UMMAs into the hi
  // token columns, staged in the ring's next stage (free by then).
  // Replaces 256 FMAs per epilogue thread on the tail (8.36 -> 8.30 us per
  // evaluation, A/B on one box).
  static constexpr int kFoldPlanes = SPLIT ? 2 : 1;
  // stage offsets: B̄ boxes (2 x 2 KB per plane), XA_s^T tile (2 KB)
  static constexpr uint32_t kFoldB = 0, kFoldX = kFoldPlanes * 4096;

  static_assert(kStage % 1024 == 0, "stages must keep the 1024-B swizzle alignment");
};

constexpr int kMaxStages = 12;

struct __align__(8) Bars {
  uint64_t full[kMaxStages], empty[kMaxStages], xg_full[kMaxStages], b_full[kMaxStages];
  uint64_t tmem_full, recv, recv_side, xa_full;
  uint64_t xb_full, xa_ready;  // LoRA fold: B̄ landed; XA_s^T tile written
  uint32_t tmem_base;
};

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// remote (DSMEM) 16-byte store that completes `bytes` on the peer's mbarrier
__device__ __forceinline__ void st_async4(uint32_t addr, float a, float b, float c, float d,
                                          uint32_t mbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
          addr),
      "f"(a), "f"(b), "f"(c), "f"(d), "r"(mbar)
      : "memory");
}

// MINB = 2: a shallow pipeline (<= 113 KB smem) so that two CTAs fit one SM.
// With PDL the next evaluation's CTAs then become resident while this one
// drains; when the weights are declared static (p.prefetch_static) they
// start streaming their first pipeline stages before the grid dependency
// resolves, so HBM stays busy across back-to-back µGraph evaluations.
template <int MODE, int STAGES, int S, int MINB, bool SPLIT>
__global__ void __launch_bounds__(kThreads, MINB)
    skinny_kernel(const __grid_constant__ CUtensorMap tmW0, const __grid_constant__ CUtensorMap tmW1,
                  const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmA,
                  const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmW3,
                  const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmO,
                  const SkinnyParams p) {
  using C = Cfg<MODE, SPLIT>;
  // weight plane maps: bf16 {W} / {W1, W3}; SPLIT {W hi, W lo} / {W1 hi, W1 lo, W3 hi, W3 lo}
  const CUtensorMap *wmap[4] = {&tmW0, &tmW1, &tmW2, &tmW3};
  static_assert(STAGES <= kMaxStages, "pipeline deeper than the barrier arrays");
  constexpr int kSide = C::kSide;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nkb = p.k_per_cta / kBK;
  constexpr int rows_per = kTileN / S;                                     // rows owned per CTA
  uint8_t *stages = smem;
  float *red = reinterpret_cast<float *>(stages + STAGES * C::kStage);
  // red: [S-1 peers][NV/4][rows_per][4] incoming row partials (peer slot:
  // its rank, minus one above the owner's own)
  float *side = red + (S > 1 ? (S - 1) * (kTileN / S) * 16 : 0);
  float *xa_w = side + S * kSide;  // side: [S][kSide]; xa_w: LoRA per-warp XA partials [4][16][16]
  Bars *bars = reinterpret_cast<Bars *>(xa_w + (C::kXaRing ? 1024 : 0));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  unsigned long long *dbg = p.dbg ? p.dbg + blockIdx.x * 16 : nullptr;
#define TPO_T(slot) \
  if (dbg) dbg[slot] = globaltimer();
  if (threadIdx.x == 0) TPO_T(0);
  if (dbg && threadIdx.x == 0) {  // ring slot 14: the SM this CTA runs on
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    dbg[14] = sm + 1;
  }
  const uint32_t rank = S > 1 ? cluster_rank() : 0;
  const int n0 = (blockIdx.x / S) * kTileN;
  const int kbase = int(rank) * p.k_per_cta;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&bars->full[s], 1);
      // experiment 16 (LoRA): stages released by the UMMA commit alone (no XA)
      mbar_init(&bars->empty[s], (p.dbg_flags & 16) ? 1u : C::kEmptyCount);
      mbar_init(&bars->xg_full[s], 1);
      mbar_init(&bars->b_full[s], 4);
    }
    mbar_init(&bars->tmem_full, 1);
    mbar_init(&bars->xb_full, 1);
    mbar_init(&bars->xa_ready, 4);
    mbar_init(&bars->recv, 1);
    mbar_init(&bars->recv_side, 1);
    mbar_init(&bars->xa_full, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
#pragma unroll
    for (int w = 0; w < C::NP; ++w) tma_prefetch(wmap[w]);
    tma_prefetch(&tmX);
    if (MODE != MODE_GATED) tma_prefetch(&tmA);
    if (MODE == MODE_LORA && SPLIT) tma_prefetch(&tmA1);
  }
  if (warp == 1) tmem_alloc<32>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  if (threadIdx.x == 0) TPO_T(1);
  if (S > 1) cluster_arrive();  // peers' mbarriers are initialised once the wait returns
  // incoming DSMEM bytes: (S-1) peers x the owned rows' partials; side blocks
  if (threadIdx.x == 0 && S > 1) {
    mbar_expect_tx(&bars->recv, uint32_t((S - 1) * rows_per * (MODE == MODE_RMS ? 8 : 16) * 4));
    if (kSide) mbar_expect_tx(&bars->recv_side, uint32_t((S - 1) * kSide * 4));
  }
  // Weights declared static (never written by preceding work on the
  // stream) may stream before the programmatic dependency resolves: the
  // producer issues the W (and LoRA A) boxes of the first pipeline stages,
  // then waits; X is read only after the wait.
  // LoRA A box(es) of k block k0 into stage st: [64 k][16 r] per plane
  auto lora_a = [&](uint8_t *st, uint64_t *bar, int k0) {
#pragma unroll
    for (int h = 0; h < C::kNABox; ++h) tma_load_2d(st + C::kLAOff + h * C::kABox, h ? &tmA1 : &tmA, bar, 0, k0);
  };
  const int npre_max = (nkb < STAGES ? nkb : STAGES) - p.pre_cut;
  const int npre = p.prefetch_static ? (npre_max > 0 ? npre_max : 0) : 0;
  if (warp == 0 && elect_one()) {
    for (int kb = 0; kb < npre; ++kb) {
      uint8_t *st = stages + kb * C::kStage;
      mbar_expect_tx(&bars->full[kb], C::kFullBytes);
      const int k0 = kbase + kb * kBK;
      uint8_t *wt = st + C::kAOff;
#pragma unroll
      for (int w = 0; w < C::NP; ++w) {
        tma_load_2d(wt + 2 * w * kWBox, wmap[w], &bars->full[kb], n0, k0);
        tma_load_2d(wt + (2 * w + 1) * kWBox, wmap[w], &bars->full[kb], n0 + 64, k0);
      }
      if (MODE == MODE_LORA) lora_a(st, &bars->full[kb], k0);  // A: static
    }
    // The activations (RMS: and G) are requested into L2 before the wait —
    // a hint only, no data reaches the SM: L2 is the point of coherence, so
    // a write by the preceding grid still lands in (or updates) those lines,
    // and every read that uses them comes after the wait.  It turns the
    // post-wait activation loads from HBM misses into L2 hits (an activation
    // the preceding grid just wrote is there already).  RMS / LoRA: the
    // CTA's whole K range (16 boxes); GatedMLP (64 k blocks per CTA): the
    // prefetched stages' (more costs 1.1 us).  TPO_X_L2=0 disables.
    if (p.x_l2) {
      const int nx = MODE == MODE_GATED ? npre : nkb;
      for (int kb = 0; kb < nx; ++kb) {
        tma_prefetch_l2_2d(&tmX, kbase + kb * kBK, 0);
        if (MODE == MODE_RMS) tma_prefetch_l2_2d(&tmA, kbase + kb * kBK, 0);
      }
    }
  }
  pdl_wait();  // inputs may be produced by the preceding kernel
  // PDL trigger: by default late — each warp triggers once its streaming
  // role is done (last TMA issued / last MMA issued / last stage consumed),
  // so the next evaluation's CTAs become resident (two-per-SM configs) and
  // prefetch their static weights while this grid drains.  Experiment flag
  // 8: trigger at once.
  const bool early_trigger = p.dbg_flags & 8;
  if (early_trigger) pdl_launch();
  // Atomic epilogue (RMS / LoRA, split clusters): every CTA adds its scaled
  // partial into the output with fp32 reductions instead of routing it to
  // an owner CTA; rank 0 zeroes the tile first, ordered before the other
  // ranks' adds by a second cluster-barrier phase.
  const bool atomic_epi = MODE != MODE_GATED && S > 1 && p.epi_atomic;
  if (atomic_epi && rank == 0 && warp >= 2) {
    const int col = n0 + (threadIdx.x - 64);
    for (int tk = 0; tk < p.tokens; ++tk) p.out[size_t(tk) * p.N + col] = 0.f;
  }

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (elect_one()) {
      // X (and RMS: G) boxes of the prefetched stages
      for (int kb = 0; kb < npre; ++kb) {
        uint8_t *st = stages + kb * C::kStage;
        if (C::kTmaX) {
          tma_load_2d(st + C::kBOff, &tmX, &bars->full[kb], kbase + kb * kBK, 0);
        } else {
          mbar_expect_tx(&bars->xg_full[kb], C::kXGBytes);
          tma_load_2d(st + C::kXRawOff, &tmX, &bars->xg_full[kb], kbase + kb * kBK, 0);
          tma_load_2d(st + C::kGOff, &tmA, &bars->xg_full[kb], kbase + kb * kBK, 0);
        }
      }
      // run ahead of the ring through L2: more weight bytes in flight per
      // CTA than the ring holds, issued only after this evaluation's X
      auto l2_pre = [&](int kb) {
        const int k0 = kbase + kb * kBK;
#pragma unroll
        for (int w = 0; w < C::NP; ++w) {
          tma_prefetch_l2_2d(wmap[w], n0, k0);
          tma_prefetch_l2_2d(wmap[w], n0 + 64, k0);
        }
      };
      const int l2a = p.l2_ahead;
      for (int kb = STAGES; kb < STAGES + l2a && kb < nkb; ++kb) l2_pre(kb);
      for (int kb = npre; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        if (l2a > 0 && kb >= STAGES && kb + l2a < nkb) l2_pre(kb + l2a);
        mbar_wait(&bars->empty[s], ((kb / STAGES) & 1) ^ 1);
        uint8_t *st = stages + s * C::kStage;
        if (MODE == MODE_RMS) {  // raw X and G first: the B-tile build is on the critical path
          mbar_expect_tx(&bars->xg_full[s], C::kXGBytes);
          tma_load_2d(st + C::kXRawOff, &tmX, &bars->xg_full[s], kbase + kb * kBK, 0);
          tma_load_2d(st + C::kGOff, &tmA, &bars->xg_full[s], kbase + kb * kBK, 0);
        }
        mbar_expect_tx(&bars->full[s], C::kFullBytes);
        const int k0 = kbase + kb * kBK;
        uint8_t *wt = st + C::kAOff;
#pragma unroll
        for (int w = 0; w < C::NP; ++w) {
          tma_load_2d(wt + 2 * w * kWBox, wmap[w], &bars->full[s], n0, k0);
          tma_load_2d(wt + (2 * w + 1) * kWBox, wmap[w], &bars->full[s], n0 + 64, k0);
        }
        if (C::kTmaX) tma_load_2d(st + C::kBOff, &tmX, &bars->full[s], k0, 0);
        if (MODE == MODE_LORA) lora_a(st, &bars->full[s], k0);
        // experiment (TPO_TRIG_EARLY = D): release the dependent grid D
        // k blocks before the last issue (one thread triggers the CTA)
        if (p.trig_early > 0 && kb == nkb - 1 - p.trig_early) pdl_launch();
      }
      if (C::kXaRing) {  // B̄ (static) into the stage after the last k block's, once it drains
        const int s = nkb % STAGES;
        mbar_wait(&bars->empty[s], ((nkb / STAGES) & 1) ^ 1);
        uint8_t *st = stages + s * C::kStage;
        mbar_expect_tx(&bars->xb_full, C::kFoldPlanes * 4096);
#pragma unroll
        for (int h = 0; h < C::kFoldPlanes; ++h) {
          const CUtensorMap *m = h ? &tmW3 : &tmW2;
          tma_load_2d(st + C::kFoldB + h * 4096, m, &bars->xb_full, n0, 0);
          tma_load_2d(st + C::kFoldB + h * 4096 + 2048, m, &bars->xb_full, n0 + 64, 0);
        }
      }
      TPO_T(10);
    }
    __syncwarp();
    if (!early_trigger) pdl_launch();
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16(kTileN, C::kTokN, /*a MN-major*/ true, /*b K-major*/ false);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&bars->full[s], (kb / STAGES) & 1);
      if (kb == 0 && lane == 0) TPO_T(8);
      if (MODE == MODE_RMS) mbar_wait(&bars->b_full[s], (kb / STAGES) & 1);
      if (kb == 0 && lane == 0) TPO_T(9);
      tc_fence_after();
      if (p.dbg_flags & 4) {  // experiment: free stages without the MMA
        if (elect_one()) {
          mbar_arrive(&bars->empty[s]);
          if (kb == nkb - 1) mbar_arrive(&bars->tmem_full);
        }
        __syncwarp();
        continue;
      }
      if (elect_one()) {
        uint8_t *st = stages + s * C::kStage;
        uint8_t *wt = st + C::kAOff;
        const uint32_t xs = smem_u32(st + C::kBOff);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) {
          const uint64_t bdesc = sdesc_sw128(xs + kk * 32, 16, 1024);
#pragma unroll
          for (int w = 0; w < C::NP; ++w) {
            // plane w accumulates into matrix w / 2 (SPLIT: hi then lo plane)
            const int acc = SPLIT ? w / 2 : w;
            const uint64_t adesc = sdesc_sw128(smem_u32(wt + w * 2 * kWBox) + kk * 16 * 128, kWBox, 1024);
            umma_bf16(tmem + acc * C::kTokN, adesc, bdesc, idesc, (kb | kk) != 0 || (SPLIT && (w & 1)));
          }
        }
        umma_commit(&bars->empty[s]);
        if (kb == nkb - 1 && !C::kXaRing) {  // LoRA: after the fold below
          umma_commit(&bars->tmem_full);
          TPO_T(3);
        }
      }
      __syncwarp();
    }
    if (C::kXaRing && !(p.dbg_flags & 4)) {
      // acc[n][t] += Σ_r B̄[r][n]·XA_s[t][r] (hi, then lo)
      uint8_t *st = stages + (nkb % STAGES) * C::kStage;
      mbar_wait(&bars->xb_full, 0);
      mbar_wait(&bars->xa_ready, 0);
      tc_fence_after();
      if (elect_one()) {
        // N = 16: the hi token columns (SPLIT's lo tokens sit in 16-31)
        constexpr uint32_t fold_idesc = idesc_bf16(kTileN, 16, true, false);
#pragma unroll
        for (int hb = 0; hb < C::kFoldPlanes; ++hb)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            umma_bf16(tmem, sdesc_sw128(smem_u32(st + C::kFoldB + hb * 4096), 2048, 1024),
                      sdesc_sw128(smem_u32(st + C::kFoldX) + h * 32, 16, 1024), fold_idesc, 1u);
        umma_commit(&bars->tmem_full);
        TPO_T(3);
      }
      __syncwarp();
    }
    if (!early_trigger) pdl_launch();
  } else {
    // ------------------------------------- auxiliary / epilogue warps 2..5
    const int t = threadIdx.x - 64;
    float sumsq = 0.f;       // RMS: Σx² of token t/16 over this CTA's K range
    // Epilogue operands from global memory are loaded now, off the critical
    // path (under a saturated HBM a dependent load costs ~1 µs): RMS D.
    float dsc = 0.f;
    if (MODE == MODE_RMS) dsc = SPLIT ? p.dscale_f32[0] : __bfloat162float(p.dscale[0]);
    if (MODE == MODE_RMS) {
      // Per stage: B tile rows 0-7 = bf16(x·g) (hi), rows 8-15 = the
      // residual x·g - hi (lo), K-major with the 128-B swizzle.  Thread t
      // owns token t/16 and k = 4·(t%16) .. +3, so Σx² stays per token.
      // bf16 X, G: the product is exact in fp32 and so is the residual;
      // SPLIT (fp32 X, G): the fp32 product, split the same way.
      const int tok = t >> 4, sub = t & 15;
      const int c = sub >> 1, half = (sub & 1) * 8;
      const uint32_t off_hi = (tok >> 3) * 1024 + (tok & 7) * 128 + ((c ^ (tok & 7)) << 4) + half;
      const int rl = tok + 8;
      const uint32_t off_lo = (rl >> 3) * 1024 + (rl & 7) * 128 + ((c ^ (rl & 7)) << 4) + half;
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&bars->xg_full[s], (kb / STAGES) & 1);
        uint8_t *st = stages + s * C::kStage;
        float xf[4], gf[4];
        if (SPLIT) {
          const float4 xr = *reinterpret_cast<const float4 *>(st + C::kXRawOff + tok * 256 + sub * 16);
          const float4 gr = *reinterpret_cast<const float4 *>(st + C::kGOff + sub * 16);
          xf[0] = xr.x, xf[1] = xr.y, xf[2] = xr.z, xf[3] = xr.w;
          gf[0] = gr.x, gf[1] = gr.y, gf[2] = gr.z, gf[3] = gr.w;
        } else {
          const uint2 xr = *reinterpret_cast<const uint2 *>(st + C::kXRawOff + tok * 128 + sub * 8);
          const uint2 gr = *reinterpret_cast<const uint2 *>(st + C::kGOff + sub * 8);
          const __nv_bfloat162 *x2 = reinterpret_cast<const __nv_bfloat162 *>(&xr);
          const __nv_bfloat162 *g2 = reinterpret_cast<const __nv_bfloat162 *>(&gr);
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const float2 a = __bfloat1622float2(x2[j]), b = __bfloat1622float2(g2[j]);
            xf[2 * j] = a.x, xf[2 * j + 1] = a.y, gf[2 * j] = b.x, gf[2 * j + 1] = b.y;
          }
        }
        uint32_t hi[2], lo[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          sumsq += xf[2 * j] * xf[2 * j] + xf[2 * j + 1] * xf[2 * j + 1];
          const float p0 = xf[2 * j] * gf[2 * j], p1 = xf[2 * j + 1] * gf[2 * j + 1];
          __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
          float2 hf = __bfloat1622float2(h);
          __nv_bfloat162 l = __floats2bfloat162_rn(p0 - hf.x, p1 - hf.y);
          hi[j] = *reinterpret_cast<uint32_t *>(&h);
          lo[j] = *reinterpret_cast<uint32_t *>(&l);
        }
        *reinterpret_cast<uint2 *>(st + C::kBOff + off_hi) = make_uint2(hi[0], hi[1]);
        *reinterpret_cast<uint2 *>(st + C::kBOff + off_lo) = make_uint2(lo[0], lo[1]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->b_full[s]);
      }
#pragma unroll
      for (int o = 8; o; o >>= 1) sumsq += __shfl_xor_sync(0xffffffffu, sumsq, o);
    }
    if (MODE == MODE_LORA && C::kXaRing) {
      // XA_s = X·A over this CTA's K range (16 tokens x 16 ranks) on the
      // warp MMA path of the otherwise idle epilogue warps, stage by stage
      // from the ring's X^T tile (K-major, 128-B swizzle) and A box
      // ([64 k][16 r]): warp q takes k16 step q of every k block, two
      // m16n8k16 bf16 MMAs with fp32 accumulation (exact products), then
      // releases the stage.  XA·B̄ is linear, so each CTA later adds
      // XA_s·B̄ to its own partial rows: no XA exchange.
      const int q = warp & 3;
      float c[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      const int mi = lane >> 3, ri = lane & 7;
      const int tok = ri + 8 * (mi & 1);
      const int kch = 2 * q + (mi >> 1);
      const uint32_t a_off = (tok >> 3) * 1024 + (tok & 7) * 128 + ((kch ^ (tok & 7)) << 4);
      const uint32_t b_off = (16 * q + ri + 8 * (mi & 1)) * 32 + (mi >> 1) * 16;
      for (int kb = 0; kb < ((p.dbg_flags & 16) ? 0 : nkb); ++kb) {  // experiment 16: no XA
        const int s = kb % STAGES;
        mbar_wait(&bars->full[s], (kb / STAGES) & 1);
        const uint32_t st = smem_u32(stages + s * C::kStage);
        // SPLIT: X^T hi rows 0-15 / lo rows 16-31 (+2 KB), A hi / lo boxes:
        // XA = Σ over the hi/lo products
        constexpr int NX = SPLIT ? 2 : 1;
        uint32_t af[NX][4], bf[NX][4];
#pragma unroll
        for (int h = 0; h < NX; ++h) {
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(af[h][0]), "=r"(af[h][1]), "=r"(af[h][2]), "=r"(af[h][3])
                       : "r"(st + C::kBOff + h * 2048 + a_off));
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(bf[h][0]), "=r"(bf[h][1]), "=r"(bf[h][2]), "=r"(bf[h][3])
                       : "r"(st + C::kLAOff + h * C::kABox + b_off));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->empty[s]);
#pragma unroll
        for (int ha = 0; ha < NX; ++ha)
#pragma unroll
          for (int hb = 0; hb < NX; ++hb)
#pragma unroll
            for (int j = 0; j < 2; ++j)
              asm volatile(
                  "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                  "{%8,%9}, {%0,%1,%2,%3};"
                  : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                  : "r"(af[ha][0]), "r"(af[ha][1]), "r"(af[ha][2]), "r"(af[ha][3]), "r"(bf[hb][2 * j]),
                    "r"(bf[hb][2 * j + 1]));
      }
      // per-warp partials -> xa_w[q][token][r]
      float *xw = xa_w + q * 256;
      const int g = lane >> 2, cc = 2 * (lane & 3);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        *reinterpret_cast<float2 *>(xw + g * 16 + 8 * j + cc) = make_float2(c[j][0], c[j][1]);
        *reinterpret_cast<float2 *>(xw + (g + 8) * 16 + 8 * j + cc) = make_float2(c[j][2], c[j][3]);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      // thread t: XA_s[t/8][2(t%8)..+1] = Σ over the 4 warps
      const int i0 = (t >> 3) * 16 + (t & 7) * 2;
      const float xa0 = (xa_w[i0] + xa_w[256 + i0]) + (xa_w[512 + i0] + xa_w[768 + i0]);
      const float xa1 = (xa_w[i0 + 1] + xa_w[256 + i0 + 1]) + (xa_w[512 + i0 + 1] + xa_w[768 + i0 + 1]);
      {
        // XA_s^T tile for the tensor-core fold: row = token, k = r (hi,
        // chunks 0-1) and 16 + r (lo, chunks 2-3), 128-B swizzle
        const __nv_bfloat162 h = __floats2bfloat162_rn(xa0, xa1);
        const float2 hf = __bfloat1622float2(h);
        const __nv_bfloat162 l = __floats2bfloat162_rn(xa0 - hf.x, xa1 - hf.y);
        const int tok = t >> 3, r = (t & 7) * 2, c = r >> 3;
        const uint32_t row_off = (tok >> 3) * 1024 + (tok & 7) * 128 + (r & 7) * 2;
        uint8_t *xt = stages + (nkb % STAGES) * C::kStage + C::kFoldX;
        mbar_wait(&bars->xb_full, 0);  // the stage has drained (and B̄ landed)
        *reinterpret_cast<__nv_bfloat162 *>(xt + row_off + ((c ^ (tok & 7)) << 4)) = h;
        *reinterpret_cast<__nv_bfloat162 *>(xt + row_off + (((c + 2) ^ (tok & 7)) << 4)) = l;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->xa_ready);
      }
    }

    if (!early_trigger) pdl_launch();
    // ---------------------------------------------------------- epilogue
    // Row `row` of the 128-column tile is held (in TMEM lane `row`) by the
    // thread (warp quarter q, lane); CTA `row / rows_per` of the cluster owns
    // it: non-owners push their partial row to the owner over DSMEM, owners
    // sum the S partials and run the post-loop ops.  Side data (RMS Σx² per
    // token, LoRA XA partials) is exchanged and reduced *before* the last
    // MMA completes, off the critical path.
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;       // UMMA M index = output column in the tile
    const int n = n0 + row;
    const int owner = row / rows_per;    // CTA of the cluster finishing this row
    const bool mine = owner == int(rank);
    constexpr int NV = MODE == MODE_RMS ? 8 : 16;  // floats per row partial
    constexpr int T = MODE == MODE_LORA ? 16 : 8;  // tokens
    float post[T];                        // RMS: 1/sqrt(Σx²·D) per token; LoRA: (XA·B̄)[t, n]
    if (MODE == MODE_RMS) {
      if ((t & 15) == 0) side[rank * kSide + (t >> 4)] = sumsq;
    }
    if (MODE != MODE_GATED) asm volatile("bar.sync 1, 128;" ::: "memory");  // own side block / XA_s written
    const bool xchg = !(p.dbg_flags & 2);  // experiment 2: no DSMEM exchange
    if (S > 1) {
      cluster_wait();  // every peer has initialised its barriers
      if (xchg && kSide > 0 && t * 4 < kSide) {
        const float *src = side + rank * kSide + t * 4;
        for (int o = 1; o < S; ++o) {
          const uint32_t dst_rank = (rank + o) % S;
          st_async4(map_rank(src, dst_rank), src[0], src[1], src[2], src[3],
                    map_rank(&bars->recv_side, dst_rank));
        }
      }
      if (xchg && kSide > 0) mbar_wait(&bars->recv_side, 0);
      if (atomic_epi) cluster_arrive();  // phase 2: rank 0's zeroed tile precedes every add
    }
    if (MODE == MODE_RMS && (mine || atomic_epi)) {
#pragma unroll
      for (int tk = 0; tk < 8; ++tk) {
        float ss = 0.f;
        for (int rr = 0; rr < S; ++rr) ss += side[rr * kSide + tk];
        post[tk] = 1.0f / sqrtf(ss * dsc);
      }
    }
    if (MODE == MODE_LORA) {
#pragma unroll
      for (int tk = 0; tk < 16; ++tk) post[tk] = 0.f;  // XA_s·B̄ is folded into the accumulator
    }

    // ---- critical path: last MMA -> TMEM -> DSMEM -> owner -> HBM
    // pin the post-loop operands here: without this the compiler may sink
    // their computation past the waits below, onto the critical path
    if (MODE == MODE_RMS && (mine || atomic_epi)) {
#pragma unroll
      for (int tk = 0; tk < T; ++tk) asm volatile("" : "+f"(post[tk]));
    }
    mbar_wait(&bars->tmem_full, 0);
    if (threadIdx.x == 64) TPO_T(5);
    __syncwarp();  // tcgen05.ld is .sync.aligned: the warp must be converged
    tc_fence_after();
    float acc[16];
    {
      float v[16];
      tmem_ld16(tmem + (uint32_t(q * 32) << 16), v);
      if (MODE == MODE_GATED) {
        float v3[16];
        tmem_ld16(tmem + (uint32_t(q * 32) << 16) + C::kTokN, v3);
#pragma unroll
        for (int i = 0; i < 8; ++i)  // SPLIT: hi tokens 0-7 + lo tokens 8-15
          acc[i] = SPLIT ? v[i] + v[8 + i] : v[i], acc[8 + i] = SPLIT ? v3[i] + v3[8 + i] : v3[i];
      } else if (MODE == MODE_RMS) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = v[i] + v[8 + i], acc[8 + i] = 0.f;
      } else {
        if (SPLIT) {  // lo tokens in columns 16-31
          float v2[16];
          tmem_ld16(tmem + (uint32_t(q * 32) << 16) + 16, v2);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += v2[i];
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = v[i] + post[i];  // partial XW_s + XA_s·B̄
      }
    }
    if (atomic_epi) {
      cluster_wait();  // phase 2
      if (!(p.dbg_flags & 1)) {
#pragma unroll
        for (int tk = 0; tk < T; ++tk)
          if (tk < p.tokens)
            atomicAdd(p.out + size_t(tk) * p.N + n, MODE == MODE_RMS ? acc[tk] * post[tk] : acc[tk]);
      }
    } else if (S > 1 && xchg) {
      if (!mine) {
        // red layout [src rank][NV/4 chunks][rows_per][4]: the owner warp's
        // lanes read consecutive 16-byte chunks (bank-conflict free)
        const uint32_t mb = map_rank(&bars->recv, owner);
        const int lr = row - owner * rows_per;
#pragma unroll
        for (int i = 0; i < NV; i += 4) {
          const int slot = int(rank) < owner ? int(rank) : int(rank) - 1;
          const uint32_t dst = map_rank(red + ((slot * (NV / 4) + i / 4) * rows_per + lr) * 4, owner);
          st_async4(dst, acc[i], acc[i + 1], acc[i + 2], acc[i + 3], mb);
        }
        if (threadIdx.x == 64) TPO_T(4);
      } else {
        mbar_wait(&bars->recv, 0);  // all peers' partials of the owned rows have landed
        if (lane == 0) TPO_T(6);
        const int lr = row - int(rank) * rows_per;
        for (int rr = 0; rr < S; ++rr) {
          if (rr == int(rank)) continue;
#pragma unroll
          for (int i = 0; i < NV / 4; ++i) {
            const int slot = rr < int(rank) ? rr : rr - 1;
            const float4 v = *reinterpret_cast<const float4 *>(red + ((slot * (NV / 4) + i) * rows_per + lr) * 4);
            acc[4 * i] += v.x, acc[4 * i + 1] += v.y, acc[4 * i + 2] += v.z, acc[4 * i + 3] += v.w;
          }
        }
        if (lane == 0) TPO_T(15);
      }
    }
    if (mine && !atomic_epi && !(p.dbg_flags & 1)) {
      // the warp's [T][32] output tile through a drained stage and one TMA
      // store (rows past p.tokens clip); TPO_TMA_OUT=0: T coalesced row stores
      float *tile = reinterpret_cast<float *>(stages) + q * 32 * T;
#pragma unroll
      for (int tk = 0; tk < T; ++tk) {
        float o;
        if (MODE == MODE_GATED) o = silu(acc[tk]) * acc[8 + tk];
        else if (MODE == MODE_RMS) o = acc[tk] * post[tk];
        else o = acc[tk];
        if (p.tma_out) tile[tk * 32 + lane] = o;
        else if (tk < p.tokens) p.out[size_t(tk) * p.N + n] = o;
      }
      if (p.tma_out) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmO, tile, n0 + q * 32, 0);
          bulk_commit();
          bulk_wait_read();
        }
        __syncwarp();
      }
      if (lane == 0 && (S == 1 || q == int(rank) * (4 / S))) TPO_T(11);
    }
  }
  if (threadIdx.x == 64) TPO_T(2);
  if (S > 1 && warp < 2) {
    __syncwarp();
    cluster_wait();  // complete the start-up barrier phase for warps 0/1
    if (atomic_epi) cluster_arrive();  // phase 2 (the epilogue warps wait on it)
  }
  if (threadIdx.x == 0) TPO_T(13);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) TPO_T(12);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<32>(tmem);
  }
  if (threadIdx.x == 0) TPO_T(7);
#undef TPO_T
}

template <int MODE, int STAGES, int S, bool SPLIT>
size_t skinny_smem(const SkinnyParams &p) {
  using C = Cfg<MODE, SPLIT>;
  const int nkb = p.k_per_cta / kBK;
  (void)nkb;
  size_t b = size_t(STAGES) * C::kStage +
             (S > 1 ? size_t(S - 1) * (kTileN / S) * 16 * 4 : 0) + size_t(S) * C::kSide * 4 +
             (MODE == MODE_LORA ? 1024 * 4 : 0) + sizeof(Bars);
  return b + 1024;
}

template <int MODE, int STAGES, int S, int MINB, bool SPLIT>
cudaError_t launch_t(const CUtensorMap *maps, const SkinnyParams &p, cudaStream_t st) {
  if (p.ksplit != S) return cudaErrorInvalidValue;
  const size_t smem = skinny_smem<MODE, STAGES, S, SPLIT>(p);
  auto kern = skinny_kernel<MODE, STAGES, S, MINB, SPLIT>;
  if (cudaError_t e = tpo_ensure_smem(reinterpret_cast<const void *>(kern), smem)) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((p.N / kTileN) * p.ksplit);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.ksplit;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = std::getenv("TPO_NO_PDL") ? 1 : 2;
  return cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], maps[7], p);
}

}  // namespace tpo_fused

using namespace tpo_fused;

// (mode, stages, cluster split, CTAs per SM, split precision)
#define TPO_SKINNY_CASES(X)                                                                           \
  X(MODE_GATED, 4, 1, 1, false) X(MODE_GATED, 6, 1, 1, false) X(MODE_GATED, 3, 1, 2, false)           \
  X(MODE_GATED, 3, 2, 1, false) X(MODE_GATED, 6, 2, 1, false) X(MODE_RMS, 4, 4, 2, false)             \
  X(MODE_RMS, 5, 4, 2, false) X(MODE_RMS, 3, 4, 2, false) X(MODE_RMS, 6, 4, 1, false)                 \
  X(MODE_RMS, 8, 4, 1, false) X(MODE_RMS, 10, 4, 1, false) X(MODE_RMS, 4, 2, 1, false)                \
  X(MODE_RMS, 6, 2, 1, false) X(MODE_RMS, 8, 2, 1, false) X(MODE_RMS, 6, 1, 1, false)                 \
  X(MODE_LORA, 4, 4, 2, false) X(MODE_LORA, 5, 4, 2, false) X(MODE_LORA, 6, 4, 1, false)              \
  X(MODE_LORA, 8, 4, 1, false) X(MODE_LORA, 10, 4, 1, false) X(MODE_LORA, 6, 2, 1, false)             \
  X(MODE_LORA, 8, 2, 1, false) X(MODE_LORA, 6, 1, 1, false)                                           \
  X(MODE_GATED, 3, 1, 1, true) X(MODE_GATED, 3, 2, 1, true) X(MODE_RMS, 5, 1, 1, true)                \
  X(MODE_RMS, 5, 2, 1, true) X(MODE_RMS, 5, 4, 1, true) X(MODE_LORA, 5, 1, 1, true)                   \
  X(MODE_LORA, 5, 2, 1, true) X(MODE_LORA, 5, 4, 1, true)                                           \
  X(MODE_RMS, 5, 8, 2, false) X(MODE_RMS, 4, 8, 2, false) X(MODE_RMS, 3, 8, 3, false)                 \
  X(MODE_LORA, 5, 8, 2, false) X(MODE_LORA, 4, 8, 2, false)

extern "C" int tpo_skinny_launch(int mode, int stages, int minb, int split, const CUtensorMap *maps,
                                 const SkinnyParams *p, cudaStream_t st) {
#define TPO_CASE(M, ST, S, MB, SP)                                                           \
  if (mode == M && stages == ST && p->ksplit == S && minb == MB && bool(split) == SP) \
    return int(launch_t<M, ST, S, MB, SP>(maps, *p, st));
  TPO_SKINNY_CASES(TPO_CASE)
#undef TPO_CASE
  return int(cudaErrorInvalidValue);
}

// Shared memory of (mode, stages, split, CTAs per SM, precision) for `p`; 0
// when that configuration is not instantiated.
extern "C" size_t tpo_skinny_smem(int mode, int stages, int minb, int split, const SkinnyParams *p) {
#define TPO_CASE(M, ST, S, MB, SP)                                                           \
  if (mode == M && stages == ST && p->ksplit == S && minb == MB && bool(split) == SP) \
    return skinny_smem<M, ST, S, SP>(*p);
  TPO_SKINNY_CASES(TPO_CASE)
#undef TPO_CASE
  return 0;
}
