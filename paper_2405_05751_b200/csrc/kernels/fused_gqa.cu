// B200 backend — fused GQA-decode µGraph kernel (sm_100a, tcgen05 + TMA).
//
// µGraph (fixtures.gqa_mugraph): per KV group g,
//   out = Matmul(EwExp(Matmul(Q̄, K̄)), V̄) / Sum(EwExp(Matmul(Q̄, K̄)), dim 2)
// with φ-Accums N (numerator) and D (denominator) over the kv for-loop and
// no max subtraction (the Lax fragment has a single exp).
// N and D are sums over kv, so the loop is split across a CTA cluster
// (flash-decoding inside one block-graph instance); partials are combined
// point-to-point over DSMEM before the post-loop EwDiv.
//
// Per 128-kv block, two chained UMMAs (swap-AB, M=128, N=16):
//   S^T[l, q]  = K̄[l, d]   · Q^T[d, q]     A = K^T tile, MN-major (l contiguous)
//   O^T[d, q] += V̄^T[d, l] · P^T[l, q]     A = V tile,   MN-major (d contiguous)
// P = exp(S) is computed in fp32 by the epilogue warps from TMEM, split into
// bf16 hi + lo rows of the second B operand (q hi rows 0-7, lo rows 8-15) so
// the P·V product carries ~16 mantissa bits; D accumulates the fp32 p.
// S^T is double-buffered in TMEM and P^T in shared memory, so exp of block
// j overlaps S of block j+1 and P·V of block j-1.
//
// SPLIT (fp32 / fp64 callers): K and V arrive as bf16 hi + lo planes (each
// ring slot holds both planes of a block, 64 KB) and Q as hi rows 0-7 + lo
// rows 8-15 of the Q^T tile; both planes of a block accumulate into the same
// TMEM accumulator, and S = S[hi rows] + S[lo rows] before the exp, so
// every product carries ~16 mantissa bits per operand.
//
// Warps: 0 TMA producer, 1 MMA issuer + TMEM owner, 2-5 exp / epilogue.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fused.cuh"
#include "sm100.cuh"
#include "smem_limit.cuh"

namespace tpo_gqa {

using namespace sm100;

constexpr int kBL = 128;                    // kv per block (UMMA M of S^T)
constexpr int kHD = 128;                    // head dim (UMMA M of O^T, K of S^T)
constexpr int kTok = 16;                    // UMMA N: 8 q rows (+ lo rows / zero pad)
constexpr uint32_t kHalf = 64 * kBL * 2;    // one 64-wide box of 128 rows: 16 KB
constexpr uint32_t kSlot = 2 * kHalf;       // one ring slot: a K^T block or a V block (2 boxes)
constexpr uint32_t kQBytes = 2 * kTok * 128;  // Q^T: 2 K-major atoms of 16 rows
constexpr uint32_t kPBytes = 2 * kTok * 128;  // P^T buffer: 2 K-major atoms of 16 rows
constexpr int kThreads = 192;

struct __align__(8) Bars {
  uint64_t full[8], empty[8], s_full[2], s_empty[2], p_full[2], p_empty[2], o_full, q_full, recv;
  uint32_t tmem_base;
};

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void st_async4(uint32_t addr, float a, float b, float c, float d,
                                          uint32_t mbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
          addr),
      "f"(a), "f"(b), "f"(c), "f"(d), "r"(mbar)
      : "memory");
}
// byte offset of element (row, col) inside a K-major, 128-B-swizzled tile of
// 16 rows x 128 columns (two 64-column atoms of 2 KB)
__device__ __forceinline__ uint32_t kmaj_off(int row, int col) {
  const int atom = col >> 6, c = (col & 63) >> 3, e = col & 7;
  return atom * 2048 + (row >> 3) * 1024 + (row & 7) * 128 + ((c ^ (row & 7)) << 4) + e * 2;
}

// The ring holds SLOTS 32-KB slots filled in the order K_0, V_0, K_1, V_1, ...
// (slot index 2j for K_j, 2j+1 for V_j).  K_j's slot frees when S_j's MMA
// completes, V_j's when P_j·V_j's does.  MINB = 2: three slots (≈113 KB) so
// that the next decode step's CTAs become resident beside this one's and
// wait at the programmatic dependency instead of behind this grid's exit.
template <int SLOTS, int S, int MINB, bool SPLIT>
__global__ void __launch_bounds__(kThreads, MINB)
    gqa_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
               const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK1,
               const __grid_constant__ CUtensorMap tmV1, const GqaParams p) {
  constexpr int NPL = SPLIT ? 2 : 1;             // planes per K / V block
  constexpr uint32_t kSlotB = NPL * kSlot;       // ring slot bytes
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *stages = smem;
  uint8_t *qt = stages + SLOTS * kSlotB;
  uint8_t *pbuf = qt + kQBytes;                         // 2 x kPBytes
  constexpr int rows_per = kHD / S;
  // [S-1 peers][rows_per][8] (peer slot: its rank, minus one above the owner's)
  float *red = reinterpret_cast<float *>(pbuf + 2 * kPBytes);
  float *dpart = red + (S > 1 ? (S - 1) * rows_per * 8 : 0);  // [S][8] denominators
  float *wsum = dpart + 4 * 8;                                 // [4 warps][8]
  Bars *bars = reinterpret_cast<Bars *>(wsum + 4 * 8);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  unsigned long long *dbg = p.dbg ? p.dbg + blockIdx.x * 16 : nullptr;
#define TPO_T(slot) \
  if (dbg) dbg[slot] = globaltimer();
  if (threadIdx.x == 0) TPO_T(0);
  const uint32_t rank = S > 1 ? cluster_rank() : 0;
  const int g = blockIdx.x / S;
  const int nb = p.l_per_cta / kBL;
  const int l0 = int(rank) * p.l_per_cta;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SLOTS; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars->s_full[b], 1);
      mbar_init(&bars->s_empty[b], 4);
      mbar_init(&bars->p_full[b], 4);
      mbar_init(&bars->p_empty[b], 1);
    }
    mbar_init(&bars->o_full, 1);
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->recv, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmQ);
    if (SPLIT) tma_prefetch(&tmK1), tma_prefetch(&tmV1);
  }
  if (warp == 1) tmem_alloc<64>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;  // cols [0,16) S0, [16,32) S1, [32,48) O
  if (threadIdx.x == 0) TPO_T(1);
  if (S > 1) cluster_arrive();
  if (threadIdx.x == 0 && S > 1) mbar_expect_tx(&bars->recv, uint32_t((S - 1) * (rows_per * 32 + 32)));
  // The first ring units (and Q) requested into L2 before the wait: a hint
  // only — L2 is the point of coherence, every read that uses the data comes
  // after the wait — so a CTA that becomes resident while the previous grid
  // drains turns its first post-wait loads into L2 hits.
  auto unit = [&](int u, bool &isk, int &blk) {
    // slot u carries K_j or V_j: K_0 V_0 K_1 V_1 ..., or in the MMA issue
    // order K_0 K_1 V_0 K_2 V_1 ... K_{nb-1} V_{nb-2} V_{nb-1}
    if (!p.consume_order) isk = !(u & 1), blk = u >> 1;
    else if (u == 0) isk = true, blk = 0;
    else if (u & 1) isk = (u + 1) / 2 < nb, blk = isk ? (u + 1) / 2 : nb - 1;
    else isk = false, blk = u / 2 - 1;
  };
  if (warp == 0 && p.l2_units > 0 && elect_one()) {
    tma_prefetch_l2_3d(&tmQ, 0, 0, g);
    tma_prefetch_l2_3d(&tmQ, 64, 0, g);
    for (int u = 0; u < p.l2_units && u < 2 * nb; ++u) {
      bool isk;
      int blk;
      unit(u, isk, blk);
      const int l = l0 + blk * kBL;
      if (isk) tma_prefetch_l2_3d(&tmK, l, 0, g), tma_prefetch_l2_3d(&tmK, l + 64, 0, g);
      else tma_prefetch_l2_3d(&tmV, 0, l, g), tma_prefetch_l2_3d(&tmV, 64, l, g);
    }
  }
  pdl_wait();
  pdl_launch();  // every thread: the dependent grid may become resident early

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (elect_one()) {
      mbar_expect_tx(&bars->q_full, kQBytes);
      tma_load_3d(qt, &tmQ, &bars->q_full, 0, 0, g);
      tma_load_3d(qt + kTok * 128, &tmQ, &bars->q_full, 64, 0, g);
      for (int u = 0; u < 2 * nb; ++u) {
        const int s = u % SLOTS;
        mbar_wait(&bars->empty[s], ((u / SLOTS) & 1) ^ 1);
        uint8_t *st = stages + s * kSlotB;
        mbar_expect_tx(&bars->full[s], kSlotB);
        bool isk;
        int blk;
        unit(u, isk, blk);
        const int l = l0 + blk * kBL;
        if (isk) {
          tma_load_3d(st, &tmK, &bars->full[s], l, 0, g);              // K^T[d, l..l+63]
          tma_load_3d(st + kHalf, &tmK, &bars->full[s], l + 64, 0, g); // K^T[d, l+64..]
          if (SPLIT) {                                                  // lo plane
            tma_load_3d(st + kSlot, &tmK1, &bars->full[s], l, 0, g);
            tma_load_3d(st + kSlot + kHalf, &tmK1, &bars->full[s], l + 64, 0, g);
          }
        } else {
          tma_load_3d(st, &tmV, &bars->full[s], 0, l, g);              // V[l.., d 0..63]
          tma_load_3d(st + kHalf, &tmV, &bars->full[s], 64, l, g);     // V[l.., d 64..]
          if (SPLIT) {
            tma_load_3d(st + kSlot, &tmV1, &bars->full[s], 0, l, g);
            tma_load_3d(st + kSlot + kHalf, &tmV1, &bars->full[s], 64, l, g);
          }
        }
      }
      TPO_T(10);
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16(128, kTok, /*a MN-major*/ true, /*b K-major*/ false);
    mbar_wait(&bars->q_full, 0);
    auto mma2 = [&](int i) {  // O^T += V^T · P^T for block i
      const int u = !p.consume_order ? 2 * i + 1 : i < nb - 1 ? 2 * i + 2 : 2 * nb - 1;
      const int s = u % SLOTS, b = i & 1;
      mbar_wait(&bars->full[s], (u / SLOTS) & 1);
      mbar_wait(&bars->p_full[b], (i >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t vt = smem_u32(stages + s * kSlotB);
        const uint32_t pt = smem_u32(pbuf + b * kPBytes);
#pragma unroll
        for (int kk = 0; kk < kBL / 16; ++kk) {
          const uint64_t bdesc = sdesc_sw128(pt + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024);
#pragma unroll
          for (int pl = 0; pl < NPL; ++pl) {
            const uint64_t adesc = sdesc_sw128(vt + pl * kSlot + kk * 16 * 128, kHalf, 1024);
            umma_bf16(tmem + 32, adesc, bdesc, idesc, (i | kk | pl) != 0);
          }
        }
        umma_commit(&bars->empty[s]);
        umma_commit(&bars->p_empty[b]);
      }
      __syncwarp();
    };
    for (int j = 0; j < nb; ++j) {
      const int u = !p.consume_order ? 2 * j : j == 0 ? 0 : 2 * j - 1;
      const int s = u % SLOTS, b = j & 1;
      mbar_wait(&bars->full[s], (u / SLOTS) & 1);
      if (j == 0 && lane == 0) TPO_T(8);
      if (j >= 2) mbar_wait(&bars->s_empty[b], ((j - 2) >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t kt = smem_u32(stages + s * kSlotB);
        const uint32_t qs = smem_u32(qt);
#pragma unroll
        for (int kk = 0; kk < kHD / 16; ++kk) {
          const uint64_t bdesc = sdesc_sw128(qs + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024);
#pragma unroll
          for (int pl = 0; pl < NPL; ++pl) {
            const uint64_t adesc = sdesc_sw128(kt + pl * kSlot + kk * 16 * 128, kHalf, 1024);
            umma_bf16(tmem + b * kTok, adesc, bdesc, idesc, (kk | pl) != 0);
          }
        }
        umma_commit(&bars->s_full[b]);
        umma_commit(&bars->empty[s]);
      }
      __syncwarp();
      if (j >= 1) mma2(j - 1);
    }
    mma2(nb - 1);
    if (elect_one()) umma_commit(&bars->o_full);
    __syncwarp();
  } else {
    // --------------------------------------------- exp / epilogue warps
    const int t = threadIdx.x - 64;
    const int q4 = warp & 3;             // TMEM lane quarter
    const int row = q4 * 32 + lane;      // kv row of S^T, then head-dim row of O^T
    float dsum[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) dsum[i] = 0.f;
    for (int j = 0; j < nb; ++j) {
      const int b = j & 1;
      mbar_wait(&bars->s_full[b], (j >> 1) & 1);
      __syncwarp();
      tc_fence_after();
      float sv[16];
      tmem_ld16(tmem + (uint32_t(q4 * 32) << 16) + b * kTok, sv);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->s_empty[b]);
      if (j >= 2) mbar_wait(&bars->p_empty[b], ((j - 2) >> 1) & 1);
      uint8_t *pb = pbuf + b * kPBytes;
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) {
        const float e = expf(SPLIT ? sv[qq] + sv[qq + 8] : sv[qq]);  // SPLIT: Q hi + lo rows
        dsum[qq] += e;
        const __nv_bfloat16 hi = __float2bfloat16_rn(e);
        const __nv_bfloat16 lo = __float2bfloat16_rn(e - __bfloat162float(hi));
        *reinterpret_cast<__nv_bfloat16 *>(pb + kmaj_off(qq, row)) = hi;
        *reinterpret_cast<__nv_bfloat16 *>(pb + kmaj_off(qq + 8, row)) = lo;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->p_full[b]);
    }
    // denominator partial of this CTA: reduce the 128 kv rows
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int o = 16; o; o >>= 1) dsum[i] += __shfl_xor_sync(0xffffffffu, dsum[i], o);
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < 8; ++i) wsum[q4 * 8 + i] = dsum[i];
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (t < 8) dpart[rank * 8 + t] = wsum[t] + wsum[8 + t] + wsum[16 + t] + wsum[24 + t];
    asm volatile("bar.sync 1, 128;" ::: "memory");

    mbar_wait(&bars->o_full, 0);
    if (threadIdx.x == 64) TPO_T(5);
    __syncwarp();
    tc_fence_after();
    float ov[16], o[8];
    tmem_ld16(tmem + (uint32_t(q4 * 32) << 16) + 32, ov);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = ov[i] + ov[8 + i];
    const int owner = row / rows_per;
    if (S > 1) {
      cluster_wait();
      if (owner != int(rank)) {
        const int slot = int(rank) < owner ? int(rank) : int(rank) - 1;
        const uint32_t dst = map_rank(red + (slot * rows_per + (row - owner * rows_per)) * 8, owner);
        const uint32_t mb = map_rank(&bars->recv, owner);
        st_async4(dst, o[0], o[1], o[2], o[3], mb);
        st_async4(dst + 16, o[4], o[5], o[6], o[7], mb);
      }
      if (t < 2) {
        const float *src = dpart + rank * 8 + t * 4;
        for (int pr = 0; pr < S; ++pr) {
          if (pr == int(rank)) continue;
          st_async4(map_rank(src, pr), src[0], src[1], src[2], src[3], map_rank(&bars->recv, pr));
        }
      }
      mbar_wait(&bars->recv, 0);
      if (threadIdx.x == 64) TPO_T(6);
    }
    if (owner == int(rank)) {
      for (int rr = 0; rr < S; ++rr) {
        if (rr == int(rank)) continue;
        const int slot = rr < int(rank) ? rr : rr - 1;
        const float *src = red + (slot * rows_per + (row - owner * rows_per)) * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] += src[i];
      }
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) {
        if (qq >= p.qh) break;
        float den = 0.f;
        for (int rr = 0; rr < S; ++rr) den += dpart[rr * 8 + qq];
        p.out[(size_t(g) * p.qh + qq) * kHD + row] = o[qq] / den;
      }
    }
  }
  if (S > 1 && warp < 2) {
    __syncwarp();
    cluster_wait();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<64>(tmem);
  }
  if (threadIdx.x == 0) TPO_T(7);
#undef TPO_T
}

template <int SLOTS, int S, bool SPLIT>
size_t gqa_smem() {
  return size_t(SLOTS) * kSlot * (SPLIT ? 2 : 1) + kQBytes + 2 * kPBytes + (S - 1) * (kHD / S) * 8 * 4 + 4 * 8 * 4 +
         4 * 8 * 4 + sizeof(Bars) + 1024;
}

template <int SLOTS, int S, int MINB, bool SPLIT>
cudaError_t launch_t(const CUtensorMap *maps, const GqaParams &p, cudaStream_t st) {
  const size_t smem = gqa_smem<SLOTS, S, SPLIT>();
  auto kern = gqa_kernel<SLOTS, S, MINB, SPLIT>;
  if (cudaError_t e = tpo_ensure_smem(reinterpret_cast<const void *>(kern), smem)) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.groups * S);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = S;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], maps[4], p);
}

}  // namespace tpo_gqa

// maps: {K^T, V, Q^T, K^T lo plane, V lo plane}; split = 1: the SPLIT kernel
extern "C" int tpo_gqa_launch(int slots, int minb, int split, const CUtensorMap *maps,
                              const GqaParams *p, cudaStream_t st) {
  using namespace tpo_gqa;
#define TPO_CASE(SL, S, MB, SP)                                                 \
  if (slots == SL && p->ksplit == S && minb == MB && bool(split) == SP) \
    return int(launch_t<SL, S, MB, SP>(maps, *p, st));
  TPO_CASE(5, 1, 1, false) TPO_CASE(6, 1, 1, false) TPO_CASE(6, 2, 1, false) TPO_CASE(5, 4, 1, false)
  TPO_CASE(6, 4, 1, false) TPO_CASE(4, 2, 1, false) TPO_CASE(5, 2, 1, false) TPO_CASE(3, 2, 2, false)
  TPO_CASE(3, 4, 2, false) TPO_CASE(3, 1, 1, true) TPO_CASE(3, 2, 1, true) TPO_CASE(3, 4, 1, true)
#undef TPO_CASE
  return int(cudaErrorInvalidValue);
}

extern "C" size_t tpo_gqa_smem(int slots, int ksplit) {
  using namespace tpo_gqa;
  if (slots == 3 && ksplit == 2) return gqa_smem<3, 2, false>();
  if (slots == 3 && ksplit == 4) return gqa_smem<3, 4, false>();
  return 0;
}
