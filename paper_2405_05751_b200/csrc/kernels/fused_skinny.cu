// B200 backend — fused skinny-GEMM µGraph kernels (sm_100a, tcgen05 + TMA).
//
// One kernel family executes the GraphDefs of three benchmark µGraphs
// (fixtures.py):
//   GATED   : out = SiLU(X·W1) ⊙ (X·W3)                    (GatedMLP)
//   RMS     : out = (X·G)·W / sqrt(Σ_k X² · D)             (RMSNorm -> MatMul)
//   LORA    : out = X·W + (X·A)·B                           (single-kernel LoRA)
// Each µGraph block graph accumulates φ-Accums over its for-loop; all of them
// are linear, so a block graph instance maps onto a CTA *cluster* that
// splits the for-loop (the K range) S ways: every CTA accumulates its share
// of the loop in TMEM, partial accumulators are summed over DSMEM, and the
// post-loop ops (SiLU·, /sqrt, +XA·B̄) run once in the leader's epilogue.
//
// Block matmuls run on the 5th-gen tensor cores with swap-AB (weights on
// UMMA M=128, the 8 or 16 tokens on N=16): D^T[n, t] = W^T[n, k] · X^T[k, t].
// W tiles are TMA-staged MN-major with 128-byte swizzle; X^T is K-major.
// For RMS the B operand is the exact fp32 product x·g split into bf16
// hi + lo rows (tokens 0-7 = hi, 8-15 = lo), so the tensor cores see no
// rounding of the elementwise product; the two halves are summed in the
// epilogue.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer + TMEM
// owner, warps 2-5 auxiliary (B-tile / side products) and epilogue.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fused.cuh"
#include "sm100.cuh"

namespace tpo_fused {

using namespace sm100;

constexpr int kBK = 64;                   // K per pipeline stage (one 128-B swizzle atom)
constexpr int kTileN = 128;               // UMMA M (weight columns per CTA)
constexpr int kTok = 16;                  // UMMA N (tokens, zero padded)
constexpr uint32_t kWBox = kBK * 128;     // bytes of one 64-col x kBK-row W box
constexpr uint32_t kXTile = kTok * 128;   // bytes of a 16-row x 64-k B tile
constexpr uint32_t kATile = kBK * 32;     // LoRA A tile: kBK rows x 16 cols
constexpr int kThreads = 192;

template <int MODE>
struct Cfg {
  static constexpr int NA = MODE == MODE_GATED ? 2 : 1;              // weight matrices
  static constexpr bool kTmaX = MODE != MODE_RMS;                    // B tile via TMA
  static constexpr uint32_t kStage =
      NA * 2 * kWBox + (kTmaX ? kXTile : 0) + (MODE == MODE_LORA ? kATile : 0);
};

struct __align__(8) Bars {
  uint64_t full[8], empty[8], tmem_full, b_ready;
  uint32_t tmem_base;
};

template <int MODE, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    skinny_kernel(const __grid_constant__ CUtensorMap tmW0, const __grid_constant__ CUtensorMap tmW1,
                  const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmA,
                  const SkinnyParams p) {
  using C = Cfg<MODE>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *stages = smem;
  const int nkb = p.k_per_cta / kBK;
  uint8_t *bregion = stages + STAGES * C::kStage;                       // RMS: all B tiles
  float *red = reinterpret_cast<float *>(bregion + (MODE == MODE_RMS ? nkb * kXTile : 0));
  // red: [S-1][128][16] row partials, then side: [S][kSide]
  constexpr int kSide = MODE == MODE_LORA ? 256 : 8;
  float *side = red + (p.ksplit - 1) * kTileN * 16;
  Bars *bars = reinterpret_cast<Bars *>(side + p.ksplit * kSide);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = p.ksplit > 1 ? cluster_rank() : 0;
  const int tile = blockIdx.x / p.ksplit;
  const int n0 = tile * kTileN;
  const int kbase = int(rank) * p.k_per_cta;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], MODE == MODE_LORA ? 1 + 4 : 1);
    }
    mbar_init(&bars->tmem_full, 1);
    mbar_init(&bars->b_ready, 4);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmW0);
    if (C::NA > 1) tma_prefetch(&tmW1);
    if (C::kTmaX) tma_prefetch(&tmX);
    if (MODE == MODE_LORA) tma_prefetch(&tmA);
  }
  if (warp == 1) tmem_alloc<32>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  if (p.ksplit > 1) cluster_arrive();  // paired with the wait before DSMEM stores
  float acc[16];                       // epilogue warps: this row's accumulator values

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint32_t bytes = C::kStage;
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&bars->empty[s], ((kb / STAGES) & 1) ^ 1);
        uint8_t *st = stages + s * C::kStage;
        mbar_expect_tx(&bars->full[s], bytes);
        const int k0 = kbase + kb * kBK;
        tma_load_2d(st, &tmW0, &bars->full[s], n0, k0);
        tma_load_2d(st + kWBox, &tmW0, &bars->full[s], n0 + 64, k0);
        uint8_t *nx = st + 2 * kWBox;
        if (C::NA > 1) {
          tma_load_2d(nx, &tmW1, &bars->full[s], n0, k0);
          tma_load_2d(nx + kWBox, &tmW1, &bars->full[s], n0 + 64, k0);
          nx += 2 * kWBox;
        }
        if (C::kTmaX) {
          tma_load_2d(nx, &tmX, &bars->full[s], k0, 0);
          nx += kXTile;
        }
        if (MODE == MODE_LORA) tma_load_2d(nx, &tmA, &bars->full[s], 0, k0);
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16(kTileN, kTok, /*a MN-major*/ true, /*b K-major*/ false);
    if (MODE == MODE_RMS) mbar_wait(&bars->b_ready, 0);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&bars->full[s], (kb / STAGES) & 1);
      tc_fence_after();
      if (elect_one()) {
        uint8_t *st = stages + s * C::kStage;
        const uint32_t xs = MODE == MODE_RMS ? smem_u32(bregion + kb * kXTile)
                                             : smem_u32(st + C::NA * 2 * kWBox);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) {
          const uint64_t bdesc = sdesc_sw128(xs + kk * 32, 16, 1024);
#pragma unroll
          for (int w = 0; w < C::NA; ++w) {
            const uint64_t adesc = sdesc_sw128(smem_u32(st + w * 2 * kWBox) + kk * 16 * 128, kWBox, 1024);
            umma_bf16(tmem + w * kTok, adesc, bdesc, idesc, (kb | kk) != 0);
          }
        }
        umma_commit(&bars->empty[s]);
        if (kb == nkb - 1) umma_commit(&bars->tmem_full);
      }
      __syncwarp();
    }
  } else {
    // -------------------------------------- auxiliary warps (2..5): 128 thr
    const int t = threadIdx.x - 64;
    float sidev[kSide > 8 ? 2 : 1] = {};
    float sumsq = 0.f;
    if (MODE == MODE_RMS) {
      // B region: for every k block, 16 rows (x*g hi for tokens 0-7, lo for
      // tokens 8-15) x 64 k, K-major 128-B swizzled like a TMA box.
      // Work item = (k block, token, 16-byte chunk of 8 k): thread t owns a
      // fixed token (t / 16) so its running sum of squares stays per token.
      const int tok = t >> 4;           // 0..7
      const int sub = t & 15;           // 16 threads per token
      for (int item = sub; item < nkb * 8; item += 16) {
        const int kb = item >> 3, c = item & 7;
        const int k = kbase + kb * kBK + c * 8;
        const uint4 xv = tok < p.tokens ? *reinterpret_cast<const uint4 *>(p.x + size_t(tok) * p.K + k)
                                        : make_uint4(0, 0, 0, 0);
        const uint4 gv = *reinterpret_cast<const uint4 *>(p.g + k);
        const __nv_bfloat162 *x2 = reinterpret_cast<const __nv_bfloat162 *>(&xv);
        const __nv_bfloat162 *g2 = reinterpret_cast<const __nv_bfloat162 *>(&gv);
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 xf = __bfloat1622float2(x2[j]), gf = __bfloat1622float2(g2[j]);
          sumsq += xf.x * xf.x + xf.y * xf.y;
          float p0 = xf.x * gf.x, p1 = xf.y * gf.y;  // exact in fp32 (8b x 8b mantissas)
          __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
          float2 hf = __bfloat1622float2(h);
          __nv_bfloat162 l = __floats2bfloat162_rn(p0 - hf.x, p1 - hf.y);  // exact residual
          hi[j] = *reinterpret_cast<uint32_t *>(&h);
          lo[j] = *reinterpret_cast<uint32_t *>(&l);
        }
        uint8_t *tb = bregion + kb * kXTile;
        const int rh = tok, rl = tok + 8;
        *reinterpret_cast<uint4 *>(tb + (rh >> 3) * 1024 + (rh & 7) * 128 + ((c ^ (rh & 7)) << 4)) =
            make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4 *>(tb + (rl >> 3) * 1024 + (rl & 7) * 128 + ((c ^ (rl & 7)) << 4)) =
            make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->b_ready);
      // per-token sum of squares: reduce the 16 threads of each token
#pragma unroll
      for (int o = 8; o; o >>= 1) sumsq += __shfl_xor_sync(0xffffffffu, sumsq, o);
    }
    if (MODE == MODE_LORA) {
      // XA partial (16 tokens x 16 ranks) from the staged X / A tiles while
      // the tensor cores stream W: thread t owns (token t/8, ranks 2*(t%8)..+1).
      const int tok = t >> 3, r0 = (t & 7) * 2;
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&bars->full[s], (kb / STAGES) & 1);
        const uint8_t *xt = stages + s * C::kStage + 2 * kWBox;
        const uint8_t *at = xt + kXTile;
#pragma unroll 8
        for (int k = 0; k < kBK; ++k) {
          // X tile: row tok, element k (K-major SW128); A tile: row k, cols r0, r0+1 (unswizzled)
          const int c = k >> 3;
          const __nv_bfloat16 xv = *reinterpret_cast<const __nv_bfloat16 *>(
              xt + (tok >> 3) * 1024 + (tok & 7) * 128 + ((c ^ (tok & 7)) << 4) + (k & 7) * 2);
          const __nv_bfloat162 av = *reinterpret_cast<const __nv_bfloat162 *>(at + k * 32 + r0 * 2);
          const float xf = __bfloat162float(xv);
          const float2 af = __bfloat1622float2(av);
          sidev[0] += xf * af.x;
          sidev[1] += xf * af.y;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->empty[s]);
      }
    }

    // ---------------------------------------------------------- epilogue
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;       // output column within the tile (UMMA M index)
    mbar_wait(&bars->tmem_full, 0);
    __syncwarp();  // tcgen05.ld is .sync.aligned: the warp must be converged
    tc_fence_after();
    {
      float v[16];
      tmem_ld16(tmem + (uint32_t(q * 32) << 16), v);
      if (MODE == MODE_GATED) {
        float v3[16];
        tmem_ld16(tmem + (uint32_t(q * 32) << 16) + kTok, v3);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = v[i], acc[8 + i] = v3[i];
      } else if (MODE == MODE_RMS) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = v[i] + v[8 + i], acc[8 + i] = 0.f;
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = v[i];
      }
    }
    if (p.ksplit > 1) {
      cluster_wait();  // every CTA of the cluster has started: DSMEM is live
      if (rank != 0) {
        const uint32_t dst = map_rank(red + ((rank - 1) * kTileN + row) * 16, 0);
#pragma unroll
        for (int i = 0; i < 16; i += 4) st_cluster_v4(dst + i * 4, acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
      }
    }
    // side partials (sum of squares / XA) of every rank -> leader
    if (MODE == MODE_RMS && (t & 15) == 0) {
      const uint32_t dst = map_rank(side + rank * kSide + (t >> 4), 0);
      if (p.ksplit > 1)
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dst), "f"(sumsq) : "memory");
      else
        side[t >> 4] = sumsq;
    }
    if (MODE == MODE_LORA) {
      const int tok = t >> 3, r0 = (t & 7) * 2;
      float *loc = side + rank * kSide + tok * 16 + r0;
      if (p.ksplit > 1) {
        const uint32_t dst = map_rank(loc, 0);
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dst), "f"(sidev[0]) : "memory");
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dst + 4), "f"(sidev[1]) : "memory");
      } else {
        loc[0] = sidev[0];
        loc[1] = sidev[1];
      }
    }
  }

  __syncwarp();
  // all partials have landed in the leader once every thread passed this
  if (p.ksplit > 1) {
    if (warp < 2) cluster_wait();  // warps 0/1 still owe the first wait
    cluster_sync();
  } else {
    __syncthreads();
  }

  if (warp >= 2 && rank == 0) {
    const int t = threadIdx.x - 64;
    const int q = warp & 3, row = q * 32 + lane;
    for (int r = 1; r < p.ksplit; ++r) {
      const float4 *src = reinterpret_cast<const float4 *>(red + ((r - 1) * kTileN + row) * 16);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float4 x = src[i];
        acc[4 * i] += x.x, acc[4 * i + 1] += x.y, acc[4 * i + 2] += x.z, acc[4 * i + 3] += x.w;
      }
    }
    const int n = n0 + row;
    if (MODE == MODE_GATED) {
#pragma unroll
      for (int tk = 0; tk < 8; ++tk)
        if (tk < p.tokens) p.out[size_t(tk) * p.N + n] = silu(acc[tk]) * acc[8 + tk];
    } else if (MODE == MODE_RMS) {
      const float dsc = __bfloat162float(p.dscale[0]);
#pragma unroll
      for (int tk = 0; tk < 8; ++tk) {
        float ss = 0.f;
        for (int r = 0; r < p.ksplit; ++r) ss += side[r * kSide + tk];
        if (tk < p.tokens) p.out[size_t(tk) * p.N + n] = acc[tk] / sqrtf(ss * dsc);
      }
    } else {
      // post: XW + XA · B̄   (XA summed over ranks; B̄ = B[:, n] column)
      float bcol[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) bcol[r] = __bfloat162float(p.lora_b[size_t(r) * p.N + n]);
#pragma unroll 4
      for (int tk = 0; tk < 16; ++tk) {
        float s = acc[tk];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          float xa = 0.f;
          for (int rr = 0; rr < p.ksplit; ++rr) xa += side[rr * kSide + tk * 16 + r];
          s += xa * bcol[r];
        }
        if (tk < p.tokens) p.out[size_t(tk) * p.N + n] = s;
      }
    }
    (void)t;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<32>(tmem);
  }
}

template <int MODE, int STAGES>
size_t skinny_smem(const SkinnyParams &p) {
  using C = Cfg<MODE>;
  const int nkb = p.k_per_cta / kBK;
  const int kSide = MODE == MODE_LORA ? 256 : 8;
  size_t b = size_t(STAGES) * C::kStage + (MODE == MODE_RMS ? size_t(nkb) * kXTile : 0) +
             size_t(p.ksplit - 1) * kTileN * 16 * 4 + size_t(p.ksplit) * kSide * 4 + sizeof(Bars);
  return b + 1024;
}

template <int MODE, int STAGES>
cudaError_t launch_t(const CUtensorMap *maps, const SkinnyParams &p, cudaStream_t st) {
  const size_t smem = skinny_smem<MODE, STAGES>(p);
  auto kern = skinny_kernel<MODE, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e) return e;
  if (p.ksplit > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((p.N / kTileN) * p.ksplit);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.ksplit;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], p);
}

}  // namespace tpo_fused

using namespace tpo_fused;

extern "C" int tpo_skinny_launch(int mode, int stages, const CUtensorMap *maps,
                                 const SkinnyParams *p, cudaStream_t st) {
#define TPO_CASE(M, S) \
  if (mode == M && stages == S) return int(launch_t<M, S>(maps, *p, st));
  TPO_CASE(MODE_GATED, 2)
  TPO_CASE(MODE_GATED, 3)
  TPO_CASE(MODE_GATED, 4)
  TPO_CASE(MODE_GATED, 6)
  TPO_CASE(MODE_RMS, 3)
  TPO_CASE(MODE_RMS, 4)
  TPO_CASE(MODE_RMS, 6)
  TPO_CASE(MODE_RMS, 8)
  TPO_CASE(MODE_LORA, 3)
  TPO_CASE(MODE_LORA, 4)
  TPO_CASE(MODE_LORA, 6)
  TPO_CASE(MODE_LORA, 8)
#undef TPO_CASE
  return int(cudaErrorInvalidValue);
}

extern "C" size_t tpo_skinny_smem(int mode, int stages, const SkinnyParams *p) {
  switch (mode * 16 + stages) {
    case MODE_GATED * 16 + 2: return skinny_smem<MODE_GATED, 2>(*p);
    case MODE_GATED * 16 + 3: return skinny_smem<MODE_GATED, 3>(*p);
    case MODE_GATED * 16 + 4: return skinny_smem<MODE_GATED, 4>(*p);
    case MODE_GATED * 16 + 6: return skinny_smem<MODE_GATED, 6>(*p);
    case MODE_RMS * 16 + 3: return skinny_smem<MODE_RMS, 3>(*p);
    case MODE_RMS * 16 + 4: return skinny_smem<MODE_RMS, 4>(*p);
    case MODE_RMS * 16 + 6: return skinny_smem<MODE_RMS, 6>(*p);
    case MODE_RMS * 16 + 8: return skinny_smem<MODE_RMS, 8>(*p);
    case MODE_LORA * 16 + 3: return skinny_smem<MODE_LORA, 3>(*p);
    case MODE_LORA * 16 + 4: return skinny_smem<MODE_LORA, 4>(*p);
    case MODE_LORA * 16 + 6: return skinny_smem<MODE_LORA, 6>(*p);
    case MODE_LORA * 16 + 8: return skinny_smem<MODE_LORA, 8>(*p);
  }
  return 0;
}
