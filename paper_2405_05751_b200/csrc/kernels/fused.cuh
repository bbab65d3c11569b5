// B200 backend — launch contract of the fused µGraph kernels.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

enum { MODE_GATED = 1, MODE_RMS = 2, MODE_LORA = 3 };

struct SkinnyParams {
  int N, K, tokens;          // out columns, reduction dim, live tokens (<= 8, LoRA <= 16)
  int ksplit, k_per_cta;     // cluster size along K and K elements per CTA
  const __nv_bfloat16 *x;    // RMS: X [tokens, K]
  const __nv_bfloat16 *g;    // RMS: G [1, K]
  const __nv_bfloat16 *dscale;  // RMS: D [1, 1]
  const __nv_bfloat16 *lora_a;  // LoRA: A [K, 16]
  const float *dscale_f32;   // SPLIT RMS: D [1, 1] fp32
  float *out;                // [tokens, N] fp32
  unsigned long long *dbg;   // optional per-CTA phase timestamps (TPO_DEBUG_TIMES)
  int dbg_flags;             // experiments (TPO_DBG_FLAGS): 1 skip finalize
  int prefetch_static;       // weights are static: stream them before the PDL wait
  int epi_atomic;            // RMS/LoRA split clusters: fp32-reduction epilogue
  int trig_early;            // experiment: producer triggers dependents this many k blocks early
  int pre_cut;               // experiment: prefetch this many fewer static stages
  int l2_ahead;              // weight k blocks requested into L2 ahead of the ring (after the wait)
  int tma_out;               // outputs by one TMA tile store per owner warp (map 7)
  int x_l2;                  // activations requested into L2 before the PDL wait
};

struct GqaParams {
  int groups, qh, hd, L;     // Q [g, qh, hd], K^T [g, hd, L], V [g, L, hd]
  int ksplit, l_per_cta;     // cluster split of the kv loop
  const __nv_bfloat16 *q;
  float *out;                // [g, qh, hd]
  unsigned long long *dbg;   // optional per-CTA phase timestamps (TPO_DEBUG_TIMES)
  int consume_order;         // ring filled K_0, K_1, V_0, K_2, V_1, ... (the MMA issue order)
  int l2_units;              // ring units (and Q) requested into L2 before the PDL wait
};

// maps: {W plane 0, W plane 1, X, A / G, W plane 2 | LoRA B̄ (hi), W plane 3 | LoRA B̄ lo, A lo plane, out (fp32, TPO_TMA_OUT)}
extern "C" int tpo_skinny_launch(int mode, int stages, int minb, int split, const CUtensorMap *maps,
                                 const SkinnyParams *p, cudaStream_t st);
extern "C" size_t tpo_skinny_smem(int mode, int stages, int minb, int split, const SkinnyParams *p);
extern "C" int tpo_gqa_launch(int slots, int minb, int split, const CUtensorMap *maps,
                              const GqaParams *p, cudaStream_t st);
extern "C" size_t tpo_gqa_smem(int slots, int ksplit);
