// B200 backend — recognition of the benchmark µGraphs and launch of their
// hand-written fused sm_100a kernels (csrc/kernels/fused_*.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "tpo/ir/graph.hpp"

namespace tpo::gpu {

struct FusedPlan {
  int kind = 0;           // TPO_FUSED_* (include/tpo_gpu.h)
  // problem sizes (meaning per kind)
  int64_t b = 0, h = 0, n = 0, r = 0;   // tokens, reduction dim, out columns, LoRA rank
  int64_t groups = 0, qh = 0, hd = 0, L = 0;  // GQA
  int64_t grid = 0, forloop = 0;        // the µGraph's block-graph schedule
  std::string why;                      // reason when kind == 0
  uint64_t static_inputs = 0;           // bit i: input i is never written by work
                                        // enqueued before an evaluation (weights)
};

// Structural match of a KernelGraph against the four benchmark µGraph forms
// (SURVEY §8d).  Never throws.
FusedPlan match_fused(const ir::KernelGraph &g);

// Launches the fused kernel for `plan` on `stream`; inputs in graph-input
// order (bf16 unless stated), output fp32.  Returns cudaError_t.
int launch_fused(const FusedPlan &plan, const void *const *in, const int32_t *in_dtype,
                 float *const *out, void *workspace, size_t ws_bytes, cudaStream_t stream);

size_t fused_workspace_bytes(const FusedPlan &plan);

}  // namespace tpo::gpu
