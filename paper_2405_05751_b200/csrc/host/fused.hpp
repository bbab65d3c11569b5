// B200 backend — recognition of the benchmark µGraphs and launch of their
// hand-written fused sm_100a kernels (csrc/kernels/fused_*.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
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

// One fused evaluation: device inputs in graph-input order with their
// TPO_DTYPE_*, fp32 outputs, the graph's TPO_PREC_* policy.
struct FusedIO {
  const void *const *in = nullptr;
  const int32_t *dt = nullptr;
  float *const *out = nullptr;
  int precision = 0;         // TPO_PREC_AUTO / _BF16
  // the caller's inputs are used in place (no library conversion wrote
  // them on this stream): static weights may stream before the PDL wait
  bool caller_inputs = true;
  int num_sms = 148;
  // device scratch slot `i` of at least `bytes` (operand conversions)
  std::function<void *(int, size_t)> scratch;
};

// Launches the fused kernel for `plan` on `stream`.  Precision (tpo_gpu.h):
// all-bf16 inputs run the bf16 kernel; TPO_PREC_AUTO with any fp32 / fp64
// input converts every input to the split operand forms (bf16 hi + lo) and
// runs the SPLIT kernel; TPO_PREC_BF16 rounds non-bf16 inputs to bf16.
// Returns cudaError_t.
int launch_fused(const FusedPlan &plan, const FusedIO &io, cudaStream_t stream);

}  // namespace tpo::gpu
