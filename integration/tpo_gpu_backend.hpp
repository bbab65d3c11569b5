// Reference-side binding of the B200 backend (a file a maintainer adds to the
// reference's tpo_core).  Re-exposes the reference entry
// points of the µGraph-evaluation hot path with their own types, backed by
// the C-ABI in include/tpo_gpu.h:
//
//   tpo::interp::eval_mugraph                proj/core/include/tpo/interp/interp.hpp:47-48
//   tpo::verify::random_test_equivalence     proj/core/include/tpo/verify/equiv.hpp:50-53
//   (batched) the search loop's per-candidate verification
//
// Graphs cross the ABI in the reference's own wire format
// (tpo::ir::to_json, proj/core/include/tpo/ir/serialize.hpp:33).  Errors come
// back as the reference's tpo::Error with the same ErrCode.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "tpo/interp/interp.hpp"
#include "tpo/ir/graph.hpp"
#include "tpo/verify/equiv.hpp"
#include "tpo_gpu.h"

namespace tpo::gpu {

/// A compiled graph handle (validated with B200 limits, lowered).
class CompiledGraph {
 public:
  CompiledGraph(tpo_gpu_ctx *ctx, const ir::KernelGraph &g);
  ~CompiledGraph();
  CompiledGraph(const CompiledGraph &) = delete;
  CompiledGraph &operator=(const CompiledGraph &) = delete;
  /// Adopts a handle from tpo_gpu_compile_many.
  explicit CompiledGraph(tpo_gpu_graph *h) : h_(h) {}
  tpo_gpu_graph *handle() const { return h_; }
  int64_t op_madds() const;
  bool has_fused_kernel() const;

 private:
  tpo_gpu_graph *h_ = nullptr;
};

/// One device (and its stream).  Not thread-safe: use one Backend per host
/// thread, as the reference API is re-entrant per call.
class Backend {
 public:
  explicit Backend(int device = 0);
  ~Backend();
  Backend(const Backend &) = delete;
  Backend &operator=(const Backend &) = delete;

  /// eval_mugraph for host tensors (tpo_gpu_eval_mugraph_f64: doubles in,
  /// doubles out).  A benchmark µGraph runs its fused sm_100a kernel under
  /// the precision policy (default TPO_PREC_AUTO: fp64 operands enter as
  /// bf16 hi + lo, fp32 accumulation; |o - r| <= 1e-3·max(|r|, rms(r))
  /// against interp::eval_mugraph on arbitrary inputs); any other µGraph, or
  /// `precision` = TPO_PREC_VM, runs on the generic GPU VM in double
  /// arithmetic in the reference's operation order (bit-identical except
  /// exp / SiLU).  TPO_PREC_BF16 rounds the inputs to bf16 instead.
  std::vector<interp::FTensor> eval_mugraph(const ir::KernelGraph &g,
                                            const std::vector<interp::FTensor> &inputs,
                                            int precision = TPO_PREC_AUTO);

  /// random_test_equivalence on the GPU; the verdict (kind, witness,
  /// rounds_run, resamples) is bit-identical to the CPU reference's.
  verify::EquivVerdict random_test_equivalence(const ir::KernelGraph &g1,
                                               const ir::KernelGraph &g2,
                                               const verify::VerifyConfig &cfg,
                                               const verify::FieldParams &fp = verify::FieldParams());

  /// The search loop's batch: candidate k against `program` with
  /// {cfg.num_tests, seeds[k], cfg.max_resamples}.
  std::vector<verify::EquivVerdict> verify_batch(const ir::KernelGraph &program,
                                                 const std::vector<const ir::KernelGraph *> &cands,
                                                 const std::vector<uint64_t> &seeds,
                                                 const verify::VerifyConfig &cfg,
                                                 const verify::FieldParams &fp = verify::FieldParams());

  tpo_gpu_ctx *ctx() const { return ctx_; }

 private:
  tpo_gpu_ctx *ctx_ = nullptr;
};

}  // namespace tpo::gpu
