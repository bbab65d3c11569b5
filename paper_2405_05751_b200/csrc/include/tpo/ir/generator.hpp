// B200 backend — fused-kernel candidate generator (first slice of the
// reference's absent generator.cpp, proj/core/CMakeLists.txt:16;
// SPEC.md:254-352, Algorithm 1).
//
// Algorithm 1 enumerates µGraph prefixes op by op and prunes them with
// abstract expressions (the expr engine, out of scope here).  This slice
// targets the candidates the GPU verifier and the fused kernels consume:
// single-GraphDef µGraphs that fuse a whole computation graph into one
// kernel.  It enumerates the data partition instead of op sequences:
//
//  * dimension labels: (tensor, dim) pairs unified through the ops
//    (broadcast elementwise, matmul m/n/k and batch, full-group Sum);
//  * a grid label (an output dimension, split over grid x) and a for-loop
//    label (a contracted dimension, split over the loop) with extents from
//    the config; every input's imap / fmap follows from its labels;
//  * ops are placed by partition state: loop-sliced values stay in the
//    loop body, contractions over the loop label yield partial sums, which
//    flow through linear ops (scaling by loop-invariant values, sums,
//    matmuls with invariant operands) and are accumulated (φ-Accum) before
//    the first non-linear use — "late" placement — or right after the
//    contraction — "early" placement; post-loop ops follow;
//  * one algebraic rewrite exposes more fusion: a matmul of a row-scaled
//    operand, Matmul(A ∘ s, W) with s broadcast along the contracted dim,
//    becomes (Matmul(A, W)) ∘ s for ∘ ∈ {EwMul, EwDiv} (Fig. 2's RMSNorm).
//
// Every emitted graph passes validate (B200 limits); equivalence with the
// program is the verifier's job (tpo_gpu_verify_batch), as in the search
// loop.  Candidates are deduplicated by canonical key and emitted in a
// deterministic order.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "tpo/ir/graph.hpp"
#include "tpo/ir/validate.hpp"

namespace tpo::ir {

struct GenConfig {
  std::vector<int64_t> grids{1, 2, 4, 8, 16, 32, 64, 128};
  std::vector<int64_t> loops{1, 2, 4, 8, 16, 32, 64};
  bool rewrite = true;          // also try the row-scale rewrite of the program
  size_t max_candidates = 4096;
  MemLimits limits = kB200Limits;
  // Multi-kernel µGraphs (generate_multi): at most this many kernels, each a
  // contiguous single-output segment of the program's op list lowered as a
  // pre-defined kernel op (one-op segments) or one of the first
  // `per_segment` fused GraphDef candidates of the segment.
  int max_kernels = 1;
  int per_segment = 3;
};

struct GenStats {
  int64_t partitions = 0;       // (program form, grid label/extent, loop label/extent) tried
  int64_t placements = 0;       // block graphs built
  int64_t rejected_structure = 0;  // partition state conflicts (e.g. a loop slice used post-loop)
  int64_t rejected_validate = 0;   // Definition-1 / memory violations
  int64_t duplicates = 0;
};

// Throws Error(Unsupported) for a program that is not a single-output
// computation graph of Matmul / Ew* / Sqr / Sqrt / SiLU / full-group Sum.
std::vector<KernelGraph> generate_fused(const KernelGraph &program, const GenConfig &cfg,
                                        GenStats *stats = nullptr);

// Algorithm 1's kernel level: µGraphs of up to cfg.max_kernels kernels.  The
// program's op list (a topological order) is cut into contiguous segments
// with one externally used output each; every segment becomes a
// pre-defined kernel op (a one-op segment) or a fused GraphDef from
// generate_fused on the segment's sub-program; the kernels are chained
// through device tensors.  Includes generate_fused's single-kernel
// candidates; deduplicated by canonical key; deterministic.
std::vector<KernelGraph> generate_multi(const KernelGraph &program, const GenConfig &cfg,
                                        GenStats *stats = nullptr);

}  // namespace tpo::ir
