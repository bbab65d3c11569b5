// B200 backend — Algorithm 1 (§4, SPEC.md generator module): op-by-op
// enumeration of µGraphs in canonical form with abstract-expression pruning.
// The reference lists generator.cpp but does not ship it
// (proj/core/CMakeLists.txt:16)
// specify it.
//
// Kernel level: up to `max_kernel_ops` pre-defined kernel operators
// (Matmul, Ew*, Sqr, Sqrt, SiLU, full Sum) added in increasing rank, each
// kept only if its abstract expression is a subexpression of the
// program's (ConstructOp's expr check), followed by ONE graph-defined
// operator whose block graph computes the program output from the
// remaining kernel tensors.
//
// Block level (GenerateNextBlockOperator): for every data partition — a
// grid label over gx blocks and a set of loop labels over the for-loop —
// the InIters are fixed by the partition and block operators are added
// one at a time in increasing rank (input tensor indices, then type) from
// the pool {EwAdd, EwMul, EwDiv, EwExp, Sqr, Sqrt, SiLU, Matmul,
// ConcatMatmul, Sum, Accum (φ or concatenating)}.  An operator is
// constructed only if
//   * its output shape infers (shape check),
//   * its abstract expression (absexpr.hpp) is a subexpression of the
//     program's (expression check),
//   * shared memory stays within the limit (memory check),
// and the prefix stays completable: every InIter -> tensor path crosses at
// most one Accum and paths of 0 and 1 Accums never merge (Definition 1's
// accumulation rule, decided per prefix), no tensor duplicates an existing
// one's (shape, expression, phase), and the unconsumed tensors can still
// be consumed within the operator budget.  A block graph is complete when
// its only unconsumed tensor carries the program's abstract expression
// behind exactly one Accum on every path ("all shared tensors consumed");
// its OutSaver assembles the kernel output by the grid label.
//
// Equal abstract expressions do not imply equivalence: every emitted
// candidate is for the Z_p×Z_q verifier to decide (tpo_gpu_verify_batch),
// as in the paper's search loop.  Candidates are valid (validate, B200
// limits), deduplicated by canonical key and emitted deterministically.
#pragma once

#include <cstdint>
#include <vector>

#include "tpo/ir/graph.hpp"
#include "tpo/ir/validate.hpp"

namespace tpo::ir {

struct EnumConfig {
  std::vector<int64_t> grids{1, 2, 4, 8, 16};
  std::vector<int64_t> loops{1, 2, 4, 8, 16};
  int max_block_ops = 9;          // compute ops per block graph (InIter / OutSaver excluded)
  int max_kernel_ops = 1;         // pre-defined kernel ops before the GraphDef
  int max_loop_labels = 2;        // loop labels partitioned at once (2: concatenated K, LoRA)
  bool concat_matmul = true;      // the ConcatMatmul operator
  size_t max_candidates = 4096;
  uint64_t max_prefixes = 4000000;  // block prefixes explored, over all partitions
  int threads = 0;                // <= 0: all host cores
  MemLimits limits = kB200Limits;
};

struct EnumStats {
  uint64_t kernel_prefixes = 0;   // kernel-level prefixes (pre-defined ops) kept
  uint64_t partitions = 0;        // (GraphDef inputs, grid, loop) block searches
  uint64_t prefixes = 0;          // block prefixes constructed
  uint64_t pruned_expr = 0;       // ConstructOp: not a subexpression of the program's
  uint64_t pruned_shape = 0;      // ConstructOp: no output shape
  uint64_t pruned_memory = 0;     // ConstructOp: shared memory
  uint64_t pruned_structure = 0;  // accumulation rule / duplicate value / unconsumable
  uint64_t completed = 0;         // complete block graphs (before validate / dedup)
  uint64_t rejected_validate = 0;
  uint64_t duplicates = 0;
  bool budget_exhausted = false;
};

// Throws Error(Unsupported) for a program that is not a single-output
// computation graph of Matmul / Ew* / Sqr / Sqrt / SiLU / full-group Sum.
std::vector<KernelGraph> enumerate_mugraphs(const KernelGraph &program, const EnumConfig &cfg,
                                            EnumStats *stats = nullptr);

// The abstract expression of `g`'s first output, printed (debugging, tests).
std::string abstract_expression(const KernelGraph &g);

}  // namespace tpo::ir
