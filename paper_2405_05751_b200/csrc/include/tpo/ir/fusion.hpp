// B200 backend — thread-graph construction (the reference's absent
// core/src/fusion.cpp, proj/core/CMakeLists.txt:17).
#pragma once

#include "tpo/ir/graph.hpp"

namespace tpo::ir {

// Greedily fuses maximal chains of elementwise block ops (op_elementwise:
// EwAdd, EwMul, EwDiv, EwExp, Sqr, Sqrt, SiLU) of one block graph into
// ThreadGroups whose interior edges are register-resident: an op joins its
// producer's group when it is that producer's only consumer (no fusing past
// a fan-out point) and both run in the same phase (for-loop body or
// post-loop).  Replaces any existing groups; the fixpoint of the pairwise
// rule is reached in one union-find pass.  Semantics are unchanged (the
// evaluator ignores thread groups, eval_core.hpp); only the shared-memory
// accounting (block_shared_bytes, validate.cpp:115-140) changes.
void construct_thread_groups(BlockGraph &bg);

// construct_thread_groups on every GraphDef of `g` (SPEC construct_thread_graphs).
KernelGraph construct_thread_graphs(const KernelGraph &g);

}  // namespace tpo::ir
