// B200 backend — block-graph operator scheduling and shared-memory planning
// (the reference's absent core/src/schedule.cpp and memplan.cpp,
// proj/core/CMakeLists.txt:19-20).
//
// schedule_ops orders a block graph's operators by depth (longest path
// from an operator without producers) so that synchronisation is needed
// only between consecutive depth levels; plan_memory assigns shared-memory
// offsets from the schedule's tensor lifetimes (exhaustive over placement
// orders for <= 8 tensors, first-fit-decreasing above).  The VM lowering
// (csrc/host/lower.cpp) emits block ops in this order, places its buffers
// with plan_intervals, and the VM interpreters synchronise only between
// dependent phases (VM_NOSYNC).
#pragma once

#include <cstdint>
#include <vector>

#include "tpo/ir/graph.hpp"
#include "tpo/ir/validate.hpp"

namespace tpo::ir {

struct Schedule {
  std::vector<int> order;       // op ids, execution order (a topological order)
  std::vector<int> depth;       // per op id: 1 + max depth of its producers (0 if none)
  std::vector<int> post;        // per op id: 1 iff post-loop (eval_core.hpp:277-294)
  std::vector<int> sync_after;  // positions p in `order` followed by a sync point
};

// Depth schedule of one block graph (SPEC schedule_ops).  Ops are sorted
// ascending by depth within each execution phase (for-loop body, then
// post-loop); ties keep the canonical rank (input (producer op, output)
// tuples, then op type, then list position).  OutSavers close the post
// phase in list order (OutSaver #k writes GraphDef output k).  A sync point
// separates consecutive ops of different depth, and the two phases.
Schedule schedule_ops(const BlockGraph &bg);

// One buffer for the planner: `size` bytes (or words) live over the
// inclusive schedule positions [start, end].  Two buffers conflict iff
// their lifetimes intersect.
struct Lifetime {
  int64_t size, start, end;
};

struct MemoryPlan {
  std::vector<int64_t> offset;  // per buffer (-1: not in shared memory)
  int64_t peak = 0;
  bool exhaustive = false;      // optimal (all placement orders tried)
};

// Minimal-peak placement of `buf` (SPEC plan_memory): for n <= exhaustive_max
// every placement order is tried with lowest-offset first fit (optimal for
// interval lifetimes: the first fit of an optimal packing sorted by offset
// never lands higher); above, first-fit-decreasing by size.
MemoryPlan plan_intervals(const std::vector<Lifetime> &buf, int exhaustive_max = 8);

// Shared-memory plan of one block graph under `sched`: one buffer per
// block tensor outside the register-resident interior edges of its thread
// groups (validate.cpp:115-140 accounting), elem_size bytes per element.
// Lifetimes run from the producer's barrier phase (depth level) to the last
// consumer's — ops of one phase run without a sync between them, so their
// buffers may not alias — and accumulators are live over the whole loop body.  Throws
// Error(DoesNotFit) when the optimal peak exceeds limits.smem_bytes.
MemoryPlan plan_memory(const BlockGraph &bg, const Schedule &sched, const MemLimits &limits);

}  // namespace tpo::ir
