// B200 backend — depth scheduling and shared-memory planning of block
// graphs; see tpo/ir/schedule.hpp.
#include "tpo/ir/schedule.hpp"

#include <algorithm>
#include <numeric>
#include <tuple>

#include "tpo/ir/ops.hpp"

namespace tpo::ir {

namespace {

// Interior edges of thread groups live in registers (validate.cpp:115-140).
std::vector<char> register_resident(const BlockGraph &bg) {
  std::vector<char> reg(bg.tensors.size(), 0);
  for (const ThreadGroup &tg : bg.thread_groups) {
    std::vector<char> member(bg.ops.size(), 0);
    for (int id : tg.op_ids) member[size_t(id)] = 1;
    for (int id : tg.op_ids)
      for (TensorId out : bg.ops[size_t(id)].outputs) {
        bool any = false, inside = true;
        for (const Op &o : bg.ops)
          for (TensorId t : o.inputs)
            if (t == out) {
              any = true;
              if (!member[size_t(o.id)]) inside = false;
            }
        if (any && inside) reg[size_t(out)] = 1;
      }
  }
  return reg;
}

}  // namespace

Schedule schedule_ops(const BlockGraph &bg) {
  const size_t n = bg.ops.size(), nt = bg.tensors.size();
  Schedule s;
  s.depth.assign(n, 0);
  s.post.assign(n, 0);
  std::vector<int> prod(nt, -1), prod_out(nt, 0);
  for (size_t k = 0; k < n; ++k)
    for (size_t j = 0; j < bg.ops[k].outputs.size(); ++j) {
      prod[size_t(bg.ops[k].outputs[j])] = int(k);
      prod_out[size_t(bg.ops[k].outputs[j])] = int(j);
    }
  // post phase: Accum outputs and their descendants (eval_core.hpp:277-294)
  std::vector<char> post_t(nt, 0);
  for (size_t k = 0; k < n; ++k) {
    const Op &op = bg.ops[k];
    if (op.type == OpType::Accum) {
      post_t[size_t(op.outputs[0])] = 1;
      continue;
    }
    bool p = op.type == OpType::OutSaver;
    for (TensorId t : op.inputs) p = p || post_t[size_t(t)];
    if (op.type != OpType::InIter && p) {
      s.post[k] = 1;
      for (TensorId t : op.outputs) post_t[size_t(t)] = 1;
    }
  }
  // longest path (list order is topological: builders append ops after
  // their inputs, validate.cpp)
  for (size_t k = 0; k < n; ++k) {
    int d = 0;
    for (TensorId t : bg.ops[k].inputs)
      if (prod[size_t(t)] >= 0) d = std::max(d, s.depth[size_t(prod[size_t(t)])]);
    s.depth[k] = d + 1;
  }
  auto rank = [&](int k) {
    std::vector<std::pair<int, int>> in;
    for (TensorId t : bg.ops[size_t(k)].inputs) in.emplace_back(prod[size_t(t)], prod_out[size_t(t)]);
    return std::make_tuple(in, int(bg.ops[size_t(k)].type), k);
  };
  std::vector<int> loop_ops, post_ops, savers;
  for (size_t k = 0; k < n; ++k) {
    if (bg.ops[k].type == OpType::OutSaver)
      savers.push_back(int(k));
    else
      (s.post[k] ? post_ops : loop_ops).push_back(int(k));
  }
  auto by_depth = [&](std::vector<int> &v) {
    std::stable_sort(v.begin(), v.end(), [&](int a, int b) {
      if (s.depth[size_t(a)] != s.depth[size_t(b)]) return s.depth[size_t(a)] < s.depth[size_t(b)];
      return rank(a) < rank(b);
    });
  };
  by_depth(loop_ops);
  by_depth(post_ops);
  s.order = loop_ops;
  s.order.insert(s.order.end(), post_ops.begin(), post_ops.end());
  s.order.insert(s.order.end(), savers.begin(), savers.end());
  for (size_t p = 0; p + 1 < s.order.size(); ++p) {
    const int a = s.order[p], b = s.order[p + 1];
    const bool phase_change = s.post[size_t(a)] != s.post[size_t(b)] ||
                              (bg.ops[size_t(a)].type == OpType::OutSaver) !=
                                  (bg.ops[size_t(b)].type == OpType::OutSaver);
    if (phase_change || s.depth[size_t(a)] != s.depth[size_t(b)]) s.sync_after.push_back(int(p));
  }
  return s;
}

MemoryPlan plan_intervals(const std::vector<Lifetime> &buf, int exhaustive_max) {
  const size_t n = buf.size();
  MemoryPlan best;
  best.offset.assign(n, -1);
  if (!n) {
    best.exhaustive = true;
    return best;
  }
  auto conflict = [&](size_t a, size_t b) {
    return buf[a].start <= buf[b].end && buf[b].start <= buf[a].end;
  };
  // lowest-offset first fit in `order`; returns the peak
  std::vector<int64_t> off(n);
  std::vector<std::pair<int64_t, int64_t>> busy;
  auto place = [&](const std::vector<size_t> &order, int64_t cut) {
    int64_t peak = 0;
    for (size_t i = 0; i < order.size(); ++i) {
      const size_t v = order[i];
      busy.clear();
      for (size_t j = 0; j < i; ++j)
        if (conflict(v, order[j])) busy.emplace_back(off[order[j]], off[order[j]] + buf[order[j]].size);
      std::sort(busy.begin(), busy.end());
      int64_t at = 0;
      for (auto [lo, hi] : busy) {
        if (at + buf[v].size <= lo) break;
        at = std::max(at, hi);
      }
      off[v] = at;
      peak = std::max(peak, at + buf[v].size);
      if (peak >= cut) return peak;  // cannot beat the incumbent
    }
    return peak;
  };
  std::vector<size_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  if (int(n) <= exhaustive_max) {
    int64_t bp = INT64_MAX;
    do {
      const int64_t pk = place(order, bp);
      if (pk < bp) {
        bp = pk;
        best.offset = off;
      }
    } while (std::next_permutation(order.begin(), order.end()));
    best.peak = bp;
    best.exhaustive = true;
    return best;
  }
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return buf[a].size > buf[b].size; });
  best.peak = place(order, INT64_MAX);
  best.offset = off;
  return best;
}

MemoryPlan plan_memory(const BlockGraph &bg, const Schedule &sched, const MemLimits &limits) {
  const size_t nt = bg.tensors.size();
  const std::vector<char> reg = register_resident(bg);
  // lifetimes in barrier phases, not positions: ops of one depth run
  // without a sync between them, so a buffer read in a phase may not be
  // reused by a write in that same phase
  std::vector<int> phase_of(sched.order.size(), 0);
  {
    int ph = 0;
    size_t k = 0;
    for (size_t p = 0; p < sched.order.size(); ++p) {
      phase_of[p] = ph;
      if (k < sched.sync_after.size() && sched.sync_after[k] == int(p)) ++ph, ++k;
    }
  }
  std::vector<int> pos(bg.ops.size(), -1);
  for (size_t p = 0; p < sched.order.size(); ++p) pos[size_t(sched.order[p])] = phase_of[p];
  int loop_end = -1;  // last phase of the for-loop body
  for (size_t p = 0; p < sched.order.size(); ++p)
    if (!sched.post[size_t(sched.order[p])] && bg.ops[size_t(sched.order[p])].type != OpType::OutSaver)
      loop_end = phase_of[p];
  std::vector<int64_t> start(nt, -1), end(nt, -1);
  for (const Op &op : bg.ops) {
    const int p = pos[size_t(op.id)];
    for (TensorId t : op.outputs) {
      start[size_t(t)] = op.type == OpType::Accum ? 0 : p;  // accumulators persist over the loop
      end[size_t(t)] = std::max<int64_t>(end[size_t(t)], op.type == OpType::Accum ? loop_end : p);
    }
    for (TensorId t : op.inputs) end[size_t(t)] = std::max<int64_t>(end[size_t(t)], p);
  }
  std::vector<Lifetime> buf;
  std::vector<size_t> who;
  for (size_t t = 0; t < nt; ++t) {
    if (reg[t] || start[t] < 0) continue;
    buf.push_back({bg.tensors[t].shape.elem_count() * limits.elem_size, start[t], std::max(start[t], end[t])});
    who.push_back(t);
  }
  MemoryPlan pb = plan_intervals(buf);
  MemoryPlan out;
  out.offset.assign(nt, -1);
  for (size_t i = 0; i < who.size(); ++i) out.offset[who[i]] = pb.offset[i];
  out.peak = pb.peak;
  out.exhaustive = pb.exhaustive;
  if (out.peak > limits.smem_bytes)
    throw Error(ErrCode::DoesNotFit, "block graph needs " + std::to_string(out.peak) +
                                         " B of shared memory, limit " + std::to_string(limits.smem_bytes));
  return out;
}

}  // namespace tpo::ir
