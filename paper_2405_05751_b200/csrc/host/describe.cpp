// B200 backend — `describe`: a human-readable pseudo-kernel listing of a
// µGraph (the reference's absent describe.cpp, proj/core/CMakeLists.txt:25;
// SPEC.md:686-692): per kernel op its grid and for-loop, the InIter /
// Accum / OutSaver maps, the block ops in schedule order with sync markers
// and shared-memory offsets (tpo/ir/schedule.hpp), and how this backend
// runs it on B200 (the fused sm_100a kernel it matches, else the VM
// bytecode: instructions, barrier phases, working-set words).
#include <sstream>
#include <string>

#include "fused.hpp"
#include "lower.hpp"
#include "tpo/ir/schedule.hpp"
#include "tpo/ir/validate.hpp"

namespace tpo::gpu {

using namespace ir;

namespace {

std::string shape_str(const TensorShape &s) {
  std::ostringstream o;
  o << "[";
  for (size_t i = 0; i < s.dims.size(); ++i) o << (i ? ", " : "") << s.dims[i];
  o << "]";
  return o.str();
}

// {x: 1, y: φ} for grid maps, {i: 0} for the for-loop map
std::string map_str(const DimMap &m, bool grid_axes) {
  static const char *ax[3] = {"x", "y", "z"};
  std::ostringstream o;
  o << "{";
  for (int a = 0; a < m.axes(); ++a) {
    o << (a ? ", " : "") << (grid_axes ? ax[a] : "i") << ": ";
    if (m.targets[size_t(a)] == kReplica)
      o << "phi";
    else
      o << m.targets[size_t(a)];
  }
  o << "}";
  return o.str();
}

std::string attrs_str(const Op &op) {
  std::ostringstream o;
  if (auto *a = std::get_if<InIterAttrs>(&op.attrs))
    o << " operand " << a->operand << " imap " << map_str(a->imap, true) << " fmap " << map_str(a->fmap, false);
  else if (auto *a = std::get_if<OutSaverAttrs>(&op.attrs))
    o << " omap " << map_str(a->omap, true);
  else if (auto *a = std::get_if<AccumAttrs>(&op.attrs))
    o << " fmap " << map_str(a->fmap, false);
  else if (auto *a = std::get_if<SumAttrs>(&op.attrs))
    o << " dim " << a->dim << " group " << a->group;
  else if (auto *a = std::get_if<ReshapeAttrs>(&op.attrs))
    o << " to " << shape_str(a->target);
  else if (auto *a = std::get_if<RepeatAttrs>(&op.attrs))
    o << " to " << shape_str(a->target);
  return o.str();
}

std::string ids(const std::vector<TensorId> &v, char tag) {
  std::ostringstream o;
  for (size_t i = 0; i < v.size(); ++i) o << (i ? ", " : "") << tag << v[i];
  return o.str();
}

}  // namespace

std::string describe(const KernelGraph &g, const MemLimits &lim) {
  std::ostringstream o;
  if (g.ops.empty() && g.inputs.empty()) return "";
  o << "kernel graph: " << g.inputs.size() << " input(s), " << g.outputs.size() << " output(s), "
    << g.ops.size() << " op(s)\n";
  for (TensorId t : g.inputs) o << "  input t" << t << " " << shape_str(g.tensor(t).shape) << "\n";
  for (size_t k = 0; k < g.ops.size(); ++k) {
    const Op &op = g.ops[k];
    o << "op " << k << ": " << op_name(op.type) << "(" << ids(op.inputs, 't') << ") -> " << ids(op.outputs, 't');
    for (TensorId t : op.outputs) o << " " << shape_str(g.tensor(t).shape);
    o << attrs_str(op) << "\n";
    if (op.type != OpType::GraphDef || !op.block) continue;
    const BlockGraph &bg = *op.block;
    o << "  grid (" << bg.grid[0] << ", " << bg.grid[1] << ", " << bg.grid[2] << ")  forloop i=" << bg.forloop
      << "  block ops " << bg.ops.size() << "  thread groups " << bg.thread_groups.size() << "\n";
    const Schedule s = schedule_ops(bg);
    MemoryPlan m;
    std::string mem_err;
    try {
      m = plan_memory(bg, s, lim);
    } catch (const Error &e) {
      mem_err = e.what();
    }
    int acc = 0;
    for (const Op &b : bg.ops) acc += b.type == OpType::Accum;
    o << "  accumulators " << acc << "  sync points " << s.sync_after.size();
    if (mem_err.empty())
      o << "  shared memory peak " << m.peak << " B (" << (m.exhaustive ? "optimal" : "first-fit-decreasing")
        << ")\n";
    else
      o << "  shared memory: " << mem_err << "\n";
    int phase = -1;  // 0 loop body, 1 post-loop, 2 outsavers
    for (size_t p = 0; p < s.order.size(); ++p) {
      const int id = s.order[p];
      const Op &b = bg.ops[size_t(id)];
      const int ph = b.type == OpType::OutSaver ? 2 : s.post[size_t(id)];
      if (ph != phase) {
        o << (ph == 0 ? "  for i in [0, " + std::to_string(bg.forloop) + "):\n"
                      : ph == 1 ? "  after the loop:\n" : "  save:\n");
        phase = ph;
      }
      o << "    [d" << s.depth[size_t(id)] << "] " << op_name(b.type) << "(" << ids(b.inputs, 'b') << ") -> "
        << ids(b.outputs, 'b');
      for (TensorId t : b.outputs) {
        o << " " << shape_str(bg.tensor(t).shape);
        if (mem_err.empty()) {
          const int64_t off = m.offset[size_t(t)];
          if (off < 0)
            o << " @reg";
          else
            o << " @smem+" << off;
        }
      }
      o << attrs_str(b) << "\n";
      for (int sp : s.sync_after)
        if (sp == int(p)) o << "    ---- sync\n";
    }
  }
  o << "outputs: " << ids(g.outputs, 't') << "\n";
  // how the B200 backend runs it
  const FusedPlan fp = match_fused(g);
  if (fp.kind) {
    static const char *kn[] = {"", "rmsnorm_matmul", "gated_mlp", "gqa_decode", "lora"};
    o << "B200: fused sm_100a kernel " << (fp.kind >= 1 && fp.kind <= 4 ? kn[fp.kind] : "?")
      << " (tcgen05 + TMA, one launch per evaluation)\n";
  } else {
    o << "B200: no fused kernel (" << fp.why << ")";
    try {
      const VmProgram vp = lower_vm(g, 0, uint32_t(input_elems(g)), false, /*field=*/false);
      int instrs = 0, phases = 0, chained = 0;
      for (const TpoVmInstr &I : vp.code) {
        if (I.op == VM_LOOP || I.op == VM_ENDLOOP) continue;
        ++instrs;
        phases += !(I.flags & VM_NOSYNC);
        chained += (I.pre_a != 0) + (I.pre_b != 0);
      }
      o << "; VM bytecode: " << instrs << " instructions in " << phases << " barrier phases, "
        << (input_elems(g) + vp.region_words) << " words";
      if (chained) o << "; " << chained << " thread-graph unary(s) fused into their consumers (registers)";
    } catch (const Error &e) {
      o << "; VM: " << e.what();
    }
    o << "\n";
  }
  return o.str();
}

}  // namespace tpo::gpu
