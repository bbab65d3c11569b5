// B200 backend — fused-kernel candidate generator; see tpo/ir/generator.hpp.
#include "tpo/ir/generator.hpp"

#include <algorithm>
#include <map>
#include <numeric>
#include <set>

#include "labels.hpp"
#include "tpo/ir/shape_infer.hpp"

namespace tpo::ir {

namespace {

using labels::Labels;
using labels::label;
using labels::supported;
using labels::unary;

// ------------------------------------------------------------ rewrite
// Matmul(A ∘ s, W) -> Matmul(A, W) ∘ s for ∘ in {EwMul, EwDiv} when s
// broadcasts along A's last (contracted) dim and A ∘ s feeds only the
// matmul.  Row scaling commutes with the contraction exactly in Z_p and
// up to rounding in floating point (the stability filter's concern).
KernelGraph rewrite_rowscale(const KernelGraph &p, bool &changed) {
  changed = false;
  std::vector<int> uses(p.tensors.size(), 0);
  for (const Op &op : p.ops)
    for (TensorId t : op.inputs) ++uses[size_t(t)];
  for (TensorId t : p.outputs) ++uses[size_t(t)];
  std::vector<int> prod(p.tensors.size(), -1);
  for (size_t k = 0; k < p.ops.size(); ++k) prod[size_t(p.ops[k].outputs[0])] = int(k);
  // matmul op -> (scale op, A, s)
  struct Hit {
    int scale_op;
    TensorId a, s;
  };
  std::map<int, Hit> hits;
  std::set<int> skipped;
  for (size_t k = 0; k < p.ops.size(); ++k) {
    const Op &m = p.ops[k];
    if (m.type != OpType::Matmul) continue;
    const TensorId x = m.inputs[0];
    const int e = prod[size_t(x)];
    if (e < 0 || uses[size_t(x)] != 1) continue;
    const Op &so = p.ops[size_t(e)];
    if (so.type != OpType::EwMul && so.type != OpType::EwDiv) continue;
    for (int side = 0; side < (so.type == OpType::EwMul ? 2 : 1); ++side) {
      const TensorId a = so.inputs[size_t(side)], s = so.inputs[size_t(1 - side)];
      const TensorShape &as = p.tensor(a).shape, &ss = p.tensor(s).shape, &xs = p.tensor(x).shape;
      if (as != xs || ss.rank() != as.rank() || ss.dims.back() != 1 || as.dims.back() == 1) continue;
      bool ok = true;  // s broadcasts only along the last dim: [.., m or 1, 1]
      for (int d = 0; d + 1 < ss.rank(); ++d)
        if (ss.dims[size_t(d)] != 1 && ss.dims[size_t(d)] != as.dims[size_t(d)]) ok = false;
      if (!ok) continue;
      hits[int(k)] = {e, a, s};
      skipped.insert(e);
      break;
    }
  }
  if (hits.empty()) return p;
  changed = true;
  GraphBuilder gb;
  std::vector<TensorId> map(p.tensors.size(), -1);
  for (TensorId t : p.inputs) map[size_t(t)] = gb.input(p.tensor(t).shape);
  for (size_t k = 0; k < p.ops.size(); ++k) {
    const Op &op = p.ops[k];
    if (skipped.count(int(k))) continue;
    auto it = hits.find(int(k));
    if (it != hits.end()) {
      const Hit &h = it->second;
      const TensorId mm = gb.op(OpType::Matmul, {map[size_t(h.a)], map[size_t(op.inputs[1])]});
      map[size_t(op.outputs[0])] = gb.op(p.ops[size_t(h.scale_op)].type, {mm, map[size_t(h.s)]});
      continue;
    }
    std::vector<TensorId> in;
    for (TensorId t : op.inputs) in.push_back(map[size_t(t)]);
    map[size_t(op.outputs[0])] = gb.op(op.type, in, op.attrs);
  }
  std::vector<TensorId> outs;
  for (TensorId t : p.outputs) outs.push_back(map[size_t(t)]);
  return gb.finish(outs);
}

enum St { INV = 0, SLICE = 1, PARTIAL = 2, ACC = 3 };

struct Fail {};

struct Built {
  KernelGraph g;
  bool ok = false;
};

// One block graph for (grid label g over gx blocks, loop label f over fl
// iterations); `late`: carry partial sums through linear ops.
Built build(const KernelGraph &p, Labels &L, int g, int64_t gx, int f, int64_t fl, bool late) {
  auto lab = [&](TensorId t, int d) -> int {
    return p.tensor(t).shape.dims[size_t(d)] > 1 ? L.find(L.off[size_t(t)] + d) : -1;
  };
  auto dim_of = [&](TensorId t, int l) -> int {  // the (unique) dim of t carrying label l
    if (l < 0) return -1;
    int found = -1;
    for (int d = 0; d < p.tensor(t).shape.rank(); ++d)
      if (lab(t, d) == l) {
        if (found >= 0) throw Fail{};
        found = d;
      }
    return found;
  };
  const DimMap PHI({kReplica});
  std::vector<TensorShape> in_shapes;
  for (TensorId t : p.inputs) in_shapes.push_back(p.tensor(t).shape);
  BlockBuilder bb({gx, 1, 1}, fl, in_shapes);
  struct V {
    TensorId bt = -1;
    St st = INV;
  };
  std::vector<V> v(p.tensors.size());
  std::map<TensorId, TensorId> acc_of;  // partial block tensor -> its Accum
  auto accum = [&](V &x) {
    if (x.st == ACC) return;
    if (x.st != PARTIAL && !(fl == 1 && x.st != ACC)) throw Fail{};  // a loop slice or invariant over >1 iterations
    auto it = acc_of.find(x.bt);
    const TensorId a = it != acc_of.end() ? it->second : bb.op(OpType::Accum, {x.bt}, AccumAttrs{PHI});
    acc_of[x.bt] = a;
    x = {a, ACC};
  };
  for (size_t i = 0; i < p.inputs.size(); ++i) {
    const TensorId t = p.inputs[i];
    const int dg = dim_of(t, g), df = dim_of(t, f);
    const DimMap imap(std::vector<int>{dg >= 0 ? dg : kReplica});
    const DimMap fmap(std::vector<int>{df >= 0 ? df : kReplica});
    v[size_t(t)] = {bb.initer(int(i), imap, fmap), df >= 0 ? SLICE : INV};
  }
  for (const Op &op : p.ops) {
    std::vector<V> in;
    for (TensorId t : op.inputs) in.push_back(v[size_t(t)]);
    auto any = [&](St s) {
      for (const V &x : in)
        if (x.st == s) return true;
      return false;
    };
    const TensorId a0 = op.inputs[0];
    const bool contracts_f =
        f >= 0 && ((op.type == OpType::Matmul && lab(a0, p.tensor(a0).shape.rank() - 1) == f) ||
                   (op.type == OpType::Sum && lab(a0, std::get<SumAttrs>(op.attrs).dim) == f));
    St out = INV;
    if (any(PARTIAL) && !any(ACC)) {
      // linear in the partial sums (and the loop-invariant other operands)?
      bool lin = late && !contracts_f;
      if (lin) {
        if (unary(op.type)) lin = false;
        else if (op.type == OpType::EwAdd) lin = in[0].st == PARTIAL && in[1].st == PARTIAL;
        else if (op.type == OpType::EwMul) lin = (in[0].st == PARTIAL) != (in[1].st == PARTIAL) &&
                                                 (in[0].st == INV || in[1].st == INV);
        else if (op.type == OpType::EwDiv) lin = in[0].st == PARTIAL && in[1].st == INV;
        else if (op.type == OpType::Matmul) lin = (in[0].st == PARTIAL) != (in[1].st == PARTIAL) &&
                                                  (in[0].st == INV || in[1].st == INV);
        else if (op.type == OpType::Sum) lin = true;
      }
      if (lin) {
        out = PARTIAL;
      } else {
        for (V &x : in)
          if (x.st == PARTIAL) accum(x);
      }
    }
    if (out != PARTIAL) {
      if (any(ACC)) {  // post-loop: no loop slices may reach it
        for (V &x : in) {
          if (x.st == PARTIAL) accum(x);
          if (x.st == SLICE) throw Fail{};
        }
        out = ACC;
      } else if (contracts_f) {
        out = PARTIAL;
      } else {
        out = any(SLICE) ? SLICE : INV;
      }
    }
    std::vector<TensorId> bin;
    for (const V &x : in) bin.push_back(x.bt);
    OpAttrs at = op.attrs;
    if (op.type == OpType::Sum) {
      auto sa = std::get<SumAttrs>(op.attrs);
      if (g >= 0 && lab(a0, sa.dim) == g) throw Fail{};  // a reduction across grid blocks
      BlockGraph &bgr = *bb.finish();
      sa.group = bgr.tensor(bin[0]).shape.dims[size_t(sa.dim)];  // the tile's extent
      at = sa;
    }
    v[size_t(op.outputs[0])] = {bb.op(op.type, bin, at), out};
  }
  const TensorId o = p.outputs[0];
  V &vo = v[size_t(o)];
  accum(vo);
  const int og = dim_of(o, g);
  bb.outsaver(vo.bt, DimMap(std::vector<int>{og >= 0 ? og : 0}));
  GraphBuilder gb;
  std::vector<TensorId> ins;
  for (TensorId t : p.inputs) ins.push_back(gb.input(p.tensor(t).shape));
  const TensorId out = gb.graphdef(ins, bb.finish(), bb.out_shapes());
  Built b;
  b.g = gb.finish({out});
  b.ok = true;
  return b;
}

}  // namespace

std::vector<KernelGraph> generate_fused(const KernelGraph &program, const GenConfig &cfg, GenStats *stats) {
  GenStats st;
  if (program.outputs.size() != 1) throw Error(ErrCode::Unsupported, "generator: single-output programs");
  for (const Op &op : program.ops)
    if (!supported(op.type)) throw Error(ErrCode::Unsupported, std::string("generator: op ") + op_name(op.type));
  std::vector<KernelGraph> forms{program};
  if (cfg.rewrite) {
    bool changed = false;
    KernelGraph r = rewrite_rowscale(program, changed);
    if (changed) forms.push_back(std::move(r));
  }
  std::vector<KernelGraph> out;
  std::set<std::string> seen;
  for (const KernelGraph &p : forms) {
    Labels L = label(p);
    const TensorId o = p.outputs[0];
    auto size_of = [&](int l) -> int64_t {
      for (size_t t = 0; t < p.tensors.size(); ++t)
        for (int d = 0; d < p.tensors[t].shape.rank(); ++d)
          if (p.tensors[t].shape.dims[size_t(d)] > 1 && L.find(L.off[t] + d) == l)
            return p.tensors[t].shape.dims[size_t(d)];
      return 1;
    };
    std::vector<int> glabels{-1}, flabels{-1};
    for (int d = 0; d < p.tensor(o).shape.rank(); ++d) {
      if (p.tensor(o).shape.dims[size_t(d)] <= 1) continue;
      const int l = L.find(L.off[size_t(o)] + d);
      if (!L.contracted.count(l) && std::find(glabels.begin(), glabels.end(), l) == glabels.end())
        glabels.push_back(l);
    }
    for (int l : L.contracted) flabels.push_back(l);
    for (int g : glabels)
      for (int64_t gx : (g < 0 ? std::vector<int64_t>{1} : cfg.grids)) {
        if (g >= 0 && (gx <= 1 || size_of(g) % gx)) continue;
        for (int f : flabels)
          for (int64_t fl : (f < 0 ? std::vector<int64_t>{1} : cfg.loops)) {
            if (f >= 0 && (fl <= 1 || size_of(f) % fl || f == g)) continue;
            ++st.partitions;
            for (int late = 1; late >= 0; --late) {
              if (out.size() >= cfg.max_candidates) break;
              Built b;
              try {
                b = build(p, L, g, gx, f, fl, late != 0);
              } catch (const Fail &) {
                ++st.rejected_structure;
                continue;
              } catch (const Error &) {
                ++st.rejected_structure;  // shape / divisibility
                continue;
              }
              ++st.placements;
              if (!validate(b.g, cfg.limits).valid()) {
                ++st.rejected_validate;
                continue;
              }
              if (!seen.insert(canonical_key(b.g)).second) {
                ++st.duplicates;
                continue;
              }
              out.push_back(std::move(b.g));
            }
          }
      }
  }
  if (stats) *stats = st;
  return out;
}

namespace {

// The sub-program of ops [b, e): inputs are the tensors it reads that it does
// not produce (in first-use order), the output is `out`.
KernelGraph segment_program(const KernelGraph &p, size_t b, size_t e, TensorId out,
                            std::vector<TensorId> &seg_inputs) {
  GraphBuilder gb;
  std::vector<TensorId> map(p.tensors.size(), -1);
  seg_inputs.clear();
  for (size_t k = b; k < e; ++k)
    for (TensorId t : p.ops[k].inputs)
      if (map[size_t(t)] < 0) {
        bool inner = false;
        for (size_t j = b; j < k; ++j) inner = inner || p.ops[j].outputs[0] == t;
        if (!inner) {
          map[size_t(t)] = gb.input(p.tensor(t).shape);
          seg_inputs.push_back(t);
        }
      }
  for (size_t k = b; k < e; ++k) {
    std::vector<TensorId> in;
    for (TensorId t : p.ops[k].inputs) in.push_back(map[size_t(t)]);
    map[size_t(p.ops[k].outputs[0])] = gb.op(p.ops[k].type, in, p.ops[k].attrs);
  }
  return gb.finish({map[size_t(out)]});
}

}  // namespace

std::vector<KernelGraph> generate_multi(const KernelGraph &program, const GenConfig &cfg, GenStats *stats) {
  GenStats st;
  std::vector<KernelGraph> out = generate_fused(program, cfg, &st);
  std::set<std::string> seen;
  for (const KernelGraph &g : out) seen.insert(canonical_key(g));
  const KernelGraph &p = program;
  const size_t n = p.ops.size();
  if (cfg.max_kernels < 2 || n < 2 || n > 16) {
    if (stats) *stats = st;
    return out;
  }
  std::vector<int> prod(p.tensors.size(), -1);
  for (size_t k = 0; k < n; ++k) prod[size_t(p.ops[k].outputs[0])] = int(k);
  // segment [b, e) -> its single externally used output, or -1
  auto seg_out = [&](size_t b, size_t e) -> TensorId {
    TensorId o = -1;
    for (size_t k = b; k < e; ++k) {
      const TensorId t = p.ops[k].outputs[0];
      bool ext = std::find(p.outputs.begin(), p.outputs.end(), t) != p.outputs.end();
      for (size_t j = e; j < n && !ext; ++j)
        for (TensorId x : p.ops[j].inputs) ext = ext || x == t;
      if (ext) {
        if (o >= 0) return -2;
        o = t;
      }
    }
    return o;
  };
  // per segment: the options (kernel-level op, fused candidates), memoised
  std::map<std::pair<size_t, size_t>, std::vector<KernelGraph>> fused;
  auto options = [&](size_t b, size_t e, TensorId o, std::vector<TensorId> &ins) -> const std::vector<KernelGraph> & {
    auto key = std::make_pair(b, e);
    auto it = fused.find(key);
    KernelGraph sp = segment_program(p, b, e, o, ins);
    if (it != fused.end()) return it->second;
    GenConfig c = cfg;
    c.max_candidates = size_t(cfg.per_segment);
    std::vector<KernelGraph> v;
    try {
      v = generate_fused(sp, c, nullptr);
    } catch (const Error &) {
    }
    return fused.emplace(key, std::move(v)).first->second;
  };
  // every cut of the op list into 2..max_kernels contiguous segments
  for (uint32_t mask = 1; mask < (1u << (n - 1)) && out.size() < cfg.max_candidates; ++mask) {
    if (__builtin_popcount(mask) + 1 > cfg.max_kernels) continue;
    std::vector<std::pair<size_t, size_t>> segs;
    size_t b = 0;
    for (size_t k = 1; k <= n; ++k)
      if (k == n || (mask >> (k - 1)) & 1u) segs.push_back({b, k}), b = k;
    ++st.partitions;
    struct Seg {
      TensorId out;
      std::vector<TensorId> ins;
      std::vector<const KernelGraph *> fused;
      bool flat;  // one op: a pre-defined kernel op is an option
    };
    std::vector<Seg> S;
    bool ok = true;
    for (auto [sb, se] : segs) {
      Seg sg;
      sg.out = seg_out(sb, se);
      if (sg.out < 0) {
        ok = false;
        break;
      }
      for (const KernelGraph &g : options(sb, se, sg.out, sg.ins)) sg.fused.push_back(&g);
      sg.flat = se - sb == 1;
      if (sg.fused.empty() && !sg.flat) {
        ok = false;
        break;
      }
      S.push_back(std::move(sg));
    }
    if (!ok) {
      ++st.rejected_structure;
      continue;
    }
    // mixed-radix walk over the per-segment choices (flat op first)
    std::vector<size_t> radix, idx(S.size(), 0);
    for (const Seg &sg : S) radix.push_back(sg.fused.size() + (sg.flat ? 1 : 0));
    for (;;) {
      if (out.size() >= cfg.max_candidates) break;
      bool any_fused = false;
      GraphBuilder gb;
      std::vector<TensorId> map(p.tensors.size(), -1);
      for (TensorId t : p.inputs) map[size_t(t)] = gb.input(p.tensor(t).shape);
      for (size_t s = 0; s < S.size(); ++s) {
        const Seg &sg = S[s];
        std::vector<TensorId> in;
        for (TensorId t : sg.ins) in.push_back(map[size_t(t)]);
        const size_t c = idx[s];
        if (sg.flat && c == 0) {
          const Op &op = p.ops[size_t(segs[s].first)];
          map[size_t(sg.out)] = gb.op(op.type, in, op.attrs);
        } else {
          const KernelGraph &fg = *sg.fused[c - (sg.flat ? 1 : 0)];
          const Op &gd = fg.ops.at(0);
          std::vector<TensorShape> oshapes{fg.tensor(fg.outputs[0]).shape};
          map[size_t(sg.out)] = gb.graphdef(in, gd.block, oshapes);
          any_fused = true;
        }
      }
      if (any_fused) {
        KernelGraph g = gb.finish({map[size_t(p.outputs[0])]});
        ++st.placements;
        if (!validate(g, cfg.limits).valid()) {
          ++st.rejected_validate;
        } else if (!seen.insert(canonical_key(g)).second) {
          ++st.duplicates;
        } else {
          out.push_back(std::move(g));
        }
      }
      size_t s = 0;
      while (s < idx.size() && ++idx[s] == radix[s]) idx[s++] = 0;
      if (s == idx.size()) break;
    }
  }
  if (stats) *stats = st;
  return out;
}

}  // namespace tpo::ir
