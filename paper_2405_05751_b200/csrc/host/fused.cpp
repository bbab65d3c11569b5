// B200 backend — benchmark µGraph recognition and fused-kernel launch.
//
// A KernelGraph is lowered to a hand-written fused kernel when it is,
// structurally, one of the benchmark µGraphs of SURVEY §8d (any shapes, any
// grid / for-loop schedule): the graph is rebuilt from its own input shapes
// with the fixture builders below and compared by canonical_key (the
// reference's structural identity, graph.cpp:128-157).  The kernel computes
// the same block-graph function; the µGraph's (grid, forloop) schedule is
// re-tiled for B200 (see fused_skinny.cu / fused_gqa.cu headers).
#include "fused.hpp"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <array>
#include <functional>
#include <map>
#include <mutex>

#include "../../../include/tpo_gpu.h"
#include "../kernels/fused.cuh"
#include "tpo/ir/graph.hpp"

namespace tpo::gpu {

using namespace ir;

namespace {

const DimMap PHI1({kReplica});
DimMap dm(std::vector<int> v) { return DimMap(std::move(v)); }

// ---- fixture builders (C++ mirror of paper_2405_05751_b200/fixtures.py) ----

KernelGraph rmsnorm_mugraph(int64_t b, int64_t h, int64_t n, int64_t grid, int64_t fl) {
  GraphBuilder gb;
  TensorId X = gb.input({b, h}), G = gb.input({1, h}), W = gb.input({h, n}), D = gb.input({1, 1});
  BlockBuilder bb({grid, 1, 1}, fl, {{b, h}, {1, h}, {h, n}, {1, 1}});
  TensorId xb = bb.initer(0, PHI1, dm({1}));
  TensorId gbar = bb.initer(1, PHI1, dm({1}));
  TensorId wb = bb.initer(2, dm({1}), dm({0}));
  TensorId db = bb.initer(3, PHI1, PHI1);
  TensorId xg = bb.op(OpType::EwMul, {xb, gbar});
  TensorId B = bb.op(OpType::Accum, {bb.op(OpType::Matmul, {xg, wb})}, AccumAttrs{PHI1});
  TensorId ss = bb.op(OpType::Sum, {bb.op(OpType::Sqr, {xb})}, SumAttrs{1, h / fl});
  TensorId A = bb.op(OpType::Accum, {bb.op(OpType::EwMul, {ss, db})}, AccumAttrs{PHI1});
  bb.outsaver(bb.op(OpType::EwDiv, {B, bb.op(OpType::Sqrt, {A})}), dm({1}));
  TensorId o = gb.graphdef({X, G, W, D}, bb.finish(), bb.out_shapes());
  return gb.finish({o});
}

KernelGraph gatedmlp_mugraph(int64_t b, int64_t h, int64_t n, int64_t grid, int64_t fl) {
  GraphBuilder gb;
  TensorId X = gb.input({b, h}), W1 = gb.input({h, n}), W3 = gb.input({h, n});
  BlockBuilder bb({grid, 1, 1}, fl, {{b, h}, {h, n}, {h, n}});
  TensorId xb = bb.initer(0, PHI1, dm({1}));
  TensorId w1 = bb.initer(1, dm({1}), dm({0}));
  TensorId w3 = bb.initer(2, dm({1}), dm({0}));
  TensorId A1 = bb.op(OpType::Accum, {bb.op(OpType::Matmul, {xb, w1})}, AccumAttrs{PHI1});
  TensorId A3 = bb.op(OpType::Accum, {bb.op(OpType::Matmul, {xb, w3})}, AccumAttrs{PHI1});
  bb.outsaver(bb.op(OpType::EwMul, {bb.op(OpType::SiLU, {A1}), A3}), dm({1}));
  TensorId o = gb.graphdef({X, W1, W3}, bb.finish(), bb.out_shapes());
  return gb.finish({o});
}

KernelGraph gqa_mugraph(int64_t g, int64_t qh, int64_t hd, int64_t L, int64_t grid, int64_t fl) {
  GraphBuilder gb;
  TensorId Q = gb.input({g, qh, hd}), K = gb.input({g, hd, L}), V = gb.input({g, L, hd});
  BlockBuilder bb({grid, 1, 1}, fl, {{g, qh, hd}, {g, hd, L}, {g, L, hd}});
  TensorId qb = bb.initer(0, dm({0}), PHI1);
  TensorId kb = bb.initer(1, dm({0}), dm({2}));
  TensorId vb = bb.initer(2, dm({0}), dm({1}));
  TensorId e = bb.op(OpType::EwExp, {bb.op(OpType::Matmul, {qb, kb})});
  TensorId N = bb.op(OpType::Accum, {bb.op(OpType::Matmul, {e, vb})}, AccumAttrs{PHI1});
  TensorId D = bb.op(OpType::Accum, {bb.op(OpType::Sum, {e}, SumAttrs{2, L / fl})}, AccumAttrs{PHI1});
  bb.outsaver(bb.op(OpType::EwDiv, {N, D}), dm({0}));
  TensorId o = gb.graphdef({Q, K, V}, bb.finish(), bb.out_shapes());
  return gb.finish({o});
}

KernelGraph lora_mugraph(int64_t b, int64_t h, int64_t n, int64_t r, int64_t grid, int64_t fl) {
  GraphBuilder gb;
  TensorId X = gb.input({b, h}), W = gb.input({h, n}), A = gb.input({h, r}), B = gb.input({r, n});
  BlockBuilder bb({grid, 1, 1}, fl, {{b, h}, {h, n}, {h, r}, {r, n}});
  TensorId xb = bb.initer(0, PHI1, dm({1}));
  TensorId wb = bb.initer(1, dm({1}), dm({0}));
  TensorId ab = bb.initer(2, PHI1, dm({0}));
  TensorId bbar = bb.initer(3, dm({1}), dm({0}));
  TensorId XW = bb.op(OpType::Accum, {bb.op(OpType::Matmul, {xb, wb})}, AccumAttrs{PHI1});
  TensorId XA = bb.op(OpType::Accum, {bb.op(OpType::Matmul, {xb, ab})}, AccumAttrs{PHI1});
  TensorId Bc = bb.op(OpType::Accum, {bbar}, AccumAttrs{dm({0})});
  bb.outsaver(bb.op(OpType::EwAdd, {XW, bb.op(OpType::Matmul, {XA, Bc})}), dm({1}));
  TensorId o = gb.graphdef({X, W, A, B}, bb.finish(), bb.out_shapes());
  return gb.finish({o});
}

// LoRA as the fusion generator emits it: one φ-accumulator of the sum,
// XA·B̄ applied per iteration (linear in the loop's partial sums); same
// kernel, XA·B̄ = Σ_i XA_i·B̄.
KernelGraph lora_single_mugraph(int64_t b, int64_t h, int64_t n, int64_t r, int64_t grid, int64_t fl) {
  GraphBuilder gb;
  TensorId X = gb.input({b, h}), W = gb.input({h, n}), A = gb.input({h, r}), B = gb.input({r, n});
  BlockBuilder bb({grid, 1, 1}, fl, {{b, h}, {h, n}, {h, r}, {r, n}});
  TensorId xb = bb.initer(0, PHI1, dm({1}));
  TensorId wb = bb.initer(1, dm({1}), dm({0}));
  TensorId ab = bb.initer(2, PHI1, dm({0}));
  TensorId bbar = bb.initer(3, dm({1}), PHI1);
  TensorId xw = bb.op(OpType::Matmul, {xb, wb});
  TensorId xab = bb.op(OpType::Matmul, {bb.op(OpType::Matmul, {xb, ab}), bbar});
  TensorId acc = bb.op(OpType::Accum, {bb.op(OpType::EwAdd, {xw, xab})}, AccumAttrs{PHI1});
  bb.outsaver(acc, dm({1}));
  TensorId o = gb.graphdef({X, W, A, B}, bb.finish(), bb.out_shapes());
  return gb.finish({o});
}

// `key`: canonical_key(g), computed once by the caller
// Order-insensitive structure of a single-GraphDef µGraph: grid, for-loop,
// operand shapes and, per OutSaver, the expression tree of its value (op
// names with attributes; InIter leaves carry operand / imap / fmap).  Two
// µGraphs that differ only in the list order of independent block ops (a
// generator's output vs a hand-built fixture) get the same key.
std::string structural_key(const KernelGraph &g) {
  if (g.ops.size() != 1 || !g.ops[0].block) return canonical_key(g);
  const BlockGraph &bg = *g.ops[0].block;
  std::vector<int> prod(bg.tensors.size(), -1);
  for (size_t k = 0; k < bg.ops.size(); ++k)
    for (TensorId t : bg.ops[k].outputs) prod[size_t(t)] = int(k);
  std::vector<std::string> memo(bg.tensors.size());
  std::function<const std::string &(TensorId)> expr = [&](TensorId t) -> const std::string & {
    std::string &m = memo[size_t(t)];
    if (!m.empty()) return m;
    const Op &op = bg.ops[size_t(prod[size_t(t)])];
    std::string e = std::string(op_name(op.type)) + attr_key(op.attrs) + "(";
    std::vector<std::string> args;
    for (TensorId x : op.inputs) args.push_back(expr(x));
    // commutative operators: operand order is not structure
    if (op.type == OpType::EwAdd || op.type == OpType::EwMul) std::sort(args.begin(), args.end());
    for (const std::string &a : args) e += a + ",";
    m = e + ")";
    return m;
  };
  std::string key = "S(";
  for (TensorId t : g.inputs) key += to_string(g.tensor(t).shape) + ";";
  key += std::to_string(bg.grid[0]) + "," + std::to_string(bg.grid[1]) + "," + std::to_string(bg.grid[2]) + ";" +
         std::to_string(bg.forloop) + ";";
  std::vector<std::string> outs;
  for (const Op &op : bg.ops)
    if (op.type == OpType::OutSaver) outs.push_back(std::string(attr_key(op.attrs)) + expr(op.inputs[0]));
  for (const auto &o : outs) key += o + "|";  // OutSaver #k -> output k: list order kept
  return key + ")";
}

// structural keys of the reference forms, memoised by (form, sizes): a
// search stream matches thousands of candidates against the same few
template <class F>
bool same(const std::string &key, const std::array<int64_t, 7> &form, F &&build) {
  static std::mutex mu;
  static std::map<std::array<int64_t, 7>, std::string> memo;
  std::string want;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = memo.find(form);
    if (it != memo.end()) want = it->second;
  }
  if (want.empty()) {
    try {
      want = structural_key(build());
    } catch (const Error &) {
      want = "-";  // not constructible: never matches
    }
    std::lock_guard<std::mutex> lk(mu);
    if (memo.size() > 4096) memo.clear();
    memo.emplace(form, want);
  }
  return key == want;
}

int env_int(const char *name, int dflt) {
  const char *v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// K split (= cluster size) for the skinny kernels: the largest split whose
// grid still fits in ONE wave (every CTA streams weights from the first
// cycle; a second wave would idle SMs), K per CTA a multiple of 64.  Cluster
// packing on 148 SMs: size 1/2 -> 148 slots per CTA-per-SM, size 4 -> 132,
// size 8 -> 120 (GPC granularity).
int pick_ksplit(int64_t ntiles, int64_t K, int ctas_per_sm) {
  int forced = env_int("TPO_KSPLIT", 0);
  if (forced > 0) return forced;
  int best = 1;
  for (int s = 1; s <= 4; s *= 2) {
    if (K % (64 * s)) break;
    int64_t slots = (s <= 2 ? 148 : s == 4 ? 132 : 120) * int64_t(ctas_per_sm);
    if (ntiles * s <= slots) best = s;
  }
  return best;
}

}  // namespace

namespace {

// The paper's LoRA µGraph (Algorithm 1 rediscovers it,
// tests/test_enumerate.py): kernel op T = Matmul(X, A), then ONE GraphDef
// over (X, W, B, T) whose for-loop runs ConcatMatmul(X̄, T̄, W̄, B̄) =
// X̄·W̄ + T̄·B̄ into one φ-Accum — i.e. X·W + (X·A)·B, the function the
// fused LoRA kernel computes (graph inputs X, W, A, B as in the
// single-kernel form).  Matched structurally, independent of list order
// and tensor ids; every InIter map is checked so that the partition covers
// exactly that function: the loop slices both contractions (X̄ / T̄ along
// dim 1, W̄ / B̄ along dim 0, or no loop split), the grid splits either the
// output columns (W̄, B̄, OutSaver along dim 1) or the tokens (X̄, T̄,
// OutSaver along dim 0).
bool match_lora_concat(const KernelGraph &g, FusedPlan &p) {
  if (g.ops.size() != 2 || g.inputs.size() != 4 || g.outputs.size() != 1) return false;
  const Op &mm = g.ops[0], &gd = g.ops[1];
  if (mm.type != OpType::Matmul || gd.type != OpType::GraphDef || !gd.block) return false;
  const TensorId X = g.inputs[0], W = g.inputs[1], A = g.inputs[2], B = g.inputs[3];
  if (mm.inputs != std::vector<TensorId>{X, A} || mm.outputs.size() != 1) return false;
  const TensorId T = mm.outputs[0];
  if (gd.outputs.size() != 1 || gd.outputs[0] != g.outputs[0]) return false;
  for (TensorId t : {X, W, A, B})
    if (g.tensor(t).shape.rank() != 2) return false;
  const int64_t b = g.tensor(X).shape.dims[0], h = g.tensor(X).shape.dims[1];
  const int64_t n = g.tensor(W).shape.dims[1], r = g.tensor(A).shape.dims[1];
  if (g.tensor(W).shape.dims[0] != h || g.tensor(A).shape.dims[0] != h || g.tensor(B).shape.dims != std::vector<int64_t>{r, n})
    return false;
  const BlockGraph &bg = *gd.block;
  if (bg.grid[1] != 1 || bg.grid[2] != 1) return false;
  const int64_t grid = bg.grid[0], fl = bg.forloop;
  // block tensor -> role (0 X̄, 1 W̄, 2 B̄, 3 T̄) through its InIter
  std::vector<int> role(bg.tensors.size(), -1);
  int seen[4] = {0, 0, 0, 0}, n_in = 0, n_cm = 0, n_acc = 0, n_out = 0;
  const Op *cm = nullptr, *acc = nullptr, *sav = nullptr;
  const InIterAttrs *it[4] = {nullptr, nullptr, nullptr, nullptr};
  for (const Op &o : bg.ops) {
    switch (o.type) {
      case OpType::InIter: {
        const auto &a = std::get<InIterAttrs>(o.attrs);
        if (a.operand < 0 || size_t(a.operand) >= gd.inputs.size()) return false;
        const TensorId src = gd.inputs[size_t(a.operand)];
        const int rl = src == X ? 0 : src == W ? 1 : src == B ? 2 : src == T ? 3 : -1;
        if (rl < 0 || seen[rl]++) return false;
        role[size_t(o.outputs.at(0))] = rl;
        it[rl] = &a;
        ++n_in;
        break;
      }
      case OpType::ConcatMatmul: cm = &o, ++n_cm; break;
      case OpType::Accum: acc = &o, ++n_acc; break;
      case OpType::OutSaver: sav = &o, ++n_out; break;
      default: return false;
    }
  }
  if (n_in != 4 || n_cm != 1 || n_acc != 1 || n_out != 1 || cm->inputs.size() != 4) return false;
  // ConcatMatmul(a0, a1, b0, b1) = a0·b0 + a1·b1: pairs (X̄, W̄) and (T̄, B̄)
  std::array<int, 4> cr;
  for (int k = 0; k < 4; ++k) cr[size_t(k)] = role[size_t(cm->inputs[size_t(k)])];
  const bool pairs = (cr == std::array<int, 4>{0, 3, 1, 2}) || (cr == std::array<int, 4>{3, 0, 2, 1});
  if (!pairs) return false;
  const auto &aa = std::get<AccumAttrs>(acc->attrs);
  if (acc->inputs.at(0) != cm->outputs.at(0) || aa.fmap.axes() != 1 || aa.fmap.targets[0] != kReplica) return false;
  if (sav->inputs.at(0) != acc->outputs.at(0)) return false;
  const auto &om = std::get<OutSaverAttrs>(sav->attrs).omap;
  auto t0 = [](const DimMap &m) { return m.axes() ? m.targets[0] : kReplica; };
  // the loop: both contractions sliced consistently, or not split at all
  const bool loop_ok = fl == 1 || (t0(it[0]->fmap) == 1 && t0(it[3]->fmap) == 1 && t0(it[1]->fmap) == 0 &&
                                   t0(it[2]->fmap) == 0 && h % fl == 0 && r % fl == 0);
  // the grid: output columns (W̄, B̄, OutSaver along dim 1) or tokens
  const bool cols = t0(it[0]->imap) == kReplica && t0(it[3]->imap) == kReplica && t0(it[1]->imap) == 1 &&
                    t0(it[2]->imap) == 1 && t0(om) == 1;
  const bool toks = t0(it[0]->imap) == 0 && t0(it[3]->imap) == 0 && t0(it[1]->imap) == kReplica &&
                    t0(it[2]->imap) == kReplica && t0(om) == 0;
  if (!loop_ok || !(cols || toks || grid == 1)) return false;
  p.kind = TPO_FUSED_LORA;
  p.b = b, p.h = h, p.n = n, p.r = r, p.grid = grid, p.forloop = fl;
  return true;
}

}  // namespace

FusedPlan match_fused(const KernelGraph &g) {
  FusedPlan p;
  if (g.ops.size() == 2) {
    try {
      if (match_lora_concat(g, p)) {
        if (p.r != 16 || p.n % 128 || p.h % 64) {
          p.kind = TPO_FUSED_NONE;
          p.why = "LoRA µGraph outside kernel limits (r==16, n%128, h%64)";
        }
        return p;
      }
    } catch (const std::exception &) {
    }
  }
  if (g.ops.size() != 1 || g.ops[0].type != OpType::GraphDef || !g.ops[0].block ||
      g.outputs.size() != 1) {
    p.why = "not a single-GraphDef µGraph";
    return p;
  }
  const BlockGraph &bg = *g.ops[0].block;
  const int64_t grid = bg.grid[0], fl = bg.forloop;
  std::string key;
  try {
    key = structural_key(g);
  } catch (const Error &) {
    p.why = "no canonical form";
    return p;
  }
  std::vector<TensorShape> in;
  for (TensorId t : g.inputs) in.push_back(g.tensor(t).shape);
  auto r2 = [&](size_t i) { return in[i].rank() == 2; };
  if (in.size() == 4 && r2(0) && r2(1) && r2(2) && r2(3) && in[1].dims[0] == 1 &&
      in[3].dims == std::vector<int64_t>{1, 1}) {
    int64_t b = in[0].dims[0], h = in[0].dims[1], n = in[2].dims[1];
    if (same(key, {1, b, h, n, 0, grid, fl}, [&] { return rmsnorm_mugraph(b, h, n, grid, fl); })) {
      if (n % 128 || h % 64) {
        p.why = "RMSNorm µGraph outside kernel limits (n%128, h%64)";
        return p;
      }
      p.kind = TPO_FUSED_RMSNORM_MATMUL;
      p.b = b, p.h = h, p.n = n, p.grid = grid, p.forloop = fl;
      return p;
    }
  }
  if (in.size() == 3 && r2(0) && r2(1) && r2(2)) {
    int64_t b = in[0].dims[0], h = in[0].dims[1], n = in[1].dims[1];
    if (same(key, {2, b, h, n, 0, grid, fl}, [&] { return gatedmlp_mugraph(b, h, n, grid, fl); })) {
      if (n % 128 || h % 64) {
        p.why = "GatedMLP µGraph outside kernel limits (n%128, h%64)";
        return p;
      }
      p.kind = TPO_FUSED_GATED_MLP;
      p.b = b, p.h = h, p.n = n, p.grid = grid, p.forloop = fl;
      return p;
    }
  }
  if (in.size() == 3 && in[0].rank() == 3 && in[1].rank() == 3 && in[2].rank() == 3) {
    int64_t G = in[0].dims[0], qh = in[0].dims[1], hd = in[0].dims[2], L = in[1].dims[2];
    if (same(key, {3, G, qh, hd, L, grid, fl}, [&] { return gqa_mugraph(G, qh, hd, L, grid, fl); })) {
      if (qh > 8 || hd != 128 || L % 128) {
        p.why = "GQA µGraph outside kernel limits (qh<=8, hd==128, L%128)";
        return p;
      }
      p.kind = TPO_FUSED_GQA_DECODE;
      p.groups = G, p.qh = qh, p.hd = hd, p.L = L, p.grid = grid, p.forloop = fl;
      return p;
    }
  }
  if (in.size() == 4 && r2(0) && r2(1) && r2(2) && r2(3)) {
    int64_t b = in[0].dims[0], h = in[0].dims[1], n = in[1].dims[1], r = in[2].dims[1];
    if (same(key, {4, b, h, n, r, grid, fl}, [&] { return lora_mugraph(b, h, n, r, grid, fl); }) ||
        same(key, {5, b, h, n, r, grid, fl}, [&] { return lora_single_mugraph(b, h, n, r, grid, fl); })) {
      if (r != 16 || n % 128 || h % 64) {
        p.why = "LoRA µGraph outside kernel limits (r==16, n%128, h%64)";
        return p;
      }
      p.kind = TPO_FUSED_LORA;
      p.b = b, p.h = h, p.n = n, p.r = r, p.grid = grid, p.forloop = fl;
      return p;
    }
  }
  p.why = "µGraph does not match a benchmark kernel structurally";
  return p;
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// 2-D bf16 tensor map: rows x cols row-major, box (box_cols x box_rows).
// Encoded maps are cached by (pointer, shape, box, swizzle): repeated
// evaluations on the same buffers skip the driver call.
bool tmap_2d(CUtensorMap *m, const void *ptr, uint64_t rows, uint64_t cols, uint32_t box_cols,
             uint32_t box_rows, CUtensorMapSwizzle sw, bool f32 = false) {
  struct Key {
    const void *p;
    uint64_t r, c;
    uint32_t bc, br;
    int sw;
    bool f32;
    bool operator==(const Key &o) const {
      return p == o.p && r == o.r && c == o.c && bc == o.bc && br == o.br && sw == o.sw && f32 == o.f32;
    }
  };
  static std::mutex mu;
  static std::vector<std::pair<Key, CUtensorMap>> cache;
  const Key key{ptr, rows, cols, box_cols, box_rows, int(sw), f32};
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto &e : cache)
      if (e.first == key) {
        *m = e.second;
        return true;
      }
  }
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() >= 256) cache.erase(cache.begin());
  cache.emplace_back(key, *m);
  return true;
}

// 3-D bf16 tensor map, dims innermost first (cached like tmap_2d).
bool tmap_3d(CUtensorMap *m, const void *ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0,
             uint32_t b1, uint32_t b2, CUtensorMapSwizzle sw) {
  struct Key {
    const void *p;
    uint64_t d0, d1, d2;
    uint32_t b0, b1, b2;
    int sw;
    bool operator==(const Key &o) const {
      return p == o.p && d0 == o.d0 && d1 == o.d1 && d2 == o.d2 && b0 == o.b0 && b1 == o.b1 &&
             b2 == o.b2 && sw == o.sw;
    }
  };
  static std::mutex mu;
  static std::vector<std::pair<Key, CUtensorMap>> cache;
  const Key key{ptr, d0, d1, d2, b0, b1, b2, int(sw)};
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto &e : cache)
      if (e.first == key) {
        *m = e.second;
        return true;
      }
  }
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * 2, d0 * d1 * 2};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(ptr), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() >= 256) cache.erase(cache.begin());
  cache.emplace_back(key, *m);
  return true;
}

// TPO_DEBUG_TIMES: per-CTA %globaltimer phase stamps (16 slots per CTA)
// written by the kernels, summarised on stderr (µs since the first CTA
// started).  Debug only: the launch is followed by a synchronising copy.
// TPO_DEBUG_RING=1 instead gives every launch its own slot of a ring of
// kRing launches (no copy, no sync: usable inside CUDA graphs and
// back-to-back streams); read it with tpo_debug_ring_read.
constexpr int kRing = 16, kRingCtas = 4096;
unsigned long long *g_ring = nullptr;
unsigned g_ring_seq = 0;

unsigned long long *debug_begin(int nct, cudaStream_t st) {
  static unsigned long long *dbg = nullptr;
  if (std::getenv("TPO_DEBUG_RING")) {
    if (!g_ring) {
      cudaMalloc(&g_ring, size_t(kRing) * kRingCtas * 16 * 8);
      cudaMemset(g_ring, 0, size_t(kRing) * kRingCtas * 16 * 8);
    }
    return g_ring + size_t(g_ring_seq++ % kRing) * kRingCtas * 16;
  }
  if (!std::getenv("TPO_DEBUG_TIMES")) return nullptr;
  if (!dbg) cudaMalloc(&dbg, 16 * 8 * 4096);
  cudaMemsetAsync(dbg, 0, size_t(nct) * 128, st);
  return dbg;
}

void debug_end(const char *tag, unsigned long long *dbg, int nct, cudaStream_t st) {
  if (std::getenv("TPO_DEBUG_RING")) return;
  std::vector<unsigned long long> h(size_t(nct) * 16);
  cudaMemcpyAsync(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  unsigned long long t0 = ~0ull;
  for (int c = 0; c < nct; ++c)
    if (h[size_t(c) * 16]) t0 = std::min(t0, h[size_t(c) * 16]);
  static const char *names[14] = {"start", "setup", "epi_done", "last_mma", "sent", "tmem_full",
                                  "recv_done", "end", "first_full", "b_ready", "last_tma",
                                  "owner_done", "after_sync", "w0_at_sync"};
  std::fprintf(stderr, "[tpo debug] %s ctas %d (us since first start)\n", tag, nct);
  for (int k = 0; k < 14; ++k) {
    double mn = 1e30, mx = 0, sum = 0;
    int cnt = 0;
    for (int c = 0; c < nct; ++c) {
      unsigned long long v = h[size_t(c) * 16 + k];
      if (!v) continue;
      double d = double(v - t0) / 1e3;
      mn = std::min(mn, d), mx = std::max(mx, d), sum += d, ++cnt;
    }
    if (cnt)
      std::fprintf(stderr, "  %-12s n=%4d min %7.2f mean %7.2f max %7.2f\n", names[k], cnt, mn, sum / cnt, mx);
  }
  // skew within clusters of `cl` consecutive CTAs vs across clusters (slot 5)
  const char *cs = std::getenv("TPO_DEBUG_CLUSTER");
  const int cl = cs ? std::atoi(cs) : 0;
  if (cl > 1) {
    double within = 0, across_mx = 0, across_mn = 1e30;
    int nc = 0;
    for (int c0 = 0; c0 + cl <= nct; c0 += cl) {
      double mx = 0, mn = 1e30;
      for (int c = c0; c < c0 + cl; ++c) {
        const double d = double(h[size_t(c) * 16 + 5] - t0) / 1e3;
        mx = std::max(mx, d), mn = std::min(mn, d);
      }
      within += mx - mn, ++nc;
      across_mx = std::max(across_mx, mx), across_mn = std::min(across_mn, mx);
    }
    std::fprintf(stderr, "  slot5 skew: mean within-cluster %.2f us, cluster-max range %.2f .. %.2f us\n",
                 within / nc, across_mn, across_mx);
  }
}

}  // namespace

namespace {
extern "C" int tpo_convert_planes(const void *in, int dtype, void *hi, void *lo, size_t n, int num_sms,
                                  cudaStream_t st);
extern "C" int tpo_convert_rows(const void *in, int dtype, void *out, size_t batch, size_t R, size_t C,
                                size_t P, int num_sms, cudaStream_t st);
extern "C" int tpo_convert_to_f32(const void *in, int dtype, float *out, size_t n, int num_sms,
                                  cudaStream_t st);
extern "C" int tpo_convert_to_bf16(const void *in, int dtype, void *out, size_t n, int num_sms,
                                   cudaStream_t st);

// Operand conversions of one evaluation into scratch slots (slot 2i, 2i+1
// for input i).  Each returns false on a CUDA error.
struct Convert {
  const FusedIO &io;
  cudaStream_t st;
  int err = 0;
  // hi / lo bf16 planes of input i (n elements)
  std::pair<void *, void *> planes(int i, size_t n) {
    void *hi = io.scratch(2 * i, n * 2), *lo = io.scratch(2 * i + 1, n * 2);
    if (!err) err = tpo_convert_planes(io.in[i], io.dt[i], hi, lo, n, io.num_sms, st);
    return {hi, lo};
  }
  // [batch][2P][C] hi / lo token rows of input i ([batch][R][C])
  void *rows(int i, size_t batch, size_t R, size_t C, size_t P) {
    void *o = io.scratch(2 * i, batch * 2 * P * C * 2);
    if (!err) err = tpo_convert_rows(io.in[i], io.dt[i], o, batch, R, C, P, io.num_sms, st);
    return o;
  }
  const float *f32(int i, size_t n) {
    if (io.dt[i] == TPO_DTYPE_F32) return static_cast<const float *>(io.in[i]);
    float *o = static_cast<float *>(io.scratch(2 * i, n * 4));
    if (!err) err = tpo_convert_to_f32(io.in[i], io.dt[i], o, n, io.num_sms, st);
    return o;
  }
  const void *bf16(int i, size_t n) {
    if (io.dt[i] == TPO_DTYPE_BF16) return io.in[i];
    void *o = io.scratch(2 * i, n * 2);
    if (!err) err = tpo_convert_to_bf16(io.in[i], io.dt[i], o, n, io.num_sms, st);
    return o;
  }
};

// Input element counts of a fused plan, in graph-input order.
std::vector<size_t> input_elems(const FusedPlan &p) {
  switch (p.kind) {
    case TPO_FUSED_GATED_MLP: return {size_t(p.b * p.h), size_t(p.h * p.n), size_t(p.h * p.n)};
    case TPO_FUSED_RMSNORM_MATMUL: return {size_t(p.b * p.h), size_t(p.h), size_t(p.h * p.n), 1};
    case TPO_FUSED_LORA: return {size_t(p.b * p.h), size_t(p.h * p.n), size_t(p.h * p.r), size_t(p.r * p.n)};
    case TPO_FUSED_GQA_DECODE:
      return {size_t(p.groups * p.qh * p.hd), size_t(p.groups * p.hd * p.L), size_t(p.groups * p.L * p.hd)};
  }
  return {};
}

}  // namespace

int launch_fused(const FusedPlan &p, const FusedIO &io, cudaStream_t st) {
  // More tokens than one kernel tile holds (8 for RMSNorm / GatedMLP, 16
  // for LoRA): one launch per token chunk, X and the output offset by whole
  // rows — every per-token quantity (Σx², SiLU gate, XA) is row-local, so
  // the chunks are independent; each re-streams the weights.
  const int64_t chunk = p.kind == TPO_FUSED_LORA ? 16 : 8;
  if ((p.kind == TPO_FUSED_RMSNORM_MATMUL || p.kind == TPO_FUSED_GATED_MLP || p.kind == TPO_FUSED_LORA) &&
      p.b > chunk) {
    const size_t xel = io.dt[0] == TPO_DTYPE_BF16 ? 2 : io.dt[0] == TPO_DTYPE_F32 ? 4 : 8;
    const size_t nin = input_elems(p).size();
    for (int64_t c = 0; c < p.b; c += chunk) {
      FusedPlan pc = p;
      pc.b = std::min(chunk, p.b - c);
      std::vector<const void *> in(io.in, io.in + nin);
      in[0] = static_cast<const char *>(io.in[0]) + size_t(c) * size_t(p.h) * xel;
      float *out = io.out[0] + size_t(c) * size_t(p.n);
      FusedIO ic = io;
      ic.in = in.data();
      ic.out = &out;
      if (int e = launch_fused(pc, ic, st)) return e;
    }
    return 0;
  }
  const std::vector<size_t> ne = input_elems(p);
  const int n_in = int(ne.size());
  bool all_bf16 = true;
  for (int i = 0; i < n_in; ++i) {
    if (io.dt[i] != TPO_DTYPE_BF16 && io.dt[i] != TPO_DTYPE_F32 && io.dt[i] != TPO_DTYPE_F64)
      return int(cudaErrorInvalidValue);
    all_bf16 &= io.dt[i] == TPO_DTYPE_BF16;
  }
  const bool split = !all_bf16 && io.precision == TPO_PREC_AUTO;
  Convert cv{io, st};
  // operands as the kernels read them: the caller's bf16 buffers, rounded
  // copies (TPO_PREC_BF16), or the split forms
  std::vector<const void *> in(n_in);
  for (int i = 0; i < n_in; ++i) in[i] = split ? nullptr : cv.bf16(i, ne[i]);
  // the library wrote an operand on this stream just now: no weight may be
  // read before the PDL wait
  const bool converted = !all_bf16;
  CUtensorMap maps[8];
  std::memset(maps, 0, sizeof(maps));
  if (p.kind == TPO_FUSED_GQA_DECODE) {
    // K^T [G, hd, L], V [G, L, hd], Q [G, qh, hd]
    GqaParams gp{};
    gp.groups = int(p.groups), gp.qh = int(p.qh), gp.hd = int(p.hd), gp.L = int(p.L);
    int S = env_int("TPO_KSPLIT", 0);
    if (S <= 0) {
      S = 1;
      while (S < 4 && p.groups * S * 2 <= 148 && p.L % (128 * S * 2) == 0) S *= 2;
    }
    gp.ksplit = S;
    gp.l_per_cta = int(p.L / S);
    gp.out = io.out[0];
    // ring of 32-KB slots (K or V blocks) filled in the MMA issue order;
    // TPO_STAGES counts K+V pairs (sweep, profiles/r01/ring/sweep_gqa_slots*:
    // 5 slots in issue order 22.95 us; 6 slots K,V-paired 23.25; 3 slots at
    // two CTAs per SM 24.1).  SPLIT: three 64-KB slots (hi + lo planes).
    int slots = env_int("TPO_GQA_SLOTS", env_int("TPO_STAGES", 0) > 0 ? 2 * env_int("TPO_STAGES", 0) : 5);
    int minb = env_int("TPO_MINB", 1);
    if (split) slots = 3, minb = 1;
    gp.consume_order = env_int("TPO_GQA_ORDER", 1);
    // first ring units + Q into L2 before the PDL wait (22.80 -> 22.26 us
    // per evaluation at 3 units; 1: 22.47, 2: 22.31, 4: 22.34, all: 28.3)
    gp.l2_units = env_int("TPO_GQA_L2", 3);
    const int nct_g = int(p.groups) * S;
    gp.dbg = debug_begin(nct_g, st);
    bool ok;
    if (split) {
      const void *qs = cv.rows(0, size_t(p.groups), size_t(p.qh), size_t(p.hd), 8);
      auto kp = cv.planes(1, ne[1]);
      auto vp = cv.planes(2, ne[2]);
      if (cv.err) return cv.err;
      ok = tmap_3d(&maps[0], kp.first, p.L, p.hd, p.groups, 64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B) &&
           tmap_3d(&maps[3], kp.second, p.L, p.hd, p.groups, 64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B) &&
           tmap_3d(&maps[1], vp.first, p.hd, p.L, p.groups, 64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B) &&
           tmap_3d(&maps[4], vp.second, p.hd, p.L, p.groups, 64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B) &&
           tmap_3d(&maps[2], qs, p.hd, 16, p.groups, 64, 16, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    } else {
      if (cv.err) return cv.err;
      ok = tmap_3d(&maps[0], in[1], p.L, p.hd, p.groups, 64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B) &&
           tmap_3d(&maps[1], in[2], p.hd, p.L, p.groups, 64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B) &&
           tmap_3d(&maps[2], in[0], p.hd, p.qh, p.groups, 64, 16, 1, CU_TENSOR_MAP_SWIZZLE_128B);
      maps[3] = maps[0], maps[4] = maps[1];
    }
    if (!ok) return int(cudaErrorInvalidValue);
    int rc_g = tpo_gqa_launch(slots, minb, split, maps, &gp, st);
    if (gp.dbg && !rc_g) {
      char tag[96];
      std::snprintf(tag, sizeof(tag), "gqa ksplit %d slots %d minb %d split %d", S, slots, minb, int(split));
      debug_end(tag, gp.dbg, nct_g, st);
    }
    return rc_g;
  }
  SkinnyParams sp{};
  int mode = 0;
  bool ok = true;
  const auto SW = CU_TENSOR_MAP_SWIZZLE_128B, NOSW = CU_TENSOR_MAP_SWIZZLE_NONE;
  if (p.kind == TPO_FUSED_GATED_MLP) {
    mode = MODE_GATED;
    sp.ksplit = std::min(2, pick_ksplit(p.n / 128, p.h, 1));
    if (split) {  // W1 hi, W1 lo | X rows (hi 0-7, lo 8-15) | W3 hi, W3 lo
      const void *xs = cv.rows(0, 1, size_t(p.b), size_t(p.h), 8);
      auto w1 = cv.planes(1, ne[1]);
      auto w3 = cv.planes(2, ne[2]);
      if (cv.err) return cv.err;
      ok = tmap_2d(&maps[0], w1.first, p.h, p.n, 64, 64, SW) && tmap_2d(&maps[1], w1.second, p.h, p.n, 64, 64, SW) &&
           tmap_2d(&maps[4], w3.first, p.h, p.n, 64, 64, SW) && tmap_2d(&maps[5], w3.second, p.h, p.n, 64, 64, SW) &&
           tmap_2d(&maps[2], xs, 16, p.h, 64, 16, SW);
    } else {
      if (cv.err) return cv.err;
      ok = tmap_2d(&maps[0], in[1], p.h, p.n, 64, 64, SW) && tmap_2d(&maps[1], in[2], p.h, p.n, 64, 64, SW) &&
           tmap_2d(&maps[2], in[0], p.b, p.h, 64, 16, SW);
    }
    maps[3] = maps[2];
  } else if (p.kind == TPO_FUSED_RMSNORM_MATMUL) {
    mode = MODE_RMS;
    sp.ksplit = pick_ksplit(p.n / 128, p.h, 1);
    if (split) {  // W hi, W lo | fp32 X, G, D
      const float *x = cv.f32(0, ne[0]), *g = cv.f32(1, ne[1]);
      auto w = cv.planes(2, ne[2]);
      sp.dscale_f32 = cv.f32(3, 1);
      if (cv.err) return cv.err;
      ok = tmap_2d(&maps[0], w.first, p.h, p.n, 64, 64, SW) && tmap_2d(&maps[1], w.second, p.h, p.n, 64, 64, SW) &&
           tmap_2d(&maps[2], x, p.b, p.h, 64, 8, NOSW, true) && tmap_2d(&maps[3], g, 1, p.h, 64, 1, NOSW, true);
    } else {
      if (cv.err) return cv.err;
      ok = tmap_2d(&maps[0], in[2], p.h, p.n, 64, 64, SW) && tmap_2d(&maps[2], in[0], p.b, p.h, 64, 8, NOSW) &&
           tmap_2d(&maps[3], in[1], 1, p.h, 64, 1, NOSW);
      maps[1] = maps[0];
      sp.x = static_cast<const __nv_bfloat16 *>(in[0]);
      sp.g = static_cast<const __nv_bfloat16 *>(in[1]);
      sp.dscale = static_cast<const __nv_bfloat16 *>(in[3]);
    }
  } else if (p.kind == TPO_FUSED_LORA) {
    mode = MODE_LORA;
    sp.ksplit = pick_ksplit(p.n / 128, p.h, 1);
    const int abox = 16;  // A box [64 k][16 r]
    if (split) {  // W hi, W lo | X rows (hi 0-15, lo 16-31) | A hi, A lo | fp32 B
      const void *xs = cv.rows(0, 1, size_t(p.b), size_t(p.h), 16);
      auto w = cv.planes(1, ne[1]);
      auto a = cv.planes(2, ne[2]);
      auto b = cv.planes(3, ne[3]);  // B̄ hi, lo: the tensor-core fold's A operand
      if (cv.err) return cv.err;
      ok = tmap_2d(&maps[0], w.first, p.h, p.n, 64, 64, SW) && tmap_2d(&maps[1], w.second, p.h, p.n, 64, 64, SW) &&
           tmap_2d(&maps[2], xs, 32, p.h, 64, 32, SW) && tmap_2d(&maps[3], a.first, p.h, p.r, abox, 64, NOSW) &&
           tmap_2d(&maps[6], a.second, p.h, p.r, abox, 64, NOSW) &&
           tmap_2d(&maps[4], b.first, p.r, p.n, 64, 16, SW) && tmap_2d(&maps[5], b.second, p.r, p.n, 64, 16, SW);
    } else {
      if (cv.err) return cv.err;
      ok = tmap_2d(&maps[0], in[1], p.h, p.n, 64, 64, SW) && tmap_2d(&maps[2], in[0], p.b, p.h, 64, 16, SW) &&
           tmap_2d(&maps[3], in[2], p.h, p.r, abox, 64, NOSW);
      maps[1] = maps[0];
      sp.x = static_cast<const __nv_bfloat16 *>(in[0]);
      sp.lora_a = static_cast<const __nv_bfloat16 *>(in[2]);
    }
  } else {
    return int(cudaErrorNotSupported);
  }
  if (!ok) return int(cudaErrorInvalidValue);
  for (int i = 4; i < 7; ++i)  // unused plane maps: any valid map
    if (!split) maps[i] = maps[0];
  if (split && mode == MODE_RMS) maps[4] = maps[5] = maps[0];
  if (split && mode != MODE_LORA) maps[6] = maps[0];
  // bf16 LoRA: B̄ [r][n] for the tensor-core fold of XA_s·B̄ (box [16 r][64 n];
  // SPLIT: its hi / lo planes, maps 4 and 5)
  if (!split && mode == MODE_LORA && !tmap_2d(&maps[4], in[3], p.r, p.n, 64, 16, SW))
    return int(cudaErrorInvalidValue);
  sp.N = int(p.n);
  sp.K = int(p.h);
  sp.tokens = int(p.b);
  sp.k_per_cta = int(p.h / sp.ksplit);
  sp.out = io.out[0];
  // outputs: one TMA tile store per owner warp (TPO_TMA_OUT=0: T coalesced
  // row stores per thread; LoRA 8.18-8.37 vs 8.20-8.24 us, same box)
  sp.tma_out = env_int("TPO_TMA_OUT", 1);
  // activations into L2 before the PDL wait (RMS 7.48 -> 7.39, LoRA 8.21 ->
  // 8.05, GatedMLP 35.4 -> 35.25 us per evaluation, same boxes)
  sp.x_l2 = env_int("TPO_X_L2", 1);
  maps[7] = maps[0];
  if (sp.tma_out) {
    const int T = mode == MODE_LORA ? 16 : 8;
    if (!tmap_2d(&maps[7], sp.out, p.b, p.n, 32, uint32_t(T), NOSW, /*f32*/ true)) return int(cudaErrorInvalidValue);
  }
  // Weights (W / W1,W3 / A) declared static may stream before the PDL wait,
  // unless the library itself just wrote them (converted operands).
  const uint64_t weights = p.kind == TPO_FUSED_GATED_MLP ? 0x6 : p.kind == TPO_FUSED_LORA ? 0x6 : 0x4;
  sp.prefetch_static = (p.static_inputs & weights) == weights && io.caller_inputs && !converted &&
                       !std::getenv("TPO_NO_PREFETCH");
  // Pipeline depth: the measured-best depth that fits (profiles/r01:
  // sweeps, steady-state ring timelines).  Two CTAs per SM (TPO_MINB=2) pay
  // off for RMS only; GatedMLP / LoRA run one CTA per SM with deeper rings.
  int stages = env_int("TPO_STAGES", 0), minb = env_int("TPO_MINB", 0);
  const size_t kOnePerSm = 232448;
  if (split) {
    stages = mode == MODE_GATED ? 3 : 5;  // the instantiated SPLIT rings (one CTA per SM)
    minb = 1;
  }
  // RMS / LoRA with static weights: two CTAs per SM (5-stage ring, <= 113 KB) so
  // the next evaluation's CTAs become resident and prefetch their weight
  // stages while this one drains (ring timeline, profiles/r01/ring_rms.txt:
  // 8.07 vs 8.63 us per evaluation).
  if (stages <= 0 && minb <= 0 && mode != MODE_GATED && sp.prefetch_static) minb = 2;
  if (stages <= 0) {
    if (minb == 2) {
      for (int s : {5, 4, 3}) {
        const size_t b = tpo_skinny_smem(mode, s, 2, 0, &sp);
        if (b && b <= 115712) {
          stages = s;
          break;
        }
      }
    }
    if (stages <= 0) {
      minb = 1;
      const int pref_g[] = {4, 6, 3}, pref_r[] = {6, 8, 4, 10}, pref_l[] = {8, 6, 4, 10};
      const int *pref = mode == MODE_GATED ? pref_g : mode == MODE_RMS ? pref_r : pref_l;
      const int np = mode == MODE_GATED ? 3 : 4;
      for (int i = 0; i < np; ++i) {
        const size_t b = tpo_skinny_smem(mode, pref[i], 1, 0, &sp);
        if (b && b <= kOnePerSm) {
          stages = pref[i];
          break;
        }
      }
    }
  } else if (minb <= 0) {
    minb = tpo_skinny_smem(mode, stages, 2, int(split), &sp) ? 2 : 1;
  }
  sp.dbg_flags = env_int("TPO_DBG_FLAGS", 0);
  sp.epi_atomic = env_int("TPO_EPI_ATOMIC", 0);
  // two CTAs per SM: the producer releases the next evaluation a few k
  // blocks before its last issue (RMS 5, LoRA 4), so the next grid's weight
  // prefetch overlaps this one's last stages (sweeps: RMS 7.59 vs 7.87 us,
  // LoRA 8.54 vs 8.84 us; with the L2 hints LoRA 8.06 at 4 vs 8.11 at 3)
  sp.trig_early = env_int("TPO_TRIG_EARLY", !sp.prefetch_static || minb != 2 ? 0 : mode == MODE_RMS ? 5 : 4);
  sp.pre_cut = env_int("TPO_PRE_CUT", 0);
  // and, behind this evaluation's X, runs two weight k blocks ahead of the
  // ring through L2 (sweeps: RMS 7.52 vs 7.67 us, LoRA 8.37 vs 8.60 us;
  // deeper run-ahead is slower, GatedMLP's deep ring gains nothing; with
  // the activation L2 hints LoRA prefers one block: 7.98 vs 8.06 us at 2)
  sp.l2_ahead = env_int("TPO_L2_AHEAD", !sp.prefetch_static || minb != 2 || mode == MODE_GATED ? 0
                                        : mode == MODE_LORA                                     ? 1
                                                                                                : 2);
  const int nct = int(p.n / 128) * sp.ksplit;
  unsigned long long *dbg = debug_begin(nct, st);
  sp.dbg = dbg;
  int rc = tpo_skinny_launch(mode, stages, minb, int(split), maps, &sp, st);
  if (dbg && !rc) {
    char tag[128];
    std::snprintf(tag, sizeof(tag), "mode %d ksplit %d stages %d minb %d prefetch %d split %d", mode,
                  sp.ksplit, stages, minb, sp.prefetch_static, int(split));
    debug_end(tag, dbg, nct, st);
  }
  return rc;
}

}  // namespace tpo::gpu

// Debug: copy the launch-timestamp ring (kRing launches x kRingCtas CTAs x
// 16 slots) to `host` and reset it; returns the launch count so far.
extern "C" int tpo_debug_ring_read(unsigned long long *host, size_t n) {
  if (!tpo::gpu::g_ring) return -1;
  const size_t tot = size_t(tpo::gpu::kRing) * tpo::gpu::kRingCtas * 16;
  cudaDeviceSynchronize();
  cudaMemcpy(host, tpo::gpu::g_ring, std::min(n, tot) * 8, cudaMemcpyDeviceToHost);
  cudaMemset(tpo::gpu::g_ring, 0, tot * 8);
  return int(tpo::gpu::g_ring_seq);
}
