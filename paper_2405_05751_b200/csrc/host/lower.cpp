// B200 backend — µGraph -> block-batched VM bytecode.
//
// Semantics follow the reference evaluator (eval_core.hpp:81-376) op for op:
//   * kernel ops in list order (:91-100); GraphDef outputs zero-initialised
//     (:229-231);
//   * block graph: post-loop set = Accum outputs and their descendants
//     (:277-294); accumulators zeroed (:296-301); loop body = InIter loads,
//     Accum updates and non-post ops in list order (:303-341); then post ops
//     and OutSavers in list order (:348-375);
//   * InIter tile offsets (load_tile, :244-270), OutSaver offsets (:350-366),
//     concat Accum slices (:321-333).
// The only structural change is that all grid blocks run as one batch
// dimension (see kernels/vm.h); results are identical because blocks never
// read each other's state and the last-writer rule is encoded in `wmask`.
#include "lower.hpp"
#include "tpo/ir/schedule.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "tpo/ir/shape_infer.hpp"

namespace tpo::gpu {

using namespace ir;

namespace {

std::vector<int64_t> contiguous(const std::vector<int64_t> &d) {
  std::vector<int64_t> s(d.size(), 1);
  for (int i = int(d.size()) - 2; i >= 0; --i) s[size_t(i)] = s[size_t(i + 1)] * d[size_t(i + 1)];
  return s;
}

int64_t numel(const TensorShape &s) { return s.elem_count(); }

// Right-aligned broadcast strides of `shape` (contiguous buffer) inside an
// index space whose trailing dims are `out` (rank R).
std::vector<int64_t> bcast_strides(const TensorShape &shape, const std::vector<int64_t> &out) {
  auto cs = contiguous(shape.dims);
  std::vector<int64_t> st(out.size(), 0);
  int shift = int(out.size()) - shape.rank();
  for (int i = 0; i < shape.rank(); ++i)
    if (shape.dims[size_t(i)] != 1) st[size_t(i + shift)] = cs[size_t(i)];
  return st;
}

struct View {
  std::vector<int64_t> dims;               // index space
  std::vector<std::vector<int64_t>> st;    // per operand (dst first)
  std::vector<char> wm;                    // per dim write-mask bit
};

// Drop unit dims and merge dims that are jointly contiguous for all operands.
// In place: the kept dims are compacted to the front (w <= k), so no
// second View is allocated.
void collapse(View &v) {
  size_t w = 0;  // dims kept so far
  for (size_t k = 0; k < v.dims.size(); ++k) {
    if (v.dims[k] == 1) continue;
    bool merge = w > 0 && !v.wm[k] && !v.wm[w - 1];
    if (merge)
      for (size_t p = 0; p < v.st.size(); ++p)
        if (v.st[p][w - 1] != v.st[p][k] * v.dims[k]) merge = false;
    if (merge) {
      v.dims[w - 1] *= v.dims[k];
      for (size_t p = 0; p < v.st.size(); ++p) v.st[p][w - 1] = v.st[p][k];
    } else {
      v.dims[w] = v.dims[k];
      v.wm[w] = v.wm[k];
      for (size_t p = 0; p < v.st.size(); ++p) v.st[p][w] = v.st[p][k];
      ++w;
    }
  }
  v.dims.resize(w);
  v.wm.resize(w);
  for (auto &s : v.st) s.resize(w);
}

int32_t i32(int64_t x) {
  if (x > INT32_MAX || x < INT32_MIN) throw Error(ErrCode::DoesNotFit, "VM stride overflow");
  return int32_t(x);
}

TpoVmInstr make(uint8_t op, uint8_t sub, View &v, uint32_t dst, uint32_t a, uint32_t b) {  // collapses v
  collapse(v);
  if (v.dims.size() > TPO_VM_DIMS) throw Error(ErrCode::Unsupported, "VM index rank > 7");
  TpoVmInstr in;
  std::memset(&in, 0, sizeof(in));
  in.op = op;
  in.sub = sub;
  in.dst = dst;
  in.a = a;
  in.b = b;
  in.ndim = uint8_t(v.dims.size());
  int64_t n = 1;
  bool flat = true;
  for (size_t k = 0; k < v.dims.size(); ++k) {
    n *= v.dims[k];
    in.dims[k] = uint32_t(v.dims[k]);
    in.sd[k] = i32(v.st[0][k]);
    if (v.st.size() > 1) in.sa[k] = i32(v.st[1][k]);
    if (v.st.size() > 2) in.sb[k] = i32(v.st[2][k]);
    if (v.wm[k]) in.wmask |= uint8_t(1u << k);
    for (auto &s : v.st)
      if (s[k] != 1) flat = false;
  }
  if (v.dims.size() > 1 || in.wmask) flat = false;
  if (n > INT32_MAX) throw Error(ErrCode::DoesNotFit, "VM index space too large");
  in.n = uint32_t(n);
  if (flat) in.flags |= VM_FLAT;
  return in;
}

// Word intervals an instruction may touch, over every for-loop iteration
// (hulls of its strided views; conservative).
struct Span {
  int64_t lo, hi;  // [lo, hi)
};

// at most 3 operand reads and 1 write per instruction: fixed storage, no
// allocation (the lowering runs per candidate of a search stream)
struct SpanList {
  Span s[3];
  int n = 0;
  void push_back(Span x) { s[n++] = x; }
  Span &back() { return s[n - 1]; }
  const Span *begin() const { return s; }
  const Span *end() const { return s + n; }
};

struct Access {
  SpanList rd, wr;
  bool opaque = false;  // treat as touching everything
};

// Hull of base + it*iter + sum_k c_k * st[k] over c_k < dims[k], it < trips.
Span view_span(uint32_t base, int64_t iter, int64_t trips, const uint32_t *dims, const int32_t *st,
               const int *ks, int nk) {
  int64_t lo = int64_t(base), hi = int64_t(base);
  const int64_t ti = (trips - 1) * iter;
  (ti < 0 ? lo : hi) += ti;
  for (int j = 0; j < nk; ++j) {
    const int k = ks[j];
    if (dims[k] == 0) return {0, 0};
    const int64_t e = int64_t(dims[k] - 1) * st[k];
    (e < 0 ? lo : hi) += e;
  }
  return {lo, hi + 1};
}

Access instr_access(const TpoVmInstr &I, int64_t trips) {
  Access A;
  static const int all[TPO_VM_DIMS] = {0, 1, 2, 3, 4, 5, 6};
  const bool flat = I.flags & VM_FLAT;
  const int64_t n = I.n;
  switch (I.op) {
    case VM_ZERO:
      A.wr.push_back({I.dst, I.dst + n});
      break;
    case VM_UNARY:
      A.rd.push_back({I.a, I.a + n});
      A.wr.push_back({I.dst, I.dst + n});
      break;
    case VM_COPY:
      if (flat) {
        A.rd.push_back(view_span(I.a, I.a_iter, trips, nullptr, nullptr, nullptr, 0));
        A.rd.back().hi += n - 1;
        A.wr.push_back(view_span(I.dst, I.d_iter, trips, nullptr, nullptr, nullptr, 0));
        A.wr.back().hi += n - 1;
      } else {
        A.rd.push_back(view_span(I.a, I.a_iter, trips, I.dims, I.sa, all, I.ndim));
        A.wr.push_back(view_span(I.dst, I.d_iter, trips, I.dims, I.sd, all, I.ndim));
      }
      break;
    case VM_BINARY:
      if (flat) {
        A.rd.push_back({I.a, I.a + n});
        A.rd.push_back({I.b, I.b + n});
        A.wr.push_back({I.dst, I.dst + n});
      } else {
        A.rd.push_back(view_span(I.a, 0, 1, I.dims, I.sa, all, I.ndim));
        A.rd.push_back(view_span(I.b, 0, 1, I.dims, I.sb, all, I.ndim));
        A.wr.push_back(view_span(I.dst, 0, 1, I.dims, I.sd, all, I.ndim));
      }
      break;
    case VM_MATMUL: {
      if (!(I.flags & VM_STRIDED)) {
        A.opaque = true;
        break;
      }
      static const int ka[6] = {0, 1, 2, 3, 4, 5}, kb[6] = {0, 1, 2, 3, 5, 6};
      A.rd.push_back(view_span(I.a, I.a_iter, trips, I.dims, I.sa, ka, 6));
      A.rd.push_back(view_span(I.b, I.b_iter, trips, I.dims, I.sb, kb, 6));
      const int64_t out = int64_t(I.dims[0]) * I.dims[1] * I.dims[2] * I.dims[3] * I.dims[4] * I.dims[6];
      A.wr.push_back({I.dst, I.dst + out});
      if (I.flags & VM_ACCUM) A.rd.push_back(A.wr.back());
      break;
    }
    case VM_SUM:
      A.rd.push_back({I.a, I.a + int64_t(I.dims[0]) * I.dims[1] * I.dims[2] * I.dims[3]});
      A.wr.push_back({I.dst, I.dst + n});
      break;
    default:
      A.opaque = true;
  }
  return A;
}

bool overlaps(const SpanList &x, const SpanList &y) {
  for (const Span &a : x)
    for (const Span &b : y)
      if (a.lo < b.hi && b.lo < a.hi) return true;
  return false;
}

}  // namespace

// Barrier placement (synchronisation only between
// dependent levels).  Consecutive instructions form one phase while none
// reads or writes a word another member of the phase writes; the CTA
// interpreters skip the barrier after every instruction but a phase's
// last (VM_NOSYNC).  Phases never span VM_LOOP / VM_ENDLOOP, and the last
// instruction of a program always synchronises.  TPO_VM_NOSYNC=0 disables.
void mark_phases(std::vector<TpoVmInstr> &code) {
  static const bool off = [] {
    const char *e = std::getenv("TPO_VM_NOSYNC");
    return e && e[0] == '0';
  }();
  for (TpoVmInstr &I : code) I.flags &= uint8_t(~VM_NOSYNC);
  if (off) return;
  int64_t trips = 1;
  std::vector<Access> phase;
  int prev = -1;  // last compute instruction of the current phase
  for (size_t k = 0; k < code.size(); ++k) {
    TpoVmInstr &I = code[k];
    if (I.op == VM_RAISE) {  // checks the event flag after a barrier of its own
      phase.clear();
      prev = -1;
      continue;
    }
    if (I.op == VM_LOOP || I.op == VM_ENDLOOP) {
      trips = I.op == VM_LOOP ? int64_t(I.n) : 1;
      phase.clear();
      prev = -1;
      continue;
    }
    Access A = instr_access(I, trips);
    bool join = prev >= 0 && !A.opaque;
    for (const Access &P : phase) {
      if (!join) break;
      if (P.opaque || overlaps(P.wr, A.rd) || overlaps(P.wr, A.wr) || overlaps(P.rd, A.wr)) join = false;
    }
    if (join) {
      code[size_t(prev)].flags |= VM_NOSYNC;
    } else {
      phase.clear();
    }
    phase.push_back(std::move(A));
    prev = int(k);
  }
}

namespace {

class Lowerer {
 public:
  Lowerer(const KernelGraph &g, uint32_t in_base, uint32_t region, bool pin, bool field,
          bool list_order = false)
      : g_(g), region_(region), pin_(pin), field_(field), list_order_(list_order) {
    kbuf_.assign(g.tensors.size(), UINT32_MAX);
    kqd_.assign(g.tensors.size(), 1);
    uint32_t off = in_base;
    lazy_ok_ = in_base == 0 && g.inputs.size() <= TPO_VM_MAX_GEN;
    for (TensorId t : g.inputs) {
      if (kbuf_[size_t(t)] == UINT32_MAX) {
        kbuf_[size_t(t)] = off;
        in_ranges_.push_back({off, uint32_t(numel(g.tensor(t).shape))});
        off += uint32_t(numel(g.tensor(t).shape));
      } else {
        lazy_ok_ = false;  // a repeated input: words and draw order differ
      }
      p_.in_shapes.push_back(g.tensor(t).shape);
    }
  }

  VmProgram run() {
    for (const Op &op : g_.ops) {
      if (op.type == OpType::GraphDef) {
        graphdef(op);
        continue;
      }
      std::vector<uint32_t> ins;
      std::vector<TensorShape> shapes;
      std::vector<uint8_t> qds;
      for (TensorId t : op.inputs) {
        ins.push_back(buf(t));
        shapes.push_back(g_.tensor(t).shape);
        qds.push_back(kqd_[size_t(t)]);
      }
      const TensorId out = op.outputs.at(0);
      kbuf_[size_t(out)] = alloc(numel(g_.tensor(out).shape));
      kqd_[size_t(out)] = compute(op, ins, shapes, qds, std::vector<uint8_t>(ins.size(), 1),
                                  kbuf_[size_t(out)], g_.tensor(out).shape, {1, 1, 1});
    }
    if (g_.outputs.size() > TPO_VM_MAX_OUTPUTS) throw Error(ErrCode::Unsupported, "too many outputs");
    p_.desc.n_out = uint32_t(g_.outputs.size());
    for (size_t i = 0; i < g_.outputs.size(); ++i) {
      TensorId t = g_.outputs[i];
      p_.desc.out_off[i] = buf(t);
      p_.desc.out_len[i] = uint32_t(numel(g_.tensor(t).shape));
      p_.desc.out_qd[i] = kqd_[size_t(t)];
      p_.out_shapes.push_back(g_.tensor(t).shape);
    }
    // DivByZero / NonResidue events count toward a VM_RAISE only when the
    // reference evaluates them before the raising op: every earlier op
    // outside the raising GraphDef, grid block 0 inside it
    for (size_t k = 0; k < p_.code.size(); ++k)
      if (raise_at_ < 0 || int64_t(k) > raise_at_ || gd_of_[k] != raise_gd_) p_.code[k].b0n = 0;
    plan_memory();
    mark_phases(p_.code);
    if (field_ && lazy_ok_) lazy_inputs();
    p_.desc.words = p_.region_words;
    p_.desc.code_len = uint32_t(p_.code.size());
    p_.desc.poisoned = p_.poisoned;
    p_.desc.has_silu = p_.has_silu;
    p_.madds = graph_madds(g_);
    return std::move(p_);
  }

 private:
  const KernelGraph &g_;
  uint32_t region_;
  bool pin_;
  bool field_;
  bool list_order_;                               // emit block ops in list order (VM_RAISE graphs)
  int gd_ = -1;                                   // GraphDef being lowered (-1: kernel level)
  std::vector<int> gd_of_;                        // per instruction: its GraphDef
  int64_t raise_at_ = -1;                         // index of the VM_RAISE, if any
  int raise_gd_ = -1;
  int gd_count_ = -1;
  static constexpr uint32_t kVirt = 0x80000000u;  // virtual buffer id tag
  std::vector<int64_t> vsize_;                    // words per virtual buffer
  std::vector<uint32_t> kbuf_;
  std::vector<uint8_t> kqd_;
  std::vector<std::pair<uint32_t, uint32_t>> in_ranges_;  // input words (offset, count), input order
  bool lazy_ok_ = false;
  VmProgram p_;

  // Buffers are virtual until plan_memory() assigns addresses.
  uint32_t alloc(int64_t words) {
    if (words > int64_t(INT32_MAX / 2)) throw Error(ErrCode::DoesNotFit, "VM buffer too large");
    vsize_.push_back(words);
    return kVirt | uint32_t(vsize_.size() - 1);
  }

  // Liveness-based placement (the role of the reference's absent memplan,
  // SPEC.md:527-545): interval [first use, last use] over the instruction
  // stream, widened to the whole loop body for buffers touched inside the
  // for-loop; graph outputs live to the end (or are pinned at the region
  // start when `pin_`, so a later program may reuse the scratch above them).
  // First-fit placement; a buffer may reuse space only after the previous
  // occupant's last use (strictly earlier instruction).
  void plan_memory() {
    const size_t nv = vsize_.size(), nc = p_.code.size();
    std::vector<int64_t> lo(nv, INT64_MAX), hi(nv, -1);
    std::vector<std::pair<size_t, size_t>> loops;
    size_t lb = 0;
    for (size_t k = 0; k < nc; ++k) {
      if (p_.code[k].op == VM_LOOP) lb = k;
      if (p_.code[k].op == VM_ENDLOOP) loops.emplace_back(lb, k);
    }
    auto touch = [&](uint32_t b, size_t k) {
      if (!(b & kVirt)) return;
      uint32_t v = b & ~kVirt;
      lo[v] = std::min<int64_t>(lo[v], int64_t(k));
      hi[v] = std::max<int64_t>(hi[v], int64_t(k));
    };
    for (size_t k = 0; k < nc; ++k) {
      const TpoVmInstr &I = p_.code[k];
      if (I.op == VM_LOOP || I.op == VM_ENDLOOP) continue;
      touch(I.dst, k);
      if (I.op != VM_ZERO) touch(I.a, k);
      if (I.op == VM_BINARY || I.op == VM_MATMUL) touch(I.b, k);
    }
    for (size_t v = 0; v < nv; ++v)
      for (auto [a, b] : loops)
        if (hi[v] >= int64_t(a) && lo[v] <= int64_t(b)) {
          lo[v] = std::min<int64_t>(lo[v], int64_t(a));
          hi[v] = std::max<int64_t>(hi[v], int64_t(b));
        }
    std::vector<int64_t> addr(nv, -1);
    int64_t pinned = 0;
    for (uint32_t i = 0; i < p_.desc.n_out; ++i) {
      uint32_t b = p_.desc.out_off[i];
      if (!(b & kVirt)) continue;
      uint32_t v = b & ~kVirt;
      hi[v] = int64_t(nc);
      if (pin_ && addr[v] < 0) {
        addr[v] = region_ + pinned;
        pinned += vsize_[v];
      }
    }
    std::vector<size_t> order;
    for (size_t v = 0; v < nv; ++v)
      if (addr[v] < 0 && hi[v] >= 0) order.push_back(v);
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return lo[a] < lo[b]; });
    struct Live {
      int64_t off, size, end;
    };
    std::vector<Live> live;
    const int64_t base = int64_t(region_) + pinned;
    int64_t peak = base;
    for (size_t v : order) {
      live.erase(std::remove_if(live.begin(), live.end(), [&](const Live &l) { return l.end < lo[v]; }),
                 live.end());
      std::sort(live.begin(), live.end(), [](const Live &a, const Live &b) { return a.off < b.off; });
      int64_t at = base;
      for (const Live &l : live) {
        if (at + vsize_[v] <= l.off) break;
        at = std::max(at, l.off + l.size);
      }
      addr[v] = at;
      live.push_back({at, vsize_[v], hi[v]});
      peak = std::max(peak, at + vsize_[v]);
    }
    // the SPEC planner (exhaustive over placement orders up to 8 buffers,
    // first-fit-decreasing above) on the same lifetimes: keep the lower peak
    static const bool ffd = [] {
      const char *e = std::getenv("TPO_VM_FFD");
      return !(e && e[0] == '0');
    }();
    // skip it when first fit already meets the load bound (the largest
    // total size live at one instruction: no placement can go below it)
    int64_t load = 0;
    if (ffd) {
      std::vector<std::pair<int64_t, int64_t>> ev;  // (position, +size at start / -size after end)
      for (size_t v : order) ev.emplace_back(lo[v] * 2, vsize_[v]), ev.emplace_back(hi[v] * 2 + 1, -vsize_[v]);
      std::sort(ev.begin(), ev.end());
      int64_t cur = 0;
      for (auto &e : ev) load = std::max(load, cur += e.second);
    }
    if (ffd && peak - base > load) {
      std::vector<Lifetime> lt;
      for (size_t v : order) lt.push_back({vsize_[v], lo[v], hi[v]});
      const MemoryPlan mp = plan_intervals(lt, 0);  // first-fit-decreasing (host cost: lowering runs per batch)
      if (base + mp.peak < peak) {
        for (size_t i = 0; i < order.size(); ++i) addr[order[i]] = base + mp.offset[i];
        peak = base + mp.peak;
      }
    }
    for (size_t v = 0; v < nv; ++v) {
      if (addr[v] < 0) addr[v] = base;  // never referenced
      if (addr[v] + vsize_[v] > int64_t(INT32_MAX)) throw Error(ErrCode::DoesNotFit, "VM region overflow");
    }
    auto fix = [&](uint32_t &b) {
      if (b & kVirt) b = uint32_t(addr[b & ~kVirt]);
    };
    for (TpoVmInstr &I : p_.code) {
      if (I.op == VM_LOOP || I.op == VM_ENDLOOP) continue;
      fix(I.dst);
      if (I.op != VM_ZERO) fix(I.a);
      if (I.op == VM_BINARY || I.op == VM_MATMUL) fix(I.b);
    }
    for (uint32_t i = 0; i < p_.desc.n_out; ++i) fix(p_.desc.out_off[i]);
    p_.pinned_words = uint32_t(pinned);
    p_.region_words = uint32_t(std::max(peak, base) - region_);
  }

  // Lazy input sampling (FF verifier): per input, the first instruction
  // whose read hull (instr_access, over every loop iteration) touches its
  // words; opaque instructions count as reading everything.  The draws of
  // an input are independent of when they are made (closed-form stream),
  // so drawing it right before its first reader gives the reference's
  // values; an attempt that resamples earlier never draws it.  Inputs whose
  // first readers are not separated by an instruction that can resample
  // (sqrt, division, a fused sqrt, VM_RAISE) are drawn together at the
  // earlier point, contiguous ranges merged; when that leaves one group the
  // graph draws everything up front (n_gen = 0: no barrier overhead).
  void lazy_inputs() {
    const size_t ni = in_ranges_.size(), nc = p_.code.size();
    std::vector<uint32_t> first(ni, uint32_t(nc));
    std::vector<char> event(nc, 0);
    int64_t trips = 1;
    for (size_t k = 0; k < nc; ++k) {
      const TpoVmInstr &I = p_.code[k];
      if (I.op == VM_LOOP) {
        trips = int64_t(I.n);
        continue;
      }
      if (I.op == VM_ENDLOOP) {
        trips = 1;
        continue;
      }
      event[k] = I.op == VM_RAISE || (I.op == VM_UNARY && I.sub == VM_SQRT) ||
                 (I.op == VM_BINARY && (I.sub == VM_DIV || I.pre_a == 1 + VM_SQRT || I.pre_b == 1 + VM_SQRT));
      if (I.op == VM_RAISE) continue;
      const Access A = instr_access(I, trips);
      for (size_t i = 0; i < ni; ++i) {
        if (first[i] != nc) continue;
        const int64_t lo = in_ranges_[i].first, hi = lo + in_ranges_[i].second;
        bool rd = A.opaque;
        for (const Span &sp : A.rd) rd = rd || (sp.lo < hi && lo < sp.hi);
        if (rd) first[i] = uint32_t(k);
      }
    }
    std::vector<size_t> ord(ni);
    std::iota(ord.begin(), ord.end(), size_t(0));
    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return first[a] < first[b]; });
    // group: an input joins the current group unless an event-capable
    // instruction lies between the group's draw point and its first reader
    std::vector<uint32_t> at(ni);
    uint32_t gpc = ni ? first[ord[0]] : 0;
    int groups = ni ? 1 : 0;
    for (size_t j = 0; j < ni; ++j) {
      const uint32_t f = first[ord[j]];
      bool ev = false;
      for (uint32_t k = gpc; k < f && k < nc; ++k) ev = ev || event[k];
      static const bool nogroup = [] {  // experiment: one draw point per input
        const char *e = std::getenv("TPO_VM_LAZY_GROUP");
        return e && e[0] == '0';
      }();
      if (ev || (nogroup && f != gpc)) {
        gpc = f;
        ++groups;
      }
      at[ord[j]] = gpc;
    }
    if (groups <= 1) return;
    // entries by (draw point, word offset), contiguous ranges of one point merged
    std::vector<size_t> ent(ni);
    std::iota(ent.begin(), ent.end(), size_t(0));
    std::sort(ent.begin(), ent.end(), [&](size_t a, size_t b) {
      return at[a] != at[b] ? at[a] < at[b] : in_ranges_[a].first < in_ranges_[b].first;
    });
    uint8_t n = 0;
    for (size_t i : ent) {
      if (n && p_.desc.gen_pc[n - 1] == at[i] && p_.desc.gen_e0[n - 1] + p_.desc.gen_len[n - 1] == in_ranges_[i].first) {
        p_.desc.gen_len[n - 1] += in_ranges_[i].second;
        continue;
      }
      p_.desc.gen_pc[n] = at[i];
      p_.desc.gen_e0[n] = in_ranges_[i].first;
      p_.desc.gen_len[n] = in_ranges_[i].second;
      ++n;
    }
    p_.desc.n_gen = n;
  }

  uint32_t buf(TensorId t) {
    if (kbuf_[size_t(t)] == UINT32_MAX)
      throw Error(ErrCode::ShapeMismatch, "tensor " + std::to_string(t) + " used before defined");
    return kbuf_[size_t(t)];
  }

  void emit(TpoVmInstr in) {
    static const uint32_t tile_min = [] {
      const char *e = std::getenv("TPO_VM_TILE_MIN");
      return e ? uint32_t(std::atoi(e)) : 64u;  // measured: 64 best (profiles)
    }();
    if (in.op == VM_MATMUL && (in.flags & VM_STRIDED) && in.dims[4] % 2 == 0 && in.dims[6] % 2 == 0 &&
        in.n / 4 >= tile_min) {
      in.flags |= VM_TILE22;  // one thread, 2 x 2 outputs: shared operand loads
      in.n /= 4;
    }
    tpo_vm_set_divisors(&in);
    p_.code.push_back(in);
    gd_of_.push_back(gd_);
  }

  // Grid dims (bx, by, bz) and the strides of a block tensor of E elements.
  // Block-invariant tensors (identical in every block) are stored once:
  // their grid strides are 0.
  static void grid_part(const std::array<int64_t, 3> &G, int64_t E, bool inv,
                        std::vector<int64_t> &dims, std::vector<int64_t> &st) {
    dims = {G[0], G[1], G[2]};
    if (inv)
      st = {0, 0, 0};
    else
      st = {G[1] * G[2] * E, G[2] * E, E};
  }

  static std::vector<int64_t> cat(std::vector<int64_t> a, const std::vector<int64_t> &b) {
    a.insert(a.end(), b.begin(), b.end());
    return a;
  }

  // Matmul over contiguous (block-batched) operands, expressed in the
  // strided form every VM matmul uses (kernels/vm.h VM_STRIDED).
  void emit_matmul(uint32_t d, uint32_t a, uint32_t b, const TensorShape &sa, const TensorShape &sb,
                   int64_t nb, bool inv_a, bool inv_b, uint8_t q) {
    const int r = sa.rank();
    const int64_t M = sa.dims[size_t(r - 2)], K = sa.dims[size_t(r - 1)], N = sb.dims[size_t(r - 1)];
    const int64_t Bi = numel(sa) / (M * K);
    TpoVmInstr i;
    std::memset(&i, 0, sizeof(i));
    i.op = VM_MATMUL;
    i.flags = VM_STRIDED;
    i.dst = d;
    i.a = a;
    i.b = b;
    i.ndim = 7;
    const int64_t d7[7] = {nb, 1, 1, Bi, M, K, N};
    for (int k = 0; k < 7; ++k) i.dims[k] = uint32_t(d7[k]);
    i.sa[0] = inv_a ? 0 : i32(Bi * M * K);
    i.sb[0] = inv_b ? 0 : i32(Bi * K * N);
    i.sa[3] = i32(M * K), i.sa[4] = i32(K), i.sa[5] = 1;
    i.sb[3] = i32(K * N), i.sb[5] = i32(N), i.sb[6] = 1;
    if (nb * Bi * M * N > INT32_MAX) throw Error(ErrCode::DoesNotFit, "VM matmul too large");
    i.n = uint32_t(nb * Bi * M * N);
    i.qd = q;
    emit(i);
  }

  // Pre-defined op at kernel level (G = {1,1,1}) or block level (block-
  // batched).  `inv[k]`: input k is block-invariant; the output is invariant
  // iff every input is (then it is computed once).  Returns q-definedness.
  // `pre` (nullable): per input, a fused thread-graph unary (vm.h pre_a /
  // pre_b) applied to it in registers.
  uint8_t compute(const Op &op, const std::vector<uint32_t> &in, const std::vector<TensorShape> &s,
                  const std::vector<uint8_t> &qd, const std::vector<uint8_t> &inv, uint32_t dst,
                  const TensorShape &out, const std::array<int64_t, 3> &G,
                  const std::vector<uint8_t> *pre = nullptr) {
    bool inv_out = true;
    for (uint8_t x : inv) inv_out = inv_out && x;
    const std::array<int64_t, 3> Go = inv_out ? std::array<int64_t, 3>{1, 1, 1} : G;
    const int64_t nb = Go[0] * Go[1] * Go[2];
    std::vector<int64_t> gd, d_g;
    grid_part(Go, numel(out), false, gd, d_g);
    auto flat = [&](uint8_t opc, uint8_t sub, int nops) {
      View v;
      v.dims = {nb * numel(out)};
      v.st.assign(size_t(nops), {1});
      v.wm = {0};
      return make(opc, sub, v, dst, in[0], nops > 2 ? in[1] : 0);
    };
    auto elementwise2 = [&](uint8_t sub) {
      View v;
      std::vector<int64_t> a_g, b_g;
      grid_part(Go, numel(s[0]), inv[0], gd, a_g);
      grid_part(Go, numel(s[1]), inv[1], gd, b_g);
      v.dims = cat(gd, out.dims);
      v.st = {cat(d_g, contiguous(out.dims)), cat(a_g, bcast_strides(s[0], out.dims)),
              cat(b_g, bcast_strides(s[1], out.dims))};
      v.wm.assign(v.dims.size(), 0);
      TpoVmInstr i = make(VM_BINARY, sub, v, dst, in[0], in[1]);
      i.b0n = uint32_t(numel(out));  // grid-block-major index space: block 0 first
      if (pre) {
        i.pre_a = (*pre)[0], i.pre_b = (*pre)[1];
        if (i.pre_a == 1 + VM_SILU || i.pre_b == 1 + VM_SILU) p_.has_silu = true;
      }
      i.qd = qd[0] & qd[1];
      i.flags |= (qd[0] ? VM_A_QD : 0) | (qd[1] ? VM_B_QD : 0);
      emit(i);
      return uint8_t(qd[0] & qd[1]);
    };
    auto unary = [&](uint8_t sub) {
      TpoVmInstr i = flat(VM_UNARY, sub, 2);
      i.b0n = uint32_t(numel(out));
      uint8_t q = sub == VM_EXP ? 0 : qd[0];
      if (sub == VM_EXP && !qd[0]) {
        // the reference throws Error(PoisonedExponent) here (field.cpp:105-108)
        // unless a ResampleNeeded came first: stop the program at this op
        if (field_ && raise_at_ < 0) {
          TpoVmInstr r;
          std::memset(&r, 0, sizeof(r));
          r.op = VM_RAISE;
          raise_at_ = int64_t(p_.code.size());
          raise_gd_ = gd_;
          emit(r);
        }
        p_.poisoned = true;
      }
      if (sub == VM_SILU) p_.has_silu = true;
      i.qd = q;
      i.flags |= qd[0] ? VM_A_QD : 0;
      emit(i);
      return q;
    };
    switch (op.type) {
      case OpType::EwAdd:
        return elementwise2(VM_ADD);
      case OpType::EwMul:
        return elementwise2(VM_MUL);
      case OpType::EwDiv:
        return elementwise2(VM_DIV);
      case OpType::EwExp:
        return unary(VM_EXP);
      case OpType::Sqr:
        return unary(VM_SQR);
      case OpType::Sqrt:
        return unary(VM_SQRT);
      case OpType::SiLU:
        return unary(VM_SILU);
      case OpType::Matmul: {
        uint8_t q = qd[0] & qd[1];
        emit_matmul(dst, in[0], in[1], s[0], s[1], nb, inv[0], inv[1], q);
        return q;
      }
      case OpType::ConcatMatmul: {
        // W x Y + X x Z (eval_core.hpp:116-122); temporaries share the output's batching
        uint32_t t1 = alloc(nb * numel(out)), t2 = alloc(nb * numel(out));
        uint8_t q1 = qd[0] & qd[2], q2 = qd[1] & qd[3];
        emit_matmul(t1, in[0], in[2], s[0], s[2], nb, inv[0], inv[2], q1);
        emit_matmul(t2, in[1], in[3], s[1], s[3], nb, inv[1], inv[3], q2);
        View v;
        v.dims = {nb * numel(out)};
        v.st = {{1}, {1}, {1}};
        v.wm = {0};
        TpoVmInstr i = make(VM_BINARY, VM_ADD, v, dst, t1, t2);
        i.qd = q1 & q2;
        i.flags |= (q1 ? VM_A_QD : 0) | (q2 ? VM_B_QD : 0);
        emit(i);
        return q1 & q2;
      }
      case OpType::Sum: {
        const auto &a = std::get<SumAttrs>(op.attrs);
        int64_t outer = nb, inner = 1;
        for (int k = 0; k < a.dim; ++k) outer *= s[0].dims[size_t(k)];
        for (int k = a.dim + 1; k < s[0].rank(); ++k) inner *= s[0].dims[size_t(k)];
        TpoVmInstr i;
        std::memset(&i, 0, sizeof(i));
        i.op = VM_SUM;
        i.dst = dst;
        i.a = in[0];
        i.ndim = 4;
        i.dims[0] = uint32_t(outer);
        i.dims[1] = uint32_t(s[0].dims[size_t(a.dim)] / a.group);
        i.dims[2] = uint32_t(a.group);
        i.dims[3] = uint32_t(inner);
        i.n = uint32_t(outer * i.dims[1] * inner);
        i.qd = qd[0];
        emit(i);
        return qd[0];
      }
      case OpType::Repeat: {
        View v;
        std::vector<int64_t> a_g;
        grid_part(Go, numel(s[0]), inv[0], gd, a_g);
        v.dims = cat(gd, out.dims);
        v.st = {cat(d_g, contiguous(out.dims)), cat(a_g, bcast_strides(s[0], out.dims))};
        v.wm.assign(v.dims.size(), 0);
        TpoVmInstr i = make(VM_COPY, 0, v, dst, in[0], 0);
        i.qd = qd[0];
        emit(i);
        return qd[0];
      }
      case OpType::Reshape: {
        TpoVmInstr i = flat(VM_COPY, 0, 2);
        i.qd = qd[0];
        emit(i);
        return qd[0];
      }
      default:
        throw Error(ErrCode::Unsupported, std::string("VM lowering of ") + op_name(op.type));
    }
  }

  void graphdef(const Op &op) {
    if (!op.block) throw Error(ErrCode::Unsupported, "graphdef without block");
    struct GdScope {
      int &g;
      int saved;
      GdScope(int &x, int v) : g(x), saved(x) { g = v; }
      ~GdScope() { g = saved; }
    } scope(gd_, ++gd_count_);
    const BlockGraph &bg = *op.block;
    const std::array<int64_t, 3> G = bg.grid;
    for (int a = 0; a < 3; ++a)
      if (G[size_t(a)] < 1) throw Error(ErrCode::Unsupported, "grid extent < 1");
    if (bg.forloop < 1) throw Error(ErrCode::Unsupported, "forloop < 1");
    const int64_t nb = G[0] * G[1] * G[2];

    // kernel-level outputs, zero-initialised (eval_core.hpp:229-231)
    for (TensorId t : op.outputs) {
      kbuf_[size_t(t)] = alloc(numel(g_.tensor(t).shape));
      kqd_[size_t(t)] = 1;
      View v;
      v.dims = {numel(g_.tensor(t).shape)};
      v.st = {{1}};
      v.wm = {0};
      TpoVmInstr z = make(VM_ZERO, 0, v, kbuf_[size_t(t)], 0, 0);
      z.qd = 1;
      emit(z);
    }

    const size_t nt = bg.tensors.size();
    std::vector<uint32_t> bbuf(nt, UINT32_MAX);
    std::vector<uint8_t> bqd(nt, 1), binv(nt, 1);
    std::vector<char> post(nt, 0);
    for (const Op &b : bg.ops) {  // eval_core.hpp:277-294
      if (b.type == OpType::Accum) {
        post[size_t(b.outputs[0])] = 1;
        continue;
      }
      if (b.type == OpType::InIter || b.type == OpType::OutSaver) continue;
      for (TensorId t : b.inputs)
        if (post[size_t(t)]) post[size_t(b.outputs[0])] = 1;
    }
    auto is_post = [&](const Op &b) {
      for (TensorId t : b.inputs)
        if (post[size_t(t)]) return true;
      return false;
    };
    auto bshape = [&](TensorId t) -> const TensorShape & { return bg.tensor(t).shape; };
    auto bget = [&](TensorId t) {
      if (bbuf[size_t(t)] == UINT32_MAX)
        throw Error(ErrCode::ShapeMismatch, "block tensor used before defined");
      return bbuf[size_t(t)];
    };
    auto copies = [&](TensorId t) { return binv[size_t(t)] ? int64_t(1) : nb; };

    // Block invariance (list order = topological order): an InIter whose
    // imap replicates every grid axis of extent > 1 loads the same tile in
    // every block; ops / accumulators fed only by invariant values are
    // invariant.
    for (const Op &b : bg.ops) {
      if (b.type == OpType::OutSaver) continue;
      bool inv = true;
      if (b.type == OpType::InIter) {
        const auto &a = std::get<InIterAttrs>(b.attrs);
        for (int ax = 0; ax < 3; ++ax)
          if (G[size_t(ax)] > 1 && ax < a.imap.axes() && a.imap.targets[size_t(ax)] != kReplica)
            inv = false;
      } else {
        for (TensorId t : b.inputs) inv = inv && binv[size_t(t)];
      }
      for (TensorId t : b.outputs) binv[size_t(t)] = inv;
    }

    std::vector<std::vector<const Op *>> cons(nt);
    for (const Op &b : bg.ops)
      for (TensorId t : b.inputs) cons[size_t(t)].push_back(&b);
    // Thread-graph chains (the graph's ThreadGroups, or the
    // fuser's rule — a single-consumer elementwise chain — when it has none):
    // a Sqr / Sqrt / SiLU whose only consumer is an elementwise binary of the
    // same group runs inside that binary's instruction (pre_a / pre_b), its
    // result staying in registers: the chain's interior tensor gets no VM
    // words and no instruction.  Graphs that raise (list order kept for the
    // PoisonedExponent ordering) are not fused.
    std::vector<uint8_t> pre_sub(nt, 0);
    std::vector<TensorId> pre_src(nt, -1);
    {
      static const bool off = [] {
        const char *e = std::getenv("TPO_VM_CHAINS");
        return e && e[0] == '0';
      }();
      std::vector<int> group(bg.ops.size(), -1);
      for (size_t gi = 0; gi < bg.thread_groups.size(); ++gi)
        for (int id : bg.thread_groups[gi].op_ids)
          if (id >= 0 && size_t(id) < group.size()) group[size_t(id)] = int(gi);
      const bool explicit_groups = !bg.thread_groups.empty();
      for (const Op &u : bg.ops) {
        if (off || list_order_) break;
        uint8_t sub;
        switch (u.type) {
          case OpType::Sqr: sub = VM_SQR; break;
          case OpType::Sqrt: sub = VM_SQRT; break;
          case OpType::SiLU: sub = VM_SILU; break;
          default: continue;
        }
        const TensorId o = u.outputs[0];
        if (cons[size_t(o)].size() != 1) continue;
        const Op &b = *cons[size_t(o)][0];
        if (b.type != OpType::EwAdd && b.type != OpType::EwMul && b.type != OpType::EwDiv) continue;
        if (explicit_groups && (group[size_t(u.id)] < 0 || group[size_t(u.id)] != group[size_t(b.id)])) continue;
        pre_sub[size_t(o)] = uint8_t(1 + sub);
        pre_src[size_t(o)] = u.inputs[0];
      }
    }
    auto chained = [&](const Op &b) {
      return b.outputs.size() == 1 && pre_sub[size_t(b.outputs[0])] != 0;
    };

    // A concat-Accum of an InIter tile along that tile's own fmap dim is the
    // untiled tile over the whole loop range (the concat is an address
    // offset): when only Matmuls consume it, it is a view of
    // the kernel input — no per-iteration copy, no accumulator buffer.
    std::vector<char> concat_view(nt, 0), concat_src(nt, 0);
    for (const Op &b : bg.ops) {
      if (b.type != OpType::Accum) continue;
      const auto &fa = std::get<AccumAttrs>(b.attrs);
      if (!fa.fmap.axes() || fa.fmap.targets[0] == kReplica) continue;
      const TensorId val = b.inputs[0], acc = b.outputs[0];
      const Op *prod = nullptr;
      for (const Op &c : bg.ops)
        for (TensorId t : c.outputs)
          if (t == val) prod = &c;
      if (!prod || prod->type != OpType::InIter || cons[size_t(val)].size() != 1) continue;
      const auto &ia = std::get<InIterAttrs>(prod->attrs);
      if (!ia.fmap.axes() || ia.fmap.targets[0] != fa.fmap.targets[0]) continue;
      if (cons[size_t(acc)].empty() || bshape(acc).rank() < 2) continue;
      bool ok = true;
      for (const Op *c : cons[size_t(acc)]) ok = ok && c->type == OpType::Matmul;
      const TensorShape &dev = g_.tensor(op.inputs[size_t(ia.operand)]).shape;
      if (!ok || dev.rank() != bshape(acc).rank()) continue;
      concat_view[size_t(acc)] = 1;
      concat_src[size_t(val)] = 1;
    }

    // accumulators: the Accum output buffer is the running state
    for (const Op &b : bg.ops)
      if (b.type == OpType::Accum) {
        TensorId t = b.outputs[0];
        if (concat_view[size_t(t)]) continue;
        bbuf[size_t(t)] = alloc(copies(t) * numel(bshape(t)));
        View v;
        v.dims = {copies(t) * numel(bshape(t))};
        v.st = {{1}};
        v.wm = {0};
        TpoVmInstr z = make(VM_ZERO, 0, v, bbuf[size_t(t)], 0, 0);
        z.qd = 1;
        emit(z);
      }
    for (const Op &b : bg.ops)
      for (TensorId t : b.outputs)
        if (bbuf[size_t(t)] == UINT32_MAX && !pre_sub[size_t(t)])  // chain interiors: registers
          bbuf[size_t(t)] = alloc(copies(t) * numel(bshape(t)));

    // ---- operand views and fused accumulation (thread-graph-free fusion of
    // the block graph's data movement into its matmuls):
    //  * an InIter tile consumed only by in-loop Matmuls is not copied: the
    //    Matmul reads it in place through strides (VM_STRIDED);
    //  * a Matmul whose only consumer is a φ-Accum accumulates straight into
    //    the accumulator (VM_ACCUM: acc = add(acc, A·B), the reference's
    //    Accum update, eval_core.hpp:311-320).
    struct Operand {
      uint32_t base;
      int64_t g[3];
      std::vector<int64_t> dims, st;
      int32_t it_step;
    };
    std::vector<char> is_view(nt, 0);
    std::vector<Operand> views(nt);
    std::vector<char> acc_fused(nt, 0);  // Accum output fed by a fused Matmul
    std::vector<TpoVmInstr> hoisted;     // field mode: loop-spanning Matmuls
    auto collapsible = [](const std::vector<int64_t> &d, const std::vector<int64_t> &st) {
      // batch dims (all but the last two) must flatten to one stride
      const int r = int(d.size());
      int64_t prev = -1, prev_d = 1;
      for (int i = r - 3; i >= 0; --i) {
        if (d[size_t(i)] == 1) continue;
        if (prev >= 0 && st[size_t(i)] != prev * prev_d) return false;
        prev = st[size_t(i)], prev_d = d[size_t(i)];
      }
      return true;
    };
    for (const Op &b : bg.ops) {
      if (b.type != OpType::InIter) continue;
      const TensorId o = b.outputs[0];
      if (cons[size_t(o)].empty() || bshape(o).rank() < 2) continue;
      bool ok = true;
      for (const Op *c : cons[size_t(o)]) ok = ok && c->type == OpType::Matmul && !is_post(*c);
      if (!ok) continue;
      const auto &a = std::get<InIterAttrs>(b.attrs);
      const TensorShape &dev = g_.tensor(op.inputs[size_t(a.operand)]).shape;
      if (dev.rank() != bshape(o).rank()) continue;
      if (!collapsible(bshape(o).dims, contiguous(dev.dims))) continue;
      is_view[size_t(o)] = 1;
    }
    auto operand = [&](TensorId t) {
      Operand d;
      if (is_view[size_t(t)]) return views[size_t(t)];
      d.base = bget(t);
      const int64_t E = numel(bshape(t));
      const bool inv = binv[size_t(t)];
      d.g[0] = inv ? 0 : G[1] * G[2] * E;
      d.g[1] = inv ? 0 : G[2] * E;
      d.g[2] = inv ? 0 : E;
      d.dims = bshape(t).dims;
      d.st = contiguous(d.dims);
      d.it_step = 0;
      return d;
    };
    auto matmul_fusable = [&](const Op &b) {
      if (b.type != OpType::Matmul) return false;
      bool any_view = is_view[size_t(b.inputs[0])] || is_view[size_t(b.inputs[1])];
      if (is_post(b)) return any_view;  // post-loop: only concat views (loop-invariant)
      const auto &oc = cons[size_t(b.outputs[0])];
      bool to_acc = false;
      if (oc.size() == 1 && oc[0]->type == OpType::Accum) {
        const auto &fa = std::get<AccumAttrs>(oc[0]->attrs);
        to_acc = !fa.fmap.axes() || fa.fmap.targets[0] == kReplica;
      }
      return any_view || to_acc;
    };
    auto emit_strided_matmul = [&](const Op &b) {
      const TensorId ta = b.inputs[0], tb = b.inputs[1], to = b.outputs[0];
      const Operand A = operand(ta), B = operand(tb);
      const int r = bshape(ta).rank();
      const int64_t M = A.dims[size_t(r - 2)], K = A.dims[size_t(r - 1)], N = B.dims[size_t(r - 1)];
      // batch dims flatten to one index whose stride is the innermost
      // non-unit batch dim's (layouts were checked collapsible)
      int64_t Bi = 1, sab = 0, sbb = 0;
      for (int i = 0; i < r - 2; ++i) {
        Bi *= A.dims[size_t(i)];
        if (A.dims[size_t(i)] != 1) sab = A.st[size_t(i)], sbb = B.st[size_t(i)];
      }
      const bool inv_out = binv[size_t(ta)] && binv[size_t(tb)];
      const std::array<int64_t, 3> Go = inv_out ? std::array<int64_t, 3>{1, 1, 1} : G;
      const auto &oc = cons[size_t(to)];
      bool to_acc = false;
      TensorId acc = -1;
      if (oc.size() == 1 && oc[0]->type == OpType::Accum) {
        const auto &fa = std::get<AccumAttrs>(oc[0]->attrs);
        if (!fa.fmap.axes() || fa.fmap.targets[0] == kReplica) to_acc = true, acc = oc[0]->outputs[0];
      }
      TpoVmInstr i;
      std::memset(&i, 0, sizeof(i));
      i.op = VM_MATMUL;
      i.flags = VM_STRIDED | (to_acc ? VM_ACCUM : 0);
      i.dst = to_acc ? bbuf[size_t(acc)] : bbuf[size_t(to)];
      i.a = A.base;
      i.b = B.base;
      i.ndim = 7;
      const int64_t d7[7] = {Go[0], Go[1], Go[2], Bi, M, K, N};
      for (int k = 0; k < 7; ++k) i.dims[k] = uint32_t(d7[k]);
      for (int k = 0; k < 3; ++k) i.sa[k] = i32(A.g[k]), i.sb[k] = i32(B.g[k]);
      i.sa[3] = i32(sab), i.sb[3] = i32(sbb);
      i.sa[4] = i32(A.st[size_t(r - 2)]), i.sa[5] = i32(A.st[size_t(r - 1)]);
      i.sb[5] = i32(B.st[size_t(r - 2)]), i.sb[6] = i32(B.st[size_t(r - 1)]);
      i.a_iter = A.it_step;
      i.b_iter = B.it_step;
      const int64_t n = Go[0] * Go[1] * Go[2] * Bi * M * N;
      if (n > INT32_MAX) throw Error(ErrCode::DoesNotFit, "VM matmul too large");
      i.n = uint32_t(n);
      const uint8_t q = bqd[size_t(ta)] & bqd[size_t(tb)];
      i.qd = q;
      bqd[size_t(to)] = q;
      if (to_acc) acc_fused[size_t(acc)] = 1;
      static const bool fp_hoist = [] {  // experiments: TPO_VM_FP_HOIST=0 keeps fp matmuls in the loop
        const char *e = std::getenv("TPO_VM_FP_HOIST");
        return !(e && e[0] == '0');
      }();
      if ((field_ || fp_hoist) && to_acc && bg.forloop > 1 && int64_t(i.a_iter) == K * i.sa[5] &&
          int64_t(i.b_iter) == K * i.sb[5] && K * bg.forloop <= INT32_MAX) {
        // both operands walk one k tile per iteration: the loop is just the
        // continuation of the k sum — one Matmul over K·forloop after it.
        // Field sums reassociate freely; fp keeps the reference's order:
        // each iteration's K-segment sum is added to the accumulator in
        // iteration order (kseg, kernels/vm.h)
        i.dims[5] = uint32_t(K * bg.forloop);
        i.a_iter = i.b_iter = 0;
        if (!field_) i.kseg = uint32_t(K);
        hoisted.push_back(i);
        return;
      }
      emit(i);
    };

    auto run_compute = [&](const Op &b) {
      std::vector<uint32_t> ins;
      std::vector<TensorShape> shapes;
      std::vector<uint8_t> qds, invs, pres;
      bool any_pre = false;
      for (TensorId t : b.inputs) {
        const TensorId src = pre_sub[size_t(t)] ? pre_src[size_t(t)] : t;  // chained unary: its input
        ins.push_back(bget(src));
        shapes.push_back(bshape(src));
        qds.push_back(bqd[size_t(src)]);  // Sqr / Sqrt / SiLU keep q-definedness
        invs.push_back(binv[size_t(src)]);
        pres.push_back(pre_sub[size_t(t)]);
        any_pre = any_pre || pre_sub[size_t(t)];
      }
      TensorId o = b.outputs.at(0);
      bqd[size_t(o)] = compute(b, ins, shapes, qds, invs, bbuf[size_t(o)], bshape(o), G, any_pre ? &pres : nullptr);
    };

    // Emission order: the depth schedule (SPEC schedule_ops, tpo/ir/schedule.hpp)
    // groups independent ops of one level next to each other, so that
    // mark_phases can drop the barriers between them.  Only data dependences
    // order pure ops, so the results are those of the reference's list order;
    // OutSavers keep their list order (OutSaver #k -> output k).
    std::vector<const Op *> sched_ops;
    {
      static const bool keep = [] {
        const char *e = std::getenv("TPO_VM_SCHED");
        return e && e[0] == '0';
      }();
      if (keep || list_order_) {
        for (const Op &b : bg.ops) sched_ops.push_back(&b);
      } else {
        for (int k : schedule_ops(bg).order) sched_ops.push_back(&bg.ops[size_t(k)]);
      }
    }

    // ---- loop body (eval_core.hpp:303-341)
    {
      TpoVmInstr L;
      std::memset(&L, 0, sizeof(L));
      L.op = VM_LOOP;
      L.n = uint32_t(bg.forloop);
      emit(L);
    }
    for (const Op *bp : sched_ops) {
      const Op &b = *bp;
      if (b.type == OpType::InIter) {
        const auto &a = std::get<InIterAttrs>(b.attrs);
        if (a.operand < 0 || size_t(a.operand) >= op.inputs.size())
          throw Error(ErrCode::ShapeMismatch, "initer operand range");
        TensorId src = op.inputs[size_t(a.operand)], o = b.outputs[0];
        const TensorShape &dev = g_.tensor(src).shape;
        const TensorShape &tile = bshape(o);
        if (tile.rank() != dev.rank()) throw Error(ErrCode::ShapeMismatch, "initer rank");
        const bool inv = binv[size_t(o)];
        const std::array<int64_t, 3> Go = inv ? std::array<int64_t, 3>{1, 1, 1} : G;
        auto ds = contiguous(dev.dims);
        View v;
        std::vector<int64_t> d_g;
        grid_part(Go, numel(tile), false, v.dims, d_g);
        std::vector<int64_t> a_g(3, 0);
        std::vector<int64_t> part = dev.dims;  // dims after the imap division
        for (int ax = 0; ax < a.imap.axes() && ax < 3; ++ax) {
          int t = a.imap.targets[size_t(ax)];
          if (t == kReplica) continue;
          if (t < 0 || t >= dev.rank()) throw Error(ErrCode::ShapeMismatch, "imap target");
          part[size_t(t)] /= G[size_t(ax)];
          a_g[size_t(ax)] = inv ? 0 : part[size_t(t)] * ds[size_t(t)];
        }
        int ft = a.fmap.axes() ? a.fmap.targets[0] : kReplica;
        int32_t it_step = 0;
        if (ft != kReplica) {
          if (ft < 0 || ft >= dev.rank()) throw Error(ErrCode::ShapeMismatch, "fmap target");
          it_step = i32((part[size_t(ft)] / bg.forloop) * ds[size_t(ft)]);
        }
        if (concat_src[size_t(o)]) {  // feeds a concat-Accum view: the accumulator is a view
          const Op *acc_op = cons[size_t(o)][0];
          const TensorId acc = acc_op->outputs[0];
          Operand w;
          w.base = buf(src);
          for (int k = 0; k < 3; ++k) w.g[k] = a_g[size_t(k)];
          w.dims = bshape(acc).dims;
          w.st = ds;
          w.it_step = 0;
          views[size_t(acc)] = w;
          is_view[size_t(acc)] = 1;
          bqd[size_t(o)] = kqd_[size_t(src)];
          continue;
        }
        if (is_view[size_t(o)]) {  // read in place by its Matmul consumers
          Operand w;
          w.base = buf(src);
          for (int k = 0; k < 3; ++k) w.g[k] = a_g[size_t(k)];
          w.dims = tile.dims;
          w.st = ds;
          w.it_step = it_step;
          views[size_t(o)] = w;
          bqd[size_t(o)] = kqd_[size_t(src)];
          continue;
        }
        v.dims = cat(v.dims, tile.dims);
        v.st = {cat(d_g, contiguous(tile.dims)), cat(a_g, ds)};
        v.wm.assign(v.dims.size(), 0);
        TpoVmInstr i = make(VM_COPY, 0, v, bbuf[size_t(o)], buf(src), 0);
        i.a_iter = it_step;
        i.qd = kqd_[size_t(src)];
        bqd[size_t(o)] = i.qd;
        emit(i);
        continue;
      }
      if (b.type == OpType::Accum) {
        const auto &a = std::get<AccumAttrs>(b.attrs);
        TensorId val = b.inputs.at(0), acc = b.outputs[0];
        const TensorShape &vs = bshape(val);
        int t = a.fmap.axes() ? a.fmap.targets[0] : kReplica;
        if (t == kReplica && acc_fused[size_t(acc)]) {
          // already accumulated by the producing Matmul (VM_ACCUM)
        } else if (t != kReplica && concat_view[size_t(acc)]) {
          // a view of the kernel input (see concat_view)
        } else if (t == kReplica) {
          View v;
          v.dims = {copies(val) * numel(vs)};
          v.st = {{1}, {1}, {1}};
          v.wm = {0};
          TpoVmInstr i = make(VM_BINARY, VM_ADD, v, bbuf[size_t(acc)], bbuf[size_t(acc)], bget(val));
          i.qd = bqd[size_t(val)];
          i.flags |= VM_A_QD | (bqd[size_t(val)] ? VM_B_QD : 0);
          emit(i);
        } else {
          const TensorShape &as = bshape(acc);
          const std::array<int64_t, 3> Go =
              binv[size_t(val)] ? std::array<int64_t, 3>{1, 1, 1} : G;
          View v;
          std::vector<int64_t> d_g, a_g;
          grid_part(Go, numel(as), false, v.dims, d_g);
          grid_part(Go, numel(vs), false, v.dims, a_g);
          auto cs_acc = contiguous(as.dims);
          v.dims = cat(v.dims, vs.dims);
          v.st = {cat(d_g, cs_acc), cat(a_g, contiguous(vs.dims))};
          v.wm.assign(v.dims.size(), 0);
          TpoVmInstr i = make(VM_COPY, 0, v, bbuf[size_t(acc)], bget(val), 0);
          i.d_iter = i32(vs.dims[size_t(t)] * cs_acc[size_t(t)]);
          i.qd = bqd[size_t(val)];
          emit(i);
        }
        bqd[size_t(acc)] = bqd[size_t(val)];
        continue;
      }
      if (b.type == OpType::OutSaver || is_post(b) || chained(b)) continue;
      if (matmul_fusable(b)) {
        emit_strided_matmul(b);
        continue;
      }
      run_compute(b);
    }
    {
      TpoVmInstr E;
      std::memset(&E, 0, sizeof(E));
      E.op = VM_ENDLOOP;
      emit(E);
    }
    for (const TpoVmInstr &h : hoisted) emit(h);

    // ---- post-loop ops and OutSavers (eval_core.hpp:348-375)
    size_t saver = 0;
    for (const Op *bp : sched_ops) {
      const Op &b = *bp;
      if (b.type == OpType::OutSaver) {
        if (saver >= op.outputs.size()) throw Error(ErrCode::ShapeMismatch, "outsaver count");
        const auto &a = std::get<OutSaverAttrs>(b.attrs);
        TensorId val = b.inputs.at(0), out = op.outputs[saver++];
        const TensorShape &vs = bshape(val), &os = g_.tensor(out).shape;
        if (vs.rank() != os.rank()) throw Error(ErrCode::ShapeMismatch, "outsaver rank");
        auto ods = contiguous(os.dims);
        View v;
        std::vector<int64_t> a_g;
        grid_part(G, numel(vs), binv[size_t(val)], v.dims, a_g);
        std::vector<int64_t> d_g(3, 0);
        v.wm.assign(3, 0);
        for (int ax = 0; ax < 3; ++ax) {
          if (ax < a.omap.axes()) {
            int t = a.omap.targets[size_t(ax)];
            if (t == kReplica || t < 0 || t >= vs.rank())
              throw Error(ErrCode::ReplicaInOmap, "omap target");
            d_g[size_t(ax)] = vs.dims[size_t(t)] * ods[size_t(t)];
          } else if (G[size_t(ax)] > 1) {
            v.wm[size_t(ax)] = 1;  // last block along this axis wins
          }
        }
        v.dims = cat(v.dims, vs.dims);
        v.wm.resize(v.dims.size(), 0);
        v.st = {cat(d_g, ods), cat(a_g, contiguous(vs.dims))};
        TpoVmInstr i = make(VM_COPY, 0, v, kbuf_[size_t(out)], bget(val), 0);
        i.qd = bqd[size_t(val)];
        kqd_[size_t(out)] = i.qd;
        emit(i);
        continue;
      }
      if (b.type == OpType::InIter || b.type == OpType::Accum || !is_post(b) || chained(b)) continue;
      if (matmul_fusable(b)) {
        emit_strided_matmul(b);
        continue;
      }
      run_compute(b);
    }
  }
};

}  // namespace

VmProgram lower_vm(const KernelGraph &g, uint32_t input_base, uint32_t region_base,
                   bool pin_outputs, bool field) {
  VmProgram p = Lowerer(g, input_base, region_base, pin_outputs, field).run();
  // a raising graph keeps the reference's list order, so that exactly the
  // ops evaluated before the raising EwExp precede the VM_RAISE
  if (field && p.poisoned) p = Lowerer(g, input_base, region_base, pin_outputs, field, true).run();
  return p;
}

int64_t input_elems(const KernelGraph &g) {
  int64_t n = 0;
  for (TensorId t : g.inputs) n += numel(g.tensor(t).shape);
  return n;
}

// Reference work counter (shape_infer.cpp:195-217) summed over the graph,
// block ops scaled by the grid and, for in-loop ops, the for-loop trip count.
int64_t graph_madds(const KernelGraph &g) {
  int64_t total = 0;
  for (const Op &op : g.ops) {
    if (op.type != OpType::GraphDef) {
      std::vector<TensorShape> in;
      for (TensorId t : op.inputs) in.push_back(g.tensor(t).shape);
      total += op_madds(op.type, op.attrs, in, g.tensor(op.outputs[0]).shape);
      continue;
    }
    const BlockGraph &bg = *op.block;
    std::vector<char> post(bg.tensors.size(), 0);
    for (const Op &b : bg.ops) {
      if (b.type == OpType::Accum) {
        post[size_t(b.outputs[0])] = 1;
        continue;
      }
      if (b.type == OpType::InIter || b.type == OpType::OutSaver) continue;
      for (TensorId t : b.inputs)
        if (post[size_t(t)]) post[size_t(b.outputs[0])] = 1;
    }
    for (const Op &b : bg.ops) {
      if (b.type == OpType::InIter || b.type == OpType::OutSaver) continue;
      std::vector<TensorShape> in;
      for (TensorId t : b.inputs) in.push_back(bg.tensor(t).shape);
      int64_t m = op_madds(b.type, b.attrs, in, bg.tensor(b.outputs[0]).shape);
      bool p = b.type != OpType::Accum && post[size_t(b.outputs[0])];
      total += m * bg.grid_product() * (p ? 1 : bg.forloop);
    }
  }
  return total;
}

}  // namespace tpo::gpu
