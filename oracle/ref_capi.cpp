// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C shim over the *unmodified* reference ("tpo" core, compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/).  Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg load this library, and only as the checker or the CPU
// baseline.  Each entry point is a thin adapter around one reference call:
//
//   ref_eval_mugraph      -> tpo::interp::eval_mugraph / eval_mugraph_f32 /
//                            eval_program           (interp.hpp:41-53)
//   ref_ff_attempt        -> one attempt of random_test_equivalence's inner
//                            loop (equiv.cpp:57-68): derive, sample_inputs,
//                            sample_omega, SiluTables::sample, ff_eval
//   ref_random_test_equivalence -> tpo::verify::random_test_equivalence
//                            (equiv.hpp:50-53)
//   ref_verify_batch      -> the same call over a candidate pool on a
//                            std::thread pool (the call is pure)
//   ref_float_stability_filter -> tpo::verify::float_stability_filter
//   ref_validate / ref_op_madds / ref_canonical_key -> ir helpers
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tpo/interp/interp.hpp"
#include "tpo/ir/serialize.hpp"
#include "tpo/ir/shape_infer.hpp"
#include "tpo/ir/validate.hpp"
#include "tpo/util/rng.hpp"
#include "tpo/verify/equiv.hpp"
#include "tpo/verify/ffeval.hpp"
#include "tpo/verify/field.hpp"
#include "tpo/verify/stability.hpp"

using namespace tpo;

namespace {
thread_local std::string g_err;

int fail_code(const Error &e) {
  g_err = e.what();
  return 1000 + int(e.code);
}

ir::KernelGraph parse(const char *json) {
  try {
    return ir::kernel_graph_from_json(nlohmann::json::parse(json));
  } catch (const nlohmann::json::exception &e) {
    throw Error(ErrCode::ParseError, e.what());
  }
}

bool graph_has_silu(const ir::KernelGraph &g) {
  for (const ir::Op &op : g.ops) {
    if (op.type == ir::OpType::SiLU) return true;
    if (op.block)
      for (const ir::Op &bop : op.block->ops)
        if (bop.type == ir::OpType::SiLU) return true;
  }
  return false;
}
}  // namespace

extern "C" {

// Verdict record shared with the product ABI layout (see include/tpo_gpu.h).
struct ref_verdict {
  int32_t kind;  // 0 Equivalent, 1 NotEquivalent, 2 Inconclusive, 3 Error
  int32_t rounds_run;
  int32_t resamples;
  int32_t has_witness;
  uint64_t w_seed;
  int32_t w_round;
  uint32_t w_omega;
  int32_t w_tensor;
  int32_t err_code;  // 1000 + ErrCode when kind == 3
  int64_t w_index;
};

const char *ref_last_error() { return g_err.c_str(); }

int ref_abi_version() { return 1; }

// splitmix64 stream: n draws of Rng(seed) (derive==1 -> Rng::derive(seed, stream)).
void ref_rng_draws(uint64_t seed, uint64_t stream, int derive, int n, uint64_t *out) {
  Rng r = derive ? Rng::derive(seed, stream) : Rng(seed);
  for (int i = 0; i < n; ++i) out[i] = r.next();
}

void ref_rng_normals(uint64_t seed, uint64_t stream, int n, double *out) {
  Rng r = Rng::derive(seed, stream);
  for (int i = 0; i < n; ++i) out[i] = r.normal();
}

// Field tables: inv_p[p], inv_q[q], sqrt_p[p], sqrt_q[q].
int ref_field_tables(uint32_t p, uint32_t q, uint32_t wbase, uint32_t *inv_p, uint32_t *inv_q,
                     int32_t *sqrt_p, int32_t *sqrt_q) {
  try {
    verify::FieldParams fp(p, q, wbase);
    for (uint32_t x = 0; x < p; ++x) inv_p[x] = fp.inv_p(x), sqrt_p[x] = fp.sqrt_p(x);
    for (uint32_t x = 0; x < q; ++x) inv_q[x] = fp.inv_q(x), sqrt_q[x] = fp.sqrt_q(x);
    return 0;
  } catch (const Error &e) {
    return fail_code(e);
  }
}

// Scalar field op for exhaustive checks: op 0 add 1 sub 2 mul 3 div 4 exp 5 sqrt.
// Returns 0, 2000+ErrCode for ResampleNeeded, 1000+ErrCode for Error.
int ref_field_op(uint32_t p, uint32_t q, uint32_t wbase, int op, uint32_t omega,
                 const uint16_t *a, const uint16_t *b, uint16_t *r) {
  verify::FieldParams fp(p, q, wbase);
  verify::FFValue x{a[0], a[1], a[2] != 0}, y{b[0], b[1], b[2] != 0}, z;
  try {
    switch (op) {
      case 0: z = fp.add(x, y); break;
      case 1: z = fp.sub(x, y); break;
      case 2: z = fp.mul(x, y); break;
      case 3: z = fp.div(x, y); break;
      case 4: z = fp.exp(x, omega); break;
      case 5: z = fp.sqrt(x); break;
      default: return -1;
    }
  } catch (const verify::ResampleNeeded &rn) {
    return 2000 + int(rn.code);
  } catch (const Error &e) {
    return fail_code(e);
  }
  r[0] = z.xp;
  r[1] = z.xq;
  r[2] = z.q_defined;
  return 0;
}

// Float evaluation. mode 0 eval_mugraph (double), 1 eval_program, 2 eval_mugraph_f32.
// Inputs/outputs are flat row-major double arrays in graph input/output order.
int ref_eval_mugraph(const char *json, int mode, const double *const *inputs,
                     double *const *outputs) {
  try {
    ir::KernelGraph g = parse(json);
    if (mode == 2) {
      std::vector<interp::F32Tensor> in;
      for (size_t i = 0; i < g.inputs.size(); ++i) {
        interp::F32Tensor t(g.tensor(g.inputs[i]).shape);
        for (size_t k = 0; k < t.data.size(); ++k) t.data[k] = float(inputs[i][k]);
        in.push_back(std::move(t));
      }
      auto out = interp::eval_mugraph_f32(g, in);
      for (size_t i = 0; i < out.size(); ++i)
        for (size_t k = 0; k < out[i].data.size(); ++k) outputs[i][k] = out[i].data[k];
      return 0;
    }
    std::vector<interp::FTensor> in;
    for (size_t i = 0; i < g.inputs.size(); ++i) {
      interp::FTensor t(g.tensor(g.inputs[i]).shape);
      std::memcpy(t.data.data(), inputs[i], t.data.size() * sizeof(double));
      in.push_back(std::move(t));
    }
    auto out = mode == 1 ? interp::eval_program(g, in) : interp::eval_mugraph(g, in);
    for (size_t i = 0; i < out.size(); ++i)
      std::memcpy(outputs[i], out[i].data.data(), out[i].data.size() * sizeof(double));
    return 0;
  } catch (const Error &e) {
    return fail_code(e);
  }
}

// Wall-clock milliseconds of `reps` eval_mugraph calls on the given inputs
// (parse and input marshalling outside the timed region).
double ref_time_eval_mugraph(const char *json, const double *const *inputs, int reps) {
  ir::KernelGraph g = parse(json);
  std::vector<interp::FTensor> in;
  for (size_t i = 0; i < g.inputs.size(); ++i) {
    interp::FTensor t(g.tensor(g.inputs[i]).shape);
    std::memcpy(t.data.data(), inputs[i], t.data.size() * sizeof(double));
    in.push_back(std::move(t));
  }
  auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) {
    auto out = interp::eval_mugraph(g, in);
    (void)out;
  }
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(t1 - t0).count();
}

// Time `reps` eval_mugraph calls per thread on `threads` graphs concurrently
// (each thread its own graph + inputs). Returns wall ms of the slowest thread.
double ref_time_eval_parallel(const char *const *jsons, const double *const *const *inputs,
                              int threads, int reps) {
  std::vector<ir::KernelGraph> gs;
  std::vector<std::vector<interp::FTensor>> ins; ins.resize(size_t(threads));
  for (int t = 0; t < threads; ++t) {
    gs.push_back(parse(jsons[t]));
    const ir::KernelGraph &g = gs.back();
    for (size_t i = 0; i < g.inputs.size(); ++i) {
      interp::FTensor x(g.tensor(g.inputs[i]).shape);
      std::memcpy(x.data.data(), inputs[t][i], x.data.size() * sizeof(double));
      ins[size_t(t)].push_back(std::move(x));
    }
  }
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      for (int r = 0; r < reps; ++r) {
        auto out = interp::eval_mugraph(gs[size_t(t)], ins[size_t(t)]);
        (void)out;
      }
    });
  for (auto &th : pool) th.join();
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(t1 - t0).count();
}

// One verifier attempt exactly as equiv.cpp:57-68 performs it for graph g:
// rng = derive(seed, stream); inputs; omega; SiLU tables iff with_silu.
// Writes FF outputs (xp, xq, q_defined planes, concatenated over outputs),
// sampled inputs (xp, xq planes, concatenated) and omega.
// Returns 0, 2000+code on ResampleNeeded, 1000+code on Error.
int ref_ff_attempt(const char *json, uint32_t p, uint32_t q, uint32_t wbase, uint64_t seed,
                   uint64_t stream, int with_silu, uint16_t *in_xp, uint16_t *in_xq,
                   uint16_t *out_xp, uint16_t *out_xq, uint8_t *out_qd, uint32_t *omega_out) {
  try {
    ir::KernelGraph g = parse(json);
    verify::FieldParams fp(p, q, wbase);
    std::vector<ir::TensorShape> shapes;
    for (ir::TensorId t : g.inputs) shapes.push_back(g.tensor(t).shape);
    Rng rng = Rng::derive(seed, stream);
    auto inputs = verify::sample_inputs(fp, shapes, rng);
    uint32_t omega = fp.sample_omega(rng);
    *omega_out = omega;
    verify::SiluTables tables;
    const verify::SiluTables *tp = nullptr;
    if (with_silu) {
      tables = verify::SiluTables::sample(fp, rng);
      tp = &tables;
    }
    size_t c = 0;
    for (const auto &t : inputs)
      for (const auto &v : t.data) {
        if (in_xp) in_xp[c] = v.xp;
        if (in_xq) in_xq[c] = v.xq;
        ++c;
      }
    std::vector<verify::FFTensor> out;
    try {
      out = verify::ff_eval(g, inputs, fp, omega, tp);
    } catch (const verify::ResampleNeeded &rn) {
      return 2000 + int(rn.code);
    }
    c = 0;
    for (const auto &t : out)
      for (const auto &v : t.data) {
        out_xp[c] = v.xp;
        out_xq[c] = v.xq;
        out_qd[c] = v.q_defined;
        ++c;
      }
    return 0;
  } catch (const Error &e) {
    return fail_code(e);
  }
}

static void fill_verdict(const verify::EquivVerdict &v, ref_verdict *o) {
  std::memset(o, 0, sizeof(*o));
  o->kind = int32_t(v.kind);
  o->rounds_run = v.rounds_run;
  o->resamples = v.resamples;
  if (v.witness) {
    o->has_witness = 1;
    o->w_seed = v.witness->seed;
    o->w_round = v.witness->round;
    o->w_omega = v.witness->omega;
    o->w_tensor = v.witness->tensor;
    o->w_index = v.witness->index;
  }
}

int ref_random_test_equivalence(const char *j1, const char *j2, int num_tests, uint64_t seed,
                                int max_resamples, uint32_t p, uint32_t q, uint32_t wbase,
                                ref_verdict *out) {
  try {
    ir::KernelGraph g1 = parse(j1), g2 = parse(j2);
    verify::VerifyConfig cfg;
    cfg.num_tests = num_tests;
    cfg.seed = seed;
    cfg.max_resamples = max_resamples;
    verify::FieldParams fp(p, q, wbase);
    fill_verdict(verify::random_test_equivalence(g1, g2, cfg, fp), out);
    return 0;
  } catch (const Error &e) {
    std::memset(out, 0, sizeof(*out));
    out->kind = 3;
    out->err_code = fail_code(e);
    return out->err_code;
  }
}

// Candidate i (i in [first, first+n)) = pool[i % pool_n] verified against
// `program` with cfg {num_tests, seed = i, max_resamples}.  `threads` workers
// pull indices from an atomic counter.  Returns wall milliseconds.
double ref_verify_batch(const char *program, const char *const *pool, int pool_n,
                        uint64_t first, uint64_t n, int num_tests, int max_resamples,
                        uint32_t p, uint32_t q, uint32_t wbase, int threads,
                        ref_verdict *out) {
  ir::KernelGraph prog = parse(program);
  std::vector<ir::KernelGraph> cands;
  for (int i = 0; i < pool_n; ++i) cands.push_back(parse(pool[i]));
  verify::FieldParams fp(p, q, wbase);
  std::atomic<uint64_t> next{0};
  auto t0 = std::chrono::steady_clock::now();
  auto work = [&] {
    for (;;) {
      uint64_t k = next.fetch_add(1);
      if (k >= n) return;
      uint64_t i = first + k;
      verify::VerifyConfig cfg;
      cfg.num_tests = num_tests;
      cfg.seed = i;
      cfg.max_resamples = max_resamples;
      ref_verdict *o = out ? out + k : nullptr;
      try {
        auto v = verify::random_test_equivalence(prog, cands[size_t(i % uint64_t(pool_n))], cfg, fp);
        if (o) fill_verdict(v, o);
      } catch (const Error &e) {
        if (o) {
          std::memset(o, 0, sizeof(*o));
          o->kind = 3;
          o->err_code = 1000 + int(e.code);
        }
      }
    }
  };
  std::vector<std::thread> pool_t;
  for (int t = 0; t < threads; ++t) pool_t.emplace_back(work);
  for (auto &th : pool_t) th.join();
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(t1 - t0).count();
}

int ref_float_stability_filter(const char *g_json, const char *prog_json, int trials,
                               double tol, uint64_t seed, double scale) {
  try {
    ir::KernelGraph g = parse(g_json), prog = parse(prog_json);
    return verify::float_stability_filter(g, prog, trials, tol, seed, scale) ? 1 : 0;
  } catch (const Error &e) {
    return -fail_code(e);
  }
}

// Number of violations of validate(g, {smem_bytes, reg_elems, elem_size}); -code on parse error.
int ref_validate(const char *json, int64_t smem_bytes, int64_t elem_size) {
  try {
    ir::KernelGraph g = parse(json);
    ir::MemLimits lim;
    lim.smem_bytes = smem_bytes;
    lim.elem_size = elem_size;
    auto rep = ir::validate(g, lim);
    g_err.clear();
    for (auto &v : rep.violations) g_err += v.detail + "; ";
    return int(rep.violations.size());
  } catch (const Error &e) {
    return -fail_code(e);
  }
}

int64_t ref_block_shared_bytes(const char *json, int op_index, int64_t elem_size) {
  ir::KernelGraph g = parse(json);
  return ir::block_shared_bytes(*g.ops[size_t(op_index)].block, elem_size);
}

// Reference work counter: sum of op_madds over kernel ops, with GraphDef
// block ops scaled by grid product (and forloop for in-loop ops), as SURVEY
// §8d defines the verifier's algorithmic unit.
int64_t ref_op_madds(const char *json) {
  ir::KernelGraph g = parse(json);
  int64_t total = 0;
  for (const ir::Op &op : g.ops) {
    if (op.type != ir::OpType::GraphDef) {
      std::vector<ir::TensorShape> ins;
      for (auto t : op.inputs) ins.push_back(g.tensor(t).shape);
      total += ir::op_madds(op.type, op.attrs, ins, g.tensor(op.outputs[0]).shape);
      continue;
    }
    const ir::BlockGraph &bg = *op.block;
    std::vector<bool> post(bg.tensors.size(), false);
    for (const ir::Op &bop : bg.ops) {
      if (bop.type == ir::OpType::Accum) {
        post[size_t(bop.outputs[0])] = true;
        continue;
      }
      if (bop.type == ir::OpType::InIter || bop.type == ir::OpType::OutSaver) continue;
      for (auto t : bop.inputs)
        if (post[size_t(t)]) post[size_t(bop.outputs[0])] = true;
    }
    for (const ir::Op &bop : bg.ops) {
      if (bop.type == ir::OpType::InIter || bop.type == ir::OpType::OutSaver) continue;
      std::vector<ir::TensorShape> ins;
      for (auto t : bop.inputs) ins.push_back(bg.tensor(t).shape);
      int64_t m = ir::op_madds(bop.type, bop.attrs, ins, bg.tensor(bop.outputs[0]).shape);
      bool is_post = bop.type != ir::OpType::Accum && post[size_t(bop.outputs[0])];
      total += m * bg.grid_product() * (is_post ? 1 : bg.forloop);
    }
  }
  return total;
}

// canonical_key into buf (returns required length).
int ref_canonical_key(const char *json, char *buf, int cap) {
  std::string k = ir::canonical_key(parse(json));
  if (buf && cap > 0) {
    std::strncpy(buf, k.c_str(), size_t(cap - 1));
    buf[cap - 1] = 0;
  }
  return int(k.size()) + 1;
}

// JSON round trip through the reference's serializer (for wire-format tests).
int ref_roundtrip_json(const char *json, char *buf, int cap) {
  std::string s = ir::to_json(parse(json)).dump();
  if (buf && cap > 0) {
    std::strncpy(buf, s.c_str(), size_t(cap - 1));
    buf[cap - 1] = 0;
  }
  return int(s.size()) + 1;
}

}  // extern "C"
