// Reference-side binding of the B200 backend — see tpo_gpu_backend.hpp.
#include "tpo_gpu_backend.hpp"

#include <algorithm>
#include <string>
#include <thread>

#include "tpo/ir/serialize.hpp"

namespace tpo::gpu {

namespace {

// C-ABI status -> the reference's exception (shape.hpp:27-50).
void check(int rc) {
  if (rc == 0) return;
  const char *msg = tpo_gpu_last_error();
  if (rc >= 1000 && rc < 2000) throw Error(ErrCode(rc - 1000), msg ? msg : "");
  throw Error(ErrCode::Unsupported, std::string("tpo_gpu status ") + std::to_string(rc) + ": " +
                                        (msg ? msg : ""));
}

tpo_field_params field(const verify::FieldParams &fp) {
  return tpo_field_params{fp.p(), fp.q(), fp.omega_base()};
}

verify::EquivVerdict to_verdict(const tpo_verdict &v) {
  if (v.kind == 3) throw Error(ErrCode(v.err_code - 1000), tpo_gpu_last_error());
  verify::EquivVerdict r;
  r.kind = verify::EquivVerdict::Kind(v.kind);
  r.rounds_run = v.rounds_run;
  r.resamples = v.resamples;
  if (v.has_witness) r.witness = verify::Witness{v.w_seed, v.w_round, v.w_omega, v.w_tensor, v.w_index};
  return r;
}

}  // namespace

CompiledGraph::CompiledGraph(tpo_gpu_ctx *ctx, const ir::KernelGraph &g) {
  const std::string js = ir::to_json(g).dump();
  check(tpo_gpu_compile(ctx, js.c_str(), &h_));
}

CompiledGraph::~CompiledGraph() {
  if (h_) tpo_gpu_graph_free(h_);
}

int64_t CompiledGraph::op_madds() const { return tpo_gpu_op_madds(h_); }

bool CompiledGraph::has_fused_kernel() const {
  tpo_graph_info info{};
  tpo_gpu_graph_info(h_, &info);
  return info.fused_kind != TPO_FUSED_NONE;
}

Backend::Backend(int device) { check(tpo_gpu_open(device, &ctx_)); }

Backend::~Backend() {
  if (ctx_) tpo_gpu_close(ctx_);
}

std::vector<interp::FTensor> Backend::eval_mugraph(const ir::KernelGraph &g,
                                                   const std::vector<interp::FTensor> &inputs,
                                                   int precision) {
  if (inputs.size() != g.inputs.size()) throw Error(ErrCode::ShapeMismatch, "input count");
  CompiledGraph cg(ctx_, g);
  check(tpo_gpu_graph_set_precision(cg.handle(), precision));
  std::vector<const double *> pin(inputs.size());
  for (size_t i = 0; i < inputs.size(); ++i) {
    if (inputs[i].shape.dims != g.tensor(g.inputs[i]).shape.dims)
      throw Error(ErrCode::ShapeMismatch, "input tensor shape");
    pin[i] = inputs[i].data.data();
  }
  std::vector<interp::FTensor> out;
  std::vector<double *> pout(g.outputs.size());
  for (size_t o = 0; o < g.outputs.size(); ++o) out.emplace_back(g.tensor(g.outputs[o]).shape);
  for (size_t o = 0; o < g.outputs.size(); ++o) pout[o] = out[o].data.data();
  check(tpo_gpu_eval_mugraph_f64(ctx_, cg.handle(), pin.data(), pout.data(), nullptr));
  return out;
}

verify::EquivVerdict Backend::random_test_equivalence(const ir::KernelGraph &g1,
                                                      const ir::KernelGraph &g2,
                                                      const verify::VerifyConfig &cfg,
                                                      const verify::FieldParams &fp) {
  CompiledGraph a(ctx_, g1), b(ctx_, g2);
  const tpo_verify_cfg c{cfg.num_tests, cfg.max_resamples, cfg.seed, cfg.float_tolerance};
  const tpo_field_params f = field(fp);
  tpo_verdict v{};
  const int rc = tpo_gpu_random_test_equivalence(ctx_, a.handle(), b.handle(), &c, &f, &v);
  if (rc && v.kind != 3) check(rc);
  return to_verdict(v);
}

std::vector<verify::EquivVerdict> Backend::verify_batch(
    const ir::KernelGraph &program, const std::vector<const ir::KernelGraph *> &cands,
    const std::vector<uint64_t> &seeds, const verify::VerifyConfig &cfg,
    const verify::FieldParams &fp) {
  if (seeds.size() != cands.size()) throw Error(ErrCode::ShapeMismatch, "one seed per candidate");
  CompiledGraph prog(ctx_, program);
  // the candidate stream: wire format on all host cores, then one parallel
  // compile (tpo_gpu_compile_many); a candidate that does not compile
  // rethrows its tpo::Error, as the CPU path would on that candidate
  const size_t n = cands.size();
  std::vector<std::string> js(n);
  {
    const size_t nt = std::max<size_t>(1, std::min<size_t>(std::thread::hardware_concurrency(), n / 64 + 1));
    std::vector<std::thread> pool;
    for (size_t t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        for (size_t i = t; i < n; i += nt) js[i] = ir::to_json(*cands[i]).dump();
      });
    for (auto &th : pool) th.join();
  }
  std::vector<const char *> jp(n);
  for (size_t i = 0; i < n; ++i) jp[i] = js[i].c_str();
  std::vector<tpo_gpu_graph *> raw(n, nullptr);
  std::vector<int32_t> st(n, 0);
  check(tpo_gpu_compile_many(ctx_, jp.data(), int64_t(n), 0, raw.data(), st.data()));
  std::vector<std::unique_ptr<CompiledGraph>> owned;
  std::vector<const tpo_gpu_graph *> hs;
  for (size_t i = 0; i < n; ++i) owned.push_back(std::make_unique<CompiledGraph>(raw[i]));
  for (size_t i = 0; i < n; ++i) {
    check(st[i]);
    hs.push_back(raw[i]);
  }
  const tpo_verify_cfg c{cfg.num_tests, cfg.max_resamples, cfg.seed, cfg.float_tolerance};
  const tpo_field_params f = field(fp);
  std::vector<tpo_verdict> v(cands.size());
  check(tpo_gpu_verify_batch(ctx_, prog.handle(), hs.data(), seeds.data(), uint64_t(cands.size()), &c,
                             &f, v.data(), nullptr));
  std::vector<verify::EquivVerdict> out;
  out.reserve(v.size());
  for (const tpo_verdict &x : v) out.push_back(to_verdict(x));  // kind 3 rethrows the tpo::Error
  return out;
}

}  // namespace tpo::gpu
