// B200 backend — C-ABI (include/tpo_gpu.h) over the host runtime.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../../include/tpo_gpu.h"
#include "runtime.hpp"
#include "tpo/ir/enumerate.hpp"
#include "tpo/ir/serialize.hpp"
#include "tpo/ir/shape_infer.hpp"
#include "tpo/ir/validate.hpp"

struct tpo_gpu_ctx {
  tpo::gpu::Ctx c;
};
struct tpo_gpu_graph {
  tpo::gpu::Graph g;
};

namespace tpo::gpu {

namespace {
thread_local std::string g_last;

int fail(int code, const std::string &msg) {
  g_last = msg;
  return code;
}

template <class F>
int guard(F &&f) {
  try {
    return f();
  } catch (const Error &e) {
    return fail(1000 + int(e.code), e.what());
  } catch (const std::exception &e) {
    return fail(1000 + int(ErrCode::Unsupported), e.what());
  }
}

int host_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return int(std::max(1u, std::min(h ? h : 1u, 64u)));
}

// fn(i) for i in [0, n) over `threads` host threads (atomic work counter)
template <class Fn>
void parallel_for(int64_t n, int threads, Fn &&fn) {
  if (threads <= 1 || n < 2) {
    for (int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int64_t> next{0};
  auto work = [&] {
    for (int64_t i; (i = next.fetch_add(1)) < n;) fn(i);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work);
  work();
  for (auto &t : pool) t.join();
}

bool is_prime(uint32_t n) {
  if (n < 2) return false;
  for (uint32_t d = 2; d * d <= n; ++d)
    if (n % d == 0) return false;
  return true;
}

uint32_t pow_mod(uint64_t b, uint64_t e, uint32_t m) {
  uint64_t r = 1;
  b %= m;
  while (e) {
    if (e & 1) r = r * b % m;
    b = b * b % m;
    e >>= 1;
  }
  return uint32_t(r);
}
}  // namespace

void check_cuda(cudaError_t e, const char *what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(ErrCode::Unsupported, std::string("CUDA ") + what + ": " + cudaGetErrorString(e));
  }
}

void *DevBuf::get(size_t bytes) {
  if (bytes > cap) {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    size_t c = std::max(bytes, cap * 2);
    c = std::max<size_t>(c, 256);
    check_cuda(cudaMalloc(&ptr, c), "cudaMalloc");
    cap = c;
  }
  return ptr;
}

DevBuf::~DevBuf() {
  if (ptr) cudaFree(ptr);
}

// FieldParams (field.cpp:43-67): same validity checks and tables, plus the
// device constants of the lazy-reduction scheme.
FieldState &Ctx::field(uint32_t p, uint32_t q, uint32_t wbase) {
  const auto key = std::make_tuple(p, q, wbase);
  auto it = fields.find(key);
  if (it != fields.end()) return *it->second;
  if (!is_prime(p) || !is_prime(q)) throw Error(ErrCode::ConfigError, "p and q must be prime");
  if ((p - 1) % q != 0) throw Error(ErrCode::ConfigError, "q must divide p-1");
  if (wbase % p == 0 || wbase % p == 1 || pow_mod(wbase, q, p) != 1)
    throw Error(ErrCode::ConfigError, "omega base must have multiplicative order q in Z_p");
  if (p > 4093) throw Error(ErrCode::Unsupported, "device field tables limited to p < 4096");
  auto fs = std::make_unique<FieldState>();
  auto &f = fs->fc;
  f.p = p;
  f.q = q;
  f.wbase = wbase;
  f.magic_p = uint32_t((1ull << 32) / p);
  f.magic_q = uint32_t((1ull << 32) / q);
  f.two32_p = uint32_t((1ull << 32) % p);
  f.two32_q = uint32_t((1ull << 32) % q);
  uint64_t pm1 = p - 1;
  f.lazy = uint32_t(std::max<uint64_t>(1, (0xFFFFFFFFull - p) / (pm1 * pm1)));
  f.lazy_sum = uint32_t(std::max<uint64_t>(1, (0xFFFFFFFFull - p) / pm1));
  f.thr_p = (0 - uint64_t(p)) % p;
  f.thr_q = (0 - uint64_t(q)) % q;
  f.k24_p = uint32_t((1ull << 24) % p);
  f.k48_p = uint32_t((1ull << 48) % p);
  f.k24_q = uint32_t((1ull << 24) % q);
  f.k48_q = uint32_t((1ull << 48) % q);
  f.small = p < 256 && q < 256;
  uint32_t tb = 2 * (5 * 0 + p + q + p + q + q) + 2 * (p + q);
  f.table_bytes = (tb + 15) & ~15u;
  auto &t = fs->host_tables;
  t.assign(2 * (p + q), 0);
  for (uint32_t x = 1; x < p; ++x) t[x] = uint16_t(pow_mod(x, p - 2, p));
  for (uint32_t x = 1; x < q; ++x) t[p + x] = uint16_t(pow_mod(x, q - 2, q));
  std::vector<int32_t> sp(p, -1), sq(q, -1);
  for (int64_t r = int64_t(p) - 1; r >= 0; --r) sp[size_t(uint64_t(r) * uint64_t(r) % p)] = int32_t(r);
  for (int64_t r = int64_t(q) - 1; r >= 0; --r) sq[size_t(uint64_t(r) * uint64_t(r) % q)] = int32_t(r);
  for (uint32_t x = 0; x < p; ++x) t[p + q + x] = uint16_t(int16_t(sp[x]));
  for (uint32_t x = 0; x < q; ++x) t[2 * p + q + x] = uint16_t(int16_t(sq[x]));
  check_cuda(cudaSetDevice(device), "cudaSetDevice");
  void *d = fs->dev.get(t.size() * 2);
  check_cuda(cudaMemcpy(d, t.data(), t.size() * 2, cudaMemcpyHostToDevice), "tables");
  auto &ref = *fs;
  fields[key] = std::move(fs);
  return ref;
}

namespace {

// A verification batch: the program plus unique candidate graphs lowered
// into one device upload.
struct Batch {
  std::vector<TpoVmInstr> code;
  std::vector<TpoVmGraph> graphs;
  uint32_t n_in = 0;
  uint32_t max_words = 0;  // words of VM memory needed
  uint32_t max_code = 0;   // program + largest candidate, instructions (staged in smem)
  uint32_t cand_base = 0;  // inputs + the program's pinned outputs (words)
};

void check_pair(const ir::KernelGraph &a, const ir::KernelGraph &b) {
  // equiv.cpp:38-49
  if (a.inputs.size() != b.inputs.size() || a.outputs.size() != b.outputs.size())
    throw Error(ErrCode::ShapeMismatch, "graph arity");
  for (size_t i = 0; i < a.inputs.size(); ++i)
    if (a.tensor(a.inputs[i]).shape != b.tensor(b.inputs[i]).shape)
      throw Error(ErrCode::ShapeMismatch, "input shapes");
  for (size_t i = 0; i < a.outputs.size(); ++i)
    if (a.tensor(a.outputs[i]).shape != b.tensor(b.outputs[i]).shape)
      throw Error(ErrCode::ShapeMismatch, "output shapes");
}

void add_graph(Batch &bt, const VmProgram &p) {
  TpoVmGraph d = p.desc;
  d.code_off = uint32_t(bt.code.size());
  d.code_len = uint32_t(p.code.size());
  bt.code.insert(bt.code.end(), p.code.begin(), p.code.end());
  bt.graphs.push_back(d);
}

TpoVmGraph error_graph(ErrCode c) {
  TpoVmGraph d;
  std::memset(&d, 0, sizeof(d));
  d.err = uint8_t(1 + int(c));
  return d;
}

// Lowers program + unique candidates; returns candidate graph index per
// unique handle in `index`.
Batch build_batch(const Graph &prog, const std::vector<const Graph *> &uniq) {
  Batch bt;
  bt.graphs.reserve(uniq.size() + 1);
  bt.n_in = uint32_t(prog.in_elems);
  // program outputs pinned right after the inputs; program scratch above
  // them is dead once the candidate starts, so the candidate region reuses it
  VmProgram pp = lowered_ff(prog, bt.n_in, /*pin_outputs=*/true);
  const uint32_t cbase = bt.n_in + pp.pinned_words;
  bt.cand_base = cbase;
  add_graph(bt, pp);
  uint32_t maxw = bt.n_in + pp.region_words;
  // lower the distinct candidates on all host cores (memoised per handle),
  // then lay the batch out by a prefix sum and copy the bytecode in parallel
  const size_t nu = uniq.size();
  const int th = nu >= 16 ? host_threads() : 1;
  std::vector<const VmProgram *> low(nu, nullptr);
  std::vector<ErrCode> err(nu, ErrCode::ShapeMismatch);
  parallel_for(int64_t(nu), th, [&](int64_t i) {
    try {
      check_pair(prog.g, uniq[size_t(i)]->g);
      low[size_t(i)] = &lowered_ff(*uniq[size_t(i)], cbase, false);
    } catch (const Error &e) {
      err[size_t(i)] = e.code;
    }
  });
  std::vector<size_t> at(nu);
  size_t ncode = bt.code.size();
  for (size_t i = 0; i < nu; ++i) {
    const VmProgram *cp = low[i];
    if (!cp) {
      bt.graphs.push_back(error_graph(err[i]));
      continue;
    }
    TpoVmGraph d = cp->desc;
    d.code_off = uint32_t(ncode);
    d.code_len = uint32_t(cp->code.size());
    bt.graphs.push_back(d);
    at[i] = ncode;
    ncode += cp->code.size();
    maxw = std::max(maxw, cbase + cp->region_words);
  }
  bt.code.resize(ncode);
  parallel_for(int64_t(nu), th, [&](int64_t i) {
    if (const VmProgram *cp = low[size_t(i)])
      std::copy(cp->code.begin(), cp->code.end(), bt.code.begin() + ptrdiff_t(at[size_t(i)]));
  });
  bt.max_words = maxw;
  uint32_t mc = 0;
  for (size_t i = 1; i < bt.graphs.size(); ++i) mc = std::max(mc, bt.graphs[i].code_len);
  bt.max_code = bt.graphs[0].code_len + mc;
  return bt;
}

struct VerifyRun {
  const uint32_t *pool_host = nullptr;  // pool mode
  uint32_t pool_n = 0;
  const std::vector<uint32_t> *cand_graph = nullptr;  // explicit mode
  const uint64_t *seeds = nullptr;
  uint64_t first = 0, n = 0;
  tpo_verdict *verdicts_host = nullptr;
  uint32_t *accept_host = nullptr;
  uint32_t *accept_dev = nullptr;
  uint64_t *attempts = nullptr;
  cudaStream_t stream = nullptr;
};

void run_verify(Ctx &C, const Batch &bt, const tpo_verify_cfg &cfg, const tpo_field_params &fpp,
                const VerifyRun &r) {
  check_cuda(cudaSetDevice(C.device), "cudaSetDevice");
  FieldState &fs = C.field(fpp.p, fpp.q, fpp.omega_base);
  const size_t code_bytes = size_t(bt.max_code) * sizeof(TpoVmInstr);
  // 16-bit VM words when both primes are below 256 (TPO_VM_WIDE keeps 32)
  const int narrow = fs.fc.small && !std::getenv("TPO_VM_WIDE");
  const size_t smem = fs.fc.table_bytes + code_bytes + size_t(bt.max_words) * (narrow ? 2 : 4);
  if (smem > 232448)
    throw Error(ErrCode::DoesNotFit,
                "verifier working set " + std::to_string(smem) + " B exceeds 227 KiB of shared memory");
  if (cfg.num_tests < 1) throw Error(ErrCode::ConfigError, "num_tests must be >= 1");
  cudaStream_t st = r.stream ? r.stream : C.stream;
  tpo_ff::VerifyArgs a{};
  a.field = fs.fc;
  a.tables = static_cast<const uint16_t *>(fs.dev.ptr);
  static const bool eager = std::getenv("TPO_VM_EAGER") != nullptr;  // A/B: no lazy input sampling
  a.eager_inputs = eager ? 1 : 0;
  auto *dcode = static_cast<TpoVmInstr *>(C.code.get(bt.code.size() * sizeof(TpoVmInstr) + 1));
  auto *dgraphs = static_cast<TpoVmGraph *>(C.graphs.get(bt.graphs.size() * sizeof(TpoVmGraph)));
  check_cuda(cudaMemcpyAsync(dcode, bt.code.data(), bt.code.size() * sizeof(TpoVmInstr),
                             cudaMemcpyHostToDevice, st), "upload code");
  check_cuda(cudaMemcpyAsync(dgraphs, bt.graphs.data(), bt.graphs.size() * sizeof(TpoVmGraph),
                             cudaMemcpyHostToDevice, st), "upload graphs");
  a.code = dcode;
  a.graphs = dgraphs;
  a.program = 0;
  a.code_smem_bytes = uint32_t(code_bytes);
  if (r.pool_host) {
    auto *dp = static_cast<uint32_t *>(C.pool.get(r.pool_n * 4));
    check_cuda(cudaMemcpyAsync(dp, r.pool_host, r.pool_n * 4, cudaMemcpyHostToDevice, st), "pool");
    a.pool = dp;
    a.pool_n = r.pool_n;
  } else {
    auto *dc = static_cast<uint32_t *>(C.cand.get(r.n * 4));
    check_cuda(cudaMemcpyAsync(dc, r.cand_graph->data(), r.n * 4, cudaMemcpyHostToDevice, st), "cands");
    a.cand_graph = dc;
  }
  a.n_in = bt.n_in;
  if (r.seeds) {
    auto *ds = static_cast<uint64_t *>(C.seeds.get(r.n * 8));
    check_cuda(cudaMemcpyAsync(ds, r.seeds, r.n * 8, cudaMemcpyHostToDevice, st), "seeds");
    a.seeds = ds;
    // a search loop verifies every candidate with the same VerifyConfig
    // seed: the first attempt's inputs and program outputs are then common
    // to the batch — compute them once (TPO_VM_NO_SHARED disables)
    bool same = r.n >= 32 && !bt.graphs[0].err && !std::getenv("TPO_VM_NO_SHARED");
    for (uint64_t k = 1; same && k < r.n; ++k) same = r.seeds[k] == r.seeds[0];
    if (same) {
      a.shared_len = bt.cand_base;
      auto *sw = static_cast<uint32_t *>(C.shared_w.get(size_t(bt.cand_base) * 4 + 16));
      auto *stab = static_cast<uint16_t *>(C.shared_tab.get(size_t(fs.fc.p + 2 * fs.fc.q) * 2 + 16));
      auto *smeta = static_cast<uint32_t *>(C.shared_meta.get(16));
      check_cuda(cudaError_t(tpo_ff_launch_shared(&a, r.seeds[0], smem, sw, stab, smeta, narrow, st)), "shared attempt");
      a.shared_w = sw;
      a.shared_tab = stab;
      a.shared_meta = smeta;
      a.shared_seed = r.seeds[0];
    }
  }
  a.first = r.first;
  a.n = r.n;
  a.n_in = bt.n_in;
  a.num_tests = cfg.num_tests;
  a.max_resamples = cfg.max_resamples;
  auto *cnt = static_cast<unsigned long long *>(C.counter.get(24));
  check_cuda(cudaMemsetAsync(cnt, 0, 24, st), "counter");
  a.counter = cnt;
  a.work = cnt + 1;
  a.drawn = cnt + 2;
  if (r.verdicts_host) a.verdicts = static_cast<TpoVerdict *>(C.verdicts.get(r.n * sizeof(TpoVerdict)));
  const size_t words = (r.n + 31) / 32;
  uint32_t *acc = r.accept_dev;
  if (!acc && r.accept_host) acc = static_cast<uint32_t *>(C.accept.get(words * 4));
  if (acc) check_cuda(cudaMemsetAsync(acc, 0, words * 4, st), "accept");
  a.accept = acc;
  // 128-thread candidate CTAs when twice as many of them fit an SM (small
  // working sets, e.g. the RMSNorm pool: many short instructions, so more
  // independent barrier domains per SM win: 8.6 vs 6.5 M cand/s measured);
  // TPO_VM_THREADS overrides
  int nthr = 256;
  int occ = tpo_ff_verify_occupancy(smem, 256, narrow);
  {
    const char *e = std::getenv("TPO_VM_THREADS");
    const int forced = e ? std::atoi(e) : 0;
    const int occ128 = tpo_ff_verify_occupancy(smem, 128, narrow);
    if (forced == 128 || (forced == 0 && occ128 >= 2 * occ)) nthr = 128, occ = occ128;
    // graphs of tiny instructions (mean index space < 64 items: the RMSNorm
    // pool) run a candidate per 64 threads when that raises residency 1.5x
    // (10.3 vs 9.1 M cand/s measured; larger graphs lose by it)
    double sn = 0, cnt = 0;
    for (const TpoVmInstr &I : bt.code)
      if (I.op != VM_LOOP && I.op != VM_ENDLOOP) sn += I.n, cnt += 1;
    const int occ64 = tpo_ff_verify_occupancy(smem, 64, narrow);
    if (forced == 64 || (forced == 0 && nthr == 128 && cnt > 0 && sn / cnt < 64 && 2 * occ64 >= 3 * occ))
      nthr = 64, occ = occ64;
  }
  if (occ < 1) throw Error(ErrCode::DoesNotFit, "verifier kernel does not fit on an SM");
  // Bytecode read in place from global memory (block-uniform loads that
  // stay L1-resident) instead of staged in shared memory: the staging
  // copies and their barriers go, and the smaller working set raises
  // residency where shared memory bounds it (the GQA pool: 6 -> 7 CTAs per
  // SM).  A/B on one box, 250k candidates per pool: GQA 31.0 -> 29.7 ms,
  // RMSNorm 17.7 -> 17.5, GatedMLP and LoRA unchanged
  // (profiles/r02/verify_code_global_ab.txt).  TPO_VM_CODE_GLOBAL=0 stages.
  size_t smem_run = smem;
  {
    const char *e = std::getenv("TPO_VM_CODE_GLOBAL");
    const size_t smem_nc = smem - code_bytes;
    const int occ_nc = tpo_ff_verify_occupancy(smem_nc, nthr, narrow);
    if (!e || std::atoi(e) != 0) {
      a.code_global = 1;
      a.code_smem_bytes = 0;
      smem_run = smem_nc;
      occ = occ_nc;
    }
  }
  if (std::getenv("TPO_VM_DEBUG")) {
    double sn = 0, cnt = 0, mm = 0;
    for (const TpoVmInstr &I : bt.code) {
      if (I.op == VM_LOOP || I.op == VM_ENDLOOP) continue;
      sn += I.n, cnt += 1;
      if (I.op == VM_MATMUL) mm += double(I.n) * I.dims[5] * ((I.flags & VM_TILE22) ? 4 : 1);
    }
    std::fprintf(stderr, "[tpo vm] smem %zu occ256 %d occ128 %d instrs %.0f avg_n %.1f matmul_macs/instr %.1f\n", smem,
                 tpo_ff_verify_occupancy(smem, 256, narrow), tpo_ff_verify_occupancy(smem, 128, narrow), cnt, sn / cnt, mm / cnt);
  }
  uint64_t grid = std::min<uint64_t>(uint64_t(C.num_sms) * uint64_t(occ), r.n);
  grid = std::max<uint64_t>(grid, 1);
  // TPO_VM_PROFILE: per-opcode cycle breakdown of the verifier (thread 0 of
  // each CTA; slot 0 = input/omega/SiLU generation, 9 = output compare)
  static unsigned long long *prof = nullptr;
  const bool profile = std::getenv("TPO_VM_PROFILE") != nullptr;
  if (profile) {
    if (!prof) check_cuda(cudaMalloc(&prof, 32 * 8), "prof");
    check_cuda(cudaMemsetAsync(prof, 0, 32 * 8, st), "prof");
    a.prof = prof;
  }
  const bool dbg = std::getenv("TPO_VM_DEBUG") != nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::chrono::steady_clock::time_point tu;
  if (dbg) {
    cudaStreamSynchronize(st);
    tu = std::chrono::steady_clock::now();
    cudaEventCreate(&ev0);
    cudaEventCreate(&ev1);
    cudaEventRecord(ev0, st);
  }
  check_cuda(cudaError_t(tpo_ff_launch_verify(&a, int(grid), smem_run, st, nthr, narrow)), "verify launch");
  if (dbg) {
    cudaEventRecord(ev1, st);
    cudaEventSynchronize(ev1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev0, ev1);
    std::fprintf(stderr, "[tpo run_verify] kernel %.3f ms (grid %llu x %d thr, smem %zu B), host after upload %.3f ms\n",
                 ms, (unsigned long long)grid, nthr, smem,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tu).count());
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
  }
  if (profile) {
    unsigned long long h[32];
    check_cuda(cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, st), "prof");
    check_cuda(cudaStreamSynchronize(st), "prof");
    static const char *nm[16] = {"gen_inputs", "ZERO", "COPY", "UNARY", "BINARY", "MATMUL", "SUM",
                                 "LOOP", "ENDLOOP", "compare", "", "", "", "", "", ""};
    unsigned long long tot = 0;
    for (int i = 0; i < 16; ++i) tot += h[i];
    std::fprintf(stderr, "[tpo vm profile] n=%llu candidates, %d CTAs\n", (unsigned long long)r.n, int(grid));
    for (int i = 0; i < 16; ++i)
      if (h[i])
        std::fprintf(stderr, "  %-11s %6.2f%%  cycles/exec %9.1f  execs %llu\n", nm[i], 100.0 * double(h[i]) / double(tot),
                     double(h[i]) / double(h[16 + i] ? h[16 + i] : 1), h[16 + i]);
  }
  if (r.verdicts_host)
    check_cuda(cudaMemcpyAsync(r.verdicts_host, a.verdicts, r.n * sizeof(TpoVerdict),
                               cudaMemcpyDeviceToHost, st), "verdicts");
  if (r.accept_host)
    check_cuda(cudaMemcpyAsync(r.accept_host, acc, words * 4, cudaMemcpyDeviceToHost, st), "accept");
  unsigned long long counters[3] = {0, 0, 0};
  if (r.attempts)
    check_cuda(cudaMemcpyAsync(counters, cnt, 24, cudaMemcpyDeviceToHost, st), "attempts");
  check_cuda(cudaStreamSynchronize(st), "verify sync");
  if (r.attempts) {
    *r.attempts = counters[1];
    C.last_draws = counters[2];
  }
}

}  // namespace

const VmProgram &lowered_fp(const Graph &G) {
  std::lock_guard<std::mutex> lk(G.ff_mu);
  const auto key = std::make_pair(uint32_t(G.in_elems), 2);
  auto it = G.ff_cache.find(key);
  if (it == G.ff_cache.end())
    it = G.ff_cache.emplace(key, std::make_shared<const VmProgram>(lower_vm(G.g, 0, uint32_t(G.in_elems)))).first;
  return *it->second;
}

const VmProgram &lowered_ff(const Graph &G, uint32_t region, bool pin) {
  std::lock_guard<std::mutex> lk(G.ff_mu);
  const auto key = std::make_pair(region, int(pin));
  auto it = G.ff_cache.find(key);
  if (it == G.ff_cache.end())
    it = G.ff_cache.emplace(key, std::make_shared<const VmProgram>(lower_vm(G.g, 0, region, pin, true))).first;
  return *it->second;
}

}  // namespace tpo::gpu

using namespace tpo;
using namespace tpo::gpu;

extern "C" {

int tpo_gpu_abi_version(void) { return TPO_GPU_ABI_VERSION; }

const char *tpo_gpu_last_error(void) { return g_last.c_str(); }

int tpo_gpu_open(int device, tpo_gpu_ctx **out) {
  return guard([&] {
    auto *c = new tpo_gpu_ctx();
    c->c.device = device;
    try {
      check_cuda(cudaSetDevice(device), "cudaSetDevice");
      check_cuda(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking), "stream");
      check_cuda(cudaDeviceGetAttribute(&c->c.num_sms, cudaDevAttrMultiProcessorCount, device), "attr");
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
    return 0;
  });
}

void tpo_gpu_close(tpo_gpu_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  if (ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
  delete ctx;
}

}  // extern "C"

namespace {

// the per-graph facts every entry point reads; `match`: also the fused
// kernel match (a search candidate defers it until it is accepted)
void finish_graph(Graph &G, bool match) {
  G.lax = ir::mugraph_lax_check(G.g).lax;
  G.madds = graph_madds(G.g);
  G.in_elems = input_elems(G.g);
  G.out_elems = 0;
  for (ir::TensorId t : G.g.outputs) G.out_elems += G.g.tensor(t).shape.elem_count();
  if (match) G.fused_plan();
  G.vm_words = -2;  // computed on first tpo_gpu_graph_info (an fp lowering)
}

// parse + validate (B200 limits) + fused match + VM footprint; throws
tpo_gpu_graph *compile_one(const char *json) {
  auto h = std::make_unique<tpo_gpu_graph>();
  Graph &G = h->g;
  static const bool slow_only = std::getenv("TPO_JSON_SLOW") != nullptr;
  if (slow_only || !ir::kernel_graph_from_text_fast(json, std::strlen(json), G.g)) {
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(json);
    } catch (const nlohmann::json::exception &e) {
      throw Error(ErrCode::ParseError, e.what());
    }
    G.g = ir::kernel_graph_from_json(j);
  }
  ir::ValidityReport rep = ir::validate(G.g, ir::kB200Limits);
  if (!rep.valid()) {
    std::string msg;
    for (auto &v : rep.violations) msg += v.detail + "; ";
    ErrCode c = rep.violations[0].kind == ir::ViolationKind::MemoryCapacity ? ErrCode::DoesNotFit
                                                                           : ErrCode::ShapeMismatch;
    throw Error(c, "invalid µGraph: " + msg);
  }
  finish_graph(G, false);  // the fused match runs on first use
  return h.release();
}

}  // namespace

extern "C" {

int tpo_gpu_compile(tpo_gpu_ctx *, const char *json, tpo_gpu_graph **out) {
  return guard([&] {
    *out = compile_one(json);
    return 0;
  });
}

int tpo_gpu_compile_many(tpo_gpu_ctx *, const char *const *json, int64_t n, int32_t threads,
                         tpo_gpu_graph **out, int32_t *status) {
  return guard([&] {
    if (n < 0 || (n && (!json || !out || !status))) throw Error(ErrCode::ShapeMismatch, "compile_many: bad arguments");
    const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(threads > 0 ? threads : host_threads(), n / 8 + 1));
    parallel_for(n, int(nt), [&](int64_t i) {
      out[i] = nullptr;
      status[i] = guard([&] {
        out[i] = compile_one(json[i]);
        return 0;
      });
    });
    return 0;
  });
}

void tpo_gpu_graph_free(tpo_gpu_graph *g) { delete g; }

int tpo_gpu_graph_info(const tpo_gpu_graph *h, tpo_graph_info *o) {
  const Graph &G = h->g;
  o->n_inputs = int32_t(G.g.inputs.size());
  o->n_outputs = int32_t(G.g.outputs.size());
  o->fused_kind = G.fused_plan().kind;
  o->lax = G.lax;
  o->madds = G.madds;
  o->input_elems = G.in_elems;
  o->output_elems = G.out_elems;
  {
    std::lock_guard<std::mutex> lk(G.ff_mu);
    if (G.vm_words == -2) {
      try {
        G.vm_words = G.in_elems + lower_vm(G.g, 0, uint32_t(G.in_elems)).region_words;
      } catch (const Error &) {
        G.vm_words = -1;
      }
    }
  }
  o->vm_words = G.vm_words;
  return 0;
}

int tpo_gpu_graph_set_static_inputs(tpo_gpu_graph *h, uint64_t mask) {
  return guard([&] {
    if (h->g.g.inputs.size() < 64 && (mask >> h->g.g.inputs.size()))
      throw Error(ErrCode::ShapeMismatch, "static-input mask names a non-existent input");
    h->g.plan.static_inputs = mask;
    return 0;
  });
}

int tpo_gpu_graph_shape(const tpo_gpu_graph *h, int is_output, int index, int64_t *dims) {
  const auto &v = is_output ? h->g.g.outputs : h->g.g.inputs;
  if (index < 0 || size_t(index) >= v.size()) return -1;
  const auto &s = h->g.g.tensor(v[size_t(index)]).shape;
  for (int i = 0; i < s.rank(); ++i) dims[i] = s.dims[size_t(i)];
  return s.rank();
}

int tpo_gpu_validate(const char *json, int64_t smem_bytes, int64_t elem_size, char *buf, int cap) {
  return guard([&] {
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(json);
    } catch (const nlohmann::json::exception &e) {
      throw Error(ErrCode::ParseError, e.what());
    }
    ir::KernelGraph g = ir::kernel_graph_from_json(j);
    ir::MemLimits lim;
    lim.smem_bytes = smem_bytes;
    lim.elem_size = elem_size;
    auto rep = ir::validate(g, lim);
    std::string msg;
    for (auto &v : rep.violations) msg += v.detail + "; ";
    if (buf && cap > 0) {
      std::strncpy(buf, msg.c_str(), size_t(cap - 1));
      buf[cap - 1] = 0;
    }
    return int(rep.violations.size());
  });
}

int64_t tpo_gpu_op_madds(const tpo_gpu_graph *g) { return g->g.madds; }

}  // extern "C"

extern "C" int tpo_convert_to_f32(const void *in, int dtype, float *out, size_t n, int num_sms,
                                  cudaStream_t st);
extern "C" int tpo_convert_to_f64(const void *in, int dtype, double *out, size_t n, int num_sms,
                                  cudaStream_t st);

namespace {
int eval_vm_impl(tpo_gpu_ctx *ctx, const tpo_gpu_graph *h, int32_t mode, const void *in, void *out,
                 bool host, cudaStream_t stream);

size_t dtype_bytes(int32_t dt) {
  switch (dt) {
    case TPO_DTYPE_F32: return 4;
    case TPO_DTYPE_BF16: return 2;
    case TPO_DTYPE_F64: return 8;
  }
  throw Error(ErrCode::Unsupported, "input dtype must be TPO_DTYPE_BF16, TPO_DTYPE_F32 or TPO_DTYPE_F64");
}

// A µGraph without a hand-written kernel (or TPO_PREC_VM): the generic VM on
// the device in the reference's operation order — double arithmetic
// (eval_mugraph, interp.hpp:47-48) when any input is fp64, else fp32
// (eval_mugraph_f32, interp.hpp:51-53).  Inputs are widened into one
// contiguous buffer; outputs are written as fp32 (out_dev) or, with
// out_f64, as the VM's doubles.
void eval_generic_dev(tpo_gpu_ctx *ctx, const tpo_gpu_graph *h, const void *const *in_dev,
                      const int32_t *in_dtype, float *const *out_dev, cudaStream_t st,
                      double *const *out_f64 = nullptr) {
  Ctx &C = ctx->c;
  const Graph &G = h->g;
  bool f64 = out_f64 != nullptr;
  for (size_t i = 0; i < G.g.inputs.size(); ++i) f64 |= dtype_bytes(in_dtype[i]) == 8;
  const size_t el = f64 ? 8 : 4;
  char *vin = static_cast<char *>(C.vm_in.get(size_t(G.in_elems) * el + 16));
  char *vout = static_cast<char *>(C.vm_out.get(size_t(G.out_elems) * el + 16));
  size_t off = 0;
  for (size_t i = 0; i < G.g.inputs.size(); ++i) {
    const size_t n = size_t(G.g.tensor(G.g.inputs[i]).shape.elem_count());
    const int32_t dt = in_dtype[i];
    if ((f64 && dt == TPO_DTYPE_F64) || (!f64 && dt == TPO_DTYPE_F32))
      check_cuda(cudaMemcpyAsync(vin + off * el, in_dev[i], n * el, cudaMemcpyDeviceToDevice, st), "in");
    else if (f64)
      check_cuda(cudaError_t(tpo_convert_to_f64(in_dev[i], dt, reinterpret_cast<double *>(vin) + off, n,
                                                C.num_sms, st)), "in->f64");
    else
      check_cuda(cudaError_t(tpo_convert_to_f32(in_dev[i], dt, reinterpret_cast<float *>(vin) + off, n,
                                                C.num_sms, st)), "in->f32");
    off += n;
  }
  const int rc = eval_vm_impl(ctx, h, f64 ? 0 : 2, vin, vout, false, st);
  if (rc) throw Error(ErrCode::Unsupported, "generic VM: " + std::string(tpo_gpu_last_error()));
  off = 0;
  for (size_t o = 0; o < G.g.outputs.size(); ++o) {
    const size_t n = size_t(G.g.tensor(G.g.outputs[o]).shape.elem_count());
    if (out_f64)
      check_cuda(cudaMemcpyAsync(out_f64[o], vout + off * 8, n * 8, cudaMemcpyDeviceToDevice, st), "out");
    else if (f64)
      check_cuda(cudaError_t(tpo_convert_to_f32(vout + off * 8, TPO_DTYPE_F64, out_dev[o], n, C.num_sms, st)),
                 "out->f32");
    else
      check_cuda(cudaMemcpyAsync(out_dev[o], vout + off * 4, n * 4, cudaMemcpyDeviceToDevice, st), "out");
    off += n;
  }
}

// Fused evaluation with the graph's precision policy; operand conversions
// land in context scratch.  caller_inputs: the buffers are the caller's
// (not written by the library on this stream).
int run_fused(Ctx &C, const Graph &G, const void *const *in, const int32_t *dt, float *const *out,
              bool caller_inputs, cudaStream_t st) {
  FusedIO io;
  io.in = in;
  io.dt = dt;
  io.out = out;
  io.precision = G.precision;
  io.caller_inputs = caller_inputs;
  io.num_sms = C.num_sms;
  io.scratch = [&C](int slot, size_t bytes) {
    if (C.fused_scratch.size() <= size_t(slot)) C.fused_scratch.resize(size_t(slot) + 1);
    return C.fused_scratch[size_t(slot)].get(bytes);
  };
  return launch_fused(G.fused_plan(), io, st);
}

bool use_fused(const Graph &G) { return G.fused_plan().kind != 0 && G.precision != TPO_PREC_VM; }

}  // namespace

extern "C" {

int tpo_gpu_graph_set_precision(tpo_gpu_graph *h, int32_t policy) {
  return guard([&] {
    if (!h) throw Error(ErrCode::ConfigError, "null graph");
    if (policy < TPO_PREC_AUTO || policy > TPO_PREC_VM) throw Error(ErrCode::ConfigError, "unknown TPO_PREC_* policy");
    h->g.precision = policy;
    return 0;
  });
}

int tpo_gpu_eval_mugraph(tpo_gpu_ctx *ctx, const tpo_gpu_graph *h, const void *const *in_dev,
                         const int32_t *in_dtype, float *const *out_dev, void *stream) {
  return guard([&] {
    const Graph &G = h->g;
    for (size_t i = 0; i < G.g.inputs.size(); ++i) dtype_bytes(in_dtype[i]);
    check_cuda(cudaSetDevice(ctx->c.device), "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL = legacy default stream
    if (!use_fused(G)) {
      eval_generic_dev(ctx, h, in_dev, in_dtype, out_dev, st);
      return 0;
    }
    int e = run_fused(ctx->c, G, in_dev, in_dtype, out_dev, true, st);
    if (e) return fail(3000 + e, std::string("fused launch: ") + cudaGetErrorString(cudaError_t(e)));
    return 0;
  });
}

int tpo_gpu_eval_mugraph_host(tpo_gpu_ctx *ctx, const tpo_gpu_graph *h, const void *const *in_host,
                              const int32_t *in_dtype, float *const *out_host, void *stream) {
  return guard([&] {
    Ctx &C = ctx->c;
    const Graph &G = h->g;
    check_cuda(cudaSetDevice(C.device), "cudaSetDevice");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : C.stream;
    const size_t ni = G.g.inputs.size(), no = G.g.outputs.size();
    if (C.h_in.size() < ni) C.h_in.resize(ni);
    if (C.h_out.size() < no) C.h_out.resize(no);
    // inputs cross PCIe in the caller's dtype; conversions run on the device
    std::vector<const void *> din(ni);
    for (size_t i = 0; i < ni; ++i) {
      const size_t n = size_t(G.g.tensor(G.g.inputs[i]).shape.elem_count()) * dtype_bytes(in_dtype[i]);
      void *d = C.h_in[i].get(n);
      check_cuda(cudaMemcpyAsync(d, in_host[i], n, cudaMemcpyHostToDevice, st), "H2D");
      din[i] = d;
    }
    std::vector<float *> dout(no);
    for (size_t o = 0; o < no; ++o)
      dout[o] = static_cast<float *>(
          C.h_out[o].get(size_t(G.g.tensor(G.g.outputs[o]).shape.elem_count()) * 4));
    if (use_fused(G)) {
      // the copies above wrote the operands on this stream: nothing may be
      // read before the kernel's dependency resolves (no static prefetch)
      int e = run_fused(C, G, din.data(), in_dtype, dout.data(), false, st);
      if (e) return fail(3000 + e, std::string("fused launch: ") + cudaGetErrorString(cudaError_t(e)));
    } else {
      eval_generic_dev(ctx, h, din.data(), in_dtype, dout.data(), st);
    }
    for (size_t o = 0; o < no; ++o)
      check_cuda(cudaMemcpyAsync(out_host[o], dout[o],
                                 size_t(G.g.tensor(G.g.outputs[o]).shape.elem_count()) * 4,
                                 cudaMemcpyDeviceToHost, st),
                 "D2H");
    check_cuda(cudaStreamSynchronize(st), "sync");
    return 0;
  });
}

int tpo_gpu_eval_mugraph_f64(tpo_gpu_ctx *ctx, const tpo_gpu_graph *h, const double *const *in_host,
                             double *const *out_host, void *stream) {
  return guard([&] {
    Ctx &C = ctx->c;
    const Graph &G = h->g;
    check_cuda(cudaSetDevice(C.device), "cudaSetDevice");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : C.stream;
    const size_t ni = G.g.inputs.size(), no = G.g.outputs.size();
    if (C.h_in.size() < ni) C.h_in.resize(ni);
    if (C.h_out.size() < 2 * no) C.h_out.resize(2 * no);
    std::vector<const void *> din(ni);
    std::vector<int32_t> dt(ni, TPO_DTYPE_F64);
    for (size_t i = 0; i < ni; ++i) {
      const size_t n = size_t(G.g.tensor(G.g.inputs[i]).shape.elem_count()) * 8;
      void *d = C.h_in[i].get(n);
      check_cuda(cudaMemcpyAsync(d, in_host[i], n, cudaMemcpyHostToDevice, st), "H2D");
      din[i] = d;
    }
    std::vector<double *> d64(no);
    for (size_t o = 0; o < no; ++o)
      d64[o] = static_cast<double *>(C.h_out[no + o].get(size_t(G.g.tensor(G.g.outputs[o]).shape.elem_count()) * 8));
    if (use_fused(G)) {
      std::vector<float *> d32(no);
      for (size_t o = 0; o < no; ++o)
        d32[o] = static_cast<float *>(C.h_out[o].get(size_t(G.g.tensor(G.g.outputs[o]).shape.elem_count()) * 4));
      int e = run_fused(C, G, din.data(), dt.data(), d32.data(), false, st);
      if (e) return fail(3000 + e, std::string("fused launch: ") + cudaGetErrorString(cudaError_t(e)));
      for (size_t o = 0; o < no; ++o)
        check_cuda(cudaError_t(tpo_convert_to_f64(d32[o], TPO_DTYPE_F32, d64[o],
                                                  size_t(G.g.tensor(G.g.outputs[o]).shape.elem_count()),
                                                  C.num_sms, st)), "out->f64");
    } else {
      eval_generic_dev(ctx, h, din.data(), dt.data(), nullptr, st, d64.data());
    }
    for (size_t o = 0; o < no; ++o)
      check_cuda(cudaMemcpyAsync(out_host[o], d64[o], size_t(G.g.tensor(G.g.outputs[o]).shape.elem_count()) * 8,
                                 cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaStreamSynchronize(st), "sync");
    return 0;
  });
}

int tpo_gpu_ff_eval(tpo_gpu_ctx *ctx, const tpo_gpu_graph *h, const tpo_field_params *fpp,
                    uint64_t seed, uint64_t stream, int32_t with_silu, uint16_t *out_xp,
                    uint16_t *out_xq, uint8_t *out_qd, uint32_t *omega_out, uint16_t *in_xp,
                    uint16_t *in_xq) {
  return guard([&] {
    Ctx &C = ctx->c;
    check_cuda(cudaSetDevice(C.device), "cudaSetDevice");
    const Graph &G = h->g;
    FieldState &fs = C.field(fpp->p, fpp->q, fpp->omega_base);
    const uint32_t n_in = uint32_t(G.in_elems);
    VmProgram p = lower_vm(G.g, 0, n_in, false, /*field=*/true);
    const size_t smem = fs.fc.table_bytes + size_t(n_in + p.region_words) * 4;
    if (smem > 232448) throw Error(ErrCode::DoesNotFit, "graph exceeds shared memory");
    TpoVmGraph d = p.desc;
    d.code_off = 0;
    cudaStream_t st = C.stream;
    auto *dcode = static_cast<TpoVmInstr *>(C.code.get(p.code.size() * sizeof(TpoVmInstr) + 1));
    auto *dg = static_cast<TpoVmGraph *>(C.graphs.get(sizeof(TpoVmGraph)));
    check_cuda(cudaMemcpyAsync(dcode, p.code.data(), p.code.size() * sizeof(TpoVmInstr),
                               cudaMemcpyHostToDevice, st), "code");
    check_cuda(cudaMemcpyAsync(dg, &d, sizeof(d), cudaMemcpyHostToDevice, st), "graph");
    const size_t n_out = size_t(G.out_elems);
    auto *dout = static_cast<uint32_t *>(C.out.get((n_out + n_in) * 4 + 4));
    auto *dstat = static_cast<int *>(C.status.get(16));
    tpo_ff::EvalArgs a{};
    a.field = fs.fc;
    a.tables = static_cast<const uint16_t *>(fs.dev.ptr);
    a.code = dcode;
    a.graphs = dg;
    a.n_in = n_in;
    a.seed = seed;
    a.stream = stream;
    a.with_silu = with_silu;
    a.out = dout;
    a.in_dump = dout + n_out;
    a.status = dstat;
    check_cuda(cudaError_t(tpo_ff_launch_eval(&a, smem, st)), "eval launch");
    std::vector<uint32_t> hout(n_out + n_in);
    int hs[2];
    check_cuda(cudaMemcpyAsync(hs, dstat, 8, cudaMemcpyDeviceToHost, st), "status");
    check_cuda(cudaMemcpyAsync(hout.data(), dout, (n_out + n_in) * 4, cudaMemcpyDeviceToHost, st), "out");
    check_cuda(cudaStreamSynchronize(st), "eval sync");
    if (omega_out) *omega_out = uint32_t(hs[1]);
    for (uint32_t e = 0; e < n_in; ++e) {
      if (in_xp) in_xp[e] = uint16_t(hout[n_out + e] & 0xffff);
      if (in_xq) in_xq[e] = uint16_t(hout[n_out + e] >> 16);
    }
    // a VM_RAISE reached with no event before it: the reference's Error
    if (hs[0] == 3) throw Error(ErrCode::PoisonedExponent, "exponent depends on a prior exponentiation");
    if (hs[0]) return 2000 + int(hs[0] == 2 ? ErrCode::NonResidue : ErrCode::DivByZero);
    size_t c = 0;
    for (uint32_t t = 0; t < p.desc.n_out; ++t)
      for (uint32_t i = 0; i < p.desc.out_len[t]; ++i, ++c) {
        out_xp[c] = uint16_t(hout[c] & 0xffff);
        out_xq[c] = uint16_t(hout[c] >> 16);
        out_qd[c] = p.desc.out_qd[t];
      }
    return 0;
  });
}

}  // extern "C"

namespace {
TpoVerdict verdict_global(Ctx &C, const Graph &P, const Graph &G2, const tpo_verify_cfg &cfg, FieldState &fs);
}

extern "C" {

int tpo_gpu_verify_batch(tpo_gpu_ctx *ctx, const tpo_gpu_graph *program,
                         const tpo_gpu_graph *const *cands, const uint64_t *seeds, uint64_t n,
                         const tpo_verify_cfg *cfg, const tpo_field_params *fp,
                         tpo_verdict *verdicts, uint32_t *accept_bits) {
  return guard([&] {
    if (n == 0) return 0;
    // seeds == NULL: cfg->seed for every candidate (one VerifyConfig for the
    // whole batch, as the search loop calls it) on either
    // executor
    std::vector<uint64_t> one_seed;
    if (!seeds) {
      one_seed.assign(size_t(n), cfg->seed);
      seeds = one_seed.data();
    }
    // graphs beyond shared memory: the global-memory field executor, one
    // candidate at a time (same verdicts; BASELINE-shape pairs)
    auto global_loop = [&] {
      Ctx &C = ctx->c;
      check_cuda(cudaSetDevice(C.device), "cudaSetDevice");
      if (cfg->num_tests < 1) throw Error(ErrCode::ConfigError, "num_tests must be >= 1");
      FieldState &fs = C.field(fp->p, fp->q, fp->omega_base);
      if (accept_bits) std::memset(accept_bits, 0, size_t((n + 31) / 32) * 4);
      for (uint64_t k = 0; k < n; ++k) {
        tpo_verify_cfg c = *cfg;
        c.seed = seeds[k];
        TpoVerdict v;
        try {
          check_pair(program->g.g, cands[k]->g.g);
          v = verdict_global(C, program->g, cands[k]->g, c, fs);
        } catch (const Error &e) {
          v = TpoVerdict{};
          v.kind = 3;
          v.err_code = 1000 + int(e.code);
        }
        if (verdicts) std::memcpy(&verdicts[k], &v, sizeof(v));
        if (accept_bits && v.kind == 0) accept_bits[k >> 5] |= 1u << (k & 31);
      }
      return 0;
    };
    if (std::getenv("TPO_VM_GLOBAL")) return global_loop();  // test hook: force the HBM executor
    std::unordered_map<const tpo_gpu_graph *, uint32_t> idx;
    std::vector<const Graph *> uniq;
    std::vector<uint32_t> cg(n);
    for (uint64_t k = 0; k < n; ++k) {
      auto it = idx.find(cands[k]);
      if (it == idx.end()) {
        it = idx.emplace(cands[k], uint32_t(uniq.size() + 1)).first;
        uniq.push_back(&cands[k]->g);
      }
      cg[k] = it->second;
    }
    const auto t0 = std::chrono::steady_clock::now();
    Batch bt = build_batch(program->g, uniq);
    const auto t1 = std::chrono::steady_clock::now();
    VerifyRun r;
    r.cand_graph = &cg;
    r.seeds = seeds;
    r.n = n;
    r.verdicts_host = verdicts;
    r.accept_host = accept_bits;
    try {
      run_verify(ctx->c, bt, *cfg, *fp, r);
    } catch (const Error &e) {
      if (e.code != ErrCode::DoesNotFit) throw;
      return global_loop();
    }
    if (std::getenv("TPO_VM_DEBUG")) {
      const auto t2 = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[tpo verify_batch] n %llu distinct %zu build %.2f ms, upload+run %.2f ms, code %.1f MB\n",
                   (unsigned long long)n, uniq.size(),
                   std::chrono::duration<double, std::milli>(t1 - t0).count(),
                   std::chrono::duration<double, std::milli>(t2 - t1).count(),
                   double(bt.code.size() * sizeof(TpoVmInstr)) / 1e6);
    }
    return 0;
  });
}

}  // extern "C"

namespace {

// Walk one graph's bytecode on the global-memory field executor.  Returns
// true when the walk stopped at a VM_RAISE (the caller reads the event flag).
bool run_global_ff(Ctx &C, const VmProgram &p, const tpo_ff::GlobalFF &g, cudaStream_t st) {
  for (size_t pc = 0; pc < p.code.size(); ++pc) {
    const TpoVmInstr &I = p.code[pc];
    if (I.op == VM_RAISE) return true;
    if (I.op == VM_LOOP) {
      size_t end = pc + 1;
      while (end < p.code.size() && p.code[end].op != VM_ENDLOOP) ++end;
      for (uint32_t it = 0; it < I.n; ++it)
        for (size_t k = pc + 1; k < end; ++k) {
          if (p.code[k].op == VM_RAISE) return true;  // reached in the first iteration
          check_cuda(cudaError_t(tpo_ff_global_launch(0, &g, &p.code[k], it, uint32_t(k), 0, 0, 0, C.num_sms, st)),
                     "ff instr");
        }
      pc = end;
      continue;
    }
    check_cuda(cudaError_t(tpo_ff_global_launch(0, &g, &I, 0, uint32_t(pc), 0, 0, 0, C.num_sms, st)), "ff instr");
  }
  return false;
}

// random_test_equivalence (equiv.cpp:34-94) for graphs beyond shared
// memory: the same draws, arithmetic, resample and witness rules as the
// batched kernel, with VM memory in HBM and one launch per instruction.
TpoVerdict verdict_global(Ctx &C, const Graph &P, const Graph &G2, const tpo_verify_cfg &cfg, FieldState &fs) {
  TpoVerdict v{};
  const uint32_t n_in = uint32_t(P.in_elems);
  VmProgram pp, cp;
  try {
    pp = lower_vm(P.g, 0, n_in, /*pin_outputs=*/true, /*field=*/true);
    cp = lower_vm(G2.g, 0, n_in + pp.pinned_words, false, true);
  } catch (const Error &e) {
    v.kind = 3;
    v.err_code = 1000 + int(e.code);
    return v;
  }
  const uint64_t words = std::max<uint64_t>(uint64_t(n_in) + pp.region_words,
                                            uint64_t(n_in) + pp.pinned_words + cp.region_words);
  cudaStream_t st = C.stream;
  tpo_ff::GlobalFF g{};
  g.field = fs.fc;
  g.tables = static_cast<const uint16_t *>(fs.dev.ptr);
  g.attempt_tab = static_cast<uint16_t *>(C.shared_tab.get(size_t(fs.fc.p + 2 * fs.fc.q) * 2 + 16));
  g.W = static_cast<uint32_t *>(C.ws.get(words * 4 + 16));
  g.flag = static_cast<int *>(C.status.get(16));
  g.meta = static_cast<uint32_t *>(C.shared_meta.get(16));
  auto *key = static_cast<unsigned long long *>(C.counter.get(16));
  const uint64_t seed = cfg.seed;
  bool finished = false;
  for (int round = 0; round < cfg.num_tests && !finished; ++round) {
    bool round_done = false;
    for (int att = 0; att <= cfg.max_resamples && !round_done; ++att) {
      const uint64_t stream = uint64_t(round) * 131071ull + uint64_t(att);
      check_cuda(cudaMemsetAsync(g.meta, 0, 16, st), "meta");
      for (int what : {1, 2, 3})
        check_cuda(cudaError_t(tpo_ff_global_launch(what, &g, nullptr, 0, 0, seed, stream, n_in, C.num_sms, st)),
                   "ff gen");
      bool ok = true;
      for (const VmProgram *prog : {&pp, &cp}) {
        check_cuda(cudaMemsetAsync(g.flag, 0, 4, st), "flag");
        const bool raised = run_global_ff(C, *prog, g, st);
        int h = 0;
        check_cuda(cudaMemcpyAsync(&h, g.flag, 4, cudaMemcpyDeviceToHost, st), "flag");
        check_cuda(cudaStreamSynchronize(st), "sync");
        if (h) {  // g1 then g2: any ResampleNeeded resamples (equiv.cpp:67-83)
          ok = false;
          break;
        }
        if (raised) {  // Error(PoisonedExponent) escapes random_test_equivalence
          TpoVerdict e{};
          e.kind = 3;
          e.err_code = 1000 + int(ErrCode::PoisonedExponent);
          return e;
        }
      }
      if (!ok) {
        ++v.resamples;
        continue;
      }
      uint32_t omega = 0;
      check_cuda(cudaMemcpyAsync(&omega, g.meta + 1, 4, cudaMemcpyDeviceToHost, st), "omega");
      for (uint32_t t = 0; t < pp.desc.n_out && !finished; ++t) {
        const unsigned long long none = ~0ull;
        check_cuda(cudaMemcpyAsync(key, &none, 8, cudaMemcpyHostToDevice, st), "key");
        check_cuda(cudaError_t(tpo_ff_global_mismatch(g.W + pp.desc.out_off[t], g.W + cp.desc.out_off[t],
                                                      pp.desc.out_len[t], pp.desc.out_qd[t] && cp.desc.out_qd[t],
                                                      key, C.num_sms, st)),
                   "mismatch");
        unsigned long long k = 0;
        check_cuda(cudaMemcpyAsync(&k, key, 8, cudaMemcpyDeviceToHost, st), "key");
        check_cuda(cudaStreamSynchronize(st), "sync");
        if (k != none) {
          v.kind = 1;
          v.has_witness = 1;
          v.w_seed = seed;
          v.w_round = round;
          v.w_omega = omega;
          v.w_tensor = int32_t(t);
          v.w_index = int64_t(k);
          v.rounds_run = round + 1;
          finished = true;
        }
      }
      round_done = true;
    }
    if (!round_done && !finished) {
      v.kind = 2;
      v.rounds_run = round;
      finished = true;
    }
  }
  if (!finished) {
    v.kind = 0;
    v.rounds_run = cfg.num_tests;
  }
  return v;
}

}  // namespace

extern "C" {

int tpo_gpu_random_test_equivalence(tpo_gpu_ctx *ctx, const tpo_gpu_graph *g1,
                                    const tpo_gpu_graph *g2, const tpo_verify_cfg *cfg,
                                    const tpo_field_params *fp, tpo_verdict *out) {
  return guard([&] {
    check_pair(g1->g.g, g2->g.g);  // throws ShapeMismatch before sampling, like equiv.cpp:38-49
    uint64_t seed = cfg->seed;
    const tpo_gpu_graph *c = g2;
    // (beyond shared memory verify_batch takes the global-memory executor)
    int rc = tpo_gpu_verify_batch(ctx, g1, &c, &seed, 1, cfg, fp, out, nullptr);
    if (rc) return rc;
    if (out->kind == 3) return out->err_code;
    return 0;
  });
}

int tpo_gpu_verify_pool(tpo_gpu_ctx *ctx, const tpo_gpu_graph *program,
                        const tpo_gpu_graph *const *pool, int32_t pool_n, uint64_t first,
                        uint64_t n, const tpo_verify_cfg *cfg, const tpo_field_params *fp,
                        uint32_t *accept_dev, tpo_verdict *verdicts, uint64_t *attempts,
                        void *cuda_stream) {
  return guard([&] {
    if (n == 0) return 0;
    if (pool_n < 1) throw Error(ErrCode::ConfigError, "empty pool");
    std::unordered_map<const tpo_gpu_graph *, uint32_t> idx;
    std::vector<const Graph *> uniq;
    std::vector<uint32_t> pg(static_cast<size_t>(pool_n));
    for (int32_t k = 0; k < pool_n; ++k) {
      auto it = idx.find(pool[k]);
      if (it == idx.end()) {
        it = idx.emplace(pool[k], uint32_t(uniq.size() + 1)).first;
        uniq.push_back(&pool[k]->g);
      }
      pg[size_t(k)] = it->second;
    }
    Batch bt = build_batch(program->g, uniq);
    VerifyRun r;
    r.pool_host = pg.data();
    r.pool_n = uint32_t(pool_n);
    r.first = first;
    r.n = n;
    r.verdicts_host = verdicts;
    r.accept_dev = accept_dev;
    r.attempts = attempts;
    r.stream = static_cast<cudaStream_t>(cuda_stream);
    run_verify(ctx->c, bt, *cfg, *fp, r);
    return 0;
  });
}

int tpo_gpu_verify_draws(tpo_gpu_ctx *ctx, uint64_t *draws) {
  return guard([&] {
    if (!draws) throw Error(ErrCode::ShapeMismatch, "draws is NULL");
    *draws = ctx->c.last_draws;
    return 0;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Floating-point VM (kernels/fp_vm.cu): generic eval_mugraph / eval_program /
// eval_mugraph_f32 and the batched float stability filter.
// ---------------------------------------------------------------------------
#include "../kernels/fp_vm.cuh"

namespace tpo::gpu {
namespace {

size_t fp_smem(uint32_t code_len, uint64_t words, size_t elem) {
  return size_t(code_len) * sizeof(TpoVmInstr) + size_t(words) * elem;
}

}  // namespace
}  // namespace tpo::gpu

extern "C" {

}  // extern "C"

namespace {

// Generic fp VM evaluation.  host: in/out are host buffers (copied and
// synchronised); else device buffers, asynchronous on `stream`.
int eval_vm_impl(tpo_gpu_ctx *ctx, const tpo_gpu_graph *h, int32_t mode, const void *in, void *out,
                 bool host, cudaStream_t stream) {
  return guard([&] {
    Ctx &C = ctx->c;
    const Graph &G = h->g;
    if (mode < 0 || mode > 2) throw Error(ErrCode::ConfigError, "mode: 0 eval_mugraph, 1 eval_program, 2 f32");
    if (mode == 1)  // interp.cpp:20-28: the flat evaluator rejects GraphDefs
      for (const ir::Op &op : G.g.ops)
        if (op.type == ir::OpType::GraphDef)
          throw Error(ErrCode::Unsupported, "eval_program: graph contains a GraphDef");
    check_cuda(cudaSetDevice(C.device), "cudaSetDevice");
    const size_t elem = mode == 2 ? 4 : 8;
    const uint32_t n_in = uint32_t(G.in_elems);
    const VmProgram &p = lowered_fp(G);
    const size_t smem = fp_smem(uint32_t(p.code.size()), uint64_t(n_in) + p.region_words, elem);
    cudaStream_t st = host ? C.stream : stream;
    const cudaMemcpyKind h2d = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const cudaMemcpyKind d2h = host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (smem > 232448 || std::getenv("TPO_VM_GLOBAL")) {
      // global-memory executor: VM memory in HBM, one launch per instruction
      const uint64_t words = uint64_t(n_in) + p.region_words;
      void *W = C.ws.get(words * elem + 16);
      check_cuda(cudaMemcpyAsync(W, in, size_t(n_in) * elem, h2d, st), "in");
      auto launch_all = [&](cudaStream_t s2) {
        for (size_t pc = 0; pc < p.code.size(); ++pc) {
          const TpoVmInstr &I = p.code[pc];
          if (I.op == VM_LOOP) {  // run the body I.n times
            size_t end = pc + 1;
            while (end < p.code.size() && p.code[end].op != VM_ENDLOOP) ++end;
            for (uint32_t it = 0; it < I.n; ++it)
              for (size_t k = pc + 1; k < end; ++k)
                check_cuda(cudaError_t(tpo_fp_launch_instr(W, mode == 2, &p.code[k], it, C.num_sms, s2)),
                           "vm instr");
            pc = end;  // skip ENDLOOP
            continue;
          }
          check_cuda(cudaError_t(tpo_fp_launch_instr(W, mode == 2, &I, 0, C.num_sms, s2)), "vm instr");
        }
      };
      // the launch sequence is fixed per (graph, mode, arena): captured once
      // into a CUDA graph (the per-instruction kernels are µs-scale, so host
      // launch overhead would otherwise bound the executor)
      cudaGraphExec_t exec = nullptr;
      {
        std::lock_guard<std::mutex> lk(G.ff_mu);
        auto it = G.vm_graphs.find({mode, W});
        if (it != G.vm_graphs.end()) exec = it->second;
      }
      if (!exec && !std::getenv("TPO_VM_NO_GRAPH")) {
        cudaStream_t cap;
        check_cuda(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "capture stream");
        cudaGraph_t graph = nullptr;
        if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
          launch_all(cap);
          if (cudaStreamEndCapture(cap, &graph) == cudaSuccess && graph) {
            if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) exec = nullptr;
            cudaGraphDestroy(graph);
          }
        }
        cudaStreamDestroy(cap);
        (void)cudaGetLastError();
        if (exec) {
          std::lock_guard<std::mutex> lk(G.ff_mu);
          G.vm_graphs[{mode, W}] = exec;
        }
      }
      if (exec)
        check_cuda(cudaGraphLaunch(exec, st), "vm graph");
      else
        launch_all(st);
      size_t c = 0;
      for (uint32_t t = 0; t < p.desc.n_out; ++t) {
        check_cuda(cudaMemcpyAsync(static_cast<char *>(out) + c * elem,
                                   static_cast<char *>(W) + size_t(p.desc.out_off[t]) * elem,
                                   size_t(p.desc.out_len[t]) * elem, d2h, st), "out");
        c += p.desc.out_len[t];
      }
      if (host) check_cuda(cudaStreamSynchronize(st), "vm sync");
      return 0;
    }
    auto *dcode = static_cast<TpoVmInstr *>(C.code.get(p.code.size() * sizeof(TpoVmInstr) + 16));
    check_cuda(cudaMemcpyAsync(dcode, p.code.data(), p.code.size() * sizeof(TpoVmInstr),
                               cudaMemcpyHostToDevice, st), "code");
    const void *din = in;
    if (host) {
      void *d = C.inputs.get(size_t(n_in) * elem + 16);
      check_cuda(cudaMemcpyAsync(d, in, size_t(n_in) * elem, h2d, st), "in");
      din = d;
    }
    const size_t n_out = size_t(G.out_elems);
    void *dout = host ? C.out.get(n_out * elem + 16) : out;
    tpo_fp::EvalArgs a{};
    a.code = dcode;
    a.code_len = uint32_t(p.code.size());
    a.code_bytes = uint32_t(p.code.size() * sizeof(TpoVmInstr));
    a.graph = p.desc;
    a.n_in = n_in;
    a.inputs = din;
    a.out = dout;
    check_cuda(cudaError_t(tpo_fp_launch_eval(&a, mode == 2, smem, st)), "fp eval launch");
    if (host) {
      check_cuda(cudaMemcpyAsync(out, dout, n_out * elem, d2h, st), "out");
      check_cuda(cudaStreamSynchronize(st), "fp eval sync");
    }
    return 0;
  });
}

}  // namespace

extern "C" {

int tpo_gpu_eval_vm(tpo_gpu_ctx *ctx, const tpo_gpu_graph *h, int32_t mode, const void *in_host,
                    void *out_host) {
  return eval_vm_impl(ctx, h, mode, in_host, out_host, true, nullptr);
}

int tpo_gpu_eval_vm_dev(tpo_gpu_ctx *ctx, const tpo_gpu_graph *h, int32_t mode, const void *in_dev,
                        void *out_dev, void *cuda_stream) {
  return eval_vm_impl(ctx, h, mode, in_dev, out_dev, false, static_cast<cudaStream_t>(cuda_stream));
}

}  // extern "C"

namespace {
int8_t stability_global(tpo_gpu_ctx *ctx, const tpo_gpu_graph *prog, const tpo_gpu_graph *cand, int trials,
                        double tol, uint64_t seed, double scale);
int stability_batch_smem(tpo_gpu_ctx *ctx, const tpo_gpu_graph *program, const tpo_gpu_graph *const *cands,
                         const uint64_t *seeds, uint64_t n, int32_t trials, double tol, uint64_t seed,
                         double input_scale, int8_t *ok);
}  // namespace

extern "C" {

int tpo_gpu_stability_batch(tpo_gpu_ctx *ctx, const tpo_gpu_graph *program,
                            const tpo_gpu_graph *const *cands, const uint64_t *seeds, uint64_t n,
                            int32_t trials, double tol, uint64_t seed, double input_scale,
                            int8_t *ok) {
  const int rc = stability_batch_smem(ctx, program, cands, seeds, n, trials, tol, seed, input_scale, ok);
  if (rc != 1000 + int(ErrCode::DoesNotFit)) return rc;
  // graphs beyond shared memory: the global-memory fp64 executor, one candidate at a time
  return guard([&] {
    check_cuda(cudaSetDevice(ctx->c.device), "cudaSetDevice");
    for (uint64_t k = 0; k < n; ++k) {
      try {
        ok[k] = stability_global(ctx, program, cands[k], trials, tol, seeds ? seeds[k] : seed, input_scale);
      } catch (const Error &e) {
        if (e.code != ErrCode::ShapeMismatch) throw;
        ok[k] = -1;
      }
    }
    return 0;
  });
}

}  // extern "C"

namespace {
int stability_batch_smem(tpo_gpu_ctx *ctx, const tpo_gpu_graph *program, const tpo_gpu_graph *const *cands,
                         const uint64_t *seeds, uint64_t n, int32_t trials, double tol, uint64_t seed,
                         double input_scale, int8_t *ok) {
  return guard([&] {
    if (n == 0) return 0;
    Ctx &C = ctx->c;
    check_cuda(cudaSetDevice(C.device), "cudaSetDevice");
    const Graph &P = program->g;
    const uint32_t n_in = uint32_t(P.in_elems);
    // program outputs pinned after the inputs; candidate region above them
    VmProgram pp = lower_vm(P.g, 0, n_in, /*pin_outputs=*/true);
    const uint32_t cbase = n_in + pp.pinned_words;
    std::vector<TpoVmInstr> code(pp.code);
    std::vector<TpoVmGraph> graphs;
    TpoVmGraph d0 = pp.desc;
    d0.code_off = 0;
    d0.code_len = uint32_t(pp.code.size());
    graphs.push_back(d0);
    uint64_t maxw = uint64_t(n_in) + pp.region_words;
    uint32_t max_cl = 0;
    std::unordered_map<const tpo_gpu_graph *, uint32_t> idx;
    std::vector<uint32_t> cg(n);
    for (uint64_t k = 0; k < n; ++k) {
      auto it = idx.find(cands[k]);
      if (it == idx.end()) {
        TpoVmGraph d;
        try {
          check_pair(P.g, cands[k]->g.g);
          VmProgram cp = lower_vm(cands[k]->g.g, 0, cbase);
          d = cp.desc;
          d.code_off = uint32_t(code.size());
          d.code_len = uint32_t(cp.code.size());
          code.insert(code.end(), cp.code.begin(), cp.code.end());
          maxw = std::max<uint64_t>(maxw, uint64_t(cbase) + cp.region_words);
          max_cl = std::max(max_cl, d.code_len);
        } catch (const Error &e) {
          d = error_graph(e.code);
        }
        it = idx.emplace(cands[k], uint32_t(graphs.size())).first;
        graphs.push_back(d);
      }
      cg[k] = it->second;
    }
    // bytecode read in place (as the field verifier does) unless
    // TPO_VM_CODE_GLOBAL=0 stages it into shared memory
    const char *cg_env = std::getenv("TPO_VM_CODE_GLOBAL");
    const bool code_in_place = !cg_env || std::atoi(cg_env) != 0;
    const size_t code_bytes = code_in_place ? 0 : size_t(d0.code_len + max_cl) * sizeof(TpoVmInstr);
    const size_t smem = code_bytes + size_t(maxw) * 8;
    if (smem > 232448)
      throw Error(ErrCode::DoesNotFit, "stability working set " + std::to_string(smem) +
                                           " B exceeds 227 KiB of shared memory");
    cudaStream_t st = C.stream;
    auto *dcode = static_cast<TpoVmInstr *>(C.code.get(code.size() * sizeof(TpoVmInstr) + 16));
    auto *dgraphs = static_cast<TpoVmGraph *>(C.graphs.get(graphs.size() * sizeof(TpoVmGraph)));
    auto *dcg = static_cast<uint32_t *>(C.cand.get(n * 4));
    auto *dok = static_cast<int8_t *>(C.verdicts.get(n));
    auto *cnt = static_cast<unsigned long long *>(C.counter.get(16));
    check_cuda(cudaMemcpyAsync(dcode, code.data(), code.size() * sizeof(TpoVmInstr), cudaMemcpyHostToDevice, st), "code");
    check_cuda(cudaMemcpyAsync(dgraphs, graphs.data(), graphs.size() * sizeof(TpoVmGraph), cudaMemcpyHostToDevice, st), "graphs");
    check_cuda(cudaMemcpyAsync(dcg, cg.data(), n * 4, cudaMemcpyHostToDevice, st), "cands");
    check_cuda(cudaMemsetAsync(cnt, 0, 16, st), "counter");
    tpo_fp::StabilityArgs a{};
    a.code = dcode;
    a.graphs = dgraphs;
    a.code_bytes = uint32_t(code_bytes);
    a.cand_graph = dcg;
    if (seeds) {
      auto *ds = static_cast<uint64_t *>(C.seeds.get(n * 8));
      check_cuda(cudaMemcpyAsync(ds, seeds, n * 8, cudaMemcpyHostToDevice, st), "seeds");
      a.seeds = ds;
    }
    a.seed = seed;
    a.n = n;
    a.n_in = n_in;
    a.trials = trials;
    a.tol = tol;
    a.scale = input_scale;
    a.counter = cnt;
    a.ok = dok;
    const int occ = tpo_fp_stability_occupancy(smem);
    if (occ < 1) throw Error(ErrCode::DoesNotFit, "stability kernel does not fit on an SM");
    const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(C.num_sms) * occ, n));
    check_cuda(cudaError_t(tpo_fp_launch_stability(&a, int(grid), smem, st)), "stability launch");
    check_cuda(cudaMemcpyAsync(ok, dok, n, cudaMemcpyDeviceToHost, st), "ok");
    check_cuda(cudaStreamSynchronize(st), "stability sync");
    return 0;
  });
}

}  // namespace

namespace {
// float_stability_filter (stability.cpp:25-50) for graphs beyond shared
// memory: per trial the normals in HBM, program and candidate on the
// global-memory fp64 executor, the comparison as a device flag.
int8_t stability_global(tpo_gpu_ctx *ctx, const tpo_gpu_graph *prog, const tpo_gpu_graph *cand, int trials,
                        double tol, uint64_t seed, double scale) {
  Ctx &C = ctx->c;
  const Graph &P = prog->g, &G = cand->g;
  check_pair(P.g, G.g);
  cudaStream_t st = C.stream;
  double *in = static_cast<double *>(C.vm_in.get(size_t(P.in_elems) * 8 + 16));
  double *ro = static_cast<double *>(C.vm_out.get(size_t(P.out_elems) * 2 * 8 + 16));
  double *co = ro + P.out_elems;
  int *fail = static_cast<int *>(C.status.get(16));
  for (int trial = 0; trial < trials; ++trial) {
    check_cuda(cudaError_t(tpo_fp_launch_normals(in, seed, trial, uint64_t(P.in_elems), scale, C.num_sms, st)),
               "normals");
    int rc = eval_vm_impl(ctx, prog, 0, in, ro, false, st);
    if (!rc) rc = eval_vm_impl(ctx, cand, 0, in, co, false, st);
    if (rc) throw Error(ErrCode::Unsupported, "stability filter: " + std::string(tpo_gpu_last_error()));
    check_cuda(cudaMemsetAsync(fail, 0, 4, st), "flag");
    check_cuda(cudaError_t(tpo_fp_launch_stab_compare(ro, co, uint64_t(P.out_elems), tol, fail, C.num_sms, st)),
               "compare");
    int h = 0;
    check_cuda(cudaMemcpyAsync(&h, fail, 4, cudaMemcpyDeviceToHost, st), "flag");
    check_cuda(cudaStreamSynchronize(st), "sync");
    if (h) return 0;  // stability.cpp returns at the first failing trial
  }
  return 1;
}
}  // namespace

extern "C" {

int tpo_gpu_float_stability_filter(tpo_gpu_ctx *ctx, const tpo_gpu_graph *g,
                                   const tpo_gpu_graph *program, int32_t trials, double tol,
                                   uint64_t seed, double input_scale, int32_t *out_ok) {
  int8_t ok = 0;
  const tpo_gpu_graph *c = g;
  // (beyond shared memory the batch takes the global-memory executor)
  const int rc = tpo_gpu_stability_batch(ctx, program, &c, nullptr, 1, trials, tol, seed, input_scale, &ok);
  if (rc) return rc;
  if (ok < 0) return fail(1000 + int(ErrCode::ShapeMismatch), "candidate does not match the program's interface");
  *out_ok = ok;
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Thread-graph construction over the JSON wire format.
// ---------------------------------------------------------------------------
#include "tpo/ir/fusion.hpp"

extern "C" int tpo_gpu_construct_thread_graphs(const char *json_in, char *json_out, int64_t cap,
                                               int64_t *needed) {
  return guard([&] {
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(json_in);
    } catch (const nlohmann::json::exception &e) {
      throw Error(ErrCode::ParseError, e.what());
    }
    const ir::KernelGraph g = ir::construct_thread_graphs(ir::kernel_graph_from_json(j));
    const std::string s = ir::to_json(g).dump();
    if (needed) *needed = int64_t(s.size()) + 1;
    if (json_out && cap > int64_t(s.size())) std::memcpy(json_out, s.c_str(), s.size() + 1);
    return 0;
  });
}

// ------------------------------------------------- schedule / memory plan
#include "tpo/ir/schedule.hpp"

extern "C" int tpo_gpu_plan_block_graphs(const char *json_in, int64_t smem_bytes, int32_t elem_size,
                                         char *json_out, int64_t cap, int64_t *needed) {
  return guard([&] {
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(json_in);
    } catch (const nlohmann::json::exception &e) {
      throw Error(ErrCode::ParseError, e.what());
    }
    const ir::KernelGraph g = ir::kernel_graph_from_json(j);
    ir::MemLimits lim;
    lim.smem_bytes = smem_bytes > 0 ? smem_bytes : ir::kB200Limits.smem_bytes;
    lim.elem_size = elem_size > 0 ? elem_size : 2;
    nlohmann::json out = nlohmann::json::array();
    for (size_t k = 0; k < g.ops.size(); ++k) {
      const ir::Op &op = g.ops[k];
      if (op.type != ir::OpType::GraphDef || !op.block) continue;
      const ir::Schedule s = ir::schedule_ops(*op.block);
      const ir::MemoryPlan m = ir::plan_memory(*op.block, s, lim);
      out.push_back({{"op", int(k)},
                     {"order", s.order},
                     {"depth", s.depth},
                     {"post", s.post},
                     {"sync_after", s.sync_after},
                     {"syncs", s.sync_after.size()},
                     {"offset", m.offset},
                     {"peak", m.peak},
                     {"exhaustive", m.exhaustive}});
    }
    const std::string str = nlohmann::json{{"graphdefs", out}}.dump();
    if (needed) *needed = int64_t(str.size()) + 1;
    if (json_out && cap > int64_t(str.size())) std::memcpy(json_out, str.c_str(), str.size() + 1);
    return 0;
  });
}

extern "C" int tpo_gpu_plan_intervals(int32_t n, const int64_t *size, const int64_t *start,
                                      const int64_t *end, int32_t exhaustive_max, int64_t *offset,
                                      int64_t *peak, int32_t *exhaustive) {
  return guard([&] {
    if (n < 0 || (n && (!size || !start || !end || !offset)))
      throw Error(ErrCode::ShapeMismatch, "plan_intervals: bad arguments");
    std::vector<ir::Lifetime> b(static_cast<size_t>(n));
    for (int32_t i = 0; i < n; ++i) {
      if (size[i] < 0 || end[i] < start[i]) throw Error(ErrCode::ShapeMismatch, "plan_intervals: bad lifetime");
      b[size_t(i)] = {size[i], start[i], end[i]};
    }
    const ir::MemoryPlan m = ir::plan_intervals(b, exhaustive_max);
    for (int32_t i = 0; i < n; ++i) offset[i] = m.offset[size_t(i)];
    if (peak) *peak = m.peak;
    if (exhaustive) *exhaustive = m.exhaustive;
    return 0;
  });
}

// ------------------------------------------------------------- describe
namespace tpo::gpu {
std::string describe(const ir::KernelGraph &g, const ir::MemLimits &lim);
}

extern "C" int tpo_gpu_describe(const char *json_in, int64_t smem_bytes, char *text_out, int64_t cap,
                                int64_t *needed) {
  return guard([&] {
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(json_in);
    } catch (const nlohmann::json::exception &e) {
      throw Error(ErrCode::ParseError, e.what());
    }
    ir::MemLimits lim;
    lim.smem_bytes = smem_bytes > 0 ? smem_bytes : ir::kB200Limits.smem_bytes;
    const std::string str = tpo::gpu::describe(ir::kernel_graph_from_json(j), lim);
    if (needed) *needed = int64_t(str.size()) + 1;
    if (text_out && cap > int64_t(str.size())) std::memcpy(text_out, str.c_str(), str.size() + 1);
    return 0;
  });
}

// ----------------------------------------------- wire-format parity (debug)
extern "C" int tpo_gpu_parse_check(const char *json_in, int32_t *fast_accepted, int32_t *same) {
  return guard([&] {
    ir::KernelGraph a;
    const bool fast = ir::kernel_graph_from_text_fast(json_in, std::strlen(json_in), a);
    if (fast_accepted) *fast_accepted = fast;
    if (same) *same = 0;
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(json_in);
    } catch (const nlohmann::json::exception &e) {
      throw Error(ErrCode::ParseError, e.what());
    }
    const ir::KernelGraph b = ir::kernel_graph_from_json(j);
    if (fast && same) {
      bool eq = ir::to_json(a).dump() == ir::to_json(b).dump() && a.tensors.size() == b.tensors.size();
      for (size_t t = 0; eq && t < a.tensors.size(); ++t)
        eq = a.tensors[t].producer_op == b.tensors[t].producer_op &&
             a.tensors[t].producer_out == b.tensors[t].producer_out;
      *same = eq;
    }
    return 0;
  });
}

// ------------------------------------------------------------- generator
#include "tpo/ir/generator.hpp"

namespace {
ir::EnumConfig enum_config(const char *config_json) {
  nlohmann::json c;
  try {
    c = config_json && *config_json ? nlohmann::json::parse(config_json) : nlohmann::json::object();
  } catch (const nlohmann::json::exception &e) {
    throw Error(ErrCode::ParseError, e.what());
  }
  ir::EnumConfig cfg;
  if (c.contains("grids")) cfg.grids = c.at("grids").get<std::vector<int64_t>>();
  if (c.contains("loops")) cfg.loops = c.at("loops").get<std::vector<int64_t>>();
  if (c.contains("max_block_ops")) cfg.max_block_ops = c.at("max_block_ops").get<int>();
  if (c.contains("max_kernel_ops")) cfg.max_kernel_ops = c.at("max_kernel_ops").get<int>();
  if (c.contains("max_loop_labels")) cfg.max_loop_labels = c.at("max_loop_labels").get<int>();
  if (c.contains("concat_matmul")) cfg.concat_matmul = c.at("concat_matmul").get<bool>();
  if (c.contains("max_candidates")) cfg.max_candidates = c.at("max_candidates").get<size_t>();
  if (c.contains("max_prefixes")) cfg.max_prefixes = c.at("max_prefixes").get<uint64_t>();
  if (c.contains("threads")) cfg.threads = c.at("threads").get<int>();
  if (c.contains("smem_bytes")) cfg.limits.smem_bytes = c.at("smem_bytes").get<int64_t>();
  return cfg;
}

nlohmann::json enum_stats_json(const ir::EnumStats &st) {
  return {{"kernel_prefixes", st.kernel_prefixes}, {"partitions", st.partitions}, {"prefixes", st.prefixes},
          {"pruned_expr", st.pruned_expr},         {"pruned_shape", st.pruned_shape},
          {"pruned_memory", st.pruned_memory},     {"pruned_structure", st.pruned_structure},
          {"completed", st.completed},             {"rejected_validate", st.rejected_validate},
          {"duplicates", st.duplicates},           {"budget_exhausted", st.budget_exhausted}};
}
}  // namespace

extern "C" int tpo_gpu_enumerate(const char *program_json, const char *config_json, char *json_out, int64_t cap,
                                 int64_t *needed) {
  return guard([&] {
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(program_json);
    } catch (const nlohmann::json::exception &e) {
      throw Error(ErrCode::ParseError, e.what());
    }
    ir::EnumStats st;
    const auto cands = ir::enumerate_mugraphs(ir::kernel_graph_from_json(j), enum_config(config_json), &st);
    nlohmann::json arr = nlohmann::json::array();
    for (const auto &g : cands) arr.push_back(ir::to_json(g));
    const std::string s = nlohmann::json{{"candidates", arr}, {"stats", enum_stats_json(st)}}.dump();
    if (needed) *needed = int64_t(s.size()) + 1;
    if (json_out && cap > int64_t(s.size())) std::memcpy(json_out, s.c_str(), s.size() + 1);
    return 0;
  });
}

extern "C" int tpo_gpu_search(tpo_gpu_ctx *ctx, const tpo_gpu_graph *program, const char *config_json,
                              const tpo_verify_cfg *cfg, const tpo_field_params *fp, tpo_gpu_graph **accepted,
                              int64_t cap, int64_t *n_accepted, tpo_search_stats *stats) {
  return guard([&] {
    if (!ctx || !program || !cfg || !fp) throw Error(ErrCode::ConfigError, "search: null argument");
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    ir::EnumStats est;
    std::vector<ir::KernelGraph> cands = ir::enumerate_mugraphs(program->g.g, enum_config(config_json), &est);
    const auto t1 = clk::now();
    // candidates become handles directly: no wire format; enumerated graphs
    // are valid by construction, the fused-kernel match waits for acceptance
    const int64_t n = int64_t(cands.size());
    std::vector<std::unique_ptr<tpo_gpu_graph>> hs(static_cast<size_t>(n));
    parallel_for(n, n >= 64 ? host_threads() : 1, [&](int64_t i) {
      auto h = std::make_unique<tpo_gpu_graph>();
      h->g.g = std::move(cands[size_t(i)]);
      finish_graph(h->g, false);
      hs[size_t(i)] = std::move(h);
    });
    const auto t2 = clk::now();
    std::vector<tpo_verdict> v(static_cast<size_t>(n));
    std::vector<const tpo_gpu_graph *> hp(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) hp[size_t(i)] = hs[size_t(i)].get();
    // the search loop's single VerifyConfig: cfg->seed for every candidate
    if (n) {
      const int rc = tpo_gpu_verify_batch(ctx, program, hp.data(), nullptr, uint64_t(n), cfg, fp, v.data(), nullptr);
      if (rc) throw Error(ErrCode::Unsupported, std::string("search verify: ") + tpo_gpu_last_error());
    }
    const auto t3 = clk::now();
    int64_t acc = 0, kinds[4] = {0, 0, 0, 0};
    for (int64_t i = 0; i < n; ++i) {
      const int k = v[size_t(i)].kind;
      if (k >= 0 && k < 4) ++kinds[k];
      if (k != 0) continue;
      if (accepted && acc < cap) {
        Graph &G = hs[size_t(i)]->g;
        G.fused_plan();
        accepted[acc] = hs[size_t(i)].release();
      }
      ++acc;
    }
    if (n_accepted) *n_accepted = acc;
    if (stats) {
      *stats = tpo_search_stats{};
      stats->candidates = n;
      stats->equivalent = kinds[0];
      stats->not_equivalent = kinds[1];
      stats->inconclusive = kinds[2];
      stats->errors = kinds[3];
      stats->prefixes = int64_t(est.prefixes);
      stats->partitions = int64_t(est.partitions);
      stats->pruned_expr = int64_t(est.pruned_expr);
      stats->budget_exhausted = est.budget_exhausted;
      stats->enumerate_s = std::chrono::duration<double>(t1 - t0).count();
      stats->compile_s = std::chrono::duration<double>(t2 - t1).count();
      stats->verify_s = std::chrono::duration<double>(t3 - t2).count();
    }
    return 0;
  });
}

extern "C" int tpo_gpu_graph_json(const tpo_gpu_graph *h, char *json_out, int64_t cap, int64_t *needed) {
  return guard([&] {
    if (!h) throw Error(ErrCode::ConfigError, "null graph");
    const std::string s = ir::to_json(h->g.g).dump();
    if (needed) *needed = int64_t(s.size()) + 1;
    if (json_out && cap > int64_t(s.size())) std::memcpy(json_out, s.c_str(), s.size() + 1);
    return 0;
  });
}

extern "C" int tpo_gpu_abstract_expression(const char *graph_json, char *out, int64_t cap, int64_t *needed) {
  return guard([&] {
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(graph_json);
    } catch (const nlohmann::json::exception &e) {
      throw Error(ErrCode::ParseError, e.what());
    }
    const std::string s = ir::abstract_expression(ir::kernel_graph_from_json(j));
    if (needed) *needed = int64_t(s.size()) + 1;
    if (out && cap > int64_t(s.size())) std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
  });
}

extern "C" int tpo_gpu_generate(const char *program_json, const char *config_json, char *json_out,
                                int64_t cap, int64_t *needed) {
  return guard([&] {
    nlohmann::json j, c;
    try {
      j = nlohmann::json::parse(program_json);
      c = config_json && *config_json ? nlohmann::json::parse(config_json) : nlohmann::json::object();
    } catch (const nlohmann::json::exception &e) {
      throw Error(ErrCode::ParseError, e.what());
    }
    ir::GenConfig cfg;
    if (c.contains("grids")) cfg.grids = c.at("grids").get<std::vector<int64_t>>();
    if (c.contains("loops")) cfg.loops = c.at("loops").get<std::vector<int64_t>>();
    if (c.contains("rewrite")) cfg.rewrite = c.at("rewrite").get<bool>();
    if (c.contains("max_candidates")) cfg.max_candidates = c.at("max_candidates").get<size_t>();
    if (c.contains("smem_bytes")) cfg.limits.smem_bytes = c.at("smem_bytes").get<int64_t>();
    if (c.contains("max_kernels")) cfg.max_kernels = c.at("max_kernels").get<int>();
    if (c.contains("per_segment")) cfg.per_segment = c.at("per_segment").get<int>();
    ir::GenStats st;
    const auto cands = ir::generate_multi(ir::kernel_graph_from_json(j), cfg, &st);
    nlohmann::json arr = nlohmann::json::array();
    for (const auto &g : cands) arr.push_back(ir::to_json(g));
    const std::string s = nlohmann::json{{"candidates", arr},
                                         {"stats",
                                          {{"partitions", st.partitions},
                                           {"placements", st.placements},
                                           {"rejected_structure", st.rejected_structure},
                                           {"rejected_validate", st.rejected_validate},
                                           {"duplicates", st.duplicates}}}}
                              .dump();
    if (needed) *needed = int64_t(s.size()) + 1;
    if (json_out && cap > int64_t(s.size())) std::memcpy(json_out, s.c_str(), s.size() + 1);
    return 0;
  });
}
