/* tpo_gpu.h — C-ABI of the B200 µGraph evaluation backend.
 *
 * Drop-in boundary for the reference's µGraph evaluation hot path
 * (/root/reference/proj/core).  Plain C: opaque handles, plain pointers and
 * sizes, no exceptions across the ABI.  Every entry point returns 0 on
 * success or a status:
 *     1000 + tpo::ErrCode ordinal  (reference proj/core/include/tpo/ir/shape.hpp:27-42)
 *     2000 + ErrCode               "resample needed" (DivByZero / NonResidue) for the
 *                                   single-attempt debug entry point
 *     3000 + cudaError_t            CUDA failure
 * and tpo_gpu_last_error() returns the message of the calling thread's last
 * failure.  A context is bound to one device and one CUDA stream; use one
 * context per host thread for concurrency (the reference API is pure and
 * re-entrant).
 *
 * Reference interfaces replaced (file:line in /root/reference):
 *   tpo_gpu_eval_mugraph(_host)     <- tpo::interp::eval_mugraph
 *                                      proj/core/include/tpo/interp/interp.hpp:47-48
 *   tpo_gpu_ff_eval                 <- tpo::verify::ff_eval (+ sample_inputs, sample_omega,
 *                                      SiluTables::sample) proj/core/include/tpo/verify/ffeval.hpp:58-67,
 *                                      proj/core/src/equiv.cpp:57-68
 *   tpo_gpu_random_test_equivalence <- tpo::verify::random_test_equivalence
 *                                      proj/core/include/tpo/verify/equiv.hpp:50-53
 *   tpo_gpu_verify_batch/_pool      <- the search loop's per-candidate calls of the same
 *                                      (SPEC.md:664-668), batched
 *   tpo_gpu_compile                 <- tpo::ir::kernel_graph_from_json + tpo::ir::validate
 *                                      proj/core/include/tpo/ir/serialize.hpp:33-34,
 *                                      proj/core/include/tpo/ir/validate.hpp:51
 *   tpo_gpu_validate                <- tpo::ir::validate (B200 MemLimits)
 *   tpo_gpu_op_madds                <- tpo::ir::op_madds summed over a µGraph
 *                                      proj/core/include/tpo/ir/shape_infer.hpp:67-69
 *   tpo_gpu_eval_vm                 <- tpo::interp::eval_mugraph / eval_program / eval_mugraph_f32
 *                                      (generic GPU VM) proj/core/include/tpo/interp/interp.hpp:41-53
 *   tpo_gpu_float_stability_filter  <- tpo::verify::float_stability_filter
 *   tpo_gpu_stability_batch            proj/core/include/tpo/verify/stability.hpp:29-31
 */
#ifndef TPO_GPU_H
#define TPO_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPO_GPU_ABI_VERSION 1

typedef struct tpo_gpu_ctx tpo_gpu_ctx;
typedef struct tpo_gpu_graph tpo_gpu_graph;

/* FieldParams(p, q, omega_base) — proj/core/include/tpo/verify/field.hpp:50-79 */
typedef struct {
  uint32_t p, q, omega_base;
} tpo_field_params;

/* VerifyConfig — proj/core/include/tpo/verify/equiv.hpp:25-30 */
typedef struct {
  int32_t num_tests;
  int32_t max_resamples;
  uint64_t seed;
  double float_tolerance;
} tpo_verify_cfg;

/* EquivVerdict + Witness — proj/core/include/tpo/verify/equiv.hpp:32-45 (48 bytes) */
typedef struct {
  int32_t kind; /* 0 Equivalent, 1 NotEquivalent, 2 Inconclusive, 3 Error (err_code) */
  int32_t rounds_run;
  int32_t resamples;
  int32_t has_witness;
  uint64_t w_seed;
  int32_t w_round;
  uint32_t w_omega;
  int32_t w_tensor;
  int32_t err_code;
  int64_t w_index;
} tpo_verdict;

/* Lowering chosen for a compiled graph by tpo_gpu_eval_mugraph. */
enum {
  TPO_FUSED_NONE = 0, /* generic VM path only */
  TPO_FUSED_RMSNORM_MATMUL = 1,
  TPO_FUSED_GATED_MLP = 2,
  TPO_FUSED_GQA_DECODE = 3,
  TPO_FUSED_LORA = 4,
};

enum { TPO_DTYPE_F32 = 0, TPO_DTYPE_BF16 = 1, TPO_DTYPE_F64 = 2 };

/* Precision policy of the fused kernels (tpo_gpu_graph_set_precision).
 * The reference evaluates in double (interp.hpp:47-48); the fused kernels
 * multiply bf16 operands on the tensor cores with fp32 accumulation.
 *   TPO_PREC_AUTO (default): all-bf16 inputs run the bf16 kernel (bf16 x
 *     bf16 products are exact in fp32).  Any fp32 / fp64 input selects the
 *     SPLIT kernel: every operand enters as bf16 hi + lo (x = hi + lo to
 *     ~2^-16 relative), all hi/lo products accumulate in fp32, so the
 *     result meets |o - r| <= 1e-3 * max(|r|, rms(r)) against the double
 *     reference on arbitrary inputs (tests/test_precision_gpu.py), at twice
 *     the weight bytes of the bf16 kernel.
 *   TPO_PREC_BF16: round every input to bf16 and run the bf16 kernel (the
 *     fast path for callers whose operands are bf16 by construction).
 *   TPO_PREC_VM: no fused kernel — the generic GPU VM in the reference's
 *     operation order (fp64 for fp64 inputs, else fp32 semantics). */
enum { TPO_PREC_AUTO = 0, TPO_PREC_BF16 = 1, TPO_PREC_VM = 2 };

typedef struct {
  int32_t n_inputs, n_outputs;
  int32_t fused_kind;      /* TPO_FUSED_* */
  int32_t lax;             /* 1 when no EwExp consumes an exponentiated value */
  int64_t madds;           /* reference op_madds work of the graph */
  int64_t input_elems;     /* total elements over all inputs */
  int64_t output_elems;
  int64_t vm_words;        /* verifier VM words (inputs + graph region); -1 if not lowerable */
} tpo_graph_info;

int tpo_gpu_abi_version(void);
const char *tpo_gpu_last_error(void);

int tpo_gpu_open(int device, tpo_gpu_ctx **out);
void tpo_gpu_close(tpo_gpu_ctx *ctx);

/* Parse (serialize.hpp schema), validate against B200 limits (227 KiB smem),
 * lower.  The handle owns host IR + lowering plans; device bytecode is
 * uploaded per batch. */
int tpo_gpu_compile(tpo_gpu_ctx *ctx, const char *graph_json, tpo_gpu_graph **out);

/* tpo_gpu_compile of n graphs on `threads` host threads (<= 0: all cores) —
 * the search loop's candidate stream (each candidate is a distinct graph, so
 * host-side parsing and lowering, not the GPU, bound the batch).  out[i]
 * receives the handle or NULL, status[i] the per-graph status (0 or
 * 1000 + ErrCode); returns nonzero only for bad arguments. */
int tpo_gpu_compile_many(tpo_gpu_ctx *ctx, const char *const *graph_json, int64_t n, int32_t threads,
                         tpo_gpu_graph **out, int32_t *status);
void tpo_gpu_graph_free(tpo_gpu_graph *g);
int tpo_gpu_graph_info(const tpo_gpu_graph *g, tpo_graph_info *out);
/* Declares graph inputs (bit i = input i) as static parameters: never
 * written by work enqueued on the stream before an evaluation (weights).  A
 * fused kernel may then start streaming them before its programmatic
 * dependency on the preceding kernel resolves (PDL), overlapping
 * back-to-back evaluations.  Default 0: every input is ordered after the
 * preceding work.  No reference counterpart (a launch-time property). */
int tpo_gpu_graph_set_static_inputs(tpo_gpu_graph *g, uint64_t mask);

/* Sets the graph's TPO_PREC_* policy (default TPO_PREC_AUTO). */
int tpo_gpu_graph_set_precision(tpo_gpu_graph *g, int32_t policy);

/* Shape of input/output `index` (is_output 0/1): writes rank dims, returns rank or <0. */
int tpo_gpu_graph_shape(const tpo_gpu_graph *g, int is_output, int index, int64_t *dims);

/* validate(g, {smem_bytes, 512, elem_size}); returns number of violations
 * (>= 0) with details in `buf`, or a status (>= 1000) on parse errors. */
int tpo_gpu_validate(const char *graph_json, int64_t smem_bytes, int64_t elem_size, char *buf,
                     int cap);

/* Floating-point µGraph evaluation on device buffers (row-major, caller
 * owns).  Inputs are TPO_DTYPE_BF16, _F32 or _F64 per `in_dtype`; outputs
 * fp32.  Benchmark µGraphs run as one fused sm_100a kernel (fused_kind != 0)
 * under the graph's precision policy (TPO_PREC_*: bf16 operands for bf16
 * inputs, split hi + lo operands for fp32 / fp64 inputs); any other µGraph,
 * or TPO_PREC_VM, runs on the generic GPU VM in the reference's operation
 * order: fp64 arithmetic (eval_mugraph, interp.hpp:47-48) when an input is
 * fp64, else fp32 (eval_mugraph_f32, interp.hpp:51-53).  Operand conversions
 * use context scratch.  Enqueued on `cuda_stream` (NULL = the legacy default
 * stream); asynchronous. */
int tpo_gpu_eval_mugraph(tpo_gpu_ctx *ctx, const tpo_gpu_graph *g, const void *const *in_dev,
                         const int32_t *in_dtype, float *const *out_dev, void *cuda_stream);

/* Same evaluation from and to HOST buffers (pageable or pinned): inputs are
 * copied host->device in their dtype, converted on the device as the
 * precision policy requires, evaluated, and the fp32 outputs copied back;
 * synchronous on `cuda_stream` (NULL = the context stream). */
int tpo_gpu_eval_mugraph_host(tpo_gpu_ctx *ctx, const tpo_gpu_graph *g, const void *const *in_host,
                              const int32_t *in_dtype, float *const *out_host, void *cuda_stream);

/* The exact types of tpo::interp::eval_mugraph
 * (proj/core/include/tpo/interp/interp.hpp:47-48): fp64 host tensors in,
 * fp64 host tensors out.  A fused µGraph runs its SPLIT kernel (TPO_PREC_AUTO;
 * tolerance above; TPO_PREC_BF16 rounds instead), any other µGraph — or
 * TPO_PREC_VM — the generic VM in double arithmetic, bit-identical to the
 * reference except exp / SiLU (last ulp).  Synchronous. */
int tpo_gpu_eval_mugraph_f64(tpo_gpu_ctx *ctx, const tpo_gpu_graph *g, const double *const *in_host,
                             double *const *out_host, void *cuda_stream);

/* One verifier attempt for one graph, exactly as equiv.cpp:57-68 draws it
 * (Rng::derive(seed, stream); inputs; omega; SiLU tables iff with_silu).
 * Outputs are concatenated over the graph outputs.  in_xp/in_xq (nullable)
 * receive the sampled inputs.  Returns 0, or 2000 + ErrCode when an undefined
 * field op requires a resample. */
int tpo_gpu_ff_eval(tpo_gpu_ctx *ctx, const tpo_gpu_graph *g, const tpo_field_params *fp,
                    uint64_t seed, uint64_t stream, int32_t with_silu, uint16_t *out_xp,
                    uint16_t *out_xq, uint8_t *out_qd, uint32_t *omega_out, uint16_t *in_xp,
                    uint16_t *in_xq);

/* random_test_equivalence(g1, g2, cfg, fp) on the GPU. */
int tpo_gpu_random_test_equivalence(tpo_gpu_ctx *ctx, const tpo_gpu_graph *g1,
                                    const tpo_gpu_graph *g2, const tpo_verify_cfg *cfg,
                                    const tpo_field_params *fp, tpo_verdict *out);

/* Batched verification: candidate k (k < n) is checked against `program`
 * with cfg {num_tests, seeds[k], max_resamples} (seeds NULL: cfg->seed for
 * every candidate, whatever executor the graphs need); one verdict per candidate
 * (host array, nullable) and packed accept bits (host, nullable; bit k set
 * iff Equivalent). */
int tpo_gpu_verify_batch(tpo_gpu_ctx *ctx, const tpo_gpu_graph *program,
                         const tpo_gpu_graph *const *cands, const uint64_t *seeds, uint64_t n,
                         const tpo_verify_cfg *cfg, const tpo_field_params *fp,
                         tpo_verdict *verdicts, uint32_t *accept_bits);

/* Sharding form: candidate i in [first, first + n) is pool[i % pool_n] with
 * seed i.  `accept_dev` (nullable) is a DEVICE buffer of ceil(n/32) words
 * receiving accept bits (ready for a collective gather); `verdicts` (host,
 * nullable); `attempts` (host, nullable) receives the attempts consumed.
 * Runs on `cuda_stream` (null: the context stream) and synchronises. */
int tpo_gpu_verify_pool(tpo_gpu_ctx *ctx, const tpo_gpu_graph *program,
                        const tpo_gpu_graph *const *pool, int32_t pool_n, uint64_t first,
                        uint64_t n, const tpo_verify_cfg *cfg, const tpo_field_params *fp,
                        uint32_t *accept_dev, tpo_verdict *verdicts, uint64_t *attempts,
                        void *cuda_stream);

/* splitmix64 draws made by the context's last tpo_gpu_verify_pool call that
 * requested `attempts` (2 per input element drawn, omega, the SiLU tables):
 * the verifier's RNG work term.  Inputs are drawn lazily — an
 * attempt the program resamples before an input's first reader never draws
 * it — so this is the work actually done, not 2 x inputs x attempts.
 * Replaces: no reference counterpart (instrumentation). */
int tpo_gpu_verify_draws(tpo_gpu_ctx *ctx, uint64_t *draws);

/* Generic floating-point evaluation on the GPU µGraph VM (any graph; working
 * sets that fit shared memory run in one CTA, larger ones on the
 * global-memory executor, one grid-wide launch per VM instruction),
 * semantics of the reference evaluator:
 *   mode 0  tpo::interp::eval_mugraph      (double)   interp.hpp:47-48
 *   mode 1  tpo::interp::eval_program      (double; rejects GraphDefs) interp.hpp:41-42
 *   mode 2  tpo::interp::eval_mugraph_f32  (float)    interp.hpp:51-53
 * Inputs / outputs are HOST arrays of double (float for mode 2), inputs
 * concatenated in graph-input order, outputs in graph-output order.
 * Matmul/Sum/Accum accumulate in the reference's order with individually
 * rounded ops (no FMA): add/mul/div/sqrt results are bit-identical to the
 * reference; exp/SiLU may differ in the last ulp. */
int tpo_gpu_eval_vm(tpo_gpu_ctx *ctx, const tpo_gpu_graph *g, int32_t mode, const void *in_host,
                    void *out_host);

/* tpo_gpu_eval_vm on device buffers (inputs concatenated in graph-input
 * order, outputs concatenated; fp64, or fp32 for mode 2), asynchronous on
 * cuda_stream (NULL: the legacy stream). */
int tpo_gpu_eval_vm_dev(tpo_gpu_ctx *ctx, const tpo_gpu_graph *g, int32_t mode, const void *in_dev,
                        void *out_dev, void *cuda_stream);

/* tpo::verify::float_stability_filter(g, program, trials, tol, seed, input_scale)
 * proj/core/include/tpo/verify/stability.hpp:29-31 on the GPU; *out_ok = 1/0. */
int tpo_gpu_float_stability_filter(tpo_gpu_ctx *ctx, const tpo_gpu_graph *g,
                                   const tpo_gpu_graph *program, int32_t trials, double tol,
                                   uint64_t seed, double input_scale, int32_t *out_ok);

/* The same for n candidates in one launch: ok[k] = 1 pass, 0 fail, -1 the
 * candidate's interface differs from the program's.  seeds (nullable): a
 * seed per candidate, else `seed` for all (the reference default is 17). */
int tpo_gpu_stability_batch(tpo_gpu_ctx *ctx, const tpo_gpu_graph *program,
                            const tpo_gpu_graph *const *cands, const uint64_t *seeds, uint64_t n,
                            int32_t trials, double tol, uint64_t seed, double input_scale,
                            int8_t *ok);

/* Thread-graph construction (the reference's absent fusion.cpp):
 * greedily fuses maximal single-consumer chains of elementwise block ops of
 * every GraphDef into ThreadGroups (register-resident interior edges).
 * Writes the resulting graph JSON into json_out when cap suffices; *needed
 * receives the byte count including the terminator. */
int tpo_gpu_construct_thread_graphs(const char *json_in, char *json_out, int64_t cap,
                                    int64_t *needed);

/* Post-verification block-graph planning (the reference's absent
 * schedule.cpp / memplan.cpp, proj/core/CMakeLists.txt:19-20):
 * for every GraphDef, the depth schedule (SPEC schedule_ops: ops ascending by
 * longest-path depth per phase, sync points only between depth levels) and
 * the shared-memory plan over its lifetimes (SPEC plan_memory: exhaustive
 * for <= 8 tensors, first-fit-decreasing above).  Output JSON:
 * {"graphdefs": [{"op", "order", "depth", "post", "sync_after", "syncs",
 * "offset" (bytes per block tensor, -1 = register), "peak", "exhaustive"}]}.
 * smem_bytes <= 0 selects the B200 limit (232448); elem_size <= 0 selects 2.
 * Returns 1000 + DoesNotFit when a plan exceeds smem_bytes. */
int tpo_gpu_plan_block_graphs(const char *json_in, int64_t smem_bytes, int32_t elem_size,
                              char *json_out, int64_t cap, int64_t *needed);

/* The planner on explicit lifetimes: n buffers of size[i] live over the
 * inclusive positions [start[i], end[i]]; writes offset[i], *peak and
 * *exhaustive (1 when every placement order was tried). */
int tpo_gpu_plan_intervals(int32_t n, const int64_t *size, const int64_t *start, const int64_t *end,
                           int32_t exhaustive_max, int64_t *offset, int64_t *peak,
                           int32_t *exhaustive);

/* `describe` (the reference's absent describe.cpp): a
 * human-readable pseudo-kernel listing — per kernel op its grid, for-loop,
 * InIter/Accum/OutSaver maps, the block ops in schedule order with sync
 * markers and shared-memory offsets — followed by how the B200 backend runs
 * the graph (the fused kernel it matches, else VM instructions, barrier
 * phases and working set).  An empty graph yields an empty listing.
 * smem_bytes <= 0 selects the B200 limit. */
int tpo_gpu_describe(const char *json_in, int64_t smem_bytes, char *text_out, int64_t cap,
                     int64_t *needed);

/* Debug / parity of the JSON fast path (host/fastjson.cpp): parses
 * json_in with the fast path and with the generic parser; *fast_accepted =
 * 1 if the fast path took it, *same = 1 if both give the identical graph.
 * Returns the generic parser's status (1000 + ParseError on invalid text). */
int tpo_gpu_parse_check(const char *json_in, int32_t *fast_accepted, int32_t *same);

/* Fused-kernel candidate generator (first slice of the reference's absent
 * generator.cpp): single-GraphDef µGraphs for a
 * single-output computation graph, by enumerating grid / for-loop
 * partitions of its dimension labels and placing φ-Accums by partition
 * state (tpo/ir/generator.hpp); with "max_kernels" > 1 also µGraphs of up
 * to that many kernels chained through device tensors (contiguous
 * single-output segments of the op list, each a pre-defined kernel op or
 * one of its first "per_segment" fused GraphDefs; Algorithm 1's kernel
 * level).  config_json (nullable): {"grids": [..], "loops": [..],
 * "rewrite": bool, "max_candidates": n, "smem_bytes": n, "max_kernels": n,
 * "per_segment": n}.
 * Output JSON: {"candidates": [graph, ...], "stats": {...}}; every candidate
 * passes validate; equivalence is the verifier's job. */
int tpo_gpu_generate(const char *program_json, const char *config_json, char *json_out, int64_t cap,
                     int64_t *needed);

/* Algorithm 1 (§4; the reference's absent
 * generator.cpp): µGraphs generated op by op in canonical form — up to
 * "max_kernel_ops" pre-defined kernel operators, then one graph-defined
 * operator whose block graph is enumerated operator by operator over every
 * grid / for-loop partition — pruned by abstract expressions (a prefix's
 * expression must be a subexpression of the program's, Tables 2-3),
 * shape and shared memory.  config_json (nullable): {"grids", "loops",
 * "max_block_ops", "max_kernel_ops", "max_loop_labels", "concat_matmul",
 * "max_candidates", "max_prefixes", "threads", "smem_bytes"}.  Output JSON:
 * {"candidates": [graph, ...], "stats": {...}}; every candidate is valid and
 * carries the program's abstract expression — equivalence is the verifier's. */
int tpo_gpu_enumerate(const char *program_json, const char *config_json, char *json_out, int64_t cap,
                      int64_t *needed);

/* The abstract expression of a graph's first output (normal form text). */
int tpo_gpu_abstract_expression(const char *graph_json, char *text_out, int64_t cap, int64_t *needed);

typedef struct {
  int64_t candidates, equivalent, not_equivalent, inconclusive, errors;
  int64_t prefixes, partitions, pruned_expr;
  int32_t budget_exhausted, pad;
  double enumerate_s, compile_s, verify_s;  /* host enumeration, handle construction, GPU verification */
} tpo_search_stats;

/* The search loop end to end (SPEC.md:664-668 generate -> verify): the
 * candidates of tpo_gpu_enumerate become graph handles directly (no wire
 * format) and are verified in one batch against `program` with `cfg`
 * (cfg->seed for every candidate: the loop's single VerifyConfig).
 * accepted (nullable) receives up to `cap` handles of the Equivalent
 * candidates (caller frees them); *n_accepted their count. */
int tpo_gpu_search(tpo_gpu_ctx *ctx, const tpo_gpu_graph *program, const char *config_json,
                   const tpo_verify_cfg *cfg, const tpo_field_params *fp, tpo_gpu_graph **accepted,
                   int64_t cap, int64_t *n_accepted, tpo_search_stats *stats);

/* A handle's graph in the wire format (serialize.hpp schema). */
int tpo_gpu_graph_json(const tpo_gpu_graph *g, char *json_out, int64_t cap, int64_t *needed);

/* Reference op_madds work of a graph (SURVEY §8d verifier work unit). */
int64_t tpo_gpu_op_madds(const tpo_gpu_graph *g);

#ifdef __cplusplus
}
#endif
#endif /* TPO_GPU_H */
