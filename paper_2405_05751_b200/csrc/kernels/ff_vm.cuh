// B200 backend — launch contract of the batched finite-field verifier.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "vm.h"

// Identical layout to tpo_verdict in include/tpo_gpu.h (48 bytes).
struct TpoVerdict {
  int32_t kind;  // 0 Equivalent, 1 NotEquivalent, 2 Inconclusive, 3 Error
  int32_t rounds_run;
  int32_t resamples;
  int32_t has_witness;
  uint64_t w_seed;
  int32_t w_round;
  uint32_t w_omega;
  int32_t w_tensor;
  int32_t err_code;
  int64_t w_index;
};

namespace tpo_ff {

constexpr int kThreads = 256;

struct FieldConst {
  uint32_t p, q, wbase;
  uint32_t magic_p, magic_q;   // floor(2^32 / p), floor(2^32 / q)
  uint32_t two32_p, two32_q;   // 2^32 mod p, 2^32 mod q
  uint32_t lazy, lazy_sum;     // products / values summable before a reduction
  uint32_t table_bytes;        // smem bytes of the field tables (16-B aligned)
  uint64_t thr_p, thr_q;       // uniform() rejection thresholds (2^64 - n) mod n
  // p, q < 256: a 64-bit draw r = A*2^48 + B*2^24 + C reduces as
  // A*k48 + B*k24 + C < 2^32 (k24 = 2^24 mod n, k48 = 2^48 mod n), one mod32
  uint32_t k24_p, k48_p, k24_q, k48_q;
  uint32_t small;
};

struct VerifyArgs {
  FieldConst field;
  const uint16_t *tables;        // inv_p, inv_q, sqrt_p, sqrt_q
  const TpoVmInstr *code;
  const TpoVmGraph *graphs;
  uint32_t program;              // index of the program graph in `graphs`
  const uint32_t *pool;          // pool mode: candidate graph = pool[(first+k) % pool_n]
  uint32_t pool_n;
  const uint32_t *cand_graph;    // explicit mode (non-null): graph index per candidate
  const uint64_t *seeds;         // explicit seeds (null: seed = first + k)
  uint64_t first, n;
  uint32_t n_in;                 // input elements (shared by both graphs)
  int num_tests, max_resamples;
  unsigned long long *counter;   // work queue head
  TpoVerdict *verdicts;          // optional
  uint32_t *accept;              // optional packed accept bits (Equivalent)
  unsigned long long *work;      // optional: attempts actually consumed
  unsigned long long *prof;      // optional (TPO_VM_PROFILE): [16] cycles, [16] counts per opcode
  uint32_t code_smem_bytes;      // smem staging of program + candidate bytecode
  uint32_t code_global;          // 1: bytecode read in place from `code` (no smem staging)
  // Same-seed batches (a search loop verifying every candidate with the
  // VerifyConfig seed): attempt (shared_seed, round 0, attempt 0) is
  // generated and the program evaluated ONCE (shared_attempt_kernel); the
  // candidates copy its inputs, tables and program outputs.
  const void *shared_w;          // VM words [0, shared_len): inputs + pinned program outputs
  const uint16_t *shared_tab;    // silu_p[p], silu_q[q], pow_w[q]
  const uint32_t *shared_meta;   // [0] program ok on that stream, [1] omega
  uint64_t shared_seed;
  uint32_t shared_len;
  int eager_inputs;              // 1: draw every input at attempt start (TPO_VM_EAGER, A/B)
  unsigned long long *drawn;     // optional: splitmix64 draws made (inputs 2 per element, omega, SiLU tables)
};

struct EvalArgs {
  FieldConst field;
  const uint16_t *tables;
  const TpoVmInstr *code;
  const TpoVmGraph *graphs;      // graphs[0] is evaluated
  uint32_t n_in;
  uint64_t seed, stream;
  int with_silu;
  const uint32_t *inputs;        // optional explicit packed inputs
  const uint16_t *silu_tables;   // optional explicit tp[p] ++ tq[q]
  uint32_t omega;                // used with explicit inputs
  uint32_t *out;                 // packed outputs, concatenated
  uint32_t *in_dump;             // optional: sampled inputs
  int *status;                   // [0] 0 ok / 1 resample, [1] omega
};

// Global-memory field executor state (graphs beyond shared memory).
struct GlobalFF {
  FieldConst field;
  const uint16_t *tables;  // inv_p, inv_q, sqrt_p, sqrt_q (field state)
  uint16_t *attempt_tab;   // silu_p[p], silu_q[q], pow_w[q] of the current attempt
  uint32_t *W;             // 32-bit VM words: inputs, program, candidate regions
  int *flag;               // resample flag ((0xffff - pc) << 3 | code), max
  uint32_t *meta;          // [1] omega, [2] rejection-zone replay needed
};

}  // namespace tpo_ff

// narrow: 16-bit VM words (p, q < 256)
extern "C" int tpo_ff_launch_verify(const tpo_ff::VerifyArgs *a, int grid, size_t smem,
                                    cudaStream_t st, int nthreads, int narrow);
extern "C" int tpo_ff_launch_eval(const tpo_ff::EvalArgs *a, size_t smem, cudaStream_t st);
// One CTA: attempt (seed, stream 0) of the program -> words / tables / meta.
extern "C" int tpo_ff_launch_shared(const tpo_ff::VerifyArgs *a, uint64_t seed, size_t smem,
                                    void *w_out, uint16_t *tab_out, uint32_t *meta, int narrow,
                                    cudaStream_t st);
extern "C" int tpo_ff_verify_occupancy(size_t smem, int nthreads, int narrow);
// what: 0 one VM instruction, 1 inputs of (seed, stream), 2 rejection check
// of the ω / SiLU draws, 3 ω + SiLU + power tables (sequential replay when
// meta[2] is set).
extern "C" int tpo_ff_global_launch(int what, const tpo_ff::GlobalFF *g, const TpoVmInstr *I, uint32_t it,
                                    uint32_t pc, uint64_t seed, uint64_t stream, uint64_t n, int num_sms,
                                    cudaStream_t st);
extern "C" int tpo_ff_global_mismatch(const uint32_t *a, const uint32_t *b, uint64_t n, int cmp_q,
                                      unsigned long long *key, int num_sms, cudaStream_t st);
