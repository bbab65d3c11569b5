// B200 backend — block-batched µGraph VM bytecode (host <-> device contract).
//
// A µGraph is lowered (csrc/host/lower.cpp) into a straight-line program of
// tensor instructions.  Every GraphDef's block graph is executed for *all*
// grid blocks at once: each block-level tensor gets three leading grid dims
// (bx, by, bz), so one instruction is one data-parallel loop over
// grid x tile elements, and the reference's sequential block loop
// (eval_core.hpp:234-237) becomes a batch dimension.  Only the for-loop
// (eval_core.hpp:303-341) stays sequential: VM_LOOP / VM_ENDLOOP.
//
// Addressing: an instruction's index space has up to kVmDims dims (outer to
// inner).  Operand offsets are base + sum(coord_k * stride_k) (+ iter *
// iter_stride); a zero stride broadcasts.  `wmask` marks grid dims whose
// coordinate must be maximal for the store to happen — the reference's
// "last block in grid-major order wins" rule for grid axes absent from an
// omap (eval_core.hpp:355-366).
#pragma once

#include <stdint.h>

#define TPO_VM_DIMS 7
#define TPO_VM_MAX_OUTPUTS 8
#define TPO_VM_MAX_GEN 8

enum TpoVmOp {
  VM_ZERO = 1,   // dst[0..n) = 0 (field zero (0,0,defined) / 0.0)
  VM_COPY,       // dst[view] = a[view]           (InIter, Repeat, Reshape, concat Accum, OutSaver)
  VM_UNARY,      // dst[i] = f(a[view])           sub: VM_EXP, VM_SQR, VM_SQRT, VM_SILU
  VM_BINARY,     // dst[i] = f(a[view], b[view])  sub: VM_ADD, VM_MUL, VM_DIV
  VM_MATMUL,     // dims {B, M, K, N}; a [B,M,K], b [B,K,N], dst [B,M,N] contiguous
                 // VM_STRIDED: dims {gx, gy, gz, B, M, K, N} with per-operand grid /
                 // batch / row / k strides (operands read in place: InIter views)
  VM_SUM,        // dims {outer, mid, group, inner}: dst[o,m,i] = sum_t a[o, m*group+t, i]
  VM_LOOP,       // n = trip count; body follows
  VM_ENDLOOP,    // jump back to the instruction after the matching VM_LOOP
  VM_RAISE,      // FF: the first EwExp of a q-undefined value (field.cpp:105-108) — the
                 // program stops; it is a resample if a counted event preceded it, else
                 // Error(PoisonedExponent)
};

enum TpoVmSub { VM_ADD = 0, VM_MUL, VM_DIV, VM_EXP, VM_SQR, VM_SQRT, VM_SILU };

enum TpoVmFlags {
  VM_FLAT = 1,    // all operands contiguous over the index space: no index math
  VM_A_QD = 2,    // operand a is q-defined (FF mode, static)
  VM_B_QD = 4,    // operand b is q-defined
  VM_STRIDED = 8, // MATMUL: strided operand views (see VM_MATMUL)
  VM_ACCUM = 16,  // MATMUL: dst = dst + A·B (a fused φ-Accum, acc = add(acc, val))
  VM_TILE22 = 32, // MATMUL: each index is a 2 x 2 output tile (rows 2i, 2i+1; cols 2j, 2j+1)
  VM_NOSYNC = 64, // no CTA barrier after this instruction: the next one neither reads nor
                  // writes any word this phase writes, nor writes a word it reads (lowering
                  // mark_phases, the depth-schedule sync placement of SPEC.md:527-536)
};

struct TpoVmInstr {
  uint8_t op, sub, qd, flags;  // qd: result q-defined (static, FF mode)
  // VM_BINARY: a thread-graph chain fused into the instruction — operand a
  // (pre_a) / b (pre_b) first goes through the unary 1 + TpoVmSub (VM_SQR,
  // VM_SQRT, VM_SILU) in registers: the intermediate tensor of the chain
  // has no VM words (register-resident); 0 = none
  uint8_t ndim, wmask, pre_a, pre_b;
  uint32_t n;                  // elements in the index space
  uint32_t dst, a, b;          // buffer base offsets (words)
  int32_t a_iter, d_iter;      // per-iteration offsets added to a / dst
  uint32_t dims[TPO_VM_DIMS];
  int32_t sd[TPO_VM_DIMS], sa[TPO_VM_DIMS], sb[TPO_VM_DIMS];
  // Division by invariant integers (index math without IDIV):
  // x / d = __umulhi(x, dmul) >> dsh for x < 2^31; dmul = 0 means d = 1.
  // COPY / BINARY / UNARY: one per index dim.  MATMUL: {B*M*N, M*N, N}.
  // SUM: {inner, mid}.  Filled by the lowering (tpo_vm_set_divisors).
  uint32_t dmul[TPO_VM_DIMS];
  uint8_t dsh[TPO_VM_DIMS];
  uint8_t pad2;
  int32_t b_iter;              // MATMUL VM_STRIDED: per-iteration offset added to b
  // FF, graphs with a VM_RAISE: a DivByZero / NonResidue event counts only at
  // indices < b0n (grid block 0 of the raising GraphDef: the reference's
  // grid-major evaluation reaches the raising op before any later block);
  // 0 = every index counts
  uint32_t b0n;
  // fp MATMUL hoisted out of the for-loop (VM_ACCUM, K = the loop's whole
  // contraction): the reference adds each iteration's k-segment sum to the
  // accumulator, acc = add(acc, Σ_{k in segment} a·b), so the executors sum
  // every `kseg` consecutive k (ascending) before adding; 0 = one segment
  uint32_t kseg;               // 192 bytes: copied to shared memory as uint4
};

// Host helper: the (mul, shift) pair of divisor d >= 1 (CUTLASS-style
// round-up reciprocal, exact for numerators < 2^31).
static inline void tpo_vm_divisor(uint32_t d, uint32_t *mul, uint8_t *sh) {
  if (d <= 1) {
    *mul = 0;
    *sh = 0;
    return;
  }
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;  // ceil(log2 d)
  const unsigned long long p = 1ull << (31 + l);
  *mul = (uint32_t)((p + d - 1) / d);
  *sh = (uint8_t)(l - 1);
}

static inline void tpo_vm_set_divisors(TpoVmInstr *I) {
  for (int k = 0; k < TPO_VM_DIMS; ++k) I->dmul[k] = 0, I->dsh[k] = 0;
  if (I->op == VM_MATMUL && (I->flags & VM_STRIDED)) {
    // {B*M*N, M*N, N, gy*gz, gz}; with VM_TILE22 over M/2 x N/2 tiles
    const uint32_t t = (I->flags & VM_TILE22) ? 2u : 1u;
    const uint32_t Mt = I->dims[4] / t, Nt = I->dims[6] / t, MN = Mt * Nt;
    tpo_vm_divisor(I->dims[3] * MN, &I->dmul[0], &I->dsh[0]);
    tpo_vm_divisor(MN, &I->dmul[1], &I->dsh[1]);
    tpo_vm_divisor(Nt, &I->dmul[2], &I->dsh[2]);
    tpo_vm_divisor(I->dims[1] * I->dims[2], &I->dmul[3], &I->dsh[3]);
    tpo_vm_divisor(I->dims[2], &I->dmul[4], &I->dsh[4]);
  } else if (I->op == VM_MATMUL) {
    const uint32_t MN = I->dims[2] * I->dims[4];
    tpo_vm_divisor(I->dims[1] * MN, &I->dmul[0], &I->dsh[0]);
    tpo_vm_divisor(MN, &I->dmul[1], &I->dsh[1]);
    tpo_vm_divisor(I->dims[4], &I->dmul[2], &I->dsh[2]);
  } else if (I->op == VM_SUM) {
    tpo_vm_divisor(I->dims[3], &I->dmul[0], &I->dsh[0]);
    tpo_vm_divisor(I->dims[1], &I->dmul[1], &I->dsh[1]);
  } else if (I->op == VM_COPY || I->op == VM_BINARY || I->op == VM_UNARY) {
    for (int k = 0; k < I->ndim && k < TPO_VM_DIMS; ++k) tpo_vm_divisor(I->dims[k], &I->dmul[k], &I->dsh[k]);
  }
}

// One compiled graph inside a batch upload.
struct TpoVmGraph {
  uint32_t code_off, code_len;  // into the batch instruction array
  uint32_t n_out;
  uint32_t words;               // words used past the graph's region base
  uint32_t out_off[TPO_VM_MAX_OUTPUTS];
  uint32_t out_len[TPO_VM_MAX_OUTPUTS];
  uint8_t out_qd[TPO_VM_MAX_OUTPUTS];
  uint8_t has_silu, poisoned;
  uint8_t err;                  // 0, or 1 + tpo::ErrCode: candidate rejected up front
  // FF, lazy input sampling: input words [gen_e0[i], + gen_len[i]) are drawn
  // right before instruction gen_pc[i], their first reader (gen_pc ascending;
  // gen_pc == code_len: never read by this graph).  An attempt that resamples
  // before an input is read never draws it.  n_gen = 0: draw all up front.
  uint8_t n_gen;
  uint8_t pad[4];
  uint32_t gen_pc[TPO_VM_MAX_GEN];
  uint32_t gen_e0[TPO_VM_MAX_GEN], gen_len[TPO_VM_MAX_GEN];
};
