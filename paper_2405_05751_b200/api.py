"""Python host API over the C-ABI, mirroring the reference entry points.

==============================  ===============================================
this module                     reference (proj/core/include/tpo/...)
==============================  ===============================================
``Context.eval_mugraph``        ``interp::eval_mugraph`` (interp/interp.hpp:47-48)
``Context.ff_eval``             ``verify::ff_eval`` + sampling (verify/ffeval.hpp:58-67)
``Context.random_test_equivalence`` ``verify::random_test_equivalence`` (verify/equiv.hpp:50-53)
``Context.verify_batch``        the search loop's per-candidate verification, batched
``Context.verify_pool``         same, sharding form (candidate i = pool[i % n], seed i)
``validate``                    ``ir::validate`` (ir/validate.hpp:51)
==============================  ===============================================

Graphs are wire-format dicts (see ``graph.py``) or JSON strings.  Errors raise
:class:`~paper_2405_05751_b200._native.NativeError` carrying the C-ABI status
(1000 + ErrCode).  All compute runs on the GPU through ``libtpo_b200.so``.
"""
from __future__ import annotations

import ctypes as C
import json
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _native as N

VERDICT_DTYPE = np.dtype([("kind", "<i4"), ("rounds_run", "<i4"), ("resamples", "<i4"),
                          ("has_witness", "<i4"), ("w_seed", "<u8"), ("w_round", "<i4"),
                          ("w_omega", "<u4"), ("w_tensor", "<i4"), ("err_code", "<i4"),
                          ("w_index", "<i8")])
KIND = {0: "Equivalent", 1: "NotEquivalent", 2: "Inconclusive", 3: "Error"}
FUSED = {0: None, 1: "rmsnorm", 2: "gatedmlp", 3: "gqa", 4: "lora"}
# tpo_gpu.h TPO_PREC_*: precision policy of the fused kernels
PRECISION = {"auto": 0, "bf16": 1, "vm": 2}


def _dtype_code(x) -> int:
    """TPO_DTYPE_* of a torch tensor; anything else is rejected (the C-ABI
    would read the buffer with the wrong element size)."""
    import torch
    codes = {torch.float32: 0, torch.bfloat16: 1, torch.float64: 2}
    if x.dtype not in codes:
        raise ValueError(f"input dtype {x.dtype} unsupported: use bfloat16, float32 or float64")
    return codes[x.dtype]


def _js(g) -> bytes:
    if isinstance(g, Graph):
        g = g.spec
    return (g if isinstance(g, str) else json.dumps(g, separators=(",", ":"))).encode()


def validate(g, smem_bytes: int = 232448, elem_size: int = 2):
    """Number of Definition-1 violations and their text (B200 limits by default)."""
    buf = C.create_string_buffer(4096)
    rc = N.lib().tpo_gpu_validate(_js(g), smem_bytes, elem_size, buf, 4096)
    if rc >= 1000:
        raise N.NativeError(rc, N.last_error())
    return rc, buf.value.decode()


def construct_thread_graphs(g) -> dict:
    """SPEC construct_thread_graphs: the graph with every
    GraphDef's maximal single-consumer elementwise chains grouped into
    register-resident ThreadGroups (``tpo_gpu_construct_thread_graphs``)."""
    need = C.c_int64(0)
    N.check(N.lib().tpo_gpu_construct_thread_graphs(_js(g), None, 0, C.byref(need)))
    buf = C.create_string_buffer(int(need.value))
    N.check(N.lib().tpo_gpu_construct_thread_graphs(_js(g), buf, need.value, C.byref(need)))
    return json.loads(buf.value.decode())


def plan_block_graphs(g, smem_bytes: int = 0, elem_size: int = 2) -> dict:
    """SPEC schedule_ops + plan_memory for every GraphDef of
    ``g`` (``tpo_gpu_plan_block_graphs``): depth order, sync points, shared-
    memory offsets and peak.  Raises NativeError(DoesNotFit) past smem_bytes."""
    need = C.c_int64(0)
    N.check(N.lib().tpo_gpu_plan_block_graphs(_js(g), C.c_int64(smem_bytes), C.c_int32(elem_size),
                                              None, 0, C.byref(need)))
    buf = C.create_string_buffer(int(need.value))
    N.check(N.lib().tpo_gpu_plan_block_graphs(_js(g), C.c_int64(smem_bytes), C.c_int32(elem_size),
                                              buf, need.value, C.byref(need)))
    return json.loads(buf.value.decode())


def generate(program, grids=None, loops=None, rewrite: bool = True, max_candidates: int = 4096,
             with_stats: bool = False, max_kernels: int = 1, per_segment: int = 3):
    """µGraph candidates for a computation graph (``tpo_gpu_generate``):
    single-GraphDef µGraphs over grid / for-loop partitions and, with
    ``max_kernels`` > 1, µGraphs of up to that many kernels (contiguous
    single-output segments of the op list, each a pre-defined kernel op or
    one of its first ``per_segment`` fused GraphDefs).  Each is valid under
    B200 limits; equivalence is left to the verifier."""
    cfg = {"rewrite": rewrite, "max_candidates": max_candidates, "max_kernels": max_kernels,
           "per_segment": per_segment}
    if grids is not None:
        cfg["grids"] = list(grids)
    if loops is not None:
        cfg["loops"] = list(loops)
    cj = json.dumps(cfg).encode()
    need = C.c_int64(0)
    N.check(N.lib().tpo_gpu_generate(_js(program), cj, None, 0, C.byref(need)))
    buf = C.create_string_buffer(int(need.value))
    N.check(N.lib().tpo_gpu_generate(_js(program), cj, buf, need.value, C.byref(need)))
    res = json.loads(buf.value.decode())
    return (res["candidates"], res["stats"]) if with_stats else res["candidates"]


def enumerate_mugraphs(program, grids=(1, 2, 4, 8, 16), loops=(1, 2, 4, 8, 16), max_block_ops: int = 9,
                       max_kernel_ops: int = 1, max_loop_labels: int = 2, concat_matmul: bool = True,
                       max_candidates: int = 4096, max_prefixes: int = 4_000_000, threads: int = 0,
                       with_stats: bool = False):
    """Algorithm 1 (§4; ``tpo_gpu_enumerate``): µGraphs generated op
    by op in canonical form — up to ``max_kernel_ops`` pre-defined kernel ops,
    then one GraphDef whose block graph is enumerated operator by operator —
    pruned by abstract expressions (subexpressions of the program's), shape
    and shared memory.  Candidates carry the program's abstract expression;
    equivalence is the verifier's job."""
    cfg = {"grids": list(grids), "loops": list(loops), "max_block_ops": max_block_ops,
           "max_kernel_ops": max_kernel_ops, "max_loop_labels": max_loop_labels,
           "concat_matmul": concat_matmul, "max_candidates": max_candidates,
           "max_prefixes": max_prefixes, "threads": threads}
    cj = json.dumps(cfg).encode()
    need = C.c_int64(0)
    N.check(N.lib().tpo_gpu_enumerate(_js(program), cj, None, 0, C.byref(need)))
    buf = C.create_string_buffer(int(need.value))
    N.check(N.lib().tpo_gpu_enumerate(_js(program), cj, buf, need.value, C.byref(need)))
    res = json.loads(buf.value.decode())
    return (res["candidates"], res["stats"]) if with_stats else res["candidates"]


def abstract_expression(g) -> str:
    """The abstract expression (Table 2) of ``g``'s output in the
    enumerator's normal form (``tpo_gpu_abstract_expression``)."""
    need = C.c_int64(0)
    N.check(N.lib().tpo_gpu_abstract_expression(_js(g), None, 0, C.byref(need)))
    buf = C.create_string_buffer(int(need.value))
    N.check(N.lib().tpo_gpu_abstract_expression(_js(g), buf, need.value, C.byref(need)))
    return buf.value.decode()


def describe(g, smem_bytes: int = 0) -> str:
    """SPEC describe: pseudo-kernel listing of ``g`` plus
    its B200 execution (``tpo_gpu_describe``)."""
    need = C.c_int64(0)
    N.check(N.lib().tpo_gpu_describe(_js(g), C.c_int64(smem_bytes), None, 0, C.byref(need)))
    buf = C.create_string_buffer(int(need.value))
    N.check(N.lib().tpo_gpu_describe(_js(g), C.c_int64(smem_bytes), buf, need.value, C.byref(need)))
    return buf.value.decode()


def plan_intervals(sizes, starts, ends, exhaustive_max: int = 8):
    """The memory planner on explicit inclusive lifetimes: (offsets, peak,
    exhaustive) (``tpo_gpu_plan_intervals``)."""
    n = len(sizes)
    arr = C.c_int64 * max(n, 1)
    off = arr()
    peak = C.c_int64(0)
    ex = C.c_int32(0)
    N.check(N.lib().tpo_gpu_plan_intervals(C.c_int32(n), arr(*sizes), arr(*starts), arr(*ends),
                                           C.c_int32(exhaustive_max), off, C.byref(peak), C.byref(ex)))
    return [int(off[i]) for i in range(n)], int(peak.value), bool(ex.value)


class GraphBatch:
    """n compiled graph handles in one ctypes array (``compile_many(...,
    batch=True)``); frees them when collected.  ``st[i]`` != 0: graph i did
    not compile (its handle is NULL)."""

    def __init__(self, n: int):
        self.n = n
        self.arr = (C.c_void_p * max(n, 1))()
        self.st = (C.c_int32 * max(n, 1))()

    def __len__(self):
        return self.n

    def __del__(self):
        try:
            if N is not None and N._lib is not None:
                free = N.lib().tpo_gpu_graph_free
                for i in range(self.n):
                    if self.arr[i]:
                        free(C.c_void_p(self.arr[i]))
        except (AttributeError, TypeError):  # interpreter shutdown: module globals gone
            pass
        self.n = 0


class Graph:
    """A compiled µGraph handle (``tpo_gpu_compile``)."""

    def __init__(self, ctx: "Context", g):
        self.ctx = ctx
        self._spec = g
        h = C.c_void_p()
        N.check(N.lib().tpo_gpu_compile(ctx.h, _js(g), C.byref(h)))
        self.h = h
        self._info = None

    @property
    def spec(self) -> dict:
        """The graph as a dict (parsed on first use when built from JSON text;
        fetched from the handle for graphs the library built, e.g. search results)."""
        if self._spec is None:
            need = C.c_int64(0)
            N.check(N.lib().tpo_gpu_graph_json(self.h, None, 0, C.byref(need)))
            buf = C.create_string_buffer(int(need.value))
            N.check(N.lib().tpo_gpu_graph_json(self.h, buf, need.value, C.byref(need)))
            self._spec = buf.value.decode()
        if isinstance(self._spec, (str, bytes)):
            self._spec = json.loads(self._spec)
        return self._spec

    @classmethod
    def _wrap(cls, ctx: "Context", spec, h) -> "Graph":
        self = cls.__new__(cls)
        self.ctx = ctx
        self._spec = spec
        self.h = h
        self._info = None
        return self

    @property
    def info(self):
        """tpo_graph_info, fetched on first use."""
        if self._info is None:
            info = N.GraphInfo()
            N.lib().tpo_gpu_graph_info(self.h, C.byref(info))
            self._info = info
        return self._info

    def __del__(self):
        h = getattr(self, "h", None)
        try:
            if h and N is not None and N._lib is not None:
                N.lib().tpo_gpu_graph_free(h)
        except (AttributeError, TypeError):  # interpreter shutdown: module globals gone
            pass
        self.h = None

    def shapes(self, outputs: bool) -> List[List[int]]:
        n = self.info.n_outputs if outputs else self.info.n_inputs
        out = []
        for i in range(n):
            dims = (C.c_int64 * 4)()
            r = N.lib().tpo_gpu_graph_shape(self.h, int(outputs), i, dims)
            out.append([dims[k] for k in range(r)])
        return out

    def set_static_inputs(self, indices: Sequence[int]) -> "Graph":
        """Declare inputs that no earlier work on the stream writes (weights):
        the fused kernel may stream them before the preceding kernel ends."""
        mask = 0
        for i in indices:
            mask |= 1 << int(i)
        N.check(N.lib().tpo_gpu_graph_set_static_inputs(self.h, mask))
        return self

    def set_precision(self, policy: str) -> "Graph":
        """TPO_PREC_* policy of the fused kernels: "auto" (bf16 inputs -> bf16
        kernel, fp32/fp64 inputs -> split hi+lo kernel), "bf16" (round every
        input to bf16), "vm" (generic VM in the reference's operation order)."""
        N.check(N.lib().tpo_gpu_graph_set_precision(self.h, PRECISION[policy]))
        return self

    @property
    def fused(self) -> Optional[str]:
        return FUSED.get(self.info.fused_kind)

    @property
    def madds(self) -> int:
        return int(self.info.madds)


class Context:
    """One device + stream (``tpo_gpu_open``)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        N.check(N.lib().tpo_gpu_open(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            N.lib().tpo_gpu_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def compile(self, g) -> Graph:
        return g if isinstance(g, Graph) else Graph(self, g)

    def compile_many(self, graphs: Sequence, threads: int = 0, batch: bool = False):
        """Compile n graphs on all host cores (``tpo_gpu_compile_many``):
        (list of Graph or None, list of per-graph status).  ``batch=True``
        returns a GraphBatch instead of the list (one handle array, no
        per-graph Python object: the search-stream fast path; verify_batch
        takes it as ``cands``)."""
        n = len(graphs)
        if batch:
            js = [g.encode() for g in graphs] if all(type(g) is str for g in graphs) else [_js(g) for g in graphs]
            gb = GraphBatch(n)
            N.check(N.lib().tpo_gpu_compile_many(self.h, (C.c_char_p * max(n, 1))(*js), C.c_int64(n),
                                                 C.c_int32(threads), gb.arr, gb.st))
            return gb, list(gb.st)[:n]
        js = [_js(g) for g in graphs]
        arr = (C.c_char_p * max(n, 1))(*js)
        hs = (C.c_void_p * max(n, 1))()
        st = (C.c_int32 * max(n, 1))()
        N.check(N.lib().tpo_gpu_compile_many(self.h, arr, C.c_int64(n), C.c_int32(threads), hs, st))
        out = []
        for i in range(n):
            if st[i] == 0:
                out.append(Graph._wrap(self, graphs[i], C.c_void_p(hs[i])))
            else:
                out.append(None)
        return out, [int(st[i]) for i in range(n)]

    # ---- floating point -------------------------------------------------
    def eval_mugraph(self, g, inputs: Sequence, outputs=None, stream=None):
        """fp evaluation on torch CUDA tensors (bf16, fp32 or fp64 inputs,
        fp32 outputs) under the graph's precision policy."""
        import torch
        g = self.compile(g)
        ins = list(inputs)
        if len(ins) != g.info.n_inputs:
            raise ValueError("input count")
        for x, s in zip(ins, g.shapes(False)):
            if list(x.shape) != s or not x.is_cuda or not x.is_contiguous():
                raise ValueError(f"input must be a contiguous CUDA tensor of shape {s}")
        codes = [_dtype_code(x) for x in ins]
        if outputs is None:
            outputs = [torch.empty(s, device=ins[0].device, dtype=torch.float32)
                       for s in g.shapes(True)]
        for o, s in zip(outputs, g.shapes(True)):
            if list(o.shape) != s or o.dtype != torch.float32 or not o.is_cuda or not o.is_contiguous():
                raise ValueError(f"output must be a contiguous fp32 CUDA tensor of shape {s}")
        dt = (C.c_int32 * len(ins))(*codes)
        pin = (C.c_void_p * len(ins))(*[x.data_ptr() for x in ins])
        pout = (C.c_void_p * len(outputs))(*[o.data_ptr() for o in outputs])
        st = stream if stream is not None else torch.cuda.current_stream(ins[0].device).cuda_stream
        N.check(N.lib().tpo_gpu_eval_mugraph(self.h, g.h, pin, dt, pout, C.c_void_p(st)))
        return outputs

    def eval_mugraph_host(self, g, inputs: Sequence, outputs=None, stream=None):
        """fp evaluation from/to HOST tensors (``tpo_gpu_eval_mugraph_host``):
        bf16, fp32 or fp64 CPU torch tensors in (pinned for full PCIe speed),
        fp32 CPU tensors out; the host<->device copies are part of the call."""
        import torch
        g = self.compile(g)
        ins = list(inputs)
        if len(ins) != g.info.n_inputs:
            raise ValueError("input count")
        for x, s in zip(ins, g.shapes(False)):
            if list(x.shape) != s or x.is_cuda or not x.is_contiguous():
                raise ValueError(f"input must be a contiguous host tensor of shape {s}")
        codes = [_dtype_code(x) for x in ins]
        if outputs is None:
            outputs = [torch.empty(s, dtype=torch.float32) for s in g.shapes(True)]
        dt = (C.c_int32 * len(ins))(*codes)
        pin = (C.c_void_p * len(ins))(*[x.data_ptr() for x in ins])
        pout = (C.c_void_p * len(outputs))(*[o.data_ptr() for o in outputs])
        N.check(N.lib().tpo_gpu_eval_mugraph_host(self.h, g.h, pin, dt, pout,
                                                  C.c_void_p(stream) if stream else None))
        return outputs

    def eval_mugraph_f64(self, g, inputs: Sequence, stream=None) -> List[np.ndarray]:
        """``interp::eval_mugraph`` with its own types (interp.hpp:47-48):
        float64 numpy inputs, float64 numpy outputs (``tpo_gpu_eval_mugraph_f64``).
        Fused µGraphs run their split kernel (TPO_PREC_AUTO), others the
        generic VM in double arithmetic."""
        g = self.compile(g)
        shapes = g.shapes(False)
        if len(inputs) != len(shapes):
            raise ValueError("input count")
        ins = []
        for x, s in zip(inputs, shapes):
            a = np.ascontiguousarray(x, dtype=np.float64)
            if list(a.shape) != s:
                raise ValueError(f"input shape {list(a.shape)} != {s}")
            ins.append(a)
        outs = [np.zeros(s, np.float64) for s in g.shapes(True)]
        pin = (C.c_void_p * max(len(ins), 1))(*[a.ctypes.data for a in ins])
        pout = (C.c_void_p * max(len(outs), 1))(*[o.ctypes.data for o in outs])
        N.check(N.lib().tpo_gpu_eval_mugraph_f64(self.h, g.h, pin, pout,
                                                 C.c_void_p(stream) if stream else None))
        return outs

    def eval_vm(self, g, inputs: Sequence, mode: int = 0):
        """Generic GPU µGraph VM (``tpo_gpu_eval_vm``): mode 0 eval_mugraph
        (double), 1 eval_program (double, rejects GraphDefs), 2
        eval_mugraph_f32 (float).  numpy inputs in graph-input order; returns
        numpy outputs."""
        g = self.compile(g)
        dt = np.float32 if mode == 2 else np.float64
        shapes = g.shapes(False)
        if len(inputs) != len(shapes):
            raise ValueError("input count")
        flat = np.concatenate([np.ascontiguousarray(x, dtype=dt).reshape(-1) for x in inputs]) \
            if inputs else np.zeros(0, dt)
        oshapes = g.shapes(True)
        out = np.zeros(sum(int(np.prod(s)) for s in oshapes), dt)
        N.check(N.lib().tpo_gpu_eval_vm(self.h, g.h, mode, flat.ctypes.data, out.ctypes.data))
        res, c = [], 0
        for s in oshapes:
            k = int(np.prod(s))
            res.append(out[c:c + k].reshape(s))
            c += k
        return res

    def eval_vm_dev(self, g, inputs, mode: int = 0, stream=None):
        """tpo_gpu_eval_vm on torch CUDA tensors (``tpo_gpu_eval_vm_dev``):
        inputs fp64 (fp32 for mode 2) in graph-input order; returns the
        outputs as torch CUDA tensors, asynchronously on ``stream``."""
        import torch
        g = self.compile(g)
        dt = torch.float32 if mode == 2 else torch.float64
        flat = torch.cat([x.to(dt).reshape(-1) for x in inputs]).contiguous()
        oshapes = g.shapes(True)
        out = torch.empty(sum(int(np.prod(s)) for s in oshapes), dtype=dt, device=flat.device)
        N.check(N.lib().tpo_gpu_eval_vm_dev(self.h, g.h, mode, C.c_void_p(flat.data_ptr()),
                                            C.c_void_p(out.data_ptr()), C.c_void_p(stream) if stream else None))
        res, c = [], 0
        for s in oshapes:
            k = int(np.prod(s))
            res.append(out[c:c + k].view(*s))
            c += k
        return res

    def float_stability_filter(self, g, program, trials: int = 1, tol: float = 1e-3, seed: int = 17,
                               scale: float = 1.0) -> bool:
        """verify::float_stability_filter (stability.hpp:29-31) on the GPU."""
        g, program = self.compile(g), self.compile(program)
        ok = C.c_int32(0)
        N.check(N.lib().tpo_gpu_float_stability_filter(self.h, g.h, program.h, trials, tol, seed,
                                                         scale, C.addressof(ok)))
        return bool(ok.value)

    def stability_batch(self, program, cands: Sequence, seeds=None, trials: int = 1,
                        tol: float = 1e-3, seed: int = 17, scale: float = 1.0) -> np.ndarray:
        """The stability filter for many candidates in one launch: int8 per
        candidate (1 pass, 0 fail, -1 interface mismatch)."""
        prog = self.compile(program)
        handles, hs = {}, []
        for c in cands:
            if id(c) not in handles:
                handles[id(c)] = self.compile(c)
            hs.append(handles[id(c)].h.value)
        n = len(hs)
        arr = (C.c_void_p * n)(*hs)
        sd = None
        if seeds is not None:
            sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        ok = np.zeros(n, np.int8)
        N.check(N.lib().tpo_gpu_stability_batch(self.h, prog.h, arr,
                                                 sd.ctypes.data if sd is not None else None, n,
                                                 trials, tol, seed, scale, ok.ctypes.data))
        return ok

    # ---- search ---------------------------------------------------------------
    def search(self, program, cap: int = 1 << 16, num_tests=1, seed=0, max_resamples=16, p=227, q=113,
               wbase=4, **enum_cfg):
        """The search loop (``tpo_gpu_search``): Algorithm 1's candidates
        (``enumerate_mugraphs`` options as keywords) become handles without
        the wire format and are verified in one GPU batch with one
        VerifyConfig.  Returns (accepted Graphs, stats dict)."""
        prog = self.compile(program)
        cj = json.dumps(enum_cfg).encode()
        arr = (C.c_void_p * max(cap, 1))()
        na = C.c_int64(0)
        st = N.SearchStats()
        cfg = N.VerifyCfg(num_tests, max_resamples, seed, 1e-3)
        fp = N.FieldParams(p, q, wbase)
        N.check(N.lib().tpo_gpu_search(self.h, prog.h, cj, C.byref(cfg), C.byref(fp), arr, cap,
                                       C.byref(na), C.byref(st)))
        acc = [Graph._wrap(self, None, C.c_void_p(arr[i])) for i in range(min(na.value, cap))]
        return acc, {k: getattr(st, k) for k, _ in N.SearchStats._fields_ if k != "pad"}

    # ---- finite field -------------------------------------------------------
    def ff_eval(self, g, seed: int, stream: int, with_silu: Optional[bool] = None, p=227, q=113,
                wbase=4):
        """One verifier attempt on one graph; mirrors oracle.ref.ff_attempt's return."""
        from .graph import has_silu
        g = self.compile(g)
        if with_silu is None:
            with_silu = has_silu(g.spec)
        n_in, n_out = g.info.input_elems, g.info.output_elems
        oxp, oxq = np.zeros(n_out, np.uint16), np.zeros(n_out, np.uint16)
        oqd = np.zeros(n_out, np.uint8)
        ixp, ixq = np.zeros(n_in, np.uint16), np.zeros(n_in, np.uint16)
        om = C.c_uint32(0)
        fp = N.FieldParams(p, q, wbase)
        rc = N.lib().tpo_gpu_ff_eval(self.h, g.h, C.byref(fp), seed, stream, int(with_silu),
                                     oxp.ctypes.data, oxq.ctypes.data, oqd.ctypes.data,
                                     C.addressof(om), ixp.ctypes.data, ixq.ctypes.data)
        if rc and rc < 2000:
            raise N.NativeError(rc, N.last_error())
        outs, c = [], 0
        for s in g.shapes(True):
            n = int(np.prod(s))
            outs.append((oxp[c:c + n].reshape(s), oxq[c:c + n].reshape(s), oqd[c:c + n].reshape(s)))
            c += n
        return dict(rc=rc, omega=om.value, in_xp=ixp, in_xq=ixq, out=outs)

    def random_test_equivalence(self, g1, g2, num_tests=1, seed=0, max_resamples=16, p=227,
                                q=113, wbase=4) -> Dict[str, int]:
        g1, g2 = self.compile(g1), self.compile(g2)
        v = N.Verdict()
        cfg = N.VerifyCfg(num_tests, max_resamples, seed, 1e-3)
        fp = N.FieldParams(p, q, wbase)
        rc = N.lib().tpo_gpu_random_test_equivalence(self.h, g1.h, g2.h, C.byref(cfg), C.byref(fp),
                                                     C.byref(v))
        if rc and v.kind != 3:
            raise N.NativeError(rc, N.last_error())
        return {k: getattr(v, k) for k, _ in N.Verdict._fields_}

    def verify_batch(self, program, cands: Sequence, seeds: Sequence[int], num_tests=1,
                     max_resamples=16, p=227, q=113, wbase=4, want_verdicts=True):
        """Returns (verdicts structured array | None, accept bool array)."""
        prog = self.compile(program)
        if isinstance(cands, GraphBatch):  # compile_many(batch=True): the handle array as is
            if any(cands.st[i] for i in range(cands.n)):
                raise ValueError("verify_batch: the batch holds graphs that failed to compile")
            n, arr = cands.n, cands.arr
        else:
            handles = {}
            hs = []
            for c in cands:
                key = id(c)
                if key not in handles:
                    handles[key] = self.compile(c)
                hs.append(handles[key].h.value)
            n = len(hs)
            arr = (C.c_void_p * n)(*hs)
        sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        out = np.zeros(n, VERDICT_DTYPE) if want_verdicts else None
        acc = np.zeros((n + 31) // 32, np.uint32)
        cfg = N.VerifyCfg(num_tests, max_resamples, 0, 1e-3)
        fp = N.FieldParams(p, q, wbase)
        N.check(N.lib().tpo_gpu_verify_batch(self.h, prog.h, arr, sd.ctypes.data, n, C.byref(cfg),
                                             C.byref(fp), out.ctypes.data if want_verdicts else None,
                                             acc.ctypes.data))
        bits = np.unpackbits(acc.view(np.uint8), bitorder="little")[:n].astype(bool)
        return out, bits

    def verify_pool(self, program, pool: Sequence, first: int, n: int, num_tests=1,
                    max_resamples=16, p=227, q=113, wbase=4, want_verdicts=False,
                    accept_dev=None, stream=None):
        """Sharding form: candidate i in [first, first+n) = pool[i % len(pool)], seed i.
        ``accept_dev``: optional int32 torch CUDA tensor of ceil(n/32) words.
        Returns (verdicts | None, attempts)."""
        prog = self.compile(program)
        gs = [self.compile(c) for c in pool]
        arr = (C.c_void_p * len(gs))(*[g.h.value for g in gs])
        out = np.zeros(n, VERDICT_DTYPE) if want_verdicts else None
        att = C.c_uint64(0)
        cfg = N.VerifyCfg(num_tests, max_resamples, 0, 1e-3)
        fp = N.FieldParams(p, q, wbase)
        N.check(N.lib().tpo_gpu_verify_pool(
            self.h, prog.h, arr, len(gs), first, n, C.byref(cfg), C.byref(fp),
            C.c_void_p(accept_dev.data_ptr()) if accept_dev is not None else None,
            out.ctypes.data if want_verdicts else None, C.addressof(att),
            C.c_void_p(stream) if stream else None))
        return out, att.value

    def last_verify_draws(self) -> int:
        """splitmix64 draws of the last verify_pool call (tpo_gpu_verify_draws)."""
        d = C.c_uint64(0)
        N.check(N.lib().tpo_gpu_verify_draws(self.h, C.byref(d)))
        return d.value
