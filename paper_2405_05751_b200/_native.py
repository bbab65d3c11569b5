"""ctypes binding of the C-ABI (include/tpo_gpu.h) exported by the in-tree
``libtpo_b200.so``.  There is no fallback: if the library is missing, or a
GPU call is made without a CUDA device, the call raises."""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.path.join(PKG, "libtpo_b200.so")
# experiments only (A/B of build variants): TPO_NATIVE_LIB names another in-tree build
if os.environ.get("TPO_NATIVE_LIB"):
    LIB_PATH = os.path.join(PKG, os.path.basename(os.environ["TPO_NATIVE_LIB"]))
HEADER = os.path.join(ROOT, "include", "tpo_gpu.h")


class FieldParams(C.Structure):
    _fields_ = [("p", C.c_uint32), ("q", C.c_uint32), ("omega_base", C.c_uint32)]


class VerifyCfg(C.Structure):
    _fields_ = [("num_tests", C.c_int32), ("max_resamples", C.c_int32), ("seed", C.c_uint64),
                ("float_tolerance", C.c_double)]


class Verdict(C.Structure):
    _fields_ = [("kind", C.c_int32), ("rounds_run", C.c_int32), ("resamples", C.c_int32),
                ("has_witness", C.c_int32), ("w_seed", C.c_uint64), ("w_round", C.c_int32),
                ("w_omega", C.c_uint32), ("w_tensor", C.c_int32), ("err_code", C.c_int32),
                ("w_index", C.c_int64)]


class GraphInfo(C.Structure):
    _fields_ = [("n_inputs", C.c_int32), ("n_outputs", C.c_int32), ("fused_kind", C.c_int32),
                ("lax", C.c_int32), ("madds", C.c_int64), ("input_elems", C.c_int64),
                ("output_elems", C.c_int64), ("vm_words", C.c_int64)]


class SearchStats(C.Structure):
    _fields_ = [("candidates", C.c_int64), ("equivalent", C.c_int64), ("not_equivalent", C.c_int64),
                ("inconclusive", C.c_int64), ("errors", C.c_int64), ("prefixes", C.c_int64),
                ("partitions", C.c_int64), ("pruned_expr", C.c_int64), ("budget_exhausted", C.c_int32),
                ("pad", C.c_int32), ("enumerate_s", C.c_double), ("compile_s", C.c_double),
                ("verify_s", C.c_double)]


assert C.sizeof(Verdict) == 48

_lib = None


class NativeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"tpo_gpu status {status}: {msg}")
        self.status = status


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"native library missing: {LIB_PATH} — run paper_2405_05751_b200/build.py "
                           "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u64, i32, i64 = C.c_void_p, C.c_uint64, C.c_int32, C.c_int64
    L.tpo_gpu_last_error.restype = C.c_char_p
    L.tpo_gpu_open.argtypes = [C.c_int, C.POINTER(vp)]
    L.tpo_gpu_close.argtypes = [vp]
    L.tpo_gpu_close.restype = None
    L.tpo_gpu_compile.argtypes = [vp, C.c_char_p, C.POINTER(vp)]
    L.tpo_gpu_graph_free.argtypes = [vp]
    L.tpo_gpu_graph_free.restype = None
    L.tpo_gpu_graph_info.argtypes = [vp, C.POINTER(GraphInfo)]
    L.tpo_gpu_graph_shape.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_int64)]
    L.tpo_gpu_graph_set_static_inputs.argtypes = [vp, u64]
    L.tpo_gpu_validate.argtypes = [C.c_char_p, i64, i64, C.c_char_p, C.c_int]
    L.tpo_gpu_eval_mugraph.argtypes = [vp, vp, vp, vp, vp, vp]
    L.tpo_gpu_eval_mugraph_host.argtypes = [vp, vp, vp, vp, vp, vp]
    L.tpo_gpu_eval_mugraph_f64.argtypes = [vp, vp, vp, vp, vp]
    L.tpo_gpu_graph_set_precision.argtypes = [vp, i32]
    L.tpo_gpu_eval_vm.argtypes = [vp, vp, i32, vp, vp]
    L.tpo_gpu_construct_thread_graphs.argtypes = [C.c_char_p, C.c_char_p, i64, C.POINTER(i64)]
    L.tpo_gpu_float_stability_filter.argtypes = [vp, vp, vp, i32, C.c_double, u64, C.c_double, vp]
    L.tpo_gpu_stability_batch.argtypes = [vp, vp, vp, vp, u64, i32, C.c_double, u64, C.c_double, vp]
    L.tpo_gpu_ff_eval.argtypes = [vp, vp, C.POINTER(FieldParams), u64, u64, i32] + [vp] * 6
    L.tpo_gpu_random_test_equivalence.argtypes = [vp, vp, vp, C.POINTER(VerifyCfg),
                                                  C.POINTER(FieldParams), C.POINTER(Verdict)]
    L.tpo_gpu_verify_batch.argtypes = [vp, vp, vp, vp, u64, C.POINTER(VerifyCfg),
                                       C.POINTER(FieldParams), vp, vp]
    L.tpo_gpu_verify_pool.argtypes = [vp, vp, vp, i32, u64, u64, C.POINTER(VerifyCfg),
                                      C.POINTER(FieldParams), vp, vp, vp, vp]
    L.tpo_gpu_verify_draws.argtypes = [vp, C.POINTER(u64)]
    L.tpo_gpu_enumerate.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, i64, C.POINTER(i64)]
    L.tpo_gpu_abstract_expression.argtypes = [C.c_char_p, C.c_char_p, i64, C.POINTER(i64)]
    L.tpo_gpu_search.argtypes = [vp, vp, C.c_char_p, C.POINTER(VerifyCfg), C.POINTER(FieldParams), vp, i64,
                                 C.POINTER(i64), C.POINTER(SearchStats)]
    L.tpo_gpu_graph_json.argtypes = [vp, C.c_char_p, i64, C.POINTER(i64)]
    L.tpo_gpu_op_madds.argtypes = [vp]
    L.tpo_gpu_op_madds.restype = i64
    _lib = L
    return L


def last_error() -> str:
    return lib().tpo_gpu_last_error().decode(errors="replace")


def check(status: int):
    if status:
        raise NativeError(status, last_error())
    return status


def declared_symbols():
    """Entry points declared in include/tpo_gpu.h."""
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tpo_gpu_\w+)\s*\(", src)))
