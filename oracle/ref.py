"""TEST INFRASTRUCTURE ONLY: ctypes access to the compiled reference.

Loads ``oracle/_ref/libtpo_ref.so`` (the unmodified reference sources built by
``oracle/Makefile`` plus the adapter ``oracle/ref_capi.cpp``).  Imported only
by tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs, as the
checker / the reference arm — never by the product package.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libtpo_ref.so")


class RefVerdict(C.Structure):
    _fields_ = [("kind", C.c_int32), ("rounds_run", C.c_int32), ("resamples", C.c_int32),
                ("has_witness", C.c_int32), ("w_seed", C.c_uint64), ("w_round", C.c_int32),
                ("w_omega", C.c_uint32), ("w_tensor", C.c_int32), ("err_code", C.c_int32),
                ("w_index", C.c_int64)]


VERDICT_NP = np.dtype([("kind", "<i4"), ("rounds_run", "<i4"), ("resamples", "<i4"),
                       ("has_witness", "<i4"), ("w_seed", "<u8"), ("w_round", "<i4"),
                       ("w_omega", "<u4"), ("w_tensor", "<i4"), ("err_code", "<i4"),
                       ("w_index", "<i8")])
assert VERDICT_NP.itemsize == C.sizeof(RefVerdict) == 48

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint64)]
        L.ref_rng_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_double)]
        L.ref_field_tables.argtypes = [C.c_uint32] * 3 + [C.c_void_p] * 4
        L.ref_field_op.argtypes = [C.c_uint32] * 3 + [C.c_int, C.c_uint32] + [C.c_void_p] * 3
        L.ref_eval_mugraph.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_time_eval_mugraph.argtypes = [C.c_char_p, C.c_void_p, C.c_int]
        L.ref_time_eval_mugraph.restype = C.c_double
        L.ref_time_eval_parallel.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.ref_time_eval_parallel.restype = C.c_double
        L.ref_ff_attempt.argtypes = ([C.c_char_p] + [C.c_uint32] * 3 + [C.c_uint64, C.c_uint64, C.c_int]
                                     + [C.c_void_p] * 6)
        L.ref_random_test_equivalence.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_uint64, C.c_int,
                                                  C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]
        L.ref_verify_batch.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_uint64, C.c_uint64,
                                       C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                       C.c_void_p]
        L.ref_verify_batch.restype = C.c_double
        L.ref_float_stability_filter.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_double,
                                                 C.c_uint64, C.c_double]
        L.ref_validate.argtypes = [C.c_char_p, C.c_int64, C.c_int64]
        L.ref_block_shared_bytes.argtypes = [C.c_char_p, C.c_int, C.c_int64]
        L.ref_block_shared_bytes.restype = C.c_int64
        L.ref_op_madds.argtypes = [C.c_char_p]
        L.ref_op_madds.restype = C.c_int64
        L.ref_canonical_key.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        L.ref_roundtrip_json.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        _lib = L
    return _lib


def _js(g) -> bytes:
    return (g if isinstance(g, str) else json.dumps(g, separators=(",", ":"))).encode()


def _shapes(g, key):
    return [list(g["tensors"][t]["shape"]) for t in g[key]]


def last_error() -> str:
    return lib().ref_last_error().decode()


def rng_draws(seed: int, n: int, stream: Optional[int] = None) -> np.ndarray:
    out = np.zeros(n, np.uint64)
    lib().ref_rng_draws(seed, stream or 0, int(stream is not None), n,
                        out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return out


def rng_normals(seed: int, stream: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.float64)
    lib().ref_rng_normals(seed, stream, n, out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def field_tables(p=227, q=113, wbase=4):
    ip, iq = np.zeros(p, np.uint32), np.zeros(q, np.uint32)
    sp, sq = np.zeros(p, np.int32), np.zeros(q, np.int32)
    rc = lib().ref_field_tables(p, q, wbase, ip.ctypes.data, iq.ctypes.data, sp.ctypes.data,
                                sq.ctypes.data)
    if rc:
        raise RuntimeError(last_error())
    return ip, iq, sp, sq


def field_op(op: int, a, b=(0, 0, 1), omega=4, p=227, q=113, wbase=4):
    """op 0 add 1 sub 2 mul 3 div 4 exp 5 sqrt; returns (rc, (xp, xq, qd))."""
    A = np.array(a, np.uint16)
    B = np.array(b, np.uint16)
    R = np.zeros(3, np.uint16)
    rc = lib().ref_field_op(p, q, wbase, op, omega, A.ctypes.data, B.ctypes.data, R.ctypes.data)
    return rc, tuple(int(x) for x in R)


def eval_mugraph(g, inputs: Sequence[np.ndarray], mode: int = 0) -> List[np.ndarray]:
    """mode 0 eval_mugraph (double), 1 eval_program, 2 eval_mugraph_f32."""
    ins = [np.ascontiguousarray(x, dtype=np.float64) for x in inputs]
    outs = [np.zeros(s, np.float64) for s in _shapes(g, "outputs")]
    pin = (C.c_void_p * len(ins))(*[x.ctypes.data for x in ins])
    pout = (C.c_void_p * len(outs))(*[x.ctypes.data for x in outs])
    rc = lib().ref_eval_mugraph(_js(g), mode, pin, pout)
    if rc:
        raise RuntimeError(f"ref eval failed {rc}: {last_error()}")
    return outs


def time_eval_mugraph(g, inputs, reps=1) -> float:
    ins = [np.ascontiguousarray(x, dtype=np.float64) for x in inputs]
    pin = (C.c_void_p * len(ins))(*[x.ctypes.data for x in ins])
    return lib().ref_time_eval_mugraph(_js(g), pin, reps)


def time_eval_parallel(graphs, inputs_per_graph, reps=1) -> float:
    js = [_js(g) for g in graphs]
    arrs = [[np.ascontiguousarray(x, dtype=np.float64) for x in ins] for ins in inputs_per_graph]
    inner = [(C.c_void_p * len(a))(*[x.ctypes.data for x in a]) for a in arrs]
    pj = (C.c_char_p * len(js))(*js)
    pi = (C.c_void_p * len(inner))(*[C.addressof(x) for x in inner])
    return lib().ref_time_eval_parallel(pj, pi, len(js), reps)


def ff_attempt(g, seed: int, stream: int, with_silu: Optional[bool] = None, p=227, q=113, wbase=4):
    """One verifier attempt (equiv.cpp:57-68) on a single graph.
    Returns dict(rc, omega, in_xp, in_xq, out=[(xp, xq, qd) per output])."""
    from .restate import graph_has_silu
    if with_silu is None:
        with_silu = graph_has_silu(g)
    n_in = sum(int(np.prod(s)) for s in _shapes(g, "inputs"))
    oshapes = _shapes(g, "outputs")
    n_out = sum(int(np.prod(s)) for s in oshapes)
    ixp, ixq = np.zeros(n_in, np.uint16), np.zeros(n_in, np.uint16)
    oxp, oxq, oqd = np.zeros(n_out, np.uint16), np.zeros(n_out, np.uint16), np.zeros(n_out, np.uint8)
    om = C.c_uint32(0)
    rc = lib().ref_ff_attempt(_js(g), p, q, wbase, seed, stream, int(with_silu), ixp.ctypes.data,
                              ixq.ctypes.data, oxp.ctypes.data, oxq.ctypes.data, oqd.ctypes.data,
                              C.addressof(om))
    outs, c = [], 0
    for s in oshapes:
        n = int(np.prod(s))
        outs.append((oxp[c:c + n].reshape(s), oxq[c:c + n].reshape(s), oqd[c:c + n].reshape(s)))
        c += n
    return dict(rc=rc, omega=om.value, in_xp=ixp, in_xq=ixq, out=outs)


def random_test_equivalence(g1, g2, num_tests=1, seed=0, max_resamples=16, p=227, q=113, wbase=4):
    v = RefVerdict()
    lib().ref_random_test_equivalence(_js(g1), _js(g2), num_tests, seed, max_resamples, p, q, wbase,
                                      C.addressof(v))
    return {k: getattr(v, k) for k, _ in RefVerdict._fields_}


def verify_batch(program, pool, first: int, n: int, threads: int = 1, num_tests=1,
                 max_resamples=16, p=227, q=113, wbase=4, want=True):
    """Candidate i = pool[i % len(pool)], seed i, for i in [first, first+n).
    Returns (verdicts structured array or None, wall_ms)."""
    js = [_js(g) for g in pool]
    pj = (C.c_char_p * len(js))(*js)
    out = np.zeros(n, VERDICT_NP) if want else None
    ms = lib().ref_verify_batch(_js(program), pj, len(js), first, n, num_tests, max_resamples,
                                p, q, wbase, threads, out.ctypes.data if want else None)
    return out, ms


def float_stability_filter(g, program, trials=1, tol=1e-3, seed=17, scale=1.0) -> bool:
    rc = lib().ref_float_stability_filter(_js(g), _js(program), trials, tol, seed, scale)
    if rc < 0:
        raise RuntimeError(last_error())
    return bool(rc)


def validate(g, smem_bytes=232448, elem_size=2) -> int:
    return lib().ref_validate(_js(g), smem_bytes, elem_size)


def op_madds(g) -> int:
    return lib().ref_op_madds(_js(g))


def canonical_key(g) -> str:
    n = lib().ref_canonical_key(_js(g), None, 0)
    buf = C.create_string_buffer(n)
    lib().ref_canonical_key(_js(g), buf, n)
    return buf.value.decode()


def roundtrip_json(g) -> dict:
    n = lib().ref_roundtrip_json(_js(g), None, 0)
    buf = C.create_string_buffer(n)
    lib().ref_roundtrip_json(_js(g), buf, n)
    return json.loads(buf.value.decode())


def block_shared_bytes(g, op_index: int, elem_size: int = 2) -> int:
    """validate.cpp:115-140 for the GraphDef at kernel op `op_index`."""
    return lib().ref_block_shared_bytes(_js(g), op_index, elem_size)
