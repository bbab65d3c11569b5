"""CPU checks of the C-ABI library: it loads, exports every entry point
include/tpo_gpu.h declares, and its host-side pieces (JSON parse, validate,
op_madds, fused-pattern matching) agree with the reference — no GPU calls."""
import ctypes as C
import json

import pytest

from oracle import ref
from paper_2405_05751_b200 import _native as N
from paper_2405_05751_b200 import api, fixtures as F


def test_library_exports_declared_symbols():
    lib = N.lib()
    syms = N.declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.tpo_gpu_abi_version() == 1


def _compile_host(g):
    """tpo_gpu_compile needs no device: ctx may be NULL."""
    h = C.c_void_p()
    rc = N.lib().tpo_gpu_compile(None, json.dumps(g).encode(), C.byref(h))
    return rc, h


@pytest.mark.parametrize("fam", list(F.VERIFY_SHAPES))
def test_compile_validate_madds_match_reference(fam):
    prog, pool = F.verify_families()[fam]
    for tag, g in [("program", prog)] + pool[::5]:
        rc, h = _compile_host(g)
        assert rc == 0, (tag, N.last_error())
        info = N.GraphInfo()
        N.lib().tpo_gpu_graph_info(h, C.byref(info))
        assert info.madds == ref.op_madds(g), tag
        assert info.lax == 1
        N.lib().tpo_gpu_graph_free(h)
        for smem in (48 * 1024, 232448):
            n, _ = api.validate(g, smem_bytes=smem)
            assert n == ref.validate(g, smem_bytes=smem), (tag, smem)


def test_bench_graphs_validate_and_match():
    for name in F.BENCH:
        prog, mu = F.bench_pair(name)
        assert api.validate(mu)[0] == 0 == ref.validate(mu)
        assert api.validate(mu, smem_bytes=48 * 1024)[0] == ref.validate(mu, smem_bytes=48 * 1024)
        rc, h = _compile_host(mu)
        assert rc == 0, N.last_error()
        N.lib().tpo_gpu_graph_free(h)


def test_compile_errors_are_statuses():
    rc, _ = _compile_host({"tensors": [], "ops": [{"id": 0, "type": "nope"}], "inputs": [],
                           "outputs": []})
    assert rc == 1000 + 10  # ParseError
    rc = N.lib().tpo_gpu_compile(None, b"{not json", C.byref(C.c_void_p()))
    assert rc == 1010
    assert "parse" in N.last_error().lower() or "syntax" in N.last_error().lower()


def test_compile_many_matches_compile():
    """tpo_gpu_compile_many (parallel host compile of a candidate stream):
    per-graph handles and statuses equal one-at-a-time tpo_gpu_compile,
    including parse and validation failures."""
    graphs = []
    for fam in F.VERIFY_SHAPES:
        prog, pool = F.verify_families()[fam]
        graphs += [json.dumps(g) for _, g in pool[::7]]
    bad_shape = json.loads(graphs[0])
    bad_shape["tensors"][0]["shape"] = [3, 5, 7, 11, 13]   # rank 5: rejected
    graphs += ["{not json", json.dumps(bad_shape)]
    n = len(graphs)
    lib = N.lib()
    arr = (C.c_char_p * n)(*[g.encode() for g in graphs])
    hs = (C.c_void_p * n)()
    st = (C.c_int32 * n)()
    assert lib.tpo_gpu_compile_many(None, arr, C.c_int64(n), C.c_int32(4), hs, st) == 0
    for i, g in enumerate(graphs):
        h1 = C.c_void_p()
        rc = lib.tpo_gpu_compile(None, g.encode(), C.byref(h1))
        assert st[i] == rc, (i, st[i], rc)
        if rc == 0:
            a, b = N.GraphInfo(), N.GraphInfo()
            lib.tpo_gpu_graph_info(C.c_void_p(hs[i]), C.byref(a))
            lib.tpo_gpu_graph_info(h1, C.byref(b))
            assert (a.madds, a.vm_words, a.fused_kind) == (b.madds, b.vm_words, b.fused_kind)
            lib.tpo_gpu_graph_free(C.c_void_p(hs[i]))
            lib.tpo_gpu_graph_free(h1)
        else:
            assert not hs[i]
    from paper_2405_05751_b200.graph import ErrCode
    assert st[n - 2] == 1000 + int(ErrCode.ParseError)
    assert st[n - 1] != 0


def _parse_check(text):
    fa, same = C.c_int32(-1), C.c_int32(-1)
    rc = N.lib().tpo_gpu_parse_check(text.encode(), C.byref(fa), C.byref(same))
    return rc, fa.value, same.value


def test_json_fast_path_equals_generic_parser():
    """The wire-format fast path (host/fastjson.cpp) yields exactly the
    generic parser's graph on every golden graph and pool graph, and hands
    everything outside its strict subset to the generic parser."""
    import os
    here = os.path.dirname(os.path.abspath(__file__))
    golden = json.load(open(os.path.join(here, "golden", "graphs.json")))
    texts = [json.dumps(g) for g in (golden.values() if isinstance(golden, dict) else golden)]
    for fam in F.VERIFY_SHAPES:
        prog, pool = F.verify_families()[fam]
        texts += [json.dumps(prog)] + [json.dumps(g) for _, g in pool]
    for t in texts:
        t = t if isinstance(t, str) else json.dumps(t)
        rc, fa, same = _parse_check(t)
        if rc != 0:
            continue  # invalid golden entries: both paths reject (status checked below)
        assert fa == 1 and same == 1, t[:200]
    # outside the subset: floats, escapes, pretty-printing with tabs, leading zeros
    g = json.loads(texts[0])
    alt = json.dumps(g, indent="\t")
    assert _parse_check(alt)[1:] == (1, 1)
    flt = json.dumps(g).replace('"forloop": 4', '"forloop": 4.0', 1)
    rc, fa, _ = _parse_check(flt)
    assert rc == 0 and (fa == 0 or flt == json.dumps(g))
    rc, fa, _ = _parse_check(json.dumps(g).replace('"shape": [', '"shape": [0', 1))
    assert fa == 0
    rc, fa, _ = _parse_check("{not json")
    from paper_2405_05751_b200.graph import ErrCode
    assert rc == 1000 + int(ErrCode.ParseError) and fa == 0


def test_compile_many_batch_handles():
    """compile_many(batch=True): one GraphBatch (handle array + statuses, no
    per-graph Python objects) whose statuses match the list form; a graph
    that fails to compile leaves a NULL handle; collecting the batch frees
    the handles."""
    from paper_2405_05751_b200 import api

    class _NoDevice:  # compile_many needs no device (the C-ABI ignores ctx)
        h = None

    texts = [json.dumps(g) for _, g in F.verify_families()["lora"][1][::5]] + ["{not json"]
    gb, st = api.Context.compile_many(_NoDevice(), texts, batch=True)
    assert len(gb) == len(texts)
    assert st[:-1] == [0] * (len(texts) - 1) and st[-1] == 1010
    assert all(gb.arr[i] for i in range(len(texts) - 1)) and not gb.arr[len(texts) - 1]
    gl, stl = api.Context.compile_many(_NoDevice(), texts)
    assert stl == st and gl[-1] is None
    del gb, gl
