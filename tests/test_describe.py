"""`describe` (the reference's absent describe.cpp): the
SPEC's examples — the Fig. 2(b) µGraph lists grid 128, loop i=16 and two
accumulators; an empty graph lists nothing; every DimMap of the JSON
appears in the listing — plus the B200 execution line."""
import re

import pytest

from paper_2405_05751_b200 import api
from paper_2405_05751_b200 import fixtures as F


def _maps(g):
    out = []
    for op in g["ops"]:
        for b in op.get("blockGraph", {}).get("ops", []):
            for k in ("imap", "fmap", "omap"):
                if k in b.get("attrs", {}):
                    out.append((b["type"], k, b["attrs"][k]))
    return out


def _fmt(m, grid):
    axes = ["x", "y", "z"] if grid else ["i"]
    items = sorted(m.items(), key=lambda kv: (axes + list(m)).index(kv[0]))
    return "{" + ", ".join(f"{a}: {'phi' if v == 'phi' else v}" for a, v in items) + "}"


def test_fig2b_listing():
    _, mu = F.bench_pair("rmsnorm")
    txt = api.describe(mu)
    assert "grid (128, 1, 1)  forloop i=16" in txt
    assert "accumulators 2" in txt
    assert txt.count("accum(") == 2
    assert "---- sync" in txt and "@smem+" in txt
    assert "fused sm_100a kernel rmsnorm_matmul" in txt


def test_empty_graph():
    assert api.describe({"tensors": [], "ops": [], "inputs": [], "outputs": []}) == ""


def test_all_dimmaps_round_trip():
    for fam in ("rmsnorm", "gatedmlp", "gqa", "lora"):
        for _, g in F.verify_families()[fam][1][:10]:
            txt = api.describe(g)
            for typ, k, m in _maps(g):
                assert f"{k} {_fmt(m, k != 'fmap')}" in txt, (fam, typ, k, m)


def test_vm_line_for_unfused_graphs():
    prog, _ = F.verify_families()["gqa"]
    txt = api.describe(prog)
    m = re.search(r"VM bytecode: (\d+) instructions in (\d+) barrier phases", txt)
    assert m and 0 < int(m.group(2)) <= int(m.group(1))


@pytest.mark.parametrize("fam", ["rmsnorm", "gatedmlp", "gqa", "lora"])
def test_mutants_never_take_a_fused_kernel(fam):
    """An op-rewrite mutant of a BASELINE µGraph computes something else: the
    structural fused-kernel match must reject it (the generic VM runs it)."""
    from paper_2405_05751_b200 import fixtures as F
    _, mu = F.bench_pair(fam)
    assert "B200: fused" in api.describe(mu)
    for g in F.search_stream([mu], 40, seed=2)[1:]:
        assert "no fused kernel" in api.describe(g)
