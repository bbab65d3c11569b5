"""Thread-graph chains change GPU execution (§4.2):
the VM lowering folds a Sqr / Sqrt / SiLU whose only consumer is an
elementwise binary of the same thread group (the graph's ThreadGroups, or
the fuser's rule) into that binary's instruction (kernels/vm.h pre_a /
pre_b): one instruction and one barrier phase fewer, the interior tensor
in registers.  Checked on CPU through `describe` with the chains on and off
(TPO_VM_CHAINS=0 in a subprocess); parity with the reference is covered by
the GPU suites (verdicts, ff_eval outputs, fp64 VM) that run with chains on."""
import json
import os
import re
import subprocess
import sys

from paper_2405_05751_b200 import api
from paper_2405_05751_b200 import fixtures as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def vm_stats(graphs, chains=True):
    code = ("import json, sys; sys.path.insert(0, %r); from paper_2405_05751_b200 import api; "
            "gs = json.load(sys.stdin); print(json.dumps([api.describe(g).splitlines()[-1] for g in gs]))" % ROOT)
    env = dict(os.environ, TPO_VM_CHAINS="1" if chains else "0")
    r = subprocess.run([sys.executable, "-c", code], input=json.dumps(graphs), capture_output=True, text=True,
                       env=env, check=True)
    out = []
    for line in json.loads(r.stdout):
        m = re.search(r"VM bytecode: (\d+) instructions in (\d+) barrier phases, (\d+) words", line)
        fused = re.search(r"(\d+) thread-graph unary", line)
        out.append((int(m.group(1)), int(m.group(2)), int(m.group(3)), int(fused.group(1)) if fused else 0))
    return out


def test_chains_fold_into_their_consumers():
    graphs = []
    for fam in ("rmsnorm", "gatedmlp"):
        _, pool = F.verify_families()[fam]
        graphs += [g for tag, g in pool if tag.endswith("/eq")][:8]
    on, off = vm_stats(graphs, True), vm_stats(graphs, False)
    for (i1, p1, w1, f1), (i0, p0, w0, f0) in zip(on, off):
        assert f1 >= 1 and f0 == 0
        assert i1 == i0 - f1 and p1 <= p0 and w1 <= w0


def test_explicit_thread_groups_drive_the_fusion():
    """With ThreadGroups present only their chains are fused: the fuser's
    groups (construct_thread_graphs) fold; a graph whose groups leave the
    unary alone keeps it."""
    _, pool = F.verify_families()["rmsnorm"]
    g = pool[4][1]
    tg = api.construct_thread_graphs(g)
    assert any(op.get("blockGraph", {}).get("threadGroups") for op in tg["ops"])
    (a,) = vm_stats([tg])
    assert a[3] >= 1
    lone = json.loads(json.dumps(g))
    for op in lone["ops"]:
        if op["type"] == "graphdef":
            first = op["blockGraph"]["ops"][4]["id"]
            op["blockGraph"]["threadGroups"] = [{"ops": [first], "blockDims": [128, 1, 1], "forloop": 1}]
    if api.validate(lone)[0] == 0:
        (b,) = vm_stats([lone])
        assert b[3] == 0
