"""The reference-side binding (integration/tpo_gpu_backend.*), compiled
against the reference's own headers and objects into
oracle/_ref/integration_check by oracle/Makefile, checked against the
reference entry points it replaces: graphs parsed by the reference's JSON
reader, op_madds equal (CPU), verdicts bit-exact and eval_mugraph within
tolerance (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "integration_check")
GRAPHS = os.path.join(ROOT, "tests", "golden", "graphs.json")

needs_exe = pytest.mark.skipif(not os.path.exists(EXE),
                               reason="integration_check not built (make -C oracle integration)")


@needs_exe
def test_binding_host_side():
    r = subprocess.run([EXE, "host", GRAPHS], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "op_madds equal to the reference" in r.stdout


@needs_exe
@pytest.mark.gpu
def test_binding_on_gpu_matches_reference():
    r = subprocess.run([EXE, "gpu", GRAPHS], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "verdicts bit-exact" in r.stdout
