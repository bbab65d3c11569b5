"""Builds the in-tree native library ``paper_2405_05751_b200/libtpo_b200.so``.

CUDA sources are compiled for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a -lineinfo``); host C++ with g++.
The CUDA runtime is linked statically so the library does not depend on the
runtime version torch bundles.  nlohmann/json 3.11.3 (the reference's JSON
dependency) comes from the image's cudnn_frontend copy.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libtpo_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
JSON_DIR = os.environ.get(
    "TPO_JSON_DIR",
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = ["-I", os.path.join(CSRC, "include"), "-I", JSON_DIR, "-I", os.path.join(ROOT, "include"),
       "-I", os.path.join(CUDA, "include")]


def _sources():
    cu = sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu")))
    cpp = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    hdr = (glob.glob(os.path.join(CSRC, "**", "*.h*"), recursive=True)
           + glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
           + glob.glob(os.path.join(ROOT, "include", "*.h")))
    return cu, cpp, hdr


def _obj(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(BUILD, rel + ".o")


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def _cmd_cu(src, obj):
    return [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
            "--expt-relaxed-constexpr", "-Xptxas", "-v", *INC, "-c", src, "-o", obj]


def _cmd_cpp(src, obj):
    return ["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-Wno-unused-function", *INC, "-c",
            src, "-o", obj]


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    cu, cpp, hdr = _sources()
    jobs = []
    for s in cu:
        o = _obj(s)
        if force or _stale(o, [s] + hdr):
            jobs.append((s, o, _cmd_cu(s, o)))
    for s in cpp:
        o = _obj(s)
        if force or _stale(o, [s] + hdr):
            jobs.append((s, o, _cmd_cpp(s, o)))

    def run(job):
        s, o, cmd = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"compile failed: {s}\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        with open(o + ".log", "w") as f:
            f.write(r.stdout + r.stderr)
        if verbose:
            print(f"compiled {os.path.relpath(s, PKG)}", file=sys.stderr)
        return s

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(run, jobs))
    objs = [_obj(s) for s in cu + cpp]
    if jobs or force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lpthread", "-ldl",
               "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"link failed\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"linked {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
