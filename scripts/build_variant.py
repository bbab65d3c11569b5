#!/usr/bin/env python
"""Experiment builds: link a copy of the library in which ONE CUDA source is
compiled with extra nvcc flags (A/B of compile-time knobs on the GPU box via
TPO_NATIVE_LIB=<name>).  Not a product artefact.
  python scripts/build_variant.py libtpo_b200_rc0.so ff_vm.cu -DTPO_VM_REGCAP=0
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_05751_b200 import build as B  # noqa: E402


def main():
    name, src_name, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build()
    cu, cpp, _ = B._sources()
    objs = []
    for s in cu + cpp:
        o = B._obj(s)
        if os.path.basename(s) == src_name:
            o = o[:-2] + "." + name + ".o"
            cmd = B._cmd_cu(s, o)
            cmd[1:1] = flags
            subprocess.run(cmd, check=True, capture_output=True)
        objs.append(o)
    out = os.path.join(B.PKG, name)
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", out, *objs, "-lpthread",
                    "-ldl", "-lrt"], check=True)
    print(out)


if __name__ == "__main__":
    main()
