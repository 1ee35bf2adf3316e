#!/usr/bin/env python
"""Builds librpgpu.so with extra nvcc defines into build/<name>/ (A/B
measurements of compile-time variants; load with RPG_LIBRARY=...).

Usage: python tools/build_variant.py NAME -DMACRO=VALUE [...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as G  # noqa: E402


def main():
    name, defines = sys.argv[1], sys.argv[2:]
    G._embed_sources()
    out = os.path.join(ROOT, "build", name)
    os.makedirs(out, exist_ok=True)
    lib = os.path.join(out, "librpgpu.so")
    srcs = ["rpg_search.cu", "rpg_jit.cu", "rpg_fit.cu", "rpg_altarr.cu", "rpg_multi.cu", "rpg_csv.cpp"]
    cmd = [G._nvcc()] + G.NVCC_FLAGS + defines + ["-I", os.path.join(ROOT, "include"), "-shared", "-o", lib] + \
        [os.path.join(G.CSRC, f) for f in srcs] + ["-lnvrtc"]
    subprocess.run(cmd, check=True, cwd=ROOT)
    print(lib)


if __name__ == "__main__":
    main()
