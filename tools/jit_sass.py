#!/usr/bin/env python
"""Dump a bench model's specialized kernel source and compile it with nvcc
(-Xptxas -v) for register / SASS inspection.  Usage:
  jit_sass.py [gemm|2dconv|atax1] [fast|fastcm|exact] [min_blocks] [threads]
(defaults: the JIT's — FAST 32 threads x 24 blocks, FASTCM 512 x 1, EXACT 256 x 3)"""
import ctypes as C
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1906_00142_b200 import abi as A, formats as F  # noqa: E402

kern = sys.argv[1] if len(sys.argv) > 1 else "gemm"
mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
th = sys.argv[4] if len(sys.argv) > 4 else {"fast": "32", "fastcm": "512"}.get(mode, "256")
mb = sys.argv[3] if len(sys.argv) > 3 else str((512 if mode == "fastcm" else 768) // int(th))
out = "/tmp/rpg_jit_sass"
os.makedirs(out, exist_ok=True)
lib = A.load_library()
spec = F.models_to_metric_spec(F.read_models(os.path.join(ROOT, "data", "polybench", f"{kern}.models.json")))
pk = A.PackedModel(spec)
hw = A.profile_struct(F.load_profile(os.path.join(ROOT, "data", "b200.profile")))
opts = A.options_struct(arith={"fast": A.RPG_ARITH_FAST, "fastcm": A.RPG_ARITH_FAST_CM}.get(mode, A.RPG_ARITH_EXACT))
buf = C.create_string_buffer(1 << 21)
err = C.create_string_buffer(4096)
n = lib.rpg_emit_cuda_source(C.byref(pk.struct), C.byref(hw), C.byref(opts), 0, buf, len(buf), None, err, len(err))
assert n > 0, err.value
src = os.path.join(out, f"{kern}_{mode}.cu")
with open(src, "w") as f:
    f.write("#include <cstdint>\n" + buf.value.decode())
for h in ("paper_1906_00142_b200/csrc/rpg_device.cuh", "paper_1906_00142_b200/csrc/rpg_kernels.cuh", "include/rpg.h"):
    shutil.copy(os.path.join(ROOT, h), out)
cubin = src.replace(".cu", f"_{mb}.cubin")
r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-fmad=false",
                    f"-DRPG_MIN_BLOCKS={mb}", f"-DRPG_THREADS={th}", "-cubin", "-Xptxas", "-v", "-o", cubin, src],
                   capture_output=True, text=True)
print("\n".join(l for l in r.stderr.splitlines() if "registers" in l or "spill" in l or "error" in l))
print(cubin)
