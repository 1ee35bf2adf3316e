#!/usr/bin/env python
"""Regenerates tests/golden/std_vectors.json from gen_std_vectors.cpp
(g++ -std=c++17 -O2 -ffp-contract=off)."""
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
with tempfile.TemporaryDirectory() as d:
    exe = os.path.join(d, "gen")
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-o", exe,
                           os.path.join(HERE, "gen_std_vectors.cpp")])
    out = subprocess.check_output([exe]).decode()
with open(os.path.join(HERE, "std_vectors.json"), "w") as f:
    f.write(out)
print("wrote std_vectors.json")
