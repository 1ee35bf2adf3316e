"""Per-call latency of the drop-in on the reference's real usage: one
`ratprog search --models M --profile P --size N` process per data size
(ratprog_cli.cpp:277-332), one tuple x the 51 default configurations.

Prints one JSON line per case (wall seconds of the whole process, cold =
fresh persistent cubin cache directory):
  exact_auto        the default path: ahead-of-time generic kernel, no NVRTC
  fastcm_cold       specialized kernel, NVRTC compile (empty cache)
  fastcm_warm       specialized kernel loaded from the on-disk cubin cache
  specialized_cold / specialized_warm   exact arithmetic, specialized kernel
and the CPU path for the same call: oracle O1 (the reference's FP64 direct
path) searching one tuple x 51 configurations in-process, and the process
wall time of a Python process doing only that (for scale)."""
from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CLI = os.path.join(ROOT, "paper_1906_00142_b200", "ratprog-b200")
MODELS = os.path.join(ROOT, "data", "polybench", "gemm.models.json")
PROFILE = os.path.join(ROOT, "data", "b200.profile")


def run(args, env, reps=1):
    best = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = subprocess.run([CLI] + args, capture_output=True, text=True, env=env, timeout=600)
        best.append(time.perf_counter() - t0)
        if r.returncode != 0:
            raise RuntimeError(r.stderr)
    return best, r.stderr.strip()


def main():
    base = ["search", "--models", MODELS, "--profile", PROFILE, "--size", "1024", "--format", "csv",
            "-o", os.devnull]
    cache = tempfile.mkdtemp(prefix="rpgcache")
    env = dict(os.environ, RPG_CACHE_DIR=cache)
    out = {}
    try:
        # CUDA/driver warm-up of the box (first process pays module loading)
        run(base, env)
        t, _ = run(base, env, reps=5)
        out["exact_auto"] = min(t)
        t, _ = run(base + ["--arith", "fastcm"], env)
        out["fastcm_cold"] = t[0]
        t, _ = run(base + ["--arith", "fastcm"], env, reps=3)
        out["fastcm_warm"] = min(t)
        t, _ = run(base + ["--kernel", "specialized"], env)
        out["specialized_cold"] = t[0]
        t, msg = run(base + ["--kernel", "specialized"], env, reps=3)
        out["specialized_warm"] = min(t)
        out["chosen"] = msg
    finally:
        shutil.rmtree(cache, ignore_errors=True)
    # CPU path: O1 in-process for the same call
    import numpy as np
    from oracle import o1
    from paper_1906_00142_b200 import abi as A
    from paper_1906_00142_b200 import formats as F
    spec = F.models_to_metric_spec(F.read_models(MODELS))
    hw = F.load_profile(PROFILE)
    space = F.enumerate_configs()
    pk = A.PackedModel(spec, drop_zero_terms=False)
    hws, opts = A.profile_struct(hw), A.rpg_options()
    opts.tie_rel_tol = 1e-12
    cfg = A.config_array(space)
    data = np.array([1024], dtype=np.int64)
    o1.search_one(pk, hws, opts, cfg, data)
    t0 = time.perf_counter()
    for _ in range(100):
        o1.search_one(pk, hws, opts, cfg, data)
    out["o1_inprocess_per_call"] = (time.perf_counter() - t0) / 100
    t0 = time.perf_counter()
    subprocess.run([sys.executable, "-c", "import sys; sys.path.insert(0, %r); "
                    "from oracle import o1; o1.lib()" % ROOT], check=True)
    out["python_o1_process_startup"] = time.perf_counter() - t0
    probe = os.path.join(ROOT, "tools", "percall_probe")
    if os.path.exists(probe):
        cache2 = tempfile.mkdtemp(prefix="rpgcache")
        env2 = dict(os.environ, RPG_CACHE_DIR=cache2)
        out["phases_ms"] = []
        for mode in ("generic", "specialized", "specialized", "fastcm", "fastcm"):
            t0 = time.perf_counter()
            r = subprocess.run([probe, MODELS, PROFILE, mode], capture_output=True, text=True, env=env2)
            wall = time.perf_counter() - t0
            d = json.loads(r.stdout) if r.returncode == 0 else {"error": r.stderr[-300:]}
            d["process_wall_ms"] = 1e3 * wall
            out["phases_ms"].append(d)
        shutil.rmtree(cache2, ignore_errors=True)
    print(json.dumps({"metric": "cold single-call wall time (1 tuple x 51 configs)", "unit": "s",
                      "workload": "ratprog-b200 search --models gemm --size 1024", **out}))


if __name__ == "__main__":
    main()
