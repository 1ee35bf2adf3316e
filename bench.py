#!/usr/bin/env python
"""Benchmark: MWP-CWP config evaluations/s (BASELINE.json metric), config C2.

Workload (BASELINE.json configs[1]): the 2DCONV + GEMM + ATAX rational
programs (data/polybench/*.models.json — synthetic, default-bound fitted
form, see data/polybench/make_specs.py) on the B200 device profile
(data/b200.profile); a dense data-size sweep of 65,473 consecutive N values
(N = 64..65,536) x all 7,262 integer block shapes bx*by <= 1024.  One step
= search every (kernel, N) tuple for its best configuration (evaluator +
per-N argmin) = 1.426e9 (N, bx, by) evaluations.  Multi-GPU: the same N
range is split into contiguous blocks, one per rank (strong scaling along the
data-parameter axis, the reference's static partition, pipeline.hpp:602),
and the per-N winner records are all-gathered over NCCL inside the timed
region.

`--workload c4` times the parameter-estimation fit (configs[3]: 5 metrics x
10^6 samples; samples/s; CPU baseline = O3 on a bounded sample) and
`--workload dump` the Ec-table dump (GB/s).
`--workload c3` sweeps the full 27-kernel PolyBench-GPU suite (configs[2]:
N = 64..65,536 split over the GPUs, strong scaling) and `--workload c5` the
5-variable stress model over a 182 x 182 (N, M) grid x 30,343 3-D blocks
(configs[4], 1.005e9 evaluations, strong scaling); they are extra lines, the
default stays C2.

Prints one JSON line (rank 0).  `--impl reference` times the CPU
restatement of the reference path (oracle O1, all host cores) on a bounded
sample of the same workload instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

KERNELS = ("2dconv", "gemm", "atax1")
N_PER_RANK = 65473          # 2^16 - 2^6 + 1
N0 = 64
METRIC = "MWP-CWP config evaluations/sec"
UNIT = "evals/s"

# Full PolyBench-GPU suite, paper kernel-ID order (config C3).
SUITE = ("2dconv", "fdtd2d_step1", "fdtd2d_step2", "fdtd2d_step3", "2mm1", "3mm1", "bicg1", "bicg2",
         "gemm", "3dconv", "atax1", "atax2", "gesummv", "syrk", "mvt1", "mvt2", "syr2k",
         "corr", "corr_mean", "corr_reduce", "corr_std", "covar", "covar_mean", "covar_reduce",
         "gramschmidt1", "gramschmidt2", "gramschmidt3")
C5_GRID = 182               # (N, M) grid 182 x 182 = 33,124 tuples


class Workload:
    """One BASELINE.json config: models, config space and the data tuples
    each rank sweeps.  c2 = configs[1] (the bench default, weak scaling along
    N), c3 = configs[2] (all 27 suite kernels, fixed N range split over the
    ranks), c5 = configs[4] (5-variable model, 3-D blocks, (N, M) grid split
    over the ranks)."""

    def __init__(self, name: str):
        from paper_1906_00142_b200 import formats as F
        self.name = name
        self.hw = F.load_profile(os.path.join(ROOT, "data", "b200.profile"))
        if name == "c6":
            self.kernels = ("c6_stencil", "c6_kloop", "c6_reduce")
            path = os.path.join(ROOT, "data", "stressed", "{}.models.json")
            self.space = F.integer_configs(1024, dims=2)
            self.scaling = "strong"
            self.describe = ("C6 non-degenerate landscape (data/stressed/make_c6.py): 3 T-symmetric synthetic "
                             "kernels (default-bound fitted form), regs 80 (22.5% of points infeasible), "
                             "exact multi-member tie groups, all three MWP-CWP cases; N = 64..65536 x 7262 "
                             "integer (bx,by), B200 profile")
        elif name == "c5":
            self.kernels = ("stencil3d_nm",)
            path = os.path.join(ROOT, "data", "stress", "{}.models.json")
            self.space = F.integer_configs(1024, dims=3)
            self.scaling = "strong"
            self.describe = ("C5 stress: 5-variable (D1,D2,bx,by,bz) 3-D stencil rational program (synthetic "
                             "fitted form, default bounds 243+32 terms/metric), (N,M) grid 182x182 over "
                             "[64,65536]^2 x 30343 integer (bx,by,bz), B200 profile")
        else:
            self.kernels = KERNELS if name == "c2" else SUITE
            path = os.path.join(ROOT, "data", "polybench", "{}.models.json")
            self.space = F.integer_configs(1024, dims=2)
            self.scaling = "strong"   # N = 64..65536 split over the ranks (C2 and C3)
            self.describe = ("C2: 2DCONV+GEMM+ATAX rational programs (synthetic fitted-form models, default "
                             "bounds), N = 64..65536 every integer split over the GPUs, 7262 integer (bx,by) configs, "
                             "B200 profile" if name == "c2" else
                             "C3: full PolyBench-GPU suite, 27 kernels (synthetic fitted-form models, default "
                             "bounds), N = 64..65536 every integer split over the GPUs, 7262 integer (bx,by)")
        self.specs = {k: F.models_to_metric_spec(F.read_models(path.format(k))) for k in self.kernels}

    def all_tuples(self) -> np.ndarray:
        if self.name == "c5":
            v = np.unique(np.linspace(N0, 65536, C5_GRID).round().astype(np.int64))
            nn, mm = np.meshgrid(v, v, indexing="ij")
            return np.stack([nn.ravel(), mm.ravel()], axis=1)
        return np.arange(N0, N0 + N_PER_RANK, dtype=np.int64).reshape(-1, 1)

    def tuples(self, rank: int, world: int) -> np.ndarray:
        if self.scaling == "weak":
            lo = N0 + rank * N_PER_RANK
            return np.arange(lo, lo + N_PER_RANK, dtype=np.int64).reshape(-1, 1)
        t = self.all_tuples()
        per = -(-len(t) // world)   # contiguous blocks, as pipeline.hpp:602 partitions
        return t[rank * per: (rank + 1) * per]


def load_workload():
    w = Workload("c2")
    return w.hw, w.specs, w.space


def official_flops(spec) -> int:
    """F = sum over modelled metrics (2 k_num + 2 k_den + 1)
    + 35, k = distinct block-dimension monomials with a nonzero coefficient."""
    from paper_1906_00142_b200 import formats as F
    cfg_idx = [i for i, v in enumerate(spec.variables) if v in ("bx", "by", "bz")]
    total = 35
    for name in F.METRIC_SLOTS:
        if name in spec.constants:
            continue
        f = spec.models[name]
        ks = []
        for p in (f.num, f.den):
            pats = {tuple(m[i] for i in cfg_idx) for m, c in zip(p.basis, p.coeffs) if c != 0.0}
            ks.append(len(pats))
        total += 2 * ks[0] + 2 * ks[1] + 1
    return total


def default_arith(workload: str, kernel: str) -> str:
    """The arithmetic mode a workload is benchmarked in: the configuration-
    major FAST_CM search for the one-data-parameter C2/C3/C6 models (specialized
    kernels only; also the Ec dump), FAST otherwise (C5's two data parameters)."""
    return "fastcm" if workload in ("c2", "c3", "c6", "dump") and kernel == "specialized" else "fast"


def count_kernel_launches(fn, prefix="rpg_"):
    """Kernels whose name starts with `prefix` that one call of fn launches,
    counted by the CUDA activity trace (torch.profiler / CUPTI) outside the
    timed region; None if tracing is unavailable."""
    try:
        import torch
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        return sum(1 for e in prof.events() if e.device_type.name == "CUDA" and e.name.startswith(prefix))
    except Exception:  # noqa: BLE001 - diagnostics only
        return None


def fp64_peak_tflops():
    """Measured FP64 (DFMA) peak: live run of tools/fp64_peak when built,
    else the committed measurement."""
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    if os.path.exists(exe):
        try:
            out = subprocess.run([exe], capture_output=True, text=True, timeout=60, check=True).stdout
            return json.loads(out.strip().splitlines()[-1])["fp64_fma_tflops"], "measured live (tools/fp64_peak, DFMA)"
        except Exception:
            pass
    with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")) as f:
        return json.load(f)["fp64_fma_tflops"], "measured (profiles/fp64_peak_r01.json, DFMA)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i] == "Active"})
        loaded = [v for v in sm if v > 0.5 * (max(mx) if mx else 0)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU arms (oracle O1 = the CPU restatement of the reference path)

def cpu_rate(wl: Workload, seconds_target: float, threads: int):
    """Sizes a bounded sample of the workload for O1's batched search
    (~seconds_target of CPU work): an evenly spread subset of the tuples."""
    from oracle import o1
    from paper_1906_00142_b200 import abi as A
    sp = A.config_array(wl.space)
    hws = A.profile_struct(wl.hw)
    opts = A.options_struct()
    packed = {k: A.PackedModel(wl.specs[k], drop_zero_terms=False) for k in wl.kernels}
    allt = wl.all_tuples()
    probe = max(threads, 8)
    pick = lambda n: np.ascontiguousarray(allt[np.linspace(0, len(allt) - 1, n).round().astype(np.int64)])
    ns = pick(probe)
    t = time.perf_counter()
    for k in wl.kernels:
        o1.search_batch(packed[k], hws, opts, sp, ns, threads)
    dt = time.perf_counter() - t
    per_tuple = dt / (probe * len(wl.kernels))
    n = min(len(allt), max(threads, int(seconds_target / per_tuple / len(wl.kernels))))
    return packed, hws, opts, sp, pick(n)


def run_cpu_sample(packed, hws, opts, sp, ns, threads):
    from oracle import o1
    t = time.perf_counter()
    for k in packed:
        o1.search_batch(packed[k], hws, opts, sp, ns, threads)
    dt = time.perf_counter() - t
    evals = len(packed) * len(ns) * len(sp)
    return evals / dt, dt, evals


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    wl = Workload(args.workload)
    threads = host_threads()
    packed, hws, opts, sp, ns = cpu_rate(wl, args.cpu_seconds / 2.5, threads)
    for _ in range(args.warmup):
        run_cpu_sample(packed, hws, opts, sp, ns[: max(threads, len(ns) // 4)], threads)
    times = []
    for _ in range(args.steps):
        _, dt, _ = run_cpu_sample(packed, hws, opts, sp, ns, threads)
        times.append(dt)
    value = len(packed) * len(ns) * len(sp) * args.steps / sum(times)
    sample = (f"{len(ns)} data tuples spread evenly over the workload's tuples x {len(sp)} configs "
              f"x {len(packed)} kernels per step (O1 batched search, {threads} threads)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": wl.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": wl.describe + " (bounded CPU sample)",
                   "oracle": "O1 (oracle/o1.c): FP64 CPU restatement of the reference path; the reference "
                             "itself (Eigen/Boost) cannot be built in this image"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm

def gpu_arm(args):
    import torch
    import torch.distributed as dist
    from paper_1906_00142_b200 import abi as A
    from paper_1906_00142_b200 import search as S

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:  # test mode: every rank on cuda:0 (multi-rank path on one GPU)
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    dev = torch.device("cuda", local)
    cdev = dev if args.dist_backend == "nccl" else torch.device("cpu")  # collective buffers

    wl = Workload(args.workload)
    hw, specs, space = wl.hw, wl.specs, wl.space
    opts = S.SearchOptions(arith=args.arith, kernel=args.kernel, device=local)
    plans = {k: S.Plan(specs[k], hw, space, opts) for k in wl.kernels}
    data_host = wl.tuples(rank, world)
    n_real = len(data_host)
    if wl.scaling == "strong":   # equal-sized blocks for the all-gather; padding is not counted
        per = -(-len(wl.all_tuples()) // world)
        if n_real < per:
            data_host = np.concatenate([data_host, np.repeat(data_host[-1:], per - n_real, axis=0)])
    data_host = np.ascontiguousarray(data_host)
    n, d = data_host.shape
    data_dev = torch.from_numpy(data_host).to(dev)
    out_dev = {k: torch.empty(n * A.WINNER_DTYPE.itemsize, dtype=torch.uint8, device=dev) for k in wl.kernels}
    gathered = {k: torch.empty(world * n * A.WINNER_DTYPE.itemsize, dtype=torch.uint8, device=cdev)
                for k in wl.kernels} if world > 1 else None
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    def search_only():
        for k in wl.kernels:
            plans[k].search_batch_device(data_dev.data_ptr(), n, d, out_dev[k].data_ptr(), sptr)

    # rpg_* kernels one step launches (a FAST_CM batch may run as J = 3 full
    # waves + a J = 2 remainder), counted by the CUDA activity trace outside
    # the timed region; one launch per kernel model if tracing is unavailable
    launches_per_step = count_kernel_launches(search_only) or len(wl.kernels)

    def step():
        for k in wl.kernels:
            plans[k].search_batch_device(data_dev.data_ptr(), n, d, out_dev[k].data_ptr(), sptr)
        if world > 1:
            for k in wl.kernels:
                dist.all_gather_into_tensor(gathered[k], out_dev[k].to(cdev))

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---- device-timed region (inputs resident in HBM)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.fill_(1.0)  # L2 flush between timed steps (256 MiB > 126 MB L2)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = torch.tensor([sum(times)], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    total_ms = float(total_ms.item())
    evals_per_rank_step = len(wl.kernels) * n * len(space)
    # whole-job evaluations per step (padding of strong-scaling blocks not counted)
    evals_job_step = len(wl.kernels) * len(space) * (world * n if wl.scaling == "weak" else len(wl.all_tuples()))
    value = evals_job_step * args.steps / (total_ms / 1e3)

    # Kernel-only timing of the dominant kernel (the fused search kernel) on
    # the launching stream, for the roofline.
    kt = []
    for _ in range(max(3, min(args.steps, 10))):
        flush.fill_(1.0)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(stream)
        for k in wl.kernels:
            plans[k].search_batch_device(data_dev.data_ptr(), n, d, out_dev[k].data_ptr(), sptr)
        ev[1].record(stream)
        ev[1].synchronize()
        kt.append(ev[0].elapsed_time(ev[1]) / len(wl.kernels))
    kernel_ms = statistics.median(kt)
    flops_per_launch = statistics.mean(official_flops(specs[k]) for k in wl.kernels) * n * len(space)
    achieved_tf = flops_per_launch / (kernel_ms / 1e3) / 1e12
    peak_tf, peak_src = fp64_peak_tflops()
    # Per-workload ncu evidence (null when this workload has no capture):
    # DRAM bytes of one launch (--set full) and executed FP64 FLOPs per
    # evaluation (instruction-mix metrics).
    traffic = executed_flops = None
    tfile = os.path.join(ROOT, "profiles", f"search_kernel_traffic_{wl.name}.json")
    if os.path.exists(tfile):
        with open(tfile) as f:
            traffic = json.load(f).get("bytes_per_launch")
    mfile = os.path.join(ROOT, "profiles", f"search_kernel_mix_{wl.name}.json")
    if os.path.exists(mfile):
        with open(mfile) as f:
            executed_flops = json.load(f).get("executed_flops_per_eval")

    # ---- end-to-end through the public C-ABI host API (pinned host buffers)
    pinned = torch.from_numpy(data_host).pin_memory()
    pinned_np = pinned.numpy()
    # Output records land in pinned host buffers too (search_batch(out=...)).
    e2e_out = {k: torch.empty(n * A.WINNER_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
               .numpy().view(A.WINNER_DTYPE) for k in wl.kernels}
    for k in wl.kernels:  # warm the host-API staging buffers
        plans[k].search_batch(pinned_np, out=e2e_out[k])
    if world > 1:
        dist.barrier()
    e2e_times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        for k in wl.kernels:
            plans[k].search_batch(pinned_np, out=e2e_out[k])
        e2e_times.append(time.perf_counter() - t0)
    e2e_total = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(e2e_total, op=dist.ReduceOp.MAX)
    e2e_value = evals_job_step * args.steps / float(e2e_total.item())
    h2d = len(wl.kernels) * data_host.nbytes
    d2h = len(wl.kernels) * n * A.WINNER_DTYPE.itemsize

    # ---- agreement spot check against the device-API winners
    chk = {k: out_dev[k].cpu().numpy().view(A.WINNER_DTYPE) for k in wl.kernels}
    agree = all(np.array_equal(chk[k], e2e_out[k]) for k in wl.kernels)

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = host_threads()
        packed, hws, o, sp, ns = cpu_rate(wl, args.cpu_seconds, threads)
        rate, dt, evals = run_cpu_sample(packed, hws, o, sp, ns, threads)
        cpu_baseline = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                        "sample": f"O1 batched search, {len(ns)} data tuples x {len(sp)} configs x "
                                  f"{len(wl.kernels)} kernels ({evals:.3g} evals, {dt:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": wl.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl.describe, "id": wl.name,
                       "tuples_per_gpu": n_real, "tuples_rank0": [data_host[0].tolist(), data_host[n_real - 1].tolist()],
                       "configs": len(space), "evals_job_step": evals_job_step,
                       "kernels": list(wl.kernels), "evals_per_gpu_step": evals_per_rank_step,
                       "arith": args.arith, "kernel": args.kernel,
                       "parallelism": f"data-tuple shard x{world} ({wl.scaling}), NCCL all-gather of winners",
                       "l2": "flushed between timed steps (256 MiB write)"},
            "roofline": {"bound": "fp64", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved_tf / peak_tf, "traffic": traffic,
                         "kernel": "search_kernel (fused evaluator + per-N argmin)",
                         "flops_per_eval": statistics.mean(official_flops(specs[k]) for k in wl.kernels),
                         "flops_basis": "FLOP-equivalent: SURVEY 8(d) official F per evaluation (minimal "
                                        "per-point work after the per-N collapse), not the FP64 FLOPs "
                                        "the kernel executes",
                         "executed_flops_per_eval_ncu": executed_flops,
                         "kernel_ms": kernel_ms, "peak_source": peak_src},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "api": "rpg_search_batch (pinned host buffers in and out)"},
            "cpu_baseline": cpu_baseline,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks.summary(),
            "agreement_device_vs_host_api": agree,
        }
        print(json.dumps(line), flush=True)
    for p in plans.values():
        p.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# C4: the parameter-estimation fit (BASELINE.json configs[3])

C4_SAMPLES = 1_000_000
C4_CPU_SAMPLES = 20_000     # bounded sample for the O3 CPU legs


def c4_data(m: int, noise: float = 0.01, seed: int = 1906):
    """Synthetic profiled samples: D1 uniform over [64, 65536], (bx, by)
    uniform over the 7,262 integer configs, y = the GEMM ground truth x
    (1 + U(-noise, noise)) per metric.  numpy, seeded."""
    from paper_1906_00142_b200 import formats as F
    rng = np.random.default_rng(seed)
    D = rng.integers(64, 65537, m).astype(float)
    cfg = np.array(F.integer_configs(), dtype=float)[rng.integers(0, 7262, m)][:, :2]
    X = np.ascontiguousarray(np.column_stack([D, cfg]))
    spec = F.load_kernel_spec(os.path.join(ROOT, "data", "polybench", "gemm.kernel.json"))

    def poly(p):
        out = np.zeros(m)
        for mono, c in zip(p.basis, p.coeffs):
            if c != 0.0:
                out += c * np.prod(X ** np.asarray(mono, dtype=float), axis=1)
        return out

    ys = {}
    for name in F.REQUIRED_METRICS:
        f = spec.ground_truth[name]
        y = poly(f.num) / poly(f.den)
        if noise > 0:
            y = y * (1 + rng.uniform(-noise, noise, m))
        ys[name] = np.ascontiguousarray(y)
    return X, ys, spec.variables


def c4_cpu(threads: int, m: int = C4_CPU_SAMPLES):
    """O3 (numpy/LAPACK restatement of fit_rational) on a bounded sample."""
    from oracle import o3_fit as O3
    X, ys, var = c4_data(m)
    t0 = time.perf_counter()
    for y in ys.values():
        try:
            O3.fit_rational(X, y, var, [2, 2, 2], [1, 1, 1])
        except O3.DegenerateFit:
            pass
    dt = time.perf_counter() - t0
    return len(ys) * m / dt, dt, m


def c4_arm(args):
    """C4 fit: fit_all_metrics over the 5 GEMM metrics (host buffers in, the
    H2D copies inside the step).  Under torch.distributed.run the metrics are
    sharded over the ranks (dist.sharded_fit_all_metrics: strong scaling, the
    fitted models all-gathered inside the step); the step time is the max
    over ranks."""
    import torch
    import torch.distributed as dist
    from paper_1906_00142_b200 import dist as D
    from paper_1906_00142_b200 import fit as G

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if args.same_device else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    X, ys, var = c4_data(C4_SAMPLES)
    # The samples live in pinned host buffers (as the C2 e2e line's tuples
    # do); the fit API reads them in place (contiguous float64: no copy), so
    # its H2D inside the step runs at DMA speed.
    X = torch.from_numpy(X).pin_memory().numpy()
    ys = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in ys.items()}
    bounds = {k: ([2, 2, 2], [1, 1, 1]) for k in ys}

    def step():
        if world > 1:
            return D.sharded_fit_all_metrics(X, ys, var, bounds, {}, device=local)
        return G.fit_all_metrics(X, ys, var, bounds, {}, device=local)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(max(1, args.warmup)):
        models = step()
    times = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            barrier()
            t0 = time.perf_counter()
            models = step()
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
    t = torch.tensor([statistics.median(times)], dtype=torch.float64)
    if world > 1:
        if args.dist_backend == "nccl":
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_s = float(t.cpu()[0])
    per_step = count_kernel_launches(step) if world == 1 else None  # (a collective step cannot run on one rank)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    # Parity at the benchmarked arrays (untimed): each metric's GPU outcome,
    # stage by stage, against oracle O3's committed outcome on the same
    # arrays (tests/golden/c4_o3_noisy.json; rule in tools/fit_c4_compare.py
    # agreement / tests/test_gpu_fit_c4.py).
    parity = None
    fx = os.path.join(ROOT, "tests", "golden", "c4_o3_noisy.json")
    if os.path.exists(fx):
        sys.path.insert(0, ROOT)
        from tools.fit_c4_compare import agreement, holdout_points, monomials, outcome
        with open(fx) as f:
            o3 = json.load(f)["metrics"]
        from paper_1906_00142_b200 import formats as F
        Dm = monomials(F.monomial_basis([1, 1, 1]), X)
        H = holdout_points()
        parity = {}
        for name in sorted(ys):
            g = outcome(G.fit_rational, X, ys[name], var, (G.DegenerateFit, G.SvdFailure))
            a = agreement(g, o3[name], Dm, H)
            parity[name] = {k: a[k] for k in ("agree", "gpu_status", "o3_status", "gpu_stop", "o3_stop",
                                              "stages_compared", "stage_max_diff", "diverged_at", "ill_posed_guard")}
            if g["status"] == "failed":
                parity[name]["gpu_message"] = g["message"]
    samples = len(ys) * C4_SAMPLES
    n = 35
    qr_flops = len(ys) * (2 * C4_SAMPLES * n * n - 2 * n ** 3 / 3 + 3 * C4_SAMPLES * n)
    peak_tf, peak_src = fp64_peak_tflops()
    cpu = None
    if not args.no_cpu:
        threads = host_threads()
        rate, dt, m = c4_cpu(threads)
        cpu = {"value": rate, "unit": "samples/s", "cores": threads, "kind": "port",
               "sample": f"O3 (numpy/LAPACK fit_rational restatement), 5 metrics x {m} samples ({dt:.1f} s)"}
    print(json.dumps({
        "metric": "C4 rational-fit throughput (samples fitted per second)", "value": samples / step_s,
        "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * step_s, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C4: 5 GEMM metrics x 10^6 samples each, variables (D1,bx,by), bounds num "
                               "(2,2,2) / den (1,1,1) -> 10^6 x 35 sample matrices, 1% uniform noise "
                               "(positivity safeguard active)", "id": "c4",
                   "api": "fit_all_metrics -> rpg_fit_rational_multi (pinned host buffers, H2D inside the step)"
                          + (f"; metrics sharded over {world} ranks, models all-gathered" if world > 1 else ""),
                   "fitted": sorted(models.models), "failed": sorted(models.failures),
                   "o3_parity": parity},
        "roofline": {"bound": "fp64", "achieved": qr_flops / step_s / 1e12, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": qr_flops / step_s / 1e12 / peak_tf, "traffic": None,
                     "note": "QR-equivalent FLOPs (2mn^2 - 2n^3/3 + 3mn per metric); the positivity "
                             "minimizer's sample passes are extra work not counted", "peak_source": peak_src},
        "e2e": {"value": samples / step_s, "unit": "samples/s",
                "h2d_bytes_per_step": int(X.nbytes + sum(v.nbytes for v in ys.values())),  # X once
                "d2h_bytes_per_step": len(ys) * n * 8},
        "gpu_launches": per_step * args.steps if per_step is not None else None,
        "gpu_launches_note": "rank 0's rpg_* kernels per step (CUDA activity trace of one extra untimed step) x steps",
        "cpu_baseline": cpu, "clocks": clocks.summary()}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def c4_reference_arm(args):
    """The reference's fit path (O3 port: numpy/LAPACK) on a bounded sample."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    threads = host_threads()
    c4_cpu(threads, 2000)  # warm-up
    times, rate = [], 0.0
    for _ in range(args.steps):
        rate, dt, m = c4_cpu(threads)
        times.append(dt)
    value = 5 * C4_CPU_SAMPLES * args.steps / sum(times)
    sample = f"O3 fit_rational, 5 metrics x {C4_CPU_SAMPLES} samples per step"
    print(json.dumps({
        "metric": "C4 rational-fit throughput (samples fitted per second)", "value": value,
        "unit": "samples/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": "C4 (bounded CPU sample)", "id": "c4"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
        flush=True)
    return 0


def dump_arm(args):
    """Ec-table dump (BASELINE.md §3 last row): rpg_evaluate_device writes the
    full per-point table — f64 Ec + u8 case tag + i32 occupancy warps, 13 B per
    point — for the C2 2DCONV model over 8,192 consecutive N x 7,262 configs
    (59.5 M points, 773 MB per step).  Reported as HBM GB/s against the
    measured copy bandwidth; the point model bounds it, not HBM."""
    import torch
    from paper_1906_00142_b200 import search as S
    torch.cuda.set_device(0)
    wl = Workload("c2")
    spec = wl.specs["2dconv"]
    n = 8192
    data = torch.arange(N0, N0 + n, dtype=torch.int64, device="cuda").reshape(n, 1)
    pts = n * len(wl.space)
    ec = torch.empty(pts, dtype=torch.float64, device="cuda")
    tag = torch.empty(pts, dtype=torch.uint8, device="cuda")
    wocc = torch.empty(pts, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    with S.Plan(spec, wl.hw, wl.space, S.SearchOptions(arith=args.arith)) as plan:
        run = lambda: plan.evaluate_device(data.data_ptr(), n, 1, ec.data_ptr(), tag.data_ptr(),
                                           wocc.data_ptr(), stream.cuda_stream)
        for _ in range(max(3, args.warmup)):
            run()
        torch.cuda.synchronize()
        times = []
        with ClockSampler(0) as clocks:
            for _ in range(args.steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                run()
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
    ms = statistics.median(times)
    nbytes = pts * 13
    gbs = nbytes / (ms / 1e3) / 1e9
    peak = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = json.load(f)["hbm_gbs"]
    except (OSError, KeyError, ValueError):
        pass
    print(json.dumps({
        "metric": "Ec-table dump bandwidth", "value": gbs, "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 2DCONV model, N = 64..8255 x 7262 integer (bx,by): Ec f64 + tag u8 + "
                               "occupancy i32 per point (13 B)", "points": pts, "bytes_per_step": nbytes,
                   "points_per_s": pts / (ms / 1e3), "arith": args.arith},
        "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                     "frac": (gbs / peak) if peak else None, "traffic": None,
                     "note": "store traffic of the evaluate kernel; the FP64 point model, not HBM, bounds it"},
        "gpu_launches": args.steps, "clocks": clocks.summary()}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["c2", "c3", "c4", "c5", "c6", "dump"], default="c2",
                    help="BASELINE.json config: c2 (default, configs[1]), c3 (full suite), c5 (stress)")
    ap.add_argument("--arith", choices=["exact", "fast", "fastcm"], default=None,
                    help="default: fastcm (configuration-major) for the one-data-parameter C2/C3 "
                         "searches, fast otherwise (C5's two data parameters, the Ec dump)")
    ap.add_argument("--kernel", choices=["specialized", "generic"], default="specialized")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default) | gloo (test mode)")
    ap.add_argument("--same-device", action="store_true",
                    help="test mode: all ranks on cuda:0 (with --dist-backend gloo)")
    args = ap.parse_args()
    if args.arith is None:
        args.arith = default_arith(args.workload, args.kernel)
    if args.impl == "reference":
        if args.workload == "c4":
            return c4_reference_arm(args)
        if args.workload == "dump":
            args.workload = "c2"
        return reference_arm(args)
    if args.workload == "dump":
        return dump_arm(args)
    if args.workload == "c4":
        return c4_arm(args)
    return gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
