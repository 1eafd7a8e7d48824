"""FasterTucker SGD epoch benchmark (BASELINE.json metric: nonzeros/sec per SGD epoch, factor
update + core update), Netflix-shaped synthetic tensor, J = R = 32 on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config netflix32]

A step is one SGD epoch: N factor sweeps (+ C refresh + guard) then N core sweeps (+ apply +
refresh + guard) over the whole training tensor, evaluation excluded (train.py:263-277).
Rank 0 prints ONE JSON line.  See DESIGN.md "Measurement" for every field.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "nonzeros/sec per SGD epoch (factor update, core update)"

CONFIGS = {
    # BASELINE.json configs[1]: Netflix-shaped, |Omega| / |Gamma| of PAPER.md:918-919
    "netflix32": dict(dims=(480_189, 17_770, 2_182), nnz_train=99_072_112, nnz_test=1_408_395,
                      J=32, R=32, value_range=(1.0, 5.0)),
    "netflix16": dict(dims=(480_189, 17_770, 2_182), nnz_train=99_072_112, nnz_test=1_408_395,
                      J=16, R=16, value_range=(1.0, 5.0)),
    "yahoo32": dict(dims=(1_000_990, 624_961, 3_075), nnz_train=250_272_286, nnz_test=2_527_989,
                    J=32, R=32, value_range=(0.025, 5.0)),
    "config1": dict(dims=(1000, 1000, 1000), nnz_train=90_000, nnz_test=10_000, J=8, R=8,
                    value_range=(1.0, 5.0)),
    # BASELINE.json configs[3]: high order, 10 K per mode, 200 M entries, J = R = 16
    "order6": dict(dims=(10_000,) * 6, nnz_train=198_000_000, nnz_test=2_000_000, J=16, R=16,
                   value_range=(1.0, 5.0)),
    "order10": dict(dims=(10_000,) * 10, nnz_train=198_000_000, nnz_test=2_000_000, J=16, R=16,
                    value_range=(1.0, 5.0)),
    # BASELINE.json configs[4] shape (order 4, 10 K per mode, J = R = 32) at the size one GPU
    # holds with the full forest; the 1 B-entry sweep runs sharded (dist.py) over 2-8 GPUs
    "order4": dict(dims=(10_000,) * 4, nnz_train=495_000_000, nnz_test=5_000_000, J=32, R=32,
                   value_range=(1.0, 5.0)),
    "order4_1b": dict(dims=(10_000,) * 4, nnz_train=990_000_000, nnz_test=10_000_000, J=32,
                      R=32, value_range=(1.0, 5.0), keep_fibers=False),
}

# one sample size for the reference arm and the cpu_baseline leg: BASELINE.md section 4 step 3
# (10 M entries of the benchmarked dims, the fiber density the full tensor's sweeps see)
CPU_SAMPLE_NNZ = 10_000_000


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------------------------------
# algorithmic bytes (variant B = the exact row-owner schedule that runs here)
# ------------------------------------------------------------------------------------------


def kernel_bytes(kind, tree, dims, J, R):
    """Logical bytes one launch of the row-owner kernel moves over tree u (fp32 values,
    int32 indices, no cache dedup): leaves (coord + value), fibers (ptr + N-1 coords),
    prefix C rows once per fiber, the leaf-level C row per leaf, and per row its A row
    (read + write for the factor sweep; A read + C_u read for the core sweep) and row index."""
    N = len(dims)
    nnz, F, rows = tree.nnz, tree.num_fibers, tree.num_rows
    b = nnz * 8 + F * (4 + 4 * (N - 1)) + F * (N - 2) * R * 4 + nnz * R * 4 + rows * 8
    if kind == "factor_rows":
        b += rows * 2 * J * 4
    else:
        b += rows * (J + R) * 4
    return b


def refresh_bytes(I, J, R):
    return I * (J + R) * 4


# ------------------------------------------------------------------------------------------
# clocks sampler
# ------------------------------------------------------------------------------------------


class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.path = os.path.join(REPO, "gpurun_out", f"clocks_{os.getpid()}.csv")
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        self.gpu = gpu_index
        self.proc = None

    def _lines(self):
        try:
            with open(self.path) as fh:
                return sum(1 for _ in fh)
        except OSError:
            return 0

    def start(self):
        """Start sampling and wait for nvidia-smi's first line (it takes ~0.1-1 s to come up),
        so the timed region that follows is covered."""
        self.mark = 0
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            t0 = time.time()
            while self._lines() == 0 and time.time() - t0 < 10 and self.proc.poll() is None:
                time.sleep(0.05)
        except Exception:
            self.proc = None

    def begin(self):
        """The timed region starts: only samples taken from here on count."""
        self.mark = self._lines()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        # a timed region shorter than the sampling interval still gets the sample taken right
        # after it (same load, clocks do not move that fast)
        t0 = time.time()
        while self._lines() <= self.mark and time.time() - t0 < 2 and self.proc.poll() is None:
            time.sleep(0.02)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for n_line, line in enumerate(open(self.path)):
            if n_line < self.mark:
                continue
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for k, name in enumerate(names):
                if f[5 + k].lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# CPU side (reference arm and cpu_baseline): the reference's own kernels (oracle/_ref, built
# from /root/reference's _ckern.pyx) driven by the restated trainer, on a bounded sample.
# ------------------------------------------------------------------------------------------


def host_sample(dims, nnz, value_range, seed=0):
    """nnz distinct uniform cells of `dims` with U[lo,hi] values (host numpy)."""
    rng = np.random.default_rng([seed, 99])
    cap = math.prod(dims)
    if cap < 2**62:
        lin = np.unique(rng.integers(0, cap, size=int(nnz * 1.02) + 1000))
        rng.shuffle(lin)
        lin = lin[:nnz]
        idx = np.stack(np.unravel_index(lin, dims), axis=1).astype(np.int64)
    else:  # > 62-bit index space: i.i.d. cells, drop the (improbable) repeats
        idx = np.stack([rng.integers(0, d, size=nnz) for d in dims], axis=1)
        _, first = np.unique(idx, axis=0, return_index=True)
        idx = idx[np.sort(first)]
    vals = rng.uniform(value_range[0], value_range[1], size=idx.shape[0])
    return idx, vals


def cpu_epoch_rate(cfg, nnz, repeats=1, threads=None):
    """Time factor pass + core pass of the reference CPU path on a sample, on all host cores:
    the reference's compiled kernels (oracle/_ref _ckern; our C restatement if absent) driven
    over row-partitioned sub-trees (oracle.RowParallelRef: bitwise the serial factor sweep, the
    reference's own per-worker core reduction).  Returns (kind, threads, [(factor_s, core_s)])."""
    from oracle import oracle as O

    O.build()
    K = O.ref_kernels()
    kind = "reference"
    if K is None:
        K, kind = O.CKernels, "port"
    idx, vals = host_sample(cfg["dims"], nnz, cfg["value_range"])
    N = len(cfg["dims"])
    ref = O.RowParallelRef(idx, vals, cfg["dims"], threads=threads, K=K)
    model = O.default_init_model(cfg["dims"], (cfg["J"],) * N, cfg["R"], seed=0)
    ocfg = O.OracleConfig()
    cache = O.precompute_cache(model, K=K)
    times = []
    try:
        for _ in range(repeats):
            t0 = time.perf_counter()
            for t in range(N):
                ref.update_factor_mode(model, cache, t, ocfg)
            t1 = time.perf_counter()
            for t in range(N):
                ref.update_core_mode(model, cache, t, ocfg)
            t2 = time.perf_counter()
            times.append((t1 - t0, t2 - t1))
    finally:
        ref.close()
    return kind, ref.T, times


def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nnz = int(os.environ.get("FT_REF_SAMPLE", CPU_SAMPLE_NNZ))
    kind, threads, times = cpu_epoch_rate(cfg, nnz, repeats=max(args.warmup - 1, 0) + args.steps)
    timed = times[-args.steps:]
    t = sum(a + b for a, b in timed)
    value = nnz * len(timed) / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / len(timed), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (host numpy, uniform distinct cells)",
        "config": {"workload": args.config, "sample_nnz": nnz, "J": cfg["J"], "R": cfg["R"],
                   "dims": list(cfg["dims"]), "threads": threads},
        "factor_nnz_per_s": nnz * len(timed) / sum(a for a, _ in timed),
        "core_nnz_per_s": nnz * len(timed) / sum(b for _, b in timed),
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": threads, "kind": kind,
                         "sample": f"{nnz} uniform entries of the {args.config} dims, one factor "
                                   f"+ core pass per step, the reference's compiled kernels over "
                                   f"{threads} row-partitioned groups on {threads} host threads "
                                   f"(bitwise its serial factor sweep; its own `workers` hogwild "
                                   f"mode holds the GIL and measured slower than serial)"},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------


def measured_peak():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------------------------------
# the memory hierarchy as the sweeps see it: measured on-chip peaks + live per-launch traffic
# ------------------------------------------------------------------------------------------


def onchip_peaks():
    """L2 -> SM, L1-hit and shared-memory read bandwidth of this GPU (tools/peaks.cu, best of
    5 CUDA-event timed launches each).  The HBM peak is MEASURED_PEAKS.json's."""
    import ctypes

    path = os.path.join(REPO, "tools", "libft_peaks.so")
    if not os.path.exists(path):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                        "-Xcompiler", "-fPIC", "-o", path, os.path.join(REPO, "tools", "peaks.cu")],
                       capture_output=True)
    out = {}
    try:
        L = ctypes.CDLL(path)
        for name in ("l2", "l1", "smem"):
            v = ctypes.c_double(0.0)
            if getattr(L, f"ftp_{name}_read_gbs")(5, ctypes.byref(v)) == 0:
                out[name] = v.value
    except OSError as exc:
        out["error"] = str(exc)
    return out


# per launch, summed over the sweep launches of one epoch; one ncu pass group, kernel replay
NCU_METRICS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "lts__t_bytes.sum", "l1tex__t_bytes.sum",
               "l1tex__data_pipe_lsu_wavefronts.sum",
               "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
               "dram__throughput.avg.pct_of_peak_sustained_elapsed",
               "lts__throughput.avg.pct_of_peak_sustained_elapsed",
               "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
               "sm__inst_executed.avg.per_cycle_elapsed",
               "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed")


def live_traffic(args, N, timeout=420):
    """Run ncu on THIS config: a child bench process (same workload, `--ncu-child`) does one
    untimed epoch then one profiled epoch; ncu records the 2N sweep launches of the second.
    Returns [{kernel, metrics...}] in launch order (factor t = 0..N-1, core t = 0..N-1), or
    {"error": ...}.  Per-launch byte counts do not depend on timing, so they are combined with
    this run's own CUDA-event launch times."""
    import csv
    import io
    import shutil

    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return {"error": "ncu not found"}
    logf = os.path.join(REPO, "gpurun_out", f"ncu_traffic_{os.getpid()}.csv")
    os.makedirs(os.path.dirname(logf), exist_ok=True)
    cmd = [ncu, "--metrics", ",".join(NCU_METRICS), "--clock-control", "none",
           "-k", "regex:factor_rows|core_rows", "--launch-skip", str(2 * N),
           "--launch-count", str(2 * N), "--csv", "--page", "raw", "--print-units", "base",
           "--log-file", logf, sys.executable, os.path.join(REPO, "bench.py"), "--config",
           args.config, "--schedule", args.schedule, "--ncu-child"]
    t0 = time.perf_counter()
    # own process group: on a timeout the whole group (ncu AND its bench child, which holds the
    # workload's device memory) is killed, never left running under the next command
    proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                            start_new_session=True)
    try:
        _, err = proc.communicate(timeout=timeout)
        proc.stderr_tail = err
    except subprocess.TimeoutExpired:
        import signal

        os.killpg(proc.pid, signal.SIGKILL)
        proc.communicate()
        return {"error": f"ncu timed out after {timeout} s"}
    try:
        rows = list(csv.reader(io.StringIO(open(logf).read())))
    except OSError:
        return {"error": f"ncu produced no log (rc {proc.returncode}): {proc.stderr_tail[-300:]}"}
    hi = next((i for i, r in enumerate(rows) if "Kernel Name" in r), None)
    if hi is None:
        return {"error": f"ncu log without a header (rc {proc.returncode})"}
    h = rows[hi]
    out = []
    for r in rows[hi + 1:]:
        if len(r) != len(h) or not r[h.index("ID")].strip().isdigit():
            continue
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].split("<")[0].split("::")[-1]}
        for m in NCU_METRICS:
            try:
                d[m] = float(r[h.index(m)].replace(",", ""))
            except (ValueError, IndexError):
                d[m] = None
        out.append(d)
    if len(out) != 2 * N:
        return {"error": f"ncu recorded {len(out)} sweep launches, expected {2 * N}"}
    return {"launches": out, "seconds": time.perf_counter() - t0}


def ncu_child(args, cfg):
    """The process live_traffic profiles: the bench workload, one untimed + one profiled epoch."""
    import torch

    import paper_2210_06014_b200 as ft

    dims, J, R = cfg["dims"], cfg["J"], cfg["R"]
    N = len(dims)
    nnz_total = cfg["nnz_train"] + cfg["nnz_test"]
    split = ft.generate_synthetic(dims, nnz_total, cfg["value_range"], seed=0,
                                  test_fraction=cfg["nnz_test"] / nnz_total)
    forest = ft.build_forest(split.train, 128, compact=True)
    model = ft.default_init_model(dims, (J,) * N, R, seed=0)
    cache = ft.precompute_cache(model)
    tcfg = ft.TrainConfig(epochs=1, schedule=args.schedule)
    for _ in range(2):
        for n in range(N):
            ft.update_factor_mode(model, forest, cache, n, tcfg)
        for n in range(N):
            ft.update_core_mode(model, forest, cache, n, tcfg)
    torch.cuda.synchronize()


def hierarchy_roofline(name, launches, secs, peaks):
    """Per memory level, measured bytes of the given ncu launches over their live CUDA-event
    time: DRAM (read + write) vs the HBM peak, L2 (lts__t_bytes) vs the L2 peak, the L1 / shared
    data pipe (LSU wavefronts x 128 B, the pipe's width per cycle) vs the shared-memory peak.
    bound = the level with the largest fraction."""
    n = len(launches)

    def tot(m):
        return sum(x[m] or 0.0 for x in launches)

    lv = {
        "hbm": (tot("dram__bytes_read.sum") + tot("dram__bytes_write.sum"), peaks.get("hbm")),
        "l2": (tot("lts__t_bytes.sum"), peaks.get("l2")),
        "l1": (tot("l1tex__data_pipe_lsu_wavefronts.sum") * 128.0, peaks.get("smem")),
    }
    levels = {}
    for k, (b, pk) in lv.items():
        ach = b / secs / 1e9
        levels[k] = {"bytes_per_launch": b / n, "achieved": ach, "peak": pk,
                     "frac": ach / pk if pk else None}
    bound = max((k for k in levels if levels[k]["frac"] is not None),
                key=lambda k: levels[k]["frac"])
    ncu_pct = {k: sum(x[m] or 0.0 for x in launches) / n for k, m in (
        ("dram", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("l2", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("l1", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("tensor_hmma", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed"))}
    ipc = sum(x["sm__inst_executed.avg.per_cycle_elapsed"] or 0.0 for x in launches) / n
    return {"kernel": name, "bound": bound, "achieved": levels[bound]["achieved"],
            "peak": levels[bound]["peak"], "unit": "GB/s", "frac": levels[bound]["frac"],
            "traffic": levels["hbm"]["bytes_per_launch"], "levels": levels,
            "ncu_pct_of_peak": ncu_pct, "ncu_issue_ipc": ipc,
            "ncu_ms_per_launch": 1e3 * sum(x["gpu__time_duration.sum"] or 0 for x in launches)
                                 / 1e9 / n}


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import importlib

    import paper_2210_06014_b200 as ft

    T = importlib.import_module("paper_2210_06014_b200.train")

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    if world > 1:
        from paper_2210_06014_b200 import dist as D

        # NCCL over NVLink on a real multi-GPU box; FT_DIST_BACKEND=gloo lets several ranks
        # share one GPU to exercise this path (its timing is then meaningless)
        dist.init_process_group(os.environ.get("FT_DIST_BACKEND", "nccl"))
        return D.bench_distributed(args, cfg, rank, world)

    dims, J, R = cfg["dims"], cfg["J"], cfg["R"]
    N = len(dims)
    nnz_total = cfg["nnz_train"] + cfg["nnz_test"]
    t0 = time.perf_counter()
    split = ft.generate_synthetic(dims, nnz_total, cfg["value_range"], seed=0,
                                  test_fraction=cfg["nnz_test"] / nnz_total)
    train_t, test_t = split.train, split.test
    nnz = train_t.nnz
    torch.cuda.synchronize()
    log(f"generated {nnz_total} entries in {time.perf_counter() - t0:.2f}s")
    t0 = time.perf_counter()
    # the arrays the sweeps read (keep_fibers=False: without the fiber arrays, 16 B per leaf at
    # order 4 -- what fits the 1 B-entry order-4 forest on one GPU)
    forest = ft.build_forest(train_t, 128, compact=True, keep_fibers=cfg.get("keep_fibers", True))
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    log(f"forest built in {build_s:.2f}s; fibers {[t.num_fibers for t in forest.trees]}, "
        f"rows {[t.num_rows for t in forest.trees]}")
    model = ft.default_init_model(dims, (J,) * N, R, seed=0)
    counter = ft.OpCounter()
    cache = ft.precompute_cache(model, counter)
    tcfg = ft.TrainConfig(epochs=1, schedule=args.schedule)
    guards = T.GuardBank(N)

    def epoch(ev=None):
        guards.reset()
        if ev:
            ev[0].record()
        for n in range(N):
            T.update_factor_mode(model, forest, cache, n, tcfg, counter, guards=guards, slot=n)
        if ev:
            ev[1].record()
        for n in range(N):
            T.update_core_mode(model, forest, cache, n, tcfg, counter, guards=guards, slot=N + n)
        if ev:
            ev[2].record()

    clocks = Clocks(local)
    clocks.start()  # before the warm-up: the sampler is up and the clocks ramped when timing starts
    for _ in range(args.warmup):
        epoch()
    torch.cuda.synchronize()
    guards.check(tcfg.divergence_limit)
    rmse0 = ft.evaluate(model, train_t, cache)[0]

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    T.KERNEL_TIMER = T.KernelTimer()
    torch.cuda.synchronize()
    clocks.begin()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for k in range(args.steps):
        epoch(evs[k])
    stop.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    krec = T.KERNEL_TIMER.elapsed()
    T.KERNEL_TIMER = None
    guards.check(tcfg.divergence_limit)
    total_s = start.elapsed_time(stop) / 1e3
    f_s = sum(e[0].elapsed_time(e[1]) for e in evs) / 1e3
    c_s = sum(e[1].elapsed_time(e[2]) for e in evs) / 1e3
    tr_rmse = ft.evaluate(model, train_t, cache)[0]
    te_rmse = ft.evaluate(model, test_t, cache)[0]

    # CPU baseline (rank 0, N = 1): the reference's compiled kernels on a bounded sample
    cpu = None
    if not args.no_cpu:
        nnz_s = int(os.environ.get("FT_REF_SAMPLE", CPU_SAMPLE_NNZ))
        kind, threads, times = cpu_epoch_rate(cfg, nnz_s)
        tf, tc = times[0]
        cpu = {"value": nnz_s / (tf + tc), "unit": "nnz/s", "cores": threads, "kind": kind,
               "sample": f"{nnz_s} uniform entries of the {args.config} dims (the reference arm's "
                         f"sample), one factor + core pass, the reference's compiled kernels over "
                         f"row-partitioned groups on {threads} host threads",
               "factor_nnz_per_s": nnz_s / tf, "core_nnz_per_s": nnz_s / tc}

    e2e = run_e2e(ft, T, cfg, train_t, args) if not args.no_e2e else None
    from types import SimpleNamespace

    trees = [SimpleNamespace(nnz=t.nnz, num_fibers=t.num_fibers, num_rows=t.num_rows,
                             leaf_mode=t.leaf_mode, root_mode=t.root_mode) for t in forest.trees]
    l2_note = ("inputs larger than L2 (forest arrays "
               f"{sum(t.nnz * 8 + t.num_fibers * 12 for t in forest.trees) / 1e9:.1f} GB "
               "streamed per epoch vs 126 MB L2)")
    test_nnz = test_t.nnz

    # roofline of the dominant kernel (largest share of the timed region)
    peak, peak_src = measured_peak()
    by = {}
    per_launch = {}  # (name, mode) -> mean live seconds per launch
    for name, mode, sec in krec:
        tree = trees[mode]
        b = kernel_bytes(name, tree, dims, J, R)
        agg = by.setdefault(name, {"bytes": 0, "sec": 0.0, "launches": 0})
        agg["bytes"] += b
        agg["sec"] += sec
        agg["launches"] += 1
        per_launch[(name, mode)] = per_launch.get((name, mode), 0.0) + sec / args.steps
    dom = max(by, key=lambda k: by[k]["sec"])
    d = by[dom]
    logical = {"bytes_per_launch": d["bytes"] / d["launches"],
               "achieved": d["bytes"] / d["sec"] / 1e9, "peak": peak,
               "frac_of_hbm": d["bytes"] / d["sec"] / 1e9 / peak,
               "what": "SURVEY 8d variant-B algorithmic bytes (every gathered C row counted, no "
                       "cache dedup) over the live launch time: a schedule-efficiency figure -- "
                       "the C rows are L2 / L1 hits, so it is not a DRAM utilisation"}
    # the ncu child rebuilds this workload in its own process: free ours first
    del model, cache, train_t, test_t, split, forest
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    peaks = dict(onchip_peaks()) if not args.no_ncu else {}
    peaks["hbm"] = peak
    traffic = live_traffic(args, N) if not args.no_ncu else {"error": "--no-ncu"}
    order = [("factor_rows", trees[t].leaf_mode) for t in range(N)] + \
            [("core_rows", trees[t].leaf_mode) for t in range(N)]
    kernels = {k: {"ms_total": 1e3 * v["sec"] / args.steps,
                   "logical_GB_per_s": v["bytes"] / v["sec"] / 1e9} for k, v in by.items()}
    per_mode = {}
    for (name, mode), sec in per_launch.items():
        per_mode[f"{name}:{mode}"] = {"ms": 1e3 * sec, "logical_bytes": kernel_bytes(
            name, trees[mode], dims, J, R)}
    if "launches" in traffic:
        launches = traffic["launches"]
        for k, (name, mode) in enumerate(order):
            per_mode[f"{name}:{mode}"]["hierarchy"] = hierarchy_roofline(
                launches[k]["kernel"], [launches[k]], per_launch[(name, mode)], peaks)
        for name in ("factor_rows", "core_rows"):
            sel = [k for k, o in enumerate(order) if o[0] == name]
            kernels[name]["hierarchy"] = hierarchy_roofline(
                "+".join(sorted({launches[k]["kernel"] for k in sel})), [launches[k] for k in sel],
                sum(per_launch[order[k]] for k in sel), peaks)
        roof = dict(kernels[dom]["hierarchy"])
        roof["traffic_source"] = (f"live: ncu on this config ({traffic['seconds']:.0f} s, "
                                  f"launches of one epoch, kernel replay)")
    else:
        roof = {"kernel": dom, "bound": "hbm", "achieved": logical["achieved"], "peak": peak,
                "unit": "GB/s", "frac": logical["frac_of_hbm"], "traffic": None,
                "traffic_source": traffic.get("error")}
    roof.update({"peak_source": {"hbm": peak_src, "l2/l1/smem": "tools/peaks.cu, measured here"},
                 "peaks_GB_per_s": peaks, "logical": logical,
                 "ms_per_launch": 1e3 * d["sec"] / d["launches"],
                 "share_of_step": d["sec"] / total_s})
    kernels["by_mode"] = per_mode
    pass_bytes = {"factor": 0, "core": 0}
    for tree_u in trees:
        u = tree_u.root_mode
        rb = refresh_bytes(dims[u], J, R)
        pass_bytes["factor"] += kernel_bytes("factor_rows", tree_u, dims, J, R) + rb
        pass_bytes["core"] += kernel_bytes("core_rows", tree_u, dims, J, R) + rb
    launches_per_epoch = 5 * N  # per mode: factor sweep, refresh, core sweep, apply, refresh

    line = {
        "metric": METRIC, "value": nnz * args.steps / total_s, "unit": "nnz/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (GPU generator: distinct uniform cells, U[1,5] values; random init)",
        "config": {"workload": args.config, "dims": list(dims), "nnz_train": nnz,
                   "nnz_test": test_nnz, "J": J, "R": R, "schedule": tcfg.resolved_schedule,
                   "fiber_threshold": 128, "parallelism": "1 GPU",
                   "l2": l2_note},
        "factor_nnz_per_s": nnz * args.steps / f_s, "core_nnz_per_s": nnz * args.steps / c_s,
        "factor_ms": 1e3 * f_s / args.steps, "core_ms": 1e3 * c_s / args.steps,
        # SURVEY 8d's logical (algorithmic-byte) fractions of the HBM peak, per pass and for the
        # epoch -- schedule-efficiency figures (see roofline.logical), not DRAM utilisation
        "logical_pass_frac_of_hbm": {k: pass_bytes[k] / ((f_s if k == "factor" else c_s)
                                                         / args.steps) / 1e9 / peak
                                     for k in pass_bytes},
        "logical_epoch_frac_of_hbm": (pass_bytes["factor"] + pass_bytes["core"])
                                     / (total_s / args.steps) / 1e9 / peak,
        "train_rmse_before": rmse0, "train_rmse": tr_rmse, "test_rmse": te_rmse,
        "build_forest_s": build_s,
        "roofline": roof, "kernels": kernels,
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
        "gpu_launches": launches_per_epoch * args.steps,
    }
    print(json.dumps(line), flush=True)


def run_e2e(ft, T, cfg, train_dev, args):
    """Same metric through the public API from HOST buffers.  Every step takes its training COO
    from pinned host memory (H2D), builds the B-CSF forest on the GPU, fills the cache, runs one
    epoch and reads the training RMSE back (a `train(epochs=1)` call minus its epoch-0 row).
    The input pipeline is double-buffered: step k+1's H2D runs on a copy stream under step k's
    compute, as a streaming trainer would; step 0's copy is inside the timed region."""
    import torch

    idx_h = train_dev.idx.cpu().pin_memory()
    vals_h = train_dev.vals.cpu().pin_memory()
    dims, J, R = cfg["dims"], cfg["J"], cfg["R"]
    N = len(dims)
    nnz = int(vals_h.shape[0])
    steps = max(2, min(args.steps, 10))  # the same K as the device-timed loop (bounded)
    bufs = [(torch.empty_like(idx_h, device="cuda"), torch.empty_like(vals_h, device="cuda"))
            for _ in range(2)]
    copy_stream = torch.cuda.Stream()
    main_stream = torch.cuda.current_stream()
    tcfg = ft.TrainConfig(epochs=1, schedule=args.schedule)

    def h2d(slot, after=None):
        with torch.cuda.stream(copy_stream):
            if after is not None:
                copy_stream.wait_event(after)
            bufs[slot][0].copy_(idx_h, non_blocking=True)
            bufs[slot][1].copy_(vals_h, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
        return ev

    def step(slot, ready):
        main_stream.wait_event(ready)
        dev = ft.DeviceCoo(tuple(dims), bufs[slot][0], bufs[slot][1])
        model = ft.Model(dims, (J,) * N, R, init_f, init_c)
        # the exact schedule reads the leaf-major index only: no fiber coordinates (hogwild
        # walks the fibers)
        forest = ft.build_forest(dev, 128, compact=True, keep_fibers=args.schedule != "exact")
        counter = ft.OpCounter()
        cache = ft.precompute_cache(model, counter)
        m = T.run_epoch(model, forest, cache, dev, tcfg, counter, 1, None, evaluate_metrics=True)
        _ = m.train_rmse  # the step's result, read back to the host
        done = torch.cuda.Event()
        done.record(main_stream)
        return done

    base = ft.default_init_model(dims, (J,) * N, R, seed=0)
    init_f, init_c = [a.clone() for a in base.factors], [b.clone() for b in base.cores_t]
    step(0, h2d(0))  # warm-up (allocator pools, lazy module loading)
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(main_stream)
    ready = h2d(0)
    free = [None, None]
    for k in range(steps):
        slot = k % 2
        nxt = None
        if k + 1 < steps:
            nxt = h2d((k + 1) % 2, after=free[(k + 1) % 2])
        free[slot] = step(slot, ready)
        ready = nxt
    stop.record(main_stream)
    torch.cuda.synchronize()
    t = start.elapsed_time(stop) / 1e3 / steps
    return {"value": nnz / t, "unit": "nnz/s", "h2d_bytes_per_step": nnz * (4 * N + 4),
            "d2h_bytes_per_step": 16, "ms_per_step": 1e3 * t, "steps": steps,
            "includes": "H2D COO (pinned, double-buffered on a copy stream) + GPU B-CSF build + "
                        "cache + 1 epoch + train RMSE readback"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="netflix32", choices=sorted(CONFIGS))
    ap.add_argument("--schedule", default="exact", choices=["exact", "hogwild"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ncu", action="store_true", help="skip the live ncu traffic capture")
    ap.add_argument("--ncu-child", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.ncu_child:
        return ncu_child(args, cfg)
    if args.impl == "reference":
        run_reference_arm(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
