"""SGD training sweeps over the B-CSF forest on the GPU -- the drop-in for the reference
trainer (/root/reference/pkg/src/fastertucker/train.py:40-336).

Same public surface and semantics: ``TrainConfig``, ``EpochMetrics``, ``evaluate``,
``update_factor_mode`` (sweep the tree rooted at n, update its leaf mode u = (n+N-1) mod N,
then refresh C_u), ``update_core_mode`` (accumulate the full-sweep core gradient of mode u,
one step normalised by |Omega|, refresh C_u), ``run_epoch`` (N factor sweeps then N core
sweeps, timed without evaluation) and ``train`` (row 0 evaluates the initial model, optional
early stop).  ``DivergenceError`` names the mode and the epoch.

Schedules (``TrainConfig.schedule``):
  "exact"   (default; the reference's workers <= 1): kernel K3b, one warp owns one row of A_u
            and replays its updates in the serial order -- deterministic, equal to the
            reference up to fp32 rounding.
  "hogwild" (the reference's workers > 1): kernel K3a, the reference's own fiber traversal
            with racing lock-free row updates.
The core sweep is always K4 (deterministic row form) + K5.

Divergence guards (train.py:101-110) are fused into the refresh (|A_u|) and the core apply
(|Bt_u|): each writes a max-abs word per sweep on the device.  ``run_epoch`` reads the words
once per epoch (``TrainConfig.sync_guards`` checks after every sweep instead) and raises for
the first sweep over the limit, naming that sweep's mode.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .cache import DotCache, fresh_dots, precompute_cache, refresh_count, refresh_into
from .coo import as_device
from .counter import (CH_DOT, CHANNELS, OpCounter, apply_counts, new_raw_counts,
                      sweep_counts)
from .csf import CsfForest, build_forest
from .errors import ConfigError, DivergenceError, ValidationError


@dataclass(frozen=True)
class TrainConfig:
    """Learning rates, regularizers, plan and execution mode (train.py:40-67) plus the
    B200 schedule switches."""

    lr_a: float = 1e-3
    lr_b: float = 1e-3
    reg_a: float = 1e-2
    reg_b: float = 1e-2
    epochs: int = 10
    plan: str = "cached"
    workers: int = 0
    seed: int = 0
    fiber_threshold: int | None = 128
    divergence_limit: float = 1e12
    rmse_delta_stop: float | None = None
    schedule: str | None = None   # None: "exact" if workers <= 1 else "hogwild"
    sync_guards: bool = False
    # hogwild concurrency: at most dims[u] / hogwild_rows_per_warp warps update A_u at once
    # (each warp is one serial worker; fewer rows per warp = more racing writers per row).
    # Measured (profiles/r02_hogwild_ab.md): on Netflix dims at lr 1e-3 every level from 256 to
    # 1 row per warp stays within 0.005 % of the exact schedule's RMSE, but the reference's own
    # hogwild fixture (20 rows per mode, lr 0.05) diverges with 20 racing warps; 16 rows per
    # warp keeps tiny modes serial and is 15x faster than the round-1 cap of 256 at Netflix dims
    hogwild_rows_per_warp: int = 16

    def __post_init__(self):
        if self.plan not in ("cached", "uncached"):
            raise ConfigError(f"plan must be 'cached' or 'uncached', got {self.plan!r}")
        if self.lr_a < 0 or self.lr_b < 0 or self.reg_a < 0 or self.reg_b < 0:
            raise ConfigError("learning rates and regularizers must be non-negative")
        if self.epochs < 0:
            raise ConfigError("epochs must be >= 0")
        if self.schedule not in (None, "exact", "hogwild"):
            raise ConfigError(f"schedule must be 'exact' or 'hogwild', got {self.schedule!r}")
        if self.hogwild_rows_per_warp < 1:
            raise ConfigError("hogwild_rows_per_warp must be >= 1")

    @property
    def resolved_schedule(self) -> str:
        if self.schedule is not None:
            return self.schedule
        return "hogwild" if self.workers > 1 else "exact"


@dataclass
class EpochMetrics:
    epoch: int
    train_rmse: float
    train_mae: float
    test_rmse: float
    test_mae: float
    seconds: float
    multiplies: int
    counts: dict = field(default_factory=dict)
    factor_seconds: float = 0.0
    core_seconds: float = 0.0

    def csv_row(self) -> str:
        return (f"{self.epoch},{self.train_rmse!r},{self.test_rmse!r},"
                f"{self.train_mae!r},{self.test_mae!r},{self.seconds:.6f},{self.multiplies}")


METRICS_CSV_HEADER = "epoch,train_rmse,test_rmse,train_mae,test_mae,seconds,multiplies"


# ----------------------------------------------------------------------------------------
# divergence guards
# ----------------------------------------------------------------------------------------


class GuardBank:
    """One device uint32 max-abs word per sweep of an epoch (2N words)."""

    def __init__(self, order: int):
        import torch

        self.order = order
        self.words = torch.zeros(2 * order, dtype=torch.int32, device="cuda")
        self.modes = [None] * (2 * order)

    def reset(self):
        self.words.zero_()
        self.modes = [None] * (2 * self.order)

    def slot(self, k: int, mode: int):
        self.modes[k] = mode
        return self.words[k:k + 1]

    def check(self, limit: float, upto: int | None = None) -> None:
        lim_bits = int(np.array([min(limit, 3.4028234663852886e38)], np.float32).view(np.uint32)[0])
        words = self.words.cpu().numpy().view(np.uint32)
        n = len(words) if upto is None else upto
        for k in range(n):
            if self.modes[k] is None:
                continue
            if int(words[k]) > lim_bits:
                kind = "factor" if k < self.order else "core"
                raise DivergenceError(f"{kind} mode {self.modes[k]} diverged", mode=self.modes[k])


# ----------------------------------------------------------------------------------------
# evaluation
# ----------------------------------------------------------------------------------------


def _sse(model, dev, dots):
    import torch

    L = _lib.lib()
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    _lib.check(L.ft_sse(ctypes.byref(model.view(dots)), dev.nnz, dev.idx.data_ptr(),
                        dev.vals.data_ptr(), out.data_ptr(), _lib.stream_handle()), "ft_sse")
    return out


def _sse_tree(model, tree, dots):
    """K6b: the same sums over the entries a B-CSF tree holds, walked in tree order (two C-row
    gathers per entry; None when the tree / shape is outside that kernel's cover)."""
    import torch

    if (not 3 <= model.order <= 6 or model.core_rank % 4 or tree.leaf_pc is None
            or tree.seg_coord is None):
        return None
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().ft_sse_tree(ctypes.byref(tree.view()), ctypes.byref(model.view(dots)),
                                      out.data_ptr(), _lib.stream_handle()), "ft_sse_tree")
    return out


def evaluate(model, tensor, cache: DotCache | None = None, forest: CsfForest | None = None) -> tuple:
    """RMSE and MAE over a tensor's entries (train.py:91-98), reduced in fp64 on the GPU.
    Uses ``cache`` when it is coherent (all modes clean), else fresh C_n.  ``forest``: a forest
    built from exactly this tensor (as ``train`` has for the training set) -- its first tree is
    scored in tree order (K6b) instead of the COO order."""
    if tensor is None:
        raise ValidationError("cannot evaluate on an empty entry set")
    dev = as_device(tensor)
    if dev.nnz == 0:
        raise ValidationError("cannot evaluate on an empty entry set")
    dots = cache.arrays if cache is not None and not cache.dirty.any() else fresh_dots(model)
    out = None
    if forest is not None and forest.omega is None and forest.trees[0].nnz == dev.nnz:
        out = _sse_tree(model, forest.trees[0], dots)
    if out is None:
        out = _sse(model, dev, dots)
    sse, sae = out.cpu().numpy()
    return math.sqrt(float(sse) / dev.nnz), float(sae) / dev.nnz


# ----------------------------------------------------------------------------------------
# sweeps
# ----------------------------------------------------------------------------------------


class KernelTimer:
    """Optional CUDA-event timing of the sweep kernels (installed by bench.py): events are
    recorded on the launching (current) stream around each sweep launch."""

    def __init__(self):
        self.records = []  # (name, mode, start_event, end_event)

    def elapsed(self):
        out = []
        for name, mode, a, b in self.records:
            b.synchronize()
            out.append((name, mode, a.elapsed_time(b) / 1e3))
        return out


KERNEL_TIMER: KernelTimer | None = None


class _ktime:
    __slots__ = ("name", "mode", "a")

    def __init__(self, name, mode):
        self.name, self.mode = name, mode

    def __enter__(self):
        if KERNEL_TIMER is not None:
            import torch

            self.a = torch.cuda.Event(enable_timing=True)
            self.a.record()

    def __exit__(self, *exc):
        if KERNEL_TIMER is not None and exc[0] is None:
            import torch

            b = torch.cuda.Event(enable_timing=True)
            b.record()
            KERNEL_TIMER.records.append((self.name, self.mode, self.a, b))
        return False


def _dots_for(model, cache, cfg):
    if cfg.plan == "cached":
        if cache is None:
            raise ConfigError("the cached plan needs a DotCache (precompute_cache)")
        return cache.arrays
    return fresh_dots(model)


def update_factor_mode(model, forest: CsfForest, cache: DotCache | None, n: int,
                       cfg: TrainConfig, counter: OpCounter | None = None, *,
                       guards: GuardBank | None = None, slot: int | None = None) -> np.ndarray:
    """Sweep the tree rooted at mode n, updating its leaf mode's factor rows
    (train.py:152-197); refresh the leaf mode's C (cached plan).  Returns the raw tallies."""
    L = _lib.lib()
    tree = forest.trees[n]
    u = tree.leaf_mode
    N = model.order
    dots = _dots_for(model, cache, cfg)
    mv = model.view(dots)
    stream = _lib.stream_handle()
    if cfg.resolved_schedule == "exact":
        forest.trees[u].ensure_slots(model.ranks[u], model.core_rank)  # once per tree (K1d)
        with _ktime("factor_rows", u):
            _lib.check(L.ft_factor_sweep_rows(ctypes.byref(forest.trees[u].view()),
                                              ctypes.byref(mv), cfg.lr_a, cfg.reg_a, stream),
                       "ft_factor_sweep_rows")
    else:
        with _ktime("factor_fibers", u):
            # staleness bound: one serial worker (warp) per hogwild_rows_per_warp rows of A_u
            cap = max(1, model.dims[u] // cfg.hogwild_rows_per_warp)
            _lib.check(L.ft_factor_sweep_fibers(ctypes.byref(tree.view()), ctypes.byref(mv), 0,
                                                tree.num_fibers, cfg.lr_a, cfg.reg_a, cap, stream),
                       "ft_factor_sweep_fibers")
    total = sweep_counts("factor", cfg.plan, N, model.core_rank, model.ranks, tree.prefix_modes,
                         u, tree.nnz, tree.num_fibers)
    own = guards is None
    if own:
        guards = GuardBank(1)
        slot = 0
    word = guards.slot(slot, u)
    if cache is not None:
        cache.mark_dirty(u)
    if cfg.plan == "cached":
        refresh_into(model, u, cache.arrays[u], guard=word)
        cache.dirty[u] = False
        total[CH_DOT] += refresh_count(model, u)
    else:
        import torch

        scratch = torch.empty((model.dims[u], model.core_rank), dtype=torch.float32, device="cuda")
        refresh_into(model, u, scratch, guard=word)
    if own or cfg.sync_guards:
        guards.check(cfg.divergence_limit, upto=slot + 1)
    if counter is not None:
        counter.merge(total)
    return total


def update_core_mode(model, forest: CsfForest, cache: DotCache | None, n: int,
                     cfg: TrainConfig, counter: OpCounter | None = None, *,
                     guards: GuardBank | None = None, slot: int | None = None,
                     acc_out=None, reduce_fn=None) -> np.ndarray:
    """Accumulate the leaf mode's full-sweep core gradient, apply one step normalised by
    |Omega| (train.py:200-248), refresh C_u.  ``acc_out`` (device R x J_u) receives the
    reference's ``acc``; ``reduce_fn(acc)`` (multi-GPU) allreduces it before the step."""
    import torch

    L = _lib.lib()
    tree = forest.trees[n]
    u = tree.leaf_mode
    N, R, Ju = model.order, model.core_rank, model.ranks[u]
    dots = _dots_for(model, cache, cfg)
    mv = model.view(dots)
    stream = _lib.stream_handle()
    cap = int(L.ft_core_partials_size(R, Ju))
    partials = _scratch(model, "partials", cap)
    nblocks = ctypes.c_int32(0)
    rows_tree = forest.trees[u]
    with _ktime("core_rows", u):
        _lib.check(L.ft_core_sweep_rows(ctypes.byref(rows_tree.view()), ctypes.byref(mv),
                                        partials.data_ptr(), cap, ctypes.byref(nblocks), stream),
                   "ft_core_sweep_rows")
    own = guards is None
    if own:
        guards = GuardBank(1)
        slot = 0
    word = guards.slot(slot, u)
    omega = float(tree.nnz if forest.omega is None else forest.omega)
    if reduce_fn is None:
        _lib.check(L.ft_core_apply(R, Ju, model.cores_t[u].data_ptr(), partials.data_ptr(),
                                   nblocks.value, 1, omega, cfg.lr_b, cfg.reg_b,
                                   None if acc_out is None else acc_out.data_ptr(),
                                   word.data_ptr(), stream), "ft_core_apply")
    else:
        acc = torch.empty((R, Ju), dtype=torch.float32, device="cuda")
        _lib.check(L.ft_core_reduce(R, Ju, partials.data_ptr(), nblocks.value, acc.data_ptr(),
                                    stream), "ft_core_reduce")
        reduce_fn(acc)
        _lib.check(L.ft_core_apply(R, Ju, model.cores_t[u].data_ptr(), acc.data_ptr(), 1, 1,
                                   omega, cfg.lr_b, cfg.reg_b,
                                   None if acc_out is None else acc_out.data_ptr(),
                                   word.data_ptr(), stream), "ft_core_apply")
    total = sweep_counts("core", cfg.plan, N, R, model.ranks, tree.prefix_modes, u, tree.nnz,
                         tree.num_fibers)
    total += apply_counts(R, Ju)
    if cache is not None:
        cache.mark_dirty(u)
        if cfg.plan == "cached":
            refresh_into(model, u, cache.arrays[u])
            cache.dirty[u] = False
            total[CH_DOT] += refresh_count(model, u)
    if own or cfg.sync_guards:
        guards.check(cfg.divergence_limit, upto=slot + 1)
    if counter is not None:
        counter.merge(total)
    return total


_SCRATCH = {}


def _scratch(model, name, numel):
    import torch

    key = (name, torch.cuda.current_device())
    buf = _SCRATCH.get(key)
    if buf is None or buf.numel() < numel:
        buf = torch.empty(numel, dtype=torch.float32, device="cuda")
        _SCRATCH[key] = buf
    return buf


def _log_sweep(sweep_log, plan, kind, mode, raw):
    for i, name in enumerate(CHANNELS):
        sweep_log.append((plan, f"{kind}:{mode}", name, int(raw[i])))


class _Timer:
    """CUDA-event timing on the current stream."""

    def __init__(self):
        import torch

        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]

    def mark(self, k):
        self.ev[k].record()

    def seconds(self):
        self.ev[2].synchronize()
        f = self.ev[0].elapsed_time(self.ev[1]) / 1e3
        c = self.ev[1].elapsed_time(self.ev[2]) / 1e3
        return f, c


def run_epoch(model, forest: CsfForest, cache: DotCache | None, train_tensor, cfg: TrainConfig,
              counter: OpCounter, epoch_no: int, test_tensor=None, sweep_log=None,
              evaluate_metrics: bool = True, _guards: GuardBank | None = None) -> EpochMetrics:
    """One factor pass then one core pass (train.py:251-278), CUDA-event timed without the
    evaluation, then evaluation."""
    N = model.order
    guards = _guards if _guards is not None else GuardBank(N)
    guards.reset()
    timer = _Timer()
    t0 = time.perf_counter()
    try:
        timer.mark(0)
        for n in range(N):
            raw = update_factor_mode(model, forest, cache, n, cfg, counter, guards=guards, slot=n)
            if sweep_log is not None:
                _log_sweep(sweep_log, cfg.plan, "factor", forest.trees[n].leaf_mode, raw)
        timer.mark(1)
        for n in range(N):
            raw = update_core_mode(model, forest, cache, n, cfg, counter, guards=guards,
                                   slot=N + n)
            if sweep_log is not None:
                _log_sweep(sweep_log, cfg.plan, "core", forest.trees[n].leaf_mode, raw)
        timer.mark(2)
        fsec, csec = timer.seconds()
        guards.check(cfg.divergence_limit)
    except DivergenceError as exc:
        raise DivergenceError(f"divergence at epoch {epoch_no}, mode {exc.mode}", mode=exc.mode,
                              epoch=epoch_no) from None
    wall = time.perf_counter() - t0
    m = _metrics(model, cache, train_tensor, test_tensor, counter, epoch_no, fsec + csec,
                 evaluate_metrics, forest)
    m.factor_seconds, m.core_seconds = fsec, csec
    del wall
    return m


def _metrics(model, cache, train_tensor, test_tensor, counter, epoch_no, seconds, do_eval=True,
             forest=None):
    if do_eval:
        train_rmse, train_mae = evaluate(model, train_tensor, cache, forest)
        if test_tensor is not None:
            test_rmse, test_mae = evaluate(model, test_tensor, cache)
        else:
            test_rmse = test_mae = float("nan")
    else:
        train_rmse = train_mae = test_rmse = test_mae = float("nan")
    return EpochMetrics(epoch=epoch_no, train_rmse=train_rmse, train_mae=train_mae,
                        test_rmse=test_rmse, test_mae=test_mae, seconds=seconds,
                        multiplies=counter.total_multiplies, counts=counter.snapshot())


def train(model, train_tensor, cfg: TrainConfig, test_tensor=None, forest: CsfForest | None = None,
          counter: OpCounter | None = None, sweep_log=None) -> list:
    """Full training loop (train.py:306-336); row 0 evaluates the initial model."""
    if forest is None:
        forest = build_forest(train_tensor, cfg.fiber_threshold)
    if counter is None:
        counter = OpCounter()
    cache = precompute_cache(model, counter) if cfg.plan == "cached" else None
    metrics = [_metrics(model, cache, train_tensor, test_tensor, counter, 0, 0.0, True, forest)]
    guards = GuardBank(model.order)
    for epoch_no in range(1, cfg.epochs + 1):
        m = run_epoch(model, forest, cache, train_tensor, cfg, counter, epoch_no, test_tensor,
                      sweep_log, _guards=guards)
        metrics.append(m)
        if cfg.rmse_delta_stop is not None and len(metrics) >= 2:
            monitored = "test_rmse" if test_tensor is not None else "train_rmse"
            prev, cur = getattr(metrics[-2], monitored), getattr(metrics[-1], monitored)
            if abs(prev - cur) < cfg.rmse_delta_stop:
                break
    return metrics
