"""The reusable intermediates C^(n) = A^(n) B^(n) in HBM (mirrors cache.DotCache /
refresh_mode / precompute_cache, /root/reference/pkg/src/fastertucker/cache.py:28-78).

``arrays[n]`` is an I_n x R fp32 device matrix; ``arrays[n][i, r] == factors[n][i] .
cores_t[n][r]`` whenever mode n is clean.  Refresh runs kernel K2 (ft_refresh), which also
max-reduces |A_n| into an optional divergence-guard word in the same pass.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .counter import CH_DOT, OpCounter, new_raw_counts


class DotCache:
    __slots__ = ("arrays", "dirty")

    def __init__(self, model):
        import torch

        self.arrays = [torch.zeros((model.dims[n], model.core_rank), dtype=torch.float32,
                                   device="cuda") for n in range(model.order)]
        self.dirty = np.ones(model.order, dtype=bool)

    @property
    def order(self) -> int:
        return len(self.arrays)

    def mark_dirty(self, mode: int) -> None:
        self.dirty[mode] = True

    def max_error(self, model) -> float:
        """Largest deviation from freshly computed dot products (probe, cache.py:50-57)."""
        worst = 0.0
        for n in range(self.order):
            fresh = model.factors[n].double() @ model.cores_t[n].double().T
            worst = max(worst, float((fresh - self.arrays[n].double()).abs().max()))
        return worst

    def host(self):
        return [a.cpu().numpy().astype(np.float64) for a in self.arrays]


def refresh_into(model, mode: int, out, guard=None, stream=None) -> None:
    """C_mode = A_mode Bt_mode^T into ``out`` (K2), guard word optional."""
    L = _lib.lib()
    A, Bt = model.factors[mode], model.cores_t[mode]
    _lib.check(L.ft_refresh(A.shape[0], A.shape[1], Bt.shape[0], A.data_ptr(), Bt.data_ptr(),
                            out.data_ptr(), None if guard is None else guard.data_ptr(),
                            _lib.stream_handle(stream)), "ft_refresh")


def refresh_count(model, mode: int) -> int:
    return model.dims[mode] * model.ranks[mode] * model.core_rank


def refresh_mode(cache: DotCache, model, mode: int, counter: OpCounter | None = None,
                 guard=None) -> np.ndarray:
    raw = new_raw_counts()
    refresh_into(model, mode, cache.arrays[mode], guard)
    raw[CH_DOT] += refresh_count(model, mode)
    if counter is not None:
        counter.merge(raw)
    cache.dirty[mode] = False
    return raw


def precompute_cache(model, counter: OpCounter | None = None) -> DotCache:
    """Fill all modes; costs exactly sum_n I_n J_n R multiplies (cache.py:73-78)."""
    cache = DotCache(model)
    for n in range(model.order):
        refresh_mode(cache, model, n, counter)
    return cache


def fresh_dots(model):
    """C_n for every mode, computed now (the uncached plan's dots and predict_batch's)."""
    import torch

    out = []
    for n in range(model.order):
        c = torch.empty((model.dims[n], model.core_rank), dtype=torch.float32, device="cuda")
        refresh_into(model, n, c)
        out.append(c)
    return out


def counted_sweep_cost(plan: str, tensor, model, forest=None, fiber_threshold=None,
                       counter: OpCounter | None = None) -> int:
    """One full factor pass at zero learning rate; returns the dot-product multiplies it tallied
    (cache.py:132-165).  With lr = 0 every step adds exactly 0 (the sweeps' a + (-0) a + 0 e v),
    so the device model is untouched while the real kernels run.  The cached figure covers the
    per-mode refreshes; the one-time precompute is counted by `precompute_cache`."""
    from .csf import DEFAULT_FIBER_THRESHOLD, build_forest
    from .errors import ConfigError
    from .train import TrainConfig, update_factor_mode

    if plan not in ("cached", "uncached"):
        raise ConfigError(f"plan must be 'cached' or 'uncached', got {plan!r}")
    if forest is None:
        forest = build_forest(
            tensor, DEFAULT_FIBER_THRESHOLD if fiber_threshold is None else fiber_threshold)
    if counter is None:
        counter = OpCounter()
    cache = precompute_cache(model) if plan == "cached" else None
    cfg = TrainConfig(lr_a=0.0, lr_b=0.0, reg_a=0.0, reg_b=0.0, epochs=1, plan=plan)
    before = counter.snapshot()
    for n in range(model.order):
        update_factor_mode(model, forest, cache, n, cfg, counter)
    return counter.delta(before)["dot"]


def count_report(tensor, model, forest=None, fiber_threshold=None) -> list:
    """The reference's `count` command checks (cli.py:234-289) as a function: measured tallies
    of an uncached and a cached factor pass, the precompute and each tree's `shared` channel
    against their closed forms.  Returns the report lines (the uncached / cached dot-cost
    ratio last); raises CountMismatchError when any figure disagrees."""
    from .csf import DEFAULT_FIBER_THRESHOLD, build_forest
    from .errors import CountMismatchError
    from .train import TrainConfig, update_factor_mode

    thr = DEFAULT_FIBER_THRESHOLD if fiber_threshold is None else fiber_threshold
    if forest is None:
        forest = build_forest(tensor, thr)
    N, R, nnz, ranks = model.order, model.core_rank, tensor.nnz, model.ranks
    sum_jr = sum(j * R for j in ranks)
    sum_ijr = sum(d * j * R for d, j in zip(model.dims, ranks))

    def line(label, measured, formula, expected):
        status = "ok" if measured == expected else "MISMATCH"
        return f"{label:<22} measured={measured:<15} {formula}={expected:<15} {status}", \
            measured == expected

    checks = [
        line("uncached factor pass", counted_sweep_cost("uncached", tensor, model, forest),
             "(N-1)*nnz*sum(JnR)", (N - 1) * nnz * sum_jr),
        line("cached factor pass", counted_sweep_cost("cached", tensor, model, forest),
             "sum(In*Jn*R)", sum_ijr),
    ]
    pre = OpCounter()
    cache = precompute_cache(model, pre)
    checks.append(line("precompute", pre["dot"], "sum(In*Jn*R)", sum_ijr))
    cfg = TrainConfig(lr_a=0.0, lr_b=0.0, reg_a=0.0, reg_b=0.0, plan="cached",
                      fiber_threshold=thr)
    for n in range(N):
        c = OpCounter()
        update_factor_mode(model, forest, cache, n, cfg, c)
        tree = forest.trees[n]
        u = tree.leaf_mode
        checks.append(line(f"shared tree={n} mode={u}", c["shared"], "fibers*(JuR+N-2)",
                           tree.num_fibers * (ranks[u] * R + N - 2)))
    lines = [text for text, _ in checks]
    if not all(ok for _, ok in checks):
        raise CountMismatchError("measured operation counts disagree with closed forms\n" +
                                 "\n".join(lines))
    lines.append(f"uncached/cached dot-cost ratio: {((N - 1) * nnz * sum_jr) / sum_ijr:.2f}x")
    return lines
