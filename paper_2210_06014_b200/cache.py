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
