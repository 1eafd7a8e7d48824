"""Multiply counters (mirrors counter.OpCounter, /root/reference/pkg/src/fastertucker/counter.py).

The reference kernels tally five channels with one integer add per tree node
(_ckern.pyx:167-191, 236-261, 282, 33).  The GPU kernels do not count: these tallies are
ANALYTIC, closed forms of the tree shape evaluated on the host per sweep.
They equal the reference's counted tallies exactly on every golden case
(tests/test_host_cpu.py, tests/test_gpu_parity.py::test_config1_per_sweep_and_epoch), but they
cannot detect a kernel doing extra or missing work -- the parity tests on the values do that.
"""

from __future__ import annotations

import numpy as np

CHANNELS = ("dot", "chain", "combine", "shared", "update")
CH_DOT, CH_CHAIN, CH_COMBINE, CH_SHARED, CH_UPDATE = range(len(CHANNELS))


class OpCounter:
    """Monotone per-channel multiply tallies."""

    __slots__ = ("counts",)

    def __init__(self):
        self.counts = np.zeros(len(CHANNELS), dtype=np.int64)

    def __getitem__(self, channel: str) -> int:
        return int(self.counts[CHANNELS.index(channel)])

    @property
    def total_multiplies(self) -> int:
        return int(self.counts.sum() - self.counts[CH_SHARED])

    def merge(self, raw) -> None:
        self.counts += raw

    def snapshot(self) -> dict:
        return {name: int(self.counts[i]) for i, name in enumerate(CHANNELS)}

    def delta(self, before: dict) -> dict:
        return {name: int(self.counts[i]) - before[name] for i, name in enumerate(CHANNELS)}

    def reset(self) -> None:
        self.counts[:] = 0

    def csv_rows(self, plan: str, mode) -> list:
        return [f"{plan},{mode},{name},{int(self.counts[i])}" for i, name in enumerate(CHANNELS)]

    def __repr__(self):
        inner = ", ".join(f"{k}={v}" for k, v in self.snapshot().items())
        return f"OpCounter({inner})"


def new_raw_counts() -> np.ndarray:
    return np.zeros(len(CHANNELS), dtype=np.int64)


def sweep_counts(kind: str, plan: str, N: int, R: int, ranks, prefix_modes, leaf_mode: int,
                 nnz: int, num_fibers: int) -> np.ndarray:
    """Tallies of one factor_sweep / core_sweep over a whole tree (_pykern.py:98-137, 167-207).

    cached:   per fiber chain (N-2)R, combine J_u R, shared J_u R + N-2
    uncached: the same per LEAF, plus dot R * sum_{m in prefix} J_m per leaf
    update:   factor 4 J_u per leaf; core J_u + R(1 + J_u) per leaf
    """
    raw = new_raw_counts()
    Ju = int(ranks[leaf_mode])
    evals = num_fibers if plan == "cached" else nnz
    if plan != "cached":
        raw[CH_DOT] += nnz * R * sum(int(ranks[int(m)]) for m in prefix_modes)
    raw[CH_CHAIN] += evals * (N - 2) * R
    raw[CH_COMBINE] += evals * Ju * R
    raw[CH_SHARED] += evals * (Ju * R + N - 2)
    if kind == "factor":
        raw[CH_UPDATE] += nnz * 4 * Ju
    else:
        raw[CH_UPDATE] += nnz * (Ju + R * (1 + Ju))
    return raw


def apply_counts(R: int, Ju: int) -> np.ndarray:
    raw = new_raw_counts()
    raw[CH_UPDATE] += 2 * R * Ju
    return raw
