"""Host-side logic on CPU: config validation, the closed-form op counts (the GPU kernels do not
count; counter.sweep_counts must reproduce the reference's tallies exactly), and the split."""

import numpy as np
import pytest

from helpers import manifest, model_arrays
from oracle import oracle as O
from paper_2210_06014_b200.counter import CH_DOT, OpCounter, apply_counts, sweep_counts
from paper_2210_06014_b200.errors import ConfigError
from paper_2210_06014_b200.train import TrainConfig


def test_train_config_validation():
    with pytest.raises(ConfigError):
        TrainConfig(plan="nope")
    with pytest.raises(ConfigError):
        TrainConfig(lr_a=-1)
    with pytest.raises(ConfigError):
        TrainConfig(epochs=-1)
    with pytest.raises(ConfigError):
        TrainConfig(schedule="fast")
    assert TrainConfig().resolved_schedule == "exact"
    assert TrainConfig(workers=8).resolved_schedule == "hogwild"


def _closed_form_epoch_counts(forest, dims, ranks, R, plan, epochs):
    N = len(dims)
    total = np.zeros(5, np.int64)
    if plan == "cached":
        total[CH_DOT] += sum(dims[n] * ranks[n] * R for n in range(N))
    for _ in range(epochs):
        for kind in ("factor", "core"):
            for tree in forest:
                u = tree.leaf_mode
                total += sweep_counts(kind, plan, N, R, ranks, tree.prefix_modes, u, tree.nnz,
                                      tree.num_fibers)
                if kind == "core":
                    total += apply_counts(R, ranks[u])
                if plan == "cached":
                    total[CH_DOT] += dims[u] * ranks[u] * R
    return total


@pytest.mark.parametrize("name", ["backends_cached", "backends_uncached", "counters_cached",
                                  "counters_uncached", "order5", "order6", "rank32"])
def test_closed_form_counts_equal_reference(golden_cases, name):
    z = golden_cases
    case = next(c for c in manifest(z) if c["name"] == name)
    cfg = case["cfg"]
    forest = O.build_forest(z[name + "/idx"].astype(np.int64), z[name + "/vals"],
                            cfg.get("fiber_threshold", 128))
    got = _closed_form_epoch_counts(forest, case["dims"], case["ranks"], case["R"],
                                    cfg.get("plan", "cached"), cfg["epochs"])
    np.testing.assert_array_equal(got, z[name + "/counts"])


def test_closed_form_counts_config1(golden_config1):
    z = golden_config1
    forest = O.build_forest(z["train_idx"].astype(np.int64), z["train_vals"], 128)
    got = _closed_form_epoch_counts(forest, (1000,) * 3, (8, 8, 8), 8, "cached", 5)
    np.testing.assert_array_equal(got, z["counts"])


def test_op_counter_total_excludes_shared():
    c = OpCounter()
    c.merge(np.array([1, 2, 3, 100, 4], np.int64))
    assert c.total_multiplies == 10 and c["shared"] == 100
