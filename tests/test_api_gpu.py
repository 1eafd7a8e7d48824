"""Public-API behaviours beyond the sweeps: FTMODEL checkpoints in the reference's format,
the low-rank GPU generator, train() metrics / early stop / CSV rows, and the uncached plan."""

import os
import struct

import numpy as np
import pytest

from helpers import assert_rel, manifest, model_arrays

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ft():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2210_06014_b200 as ft

    return ft


def test_checkpoint_round_trip_reference_format(ft, tmp_path, golden_cases):
    f, c = model_arrays(golden_cases, "order5/init/", 5)
    m = ft.Model(tuple(a.shape[0] for a in f), tuple(a.shape[1] for a in f), 4, f, c)
    p = tmp_path / "m.ftm"
    ft.save_model(p, m)
    raw = open(p, "rb").read()
    assert raw[:8] == b"FTMODEL\x00"
    assert struct.unpack_from("<IIII", raw, 8) == (1, 5, 4, 0)
    back = ft.load_model(p)
    for a, b in zip(m.factors + m.cores_t, back.factors + back.cores_t):
        assert np.array_equal(a.cpu().numpy(), b.cpu().numpy())
    # the payload is the fp64 widening of the fp32 parameters, in the reference's order
    off = 24 + 16 * 5
    a0 = np.frombuffer(raw, "<f8", f[0].size, off).reshape(f[0].shape)
    assert np.array_equal(a0, m.factors[0].cpu().numpy().astype(np.float64))


def test_low_rank_generator_is_learnable(ft):
    dims = (300, 200, 100)
    t = ft.generate_low_rank_device(dims, 60_000, (4, 4, 4), 4, seed=7)
    idx = t.idx.cpu().numpy().astype(np.int64)
    key = (idx[:, 0] * dims[1] + idx[:, 1]) * dims[2] + idx[:, 2]
    assert np.unique(key).size == key.size
    model = ft.default_init_model(dims, (4, 4, 4), 4, seed=1)
    rows = ft.train(model, t, ft.TrainConfig(lr_a=0.5, lr_b=0.5, reg_a=0.0, reg_b=0.0, epochs=6))
    rmse = [r.train_rmse for r in rows]
    assert all(b < a for a, b in zip(rmse, rmse[1:])), rmse


def test_train_metrics_rows_and_early_stop(ft, golden_config1):
    z = golden_config1
    train = ft.SparseCooTensor((1000,) * 3, z["train_idx"].astype(np.int64), z["train_vals"])
    f, c = model_arrays(z, "init/", 3)
    model = ft.Model((1000,) * 3, (8, 8, 8), 8, f, c)
    rows = ft.train(model, train, ft.TrainConfig(epochs=10, rmse_delta_stop=1.0))
    assert len(rows) == 2  # the first epoch already moves RMSE by less than 1.0
    assert np.isnan(rows[1].test_rmse)
    line = rows[1].csv_row().split(",")
    assert line[0] == "1" and len(line) == len(ft.METRICS_CSV_HEADER.split(","))
    assert rows[1].factor_seconds > 0 and rows[1].core_seconds > 0


def test_uncached_plan_matches_cached(ft, golden_cases):
    """plan_eq (test_trainer.py:162-170): cached and uncached plans give the same parameters."""
    z = golden_cases
    case = next(c for c in manifest(z) if c["name"] == "plan_eq")
    import torch

    dev = ft.DeviceCoo(tuple(case["dims"]), torch.from_numpy(z["plan_eq/idx"].astype(np.int32)).cuda(),
                       torch.from_numpy(z["plan_eq/vals"].astype(np.float32)).cuda())
    outs = []
    for plan in ("cached", "uncached"):
        f, c = model_arrays(z, "plan_eq/init/", 3)
        m = ft.Model(tuple(case["dims"]), tuple(case["ranks"]), case["R"], f, c)
        ft.train(m, dev, ft.TrainConfig(**case["cfg"], plan=plan))
        outs.append(m)
    for a, b in zip(outs[0].factors + outs[0].cores_t, outs[1].factors + outs[1].cores_t):
        assert_rel(b.cpu().numpy(), a.cpu().numpy(), 1e-6, "plan equivalence")
    f, c = model_arrays(z, "plan_eq/final/", 3)
    for n in range(3):
        assert_rel(outs[1].factors[n].cpu().numpy(), f[n], 1e-4, f"uncached A{n}")


def test_counted_sweep_cost_formulas(ft):
    """test_intermediates.py:109-120 on the device sweeps."""
    dims, ranks, R = (20, 25, 30), (3, 4, 5), 3
    t = ft.generate_synthetic(dims, 700, seed=4)
    m = ft.default_init_model(dims, ranks, R, seed=4)
    sum_jr = sum(j * R for j in ranks)
    want_uncached = (t.order - 1) * t.nnz * sum_jr
    want_cached = sum(d * j * R for d, j in zip(dims, ranks))
    assert ft.counted_sweep_cost("uncached", t, m) == want_uncached
    assert ft.counted_sweep_cost("cached", t, m) == want_cached
    assert want_cached < want_uncached


def test_counted_sweep_cost_leaves_model_untouched(ft):
    """test_intermediates.py:123-129: the zero-lr passes change no parameter bit."""
    t = ft.generate_synthetic((10, 10, 10), 200, seed=6)
    m = ft.default_init_model(t.dims, (2, 2, 2), 2, seed=6)
    before = [a.clone() for a in m.factors + m.cores_t]
    ft.counted_sweep_cost("uncached", t, m)
    ft.counted_sweep_cost("cached", t, m)
    for a, b in zip(before, m.factors + m.cores_t):
        assert np.array_equal(a.cpu().numpy().view(np.uint32), b.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("dims,ranks,R,nnz", [((40, 30, 20), (4, 4, 4), 4, 3000),
                                              ((12, 10, 9, 8), (3, 2, 4, 2), 3, 1500)])
def test_count_report_closed_forms(ft, dims, ranks, R, nnz):
    """The `count` command's checks (cli.py:234-289) all report ok."""
    t = ft.generate_synthetic(dims, nnz, seed=2)
    m = ft.default_init_model(dims, ranks, R, seed=2)
    lines = ft.count_report(t, m, fiber_threshold=8)
    assert len(lines) == 3 + len(dims) + 1
    assert all(l.endswith("ok") for l in lines[:-1]), lines
    assert lines[-1].startswith("uncached/cached dot-cost ratio:")
