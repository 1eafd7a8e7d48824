"""The BASELINE.json configs beyond Netflix, as parity cases at sizes the fp64 oracle replays in
seconds: order 6 and order 10 at 10 K per mode (> 64-bit keys: multi-pass LSD build, i.i.d.
generator), order 4 at 10 K per mode with J = R = 32, and the Yahoo!Music shape -- one exact
epoch each against the oracle at rel 1e-4, plus the compact forest."""

import numpy as np
import pytest

from helpers import assert_rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ft():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2210_06014_b200 as ft

    return ft


CASES = {
    "order6_16": ((10_000,) * 6, 120_000, 16),
    "order10_16": ((10_000,) * 10, 60_000, 16),
    "order4_32": ((10_000,) * 4, 150_000, 32),
    "yahoo_shape_32": ((1_000_990, 624_961, 3_075), 150_000, 32),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_config_shape_one_epoch_matches_oracle(ft, name):
    from oracle import oracle as O

    dims, nnz, JR = CASES[name]
    N = len(dims)
    t = ft.generate_device(dims, nnz, (1.0, 5.0), seed=3)
    idx = t.idx.cpu().numpy().astype(np.int64)
    vals = t.vals.cpu().numpy().astype(np.float64)
    assert (idx >= 0).all() and (idx < np.array(dims)).all()
    assert np.unique(idx, axis=0).shape[0] == nnz
    om = O.default_init_model(dims, (JR,) * N, JR, seed=1)
    model = ft.Model(dims, (JR,) * N, JR, om.factors, om.cores_t)
    oforest = O.build_forest(idx, vals, 128)
    forest = ft.build_forest(t, 128, compact=True)
    for tree, otree in zip(forest.trees, oforest):
        np.testing.assert_array_equal(tree.fiber_ptr.cpu().numpy(), otree.fiber_ptr)
        np.testing.assert_array_equal(tree.leaf_coord.cpu().numpy(), otree.leaf_coord)
    cfg = ft.TrainConfig(lr_a=1e-3, lr_b=1e-3, reg_a=1e-2, reg_b=1e-2)
    ocfg = O.OracleConfig(lr_a=1e-3, lr_b=1e-3, reg_a=1e-2, reg_b=1e-2)
    cache = ft.precompute_cache(model)
    ocache = O.precompute_cache(om)
    for n in range(N):
        ft.update_factor_mode(model, forest, cache, n, cfg)
        O.update_factor_mode(om, oforest, ocache, n, ocfg)
    for n in range(N):
        ft.update_core_mode(model, forest, cache, n, cfg)
        O.update_core_mode(om, oforest, ocache, n, ocfg)
    for n in range(N):
        assert_rel(model.factors[n].cpu().numpy(), om.factors[n], 1e-4, f"{name} A{n}")
        assert_rel(model.cores_t[n].cpu().numpy(), om.cores_t[n], 1e-4, f"{name} B{n}")


def test_compact_forest_equals_full(ft):
    t = ft.generate_device((3000, 400, 90, 7), 200_000, (1.0, 5.0), seed=9)
    full = ft.build_forest(t, 8)
    comp = ft.build_forest(t, 8, compact=True)
    for a, b in zip(full.trees, comp.trees):
        for name in ("fiber_ptr", "fiber_coord", "row_fiber_ptr", "row_coord", "vals"):
            assert bool((getattr(a, name) == getattr(b, name)).all()), name
        assert bool((a.leaf_coord == b.leaf_coord).all())
        assert a.num_subtensors == b.num_subtensors
