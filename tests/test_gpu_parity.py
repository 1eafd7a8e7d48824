"""GPU parity of the sm_100a path against the reference (goldens made by the reference itself,
tests/golden/make_golden.py) and the pinned fp64 oracle (oracle/).

Contract (SURVEY.md 8c / BASELINE.json north_star):
  * layout: exact integer equality with csf.build_tree (csf.py:101-196);
  * deterministic ("exact") schedule: per-sweep and per-epoch factors and cores at rel 1e-4
    (Frobenius and max-abs / max|ref|) against the fp64 reference;
  * hogwild schedule: train / test RMSE within 1% of the reference after E epochs;
  * op counts: exactly the reference's tallies.
"""

import json

import numpy as np
import pytest

from conftest import parse_root, parse_thr, tree_case_keys
from helpers import assert_rel, manifest, model_arrays, rel_errors

pytestmark = pytest.mark.gpu

TOL = 1e-4  # the contract's fp32 tolerance (measured headroom ~1e-6)


@pytest.fixture(scope="module")
def ft():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2210_06014_b200 as ft

    return ft


def _dev_coo(ft, idx, vals, dims=None):
    import torch

    idx = np.asarray(idx, dtype=np.int64)
    dims = dims or tuple(int(d) + 1 for d in idx.max(axis=0))
    return ft.DeviceCoo(tuple(dims), torch.from_numpy(idx.astype(np.int32)).cuda(),
                        torch.from_numpy(np.asarray(vals, np.float32)).cuda())


# ------------------------------------------------------------------------------------------
# K1 layout
# ------------------------------------------------------------------------------------------


def test_build_tree_bit_exact_all_golden_cases(ft, golden_trees):
    z = golden_trees
    keys = tree_case_keys(z)
    assert len(keys) > 80
    for key in keys:
        idx = z[key + "in_idx"].astype(np.int64)
        N = idx.shape[1]
        dims = tuple(int(d) + 1 for d in idx.max(axis=0))
        tree = ft.build_tree(_dev_coo(ft, idx, z[key + "in_vals"], dims), parse_root(key),
                             parse_thr(key))
        h = tree.host()
        for name in ("fiber_ptr", "fiber_coord", "sub_fiber_ptr", "sub_leaf_ptr"):
            np.testing.assert_array_equal(h[name], z[key + name], err_msg=key + name)
        for d in range(N):
            np.testing.assert_array_equal(h["inds"][d], z[key + f"inds{d}"], err_msg=f"{key}inds{d}")
        for d in range(N - 1):
            np.testing.assert_array_equal(h["ptrs"][d], z[key + f"ptrs{d}"], err_msg=f"{key}ptrs{d}")
        np.testing.assert_array_equal(h["vals"], z[key + "vals"].astype(np.float32), err_msg=key)
        # rows = unsplit root slices
        fc0 = h["fiber_coord"][:, 0]
        starts = np.flatnonzero(np.r_[True, fc0[1:] != fc0[:-1]])
        np.testing.assert_array_equal(h["row_fiber_ptr"], np.r_[starts, len(fc0)], err_msg=key)
        np.testing.assert_array_equal(h["row_coord"], fc0[starts], err_msg=key)


def test_build_forest_config1_digests(ft, golden_config1):
    import hashlib

    z = golden_config1
    meta = json.loads(bytes(z["meta"]).decode())
    dev = _dev_coo(ft, z["train_idx"], z["train_vals"], (1000, 1000, 1000))
    forest = ft.build_forest(dev, 128)

    def dg(a):
        return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()

    for t, want in enumerate(meta["forest"]):
        h = forest.trees[t].host()
        assert forest.trees[t].num_fibers == want["F"]
        assert forest.trees[t].num_subtensors == want["S"]
        for name in ("fiber_ptr", "fiber_coord", "sub_fiber_ptr", "sub_leaf_ptr"):
            assert dg(h[name]) == want[name], (t, name)
        assert [dg(a) for a in h["inds"]] == want["inds"]
        assert [dg(a) for a in h["ptrs"]] == want["ptrs"]


def test_build_rejects_duplicates_and_empty(ft):
    from paper_2210_06014_b200.errors import ValidationError

    idx = np.array([[0, 1, 2], [3, 1, 0], [0, 1, 2]])
    with pytest.raises(ValidationError, match=r"duplicate coordinate \(1, 2, 3\)"):
        ft.build_tree(_dev_coo(ft, idx, np.ones(3), (4, 4, 4)), 0)
    with pytest.raises(ValidationError):
        ft.SparseCooTensor((4, 4, 4), idx, np.ones(3))


def test_build_matches_oracle_random_large(ft):
    """Bit-exact against the pinned oracle builder on a 300K-entry random order-4 tensor with
    key bits > 32 and split rows."""
    from oracle import oracle as O

    rng = np.random.default_rng(7)
    dims = (3000, 50, 700, 9)
    lin = rng.choice(np.prod(dims), size=300_000, replace=False)
    idx = np.stack(np.unravel_index(lin, dims), axis=1).astype(np.int64)
    vals = rng.uniform(1, 5, size=idx.shape[0])
    dev = _dev_coo(ft, idx, vals, dims)
    for root in range(4):
        for thr in (128, 5, None):
            want = O.build_tree(idx, vals, root, thr)
            h = ft.build_tree(dev, root, thr).host()
            np.testing.assert_array_equal(h["fiber_ptr"], want.fiber_ptr)
            np.testing.assert_array_equal(h["fiber_coord"], want.fiber_coord)
            np.testing.assert_array_equal(h["sub_fiber_ptr"], want.sub_fiber_ptr)
            for d in range(4):
                np.testing.assert_array_equal(h["inds"][d], want.inds[d])
            for d in range(3):
                np.testing.assert_array_equal(h["ptrs"][d], want.ptrs[d])


def test_build_multi_pass_keys_order10(ft):
    """> 64 key bits (order 10, 10K per mode = 140 bits) -> 3 stable LSD passes; bit-exact."""
    from oracle import oracle as O

    rng = np.random.default_rng(3)
    dims = (10_000,) * 10
    idx = np.stack([rng.integers(0, d, size=20_000) for d in dims], axis=1).astype(np.int64)
    idx[1::7, :5] = idx[0::7, :5][: idx[1::7].shape[0]]  # shared prefixes -> real fibers
    idx = np.unique(idx, axis=0)
    rng.shuffle(idx)
    vals = rng.uniform(1, 5, size=idx.shape[0])
    dev = _dev_coo(ft, idx, vals, dims)
    for root in (0, 3, 9):
        want = O.build_tree(idx, vals, root, 4)
        h = ft.build_tree(dev, root, 4).host()
        np.testing.assert_array_equal(h["fiber_ptr"], want.fiber_ptr)
        np.testing.assert_array_equal(h["inds"][9], want.inds[9])
        np.testing.assert_array_equal(h["sub_fiber_ptr"], want.sub_fiber_ptr)


# ------------------------------------------------------------------------------------------
# K2-K6: training parity
# ------------------------------------------------------------------------------------------


def _model(ft, z, prefix, N):
    f, c = model_arrays(z, prefix, N)
    return ft.Model(tuple(a.shape[0] for a in f), tuple(a.shape[1] for a in f), c[0].shape[0], f, c)


def test_config1_per_sweep_and_epoch(ft, golden_config1):
    """BASELINE config 1 (1000^3, 90K train, J=R=8): every sweep of epochs 1-2 and the model
    after epochs 1, 2, 5 within rel 1e-4 of the reference; metrics and counts match."""
    z = golden_config1
    train = _dev_coo(ft, z["train_idx"], z["train_vals"], (1000,) * 3)
    test = _dev_coo(ft, z["test_idx"], z["test_vals"], (1000,) * 3)
    forest = ft.build_forest(train, 128)
    model = _model(ft, z, "init/", 3)
    cfg = ft.TrainConfig(lr_a=1e-3, lr_b=1e-3, reg_a=1e-2, reg_b=1e-2, epochs=5)
    counter = ft.OpCounter()
    cache = ft.precompute_cache(model, counter)
    worst = 0.0
    for epoch in range(1, 6):
        for n in range(3):
            ft.update_factor_mode(model, forest, cache, n, cfg, counter)
            u = forest.trees[n].leaf_mode
            if epoch <= 2:
                fro, mx = assert_rel(model.factors[u].cpu().numpy(), z[f"e{epoch}/factor{n}/A"],
                                     TOL, f"e{epoch} factor{n} A")
                worst = max(worst, fro, mx)
                assert_rel(cache.arrays[u].cpu().numpy(), z[f"e{epoch}/factor{n}/C"], TOL,
                           f"e{epoch} factor{n} C")
        for n in range(3):
            ft.update_core_mode(model, forest, cache, n, cfg, counter)
            u = forest.trees[n].leaf_mode
            if epoch <= 2:
                fro, mx = assert_rel(model.cores_t[u].cpu().numpy(), z[f"e{epoch}/core{n}/B"],
                                     TOL, f"e{epoch} core{n} B")
                worst = max(worst, fro, mx)
        if epoch in (1, 2, 5):
            f, c = model_arrays(z, f"epoch{epoch}/", 3)
            for n in range(3):
                assert_rel(model.factors[n].cpu().numpy(), f[n], TOL, f"epoch{epoch} A{n}")
                assert_rel(model.cores_t[n].cpu().numpy(), c[n], TOL, f"epoch{epoch} B{n}")
        tr = ft.evaluate(model, train, cache)
        te = ft.evaluate(model, test, cache)
        np.testing.assert_allclose([tr[0], te[0], tr[1], te[1]], z["metrics"][epoch, 1:],
                                   rtol=1e-5)
    np.testing.assert_array_equal(counter.counts, z["counts"])
    print(f"config1 worst per-sweep rel err {worst:.3e}")


def test_config1_train_api(ft, golden_config1):
    """train() end to end: row 0 + 5 epochs of metrics, reference within 1e-5 rel."""
    z = golden_config1
    train = ft.SparseCooTensor((1000,) * 3, z["train_idx"].astype(np.int64), z["train_vals"])
    test = ft.SparseCooTensor((1000,) * 3, z["test_idx"].astype(np.int64), z["test_vals"])
    model = _model(ft, z, "init/", 3)
    cfg = ft.TrainConfig(lr_a=1e-3, lr_b=1e-3, reg_a=1e-2, reg_b=1e-2, epochs=5)
    rows = ft.train(model, train, cfg, test)
    assert [m.epoch for m in rows] == list(range(6))
    got = np.array([[m.train_rmse, m.test_rmse, m.train_mae, m.test_mae] for m in rows])
    np.testing.assert_allclose(got, z["metrics"][:, 1:], rtol=1e-5)
    assert all(m.seconds > 0 for m in rows[1:])
    assert rows[-1].multiplies == int(z["counts"].sum() - z["counts"][3])


@pytest.mark.parametrize("name", ["backends_cached", "backends_uncached", "counters_cached",
                                  "counters_uncached", "plan_eq", "lowrank", "hogwild", "order5",
                                  "order6", "rank32", "rank16"])
def test_reference_cases(ft, golden_cases, name):
    z = golden_cases
    case = next(c for c in manifest(z) if c["name"] == name)
    key = name + "/"
    cfgkw = dict(case["cfg"])
    N = len(case["dims"])
    dev = _dev_coo(ft, z[key + "idx"], z[key + "vals"], tuple(case["dims"]))
    forest = ft.build_forest(dev, cfgkw.get("fiber_threshold", 128))
    model = _model(ft, z, key + "init/", N)
    cfg = ft.TrainConfig(**cfgkw)
    counter = ft.OpCounter()
    cache = ft.precompute_cache(model, counter) if cfg.plan == "cached" else None
    tol = TOL
    for epoch in range(1, cfg.epochs + 1):
        for n in range(N):
            ft.update_factor_mode(model, forest, cache, n, cfg, counter)
            u = forest.trees[n].leaf_mode
            if epoch == 1 and key + f"e1/factor{n}/A" in z.files:
                assert_rel(model.factors[u].cpu().numpy(), z[key + f"e1/factor{n}/A"], tol,
                           f"{name} e1 factor{n}")
        for n in range(N):
            ft.update_core_mode(model, forest, cache, n, cfg, counter)
            u = forest.trees[n].leaf_mode
            if epoch == 1 and key + f"e1/core{n}/B" in z.files:
                assert_rel(model.cores_t[u].cpu().numpy(), z[key + f"e1/core{n}/B"], tol,
                           f"{name} e1 core{n}")
        tr = ft.evaluate(model, dev)
        np.testing.assert_allclose(tr[0], z[key + "metrics"][epoch - 1, 1], rtol=1e-4)
    f, c = model_arrays(z, key + "final/", N)
    for n in range(N):
        assert_rel(model.factors[n].cpu().numpy(), f[n], tol, f"{name} final A{n}")
        assert_rel(model.cores_t[n].cpu().numpy(), c[n], tol, f"{name} final B{n}")
    np.testing.assert_array_equal(counter.counts, z[key + "counts"])


def test_predict_batch_matches_reference(ft, golden_cases):
    z = golden_cases
    m = _model(ft, z, "predict/", 4)
    out = ft.predict_batch(m, z["predict/idx"])
    np.testing.assert_allclose(out, z["predict/out"], rtol=2e-5, atol=2e-5)


def test_hogwild_rmse_fidelity(ft, golden_config1, golden_cases):
    """Hogwild schedule (K3a, racing row updates at the default, uncapped concurrency): RMSE
    after E epochs within 1 % of the reference's serial trajectory on BASELINE config 1 (north
    star), and within 2 % as the median of 3 runs on the reference's own hogwild fixture
    (its test_trainer.py:262-277 allows 15 %)."""
    z = golden_config1
    train = _dev_coo(ft, z["train_idx"], z["train_vals"], (1000,) * 3)
    test = _dev_coo(ft, z["test_idx"], z["test_vals"], (1000,) * 3)
    model = _model(ft, z, "init/", 3)
    cfg = ft.TrainConfig(lr_a=1e-3, lr_b=1e-3, reg_a=1e-2, reg_b=1e-2, epochs=5,
                         schedule="hogwild")
    rows = ft.train(model, train, cfg, test)
    ref = z["metrics"][5]
    assert abs(rows[-1].train_rmse - ref[1]) / ref[1] < 0.01
    assert abs(rows[-1].test_rmse - ref[2]) / ref[2] < 0.01
    zc = golden_cases
    case = next(c for c in manifest(zc) if c["name"] == "hogwild")
    dev = _dev_coo(ft, zc["hogwild/idx"], zc["hogwild/vals"], tuple(case["dims"]))
    ref_rmse = zc["hogwild/metrics"][-1, 1]
    gaps = []
    for _ in range(3):  # racing updates: every run differs
        model = _model(ft, zc, "hogwild/init/", 3)
        rows = ft.train(model, dev, ft.TrainConfig(**case["cfg"], schedule="hogwild"))
        gaps.append(abs(rows[-1].train_rmse - ref_rmse) / ref_rmse)
    assert float(np.median(gaps)) < 0.02, gaps


def test_exact_schedule_is_deterministic(ft, golden_cases):
    z = golden_cases
    case = next(c for c in manifest(z) if c["name"] == "rank32")
    dev = _dev_coo(ft, z["rank32/idx"], z["rank32/vals"], tuple(case["dims"]))
    forest = ft.build_forest(dev, 128)
    outs = []
    for _ in range(2):
        model = _model(ft, z, "rank32/init/", 3)
        cfg = ft.TrainConfig(**case["cfg"])
        cache = ft.precompute_cache(model)
        for n in range(3):
            ft.update_factor_mode(model, forest, cache, n, cfg)
        for n in range(3):
            ft.update_core_mode(model, forest, cache, n, cfg)
        outs.append([t.cpu().numpy() for t in model.factors + model.cores_t])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_core_accumulator_matches_reference(ft, golden_config1):
    """The reduced core gradient ``acc`` of one sweep at the initial model
    (core_sweep, _ckern.pyx:202-269) against the reference's raw accumulator."""
    import torch

    z = golden_config1
    train = _dev_coo(ft, z["train_idx"], z["train_vals"], (1000,) * 3)
    forest = ft.build_forest(train, 128)
    for n in range(3):
        model = _model(ft, z, "init/", 3)
        cache = ft.precompute_cache(model)
        acc = torch.empty((8, 8), dtype=torch.float32, device="cuda")
        cfg = ft.TrainConfig(lr_b=0.0, reg_b=0.0)
        ft.update_core_mode(model, forest, cache, n, cfg, acc_out=acc)
        assert_rel(acc.cpu().numpy(), z[f"acc0/tree{n}"], 1e-5, f"acc tree{n}")


def test_plugin_impl_matches_oracle(ft, golden_cases):
    """The reference-signature plugin (``_kernels.impl``, BACKEND 'cuda') on host arrays:
    refresh / factor_sweep / core_sweep / apply_core_update over whole trees and over single
    subtensor ranges, against the fp64 oracle at rel 1e-4."""
    from oracle import oracle as O
    from paper_2210_06014_b200 import _kernels

    z = golden_cases
    key = "order5/"
    idx = z[key + "idx"].astype(np.int64)
    vals = z[key + "vals"]
    forest = O.build_forest(idx, vals, 3)
    f0, c0 = model_arrays(z, key + "init/", 5)
    K = _kernels.get_backend("cuda")
    assert K.BACKEND == "cuda"
    for t, tree in enumerate(forest):
        u = tree.leaf_mode
        for lo, hi in ((0, tree.num_fibers),
                       (int(tree.sub_fiber_ptr[1]), int(tree.sub_fiber_ptr[2]))):
            outs = []
            for kern in (O.CKernels, K):
                f = [a.copy() for a in f0]
                c = [b.copy() for b in c0]
                dots = O.precompute_cache(O.OracleModel(tuple(a.shape[0] for a in f),
                                                          tuple(a.shape[1] for a in f), 4, f, c))
                counts = np.zeros(5, np.int64)
                kern.factor_sweep(tree.leaf_coord, tree.vals, tree.fiber_ptr, tree.fiber_coord,
                                  tree.prefix_modes, u, f, c, dots, 0.05, 0.01, counts, lo, hi)
                acc = np.zeros_like(c[u])
                kern.core_sweep(tree.leaf_coord, tree.vals, tree.fiber_ptr, tree.fiber_coord,
                                tree.prefix_modes, u, f, c, dots, acc, counts, lo, hi)
                kern.apply_core_update(c[u], acc, float(tree.nnz), 0.05, 0.01, counts)
                out = np.zeros((f[u].shape[0], 4))
                kern.refresh_dot_mode(f[u], c[u], out, counts)
                outs.append((f[u], c[u], acc, out, counts))
            for a, b in zip(outs[0][:4], outs[1][:4]):
                assert_rel(b, a, TOL, f"plugin tree{t} [{lo},{hi})")
            np.testing.assert_array_equal(outs[0][4], outs[1][4])


def test_divergence_error_names_mode_and_epoch(ft, golden_cases):
    from paper_2210_06014_b200.errors import DivergenceError

    z = golden_cases
    case = next(c for c in manifest(z) if c["name"] == "plan_eq")
    dev = _dev_coo(ft, z["plan_eq/idx"], z["plan_eq/vals"], tuple(case["dims"]))
    model = _model(ft, z, "plan_eq/init/", 3)
    cfg = ft.TrainConfig(lr_a=1e6, lr_b=1e6, epochs=3, divergence_limit=1e3)
    with pytest.raises(DivergenceError) as ei:
        ft.train(model, dev, cfg)
    assert ei.value.epoch == 1 and ei.value.mode == 2  # first factor sweep updates mode N-1


# ------------------------------------------------------------------------------------------
# full-size properties (sizes the oracle cannot replay quickly)
# ------------------------------------------------------------------------------------------


def test_generator_and_netflix_shaped_properties(ft):
    """GPU generator: distinct in-range cells, values in range; forest of a 4M-entry
    Netflix-shaped tensor conserves the entries; rows partition the leaves; one exact epoch
    lowers the training RMSE and is deterministic."""
    import torch

    dims = (480_189, 17_770, 2_182)
    t = ft.generate_device(dims, 4_000_000, (1.0, 5.0), seed=1)
    idx = t.idx.cpu().numpy().astype(np.int64)
    assert (idx >= 0).all() and (idx < np.array(dims)).all()
    key = (idx[:, 0] * dims[1] + idx[:, 1]) * dims[2] + idx[:, 2]
    assert np.unique(key).size == key.size
    v = t.vals.cpu().numpy()
    assert v.min() >= 1.0 and v.max() <= 5.0 and abs(v.mean() - 3.0) < 0.01
    forest = ft.build_forest(t, 128)
    for tree in forest.trees:
        assert tree.nnz == t.nnz
        fp = tree.fiber_ptr.cpu().numpy()
        assert fp[0] == 0 and fp[-1] == t.nnz and (np.diff(fp) > 0).all()
        rfp = tree.row_fiber_ptr.cpu().numpy()
        assert rfp[0] == 0 and rfp[-1] == tree.num_fibers and (np.diff(rfp) > 0).all()
        rc = tree.row_coord.cpu().numpy()
        assert (np.diff(rc) > 0).all()
        assert np.isclose(tree.vals.double().sum().item(), t.vals.double().sum().item(), rtol=1e-9)
    res = []
    for _ in range(2):
        model = ft.default_init_model(dims, (32, 32, 32), 32, seed=0)
        cfg = ft.TrainConfig(epochs=1)
        rows = ft.train(model, t, cfg)
        res.append((rows, torch.cat([a.flatten() for a in model.factors]).cpu().numpy()))
    assert res[0][0][1].train_rmse < res[0][0][0].train_rmse
    assert np.array_equal(res[0][1], res[1][1])


def test_row_shards_equal_unsharded(ft, golden_cases):
    """Multi-GPU partition, run as logical shards on one GPU: sweeping each row block of tree u
    separately gives bitwise the same A_u as the unsharded sweep (rows never interact), and the
    shard core gradients sum to the unsharded one."""
    import ctypes

    import torch

    from paper_2210_06014_b200 import _lib

    z = golden_cases
    case = next(c for c in manifest(z) if c["name"] == "rank32")
    dev = _dev_coo(ft, z["rank32/idx"], z["rank32/vals"], tuple(case["dims"]))
    forest = ft.build_forest(dev, 128)
    L = _lib.lib()
    for u in range(3):
        tree = forest.trees[u]
        ref = _model(ft, z, "rank32/init/", 3)
        cache = ft.precompute_cache(ref)
        L.ft_factor_sweep_rows(ctypes.byref(tree.view()), ctypes.byref(ref.view(cache.arrays)),
                               1e-3, 1e-2, None)
        sh = _model(ft, z, "rank32/init/", 3)
        cache2 = ft.precompute_cache(sh)
        cuts = np.linspace(0, tree.num_rows, 4).astype(int)
        for r0, r1 in zip(cuts[:-1], cuts[1:]):
            part = tree.slice_rows(int(r0), int(r1))
            _lib.check(L.ft_factor_sweep_rows(ctypes.byref(part.view()),
                                              ctypes.byref(sh.view(cache2.arrays)), 1e-3, 1e-2,
                                              None))
        torch.cuda.synchronize()
        assert torch.equal(ref.factors[u], sh.factors[u])


def test_long_rows_factor_and_core_sweeps_match_oracle(ft):
    """Rows with ~20K serial updates (the Netflix mode-2 regime, 45K per row at full size): one
    exact factor sweep and one core sweep of every mode against the fp64 oracle at rel 1e-4.
    Catches precision drift that only compounds on long rows."""
    from oracle import oracle as O

    rng = np.random.default_rng(11)
    dims = (4000, 300, 50)
    lin = rng.choice(np.prod(dims), size=1_000_000, replace=False)
    idx = np.stack(np.unravel_index(lin, dims), axis=1).astype(np.int64)
    vals = rng.uniform(1, 5, size=idx.shape[0])
    J = R = 16
    om = O.default_init_model(dims, (J,) * 3, R, seed=5)
    model = ft.Model(dims, (J,) * 3, R, om.factors, om.cores_t)
    oforest = O.build_forest(idx, vals, 128)
    forest = ft.build_forest(_dev_coo(ft, idx, vals, dims), 128)
    ocfg = O.OracleConfig(lr_a=2e-3, lr_b=2e-3, reg_a=1e-2, reg_b=1e-2)
    cfg = ft.TrainConfig(lr_a=2e-3, lr_b=2e-3, reg_a=1e-2, reg_b=1e-2)
    ocache = O.precompute_cache(om)
    cache = ft.precompute_cache(model)
    for n in range(3):
        O.update_factor_mode(om, oforest, ocache, n, ocfg)
        ft.update_factor_mode(model, forest, cache, n, cfg)
        u = forest.trees[n].leaf_mode
        assert_rel(model.factors[u].cpu().numpy(), om.factors[u], TOL, f"long rows factor {u}")
    for n in range(3):
        O.update_core_mode(om, oforest, ocache, n, ocfg)
        ft.update_core_mode(model, forest, cache, n, cfg)
        u = forest.trees[n].leaf_mode
        assert_rel(model.cores_t[u].cpu().numpy(), om.cores_t[u], TOL, f"long rows core {u}")


@pytest.mark.parametrize("variant", ["ws", "dual", "gram", "quadr", "quadw"])
def test_factor_kernel_variants_agree(variant, golden_cases):
    """Every warp-level K3b kernel the dispatcher can pick (FT_FACTOR_KERNEL forces one on every
    shape it covers, falling back to auto elsewhere) reproduces the reference's rank-32, order-5
    and rank-16 sweeps at 1e-4; in a subprocess because the choice is latched at first launch."""
    import os
    import subprocess
    import sys

    code = (
        "import numpy as np, sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import test_gpu_parity as t, conftest, paper_2210_06014_b200 as ft;"
        "z = np.load('tests/golden/cases.npz');"
        "t.test_reference_cases(ft, z, 'rank32'); t.test_reference_cases(ft, z, 'order5');"
        "t.test_reference_cases(ft, z, 'rank16'); print('ok')")
    env = dict(os.environ, FT_FACTOR_KERNEL=variant)
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=repo, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
