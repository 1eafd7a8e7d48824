"""Pin the CPU oracle (oracle/ft_oracle.c) to the reference's own outputs (tests/golden/).

The oracle is only trusted as the GPU path's checker because these tests show it reproduces
the reference bit-for-bit: tree layout (csf.py:101-196), the per-sweep parameters of the
serial trainer (train.py:152-278 over _ckern.pyx:21-282), the op counts (counter.py) and
predict/evaluate (model.py:219-230, train.py:91-98).
"""

import json

import numpy as np
import pytest

from conftest import parse_root, parse_thr, tree_case_keys
from oracle import oracle as O


def _model_from(z, prefix, N):
    factors = [np.array(z[f"{prefix}A{n}"]) for n in range(N)]
    cores_t = [np.array(z[f"{prefix}B{n}"]) for n in range(N)]
    dims = tuple(a.shape[0] for a in factors)
    ranks = tuple(a.shape[1] for a in factors)
    return O.OracleModel(dims, ranks, cores_t[0].shape[0], factors, cores_t)


def test_oracle_tree_layout_bit_exact(golden_trees):
    z = golden_trees
    keys = tree_case_keys(z)
    assert len(keys) > 80
    for key in keys:
        idx = z[key + "in_idx"].astype(np.int64)
        vals = z[key + "in_vals"]
        N = idx.shape[1]
        tree = O.build_tree(idx, vals, parse_root(key), parse_thr(key))
        np.testing.assert_array_equal(tree.fiber_ptr, z[key + "fiber_ptr"], err_msg=key)
        np.testing.assert_array_equal(tree.fiber_coord, z[key + "fiber_coord"], err_msg=key)
        np.testing.assert_array_equal(tree.sub_fiber_ptr, z[key + "sub_fiber_ptr"], err_msg=key)
        np.testing.assert_array_equal(tree.sub_leaf_ptr, z[key + "sub_leaf_ptr"], err_msg=key)
        assert np.array_equal(tree.vals, z[key + "vals"]), key
        for d in range(N):
            np.testing.assert_array_equal(tree.inds[d], z[key + f"inds{d}"], err_msg=key)
        for d in range(N - 1):
            np.testing.assert_array_equal(tree.ptrs[d], z[key + f"ptrs{d}"], err_msg=key)


def test_oracle_heavy_slice_split_sizes(golden_trees):
    # csf test: one root slice of 300 fibers at threshold 128 -> 128/128/44 (test_csf.py:64-74)
    idx = golden_trees["heavy300/r0/t128/in_idx"].astype(np.int64)
    tree = O.build_tree(idx, np.ones(300), 0, 128)
    assert list(np.diff(tree.sub_fiber_ptr)) == [128, 128, 44]
    assert np.array_equal(tree.inds[0], np.zeros(3, np.int64))


def test_oracle_config1_forest_digests(golden_config1):
    import hashlib

    z = golden_config1
    meta = json.loads(bytes(z["meta"]).decode())
    idx = z["train_idx"].astype(np.int64)
    vals = z["train_vals"]

    def dg(a):
        return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()

    for t, want in enumerate(meta["forest"]):
        tree = O.build_tree(idx, vals, t, 128)
        assert tree.num_fibers == want["F"] and tree.num_subtensors == want["S"]
        assert dg(tree.fiber_ptr) == want["fiber_ptr"]
        assert dg(tree.fiber_coord) == want["fiber_coord"]
        assert dg(tree.sub_fiber_ptr) == want["sub_fiber_ptr"]
        assert dg(tree.sub_leaf_ptr) == want["sub_leaf_ptr"]
        assert [dg(a) for a in tree.inds] == want["inds"]
        assert [dg(a) for a in tree.ptrs] == want["ptrs"]


def test_oracle_default_init_matches_reference(golden_config1):
    m = O.default_init_model((1000,) * 3, (8, 8, 8), 8, seed=0)
    ref = _model_from(golden_config1, "init/", 3)
    for a, b in zip(m.factors + m.cores_t, ref.factors + ref.cores_t):
        assert np.array_equal(a, b)


def test_oracle_config1_training_bitwise(golden_config1):
    z = golden_config1
    idx = z["train_idx"].astype(np.int64)
    vals = z["train_vals"]
    forest = O.build_forest(idx, vals, 128)
    model = _model_from(z, "init/", 3)
    cfg = O.OracleConfig(lr_a=1e-3, lr_b=1e-3, reg_a=1e-2, reg_b=1e-2)
    counts = np.zeros(5, np.int64)
    cache = O.precompute_cache(model, counts=counts)
    metrics = z["metrics"]
    for epoch in range(1, 6):
        for n in range(3):
            O.update_factor_mode(model, forest, cache, n, cfg, counts=counts)
            u = forest[n].leaf_mode
            if epoch <= 2:
                assert np.array_equal(model.factors[u], z[f"e{epoch}/factor{n}/A"])
                assert np.array_equal(cache[u], z[f"e{epoch}/factor{n}/C"])
        for n in range(3):
            O.update_core_mode(model, forest, cache, n, cfg, counts=counts)
            if epoch <= 2:
                assert np.array_equal(model.cores_t[forest[n].leaf_mode], z[f"e{epoch}/core{n}/B"])
        tr = O.evaluate(model, idx, vals)
        te = O.evaluate(model, z["test_idx"].astype(np.int64), z["test_vals"])
        np.testing.assert_allclose([tr[0], te[0], tr[1], te[1]], metrics[epoch, 1:], rtol=1e-12)
    ref = _model_from(z, "epoch5/", 3)
    for a, b in zip(model.factors + model.cores_t, ref.factors + ref.cores_t):
        assert np.array_equal(a, b)
    np.testing.assert_array_equal(counts, z["counts"])


def test_oracle_cases_bitwise(golden_cases):
    z = golden_cases
    manifest = json.loads(bytes(z["manifest"]).decode())
    assert len(manifest) >= 9
    for case in manifest:
        key = case["name"] + "/"
        cfgkw = case["cfg"]
        idx = z[key + "idx"].astype(np.int64)
        vals = z[key + "vals"]
        N = idx.shape[1]
        forest = O.build_forest(idx, vals, cfgkw.get("fiber_threshold", 128))
        model = _model_from(z, key + "init/", N)
        cfg = O.OracleConfig(lr_a=cfgkw["lr_a"], lr_b=cfgkw["lr_b"], reg_a=cfgkw["reg_a"],
                             reg_b=cfgkw["reg_b"], plan=cfgkw.get("plan", "cached"))
        counts = np.zeros(5, np.int64)
        cache = O.precompute_cache(model, counts=counts) if cfg.plan == "cached" else None
        for _epoch in range(cfgkw["epochs"]):
            O.run_epoch(model, forest, cache, cfg)
            # counts of the epoch, accumulated the way train() does
        final = _model_from(z, key + "final/", N)
        for a, b in zip(model.factors + model.cores_t, final.factors + final.cores_t):
            assert np.array_equal(a, b), case["name"]


def test_oracle_counts_match_reference(golden_cases):
    z = golden_cases
    for name, plan in (("counters_cached", "cached"), ("counters_uncached", "uncached")):
        key = name + "/"
        idx = z[key + "idx"].astype(np.int64)
        vals = z[key + "vals"]
        forest = O.build_forest(idx, vals, 128)
        model = _model_from(z, key + "init/", 3)
        cfg = O.OracleConfig(lr_a=0.01, lr_b=0.01, reg_a=0.001, reg_b=0.001, plan=plan)
        counts = np.zeros(5, np.int64)
        cache = O.precompute_cache(model, counts=counts) if plan == "cached" else None
        for n in range(3):
            O.update_factor_mode(model, forest, cache, n, cfg, counts=counts)
        for n in range(3):
            O.update_core_mode(model, forest, cache, n, cfg, counts=counts)
        np.testing.assert_array_equal(counts, z[key + "counts"])


def test_oracle_predict_matches_reference(golden_cases):
    z = golden_cases
    m = _model_from(z, "predict/", 4)
    out = O.predict(m, z["predict/idx"])
    np.testing.assert_allclose(out, z["predict/out"], rtol=1e-12, atol=1e-14)


def test_reference_kernels_agree_with_oracle(golden_cases):
    """oracle/_ref (the reference's compiled _ckern) and our restatement are bit-identical."""
    ref = O.ref_kernels()
    if ref is None:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    z = golden_cases
    key = "order5/"
    idx = z[key + "idx"].astype(np.int64)
    vals = z[key + "vals"]
    forest = O.build_forest(idx, vals, 3)
    outs = []
    for K in (O.CKernels, ref):
        model = _model_from(z, key + "init/", 5)
        cfg = O.OracleConfig(lr_a=0.05, lr_b=0.05, reg_a=0.01, reg_b=0.01)
        cache = O.precompute_cache(model, K=K)
        O.run_epoch(model, forest, cache, cfg, K=K)
        outs.append(model)
    for a, b in zip(outs[0].factors + outs[0].cores_t, outs[1].factors + outs[1].cores_t):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", ["oracle", "reference"])
def test_row_parallel_reference_is_the_serial_epoch(kind):
    """oracle.RowParallelRef (the at-scale checker of tests/test_netflix_parity_gpu.py): the
    row-partitioned concurrent factor sweeps are bitwise the serial sweeps of the full trees,
    and the per-group core accumulators sum to the serial core step (fp64 summation order
    only), over two epochs of an order-3 and an order-4 tensor with split root slices."""
    if kind == "reference" and O.ref_kernels() is None:
        pytest.skip("oracle/_ref not built")
    K = O.kernels(kind)
    for dims, nnz, J in (((60, 40, 30), 20_000, 8), ((12, 10, 9, 8), 5_000, 4)):
        rng = np.random.default_rng(len(dims))
        lin = rng.choice(int(np.prod(dims)), size=nnz, replace=False)
        idx = np.stack(np.unravel_index(lin, dims), axis=1).astype(np.int64)
        vals = rng.uniform(1, 5, size=nnz)
        N = len(dims)
        cfg = O.OracleConfig(lr_a=0.01, lr_b=0.01)
        serial = O.default_init_model(dims, (J,) * N, J, seed=3)
        par = serial.copy()
        forest = O.build_forest(idx, vals, 16)
        rp = O.RowParallelRef(idx, vals, dims, threads=5, K=K, fiber_threshold=16)
        c_s = O.precompute_cache(serial, K)
        c_p = O.precompute_cache(par, K)
        for _ in range(2):
            for t in range(N):
                O.update_factor_mode(serial, forest, c_s, t, cfg, K)
                rp.update_factor_mode(par, c_p, t, cfg)
                u = forest[t].leaf_mode
                assert np.array_equal(serial.factors[u], par.factors[u])
            for t in range(N):
                O.update_core_mode(serial, forest, c_s, t, cfg, K)
                rp.update_core_mode(par, c_p, t, cfg)
                u = forest[t].leaf_mode
                np.testing.assert_allclose(par.cores_t[u], serial.cores_t[u], rtol=1e-12)
                serial.cores_t[u][...] = par.cores_t[u]   # keep the factor check bitwise
                K.refresh_dot_mode(serial.factors[u], serial.cores_t[u], c_s[u],
                                   np.zeros(5, np.int64))
        rp.close()
