"""Generate the golden fixtures in tests/golden/ by running the REFERENCE package itself.

Runs only in the build container, where /root/reference exists (it does not travel to the
GPU box; the .npz outputs do).  The reference is imported read-only from
/root/reference/pkg/src with its own compiled kernel module (oracle/_ref/_ckern*.so, built
by `make -C oracle ref` from the reference's _ckern.pyx) injected as
`fastertucker._kernels._ckern`, so every number below is produced by the reference's
stock code path (BACKEND == "c").

    python tests/golden/make_golden.py

Outputs (all small, compressed):
  trees.npz     B-CSF arrays of the reference's build_tree on hand/known/random tensors
                (csf.py:101-196), plus sha256 digests of the config-1 forest arrays.
  config1.npz   BASELINE config 1: generate_synthetic((1000,)*3, 100_000, (1,5), seed=0),
                split_dataset(0.1, seed=0), default_init_model((8,8,8), 8, seed=0),
                TrainConfig(lr 1e-3, reg 1e-2, epochs 5, cached, thr 128): per-sweep
                snapshots of epoch 1 and 2, the model after every epoch, metrics, counts.
  cases.npz     Small training cases taken from the reference's own tests
                (pkg/tests/test_backends.py, test_trainer.py, test_intermediates.py).
"""

from __future__ import annotations

import glob
import hashlib
import importlib.util
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"


def load_reference():
    so = glob.glob(os.path.join(REPO, "oracle", "_ref", "_ckern*.so"))
    if not so:
        raise SystemExit("run `make -C oracle ref` first")
    spec = importlib.util.spec_from_file_location("fastertucker._kernels._ckern", so[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    sys.modules["fastertucker._kernels._ckern"] = mod
    sys.path.insert(0, REF_SRC)
    os.environ.pop("FASTERTUCKER_BACKEND", None)
    import fastertucker as ft  # noqa: E402

    assert ft.BACKEND == "c", ft.BACKEND
    return ft


def digest(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr, dtype="<i8").tobytes()).hexdigest()


def fdigest(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr, dtype="<f8").tobytes()).hexdigest()


def tree_arrays(prefix, tree, out):
    N = len(tree.level_modes)
    out[prefix + "fiber_ptr"] = tree.fiber_ptr
    out[prefix + "fiber_coord"] = tree.fiber_coord
    out[prefix + "sub_fiber_ptr"] = tree.sub_fiber_ptr
    out[prefix + "sub_leaf_ptr"] = tree.sub_leaf_ptr
    out[prefix + "vals"] = tree.vals
    for d in range(N):
        out[prefix + f"inds{d}"] = tree.inds[d]
    for d in range(N - 1):
        out[prefix + f"ptrs{d}"] = tree.ptrs[d]


def make_trees(ft):
    out = {}
    cases = []

    def add(name, tensor, root, thr):
        tree = ft.build_tree(tensor, root, thr)
        key = f"{name}/r{root}/t{thr}/"
        out[key + "in_idx"] = tensor.idx.astype(np.int32)
        out[key + "in_vals"] = tensor.vals
        tree_arrays(key, tree, out)
        out[key + "dump"] = np.frombuffer(ft.dump_tree(tree).encode(), dtype=np.uint8)
        cases.append({"key": key, "dims": list(tensor.dims), "root": root, "thr": thr})

    hand = ft.SparseCooTensor((1, 2, 2), np.array([[0, 0, 0], [0, 0, 1], [0, 1, 0]]),
                              np.array([1.0, 2.0, 3.0]))
    add("hand", hand, 0, None)
    heavy = ft.SparseCooTensor((1, 300, 1), np.array([[0, f, 0] for f in range(300)]), np.ones(300))
    for r in range(3):
        add("heavy300", heavy, r, 128)
    single = ft.SparseCooTensor((4, 4, 4, 4), np.array([[2, 3, 1, 0]]), np.array([7.0]))
    add("single", single, 1, 128)
    t = ft.generate_synthetic((9, 8, 7, 6), 350, seed=13)
    for r in range(4):
        add("forest4", t, r, 4)
    rng = np.random.default_rng(2024)
    for case in range(24):
        order = int(rng.integers(3, 7))
        dims = tuple(int(rng.integers(2, 9)) for _ in range(order))
        cap = int(np.prod(dims))
        nnz = int(rng.integers(1, min(cap, 400) + 1))
        thr = [1, 2, 3, 8, 128, None][case % 6]
        t = ft.generate_synthetic(dims, nnz, seed=int(rng.integers(0, 10_000)))
        for root in range(order):
            add(f"rand{case}", t, root, thr)
    np.savez_compressed(os.path.join(HERE, "trees.npz"), **out)
    return cases


def snapshot_model(prefix, m, out):
    for n in range(m.order):
        out[f"{prefix}A{n}"] = m.factors[n].copy()
        out[f"{prefix}B{n}"] = m.cores_t[n].copy()


def make_config1(ft):
    tensor = ft.generate_synthetic((1000, 1000, 1000), 100_000, (1.0, 5.0), seed=0)
    split = ft.split_dataset(tensor, 0.1, seed=0)
    cfg = ft.TrainConfig(lr_a=1e-3, lr_b=1e-3, reg_a=1e-2, reg_b=1e-2, epochs=5, plan="cached",
                         fiber_threshold=128)
    model = ft.default_init_model((1000,) * 3, (8, 8, 8), 8, seed=0)
    out = {
        "train_idx": split.train.idx.astype(np.uint16),
        "train_vals": split.train.vals,
        "test_idx": split.test.idx.astype(np.uint16),
        "test_vals": split.test.vals,
    }
    snapshot_model("init/", model, out)
    forest = ft.build_forest(split.train, 128)
    meta = {"forest": []}
    for tree in forest.trees:
        N = len(tree.level_modes)
        d = {"root": tree.root_mode, "F": tree.num_fibers, "S": tree.num_subtensors,
             "fiber_ptr": digest(tree.fiber_ptr), "fiber_coord": digest(tree.fiber_coord),
             "sub_fiber_ptr": digest(tree.sub_fiber_ptr), "sub_leaf_ptr": digest(tree.sub_leaf_ptr),
             "vals": fdigest(tree.vals),
             "inds": [digest(tree.inds[k]) for k in range(N)],
             "ptrs": [digest(tree.ptrs[k]) for k in range(N - 1)]}
        meta["forest"].append(d)
    counter = ft.OpCounter()
    cache = ft.precompute_cache(model, counter)
    m0 = ft.train(model.copy(), split.train, ft.TrainConfig(epochs=0), split.test, forest=forest)[0]
    metrics = [[0, m0.train_rmse, m0.test_rmse, m0.train_mae, m0.test_mae]]
    for epoch in range(1, cfg.epochs + 1):
        for n in range(3):
            ft.update_factor_mode(model, forest, cache, n, cfg, counter)
            u = forest.trees[n].leaf_mode
            if epoch <= 2:
                out[f"e{epoch}/factor{n}/A"] = model.factors[u].copy()
                out[f"e{epoch}/factor{n}/C"] = cache.arrays[u].copy()
        for n in range(3):
            ft.update_core_mode(model, forest, cache, n, cfg, counter)
            u = forest.trees[n].leaf_mode
            if epoch <= 2:
                out[f"e{epoch}/core{n}/B"] = model.cores_t[u].copy()
        if epoch in (1, 2, cfg.epochs):
            snapshot_model(f"epoch{epoch}/", model, out)
        tr = ft.evaluate(model, split.train)
        te = ft.evaluate(model, split.test)
        metrics.append([epoch, tr[0], te[0], tr[1], te[1]])
    out["metrics"] = np.asarray(metrics, dtype=np.float64)
    out["counts"] = counter.counts.copy()
    # One core sweep's raw accumulator at the initial model (fiber-form check, train.py:218-236).
    m = ft.default_init_model((1000,) * 3, (8, 8, 8), 8, seed=0)
    cache0 = ft.precompute_cache(m)
    for n in range(3):
        tree = forest.trees[n]
        u = tree.leaf_mode
        acc = np.zeros((8, 8))
        ft._kernels.impl.core_sweep(tree.leaf_coord, tree.vals, tree.fiber_ptr, tree.fiber_coord,
                                    tree.prefix_modes, u, m.factors, m.cores_t, cache0.arrays, acc,
                                    np.zeros(5, np.int64), 0, tree.num_fibers)
        out[f"acc0/tree{n}"] = acc
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "config1.npz"), **out)
    print("config1 final test rmse", metrics[-1][2])


def make_cases(ft):
    out = {}
    manifest = []

    def run(name, tensor, ranks, R, init_seed, cfg_kw, test=None, sweeps=True):
        cfg = ft.TrainConfig(**cfg_kw)
        m = ft.default_init_model(tensor.dims, ranks, R, seed=init_seed)
        key = name + "/"
        out[key + "idx"] = tensor.idx.astype(np.int32)
        out[key + "vals"] = tensor.vals
        if test is not None:
            out[key + "test_idx"] = test.idx.astype(np.int32)
            out[key + "test_vals"] = test.vals
        snapshot_model(key + "init/", m, out)
        forest = ft.build_forest(tensor, cfg.fiber_threshold)
        counter = ft.OpCounter()
        cache = ft.precompute_cache(m, counter) if cfg.plan == "cached" else None
        rows = []
        for epoch in range(1, cfg.epochs + 1):
            for n in range(m.order):
                ft.update_factor_mode(m, forest, cache, n, cfg, counter)
                if sweeps and epoch == 1:
                    u = forest.trees[n].leaf_mode
                    out[key + f"e1/factor{n}/A"] = m.factors[u].copy()
            for n in range(m.order):
                ft.update_core_mode(m, forest, cache, n, cfg, counter)
                if sweeps and epoch == 1:
                    u = forest.trees[n].leaf_mode
                    out[key + f"e1/core{n}/B"] = m.cores_t[u].copy()
            tr = ft.evaluate(m, tensor)
            te = ft.evaluate(m, test) if test is not None else (float("nan"), float("nan"))
            rows.append([epoch, tr[0], te[0], tr[1], te[1]])
        snapshot_model(key + "final/", m, out)
        out[key + "metrics"] = np.asarray(rows, np.float64)
        out[key + "counts"] = counter.counts.copy()
        manifest.append({"name": name, "dims": list(tensor.dims), "ranks": list(ranks), "R": R,
                         "init_seed": init_seed, "cfg": cfg_kw, "has_test": test is not None})

    # test_backends.py:46-63 (order 4, threshold 4), both plans.
    t = ft.generate_synthetic((9, 11, 8, 7), 350, seed=5)
    for plan in ("cached", "uncached"):
        run(f"backends_{plan}", t, (2, 3, 2, 2), 3, 2,
            dict(lr_a=0.03, lr_b=0.03, reg_a=0.005, reg_b=0.005, epochs=2, plan=plan,
                 fiber_threshold=4))
    # test_trainer.py:220-233 counter laws.
    t = ft.generate_synthetic((12, 10, 14), 500, seed=6)
    for plan in ("uncached", "cached"):
        run(f"counters_{plan}", t, (3, 4, 2), 3, 2,
            dict(lr_a=0.01, lr_b=0.01, reg_a=0.001, reg_b=0.001, epochs=1, plan=plan))
    # test_trainer.py:162-170 plan equivalence.
    t = ft.generate_synthetic((15, 18, 21), 600, seed=7)
    run("plan_eq", t, (3, 2, 4), 3, 1, dict(lr_a=0.02, lr_b=0.02, reg_a=0.01, reg_b=0.01, epochs=5))
    # test_trainer.py:236-244 low-rank fixture.
    t = ft.generate_synthetic((40, 40, 40), 3000, seed=10, low_rank=((3, 3, 3), 3))
    split = ft.split_dataset(t, 0.1, seed=10)
    run("lowrank", split.train, (3, 3, 3), 3, 11,
        dict(lr_a=0.5, lr_b=0.5, reg_a=0.0, reg_b=0.0, epochs=5), test=split.test, sweeps=False)
    # test_trainer.py:262-277 hogwild fixture (serial reference trajectory).
    t = ft.generate_synthetic((20, 20, 20), 2000, seed=8)
    run("hogwild", t, (3, 3, 3), 2, 3,
        dict(lr_a=0.05, lr_b=0.05, reg_a=0.0, reg_b=0.0, epochs=3, fiber_threshold=8))
    # Higher orders, split rows (threshold 3), unequal J_n.
    for order, seed in ((5, 31), (6, 32)):
        dims = tuple(6 + k for k in range(order))
        t = ft.generate_synthetic(dims, 900, seed=seed)
        ranks = tuple(2 + (k % 3) for k in range(order))
        run(f"order{order}", t, ranks, 4, seed,
            dict(lr_a=0.05, lr_b=0.05, reg_a=0.01, reg_b=0.01, epochs=2, fiber_threshold=3))
    # J = R = 32 (the Netflix rank) on a small tensor, heavy rows.
    t = ft.generate_synthetic((300, 40, 12), 20_000, seed=17)
    run("rank32", t, (32, 32, 32), 32, 17,
        dict(lr_a=1e-3, lr_b=1e-3, reg_a=1e-2, reg_b=1e-2, epochs=2))
    # J = R = 16 with unequal dims.
    t = ft.generate_synthetic((500, 60, 9), 15_000, seed=18)
    run("rank16", t, (16, 16, 16), 16, 18,
        dict(lr_a=1e-3, lr_b=1e-3, reg_a=1e-2, reg_b=1e-2, epochs=2))
    # predict_batch on a random order-4 model (test_model.py:174-182).
    rng = np.random.default_rng(31)
    dims, ranks, R = (5, 4, 6, 3), (3, 2, 4, 2), 3
    factors = [rng.normal(size=(dims[n], ranks[n])) for n in range(4)]
    cores_t = [rng.normal(size=(R, ranks[n])) for n in range(4)]
    pm = ft.Model(dims, ranks, R, factors, cores_t)
    idx = np.stack([rng.integers(0, d, size=64) for d in dims], axis=1).astype(np.int64)
    snapshot_model("predict/", pm, out)
    out["predict/idx"] = idx
    out["predict/out"] = ft.predict_batch(pm, idx)
    out["manifest"] = np.frombuffer(json.dumps(manifest).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "cases.npz"), **out)


def main():
    ft = load_reference()
    make_trees(ft)
    make_cases(ft)
    make_config1(ft)
    for f in sorted(glob.glob(os.path.join(HERE, "*.npz"))):
        print(f, os.path.getsize(f))


if __name__ == "__main__":
    main()
