"""The leaf-major index (K1b, ft_tree_leaf_index), the four-rows-per-warp factor kernels (K3b
`quadr`: many rows, `quadw`: few long rows) and the core kernel (K4 `quad`, direct and staged
loads) against the fp64 oracle (oracle/), at the contract's rel 1e-4 per sweep.

These cases force a kernel on every mode (FT_FACTOR_KERNEL, in a subprocess because the choice
is latched at the first launch) on shapes that exercise its edges: rows shorter than one 8-leaf
batch, rows of ~20 K serial updates, J < 32 and R < 32 padding, more rows than row slots.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ft():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2210_06014_b200 as ft

    return ft


def test_leaf_index_matches_fiber_arrays(ft, monkeypatch):
    """leaf_pc[L, :] = fiber_coord[f(L), 1:N-1] and row_leaf_ptr[r] = fiber_ptr[row_fiber_ptr[r]],
    on a skewed tensor (long and single-leaf fibers) for every root mode, orders 3 to 6."""
    import torch

    monkeypatch.setenv("FT_LEAF_INDEX_MAX_ORDER", "6")
    rng = np.random.default_rng(3)
    for dims in ((300, 40, 7), (50, 9, 11, 6), (20, 9, 7, 6, 5), (9, 8, 7, 6, 5, 4)):
        n = 20_000
        # skew: a few heavy coordinates per mode so fibers range from 1 to hundreds of leaves
        cols = [np.minimum(rng.zipf(1.6, size=4 * n) - 1, d - 1) for d in dims]
        lin = np.unique(np.ravel_multi_index(cols, dims))[:n]
        idx = np.stack(np.unravel_index(lin, dims), axis=1)
        dev = ft.DeviceCoo(dims, torch.from_numpy(idx.astype(np.int32)).cuda(),
                           torch.from_numpy(rng.uniform(1, 5, len(lin)).astype(np.float32)).cuda())
        for t in range(len(dims)):
            tree = ft.build_tree(dev, t, 128)
            fp = tree.fiber_ptr.cpu().numpy().astype(np.int64)
            fc = tree.fiber_coord.cpu().numpy()
            want = np.repeat(fc[:, 1:len(dims) - 1], np.diff(fp), axis=0)
            np.testing.assert_array_equal(tree.leaf_pc.cpu().numpy(), want)
            rfp = tree.row_fiber_ptr.cpu().numpy()
            np.testing.assert_array_equal(tree.row_leaf_ptr.cpu().numpy(), fp[rfp])


_CASE = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2210_06014_b200 as ft
from oracle import oracle as O
from helpers import assert_rel
dims, nnz, J, R, lr, seed = {dims}, {nnz}, {J}, {R}, {lr}, {seed}
rng = np.random.default_rng(seed)
lin = rng.choice(int(np.prod(dims)), size=nnz, replace=False)
idx = np.stack(np.unravel_index(lin, dims), axis=1).astype(np.int64)
vals = rng.uniform(1, 5, size=nnz)
N = len(dims)
om = O.default_init_model(dims, (J,) * N, R, seed=seed)
model = ft.Model(dims, (J,) * N, R, om.factors, om.cores_t)
dev = ft.DeviceCoo(dims, torch.from_numpy(idx.astype(np.int32)).cuda(),
                   torch.from_numpy(vals.astype(np.float32)).cuda())
oforest = O.build_forest(idx, vals, 128)
forest = ft.build_forest(dev, 128)
ocfg = O.OracleConfig(lr_a=lr, lr_b=lr, reg_a=1e-2, reg_b=1e-2)
cfg = ft.TrainConfig(lr_a=lr, lr_b=lr, reg_a=1e-2, reg_b=1e-2)
ocache, cache = O.precompute_cache(om), ft.precompute_cache(model)
worst = 0.0
for epoch in range(2):
    for n in range(N):
        O.update_factor_mode(om, oforest, ocache, n, ocfg)
        ft.update_factor_mode(model, forest, cache, n, cfg)
        u = forest.trees[n].leaf_mode
        assert_rel(model.factors[u].cpu().numpy(), om.factors[u], 1e-4, f"e{{epoch}} factor {{u}}")
    for n in range(N):
        O.update_core_mode(om, oforest, ocache, n, ocfg)
        ft.update_core_mode(model, forest, cache, n, cfg)
        u = forest.trees[n].leaf_mode
        assert_rel(model.cores_t[u].cpu().numpy(), om.cores_t[u], 1e-4, f"e{{epoch}} core {{u}}")
print('ok')
"""


@pytest.mark.parametrize("dims,nnz,J,R,lr", [
    ((4000, 300, 50), 1_000_000, 32, 32, 2e-3),   # ~20 K-update rows in mode 2, 4000 short rows
    ((20000, 700, 9), 300_000, 24, 20, 1e-3),     # J < 32, R < 32 (padding), 1-3 leaf rows
    ((60000, 64, 64), 200_000, 32, 32, 5e-3),     # more rows than row slots (row switching)
    ((4000, 300, 50), 500_000, 16, 12, 2e-3),     # J <= 16 (one m-tile), R = 12 (two k-tiles)
    ((2000, 300, 40, 25), 400_000, 32, 32, 2e-3),  # order 4 (two prefix levels), 10-16 K-update rows
])
@pytest.mark.parametrize("kernel", ["quadr", "quadr-stagedcore", "quadw", "quadw-gram", "quadw-chain"])
def test_quad_sweeps_match_oracle(kernel, dims, nnz, J, R, lr):
    """-stagedcore: the K4 quad core with cp.async-staged gathers (FT_CORE_DIRECT=0; the default
    above 64 MB of gathered C rows) instead of direct register loads.  quadw picks its form by
    the row count (the Gram / segment form for few rows, the per-step chain otherwise);
    -gram / -chain force one form on every mode (FT_QUADW_GRAM)."""
    code = _CASE.format(dims=dims, nnz=nnz, J=J, R=R, lr=lr, seed=7)
    env = dict(os.environ, FT_FACTOR_KERNEL=kernel.split("-")[0])
    env.pop("FT_CORE_KERNEL", None)
    if kernel.endswith("-stagedcore"):
        env.update(FT_CORE_DIRECT="0")
    if kernel.startswith("quadw-"):
        env.update(FT_QUADW_GRAM="1" if kernel.endswith("-gram") else "0")
    out = subprocess.run([sys.executable, "-c", code], cwd=REPO, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


def test_sse_tree_matches_coo_evaluate(ft):
    """K6b (ft_sse_tree: the training set scored in tree order) gives the COO-order evaluate's
    RMSE / MAE up to the fp64 summation order, and the reference-format path is kept for a
    tensor the forest was not built from."""
    import torch

    rng = np.random.default_rng(5)
    dims = (3000, 400, 60)
    lin = rng.choice(int(np.prod(dims)), size=400_000, replace=False)
    idx = np.stack(np.unravel_index(lin, dims), axis=1)
    dev = ft.DeviceCoo(dims, torch.from_numpy(idx.astype(np.int32)).cuda(),
                       torch.from_numpy(rng.uniform(1, 5, len(lin)).astype(np.float32)).cuda())
    model = ft.default_init_model(dims, (32, 32, 32), 32, seed=1)
    forest = ft.build_forest(dev, 128)
    cache = ft.precompute_cache(model)
    ref = ft.evaluate(model, dev, cache)
    got = ft.evaluate(model, dev, cache, forest)
    np.testing.assert_allclose(got, ref, rtol=1e-6)
    # a forest of another tensor is ignored (falls back to the COO walk)
    other = ft.DeviceCoo(dims, dev.idx[:1000].contiguous(), dev.vals[:1000].contiguous())
    np.testing.assert_allclose(ft.evaluate(model, other, cache, forest),
                               ft.evaluate(model, other, cache), rtol=0)


@pytest.mark.parametrize("dims,nnz,J,R", [
    ((60, 50, 40, 30), 300_000, 32, 32),            # order 4 (two prefix levels)
    ((30, 20, 20, 15, 12), 200_000, 16, 16),        # order 5, J = R = 16 instantiation
    ((12, 10, 10, 9, 8, 8), 150_000, 24, 20),       # order 6, padding
])
def test_quad_order_n_sweeps_match_oracle(dims, nnz, J, R):
    """The default dispatch at orders 4-6 (factor: quadr at order 4, dual / gram at orders 5-6;
    core: K4 quad over the leaf-major index, its prefix product folded level by level), every
    sweep against the fp64 oracle at rel 1e-4."""
    code = _CASE.format(dims=dims, nnz=nnz, J=J, R=R, lr=2e-3, seed=9)
    env = dict(os.environ, FT_LEAF_INDEX_MAX_ORDER="6")
    env.pop("FT_FACTOR_KERNEL", None)
    env.pop("FT_CORE_KERNEL", None)
    out = subprocess.run([sys.executable, "-c", code], cwd=REPO, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


@pytest.mark.parametrize("I,J,R", [(1000, 32, 32), (130, 32, 32), (480_189, 32, 32),
                                   (5000, 16, 16), (777, 24, 12), (300, 8, 8), (2182, 32, 20)])
def test_refresh_tensor_core_matches_fp64(ft, I, J, R):
    """K2 on tcgen05 (kind::tf32, 3xTF32, TMEM accumulator): C = A Bt^T against fp64 at the
    contract's fp32-level accuracy, the fused guard (max |A| as IEEE bits) and the two-destination
    scatter form used by the fused multi-GPU refresh."""
    import ctypes

    import torch
    from paper_2210_06014_b200 import _lib

    rng = np.random.default_rng(I + J + R)
    A = rng.normal(size=(I, J)).astype(np.float32)
    Bt = rng.normal(size=(R, J)).astype(np.float32)
    ref = A.astype(np.float64) @ Bt.astype(np.float64).T
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(Bt).cuda()
    C = torch.full((I, R), float("nan"), device="cuda")
    g = torch.zeros(1, dtype=torch.int32, device="cuda")
    L = _lib.lib()
    _lib.check(L.ft_refresh(I, J, R, Ad.data_ptr(), Bd.data_ptr(), C.data_ptr(), g.data_ptr(),
                            _lib.stream_handle()), "ft_refresh")
    got = C.cpu().numpy().astype(np.float64)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 2e-6, err
    assert int(g.cpu().numpy().view(np.uint32)[0]) == int(np.abs(A).max().view(np.uint32))
    C2 = torch.zeros((I, R), device="cuda")
    tab = (ctypes.c_void_p * 2)(C.data_ptr(), C2.data_ptr())
    C.zero_()
    _lib.check(L.ft_refresh_scatter(I, J, R, Ad.data_ptr(), Bd.data_ptr(), tab, 2, None,
                                    _lib.stream_handle()), "ft_refresh_scatter")
    np.testing.assert_array_equal(C.cpu().numpy(), C2.cpu().numpy())
    np.testing.assert_array_equal(C.cpu().numpy(), got.astype(np.float32))


@pytest.mark.parametrize("dims,compact", [((3000, 400, 60), True), ((3000, 400, 60), False),
                                          ((60, 50, 40, 30), True), ((40, 30, 20, 10), False)])
def test_derived_tree_build_is_bit_identical(ft, dims, compact):
    """K1 derived build (tree t+1 from tree t's leaf order, 32-bit-key stable sort) produces
    exactly the arrays of the COO build, reference-format fields included."""
    import torch
    from paper_2210_06014_b200 import csf

    rng = np.random.default_rng(len(dims) + int(compact))
    lin = rng.choice(int(np.prod(dims)), size=min(300_000, int(np.prod(dims)) // 3), replace=False)
    idx = np.stack(np.unravel_index(lin, dims), axis=1)
    dev = ft.DeviceCoo(dims, torch.from_numpy(idx.astype(np.int32)).cuda(),
                       torch.from_numpy(rng.uniform(1, 5, len(lin)).astype(np.float32)).cuda())
    prev = csf.build_tree(dev, 0, 16, compact=compact)
    for t in range(1, len(dims)):
        want = csf.build_tree(dev, t, 16, compact=compact)
        got = csf.build_tree_derived(prev, 16, compact=compact)
        assert got is not None
        for name in ("vals", "fiber_ptr", "fiber_coord", "row_fiber_ptr", "row_coord", "leaf_pc",
                     "row_leaf_ptr", "seg_coord", "seg_leaf_ptr", "sub_fiber_ptr", "sub_leaf_ptr"):
            np.testing.assert_array_equal(getattr(got, name).cpu().numpy(),
                                          getattr(want, name).cpu().numpy(), err_msg=name)
        for a, b in zip(got.inds + got.ptrs, want.inds + want.ptrs):
            np.testing.assert_array_equal(a.cpu().numpy(), b.cpu().numpy())
        assert got.num_subtensors == want.num_subtensors
        prev = got


@pytest.mark.parametrize("dims", [(3000, 400, 60), (60, 50, 40, 30)])
def test_forest_without_fibers_matches(ft, dims):
    """build_forest(compact=True, keep_fibers=False) -- no fiber coordinates computed at all
    (the exact-schedule e2e step) -- gives the same leaf-major trees as the full compact build,
    refuses the fiber-walking hogwild sweep loudly, and trains to the same factors."""
    import torch
    from paper_2210_06014_b200 import csf

    rng = np.random.default_rng(11 + len(dims))
    lin = rng.choice(int(np.prod(dims)), size=200_000, replace=False)
    idx = np.stack(np.unravel_index(lin, dims), axis=1)
    dev = ft.DeviceCoo(dims, torch.from_numpy(idx.astype(np.int32)).cuda(),
                       torch.from_numpy(rng.uniform(1, 5, len(lin)).astype(np.float32)).cuda())
    full = csf.build_forest(dev, 16, compact=True)
    lean = csf.build_forest(dev, 16, compact=True, keep_fibers=False)
    for a, b in zip(full.trees, lean.trees):
        assert b.fiber_coord.numel() == 0 and b.num_fibers == a.num_fibers
        for name in ("vals", "row_fiber_ptr", "row_coord", "leaf_pc", "row_leaf_ptr", "seg_coord",
                     "seg_leaf_ptr"):
            np.testing.assert_array_equal(getattr(b, name).cpu().numpy(),
                                          getattr(a, name).cpu().numpy(), err_msg=name)
        np.testing.assert_array_equal(b.inds[-1].cpu().numpy(), a.inds[-1].cpu().numpy())
    N = len(dims)
    outs = []
    for forest in (full, lean):
        model = ft.default_init_model(dims, (16,) * N, 16, seed=3)
        cache = ft.precompute_cache(model)
        cfg = ft.TrainConfig(epochs=1)
        for n in range(N):
            ft.update_factor_mode(model, forest, cache, n, cfg)
        for n in range(N):
            ft.update_core_mode(model, forest, cache, n, cfg)
        outs.append([f.cpu().numpy() for f in model.factors] + [c.cpu().numpy() for c in model.cores_t])
    # the factor sweeps run the same kernels (bit-identical); the core sweep of a tree without
    # fibers always runs K4 quad, while the full tree may take the one-row-per-warp K4 on small
    # shapes (another fixed summation order): the cores agree to fp32 rounding
    for n, (a, b) in enumerate(zip(*outs)):
        if n < N:
            np.testing.assert_array_equal(a, b)
        else:
            np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-7)
    model = ft.default_init_model(dims, (16,) * N, 16, seed=3)
    with pytest.raises(Exception):
        ft.update_factor_mode(model, lean, ft.precompute_cache(model), 0,
                              ft.TrainConfig(epochs=1, schedule="hogwild"))
