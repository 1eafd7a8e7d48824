"""The reference's OWN trainer driving this package's kernel plugin (``BACKEND == "cuda"``).

The reference package is installed from /root/reference into ``baseline/_ref`` (git-ignored,
shipped to the GPU box with the snapshot; the test skips without it).  Its callers reach the
kernels only through the module global ``fastertucker._kernels.impl`` (train.py:171, 179, 192,
219, 227, 237, 243), so binding ``impl`` to ``paper_2210_06014_b200._kernels._cudakern`` is
exactly the one-line integration INTEGRATION.md describes.

``workers = 4`` runs the reference's dynamic subtensor queue (train.py:124-149) with four
threads calling ``impl.factor_sweep`` / ``impl.core_sweep`` concurrently on different fiber
ranges over the shared host ``factors[u]`` (train.py:175-186, 222-236).
"""

import os
import sys

import numpy as np
import pytest

from helpers import assert_rel

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.isdir(os.path.join(REF, "fastertucker")):
        pytest.skip("reference package not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import fastertucker

    return fastertucker


def _tensor(R, dims, nnz, seed, edge_rows=False):
    """Distinct uniform cells.  edge_rows: in every mode m the rows D_m-4..D_m-2 hold exactly one
    entry each (their updates come from one subtensor) and row D_m-1 none (never touched)."""
    rng = np.random.default_rng(seed)
    core = tuple(d - 4 for d in dims) if edge_rows else dims
    lin = rng.choice(int(np.prod(core)), size=nnz, replace=False)
    idx = np.stack(np.unravel_index(lin, core), axis=1).astype(np.int64)
    if edge_rows:
        extra = []
        for m, d in enumerate(dims):
            for i in range(d - 4, d - 1):
                e = [int(rng.integers(0, c)) for c in core]
                e[m] = i
                extra.append(e)
        idx = np.concatenate([idx, np.asarray(extra, np.int64)])
    vals = rng.uniform(1.0, 5.0, size=idx.shape[0])
    return R.SparseCooTensor(dims, idx, vals)


def test_reference_trainer_with_workers_through_cuda_plugin(ref):
    """Per sweep, from the same starting model: the reference's serial compiled sweep vs the
    reference's 4-worker pool over the CUDA plugin.  Rows of A_u touched by exactly one
    subtensor must match the serial sweep (rel 1e-4: nothing may be lost or overwritten), rows
    no subtensor touches must keep their fp64 host values bit for bit, and the core step
    (per-worker accumulators, train.py:222-236) must match the serial step."""
    import importlib

    RK = importlib.import_module("fastertucker._kernels")
    RT = importlib.import_module("fastertucker.train")

    from paper_2210_06014_b200._kernels import _cudakern

    R = ref
    dims = (40, 30, 25)
    tensor = _tensor(R, dims, 6000, seed=4, edge_rows=True)
    forest = R.build_forest(tensor, 4)  # split root slices -> many subtensors per row
    base = R.default_init_model(dims, (8, 8, 8), 8, seed=2)
    ser_cfg = RT.TrainConfig(lr_a=0.02, lr_b=0.02, reg_a=1e-2, reg_b=1e-2, workers=0)
    par_cfg = RT.TrainConfig(lr_a=0.02, lr_b=0.02, reg_a=1e-2, reg_b=1e-2, workers=4)
    compiled = RK.impl
    assert compiled.BACKEND == "c"

    def clone(m):
        return R.Model(m.dims, m.ranks, m.core_rank, [a.copy() for a in m.factors],
                       [b.copy() for b in m.cores_t])

    for n in range(3):
        tree = forest.trees[n]
        u = tree.leaf_mode
        # which subtensors touch each row of A_u
        owners = {}
        for s in range(tree.num_subtensors):
            lo, hi = int(tree.sub_leaf_ptr[s]), int(tree.sub_leaf_ptr[s + 1])
            for i in np.unique(tree.leaf_coord[lo:hi]):
                owners.setdefault(int(i), set()).add(s)
        single = np.array(sorted(i for i, s in owners.items() if len(s) == 1))
        untouched = np.array(sorted(set(range(dims[u])) - set(owners)))
        assert single.size > 0 and untouched.size > 0

        m_ser, m_par = clone(base), clone(base)
        RT.update_factor_mode(m_ser, forest, R.precompute_cache(m_ser), n, ser_cfg)
        c_par = R.precompute_cache(m_par)
        RK.impl = _cudakern
        try:
            RT.update_factor_mode(m_par, forest, c_par, n, par_cfg)
        finally:
            RK.impl = compiled
        assert_rel(m_par.factors[u][single], m_ser.factors[u][single], 1e-4,
                   f"mode {u} single-owner rows")
        assert np.array_equal(m_par.factors[u][untouched], base.factors[u][untouched])
        assert np.isfinite(m_par.factors[u]).all()

        m_ser, m_par = clone(base), clone(base)
        RT.update_core_mode(m_ser, forest, R.precompute_cache(m_ser), n, ser_cfg)
        c_par = R.precompute_cache(m_par)
        RK.impl = _cudakern
        try:
            RT.update_core_mode(m_par, forest, c_par, n, par_cfg)
        finally:
            RK.impl = compiled
        assert_rel(m_par.cores_t[u], m_ser.cores_t[u], 1e-4, f"core mode {u}")
        assert_rel(c_par.arrays[u], R.precompute_cache(m_ser).arrays[u], 1e-4,
                   f"refreshed C mode {u}")


def test_reference_train_loop_on_cuda_plugin(ref):
    """The reference's whole ``train`` (serial) on the CUDA plugin vs on its compiled kernels:
    every epoch's metrics row within 1e-4 (the per-sweep contract) -- the plugin is a drop-in
    for ``_kernels.impl``."""
    import importlib

    RK = importlib.import_module("fastertucker._kernels")
    RT = importlib.import_module("fastertucker.train")

    from paper_2210_06014_b200._kernels import _cudakern

    R = ref
    dims = (50, 40, 30, 20)
    tensor = _tensor(R, dims, 8000, seed=9)
    cfg = RT.TrainConfig(lr_a=0.01, lr_b=0.01, epochs=3)
    m_c = R.default_init_model(dims, (8, 8, 8, 8), 8, seed=1)
    m_g = R.default_init_model(dims, (8, 8, 8, 8), 8, seed=1)
    rows_c = RT.train(m_c, tensor, cfg)
    RK.impl = _cudakern
    try:
        rows_g = RT.train(m_g, tensor, cfg)
    finally:
        RK.impl = RK.get_backend("c")
    for a, b in zip(rows_c, rows_g):
        assert abs(a.train_rmse - b.train_rmse) <= 1e-4 * a.train_rmse
        assert a.multiplies == b.multiplies
    for n in range(4):
        assert_rel(m_g.factors[n], m_c.factors[n], 1e-4, f"A{n}")
        assert_rel(m_g.cores_t[n], m_c.cores_t[n], 1e-4, f"Bt{n}")
