"""Parity at the benchmarked scale: Netflix-dims tensors with 10 M training entries, J = R = 32,
the reference's default hyper-parameters (lr 1e-3, reg 1e-2, threshold 128), against the
reference's own compiled kernels (oracle/_ref ``_ckern``; our C restatement when _ref is absent)
run over all host cores by ``oracle.RowParallelRef`` (bitwise the serial factor sweeps, see its
docstring; pinned by tests/test_oracle.py::test_row_parallel_reference_is_the_serial_epoch).

Contract (BASELINE.json north_star):
  * exact schedule: every sweep of epoch 1 (factor A_u, core Bt_u) at rel 1e-4
    (Frobenius and max-abs / max|ref|), and the model after epoch 3 at rel 1e-4;
  * train / test RMSE after 3 epochs within 1 % -- for the exact schedule AND for hogwild;
  * one tensor has the Netflix dims (480,189 x 17,770 x 2,182; 4.6 K updates per mode-2 row at
    10 M entries), the other shrinks mode 2 to 218 rows so that every mode-2 row carries
    ~46 K serial updates -- the regime of the full 99 M Netflix tensor's mode 2 (45.4 K), where
    fp32 drift would compound.
Reference paths: train.py:152-278 (sweeps, epoch), train.py:91-98 (evaluate), train.py:306-336
(train), SPEC.md:439 (hogwild fidelity).
"""

import time

import numpy as np
import pytest

from helpers import rel_errors

pytestmark = pytest.mark.gpu

TOL = 1e-4
RMSE_TOL = 0.01
NNZ = 10_000_000
NTEST = 140_000
EPOCHS = 3


@pytest.fixture(scope="module")
def ft():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2210_06014_b200 as ft

    return ft


def _inputs(ft, dims, seed):
    """Distinct uniform cells (GPU generator, the reference generator's distribution,
    coo.py:164-178), split into train / test; host copies for the reference."""
    t = ft.generate_device(dims, NNZ + NTEST, (1.0, 5.0), seed=seed)
    idx = t.idx.cpu().numpy().astype(np.int64)
    vals = t.vals.cpu().numpy().astype(np.float64)   # the fp32 values the GPU sees, widened
    return idx[:NNZ], vals[:NNZ], idx[NNZ:], vals[NNZ:]


def _dev(ft, dims, idx, vals):
    import torch

    return ft.DeviceCoo(tuple(dims), torch.from_numpy(idx.astype(np.int32)).cuda(),
                        torch.from_numpy(vals.astype(np.float32)).cuda())


def _check(got, ref, what, log):
    fro, mx = rel_errors(got, ref)
    log.append(f"{what}: fro {fro:.2e} max {mx:.2e}")
    assert fro <= TOL and mx <= TOL, f"{what}: rel fro {fro:.3e} max {mx:.3e} > {TOL:g}"


@pytest.mark.parametrize("dims", [(480_189, 17_770, 2_182), (480_189, 17_770, 218)],
                         ids=["netflix_dims", "long_rows_46k"])
def test_netflix_scale_exact_and_hogwild_vs_reference(ft, dims):
    from oracle import oracle as O

    t0 = time.perf_counter()
    log = []
    idx, vals, tidx, tvals = _inputs(ft, dims, seed=7)
    ranks = (32, 32, 32)
    om = O.default_init_model(dims, ranks, 32, seed=0)
    init_f = [a.copy() for a in om.factors]
    init_c = [b.copy() for b in om.cores_t]
    ref = O.RowParallelRef(idx, vals, dims)
    ocfg = O.OracleConfig()
    ocache = O.precompute_cache(om, ref.K)
    log.append(f"reference kernels: {getattr(ref.K, 'BACKEND', ref.K.__name__)} x {ref.T} threads"
               f" (setup {time.perf_counter() - t0:.1f} s)")

    train = _dev(ft, dims, idx, vals)
    test = _dev(ft, dims, tidx, tvals)
    forest = ft.build_forest(train, 128)
    model = ft.Model(dims, ranks, 32, init_f, init_c)
    cfg = ft.TrainConfig()
    cache = ft.precompute_cache(model)
    for epoch in range(1, EPOCHS + 1):
        for n in range(3):
            ref.update_factor_mode(om, ocache, n, ocfg)
            ft.update_factor_mode(model, forest, cache, n, cfg)
            if epoch == 1:
                u = forest.trees[n].leaf_mode
                _check(model.factors[u].cpu().numpy(), om.factors[u], f"e1 factor {u}", log)
        for n in range(3):
            ref.update_core_mode(om, ocache, n, ocfg)
            ft.update_core_mode(model, forest, cache, n, cfg)
            if epoch == 1:
                u = forest.trees[n].leaf_mode
                _check(model.cores_t[u].cpu().numpy(), om.cores_t[u], f"e1 core {u}", log)
    ref.close()
    for n in range(3):
        _check(model.factors[n].cpu().numpy(), om.factors[n], f"e{EPOCHS} A{n}", log)
        _check(model.cores_t[n].cpu().numpy(), om.cores_t[n], f"e{EPOCHS} Bt{n}", log)
    ref_train = O.evaluate(om, idx, vals)[0]
    ref_test = O.evaluate(om, tidx, tvals)[0]
    got_train = ft.evaluate(model, train, cache, forest)[0]
    got_test = ft.evaluate(model, test, cache)[0]
    log.append(f"e{EPOCHS} rmse ref {ref_train:.7f}/{ref_test:.7f} exact {got_train:.7f}/"
               f"{got_test:.7f}")
    assert abs(got_train - ref_train) / ref_train < RMSE_TOL
    assert abs(got_test - ref_test) / ref_test < RMSE_TOL

    # hogwild (the reference's workers > 1): racing lock-free row updates on the GPU
    hmodel = ft.Model(dims, ranks, 32, init_f, init_c)
    rows = ft.train(hmodel, train, ft.TrainConfig(epochs=EPOCHS, schedule="hogwild"), test,
                    forest=forest)
    h_train, h_test = rows[-1].train_rmse, rows[-1].test_rmse
    log.append(f"e{EPOCHS} rmse hogwild {h_train:.7f}/{h_test:.7f} "
               f"(rel {abs(h_train - ref_train) / ref_train:.2e} / "
               f"{abs(h_test - ref_test) / ref_test:.2e}); total {time.perf_counter() - t0:.0f} s")
    print("\n".join(log))
    assert abs(h_train - ref_train) / ref_train < RMSE_TOL
    assert abs(h_test - ref_test) / ref_test < RMSE_TOL
