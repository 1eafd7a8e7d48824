"""Multi-process (world size 2, gloo, CPU) test of the row-block sharded epoch
(paper_2210_06014_b200.dist): partition, C_u block all-gather, core-gradient all-reduce,
guards and evaluation -- with the fp64 oracle as the compute engine, so the result must equal
the single-process serial reference: factors bitwise, cores to the summation order."""

import os
import socket

import numpy as np
import pytest

from helpers import manifest, model_arrays

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class HostCoo:
    def __init__(self, dims, idx, vals):
        self.dims = tuple(dims)
        self.idx = np.ascontiguousarray(idx, dtype=np.int64)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)

    @property
    def nnz(self):
        return self.idx.shape[0]

    @property
    def order(self):
        return len(self.dims)


class HostModel:
    """Model-shaped holder of torch CPU fp64 tensors (the oracle engine's parameters)."""

    def __init__(self, factors, cores):
        import torch

        self.factors = [torch.from_numpy(np.array(a)) for a in factors]
        self.cores_t = [torch.from_numpy(np.array(b)) for b in cores]
        self.dims = tuple(a.shape[0] for a in factors)
        self.ranks = tuple(a.shape[1] for a in factors)
        self.core_rank = cores[0].shape[0]

    @property
    def order(self):
        return len(self.dims)


class OracleEngine:
    """dist.DistTrainer engine backed by the fp64 oracle (test infrastructure only)."""

    device = "cpu"

    def __init__(self):
        from oracle import oracle as O

        self.O = O

    def mode_counts(self, coo, u, I):
        return np.bincount(coo.idx[:, u], minlength=I)

    def build_shard(self, coo, u, c0, c1, thr):
        sel = (coo.idx[:, u] >= c0) & (coo.idx[:, u] < c1)
        if not sel.any():
            return None, 0, 0
        t = (u + 1) % coo.order
        tree = self.O.build_tree(coo.idx[sel], coo.vals[sel], t, thr)
        return tree, int(sel.sum()), tree.num_fibers

    def _np(self, ts):
        return [x.numpy() for x in ts]

    def factor_sweep(self, shard, model, dots, lr, reg):
        if shard.tree is None:
            return
        t = shard.tree
        self.O.CKernels.factor_sweep(t.leaf_coord, t.vals, t.fiber_ptr, t.fiber_coord,
                                     t.prefix_modes, t.leaf_mode, self._np(model.factors),
                                     self._np(model.cores_t), self._np(dots), lr, reg,
                                     np.zeros(5, np.int64), 0, t.num_fibers)

    def core_partial(self, shard, model, dots, u):
        import torch

        acc = np.zeros((model.core_rank, model.ranks[u]))
        if shard.tree is not None:
            t = shard.tree
            self.O.CKernels.core_sweep(t.leaf_coord, t.vals, t.fiber_ptr, t.fiber_coord,
                                       t.prefix_modes, t.leaf_mode, self._np(model.factors),
                                       self._np(model.cores_t), self._np(dots), acc,
                                       np.zeros(5, np.int64), 0, t.num_fibers)
        return torch.from_numpy(-acc)  # the CUDA engine's convention: +G^T A

    def core_apply(self, model, u, partial_sum, omega, lr, reg, guard):
        B = model.cores_t[u].numpy()
        self.O.CKernels.apply_core_update(B, -partial_sum.numpy(), float(omega), lr, reg,
                                          np.zeros(5, np.int64))
        self._guard(guard, B)

    def _guard(self, guard, arr):
        if guard is None or arr.size == 0:
            return
        bits = int(np.array([np.abs(arr).max()], np.float32).view(np.int32)[0])
        guard[0] = max(int(guard[0]), bits)

    def refresh_block(self, model, u, c0, c1, C, guard):
        if c1 <= c0:
            return
        A = model.factors[u].numpy()[c0:c1]
        out = C.numpy()[c0:c1]
        self.O.CKernels.refresh_dot_mode(np.ascontiguousarray(A), model.cores_t[u].numpy(), out,
                                         np.zeros(5, np.int64))
        self._guard(guard, A)

    def sse(self, model, dots, coo, lo, hi):
        import ctypes

        import torch

        O = self.O
        idx = np.ascontiguousarray(coo.idx[lo:hi])
        pred = np.empty(hi - lo)
        if hi > lo:
            tab = (ctypes.POINTER(ctypes.c_double) * model.order)(
                *[d.numpy().ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for d in dots])
            O.lib().fto_predict(model.order, model.core_rank, hi - lo,
                                idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), tab,
                                pred.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        r = coo.vals[lo:hi] - pred
        return torch.tensor([float(r @ r), float(np.abs(r).sum())], dtype=torch.float64)

    def new_guards(self, n):
        import torch

        return torch.zeros(n, dtype=torch.int32)

    def coo_from_host(self, dims, idx, vals):
        return HostCoo(dims, np.asarray(idx, dtype=np.int64), np.asarray(vals, dtype=np.float64))

    def synchronize(self):
        pass


def _worker(rank, world, port, case_name, epochs, outdir, host=False):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2210_06014_b200.dist import DistTrainer
    from paper_2210_06014_b200.train import TrainConfig

    z = np.load(os.path.join(REPO, "tests", "golden", "cases.npz"))
    case = next(c for c in manifest(z) if c["name"] == case_name)
    key = case_name + "/"
    N = len(case["dims"])
    coo = HostCoo(case["dims"], z[key + "idx"], z[key + "vals"])
    f, c = model_arrays(z, key + "init/", N)
    model = HostModel(f, c)
    kw = {k: v for k, v in case["cfg"].items() if k in ("lr_a", "lr_b", "reg_a", "reg_b")}
    cfg = TrainConfig(**kw)
    thr = case["cfg"].get("fiber_threshold", 128)
    if host:  # each rank receives only its row blocks' entries
        tr = DistTrainer.from_host(model, case["dims"], coo.idx, coo.vals, cfg,
                                   engine=OracleEngine(), fiber_threshold=thr)
    else:
        tr = DistTrainer(model, coo, cfg, engine=OracleEngine(), fiber_threshold=thr)
    rmse = []
    for e in range(epochs):
        tr.run_epoch(e + 1)
        rmse.append(tr.evaluate(coo)[0])
    factors = tr.gather_factors()
    if rank == 0:
        np.savez(os.path.join(outdir, "dist.npz"), rmse=np.array(rmse),
                 blocks=np.concatenate(tr.blocks),
                 **{f"A{n}": factors[n].numpy() for n in range(N)},
                 **{f"B{n}": model.cores_t[n].numpy() for n in range(N)})
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("case_name,epochs,host", [("rank16", 2, False), ("order5", 2, False),
                                                   ("rank16", 2, True)])
def test_row_block_sharding_equals_serial_reference(tmp_path, golden_cases, case_name, epochs,
                                                    host):
    """host=True: DistTrainer.from_host, every rank holding only its row blocks' entries."""
    import torch.multiprocessing as mp

    mp.start_processes(_worker, args=(2, _free_port(), case_name, epochs, str(tmp_path), host),
                       nprocs=2, join=True, start_method="spawn")
    out = np.load(tmp_path / "dist.npz")
    z = golden_cases
    case = next(c for c in manifest(z) if c["name"] == case_name)
    N = len(case["dims"])
    # the golden "final" model is the reference after cfg["epochs"] epochs (== epochs here)
    assert case["cfg"]["epochs"] == epochs
    f, c = model_arrays(z, case_name + "/final/", N)
    for n in range(N):
        assert np.array_equal(out[f"A{n}"], f[n]) or np.allclose(out[f"A{n}"], f[n], rtol=1e-12,
                                                                   atol=1e-15), f"A{n}"
        np.testing.assert_allclose(out[f"B{n}"], c[n], rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(out["rmse"], z[case_name + "/metrics"][:epochs, 1], rtol=1e-10)
    b = out["blocks"].reshape(N, 3)
    assert (b[:, 0] == 0).all() and (b[:, 2] == np.array(case["dims"])).all()


def test_balanced_blocks_properties():
    from paper_2210_06014_b200.dist import balanced_blocks

    rng = np.random.default_rng(0)
    for parts in (1, 2, 3, 8):
        counts = rng.poisson(50, size=997)
        b = balanced_blocks(counts, parts)
        assert b[0] == 0 and b[-1] == counts.size and (np.diff(b) >= 0).all()
        sums = np.add.reduceat(counts, b[:-1]) if parts > 1 else [counts.sum()]
        assert max(sums) <= counts.sum() / parts + counts.max() + 1
    b = balanced_blocks(np.array([0, 0, 100, 0]), 4)
    assert b[0] == 0 and b[-1] == 4
