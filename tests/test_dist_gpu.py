"""The sharded epoch with the CUDA engine: two ranks sharing cuda:0 over gloo (NCCL needs one
GPU per rank; the round's GPU tier has one), each sweeping its row blocks with the sm_100a
kernels.  Factors and cores equal the single-GPU exact schedule up to the fp32 order of the
core-gradient sum (the only arithmetic the partition changes); RMSE matches."""

import os
import socket

import numpy as np
import pytest

from helpers import assert_rel, manifest, model_arrays

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, outdir, peer=False, host=False):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2210_06014_b200 as ft
    from paper_2210_06014_b200.dist import DistTrainer

    z = np.load(os.path.join(REPO, "tests", "golden", "cases.npz"))
    case = next(c for c in manifest(z) if c["name"] == "rank32")
    coo = ft.DeviceCoo(tuple(case["dims"]), torch.from_numpy(z["rank32/idx"].astype(np.int32)).cuda(),
                       torch.from_numpy(z["rank32/vals"].astype(np.float32)).cuda())
    f, c = model_arrays(z, "rank32/init/", 3)
    model = ft.Model(tuple(case["dims"]), (32,) * 3, 32, f, c)
    cfg = ft.TrainConfig(**case["cfg"])
    if host:  # each rank copies only its row blocks' entries from host memory
        tr = DistTrainer.from_host(model, tuple(case["dims"]), z["rank32/idx"].astype(np.int32),
                                   z["rank32/vals"].astype(np.float32), cfg, peer_dots=peer)
    else:
        tr = DistTrainer(model, coo, cfg, peer_dots=peer)
    for e in range(case["cfg"]["epochs"]):
        tr.run_epoch(e + 1)
    rmse = tr.evaluate()[0]
    factors = tr.gather_factors()
    if rank == 0:
        np.savez(os.path.join(outdir, "d.npz"), rmse=rmse,
                 **{f"A{n}": factors[n].cpu().numpy() for n in range(3)},
                 **{f"B{n}": model.cores_t[n].cpu().numpy() for n in range(3)})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("peer,host", [(False, False), (True, False), (True, True)],
                         ids=["allgather", "fused-peer-refresh", "host-shards-peer"])
def test_two_ranks_on_one_gpu_equal_single_gpu(tmp_path, golden_cases, peer, host):
    """fused-peer-refresh: ft_refresh_scatter into both ranks' C_u through CUDA IPC, ordered by
    the device-side ft_peer_barrier (no host synchronize / barrier in the epoch);
    host-shards-peer: the same with DistTrainer.from_host (no rank holds the whole COO; training
    RMSE from the mode-0 shard trees, K6b)."""
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(_worker, args=(2, port, str(tmp_path), peer, host), nprocs=2, join=True,
                       start_method="spawn")
    out = np.load(tmp_path / "d.npz")

    import paper_2210_06014_b200 as ft

    z = golden_cases
    case = next(c for c in manifest(z) if c["name"] == "rank32")
    coo = ft.DeviceCoo(tuple(case["dims"]), torch.from_numpy(z["rank32/idx"].astype(np.int32)).cuda(),
                       torch.from_numpy(z["rank32/vals"].astype(np.float32)).cuda())
    f, c = model_arrays(z, "rank32/init/", 3)
    model = ft.Model(tuple(case["dims"]), (32,) * 3, 32, f, c)
    rows = ft.train(model, coo, ft.TrainConfig(**case["cfg"]))
    for n in range(3):
        assert_rel(out[f"A{n}"], model.factors[n].cpu().numpy(), 1e-5, f"A{n}")
        assert_rel(out[f"B{n}"], model.cores_t[n].cpu().numpy(), 1e-5, f"B{n}")
    np.testing.assert_allclose(float(out["rmse"]), rows[-1].train_rmse, rtol=1e-5)
    fr, cr = model_arrays(z, "rank32/final/", 3)
    for n in range(3):
        assert_rel(out[f"A{n}"], fr[n], 1e-4, f"ref A{n}")
