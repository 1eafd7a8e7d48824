"""Multi-GPU FasterTucker epoch: one process per GPU, torch.distributed (NCCL) for plumbing.

FasterTucker is block-coordinate: within the sweep of mode u only A_u (factor sweep) or Bt_u
(core sweep) changes (train.py:3-8).  So the path shards by ROWS OF THE
UPDATED MODE with no stratum rotation:

  * for every mode u the index range [0, I_u) is cut into P contiguous coordinate blocks
    balanced by nonzero count; rank p owns A_u[block p] and the root slices of the tree rooted
    at u whose coordinate falls in block p (a shard of that tree, built from the rank's entries;
    bit-identical to slicing the full tree, since root slices never interact);
  * factor sweep of u: each rank runs the exact row-owner kernel on its shard (conflict-free:
    no row is shared), refreshes C_u on its block, and the blocks are all-gathered
    (I_u x R fp32, 61 MB at Netflix mode 0) -- the only exchange;
  * core sweep of u: each rank reduces its R x J_u gradient partial, one all-reduce of
    R x J_u fp32 (4 KB), every rank applies the identical step, refreshes its C_u block,
    all-gather;
  * evaluate: each rank scores a slice of the entries, all-reduce of (SSE, SAE).

The first factor pass is bitwise equal to the single-GPU exact schedule; afterwards only the
order of the core-gradient sum differs.  With ``peer_dots=True`` the C_u all-gather is fused
into the refresh kernel (ft_refresh_scatter): every rank maps every other rank's C buffers by
CUDA IPC and writes its row block into all of them -- NVLink stores on a multi-GPU node -- then
one barrier.  The compute goes through an ``engine`` (CudaEngine on GPUs; the CPU tests inject
a CPU fp64 reference engine) so the partition / collective logic is tested with gloo.
"""

from __future__ import annotations

import ctypes
import json
import math
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .counter import OpCounter
from .errors import DivergenceError


# ------------------------------------------------------------------------------------------
# partition
# ------------------------------------------------------------------------------------------


def balanced_blocks(counts: np.ndarray, parts: int) -> np.ndarray:
    """Cut [0, len(counts)) into `parts` contiguous blocks with ~equal sums of `counts`.
    Returns the P+1 boundaries c_0 = 0 <= c_1 <= ... <= c_P = len(counts)."""
    counts = np.asarray(counts, dtype=np.int64)
    n = counts.size
    if parts <= 1:
        return np.array([0, n], dtype=np.int64)
    csum = np.cumsum(counts)
    total = int(csum[-1]) if n else 0
    cuts = [0]
    for p in range(1, parts):
        target = total * p / parts
        c = int(np.searchsorted(csum, target, side="left")) + 1
        c = min(max(c, cuts[-1]), n)
        cuts.append(c)
    cuts.append(n)
    return np.asarray(cuts, dtype=np.int64)


@dataclass
class ModeShard:
    """Rank-local state for mode u: the owned coordinate block and the tree shard."""

    mode: int
    c0: int
    c1: int
    tree: object     # engine-specific tree rooted at u restricted to rows in [c0, c1)
    nnz: int
    fibers_t: int    # fibers of the (full) tree rooted at t = u+1 restricted to the block


def plan_blocks(mode_counts: list, world: int) -> list:
    return [balanced_blocks(c, world) for c in mode_counts]


# ------------------------------------------------------------------------------------------
# engines
# ------------------------------------------------------------------------------------------


class CudaEngine:
    """The sm_100a kernels (libft_b200.so) on this rank's GPU."""

    device = "cuda"

    def __init__(self):
        self.L = _lib.lib()

    # -- data -------------------------------------------------------------------------------
    def mode_counts(self, coo, u, I):
        import torch

        return torch.bincount(coo.idx[:, u].long(), minlength=I).cpu().numpy()

    def build_shard(self, coo, u, c0, c1, thr):
        from .coo import DeviceCoo
        from .csf import build_tree

        col = coo.idx[:, u]
        mask = (col >= c0) & (col < c1)
        sub = DeviceCoo(coo.dims, coo.idx[mask].contiguous(), coo.vals[mask].contiguous())
        if sub.nnz == 0:
            return None, 0, 0
        # compact: only the arrays the row-owner kernels read (1 B entries must fit 180 GB / P)
        tree = build_tree(sub, u, thr, compact=True)
        del sub
        return tree, tree.nnz, -1

    # -- compute ----------------------------------------------------------------------------
    def factor_sweep(self, shard, model, dots, lr, reg):
        if shard.tree is None:
            return
        shard.tree.ensure_slots(model.ranks[shard.tree.root_mode], model.core_rank)
        _lib.check(self.L.ft_factor_sweep_rows(ctypes.byref(shard.tree.view()),
                                               ctypes.byref(model.view(dots)), lr, reg,
                                               _lib.stream_handle()), "ft_factor_sweep_rows")

    def core_partial(self, shard, model, dots, u):
        """+sum_i g_i (x) A_u[i] over the shard (R x J_u); acc = -(this, summed)."""
        import torch

        R, J = model.core_rank, model.ranks[u]
        out = torch.zeros((R, J), dtype=torch.float32, device="cuda")
        if shard.tree is None:
            return out
        cap = int(self.L.ft_core_partials_size(R, J))
        parts = torch.empty(cap, dtype=torch.float32, device="cuda")
        nb = ctypes.c_int32(0)
        _lib.check(self.L.ft_core_sweep_rows(ctypes.byref(shard.tree.view()),
                                             ctypes.byref(model.view(dots)), parts.data_ptr(), cap,
                                             ctypes.byref(nb), _lib.stream_handle()),
                   "ft_core_sweep_rows")
        _lib.check(self.L.ft_core_reduce(R, J, parts.data_ptr(), nb.value, out.data_ptr(),
                                         _lib.stream_handle()), "ft_core_reduce")
        return out

    def core_apply(self, model, u, partial_sum, omega, lr, reg, guard):
        R, J = model.core_rank, model.ranks[u]
        _lib.check(self.L.ft_core_apply(R, J, model.cores_t[u].data_ptr(), partial_sum.data_ptr(),
                                        1, 1, float(omega), lr, reg, None, guard.data_ptr(),
                                        _lib.stream_handle()), "ft_core_apply")

    def refresh_scatter(self, model, u, c0, c1, dsts, guard):
        """Fused refresh + all-gather: this rank's C_u rows into every rank's C_u (peer IPC)."""
        if c1 <= c0:
            return
        A, Bt = model.factors[u], model.cores_t[u]
        J, R = A.shape[1], Bt.shape[0]
        tab = (ctypes.c_void_p * len(dsts))(*[d[c0:c1].data_ptr() for d in dsts])
        _lib.check(self.L.ft_refresh_scatter(c1 - c0, J, R, A[c0:c1].data_ptr(), Bt.data_ptr(),
                                             tab, len(dsts),
                                             None if guard is None else guard.data_ptr(),
                                             _lib.stream_handle()), "ft_refresh_scatter")

    def share(self, tensors):
        """CUDA-IPC descriptors of device tensors (torch's own cross-process sharing)."""
        return [t.untyped_storage()._share_cuda_() for t in tensors]

    def open_peer(self, metas, like):
        import torch

        out = []
        for meta, ref in zip(metas, like):
            st = torch.UntypedStorage._new_shared_cuda(*meta)
            t = torch.empty(0, dtype=ref.dtype, device=ref.device)
            t.set_(st, 0, ref.shape, ref.stride())
            out.append(t)
        return out

    def refresh_block(self, model, u, c0, c1, C, guard):
        if c1 <= c0:
            return
        A, Bt = model.factors[u], model.cores_t[u]
        J, R = A.shape[1], Bt.shape[0]
        _lib.check(self.L.ft_refresh(c1 - c0, J, R, A[c0:c1].data_ptr(), Bt.data_ptr(),
                                     C[c0:c1].data_ptr(),
                                     None if guard is None else guard.data_ptr(),
                                     _lib.stream_handle()), "ft_refresh")

    def sse(self, model, dots, coo, lo, hi):
        import torch

        out = torch.zeros(2, dtype=torch.float64, device="cuda")
        if hi > lo:
            idx = coo.idx[lo:hi]
            vals = coo.vals[lo:hi]
            _lib.check(self.L.ft_sse(ctypes.byref(model.view(dots)), hi - lo, idx.data_ptr(),
                                     vals.data_ptr(), out.data_ptr(), _lib.stream_handle()),
                       "ft_sse")
        return out

    def new_guards(self, n):
        import torch

        return torch.zeros(n, dtype=torch.int32, device="cuda")

    def new_flags(self, n):
        import torch

        return torch.zeros(n, dtype=torch.int32, device="cuda")

    def peer_barrier(self, local, peers, rank, seq):
        """Stream-ordered: the next kernels wait on the device for every rank's arrival."""
        tab = (ctypes.c_void_p * len(peers))(*[p.data_ptr() for p in peers])
        _lib.check(self.L.ft_peer_barrier(local.data_ptr(), tab, len(peers), rank,
                                          seq & 0xFFFFFFFF, _lib.stream_handle()),
                   "ft_peer_barrier")

    def sse_tree(self, model, dots, tree):
        """(SSE, SAE) of a shard's entries scored in tree order (K6b); None when the shape is
        outside that kernel's cover."""
        import torch

        from .train import _sse_tree

        if tree is None:
            return torch.zeros(2, dtype=torch.float64, device="cuda")
        return _sse_tree(model, tree, dots)

    def coo_from_host(self, dims, idx, vals):
        """A rank's subset of host entries -> device (H2D from pinned memory when given)."""
        import torch

        from .coo import DeviceCoo

        t_idx = idx if isinstance(idx, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(idx, dtype=np.int32))
        t_val = vals if isinstance(vals, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float32))
        return DeviceCoo(tuple(dims), t_idx.to("cuda", non_blocking=True),
                         t_val.to("cuda", non_blocking=True))

    def synchronize(self):
        import torch

        torch.cuda.synchronize()


# ------------------------------------------------------------------------------------------
# the distributed trainer
# ------------------------------------------------------------------------------------------


class DistTrainer:
    """Row-block sharded FasterTucker epochs over torch.distributed (one rank per GPU).

    ``model``: a Model (replicated; each rank only updates its A_u blocks),
    ``coo``: the full training tensor on every rank (DeviceCoo for the CUDA engine); use
    :meth:`from_host` to give each rank only its row blocks' entries,
    ``cfg``: TrainConfig (exact schedule)."""

    def __init__(self, model, coo, cfg, group=None, engine=None, fiber_threshold=128,
                 peer_dots: bool = False, _parts=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.engine = engine if engine is not None else CudaEngine()
        self.model = model
        self.coo = coo  # None for a host-partitioned trainer (from_host): no rank holds it all
        self.cfg = cfg
        self.N = model.order
        N = self.N
        if _parts is None:
            self.omega = coo.nnz
            counts = [self.engine.mode_counts(coo, u, model.dims[u]) for u in range(N)]
            self.blocks = plan_blocks(counts, self.world)
            subsets = [coo] * N
        else:  # from_host: the blocks and this rank's per-mode entry subsets are given
            self.omega, self.blocks, subsets = _parts
        self.shards = []
        for u in range(N):
            c0, c1 = int(self.blocks[u][self.rank]), int(self.blocks[u][self.rank + 1])
            tree, nnz, ft = self.engine.build_shard(subsets[u], u, c0, c1, fiber_threshold)
            self.shards.append(ModeShard(u, c0, c1, tree, nnz, ft))
        del subsets
        self.dots = self._alloc_dots()
        # peer mode: every rank maps every other rank's C_n buffers and barrier flags (CUDA IPC;
        # NVLink peer memory on a multi-GPU node); the refresh kernel writes its block into all of
        # them and a device-side barrier (ft_peer_barrier) orders the next sweep after every
        # rank's block -- no host synchronize / barrier inside the epoch
        self.peer_dots = None
        if peer_dots and self.world > 1:
            self.flags = self.engine.new_flags(self.world)
            mine = self.dots + [self.flags]
            metas = [None] * self.world
            self.dist.all_gather_object(metas, self.engine.share(mine), group=self.group)
            peer = [mine if q == self.rank else self.engine.open_peer(metas[q], mine)
                    for q in range(self.world)]
            self.peer_dots = [pm[:N] for pm in peer]
            self.peer_flags = [pm[N] for pm in peer]
            self.seq = 0
        for u in range(N):
            self._refresh_and_gather(u, None)
        self.guards = self.engine.new_guards(2 * N)
        self.counter = OpCounter()

    @classmethod
    def from_host(cls, model, dims, idx, vals, cfg, group=None, engine=None,
                  fiber_threshold=128, peer_dots: bool = False):
        """A trainer whose rank copies only the entries of its own row blocks (one subset per
        mode, ~N/P of the tensor) from HOST arrays ``idx`` [nnz x N] / ``vals`` [nnz] (numpy or
        pinned torch tensors), instead of holding the whole COO on its device.  The blocks come
        from host bincounts, identical on every rank."""
        import torch.distributed as dist

        eng = engine if engine is not None else CudaEngine()
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        idx_np = idx.numpy() if hasattr(idx, "numpy") else np.asarray(idx)
        vals_np = vals.numpy() if hasattr(vals, "numpy") else np.asarray(vals)
        N = idx_np.shape[1]
        blocks = plan_blocks([np.bincount(idx_np[:, u], minlength=dims[u]) for u in range(N)],
                             world)
        subsets = []
        for u in range(N):
            c0, c1 = int(blocks[u][rank]), int(blocks[u][rank + 1])
            sel = np.flatnonzero((idx_np[:, u] >= c0) & (idx_np[:, u] < c1))
            subsets.append(eng.coo_from_host(dims, idx_np[sel], vals_np[sel]))
        return cls(model, None, cfg, group=group, engine=eng, fiber_threshold=fiber_threshold,
                   peer_dots=peer_dots, _parts=(int(idx_np.shape[0]), blocks, subsets))

    # -- helpers ------------------------------------------------------------------------------
    def _alloc_dots(self):
        import torch

        dev = self.engine.device
        dt = self.model.factors[0].dtype
        return [torch.zeros((self.model.dims[n], self.model.core_rank), dtype=dt, device=dev)
                for n in range(self.N)]

    def _refresh_and_gather(self, u, guard):
        """C_u on this rank's block, then all-gather the blocks (padded to equal size)."""
        import torch

        b = self.blocks[u]
        if self.peer_dots is not None:
            self.engine.refresh_scatter(self.model, u, int(b[self.rank]), int(b[self.rank + 1]),
                                        [pd[u] for pd in self.peer_dots], guard)
            # every block landed before anyone reads C_u: a device-side barrier on the stream
            self.seq += 1
            self.engine.peer_barrier(self.flags, self.peer_flags, self.rank, self.seq)
            return
        self.engine.refresh_block(self.model, u, int(b[self.rank]), int(b[self.rank + 1]),
                                  self.dots[u], guard)
        if self.world == 1:
            return
        sizes = np.diff(b)
        m = int(sizes.max())
        R = self.model.core_rank
        send = torch.zeros((m, R), dtype=self.dots[u].dtype, device=self.dots[u].device)
        mine = int(sizes[self.rank])
        if mine:
            send[:mine] = self.dots[u][int(b[self.rank]):int(b[self.rank + 1])]
        recv = [torch.empty_like(send) for _ in range(self.world)]
        self.dist.all_gather(recv, send, group=self.group)
        for p in range(self.world):
            if p != self.rank and sizes[p]:
                self.dots[u][int(b[p]):int(b[p + 1])] = recv[p][:int(sizes[p])]

    def _check_guards(self, limit):
        import torch

        g = self.guards.clone()
        if self.world > 1:
            self.dist.all_reduce(g, op=self.dist.ReduceOp.MAX, group=self.group)
        words = g.cpu().numpy().view(np.uint32)
        lim = int(np.array([min(limit, 3.4028234663852886e38)], np.float32).view(np.uint32)[0])
        order = [(n, (n + self.N - 1) % self.N) for n in range(self.N)]
        for k in range(2 * self.N):
            if int(words[k]) > lim:
                raise DivergenceError(f"{'factor' if k < self.N else 'core'} mode "
                                      f"{order[k % self.N][1]} diverged", mode=order[k % self.N][1])

    # -- the epoch ----------------------------------------------------------------------------
    def factor_pass(self):
        cfg, N = self.cfg, self.N
        for n in range(N):
            u = (n + N - 1) % N
            self.engine.factor_sweep(self.shards[u], self.model, self.dots, cfg.lr_a, cfg.reg_a)
            self._refresh_and_gather(u, self.guards[n:n + 1])

    def core_pass(self):
        cfg, N = self.cfg, self.N
        for n in range(N):
            u = (n + N - 1) % N
            part = self.engine.core_partial(self.shards[u], self.model, self.dots, u)
            if self.world > 1:
                self.dist.all_reduce(part, group=self.group)
            self.engine.core_apply(self.model, u, part, self.omega, cfg.lr_b, cfg.reg_b,
                                   self.guards[N + n:N + n + 1])
            self._refresh_and_gather(u, None)

    def run_epoch(self, epoch_no: int = 1):
        self.guards.zero_()
        try:
            self.factor_pass()
            self.core_pass()
            self._check_guards(self.cfg.divergence_limit)
        except DivergenceError as exc:
            raise DivergenceError(f"divergence at epoch {epoch_no}, mode {exc.mode}",
                                  mode=exc.mode, epoch=epoch_no) from None

    def evaluate(self, coo=None):
        """(RMSE, MAE) of ``coo`` (entries split by index across ranks), or of the training
        entries: every rank scores its mode-0 shard in tree order (the mode-0 row blocks
        partition the entries), so no rank needs the full training COO."""
        out = None
        if coo is None and hasattr(self.engine, "sse_tree"):
            out = self.engine.sse_tree(self.model, self.dots, self.shards[0].tree)
        if out is not None:
            if self.world > 1:
                self.dist.all_reduce(out, group=self.group)
            sse, sae = (float(v) for v in out.cpu().numpy())
            return math.sqrt(sse / self.omega), sae / self.omega
        coo = coo if coo is not None else self.coo
        if coo is None:
            raise ValueError("evaluate: this shape needs the training COO (K6b does not cover it)")
        n = coo.nnz
        lo = n * self.rank // self.world
        hi = n * (self.rank + 1) // self.world
        out = self.engine.sse(self.model, self.dots, coo, lo, hi)
        if self.world > 1:
            self.dist.all_reduce(out, group=self.group)
        sse, sae = (float(v) for v in out.cpu().numpy())
        return math.sqrt(sse / n), sae / n

    def gather_factors(self):
        """Full A_n on every rank (for checkpoints): all-gather the owned row blocks."""
        import torch

        if self.world == 1:
            return [a.clone() for a in self.model.factors]
        out = []
        for u in range(self.N):
            b = self.blocks[u]
            sizes = np.diff(b)
            m = int(sizes.max())
            A = self.model.factors[u]
            send = torch.zeros((m, A.shape[1]), dtype=A.dtype, device=A.device)
            mine = int(sizes[self.rank])
            if mine:
                send[:mine] = A[int(b[self.rank]):int(b[self.rank + 1])]
            recv = [torch.empty_like(send) for _ in range(self.world)]
            self.dist.all_gather(recv, send, group=self.group)
            full = A.clone()
            for p in range(self.world):
                if sizes[p]:
                    full[int(b[p]):int(b[p + 1])] = recv[p][:int(sizes[p])]
            out.append(full)
        return out


# ------------------------------------------------------------------------------------------
# bench.py --gpus N (torchrun): strong scaling of the same workload
# ------------------------------------------------------------------------------------------


def bench_distributed(args, cfg, rank, world):
    import torch
    import torch.distributed as dist

    from .coo import generate_synthetic
    from .model import default_init_model
    from .train import TrainConfig

    dims, J, R = cfg["dims"], cfg["J"], cfg["R"]
    N = len(dims)
    nnz_total = cfg["nnz_train"] + cfg["nnz_test"]
    split = generate_synthetic(dims, nnz_total, cfg["value_range"], seed=0,
                               test_fraction=cfg["nnz_test"] / nnz_total)
    model = default_init_model(dims, (J,) * N, R, seed=0)
    tcfg = TrainConfig(epochs=1)
    # the training entries go to host memory once (a sharded loader's view); every rank then
    # copies only its row blocks' entries (DistTrainer.from_host), no rank holds the whole COO
    idx_h = split.train.idx.cpu().pin_memory()
    vals_h = split.train.vals.cpu().pin_memory()
    nnz = split.train.nnz
    del split.train
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    # fused refresh + all-gather over peer memory (NVLink) by default; FT_PEER=0: NCCL all-gather
    peer = os.environ.get("FT_PEER", "1") == "1"
    trainer = DistTrainer.from_host(model, dims, idx_h, vals_h, tcfg, peer_dots=peer)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    clocks = None
    if rank == 0:
        import bench as _bench  # the driver's bench module (repo root): its nvidia-smi sampler

        clocks = _bench.Clocks(int(os.environ.get("LOCAL_RANK", "0")))
        clocks.start()
    for k in range(args.warmup):
        trainer.run_epoch(k + 1)
    torch.cuda.synchronize()
    dist.barrier()
    if clocks is not None:
        clocks.begin()
    start, mid, stop = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    fsum = 0.0
    start.record()
    for k in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        trainer.factor_pass()
        b.record()
        trainer.core_pass()
        b.synchronize()
        fsum += a.elapsed_time(b)
    stop.record()
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks is not None else None
    dist.barrier()
    mine = torch.tensor([start.elapsed_time(stop) / 1e3, fsum / 1e3], dtype=torch.float64,
                        device="cuda")
    dist.all_reduce(mine, op=dist.ReduceOp.MAX)
    total_s, f_s = (float(v) for v in mine.cpu().numpy())
    tr = trainer.evaluate()
    te = trainer.evaluate(split.test)
    init = default_init_model(dims, (J,) * N, R, seed=0)
    del trainer
    e2e = _e2e_distributed(dims, idx_h, vals_h, init, tcfg, rank, world, args, peer)
    if rank == 0:
        line = {
            "metric": "nonzeros/sec per SGD epoch (factor update, core update)",
            "value": nnz * args.steps / total_s, "unit": "nnz/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total_s / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (GPU generator: distinct uniform cells, U[1,5]; random init)",
            "config": {"workload": args.config, "dims": list(dims), "nnz_train": nnz, "J": J,
                       "R": R, "schedule": "exact", "parallelism": f"row-block x{world}",
                       "l2": "inputs larger than L2"},
            "factor_ms": 1e3 * f_s / args.steps,
            "train_rmse": tr[0], "test_rmse": te[0], "setup_s": setup_s,
            "gpu_launches": (6 * N) * args.steps,
            "e2e": e2e, "roofline": None, "cpu_baseline": None, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def _e2e_distributed(dims, idx_h, vals_h, init, tcfg, rank, world, args, peer):
    """The N-GPU end-to-end step through the public API: every rank copies ITS row blocks'
    entries (one subset per mode, ~N/P of the tensor, host-partitioned once as a sharded loader
    would deliver them) from pinned host memory, builds its shards, runs one epoch and reads the
    training RMSE back (all-reduced).  CUDA events on each rank, max over ranks."""
    import torch
    import torch.distributed as dist

    from .model import Model

    idx_np, vals_np = idx_h.numpy(), vals_h.numpy()
    N = len(dims)
    blocks = plan_blocks([np.bincount(idx_np[:, u], minlength=dims[u]) for u in range(N)], world)
    mine = []
    for u in range(N):
        c0, c1 = int(blocks[u][rank]), int(blocks[u][rank + 1])
        sel = np.flatnonzero((idx_np[:, u] >= c0) & (idx_np[:, u] < c1))
        mine.append((torch.from_numpy(idx_np[sel]).pin_memory(),
                     torch.from_numpy(vals_np[sel]).pin_memory()))
    h2d = sum(int(i.numel()) * 4 + int(v.numel()) * 4 for i, v in mine)
    eng = CudaEngine()
    steps = max(1, min(args.steps, 2))

    def step():
        subsets = [eng.coo_from_host(dims, i, v) for i, v in mine]
        m = Model(init.dims, init.ranks, init.core_rank, [a.clone() for a in init.factors],
                  [b.clone() for b in init.cores_t])
        tr = DistTrainer(m, None, tcfg, engine=eng, peer_dots=peer,
                         _parts=(int(idx_np.shape[0]), blocks, subsets))
        del subsets
        tr.run_epoch(1)
        return tr.evaluate()[0]

    step()  # warm-up (allocator pools, IPC mappings)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    mine_t = torch.tensor([a.elapsed_time(b) / 1e3 / steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(mine_t, op=dist.ReduceOp.MAX)
    t = float(mine_t.item())
    nnz = int(idx_np.shape[0])
    return {"value": nnz / t, "unit": "nnz/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": 16, "ms_per_step": 1e3 * t, "steps": steps,
            "includes": "per rank: H2D of its row blocks' entries (pinned, one subset per mode) "
                        "+ shard build + cache + one epoch + training RMSE all-reduce / readback"}
