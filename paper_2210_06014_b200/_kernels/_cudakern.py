"""The reference's kernel-plugin entry points over host numpy buffers, run on the B200.

Same names, argument order and in-place semantics as ``_ckern`` / ``_pykern``
(/root/reference/pkg/src/fastertucker/_kernels/_ckern.pyx:21-282):

  refresh_dot_mode(A, B_t, out, counts)
  factor_sweep(leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes, leaf_mode,
               factors, cores_t, dots, lr, reg, counts, fib_lo, fib_hi)
  core_sweep(leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes, leaf_mode,
             factors, cores_t, dots, acc, counts, fib_lo, fib_hi)
  apply_core_update(core_t_u, acc, omega, lr, reg, counts)

This is the CONVENIENCE boundary for code written against the reference's ``impl`` module:
every call uploads its operands (fp64 -> fp32), runs the sm_100a kernels and writes results
back in place.  The sweeps over a fiber range [fib_lo, fib_hi) of the tree rooted at
t = (leaf_mode + 1) mod N are executed exactly: the range's entries are re-indexed on the GPU
as a tree rooted at the leaf mode (kernel K1), whose root slices are the rows' update lists in
the serial order, and swept by the row-owner kernels K3b / K4.  The throughput path is the
device-resident API in :mod:`paper_2210_06014_b200.train` (no copies).

Concurrency (the reference's ``workers > 1`` pool, train.py:124-149, calls ``factor_sweep`` /
``core_sweep`` from several threads on different subtensor ranges over the shared host
``factors[u]``): each call holds a module lock from upload to write-back, so every call starts
from the rows the previous calls wrote, and ``factor_sweep`` writes back only the rows of A_u
its range touched -- other rows keep their host (fp64) values bit for bit.  The calls thus
run as some serial order of the subtensors, never losing a whole range of updates.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from .. import _lib
from ..counter import CH_DOT, apply_counts, sweep_counts

BACKEND = "cuda"

# one plugin call at a time: upload -> sweep -> write-back is atomic w.r.t. other workers
_CALL_LOCK = threading.RLock()


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _model_view(factors, cores_t, dots_dev):
    v = _lib.FtModel()
    N = len(factors)
    v.order = N
    v.core_rank = cores_t[0].shape[0]
    for n in range(N):
        v.dims[n] = factors[n].shape[0]
        v.ranks[n] = factors[n].shape[1]
        v.factors[n] = factors[n].data_ptr()
        v.cores_t[n] = cores_t[n].data_ptr()
        v.dots[n] = dots_dev[n].data_ptr() if dots_dev[n] is not None else None
    return v


def refresh_dot_mode(A, B_t, out, counts):
    """out[i, r] = A[i] . B_t[r] (K2)."""
    import torch

    L = _lib.lib()
    I, J = A.shape
    R = B_t.shape[0]
    with _CALL_LOCK:
        dA, dB = _dev(A), _dev(B_t)
        dC = torch.empty((I, R), dtype=torch.float32, device="cuda")
        _lib.check(L.ft_refresh(I, J, R, dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), None,
                                _lib.stream_handle()), "ft_refresh")
        out[...] = dC.cpu().numpy()
    counts[CH_DOT] += I * J * R


def _range_as_tree(leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes, leaf_mode, N,
                   dims, fib_lo, fib_hi):
    """The entries of fibers [fib_lo, fib_hi) re-indexed as a tree rooted at leaf_mode."""
    from ..coo import DeviceCoo
    from ..csf import build_tree

    fp = np.asarray(fiber_ptr, dtype=np.int64)
    lo, hi = int(fp[fib_lo]), int(fp[fib_hi])
    nleaf = hi - lo
    if nleaf == 0:
        return None, 0
    fib_of_leaf = np.repeat(np.arange(fib_lo, fib_hi), np.diff(fp[fib_lo:fib_hi + 1]))
    idx = np.empty((nleaf, N), dtype=np.int32)
    fc = np.asarray(fiber_coord)
    for d, m in enumerate(np.asarray(prefix_modes, dtype=np.int64)):
        idx[:, int(m)] = fc[fib_of_leaf, d]
    idx[:, int(leaf_mode)] = np.asarray(leaf_coord)[lo:hi]
    import torch

    dev = DeviceCoo(tuple(int(d) for d in dims), torch.from_numpy(idx).cuda(),
                    _dev(np.asarray(leaf_val)[lo:hi]))
    return build_tree(dev, int(leaf_mode), None), nleaf


def _dots_dev(factors_d, cores_d, dots):
    import torch

    L = _lib.lib()
    out = []
    for n in range(len(factors_d)):
        if dots is not None:
            out.append(_dev(dots[n]))
            continue
        A, B = factors_d[n], cores_d[n]
        C = torch.empty((A.shape[0], B.shape[0]), dtype=torch.float32, device="cuda")
        _lib.check(L.ft_refresh(A.shape[0], A.shape[1], B.shape[0], A.data_ptr(), B.data_ptr(),
                                C.data_ptr(), None, _lib.stream_handle()), "ft_refresh")
        out.append(C)
    return out


def factor_sweep(leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes, leaf_mode, factors,
                 cores_t, dots, lr, reg, counts, fib_lo, fib_hi):
    L = _lib.lib()
    N = len(factors)
    u = int(leaf_mode)
    dims = [a.shape[0] for a in factors]
    tree, nleaf = _range_as_tree(leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes, u,
                                 N, dims, fib_lo, fib_hi)
    R = cores_t[0].shape[0]
    ranks = [a.shape[1] for a in factors]
    plan = "cached" if dots is not None else "uncached"
    counts += sweep_counts("factor", plan, N, R, ranks, prefix_modes, u, nleaf, fib_hi - fib_lo)
    if tree is None:
        return
    fp = np.asarray(fiber_ptr, dtype=np.int64)
    rows = np.unique(np.asarray(leaf_coord)[int(fp[fib_lo]):int(fp[fib_hi])])
    with _CALL_LOCK:
        fd = [_dev(a) for a in factors]
        cd = [_dev(b) for b in cores_t]
        dd = _dots_dev(fd, cd, dots)
        mv = _model_view(fd, cd, dd)
        _lib.check(L.ft_factor_sweep_rows(ctypes.byref(tree.view()), ctypes.byref(mv), float(lr),
                                          float(reg), _lib.stream_handle()),
                   "ft_factor_sweep_rows")
        import torch

        factors[u][rows] = fd[u][torch.from_numpy(rows).cuda()].cpu().numpy()


def core_sweep(leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes, leaf_mode, factors,
               cores_t, dots, acc, counts, fib_lo, fib_hi):
    import torch

    L = _lib.lib()
    N = len(factors)
    u = int(leaf_mode)
    dims = [a.shape[0] for a in factors]
    tree, nleaf = _range_as_tree(leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes, u,
                                 N, dims, fib_lo, fib_hi)
    R = cores_t[0].shape[0]
    ranks = [a.shape[1] for a in factors]
    plan = "cached" if dots is not None else "uncached"
    counts += sweep_counts("core", plan, N, R, ranks, prefix_modes, u, nleaf, fib_hi - fib_lo)
    if tree is None:
        return
    with _CALL_LOCK:
        fd = [_dev(a) for a in factors]
        cd = [_dev(b) for b in cores_t]
        dd = _dots_dev(fd, cd, dots)
        # s = C_u[i] . cross needs C_u coherent with (A_u, Bt_u): compute it fresh
        dd[u] = _dots_dev([fd[u]], [cd[u]], None)[0]
        mv = _model_view(fd, cd, dd)
        Ju = ranks[u]
        cap = int(L.ft_core_partials_size(R, Ju))
        partials = torch.empty(cap, dtype=torch.float32, device="cuda")
        nb = ctypes.c_int32(0)
        _lib.check(L.ft_core_sweep_rows(ctypes.byref(tree.view()), ctypes.byref(mv),
                                        partials.data_ptr(), cap, ctypes.byref(nb),
                                        _lib.stream_handle()), "ft_core_sweep_rows")
        g = torch.empty((R, Ju), dtype=torch.float32, device="cuda")
        _lib.check(L.ft_core_reduce(R, Ju, partials.data_ptr(), nb.value, g.data_ptr(),
                                    _lib.stream_handle()), "ft_core_reduce")
        acc[...] -= g.cpu().numpy()


def apply_core_update(core_t_u, acc, omega, lr, reg, counts):
    L = _lib.lib()
    R, J = core_t_u.shape
    with _CALL_LOCK:
        dB, dA = _dev(core_t_u), _dev(acc)
        _lib.check(L.ft_core_apply(R, J, dB.data_ptr(), dA.data_ptr(), 1, 0, float(omega),
                                   float(lr), float(reg), None, None, _lib.stream_handle()),
                   "ft_core_apply")
        core_t_u[...] = dB.cpu().numpy()
    counts += apply_counts(R, J)
