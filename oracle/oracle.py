"""TEST INFRASTRUCTURE ONLY -- the CPU parity checker for the FasterTucker hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import this module.  The product package never does.

Two CPU implementations live behind one driver:

* ``libft_oracle.so`` -- our fp64 C restatement (``oracle/ft_oracle.c``) of the reference's
  build_tree / refresh_dot_mode / factor_sweep / core_sweep / apply_core_update /
  predict_batch, bit-identical to the reference (pinned against ``tests/golden``).
* ``oracle/_ref/_ckern*.so`` -- the reference's OWN Cython kernel module compiled from
  /root/reference (``make -C oracle ref``).  When present it is used as the reference arm.

The epoch driver below restates the reference trainer (paths relative to
/root/reference/pkg/src/fastertucker/): ``update_factor_mode`` (train.py:152-197),
``update_core_mode`` (train.py:200-248), ``run_epoch`` (train.py:251-278), ``evaluate``
(train.py:91-98), the hogwild subtensor queue (train.py:124-149) and the divergence guards
(train.py:101-110).
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import math
import os
import subprocess
import threading
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build(quiet: bool = True) -> None:
    """Compile the oracle (and oracle/_ref when /root/reference is present)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "_build", "libft_oracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.fto_build_tree.restype = ctypes.c_int
        L.fto_build_tree.argtypes = [
            ctypes.c_int, ctypes.c_int64, _i64p, _f64p, ctypes.c_int, ctypes.c_int64,
            _i64p, _f64p, _i64p, _i64p, _i64p, _i64p,
            ctypes.POINTER(_i64p), ctypes.POINTER(_i64p), _i64p,
        ]
        L.fto_refresh.argtypes = [ctypes.c_int64] * 3 + [_f64p, _f64p, _f64p, _i64p]
        sweep_args = [
            ctypes.c_int, ctypes.c_int64, _i64p, _i64p, _f64p, _i64p, _i64p, _i64p, ctypes.c_int,
            ctypes.POINTER(_f64p), ctypes.POINTER(_f64p), ctypes.POINTER(_f64p),
        ]
        L.fto_factor_sweep.argtypes = sweep_args + [
            ctypes.c_double, ctypes.c_double, _i64p, ctypes.c_int64, ctypes.c_int64]
        L.fto_core_sweep.argtypes = sweep_args + [_f64p, _i64p, ctypes.c_int64, ctypes.c_int64]
        L.fto_apply_core.argtypes = [ctypes.c_int64, ctypes.c_int64, _f64p, _f64p,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double, _i64p]
        L.fto_predict.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _i64p,
                                  ctypes.POINTER(_f64p), _f64p]
        _LIB = L
    return _LIB


def ref_kernels():
    """The reference's own compiled `_ckern` module (oracle/_ref), or None if not built."""
    global _REF
    if _REF is None:
        cands = glob.glob(os.path.join(HERE, "_ref", "_ckern*.so"))
        if not cands:
            return None
        spec = importlib.util.spec_from_file_location("_ckern", cands[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REF = mod
    return _REF


def _p64(a):
    return a.ctypes.data_as(_f64p)


def _pi(a):
    return a.ctypes.data_as(_i64p)


def _table(arrs):
    return (_f64p * len(arrs))(*[_p64(a) for a in arrs])


# ----------------------------------------------------------------------------------------
# Layout
# ----------------------------------------------------------------------------------------


@dataclass
class OracleTree:
    """Mirror of csf.CsfTree (csf.py:32-80) as plain int64/fp64 numpy arrays."""

    root_mode: int
    level_modes: tuple
    inds: list
    ptrs: list
    vals: np.ndarray
    fiber_ptr: np.ndarray
    fiber_coord: np.ndarray
    sub_fiber_ptr: np.ndarray
    sub_leaf_ptr: np.ndarray

    @property
    def nnz(self):
        return self.vals.shape[0]

    @property
    def num_fibers(self):
        return self.fiber_ptr.shape[0] - 1

    @property
    def num_subtensors(self):
        return self.sub_fiber_ptr.shape[0] - 1

    @property
    def leaf_coord(self):
        return self.inds[-1]

    @property
    def prefix_modes(self):
        return np.asarray(self.level_modes[:-1], dtype=np.int64)

    @property
    def leaf_mode(self):
        return self.level_modes[-1]


def build_tree(idx: np.ndarray, vals: np.ndarray, root_mode: int, fiber_threshold=128) -> OracleTree:
    """csf.py:101-196 restated in C (fto_build_tree)."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    nnz, N = idx.shape
    thr = 0 if fiber_threshold is None else int(fiber_threshold)
    if fiber_threshold is not None and thr < 1:
        raise ValueError("fiber_threshold must be >= 1")
    leaf = np.empty(nnz, np.int64)
    v = np.empty(nnz, np.float64)
    fptr = np.empty(nnz + 1, np.int64)
    fcoord = np.empty(nnz * (N - 1), np.int64)
    sfp = np.empty(nnz + 1, np.int64)
    slp = np.empty(nnz + 1, np.int64)
    inds = [np.empty(nnz, np.int64) for _ in range(N)]
    ptrs = [np.empty(nnz + 1, np.int64) for _ in range(N - 1)]
    counts = np.zeros(2 + N, np.int64)
    ind_tab = (_i64p * N)(*[_pi(a) for a in inds])
    ptr_tab = (_i64p * max(N - 1, 1))(*[_pi(a) for a in ptrs])
    rc = lib().fto_build_tree(N, nnz, _pi(idx), _p64(vals), root_mode, thr, _pi(leaf), _p64(v),
                              _pi(fptr), _pi(fcoord), _pi(sfp), _pi(slp), ind_tab, ptr_tab,
                              _pi(counts))
    if rc != 0:
        raise RuntimeError("fto_build_tree failed")
    F, S = int(counts[0]), int(counts[1])
    nodes = [int(c) for c in counts[2:]]
    return OracleTree(
        root_mode=root_mode,
        level_modes=tuple((root_mode + d) % N for d in range(N)),
        inds=[inds[d][: nodes[d]].copy() for d in range(N)],
        ptrs=[ptrs[d][: nodes[d] + 1].copy() for d in range(N - 1)],
        vals=v,
        fiber_ptr=fptr[: F + 1].copy(),
        fiber_coord=fcoord[: F * (N - 1)].reshape(F, N - 1).copy(),
        sub_fiber_ptr=sfp[: S + 1].copy(),
        sub_leaf_ptr=slp[: S + 1].copy(),
    )


def build_forest(idx, vals, fiber_threshold=128):
    N = idx.shape[1]
    return [build_tree(idx, vals, t, fiber_threshold) for t in range(N)]


# ----------------------------------------------------------------------------------------
# Kernel shims (same argument order as the reference `impl` module, _ckern.pyx:21-282)
# ----------------------------------------------------------------------------------------


class CKernels:
    """Our C restatement exposed with the reference `impl` signatures."""

    BACKEND = "oracle-c"

    @staticmethod
    def refresh_dot_mode(A, B_t, out, counts):
        I, J = A.shape
        R = B_t.shape[0]
        lib().fto_refresh(I, J, R, _p64(A), _p64(B_t), _p64(out), _pi(counts))

    @staticmethod
    def _common(leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes, leaf_mode, factors,
                cores_t, dots):
        N = len(factors)
        R = cores_t[0].shape[0]
        ranks = np.asarray([a.shape[1] for a in factors], np.int64)
        keep = [ranks, prefix_modes, factors, cores_t, dots]
        args = [N, R, _pi(ranks), _pi(leaf_coord), _p64(leaf_val), _pi(fiber_ptr),
                _pi(np.ascontiguousarray(fiber_coord)), _pi(prefix_modes), int(leaf_mode),
                _table(factors), _table(cores_t),
                _table(dots) if dots is not None else ctypes.POINTER(_f64p)()]
        return args, keep

    @classmethod
    def factor_sweep(cls, leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes, leaf_mode,
                     factors, cores_t, dots, lr, reg, counts, fib_lo, fib_hi):
        args, _keep = cls._common(leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes,
                                  leaf_mode, factors, cores_t, dots)
        lib().fto_factor_sweep(*args, lr, reg, _pi(counts), fib_lo, fib_hi)

    @classmethod
    def core_sweep(cls, leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes, leaf_mode,
                   factors, cores_t, dots, acc, counts, fib_lo, fib_hi):
        args, _keep = cls._common(leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes,
                                  leaf_mode, factors, cores_t, dots)
        lib().fto_core_sweep(*args, _p64(acc), _pi(counts), fib_lo, fib_hi)

    @staticmethod
    def apply_core_update(core_t_u, acc, omega, lr, reg, counts):
        R, J = core_t_u.shape
        lib().fto_apply_core(R, J, _p64(core_t_u), _p64(acc), omega, lr, reg, _pi(counts))


def kernels(kind: str = "oracle"):
    """'oracle' -> our C restatement; 'reference' -> the reference's compiled _ckern."""
    if kind == "oracle":
        return CKernels
    mod = ref_kernels()
    if mod is None:
        raise RuntimeError("oracle/_ref/_ckern*.so not built (needs /root/reference)")
    return mod


# ----------------------------------------------------------------------------------------
# Model and trainer restated (model.py:45-141, train.py:40-336)
# ----------------------------------------------------------------------------------------


class DivergenceError(Exception):
    def __init__(self, message, mode=None, epoch=None):
        super().__init__(message)
        self.mode = mode
        self.epoch = epoch


@dataclass
class OracleModel:
    dims: tuple
    ranks: tuple
    core_rank: int
    factors: list
    cores_t: list

    @property
    def order(self):
        return len(self.dims)

    def copy(self):
        return OracleModel(self.dims, self.ranks, self.core_rank,
                           [a.copy() for a in self.factors], [b.copy() for b in self.cores_t])


def default_init_model(dims, ranks, core_rank, seed) -> OracleModel:
    """model.py:121-141: U(0,1)/sqrt(J_n) factors then U(0,1)/sqrt(R) cores, one PCG64 stream."""
    rng = np.random.default_rng(seed)
    dims = tuple(int(d) for d in dims)
    ranks = tuple(int(j) for j in ranks)
    factors = [rng.uniform(0.0, 1.0, size=(dims[n], ranks[n])) / math.sqrt(ranks[n])
               for n in range(len(dims))]
    cores_t = [rng.uniform(0.0, 1.0, size=(int(core_rank), ranks[n])) / math.sqrt(int(core_rank))
               for n in range(len(dims))]
    return OracleModel(dims, ranks, int(core_rank), factors, cores_t)


@dataclass
class OracleConfig:
    lr_a: float = 1e-3
    lr_b: float = 1e-3
    reg_a: float = 1e-2
    reg_b: float = 1e-2
    plan: str = "cached"
    workers: int = 0
    divergence_limit: float = 1e12


def precompute_cache(model, K=CKernels, counts=None):
    cache = [np.zeros((model.dims[n], model.core_rank)) for n in range(model.order)]
    c = counts if counts is not None else np.zeros(5, np.int64)
    for n in range(model.order):
        K.refresh_dot_mode(model.factors[n], model.cores_t[n], cache[n], c)
    return cache


def _guard(arr, mode, cfg, what):
    if not np.isfinite(arr).all() or float(np.abs(arr).max()) > cfg.divergence_limit:
        raise DivergenceError(f"{what} mode {mode} diverged", mode=mode)


def _parallel(tree, workers, task):
    """train.py:124-149: dynamic queue of subtensors over `workers` threads."""
    state = {"next": 0}
    lock = threading.Lock()
    errors = []

    def loop(wid):
        try:
            while True:
                with lock:
                    s = state["next"]
                    if s >= tree.num_subtensors:
                        return
                    state["next"] = s + 1
                task(wid, int(tree.sub_fiber_ptr[s]), int(tree.sub_fiber_ptr[s + 1]))
        except BaseException as exc:  # pragma: no cover
            errors.append(exc)

    threads = [threading.Thread(target=loop, args=(w,)) for w in range(workers)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]


def _targs(tree):
    return (tree.leaf_coord, tree.vals, tree.fiber_ptr, tree.fiber_coord, tree.prefix_modes,
            tree.leaf_mode)


def update_factor_mode(model, forest, cache, n, cfg, K=CKernels, counts=None):
    tree = forest[n]
    u = tree.leaf_mode
    dots = cache if cfg.plan == "cached" else None
    total = np.zeros(5, np.int64)
    if cfg.workers <= 1:
        K.factor_sweep(*_targs(tree), model.factors, model.cores_t, dots, cfg.lr_a, cfg.reg_a,
                       total, 0, tree.num_fibers)
    else:
        raws = [np.zeros(5, np.int64) for _ in range(cfg.workers)]
        _parallel(tree, cfg.workers, lambda w, lo, hi: K.factor_sweep(
            *_targs(tree), model.factors, model.cores_t, dots, cfg.lr_a, cfg.reg_a, raws[w], lo, hi))
        for r in raws:
            total += r
    _guard(model.factors[u], u, cfg, "factor")
    if cache is not None and cfg.plan == "cached":
        K.refresh_dot_mode(model.factors[u], model.cores_t[u], cache[u], total)
    if counts is not None:
        counts += total
    return total


def update_core_mode(model, forest, cache, n, cfg, K=CKernels, counts=None):
    tree = forest[n]
    u = tree.leaf_mode
    dots = cache if cfg.plan == "cached" else None
    R, Ju = model.core_rank, model.ranks[u]
    total = np.zeros(5, np.int64)
    if cfg.workers <= 1:
        acc = np.zeros((R, Ju))
        K.core_sweep(*_targs(tree), model.factors, model.cores_t, dots, acc, total, 0,
                     tree.num_fibers)
    else:
        raws = [np.zeros(5, np.int64) for _ in range(cfg.workers)]
        accs = [np.zeros((R, Ju)) for _ in range(cfg.workers)]
        _parallel(tree, cfg.workers, lambda w, lo, hi: K.core_sweep(
            *_targs(tree), model.factors, model.cores_t, dots, accs[w], raws[w], lo, hi))
        for r in raws:
            total += r
        acc = accs[0]
        for extra in accs[1:]:
            acc += extra
    K.apply_core_update(model.cores_t[u], acc, float(tree.nnz), cfg.lr_b, cfg.reg_b, total)
    _guard(model.cores_t[u], u, cfg, "core")
    if cache is not None and cfg.plan == "cached":
        K.refresh_dot_mode(model.factors[u], model.cores_t[u], cache[u], total)
    if counts is not None:
        counts += total
    return total


def run_epoch(model, forest, cache, cfg, K=CKernels, epoch_no=1, snapshots=None):
    """train.py:251-278 (without the evaluation)."""
    try:
        for n in range(model.order):
            update_factor_mode(model, forest, cache, n, cfg, K)
            if snapshots is not None:
                snapshots.append(("factor", forest[n].leaf_mode,
                                  model.factors[forest[n].leaf_mode].copy()))
        for n in range(model.order):
            update_core_mode(model, forest, cache, n, cfg, K)
            if snapshots is not None:
                snapshots.append(("core", forest[n].leaf_mode,
                                  model.cores_t[forest[n].leaf_mode].copy()))
    except DivergenceError as exc:
        raise DivergenceError(f"divergence at epoch {epoch_no}, mode {exc.mode}",
                              mode=exc.mode, epoch=epoch_no) from None


class RowParallelRef:
    """The reference's serial epoch, run on all host cores at scale (10 M+ entries).

    For the factor sweep of tree t (leaf mode u) the entries are split into T groups of
    contiguous ``i_u`` blocks balanced by count, and each group gets its own tree t
    (``build_tree``, bit-identical to csf.py:101-196).  A group's tree holds exactly the leaves
    of its rows, in the full tree's relative order, under the same fibers.  Within a sweep only
    rows of A_u change and each leaf touches only its own row (train.py:152-197), so
    running the reference kernel ``K.factor_sweep`` (_ckern.pyx:132-199) over every group tree
    concurrently -- disjoint rows, no shared writes -- is **bitwise** the serial sweep of the
    full tree.  The core sweep (_ckern.pyx:202-269) accumulates one ``acc`` per group, summed
    in fixed group order before ``apply_core_update`` with omega = |Omega| -- the reference's
    own ``workers`` reduction (train.py:222-236), so it differs from the serial sweep only in
    fp64 summation order.  ``K`` defaults to the reference's compiled ``_ckern`` (oracle/_ref)
    when built, else our C restatement; both release the GIL, so Python threads run in
    parallel.
    """

    def __init__(self, idx, vals, dims, threads=None, K=None, fiber_threshold=128):
        from concurrent.futures import ThreadPoolExecutor

        idx = np.ascontiguousarray(idx, dtype=np.int64)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        self.N = idx.shape[1]
        self.nnz = idx.shape[0]
        self.dims = tuple(int(d) for d in dims)
        self.T = int(threads or min(os.cpu_count() or 1, 32))
        self.K = K if K is not None else (ref_kernels() or CKernels)
        self.pool = ThreadPoolExecutor(self.T)
        jobs = []
        for t in range(self.N):
            u = (t + self.N - 1) % self.N
            counts = np.bincount(idx[:, u], minlength=self.dims[u])
            cum = np.cumsum(counts)
            cuts = np.searchsorted(cum, np.linspace(0, self.nnz, self.T + 1)[1:-1], side="left")
            bounds = [0] + [int(c) + 1 for c in cuts] + [self.dims[u]]
            grp = np.searchsorted(np.asarray(bounds[1:-1]), idx[:, u], side="right")
            order = np.argsort(grp, kind="stable")
            starts = np.searchsorted(grp[order], np.arange(self.T + 1))
            for k in range(self.T):
                sel = order[starts[k]:starts[k + 1]]
                if sel.size:
                    jobs.append((t, idx[sel], vals[sel]))
        built = list(self.pool.map(
            lambda j: (j[0], build_tree(j[1], j[2], j[0], fiber_threshold)), jobs))
        self.groups = [[tree for (tt, tree) in built if tt == t] for t in range(self.N)]

    def leaf_mode(self, t):
        return (t + self.N - 1) % self.N

    def update_factor_mode(self, model, cache, t, cfg):
        K, u = self.K, self.leaf_mode(t)
        dots = cache if cfg.plan == "cached" else None
        raws = [np.zeros(5, np.int64) for _ in self.groups[t]]
        list(self.pool.map(lambda k: K.factor_sweep(
            *_targs(self.groups[t][k]), model.factors, model.cores_t, dots, cfg.lr_a, cfg.reg_a,
            raws[k], 0, self.groups[t][k].num_fibers), range(len(self.groups[t]))))
        _guard(model.factors[u], u, cfg, "factor")
        if cache is not None and cfg.plan == "cached":
            K.refresh_dot_mode(model.factors[u], model.cores_t[u], cache[u], raws[0])

    def update_core_mode(self, model, cache, t, cfg):
        K, u = self.K, self.leaf_mode(t)
        dots = cache if cfg.plan == "cached" else None
        R, Ju = model.core_rank, model.ranks[u]
        raws = [np.zeros(5, np.int64) for _ in self.groups[t]]
        accs = [np.zeros((R, Ju)) for _ in self.groups[t]]
        list(self.pool.map(lambda k: K.core_sweep(
            *_targs(self.groups[t][k]), model.factors, model.cores_t, dots, accs[k], raws[k], 0,
            self.groups[t][k].num_fibers), range(len(self.groups[t]))))
        acc = accs[0]
        for extra in accs[1:]:
            acc += extra
        K.apply_core_update(model.cores_t[u], acc, float(self.nnz), cfg.lr_b, cfg.reg_b, raws[0])
        _guard(model.cores_t[u], u, cfg, "core")
        if cache is not None and cfg.plan == "cached":
            K.refresh_dot_mode(model.factors[u], model.cores_t[u], cache[u], raws[0])
        return acc

    def run_epoch(self, model, cache, cfg):
        for t in range(self.N):
            self.update_factor_mode(model, cache, t, cfg)
        for t in range(self.N):
            self.update_core_mode(model, cache, t, cfg)

    def close(self):
        self.pool.shutdown()


def predict(model, idx):
    """model.py:219-230 (dots computed fresh, sequential sums)."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    dots = precompute_cache(model)
    out = np.empty(idx.shape[0])
    lib().fto_predict(model.order, model.core_rank, idx.shape[0], _pi(idx), _table(dots), _p64(out))
    return out


def evaluate(model, idx, vals):
    """train.py:91-98."""
    resid = np.asarray(vals, np.float64) - predict(model, idx)
    return math.sqrt(float(resid @ resid) / resid.size), float(np.abs(resid).sum()) / resid.size
