"""Factor / core parameters in HBM (mirrors model.Model, model.py:45-141) and prediction.

Layout (row-major fp32, one torch CUDA tensor each):
  factors[n]  A_n  I_n x J_n   (lane j of a warp owns column j of a row)
  cores_t[n]  Bt_n R x J_n     (the reference's transposed core; rows contiguous)
Initialisation draws from numpy's PCG64 exactly like the reference (model.py:106-141) in
fp64, then rounds to fp32 on upload, so a model built here starts from the reference's
numbers.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, ValidationError

_CKPT_MAGIC = b"FTMODEL\x00"
_CKPT_VERSION = 1


@dataclass(frozen=True)
class InitSpec:
    """Uniform(lo, hi) i.i.d. initialization with a fixed seed (model.py:32-42)."""

    lo: float
    hi: float
    seed: int

    def __post_init__(self):
        if not self.lo < self.hi:
            raise ConfigError(f"init range must satisfy lo < hi, got ({self.lo}, {self.hi})")


class Model:
    """Device-resident factor and transposed core matrices."""

    __slots__ = ("dims", "ranks", "core_rank", "factors", "cores_t", "_view")

    def __init__(self, dims, ranks, core_rank, factors, cores_t):
        import torch

        _lib.lib()  # fail loudly without the sm_100a library / a GPU
        dims = tuple(int(d) for d in dims)
        ranks = tuple(int(j) for j in ranks)
        core_rank = int(core_rank)
        if len(ranks) != len(dims):
            raise ConfigError("ranks must give one J per mode")
        if any(j < 1 for j in ranks) or core_rank < 1 or any(d < 1 for d in dims):
            raise ConfigError("shapes must be positive")
        if max(ranks) > _lib.FT_MAX_RANK or core_rank > _lib.FT_MAX_RANK:
            raise ConfigError(f"J_n and R must be <= {_lib.FT_MAX_RANK} on the B200 kernels")
        if len(dims) > _lib.FT_MAX_ORDER:
            raise ConfigError(f"order must be <= {_lib.FT_MAX_ORDER}")

        def dev(a):
            if isinstance(a, torch.Tensor):
                return a.to(device="cuda", dtype=torch.float32).contiguous()
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()

        self.dims, self.ranks, self.core_rank = dims, ranks, core_rank
        self.factors = [dev(a) for a in factors]
        self.cores_t = [dev(b) for b in cores_t]
        for n, (a, b) in enumerate(zip(self.factors, self.cores_t)):
            if tuple(a.shape) != (dims[n], ranks[n]):
                raise ConfigError(f"factor {n} shape {tuple(a.shape)} != {(dims[n], ranks[n])}")
            if tuple(b.shape) != (core_rank, ranks[n]):
                raise ConfigError(f"core {n} shape {tuple(b.shape)} != {(core_rank, ranks[n])}")
        self._view = None

    @property
    def order(self) -> int:
        return len(self.dims)

    def core(self, n: int):
        return self.cores_t[n].T

    def copy(self) -> "Model":
        return Model(self.dims, self.ranks, self.core_rank,
                     [a.clone() for a in self.factors], [b.clone() for b in self.cores_t])

    def to_numpy(self):
        """(factors, cores_t) as float64 numpy lists, the reference Model's layout."""
        return ([a.cpu().numpy().astype(np.float64) for a in self.factors],
                [b.cpu().numpy().astype(np.float64) for b in self.cores_t])

    @classmethod
    def from_numpy(cls, dims, ranks, core_rank, factors, cores_t) -> "Model":
        return cls(dims, ranks, core_rank, factors, cores_t)

    @classmethod
    def from_reference(cls, ref_model) -> "Model":
        """Upload a reference ``fastertucker.Model`` (or anything with the same fields)."""
        return cls(ref_model.dims, ref_model.ranks, ref_model.core_rank, ref_model.factors,
                   ref_model.cores_t)

    def max_abs(self) -> float:
        return max(float(t.abs().max()) for t in self.factors + self.cores_t)

    def all_finite(self) -> bool:
        import torch

        return all(bool(torch.isfinite(t).all()) for t in self.factors + self.cores_t)

    def view(self, dots=None) -> _lib.FtModel:
        """ft_model_t over these parameters and the given cache arrays."""
        v = _lib.FtModel()
        v.order = self.order
        v.core_rank = self.core_rank
        for n in range(self.order):
            v.dims[n] = self.dims[n]
            v.ranks[n] = self.ranks[n]
            v.factors[n] = self.factors[n].data_ptr()
            v.cores_t[n] = self.cores_t[n].data_ptr()
            v.dots[n] = dots[n].data_ptr() if dots is not None and dots[n] is not None else None
        return v


def init_model(dims, ranks, core_rank, spec: InitSpec) -> Model:
    """All entries i.i.d. U(lo, hi); draw order factors 0..N-1 then cores (model.py:106-118)."""
    rng = np.random.default_rng(int(spec.seed))
    dims = tuple(int(d) for d in dims)
    ranks = tuple(int(j) for j in ranks)
    if len(ranks) != len(dims):
        raise ConfigError("ranks must give one J per mode")
    f = [rng.uniform(spec.lo, spec.hi, size=(dims[n], ranks[n])) for n in range(len(dims))]
    c = [rng.uniform(spec.lo, spec.hi, size=(int(core_rank), ranks[n])) for n in range(len(dims))]
    return Model(dims, ranks, core_rank, f, c)


def default_init_model(dims, ranks, core_rank, seed) -> Model:
    """U(0,1)/sqrt(J_n) factors then U(0,1)/sqrt(R) cores from one PCG64 stream
    (model.py:121-141), so the fp32 start equals the reference's fp64 start rounded."""
    rng = np.random.default_rng(seed)
    dims = tuple(int(d) for d in dims)
    ranks = tuple(int(j) for j in ranks)
    if len(ranks) != len(dims):
        raise ConfigError("ranks must give one J per mode")
    f = [rng.uniform(0.0, 1.0, size=(dims[n], ranks[n])) / math.sqrt(ranks[n])
         for n in range(len(dims))]
    c = [rng.uniform(0.0, 1.0, size=(int(core_rank), ranks[n])) / math.sqrt(int(core_rank))
         for n in range(len(dims))]
    return Model(dims, ranks, core_rank, f, c)


def predict_batch(model: Model, idx, cache=None):
    """x_hat for an (m, N) coordinate array (model.py:219-230), on the GPU (kernel K6).

    Uses the coherent cache when given, otherwise computes C_n = A_n Bt_n^T fresh (K2).
    Returns a float64 numpy array for host input, a device fp32 tensor for device input."""
    import torch

    from .cache import fresh_dots

    L = _lib.lib()
    host = not isinstance(idx, torch.Tensor)
    if host:
        idx_np = np.asarray(idx)
        if idx_np.ndim != 2 or idx_np.shape[1] != model.order:
            raise ValidationError(f"idx must be (m, {model.order})")
        d_idx = torch.from_numpy(np.ascontiguousarray(idx_np, dtype=np.int32)).cuda()
    else:
        d_idx = idx.to(device="cuda", dtype=torch.int32).contiguous()
    m = int(d_idx.shape[0])
    dots = cache.arrays if cache is not None else fresh_dots(model)
    out = torch.empty(m, dtype=torch.float32, device="cuda")
    if m:
        _lib.check(L.ft_predict(ctypes_ref(model.view(dots)), m, d_idx.data_ptr(), out.data_ptr(),
                                _lib.stream_handle()), "ft_predict")
    return out.cpu().numpy().astype(np.float64) if host else out


def ctypes_ref(v):
    import ctypes

    return ctypes.byref(v)


def save_model(path, model: Model) -> None:
    """FTMODEL v1 checkpoint (model.py:266-283): magic, u32 version / N / R / reserved,
    (u64 I_n, u64 J_n) pairs, then float64 factors and transposed cores (widened from fp32),
    so checkpoints interchange with the reference's load_model."""
    factors, cores = model.to_numpy()
    with open(path, "wb") as fh:
        fh.write(_CKPT_MAGIC)
        fh.write(struct.pack("<IIII", _CKPT_VERSION, model.order, model.core_rank, 0))
        for n in range(model.order):
            fh.write(struct.pack("<QQ", model.dims[n], model.ranks[n]))
        for a in factors:
            fh.write(np.ascontiguousarray(a, dtype="<f8").tobytes())
        for b in cores:
            fh.write(np.ascontiguousarray(b, dtype="<f8").tobytes())


def load_model(path) -> Model:
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:8] != _CKPT_MAGIC:
        raise ValidationError("not an FTMODEL checkpoint")
    ver, N, R, _ = struct.unpack_from("<IIII", data, 8)
    if ver != _CKPT_VERSION:
        raise ValidationError(f"unsupported checkpoint version {ver}")
    off = 24
    dims, ranks = [], []
    for _ in range(N):
        i, j = struct.unpack_from("<QQ", data, off)
        off += 16
        dims.append(i)
        ranks.append(j)
    factors, cores = [], []
    for n in range(N):
        cnt = dims[n] * ranks[n]
        factors.append(np.frombuffer(data, "<f8", cnt, off).reshape(dims[n], ranks[n]))
        off += 8 * cnt
    for n in range(N):
        cnt = R * ranks[n]
        cores.append(np.frombuffer(data, "<f8", cnt, off).reshape(R, ranks[n]))
        off += 8 * cnt
    if off != len(data):
        raise ValidationError("trailing bytes in checkpoint")
    return Model(dims, ranks, R, factors, cores)
