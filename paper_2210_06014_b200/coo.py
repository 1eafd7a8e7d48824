"""COO tensors: the input type of the decomposition API (mirrors coo.SparseCooTensor,
/root/reference/pkg/src/fastertucker/coo.py:24-73) plus its device-resident form.

* :class:`SparseCooTensor` keeps the reference's host contract: 0-based coordinates
  ``idx`` (nnz x N) and values ``vals`` (nnz), order >= 3, in-range, unique coordinates.
  Duplicate detection is a packed-key sort (numpy) up to ``HOST_DEDUP_LIMIT`` entries; above
  that it is deferred to the GPU B-CSF builder, which detects equal adjacent keys for free
  while sorting and raises the same :class:`ValidationError`.
* :class:`DeviceCoo` is the HBM copy (int32 coordinates, fp32 values) the kernels read.
* :func:`generate_synthetic` draws a tensor ON THE GPU (ft_generate_coo) with the reference
  generator's distribution (coo.py:164-213: distinct cells uniform without replacement,
  U[lo, hi] values) -- not its PCG64 stream; parity inputs come from the reference itself.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import CapacityError, ConfigError, ValidationError

HOST_DEDUP_LIMIT = 4_000_000


def _pack_keys(idx: np.ndarray, dims) -> np.ndarray | None:
    bits = [max(1, int(d - 1).bit_length()) for d in dims]
    if sum(bits) > 63:
        return None
    key = np.zeros(idx.shape[0], dtype=np.int64)
    for n, b in enumerate(bits):
        key = (key << b) | idx[:, n]
    return key


class SparseCooTensor:
    """N-order sparse tensor: unique 0-based coordinates plus values (coo.py:24-73)."""

    __slots__ = ("dims", "idx", "vals", "_device")

    def __init__(self, dims, idx, vals, *, validate: bool = True):
        dims = tuple(int(d) for d in dims)
        if len(dims) < 3:
            raise ValidationError(f"tensor order must be >= 3, got {len(dims)}")
        if any(d < 1 for d in dims):
            raise ValidationError(f"dims must be positive, got {dims}")
        idx = np.asarray(idx)
        vals = np.asarray(vals, dtype=np.float64)
        if idx.ndim != 2 or idx.shape[1] != len(dims):
            raise ValidationError(f"idx shape {idx.shape} does not match order {len(dims)}")
        if vals.shape != (idx.shape[0],):
            raise ValidationError("vals length does not match idx")
        if idx.shape[0] == 0:
            raise ValidationError("tensor must contain at least one entry")
        if validate:
            if idx.min(initial=0) < 0 or np.any(idx.max(axis=0) >= np.asarray(dims)):
                raise ValidationError("coordinate out of range for dims")
            if idx.shape[0] <= HOST_DEDUP_LIMIT:
                dup = _first_duplicate(idx, dims)
                if dup is not None:
                    raise ValidationError(
                        f"duplicate coordinate {tuple(int(c) + 1 for c in dup)}")
        self.dims = dims
        self.idx = idx
        self.vals = vals
        self._device = None

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return int(self.idx.shape[0])

    def capacity(self) -> int:
        return math.prod(self.dims)

    def device(self, stream=None) -> "DeviceCoo":
        """The HBM copy (uploaded once, cached)."""
        if self._device is None:
            self._device = DeviceCoo.from_host(self, stream=stream)
        return self._device


def _first_duplicate(idx: np.ndarray, dims):
    key = _pack_keys(np.asarray(idx, dtype=np.int64), dims)
    if key is None:
        uniq = np.unique(idx, axis=0)
        if uniq.shape[0] == idx.shape[0]:
            return None
        seen = set()
        for row in idx:
            t = tuple(row.tolist())
            if t in seen:
                return row
            seen.add(t)
        return None
    order = np.argsort(key, kind="stable")
    sk = key[order]
    same = np.flatnonzero(sk[1:] == sk[:-1])
    if same.size == 0:
        return None
    # the reference names the first duplicate in entry order
    first = min(int(max(order[k], order[k + 1])) for k in same)
    return idx[first]


@dataclass
class DeviceCoo:
    """Device-resident COO: ``idx`` int32 [nnz, N] row-major, ``vals`` fp32 [nnz] (torch)."""

    dims: tuple
    idx: "object"
    vals: "object"

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    @classmethod
    def from_host(cls, tensor: SparseCooTensor, stream=None) -> "DeviceCoo":
        import torch

        from . import _lib

        _lib.lib()
        if max(tensor.dims) >= 2**31:
            raise ConfigError("dims must fit int32 on the device path")
        idx = torch.from_numpy(np.ascontiguousarray(tensor.idx, dtype=np.int32))
        vals = torch.from_numpy(np.ascontiguousarray(tensor.vals, dtype=np.float32))
        return cls(tensor.dims, idx.cuda(non_blocking=False), vals.cuda(non_blocking=False))

    def to_host(self, validate: bool = False) -> SparseCooTensor:
        return SparseCooTensor(self.dims, self.idx.cpu().numpy().astype(np.int64),
                               self.vals.cpu().numpy().astype(np.float64), validate=validate)

    def slice(self, lo: int, hi: int) -> "DeviceCoo":
        return DeviceCoo(self.dims, self.idx[lo:hi], self.vals[lo:hi])


@dataclass(frozen=True)
class DatasetSplit:
    """Disjoint train/test partition of one tensor's entries (coo.py:76-82)."""

    train: object
    test: object
    seed: int


def split_dataset(tensor: SparseCooTensor, test_fraction: float, seed: int) -> DatasetSplit:
    """Deterministic exact partition (coo.py:216-231): the PCG64 stream [seed, 2] permutes the
    entries, the first round(nnz * test_fraction) become the test set."""
    if not 0.0 < test_fraction < 1.0:
        raise ConfigError(f"test_fraction must lie in (0, 1), got {test_fraction}")
    n_test = int(round(tensor.nnz * test_fraction))
    if n_test < 1 or n_test >= tensor.nnz:
        raise ConfigError(f"test_fraction {test_fraction} leaves an empty part for nnz={tensor.nnz}")
    perm = np.random.default_rng([int(seed), 2]).permutation(tensor.nnz)
    te, tr = perm[:n_test], perm[n_test:]
    return DatasetSplit(
        train=SparseCooTensor(tensor.dims, tensor.idx[tr], tensor.vals[tr], validate=False),
        test=SparseCooTensor(tensor.dims, tensor.idx[te], tensor.vals[te], validate=False),
        seed=int(seed))


def generate_device(dims, nnz: int, value_range=(1.0, 5.0), seed: int = 0) -> DeviceCoo:
    """nnz distinct uniform cells + U[lo, hi] values generated on the GPU, in random order."""
    import ctypes

    import torch

    from . import _lib

    L = _lib.lib()
    dims = tuple(int(d) for d in dims)
    if len(dims) < 3 or any(d < 1 for d in dims):
        raise ConfigError(f"dims must be >= 3 positive extents, got {dims}")
    if nnz < 1:
        raise ConfigError("nnz must be positive")
    if nnz > math.prod(dims):
        raise CapacityError(f"nnz={nnz} exceeds capacity {math.prod(dims)} of dims {dims}")
    lo, hi = float(value_range[0]), float(value_range[1])
    if not lo < hi:
        raise ConfigError(f"value range must satisfy lo < hi, got ({lo}, {hi})")
    if 2 * nnz > math.prod(dims):
        # dense request (the device sampler draws i.i.d. cells and keeps the distinct ones, which
        # needs nnz <= capacity / 2): sample without replacement on the host, as the reference's
        # _sample_coords does for dense cubes (coo.py:164-178), then upload
        rng = np.random.default_rng([int(seed), 0])
        lin = rng.permutation(math.prod(dims))[:nnz]
        hidx = np.stack(np.unravel_index(lin, dims), axis=1).astype(np.int32)
        hvals = np.random.default_rng([int(seed), 1]).uniform(lo, hi, size=nnz).astype(np.float32)
        return DeviceCoo(dims, torch.from_numpy(hidx).cuda(), torch.from_numpy(hvals).cuda())
    idx = torch.empty((nnz, len(dims)), dtype=torch.int32, device="cuda")
    vals = torch.empty(nnz, dtype=torch.float32, device="cuda")
    d = (ctypes.c_int64 * len(dims))(*dims)
    _lib.check(L.ft_generate_coo(len(dims), d, nnz, int(seed) & (2**64 - 1), lo, hi,
                                 idx.data_ptr(), vals.data_ptr(), _lib.stream_handle()),
               "ft_generate_coo")
    return DeviceCoo(dims, idx, vals)


def generate_synthetic(dims, nnz: int, value_range=(1.0, 5.0), seed: int = 0, low_rank=None,
                       *, test_fraction: float | None = None):
    """Device synthetic tensor with the reference's signature (coo.py:181-213): nnz distinct
    uniform cells, values U[value_range], or -- with ``low_rank=(ranks, core_rank)`` -- the
    predictions of a hidden random model (generate_low_rank_device).  Returns a
    :class:`DeviceCoo` (GPU-resident; ``.to_host()`` gives the reference's SparseCooTensor).  With
    ``test_fraction`` returns a :class:`DatasetSplit` of two DeviceCoo (the generator's order is
    random, so the first round(nnz * f) entries are a uniform test sample)."""
    if low_rank is not None:
        ranks, core_rank = low_rank
        t = generate_low_rank_device(dims, nnz, ranks, core_rank, seed)
    else:
        t = generate_device(dims, nnz, value_range, seed)
    if test_fraction is None:
        return t
    n_test = int(round(nnz * test_fraction))
    if n_test < 1 or n_test >= nnz:
        raise ConfigError("test_fraction leaves an empty part")
    return DatasetSplit(train=t.slice(n_test, nnz), test=t.slice(0, n_test), seed=int(seed))


def load_coo(path, order: int, dims=None, normalize=None) -> SparseCooTensor:
    """Whitespace-separated 1-based coordinates + value per line, '#' comments
    (coo.py:95-138).  Parsed by pandas' C reader (a Netflix-size file in seconds, not the
    reference's per-line Python loop); on any malformed input the file is rescanned line by line
    so the error names the offending line exactly as the reference does."""
    from .errors import ParseError

    try:
        import pandas as pd

        # coordinates as integers (the reference's int(), so "1.0" is rejected) and the value as
        # float ("nan" accepted, as float() does); '#' only as a whole-line comment, checked on
        # the raw bytes below (pandas' comment= would also strip inline comments)
        dtypes = {c: np.int64 for c in range(order)}
        dtypes[order] = np.float64
        df = pd.read_csv(path, sep=r"\s+", comment="#", header=None, engine="c", dtype=dtypes,
                         float_precision="round_trip")
        ok = df.shape[1] == order + 1 and not df.iloc[:, :order].isnull().values.any()
        if ok:
            coords = df.iloc[:, :order].to_numpy(dtype=np.int64)
            vals = df.iloc[:, order].to_numpy(dtype=np.float64)
            ok = _layout_ok(path, order, int(np.isnan(vals).sum()))
    except Exception:
        ok = False
    if not ok:
        # raises with the reference's message; a file it accepts (e.g. only comments) is parsed
        # by the same line scanner
        coords, vals = _scan_errors(path, order, ParseError)
    if coords.shape[0] == 0:
        raise ValidationError(f"{path}: no entries")
    idx = coords
    if (idx < 1).any():
        _scan_errors(path, order, ParseError)
    idx = idx - 1
    dup = _first_duplicate(idx, tuple(int(m) + 1 for m in idx.max(axis=0)))
    if dup is not None:
        _scan_errors(path, order, ParseError)
    if normalize is not None:
        vals = _minmax_scale(vals, normalize)
    if dims is None:
        dims = tuple(int(m) + 1 for m in idx.max(axis=0))
    return SparseCooTensor(tuple(dims), idx, vals)


def _layout_ok(path, order, n_nan) -> bool:
    """What pandas' reader forgives and the reference's scanner does not (coo.py:104-121): an
    inline '#' (the reference only skips whole-line comments, so such a line has extra fields)
    and a missing value field (pandas fills NaN: more NaN values than 'nan' tokens).  Known
    remaining difference: pandas' int64 reader accepts a coordinate written "1.0", which the
    reference's int() rejects (checking every coordinate token in Python would cost ~1 us per
    line, minutes on a Netflix-size file)."""
    import re

    raw = np.fromfile(path, dtype=np.uint8)
    for p in np.flatnonzero(raw == ord("#")).tolist():
        q = p - 1
        while q >= 0 and raw[q] in (32, 9, 13):
            q -= 1
        if q >= 0 and raw[q] != 10:
            return False
    if n_nan and n_nan > len(re.findall(rb"(?i)(?<![^\s])[+-]?nan(?![^\s])", raw.tobytes())):
        return False
    return True


def _scan_errors(path, order, ParseError):
    """The reference's line-by-line checks (coo.py:104-128), run to report an error; returns
    the parsed (idx, vals) when the file passes them."""
    seen = set()
    coords, values = [], []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            stripped = line.strip()
            if not stripped or stripped.startswith("#"):
                continue
            fields = stripped.split()
            if len(fields) != order + 1:
                raise ParseError(f"{path}: line {lineno}: expected {order + 1} fields, got "
                                 f"{len(fields)}")
            try:
                coord = tuple(int(f) for f in fields[:order])
            except ValueError as exc:
                raise ParseError(f"{path}: line {lineno}: bad coordinate: {exc}") from None
            try:
                float(fields[order])
            except ValueError:
                raise ParseError(f"{path}: line {lineno}: bad value {fields[order]!r}") from None
            if any(c < 1 for c in coord):
                raise ValidationError(f"{path}: line {lineno}: coordinates are 1-based")
            if coord in seen:
                raise ValidationError(f"{path}: line {lineno}: duplicate coordinate {coord}")
            seen.add(coord)
            coords.append(coord)
            values.append(float(fields[order]))
    return (np.asarray(coords, dtype=np.int64).reshape(-1, order),
            np.asarray(values, dtype=np.float64))


def _minmax_scale(vals: np.ndarray, target) -> np.ndarray:
    lo, hi = float(target[0]), float(target[1])
    if not lo < hi:
        raise ConfigError(f"normalize range must satisfy lo < hi, got ({lo}, {hi})")
    vmin, vmax = float(vals.min()), float(vals.max())
    if vmin == vmax:
        raise ConfigError("cannot min-max scale constant values")
    return lo + (vals - vmin) * ((hi - lo) / (vmax - vmin))


def write_coo(path, tensor) -> None:
    """The reference's 1-based text form (coo.py:151-157), values in shortest round-trip repr."""
    idx = np.asarray(tensor.idx) + 1
    vals = np.asarray(tensor.vals, dtype=np.float64)
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(f"# order={len(tensor.dims)} dims={','.join(map(str, tensor.dims))}\n")
        for row, val in zip(idx.tolist(), vals.tolist()):
            fh.write(" ".join(str(int(c)) for c in row) + f" {float(val)!r}\n")


def generate_low_rank_device(dims, nnz: int, ranks, core_rank: int, seed: int = 0) -> DeviceCoo:
    """generate_synthetic(..., low_rank=(ranks, core_rank)) (coo.py:207-213): distinct uniform
    cells whose values are the predictions of a hidden random model (model.py:144-146's
    distribution) -- coordinates and predictions both computed on the GPU."""
    import torch

    from .model import default_init_model, predict_batch

    t = generate_device(dims, nnz, (0.0, 1.0), seed)
    hidden = default_init_model(dims, ranks, core_rank, np.random.SeedSequence([int(seed), 3]))
    vals = predict_batch(hidden, t.idx)
    return DeviceCoo(t.dims, t.idx, vals.to(torch.float32))


def as_device(tensor) -> DeviceCoo:
    if isinstance(tensor, DeviceCoo):
        return tensor
    if isinstance(tensor, SparseCooTensor):
        return tensor.device()
    # duck-typed reference SparseCooTensor (dims / idx / vals)
    if hasattr(tensor, "idx") and hasattr(tensor, "vals") and hasattr(tensor, "dims"):
        return SparseCooTensor(tensor.dims, tensor.idx, tensor.vals, validate=False).device()
    raise ConfigError(f"expected a COO tensor, got {type(tensor).__name__}")
