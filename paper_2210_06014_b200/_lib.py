"""ctypes binding of libft_b200.so (include/ft_b200.h).

This is the only place the package touches native code.  There is no CPU fallback: if the
library is missing, or no CUDA device is present, every compute entry point raises
:class:`~paper_2210_06014_b200.errors.BackendUnavailableError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import BackendUnavailableError, BuildError, ConfigError, ValidationError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libft_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "ft_b200.h")

FT_MAX_ORDER = 16
FT_MAX_RANK = 32

FT_OK, FT_ERR_ARG, FT_ERR_CUDA, FT_ERR_DUPLICATE, FT_ERR_EMPTY, FT_ERR_UNSUPPORTED = range(6)

_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_vp = ctypes.c_void_p


class FtTree(ctypes.Structure):
    """ft_tree_t"""

    _fields_ = [
        ("order", ctypes.c_int32),
        ("root_mode", ctypes.c_int32),
        ("nnz", ctypes.c_int64),
        ("num_fibers", ctypes.c_int64),
        ("num_rows", ctypes.c_int64),
        ("leaf_coord", _vp),
        ("vals", _vp),
        ("fiber_ptr", _vp),
        ("fiber_coord", _vp),
        ("row_fiber_ptr", _vp),
        ("row_coord", _vp),
        ("leaf_pc", _vp),
        ("row_leaf_ptr", _vp),
        ("num_segs", ctypes.c_int64),
        ("seg_coord", _vp),
        ("seg_leaf_ptr", _vp),
        ("slot_grid", ctypes.c_int32),
        ("slot_kb", ctypes.c_int32),
        ("slot_batch_ptr", _vp),
        ("slot_lc", _vp),
        ("slot_pc", _vp),
        ("slot_x", _vp),
    ]


class FtModel(ctypes.Structure):
    """ft_model_t"""

    _fields_ = [
        ("order", ctypes.c_int32),
        ("core_rank", ctypes.c_int32),
        ("dims", ctypes.c_int64 * FT_MAX_ORDER),
        ("ranks", ctypes.c_int32 * FT_MAX_ORDER),
        ("factors", _vp * FT_MAX_ORDER),
        ("cores_t", _vp * FT_MAX_ORDER),
        ("dots", _vp * FT_MAX_ORDER),
    ]


# name -> (restype, argtypes); every symbol include/ft_b200.h declares
SIGNATURES = {
    "ft_last_error": (ctypes.c_char_p, []),
    "ft_abi_version": (ctypes.c_int, []),
    "ft_sm_count": (ctypes.c_int, [_i32p]),
    "ft_build_tree": (ctypes.c_int, [
        ctypes.c_int32, ctypes.c_int64, _i64p, _vp, _vp, ctypes.c_int32, ctypes.c_int64, _vp,
        ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp, _vp, _vp, _vp, _vp, _vp, _i64p, _vp, _vp]),
    "ft_tree_leaf_index": (ctypes.c_int, [ctypes.POINTER(FtTree), _vp, _vp, _vp]),
    "ft_tree_slot_plan": (ctypes.c_int, [ctypes.POINTER(FtTree), ctypes.c_int32, ctypes.c_int32,
                                         _i32p, _i32p, _vp, _i64p, _vp]),
    "ft_tree_slot_fill": (ctypes.c_int, [ctypes.POINTER(FtTree), ctypes.c_int32, _vp, _vp, _vp,
                                         _vp, _vp]),
    "ft_build_tree_derived": (ctypes.c_int, [
        ctypes.POINTER(FtTree), _i64p, ctypes.c_int64, _vp, ctypes.POINTER(_vp),
        ctypes.POINTER(_vp), _vp, _vp, _vp, _vp, _vp, _vp, _i64p, _vp, _vp]),
    "ft_tree_row_segments": (ctypes.c_int, [ctypes.POINTER(FtTree), ctypes.c_int32, _vp, _vp,
                                            _i64p, _vp]),
    "ft_refresh": (ctypes.c_int, [
        ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp, _vp, _vp]),
    "ft_peer_barrier": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_uint32, _vp]),
    "ft_refresh_scatter": (ctypes.c_int, [
        ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _vp, _vp, ctypes.POINTER(_vp),
        ctypes.c_int32, _vp, _vp]),
    "ft_factor_sweep_rows": (ctypes.c_int, [
        ctypes.POINTER(FtTree), ctypes.POINTER(FtModel), ctypes.c_float, ctypes.c_float, _vp]),
    "ft_factor_sweep_fibers": (ctypes.c_int, [
        ctypes.POINTER(FtTree), ctypes.POINTER(FtModel), ctypes.c_int64, ctypes.c_int64,
        ctypes.c_float, ctypes.c_float, ctypes.c_int32, _vp]),
    "ft_core_sweep_rows": (ctypes.c_int, [
        ctypes.POINTER(FtTree), ctypes.POINTER(FtModel), _vp, ctypes.c_int64, _i32p, _vp]),
    "ft_core_partials_size": (ctypes.c_int64, [ctypes.c_int32, ctypes.c_int32]),
    "ft_core_apply": (ctypes.c_int, [
        ctypes.c_int32, ctypes.c_int32, _vp, _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
        ctypes.c_float, ctypes.c_float, _vp, _vp, _vp]),
    "ft_core_reduce": (ctypes.c_int, [
        ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_int32, _vp, _vp]),
    "ft_predict": (ctypes.c_int, [ctypes.POINTER(FtModel), ctypes.c_int64, _vp, _vp, _vp]),
    "ft_sse": (ctypes.c_int, [ctypes.POINTER(FtModel), ctypes.c_int64, _vp, _vp, _vp, _vp]),
    "ft_sse_tree": (ctypes.c_int, [ctypes.POINTER(FtTree), ctypes.POINTER(FtModel), _vp, _vp]),
    "ft_generate_coo": (ctypes.c_int, [
        ctypes.c_int32, _i64p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_float,
        _vp, _vp, _vp]),
}

_LIB = None
_LOCK = threading.Lock()


def load(require_device: bool = False):
    """Load libft_b200.so (raising loudly if it was not built)."""
    global _LIB
    with _LOCK:
        if _LIB is None:
            if not os.path.exists(LIB_PATH):
                raise BackendUnavailableError(
                    f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "or `make -C paper_2210_06014_b200/csrc` (there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _LIB = lib
    if require_device:
        import torch

        if not torch.cuda.is_available():
            raise BackendUnavailableError(
                "no CUDA device: the FasterTucker B200 path runs only on the GPU (no CPU fallback)")
    return _LIB


def lib():
    return load(require_device=True)


def check(rc: int, what: str = "") -> None:
    if rc == FT_OK:
        return
    msg = (_LIB.ft_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == FT_ERR_DUPLICATE:
        raise ValidationError(text)
    if rc == FT_ERR_EMPTY:
        raise BuildError(text)
    if rc in (FT_ERR_ARG, FT_ERR_UNSUPPORTED):
        raise ConfigError(text)
    raise RuntimeError(text)


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
