"""Kernel backend selection -- the reference's plugin boundary
(/root/reference/pkg/src/fastertucker/_kernels/__init__.py:11-65), B200 edition.

The reference picks ``impl`` between its compiled Cython module and a pure-Python twin.  This
package has exactly one backend, ``"cuda"`` (sm_100a kernels in libft_b200.so, module
:mod:`._cudakern`), exposing the same four entry points with the same signatures.  There is no
CPU fallback: ``FASTERTUCKER_BACKEND`` may name ``cuda`` (aliases ``gpu``, ``b200``) or be
unset; any other value raises ``RuntimeError`` like the reference's unknown-backend branch.
"""

import os
from contextlib import contextmanager

from . import _cudakern

_ALIASES = ("cuda", "gpu", "b200")

_forced = os.environ.get("FASTERTUCKER_BACKEND", "").lower()
if _forced and _forced not in _ALIASES:
    raise RuntimeError(f"unknown FASTERTUCKER_BACKEND={_forced!r} (this build provides 'cuda')")

impl = _cudakern
COMPILED = True
BACKEND = impl.BACKEND


def get_backend(name: str):
    """Return the kernel module for an explicit backend name."""
    if name in _ALIASES:
        return _cudakern
    raise ValueError(f"unknown backend {name!r}")


def current_backend() -> str:
    return impl.BACKEND


@contextmanager
def use_backend(name: str):
    """Temporarily run all plugin-level sweeps on the named backend."""
    global impl
    previous = impl
    impl = get_backend(name)
    try:
        yield impl
    finally:
        impl = previous
