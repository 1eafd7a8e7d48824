"""CPU checks of the drop-in boundary (no compute): the C-ABI library exists, loads, and exports
exactly what include/ft_b200.h declares; the binding covers every symbol; the product never
imports the oracle; without a GPU the product fails loudly (no CPU fallback)."""

import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(REPO, "paper_2210_06014_b200")


def header_symbols():
    text = open(os.path.join(REPO, "include", "ft_b200.h")).read()
    return sorted(set(re.findall(r"^FT_API\s+[\w\s\*]+?\b(ft_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_abi():
    syms = header_symbols()
    for s in ("ft_build_tree", "ft_refresh", "ft_factor_sweep_rows", "ft_factor_sweep_fibers",
              "ft_core_sweep_rows", "ft_core_apply", "ft_predict", "ft_sse", "ft_last_error"):
        assert s in syms


def test_library_loads_and_exports_every_header_symbol():
    import ctypes

    from paper_2210_06014_b200 import _lib

    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build() first"
    L = ctypes.CDLL(_lib.LIB_PATH)
    for s in header_symbols():
        assert hasattr(L, s), s
    assert set(header_symbols()) == set(_lib.SIGNATURES)
    lib = _lib.load()
    assert lib.ft_abi_version() == 2


def test_library_is_sm100a_only():
    import subprocess

    from paper_2210_06014_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_\d+a?", out.stdout))
    assert arches == {"sm_100a"}, arches


def test_product_never_imports_the_oracle():
    for root, _dirs, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(root, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", text).lower() or f == "__init__.py", f


def test_no_gpu_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2210_06014_b200 as ft
    from paper_2210_06014_b200.errors import BackendUnavailableError

    with pytest.raises(BackendUnavailableError):
        ft.default_init_model((4, 4, 4), (2, 2, 2), 2, seed=0)


def test_backend_selector_contract(monkeypatch):
    from paper_2210_06014_b200 import _kernels

    assert _kernels.BACKEND == "cuda" and _kernels.COMPILED
    with pytest.raises(ValueError):
        _kernels.get_backend("python")
    with _kernels.use_backend("gpu") as k:
        assert k.BACKEND == "cuda"
    for name in ("refresh_dot_mode", "factor_sweep", "core_sweep", "apply_core_update"):
        assert callable(getattr(_kernels.impl, name))
