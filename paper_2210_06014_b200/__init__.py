"""B200-native FasterTucker hot path (arXiv 2210.06014).

A drop-in for the reference package ``fastertucker``'s decomposition API on one path: the
per-epoch factor-matrix and core-matrix SGD sweeps over the B-CSF layout, the C^(n) cache
refresh, and predict / RMSE -- driven from Python, computed by hand-written sm_100a kernels in
``libft_b200.so`` through a C ABI (include/ft_b200.h).  PyTorch holds device buffers only.
Names follow /root/reference/pkg/src/fastertucker/__init__.py:9-28.
"""

from ._kernels import BACKEND, COMPILED, get_backend, use_backend
from .cache import (DotCache, count_report, counted_sweep_cost, precompute_cache,
                    refresh_mode)
from .coo import (DatasetSplit, DeviceCoo, SparseCooTensor, generate_device,
                  generate_low_rank_device, generate_synthetic, load_coo, split_dataset,
                  write_coo)
from .counter import CHANNELS, OpCounter
from .csf import CsfForest, CsfTree, build_forest, build_tree
from .errors import (BackendUnavailableError, BuildError, ConfigError, CountMismatchError,
                     DivergenceError,
                     FasterTuckerError, ValidationError)
from .model import (InitSpec, Model, default_init_model, init_model, load_model, predict_batch,
                    save_model)
from .train import (EpochMetrics, METRICS_CSV_HEADER, TrainConfig, evaluate, run_epoch, train,
                    update_core_mode, update_factor_mode)

__version__ = "0.1.0"

__all__ = [
    "BACKEND", "COMPILED", "CHANNELS", "BackendUnavailableError", "BuildError", "ConfigError",
    "CountMismatchError", "count_report", "counted_sweep_cost",
    "CsfForest", "CsfTree", "DatasetSplit", "DeviceCoo", "DivergenceError", "DotCache",
    "EpochMetrics", "FasterTuckerError", "InitSpec", "METRICS_CSV_HEADER", "Model", "OpCounter",
    "SparseCooTensor", "TrainConfig", "ValidationError", "build_forest", "build_tree",
    "default_init_model", "evaluate", "generate_device", "generate_low_rank_device",
    "generate_synthetic", "get_backend", "init_model", "load_coo", "load_model",
    "precompute_cache", "predict_batch", "refresh_mode", "run_epoch", "save_model",
    "split_dataset", "train", "update_core_mode", "update_factor_mode", "use_backend",
    "write_coo",
]
