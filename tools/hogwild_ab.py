"""MEASUREMENT TOOL (not the product): hogwild (K3a) concurrency vs fidelity on a Netflix-dims
tensor (10 M train entries, J = R = 32, lr 1e-3): factor-sweep ms per mode and train / test
RMSE after 3 epochs for several hogwild_rows_per_warp, next to the exact schedule."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2210_06014_b200 as ft  # noqa: E402
from paper_2210_06014_b200 import train as T  # noqa: E402

dims = (480_189, 17_770, 2_182)
NNZ, NTEST, EPOCHS = 10_000_000, 140_000, 3
t = ft.generate_device(dims, NNZ + NTEST, (1.0, 5.0), seed=3)
train = ft.DeviceCoo(dims, t.idx[:NNZ].contiguous(), t.vals[:NNZ].contiguous())
test = ft.DeviceCoo(dims, t.idx[NNZ:].contiguous(), t.vals[NNZ:].contiguous())
forest = ft.build_forest(train, 128)
out = {}
for label, kw in [("exact", dict(schedule="exact"))] + [
        (f"hogwild/{r}", dict(schedule="hogwild", hogwild_rows_per_warp=r))
        for r in (256, 64, 16, 4, 1)]:
    model = ft.default_init_model(dims, (32,) * 3, 32, seed=1)
    cfg = ft.TrainConfig(epochs=EPOCHS, **kw)
    T.KERNEL_TIMES.clear() if hasattr(T, "KERNEL_TIMES") else None
    t0 = time.perf_counter()
    rows = ft.train(model, train, cfg, test_tensor=test, forest=forest)
    torch.cuda.synchronize()
    r = rows[-1]
    out[label] = {"train_rmse": r.train_rmse, "test_rmse": r.test_rmse,
                  "factor_ms_per_epoch": 1e3 * float(np.mean([x.factor_seconds for x in rows[1:]])),
                  "core_ms_per_epoch": 1e3 * float(np.mean([x.core_seconds for x in rows[1:]])),
                  "wall_s": time.perf_counter() - t0}
    print(label, json.dumps(out[label]), flush=True)
ex = out["exact"]
for k, v in out.items():
    v["train_gap"] = v["train_rmse"] / ex["train_rmse"] - 1
    v["test_gap"] = v["test_rmse"] / ex["test_rmse"] - 1
json.dump(out, open("gpurun_out/hogwild_ab.json", "w"), indent=1)
for k, v in out.items():
    print(f"{k:14s} factor {v['factor_ms_per_epoch']:8.2f} ms  train {v['train_rmse']:.6f} "
          f"({100 * v['train_gap']:+.3f} %)  test {v['test_rmse']:.6f} ({100 * v['test_gap']:+.3f} %)")
