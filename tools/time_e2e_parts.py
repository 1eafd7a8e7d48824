"""Break the bench's end-to-end step (H2D, B-CSF build, cache, epoch, RMSE) into timed parts."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_06014_b200 as ft  # noqa: E402
import importlib  # noqa: E402

from paper_2210_06014_b200 import csf  # noqa: E402

T = importlib.import_module("paper_2210_06014_b200.train")


def timed(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{name:28s} {1e3 * min(ts):8.2f} ms", flush=True)
    return out


dims = (480_189, 17_770, 2_182)
split = ft.generate_synthetic(dims, 100_480_507, (1.0, 5.0), seed=0, test_fraction=1_408_395 / 100_480_507)
tr = split.train
idx_h, vals_h = tr.idx.cpu().pin_memory(), tr.vals.cpu().pin_memory()
idx_d, vals_d = torch.empty_like(idx_h, device="cuda"), torch.empty_like(vals_h, device="cuda")
timed("H2D COO (pinned)", lambda: (idx_d.copy_(idx_h, non_blocking=True), vals_d.copy_(vals_h, non_blocking=True)))
dev = ft.DeviceCoo(dims, idx_d, vals_d)
for t in range(3):
    timed(f"build_tree {t} (compact)", lambda: csf.build_tree(dev, t, 128, compact=True))
tree = csf.build_tree(dev, 0, 128, compact=True)
timed("  leaf index + segments", lambda: csf.add_leaf_index(tree))
forest = timed("build_forest (compact)", lambda: ft.build_forest(dev, 128, compact=True))
model = ft.default_init_model(dims, (32,) * 3, 32, seed=0)
cache = timed("precompute_cache", lambda: ft.precompute_cache(model, ft.OpCounter()))
tcfg = ft.TrainConfig(epochs=1)
timed("epoch (no eval)", lambda: [T.update_factor_mode(model, forest, cache, n, tcfg, ft.OpCounter()) for n in range(3)]
      + [T.update_core_mode(model, forest, cache, n, tcfg, ft.OpCounter()) for n in range(3)])
timed("evaluate train", lambda: ft.evaluate(model, dev, cache))

# the bench's e2e step, part by part (CUDA events on the current stream)
init_f, init_c = [a.clone() for a in model.factors], [b.clone() for b in model.cores_t]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record()
    dev2 = ft.DeviceCoo(dims, idx_d, vals_d)
    m2 = ft.Model(dims, (32,) * 3, 32, init_f, init_c)
    ev[1].record()
    f2 = ft.build_forest(dev2, 128, compact=True, keep_fibers=False)
    ev[2].record()
    c2 = ft.precompute_cache(m2, ft.OpCounter())
    t_s0 = time.perf_counter()
    for tt in f2.trees:  # the K3c slot layouts (K1d), otherwise built inside the first sweep
        tt.ensure_slots(32, 32)
    torch.cuda.synchronize()
    print(f"  slot layouts (K1d)        {1e3 * (time.perf_counter() - t_s0):8.2f} ms", flush=True)
    ev[3].record()
    met = T.run_epoch(m2, f2, c2, dev2, tcfg, ft.OpCounter(), 1, None, evaluate_metrics=False)
    ev[4].record()
    r = ft.evaluate(m2, dev2, c2, f2)
    ev[5].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    names = ["model/coo", "build_forest", "cache", "epoch", "evaluate(tree)"]
    print("e2e step:", " ".join(f"{n} {ev[i].elapsed_time(ev[i + 1]):.2f}" for i, n in enumerate(names)),
          f"| wall {1e3 * wall:.2f} ms", flush=True)
