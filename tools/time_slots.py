"""MEASUREMENT TOOL: K1d slot layout cost on the Netflix32 trees (plan + fill per tree)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2210_06014_b200 as ft  # noqa: E402

dims = (480_189, 17_770, 2_182)
t = ft.generate_device(dims, 99_072_112, (1.0, 5.0), seed=0)
for rep in range(3):
    forest = ft.build_forest(t, 128, compact=True)
    torch.cuda.synchronize()
    for tree in forest.trees:
        t0 = time.perf_counter()
        tree.ensure_slots(32, 32)
        torch.cuda.synchronize()
        print(f"rep {rep} tree {tree.root_mode}: rows {tree.num_rows} grid {tree.slot_grid} kb {tree.slot_kb} "
              f"{1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
