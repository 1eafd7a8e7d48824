"""MEASUREMENT TOOL: per-rank sweep times of the row-block sharded epoch (dist.py) on ONE GPU.

For P in 1, 2, 4, 8 and every mode u, the rank with the most entries in dist.plan_blocks' cut
gets its shard tree built (CudaEngine.build_shard, exactly what DistTrainer builds) and its
factor sweep and core partial timed with CUDA events (median of 5).  The slowest rank per mode
bounds the P-GPU epoch (every sweep ends in a C_u all-gather / core all-reduce), so

    T(P) = sum_u max_rank factor_u + max_rank core_u + refresh + comm

is the measured-input scaling model DESIGN.md section 6 quotes.  Prints one JSON line per
config.  python tools/time_shards.py [netflix32 ...]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2210_06014_b200 as ft  # noqa: E402
from paper_2210_06014_b200 import dist as D  # noqa: E402


def median_ms(fn, reps=5):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["netflix32"])
    ap.add_argument("--P", type=int, nargs="*", default=[1, 2, 4, 8])
    ap.add_argument("--modes", type=int, nargs="*", default=None)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    names = args.configs
    for name in names:
        cfg = bench.CONFIGS[name]
        dims, J, R = cfg["dims"], cfg["J"], cfg["R"]
        N = len(dims)
        coo = ft.generate_device(dims, cfg["nnz_train"], cfg["value_range"], seed=0)
        model = ft.default_init_model(dims, (J,) * N, R, seed=0)
        cache = ft.precompute_cache(model)
        dots = cache.arrays
        eng = D.CudaEngine()
        counts = [eng.mode_counts(coo, u, dims[u]) for u in range(N)]
        out = {"config": name, "dims": list(dims), "nnz": int(coo.nnz), "J": J, "R": R, "P": {}}
        for P in args.P:
            blocks = D.plan_blocks(counts, P)
            per = {}
            for u in (args.modes if args.modes is not None else range(N)):
                b = blocks[u]
                nnzs = [int(counts[u][b[p]:b[p + 1]].sum()) for p in range(P)]
                p = int(np.argmax(nnzs))
                tree, nnz, _ = eng.build_shard(coo, u, int(b[p]), int(b[p + 1]), 128)
                shard = D.ModeShard(u, int(b[p]), int(b[p + 1]), tree, nnz, -1)
                eng.factor_sweep(shard, model, dots, 0.0, 0.0)  # slot layout + warm-up
                torch.cuda.synchronize()
                f = median_ms(lambda: eng.factor_sweep(shard, model, dots, 0.0, 0.0), args.reps)
                c = median_ms(lambda: eng.core_partial(shard, model, dots, u))
                rf = median_ms(lambda: eng.refresh_block(model, u, int(b[p]), int(b[p + 1]),
                                                         dots[u], None))
                per[u] = {"rows": int(b[p + 1] - b[p]), "nnz": nnz, "factor_ms": f,
                          "core_ms": c, "refresh_ms": rf}
                del shard, tree
                torch.cuda.empty_cache()
            tot = sum(v["factor_ms"] + v["core_ms"] + 2 * v["refresh_ms"] for v in per.values())
            out["P"][P] = {"modes": per, "compute_ms": tot}
            print(name, P, {u: (round(v["factor_ms"], 3), round(v["core_ms"], 3)) for u, v in per.items()},
                  round(tot, 3), file=sys.stderr, flush=True)
        if 1 in out["P"]:
            base = out["P"][1]["compute_ms"]
            out["speedup_compute_only"] = {P: base / out["P"][P]["compute_ms"] for P in out["P"]}
        print(json.dumps(out), flush=True)
        del coo, model, cache
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
