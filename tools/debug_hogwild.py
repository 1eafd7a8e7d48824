import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2210_06014_b200 as ft
from paper_2210_06014_b200 import _lib
from oracle import oracle as O
z = np.load("tests/golden/config1.npz")
idx = z["train_idx"].astype(np.int64); vals = z["train_vals"]
f0 = [np.array(z[f"init/A{n}"]) for n in range(3)]; c0 = [np.array(z[f"init/B{n}"]) for n in range(3)]
dev = ft.DeviceCoo((1000,)*3, torch.from_numpy(idx.astype(np.int32)).cuda(), torch.from_numpy(vals.astype(np.float32)).cuda())
forest = ft.build_forest(dev, 128)
oforest = O.build_forest(idx, vals, 128)
L = _lib.lib()
for hi in (32, 256, 4096, None):
    m = ft.Model((1000,)*3, (8,)*3, 8, f0, c0)
    cache = ft.precompute_cache(m)
    tree = forest.trees[0]
    hi_ = tree.num_fibers if hi is None else hi
    _lib.check(L.ft_factor_sweep_fibers(ctypes.byref(tree.view()), ctypes.byref(m.view(cache.arrays)), 0, hi_, 1e-3, 1e-2, 0, None))
    torch.cuda.synchronize()
    om = O.OracleModel((1000,)*3, (8,)*3, 8, [a.copy() for a in f0], [b.copy() for b in c0])
    oc = O.precompute_cache(om)
    t = oforest[0]
    O.CKernels.factor_sweep(t.leaf_coord, t.vals, t.fiber_ptr, t.fiber_coord, t.prefix_modes, 2, om.factors, om.cores_t, oc, 1e-3, 1e-2, np.zeros(5, np.int64), 0, hi_)
    got = m.factors[2].cpu().numpy()
    d = got - om.factors[2]
    print(hi_, "max|A| gpu", np.abs(got).max(), "oracle", np.abs(om.factors[2]).max(), "max diff", np.abs(d).max(), "changed rows gpu", int((np.abs(got - f0[2]).max(1) > 0).sum()), "oracle", int((np.abs(om.factors[2]-f0[2]).max(1)>0).sum()))
