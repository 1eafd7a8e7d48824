"""K3c, the tcgen05 factor sweep (csrc/factor_tc.cu: combine on tcgen05 with the A operand in
TMEM, one thread per row, slot layout K1d), against the fp64 oracle at the contract's rel 1e-4
per sweep, and the slot layout itself against the tree it was built from.

The default dispatch runs K3c on trees with enough rows to fill the GPU (one 128-slot CTA on
>= 90 % of the SMs) when 16 < R <= 32; with FT_TC_WIDE=1 (set here), K3c-wide (16 rows x 8
leaves per batch, the chains in two 4-lanes-per-row warps) takes order-3 trees with fewer but
long rows (>= 0.9 x 16 per SM, >= 64 leaves each):
each case below has at least one such mode; the other modes run quadr / quadw as usual, so
every sweep of two epochs is checked.  Cases: short rows (1-3 leaves, J < 32 and R < 32
padding, R % 8 = 4), more rows than slots (row switching inside a slot's stream), rows of
a hundred leaves, order 4 (two prefix levels), J = 16 / R = 24, and both chain forms
(plain fp32 and the Fast2Sum-compensated one, FT_TC_COMP).
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from test_quad_gpu import _CASE

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ft():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2210_06014_b200 as ft

    return ft


@pytest.mark.parametrize("dims,nnz,J,R,lr,comp", [
    ((20000, 700, 9), 300_000, 24, 20, 1e-3, "0"),    # 1-3 leaf rows, padding, R % 8 = 4
    ((60000, 20000, 64), 1_000_000, 32, 32, 5e-3, "0"),  # two tc modes, row switching
    ((20000, 300, 50), 2_000_000, 32, 32, 2e-3, "1"),  # ~100-leaf rows, compensated chain
    ((20000, 300, 50), 2_000_000, 32, 32, 2e-3, "0"),
    ((20000, 10000, 30, 20), 600_000, 32, 32, 2e-3, "0"),  # order 4
    ((20000, 300, 40), 400_000, 16, 24, 2e-3, "1"),   # J = 16, R = 24
    # K3c-wide (KB = 8: 16 rows per CTA, a chain warp) for few long rows:
    ((3000, 2500, 400), 2_000_000, 32, 32, 2e-3, "0"),  # modes 0 and 1: 667 / 800-leaf rows
    ((2400, 500, 100), 500_000, 24, 20, 1e-3, "0"),     # padding, row switching in a batch
    ((2300, 64, 64), 1_500_000, 32, 32, 2e-3, "1"),     # 650-leaf rows, compensated chain
])
def test_tc_factor_sweeps_match_oracle(dims, nnz, J, R, lr, comp):
    code = _CASE.format(dims=dims, nnz=nnz, J=J, R=R, lr=lr, seed=11)
    # FT_TC_WIDE=1 opts the few-long-rows shapes into K3c-wide (not dispatched by default)
    env = dict(os.environ, FT_TC_COMP=comp, FT_TC_WIDE="1")
    env.pop("FT_FACTOR_KERNEL", None)
    env.pop("FT_FACTOR_TC", None)
    out = subprocess.run([sys.executable, "-c", code], cwd=REPO, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


def test_slot_layout_covers_every_leaf_once(ft):
    """K1d: slot q = c + G s owns the contiguous rows [q rows / GS, (q + 1) rows / GS); per CTA c
    and slot s the non-padding entries [batch][s] are exactly those rows' leaves in order, the
    first leaf of each row flagged, and every leaf appears once."""
    import torch

    rng = np.random.default_rng(2)
    dims = (30000, 50, 40)
    lin = rng.choice(int(np.prod(dims)), size=500_000, replace=False)
    idx = np.stack(np.unravel_index(lin, dims), axis=1)
    dev = ft.DeviceCoo(dims, torch.from_numpy(idx.astype(np.int32)).cuda(),
                       torch.from_numpy(rng.uniform(1, 5, len(lin)).astype(np.float32)).cuda())
    tree = ft.build_tree(dev, 0, 128).ensure_slots(32, 32)
    G = tree.slot_grid
    assert G > 0 and tree.slot_kb == 1
    bp = tree.slot_batch_ptr.cpu().numpy()
    lc = tree.slot_lc.cpu().numpy().view(np.uint32)
    pc = tree.slot_pc.cpu().numpy()
    x = tree.slot_x.cpu().numpy()
    rlp = tree.row_leaf_ptr.cpu().numpy()
    leaf_coord = tree.leaf_coord.cpu().numpy()
    leaf_pc = tree.leaf_pc.cpu().numpy().reshape(-1)
    vals = tree.vals.cpu().numpy()
    rows, GS = tree.num_rows, 128 * G
    seen = 0
    for c in range(G):
        for s in range(128):
            q = c + G * s
            r0, r1 = q * rows // GS, (q + 1) * rows // GS
            want = [(int(leaf_coord[L]) | (0x80000000 if L == rlp[r] else 0), int(leaf_pc[L]),
                     float(vals[L])) for r in range(r0, r1) for L in range(rlp[r], rlp[r + 1])]
            e = np.arange(bp[c], bp[c + 1]) * 128 + s
            live = lc[e] != 0xFFFFFFFF
            got = list(zip(lc[e][live].astype(int).tolist(), pc[e][live].tolist(),
                           x[e][live].astype(float).tolist()))
            assert got == want, (c, s)
            assert not live[len(want):].any()  # padding only at the end of the stream
            seen += len(got)
    assert seen == tree.nnz
    assert bp[-1] * 128 == tree.slot_lc.numel()
