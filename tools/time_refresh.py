"""MEASUREMENT TOOL: K2 (ft_refresh, tcgen05) and its CUDA-core form (FT_REFRESH=simt) on the
Netflix32 shapes, CUDA events over 200 back-to-back launches, and the HBM fraction of the
I (J + R) 4 bytes each launch must move."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2210_06014_b200 import _lib  # noqa: E402

L = _lib.lib()
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6650.0
out = {}
for I in (480_189, 17_770, 2_182):
    J = R = 32
    A = torch.randn(I, J, device="cuda")
    Bt = torch.randn(R, J, device="cuda")
    C = torch.empty(I, R, device="cuda")
    g = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = _lib.stream_handle()
    for _ in range(10):
        L.ft_refresh(I, J, R, A.data_ptr(), Bt.data_ptr(), C.data_ptr(), g.data_ptr(), s)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(200):
        L.ft_refresh(I, J, R, A.data_ptr(), Bt.data_ptr(), C.data_ptr(), g.data_ptr(), s)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 200 * 1e3
    gbs = I * (J + R) * 4 / (us * 1e-6) / 1e9
    ref = (A.double() @ Bt.double().T)
    err = float((C.double() - ref).abs().max() / ref.abs().max())
    out[I] = {"us": us, "GB_per_s": gbs, "frac_of_hbm": gbs / peak, "rel_err": err}
    print(I, json.dumps(out[I]), flush=True)
