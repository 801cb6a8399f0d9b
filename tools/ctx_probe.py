"""Probe: A·x / Aᴴ·x bandwidth vs matrix data (random vs cfg3) and call order (perf only)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_4869_b200 as ccg  # noqa: E402
from workloads import gauss_shifted_rows, cfg3_rhs  # noqa: E402

n = 32768
A = torch.empty((n, n), dtype=torch.complex64, device="cuda")
pin = torch.empty((4096, n), dtype=torch.complex64).pin_memory()
for r0 in range(0, n, 4096):
    gauss_shifted_rows(n, r0, r0 + 4096, seed=1, out=pin.numpy())
    A[r0:r0 + 4096].copy_(pin)
xs = {"cfg3rhs": torch.from_numpy(cfg3_rhs(n)).cuda(), "randn": torch.randn(n, dtype=torch.complex64, device="cuda")}
h = ccg.ccg_create("c64", n)
ccg.ccg_set_matvec_dense(h, A, 0, n)
y = torch.empty(n, dtype=torch.complex64, device="cuda")
ccg.ccg_set_timing(h, 1)
for xn, x in xs.items():
    for order in (("A",) * 6, ("AH",) * 6, ("A", "AH") * 3):
        t = {"A": [], "AH": []}
        for op in order * 2:
            ccg.ccg_apply(h, op, x, y)
            tt = ccg.ccg_get_timing(h)
            t[op].append(tt["ms_a"] + tt["ms_ah"])
        res = {k: round(n * n * 8 / (sum(v[2:]) / len(v[2:]) * 1e-3) / 1e9) for k, v in t.items() if len(v) > 2}
        print(xn, "-".join(order[:2]), res, flush=True)
# random matrix data
A.copy_(torch.randn((n, n), dtype=torch.complex64, device="cuda") * 0.002)
for order in (("A",) * 6, ("AH",) * 6):
    t = {"A": [], "AH": []}
    for op in order * 2:
        ccg.ccg_apply(h, op, xs["randn"], y)
        tt = ccg.ccg_get_timing(h)
        t[op].append(tt["ms_a"] + tt["ms_ah"])
    print("randA", order[0], {k: round(n * n * 8 / (sum(v[2:]) / len(v[2:]) * 1e-3) / 1e9) for k, v in t.items() if len(v) > 2})
