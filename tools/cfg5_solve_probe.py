"""Drive config 5 solves (CSR or matrix-free stencil) — or config 4's FFT
lattice operator (--op toeplitz4) — for an ncu launch list
(perf only): a fixed iteration count (tol 0), so `ncu --cache-control none`
sees the L2 state of a real solve.

usage: python tools/cfg5_solve_probe.py [--op stencil|csr] [--methods bicgstab] [--its 6] [--reps 1]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_4869_b200 as ccg  # noqa: E402
from workloads import helmholtz_csr, helmholtz_rhs, helmholtz_coeffs, cfg4_rhs, dda_kernel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--op", default="stencil")
ap.add_argument("--methods", default="bicgstab")
ap.add_argument("--its", type=int, default=6)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
N = 128
n = N ** 3
y = torch.from_numpy(helmholtz_rhs(N) if a.op != "toeplitz4" else cfg4_rhs()).cuda()
n = y.numel()
x = torch.empty_like(y)
h = ccg.ccg_create("c128", n)
if a.op == "toeplitz4":
    ccg.ccg_set_matvec_toeplitz3(h, 64, 32, 32, dda_kernel((64, 32, 32), 0.5), 2.5 + 0.2j)
elif a.op == "csr":
    rp, ci, v = (torch.from_numpy(t).cuda() for t in helmholtz_csr(N))
    ccg.ccg_set_matvec_csr(h, rp, ci, v, 0, n, v.numel())
else:
    d, o = helmholtz_coeffs()
    ccg.ccg_set_matvec_stencil7(h, N, N, N, d, o)
for m in a.methods.split(","):
    for _ in range(a.reps):
        r = ccg.ccg_solve(h, m, None, y, x, 0.0, a.its)
    print(m, r["iterations"], r["status"], flush=True)
ccg.ccg_destroy(h)
