"""Drive the dense matvec kernels once each for an ncu capture (perf only).

A·x split (default), A·x column-owner (CCG_GEMV=cols), Aᴴ·x (stage 1) and the
QMR dual product on a c64 n = 32768 random matrix."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_4869_b200 as ccg  # noqa: E402

n = int(os.environ.get("PROF_N", 32768))
dt = os.environ.get("PROF_DT", "c64")
tdt = torch.complex64 if dt == "c64" else torch.complex128
A = torch.randn((n, n), dtype=tdt, device="cuda") * (0.5 / n ** 0.5)
A.diagonal().add_(2 + 0.3j)
x = torch.randn(n, dtype=tdt, device="cuda")
y = torch.empty_like(x)
for mode in ("split", "cols"):
    os.environ["CCG_GEMV"] = mode
    h = ccg.ccg_create(dt, n)
    ccg.ccg_set_matvec_dense(h, A, 0, n)
    for _ in range(2):
        ccg.ccg_apply(h, "A", x, y)
    if mode == "split":
        for _ in range(2):
            ccg.ccg_apply(h, "AH", x, y)
        ccg.ccg_solve(h, "qmr", None, x, y, 0.0, 3)
    ccg.ccg_destroy(h)
torch.cuda.synchronize()
print("ok")
