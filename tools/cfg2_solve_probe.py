"""Drive config 2 dense solves for an ncu launch list / capture (perf only).

Config 2 (c128 n = 4096 DDA lattice, BJ:8) with a fixed iteration count per
method (tol 0), so an ncu capture with --cache-control none sees the L2
state a real solve has (pinned rows of A resident from product to product).

usage: python tools/cfg2_solve_probe.py [--methods bicgstab] [--its 20] [--reps 2]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_4869_b200 as ccg  # noqa: E402
from workloads import cfg2  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--methods", default="bicgstab")
ap.add_argument("--its", type=int, default=20)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--timing", action="store_true", help="per-product CUDA events (library timing mode)")
ap.add_argument("--sym", action="store_true", help="CCG_FLAG_SYMMETRIC (upper-triangle products)")
a = ap.parse_args()
A, y = cfg2()
Ad = torch.from_numpy(A).cuda()
yd = torch.from_numpy(y).cuda()
x = torch.empty_like(yd)
h = ccg.ccg_create("c128", A.shape[0])
ccg.ccg_set_matvec_dense(h, Ad, 0, A.shape[0], flags=ccg.FLAG_SYMMETRIC if a.sym else 0)
ccg.ccg_set_timing(h, a.timing)
for m in a.methods.split(","):
    for _ in range(a.reps):
        r = ccg.ccg_solve(h, m, None, yd, x, 0.0, a.its)
    line = f"{m} its={r['iterations']} {r['status']}"
    if a.timing:
        t = ccg.ccg_get_timing(h)
        line += (f" A: {1e3 * t['ms_a'] / max(1, t['n_a']):.1f} us x{t['n_a']}"
                 f" AH: {1e3 * t['ms_ah'] / max(1, t['n_ah']):.1f} us x{t['n_ah']}")
    print(os.environ.get("CCG_L2_PIN_MB", "-"), os.environ.get("CCG_SPLIT_FUSE", "-"), line, flush=True)
torch.cuda.synchronize()
ccg.ccg_destroy(h)
