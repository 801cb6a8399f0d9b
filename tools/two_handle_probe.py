"""Two handles in one process, methods run in sequence on each (debug probe)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_4869_b200 as ccg
from workloads import helmholtz_rhs, helmholtz_coeffs
N = int(sys.argv[1])
meths = sys.argv[2].split(",")
envs = sys.argv[3].split(",") if len(sys.argv) > 3 else ["1", "4"]
y = torch.from_numpy(helmholtz_rhs(N)).cuda()
d, o = helmholtz_coeffs()
hs = []
for e in envs:
    os.environ["CCG_STENCIL_MINB"] = e
    h = ccg.ccg_create("c128", N ** 3)
    ccg.ccg_set_matvec_stencil7(h, N, N, N, d, o, o, o)
    for m in meths:
        r = ccg.ccg_solve(h, m, None, y, torch.empty_like(y), 1e-8, 5000)
        torch.cuda.synchronize()
        print(e, m, r["iterations"], r["status"], flush=True)
    hs.append(h)
