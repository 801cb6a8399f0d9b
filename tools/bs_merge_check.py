"""CCG_BS_MERGE=1 (BiCGSTAB X and P passes merged, methods.cuh BsTm / BsXP) against the default path
and the oracle on the N = 16 / 24 Helmholtz lattice (stencil and CSR): iteration counts, x at equal k,
true residual.  perf: tools/ab_env.py --config 5 --op stencil --knob CCG_BS_MERGE=0,1."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from tests._gpu import Csr  # noqa: E402
from tests.test_gpu_next import Stencil  # noqa: E402
from workloads import lattice_csr, helmholtz_coeffs, helmholtz_rhs  # noqa: E402
from oracle import CsrOp  # noqa: E402

for N in (16, 24):
    d, o = helmholtz_coeffs()
    rp, ci, v = lattice_csr(N, N, N, d, o)
    y = helmholtz_rhs(N)
    op = CsrOp(rp, ci, v)
    ref = oracle.solve("bicgstab", op, y, 1e-8, 4000)
    for kind in ("stencil", "csr"):
        res = {}
        for m in ("0", "1"):
            os.environ["CCG_BS_MERGE"] = m
            with (Stencil(N, N, N, d, o) if kind == "stencil" else Csr(rp, ci, v, N ** 3)) as h:
                g = h.solve("bicgstab", y, 1e-8, 4000)
                k = min(g["iterations"], ref.iterations) - 2
                gk = h.solve("bicgstab", y, 0.0, k)
            ok = oracle.solve("bicgstab", op, y, 0.0, k)
            res[m] = (g["status"], g["iterations"], g["true_rel_res"],
                      np.linalg.norm(gk["x"] - ok.x) / np.linalg.norm(ok.x))
        print(N, kind, "oracle k", ref.iterations, "default", res["0"], "merged", res["1"], flush=True)
