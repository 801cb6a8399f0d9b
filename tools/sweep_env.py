"""Config 5 (CSR or stencil operator): sweep CCG_* environment knobs read at
set_matvec time.  Per setting: ccg_apply(A) time (CUDA events, 200 calls on
the library stream) and BiCGSTAB / COCR µs per iteration; one JSON line each.

usage: python tools/sweep_env.py --op stencil --knob CCG_STENCIL_U=1,2,4 [--knob CCG_STENCIL_ZC=4,8]
"""

import argparse
import itertools
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_4869_b200 as ccg  # noqa: E402
from workloads import helmholtz_csr, helmholtz_rhs, helmholtz_coeffs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="stencil")
    ap.add_argument("--knob", action="append", default=[])
    ap.add_argument("--dtype", default="c128")
    ap.add_argument("--methods", default="bicgstab,cocr")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    N = 128
    n = N ** 3
    cdt = torch.complex128 if a.dtype == "c128" else torch.complex64
    y = torch.from_numpy(helmholtz_rhs(N)).to(dev).to(cdt)
    x = torch.empty_like(y)
    if a.op == "csr":
        rp, ci, v = helmholtz_csr(N)
        rpd, cid = torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev)
        vd = torch.from_numpy(v).to(dev).to(cdt)
    names = [k.split("=")[0] for k in a.knob]
    values = [k.split("=")[1].split(",") for k in a.knob]
    ref = None
    for combo in itertools.product(*values):
        for k, v in zip(names, combo):
            os.environ[k] = v
        h = ccg.ccg_create(a.dtype, n)
        if a.op == "csr":
            ccg.ccg_set_matvec_csr(h, rpd, cid, vd, 0, n, len(v))
        else:
            d, o = helmholtz_coeffs()
            ccg.ccg_set_matvec_stencil7(h, N, N, N, d, o, o, o)
        stream = torch.cuda.ExternalStream(ccg.ccg_get_stream(h))
        out = torch.empty_like(y)
        for _ in range(5):
            ccg.ccg_apply(h, "A", y, out)
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        line = dict(zip(names, combo), op=a.op, dtype=a.dtype, bitwise_equal_first=bool(torch.equal(out, ref)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(200):
            ccg.ccg_apply(h, "A", y, out)
        e1.record(stream)
        torch.cuda.synchronize()
        line["apply_us"] = e0.elapsed_time(e1) * 1e3 / 200
        for meth in a.methods.split(","):
            ccg.ccg_solve(h, meth, None, y, x, 1e-8, 5000)
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            r = ccg.ccg_solve(h, meth, None, y, x, 1e-8, 5000)
            t1.record(stream)
            torch.cuda.synchronize()
            line[meth + "_us_per_it"] = t0.elapsed_time(t1) * 1e3 / max(1, r["iterations"])
            line[meth + "_its"] = r["iterations"]
        ccg.ccg_destroy(h)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
