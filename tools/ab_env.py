"""Interleaved A/B of CCG_* knobs read at set_matvec time, on config 1 / 2 dense
(c128 n = 256 / 4096) or config 5 (CSR / stencil): one handle per setting, then R
rounds alternating between the settings (median µs per iteration per method),
so clock drift and warm-up do not favour a position.

usage: python tools/ab_env.py --config 2 --knob CCG_COLS_FUSE=0,1 [--methods bicgstab,cocr] [--rounds 7]
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
from workloads import cfg1, cfg2, cfg4_rhs, dda_kernel, helmholtz_csr, helmholtz_rhs, helmholtz_coeffs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--op", default="dense")
    ap.add_argument("--knob", action="append", default=[])
    ap.add_argument("--methods", default="bicgstab,cocr")
    ap.add_argument("--rounds", type=int, default=7)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--sym", action="store_true", help="dense: pass CCG_FLAG_SYMMETRIC (A = Aᵀ)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    if a.config == 4:                    # the FFT lattice operator (64 × 32 × 32)
        y = torch.from_numpy(cfg4_rhs()).to(dev)
        n = y.numel()
        kern = dda_kernel((64, 32, 32), 0.5)
    elif a.config in (1, 2):
        A, y = cfg1() if a.config == 1 else cfg2()
        A, y = torch.from_numpy(A).to(dev), torch.from_numpy(y).to(dev)
        n = y.numel()
    else:
        N = 128
        n = N ** 3
        y = torch.from_numpy(helmholtz_rhs(N)).to(dev)
        if a.op == "csr":
            rp, ci, v = helmholtz_csr(N)
            rpd, cid, vd = (torch.from_numpy(t).to(dev) for t in (rp, ci, v))
    names = [k.split("=")[0] for k in a.knob]
    combos = list(itertools.product(*[k.split("=")[1].split(",") for k in a.knob]))
    hs = []
    for combo in combos:
        for k, v in zip(names, combo):
            os.environ[k] = v
        h = ccg.ccg_create("c128", n)
        if a.config == 4:
            ccg.ccg_set_matvec_toeplitz3(h, 64, 32, 32, kern, 2.5 + 0.2j)
        elif a.config in (1, 2):
            ccg.ccg_set_matvec_dense(h, A, 0, n, flags=ccg.FLAG_SYMMETRIC if a.sym else 0)
        elif a.op == "csr":
            ccg.ccg_set_matvec_csr(h, rpd, cid, vd, 0, n, vd.numel())
        else:
            d, o = helmholtz_coeffs()
            ccg.ccg_set_matvec_stencil7(h, N, N, N, d, o, o, o)
        # warm solves while this setting's environment is in place (workspaces
        # sized at the first solve read their knobs then)
        for m in a.methods.split(","):
            ccg.ccg_solve(h, m, None, y, torch.empty_like(y), a.tol, 5000)
        hs.append(h)
    x = torch.empty_like(y)
    streams = [torch.cuda.ExternalStream(ccg.ccg_get_stream(h)) for h in hs]
    meths = a.methods.split(",")
    torch.cuda.synchronize()
    t = {(k, m): [] for k in range(len(hs)) for m in meths}
    its = {}
    for _ in range(a.rounds):
        for k, h in enumerate(hs):
            for m in meths:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(streams[k])
                r = ccg.ccg_solve(h, m, None, y, x, a.tol, 5000)
                e1.record(streams[k])
                torch.cuda.synchronize()
                t[(k, m)].append(e0.elapsed_time(e1) * 1e3 / max(1, r["iterations"]))
                its[(k, m)] = (r["iterations"], r["status"], r["true_rel_res"])
    med = lambda v: sorted(v)[len(v) // 2]
    for k, combo in enumerate(combos):
        line = dict(zip(names, combo), config=a.config, op=a.op, rounds=a.rounds)
        for m in meths:
            line[m + "_us_per_it_median"] = med(t[(k, m)])
            line[m + "_its"], line[m + "_status"], line[m + "_true_rel_res"] = its[(k, m)]
        print(json.dumps(line), flush=True)
    for h in hs:
        ccg.ccg_destroy(h)


if __name__ == "__main__":
    main()
