"""Config 5 CSR: SELL-32 SpMV load schedule × grid waves (CCG_SELL_ONE = 0
two rows per step / 1 one row per step at ≥ 3 CTAs/SM; CCG_SELL_WAVES).  Times ccg_apply(A) alone (CUDA events, 200 launches) and a
BiCGSTAB / COCR solve per setting; one JSON line each.

usage: python tools/sweep_sell.py [--modes 0,1] [--waves 1,4]
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_4869_b200 as ccg  # noqa: E402
from workloads import helmholtz_csr, helmholtz_rhs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", default="0,1")
    ap.add_argument("--waves", default="1")
    ap.add_argument("--dtype", default="c128")
    ap.add_argument("--rounds", type=int, default=7)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    N = 128
    n = N ** 3
    cdt = torch.complex128 if a.dtype == "c128" else torch.complex64
    rp, ci, v = helmholtz_csr(N)
    rpd, cid = torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev)
    vd = torch.from_numpy(v).to(dev).to(cdt)
    y = torch.from_numpy(helmholtz_rhs(N)).to(dev).to(cdt)
    x = torch.empty_like(y)
    s = 16 if a.dtype == "c128" else 8
    b_spmv = len(v) * (s + 4) + 2 * n * s
    # every setting gets its own handle up front; the timed solves then
    # alternate between settings (R rounds, median) so clock drift and
    # warm-up do not favour one position in the sweep
    settings = [(m, w) for m in a.modes.split(",") for w in a.waves.split(",")]
    hs = []
    for m, w in settings:
        os.environ["CCG_SELL_ONE"], os.environ["CCG_SELL_WAVES"] = m, w
        h = ccg.ccg_create(a.dtype, n)
        ccg.ccg_set_matvec_csr(h, rpd, cid, vd, 0, n, len(v))
        hs.append(h)
    stream = [torch.cuda.ExternalStream(ccg.ccg_get_stream(h)) for h in hs]
    outs = [torch.empty_like(y) for _ in hs]
    for h, o in zip(hs, outs):
        for _ in range(5):
            ccg.ccg_apply(h, "A", y, o)
    torch.cuda.synchronize()
    res = {k: {"spmv_us": [], "bicgstab": [], "cocr": []} for k in range(len(hs))}
    its = {}
    for _ in range(a.rounds):
        for k, h in enumerate(hs):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream[k])
            for _ in range(100):
                ccg.ccg_apply(h, "A", y, outs[k])
            e1.record(stream[k])
            torch.cuda.synchronize()
            res[k]["spmv_us"].append(e0.elapsed_time(e1) * 1e3 / 100)
            for meth in ("bicgstab", "cocr"):
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record(stream[k])
                r = ccg.ccg_solve(h, meth, None, y, x, 1e-8, 5000)
                t1.record(stream[k])
                torch.cuda.synchronize()
                res[k][meth].append(t0.elapsed_time(t1) * 1e3 / max(1, r["iterations"]))
                its[(k, meth)] = r["iterations"]
    med = lambda v: sorted(v)[len(v) // 2]
    for k, (m, w) in enumerate(settings):
        same = bool(torch.equal(outs[k], outs[0]))
        print(json.dumps({"sell_one": int(m), "waves": int(w), "dtype": a.dtype, "rounds": a.rounds,
                          "spmv_call_us_median": med(res[k]["spmv_us"]),
                          "bicgstab_us_per_it_median": med(res[k]["bicgstab"]), "bicgstab_its": its[(k, "bicgstab")],
                          "cocr_us_per_it_median": med(res[k]["cocr"]), "cocr_its": its[(k, "cocr")],
                          "bitwise_equal_first": same, "b_spmv_bytes": b_spmv}), flush=True)
    for h in hs:
        ccg.ccg_destroy(h)


if __name__ == "__main__":
    main()
