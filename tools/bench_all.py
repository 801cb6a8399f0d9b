"""Throughput of every config × method on one B200.

For each BASELINE config: repeated tolerance-driven ccg_solve calls (graphs on,
no per-kernel timing), iterations/s = Σ iterations / Σ device time, plus the
effective bandwidth of the algorithmic bytes (SURVEY §8(a):
B_iter = m·B_mat + v·n·s).  One JSON line per (config, method).

usage: python tools/bench_all.py [--configs 1,2,3,4,5] [--reps R]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1208_4869_b200 as ccg  # noqa: E402
from workloads import (cfg1, cfg2, gauss_shifted_rows, cfg3_rhs, cfg4_rhs, helmholtz_csr,  # noqa: E402
                       helmholtz_rhs, helmholtz_coeffs, dda_kernel, CONFIGS)
from workloads.device import cfg4_rows_device  # noqa: E402

V_PASSES = {"bicgstab": 18, "cgne": 10, "qmr": 26, "bicor": 24, "cors": 24,
            "bicg": 18, "cgs": 16, "cocr": 14, "cgnr": 11, "tfqmr": 28, "gmres": 0, "bicgstabl": 16, "pbicgstab": 26}      # NEXT-3
M_MATVEC = {"bicgstab": 2, "cgne": 2, "qmr": 2, "bicor": 2, "cors": 2,
            "bicg": 2, "cgs": 2, "cocr": 1, "cgnr": 2, "tfqmr": 2, "gmres": 1, "bicgstabl": 2, "pbicgstab": 2}
if os.environ.get("CCG_QMR_DUAL", "1") != "0":
    M_MATVEC["qmr"] = 1                  # dual GEMV: A·p and Aᴴ·q in one pass
    M_MATVEC["bicg"] = 1
KNOBS = {k: v for k, v in os.environ.items() if k.startswith("CCG_")}
ALL = ("bicgstab", "cgne", "qmr", "bicor", "cors", "bicg", "cgs", "cgnr", "tfqmr", "gmres", "bicgstabl", "pbicgstab")
SYM = ALL + ("cocr",)                    # complex-symmetric configs (2, 4, 5) also run COCR
SEL = set()


def timed(h, method, y, x, tol, maxit, reps, stream):
    r = ccg.ccg_solve(h, method, None, y, x, tol, maxit)          # warm (graph capture)
    its, ms = 0, 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        e0.record(stream)
        r = ccg.ccg_solve(h, method, None, y, x, tol, maxit)
        e1.record(stream)
        e1.synchronize()
        its += r["iterations"]
        ms += e0.elapsed_time(e1)
    return r, its, ms


SYM_FLAG = False   # --sym: configs 2 / 4 dense with CCG_FLAG_SYMMETRIC (upper-triangle products)


def run_dense(cfg, A, y, methods, tol, maxit, reps, dtype, toeplitz=None):
    n = y.shape[0]
    s = 8 if dtype == "c64" else 16
    h = ccg.ccg_create(dtype, n)
    if toeplitz is None:
        # the library detects A = Aᵀ itself (CCG_SYM_DETECT=0: general kernels);
        # --sym declares it (CCG_FLAG_SYMMETRIC)
        ccg.ccg_set_matvec_dense(h, A, 0, n, flags=ccg.FLAG_SYMMETRIC if (SYM_FLAG and cfg in (2, 4)) else 0)
        sym = ccg.ccg_get_stat(h, "symmetric")
        if sym:
            b_mat = n * (n + 1) // 2 * s   # the upper triangle: what the product reads
            opname = "dense-sym" if sym == 1 else "dense-sym-detected"
        else:
            b_mat = n * n * s
            opname = "dense"
    else:
        ccg.ccg_set_matvec_toeplitz3(h, *toeplitz)
        b_mat = 2 * n * s                  # x read + y written: the FFT operator's irreducible bytes
        opname = "toeplitz"
    stream = torch.cuda.ExternalStream(ccg.ccg_get_stream(h))
    x = torch.empty_like(y)
    for m in methods:
        if SEL and m not in SEL:
            continue
        r, its, ms = timed(h, m, y, x, tol, maxit, reps, stream)
        b_iter = M_MATVEC[m] * b_mat + V_PASSES[m] * n * s
        ips = its / (ms / 1e3)
        print(json.dumps({"config": cfg, "operator": opname, "method": m, "n": n, "dtype": dtype,
                          "status": r["status"],
                          "iterations": r["iterations"], "ms_per_solve": ms / reps,
                          "us_per_iteration": 1e3 * ms / its, "iterations_per_s": ips,
                          "effective_GBs": b_iter * ips / 1e9, "true_rel_res": r["true_rel_res"],
                          "reps": reps, "knobs": KNOBS}), flush=True)
    ccg.ccg_destroy(h)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=0)
    ap.add_argument("--methods", default="")
    ap.add_argument("--no-dense4", action="store_true", help="config 4: FFT operator only")
    ap.add_argument("--ops", default="csr,stencil", help="config 5 operators")
    ap.add_argument("--ops2", default="dense,toeplitz", help="config 2 operators")
    ap.add_argument("--sym", action="store_true", help="configs 2/4 dense: CCG_FLAG_SYMMETRIC")
    ap.add_argument("--no-fft4", action="store_true", help="config 4: dense only")
    a = ap.parse_args()
    global SEL, SYM_FLAG
    SYM_FLAG = a.sym
    SEL = set(a.methods.split(",")) if a.methods else set()
    dev = "cuda:0"
    for c in [int(v) for v in a.configs.split(",")]:
        cf = CONFIGS[c]
        t0 = time.time()
        if c == 1:
            A, y = cfg1()
            run_dense(1, torch.from_numpy(A).to(dev), torch.from_numpy(y).to(dev), ALL, cf["tol"],
                      cf["maxit"], a.reps or 200, "c128")
        elif c == 2:
            A, y = cfg2()
            if "dense" in a.ops2.split(","):
                run_dense(2, torch.from_numpy(A).to(dev), torch.from_numpy(y).to(dev), SYM, cf["tol"],
                          cf["maxit"], a.reps or 50, "c128")
            if "toeplitz" in a.ops2.split(","):
                run_dense(2, None, torch.from_numpy(y).to(dev), SYM, cf["tol"], cf["maxit"], a.reps or 50, "c128",
                          toeplitz=(16, 16, 16, dda_kernel((16, 16, 16), 1.0), 3 + 0.5j))
        elif c == 3:
            n = cf["n"]
            Ad = torch.empty((n, n), dtype=torch.complex64, device=dev)
            pin = torch.empty((4096, n), dtype=torch.complex64).pin_memory()
            for r0 in range(0, n, 4096):
                gauss_shifted_rows(n, r0, r0 + 4096, seed=1, out=pin.numpy())
                Ad[r0:r0 + 4096].copy_(pin)
            run_dense(3, Ad, torch.from_numpy(cfg3_rhs(n)).to(dev), ALL, cf["tol"], cf["maxit"],
                      a.reps or 5, "c64")
            del Ad
        elif c == 4:
            n = cf["n"]
            if not a.no_fft4:
                run_dense(4, None, torch.from_numpy(cfg4_rhs()).to(dev), SYM, cf["tol"], cf["maxit"], a.reps or 5,
                          "c128", toeplitz=(64, 32, 32, dda_kernel((64, 32, 32), 0.5), 2.5 + 0.2j))
            if a.no_dense4:
                continue
            Ad = torch.empty((n, n), dtype=torch.complex128, device=dev)
            for r0 in range(0, n, 4096):
                cfg4_rows_device(r0, r0 + 4096, Ad[r0:r0 + 4096])
            torch.cuda.synchronize()
            print(json.dumps({"config": 4, "generate_s": time.time() - t0}), flush=True)
            run_dense(4, Ad, torch.from_numpy(cfg4_rhs()).to(dev), ("bicgstab", "qmr", "bicor", "cgne", "cocr", "bicg", "tfqmr", "gmres", "bicgstabl", "pbicgstab"),
                      cf["tol"], cf["maxit"], a.reps or 1, "c128")
            del Ad
        elif c == 5:
            rp, ci, v = helmholtz_csr(128)
            y = torch.from_numpy(helmholtz_rhs(128)).to(dev)
            n = 128 ** 3
            rpd, cid, vd = (torch.from_numpy(t).to(dev) for t in (rp, ci, v))
            b_csr = len(v) * (16 + 4) + 4 * (n + 1)
            for opname in [o for o in ("csr", "stencil") if o in a.ops.split(",")]:
                h = ccg.ccg_create("c128", n)
                if opname == "csr":
                    ccg.ccg_set_matvec_csr(h, rpd, cid, vd, 0, n, len(v))
                    b_mat = b_csr
                else:
                    d, o = helmholtz_coeffs()
                    ccg.ccg_set_matvec_stencil7(h, 128, 128, 128, d, o)
                    b_mat = 2 * n * 16          # x read + y write
                stream = torch.cuda.ExternalStream(ccg.ccg_get_stream(h))
                x = torch.empty_like(y)
                for m in [m for m in ("bicgstab", "cors", "cgs", "cocr", "tfqmr", "gmres", "bicgstabl", "pbicgstab") if not a.methods or m in a.methods.split(",")]:
                    r, its, ms = timed(h, m, y, x, cf["tol"], cf["maxit"], a.reps or 2, stream)
                    ips = its / (ms / 1e3)
                    b_iter = (1 if m == "cocr" else 2) * b_mat + V_PASSES[m] * n * 16
                    print(json.dumps({"config": 5, "operator": opname, "method": m, "n": n, "dtype": "c128",
                                      "status": r["status"], "iterations": r["iterations"],
                                      "ms_per_solve": ms / (a.reps or 2), "us_per_iteration": 1e3 * ms / its,
                                      "iterations_per_s": ips, "effective_GBs": b_iter * ips / 1e9,
                                      "true_rel_res": r["true_rel_res"]}), flush=True)
                ccg.ccg_destroy(h)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
