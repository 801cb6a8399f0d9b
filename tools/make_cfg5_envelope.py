"""Write tests/golden/cfg5_envelope.json: the oracle's rounding envelope of
BASELINE config 5 (sparse c128 shifted Helmholtz, 128³ CSR, BJ:11) for
BiCGSTAB and CORS at tol 1e-8 — SURVEY §8(c) P-envelope, oracle/envelope.py.

Calls only oracle/ and workloads/ (no GPU, no product code).  Runs the clean
member and the 8 noise seeds in parallel processes (~0.25 s per oracle
iteration on one core; BiCGSTAB ~1300 iterations).

    python tools/make_cfg5_envelope.py [--procs 9]
"""

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

# one BLAS thread per member: the dot products' summation order (and so, on
# this rounding-chaotic problem, the members' iteration counts) depends on the
# BLAS thread count; the committed golden was written this way
for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[_v] = "1"

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TOL, MAXIT = 1e-8, 20000          # BJ:11; maxit reading Q8
METHODS = ("bicgstab", "cors")
K_FIXED = (10, 20, 30, 40)        # D(k) at these equal iteration counts
SEEDS = 8                         # SURVEY §8(c) E = 8; --seeds overrides (reading E4)

_OP = None


def _op():
    global _OP
    if _OP is None:
        import oracle
        from workloads import cfg5
        rp, ci, v, y = cfg5()
        _OP = (oracle.CsrOp(rp, ci, v), y)
    return _OP


def _member(args):
    method, seed, tol, maxit = args
    import oracle
    from oracle.envelope import NoisyOp, rel_history
    op, y = _op()
    m = op if seed == 0 else NoisyOp(op, seed)
    t = time.time()
    r = oracle.solve(method, m, y, tol, maxit)
    out = dict(method=method, seed=seed, k=r.iterations, status=r.status_name,
               hist=rel_history(r).tolist(), true_rel_res=r.true_rel_res, secs=time.time() - t)
    if tol == 0.0:
        out["x"] = r.x
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=SEEDS + 1)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "cfg5_envelope.json"))
    ap.add_argument("--seeds", type=int, default=SEEDS)
    ap.add_argument("--methods", default=",".join(METHODS))
    ap.add_argument("--merge", action="store_true", help="keep the other methods of an existing file")
    a = ap.parse_args()
    seeds = a.seeds
    methods = a.methods.split(",")
    from oracle.envelope import agreement_window, pairwise_spread, hist_tol, history_spread, NOISE_C128
    H = hist_tol(np.complex128)
    res = {"_source": ("written by tools/make_cfg5_envelope.py from oracle/ only: BASELINE config 5 "
                       "(BJ:11; PAPER.md:95 §5 'own sparse matrix scheme'), SURVEY §8(c) P-envelope: "
                       f"clean run + noise seeds of amplitude {NOISE_C128} per matvec output"),
           "tol": TOL, "maxit": MAXIT, "H": H, "methods": {}}
    if a.merge and os.path.exists(a.out):
        res["methods"] = json.load(open(a.out))["methods"]
    ctx = mp.get_context("fork")
    with ctx.Pool(a.procs) as pool:
        for method in methods:
            t = time.time()
            runs = pool.map(_member, [(method, s, TOL, MAXIT) for s in range(seeds + 1)])
            runs.sort(key=lambda r: r["seed"])
            hists = [r["hist"] for r in runs]
            ks = [r["k"] for r in runs]
            ent = dict(seeds=seeds, k_clean=ks[0], ks=ks, k_min=min(ks), k_max=max(ks),
                       statuses=[r["status"] for r in runs],
                       true_rel_res=[r["true_rel_res"] for r in runs],
                       window=agreement_window(hists, H), hist_clean=hists[0],
                       hist_spread=history_spread(hists).tolist(), D={})
            for k in K_FIXED:
                xr = pool.map(_member, [(method, s, 0.0, k) for s in range(seeds + 1)])
                xr.sort(key=lambda r: r["seed"])
                xs = [r["x"] for r in xr]
                ent["D"][str(k)] = pairwise_spread(xs, xs[0])
            res["methods"][method] = ent
            print(method, ent["ks"], "window", ent["window"], "D", ent["D"],
                  f"{time.time() - t:.0f}s", flush=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
