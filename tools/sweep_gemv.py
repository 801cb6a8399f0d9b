"""Sweep GEMV launch knobs on one B200 (perf tuning only; no parity).

For each configuration the knobs are set in the environment and the operator is
re-registered (launch parameters are chosen in ccg_set_matvec_dense), then A·x
and Aᴴ·x are timed with the library's own CUDA events (ccg_set_timing).
Prints one JSON line per configuration.
"""

import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_4869_b200 as ccg  # noqa: E402


def run(dtype, n, reps, grid):
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    A = torch.randn((n, n), dtype=tdt, device="cuda")
    x = torch.randn(n, dtype=tdt, device="cuda")
    y = torch.empty_like(x)
    h = ccg.ccg_create(dtype, n)
    esz = 8 if dtype == "c64" else 16
    for knobs in grid:
        for k in ("CCG_GEMV", "CCG_SPLIT_KB", "CCG_SPLIT_UR", "CCG_SPLIT_WAVES", "CCG_COLS_WAVES", "CCG_COLS_RG"):
            os.environ.pop(k, None)
        os.environ.update({k: str(v) for k, v in knobs.items()})
        ccg.ccg_set_matvec_dense(h, A, 0, n)
        ccg.ccg_set_timing(h, 1)
        res = {}
        for op in ("A", "AH"):
            for _ in range(3):
                ccg.ccg_apply(h, op, x, y)
            ms = 0.0
            cnt = 0
            for _ in range(reps):
                ccg.ccg_apply(h, op, x, y)
                t = ccg.ccg_get_timing(h)
                ms += t["ms_a"] + t["ms_ah"]
                cnt += 1
            res[op] = n * n * esz / (ms / cnt * 1e-3) / 1e9
        ccg.ccg_set_timing(h, 0)
        print(json.dumps({"dtype": dtype, "n": n, **knobs, "GBs_A": round(res["A"]), "GBs_AH": round(res["AH"])}),
              flush=True)
    ccg.ccg_destroy(h)
    del A


if __name__ == "__main__":
    if "--medium" in sys.argv:
        modes = ([dict(CCG_GEMV=m) for m in ("split", "cols", "bulk", "rows")] +
                 [dict(CCG_GEMV="split", CCG_SPLIT_KB=kb, CCG_SPLIT_UR=ur, CCG_SPLIT_WAVES=w)
                  for kb in (4, 8, 16, 32) for ur in (4, 8) for w in (1, 2, 4)])
        run("c128", 4096, 100, modes)
        sys.exit(0)
    if "--modes" in sys.argv:
        modes = [dict(CCG_GEMV="split")] + [dict(CCG_GEMV="cols", CCG_COLS_RG=g, CCG_COLS_WAVES=w)
                                            for g in (1, 4) for w in (1, 2, 4)]
        run("c64", 32768, 10, modes)
        run("c128", 16384, 10, modes)
        run("c128", 4096, 50, modes)
        sys.exit(0)
    grid = [dict(CCG_GEMV="split", CCG_SPLIT_KB=kb, CCG_SPLIT_UR=ur, CCG_SPLIT_WAVES=w)
            for kb, ur, w in itertools.product((8, 16, 24), (4, 8, 16), (1, 2, 4))]
    run("c64", 32768, 10, grid)
    run("c128", 16384, 10, [g for g in grid if g["CCG_SPLIT_WAVES"] == 2])
