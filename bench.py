"""Benchmark: Krylov iterations/s of the complex-CG hot path on B200.

Workload (BASELINE.json configs[2], the config the north_star target is
quoted on): dense complex64 n = 32768, A = (2+0.3i)I + 0.5·G/sqrt(n), BiCGSTAB
and CGNE to rel. residual 1e-5 from x0 = 0 (maxit 500), A row-sharded over
the ranks.  One "step" = one tolerance-driven ccg_solve of each method (the
whole hot path: A·x, Aᴴ·x, fused dots/updates, scalar steps, finalize).
value = global Krylov iterations per second (strong scaling: the same system
for every N).

Launch: python bench.py [--gpus N --steps K --warmup W] (N > 1 under torchrun).
--impl reference times the CPU oracle (oracle/) on the host cores instead.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N = 32768
TOL = 1e-5
MAXIT = 500
METHODS = ("bicgstab", "cgne")
METRIC = "Krylov iterations/s and matvec HBM GB/s (fraction of ~8 TB/s), 1/2/4/8 B200"
WORKLOAD = "cfg3: dense c64 n=32768, A=(2+0.3i)I+0.5G/sqrt(n) (seed 1), BiCGSTAB+CGNE to 1e-5"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ccg", choices=["ccg", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--sharded-vectors", action="store_true",
                   help="N>1: row-sharded vectors (C1 allgather + scalar allgathers) instead of replicated vectors")
    p.add_argument("--force-comm", action="store_true",
                   help="N=1: run the sharded code path through a one-rank NCCL communicator (CCG_OPT_FORCE_COMM)")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md "clocks" line)
# ---------------------------------------------------------------------------
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                bits = int(parts[2], 16)
            except ValueError:
                continue
            mx = m
            if s > 0:
                sm.append(s)
            for b, name in REASON_BITS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "gemv_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU oracle (reference arm / cpu_baseline): bounded sample of the same workload
# ---------------------------------------------------------------------------
def oracle_sample(A, y, budget_s=20.0):
    import oracle
    try:
        from threadpoolctl import threadpool_info
        cores = max((d.get("num_threads", 1) for d in threadpool_info()), default=os.cpu_count())
    except Exception:
        cores = os.cpu_count()
    op = oracle.DenseOp(A)
    its, t_used, runs = 0, 0.0, []
    t0 = time.perf_counter()
    for m in METHODS:
        t1 = time.perf_counter()
        r = oracle.solve(m, op, y, TOL, MAXIT)
        dt = time.perf_counter() - t1
        its += r.iterations
        t_used += dt
        runs.append(f"{m}:{r.iterations}it/{dt:.1f}s")
        if time.perf_counter() - t0 > budget_s:
            break
    return {"value": its / t_used, "unit": "iterations/s", "cores": int(cores), "kind": "oracle",
            "sample": "one tolerance-driven oracle solve per method on the full cfg3 system (" +
                      ", ".join(runs) + "); NumPy BLAS GEMV, Aᴴx as conj(conj(x)ᵀA)"}


def bench_config(world, args):
    """The config dict both arms print (identical by construction)."""
    rep = world > 1 and not args.sharded_vectors
    return {"workload": WORKLOAD, "n": N, "methods": list(METHODS), "tol": TOL, "maxit": MAXIT,
            "parallelism": f"row-shard{world}" + ("+replicated-vectors" if rep else ""),
            "vector_mode": "replicated" if rep else "sharded",
            "l2": "A is 8.6 GB >> 126 MB L2: no flush needed"}


def gen_rows(r0, r1, out):
    from workloads import gauss_shifted_rows
    return gauss_shifted_rows(N, r0, r1, seed=1, out=out)


# ---------------------------------------------------------------------------
def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    from workloads import cfg3_rhs
    A = np.empty((N, N), dtype=np.complex64)
    gen_rows(0, N, A)
    y = cfg3_rhs(N)
    vals, secs = [], []
    cb = None
    for _ in range(min(args.warmup, 1)):           # warm BLAS / page in A
        oracle_sample(A, y, budget_s=60.0)
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cb = oracle_sample(A, y, budget_s=60.0)
        secs.append(time.perf_counter() - t0)
        vals.append(cb["value"])
    v = float(np.median(vals))
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "iterations/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.median(secs)), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c64", "data": "synthetic",
            "config": bench_config(world, args),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ccg(args):
    import torch
    import paper_1208_4869_b200 as ccg

    rank, local_rank, world = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    uses_nccl = world > 1 or args.force_comm
    if uses_nccl:   # NCCL init lines (nRanks, transport) on stderr for the record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        nid = [ccg.ccg_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        nccl_id = nid[0]
    else:
        dist = None
        nccl_id = None
    nloc = N // world
    row0 = rank * nloc

    # inputs: this rank's rows, generated on the host in chunks, copied to HBM
    keep_host = (rank == 0 and world == 1 and not args.no_cpu_baseline)
    Ahost = np.empty((N, N), dtype=np.complex64) if keep_host else None
    Ad = torch.empty((nloc, N), dtype=torch.complex64, device=dev)
    chunk = 2048
    pin = torch.empty((chunk, N), dtype=torch.complex64).pin_memory()
    for a in range(0, nloc, chunk):
        b = min(nloc, a + chunk)
        gen_rows(row0 + a, row0 + b, pin.numpy()[:b - a])
        Ad[a:b].copy_(pin[:b - a])
        if keep_host:
            Ahost[row0 + a:row0 + b] = pin.numpy()[:b - a]
    del pin
    from workloads import cfg3_rhs
    yfull = cfg3_rhs(N)
    yloc = torch.from_numpy(yfull[row0:row0 + nloc].copy()).to(dev)
    xloc = torch.empty_like(yloc)

    # N > 1: replicated vectors (SURVEY §8(f) NEXT-2 ii) — one collective per
    # product and none per reduction phase
    opts = (ccg.OPT_REPLICATED if (world > 1 and not args.sharded_vectors) else 0) | \
        (ccg.OPT_FORCE_COMM if args.force_comm else 0)
    h = ccg.ccg_create("c64", N, world=world, rank=rank, nccl_id=nccl_id, device=local_rank, options=opts)
    ccg.ccg_set_matvec_dense(h, Ad, row0, nloc)
    stream = torch.cuda.ExternalStream(ccg.ccg_get_stream(h), device=dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def step(x0=None, y=yloc, x=xloc):
        its = 0
        launches = 0
        for m in METHODS:
            r = ccg.ccg_solve(h, m, x0, y, x, TOL, MAXIT)
            assert r["status"] == "CONVERGED", r
            its += r["iterations"]
            launches += ccg.ccg_last_launch_count(h)
        return its, launches

    for _ in range(args.warmup):
        step()

    # ---- timed region: the production path (graph replay, no per-kernel
    # events); device events on the library stream, max over ranks
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    its_total, launches_total = 0, 0
    mv_a = mv_ah = 0
    for _ in range(args.steps):
        for m in METHODS:
            r = ccg.ccg_solve(h, m, None, yloc, xloc, TOL, MAXIT)
            assert r["status"] == "CONVERGED", r
            its_total += r["iterations"]
            mv_a += r["matvecs_a"] + 1          # + the true-residual product
            mv_ah += r["matvecs_ah"]
            launches_total += ccg.ccg_last_launch_count(h)
    ev1.record(stream)
    barrier()
    clocks = sampler.stop()
    stats = ccg.ccg_get_stats(h)
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = its_total / (ms / 1e3)

    # ---- kernel timing pass (separate, not the headline): CUDA events around
    # every product launch on the library stream (library timing mode)
    ccg.ccg_set_timing(h, 1)
    ms_a = ms_ah = 0.0
    n_a = n_ah = 0
    for _ in range(max(1, min(args.steps, 3))):
        for m in METHODS:
            r = ccg.ccg_solve(h, m, None, yloc, xloc, TOL, MAXIT)
            assert r["status"] == "CONVERGED", r
            t = ccg.ccg_get_timing(h)
            ms_a += t["ms_a"]; n_a += t["n_a"]; ms_ah += t["ms_ah"]; n_ah += t["n_ah"]
    ccg.ccg_set_timing(h, 0)

    # ---- e2e: host (pinned) buffers through the C-ABI, copies inside the call
    e2e = None
    if not args.no_e2e:
        yh = torch.from_numpy(yfull[row0:row0 + nloc].copy()).pin_memory()
        xh = torch.empty_like(yh).pin_memory()
        barrier()
        t0 = time.perf_counter()
        its_e = 0
        for _ in range(args.steps):
            for m in METHODS:
                r = ccg.ccg_solve(h, m, None, yh, xh, TOL, MAXIT)
                assert r["status"] == "CONVERGED", r
                its_e += r["iterations"]
        barrier()
        dt = time.perf_counter() - t0
        if dist:
            t = torch.tensor([dt], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": its_e / dt, "unit": "iterations/s",
               "h2d_bytes_per_step": int(nloc * 8 * len(METHODS)),
               "d2h_bytes_per_step": int(nloc * 8 * len(METHODS)),
               "note": "y staged H2D and x D2H by ccg_solve (host pointers), per rank"}

    # ---- roofline of the dominant kernel (gemv_n, A·x)
    peak, peak_src = measured_peak()
    s = 8
    bytes_a = nloc * N * s + N * s + nloc * s          # A + x + y per A·x launch
    bytes_ah = nloc * N * s + nloc * s + N * s         # A + x slice + full-length output
    ach_a = bytes_a / (ms_a / n_a * 1e-3) / 1e9 if n_a else None
    ach_ah = bytes_ah / (ms_ah / n_ah * 1e-3) / 1e9 if n_ah else None
    traffic = ncu_traffic()
    roof = {"bound": "hbm", "kernel": "gemv_n_split<float,256,8> (A·x, + strip-sum stage 2)",
            "achieved": ach_a, "peak": peak, "unit": "GB/s",
            "frac": (ach_a / peak) if ach_a else None,
            "frac_of_8TBs": (ach_a / 8000.0) if ach_a else None,
            "frac_of_7p7TBs_nominal": (ach_a / 7700.0) if ach_a else None,
            "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
            "algorithmic_bytes_per_launch": bytes_a, "avg_launch_ms": (ms_a / n_a) if n_a else None,
            "launches_timed": n_a, "peak_source": peak_src,
            "ah": {"kernel": "gemv_h_stage1+stage2 (Aᴴ·x)", "achieved": ach_ah,
                   "frac": (ach_ah / peak) if ach_ah else None,
                   "avg_launch_ms": (ms_ah / n_ah) if n_ah else None, "launches_timed": n_ah},
            "timing_pass": "separate pass with per-launch CUDA events (library timing mode); "
                           "the headline value is the graph-replay path without them"}
    # whole-step effective bandwidth: the products' algorithmic bytes over the
    # (production-path) step time — vector passes not counted
    step_bytes = mv_a * bytes_a + mv_ah * bytes_ah
    roof["step_effective_gbs"] = step_bytes / (ms * 1e-3) / 1e9
    roof["step_effective_frac"] = roof["step_effective_gbs"] / peak
    roof["matvec_share_of_step"] = ((ms_a / n_a * mv_a + ms_ah / n_ah * mv_ah) / ms) if (n_a and n_ah) else None

    cpu = None
    if keep_host:
        cpu = oracle_sample(Ahost, yfull)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "c64", "data": "synthetic",
                "config": bench_config(world, args),
                "iterations_per_step": its_total // args.steps,
                "comm": {"kind": {0: "none", 1: "nccl", 2: "loopback"}[stats["comm_kind"]],
                         "graph_replays": stats["graph_replays"],
                         "collectives_in_graphs_last_solve": stats["graph_collectives"],
                         "force_comm": bool(args.force_comm)},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_total, "clocks": clocks}
        print(json.dumps(line), flush=True)
    ccg.ccg_destroy(h)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ccg(args)


if __name__ == "__main__":
    sys.exit(main())
