"""N > 1 host logic on the CPU: world_size 2 and 4 over gloo (127.0.0.1).

* the sharded oracle (row blocks, rank-ordered sums, CSR halo planes) agrees
  with the unsharded oracle — pins the partition and halo index maps;
* the NCCL-id broadcast and max-over-ranks timing pattern bench.py uses.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_dense(rank, world, port, outdir):
    import oracle
    from oracle.sharded import ShardedDots, ShardedDenseOp
    from workloads import cfg1
    _init(rank, world, port)
    try:
        A, y = cfg1(n=64, seed=7)
        n = 64
        nloc = n // world
        sl = slice(rank * nloc, (rank + 1) * nloc)
        res = {}
        for m in ("bicgstab", "cgne", "qmr", "bicor", "cors"):
            full = oracle.solve(m, oracle.DenseOp(A), y, 1e-11, 200)
            sh = oracle.solve(m, ShardedDenseOp(A[sl], rank * nloc, n), y[sl].copy(), 1e-11, 200,
                              dots=ShardedDots())
            res[m] = (full.iterations, sh.iterations,
                      float(np.linalg.norm(sh.x - full.x[sl]) / np.linalg.norm(full.x)),
                      (full.matvecs_a, full.matvecs_ah), (sh.matvecs_a, sh.matvecs_ah),
                      abs(full.true_rel_res - sh.true_rel_res))
        # bench.py pattern: rank 0 makes a 128-byte id, broadcast as an object
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res["_id"] = obj[0] == bytes(range(128))
        res["_max"] = float(t.item())
        np.save(os.path.join(outdir, f"dense{rank}.npy"), np.array([res], dtype=object))
    finally:
        dist.destroy_process_group()


def _worker_csr(rank, world, port, outdir):
    import oracle
    from oracle.sharded import ShardedDots, ShardedCsrOp
    from workloads import helmholtz_csr, helmholtz_rhs
    _init(rank, world, port)
    try:
        N = 8
        zs = N // world
        rp, ci, v = helmholtz_csr(N, kh=10 / 128, z0=rank * zs, z1=(rank + 1) * zs)
        nloc = zs * N * N
        op = ShardedCsrOp(rp, ci, v, rank * nloc, N ** 3, halo=N * N)
        x = np.random.default_rng(1).standard_normal(N ** 3) + 1j
        sl = slice(rank * nloc, (rank + 1) * nloc)
        rpf, cif, vf = helmholtz_csr(N, kh=10 / 128)
        full = oracle.CsrOp(rpf, cif, vf)
        ya = op.apply(x[sl].copy())
        err_a = float(np.max(np.abs(ya - full.apply(x)[sl])))
        y = helmholtz_rhs(N)
        fs = oracle.solve("cors", full, y, 1e-10, 500)
        ss = oracle.solve("cors", op, y[sl].copy(), 1e-10, 500, dots=ShardedDots())
        np.save(os.path.join(outdir, f"csr{rank}.npy"),
                np.array([dict(err_a=err_a, k=(fs.iterations, ss.iterations),
                               dx=float(np.linalg.norm(ss.x - fs.x[sl]) / np.linalg.norm(fs.x)))],
                         dtype=object))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_oracle_dense(world, tmp_path):
    mp.spawn(_worker_dense, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        res = np.load(tmp_path / f"dense{r}.npy", allow_pickle=True)[0]
        assert res["_id"] and res["_max"] == float(world)
        for m in ("bicgstab", "cgne", "qmr", "bicor", "cors"):
            kf, ks, dx, cf, cs, dtr = res[m]
            assert kf == ks, (m, kf, ks)
            assert dx <= 1e-12, (m, dx)
            assert cf == cs, m
            assert dtr <= 1e-13


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_oracle_csr_halo(world, tmp_path):
    mp.spawn(_worker_csr, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        res = np.load(tmp_path / f"csr{r}.npy", allow_pickle=True)[0]
        assert res["err_a"] <= 1e-14
        assert res["k"][0] == res["k"][1]
        assert res["dx"] <= 1e-10
