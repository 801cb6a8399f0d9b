"""The NCCL data plane on ONE B200 (CCG_OPT_FORCE_COMM).

A world-1 handle created with CCG_OPT_FORCE_COMM takes the sharded code path
with a real one-rank NCCL communicator: every collective call site of the
multi-GPU path (allgather of the product input C1, reduce-scatter of dense Aᴴ
partials C2, allgather of the scalar partial sums C3, the CSR / stencil halo
call C4; in replicated mode the allgather of product rows / Aᴴ partials)
executes through ncclAllGather / ncclReduceScatter, captured inside the
per-iteration CUDA graph, with the fixed multi-rank chunk schedule.  Every
method runs on every operator against the CPU oracle (P-literal,
else the P-envelope), and the handle's statistics prove that NCCL ran inside
graph replays.  (Send/recv of the halo planes needs a neighbour rank, i.e. a
second GPU: the loopback tests cover that call site's index logic.)
"""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1208_4869_b200 as ccg
from oracle import DenseOp, CsrOp, ToeplitzOp
from workloads import dda_lattice_rows, dda_lattice_rhs, dda_kernel, helmholtz_rhs, lattice_csr
from tests._gpu import Dense, to_dev
from tests.test_gpu_solve import _parity

pytestmark = pytest.mark.gpu

ALL = list(ccg.METHODS)
AH_METHODS = {"cgne", "qmr", "bicor", "bicg", "cgnr"}
DIMS = (8, 8, 8)
LATTICE = (6.5 - 0.5j, -1.0)


class Forced(Dense):
    """A world-1 handle on the sharded NCCL path (optionally replicated)."""

    def __init__(self, kind, replicated):
        opts = ccg.OPT_FORCE_COMM | (ccg.OPT_REPLICATED if replicated else 0)
        self.dtype = np.complex128
        self.keep = []
        if kind == "dense":
            A = dda_lattice_rows(DIMS, 1.0, 3 + 0.5j, 0, 512)
            self.n = 512
            self.h = ccg.ccg_create("c128", self.n, options=opts)
            self.A = to_dev(A)
            ccg.ccg_set_matvec_dense(self.h, self.A, 0, self.n)
            self.op = DenseOp(A)
        elif kind == "toeplitz":
            self.n = 512
            self.h = ccg.ccg_create("c128", self.n, options=opts)
            K = dda_kernel(DIMS, 1.0)
            ccg.ccg_set_matvec_toeplitz3(self.h, *DIMS, K, 3 + 0.5j)
            self.op = ToeplitzOp(K, DIMS, 3 + 0.5j)
        else:
            # a diagonally dominant complex-symmetric 7-point lattice: the point
            # here is the data plane, not the rounding chaos of the indefinite
            # config-5 operator (tests/test_gpu_cfg5_envelope.py covers that)
            N = 16
            d, o = LATTICE
            rp, ci, v = lattice_csr(N, N, N, d, o)
            self.n = N ** 3
            self.h = ccg.ccg_create("c128", self.n, options=opts)
            if kind == "csr":
                t = [to_dev(a) for a in (rp, ci, v)]
                self.keep = t
                ccg.ccg_set_matvec_csr(self.h, *t, 0, self.n, len(v), flags=ccg.FLAG_SYMMETRIC)
            else:
                ccg.ccg_set_matvec_stencil7(self.h, N, N, N, d, o)
            self.op = CsrOp(rp, ci, v)
        self.y = dda_lattice_rhs(DIMS, 1.0) if kind in ("dense", "toeplitz") else helmholtz_rhs(16)


@pytest.mark.parametrize("replicated", [False, True], ids=["sharded", "replicated"])
@pytest.mark.parametrize("kind", ["dense", "csr", "stencil", "toeplitz"])
@pytest.mark.parametrize("method", ALL)
def test_nccl_one_rank_parity(method, kind, replicated):
    with Forced(kind, replicated) as h:
        if kind == "csr" and not replicated and method in AH_METHODS:
            with pytest.raises(ccg.CcgError) as e:      # CSR Aᴴ is not row-shardable (include/ccg.h)
                h.solve(method, h.y, 1e-8, 10)
            assert e.value.code == -3
            return
        _parity(h, h.op, h.y, method, 1e-8, 4000, np.complex128, literal=False,
                tag=f"nccl1-{kind}-{'rep' if replicated else 'shard'}")
        st = ccg.ccg_get_stats(h.h)
        assert st["comm_kind"] == 1 and st["world"] == 1 and st["replicated"] == int(replicated), st
        assert st["graph_replays"] > 0, st
        # a collective inside the iteration graph: every reduction phase
        # (sharded) or every product (replicated, except the FFT operator, which
        # transforms the whole vector on every rank with no collective)
        if not (replicated and kind == "toeplitz"):
            assert st["graph_collectives"] >= st["graph_replays"], st


def test_nccl_one_rank_apply_matches_plain():
    """Every product through the NCCL path equals the plain world-1 product
    bitwise (the collectives are identities; the reduction order is the same)."""
    from tests._gpu import Dense as Plain
    A = dda_lattice_rows(DIMS, 1.0, 3 + 0.5j, 0, 512)
    x = np.random.default_rng(4).standard_normal(512) + 1j * np.random.default_rng(5).standard_normal(512)
    for rep in (False, True):
        with Forced("dense", rep) as hf, Plain(A) as hp:
            for o in ("A", "AH", "AT"):
                assert np.array_equal(hf.apply(x, o), hp.apply(x, o)), (rep, o)


def test_nccl_debug_lines():
    """NCCL_DEBUG=INFO in a fresh process: the communicator is initialised by
    NCCL (ncclCommInitRank) and a solve runs through it."""
    code = (
        "import numpy as np, torch, paper_1208_4869_b200 as ccg\n"
        "from workloads import cfg1\n"
        "A, y = cfg1()\n"
        "h = ccg.ccg_create('c128', 256, options=ccg.OPT_FORCE_COMM)\n"
        "Ad = torch.from_numpy(A).cuda(); yd = torch.from_numpy(y).cuda(); x = torch.empty_like(yd)\n"
        "ccg.ccg_set_matvec_dense(h, Ad, 0, 256)\n"
        "r = ccg.ccg_solve(h, 'bicgstab', None, yd, x, 1e-10, 500)\n"
        "print('RESULT', r['status'], r['iterations'], ccg.ccg_get_stats(h))\n"
        "ccg.ccg_destroy(h)\n")
    env = dict(os.environ, NCCL_DEBUG="INFO")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=300)
    out = p.stdout + p.stderr
    log = os.environ.get("CCG_NCCL_LOG")
    if log:
        with open(log, "w") as f:
            f.write(out)
    assert p.returncode == 0, out[-3000:]
    assert "NCCL INFO" in out and "Init COMPLETE" in out, out[-3000:]
    assert "RESULT CONVERGED 12" in out, out[-3000:]


@pytest.mark.parametrize("kind", ["dense", "csr", "stencil"])
@pytest.mark.parametrize("method", ["bicgstab", "cgne", "qmr", "cocr", "gmres"])
def test_nccl_window_p2p(method, kind):
    """CCG_OPT_P2P through a real NCCL symmetric-memory window (one rank):
    ncclMemAlloc + ncclCommWindowRegister, ncclGetPeerPointer resolved on the
    device, the product epilogue storing into the window, release / acquire
    flags inside the captured iteration graph — bitwise equal to the plain
    replicated NCCL path, and the oracle parity of that path."""
    class P2P(Forced):
        def __init__(self, kind):
            Forced.__init__(self, kind, True)
            h0 = self.h
            opts = ccg.OPT_FORCE_COMM | ccg.OPT_REPLICATED | ccg.OPT_P2P
            self.h = ccg.ccg_create("c128", self.n, options=opts)
            if kind == "dense":
                ccg.ccg_set_matvec_dense(self.h, self.A, 0, self.n)
            elif kind == "csr":
                ccg.ccg_set_matvec_csr(self.h, *self.keep, 0, self.n, len(self.keep[2]), flags=ccg.FLAG_SYMMETRIC)
            else:
                ccg.ccg_set_matvec_stencil7(self.h, 16, 16, 16, *LATTICE)
            ccg.ccg_destroy(h0)
    with Forced(kind, True) as ref, P2P(kind) as h:
        a = h.solve(method, h.y, 1e-8, 4000)
        b = ref.solve(method, ref.y, 1e-8, 4000)
        assert a["status"] == b["status"] == "CONVERGED"
        assert a["iterations"] == b["iterations"] and np.array_equal(a["x"], b["x"]), method
        st = ccg.ccg_get_stats(h.h)
        assert st["comm_kind"] == 1 and st["p2p_exchanges"] > 0 and st["graph_replays"] > 0, st
        _parity(h, h.op, h.y, method, 1e-8, 4000, np.complex128, literal=False, tag=f"nccl1-p2p-{kind}")
