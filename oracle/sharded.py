"""Sharded oracle mode.  TEST INFRASTRUCTURE ONLY.

The same recurrences (oracle.solvers) run on G row blocks, one process per
rank over torch.distributed (gloo on the CPU), with the data movement of the
GPU path's row sharding: A·x gathers the input slices, Aᴴ·x
sums per-rank full-length partials, every inner product is a per-rank partial
summed in rank order, and the CSR z-slab operator exchanges only one halo
plane with each neighbour.  It checks the partition and halo index maps with
no GPU; it shares no code with libccg.
"""

import numpy as np
import torch
import torch.distributed as dist

from .operators import CsrOp


def _gather_rank_ordered(t):
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return parts


class ShardedDots:
    """Inner products over row-sharded vectors: local partial, rank-ordered sum."""

    def _sum(self, z):
        t = torch.tensor([complex(z).real, complex(z).imag], dtype=torch.float64)
        parts = _gather_rank_ordered(t)
        s = 0j
        for p in parts:
            s += complex(p[0].item(), p[1].item())
        return s

    def dotc(self, u, v):
        return self._sum(np.vdot(u, v))

    def dotu(self, u, v):
        return self._sum(np.dot(u, v))

    def norm_sq(self, u):
        return self._sum(np.vdot(u, u)).real


class _Counted:
    def __init__(self):
        self.n_a = self.n_ah = self.n_at = 0

    def reset_counts(self):
        self.n_a = self.n_ah = self.n_at = 0


class ShardedDenseOp(_Counted):
    """Rows [row0, row0+nloc) of a dense n×n operator."""

    def __init__(self, A_local, row0, n):
        super().__init__()
        self.A = np.asarray(A_local)
        self.row0, self.nloc, self.n = row0, self.A.shape[0], n
        self.dtype = self.A.dtype

    def _gather(self, x_local):
        parts = _gather_rank_ordered(torch.from_numpy(np.ascontiguousarray(x_local)))
        return np.concatenate([p.numpy() for p in parts])

    def _reduce_slice(self, partial):
        parts = _gather_rank_ordered(torch.from_numpy(np.ascontiguousarray(partial)))
        s = parts[0].numpy().copy()
        for p in parts[1:]:
            s = s + p.numpy()
        return s[self.row0:self.row0 + self.nloc]

    def apply(self, x):
        self.n_a += 1
        return self.A.dot(self._gather(x))

    def apply_h(self, x):
        self.n_ah += 1
        return self._reduce_slice(np.conj(np.conj(x).dot(self.A)))

    def apply_t(self, x):
        self.n_at += 1
        return self._reduce_slice(x.dot(self.A))


class ShardedCsrOp(_Counted):
    """CSR rows [row0, row0+nloc) with GLOBAL column indices; x is exchanged as
    one halo of width h with each neighbour rank (send/recv), never gathered."""

    def __init__(self, rowptr, colind, vals, row0, n, halo):
        super().__init__()
        self.row0, self.n, self.h = row0, n, halo
        self.nloc = len(rowptr) - 1
        import scipy.sparse as sp
        self._M = sp.csr_matrix((np.asarray(vals), np.asarray(colind), np.asarray(rowptr)),
                                shape=(self.nloc, n))
        self.dtype = np.asarray(vals).dtype

    def _extended(self, x):
        r, G = dist.get_rank(), dist.get_world_size()
        full = np.zeros(self.n, dtype=x.dtype)
        full[self.row0:self.row0 + self.nloc] = x
        h = self.h
        reqs = []
        lo = torch.empty(h, dtype=torch.from_numpy(x[:1]).dtype)
        hi = torch.empty(h, dtype=lo.dtype)
        if r > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(x[:h])), r - 1))
            reqs.append(dist.irecv(lo, r - 1))
        if r < G - 1:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(x[-h:])), r + 1))
            reqs.append(dist.irecv(hi, r + 1))
        for q in reqs:
            q.wait()
        if r > 0:
            full[self.row0 - h:self.row0] = lo.numpy()
        if r < G - 1:
            full[self.row0 + self.nloc:self.row0 + self.nloc + h] = hi.numpy()
        return full

    def apply(self, x):
        self.n_a += 1
        return self._M.dot(self._extended(np.asarray(x)))

    def apply_h(self, x):  # complex-symmetric operators only: Aᴴx = conj(A conj x)
        self.n_ah += 1
        return np.conj(self._M.dot(self._extended(np.conj(np.asarray(x)))))

    def apply_t(self, x):
        self.n_at += 1
        return self._M.dot(self._extended(np.asarray(x)))
