"""Device-side generation of the large closed-form inputs (no method arithmetic).

Config 4's dense DDA matrix is 68.7 GB (complex128, n = 65536): building it on
the host and copying it takes minutes, so this module evaluates the same
closed form as ``generators.dda_lattice_rows`` (A_ij = 0.1·exp(i·k·d)/d,
A_ii = diag) with torch fp64 ops on the GPU, row block by row block.  The
values agree with the NumPy generator to a few ulp (checked by
tests/test_gpu_solve.py::test_cfg4_device_generator_matches_numpy); parity
tests compare GPU outputs with oracle values the oracle computes from its own
NumPy-generated rows.
"""

import torch


def dda_lattice_rows_device(dims, k, diag, r0, r1, out, block=512):
    """Fill ``out`` (complex128 tensor (r1-r0, n) on a CUDA device) with rows [r0, r1)."""
    nx, ny, nz = dims
    n = nx * ny * nz
    dev = out.device
    j = torch.arange(n, device=dev, dtype=torch.int64)
    ix, iy, iz = j % nx, (j // nx) % ny, j // (nx * ny)
    for a in range(r0, r1, block):  # noqa: E741
        b = min(r1, a + block)
        rows = torch.arange(a, b, device=dev, dtype=torch.int64)
        dx = (ix[rows, None] - ix[None, :]).to(torch.float64)
        dy = (iy[rows, None] - iy[None, :]).to(torch.float64)
        dz = (iz[rows, None] - iz[None, :]).to(torch.float64)
        d = torch.sqrt(dx * dx + dy * dy + dz * dz)
        blk = torch.polar(0.1 / d, k * d)            # 0.1·exp(i k d)/d
        blk[torch.arange(b - a, device=dev), rows] = complex(diag)
        out[a - r0:b - r0].copy_(blk)
        del dx, dy, dz, d, blk
    return out


def cfg4_rows_device(r0, r1, out):
    return dda_lattice_rows_device((64, 32, 32), 0.5, 2.5 + 0.2j, r0, r1, out)
