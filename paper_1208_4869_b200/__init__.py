"""B200-native hot path of the CCGPAK complex-Krylov family (arXiv:1208.4869).

Thin ctypes binding over ``libccg.so`` (C-ABI declared in ``include/ccg.h``).
The functions keep the C names; they only marshal arguments (tensor / array
-> pointer, enum names -> ints, ccg_result -> dict).  Every arithmetic step
runs in libccg's CUDA kernels: there is no CPU fallback, and every call
raises if the shared library is missing (``load()``).

PyTorch is used by callers only for device memory, streams and process
groups; tensors passed here must be contiguous complex64/complex128 (CUDA or
CPU) — numpy arrays are accepted for host-side vectors.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libccg.so")

C64, C128 = 0, 1
METHODS = {"bicgstab": 0, "cgne": 1, "qmr": 2, "bicor": 3, "cors": 4,
           "bicg": 5, "cgs": 6, "cocr": 7, "cgnr": 8, "tfqmr": 9, "gmres": 10, "bicgstabl": 11,
           "pbicgstab": 12}
OPS = {"A": 0, "AH": 1, "AT": 2}
FLAG_SYMMETRIC = 1
STATUS = {0: "CONVERGED", 1: "MAXIT", 2: "BREAKDOWN", 3: "FALSE_CONVERGENCE", 4: "NONFINITE"}
BREAKDOWN = {0: None, 1: "rho", 2: "sigma", 3: "tt", 4: "omega", 5: "pi", 6: "delta",
             7: "epsilon", 8: "beta", 9: "xi", 10: "vnorm", 11: "wnorm", 12: "gamma"}
ERRORS = {0: "CCG_OK", -1: "CCG_E_ARG", -2: "CCG_E_DIM", -3: "CCG_E_CAPABILITY",
          -4: "CCG_E_STATE", -5: "CCG_E_CUDA", -6: "CCG_E_NCCL", -7: "CCG_E_OOM", -8: "CCG_E_USER"}
CB_A, CB_AH, CB_AT, CB_GRAPH_SAFE = 1, 2, 4, 8
MATVEC_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p)

# every symbol include/ccg.h declares (checked by tests/test_abi.py)
EXPORTS = ("ccg_get_unique_id", "ccg_create", "ccg_create_ex", "ccg_create_loopback_group",
           "ccg_create_loopback_group_ex",
           "ccg_set_matvec_dense", "ccg_set_matvec_csr", "ccg_set_matvec_stencil7",
           "ccg_set_matvec_toeplitz3", "ccg_set_matvec_callback", "ccg_set_gmres_restart",
           "ccg_set_bicgstab_ell", "ccg_set_jacobi",
           "ccg_apply", "ccg_solve", "ccg_get_history", "ccg_set_timing", "ccg_get_timing",
           "ccg_last_launch_count", "ccg_get_stat", "ccg_get_stream", "ccg_last_error", "ccg_destroy",
           "ccg_version")


class ccg_result(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("iterations", ctypes.c_int32),
                ("matvecs_a", ctypes.c_int32), ("matvecs_ah", ctypes.c_int32),
                ("breakdown_code", ctypes.c_int32), ("half_step", ctypes.c_int32),
                ("rec_rel_res", ctypes.c_double), ("true_rel_res", ctypes.c_double),
                ("wall_ms", ctypes.c_double)]


class CcgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


def _set_nccl_env():
    if "CCG_NCCL_LIB" in os.environ:
        return
    try:
        import nvidia.nccl as nn
        base = list(nn.__path__)[0]
        p = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(p):
            os.environ["CCG_NCCL_LIB"] = p
    except Exception:  # pragma: no cover
        pass


def load():
    """Load libccg.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    _set_nccl_env()
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u32, dbl = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                              ctypes.c_uint32, ctypes.c_double)
    sig = {
        "ccg_get_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
        "ccg_create": (ctypes.c_int, [ctypes.POINTER(vp), ctypes.c_int, i64, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_char_p, ctypes.c_int, vp]),
        "ccg_create_loopback_group": (ctypes.c_int, [ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int,
                                                     i64, ctypes.c_int]),
        "ccg_create_ex": (ctypes.c_int, [ctypes.POINTER(vp), ctypes.c_int, i64, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_char_p, ctypes.c_int, vp, u32]),
        "ccg_create_loopback_group_ex": (ctypes.c_int, [ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int,
                                                        i64, ctypes.c_int, u32]),
        "ccg_set_matvec_dense": (ctypes.c_int, [vp, vp, i64, i64, i64, u32]),
        "ccg_set_matvec_csr": (ctypes.c_int, [vp, vp, vp, vp, i64, i64, i64, u32]),
        "ccg_set_matvec_stencil7": (ctypes.c_int, [vp, i64, i64, i64, ctypes.POINTER(dbl), u32]),
        "ccg_set_matvec_toeplitz3": (ctypes.c_int, [vp, i64, i64, i64, ctypes.POINTER(dbl),
                                                    ctypes.POINTER(dbl), u32]),
        "ccg_set_matvec_callback": (ctypes.c_int, [vp, MATVEC_FN, vp, u32, u32]),
        "ccg_set_gmres_restart": (ctypes.c_int, [vp, i32]),
        "ccg_set_bicgstab_ell": (ctypes.c_int, [vp, i32]),
        "ccg_set_jacobi": (ctypes.c_int, [vp, vp, u32]),
        "ccg_apply": (ctypes.c_int, [vp, ctypes.c_int, vp, vp]),
        "ccg_solve": (ctypes.c_int, [vp, ctypes.c_int, vp, vp, vp, dbl, i32,
                                     ctypes.POINTER(ccg_result)]),
        "ccg_get_history": (ctypes.c_int, [vp, ctypes.POINTER(dbl), i32, ctypes.POINTER(i32)]),
        "ccg_set_timing": (ctypes.c_int, [vp, ctypes.c_int]),
        "ccg_get_timing": (ctypes.c_int, [vp, ctypes.POINTER(dbl), ctypes.POINTER(i32),
                                          ctypes.POINTER(dbl), ctypes.POINTER(i32)]),
        "ccg_last_launch_count": (i64, [vp]),
        "ccg_get_stat": (ctypes.c_int, [vp, i32, ctypes.POINTER(i64)]),
        "ccg_get_stream": (vp, [vp]),
        "ccg_last_error": (ctypes.c_char_p, [vp]),
        "ccg_destroy": (ctypes.c_int, [vp]),
        "ccg_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    _lib = lib
    return lib


_lib = None
_keepalive = {}   # handle -> borrowed operator buffers (the library borrows them)


# ---------------------------------------------------------------------------
# marshalling helpers
# ---------------------------------------------------------------------------
def _ptr(a, what="array"):
    """Device or host pointer of a contiguous torch tensor / numpy array."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError(f"{what} must be contiguous")
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{what} must be C-contiguous")
        return a.ctypes.data
    raise TypeError(f"{what}: expected a torch tensor or numpy array, got {type(a)}")


def _check(h, rc):
    if rc != 0:
        msg = load().ccg_last_error(h)
        raise CcgError(rc, msg.decode() if msg else "")


def _dtype_code(dt):
    s = str(dt)
    if "complex64" in s or dt in ("c64", C64):
        return C64
    if "complex128" in s or dt in ("c128", C128):
        return C128
    raise ValueError(f"unsupported dtype {dt}")


# ---------------------------------------------------------------------------
# the C-ABI, same names
# ---------------------------------------------------------------------------
def ccg_version():
    return load().ccg_version().decode()


def ccg_get_unique_id():
    buf = ctypes.create_string_buffer(128)
    _check(None, load().ccg_get_unique_id(buf))
    return buf.raw


OPT_REPLICATED = 1
OPT_FORCE_COMM = 2
OPT_P2P = 4


def ccg_create(dtype, n, world=1, rank=0, nccl_id=None, device=0, stream=None, options=0):
    h = ctypes.c_void_p()
    sp = None if stream is None else ctypes.c_void_p(getattr(stream, "cuda_stream", stream))
    if options:
        rc = load().ccg_create_ex(ctypes.byref(h), _dtype_code(dtype), int(n), int(world), int(rank),
                                  nccl_id, int(device), sp, int(options))
    else:
        rc = load().ccg_create(ctypes.byref(h), _dtype_code(dtype), int(n), int(world), int(rank),
                               nccl_id, int(device), sp)
    _check(None, rc)
    _keepalive[h.value] = []
    return h.value


def ccg_create_loopback_group(world, dtype, n, device=0, options=0):
    """`world` handles sharing an in-process loopback communicator (one GPU)."""
    hs = (ctypes.c_void_p * world)()
    _check(None, load().ccg_create_loopback_group_ex(hs, int(world), _dtype_code(dtype), int(n), int(device),
                                                     int(options)))
    out = [hs[r] for r in range(world)]
    for h in out:
        _keepalive[h] = []
    return out


def ccg_set_matvec_dense(h, A, row0, nloc, lda=None, flags=0):
    lda = A.shape[1] if lda is None else lda
    _check(h, load().ccg_set_matvec_dense(h, _ptr(A, "A"), int(row0), int(nloc), int(lda), int(flags)))
    _keepalive[h] = [A]


def ccg_set_matvec_csr(h, rowptr, colind, vals, row0, nloc, nnz=None, flags=0):
    nnz = len(vals) if nnz is None else nnz
    _check(h, load().ccg_set_matvec_csr(h, _ptr(rowptr), _ptr(colind), _ptr(vals), int(row0),
                                        int(nloc), int(nnz), int(flags)))
    _keepalive[h] = [rowptr, colind, vals]


def ccg_set_matvec_stencil7(h, nx, ny, nz, d, ox, oy=None, oz=None, flags=0):
    """Matrix-free 7-point stencil (d, ox, oy, oz complex scalars; oy, oz default to ox)."""
    oy = ox if oy is None else oy
    oz = ox if oz is None else oz
    co = (ctypes.c_double * 8)(*[float(v) for z in (d, ox, oy, oz) for v in (complex(z).real, complex(z).imag)])
    _check(h, load().ccg_set_matvec_stencil7(h, int(nx), int(ny), int(nz), co, int(flags)))
    _keepalive[h] = []


def ccg_set_matvec_toeplitz3(h, nx, ny, nz, kernel, diag, flags=0):
    """FFT block-Toeplitz operator; ``kernel``: complex128 array of K(δ) with
    shape (2nz−1, 2ny−1, 2nx−1), index [dz+nz−1, dy+ny−1, dx+nx−1]."""
    k = np.ascontiguousarray(kernel, dtype=np.complex128)
    if k.size != (2 * nx - 1) * (2 * ny - 1) * (2 * nz - 1):
        raise ValueError("kernel must have (2nx-1)(2ny-1)(2nz-1) entries")
    kp = k.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    d = (ctypes.c_double * 2)(complex(diag).real, complex(diag).imag)
    _check(h, load().ccg_set_matvec_toeplitz3(h, int(nx), int(ny), int(nz), kp, d, int(flags)))
    _keepalive[h] = []


def ccg_set_matvec_callback(h, fn, caps=CB_A, flags=0):
    """User operator: ``fn(op, x_ptr, y_ptr, n, row0, nloc, stream_ptr) -> int``
    must enqueue y[0:nloc] = (op(A)·x)[row0:row0+nloc] on the stream (device
    pointers; op 0 = A, 1 = Aᴴ, 2 = Aᵀ) and return 0."""
    def tramp(user, op, x, y, n, row0, nloc, stream):
        try:
            return int(fn(op, x, y, n, row0, nloc, stream) or 0)
        except Exception:  # pragma: no cover - reported as CCG_E_USER
            import traceback
            traceback.print_exc()
            return 1
    cfn = MATVEC_FN(tramp)
    _check(h, load().ccg_set_matvec_callback(h, cfn, None, int(caps), int(flags)))
    _keepalive[h] = [cfn, fn]


def ccg_set_matvec_callback_ptr(h, fn_addr, user_addr=None, caps=CB_A, flags=0):
    """Same, with a native function pointer (address) and an opaque user pointer."""
    cfn = ctypes.cast(ctypes.c_void_p(int(fn_addr)), MATVEC_FN)
    _check(h, load().ccg_set_matvec_callback(h, cfn, user_addr, int(caps), int(flags)))
    _keepalive[h] = [cfn]


def ccg_set_gmres_restart(h, m):
    _check(h, load().ccg_set_gmres_restart(h, int(m)))


def ccg_set_jacobi(h, diag_local, flags=0):
    """Right Jacobi preconditioning of later solves (diag_local: this rank's
    diagonal entries, host or device; None disables)."""
    _check(h, load().ccg_set_jacobi(h, None if diag_local is None else _ptr(diag_local, "diag"), int(flags)))


def ccg_set_bicgstab_ell(h, ell):
    _check(h, load().ccg_set_bicgstab_ell(h, int(ell)))


def ccg_apply(h, op, x, y):
    op = OPS[op] if isinstance(op, str) else int(op)
    _check(h, load().ccg_apply(h, op, _ptr(x, "x"), _ptr(y, "y")))


def ccg_solve(h, method, x0, y, x_out, tol, maxit):
    """Returns the ccg_result fields as a dict (status / breakdown as names)."""
    m = METHODS[method] if isinstance(method, str) else int(method)
    res = ccg_result()
    _check(h, load().ccg_solve(h, m, _ptr(x0, "x0"), _ptr(y, "y"), _ptr(x_out, "x_out"),
                               float(tol), int(maxit), ctypes.byref(res)))
    return {"status": STATUS[res.status], "iterations": res.iterations,
            "matvecs_a": res.matvecs_a, "matvecs_ah": res.matvecs_ah,
            "breakdown": BREAKDOWN.get(res.breakdown_code), "half_step": bool(res.half_step),
            "rec_rel_res": res.rec_rel_res, "true_rel_res": res.true_rel_res,
            "wall_ms": res.wall_ms}


def ccg_get_history(h, cap=1 << 20):
    buf = (ctypes.c_double * cap)()
    n = ctypes.c_int32()
    _check(h, load().ccg_get_history(h, buf, cap, ctypes.byref(n)))
    return np.array(buf[:n.value])


def ccg_set_timing(h, enable):
    _check(h, load().ccg_set_timing(h, int(bool(enable))))


def ccg_get_timing(h):
    a, ah = ctypes.c_double(), ctypes.c_double()
    na, nah = ctypes.c_int32(), ctypes.c_int32()
    _check(h, load().ccg_get_timing(h, ctypes.byref(a), ctypes.byref(na), ctypes.byref(ah),
                                    ctypes.byref(nah)))
    return {"ms_a": a.value, "n_a": na.value, "ms_ah": ah.value, "n_ah": nah.value}


def ccg_last_launch_count(h):
    return int(load().ccg_last_launch_count(h))


STATS = {"comm_kind": 0, "graph_replays": 1, "graph_collectives": 2, "eager_collectives": 3,
         "world": 4, "replicated": 5, "p2p_exchanges": 6, "symmetric": 7}


def ccg_get_stat(h, key):
    """Execution statistics of the last solve (include/ccg.h CCG_STAT_*)."""
    v = ctypes.c_int64()
    _check(h, load().ccg_get_stat(h, STATS[key], ctypes.byref(v)))
    return int(v.value)


def ccg_get_stats(h):
    return {k: ccg_get_stat(h, k) for k in STATS}


def ccg_get_stream(h):
    return load().ccg_get_stream(h)


def ccg_last_error(h=None):
    m = load().ccg_last_error(h)
    return m.decode() if m else ""


def ccg_destroy(h):
    _check(h, load().ccg_destroy(h))
    _keepalive.pop(h, None)
