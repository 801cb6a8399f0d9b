"""Build libccg.so in-tree with nvcc for sm_100a (explicit -gencode, no JIT)."""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libccg.so")
# translation units: the C-ABI, and the Engine<T> member definitions split by
# method group and compiled once per dtype (-DCCG_T), in parallel
GROUPS = ["hot", "next", "krylov", "cluster", "core"]
UNITS = [("ccg.cu", None)] + [(f"methods_{g}.cu", t) for g in GROUPS for t in ("float", "double")]
DEPS = ["ccg.cu", "engine.cuh", "common.cuh", "matvec.cuh", "methods.cuh", "bulk.cuh", "comm.cuh", "fft.cuh",
        "cluster.cuh", "gmres.cuh"] + [f"methods_{g}.cu" for g in GROUPS]


def nccl_include():
    import nvidia.nccl
    base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include")


def nccl_libdir():
    import nvidia.nccl
    base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "lib")


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(ROOT, "include", "ccg.h"), __file__]
    return all(os.path.getmtime(d) <= t for d in deps)


def _flags(verbose):
    return ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
            "-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
            "-I", os.path.join(ROOT, "include"), "-I", nccl_include()]


def build(force=False, verbose=False, jobs=None):
    if not force and up_to_date():
        return LIB
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    tmp = tempfile.mkdtemp(prefix="ccg_build_")

    def compile_unit(u):
        src, t = u
        obj = os.path.join(tmp, src.replace(".cu", "") + (f"_{t}" if t else "") + ".o")
        cmd = [nvcc(), "-c"] + _flags(verbose) + ([f"-DCCG_T={t}"] if t else []) + [
            os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return obj, r, cmd

    jobs = jobs or max(1, min(len(UNITS), os.cpu_count() or 1))
    with ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(compile_unit, UNITS))
    for obj, r, cmd in results:
        if r.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libccg.so")
        if verbose:
            sys.stderr.write(r.stderr)
    link = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB + ".tmp"] + \
        [o for o, _, _ in results] + ["-ldl", "-Xlinker", "-rpath=" + nccl_libdir()]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libccg.so")
    os.replace(LIB + ".tmp", LIB)
    for o, _, _ in results:
        os.remove(o)
    os.rmdir(tmp)
    return LIB

if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
