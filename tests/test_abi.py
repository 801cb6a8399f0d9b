"""The C-ABI library: builds/loads, exports every declared symbol (CPU only, no compute)."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ccg.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ccg_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1208_4869_b200 import build
    build.build()
    import paper_1208_4869_b200 as p
    return p.load()


def test_exports_every_declared_symbol(lib):
    import paper_1208_4869_b200 as p
    decl = declared_functions()
    assert len(decl) >= 14
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(p.EXPORTS) == decl
    out = subprocess.run(["nm", "-D", "--defined-only", p.LIB_PATH], capture_output=True, text=True).stdout
    for name in decl:
        assert re.search(rf"\bT {name}\b", out), f"{name} not exported with C linkage"


def test_binary_is_sm100a(lib):
    import paper_1208_4869_b200 as p
    out = subprocess.run(["cuobjdump", "--list-elf", p.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_enums_match_header(lib):
    import paper_1208_4869_b200 as p
    src = open(HEADER).read()
    for name, v in (("CCG_C64", p.C64), ("CCG_C128", p.C128), ("CCG_FLAG_SYMMETRIC", p.FLAG_SYMMETRIC)):
        assert re.search(rf"{name} = {v}\b", src), name
    for m, v in p.METHODS.items():
        assert re.search(rf"CCG_{m.upper()} = {v}\b", src), m
    for code, name in p.ERRORS.items():
        if code:
            assert re.search(rf"{name} = {code}\b", src), name
    for code, name in p.STATUS.items():
        nm = {"MAXIT": "CCG_MAXIT", "FALSE_CONVERGENCE": "CCG_FALSE_CONVERGENCE"}.get(name, "CCG_" + name)
        assert re.search(rf"{nm} = {code}\b", src), name
    # result struct layout: 6 int32 + 3 double
    assert ctypes.sizeof(p.ccg_result) == 6 * 4 + 3 * 8


def test_version_and_no_gpu_errors(lib):
    import paper_1208_4869_b200 as p
    assert "sm_100a" in p.ccg_version()
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    with pytest.raises(p.CcgError) as e:
        p.ccg_create("c128", 16)
    assert e.value.code == -5          # CCG_E_CUDA: no device, no CPU fallback
    with pytest.raises(p.CcgError) as e:
        p.ccg_create("c128", 15, world=2, rank=0, nccl_id=b"\0" * 128)
    assert e.value.code == -2          # n % world != 0


def test_oracle_not_imported_by_product():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_1208_4869_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "oracle/" not in txt.replace("oracle/)", ""), f
