"""CPU: the C-ABI library loads, exports every symbol include/parcop_b200.h
declares, and its host-only logic (partition, argument validation, the
no-device failure mode) behaves like the reference — no compute calls."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "parcop_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pcb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1609_05530_b200 import _lib
    lib = _lib.load()
    decl = header_functions()
    assert len(decl) >= 18
    assert set(decl) == set(_lib.SYMBOLS)
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (pcb_[a-z0-9_]+)", nm))
    for name in decl:
        assert name in exported, name
        assert getattr(lib, name) is not None


def test_abi_version_and_struct_layout():
    from paper_1609_05530_b200 import _lib
    lib = _lib.load()
    assert lib.pcb_abi_version() == 2
    assert C.sizeof(_lib.FitResultC) == 48
    assert C.sizeof(_lib.CombinedC) == 32


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1609_05530_b200 import _lib
    import paper_1609_05530_b200 as pcb
    lib = _lib.load()
    assert not lib.pcb_create(0)
    assert b"no CUDA device" in lib.pcb_last_error(None)
    devs = (C.c_int * 2)(0, 0)
    assert not lib.pcb_create_multi(devs, 2)
    assert not lib.pcb_create_multi(devs, 0)
    assert lib.pcb_device_count(None) == 0
    with pytest.raises(pcb.CudaError):
        pcb.Context(0)
    # every compute entry point refuses a NULL context instead of computing elsewhere
    assert lib.pcb_fit(None, 0, 0, None, None, 0, None, 0, None) == _lib.PCB_E_INVALID


def test_partition_contiguous_and_strided():
    import paper_1609_05530_b200 as pcb
    p = pcb.partition(10 * 30, 3)
    assert list(np.diff(p.offsets)) == [100, 100, 100]
    p = pcb.partition(100, 3)  # remainder to the last block
    assert list(np.diff(p.offsets)) == [33, 33, 34]
    assert list(pcb.partition(200000, 100).offsets[:3]) == [0, 2000, 4000]
    s = pcb.partition(100, 3, pcb.Scheme.Strided)  # row i -> block i mod M
    assert list(np.diff(s.offsets)) == [34, 33, 33]
    with pytest.raises(ValueError):
        pcb.partition(10, 3)  # 30-row floor
    with pytest.raises(ValueError):
        pcb.partition(100, 0)


def test_host_validation_before_device():
    import paper_1609_05530_b200 as pcb
    with pytest.raises(ValueError):
        pcb.normalized_ranks(pcb.DataMatrix([1.0, 2.0], [1.0]))
    with pytest.raises(ValueError):
        pcb.normalized_ranks(pcb.DataMatrix([1.0], [2.0]))
    with pytest.raises(ValueError):
        pcb.combine([])
    with pytest.raises(ValueError):
        pcb.fit_parallel(0, pcb.DataMatrix([1.0] * 100, [2.0] * 100), 0)
    assert pcb.family_from_string("Normal") == pcb.CopulaFamily.Gaussian
    assert pcb.family_from_string("gumbel") == pcb.CopulaFamily.Gumbel
    assert pcb.family_from_string("clayton") is None


def test_product_does_not_touch_oracle():
    """The product package never imports / includes / links the oracle."""
    pkg = os.path.join(ROOT, "paper_1609_05530_b200")
    bad = re.compile(r"^\s*(import oracle|from oracle|#include\s+[<\"].*oracle)", re.M)
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".hpp", ".h", ".cpp")) or f == "Makefile":
                txt = open(os.path.join(dp, f), errors="ignore").read()
                assert not bad.search(txt), f
                if f == "Makefile":
                    assert "oracle" not in txt
    from paper_1609_05530_b200 import _lib
    ldd = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in ldd and "parcop_ref" not in ldd


def test_mixed_include_translation_unit_compiles(tmp_path):
    """The reference's own headers and include/parcop_b200.hpp in ONE
    translation unit (tests/cpp/mixed_include.cpp): the header adopts the
    reference's DataMatrix / PseudoSample / CopulaFamily instead of
    redefining them. Compile-only here (run on the GPU by test_gpu_cpp)."""
    ref = "/root/reference/proj/include"
    if not os.path.isdir(ref):
        pytest.skip("reference headers not present (GPU box)")
    src = os.path.join(ROOT, "tests", "cpp", "mixed_include.cpp")
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-include",
                        os.path.join(ROOT, "oracle", "shim.hpp"), "-I" + ref, "-I" + os.path.join(ROOT, "include"),
                        src], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    # and the standalone header still defines the types itself
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "api_smoke.cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
