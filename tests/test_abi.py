"""CPU-side checks of the boundary: libmem.so builds/loads, exports exactly what
include/mem.h declares, fails loudly without a GPU, and shares no code with the oracle."""
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "mem.h")).read()
    return sorted(set(re.findall(r"MEM_API\s+[\w\s\*]+?\b(mem_\w+)\s*\(", src)))


def test_library_exports_header():
    from paper_2309_16818_b200 import build
    lib = build.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib]).decode()
    exported = sorted(set(re.findall(r" T (mem_\w+)", out)))
    declared = header_functions()
    assert declared, "no declarations parsed"
    assert exported == declared, (set(declared) ^ set(exported))
    from paper_2309_16818_b200 import mem
    assert sorted(mem.EXPORTS) == declared


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2309_16818_b200 import mem
    with pytest.raises(mem.MemError) as e:
        mem.Map(0.1, 8, 8)
    assert e.value.status == mem.MEM_ECUDA
    assert "no CPU fallback" in str(e.value)


def test_sm100a_cubin_only():
    """the library carries sm_100a SASS (no PTX JIT to other archs)."""
    from paper_2309_16818_b200 import build
    lib = build.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib]).decode()
    assert "sm_100a" in out
    # -fmad=false: the PTX of the kernels has no floating-point fma/mad (D29: fixed op order;
    # the FFMA/DFMA in the SASS are the IEEE div/sqrt Newton sequences of div.rn / sqrt.rn)
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        ptx = os.path.join(d, "k.ptx")
        subprocess.check_call([build.NVCC, *build.ARCH, "-O3", "-std=c++17", "-fmad=false", "--extended-lambda",
                               "-I", os.path.join(ROOT, "include"), "-ptx",
                               os.path.join(build.CSRC, "kernels.cu"), "-o", ptx])
        txt = open(ptx).read()
    assert not re.search(r"\b(fma|mad)\.(rn\.)?f(32|64)", txt), "floating-point fma in PTX"
    assert "div.rn.f32" in txt and "div.rn.f64" in txt  # IEEE divisions, never approximate


def test_product_and_oracle_share_nothing():
    prod = glob.glob(os.path.join(ROOT, "paper_2309_16818_b200", "**", "*.*"), recursive=True)
    for p in prod:
        if p.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
            txt = open(p).read()
            assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower() or p.endswith("build.py"), p
            assert "mem_oracle" not in txt, p
    ora = open(os.path.join(ROOT, "oracle", "mem_oracle.c")).read()
    includes = set(re.findall(r"#include\s*[<\"]([^>\"]+)", ora))
    assert includes <= {"math.h", "stdint.h", "stdlib.h", "string.h", "stdio.h"}, includes
    oracle_py = open(os.path.join(ROOT, "oracle", "oracle.py")).read()
    assert not re.search(r"^\s*(from|import)\s+paper_2309_16818_b200", oracle_py, re.M)


def test_binding_rejects_wrong_dtype_and_small_buffers():
    """the binding refuses float64 clouds / images and undersized outputs before
    anything reaches the C-ABI (no device needed: the checks run first)."""
    import numpy as np
    import pytest
    from paper_2309_16818_b200 import mem as M
    with pytest.raises(TypeError):
        M._buf(np.zeros((10, 4)), "float32", 40, "points")
    with pytest.raises(ValueError):
        M._buf(np.zeros(39, np.float32), "float32", 40, "points")
    assert M._buf(np.zeros(40, np.float32), "float32", 40, "points")
    torch = pytest.importorskip("torch")
    with pytest.raises(TypeError):
        M._buf(torch.zeros(10, 4, dtype=torch.float64), "float32", 40, "points")
