"""The drop-in boundary: librgs_cuda.so loads without a GPU, exports every symbol
include/rgs_cuda.h declares, and refuses to run (no CPU fallback) without a device."""
import os
import re
import subprocess

import pytest

from paper_2402_03307_b200 import rgs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rgs_cuda.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rgs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_python_binding_set():
    assert sorted(rgs.EXPORTS) == header_functions()


def test_library_exports_every_declared_symbol():
    lib = rgs.load_library()
    missing = [f for f in header_functions() if not hasattr(lib, f)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", rgs.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rgs_\w+)", out))
    assert set(header_functions()) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", rgs.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version():
    assert rgs.load_library().rgs_abi_version() == 1


def test_header_compiles_as_c():
    """Plain C: no CUDA / torch / C++ types in the boundary."""
    r = subprocess.run(["gcc", "-std=c99", "-fsyntax-only", "-x", "c", HEADER], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = rgs.load_library()
    assert lib.rgs_device_count() == 0
    with pytest.raises(rgs.RgsUnavailableError):
        rgs.Context(0)
    with pytest.raises(rgs.RgsUnavailableError):
        rgs.render_forward(rgs.GaussianStore.empty(1), rgs.Camera(8, 8, 8.0, 8.0, 4.0, 4.0))


def test_product_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2402_03307_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp", ".hpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "liboracle" not in text and "librgs_ref" not in text, f
