"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, and exports every
entry point include/elastobem.h declares.  No compute calls (no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "elastobem.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|int64_t|const char \*)\s*\*?\s*(\w+)\s*\(", txt)))


def test_header_declares_the_north_star_entry_points():
    names = _declared()
    for n in ("bem_kernel_direct", "fmm_build_tree", "fmm_matvec", "fmm_eval_stress", "bem_gmres_solve"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_1612_04082_b200 import _build
    lib = _build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)$", out, flags=re.M))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    # and it is an sm_100a binary
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in sass


def test_binding_loads():
    import paper_1612_04082_b200 as eb
    assert os.path.exists(eb.LIB_PATH)
    for n in _declared():
        assert hasattr(eb._lib, n)
    # the binding exposes the same names
    for n in ("bem_kernel_direct", "fmm_build_tree", "fmm_matvec", "fmm_eval_stress", "bem_gmres_solve"):
        assert callable(getattr(eb, n))


def test_errors_without_gpu_are_reported_not_silent():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_1612_04082_b200 as eb
    with pytest.raises(eb.EbemError):
        eb.bem_kernel_direct(eb.KERNEL_U, np.zeros((4, 3)), np.ones((4, 3)), f=np.ones((4, 3)))
