"""ctypes loader for oracle/c/direct_sum.c (fp64 O(N^2) direct sum, OpenMP).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Built by build_oracle() (called
from __graft_entry__.build() and on first use); pinned against oracle.kernels.direct_sum
in tests/test_oracle_kifmm.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "direct_sum.c")
LIB = os.path.join(HERE, "c", "liboracle_direct.so")
_lib = None


def build_oracle(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", LIB, SRC, "-lm"])
    return LIB


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        _lib = ctypes.CDLL(LIB)
        P = ctypes.POINTER(ctypes.c_double)
        _lib.oracle_direct_sum.argtypes = [ctypes.c_int, P, ctypes.c_long, P, P, P, P, P,
                                           ctypes.c_long, ctypes.c_double, ctypes.c_double, P]
        _lib.oracle_direct_sum.restype = None
    return _lib


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def direct_sum(kernel, trg, src, K, G, w=None, f=None, g=None, nrm=None):
    """same contract as oracle.kernels.direct_sum, computed by the C oracle."""
    lib = _load()
    trg = np.ascontiguousarray(trg, np.float64).reshape(-1, 3)
    src = np.ascontiguousarray(src, np.float64).reshape(-1, 3)
    conv = lambda a: None if a is None else np.ascontiguousarray(a, np.float64)
    w, f, g, nrm = conv(w), conv(f), conv(g), conv(nrm)
    out = np.zeros((trg.shape[0], 6 if kernel >= 3 else 3))
    lib.oracle_direct_sum(int(kernel), _ptr(trg), trg.shape[0], _ptr(src), _ptr(nrm), _ptr(w),
                          _ptr(f), _ptr(g), src.shape[0], float(K), float(G), _ptr(out))
    return out
