"""B200-native elastostatic BEM / KIFMM hot path (arXiv:1612.04082), Python binding.

Thin ctypes marshalling over the C ABI of ``lib/libelastobem.so`` (declared in
``include/elastobem.h``): the same entry points, the same argument order.  Every
computation runs in the CUDA library; there is no Python or CPU fallback -- importing
this package fails if the library has not been built (``__graft_entry__.build()``).

Arrays may be torch CUDA tensors (the call is asynchronous on the current torch stream)
or host arrays (numpy / CPU tensors; the library stages them and returns when done).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libelastobem.so")
if os.environ.get("EBEM_LIB_VARIANT"):       # A/B measurement builds (_build.py variant ...)
    LIB_PATH = os.path.join(_HERE, "lib", "variants", os.environ["EBEM_LIB_VARIANT"] + ".so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")

_lib = ctypes.CDLL(LIB_PATH)

KERNEL_U, KERNEL_P, KERNEL_UP, KERNEL_D, KERNEL_S, KERNEL_DS = range(6)
_VP = ctypes.c_void_p
_I64 = ctypes.c_int64

_lib.ebem_last_error.restype = ctypes.c_char_p
_lib.bem_kernel_direct.argtypes = [ctypes.c_int, _VP, _I64, _VP, _VP, _VP, _VP, _VP, _I64,
                                   ctypes.c_double, ctypes.c_double, _VP, _VP]
_lib.fmm_build_tree.argtypes = [_VP, _VP, _VP, _I64, _VP, _I64, ctypes.c_int, ctypes.c_int,
                                ctypes.c_double, ctypes.c_double, ctypes.POINTER(_VP), _VP]
_lib.fmm_matvec.argtypes = [_VP, ctypes.c_int, _VP, _VP, _VP, _VP]
_lib.fmm_eval_stress.argtypes = [_VP, ctypes.c_int, _VP, _VP, _VP, _VP]
_lib.fmm_tree_free.argtypes = [_VP]
_lib.fmm_tree_export.argtypes = [_VP, ctypes.c_int, _VP, _I64]
_lib.fmm_tree_export.restype = _I64
_lib.bem_create.argtypes = [_VP, _I64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                            ctypes.c_double, ctypes.POINTER(_VP), _VP]
_lib.bem_apply.argtypes = [_VP, _VP, _VP, _VP, _VP]
_lib.bem_rhs.argtypes = [_VP, _VP, _VP, _VP, _VP]
_lib.bem_gmres_solve.argtypes = [_VP, _VP, _VP, _VP, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                 ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double), _VP]
_lib.bem_free.argtypes = [_VP]
_lib.bem_gmres_history.argtypes = [_VP, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int]


class TreeInfo(ctypes.Structure):
    _fields_ = [("nsrc", _I64), ("ntrg", _I64), ("nboxes", _I64), ("nleaves", _I64),
                ("nlevels", ctypes.c_int32), ("p", ctypes.c_int32), ("max_pts", ctypes.c_int32),
                ("n_equiv", ctypes.c_int32), ("n_u", _I64), ("n_v", _I64), ("n_w", _I64),
                ("n_x", _I64), ("origin", ctypes.c_double * 3), ("side", ctypes.c_double),
                ("device_bytes", _I64)]


_lib.fmm_tree_info.argtypes = [_VP, ctypes.POINTER(TreeInfo)]


class PhaseStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 16), ("launches", ctypes.c_int32), ("fp64", ctypes.c_int32),
                ("flops", ctypes.c_double), ("flops_fp64", ctypes.c_double),
                ("interactions", ctypes.c_double), ("bytes", ctypes.c_double),
                ("ms", ctypes.c_double)]


_lib.fmm_set_profiling.argtypes = [_VP, ctypes.c_int]
_lib.fmm_phase_stats.argtypes = [_VP, ctypes.c_int, ctypes.POINTER(PhaseStat), ctypes.c_int]
_lib.ebem_launch_count.restype = _I64
_lib.ebem_trim_cache.restype = _I64


class EbemError(RuntimeError):
    pass


def _check(rc):
    if rc != 0:
        raise EbemError(f"elastobem error {rc}: {_lib.ebem_last_error().decode()}")


def _is_cuda(a):
    return a is not None and hasattr(a, "is_cuda") and a.is_cuda


def _ptr(a, keep, writes=False):
    """device or host pointer of a float32/int32 contiguous array (None -> NULL).  Inputs may
    be non-contiguous (a contiguous copy is passed); an array the library WRITES (an output,
    or GMRES's in-place x) must be contiguous, or the result would land in a temporary."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):                      # torch tensor
        if not a.is_contiguous():
            if writes:
                raise ValueError("output / in-place array must be contiguous")
            a = a.contiguous()
        keep.append(a)
        return a.data_ptr()
    if writes:
        if not (isinstance(a, np.ndarray) and a.flags["C_CONTIGUOUS"] and a.dtype == np.float32):
            raise ValueError("output array must be a C-contiguous float32 numpy array or tensor")
        return a.ctypes.data
    arr = np.ascontiguousarray(a)
    keep.append(arr)
    return arr.ctypes.data


def _bc(bc_type):
    """boundary-condition types as int32 (the C ABI reads int32_t): integer arrays of another
    width are converted explicitly; anything else is an error."""
    if hasattr(bc_type, "dtype") and hasattr(bc_type, "data_ptr"):
        import torch
        if bc_type.dtype == torch.int32:
            return bc_type
        if bc_type.dtype.is_floating_point or bc_type.dtype == torch.bool:
            raise TypeError("bc_type must be an integer tensor")
        return bc_type.to(torch.int32)
    arr = np.asarray(bc_type)
    if not np.issubdtype(arr.dtype, np.integer):
        raise TypeError("bc_type must be an integer array")
    return np.ascontiguousarray(arr, dtype=np.int32)


def _stream(*arrs):
    if any(_is_cuda(a) for a in arrs):
        import torch
        return torch.cuda.current_stream().cuda_stream
    return None


def _f32(a):
    if a is None or hasattr(a, "data_ptr"):
        if a is not None:
            import torch
            assert a.dtype == torch.float32, "float32 expected"
        return a
    return np.ascontiguousarray(a, dtype=np.float32)


def _out_like(ref, shape):
    if _is_cuda(ref):
        import torch
        return torch.empty(shape, dtype=torch.float32, device=ref.device)
    return np.empty(shape, dtype=np.float32)


def bem_kernel_direct(kernel, trg, src, nrm=None, w=None, f=None, g=None, K=1.0, G=0.5, out=None):
    """O(N^2) sum of Eq. fmm_summation on the GPU; see include/elastobem.h."""
    trg, src, nrm, w, f, g = map(_f32, (trg, src, nrm, w, f, g))
    ntrg = int(trg.shape[0]) if trg.ndim == 2 else int(trg.shape[0]) // 3
    nsrc = int(src.shape[0]) if src.ndim == 2 else int(src.shape[0]) // 3
    nc = 6 if kernel >= KERNEL_D else 3
    if out is None:
        out = _out_like(trg, (ntrg, nc))
    keep = []
    _check(_lib.bem_kernel_direct(kernel, _ptr(trg, keep), ntrg, _ptr(src, keep), _ptr(nrm, keep),
                                  _ptr(w, keep), _ptr(f, keep), _ptr(g, keep), nsrc, float(K),
                                  float(G), _ptr(out, keep, True), _stream(trg, out)))
    return out


class FmmTree:
    """owning wrapper of an ebem_tree* (fmm_build_tree / fmm_tree_free)."""

    def __init__(self, handle, nsrc, ntrg, device):
        self.handle = handle
        self.nsrc, self.ntrg, self.device = nsrc, ntrg, device

    def __del__(self):
        h = getattr(self, "handle", None)
        self.handle = None
        if h and _lib is not None:
            try:
                _lib.fmm_tree_free(h)
            except Exception:       # interpreter teardown
                pass

    def info(self):
        return fmm_tree_info(self)


def fmm_build_tree(src, nrm=None, w=None, trg=None, max_pts=64, p=6, K=1.0, G=0.5):
    trg = src if trg is None else trg
    src, nrm, w, trg = map(_f32, (src, nrm, w, trg))
    nsrc = int(src.shape[0])
    ntrg = int(trg.shape[0])
    h = _VP()
    keep = []
    _check(_lib.fmm_build_tree(_ptr(src, keep), _ptr(nrm, keep), _ptr(w, keep), nsrc, _ptr(trg, keep),
                               ntrg, int(max_pts), int(p), float(K), float(G), ctypes.byref(h),
                               _stream(src, trg)))
    return FmmTree(h.value, nsrc, ntrg, src.device if _is_cuda(src) else None)


def _fmm_eval(fn, tree, kernel, f, g, out, nc):
    f, g = _f32(f), _f32(g)
    ref = f if f is not None else g
    if out is None:
        out = _out_like(ref, (tree.ntrg, nc))
    keep = []
    _check(fn(tree.handle, kernel, _ptr(f, keep), _ptr(g, keep), _ptr(out, keep, True), _stream(f, g, out)))
    return out


def fmm_matvec(tree, kernel, f=None, g=None, out=None):
    """KIFMM sum with displacement output (U, P, UP); see include/elastobem.h."""
    return _fmm_eval(_lib.fmm_matvec, tree, kernel, f, g, out, 3)


def fmm_eval_stress(tree, kernel, f=None, g=None, out=None):
    """KIFMM sum with stress output (D, S, DS), Voigt order; see include/elastobem.h."""
    return _fmm_eval(_lib.fmm_eval_stress, tree, kernel, f, g, out, 6)


def fmm_tree_info(tree):
    info = TreeInfo()
    _check(_lib.fmm_tree_info(tree.handle, ctypes.byref(info)))
    d = {k: getattr(info, k) for k, _ in TreeInfo._fields_}
    d["origin"] = tuple(info.origin)
    return d


_EXPORT = {"keys": (0, np.int64, 1), "perm": (1, np.int32, 1), "level": (2, np.int32, 1),
           "anchor": (3, np.int32, 3), "parent": (4, np.int32, 1), "range": (5, np.int32, 2),
           "U_off": (6, np.int32, 1), "V_off": (7, np.int32, 1), "W_off": (8, np.int32, 1),
           "X_off": (9, np.int32, 1), "U": (10, np.int32, 1), "V": (11, np.int32, 1),
           "W": (12, np.int32, 1), "X": (13, np.int32, 1)}


def fmm_tree_export(tree, what):
    code, dt, width = _EXPORT[what]
    info = fmm_tree_info(tree)
    n = {0: info["nsrc"] + info["ntrg"], 1: info["nsrc"] + info["ntrg"]}.get(code)
    if n is None:
        if 6 <= code <= 9:
            n = info["nboxes"] + 1
        elif code >= 10:
            n = info[["n_u", "n_v", "n_w", "n_x"][code - 10]]
        else:
            n = info["nboxes"]
    buf = np.zeros(max(n, 1) * width, dtype=dt)
    got = _lib.fmm_tree_export(tree.handle, code, buf.ctypes.data, buf.nbytes)
    if got < 0:
        _check(got)
    buf = buf[: n * width]
    return buf.reshape(-1, width) if width > 1 else buf


def fmm_set_profiling(tree, on=True):
    """native phase profiler: on = False/0 off, True/1 "solo" (phases one after another),
    2 or "insitu" (the normal overlapped schedule, events on each phase's own stream)."""
    mode = 2 if on == "insitu" else int(on)
    _check(_lib.fmm_set_profiling(tree.handle, mode))


def fmm_phase_stats(tree, kernel):
    """per-phase launches, algorithmic flops/bytes/interactions and last profiled device ms."""
    arr = (PhaseStat * 16)()
    n = _lib.fmm_phase_stats(tree.handle, kernel, arr, 16)
    if n < 0:
        _check(n)
    return [dict(name=a.name.decode(), launches=a.launches, fp64=bool(a.fp64), flops=a.flops,
                 flops_fp64=a.flops_fp64,
                 interactions=a.interactions, bytes=a.bytes, ms=a.ms) for a in arr[:n]]


def ebem_launch_count():
    """CUDA kernel launches issued by the library since it was loaded."""
    return int(_lib.ebem_launch_count())


def ebem_trim_cache():
    """Return the library's cached device blocks to the driver; the bytes freed."""
    return int(_lib.ebem_trim_cache())


class BemOperator:
    """owning wrapper of an ebem_bem* (bem_create / bem_free): the collocation BEM operator."""

    def __init__(self, handle, npanels):
        self.handle, self.n = handle, npanels

    def __del__(self):
        h = getattr(self, "handle", None)
        self.handle = None
        if h and _lib is not None:
            try:
                _lib.bem_free(h)
            except Exception:
                pass


def bem_create(vertices, nq=16, max_pts=64, p=6, K=1.0, G=0.5):
    """vertices: (n, 3, 3) or (n, 9) float32, counter-clockwise seen from outside."""
    v = _f32(vertices)
    n = int(v.shape[0])
    h = _VP()
    keep = []
    _check(_lib.bem_create(_ptr(v, keep), n, int(nq), int(max_pts), int(p), float(K), float(G),
                           ctypes.byref(h), _stream(v)))
    return BemOperator(h.value, n)


def bem_apply(bem, bc_type, x, out=None):
    import torch
    out = torch.empty_like(x) if out is None else out
    keep = []
    _check(_lib.bem_apply(bem.handle, _ptr(_bc(bc_type), keep), _ptr(_f32(x), keep), _ptr(out, keep, True),
                          _stream(x)))
    return out


def bem_rhs(bem, bc_type, bc_val, out=None):
    import torch
    out = torch.empty_like(bc_val) if out is None else out
    keep = []
    _check(_lib.bem_rhs(bem.handle, _ptr(_bc(bc_type), keep), _ptr(_f32(bc_val), keep), _ptr(out, keep, True),
                        _stream(bc_val)))
    return out


def bem_gmres_solve(bem, bc_type, bc_val, x, restart=50, max_iter=1000, tol=1e-6, precond=0, check=True):
    """solves A x = b in place; returns (x, iterations, relative residual).
    precond: 0 none (the paper's GMRES), 1 block-Jacobi (3x3 panel blocks), 2 leaf-block
    Jacobi (the diagonal blocks of A over each octree leaf's panels) right preconditioner."""
    keep = []
    it = ctypes.c_int32(0)
    res = ctypes.c_double(0)
    rc = _lib.bem_gmres_solve(bem.handle, _ptr(_bc(bc_type), keep), _ptr(_f32(bc_val), keep), _ptr(_f32(x), keep, True),
                              int(restart),
                              int(max_iter), float(tol), int(precond), ctypes.byref(it), ctypes.byref(res),
                              _stream(x))
    if check or rc not in (0, -4):
        _check(rc)
    return x, int(it.value), float(res.value)


def bem_gmres_history(bem):
    """residual history of the last bem_gmres_solve: (Arnoldi estimate per iteration, true
    relative residual at every restart and at the end), as numpy float64 arrays."""
    out = []
    for what in (0, 1):
        n = _lib.bem_gmres_history(bem.handle, what, None, 0)
        if n < 0:
            _check(n)
        buf = (ctypes.c_double * max(n, 1))()
        _lib.bem_gmres_history(bem.handle, what, buf, n)
        out.append(np.array(buf[:n], dtype=np.float64))
    return tuple(out)


__all__ = ["bem_kernel_direct", "fmm_build_tree", "fmm_matvec", "fmm_eval_stress", "fmm_tree_info",
           "fmm_tree_export", "bem_create", "bem_apply", "bem_rhs", "bem_gmres_solve", "bem_gmres_history", "BemOperator", "fmm_set_profiling", "fmm_phase_stats",
           "ebem_launch_count", "ebem_trim_cache", "FmmTree", "EbemError", "LIB_PATH",
           "KERNEL_U", "KERNEL_P", "KERNEL_UP", "KERNEL_D", "KERNEL_S", "KERNEL_DS"]
