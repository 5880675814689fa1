"""helpers for the -m gpu parity tests (CUDA path vs oracle)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def to_dev(d):
    return {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in d.items()}


def csr_lists(off, idx):
    return [list(idx[off[b]:off[b + 1]]) for b in range(len(off) - 1)]


def per_target_error(out, ref):
    """(relative L2 error over all targets, worst per-target error): the largest norm of one
    target's error vector divided by the largest norm of a reference output vector."""
    ref = np.asarray(ref, np.float64)
    ref = ref.reshape(ref.shape[0], -1)
    out = np.asarray(out, np.float64).reshape(ref.shape)
    d = out - ref
    den = np.linalg.norm(ref)
    if den == 0:
        return float(np.abs(out).max(initial=0.0)), float(np.abs(out).max(initial=0.0))
    return float(np.linalg.norm(d) / den), float(np.linalg.norm(d, axis=1).max() / np.linalg.norm(ref, axis=1).max())


def assert_fmm_close(out, ref, tol, factor=10.0, label=""):
    """FMM / stress parity: the relative L2 error over all (sampled) targets is <= tol AND
    every single target is within factor x tol of the largest reference output
    (max_i |out_i - ref_i| <= factor tol max_i |ref_i|), so that a corrupted leaf of a few
    targets cannot hide inside the global norm.  Returns (rel_l2, worst)."""
    rel, worst = per_target_error(out, ref)
    print(f"{label} rel-L2 {rel:.3e}  worst target {worst:.3e}  (tol {tol:.1e}, per-target bound {factor * tol:.1e})")
    assert rel <= tol, f"{label}: rel-L2 {rel} > {tol}"
    assert worst <= factor * tol, f"{label}: worst target {worst} > {factor} x {tol}"
    return rel, worst
