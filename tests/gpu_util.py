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
