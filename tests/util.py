"""Parity metrics: norm-relative and max-normalised error.
Element-wise relative error is deliberately not used (a correct fp16 conv
reaches 0.18 element-wise on near-zero outputs)."""
import numpy as np


def as_np(t):
    try:
        import torch
        if isinstance(t, torch.Tensor):
            return t.detach().float().cpu().numpy()
    except ImportError:
        pass
    return np.asarray(t, dtype=np.float64)


def norm_rel(a, b):
    a, b = as_np(a).astype(np.float64), as_np(b).astype(np.float64)
    nb = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (nb if nb > 0 else 1.0))


def max_norm(a, b):
    a, b = as_np(a).astype(np.float64), as_np(b).astype(np.float64)
    mb = np.abs(b).max() if b.size else 0.0
    return float(np.abs(a - b).max() / (mb if mb > 0 else 1.0)) if b.size else 0.0


def assert_close(a, b, tol, what=""):
    nr, mn = norm_rel(a, b), max_norm(a, b)
    assert nr <= tol and mn <= tol, f"{what}: norm-rel {nr:.3e}, max-norm {mn:.3e} > {tol}"
    return nr, mn
