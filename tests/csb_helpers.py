"""Shared test helpers (importable as `csb_helpers`; tests/ is on sys.path)."""
import numpy as np


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def rel_gap(got: np.ndarray, want: np.ndarray) -> float:
    """Tensor-level parity metric of the reference tests:
    max|got - want| / max|want| (test_moments.cpp:22-24)."""
    den = max(1e-300, float(np.max(np.abs(want)))) if want.size else 1.0
    return float(np.max(np.abs(got - want))) / den if want.size else 0.0
