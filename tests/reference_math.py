"""Error measures used by the parity tests (restated from the reference's
pkg/tests/reference.py:126-145)."""
import numpy as np


def relative_error(a, b, floor=1e-6):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) / np.maximum(floor, np.maximum(np.abs(a), np.abs(b)))


def scale_error(a, b, floor=1e-9):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(floor, float(np.abs(a).max(initial=0)), float(np.abs(b).max(initial=0)))
    return np.abs(a - b) / scale
