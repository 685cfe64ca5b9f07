"""The stated numeric bar of the floating-point outputs (BASELINE.json north_star):
bf16 inputs with fp32 accumulation within 2e-2 relative error of the fp32 oracle, fp32 mode
within 1e-4 — measured PER OUTPUT ROW (token): max |y - y_ref| over the row divided by
max |y_ref| of that row, then the worst row.  A globally normalised error
(max |y - y_ref| / max |y_ref| over the whole batch) would let small-magnitude tokens hide
large relative errors, so no test uses it."""
import numpy as np

TOL_BF16 = 2e-2
TOL_FP32 = 1e-4


def row_rel_errs(y, y_ref):
    """Per-row relative errors (rows of zeros in y_ref compare absolutely)."""
    y_ref = np.asarray(y_ref, dtype=np.float64)
    if y_ref.size == 0:
        return np.zeros(0)
    y = np.asarray(y, dtype=np.float64).reshape(len(y_ref), -1)
    y_ref = y_ref.reshape(len(y_ref), -1)
    den = np.max(np.abs(y_ref), axis=1)
    den = np.where(den > 0, den, 1.0)
    return np.max(np.abs(y - y_ref), axis=1) / den


def row_rel_err(y, y_ref):
    """Worst per-row relative error (0 for an empty batch)."""
    e = row_rel_errs(y, y_ref)
    return float(e.max()) if e.size else 0.0
