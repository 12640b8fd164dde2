"""Shared test helpers: inputs in the GPU contract (float32 means, 6 unique float32 covariance
entries) and the identical float64 view the oracle receives."""
from __future__ import annotations

import numpy as np

import oracle_ctypes as O


def contract_inputs(means, covs=None):
    """Round to the GPU input contract; return (means_f64_exact, cov9_f64_exact_symmetric, cov6_f32)."""
    m = np.asarray(means, dtype=np.float32).astype(np.float64).reshape(-1, 3)
    if covs is None:
        return m, None, None
    c = np.asarray(covs, dtype=np.float64)
    if c.ndim == 3:
        c = c.reshape(len(c), 9)
    if c.shape[1] == 9:
        c6 = c[:, [0, 1, 2, 4, 5, 8]]
    else:
        c6 = c
    c6 = c6.astype(np.float32)
    c9 = O.cov9(c6.astype(np.float64))
    return m, c9, c6


def rel_block_error(got: dict, ref: dict) -> dict:
    """‖Δ‖_F / max(1, ‖H_ii,ref‖_F) per block (test_reference.cpp:85-91 normalisation)."""
    scale = max(1.0, float(np.linalg.norm(ref["H_ii"])))
    out = {k: float(np.linalg.norm(np.asarray(got[k]) - np.asarray(ref[k])) / scale) for k in ("H_ii", "H_ij", "H_jj", "b_i", "b_j")}
    out["error"] = abs(float(got["error"]) - float(ref["error"])) / max(1.0, abs(float(ref["error"])))
    return out


def lin_dict(lin) -> dict:
    return dict(H_ii=lin.H_ii, H_ij=lin.H_ij, H_jj=lin.H_jj, b_i=lin.b_i, b_j=lin.b_j, error=lin.error, inliers=lin.inliers)
