"""Host-side phi1 setup (phi1(x) = (e^x - 1)/x): scalar/elementwise values,
the phi1 tensors of the split factors and dense phi1(tau A) matrices from an
eigendecomposition.  Same names and rounding as the reference module
``curvipat.phifun`` (phifun.py:23-71); evaluated once per (tau, coefficient)
before the time loop, as north_star allows.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .operators import EigenFactorization

_TAYLOR_CUTOFF = 1e-5
# Horner coefficients of 1 + x/2 + x^2/6 + ... + x^6/5040 (highest first)
_HORNER = (1.0 / 5040.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 1.0 / 2.0, 1.0 / 1.0)


def phi1(x):
    """Elementwise phi1 (phifun.py:23-37): degree-6 Taylor below 1e-5, else
    expm1(x)/x."""
    arr = np.asarray(x, dtype=float)
    flat = np.atleast_1d(arr).ravel()
    out = np.empty_like(flat)
    near = np.abs(flat) < _TAYLOR_CUTOFF
    xs = flat[near]
    acc = np.full_like(xs, _HORNER[0])
    for coef in _HORNER[1:]:
        acc = acc * xs + coef
    out[near] = acc
    far = flat[~near]
    out[~near] = np.expm1(far) / far
    if arr.ndim == 0:
        return float(out[0])
    return out.reshape(arr.shape)


@dataclass(frozen=True)
class PhiTensor:
    """phi1 over an outer product of spectral factors (phifun.py:40-49)."""

    field: np.ndarray
    tau_scale: float


def phi1_outer(tau_coeff: float, factors) -> PhiTensor:
    """phi1(tau_coeff * f1 (x) f2 [(x) f3]) (phifun.py:52-65)."""
    if not 2 <= len(factors) <= 3:
        raise ValueError(f"need 2 or 3 factor vectors, got {len(factors)}")
    vecs = [np.asarray(f, dtype=float) for f in factors]
    if any(v.ndim != 1 or v.size == 0 for v in vecs):
        raise ValueError("each factor must be a nonempty 1-d vector")
    prod = np.multiply.outer(vecs[0], vecs[1])
    if len(vecs) == 3:
        prod = np.multiply.outer(prod, vecs[2])
    return PhiTensor(field=phi1(tau_coeff * prod), tau_scale=tau_coeff)


def phi1_matrix(tau: float, fac: EigenFactorization) -> np.ndarray:
    """Dense phi1(tau A) = V diag(phi1(tau lambda)) V^-1 (phifun.py:68-71)."""
    return (fac.V * phi1(tau * fac.lambdas)[None, :]) @ fac.V_inv
