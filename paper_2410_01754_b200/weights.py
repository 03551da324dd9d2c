"""Titration weight algebra (reference weights.py:54-85), host side.

Form rho of a site with L lambdas has weight prod_k (lambda_k if bit k of
rho else 1 - lambda_k), lambda_0 on the least significant bit.  The device
HI kernel recomputes the same products in the same order; these helpers
only build the API objects (TildeWeights) and validate shapes.
"""

from dataclasses import dataclass

import numpy as np

MAX_BRANCHES = 4


def _lams(lams):
    arr = np.asarray(lams, dtype=np.float64)
    if arr.ndim != 1 or not 1 <= arr.shape[0] <= MAX_BRANCHES:
        raise ValueError(f"need between 1 and {MAX_BRANCHES} lambda values, got shape {arr.shape}")
    return arr


@dataclass(frozen=True)
class TildeWeights:
    lambdas: tuple
    values: np.ndarray

    @property
    def num_forms(self):
        return self.values.shape[0]

    def fingerprint(self):
        return tuple(float(v) for v in self.lambdas)


def expand_weights(lams):
    arr = _lams(lams)
    nf = 1 << arr.shape[0]
    vals = np.empty(nf)
    for rho in range(nf):
        w = 1.0
        for k, lam in enumerate(arr):
            w *= lam if (rho >> k) & 1 else 1.0 - lam
        vals[rho] = w
    return TildeWeights(lambdas=tuple(float(x) for x in arr), values=vals)


def weight_gradient(lams, k):
    arr = _lams(lams)
    if not 0 <= k < arr.shape[0]:
        raise ValueError(f"branch index {k} out of range for {arr.shape[0]} lambdas")
    nf = 1 << arr.shape[0]
    out = np.empty(nf)
    for rho in range(nf):
        g = 1.0
        for i, lam in enumerate(arr):
            bit = (rho >> i) & 1
            if i == k:
                g *= 1.0 if bit else -1.0
            else:
                g *= lam if bit else 1.0 - lam
        out[rho] = g
    return out


def weight_gradient_matrix(lams):
    arr = _lams(lams)
    return np.stack([weight_gradient(arr, k) for k in range(arr.shape[0])])
