"""Seeded synthetic instances with BASELINE.json's construction
A = U diag(sigma) G / sqrt(n) (U Haar from the QR of a Gaussian, sigma
log-spaced 1 -> 1/kappa, G i.i.d. standard complex Gaussian), b Gaussian.
Host-side (numpy) for the parity tests; bench.py builds the large configs
directly on the GPU with the same recipe."""
from __future__ import annotations

import numpy as np


def haar(m: int, rng: np.random.Generator, real: bool = False) -> np.ndarray:
    if real:
        Z = rng.standard_normal((m, m))
    else:
        Z = (rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / np.sqrt(2)
    Q, R = np.linalg.qr(Z)
    d = np.diag(R)
    return Q * (d / np.abs(d))  # Haar: fix the phase of the QR


def make_instance(m: int, n: int, kappa: float, seed: int, real: bool = False):
    rng = np.random.default_rng(seed)
    U = haar(m, rng, real)
    s = np.logspace(0, -np.log10(kappa), m)
    if real:
        G = rng.standard_normal((m, n))
        b = rng.standard_normal(m).astype(np.complex128)
    else:
        G = (rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))) / np.sqrt(2)
        b = (rng.standard_normal(m) + 1j * rng.standard_normal(m)) / np.sqrt(2)
    A = np.asfortranarray((U * s) @ G / np.sqrt(n))
    return A, b
