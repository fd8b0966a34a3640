"""Seeded synthetic-input generators shared by the tests and bench.py.

This module holds none of the method's arithmetic: it only draws counter-based
random numbers (splitmix64 of seed XOR global index) and applies a
multiplicative / additive perturbation to a state array that the caller made
(by the oracle's or the product's own init_case).  Pure numpy.
"""
from __future__ import annotations

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser of (x + golden gamma), vectorised, mod 2^64."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, index: np.ndarray) -> np.ndarray:
    """U in [0,1) from (seed, global index); partition-independent."""
    z = splitmix64(np.uint64(seed) ^ index.astype(np.uint64))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def perturb(q: np.ndarray, seed: int, amp: float = 1e-2) -> np.ndarray:
    """Canonical SoA state q[4*N]: rho and e scaled by (1 + amp (2U-1)); rho u and
    rho v shifted by amp (2U-1).  Index = global position in q."""
    q = np.asarray(q, dtype=np.float64)
    n = q.size // 4
    u = 2.0 * uniform(seed, np.arange(q.size, dtype=np.uint64)) - 1.0
    out = q.copy()
    out[0:n] *= 1.0 + amp * u[0:n]
    out[n:2 * n] += amp * u[n:2 * n]
    out[2 * n:3 * n] += amp * u[2 * n:3 * n]
    out[3 * n:] *= 1.0 + amp * u[3 * n:]
    return out
