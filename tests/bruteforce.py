"""Dense brute force (numpy, complex128) for N <= 12: the checker that pins the oracle.

Statevector: psi as a (d,)*N tensor, site 0 the most significant digit (E1).
Density operator: vec(rho) as a (4,)*N tensor with site index s = 2 sigma + sigma' (E3,
PAPER.md:46-51; SURVEY.md §8(c) algorithm item 9). Gates are applied locally by tensordot on the
two affected axes, never embedded into a 2^N x 2^N matrix.
Fidelities: E7 (pure) and E9 (Wang).
"""
from __future__ import annotations

import numpy as np


def product_zero(n: int, d: int = 2) -> np.ndarray:
    psi = np.zeros((d,) * n, np.complex128)
    psi[(0,) * n] = 1.0
    return psi


def apply_2site(psi: np.ndarray, site: int, U: np.ndarray) -> np.ndarray:
    """psi'[.., s, t, ..] = sum U[s d + t, s' d + t'] psi[.., s', t', ..]."""
    d = psi.shape[site]
    U4 = np.asarray(U, np.complex128).reshape(d, d, d, d)
    out = np.tensordot(U4, psi, axes=([2, 3], [site, site + 1]))  # s,t, rest...
    return np.moveaxis(out, [0, 1], [site, site + 1])


def apply_1site(psi: np.ndarray, site: int, U: np.ndarray) -> np.ndarray:
    out = np.tensordot(np.asarray(U, np.complex128), psi, axes=([1], [site]))
    return np.moveaxis(out, 0, site)


def run_circuit(n: int, layers, d: int = 2) -> np.ndarray:
    psi = product_zero(n, d)
    for sites, us in layers:
        for i, u in zip(sites, us):
            psi = apply_2site(psi, int(i), u)
    return psi


def pure_fidelity(a: np.ndarray, b: np.ndarray) -> float:
    """E7: |<a|b>|^2 for normalised a, b (both are normalised here)."""
    a = a.ravel() / np.linalg.norm(a)
    b = b.ravel() / np.linalg.norm(b)
    return float(abs(np.vdot(a, b)) ** 2)


def rho_matrix(vec: np.ndarray) -> np.ndarray:
    """vec(rho) (4,)*N with s = 2 sigma + sigma'  ->  2^N x 2^N matrix rho[sigma, sigma']."""
    n = vec.ndim
    t = vec.reshape((2, 2) * n)  # sigma1, sigma1', sigma2, sigma2', ...
    perm = list(range(0, 2 * n, 2)) + list(range(1, 2 * n, 2))
    return t.transpose(perm).reshape(2 ** n, 2 ** n)


def wang_fidelity(rho: np.ndarray, sig: np.ndarray) -> float:
    """E9: |Tr(rho sigma)| / sqrt(Tr(rho^2) Tr(sigma^2))."""
    num = abs(np.trace(rho @ sig))
    den = np.sqrt(abs(np.trace(rho @ rho)) * abs(np.trace(sig @ sig)))
    return float(num / den)
