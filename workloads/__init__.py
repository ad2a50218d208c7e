"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no contraction, SVD, truncation or ledger).
It only draws the random inputs the paper's workloads are made of, with the recipe of
SURVEY.md §8(d) / DESIGN.md "Input recipe":

* Haar-random two-qubit gates U(4) (PAPER.md:153, 171, 183 -- "Haar-random unitary matrices";
  the sampler is the Ginibre + QR + R-diagonal phase fix of SPEC.md:157, 162).
* Brickwork layers: layer t holds gates on (i, i+1) with i = t (mod 2)  (BASELINE.json configs).
* The MPO superoperator S = (D (x) D)(U (x) U*) with the depolarising map D of SPEC.md:340
  (noise placement: after every gate).
* Config-2 microbench thetas: theta = X diag(sigma) Y^H with Haar X, Y and sigma_k ~ k^-1.5
  (BASELINE.json configs[1]), rounded to complex64.

Every value handed to both sides is rounded to complex64 first, so
the oracle (complex128) and the GPU path (complex64) consume bit-identical numbers.

Seeds: numpy default_rng([230716870, config, ...]) (PCG64 via SeedSequence).
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 230716870

# BASELINE.json configs, indexed 1..5 as in SURVEY.md §8(d)
CONFIGS = {
    1: dict(kind="mps", n_sites=12, d=2, depth=8, f_min=0.99, strategy="global", chi_cap=0),
    2: dict(kind="micro", chis=(16, 64, 256, 1024), count=4096, f_trunc=0.9999, rule="pure"),
    3: dict(kind="mps", n_sites=50, d=2, depth=20, f_min=0.9, strategy="global", chi_cap=4096),
    4: dict(kind="mpo", n_sites=40, d=4, depth=16, f_min=0.95, strategy="global", chi_cap=4096,
            p_depol=0.01),
    5: dict(kind="mps", n_sites=300, d=2, depth=75, f_min=0.9, strategy="global", chi_cap=4096),
}


def rng_for(*key: int) -> np.random.Generator:
    return np.random.default_rng([SEED_BASE, *[int(k) for k in key]])


def haar_from_ginibre(z: np.ndarray) -> np.ndarray:
    """U = Q diag(R_ii/|R_ii|) for Z = QR. Unique for a given Z."""
    q, r = np.linalg.qr(z)
    dg = np.diagonal(r, axis1=-2, axis2=-1)
    ph = dg / np.abs(dg)
    return q * ph[..., None, :]


def ginibre(rng: np.random.Generator, n: int, batch: tuple = ()) -> np.ndarray:
    """Complex Ginibre matrix; the real block is drawn first."""
    re = rng.standard_normal(batch + (n, n))
    im = rng.standard_normal(batch + (n, n))
    return (re + 1j * im) / np.sqrt(2.0)


def haar_u4(*key: int) -> np.ndarray:
    """One Haar-random U(4), rounded to complex64 (returned as complex64)."""
    return haar_from_ginibre(ginibre(rng_for(*key), 4)).astype(np.complex64)


def haar_unitary(n: int, *key: int) -> np.ndarray:
    """Haar-random U(n) in complex128 (not rounded)."""
    return haar_from_ginibre(ginibre(rng_for(*key), n))


def brickwork_sites(n_sites: int, t: int) -> list[int]:
    """Left sites of the gates of brickwork layer t: i = t (mod 2), i+1 < N."""
    return list(range(t % 2, n_sites - 1, 2))


def brickwork_circuit(config: int, n_sites: int, depth: int):
    """List of layers; each layer = (sites int32[g], gates complex64[g,4,4]).

    Gate (layer t, site i) of config c is drawn from default_rng([230716870, c, t, i]).
    """
    layers = []
    for t in range(depth):
        sites = brickwork_sites(n_sites, t)
        us = np.stack([haar_u4(config, t, i) for i in sites]) if sites else np.zeros((0, 4, 4), np.complex64)
        layers.append((np.asarray(sites, np.int32), us))
    return layers


def n_two_qubit_gates(layers) -> int:
    return int(sum(len(s) for s, _ in layers))


def adjoint_circuit(layers):
    """Mirror half: layers reversed, each gate conjugate-transposed."""
    out = []
    for sites, us in reversed(layers):
        out.append((sites[::-1].copy(), np.conj(np.transpose(us[::-1], (0, 2, 1))).astype(np.complex64)))
    return out


# ---------------------------------------------------------------------------------------------
# MPO superoperators (SURVEY.md §8(c) algorithm item 9)
# ---------------------------------------------------------------------------------------------
PAULI = {
    "X": np.array([[0, 1], [1, 0]], np.complex128),
    "Y": np.array([[0, -1j], [1j, 0]], np.complex128),
    "Z": np.array([[1, 0], [0, -1]], np.complex128),
}


def depolarizing_1q(p: float) -> np.ndarray:
    """D[(2s+s'),(2t+t')] = (1-p) d_st d_s't' + (p/3) sum_P P[s,t] conj(P[s',t'])."""
    D = (1.0 - p) * np.eye(4, dtype=np.complex128)
    for P in PAULI.values():
        D += (p / 3.0) * np.kron(P, np.conj(P))
    return D


def unitary_superop(u: np.ndarray) -> np.ndarray:
    """(U (x) U*) acting on vec(rho) with site index s = 2*sigma + sigma' (ket, bra).

    For a 2-qubit U with gate index 2*sigma1 + sigma2, the 2-site MPO index is 4*s1 + s2 with
    s_k = 2*sigma_k + sigma'_k. Returns the 16x16 matrix S[(4 s1 + s2), (4 s1' + s2')].
    """
    u = np.asarray(u, np.complex128)
    U4 = u.reshape(2, 2, 2, 2)  # [sigma1, sigma2, tau1, tau2]
    # S[s1,s1b,s2,s2b ; t1,t1b,t2,t2b] = U[s1 s2, t1 t2] conj(U[s1b s2b, t1b t2b])
    S = np.einsum("abcd,efgh->aebfcgdh", U4, np.conj(U4))
    # axes now: sigma1, sigma1', sigma2, sigma2', tau1, tau1', tau2, tau2'
    return S.reshape(16, 16)


def mpo_gate(u: np.ndarray, p: float) -> np.ndarray:
    """S = (D (x) D)(U (x) U*), rounded to complex64 (SURVEY.md §8(c) algorithm item 9)."""
    D = depolarizing_1q(p)
    S = np.kron(D, D) @ unitary_superop(u)
    return S.astype(np.complex64)


def mpo_circuit(config: int, n_sites: int, depth: int, p: float):
    layers = []
    for sites, us in brickwork_circuit(config, n_sites, depth):
        ss = np.stack([mpo_gate(u, p) for u in us]) if len(us) else np.zeros((0, 16, 16), np.complex64)
        layers.append((sites, ss))
    return layers


# ---------------------------------------------------------------------------------------------
# NEXT-3: paper-faithful noisy workloads. PAPER.md:201: the random circuits
# "alternate randomly chosen layers of one- and two-qubit gates" (Cheng's definition is not in the
# container: Haar one-qubit layers on every site alternating with Haar two-qubit brickwork layers
# stand in); one- and two-qubit depolarising noise eps_1 = eps_2 after the gates.
# ---------------------------------------------------------------------------------------------
def haar_u2(*key: int) -> np.ndarray:
    """One Haar-random U(2), rounded to complex64 (Ginibre + QR + phase fix)."""
    return haar_from_ginibre(ginibre(rng_for(*key), 2)).astype(np.complex64)


def depolarizing_2q(p: float) -> np.ndarray:
    """Two-qubit depolarising superoperator on the 2-site vectorised index (4 s1 + s2,
    s = 2 sigma + sigma'): (1 - p) rho + (p / 15) sum_{(P, Q) != (I, I)} (P (x) Q) rho (P (x) Q)^dagger
    (the two-qubit analogue of SPEC.md:340's convention). At p = 15/16 it is the full twirl
    rho -> Tr(rho) I / 4."""
    paulis = [np.eye(2, dtype=np.complex128)] + list(PAULI.values())
    D = (1.0 - p) * np.eye(16, dtype=np.complex128)
    for a in range(4):
        for b in range(4):
            if a == 0 and b == 0:
                continue
            D += (p / 15.0) * unitary_superop(np.kron(paulis[a], paulis[b]))
    return D


def superop_1q(u: np.ndarray, p: float) -> np.ndarray:
    """D_1(p) (U (x) U*) on one site's vectorised index s = 2 sigma + sigma', rounded to complex64."""
    u = np.asarray(u, np.complex128)
    return (depolarizing_1q(p) @ np.kron(u, np.conj(u))).astype(np.complex64)


def superop_2q(u: np.ndarray, p: float) -> np.ndarray:
    """D_2(p) (U (x) U*) on the 2-site vectorised index, rounded to complex64."""
    return (depolarizing_2q(p) @ unitary_superop(u)).astype(np.complex64)


def alternating_circuit(config: int, n_sites: int, depth: int, kind: str = "mps", eps1: float = 0.0,
                        eps2: float = 0.0):
    """Layers alternating a one-qubit layer (Haar U(2) on every site; seed [.., config, t, i, 1])
    and a two-qubit brickwork layer (Haar U(4) on (i, i+1), i = t mod 2; seed [.., config, t, i]),
    `depth` of each. kind = "mps": unitaries (d x d and d^2 x d^2); kind = "mpo": superoperators
    with one-qubit depolarising eps1 after each one-qubit gate and two-qubit depolarising eps2
    after each two-qubit gate. The layer's gate shape tells the two kinds apart."""
    layers = []
    for t in range(depth):
        s1 = list(range(n_sites))
        u1 = [haar_u2(config, t, i, 1) for i in s1]
        if kind == "mpo":
            u1 = [superop_1q(u, eps1) for u in u1]
        layers.append((np.asarray(s1, np.int32), np.stack(u1)))
        s2 = brickwork_sites(n_sites, t)
        u2 = [haar_u4(config, t, i) for i in s2]
        if kind == "mpo":
            u2 = [superop_2q(u, eps2) for u in u2]
        layers.append((np.asarray(s2, np.int32), np.stack(u2)))
    return layers


def n_two_qubit_gates_any(layers, d: int) -> int:
    """Two-site gates of a mixed circuit (the ledger's n): layers of d^2 x d^2 gates."""
    return int(sum(len(s) for s, u in layers if len(s) and np.asarray(u).shape[-1] == d * d))


# ---------------------------------------------------------------------------------------------
# Config-2 microbench (BASELINE.json configs[1])
# ---------------------------------------------------------------------------------------------
def powerlaw_sigma(n: int) -> np.ndarray:
    s = np.arange(1, n + 1, dtype=np.float64) ** -1.5
    return s / np.linalg.norm(s)


def micro_theta(chi: int, b: int) -> np.ndarray:
    """theta_b = X diag(sigma) Y^H, (2chi)x(2chi), rounded to complex64. Seed [.., 2, chi, b]."""
    n = 2 * chi
    rng = rng_for(2, chi, b)
    X = haar_from_ginibre(ginibre(rng, n))
    Y = haar_from_ginibre(ginibre(rng, n))
    th = (X * powerlaw_sigma(n)[None, :]) @ np.conj(Y.T)
    return th.astype(np.complex64)


def micro_pair(chi: int, b: int, with_gate: bool = True):
    """Contract-inclusive microbench input for one theta (variant 2).

    Returns (B_left (chi,2,2chi), B_right (2chi,2,chi), U (4x4)) all complex64 such that the
    two-site update of the pair, with lambda_left = 1, sees Theta' = G_U(B_left B_right) ~ theta.
    B_right = I_{2chi} reshaped; B_left = (U^dagger acting on the (s,t) index of theta).
    """
    th = micro_theta(chi, b).astype(np.complex128)
    n = 2 * chi
    if with_gate:
        U = haar_u4(2, chi, b, 1 << 20).astype(np.complex128)
    else:
        U = np.eye(4, dtype=np.complex128)
    # theta[(a,s),(t,c)] -> T[a,s,t,c]; C[a,s',t',c] = sum_{s,t} conj(U[st, s't']) T[a,s,t,c]
    T = th.reshape(chi, 2, 2, chi)
    Ud = np.conj(U).reshape(2, 2, 2, 2)  # [s,t,s',t']
    C = np.einsum("stuv,astc->auvc", Ud, T)
    B_left = C.reshape(chi, 2, n).astype(np.complex64)
    B_right = np.eye(n, dtype=np.complex64).reshape(n, 2, chi)
    return B_left, B_right, U.astype(np.complex64)


def micro_chain(chi: int, count: int, first: int = 0, with_gate: bool = True):
    """A 2*count-site chain whose even layer is `count` independent updates of config 2.

    Bond dims: chi between pairs, 2chi inside a pair. lambda on every external bond is 1
    ("lambda_{i-1} = 1"). Returns (sites list, gates, site tensors).
    """
    tensors, gates = [], []
    for b in range(first, first + count):
        L, R, U = micro_pair(chi, b, with_gate)
        tensors += [L, R]
        gates.append(U)
    return tensors, np.stack(gates)


def micro_chain_torch(chi: int, count: int, first: int = 0, device="cuda"):
    """Same recipe as micro_chain (seeds [.., 2, chi, b]), with the QRs / products batched in
    torch (complex128, on `device`) for bench-sized batches. Haar(Z) = Q diag(R_ii/|R_ii|) is
    unique for a given Z, so this equals micro_chain up to FP64 rounding before the complex64
    rounding. Returns (site tensors as one complex64 torch tensor per side, gates complex64 np)."""
    import torch

    n = 2 * chi
    Zx = np.empty((count, n, n), np.complex128)
    Zy = np.empty((count, n, n), np.complex128)
    Zu = np.empty((count, 4, 4), np.complex128)
    for x, b in enumerate(range(first, first + count)):
        rng = rng_for(2, chi, b)
        Zx[x] = ginibre(rng, n)
        Zy[x] = ginibre(rng, n)
        Zu[x] = ginibre(rng_for(2, chi, b, 1 << 20), 4)
    U = haar_from_ginibre(Zu).astype(np.complex64).astype(np.complex128)  # as micro_pair
    sig = torch.as_tensor(powerlaw_sigma(n), device=device, dtype=torch.float64)

    def haar_t(Z):
        q, r = torch.linalg.qr(Z)
        dg = torch.diagonal(r, dim1=-2, dim2=-1)
        return q * (dg / dg.abs()).unsqueeze(-2)

    X = haar_t(torch.as_tensor(Zx, device=device))
    Y = haar_t(torch.as_tensor(Zy, device=device))
    th = (X * sig.to(X.dtype)) @ Y.conj().transpose(-1, -2)
    th = th.to(torch.complex64).to(torch.complex128)
    T = th.reshape(count, chi, 2, 2, chi)
    Ud = torch.as_tensor(np.conj(U), device=device).reshape(count, 2, 2, 2, 2)
    C = torch.einsum("gstuv,gastc->gauvc", Ud, T)
    left = C.reshape(count, chi, 2, n).to(torch.complex64)
    right = torch.eye(n, dtype=torch.complex64, device=device).reshape(n, 2, chi).expand(count, n, 2, chi)
    return left, right.contiguous(), U.astype(np.complex64)
