"""Pins of the oracle's building blocks against what the paper and the mathematics fix.

Nothing here retypes the oracle's formula: the SVD is checked against closed-form spectra,
reconstruction/orthonormality identities and numpy.linalg.svd (an independent library routine);
the selector and ledger against SPEC.md's printed worked examples and the closed-form config-2
spectrum; the ledger invariants against randomized budgets.
"""
import json
import os

import numpy as np
import pytest

import oracle
import workloads

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _haar(n, seed):
    return workloads.haar_unitary(n, 99, seed)


# ------------------------------------------------------------------------------ Jacobi SVD
def test_svd_diag_closed_form():
    s, V, AV, _ = oracle.jacobi_svd(np.diag([4.0, 3.0]).astype(complex))
    assert np.allclose(np.sort(s)[::-1], [4.0, 3.0], atol=1e-15)


def test_svd_identity():
    s, V, AV, _ = oracle.jacobi_svd(np.eye(2, dtype=complex))
    assert np.allclose(s, [1.0, 1.0], atol=1e-15)


@pytest.mark.parametrize("m,n", [(8, 8), (12, 8), (6, 10), (32, 32), (16, 64)])
def test_svd_prescribed_spectrum(m, n):
    r = min(m, n)
    X = _haar(m, 1)[:, :r]
    Y = _haar(n, 2)[:, :r]
    sig = np.linspace(1.0, 0.01, r) ** 2
    A = (X * sig) @ Y.conj().T
    s, V, AV, sw = oracle.jacobi_svd(A)
    ss = np.sort(s)[::-1]
    assert np.allclose(ss[:r], sig, rtol=1e-12, atol=1e-14)
    assert np.all(ss[r:] < 1e-13)
    # V unitary, A V = AV, reconstruction A = (AV) V^H
    assert np.abs(V.conj().T @ V - np.eye(n)).max() < 1e-13
    assert np.abs(A @ V - AV).max() < 1e-13
    assert np.linalg.norm(A - AV @ V.conj().T) < 1e-13 * np.linalg.norm(A)
    # columns of AV mutually orthogonal
    G = AV.conj().T @ AV
    off = G - np.diag(np.diag(G))
    assert np.abs(off).max() < 1e-13


@pytest.mark.parametrize("m,n,seed", [(10, 7, 0), (7, 10, 1), (24, 24, 2)])
def test_svd_vs_numpy(m, n, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    s, *_ = oracle.jacobi_svd(A)
    ref = np.linalg.svd(A, compute_uv=False)
    ss = np.sort(s)[::-1][: min(m, n)]
    assert np.allclose(ss, ref, rtol=1e-12)


def test_svd_rank_deficient_parallel_columns():
    a = np.array([1.0, 2.0j, -1.0])
    A = np.stack([a, 3 * a], axis=1)
    s, *_ = oracle.jacobi_svd(A)
    ss = np.sort(s)[::-1]
    assert abs(ss[0] - np.sqrt(10) * np.linalg.norm(a)) < 1e-14
    assert ss[1] < 1e-14


def test_svd_powerlaw_theta_c2():
    """config-2 theta (complex64-rounded): sigma equals the FP64 library SVD of the same matrix."""
    th = workloads.micro_theta(16, 0)
    s, *_ = oracle.jacobi_svd(th)
    ref = np.linalg.svd(th.astype(np.complex128), compute_uv=False)
    assert np.allclose(np.sort(s)[::-1], ref, rtol=1e-11)


# ------------------------------------------------------------------------------ sort + tails
def test_sort_tails():
    rng = np.random.default_rng(3)
    s = rng.random(37)
    s[5] = s[9]  # a tie, lower index first
    pi, T = oracle.sort_tails(s)
    assert np.all(np.diff(s[pi]) <= 0)
    assert list(pi).index(5) < list(pi).index(9)
    for k in range(38):
        assert abs(T[k] - np.sum(np.sort(s)[::-1][k:] ** 2)) < 1e-14


# ------------------------------------------------------------------------------ selector
def _sel(rule, lam2, t, cap=0):
    s = np.sqrt(np.asarray(lam2, float))
    pi, T = oracle.sort_tails(s)
    return oracle.select(rule, s[pi], T, np.log(t), cap)


def test_select_spec_examples():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for ex in g["select_pure"]:
        k, f, _, _ = _sel("pure", ex["lambda2"], ex["t"])
        assert k == ex["k"], ex["cite"]
        assert abs(f - ex["f"]) < 1e-12, ex["cite"]
    for ex in g["select_wang"]:
        k, f, _, _ = _sel("wang", ex["lambda2"], ex["t"])
        assert k == ex["k"], ex["cite"]
        assert abs(f - ex["f"]) < 1e-12, ex["cite"]


def test_select_wang_reading_is_sqrt_of_kept_weight():
    # SURVEY §8(c) reading 2 (M1): f = sqrt(P_k / P); [0.8,0.2] keeping 1 gives sqrt(0.8)
    k, f, dl, _ = _sel("wang", [0.8, 0.2], 0.89)
    assert k == 1 and abs(f - np.sqrt(0.8)) < 1e-15 and abs(dl - 0.5 * np.log(0.8)) < 1e-15
    k, f, _, _ = _sel("ratio", [0.8, 0.2], 0.79)
    assert k == 1 and abs(f - 0.8) < 1e-15


def test_select_exact_mode_and_cap():
    k, f, _, cp = _sel("pure", [0.5, 0.3, 0.2, 1e-31], 1.0)
    assert k == 3 and f == pytest.approx(1.0, abs=1e-15) and not cp  # 1e-14 machine-zero rule SPEC.md:75
    k, f, _, cp = _sel("pure", [0.4, 0.3, 0.2, 0.1], 0.999, cap=2)
    assert k == 2 and cp and abs(f - 0.7) < 1e-15  # PAPER.md:214 cap fallback


@pytest.mark.parametrize("chi", [16, 64, 256, 1024])
def test_select_c2_closed_form(chi):
    g = json.load(open(os.path.join(GOLD, "c2_closed_form.json")))
    n = 2 * chi
    s = np.arange(1, n + 1, dtype=float) ** -1.5
    s /= np.linalg.norm(s)
    pi, T = oracle.sort_tails(s)
    k, f, _, _ = oracle.select("pure", s[pi], T, np.log(g["t"]))
    assert k == g["pure"][str(chi)]["k"]
    assert abs(f - g["pure"][str(chi)]["f"]) < 1e-9
    # the same rank from the definition written independently (cumulative kept weight)
    kept = np.cumsum(s ** 2)
    k_def = int(np.argmax(kept >= g["t"] - 1e-15)) + 1
    assert k == k_def
    kw, *_ = oracle.select("wang", s[pi], T, np.log(g["t"]))
    assert kw == g["wang_k"][str(chi)]


# ------------------------------------------------------------------------------ ledger
def test_ledger_spec_examples():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["ledger"]
    assert abs(np.exp(oracle.target_log("naive", 0.9, 2, 0.0, 0)) - g["naive_0.9_n2"]["value"]) < 1e-15
    v = np.exp(oracle.target_log("naive", 0.9, 480, 0.0, 0))
    assert str(v).startswith(str(g["naive_0.9_n480_prefix"]["value_prefix"]))
    v = np.exp(oracle.target_log("global", 0.9, 3, np.log(0.99), 1))
    assert abs(v - g["global_0.9_n3_after_0.99"]["value"]) < 1e-6
    v = np.exp(oracle.target_log("nearest", 0.9, 3, np.log(0.99), 1))
    assert abs(v - g["nearest_0.9_n3_after_0.99"]["value"]) < 1e-6
    # naive ignores history
    assert oracle.target_log("naive", 0.9, 3, np.log(0.5), 2) == oracle.target_log("naive", 0.9, 3, 0.0, 0)
    # exact-simulation limit
    assert oracle.target_log("global", 1.0, 10, 0.0, 3) == 0.0
    # j >= n_planned is a state error
    with pytest.raises(oracle.OracleError):
        oracle.target_log("global", 0.9, 3, 0.0, 3)


@pytest.mark.parametrize("strategy", ["naive", "nearest", "global"])
def test_ledger_budget_soundness(strategy):
    """every achieved f >= issued t  =>  final estimate >= F_min (1 - 1e-10)."""
    rng = np.random.default_rng(7)
    for trial in range(50):
        n = int(rng.integers(1, 60))
        fmin = float(rng.uniform(0.5, 0.999))
        logE = 0.0
        for j in range(n):
            lt = oracle.target_log(strategy, fmin, n, logE, j)
            assert lt <= 0.0
            t = np.exp(lt)
            f = t + (1 - t) * rng.random() ** 3
            logE += np.log(f)
        assert logE >= np.log(fmin) + np.log1p(-1e-10)


def test_ledger_strategy_ordering():
    """on identical streams exceeding targets, global ends closer to F_min than naive (Fig. 1)."""
    rng = np.random.default_rng(11)
    n, fmin = 40, 0.9
    surplus = rng.random(n)
    res = {}
    for strat in ["naive", "global"]:
        logE = 0.0
        for j in range(n):
            t = np.exp(oracle.target_log(strat, fmin, n, logE, j))
            logE += np.log(t + (1 - t) * 0.5 * surplus[j])
        res[strat] = np.exp(logE)
    assert fmin * (1 - 1e-10) <= res["global"] <= res["naive"]


def _two_pair_chain(w1, w2):
    """4-site chain of two independent pairs whose thetas have Schmidt weights w1 and w2 (lambda = 1)."""
    tensors = []
    for w in (w1, w2):
        BL = np.zeros((1, 2, 2), np.complex128)
        BL[0, 0, 0], BL[0, 1, 1] = np.sqrt(w[0]), np.sqrt(w[1])
        BR = np.eye(2, dtype=np.complex128).reshape(2, 2, 1)
        tensors += [BL, BR]
    return tensors


def test_ledger_record_example():
    """record [0.99, 0.98] -> estimate 0.9702 (E12: the running
    product of truncation fidelities). Two updates whose rank-1 cuts keep exactly 0.99 and 0.98 of
    the weight, at a fixed per-update target below both."""
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["ledger"]["record_0.99_0.98"]
    o = oracle.OracleMPS(4, strategy="fixed", f_fixed=0.975)
    for i, B in enumerate(_two_pair_chain((0.99, 0.01), (0.98, 0.02))):
        o.import_site(i, B)
    o.apply_layer(np.array([0, 2], np.int32), np.stack([np.eye(4, dtype=np.complex64)] * 2))
    fs = [r["achieved_f"] for r in o.records()]
    assert [r["chi_after"] for r in o.records()] == [1, 1]
    assert abs(fs[0] - 0.99) < 1e-14 and abs(fs[1] - 0.98) < 1e-14
    assert abs(o.estimate()["est"] - g["value"]) < 1e-14
