"""ctypes wrapper of the complex128 CPU oracle (oracle/eamps_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package. It shares no code with the CUDA path
(paper_2307_16870_b200/) and neither imports the other.

Every function of the C library cites the paper passage it follows (see eamps_oracle.c).
Parity pins: tests/test_oracle_*.py (closed forms, SPEC worked examples, numpy.linalg.svd as an
independent library routine, and the dense 2^N / 4^N brute force of tests/bruteforce.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "eamps_oracle.c")
_HDR = os.path.join(_HERE, "eamps_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

STRATEGIES = {"naive": 0, "nearest": 1, "global": 2, "fixed": 3}
RULES = {"pure": 0, "wang": 1, "ratio": 2}


def build(force: bool = False) -> str:
    """gcc -O2 -fopenmp -shared; the oracle is plain C99 (complex.h)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


class Record(C.Structure):
    _fields_ = [("gate_index", C.c_int64), ("bond", C.c_int32), ("chi_before", C.c_int32),
                ("chi_after", C.c_int32), ("capped", C.c_int32), ("target_f", C.c_double),
                ("achieved_f", C.c_double), ("discarded_weight", C.c_double)]


class Config(C.Structure):
    _fields_ = [("f_min", C.c_double), ("n_planned", C.c_int64), ("strategy", C.c_int32),
                ("rule", C.c_int32), ("chi_cap", C.c_int32), ("max_sweeps", C.c_int32),
                ("f_fixed", C.c_double)]


_P = C.c_void_p
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


def _declare(L):
    L.orc_jacobi_svd.argtypes = [C.c_int, C.c_int, _P, _P, _P, C.c_int, C.POINTER(C.c_int)]
    L.orc_sort_tails.argtypes = [C.c_int, _P, _P, _P]
    L.orc_sort_tails.restype = None
    L.orc_target_log.argtypes = [C.c_int, C.c_double, C.c_int64, C.c_double, C.c_int64, C.c_double, _dp]
    L.orc_select.argtypes = [C.c_int, C.c_int, _P, _P, C.c_double, C.c_int, C.c_int,
                             C.POINTER(C.c_int), _dp, _dp, C.POINTER(C.c_int)]
    L.orc_select.restype = None
    L.orc_create.argtypes = [C.c_int, C.c_int, C.POINTER(Config), C.POINTER(_P)]
    L.orc_destroy.argtypes = [_P]
    L.orc_destroy.restype = None
    L.orc_import_site.argtypes = [_P, C.c_int, _P, _P]
    L.orc_set_lambda.argtypes = [_P, C.c_int, _P, C.c_int]
    L.orc_export_site.argtypes = [_P, C.c_int, _P, _P]
    L.orc_apply_gate1.argtypes = [_P, C.c_int, _P]
    L.orc_set_ledger.argtypes = [_P, C.c_double, C.c_int64, C.c_int]
    L.orc_apply_gate2.argtypes = [_P, C.c_int, _P]
    L.orc_apply_layer.argtypes = [_P, C.c_int, _P, _P]
    L.orc_bond_dims.argtypes = [_P, _P]
    L.orc_schmidt_values.argtypes = [_P, C.c_int, _P, C.c_int, C.POINTER(C.c_int)]
    L.orc_estimate.argtypes = [_P, _dp, C.POINTER(C.c_int64), C.POINTER(C.c_int)]
    L.orc_records.argtypes = [_P, C.POINTER(Record), C.c_int64, C.POINTER(C.c_int64)]
    L.orc_amplitude.argtypes = [_P, _P, _dp]
    L.orc_statevector.argtypes = [_P, _P, C.c_int64]
    L.orc_last_spectrum.argtypes = [_P, C.c_int, _P, C.c_int, C.POINTER(C.c_int)]
    L.orc_overlap.argtypes = [_P, _P, _dp]
    L.orc_trace.argtypes = [_P, _dp]
    L.orc_expectation2.argtypes = [_P, C.c_int, _P, _dp]
    L.orc_canonicalize.argtypes = [_P]


class OracleError(RuntimeError):
    pass


def _ck(rc):
    if rc != 0:
        raise OracleError("oracle status %d" % rc)


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.complex128)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------------------------
# building blocks
# ---------------------------------------------------------------------------------------------
def jacobi_svd(A, max_sweeps: int = 60):
    """One-sided Jacobi on the columns of A (m x n). Returns (sigma unsorted, V, A V, sweeps)."""
    A = np.asarray(A)
    m, n = A.shape
    Af = np.asfortranarray(A.astype(np.complex128))
    V = np.zeros((n, n), np.complex128, order="F")
    sig = np.zeros(n)
    sw = C.c_int(0)
    rc = lib().orc_jacobi_svd(m, n, _ptr(Af), _ptr(V), _ptr(sig), max_sweeps, C.byref(sw))
    _ck(rc)
    return sig, V, Af, sw.value


def sort_tails(sigma):
    sigma = np.ascontiguousarray(sigma, np.float64)
    n = sigma.size
    pi = np.zeros(n, np.int32)
    T = np.zeros(n + 1)
    lib().orc_sort_tails(n, _ptr(sigma), _ptr(pi), _ptr(T))
    return pi, T


def target_log(strategy: str, f_min: float, n_planned: int, log_E: float, j: int, f_fixed: float = 1.0) -> float:
    out = C.c_double(0)
    _ck(lib().orc_target_log(STRATEGIES[strategy], float(np.log(f_min)), int(n_planned), float(log_E), int(j),
                             float(np.log(f_fixed)), C.byref(out)))
    return out.value


def select(rule: str, sigma_sorted, T, log_t: float, chi_cap: int = 0, kmax: int = 0):
    s = np.ascontiguousarray(sigma_sorted, np.float64)
    T = np.ascontiguousarray(T, np.float64)
    k = C.c_int(0); f = C.c_double(0); dl = C.c_double(0); cp = C.c_int(0)
    lib().orc_select(RULES[rule], s.size, _ptr(s), _ptr(T), float(log_t), int(chi_cap), int(kmax),
                     C.byref(k), C.byref(f), C.byref(dl), C.byref(cp))
    return k.value, f.value, dl.value, bool(cp.value)


# ---------------------------------------------------------------------------------------------
# the state
# ---------------------------------------------------------------------------------------------
class OracleMPS:
    """B-lambda MPS (d=2) / vectorised MPO (d=4) with the EA truncation ledger."""

    def __init__(self, n_sites: int, d: int = 2, f_min: float = 1.0, n_planned: int = 0,
                 strategy: str = "global", rule: str | None = None, chi_cap: int = 0,
                 max_sweeps: int = 60, f_fixed: float = 1.0):
        if rule is None:
            rule = "wang" if d == 4 else "pure"
        cfg = Config(float(f_min), int(n_planned), STRATEGIES[strategy], RULES[rule], int(chi_cap),
                     int(max_sweeps), float(f_fixed))
        h = C.c_void_p()
        _ck(lib().orc_create(int(n_sites), int(d), C.byref(cfg), C.byref(h)))
        self._h = h
        self.n_sites, self.d, self.rule = n_sites, d, rule

    def close(self):
        if getattr(self, "_h", None):
            lib().orc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def import_site(self, site: int, B):
        B = _c128(B)
        dims = np.array(B.shape, np.int32)
        _ck(lib().orc_import_site(self._h, int(site), _ptr(B), _ptr(dims)))

    def set_lambda(self, bond: int, lam):
        lam = np.ascontiguousarray(lam, np.float64)
        _ck(lib().orc_set_lambda(self._h, int(bond), _ptr(lam), lam.size))

    def export_site(self, site: int) -> np.ndarray:
        dims = np.zeros(3, np.int32)
        _ck(lib().orc_export_site(self._h, int(site), None, _ptr(dims)))
        B = np.zeros(tuple(dims), np.complex128)
        _ck(lib().orc_export_site(self._h, int(site), _ptr(B), _ptr(dims)))
        return B

    def apply_gate1(self, site: int, U):
        U = _c128(U)
        _ck(lib().orc_apply_gate1(self._h, int(site), _ptr(U)))

    def apply_gate2(self, site: int, U):
        U = _c128(U)
        _ck(lib().orc_apply_gate2(self._h, int(site), _ptr(U)))

    def apply_layer(self, sites, Us):
        sites = np.ascontiguousarray(sites, np.int32)
        Us = _c128(Us)
        _ck(lib().orc_apply_layer(self._h, sites.size, _ptr(sites), _ptr(Us)))

    def apply_layer1(self, sites, Us):
        """A layer of single-site gates (test plumbing: one orc_apply_gate1 per site)."""
        for i, u in zip(np.asarray(sites).ravel(), np.asarray(Us)):
            self.apply_gate1(int(i), u)

    def run(self, layers):
        for sites, us in layers:
            if np.asarray(us).shape[-1] == self.d and len(sites):
                self.apply_layer1(sites, us)
            else:
                self.apply_layer(sites, us)

    def bond_dims(self) -> np.ndarray:
        out = np.zeros(self.n_sites - 1, np.int32)
        _ck(lib().orc_bond_dims(self._h, _ptr(out)))
        return out

    def schmidt_values(self, bond: int) -> np.ndarray:
        n = C.c_int(0)
        buf = np.zeros(1, np.float64)
        _ck(lib().orc_schmidt_values(self._h, int(bond), _ptr(buf), 0, C.byref(n)))
        buf = np.zeros(n.value)
        _ck(lib().orc_schmidt_values(self._h, int(bond), _ptr(buf), n.value, C.byref(n)))
        return buf

    def estimate(self):
        le = C.c_double(0); nd = C.c_int64(0); gh = C.c_int(0)
        _ck(lib().orc_estimate(self._h, C.byref(le), C.byref(nd), C.byref(gh)))
        return dict(log_est=le.value, est=float(np.exp(le.value)), n_done=nd.value,
                    guarantee_held=bool(gh.value), is_lower_bound=(self.d == 4))

    def set_ledger(self, log_E: float, j: int, guarantee_held: int):
        """Ledger token plumbing (multi-rank tests): no arithmetic."""
        _ck(lib().orc_set_ledger(self._h, float(log_E), int(j), int(guarantee_held)))

    def records(self):
        ln = C.c_int64(0)
        _ck(lib().orc_records(self._h, None, 0, C.byref(ln)))
        arr = (Record * max(ln.value, 1))()
        _ck(lib().orc_records(self._h, arr, ln.value, C.byref(ln)))
        return [dict(gate_index=r.gate_index, bond=r.bond, chi_before=r.chi_before, chi_after=r.chi_after,
                     capped=bool(r.capped), target_f=r.target_f, achieved_f=r.achieved_f,
                     discarded_weight=r.discarded_weight) for r in arr[: ln.value]]

    def amplitude(self, digits) -> complex:
        dg = np.ascontiguousarray(digits, np.uint8)
        out = (C.c_double * 2)()
        _ck(lib().orc_amplitude(self._h, _ptr(dg), out))
        return complex(out[0], out[1])

    def statevector(self) -> np.ndarray:
        n = self.d ** self.n_sites
        out = np.zeros(n, np.complex128)
        _ck(lib().orc_statevector(self._h, _ptr(out), n))
        return out

    # ---- observables (NEXT-4): E7 / E9 building blocks and E5 ------------------------------
    def overlap(self, other: "OracleMPS") -> complex:
        """<self|other> (d = 2) or the Hilbert-Schmidt <<rho_self|rho_other>> (d = 4)."""
        out = (C.c_double * 2)()
        _ck(lib().orc_overlap(self._h, other._h, out))
        return complex(out[0], out[1])

    def trace(self) -> complex:
        out = (C.c_double * 2)()
        _ck(lib().orc_trace(self._h, out))
        return complex(out[0], out[1])

    def expectation2(self, site: int, O) -> complex:
        O = _c128(O)
        out = (C.c_double * 2)()
        _ck(lib().orc_expectation2(self._h, int(site), _ptr(O), out))
        return complex(out[0], out[1])

    def canonicalize(self):
        """NEXT-1: exact canonical form (right-orthonormal B, exact Schmidt lambda), no ledger entry."""
        _ck(lib().orc_canonicalize(self._h))

    def last_spectrum(self, g: int) -> np.ndarray:
        n = C.c_int(0)
        _ck(lib().orc_last_spectrum(self._h, int(g), None, 0, C.byref(n)))
        out = np.zeros(n.value)
        _ck(lib().orc_last_spectrum(self._h, int(g), _ptr(out), n.value, C.byref(n)))
        return out
