"""B200-native entanglement-aware MPS/MPO gate update (arXiv:2307.16870) -- Python binding.

Argument marshalling only: every step of the hot path runs in the CUDA kernels of
libeamps.so (csrc/), behind the C ABI of include/eamps.h, whose functions this module exposes
under the same names. PyTorch provides the device slab and the stream -- nothing else. There is
no CPU fallback: importing this package on a machine without the built library raises, and
creating a state without a CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libeamps.so")

MPS_OK, MPS_E_INVAL, MPS_E_RANGE, MPS_E_NOMEM, MPS_E_CUDA, MPS_E_NCCL = 0, -1, -2, -3, -4, -5
MPS_E_NOCONV, MPS_E_NUMERIC, MPS_E_STATE, MPS_E_TOOBIG = -6, -7, -8, -9
STRATEGIES = {"naive": 0, "nearest": 1, "global": 2, "fixed": 3}
RULES = {"pure": 0, "wang": 1, "ratio": 2}

ABI_FUNCTIONS = [
    "mps_create", "mps_destroy", "mps_apply_gate1", "mps_apply_gate2", "mps_apply_layer",
    "mps_fidelity_estimate", "mps_amplitude", "mps_to_statevector", "mps_bond_dims",
    "mps_schmidt_values", "mps_truncation_log", "mps_last_spectrum", "mps_export_site",
    "mps_import_site", "mps_import_sites", "mps_export_sites", "mps_keep_spectra", "mps_set_lambda", "mps_snapshot_save", "mps_snapshot_load",
    "mps_launch_count", "mps_last_sweeps", "mps_set_profiling", "mps_set_svd_route", "mps_phase_times", "mps_sync", "mps_last_error", "mps_status_string",
    "mps_layer_begin", "mps_layer_step", "mps_ledger_get", "mps_ledger_set", "mps_plan_regime",
    "mps_overlap", "mps_trace", "mps_expectation2", "mps_apply_layer1", "mps_canonicalize",
]


class EampsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("eamps status %d: %s" % (status, msg))
        self.status = status


class Config(C.Structure):
    _fields_ = [("f_min", C.c_double), ("n_planned", C.c_int64), ("strategy", C.c_int32),
                ("rule", C.c_int32), ("chi_cap", C.c_int32), ("max_sweeps", C.c_int32),
                ("f_fixed", C.c_double), ("stream", C.c_void_p), ("dev_slab", C.c_void_p),
                ("slab_bytes", C.c_size_t)]


class Record(C.Structure):
    _fields_ = [("gate_index", C.c_int64), ("bond", C.c_int32), ("chi_before", C.c_int32),
                ("chi_after", C.c_int32), ("capped", C.c_int32), ("target_f", C.c_double),
                ("achieved_f", C.c_double), ("discarded_weight", C.c_double)]


_P = C.c_void_p
_lib = None


def lib():
    """Load libeamps.so (fails loudly if it was not built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libeamps.so not built: run `python -m paper_2307_16870_b200._build`")
        L = C.CDLL(LIB_PATH)
        i32, i64, dbl = C.c_int32, C.c_int64, C.c_double
        sig = {
            "mps_create": [i32, i32, C.POINTER(Config), C.POINTER(_P)],
            "mps_destroy": [_P],
            "mps_apply_gate1": [_P, i32, _P],
            "mps_apply_gate2": [_P, i32, _P],
            "mps_apply_layer": [_P, i32, _P, _P],
            "mps_fidelity_estimate": [_P, _P, _P, _P, _P, _P],
            "mps_amplitude": [_P, _P, _P],
            "mps_to_statevector": [_P, _P, C.c_size_t],
            "mps_bond_dims": [_P, _P],
            "mps_schmidt_values": [_P, i32, _P, i32, _P],
            "mps_truncation_log": [_P, _P, i64, _P],
            "mps_last_spectrum": [_P, i32, _P, i32, _P],
            "mps_export_site": [_P, i32, _P, _P],
            "mps_import_site": [_P, i32, _P, _P],
            "mps_import_sites": [_P, i32, i32, _P, _P],
            "mps_export_sites": [_P, i32, i32, _P, C.c_size_t, _P, _P],
            "mps_keep_spectra": [_P, i32],
            "mps_set_lambda": [_P, i32, _P, i32],
            "mps_snapshot_save": [_P, _P, C.c_size_t, _P],
            "mps_snapshot_load": [_P, _P, C.c_size_t],
            "mps_launch_count": [_P, _P],
            "mps_set_profiling": [_P, i32],
            "mps_set_svd_route": [_P, i32],
            "mps_phase_times": [_P, _P, _P],
            "mps_last_sweeps": [_P, i32, _P],
            "mps_sync": [_P],
            "mps_last_error": [_P],
            "mps_status_string": [i32],
            "mps_layer_begin": [_P, i32, _P, _P, _P],
            "mps_layer_step": [_P, _P],
            "mps_ledger_get": [_P, _P, _P, _P],
            "mps_ledger_set": [_P, dbl, i64, i32],
            "mps_plan_regime": [i32, i32, _P, _P, _P, _P],
            "mps_overlap": [_P, _P, _P],
            "mps_trace": [_P, _P],
            "mps_expectation2": [_P, i32, _P, _P],
            "mps_apply_layer1": [_P, i32, _P, _P],
            "mps_canonicalize": [_P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_char_p if name in ("mps_last_error", "mps_status_string") else C.c_int32
        _lib = L
    return _lib


def mps_plan_regime(m: int, n: int):
    """(regime, lane group, rows per lane, n_pad) the layer planner picks for an m x n theta (host only)."""
    out = [C.c_int32(0) for _ in range(4)]
    rc = lib().mps_plan_regime(int(m), int(n), *[C.byref(o) for o in out])
    if rc != 0:
        raise EampsError(rc, lib().mps_status_string(rc).decode())
    return tuple(o.value for o in out)


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _c64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.complex64)


class MPS:
    """One EA-MPS (d=2) or vectorised EA-MPO (d=4) on one GPU.

    slab_bytes of device memory are taken from torch's caching allocator and handed to the
    library, which owns the layout (site store, device pool, per-layer workspace).
    """

    def __init__(self, n_sites: int, d: int = 2, f_min: float = 1.0, n_planned: int = 0,
                 strategy: str = "global", rule: str | None = None, chi_cap: int = 0,
                 max_sweeps: int = 60, f_fixed: float = 1.0, slab_bytes: int = 1 << 30,
                 device=None, stream=None):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_2307_16870_b200 needs a CUDA device (no CPU fallback)")
        L = lib()
        if rule is None:
            rule = "wang" if d == 4 else "pure"
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.slab = torch.empty(int(slab_bytes), dtype=torch.uint8, device=self.device)
        self.stream = torch.cuda.current_stream(self.device) if stream is None else stream
        cfg = Config(float(f_min), int(n_planned), STRATEGIES[strategy], RULES[rule], int(chi_cap),
                     int(max_sweeps), float(f_fixed), C.c_void_p(self.stream.cuda_stream),
                     C.c_void_p(self.slab.data_ptr()), int(slab_bytes))
        h = C.c_void_p()
        self._check(L.mps_create(int(n_sites), int(d), C.byref(cfg), C.byref(h)), None)
        self._h = h
        self.n_sites, self.d, self.rule = n_sites, d, rule

    # -- plumbing ---------------------------------------------------------------------------
    def _check(self, rc, h="self"):
        if rc != 0:
            hh = self._h if h == "self" else h
            msg = lib().mps_last_error(hh).decode() if hh else lib().mps_status_string(rc).decode()
            raise EampsError(rc, msg)

    def close(self):
        if getattr(self, "_h", None):
            lib().mps_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- the hot path ---------------------------------------------------------------------------
    def mps_apply_gate1(self, site: int, U):
        U = _c64(U)
        self._check(lib().mps_apply_gate1(self._h, int(site), _ptr(U)))

    def mps_apply_gate2(self, site: int, U):
        U = _c64(U)
        self._check(lib().mps_apply_gate2(self._h, int(site), _ptr(U)))

    def mps_apply_layer(self, sites, Us):
        sites = np.ascontiguousarray(sites, np.int32)
        Us = _c64(Us)
        self._check(lib().mps_apply_layer(self._h, int(sites.size), _ptr(sites), _ptr(Us)))

    def mps_apply_layer1(self, sites, Us):
        """A layer of single-site gates (distinct sites)."""
        sites = np.ascontiguousarray(sites, np.int32)
        Us = _c64(Us)
        self._check(lib().mps_apply_layer1(self._h, int(sites.size), _ptr(sites), _ptr(Us)))

    def mps_canonicalize(self):
        """NEXT-1: exact canonical form (right-orthonormal B, exact Schmidt lambda), no ledger entry."""
        self._check(lib().mps_canonicalize(self._h))

    def mps_layer_begin(self, sites, Us) -> int:
        """a0-a3 of the layer's first wave, issued without waiting (returns the waves issued)."""
        sites = np.ascontiguousarray(sites, np.int32)
        Us = _c64(Us)
        w = C.c_int32(0)
        self._check(lib().mps_layer_begin(self._h, int(sites.size), _ptr(sites), _ptr(Us), C.byref(w)))
        return w.value

    def mps_layer_step(self) -> int:
        """a4-a5 of the wave in flight (+ a0-a3 of the next); returns the gates still pending."""
        r = C.c_int32(0)
        self._check(lib().mps_layer_step(self._h, C.byref(r)))
        return r.value

    def mps_ledger_get(self):
        le, j, g = C.c_double(0), C.c_int64(0), C.c_int32(0)
        self._check(lib().mps_ledger_get(self._h, C.byref(le), C.byref(j), C.byref(g)))
        return le.value, j.value, g.value

    def mps_ledger_set(self, log_E: float, j: int, guarantee: int):
        self._check(lib().mps_ledger_set(self._h, float(log_E), int(j), int(guarantee)))

    def run(self, layers):
        """Apply layers in order: a layer whose gates are d x d is a single-site layer
        (mps_apply_layer1), d^2 x d^2 a two-site layer (mps_apply_layer)."""
        for sites, us in layers:
            if np.asarray(us).shape[-1] == self.d and len(sites):
                self.mps_apply_layer1(sites, us)
            else:
                self.mps_apply_layer(sites, us)

    # -- queries -------------------------------------------------------------------------------
    def mps_fidelity_estimate(self):
        est, le = C.c_double(0), C.c_double(0)
        nd, gh, lb = C.c_int64(0), C.c_int32(0), C.c_int32(0)
        self._check(lib().mps_fidelity_estimate(self._h, C.byref(est), C.byref(le), C.byref(nd), C.byref(gh),
                                                C.byref(lb)))
        return dict(est=est.value, log_est=le.value, n_done=nd.value, guarantee_held=bool(gh.value),
                    is_lower_bound=bool(lb.value))

    def mps_amplitude(self, digits) -> complex:
        dg = np.ascontiguousarray(digits, np.uint8)
        out = np.zeros(2)
        self._check(lib().mps_amplitude(self._h, _ptr(dg), _ptr(out)))
        return complex(out[0], out[1])

    def mps_to_statevector(self) -> np.ndarray:
        n = self.d ** self.n_sites
        out = np.zeros(n, np.complex128)
        self._check(lib().mps_to_statevector(self._h, _ptr(out), 2 * n))
        return out

    def mps_bond_dims(self) -> np.ndarray:
        out = np.zeros(self.n_sites - 1, np.int32)
        self._check(lib().mps_bond_dims(self._h, _ptr(out)))
        return out

    def mps_schmidt_values(self, bond: int) -> np.ndarray:
        ln = C.c_int32(0)
        self._check(lib().mps_schmidt_values(self._h, int(bond), None, 0, C.byref(ln)))
        out = np.zeros(ln.value, np.float32)
        self._check(lib().mps_schmidt_values(self._h, int(bond), _ptr(out), ln.value, C.byref(ln)))
        return out

    def mps_truncation_array(self, last: int = 0) -> np.ndarray:
        """The truncation records as a numpy structured array (fields of mps_record); `last` > 0
        keeps only the most recent `last` rows."""
        ln = C.c_int64(0)
        self._check(lib().mps_truncation_log(self._h, None, 0, C.byref(ln)))
        arr = (Record * max(1, ln.value))()
        self._check(lib().mps_truncation_log(self._h, arr, ln.value, C.byref(ln)))
        a = np.ctypeslib.as_array(arr)[: ln.value]
        return a[-last:] if last > 0 else a

    def mps_truncation_log(self, last: int = 0):
        a = self.mps_truncation_array(last)
        return [dict(gate_index=int(r["gate_index"]), bond=int(r["bond"]), chi_before=int(r["chi_before"]),
                     chi_after=int(r["chi_after"]), capped=bool(r["capped"]), target_f=float(r["target_f"]),
                     achieved_f=float(r["achieved_f"]), discarded_weight=float(r["discarded_weight"])) for r in a]

    def mps_last_spectrum(self, g: int) -> np.ndarray:
        ln = C.c_int32(0)
        self._check(lib().mps_last_spectrum(self._h, int(g), None, 0, C.byref(ln)))
        out = np.zeros(ln.value)
        self._check(lib().mps_last_spectrum(self._h, int(g), _ptr(out), ln.value, C.byref(ln)))
        return out

    def mps_keep_spectra(self, on: bool = True):
        """Keep every wave's spectra readable through mps_last_spectrum (tests of multi-wave layers)."""
        self._check(lib().mps_keep_spectra(self._h, int(bool(on))))

    def mps_last_sweeps(self, g: int) -> int:
        s = C.c_int32(0)
        self._check(lib().mps_last_sweeps(self._h, int(g), C.byref(s)))
        return s.value

    def mps_export_site(self, site: int) -> np.ndarray:
        dims = np.zeros(3, np.int32)
        self._check(lib().mps_export_site(self._h, int(site), None, _ptr(dims)))
        B = np.zeros(tuple(int(x) for x in dims), np.complex64)
        self._check(lib().mps_export_site(self._h, int(site), _ptr(B), _ptr(dims)))
        return B

    def mps_import_site(self, site: int, B):
        if hasattr(B, "data_ptr"):  # a torch tensor already on the device
            dims = np.array(B.shape, np.int32)
            self._check(lib().mps_import_site(self._h, int(site), _ptr(B), _ptr(dims)))
            return
        B = _c64(B)
        dims = np.array(B.shape, np.int32)
        self._check(lib().mps_import_site(self._h, int(site), _ptr(B), _ptr(dims)))

    def mps_import_sites(self, first: int, tensors):
        """Bulk import of consecutive sites (one H2D copy + one device scatter)."""
        dims = np.array([t.shape for t in tensors], np.int32).reshape(-1, 3)
        flat = np.concatenate([_c64(t).ravel() for t in tensors])
        self._check(lib().mps_import_sites(self._h, int(first), len(tensors), _ptr(flat), _ptr(dims)))

    def mps_import_sites_raw(self, first: int, count: int, flat_ptr, dims: np.ndarray):
        dims = np.ascontiguousarray(dims, np.int32)
        self._check(lib().mps_import_sites(self._h, int(first), int(count), flat_ptr, _ptr(dims)))

    def mps_export_sites(self, first: int, count: int):
        """Bulk export of consecutive sites (one device gather + one D2H copy): list of arrays."""
        dims = np.zeros((count, 3), np.int32)
        ne = C.c_size_t(0)
        self._check(lib().mps_export_sites(self._h, int(first), int(count), None, 0, _ptr(dims), C.byref(ne)))
        flat = np.empty(ne.value, np.complex64)
        self._check(lib().mps_export_sites(self._h, int(first), int(count), _ptr(flat), ne.value, _ptr(dims),
                                           C.byref(ne)))
        out, o = [], 0
        for a, d, c in dims:
            out.append(flat[o: o + int(a) * int(d) * int(c)].reshape(int(a), int(d), int(c)))
            o += int(a) * int(d) * int(c)
        return out

    def mps_export_sites_raw(self, first: int, count: int, flat_ptr, cap_elems: int, dims: np.ndarray) -> int:
        """flat_ptr: host or device pointer (c_void_p) with room for cap_elems complex64; returns elems."""
        ne = C.c_size_t(0)
        self._check(lib().mps_export_sites(self._h, int(first), int(count), flat_ptr, int(cap_elems), _ptr(dims),
                                           C.byref(ne)))
        return ne.value

    def mps_set_lambda(self, bond: int, lam):
        lam = np.ascontiguousarray(lam, np.float32)
        self._check(lib().mps_set_lambda(self._h, int(bond), _ptr(lam), int(lam.size)))

    def mps_snapshot_save(self, buf=None):
        import torch

        need = C.c_size_t(0)
        self._check(lib().mps_snapshot_save(self._h, None, 0, C.byref(need)))
        if buf is None:
            buf = torch.empty(need.value, dtype=torch.uint8, device=self.device)
        self._check(lib().mps_snapshot_save(self._h, _ptr(buf), buf.numel(), C.byref(need)))
        return buf

    def mps_snapshot_load(self, buf):
        self._check(lib().mps_snapshot_load(self._h, _ptr(buf), buf.numel()))

    def mps_launch_count(self) -> int:
        c = C.c_int64(0)
        self._check(lib().mps_launch_count(self._h, C.byref(c)))
        return c.value

    def mps_set_profiling(self, on: bool = True):
        self._check(lib().mps_set_profiling(self._h, int(bool(on))))

    def mps_set_svd_route(self, route: int):
        """0: eigen route for large theta with 256 < n <= 2048 (default); 1: tcgen05 Jacobi route."""
        self._check(lib().mps_set_svd_route(self._h, int(route)))

    PHASES = ("contract", "svd_small", "svd_blocked", "select", "reabsorb", "svd_precond", "svd_jacobi",
              "svd_spectrum", "svd_eig_tridiag", "svd_eig_other")

    def mps_phase_times(self):
        ms = np.zeros(len(self.PHASES))
        cnt = np.zeros(len(self.PHASES), np.int64)
        self._check(lib().mps_phase_times(self._h, _ptr(ms), _ptr(cnt)))
        return {p: (float(ms[i]), int(cnt[i])) for i, p in enumerate(self.PHASES)}

    # ---- observables (NEXT-4): E7 / E9 building blocks and E5, computed on the device ---------
    def mps_overlap(self, other: "MPS") -> complex:
        """<self|other> (d = 2) or the Hilbert-Schmidt <<rho_self|rho_other>> (d = 4)."""
        out = (C.c_double * 2)()
        self._check(lib().mps_overlap(self._h, other._h, out))
        return complex(out[0], out[1])

    def mps_trace(self) -> complex:
        out = (C.c_double * 2)()
        self._check(lib().mps_trace(self._h, out))
        return complex(out[0], out[1])

    def mps_expectation2(self, site: int, O) -> complex:
        O = _c64(O)
        out = (C.c_double * 2)()
        self._check(lib().mps_expectation2(self._h, int(site), _ptr(O), out))
        return complex(out[0], out[1])

    def pure_fidelity(self, other: "MPS") -> float:
        """E7 |<a|b>|^2 / (<a|a> <b|b>): three device overlaps; the division is
        the only host arithmetic."""
        ab = self.mps_overlap(other)
        return abs(ab) ** 2 / (self.mps_overlap(self).real * other.mps_overlap(other).real)

    def wang_fidelity(self, other: "MPS") -> float:
        """E9 |Tr(rho sigma)| / sqrt(Tr rho^2 Tr sigma^2) of two MPOs."""
        ab = self.mps_overlap(other)
        return abs(ab) / (self.mps_overlap(self).real * other.mps_overlap(other).real) ** 0.5

    def mps_sync(self):
        self._check(lib().mps_sync(self._h))
