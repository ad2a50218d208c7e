"""CPU-side checks of the boundary: the C-ABI library builds, loads, and exports every symbol that
include/eamps.h declares; the binding exposes the same names; the product never imports the
oracle. No compute calls (no GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "eamps.h")).read()
    return sorted(set(re.findall(r"^\s*(?:mps_status|const char\*)\s+(mps_\w+)\s*\(", src, re.M)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for must in ["mps_create", "mps_apply_gate2", "mps_apply_layer", "mps_fidelity_estimate",
                 "mps_amplitude", "mps_to_statevector"]:
        assert must in names


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2307_16870_b200 import _build
    path = _build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (mps_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing


def test_library_loads_and_binding_names_match():
    import paper_2307_16870_b200 as pk
    L = pk.lib()
    for n in _declared():
        assert hasattr(L, n)
        assert n in pk.ABI_FUNCTIONS
    assert L.mps_status_string(-6).decode() == "Jacobi SVD did not converge"


def test_sm100a_cubin_inside():
    from paper_2307_16870_b200 import _build
    path = _build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_does_not_touch_the_oracle():
    pkg = os.path.join(ROOT, "paper_2307_16870_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "eamps_oracle" not in txt, f


def test_no_cpu_fallback_without_gpu():
    import torch
    import paper_2307_16870_b200 as pk
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        pk.MPS(4)
