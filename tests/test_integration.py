"""The reference-side binding (integration/b200_backend.cpp)
compiled against the reference's own headers and linked with libequil_b200.so:
on CPU, that it builds (when /root/reference is present) and that it exports
the reference's entry points; on the GPU, the reference's cases driven through
it, each compared bit for bit with the reference's own sources
(integration/test_backend.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INTEG = os.path.join(ROOT, "integration")
EXE = os.path.join(INTEG, "_build", "test_backend")
LIB = os.path.join(INTEG, "_build", "libequil_b200_backend.so")
REFERENCE = "/root/reference/proj"


def _ensure_built():
    if os.path.isdir(REFERENCE):
        subprocess.run(["make", "-s", "-C", INTEG], check=True, capture_output=True, text=True)
    if not os.path.exists(EXE):
        pytest.fail("integration/_build/test_backend is missing: run __graft_entry__.build() "
                    "where /root/reference is present (the binary travels with the repo)")


def test_backend_builds_and_exports_reference_entry_points():
    _ensure_built()
    out = subprocess.run(["nm", "-DC", LIB], capture_output=True, text=True, check=True).stdout
    for sym in ("equil::b200::sgd_equilibrate(equil::LinearOperator const&",
                "equil::b200::lsqr(equil::LinearOperator const&",
                "equil::b200::lsqr_preconditioned(equil::LinearOperator const&",
                "equil::b200::Device::Device(equil::ExplicitMatrix const&"):
        assert sym in out, sym
    # it resolves against the product library, not against the oracle
    ldd = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "libequil_b200.so" in ldd and "oracle" not in ldd


@pytest.mark.gpu
def test_reference_cases_through_the_binding():
    _ensure_built()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("OK"), r.stdout
